"""bench.py's JSON contract on the CPU arm (--impl reference): one line with the keys the
driver reads (the B200 arm is exercised on the GPU box)."""
import json
import os
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.skipif(not os.path.exists(os.path.join(ROOT, "oracle", "_ref", "libmars_ref.so")),
                                reason="compiled reference not built")


def test_reference_arm_line():
    r = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--workload", "cfg1_sk256_pm1",
                        "--steps", "1", "--warmup", "0", "--cpu-runs", "16"],
                       cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["unit"] == "descents/s" and d["value"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["cpu_baseline"]["kind"] in ("reference", "port")
    ttb = d["time_to_best"]
    assert ttb["unit"] == "s" and 0 < ttb["value"] <= ttb["last_retirement_s"]


def test_pool_finish_times_replays_in_order_claims():
    import numpy as np
    import bench
    # 2 workers claim 0,1 at t=0; run 2 goes to whichever frees first (run 1 at 1.0)
    fin = bench.pool_finish_times(np.array([3.0, 1.0, 1.0, 0.5]), 2)
    assert fin.tolist() == [3.0, 1.0, 2.0, 2.5]
    assert bench.pool_finish_times(np.array([1.0, 2.0]), 1).tolist() == [1.0, 3.0]


def test_time_to_best_hit_rule():
    import numpy as np
    from paper_1907_05124_b200.mars import time_to_best
    e = np.array([-5.0, -7.0, -7.0, -7.0 + 1e-12, -8.0])
    st = np.array([0, 0, 0, 0, 2], np.uint8)           # the -8 run diverged: not a hit
    fin = np.array([1.0, 4.0, 3.0, 2.0, 0.5])
    assert time_to_best(e, st, fin, -7.0, 0.0) == 3.0
    assert time_to_best(e, st, fin, -7.0, 1e-9) == 2.0
    assert time_to_best(e, st, fin, -9.0, 0.0) == float("inf")
