"""The C-ABI library loads and exports every symbol include/mars_b200.h declares, the
ctypes binding declares exactly those symbols, and there is no silent CPU path: without a
device, problem creation fails loudly (CPU-only checks; no kernels are launched)."""
import ctypes
import os
import re

import pytest

from conftest import ROOT, gpu_available


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "mars_b200.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(mars_[a-z0-9_]+)\s*\(", text)))


def test_header_symbols_exported():
    from paper_1907_05124_b200 import _native
    syms = declared_symbols()
    assert len(syms) >= 25
    lib = ctypes.CDLL(_native.LIB_PATH)
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing
    assert sorted(_native.SIGNATURES) == syms


def test_native_library_is_sm100a():
    import subprocess
    from paper_1907_05124_b200 import _native
    out = subprocess.run(["cuobjdump", "--list-elf", _native.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


@pytest.mark.skipif(gpu_available(), reason="checks the no-device behaviour")
def test_no_silent_cpu_fallback():
    import paper_1907_05124_b200 as mb
    with pytest.raises(mb.CudaError):
        mb.IsingProblem.dense(2, [0, -1, -1, 0])


def test_oracle_is_not_imported_by_product():
    pkg = os.path.join(ROOT, "paper_1907_05124_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cpp", ".cu", ".cuh", ".hpp")):
                text = open(os.path.join(dirpath, f)).read()
                assert "oracle" not in re.sub(r"#.*|//.*", "", text).replace("build_oracle_problem", "").lower() \
                    or f == "workloads.py", f


def test_reference_arm_does_not_map_the_product_library():
    """bench.py --impl reference runs the reference CPU code only: everything it imports
    (workload definitions, the oracle driver, time-to-best) must leave libmars_b200.so unmapped."""
    import subprocess
    import sys
    code = ("import sys; sys.path.insert(0, %r); import bench; "
            "from paper_1907_05124_b200.workloads import WORKLOADS, build_oracle_problem, time_to_best; "
            "import oracle.oracle; "
            "maps = open('/proc/self/maps').read(); "
            "print('LOADED' if 'libmars_b200' in maps else 'CLEAN')" % ROOT)
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, cwd=ROOT)
    assert out.returncode == 0, out.stderr
    assert out.stdout.strip().endswith("CLEAN"), out.stdout
