"""Multi-process run sharding on CPU with the gloo backend, world_size 2.

The device work is replaced by a deterministic per-index record generator (the same idea as
run_batch_with's synthetic runs, test_runner.cpp:115-146), so the test exercises exactly
the host path that changes with the GPU count: contiguous sharding, all_gather of the
per-run records, index-order aggregation on every rank, and the broadcast of the winning
spins from the rank that owns them.  Results must equal the single-process aggregation --
the analogue of the reference's worker-count invariance (test_runner.cpp:60-69)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

import paper_1907_05124_b200 as mb

N_SPINS = 24


def synthetic_records(first, count, runs):
    rng = np.random.default_rng(1234)                     # same table on every rank
    status = rng.choice([0, 0, 0, 0, 1, 2], size=runs).astype(np.uint8)
    energy = -np.round(rng.uniform(0, 50, size=runs))     # integral: ties happen
    cut = -energy / 2
    spins = rng.choice(np.array([-1, 1], np.int8), size=(runs, N_SPINS))
    rec = mb.Records.empty(count, N_SPINS, True)
    sl = slice(first, first + count)
    rec.status[:] = status[sl]
    rec.energy[:] = np.where(status[sl] == 1, 0.0, energy[sl])
    rec.cut[:] = np.where(status[sl] == 1, 0.0, cut[sl])
    rec.start_temp[:] = np.arange(first, first + count) * 0.5
    rec.descent_iters[:] = np.arange(first, first + count) % 17
    rec.spins[:] = spins[sl]
    return rec


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, runs, out):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        stats = mb.distributed_batch(dist, runs, N_SPINS, 0.0,
                                     lambda f, c: synthetic_records(f, c, runs), keep_spins=True)
        out[rank] = (stats.best_energy, stats.mean_energy, stats.best_cut, stats.hit_count,
                     stats.best_index, stats.completed_runs, stats.skipped_runs, stats.failed_runs,
                     stats.best_result.spins.tolist(), stats.records.energy.tolist(),
                     stats.records.spins.tolist())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("runs", [7, 64, 101])
def test_gloo_world2_matches_single_process(runs):
    world = 2
    manager = mp.Manager()
    out = manager.dict()
    mp.start_processes(_worker, args=(world, _free_port(), runs, out), nprocs=world, join=True,
                       start_method="spawn")
    full = synthetic_records(0, runs, runs)
    ref = mb.aggregate(full, 0.0, 0.0)
    expect = (ref.best_energy, ref.mean_energy, ref.best_cut, ref.hit_count, ref.best_index,
              ref.completed_runs, ref.skipped_runs, ref.failed_runs)
    for rank in range(world):
        got = out[rank]
        assert got[:8] == expect                          # identical stats on every rank
        assert got[8] == full.spins[ref.best_index].tolist()   # winner broadcast from its owner
        assert got[9] == full.energy.tolist()            # gathered in run-index order
        assert got[10] == full.spins.tolist()


@pytest.mark.parametrize("ranks", [1, 2, 3, 8])
def test_native_multi_gpu_exchange_logic(ranks):
    """mars_run_batch_multi's C++ shard / exchange (AllReduce-min of the best energy and of the
    first index reaching it, Broadcast of the winning spins, AllGather of the records) run on a
    host transport -- one host thread per rank, the same code the NCCL transport drives --
    must reproduce the single-shard, index-order aggregation (runner.cpp:126-167) exactly."""
    runs = 203
    full = synthetic_records(0, runs, runs)
    merged, st, best = mb.debug_exchange(ranks, full, 0.0)
    for name in ("status", "energy", "cut", "descent_iters", "elapsed_seconds"):
        assert np.array_equal(getattr(merged, name), getattr(full, name)), name
    ref = mb.aggregate(full, 0.0, 0.0)
    assert st.best_index == ref.best_index
    assert st.best_energy == ref.best_energy and st.hit_count == ref.hit_count
    assert st.mean_energy == ref.mean_energy and st.completed_runs == ref.completed_runs
    assert np.array_equal(best, full.spins[ref.best_index])
