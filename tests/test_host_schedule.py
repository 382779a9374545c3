"""Host logic of the tcgen05 kernel's large-N schedule (no GPU): the split-K / tile choice by a
greedy longest-first makespan estimate (K1 "Split-K"), through the test-only C-ABI
hook mars_debug_choose_split.  The expectations are the choices measured best on the B200
(profiles/r02/README.md, cfg5)."""
import numpy as np
import pytest

import paper_1907_05124_b200 as mb

B200 = dict(resident=(74, 33, 15), num_sms=148, np_=16384)


def _temps(runs, t_max, seed=0):
    return np.random.default_rng(seed).uniform(0.0, t_max, runs)


def test_cfg5_full_schedule_prefers_fewer_faster_slots():
    # 8192 descents, start temperatures over [0, 115]: 15 tiles at split 4 (3840 slots, runs
    # queued longest first) beat 32 tiles at split 2 (measured 17.9 vs 11.2 descents/s)
    prm = mb.MarsParams(t_min=0.0, t_max=115.0, start_mode=mb.StartMode.UniformRandom)
    assert mb.debug_choose_split(_temps(8192, 115.0), prm, pairs=32, **B200) == (4, 15)


def test_short_schedule_keeps_every_run_resident():
    # t_max = 3: every descent is short and about as long as the others -- all runs at once
    prm = mb.MarsParams(t_min=0.0, t_max=3.0, start_mode=mb.StartMode.UniformRandom)
    assert mb.debug_choose_split(_temps(8192, 3.0), prm, pairs=32, **B200) == (2, 32)


def test_small_shard_uses_the_widest_split():
    # the 1024-run share of an 8-GPU cfg5 run: 4 tiles, each split over 4 pairs
    prm = mb.MarsParams(t_min=0.0, t_max=115.0, start_mode=mb.StartMode.UniformRandom)
    assert mb.debug_choose_split(_temps(1024, 115.0), prm, pairs=4, **B200) == (4, 4)


def test_forced_split_and_residency_limits():
    prm = mb.MarsParams(t_min=0.0, t_max=115.0, start_mode=mb.StartMode.UniformRandom)
    t = _temps(8192, 115.0)
    assert mb.debug_choose_split(t, prm, pairs=32, forced=2, **B200) == (2, 32)
    # fewer resident 8-CTA clusters -> fewer split-4 tiles (the grid must be one wave)
    sp, tiles = mb.debug_choose_split(t, prm, pairs=32, forced=4, resident=(74, 33, 9), num_sms=148, np_=16384)
    assert (sp, tiles) == (4, 9)
    # a K range that does not split four ways (np / 32 chunks not divisible by 4)
    sp, _ = mb.debug_choose_split(t, prm, pairs=32, forced=0, resident=(74, 33, 15), num_sms=148, np_=8256)
    assert sp in (1, 2)


def test_bad_arguments_are_input_errors():
    prm = mb.MarsParams()
    with pytest.raises(mb.InputError):
        mb.debug_choose_split(_temps(16, 3.0), prm, pairs=0, **B200)
