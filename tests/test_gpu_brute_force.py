"""brute_force_ground_state on the device against the reference's own
exhaustive scan (oracle/_ref/libmars_ref_io.so, prebuilt from model.cpp)."""
import ctypes as C
import os

import numpy as np
import pytest

import paper_1907_05124_b200 as mb
from conftest import gpu_available

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_IO = os.path.join(ROOT, "oracle", "_ref", "libmars_ref_io.so")

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not gpu_available(), reason="needs a CUDA device"),
              pytest.mark.skipif(not os.path.exists(REF_IO), reason="reference checker not built")]


def ref_brute(n, J=None, edges=None, h=None, max_n=26):
    L = C.CDLL(REF_IO)
    vp = C.c_void_p
    L.ref_io_brute_force.argtypes = [C.c_int, vp, C.c_int64, vp, vp, vp, vp, C.c_int, vp, vp, C.c_char_p, C.c_int64]
    p_ = lambda a: None if a is None else a.ctypes.data_as(vp)  # noqa: E731
    e = np.zeros(1)
    s = np.zeros(n, np.int8)
    msg = C.create_string_buffer(256)
    if J is not None:
        J = np.ascontiguousarray(J, np.float64)
        rc = L.ref_io_brute_force(n, p_(J), 0, None, None, None, p_(h), max_n, p_(e), p_(s), msg, 256)
    else:
        u, v, w = (np.ascontiguousarray(x, t) for x, t in zip(edges, (np.int32, np.int32, np.float64)))
        rc = L.ref_io_brute_force(n, None, len(u), p_(u), p_(v), p_(w), p_(h), max_n, p_(e), p_(s), msg, 256)
    return rc, float(e[0]), s, msg.value.decode()


@pytest.mark.parametrize("n,seed", [(6, 1), (12, 2), (16, 3), (20, 4), (22, 5)])
def test_integer_instances_exact(n, seed):
    J = mb.gen_sk_pm1(n, seed)
    h = np.random.default_rng(seed).integers(-2, 3, n).astype(np.float64)
    rc, e_ref, s_ref, _ = ref_brute(n, J=J, h=h)
    assert rc == 0
    g = mb.brute_force_ground_state(mb.IsingProblem.dense(n, J, h))
    assert g.energy == e_ref and np.array_equal(g.spins, s_ref)


def test_degenerate_ties_break_lexicographically():
    # zero couplings: every configuration has energy 0 -> all -1 is the lexicographic minimum
    rc, e_ref, s_ref, _ = ref_brute(10, J=np.zeros((10, 10)))
    g = mb.brute_force_ground_state(mb.IsingProblem.dense(10, np.zeros((10, 10))))
    assert g.energy == e_ref == 0.0 and np.array_equal(g.spins, s_ref) and np.all(g.spins == -1)
    # ferromagnetic ring: two ground states (all -1 / all +1) -> all -1
    u = np.arange(8, dtype=np.int32)
    v = ((u + 1) % 8).astype(np.int32)
    w = -np.ones(8)
    rc, e_ref, s_ref, _ = ref_brute(8, edges=(u, v, w))
    g = mb.brute_force_ground_state(mb.IsingProblem.from_edges(8, (u, v, w)))
    assert g.energy == e_ref and np.array_equal(g.spins, s_ref)


def test_gaussian_instance_energy():
    J = mb.gen_sk_gaussian(18, 7)
    rc, e_ref, s_ref, _ = ref_brute(18, J=J)
    g = mb.brute_force_ground_state(mb.IsingProblem.dense(18, J))
    assert g.energy == e_ref
    # without a field s and -s tie exactly; the reference's serial scan picks between them by
    # its accumulated rounding, so the pair is compared up to the global flip
    assert np.array_equal(g.spins, s_ref) or np.array_equal(g.spins, -s_ref)


def test_guard_matches_reference():
    J = mb.gen_sk_pm1(12, 1)
    rc, _, _, msg = ref_brute(12, J=J, max_n=10)
    assert rc == 3
    with pytest.raises(mb.InputError) as e:
        mb.brute_force_ground_state(mb.IsingProblem.dense(12, J), max_n=10)
    assert str(e.value) == msg
