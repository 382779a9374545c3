"""SURVEY.md 8(f) rows 1-2 on the device: instances ingested through the I/O mirror (G-set
text, dense-matrix text) run on the B200, and the JSON result document of the GPU batch is
byte-identical to the one the reference's own io.cpp writes for its CPU batch of the same
instance, parameters and seed (oracle/_ref/libmars_ref_io.so, prebuilt; the trajectories of
these small instances match run for run)."""
import ctypes as C
import os

import numpy as np
import pytest

import paper_1907_05124_b200 as mb
from conftest import gpu_available
from paper_1907_05124_b200 import io as mio

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_IO = os.path.join(ROOT, "oracle", "_ref", "libmars_ref_io.so")

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not gpu_available(), reason="needs a CUDA device"),
              pytest.mark.skipif(not os.path.exists(REF_IO), reason="reference io checker not built")]


def ref_document(inst, prm, runs, seed, detail, pid):
    L = C.CDLL(REF_IO)
    vp, i32, i64 = C.c_void_p, C.c_int32, C.c_int64
    L.ref_io_result_document.argtypes = [i32, vp, i64, vp, vp, vp, vp, vp, i64, C.c_uint64, C.c_int,
                                         C.c_char_p, C.c_char_p, i64]
    from oracle.oracle import params
    op = params(prm.t_min, prm.t_max, prm.t_step, prm.c_step, prm.d_min,
                uniform=prm.start_mode == mb.StartMode.UniformRandom)
    out = C.create_string_buffer(1 << 22)
    p_ = lambda a: None if a is None else a.ctypes.data_as(vp)  # noqa: E731
    if inst.J is not None:
        J = np.ascontiguousarray(inst.J, np.float64)
        rc = L.ref_io_result_document(inst.n, p_(J), 0, None, None, None, None, C.byref(op), runs, seed,
                                      int(detail), pid.encode(), out, 1 << 22)
    else:
        u, v, w = (np.ascontiguousarray(x, t) for x, t in zip(inst.edges, (np.int32, np.int32, np.float64)))
        rc = L.ref_io_result_document(inst.n, None, len(u), p_(u), p_(v), p_(w), None, C.byref(op), runs, seed,
                                      int(detail), pid.encode(), out, 1 << 22)
    assert rc == 0, out.value.decode()
    return out.value.decode()


def test_gset_file_to_gpu_document(tmp_path):
    # a G-set file (1-based, integer weights) -> parse -> device problem -> GPU batch -> document
    u, v, w = mb.gen_er(200, 0.03, 6)
    g = mio.GsetGraph(200, [mio.GsetEdge(int(a) + 1, int(b) + 1, int(c)) for a, b, c in zip(u, v, w)])
    path = tmp_path / "er200.gset"
    path.write_text(mio.write_gset(g))
    loaded = mio.load_problem(str(path))
    assert loaded.format == mio.InstanceFormat.GsetGraph and loaded.problem.kernel() == "csr"
    prm = mb.MarsParams(0, 10, 1, 1, 1e-4, mb.StartMode.UniformRandom)
    stats = mb.run_batch(loaded.problem, mb.BatchSpec(prm, 32, 7, keep_spins=True))
    inst = mio.HostInstance(200, edges=mio.gset_edges(g))
    assert mio.problem_hash(loaded.problem) == mio.problem_hash(inst)
    for detail in mio.DocDetail:
        doc = mio.make_result_document("er200", loaded.problem, prm, stats, detail, include_volatile=False)
        assert mio.result_document_to_string(doc) == ref_document(inst, prm, 32, 7, detail, "er200")
    out = tmp_path / "er200.json"
    mio.save_result(mio.make_result_document("er200", loaded.problem, prm, stats), str(out))
    mio.verify_result_document(mio.load_result(str(out)), loaded.problem)


def test_matrix_file_to_gpu_document(tmp_path):
    J = mb.gen_sk_pm1(20, 3)
    path = tmp_path / "sk20.txt"
    path.write_text(mio.matrix_text(J))
    loaded = mio.load_problem(str(path))
    assert loaded.format == mio.InstanceFormat.DenseMatrix
    assert mio.write_matrix(loaded.problem) == path.read_text()
    prm = mb.MarsParams(0, 8, 1, 1, 1e-4, mb.StartMode.UniformRandom)
    stats = mb.run_batch(loaded.problem, mb.BatchSpec(prm, 48, 7, keep_spins=True))
    inst = mio.HostInstance(20, J=J)
    for detail in (mio.DocDetail.Summary, mio.DocDetail.Energies):
        doc = mio.make_result_document("sk20", loaded.problem, prm, stats, detail, include_volatile=False)
        assert mio.result_document_to_string(doc) == ref_document(inst, prm, 48, 7, detail, "sk20")
