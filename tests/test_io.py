"""Instance I/O and result documents against the reference's own
io.cpp, compiled by oracle/Makefile into oracle/_ref/libmars_ref_io.so (test-only checker;
skipped where the reference sources are absent).  CPU only: parsing, writing, problem_hash
and the JSON document of a batch need no device (the batch records come from the C port,
which equals the reference bit for bit -- tests/test_oracle.py)."""
import ctypes as C
import os

import numpy as np
import pytest

import paper_1907_05124_b200 as mb
from paper_1907_05124_b200 import io as mio

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_IO = os.path.join(ROOT, "oracle", "_ref", "libmars_ref_io.so")

pytestmark = pytest.mark.skipif(not os.path.exists(REF_IO), reason="reference io checker not built")


@pytest.fixture(scope="module")
def ref():
    L = C.CDLL(REF_IO)
    vp, i32, i64 = C.c_void_p, C.c_int32, C.c_int64
    L.ref_io_parse_gset.argtypes = [C.c_char_p, vp, vp, vp, vp, vp, i64, C.c_char_p, i64]
    L.ref_io_read_matrix.argtypes = [C.c_char_p, vp, vp, i64, C.c_char_p, i64]
    L.ref_io_detect_format.argtypes = [C.c_char_p, C.c_char_p, i64]
    L.ref_io_problem_hash.argtypes = [i32, vp, i64, vp, vp, vp, vp]
    L.ref_io_problem_hash.restype = C.c_uint64
    L.ref_io_write_matrix.argtypes = [i32, vp, i64, vp, vp, vp, C.c_char_p, i64]
    L.ref_io_write_gset.argtypes = [i32, i64, vp, vp, vp, C.c_char_p, i64]
    L.ref_io_result_document.argtypes = [i32, vp, i64, vp, vp, vp, vp, vp, i64, C.c_uint64, C.c_int,
                                         C.c_char_p, C.c_char_p, i64]
    return L


def p_(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


ERR = {1: mio.ParseError, 2: mio.StructuralError, 3: mb.InputError}


def ref_gset(L, text):
    n, m = np.zeros(1, np.int32), np.zeros(1, np.int64)
    cap = 4096
    u, v, w = np.zeros(cap, np.int32), np.zeros(cap, np.int32), np.zeros(cap, np.int64)
    msg = C.create_string_buffer(512)
    rc = L.ref_io_parse_gset(text.encode(), p_(n), p_(m), p_(u), p_(v), p_(w), cap, msg, 512)
    if rc:
        return rc, msg.value.decode()
    k = int(m[0])
    return 0, (int(n[0]), list(zip(u[:k].tolist(), v[:k].tolist(), w[:k].tolist())))


def ours(fn, text):
    try:
        return 0, fn(text)
    except (mio.ParseError, mio.StructuralError, mb.InputError) as e:
        code = 1 if isinstance(e, mio.ParseError) else (2 if isinstance(e, mio.StructuralError) else 3)
        return code, str(e)


GSET_CASES = [
    "3 2\n1 2 1\n2 3 -1\n",
    "# comment\n% other\n\n4 3\n1 2\n  2 3 5\n3 4 -7\n",
    "3 2\r\n1 2 1\r\n2 3 1\r\n",          # CRLF: '\r' is whitespace to the tokenizer
    "5 0\n",
    "",                                     # missing header
    "3\n1 2 1\n",                           # header with one token
    "3 x\n",                                # bad integer
    "0 0\n",                                # vertex count must be positive
    "3 -1\n",                               # negative edge count reads as missing header
    "3 2\n1 2 1\n",                         # count mismatch
    "3 1\n1 2 1\n2 3 1\n",                  # more edge lines than declared
    "3 2\n1 2 1\n2 1 4\n",                  # duplicate edge (reversed)
    "3 1\n2 2 1\n",                         # self loop
    "3 1\n1 4 1\n",                         # out of range
    "3 1\n1 2 1 9\n",                       # four tokens
    "3 1\n1 2 +1\n",                        # from_chars rejects '+'
    "3 1\n1 2 1.5\n",                       # non-integer weight
    "3 1\n1 2 99999999999999999999\n",      # out of range long long
    "3 1\n0 2 1\n",
]


@pytest.mark.parametrize("text", GSET_CASES)
def test_parse_gset_matches_reference(ref, text):
    rc, want = ref_gset(ref, text)
    code, got = ours(mio.parse_gset, text)
    assert code == rc, (got, want)
    if rc:
        assert got == want
    else:
        assert (got.n_vertices, [(e.u, e.v, e.w) for e in got.edges]) == want


def ref_matrix(L, text):
    n = np.zeros(1, np.int32)
    cap = 64 * 64
    J = np.zeros(cap)
    msg = C.create_string_buffer(512)
    rc = L.ref_io_read_matrix(text.encode(), p_(n), p_(J), cap, msg, 512)
    if rc:
        return rc, msg.value.decode()
    k = int(n[0])
    return 0, J[:k * k].reshape(k, k)


MATRIX_CASES = [
    "2\n0 1.5\n1.5 0\n",
    "# c\n3\n0 -1 2e-3\n-1 0 0x1p-2\n0.002 0.25 0\n",
    "2\n0 inf\ninf 0\n",
    "2\n0 nan\nnan 0\n",
    "2\n0 1e999\n1e999 0\n",               # overflow -> out_of_range
    "2\n0 1e-320\n1e-320 0\n",             # underflow -> out_of_range
    "2\n0 1_0\n1_0 0\n",                   # Python float() would accept this
    "2\n0 1\n2 0\n",                        # asymmetric -> StructuralError
    "2\n1 0\n0 0\n",                        # diagonal
    "2\n0 1\n",                             # ends early
    "2 2\n0 1\n1 0\n",                      # header with two tokens
    "0\n",
    "-3\n",
    "",
    "2\n0 1 2\n1 0\n",                      # wrong row length
    "2\n0 1x\n1 0\n",
    "3\n0 1 0\n1 0 1\n0 1 0\n# trailing comment\n",
]


@pytest.mark.parametrize("text", MATRIX_CASES)
def test_read_matrix_matches_reference(ref, text):
    rc, want = ref_matrix(ref, text)
    code, got = ours(mio.parse_matrix, text)
    assert code == rc, (got, want)
    if rc:
        assert got == want
    else:
        np.testing.assert_array_equal(got, want)   # NaN == NaN positions included


@pytest.mark.parametrize("text", ["3 2\n", "# x\n4\n", "1 2 3\n", "", "\n\n% c\n", "  7  \n"])
def test_detect_format_matches_reference(ref, text):
    msg = C.create_string_buffer(512)
    rc = ref.ref_io_detect_format(text.encode(), msg, 512)
    try:
        fmt = mio.detect_format(text)
        assert rc == fmt.value
    except mio.ParseError as e:
        assert rc < 0 and str(e) == msg.value.decode()


def instances():
    rng = np.random.default_rng(3)
    J = mb.gen_sk_gaussian(40, 5)
    yield "sk_gauss", 40, dict(J=J)
    yield "sk_pm1_field", 24, dict(J=mb.gen_sk_pm1(24, 2), field=rng.standard_normal(24))
    u, v, w = mb.gen_er(300, 0.02, 9)
    yield "er_csr", 300, dict(edges=(u, v, w))
    u, v, w = mb.gen_er(60, 0.3, 4)
    yield "er_dense_storage", 60, dict(edges=(u, v, w))
    u, v, w = mb.gen_ea(8, 3, 5)
    yield "ea3d", 512, dict(edges=(u, v, w))
    # duplicate edges: dense storage accumulates, CSR keeps both entries (sorted by (j, w))
    yield "dup_csr", 100, dict(edges=(np.array([0, 1, 0], np.int32), np.array([5, 7, 5], np.int32),
                                      np.array([2.0, -1.0, -3.0])))
    yield "dup_dense", 4, dict(edges=(np.array([0, 1, 0], np.int32), np.array([3, 2, 3], np.int32),
                                      np.array([2.0, -1.0, -3.0])))


@pytest.mark.parametrize("name,n,kw", list(instances()), ids=[x[0] for x in instances()])
def test_problem_hash_matches_reference(ref, name, n, kw):
    J = kw.get("J")
    J = None if J is None else np.ascontiguousarray(J, np.float64)
    h = kw.get("field")
    h = None if h is None else np.ascontiguousarray(h, np.float64)
    if J is not None:
        want = ref.ref_io_problem_hash(n, p_(J), 0, None, None, None, p_(h))
    else:
        u, v, w = (np.ascontiguousarray(x, t) for x, t in zip(kw["edges"], (np.int32, np.int32, np.float64)))
        want = ref.ref_io_problem_hash(n, None, len(u), p_(u), p_(v), p_(w), p_(h))
    got = mio.problem_hash(mio.HostInstance(n, J, kw.get("edges"), h))
    assert got == want and mio.hash_to_hex(got) == "%016x" % want


def test_writers_match_reference(ref):
    out = C.create_string_buffer(1 << 20)
    J = mb.gen_sk_gaussian(12, 8)
    J[0, 5] = J[5, 0] = 1e-310        # subnormal and large values through %.17g
    J[1, 2] = J[2, 1] = 1.5e300
    assert ref.ref_io_write_matrix(12, p_(np.ascontiguousarray(J)), 0, None, None, None, out, 1 << 20) == 0
    assert mio.matrix_text(J) == out.value.decode()
    g = mio.parse_gset("5 3\n1 2 3\n5 1 -2\n2 4\n")
    u = np.array([e.u for e in g.edges], np.int32)
    v = np.array([e.v for e in g.edges], np.int32)
    w = np.array([e.w for e in g.edges], np.int64)
    assert ref.ref_io_write_gset(5, 3, p_(u), p_(v), p_(w), out, 1 << 20) == 0
    assert mio.write_gset(g) == out.value.decode()
    # a written G-set parses back to the same graph
    assert mio.parse_gset(mio.write_gset(g)) == g


def test_nlohmann_double_format():
    cases = [(0.0, "0.0"), (-0.0, "-0.0"), (6120.0, "6120.0"), (-135163.12840009082, "-135163.12840009082"),
             (0.001, "0.001"), (1e-05, "1e-05"), (0.5, "0.5"), (1e15, "1e+15"), (1e14, "100000000000000.0"),
             (123.456, "123.456"), (1.5e-07, "1.5e-07"), (5e-324, "5e-324"),
             (1.7976931348623157e308, "1.7976931348623157e+308"), (0.1, "0.1"), (2.5e-4, "0.00025")]
    for v, s in cases:
        assert mio._nlohmann_double(v) == s, (v, mio._nlohmann_double(v), s)


def port_stats(port, inst, prm, runs, seed):
    """The C port's batch (== the reference's bit for bit) aggregated by the native
    index-order aggregation, as BatchStats with every run's spins."""
    from oracle.oracle import params
    n = inst.n
    if inst.J is not None:
        op = port.problem_dense(inst.J, inst.field)
    else:
        op = port.problem_edges(n, *inst.edges, inst.field)
    ob = op.run_batch(params(prm.t_min, prm.t_max, prm.t_step, prm.c_step, prm.d_min,
                             uniform=prm.start_mode == mb.StartMode.UniformRandom), runs, seed)
    rec = mb.Records(ob.status.copy(), ob.energy.copy(), ob.cut.copy(), ob.start_temp.copy(),
                     ob.descent_iters.copy(), np.zeros(len(ob.status)), ob.spins.copy())
    integral = np.all(np.equal(np.mod(inst.J if inst.J is not None else inst.edges[2], 1), 0))
    st = mb.aggregate(rec, 0.0 if integral and inst.field is None else 1e-9, 0.0)
    return st


def ref_doc(L, inst, prm, runs, seed, detail, pid):
    out = C.create_string_buffer(1 << 22)
    c = np.zeros(1)   # keep alive
    from oracle.oracle import params
    op = params(prm.t_min, prm.t_max, prm.t_step, prm.c_step, prm.d_min,
                uniform=prm.start_mode == mb.StartMode.UniformRandom)
    h = None if inst.field is None else np.ascontiguousarray(inst.field, np.float64)
    if inst.J is not None:
        J = np.ascontiguousarray(inst.J, np.float64)
        rc = L.ref_io_result_document(inst.n, p_(J), 0, None, None, None, p_(h), C.byref(op), runs, seed,
                                      int(detail), pid.encode(), out, 1 << 22)
    else:
        u, v, w = (np.ascontiguousarray(x, t) for x, t in zip(inst.edges, (np.int32, np.int32, np.float64)))
        rc = L.ref_io_result_document(inst.n, None, len(u), p_(u), p_(v), p_(w), p_(h), C.byref(op), runs,
                                      seed, int(detail), pid.encode(), out, 1 << 22)
    del c
    assert rc == 0, out.value.decode()
    return out.value.decode()


DOC_CASES = [
    ("sk20_pm1_random", mio.HostInstance(20, J=None), mb.MarsParams(0, 8, 1, 1, 1e-4, mb.StartMode.UniformRandom), 48),
    ("sk12_gauss_grid", None, mb.MarsParams(0, 10, 0.5), 1),
    ("er200_csr", None, mb.MarsParams(0, 10, 1, 1, 1e-4, mb.StartMode.UniformRandom), 32),
]


def doc_instance(name):
    if name == "sk20_pm1_random":
        return mio.HostInstance(20, J=mb.gen_sk_pm1(20, 3))
    if name == "sk12_gauss_grid":
        return mio.HostInstance(12, J=mb.gen_sk_gaussian(12, 4001))
    u, v, w = mb.gen_er(200, 0.03, 6)
    return mio.HostInstance(200, edges=(u, v, w))


@pytest.mark.parametrize("name,_inst,prm,runs", DOC_CASES, ids=[c[0] for c in DOC_CASES])
@pytest.mark.parametrize("detail", list(mio.DocDetail))
def test_result_document_byte_identical(ref, port, name, _inst, prm, runs, detail):
    inst = doc_instance(name)
    st = port_stats(port, inst, prm, runs, 7)
    doc = mio.make_result_document(name, inst, prm, st, detail, include_volatile=False)
    text = mio.result_document_to_string(doc)
    assert text == ref_doc(ref, inst, prm, runs, 7, detail, name)
    # and it reads back to the same document
    back = mio.result_document_from_string(text)
    assert mio.result_document_to_string(back) == text
    mio.verify_result_document(back, inst)
    with pytest.raises(mio.IntegrityError):
        mio.verify_result_document(back, mio.HostInstance(inst.n, J=np.zeros((inst.n, inst.n))))


def test_document_errors():
    with pytest.raises(mio.ParseError, match="not a mars-result"):
        mio.result_document_from_string('{"format": "x"}')
    with pytest.raises(mio.VersionError):
        mio.result_document_from_string('{"format": "mars-result", "version": 2}')
    with pytest.raises(mio.ParseError, match="invalid result document"):
        mio.result_document_from_string("{")
