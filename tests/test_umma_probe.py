"""The tcgen05 / TMA / TMEM layer (csrc/umma.cuh, csrc/tma_host.hpp) on its own: a one-CTA
fp16 GEMM through the exact descriptors the dense relaxation kernel uses, against
torch.matmul (GPU).  Catches descriptor / swizzle / TMEM lane-mapping errors in isolation."""
import ctypes
import os

import pytest

from conftest import ROOT, gpu_available

PROBE = os.path.join(ROOT, "tests", "cuda", "libumma_probe.so")

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not gpu_available(), reason="needs a CUDA device")]


@pytest.mark.parametrize("N", [128, 256])
@pytest.mark.parametrize("K", [64, 192, 2048])
def test_umma_gemm_matches_torch(N, K):
    import torch
    lib = ctypes.CDLL(PROBE)
    lib.umma_probe.restype = ctypes.c_int
    lib.umma_probe.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_int]
    g = torch.Generator(device="cuda").manual_seed(N + K)
    A = torch.randn(128, K, device="cuda", generator=g).half()
    B = torch.randn(N, K, device="cuda", generator=g).half()
    D = torch.full((128, N), float("nan"), device="cuda")
    rc = lib.umma_probe(A.data_ptr(), B.data_ptr(), D.data_ptr(), K, N)
    assert rc == 0
    ref = A.float() @ B.float().T
    err = (D - ref).abs().max().item()
    assert err < 1e-3 * K ** 0.5, err
    # structured operands pin the row/column/K mapping exactly
    A = torch.zeros(128, K, device="cuda")
    for r in range(128):
        A[r, (r * 7) % K] = 1.0
    B = torch.arange(N * K, device="cuda").reshape(N, K).float().remainder(97).half()
    D.fill_(float("nan"))
    assert lib.umma_probe(A.half().data_ptr(), B.data_ptr(), D.data_ptr(), K, N) == 0
    assert torch.equal(D, A.half().float() @ B.float().T)


@pytest.mark.parametrize("N", [128, 256])
@pytest.mark.parametrize("K", [64, 2048])
def test_umma_ts_gemm_matches_torch(N, K):
    """A operand from TMEM (written with tcgen05.st, 2 fp16 per column), B from smem."""
    import torch
    lib = ctypes.CDLL(PROBE)
    lib.umma_probe_ts.restype = ctypes.c_int
    lib.umma_probe_ts.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_int]
    A = torch.zeros(128, K, device="cuda")
    for r in range(128):
        A[r, (r * 7) % K] = 1.0
        A[r, (r * 13 + 5) % K] += 2.0
    A = A.half()
    B = torch.arange(N * K, device="cuda").reshape(N, K).float().remainder(97).half()
    D = torch.full((128, N), float("nan"), device="cuda")
    assert lib.umma_probe_ts(A.data_ptr(), B.data_ptr(), D.data_ptr(), K, N) == 0
    assert torch.equal(D, A.float() @ B.float().T)
    g = torch.Generator(device="cuda").manual_seed(N + K)
    A = torch.randn(128, K, device="cuda", generator=g).half()
    B = torch.randn(N, K, device="cuda", generator=g).half()
    assert lib.umma_probe_ts(A.data_ptr(), B.data_ptr(), D.data_ptr(), K, N) == 0
    assert (D - A.float() @ B.float().T).abs().max().item() < 1e-3 * K ** 0.5
