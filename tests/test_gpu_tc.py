"""tcgen05 plumbing: the 3xTF32 self-test GEMM against an fp64 matmul."""

import ctypes

import pytest
import torch

from paper_2004_06231_b200 import _native

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n,k", [(16, 8), (48, 40), (160, 40), (256, 64), (48, 16)])
def test_selftest_tf32_gemm(n, k):
    lib = _native.require_cuda()
    g = torch.Generator(device="cuda").manual_seed(n * 1000 + k)
    a = torch.rand((128, k), device="cuda", generator=g, dtype=torch.float32)
    b = torch.rand((n, k), device="cuda", generator=g, dtype=torch.float32)
    d = torch.full((128, n), float("nan"), device="cuda", dtype=torch.float32)
    rc = lib.einet_selftest_tf32_gemm(ctypes.c_void_p(a.data_ptr()), ctypes.c_void_p(b.data_ptr()),
                                      ctypes.c_void_p(d.data_ptr()), n, k,
                                      ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
    _native.check(rc, "selftest")
    want = a.double() @ b.double().T
    err = ((d.double() - want).abs() / want.abs().clamp_min(1e-30)).max().item()
    assert err < 2e-6, err
