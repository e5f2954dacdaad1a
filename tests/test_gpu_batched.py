"""Tensor-core (tcgen05) batched correlation GEMM vs a torch fp32 reference of the same op."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_1412_4080_b200 import _native as nat  # noqa: E402


def _gemm(A, B, S, Nb):
    L = nat.lib()
    M, K = A.shape
    C = torch.empty((Nb, M), dtype=torch.float32, device=A.device)
    nat.check(L.dscr_batched_gemm_bf16(A.data_ptr(), M, K, B.data_ptr(), Nb, K, K, S, C.data_ptr(), M,
                                       nat.stream_ptr()))
    return C


@pytest.mark.parametrize("M,Nb,K,S", [(128, 256, 64, 1), (256, 512, 128, 1), (384, 256, 192, 2), (1024, 1024, 1024, 1)])
def test_gemm_matches_fp32_reference(M, Nb, K, S):
    g = torch.Generator(device="cuda").manual_seed(M + Nb + K + S)
    A = torch.randn(M, K, device="cuda", generator=g).to(torch.bfloat16)
    B = torch.randn(S * Nb, K, device="cuda", generator=g).to(torch.bfloat16)
    C = _gemm(A, B, S, Nb)
    torch.cuda.synchronize()
    ref = sum(B[s * Nb:(s + 1) * Nb].double() @ A.double().T for s in range(S))
    err = (C.double() - ref).abs().max().item()
    scale = (B.double().abs().max() * A.double().abs().max() * K * S).item()
    assert err <= 1e-6 * scale, (err, scale)


def test_gemm_c5_shape_throughput():
    M, Nb, K = 16384, 4096, 1024
    A = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    B = torch.randn(Nb, K, device="cuda").to(torch.bfloat16)
    C = _gemm(A, B, 1, Nb)
    torch.cuda.synchronize()
    idx = torch.randint(0, M, (64,), device="cuda")
    ref = (B.float() @ A[idx].float().T)
    assert torch.allclose(C[:, idx], ref, rtol=1e-3, atol=1e-2)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(3):
        _gemm(A, B, 1, Nb)
    ev0.record()
    for _ in range(10):
        _gemm(A, B, 1, Nb)
    ev1.record()
    torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1) / 10
    tflops = 2 * M * Nb * K / ms / 1e9
    print(f"\nc5 D^T Theta: {ms * 1e3:.1f} us, {tflops:.0f} TFLOP/s")
    assert tflops > 200
