"""cuBLAS (torch.matmul) bf16 time on the c5 correlation shape, for comparison with k_gemm_dt."""
import torch

M, N, K = 16384, 4096, 1024
a = torch.randn(N, K, device="cuda", dtype=torch.bfloat16)
b = torch.randn(M, K, device="cuda", dtype=torch.bfloat16)
for dt_out in (torch.bfloat16, torch.float32):
    for _ in range(5):
        c = torch.matmul(a, b.T)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        c = torch.matmul(a, b.T) if dt_out == torch.bfloat16 else torch.matmul(a, b.T).float()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 20
    print(f"cuBLAS {dt_out}: {ms * 1e3:.1f} us, {2 * M * N * K / ms / 1e9:.0f} TFLOP/s")
