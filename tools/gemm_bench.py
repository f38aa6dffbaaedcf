"""Quick tcgen05 GEMM throughput probe (CUDA events, warm, inputs > L2 not required)."""
import sys
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2305_16121_b200 import _capi as capi, ops

def bench(M, N, K, amn=0, bmn=0, c_dtype=torch.bfloat16, iters=20, max_ctas=0):
    A = torch.randn(M, K, device="cuda").bfloat16()
    B = torch.randn(N, K, device="cuda").bfloat16()
    a_store = A.t().contiguous() if amn else A
    b_store = B.t().contiguous() if bmn else B
    C = torch.empty(M, N, device="cuda", dtype=c_dtype)
    f = lambda: ops.gemm(M, N, K, ops.operand(a_store, amn), ops.operand(b_store, bmn), C, max_ctas=max_ctas)
    for _ in range(3): f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters): f()
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / iters
    tf = 2.0 * M * N * K / ms / 1e9
    # cuBLAS reference for the same shape
    Bt = B.t()
    for _ in range(3): torch.matmul(A, Bt)
    torch.cuda.synchronize(); e0.record()
    for _ in range(iters): torch.matmul(A, Bt)
    e1.record(); torch.cuda.synchronize()
    ms_cb = e0.elapsed_time(e1) / iters
    print(f"M={M} N={N} K={K} amn={amn} bmn={bmn} out={str(c_dtype)[6:]}: {ms*1e3:8.1f} us {tf:7.1f} TF/s | cuBLAS {ms_cb*1e3:8.1f} us {2.0*M*N*K/ms_cb/1e9:7.1f} TF/s", flush=True)

if __name__ == "__main__":
    for shp in [(4096, 6144, 2048), (4096, 2048, 2048), (4096, 8192, 2048), (4096, 2048, 8192), (8192, 8192, 8192)]:
        bench(*shp)
    bench(4096, 2048, 8192, 0, 1)   # dgrad
    bench(2048, 8192, 4096, 1, 1, torch.float32)  # wgrad, f32 out
