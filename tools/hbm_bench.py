"""Warm back-to-back timing of the HBM-bound kernels at C2 sub-batch shapes (CUDA events)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2305_16121_b200 import ops  # noqa: E402

HBM = 6532.9e9
T, h, f = 4096, 2048, 8192
bf = torch.bfloat16
x = torch.randn(T, h, device="cuda").to(bf)
r = torch.randn(T, h, device="cuda").to(bf)
y = torch.empty_like(x)
g = torch.ones(h, device="cuda", dtype=bf)
b = torch.zeros(h, device="cuda", dtype=bf)
big = torch.randn(T, f, device="cuda").to(bf)
db = torch.zeros(h, device="cuda")
dbf = torch.zeros(f, device="cuda")
dg = torch.zeros(h, device="cuda")
dbe = torch.zeros(h, device="cuda")


def timeit(fn, nbytes, name, rep=20):
    # captured into a CUDA graph so host launch overhead does not starve the GPU
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr):
        for _ in range(rep):
            fn()
    gr.replay()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    s.record()
    gr.replay()
    e.record()
    torch.cuda.synchronize()
    us = s.elapsed_time(e) / rep * 1e3
    print(f"{name:34s} {us:7.2f} us  {nbytes / us / 1e3:7.0f} GB/s  ({nbytes / (us * 1e-6) / HBM:4.2f} of HBM)")


B = 2
timeit(lambda: ops.layernorm_fwd(x, g, b, y), 2 * T * h * B, "layernorm_fwd")
timeit(lambda: ops.layernorm_bwd(x, g, r, y, dg, dbe, accumulate_dx=True), 6 * T * h * B,
       "layernorm_bwd (+dgamma/dbeta)")
timeit(lambda: ops.bias_dropout_residual_fwd(x, b, r, y, dropout_p=0.1, seed=1, offset=2), 3 * T * h * B,
       "bias_dropout_residual_fwd p=0.1")
timeit(lambda: ops.bias_dropout_residual_layernorm_fwd(x, b, r, y, g, b, r, dropout_p=0.1, seed=1, offset=2),
       4 * T * h * B, "fused bdr + layernorm_fwd p=0.1")
timeit(lambda: ops.bias_dropout_residual_bwd(x, y, db, dropout_p=0.1, seed=1, offset=2), 2 * T * h * B,
       "dropout' + dbias (col_pass)")
timeit(lambda: ops.colsum(big, dbf), T * f * B, "colsum [4096 x 8192]")
