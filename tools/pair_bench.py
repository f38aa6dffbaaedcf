"""Backward GEMM pairs at C2 sub-batch shapes, exactly as Stack::backward issues
them (wgrad f32-accumulate + dgrad with/without the dGeLU epilogue), timed
alone and grouped (CUDA events over a captured loop)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2305_16121_b200 import _capi as capi, ops  # noqa: E402

Ts, h = 4096, 2048
bf = torch.bfloat16
REP = 10


def timeit(fn, flops, name):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(REP):
            fn()
    g.replay()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    s.record()
    g.replay()
    e.record()
    torch.cuda.synchronize()
    us = s.elapsed_time(e) / REP * 1e3
    print(f"{name:44s} {us:8.1f} us  {flops / us / 1e6:7.1f} TF/s", flush=True)


def pair(nrow, ncol_name, dgelu):
    gar = torch.randn(Ts, h, device="cuda").to(bf)
    act = torch.randn(Ts, nrow, device="cuda").to(bf)
    w = torch.randn(h, nrow, device="cuda").to(bf)
    dW = torch.zeros(h, nrow, device="cuda")
    pre = torch.randn(Ts, nrow, device="cuda").to(bf)
    dcol = torch.empty(Ts, nrow, device="cuda", dtype=bf)
    dw = ops.gemm_desc(h, nrow, Ts, ops.operand(gar, True), ops.operand(act, True), dW, accumulate=True)
    kw = dict(epilogue=capi.EPI_DGELU, aux=pre) if dgelu else {}
    dd = ops.gemm_desc(Ts, nrow, h, ops.operand(gar), ops.operand(w, True), dcol, **kw)
    fl_w = 2.0 * h * nrow * Ts
    fl_d = 2.0 * Ts * nrow * h
    timeit(lambda: ops.gemm_grouped([dw]), fl_w, f"{ncol_name} wgrad f32 acc {h}x{nrow}x{Ts}")
    timeit(lambda: ops.gemm_grouped([dd]), fl_d, f"{ncol_name} dgrad {'dGeLU ' if dgelu else ''}{Ts}x{nrow}x{h}")
    timeit(lambda: ops.gemm_grouped([dw, dd]), fl_w + fl_d, f"{ncol_name} grouped pair")


def col_pair(ncol, name):
    dcol = torch.randn(Ts, ncol, device="cuda").to(bf)
    ln = torch.randn(Ts, h, device="cuda").to(bf)
    w = torch.randn(ncol, h, device="cuda").to(bf)
    dW = torch.zeros(ncol, h, device="cuda")
    out = torch.empty(Ts, h, device="cuda", dtype=bf)
    dw = ops.gemm_desc(ncol, h, Ts, ops.operand(dcol, True), ops.operand(ln, True), dW, accumulate=True)
    dd = ops.gemm_desc(Ts, h, ncol, ops.operand(dcol), ops.operand(w, True), out)
    fl = 2.0 * ncol * h * Ts
    timeit(lambda: ops.gemm_grouped([dw]), fl, f"{name} wgrad f32 acc {ncol}x{h}x{Ts}")
    timeit(lambda: ops.gemm_grouped([dd]), fl, f"{name} dgrad {Ts}x{h}x{ncol}")
    timeit(lambda: ops.gemm_grouped([dw, dd]), 2 * fl, f"{name} grouped pair")


def fwd(N, K, name, gelu=False):
    a = torch.randn(Ts, K, device="cuda").to(bf)
    w = torch.randn(N, K, device="cuda").to(bf)
    c = torch.empty(Ts, N, device="cuda", dtype=bf)
    c2 = torch.empty(Ts, N, device="cuda", dtype=bf)
    bias = torch.zeros(N, device="cuda", dtype=bf)
    kw = dict(epilogue=capi.EPI_BIAS_GELU, c2=c2, bias=bias) if gelu else {}
    d = ops.gemm_desc(Ts, N, K, ops.operand(a), ops.operand(w), c, **kw)
    timeit(lambda: ops.gemm_grouped([d]), 2.0 * Ts * N * K, f"{name} fwd {Ts}x{N}x{K}")


if __name__ == "__main__":
    fwd(3 * h, h, "QKV")
    fwd(h, h, "proj")
    fwd(4 * h, h, "FC1 +bias+GeLU", gelu=True)
    fwd(h, 4 * h, "FC2")
    pair(4 * h, "FC2 bwd", True)
    pair(h, "proj bwd", False)
    col_pair(4 * h, "FC1 bwd")
    col_pair(3 * h, "QKV bwd")
