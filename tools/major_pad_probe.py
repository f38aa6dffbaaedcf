"""Probe: does the MN/MN GEMM penalty depend on the operands' row pitch?
Times 4096x8192x2048 with both operands MN-major at pitch = width and width + PAD."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2305_16121_b200 import _capi as capi, ops  # noqa: E402

M, N, K = 4096, 8192, 2048


def operand_view(t, mn, rows, cols, ld):
    o = capi.GemmOperand()
    o.ptr, o.rows, o.cols, o.ld, o.mn_major = t.data_ptr(), rows, cols, ld, int(mn)
    return o


def run(pad, amn, bmn, nsets=4, rep=16):
    sets = []
    for _ in range(nsets):
        if amn:
            a = torch.randn(K, M + pad, device="cuda").bfloat16()
            oa = (a, K, M, M + pad)
        else:
            a = torch.randn(M, K + pad, device="cuda").bfloat16()
            oa = (a, M, K, K + pad)
        if bmn:
            b = torch.randn(K, N + pad, device="cuda").bfloat16()
            ob = (b, K, N, N + pad)
        else:
            b = torch.randn(N, K + pad, device="cuda").bfloat16()
            ob = (b, N, K, K + pad)
        sets.append((oa, ob, torch.empty(M, N, device="cuda", dtype=torch.bfloat16)))

    def fn(s):
        (a, ar, ac, al), (b, br, bc, bl), c = s
        ops.gemm(M, N, K, operand_view(a, amn, ar, ac, al), operand_view(b, bmn, br, bc, bl), c)

    for s in sets:
        fn(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for i in range(rep):
            fn(sets[i % nsets])
    g.replay()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(); g.replay(); e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / rep * 1e3


for pad in (0, 64, 128):
    for amn, bmn in ((0, 0), (1, 1), (0, 1), (1, 0)):
        us = run(pad, amn, bmn)
        print(json.dumps({"pad": pad, "major": [amn, bmn], "us": round(us, 2), "tflops": round(2 * M * N * K / us / 1e6, 1)}),
              flush=True)
