"""Our tcgen05 GEMM vs cuBLAS (torch.matmul) on the C2 layer shapes, same warm
protocol (CUDA graph of back-to-back launches over operand sets larger than L2).

    python tools/cublas_compare.py   -> one JSON line per shape
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2305_16121_b200 import ops  # noqa: E402

SHAPES = [  # (M, N, K, A MN-major, B MN-major, what)
    (4096, 6144, 2048, 0, 0, "QKV fwd"), (4096, 2048, 2048, 0, 0, "proj fwd"),
    (4096, 8192, 2048, 0, 0, "FC1 fwd"), (4096, 2048, 8192, 0, 0, "FC2 fwd"),
    (4096, 8192, 2048, 0, 1, "FC2 dgrad"), (4096, 2048, 8192, 0, 1, "FC1 dgrad"),
    (2048, 8192, 8192, 1, 1, "FC2 wgrad"), (8192, 2048, 8192, 1, 1, "FC1 wgrad"),
]


def timed(fn, sets, rep):
    for s in sets:
        fn(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for i in range(rep):
            fn(sets[i % len(sets)])
    g.replay()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / rep * 1e3


for M, N, K, amn, bmn, what in SHAPES:
    nsets = max(2, int(400e6 // (2 * (M * K + N * K + M * N))) + 1)
    sets = []
    for _ in range(nsets):
        A = torch.randn(M, K, device="cuda").bfloat16()
        B = torch.randn(N, K, device="cuda").bfloat16()
        a = A.t().contiguous() if amn else A  # stored [K, M] when MN-major
        b = B.t().contiguous() if bmn else B  # stored [K, N] when MN-major
        sets.append((a, b, torch.empty(M, N, device="cuda", dtype=torch.bfloat16)))
    ours = timed(lambda s: ops.gemm(M, N, K, ops.operand(s[0], amn), ops.operand(s[1], bmn), s[2]), sets, 4 * nsets)
    # cuBLAS on the same storage: C = A' B'^T with A' = a or a^T, B' = b or b^T (views, no copies)
    cub = timed(lambda s: torch.matmul(s[0].t() if amn else s[0], s[1] if bmn else s[1].t(), out=s[2]), sets,
                4 * nsets)
    fl = 2 * M * N * K
    print(json.dumps({"shape": [M, N, K], "what": what, "major": [amn, bmn], "ours_us": round(ours, 2),
                      "cublas_us": round(cub, 2), "ours_tflops": round(fl / ours / 1e6, 1),
                      "cublas_tflops": round(fl / cub / 1e6, 1), "ratio": round(cub / ours, 3)}), flush=True)
