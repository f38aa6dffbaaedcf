"""Warm timing of one bf16 GEMM shape (CUDA graph of back-to-back launches, operands rotated
over enough buffer sets to exceed L2).  SHAPE=M,N,K MAJOR=a,b  -> one JSON line."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2305_16121_b200 import ops  # noqa: E402

M, N, K = (int(v) for v in os.environ.get("SHAPE", "4096,2048,8192").split(","))
amn, bmn = (int(v) for v in os.environ.get("MAJOR", "0,0").split(","))
nsets = max(2, int(400e6 // (2 * (M * K + N * K + M * N))) + 1)
sets = []
for _ in range(nsets):
    A = torch.randn(M, K, device="cuda").bfloat16()
    B = torch.randn(N, K, device="cuda").bfloat16()
    sets.append((A.t().contiguous() if amn else A, B.t().contiguous() if bmn else B,
                 torch.empty(M, N, device="cuda", dtype=torch.bfloat16)))
run = lambda s: ops.gemm(M, N, K, ops.operand(s[0], amn), ops.operand(s[1], bmn), s[2])  # noqa: E731
for s in sets:
    run(s)
torch.cuda.synchronize()
rep = 4 * nsets
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    for i in range(rep):
        run(sets[i % nsets])
g.replay()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
g.replay()
e1.record()
torch.cuda.synchronize()
us = e0.elapsed_time(e1) / rep * 1e3
print(json.dumps({"shape": [M, N, K], "major": [amn, bmn], "us": us, "tflops": 2 * M * N * K / us / 1e6}))
