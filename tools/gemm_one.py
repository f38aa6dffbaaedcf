"""Run one GEMM shape a few times (for ncu captures)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2305_16121_b200 import ops  # noqa: E402

M, N, K = (int(v) for v in os.environ.get("SHAPE", "4096,8192,2048").split(","))
amn, bmn = (int(v) for v in os.environ.get("MAJOR", "0,0").split(","))
A = torch.randn(M, K, device="cuda").bfloat16()
B = torch.randn(N, K, device="cuda").bfloat16()
a = A.t().contiguous() if amn else A
b = B.t().contiguous() if bmn else B
C = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
for _ in range(int(os.environ.get("ITERS", "3"))):
    ops.gemm(M, N, K, ops.operand(a, amn), ops.operand(b, bmn), C)
torch.cuda.synchronize()
print("ok")
