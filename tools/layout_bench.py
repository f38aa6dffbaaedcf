"""B-operand majorness x epilogue at the C2 FFN dgrad shape (4096 x 8192 x 2048):
is the dgrad's lower tensor-pipe share the MN-major weight operand or the
epilogue? CUDA events over a captured loop of 10 launches."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2305_16121_b200 import _capi as capi, ops  # noqa: E402
from pair_bench import timeit  # noqa: E402

M, N, K = (int(x) for x in os.environ.get("SHAPE", "4096,8192,2048").split(","))
bf = torch.bfloat16
a = torch.randn(M, K, device="cuda").to(bf)
b_k = torch.randn(N, K, device="cuda").to(bf)   # [N, K]: K-major
b_mn = b_k.t().contiguous()                       # [K, N]: MN-major
aux = torch.rand(M, N, device="cuda").to(bf)
c = torch.empty(M, N, device="cuda", dtype=bf)
fl = 2.0 * M * N * K
for name, bop in (("B K-major", ops.operand(b_k)), ("B MN-major", ops.operand(b_mn, True))):
    for ename, kw in (("plain", {}), ("MUL", dict(epilogue=capi.EPI_MUL, aux=aux)),
                      ("DGELU", dict(epilogue=capi.EPI_DGELU, aux=aux))):
        d = ops.gemm_desc(M, N, K, ops.operand(a), bop, c, **kw)
        timeit(lambda d=d: ops.gemm_grouped([d]), fl, f"{name} {ename} {M}x{N}x{K}")
