"""One dGeLU dgrad and one f32-accumulate wgrad launch at C2 FFN shapes (ncu captures)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2305_16121_b200 import _capi as capi, ops  # noqa: E402

Ts, h, f = 4096, 2048, 8192
bf = torch.bfloat16
gar = torch.randn(Ts, h, device="cuda").to(bf)
act = torch.randn(Ts, f, device="cuda").to(bf)
w = torch.randn(h, f, device="cuda").to(bf)
dW = torch.zeros(h, f, device="cuda")
pre = torch.randn(Ts, f, device="cuda").to(bf)
dcol = torch.empty(Ts, f, device="cuda", dtype=bf)
dw = ops.gemm_desc(h, f, Ts, ops.operand(gar, True), ops.operand(act, True), dW, accumulate=True)
dd = ops.gemm_desc(Ts, f, h, ops.operand(gar), ops.operand(w, True), dcol, epilogue=capi.EPI_DGELU, aux=pre)
for _ in range(int(os.environ.get("ITERS", "2"))):
    ops.gemm_grouped([dd])
    ops.gemm_grouped([dw])
torch.cuda.synchronize()
print("ok")
