"""One launch each of the LayerNorm row kernels at a sub-batch shape (for ncu):
plain forward, bias-dropout-residual forward, backward (+ parameter finalize).

    python tools/lnp_one.py [T] [h]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2305_16121_b200 import ops  # noqa: E402

T = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
h = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
bf = torch.bfloat16
x, r, y, z = ((torch.randn(T, h, device="cuda") * 0.5 + 0.1).to(bf) for _ in range(4))
g = (torch.rand(h, device="cuda") + 0.5).to(bf)
b = (torch.randn(h, device="cuda") * 0.1).to(bf)
dg = torch.zeros(h, device="cuda")
dbe = torch.zeros(h, device="cuda")
ops.layernorm_fwd(x, g, b, y)
ops.bias_dropout_residual_layernorm_fwd(x, b, r, y, g, b, z, dropout_p=0.1, seed=1, offset=2)
ops.layernorm_bwd(x, g, r, y, dg, dbe, accumulate_dx=True)
torch.cuda.synchronize()
