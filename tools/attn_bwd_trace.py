"""Per-iteration event timeline of CTA 0 (key tile 0) of the attention dK/dV kernel (trace build)."""
import ctypes as C
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2305_16121_b200 import _capi as capi, ops  # noqa: E402

n, hl, dh, s = 4, 16, 128, 1024
p = float(os.environ.get("P", 0.1))
hd = hl * dh
qkv = torch.randn(n * s, 3 * hd, device="cuda").bfloat16()
out = torch.empty(n * s, hd, device="cuda", dtype=torch.bfloat16)
lse = torch.empty(n * hl * s, device="cuda")
dout = torch.randn_like(out)
dqkv = torch.empty_like(qkv)
ds = torch.empty(n * hl * s, s, device="cuda", dtype=torch.bfloat16)
sc = 1 / math.sqrt(dh)
# MODE 0: Philox inside the kernels; 2: cached keep bits (the stack's path)
mode = int(os.environ.get("MODE", "2"))
mbits = None
if mode == 2 and p > 0:
    d = ops._attn_desc(qkv, n, hl, dh, s, 1.0, p, 1, 2, 0, 0)
    mbits = torch.zeros(capi.lib().oases_attention_mask_bytes(C.byref(d)) // 4, dtype=torch.int32, device="cuda")
    ops.attention_masks(qkv, n, hl, dh, s, p, 1, 2, mbits)
kw = dict(mask_bits=mbits, mask_mode=2) if mbits is not None else {}
ops.attention_fwd(qkv, out, lse, n, hl, dh, s, sc, p, 1, 2, **kw)
for _ in range(3):
    ops.attention_bwd(qkv, out, lse, dout, dqkv, n, hl, dh, s, sc, p, 1, 2, ds=ds, **kw)
torch.cuda.synchronize()
buf = (C.c_ulonglong * (8 * 64))()
capi.lib().oases_attn_trace_dump(buf)
t = [[buf[e * 64 + g] for g in range(64)] for e in range(8)]
t0 = min(v for row in t for v in row if v)
names = ["ld_issue", "dV_go", "dK_go", "s_seen", "pd_arrive", "dp_seen", "buf1_ok", "ds_arrive"]
print("it  " + " ".join(f"{x:>10s}" for x in names))
for g in range(9):
    print(f"{g:3d} " + " ".join(f"{(t[e][g] - t0) if t[e][g] else -1:10d}" for e in range(8)))
