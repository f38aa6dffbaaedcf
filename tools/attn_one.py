"""Run the fused attention forward + backward at C2 shape (for ncu captures / timing).

Env: N (samples, 4), HL (local heads, 16), DH (128), SEQ (1024), P (0.1), ITERS (3).
"""
import ctypes as C
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2305_16121_b200 import ops  # noqa: E402

n, hl, dh, s = (int(os.environ.get(k, v)) for k, v in (("N", 4), ("HL", 16), ("DH", 128), ("SEQ", 1024)))
p = float(os.environ.get("P", 0.1))
hd = hl * dh
qkv = torch.randn(n * s, 3 * hd, device="cuda").bfloat16()
out = torch.empty(n * s, hd, device="cuda", dtype=torch.bfloat16)
lse = torch.empty(n * hl * s, device="cuda")
dout = torch.randn_like(out)
dqkv = torch.empty_like(qkv)
ds = torch.empty(n * hl * s, s, device="cuda", dtype=torch.bfloat16)
scale = 1 / math.sqrt(dh)
iters = int(os.environ.get("ITERS", "3"))
# MODE 0: Philox inside the kernels; 2: keep bits from the separate mask pass (the stack's path)
mode = int(os.environ.get("MODE", "0"))
mbits = None
if mode == 2 and p > 0:
    d = ops._attn_desc(qkv, n, hl, dh, s, 1.0, p, 1, 2, 0, 0)
    from paper_2305_16121_b200 import _capi as capi
    mbits = torch.zeros(capi.lib().oases_attention_mask_bytes(C.byref(d)) // 4, dtype=torch.int32, device="cuda")
    for _ in range(2):
        ops.attention_masks(qkv, n, hl, dh, s, p, 1, 2, mbits)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        ops.attention_masks(qkv, n, hl, dh, s, p, 1, 2, mbits)
    e1.record()
    torch.cuda.synchronize()
    print(f"mask pass {e0.elapsed_time(e1) / 10 * 1e3:8.1f} us")
ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
rep = int(os.environ.get("REP", "10"))  # back-to-back launches per timing (amortises host overhead)
for it in range(iters):
    torch.cuda.synchronize()
    ev[0].record()
    for _ in range(rep):
        ops.attention_fwd(qkv, out, lse, n, hl, dh, s, scale, p, 1, 2, mask_bits=mbits, mask_mode=mode if mbits is not None else 0)
    ev[1].record()
    for _ in range(rep):
        ops.attention_bwd(qkv, out, lse, dout, dqkv, n, hl, dh, s, scale, p, 1, 2, ds=ds, mask_bits=mbits,
                          mask_mode=mode if mbits is not None else 0)
    ev[2].record()
    torch.cuda.synchronize()
    fl = 4 * n * hl * s * s * dh / 2  # causal: QK^T + PV
    f_ms, b_ms = ev[0].elapsed_time(ev[1]) / rep, ev[1].elapsed_time(ev[2]) / rep
    print(f"fwd {f_ms*1e3:8.1f} us ({fl/f_ms/1e9:6.1f} TF/s)  bwd {b_ms*1e3:8.1f} us ({2.5*fl/b_ms/1e9:6.1f} TF/s)")
