"""Repeat the attention forward (cached keep bits) and check every launch is
bit-identical; write a digest of the output so runs under different env
settings (OASES_ATTN_PV_WAIT, OASES_ATTN_FWD2) can be compared.

Env: N, HL, SEQ (C2 sub-batch by default), REPS (100), OUT (digest file).
"""
import ctypes as C
import hashlib
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2305_16121_b200 import _capi as capi  # noqa: E402
from paper_2305_16121_b200 import ops  # noqa: E402

n, hl, s, reps = (int(os.environ.get(k, v)) for k, v in (("N", 4), ("HL", 16), ("SEQ", 1024), ("REPS", 100)))
dh, p = 128, 0.1
g = torch.Generator(device="cuda").manual_seed(5)
qkv = (torch.randn(n * s, 3 * hl * dh, device="cuda", generator=g) * 2).bfloat16()
out = torch.empty(n * s, hl * dh, device="cuda", dtype=torch.bfloat16)
lse = torch.empty(n * hl * s, device="cuda")
d = ops._attn_desc(qkv, n, hl, dh, s, 1.0, p, 1, 2, 0, 0)
mbits = torch.zeros(capi.lib().oases_attention_mask_bytes(C.byref(d)) // 4, dtype=torch.int32, device="cuda")
ops.attention_masks(qkv, n, hl, dh, s, p, 1, 2, mbits)
ops.attention_fwd(qkv, out, lse, n, hl, dh, s, 1 / math.sqrt(dh), p, 1, 2, mask_bits=mbits, mask_mode=2)
ref, ref_lse = out.clone(), lse.clone()
bad = 0
for _ in range(reps):
    ops.attention_fwd(qkv, out, lse, n, hl, dh, s, 1 / math.sqrt(dh), p, 1, 2, mask_bits=mbits, mask_mode=2)
    bad += int(not (torch.equal(out, ref) and torch.equal(lse, ref_lse)))
torch.cuda.synchronize()
h = hashlib.sha256(ref.view(torch.int16).cpu().numpy().tobytes() + ref_lse.cpu().numpy().tobytes()).hexdigest()
print(f"reps {reps} mismatching {bad} digest {h[:16]}")
if os.environ.get("OUT"):
    open(os.environ["OUT"], "w").write(h)
sys.exit(1 if bad else 0)
