"""Per-CTA start/end/SM of one attn_dkdv_kernel launch (trace build: OASES_LIB=liboases_trace.so,
compiled with -DOASES_EXP_TRACE): CTA duration vs its query-tile count, SM busy fraction, idle gaps.

Env as tools/attn_one.py (N, HL, DH, SEQ, P); cached keep bits (the stack's path)."""
import ctypes as C
import math
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2305_16121_b200 import _capi as capi, ops  # noqa: E402

n, hl, dh, s = (int(os.environ.get(k, v)) for k, v in (("N", 4), ("HL", 16), ("DH", 128), ("SEQ", 1024)))
p = float(os.environ.get("P", 0.1))
hd = hl * dh
qkv = torch.randn(n * s, 3 * hd, device="cuda").bfloat16()
out = torch.empty(n * s, hd, device="cuda", dtype=torch.bfloat16)
lse = torch.empty(n * hl * s, device="cuda")
dout = torch.randn_like(out)
dqkv = torch.empty_like(qkv)
ds = torch.empty(n * hl * s, s, device="cuda", dtype=torch.bfloat16)
sc = 1 / math.sqrt(dh)
d = ops._attn_desc(qkv, n, hl, dh, s, 1.0, p, 1, 2, 0, 0)
mbits = torch.zeros(capi.lib().oases_attention_mask_bytes(C.byref(d)) // 4, dtype=torch.int32, device="cuda")
ops.attention_masks(qkv, n, hl, dh, s, p, 1, 2, mbits)
kw = dict(mask_bits=mbits, mask_mode=2)
ops.attention_fwd(qkv, out, lse, n, hl, dh, s, sc, p, 1, 2, **kw)
for _ in range(3):
    ops.attention_bwd(qkv, out, lse, dout, dqkv, n, hl, dh, s, sc, p, 1, 2, ds=ds, **kw)
torch.cuda.synchronize()
buf = (C.c_ulonglong * (3 * 1024))()
capi.lib().oases_attn_cta_dump(buf)
Z, nq = n * hl, s // 128
ncta = min(Z * nq, 1024, torch.cuda.get_device_properties(0).multi_processor_count) if os.environ.get('PERSISTENT') else min(Z * nq, 1024)
t0 = [buf[i] for i in range(ncta)]
t1 = [buf[1024 + i] for i in range(ncta)]
sm = [buf[2048 + i] for i in range(ncta)]
base = min(t0)
end = max(t1)
span = end - base
print(f"CTAs {ncta}, kernel span (first start -> last end) {span / 1e3:.1f} us, SMs used {len(set(sm))}")
if ncta < Z * nq:  # persistent build: CTAs walk several items; only the SM-level figures apply
    print(f"  persistent grid ({ncta} CTAs for {Z * nq} items): CTA span mean "
          f"{statistics.mean((t1[b] - t0[b]) / 1e3 for b in range(ncta)):.1f} us, "
          f"max {max((t1[b] - t0[b]) / 1e3 for b in range(ncta)):.1f} us; "
          f"finish spread {(max(t1) - min(t1)) / 1e3:.1f} us")
    sys.exit(0)
per_tiles = {}
for b in range(ncta):
    kt = b // Z
    per_tiles.setdefault(nq - kt, []).append((t1[b] - t0[b]) / 1e3)
for ni in sorted(per_tiles):
    v = per_tiles[ni]
    print(f"  {ni} query tiles: {len(v):3d} CTAs, duration mean {statistics.mean(v):6.2f} us  (per tile {statistics.mean(v) / ni:5.2f})")
# fit duration = a + b * tiles
xs = [nq - b // Z for b in range(ncta)]
ys = [(t1[b] - t0[b]) / 1e3 for b in range(ncta)]
mx, my = statistics.mean(xs), statistics.mean(ys)
bb = sum((x - mx) * (y - my) for x, y in zip(xs, ys)) / sum((x - mx) ** 2 for x in xs)
print(f"  fit: duration = {my - bb * mx:.2f} us + {bb:.2f} us x tiles")
busy = {}
for b in range(ncta):
    busy.setdefault(sm[b], []).append((t0[b], t1[b]))
fr, gaps = [], []
for k, iv in busy.items():
    iv.sort()
    fr.append(sum(e - a for a, e in iv) / span)
    gaps += [(iv[i + 1][0] - iv[i][1]) / 1e3 for i in range(len(iv) - 1)]
    last = max(e for _, e in iv)
print(f"  SM busy fraction (CTA resident): mean {statistics.mean(fr):.3f} min {min(fr):.3f}")
print(f"  gap between consecutive CTAs on an SM: mean {statistics.mean(gaps):.2f} us, max {max(gaps):.2f} us")
ends = sorted((max(e for _, e in iv) - base) / 1e3 for iv in busy.values())
print(f"  SM finish times: first {ends[0]:.1f} us, median {ends[len(ends) // 2]:.1f}, last {ends[-1]:.1f}")
