"""Fused tcgen05 causal attention (csrc/kernels/attention.cu) vs a float64 torch
reference of the unfused chain it replaces: S = Q K^T * scale, causal softmax,
global-head keyed Philox dropout, ctx = P_drop V,
and the autograd backward of that chain."""
import math

import pytest
import torch

pytestmark = pytest.mark.gpu

from paper_2305_16121_b200 import ops  # noqa: E402
from oracle.oracle import keep_mask, keep_scale  # noqa: E402


def rel(a, b):
    a, b = a.double(), b.double()
    return ((a - b).abs().max() / b.abs().max().clamp_min(1e-30)).item()


def reference(qkv, n, hl, dh, s, scale, p, seed, off, hg, hoff):
    x = qkv.double().view(n, s, 3, hl, dh)
    q, k, v = (x[:, :, t].permute(0, 2, 1, 3) for t in range(3))  # [n, hl, s, dh]
    S = (q @ k.transpose(-1, -2)) * scale
    i = torch.arange(s, device=qkv.device)
    causal = i[None, :] <= i[:, None]
    P = torch.softmax(S.masked_fill(~causal, float("-inf")), dim=-1)
    if p > 0:
        km = torch.tensor(keep_mask(seed, off, n * hg * s * s, p), device=qkv.device).view(n, hg, s, s)
        P = P * km[:, hoff:hoff + hl].double() * keep_scale(p)
    o = P @ v  # [n, hl, s, dh]
    return o.permute(0, 2, 1, 3).reshape(n * s, hl * dh)


CASES = [
    # n, hl, hg, hoff, dh, seq, p
    (2, 2, 4, 2, 128, 256, 0.1),
    (1, 3, 3, 0, 64, 384, 0.0),
    (2, 2, 2, 0, 128, 128, 0.0),
    (1, 2, 2, 0, 64, 256, 0.25),
    (1, 2, 2, 0, 128, 1024, 0.1),
    (1, 2, 2, 0, 128, 640, 0.1),   # odd tile count: the forward's last tile pair has no second tile
    (3, 1, 2, 1, 128, 128, 0.1),   # one tile per head
]


@pytest.mark.parametrize("n,hl,hg,hoff,dh,seq,p", CASES)
def test_fused_attention_fwd_bwd(cuda, n, hl, hg, hoff, dh, seq, p):
    torch.manual_seed(seq + dh + hl)
    hd = hl * dh
    scale = 1.0 / math.sqrt(dh)
    qkv = torch.randn(n * seq, 3 * hd, device=cuda).bfloat16()
    out = torch.empty(n * seq, hd, device=cuda, dtype=torch.bfloat16)
    lse = torch.empty(n * hl * seq, device=cuda, dtype=torch.float32)
    assert ops.attention_supported(torch.bfloat16, dh, seq)
    ops.attention_fwd(qkv, out, lse, n, hl, dh, seq, scale, p, 7, 13, hg, hoff)
    x = qkv.double().requires_grad_(True)
    ref = reference(x, n, hl, dh, seq, scale, p, 7, 13, hg, hoff)
    torch.cuda.synchronize()
    assert rel(out, ref) < 2e-2
    # lse = log2 sum_j exp2(scale*log2e*S_ij) over the causal row
    xq = qkv.double().view(n, seq, 3, hl, dh)
    S = (xq[:, :, 0].permute(0, 2, 1, 3) @ xq[:, :, 1].permute(0, 2, 3, 1)) * scale
    i = torch.arange(seq, device=cuda)
    S = S.masked_fill(~(i[None, :] <= i[:, None]), float("-inf"))
    ref_lse = torch.logsumexp(S, dim=-1).reshape(-1) / math.log(2.0)
    assert (lse.double() - ref_lse).abs().max().item() < 2e-3

    dout = torch.randn(n * seq, hd, device=cuda).bfloat16()
    ref.backward(dout.double())
    dqkv = torch.empty_like(qkv)
    ops.attention_bwd(qkv, out, lse, dout, dqkv, n, hl, dh, seq, scale, p, 7, 13, hg, hoff)
    torch.cuda.synchronize()
    g = x.grad.view(n * seq, 3, hd)
    got = dqkv.view(n * seq, 3, hd)
    for t, name in enumerate("QKV"):
        assert rel(got[:, t], g[:, t]) < 3e-2, name


def test_fused_attention_deterministic_and_rejects(cuda):
    n, hl, dh, seq = 2, 2, 128, 512
    torch.manual_seed(1)
    qkv = torch.randn(n * seq, 3 * hl * dh, device=cuda).bfloat16()
    out = torch.empty(n * seq, hl * dh, device=cuda, dtype=torch.bfloat16)
    lse = torch.empty(n * hl * seq, device=cuda)
    dout = torch.randn_like(out)
    res = []
    for _ in range(2):
        ops.attention_fwd(qkv, out, lse, n, hl, dh, seq, 0.125, 0.1, 3, 5)
        dqkv = torch.empty_like(qkv)
        ops.attention_bwd(qkv, out, lse, dout, dqkv, n, hl, dh, seq, 0.125, 0.1, 3, 5)
        res.append((out.clone(), lse.clone(), dqkv))
    torch.cuda.synchronize()
    assert all(torch.equal(a, b) for a, b in zip(res[0], res[1]))
    assert not ops.attention_supported(torch.bfloat16, 96, 512)
    assert not ops.attention_supported(torch.bfloat16, 128, 200)
    assert not ops.attention_supported(torch.float32, 128, 512)
    with pytest.raises(Exception):
        ops.attention_fwd(qkv, out, lse, n, hl, dh, 500, 0.125)


@pytest.mark.parametrize("dh,hl,hg,hoff,s", [(128, 2, 4, 2, 384), (64, 3, 3, 0, 256)])
def test_keep_bit_cache_modes_bit_identical(cuda, dh, hl, hg, hoff, s):
    """The keep-bit cache stores exactly the Philox decisions: forward with
    generate / generate+store / read, and backward with generate / read, give the
    same bits."""
    torch.manual_seed(5)
    n, p, seed, off = 2, 0.1, 11, 7
    hd = hl * dh
    qkv = torch.randn(n * s, 3 * hd, device=cuda).bfloat16()
    scale = 1 / math.sqrt(dh)
    bits = torch.zeros(ops.attention_mask_bytes(n, hl, s) // 4, dtype=torch.int32, device=cuda)
    outs, lses = [], []
    for mode in (0, 1, 2):
        out = torch.empty(n * s, hd, device=cuda, dtype=torch.bfloat16)
        lse = torch.empty(n * hl * s, device=cuda)
        ops.attention_fwd(qkv, out, lse, n, hl, dh, s, scale, p, seed, off, heads_total=hg, head_offset=hoff,
                          mask_bits=bits, mask_mode=mode)
        outs.append(out)
        lses.append(lse)
    torch.cuda.synchronize()
    assert torch.equal(outs[0], outs[1]) and torch.equal(outs[0], outs[2])
    assert torch.equal(lses[0], lses[2])
    assert bits.abs().sum().item() > 0
    # the separate mask pass writes exactly the bits the forward stored (mode 1)
    bits2 = torch.zeros_like(bits)
    ops.attention_masks(qkv, n, hl, dh, s, p, seed, off, bits2, heads_total=hg, head_offset=hoff)
    torch.cuda.synchronize()
    assert torch.equal(bits, bits2)
    dout = torch.randn(n * s, hd, device=cuda).bfloat16()
    grads = []
    for mode in (0, 2):
        dqkv = torch.empty_like(qkv)
        ops.attention_bwd(qkv, outs[0], lses[0], dout, dqkv, n, hl, dh, s, scale, p, seed, off, heads_total=hg,
                          head_offset=hoff, mask_bits=bits, mask_mode=mode)
        grads.append(dqkv)
    torch.cuda.synchronize()
    assert torch.equal(grads[0], grads[1])
