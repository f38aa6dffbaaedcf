"""HBM-bound kernels vs float64 torch references, at C2-like row widths and at
toy widths (vector and scalar paths), including the workspace sizing of the
deterministic column reductions."""
import math

import pytest
import torch

pytestmark = pytest.mark.gpu

from paper_2305_16121_b200 import ops  # noqa: E402
from oracle.oracle import keep_mask, keep_scale  # noqa: E402


def rel(a, b):
    a, b = a.double(), b.double()
    return ((a - b).abs().max() / b.abs().max().clamp_min(1e-30)).item()


@pytest.mark.parametrize("dt,tol", [(torch.float32, 1e-5), (torch.bfloat16, 2e-2)])
@pytest.mark.parametrize("rows,cols", [(4096, 2048), (512, 8192), (64, 24), (3, 6)])
def test_bias_dropout_residual_and_colsum(cuda, dt, tol, rows, cols):
    torch.manual_seed(rows + cols)
    x = torch.randn(rows, cols, device=cuda).to(dt)
    b = torch.randn(cols, device=cuda).to(dt)
    r = torch.randn(rows, cols, device=cuda).to(dt)
    out = torch.empty_like(x)
    p = 0.1 if rows * cols % 4 == 0 else 0.0
    ops.bias_dropout_residual_fwd(x, b, r, out, dropout_p=p, seed=5, offset=9)
    keep = torch.tensor(keep_mask(5, 9, rows * cols, p), device=cuda).view(rows, cols).double()
    ref = r.double() + (x.double() + b.double()) * keep * keep_scale(p)
    torch.cuda.synchronize()
    assert rel(out, ref) < tol
    dx = torch.empty_like(x)
    db = torch.zeros(cols, device=cuda)
    ops.bias_dropout_residual_bwd(x, dx, db, dropout_p=p, seed=5, offset=9)
    ref_dx = x.double() * keep * keep_scale(p)
    torch.cuda.synchronize()
    assert rel(dx, ref_dx) < tol
    assert rel(db, ref_dx.sum(0)) < (1e-4 if dt == torch.float32 else 2e-2)
    s = torch.zeros(cols, device=cuda)
    ops.colsum(x, s)
    torch.cuda.synchronize()
    assert rel(s, x.double().sum(0)) < 1e-4


@pytest.mark.parametrize("dt,tol", [(torch.float32, 1e-5), (torch.bfloat16, 2e-2)])
@pytest.mark.parametrize("rows,cols", [(4096, 2048), (256, 4096), (128, 8192), (16, 64)])
def test_layernorm_fwd_bwd(cuda, dt, tol, rows, cols):
    torch.manual_seed(cols)
    x = (torch.randn(rows, cols, device=cuda) * 2 + 0.5).to(dt)
    g = (1 + 0.1 * torch.randn(cols, device=cuda)).to(dt)
    b = (0.1 * torch.randn(cols, device=cuda)).to(dt)
    y = torch.empty_like(x)
    ops.layernorm_fwd(x, g, b, y)
    xd = x.double().requires_grad_(True)
    gd, bd = g.double().requires_grad_(True), b.double().requires_grad_(True)
    ref = torch.nn.functional.layer_norm(xd, (cols,), gd, bd, eps=1e-5)
    torch.cuda.synchronize()
    assert rel(y, ref) < tol
    dy = torch.randn(rows, cols, device=cuda).to(dt)
    ref.backward(dy.double())
    dx = torch.empty_like(x)
    dg = torch.zeros(cols, device=cuda)
    dbeta = torch.zeros(cols, device=cuda)
    ops.layernorm_bwd(x, g, dy, dx, dg, dbeta)
    torch.cuda.synchronize()
    assert rel(dx, xd.grad) < tol * 2
    assert rel(dg, gd.grad) < (1e-4 if dt == torch.float32 else 3e-2)
    assert rel(dbeta, bd.grad) < (1e-4 if dt == torch.float32 else 3e-2)


@pytest.mark.parametrize("dt,tol", [(torch.float32, 1e-5), (torch.bfloat16, 2e-2)])
@pytest.mark.parametrize("seq,p", [(1024, 0.0), (256, 0.1), (2048, 0.1)])
def test_causal_softmax_fwd_bwd(cuda, dt, tol, seq, p):
    torch.manual_seed(seq)
    n, hl, hg, hoff = 2, 2, 4, 2
    rows = n * hl * seq
    s = torch.randn(rows, seq, device=cuda).to(dt)
    P = torch.empty_like(s)
    Pd = torch.empty_like(s) if p > 0 else None
    scale = 1 / math.sqrt(64)
    ops.softmax_fwd(s, P, Pd, n * hl, seq, scale, p, 3, 11, hl, hg, hoff)
    i = torch.arange(seq, device=cuda)
    causal = (i[None, :] <= i[:, None]).repeat(n * hl, 1)
    band = (i[None, :] < ((i[:, None] + 128) // 128 * 128)).repeat(n * hl, 1)
    ref = torch.softmax((s.double() * scale).masked_fill(~causal, float("-inf")), dim=-1)
    torch.cuda.synchronize()
    assert rel(P[band], ref[band]) < tol
    assert P.double()[band & ~causal].abs().max().item() == 0.0
    if p > 0:
        # global-head keyed mask: local head jl of sample k is global head hoff + jl
        keep = torch.zeros(rows, seq, dtype=torch.float64, device=cuda)
        km = torch.tensor(keep_mask(3, 11, n * hg * seq * seq, p), device=cuda).view(n, hg, seq, seq)
        keep = km[:, hoff:hoff + hl].reshape(rows, seq).double()
        assert rel(Pd[band], (ref * keep * keep_scale(p))[band]) < tol
    dpd = torch.randn(rows, seq, device=cuda).to(dt)
    ds = torch.empty_like(s)
    ops.softmax_bwd(P, dpd, ds, n * hl, seq, scale, p, 3, 11, hl, hg, hoff)
    dp = dpd.double() * (keep * keep_scale(p) if p > 0 else 1.0)
    dp = dp.masked_fill(~causal, 0.0)
    ref_ds = scale * ref * (dp - (ref * dp).sum(-1, keepdim=True))
    torch.cuda.synchronize()
    assert rel(ds[band], ref_ds[band]) < tol * 2


def test_loss_head_and_local_allreduce(cuda):
    torch.manual_seed(0)
    z = torch.randn(4096, 2048, device=cuda)
    dz = torch.empty_like(z)
    loss = torch.zeros(1, dtype=torch.float64, device=cuda)
    ops.gelu_sq_loss(z, dz, loss)
    g = 0.5 * z.double() * (1 + torch.erf(z.double() / math.sqrt(2)))
    torch.cuda.synchronize()
    assert abs(loss.item() - 0.5 * (g * g).sum().item()) < 1e-5 * loss.item()
    bufs = [torch.randn(1000, device=cuda) for _ in range(3)]
    ref = bufs[0].double() + bufs[1].double() + bufs[2].double()
    ops.local_allreduce(bufs)
    torch.cuda.synchronize()
    for b in bufs:
        assert rel(b, ref) < 1e-6


@pytest.mark.parametrize("dt", [torch.float32, torch.bfloat16])
@pytest.mark.parametrize("rows,cols", [(4096, 2048), (1000, 1024), (257, 4096), (64, 8192), (33, 512)])
@pytest.mark.parametrize("p,use_bias,use_res", [(0.1, True, True), (0.0, False, True), (0.1, True, False)])
def test_fused_bdr_layernorm_bit_identical(cuda, dt, rows, cols, p, use_bias, use_res):
    """The fused block-boundary kernel equals bias_dropout_residual_fwd followed by
    layernorm_fwd BIT FOR BIT (x and LN(x)); LN checked against float64 too."""
    torch.manual_seed(rows * 7 + cols)
    x = torch.randn(rows, cols, device=cuda).to(dt)
    b = torch.randn(cols, device=cuda).to(dt) if use_bias else None
    r = torch.randn(rows, cols, device=cuda).to(dt) if use_res else None
    g = (1 + 0.1 * torch.randn(cols, device=cuda)).to(dt)
    be = (0.1 * torch.randn(cols, device=cuda)).to(dt)
    x1, y1 = torch.empty_like(x), torch.empty_like(x)
    ops.bias_dropout_residual_fwd(x, b, r, x1, dropout_p=p, seed=3, offset=17)
    ops.layernorm_fwd(x1, g, be, y1)
    x2, y2 = torch.empty_like(x), torch.empty_like(x)
    ops.bias_dropout_residual_layernorm_fwd(x, b, r, x2, g, be, y2, dropout_p=p, seed=3, offset=17)
    torch.cuda.synchronize()
    assert torch.equal(x1, x2)
    assert torch.equal(y1, y2)
    xd = x2.double()
    ref = (xd - xd.mean(1, keepdim=True)) / torch.sqrt(xd.var(1, unbiased=False, keepdim=True) + 1e-5)
    ref = ref * g.double() + be.double()
    assert rel(y2, ref) < (1e-5 if dt == torch.float32 else 2e-2)


def test_fused_bdr_layernorm_rejects_uncovered_shape(cuda):
    from paper_2305_16121_b200 import _capi as capi

    x = torch.randn(8, 40, device=cuda)
    g, be = torch.ones(40, device=cuda), torch.zeros(40, device=cuda)
    with pytest.raises(capi.OasesError) as e:
        ops.bias_dropout_residual_layernorm_fwd(x, None, x, torch.empty_like(x), g, be, torch.empty_like(x))
    assert e.value.status == capi.ERR_CONFIG


@pytest.mark.parametrize("dt", [torch.float32, torch.bfloat16])
@pytest.mark.parametrize("rows,cols", [(1000, 1024), (257, 4096), (33, 512), (4096, 2048)])
def test_layernorm_bwd_accumulate_and_deterministic(cuda, dt, rows, cols):
    """The persistent LayerNorm backward (rowpipe.cu): dx accumulated onto an existing
    residual gradient, dgamma/dbeta from the folded column partials (per-CTA registers,
    2-CTA cluster reduction, fixed-order finalize) against float64 torch, with a ragged
    last row group, and bit-identical across repeated launches."""
    torch.manual_seed(rows + cols)
    x = (torch.randn(rows, cols, device=cuda) * 1.5 + 0.3).to(dt)
    g = (1 + 0.1 * torch.randn(cols, device=cuda)).to(dt)
    dy = torch.randn(rows, cols, device=cuda).to(dt)
    res = torch.randn(rows, cols, device=cuda).to(dt)
    xd = x.double().requires_grad_(True)
    gd = g.double().requires_grad_(True)
    bd = torch.zeros(cols, device=cuda, dtype=torch.float64, requires_grad=True)
    ref = torch.nn.functional.layer_norm(xd, (cols,), gd, bd, eps=1e-5)
    ref.backward(dy.double())
    outs = []
    for _ in range(2):
        dx = res.clone()
        dg = torch.zeros(cols, device=cuda)
        dbeta = torch.zeros(cols, device=cuda)
        ops.layernorm_bwd(x, g, dy, dx, dg, dbeta, accumulate_dx=True)
        outs.append((dx, dg, dbeta))
    torch.cuda.synchronize()
    tol = 1e-5 if dt == torch.float32 else 2e-2
    assert rel(outs[0][0], res.double() + xd.grad) < 2 * tol
    assert rel(outs[0][1], gd.grad) < (1e-4 if dt == torch.float32 else 3e-2)
    assert rel(outs[0][2], bd.grad) < (1e-4 if dt == torch.float32 else 3e-2)
    for a, b in zip(outs[0], outs[1]):
        assert torch.equal(a, b)
