"""GEMM parity: tcgen05 bf16 kernel and f32 FFMA kernel vs an f64 torch reference.

Covers every operand major-ness combination the layer uses (forward TN,
dgrad with MN-major B, wgrad with MN-major A and B), the fused epilogues
(bias, bias+GeLU, dGeLU, f32 accumulate), M/N/K tails, and the batched causal
attention contractions (QK^T tile skip, P.V and dS.K K-limits, dS^T.Q K-start).
Tolerances: bf16 output 1e-2 relative to max|ref|; f32 output 1e-5 (bf16 in) /
1e-5 (f32 FFMA).
"""
import math

import pytest
import torch

pytestmark = pytest.mark.gpu

from paper_2305_16121_b200 import _capi as capi  # noqa: E402
from paper_2305_16121_b200 import ops  # noqa: E402


def relerr(x, ref, mask=None):
    x = x.double()
    ref = ref.double()
    if mask is not None:
        x = x[mask]
        ref = ref[mask]
    return ((x - ref).abs().max() / ref.abs().max().clamp_min(1e-30)).item()


def gelu64(x):
    return 0.5 * x * (1.0 + torch.erf(x / math.sqrt(2.0)))


def gelu_grad64(x):
    return 0.5 * (1.0 + torch.erf(x / math.sqrt(2.0))) + x * torch.exp(-0.5 * x * x) / math.sqrt(2 * math.pi)


@pytest.mark.parametrize("dt", ["bf16", "f32"])
@pytest.mark.parametrize("M,N,K", [(128, 128, 64), (256, 512, 1024), (200, 296, 136), (384, 256, 320),
                                   (1024, 1536, 512)])
@pytest.mark.parametrize("amn,bmn", [(0, 0), (0, 1), (1, 0), (1, 1)])
def test_gemm_majors(cuda, dt, M, N, K, amn, bmn):
    torch.manual_seed(M + N + K + 2 * amn + bmn)
    tdt = torch.bfloat16 if dt == "bf16" else torch.float32
    A = torch.randn(M, K, device=cuda).to(tdt)
    B = torch.randn(N, K, device=cuda).to(tdt)
    a_store = A.t().contiguous() if amn else A
    b_store = B.t().contiguous() if bmn else B
    C = torch.empty(M, N, device=cuda, dtype=torch.float32)
    ops.gemm(M, N, K, ops.operand(a_store, amn), ops.operand(b_store, bmn), C,
             dtype=capi.BF16 if dt == "bf16" else capi.F32)
    torch.cuda.synchronize()
    ref = A.double() @ B.double().t()
    assert relerr(C, ref) < 1e-5


@pytest.mark.parametrize("dt", ["bf16", "f32"])
def test_gemm_epilogues(cuda, dt):
    torch.manual_seed(7)
    tdt = torch.bfloat16 if dt == "bf16" else torch.float32
    kdt = capi.BF16 if dt == "bf16" else capi.F32
    M, N, K = 256, 384, 192
    A = torch.randn(M, K, device=cuda).to(tdt)
    B = (torch.randn(N, K, device=cuda) / math.sqrt(K)).to(tdt)
    bias = torch.randn(N, device=cuda).to(tdt)
    ref = A.double() @ B.double().t()
    tol = 1e-2 if dt == "bf16" else 1e-5
    # bias
    C = torch.empty(M, N, device=cuda, dtype=tdt)
    ops.gemm(M, N, K, ops.operand(A), ops.operand(B), C, epilogue=capi.EPI_BIAS, bias=bias, dtype=kdt)
    torch.cuda.synchronize()
    assert relerr(C, ref + bias.double()) < tol
    # bias + gelu (pre and act)
    pre = torch.empty_like(C)
    act = torch.empty_like(C)
    ops.gemm(M, N, K, ops.operand(A), ops.operand(B), pre, epilogue=capi.EPI_BIAS_GELU, bias=bias, c2=act, dtype=kdt)
    torch.cuda.synchronize()
    assert relerr(pre, ref + bias.double()) < tol
    assert relerr(act, gelu64(ref + bias.double())) < tol
    # dgelu with aux
    aux = torch.randn(M, N, device=cuda).to(tdt)
    C2 = torch.empty_like(C)
    ops.gemm(M, N, K, ops.operand(A), ops.operand(B), C2, epilogue=capi.EPI_DGELU, aux=aux, dtype=kdt)
    torch.cuda.synchronize()
    assert relerr(C2, ref * gelu_grad64(aux.double())) < tol
    # f32 accumulate + alpha
    Cf = torch.randn(M, N, device=cuda, dtype=torch.float32)
    C0 = Cf.clone()
    ops.gemm(M, N, K, ops.operand(A), ops.operand(B), Cf, accumulate=True, alpha=0.5, dtype=kdt)
    torch.cuda.synchronize()
    assert relerr(Cf, C0.double() + 0.5 * ref) < 1e-5


@pytest.mark.parametrize("dt", ["bf16", "f32"])
@pytest.mark.parametrize("bsz,H,s,d", [(2, 2, 256, 128), (1, 3, 384, 64)])
def test_gemm_attention_batched(cuda, dt, bsz, H, s, d):
    """Q.K^T (skip upper), P.V (k < m_end), dS^T.Q (k >= m_begin) over a fused QKV buffer."""
    torch.manual_seed(11)
    tdt = torch.bfloat16 if dt == "bf16" else torch.float32
    kdt = capi.BF16 if dt == "bf16" else capi.F32
    T = bsz * s
    qkv = torch.randn(T, 3 * H * d, device=cuda).to(tdt)
    q = qkv[:, : H * d].reshape(bsz, s, H, d).permute(0, 2, 1, 3).double()
    k = qkv[:, H * d: 2 * H * d].reshape(bsz, s, H, d).permute(0, 2, 1, 3).double()
    v = qkv[:, 2 * H * d:].reshape(bsz, s, H, d).permute(0, 2, 1, 3).double()
    Z = bsz * H
    # S = Q K^T  -> [Z*s, s]
    S = torch.zeros(Z * s, s, device=cuda, dtype=tdt)
    ops.gemm(s, s, d, ops.operand(qkv, False, (s, 0), (0, d)), ops.operand(qkv, False, (s, 0), (0, d), col_base=H * d),
             S, batch=Z, batch_inner=H, c_row_off=(H * s, s), causal=capi.CAUSAL_SKIP_UPPER, dtype=kdt)
    torch.cuda.synchronize()
    ref = (q @ k.transpose(-1, -2)).reshape(Z * s, s)
    tri = torch.tril(torch.ones(s, s, dtype=torch.bool, device=cuda)).repeat(Z, 1)
    tol = 1e-2 if dt == "bf16" else 1e-5
    assert relerr(S, ref, tri) < tol
    # causal P (zeros above the diagonal), ctx = P V
    P = (torch.rand(Z * s, s, device=cuda) * tri).to(tdt)
    ctx = torch.empty(T, H * d, device=cuda, dtype=tdt)
    ops.gemm(s, d, s, ops.operand(P, False, (H * s, s)),
             ops.operand(qkv, True, (s, 0), (0, d), col_base=2 * H * d), ctx,
             batch=Z, batch_inner=H, c_row_off=(s, 0), c_col_off=(0, d), causal=capi.CAUSAL_K_UPTO_M, dtype=kdt)
    torch.cuda.synchronize()
    ref_ctx = (P.double().reshape(bsz, H, s, s) @ v).permute(0, 2, 1, 3).reshape(T, H * d)
    assert relerr(ctx, ref_ctx) < tol
    # dK = dS^T Q with dS causal: A = dS MN-major, B = Q MN-major, k >= m_begin
    dK = torch.empty(T, H * d, device=cuda, dtype=tdt)
    ops.gemm(s, d, s, ops.operand(P, True, (H * s, s)), ops.operand(qkv, True, (s, 0), (0, d)), dK,
             batch=Z, batch_inner=H, c_row_off=(s, 0), c_col_off=(0, d), causal=capi.CAUSAL_K_FROM_M, dtype=kdt)
    torch.cuda.synchronize()
    ref_dk = (P.double().reshape(bsz, H, s, s).transpose(-1, -2) @ q).permute(0, 2, 1, 3).reshape(T, H * d)
    assert relerr(dK, ref_dk) < tol


def test_gemm_max_ctas(cuda):
    torch.manual_seed(3)
    M, N, K = 1024, 1024, 512
    A = torch.randn(M, K, device=cuda).bfloat16()
    B = torch.randn(N, K, device=cuda).bfloat16()
    C = torch.empty(M, N, device=cuda)
    ops.gemm(M, N, K, ops.operand(A), ops.operand(B), C, max_ctas=7)
    torch.cuda.synchronize()
    assert relerr(C, A.double() @ B.double().t()) < 1e-5


def test_gemm_rejects_misaligned(cuda):
    A = torch.randn(64, 60, device=cuda).bfloat16()
    C = torch.empty(64, 64, device=cuda)
    with pytest.raises(capi.OasesError) as e:
        ops.gemm(64, 64, 60, ops.operand(A[:, :60]), ops.operand(A), C)
    assert e.value.status == capi.ERR_CONFIG


@pytest.mark.parametrize("T,h,n", [(1024, 512, 768), (640, 384, 1024)])
def test_gemm_grouped_dgrad_wgrad_bitwise(cuda, T, h, n):
    """A backward dgrad (DGELU epilogue, MN-major B) and wgrad (f32 accumulate, MN-major A and B)
    in one grouped launch give exactly the bits of two separate launches."""
    torch.manual_seed(T + n)
    g = torch.randn(T, h, device=cuda).bfloat16()       # gradient [T, h]
    w = torch.randn(h, n, device=cuda).bfloat16() / 8   # W_row [out=h, in=n]
    act = torch.randn(T, n, device=cuda).bfloat16()     # forward activation
    pre = torch.randn(T, n, device=cuda).bfloat16()     # DGELU aux
    outs = []
    for grouped in (False, True):
        dcol = torch.empty(T, n, device=cuda, dtype=torch.bfloat16)
        dw = torch.full((h, n), 0.5, device=cuda)
        dd = ops.gemm_desc(T, n, h, ops.operand(g), ops.operand(w, True), dcol, epilogue=capi.EPI_DGELU, aux=pre)
        dwd = ops.gemm_desc(h, n, T, ops.operand(g, True), ops.operand(act, True), dw, accumulate=True)
        if grouped:
            ops.gemm_grouped([dwd, dd])
        else:
            ops.gemm_grouped([dwd])
            ops.gemm_grouped([dd])
        outs.append((dcol, dw))
    torch.cuda.synchronize()
    assert torch.equal(outs[0][0], outs[1][0]) and torch.equal(outs[0][1], outs[1][1])
    ref_d = (g.double() @ w.double()) * gelu_grad64(pre.double())
    ref_w = 0.5 + g.double().t() @ act.double()
    assert relerr(outs[1][0], ref_d) < 1e-2
    assert relerr(outs[1][1], ref_w) < 1e-5


@pytest.mark.parametrize("dt", ["bf16", "f32"])
def test_gemm_gelu_activation_only(cuda, dt):
    """EPI_BIAS_GELU with no C2 stores only gelu(acc + bias) into C (the forward FC1
    under recomputation, whose pre-activation is dead)."""
    torch.manual_seed(9)
    tdt = torch.bfloat16 if dt == "bf16" else torch.float32
    kdt = capi.BF16 if dt == "bf16" else capi.F32
    M, N, K = 384, 512, 256
    A = torch.randn(M, K, device=cuda).to(tdt)
    B = (torch.randn(N, K, device=cuda) / math.sqrt(K)).to(tdt)
    bias = torch.randn(N, device=cuda).to(tdt)
    pre, act = torch.empty(M, N, device=cuda, dtype=tdt), torch.empty(M, N, device=cuda, dtype=tdt)
    ops.gemm(M, N, K, ops.operand(A), ops.operand(B), pre, epilogue=capi.EPI_BIAS_GELU, bias=bias, c2=act, dtype=kdt)
    only = torch.empty(M, N, device=cuda, dtype=tdt)
    ops.gemm(M, N, K, ops.operand(A), ops.operand(B), only, epilogue=capi.EPI_BIAS_GELU, bias=bias, dtype=kdt)
    torch.cuda.synchronize()
    assert torch.equal(only, act)


@pytest.mark.parametrize("dt", ["bf16", "f32"])
def test_gemm_gelu_grad_and_mul_epilogues(cuda, dt):
    """BIAS_GELU_GRAD stores gelu'(v) and gelu(v); MUL multiplies by AUX: together
    they equal the DGELU epilogue on the pre-activation (the FFN backward)."""
    torch.manual_seed(10)
    tdt = torch.bfloat16 if dt == "bf16" else torch.float32
    kdt = capi.BF16 if dt == "bf16" else capi.F32
    M, N, K = 384, 512, 256
    A = torch.randn(M, K, device=cuda).to(tdt)
    B = (torch.randn(N, K, device=cuda) / math.sqrt(K)).to(tdt)
    bias = torch.randn(N, device=cuda).to(tdt)
    v = A.double() @ B.double().t() + bias.double()
    dgl, act = torch.empty(M, N, device=cuda, dtype=tdt), torch.empty(M, N, device=cuda, dtype=tdt)
    ops.gemm(M, N, K, ops.operand(A), ops.operand(B), dgl, epilogue=capi.EPI_BIAS_GELU_GRAD, bias=bias, c2=act,
             dtype=kdt)
    torch.cuda.synchronize()
    tol = 1e-2 if dt == "bf16" else 1e-5
    assert relerr(dgl, gelu_grad64(v)) < tol
    assert relerr(act, gelu64(v)) < tol
    G = torch.randn(M, K, device=cuda).to(tdt)
    W = (torch.randn(N, K, device=cuda) / math.sqrt(K)).to(tdt)
    out = torch.empty(M, N, device=cuda, dtype=tdt)
    ops.gemm(M, N, K, ops.operand(G), ops.operand(W), out, epilogue=capi.EPI_MUL, aux=dgl, dtype=kdt)
    torch.cuda.synchronize()
    assert relerr(out, (G.double() @ W.double().t()) * dgl.double()) < tol


@pytest.mark.parametrize("M,N,K", [(256, 256, 128), (1000, 384, 192), (4096, 8192, 2048), (96, 2080, 64)])
def test_gemm_mul_colsum_partials(cuda, M, N, K):
    """MUL epilogue with colsum partials: COLSUM[m / 32][n] = sum of the stored bf16 C over
    rows m..m+31 (CTA-pair and single-CTA kernels, ragged M), then oases_colsum_finalize
    gives the column-bias gradient -- equal to oases_colsum over C, the unfused pass."""
    torch.manual_seed(13)
    G = torch.randn(M, K, device=cuda).bfloat16()
    W = (torch.randn(N, K, device=cuda) / math.sqrt(K)).bfloat16()
    X = torch.rand(M, N, device=cuda).bfloat16()
    out = torch.empty(M, N, device=cuda, dtype=torch.bfloat16)
    chunks = (M + 31) // 32
    part = torch.full((chunks, N), float("nan"), device=cuda)
    ops.gemm(M, N, K, ops.operand(G), ops.operand(W), out, epilogue=capi.EPI_MUL, aux=X, colsum=part)
    ref = torch.empty(M, N, device=cuda, dtype=torch.bfloat16)
    ops.gemm(M, N, K, ops.operand(G), ops.operand(W), ref, epilogue=capi.EPI_MUL, aux=X)
    torch.cuda.synchronize()
    assert torch.equal(out, ref)  # the stored C does not change
    assert torch.isfinite(part).all()
    pad = torch.zeros(chunks * 32, N, device=cuda, dtype=torch.float64)
    pad[:M] = out.double()
    assert relerr(part, pad.view(chunks, 32, N).sum(1)) < 1e-6
    db = torch.full((N,), 2.0, device=cuda)
    ops.colsum_finalize(part, db, accumulate=True)
    db2 = torch.full((N,), 2.0, device=cuda)
    ops.colsum(out, db2, accumulate=True)
    torch.cuda.synchronize()
    assert relerr(db - 2.0, out.double().sum(0)) < 1e-5
    assert relerr(db, db2) < 1e-5
    # fixed reduction order: a second run gives the same bits
    part2 = torch.empty_like(part)
    ops.gemm(M, N, K, ops.operand(G), ops.operand(W), out, epilogue=capi.EPI_MUL, aux=X, colsum=part2)
    torch.cuda.synchronize()
    assert torch.equal(part, part2)


def test_gemm_colsum_rejected_outside_mul(cuda):
    A = torch.randn(128, 64, device=cuda).bfloat16()
    C = torch.empty(128, 128, device=cuda, dtype=torch.bfloat16)
    part = torch.empty(4, 128, device=cuda)
    with pytest.raises(Exception, match="COLSUM"):
        ops.gemm(128, 128, 64, ops.operand(A), ops.operand(A[:128]), C, colsum=part)
    with pytest.raises(Exception, match="COLSUM"):
        ops.gemm(128, 120, 64, ops.operand(A), ops.operand(A[:120]), C[:, :120], epilogue=capi.EPI_MUL, aux=C,
                 colsum=part)


@pytest.mark.parametrize("dh,hl,seq,n", [(128, 4, 256, 3), (64, 6, 128, 2), (128, 16, 1024, 4)])
def test_gemm_rowdot_epilogue(cuda, dh, hl, seq, n):
    """EPI_ROWDOT: C = A B^T stored as usual, and per (sample, head, row)
    D = sum over the head's columns of bf16(C) * AUX -- the attention backward's
    rowsum(dO o O) produced by the proj dgrad GEMM."""
    torch.manual_seed(12)
    M, N, K = n * seq, hl * dh, 512
    A = torch.randn(M, K, device=cuda).bfloat16()
    B = (torch.randn(N, K, device=cuda) / math.sqrt(K)).bfloat16()
    O = torch.randn(M, N, device=cuda).bfloat16()
    C = torch.empty(M, N, device=cuda, dtype=torch.bfloat16)
    D = torch.full((n * hl * seq,), float("nan"), device=cuda)
    ops.gemm(M, N, K, ops.operand(A), ops.operand(B), C, epilogue=capi.EPI_ROWDOT, aux=O, rowdot=D,
             rowdot_group=dh, rowdot_seq=seq, rowdot_heads=hl)
    torch.cuda.synchronize()
    ref_c = A.double() @ B.double().t()
    assert relerr(C, ref_c) < 1e-2
    ref_d = (C.double() * O.double()).view(n, seq, hl, dh).sum(-1).permute(0, 2, 1).reshape(-1)
    assert torch.isfinite(D).all()
    assert relerr(D, ref_d) < 1e-4
