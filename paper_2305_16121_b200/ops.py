"""Thin torch-tensor front end over the kernel entry points of include/oases.h.

torch is used only for device memory and the current stream (plumbing); every
call lands in liboases.so. Used by the kernel-level parity tests.
"""
from __future__ import annotations

import ctypes as C

import torch

from . import _capi as capi
from ._capi import check

_DT = {torch.float32: capi.F32, torch.bfloat16: capi.BF16}


def _dtype(t: torch.Tensor) -> int:
    try:
        return _DT[t.dtype]
    except KeyError as e:
        raise TypeError(f"unsupported dtype {t.dtype}") from e


def _ptr(t):
    return None if t is None else C.c_void_p(t.data_ptr())


def _stream(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


def operand(t: torch.Tensor, mn_major: bool = False, row_off=(0, 0), col_off=(0, 0), col_base: int = 0):
    """GEMM operand over a 2-D row-major storage tensor (optionally starting at column col_base)."""
    assert t.dim() == 2 and t.stride(1) == 1
    o = capi.GemmOperand()
    o.ptr = t.data_ptr() + col_base * t.element_size()
    o.rows = t.shape[0]
    o.cols = t.shape[1] - col_base
    o.ld = t.stride(0)
    o.mn_major = int(mn_major)
    o.row_off[0], o.row_off[1] = row_off
    o.col_off[0], o.col_off[1] = col_off
    return o


def gemm_desc(M, N, K, a, b, c: torch.Tensor, *, batch=1, batch_inner=1, c_row_off=(0, 0), c_col_off=(0, 0),
              c_col_base=0, epilogue=capi.EPI_NONE, causal=capi.CAUSAL_NONE, alpha=1.0, accumulate=False,
              bias=None, aux=None, c2=None, max_ctas=0, dtype=capi.BF16, rowdot=None, rowdot_group=0,
              rowdot_seq=0, rowdot_heads=0, colsum=None):
    d = capi.GemmDesc()
    d.dtype = dtype
    d.c_dtype = _dtype(c)
    d.M, d.N, d.K = M, N, K
    d.batch, d.batch_inner = batch, batch_inner
    d.a, d.b = a, b
    esz = c.element_size()
    d.c = c.data_ptr() + c_col_base * esz
    d.ldc = c.stride(0)
    d.c_row_off[0], d.c_row_off[1] = c_row_off
    d.c_col_off[0], d.c_col_off[1] = c_col_off
    d.epilogue = epilogue
    d.causal = causal
    d.alpha = alpha
    d.accumulate = int(accumulate)
    d.bias = None if bias is None else bias.data_ptr()
    d.aux = None if aux is None else aux.data_ptr() + c_col_base * esz
    d.c2 = None if c2 is None else c2.data_ptr() + c_col_base * esz
    d.max_ctas = max_ctas
    d.rowdot = None if rowdot is None else rowdot.data_ptr()
    d.rowdot_group, d.rowdot_seq, d.rowdot_heads = rowdot_group, rowdot_seq, rowdot_heads
    d.colsum = None if colsum is None else colsum.data_ptr()
    return d


def gemm(M, N, K, a, b, c: torch.Tensor, *, stream=None, **kw):
    """dtype: operand dtype (capi.BF16 -> tcgen05 kernel, capi.F32 -> FFMA kernel)."""
    d = gemm_desc(M, N, K, a, b, c, **kw)
    check(capi.lib().oases_gemm(C.byref(d), _stream(stream)))


def gemm_grouped(descs, stream=None):
    """Independent bf16 problems (descriptors from gemm_desc) in one launch where possible."""
    arr = (capi.GemmDesc * len(descs))(*descs)
    check(capi.lib().oases_gemm_grouped(arr, len(descs), _stream(stream)))


def layernorm_fwd(x, gamma, beta, y, eps=1e-5, stream=None):
    rows, cols = x.shape
    check(capi.lib().oases_layernorm_fwd(_dtype(x), _ptr(x), _ptr(gamma), _ptr(beta), _ptr(y), rows, cols, eps,
                                         _stream(stream)))


def layernorm_bwd(x, gamma, dy, dx, dgamma, dbeta, accumulate_dx=False, acc_params=False, eps=1e-5, stream=None):
    rows, cols = x.shape
    ws = torch.empty(capi.lib().oases_layernorm_bwd_workspace(rows, cols) // 4 + 64, dtype=torch.float32,
                     device=x.device)
    check(capi.lib().oases_layernorm_bwd(_dtype(x), _ptr(x), _ptr(gamma), _ptr(dy), _ptr(dx), int(accumulate_dx),
                                         _ptr(dgamma), _ptr(dbeta), int(acc_params), _ptr(ws), rows, cols, eps,
                                         _stream(stream)))


def attention_supported(dtype: torch.dtype, head_dim: int, seq: int) -> bool:
    return bool(capi.lib().oases_attention_supported(_dtype(torch.empty(0, dtype=dtype)), head_dim, seq))


def _attn_desc(qkv, samples, heads, head_dim, seq, scale, dropout_p, seed, offset, heads_total, head_offset):
    d = capi.AttnDesc()
    d.dtype = _dtype(qkv)
    d.samples, d.heads_local, d.head_dim, d.seq = samples, heads, head_dim, seq
    d.heads_total = heads_total or heads
    d.head_offset = head_offset
    d.qkv, d.ld_qkv = _ptr(qkv), qkv.stride(0)
    d.scale, d.dropout_p, d.seed, d.offset = scale, dropout_p, seed, offset
    return d


def attention_mask_bytes(samples, heads, seq):
    """Bytes of the attention-dropout keep-bit cache (mask_bits) for this shape."""
    d = capi.AttnDesc()
    d.samples, d.heads_local, d.seq = samples, heads, seq
    return capi.lib().oases_attention_mask_bytes(C.byref(d))


def attention_fwd(qkv, out, lse, samples, heads, head_dim, seq, scale, dropout_p=0.0, seed=0, offset=0,
                  heads_total=0, head_offset=0, stream=None, mask_bits=None, mask_mode=0):
    """Fused causal attention: qkv [samples*seq, >=3*heads*head_dim] (Q|K|V blocks) -> out (ctx), lse (f32).
    mask_bits/mask_mode: keep-bit cache (0 generate, 1 generate + store, 2 read)."""
    d = _attn_desc(qkv, samples, heads, head_dim, seq, scale, dropout_p, seed, offset, heads_total, head_offset)
    d.out, d.ld_out, d.lse = _ptr(out), out.stride(0), _ptr(lse)
    d.mask_bits, d.mask_mode = _ptr(mask_bits), mask_mode
    check(capi.lib().oases_attention_fwd(C.byref(d), _stream(stream)))


def attention_masks(qkv, samples, heads, head_dim, seq, dropout_p, seed, offset, mask_bits, heads_total=0,
                    head_offset=0, stream=None):
    """Keep bits of every causal-band element into mask_bits (what mask_mode 1 stores)."""
    d = _attn_desc(qkv, samples, heads, head_dim, seq, 1.0, dropout_p, seed, offset, heads_total, head_offset)
    d.ld_out = heads * head_dim  # (no ctx written; the shared descriptor checks want a valid stride)
    d.mask_bits = _ptr(mask_bits)
    check(capi.lib().oases_attention_masks(C.byref(d), _stream(stream)))


def attention_bwd(qkv, out, lse, dout, dqkv, samples, heads, head_dim, seq, scale, dropout_p=0.0, seed=0, offset=0,
                  heads_total=0, head_offset=0, ds=None, stream=None, mask_bits=None, mask_mode=0):
    """Backward of attention_fwd: writes dQ | dK | dV into dqkv (dS scratch allocated when not given)."""
    d = _attn_desc(qkv, samples, heads, head_dim, seq, scale, dropout_p, seed, offset, heads_total, head_offset)
    d.mask_bits, d.mask_mode = _ptr(mask_bits), mask_mode
    d.out, d.ld_out, d.lse = _ptr(out), out.stride(0), _ptr(lse)
    d.dout, d.ld_dout = _ptr(dout), dout.stride(0)
    d.dqkv, d.ld_dqkv = _ptr(dqkv), dqkv.stride(0)
    if ds is None:
        ds = torch.empty(samples * heads * seq, seq, dtype=qkv.dtype, device=qkv.device)
    d.ds = _ptr(ds)
    ws = torch.empty(capi.lib().oases_attention_bwd_workspace(C.byref(d)) // 4 + 4, dtype=torch.float32,
                     device=qkv.device)
    d.workspace = _ptr(ws)
    check(capi.lib().oases_attention_bwd(C.byref(d), _stream(stream)))
    return ds


def softmax_fwd(s, p, p_drop, batch, seq, scale, dropout_p=0.0, seed=0, offset=0, heads_local=1, heads_total=1,
                head_offset=0, stream=None):
    check(capi.lib().oases_softmax_fwd(_dtype(s), _ptr(s), _ptr(p), _ptr(p_drop), batch, seq, scale, dropout_p, seed,
                                       offset, heads_local, heads_total, head_offset, _stream(stream)))


def softmax_bwd(p, dp_drop, ds, batch, seq, scale, dropout_p=0.0, seed=0, offset=0, heads_local=1, heads_total=1,
                head_offset=0, stream=None):
    check(capi.lib().oases_softmax_bwd(_dtype(p), _ptr(p), _ptr(dp_drop), _ptr(ds), batch, seq, scale, dropout_p,
                                       seed, offset, heads_local, heads_total, head_offset, _stream(stream)))


def bias_dropout_residual_fwd(x, bias, residual, out, dropout_p=0.0, seed=0, offset=0, stream=None):
    rows, cols = x.shape
    check(capi.lib().oases_bias_dropout_residual_fwd(_dtype(x), _ptr(x), _ptr(bias), _ptr(residual), _ptr(out), rows,
                                                     cols, dropout_p, seed, offset, _stream(stream)))


def bias_dropout_residual_layernorm_fwd(x, bias, residual, x_out, gamma, beta, y, dropout_p=0.0, seed=0, offset=0,
                                        eps=1e-5, stream=None):
    rows, cols = x.shape
    check(capi.lib().oases_bias_dropout_residual_layernorm_fwd(
        _dtype(x), _ptr(x), _ptr(bias), _ptr(residual), _ptr(x_out), _ptr(gamma), _ptr(beta), _ptr(y), rows, cols,
        eps, dropout_p, seed, offset, _stream(stream)))


def bias_dropout_residual_bwd(dout, dx, dbias, acc_bias=False, dropout_p=0.0, seed=0, offset=0, stream=None):
    rows, cols = dout.shape
    ws = torch.empty(capi.lib().oases_colsum_workspace(rows, cols) // 4 + 64, dtype=torch.float32,
                     device=dout.device)
    check(capi.lib().oases_bias_dropout_residual_bwd(_dtype(dout), _ptr(dout), _ptr(dx), _ptr(dbias), int(acc_bias),
                                                     _ptr(ws), rows, cols, dropout_p, seed, offset, _stream(stream)))


def colsum(x, out, accumulate=False, stream=None):
    rows, cols = x.shape
    ws = torch.empty(capi.lib().oases_colsum_workspace(rows, cols) // 4 + 64, dtype=torch.float32, device=x.device)
    check(capi.lib().oases_colsum(_dtype(x), _ptr(x), _ptr(out), int(accumulate), _ptr(ws), rows, cols,
                                  _stream(stream)))


def colsum_finalize(partials, out, accumulate=False, stream=None):
    """out (+)= partials.sum(0) in a fixed order (partials: [chunks, cols] f32, e.g. from gemm(colsum=))."""
    chunks, cols = partials.shape
    check(capi.lib().oases_colsum_finalize(_ptr(partials), chunks, cols, _ptr(out), int(accumulate),
                                           _stream(stream)))


def gelu_fwd(x, y, stream=None):
    check(capi.lib().oases_gelu_fwd(_dtype(x), _ptr(x), _ptr(y), x.numel(), _stream(stream)))


def gelu_bwd(x, dy, dx, stream=None):
    check(capi.lib().oases_gelu_bwd(_dtype(x), _ptr(x), _ptr(dy), _ptr(dx), x.numel(), _stream(stream)))


def gelu_sq_loss(z, dz, loss_out, accumulate=False, stream=None):
    ws = torch.empty(1024, dtype=torch.float64, device=z.device)
    check(capi.lib().oases_gelu_sq_loss(_dtype(z), _ptr(z), _ptr(dz), _ptr(loss_out), int(accumulate), _ptr(ws),
                                        z.numel(), _stream(stream)))


def local_allreduce(bufs, stream=None):
    arr = (C.c_void_p * len(bufs))(*[b.data_ptr() for b in bufs])
    check(capi.lib().oases_local_allreduce(_dtype(bufs[0]), arr, len(bufs), bufs[0].numel(), _stream(stream)))
