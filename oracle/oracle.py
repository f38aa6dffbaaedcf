"""TEST INFRASTRUCTURE ONLY: ctypes front end of the fp64 oracle (gpt_oracle.cpp).

Importable only by tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline leg, as the checker. The product package never imports it.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "build", "liboracle.so")

LN_GAMMA, LN_BETA, W_COL, B_COL, W_ROW, B_ROW = range(6)
PARAMS = (LN_GAMMA, LN_BETA, W_COL, B_COL, W_ROW, B_ROW)


class _Cfg(C.Structure):
    _fields_ = [
        ("hidden", C.c_int), ("ffn", C.c_int), ("heads", C.c_int), ("seq", C.c_int), ("batch", C.c_int),
        ("layers", C.c_int), ("tp", C.c_int), ("use_attention", C.c_int), ("use_layernorm", C.c_int),
        ("use_bias", C.c_int), ("use_residual", C.c_int), ("hidden_dropout", C.c_float),
        ("attention_dropout", C.c_float), ("ln_eps", C.c_double), ("seed", C.c_uint64),
    ]


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            subprocess.check_call(["make", "-C", HERE, "build/liboracle.so"])
        L = C.CDLL(LIB)
        vp = C.c_void_p
        L.oracle_create.restype = vp
        L.oracle_create.argtypes = [C.POINTER(_Cfg)]
        L.oracle_destroy.argtypes = [vp]
        L.oracle_num_blocks.argtypes = [vp]
        L.oracle_block_is_attention.argtypes = [vp, C.c_int]
        L.oracle_param_numel.restype = C.c_longlong
        L.oracle_param_numel.argtypes = [vp, C.c_int, C.c_int]
        L.oracle_param_rows.argtypes = [vp, C.c_int, C.c_int]
        for name in ("oracle_param", "oracle_grad"):
            getattr(L, name).restype = C.POINTER(C.c_double)
            getattr(L, name).argtypes = [vp, C.c_int, C.c_int, C.c_int]
        for name in ("oracle_input", "oracle_input_grad"):
            getattr(L, name).restype = C.POINTER(C.c_double)
            getattr(L, name).argtypes = [vp]
        L.oracle_activation.restype = C.POINTER(C.c_double)
        L.oracle_activation.argtypes = [vp, C.c_int]
        L.oracle_loss.restype = C.c_double
        L.oracle_loss.argtypes = [vp]
        L.oracle_init_params.argtypes = [vp, C.c_uint, C.c_int]
        L.oracle_run.argtypes = [vp]
        _lib = L
    return _lib


@dataclass
class LayerCfg:
    hidden: int
    ffn: int = 0
    heads: int = 1
    seq: int = 1
    batch: int = 2
    layers: int = 1
    tp: int = 1
    use_attention: bool = True
    use_layernorm: bool = True
    use_bias: bool = True
    use_residual: bool = True
    hidden_dropout: float = 0.0
    attention_dropout: float = 0.0
    ln_eps: float = 1e-5
    seed: int = 1234

    def __post_init__(self):
        if not self.ffn:
            self.ffn = 4 * self.hidden

    @property
    def tokens(self):
        return self.batch * self.seq


class Oracle:
    """fp64 TMP layer stack with `tp` in-process workers (literal-sum AllReduce)."""

    def __init__(self, cfg: LayerCfg):
        self.cfg = cfg
        c = _Cfg(cfg.hidden, cfg.ffn, cfg.heads, cfg.seq, cfg.batch, cfg.layers, cfg.tp, int(cfg.use_attention),
                 int(cfg.use_layernorm), int(cfg.use_bias), int(cfg.use_residual), cfg.hidden_dropout,
                 cfg.attention_dropout, cfg.ln_eps, cfg.seed)
        self._h = lib().oracle_create(C.byref(c))
        if not self._h:
            raise ValueError(f"invalid oracle config {cfg}")
        self.num_blocks = lib().oracle_num_blocks(self._h)

    def __del__(self):
        if getattr(self, "_h", None):
            lib().oracle_destroy(self._h)
            self._h = None

    def is_attention(self, b):
        return bool(lib().oracle_block_is_attention(self._h, b))

    def _view(self, ptr, n, shape=None):
        a = np.ctypeslib.as_array(ptr, shape=(n,))
        return a.reshape(shape) if shape else a

    def param_shape(self, block, p):
        n = lib().oracle_param_numel(self._h, block, p)
        rows = lib().oracle_param_rows(self._h, block, p)
        return (rows, n // rows) if rows > 1 else (n,)

    def param(self, worker, block, p):
        shape = self.param_shape(block, p)
        return self._view(lib().oracle_param(self._h, worker, block, p), int(np.prod(shape)), shape)

    def grad(self, worker, block, p):
        shape = self.param_shape(block, p)
        return self._view(lib().oracle_grad(self._h, worker, block, p), int(np.prod(shape)), shape)

    @property
    def input(self):
        return self._view(lib().oracle_input(self._h), self.cfg.tokens * self.cfg.hidden,
                          (self.cfg.tokens, self.cfg.hidden))

    @property
    def input_grad(self):
        return self._view(lib().oracle_input_grad(self._h), self.cfg.tokens * self.cfg.hidden,
                          (self.cfg.tokens, self.cfg.hidden))

    def activation(self, block):
        return self._view(lib().oracle_activation(self._h, block), self.cfg.tokens * self.cfg.hidden,
                          (self.cfg.tokens, self.cfg.hidden))

    @property
    def loss(self):
        return lib().oracle_loss(self._h)

    def init_params(self, seed, extras=True):
        lib().oracle_init_params(self._h, seed, int(extras))

    def run(self):
        lib().oracle_run(self._h)
        return self.loss


# --------------------------------------------------------------------------- Philox (numpy)
M0, M1 = np.uint64(0xD2511F53), np.uint64(0xCD9E8D57)
W0, W1 = np.uint32(0x9E3779B9), np.uint32(0xBB67AE85)


def philox4x32_10(seed: int, offset: int, ctr: np.ndarray) -> np.ndarray:
    """Vectorised Philox4x32-10 (same spec as oracle/philox.h); returns [n, 4] uint32."""
    ctr = ctr.astype(np.uint64)
    c0 = (ctr & np.uint64(0xFFFFFFFF)).astype(np.uint64)
    c1 = (ctr >> np.uint64(32)).astype(np.uint64)
    c2 = np.full_like(c0, offset & 0xFFFFFFFF)
    c3 = np.full_like(c0, (offset >> 32) & 0xFFFFFFFF)
    k0 = np.uint64(seed & 0xFFFFFFFF)
    k1 = np.uint64((seed >> 32) & 0xFFFFFFFF)
    mask = np.uint64(0xFFFFFFFF)
    for r in range(10):
        p0 = M0 * c0
        p1 = M1 * c2
        n0 = (p1 >> np.uint64(32)) ^ c1 ^ k0
        n1 = p1 & mask
        n2 = (p0 >> np.uint64(32)) ^ c3 ^ k1
        n3 = p0 & mask
        c0, c1, c2, c3 = n0 & mask, n1, n2 & mask, n3
        if r < 9:
            k0 = (k0 + np.uint64(W0)) & mask
            k1 = (k1 + np.uint64(W1)) & mask
    return np.stack([c0, c1, c2, c3], axis=-1).astype(np.uint32)


def keep_threshold(p: float) -> int:
    """thr8 = round(p * 256) in float32 arithmetic, clamped to [1, 255] (0 when p <= 0)."""
    if not p > 0:
        return 0
    t = int(np.float32(p) * np.float32(256.0) + np.float32(0.5))
    return min(255, max(1, t))


def keep_scale(p: float) -> float:
    t = keep_threshold(p)
    return 256.0 / (256.0 - t) if t else 1.0


def keep_mask(seed: int, offset: int, n: int, p: float) -> np.ndarray:
    """Keep-mask of elements 0..n-1 under (seed, offset): byte (e & 15) of Philox(e >> 4) >= thr8."""
    thr = keep_threshold(p)
    ctrs = (n + 15) // 16
    words = philox4x32_10(seed, offset, np.arange(ctrs, dtype=np.uint64))  # [ctrs, 4]
    byts = words.astype("<u4").view(np.uint8).reshape(ctrs * 16)  # byte b of word w at 4w + b (little endian)
    return byts[:n] >= np.uint8(thr)
