"""Independent float64 torch-autograd statement of the TMP layer stack.

Used to validate the fp64 oracle's extra ops (LN, causal attention, biases,
bias-dropout-residual, dropout), which the reference leaves parity-unpinned.
Reads parameters from an oracle.Oracle so both see identical inputs.
"""
import math

import numpy as np
import torch

from oracle.oracle import B_COL, B_ROW, LN_BETA, LN_GAMMA, W_COL, W_ROW, keep_mask, keep_scale


def run_torch_ref(orc):
    cfg = orc.cfg
    T, h, s = cfg.tokens, cfg.hidden, cfg.seq
    half = cfg.batch // 2 if cfg.batch % 2 == 0 else cfg.batch
    params = {}
    for b in range(orc.num_blocks):
        for r in range(cfg.tp):
            for p in (LN_GAMMA, LN_BETA, W_COL, B_COL, W_ROW, B_ROW):
                params[(r, b, p)] = torch.tensor(np.array(orc.param(r, b, p)), dtype=torch.float64, requires_grad=True)
    x0 = torch.tensor(np.array(orc.input), dtype=torch.float64, requires_grad=True)

    def hidden_mask(b):
        if cfg.hidden_dropout <= 0:
            return None
        m = np.zeros((T, h), dtype=np.float64)
        rows_per_sb = half * s
        for sb in range((T + rows_per_sb - 1) // rows_per_sb):
            k = keep_mask(cfg.seed, (b * 2 + sb) * 4 + 0, rows_per_sb * h, cfg.hidden_dropout)
            m[sb * rows_per_sb:(sb + 1) * rows_per_sb] = k.reshape(rows_per_sb, h)
        return torch.tensor(m * keep_scale(cfg.hidden_dropout))

    def attn_mask(b, r):
        Ht = cfg.heads // cfg.tp
        H = cfg.heads
        m = np.zeros((cfg.batch, Ht, s, s))
        for n in range(cfg.batch):
            sb, nl = n // half, n % half
            k = keep_mask(cfg.seed, (b * 2 + sb) * 4 + 1, half * H * s * s, cfg.attention_dropout)
            k = k.reshape(half, H, s, s)
            m[n] = k[nl, r * Ht:(r + 1) * Ht]
        return torch.tensor(m * keep_scale(cfg.attention_dropout))

    x = x0
    for b in range(orc.num_blocks):
        att = orc.is_attention(b)
        ar = torch.zeros(T, h, dtype=torch.float64)
        for r in range(cfg.tp):
            P = lambda p: params[(r, b, p)]  # noqa: E731
            if cfg.use_layernorm:
                mu = x.mean(dim=1, keepdim=True)
                var = ((x - mu) ** 2).mean(dim=1, keepdim=True)
                ln = (x - mu) / torch.sqrt(var + cfg.ln_eps) * P(LN_GAMMA) + P(LN_BETA)
            else:
                ln = x
            col = ln @ P(W_COL)
            if cfg.use_bias:
                col = col + P(B_COL)
            if att:
                Ht = cfg.heads // cfg.tp
                d = h // cfg.heads
                q, k, v = col[:, :Ht * d], col[:, Ht * d:2 * Ht * d], col[:, 2 * Ht * d:]
                shp = lambda z: z.reshape(cfg.batch, s, Ht, d).permute(0, 2, 1, 3)  # noqa: E731
                sc = shp(q) @ shp(k).transpose(-1, -2) / math.sqrt(d)
                causal = torch.tril(torch.ones(s, s, dtype=torch.bool))
                sc = sc.masked_fill(~causal, float("-inf"))
                pr = torch.softmax(sc, dim=-1)
                if cfg.attention_dropout > 0:
                    pr = pr * attn_mask(b, r)
                act = (pr @ shp(v)).permute(0, 2, 1, 3).reshape(T, Ht * d)
            else:
                act = 0.5 * col * (1.0 + torch.erf(col / math.sqrt(2.0)))
            ar = ar + act @ P(W_ROW)
        v = ar
        if cfg.use_bias:
            v = v + params[(0, b, B_ROW)]
        m = hidden_mask(b)
        if m is not None:
            v = v * m
        x = x + v if cfg.use_residual else v
    g = 0.5 * x * (1.0 + torch.erf(x / math.sqrt(2.0)))
    loss = 0.5 * (g * g).sum()
    loss.backward()
    grads = {}
    for (r, b, p), t in params.items():
        # replicated params: the oracle reports the full gradient on every worker
        grads[(r, b, p)] = t.grad.clone() if t.grad is not None else torch.zeros_like(t)
    for (r, b, p) in list(grads):
        if p in (LN_GAMMA, LN_BETA, B_ROW):
            grads[(r, b, p)] = sum(params[(rr, b, p)].grad if params[(rr, b, p)].grad is not None
                                   else torch.zeros_like(params[(rr, b, p)]) for rr in range(cfg.tp))
    return loss.item(), x.detach(), x0.grad, grads
