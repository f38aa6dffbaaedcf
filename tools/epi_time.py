"""Warm timing of the C2 FFN backward GEMMs whose epilogues read global memory:
FC2 dgrad with the gelu' product (EPI_MUL, + column-sum partials off) and with
dGeLU, the attention-projection dgrad shape with no epilogue for comparison,
and the grouped dgrad + wgrad (CUDA graph of back-to-back launches).

    [OASES_LIB=...] python tools/epi_time.py   -> one JSON line
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2305_16121_b200 import _capi as capi, ops  # noqa: E402

Ts, h, f = 4096, 2048, 8192
bf = torch.bfloat16
gar = torch.randn(Ts, h, device="cuda").to(bf)
act = torch.randn(Ts, f, device="cuda").to(bf)
w = torch.randn(h, f, device="cuda").to(bf)
dW = torch.zeros(h, f, device="cuda")
aux = [torch.randn(Ts, f, device="cuda").to(bf) for _ in range(2)]
out = [torch.empty(Ts, f, device="cuda", dtype=bf) for _ in range(2)]


def desc(i, epi):
    kw = {} if epi is None else {"epilogue": epi, "aux": aux[i]}
    return ops.gemm_desc(Ts, f, h, ops.operand(gar), ops.operand(w, True), out[i], **kw)


def timeit(fn, rep=20):
    fn(0); fn(1)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for i in range(rep):
            fn(i & 1)
    g.replay()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    s.record(); g.replay(); e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / rep * 1e3


fl = 2 * Ts * f * h
res = {}
for name, epi in (("plain", None), ("mul", capi.EPI_MUL), ("dgelu", capi.EPI_DGELU)):
    us = timeit(lambda i, epi=epi: ops.gemm_grouped([desc(i, epi)]))
    res[name] = {"us": round(us, 2), "tflops": round(fl / us / 1e6, 1)}
dw = ops.gemm_desc(h, f, Ts, ops.operand(gar, True), ops.operand(act, True), dW)
us = timeit(lambda i: ops.gemm_grouped([dw, desc(i, capi.EPI_MUL)]))
res["grouped_wgrad_mul"] = {"us": round(us, 2), "tflops": round(2 * fl / us / 1e6, 1)}
print(json.dumps({"lib": os.environ.get("OASES_LIB", "in-tree"), **res}))
