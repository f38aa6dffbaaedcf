"""Digest of one C2-shaped training step (2 layers, dropout 0.1, Oases plan): the loss,
dX and every parameter gradient, hashed. Run once per build (OASES_LIB=...) on one box;
equal digests = bit-identical results.

    python tools/bitcheck.py [layers]
"""
import hashlib
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2305_16121_b200.runtime import Context, LayerStack, ModelConfig, plan_for  # noqa: E402

layers = int(sys.argv[1]) if len(sys.argv) > 1 else 2
mc = ModelConfig(hidden=2048, heads=16, seq=1024, batch=8, layers=layers, dtype="bf16", hidden_dropout=0.1,
                 attention_dropout=0.1)
ctx = Context(tp=1, device=0)
st = LayerStack(ctx, mc)
st.init_random(1234)
st.bind(plan_for(mc, "Oases"))
res = st.step(trace=False)
h = hashlib.sha256()
h.update(np.float64(res.loss).tobytes())
h.update(np.ascontiguousarray(st.input_grad()).tobytes())
for b in range(mc.num_blocks):
    for p in range(6):  # LN_GAMMA, LN_BETA, W_COL, B_COL, W_ROW, B_ROW
        if st.param_numel(b, p):
            h.update(np.ascontiguousarray(st.grad(0, b, p)).tobytes())
print(f"loss {res.loss!r} digest {h.hexdigest()}")
st.close()
ctx.close()
