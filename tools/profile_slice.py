"""One eager step of a TMP rank slice (few layers) for ncu launch lists."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2305_16121_b200.runtime import Context, LayerStack, ModelConfig, plan_for  # noqa: E402

cfg = dict(bench.CONFIGS[os.environ.get("CONFIG", "c3")])
cfg["layers"] = int(os.environ.get("LAYERS", "1"))
mc = ModelConfig(dtype="bf16", hidden_dropout=0.1, attention_dropout=0.1, **cfg)
st = LayerStack(Context(tp=int(os.environ.get("TP", "8")), comm_disabled=True), mc)
st.init_random(1)
st.bind(plan_for(mc, "Oases"))
for _ in range(int(os.environ.get("STEPS", "2"))):
    r = st.step(trace=True)
print("makespan_ms", r.makespan * 1e3)
