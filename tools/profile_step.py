"""One eager C2-shaped step (few layers) for ncu launch lists / captures."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2305_16121_b200.runtime import Context, LayerStack, ModelConfig, plan_for  # noqa: E402

layers = int(os.environ.get("LAYERS", "2"))
steps = int(os.environ.get("STEPS", "2"))
mc = ModelConfig(hidden=2048, heads=16, seq=1024, batch=8, layers=layers, dtype="bf16", hidden_dropout=0.1,
                 attention_dropout=0.1)
st = LayerStack(Context(tp=1), mc)
st.init_random(1)
st.bind(plan_for(mc, os.environ.get("VARIANT", "Oases")))
for _ in range(steps):
    r = st.step(trace=True)
print("makespan_ms", r.makespan * 1e3)
