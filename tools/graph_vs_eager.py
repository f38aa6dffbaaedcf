"""C2 device step time: eager issue (untraced / traced) vs CUDA-graph replay."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2305_16121_b200.runtime import Context, LayerStack, ModelConfig, plan_for  # noqa: E402

layers = int(os.environ.get("LAYERS", "24"))
n = int(os.environ.get("STEPS", "8"))
mc = ModelConfig(hidden=2048, heads=16, seq=1024, batch=8, layers=layers, dtype="bf16", hidden_dropout=0.1,
                 attention_dropout=0.1)
st = LayerStack(Context(tp=1), mc)
st.init_random(1)
st.bind(plan_for(mc, os.environ.get("VARIANT", "Oases")))


def run(label, trace):
    for _ in range(3):
        st.step(trace=trace)
    t = [st.step(trace=trace).makespan * 1e3 for _ in range(n)]
    print(f"{label:14s} median {statistics.median(t):8.3f} ms  min {min(t):8.3f}  max {max(t):8.3f}", flush=True)


run("eager", False)
run("eager+trace", True)
st.capture_graph()
run("graph", False)
run("eager+trace", True)
run("graph", False)
