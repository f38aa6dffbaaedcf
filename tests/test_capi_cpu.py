"""The C-ABI boundary without a GPU: liboases.so loads, exports every function
include/oases.h declares, the ctypes binding declares exactly those, the ctypes
struct mirrors have the C layout (checked against gcc on the header), and the
host-only entry points answer. No kernel is launched here (the GPU parity
tests in test_*_gpu.py call through the same entry points)."""
import ctypes as C
import os
import re
import subprocess

import pytest

from paper_2305_16121_b200 import _capi as capi

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "oases.h")

STRUCTS = {
    "oases_gemm_operand": capi.GemmOperand,
    "oases_gemm_desc": capi.GemmDesc,
    "oases_attn_desc": capi.AttnDesc,
    "oases_ctx_desc": capi.CtxDesc,
    "oases_model_desc": capi.ModelDesc,
    "oases_plan_op": capi.PlanOp,
    "oases_flat_plan": capi.FlatPlan,
    "oases_trace_event": capi.TraceEventC,
    "oases_kernel_stats": capi.KernelStats,
    "oases_step_result": capi.StepResult,
}
# ctypes names that differ from the C member (Python keywords)
RENAME = {("oases_plan_op", "pass_"): "pass"}


def header_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    src = re.sub(r"//[^\n]*", "", src)
    return set(re.findall(r"\b(oases_\w+)\s*\(", src))


def test_binding_declares_exactly_the_header():
    declared = header_functions()
    assert len(declared) > 40
    assert declared == set(capi.SYMBOLS)


def test_library_loads_and_exports_every_symbol():
    if not os.path.exists(capi.LIB_PATH):
        pytest.skip("liboases.so not built (run __graft_entry__.build())")
    assert capi.missing_symbols() == []
    out = subprocess.check_output(["nm", "-D", "--defined-only", capi.LIB_PATH], text=True)
    exported = {line.split()[-1] for line in out.splitlines() if line.strip()}
    assert header_functions() <= exported


def test_struct_layouts_match_the_c_header(tmp_path):
    """sizeof / offsetof of every C-ABI struct, from gcc on include/oases.h, equal the ctypes mirrors."""
    lines = ["#include <stdio.h>", "#include <stddef.h>", '#include "oases.h"', "int main(void) {"]
    for cname, py in STRUCTS.items():
        lines.append(f'  printf("{cname} sizeof %zu\\n", sizeof({cname}));')
        for fname, _ in py._fields_:
            cf = RENAME.get((cname, fname), fname)
            lines.append(f'  printf("{cname} {fname} %zu\\n", offsetof({cname}, {cf}));')
    lines += ["  return 0;", "}"]
    src = tmp_path / "layout.c"
    src.write_text("\n".join(lines) + "\n")
    exe = tmp_path / "layout"
    subprocess.check_call(["gcc", "-std=c11", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)])
    got = {}
    for line in subprocess.check_output([str(exe)], text=True).splitlines():
        cname, what, v = line.split()
        got[(cname, what)] = int(v)
    for cname, py in STRUCTS.items():
        assert got[(cname, "sizeof")] == C.sizeof(py), cname
        for fname, _ in py._fields_:
            assert got[(cname, fname)] == getattr(py, fname).offset, (cname, fname)


def test_host_only_entry_points():
    if not os.path.exists(capi.LIB_PATH):
        pytest.skip("liboases.so not built")
    L = capi.lib()
    assert L.oases_version()
    assert L.oases_colsum_workspace(8192, 2048) > 0
    assert L.oases_attention_mask_bytes(None) == 0
    # null descriptors are configuration errors, reported before any device work
    assert L.oases_gemm(None, None) == capi.ERR_CONFIG
    assert b"null descriptor" in L.oases_last_error()
    assert L.oases_colsum_finalize(None, 0, 0, None, 0, None) == capi.ERR_CONFIG


CPP_CONSUMER = r"""
#include <cstdio>
#include "oases/tmpsim.hpp"
#include "oases/runtime.hpp"
using namespace tmpsim;
int main() {
  ModelSpec spec;
  spec.hidden_size = 4096; spec.num_layers = 3; spec.seq_len = 2048;
  spec.attention_heads = 32; spec.global_batch = 8; spec.bytes_per_element = 2;
  spec.recompute_enabled = true;
  const ModelGraph g = build_block_graph(build_operator_sequence(spec), spec);
  const CostVectors costs = build_cost_vectors(g, spec, b200_profile(8));
  const Strategy s{std::vector<int>(g.block_count(), 8)};
  for (ScheduleVariant v : {ScheduleVariant::Oases, ScheduleVariant::CrossPass}) {
    const SchedulePlan plan = make_schedule(g, v);
    const SimResult r = simulate(plan, costs, s);
    std::printf("%zu %d %.17g %.17g %.17g\n", validate_plan(plan).size(), comm_op_count(plan), r.makespan,
                r.comm_exposed, r.peak_memory);
  }
  try {
    make_schedule(g, static_cast<ScheduleVariant>(99));
  } catch (const ConfigError&) {
    std::printf("ConfigError\n");
  }
  return 0;
}
"""


def test_cpp_consumer_links_the_tmpsim_api(tmp_path):
    """A C++ caller of the reference's tmpsim API (its headers swapped for include/oases/*.hpp,
    INTEGRATION.md) compiles, links liboases.so and gets the same plans and simulations as the
    Python binding -- host-only, no device needed."""
    if not os.path.exists(capi.LIB_PATH):
        pytest.skip("liboases.so not built")
    import paper_2305_16121_b200.tmpsim as t

    src = tmp_path / "consumer.cpp"
    src.write_text(CPP_CONSUMER)
    exe = tmp_path / "consumer"
    libdir = os.path.dirname(capi.LIB_PATH)
    subprocess.check_call(["g++", "-std=c++17", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe),
                           "-L", libdir, "-loases", f"-Wl,-rpath,{libdir}"])
    out = subprocess.check_output([str(exe)], text=True).split("\n")
    assert out[2] == "ConfigError"
    spec = t.ModelSpec()
    spec.hidden_size, spec.num_layers, spec.seq_len = 4096, 3, 2048
    spec.attention_heads, spec.global_batch, spec.bytes_per_element = 32, 8, 2
    spec.recompute_enabled = True
    g = t.build_block_graph(t.build_operator_sequence(spec), spec)
    costs = t.build_cost_vectors(g, spec, t.b200_profile(8))
    s = t.Strategy([8] * g.block_count())
    for line, v in zip(out[:2], (t.ScheduleVariant.Oases, t.ScheduleVariant.CrossPass)):
        plan = t.make_schedule(g, v)
        r = t.simulate(plan, costs, s)
        nviol, ncomm, mk, ce, pm = line.split()
        assert int(nviol) == 0 and int(ncomm) == t.comm_op_count(plan)
        assert float(mk) == r.makespan and float(ce) == r.comm_exposed and float(pm) == r.peak_memory
