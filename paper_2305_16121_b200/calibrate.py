"""Calibration -> planner.

Measures, on this device, the per-block per-degree costs the reference's cost
model otherwise derives analytically (`build_cost_vectors`,
proj/src/costs.cpp:106-160) and emits them as measured-cost rows in the
schema `load_measured_costs` ingests (costs.cpp:174-211):

  d_fwd  per-sub-batch forward time of block b      = mean over sub-batches of F_b
  d_bwd  per-sub-batch backward time INCLUDING the  = mean of R_b + B_b
         recompute (costs.cpp:117,136 convention; sim.cpp:61-67 subtracts d_fwd)
  c_fwd, c_bwd  AllReduce of the half-batch boundary tensor at degree d; with
         one device these come from a bus-bandwidth model (alpha-beta, the
         reference's own comm_time) unless a measured table is supplied.
  m_saved  bytes of the stored post-AllReduce tensor per block (both halves)

Per-degree compute is measured by running ONE rank's shard of a d-way group on
this device with collectives disabled (`Context(tp=d, comm_disabled=True)`):
the kernels, shapes and memory traffic are exactly those of a real rank.
"""
from __future__ import annotations

import statistics

from . import tmpsim as t
from .runtime import Context, LayerStack, ModelConfig, plan_for


def measure_block_times(cfg: ModelConfig, degree: int, steps: int = 3, variant="Oases"):
    """{block: (d_fwd, d_bwd)} seconds per sub-batch for one rank at `degree`."""
    ctx = Context(tp=degree, comm_disabled=degree > 1)
    st = LayerStack(ctx, cfg)
    st.init_random(7)
    plan = plan_for(cfg, variant)
    st.bind(plan)
    st.step(trace=False)  # warm-up
    ops = list(plan.forward_ops) + list(plan.backward_ops)
    fwd = {b: [] for b in range(st.num_blocks)}
    bwd = {b: [] for b in range(st.num_blocks)}
    for _ in range(steps):
        res = st.step(trace=True)
        per = {}
        for op_id, _stream, s0, s1 in res.events:
            if op_id >= len(ops):
                continue
            op = ops[op_id]
            key = (op.block, op.sub_batch, op.pass_)
            per[key] = per.get(key, 0.0) + (s1 - s0)
        for (b, sb, ps), dur in per.items():
            if ps == t.Pass.Forward:
                fwd[b].append(dur)
        for b in range(st.num_blocks):
            for sb in (0, 1):
                rec = per.get((b, sb, t.Pass.Recompute), 0.0)
                bw = per.get((b, sb, t.Pass.Backward))
                if bw is not None:
                    bwd[b].append(rec + bw)
    st.close()
    ctx.close()
    return {b: (statistics.median(fwd[b]), statistics.median(bwd[b])) for b in fwd}


def calibrate(cfg: ModelConfig, degrees, *, steps: int = 3, profile: "t.HardwareProfile | None" = None,
              measured_allreduce=None):
    """Measured-cost rows for every block of `cfg` and every degree in `degrees`.

    measured_allreduce: optional {degree: seconds} per half-batch AllReduce
    (e.g. from an NCCL sweep on a multi-GPU box); otherwise the alpha-beta
    model of `profile` (default: tmpsim.b200_profile) is used.
    """
    profile = profile or t.b200_profile(max(degrees))
    spec = cfg.spec()
    half_bytes = cfg.batch / 2 * cfg.seq * cfg.hidden * cfg.bytes_per_element
    rows = []
    for d in degrees:
        times = measure_block_times(cfg, d, steps)
        if d == 1:
            c = 0.0
        elif measured_allreduce and d in measured_allreduce:
            c = measured_allreduce[d]
        else:
            c = t.comm_time(t.allreduce_volume(half_bytes, d), d, profile)
        for b, (df, db) in times.items():
            for field, v in (("d_fwd", df), ("d_bwd", db), ("c_fwd", c), ("c_bwd", c),
                             ("m_saved", 2 * half_bytes)):
                r = t.MeasuredRow()
                r.block_index, r.degree, r.field, r.seconds_or_bytes = b, d, field, float(v)
                rows.append(r)
    del spec
    return rows


def replicate_layers(rows, blocks_per_layer: int, layers: int):
    """Per-block rows measured on one layer, repeated over `layers` identical layers."""
    out = []
    for layer in range(layers):
        for r in rows:
            if r.block_index >= blocks_per_layer:
                continue
            n = t.MeasuredRow()
            n.block_index, n.degree, n.field, n.seconds_or_bytes = (layer * blocks_per_layer + r.block_index,
                                                                    r.degree, r.field, r.seconds_or_bytes)
            out.append(n)
    return out
