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

from . import tmpsim as t
from .runtime import ModelConfig, graph_for


def _exec_options(cfg: ModelConfig, steps: int = 1):
    o = t.ExecOptions()
    o.spec = cfg.spec()
    o.ffn_hidden, o.attention, o.layernorm, o.bias, o.residual = (cfg.ffn, cfg.attention, cfg.layernorm, cfg.bias,
                                                                   cfg.residual)
    o.hidden_dropout, o.attention_dropout, o.seed = cfg.hidden_dropout, cfg.attention_dropout, cfg.seed
    o.steps = steps
    return o


def calibrate(cfg: ModelConfig, degrees, *, steps: int = 3, profile: "t.HardwareProfile | None" = None,
              measured_allreduce=None, device: int = 0):
    """Measured-cost rows for every block of `cfg` and every degree in `degrees`
    (the C++ tmpsim::calibrate of include/oases/runtime.hpp).

    measured_allreduce: optional {degree: seconds} per half-batch AllReduce (e.g.
    tools/nccl_sweep.py on a multi-GPU node); otherwise c_fwd / c_bwd are the
    alpha-beta comm_time of `profile` (default: tmpsim.b200_profile).
    """
    o = t.ContextOptions()
    o.device = device
    ctx = t.Context(o)
    rows = list(t.calibrate(graph_for(cfg), cfg.spec(), ctx, list(degrees), _exec_options(cfg), steps))
    half_bytes = cfg.batch / 2 * cfg.seq * cfg.hidden * cfg.bytes_per_element
    for r in rows:
        if r.field in ("c_fwd", "c_bwd") and r.degree > 1:
            if measured_allreduce and r.degree in measured_allreduce:
                r.seconds_or_bytes = float(measured_allreduce[r.degree])
            elif profile is not None:
                r.seconds_or_bytes = t.comm_time(t.allreduce_volume(half_bytes, r.degree), r.degree, profile)
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
