"""Python host side of the measured TMP step (mirror of the reference's
operator API for this path, over the C-ABI of include/oases.h).

    ctx   = Context(tp=1)                       # streams, NCCL comm (tp > 1)
    stack = LayerStack(ctx, ModelConfig(...))   # weights, saved tensors, workspaces
    stack.bind(plan)                            # a tmpsim.SchedulePlan (e.g. schedule_oases)
    res   = stack.step(trace=True)              # measured SimResult + loss

`plan_for(cfg, variant)` builds the plan with the tmpsim-compatible API
(build_operator_sequence -> build_block_graph -> make_schedule).
"""
from __future__ import annotations

import atexit
import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _capi as capi
from . import tmpsim as t
from ._capi import check

LN_GAMMA, LN_BETA, W_COL, B_COL, W_ROW, B_ROW = range(6)

_SHUTTING_DOWN = [False]


@atexit.register
def _mark_shutdown():
    # Native handles still alive at interpreter exit are leaked on purpose: the
    # CUDA runtime may already be tearing down when their finalisers run.
    _SHUTTING_DOWN[0] = True

VARIANTS = {"Default": t.ScheduleVariant.Default, "IntraPass": t.ScheduleVariant.IntraPass,
            "CrossPass": t.ScheduleVariant.CrossPass, "Oases": t.ScheduleVariant.Oases}


@dataclass
class ModelConfig:
    hidden: int
    heads: int
    seq: int
    batch: int            # micro-batch, split into two sub-batches
    layers: int
    ffn: int = 0          # 0 -> 4*hidden
    dtype: str = "bf16"   # "bf16" | "f32" | "f64" (the reference's toy FFN blocks only)
    recompute: bool = True
    attention: bool = True
    layernorm: bool = True
    bias: bool = True
    residual: bool = True
    hidden_dropout: float = 0.0
    attention_dropout: float = 0.0
    ln_eps: float = 1e-5
    seed: int = 1234

    def __post_init__(self):
        if not self.ffn:
            self.ffn = 4 * self.hidden

    @property
    def bytes_per_element(self):
        return {"bf16": 2, "f32": 4, "f64": 8}[self.dtype]

    @property
    def num_blocks(self):
        return self.layers * (2 if self.attention else 1)

    def spec(self) -> "t.ModelSpec":
        s = t.ModelSpec()
        s.hidden_size, s.num_layers, s.seq_len = self.hidden, self.layers, self.seq
        s.attention_heads = self.heads if self.attention else 1
        s.global_batch, s.bytes_per_element, s.recompute_enabled = self.batch, self.bytes_per_element, self.recompute
        return s

    def desc(self) -> capi.ModelDesc:
        return capi.ModelDesc(self.hidden, self.layers, self.seq, self.heads, self.batch, self.bytes_per_element,
                              int(self.recompute), self.ffn, int(self.attention), int(self.layernorm),
                              int(self.bias), int(self.residual), self.hidden_dropout, self.attention_dropout,
                              self.ln_eps, 0, self.seed)


def graph_for(cfg: ModelConfig):
    spec = cfg.spec()
    ops = t.build_operator_sequence(spec) if cfg.attention else t.build_ffn_sequence(spec)
    return t.build_block_graph(ops, spec)


def plan_for(cfg: ModelConfig, variant="Oases", keep=None):
    """Schedule for `cfg`. keep: per layer unit, keep its interior post-AllReduce
    tensors (Oases) or replay the unit with its AllReduces (CrossPass); the
    fine-grained recomputation policy (tmpsim.schedule_oases_policy)."""
    if keep is not None:
        return t.schedule_oases_policy(graph_for(cfg), [bool(k) for k in keep])
    return t.make_schedule(graph_for(cfg), VARIANTS[variant] if isinstance(variant, str) else variant)


def recompute_policy(cfg: ModelConfig, budget_bytes: float, *, tp: int = 1, costs=None, profile=None):
    """Per-layer keep/replay choice under an HBM budget (tmpsim.choose_recompute_policy)
    on `costs` (analytic build_cost_vectors of `profile` unless given, e.g. calibrated
    rows loaded with load_measured_costs)."""
    graph = graph_for(cfg)
    if costs is None:
        costs = t.build_cost_vectors(graph, cfg.spec(), profile or t.b200_profile(max(tp, 1)))
    return t.choose_recompute_policy(graph, costs, t.Strategy([tp] * graph.block_count()), float(budget_bytes))


class _FlatPlan:
    """ctypes view of a SchedulePlan (keeps the arrays alive)."""

    def __init__(self, plan):
        ops = list(plan.forward_ops) + list(plan.backward_ops)
        deps = []
        self.ops = (capi.PlanOp * max(1, len(ops)))()
        for i, op in enumerate(ops):
            o = self.ops[i]
            o.id, o.base_id, o.kind, o.pass_ = op.id, op.base_id, int(op.kind), int(op.pass_)
            o.stream, o.block, o.sub_batch, o.blocking = int(op.stream), op.block, op.sub_batch, int(op.blocking)
            o.dep_begin, o.dep_count = len(deps), len(op.deps)
            deps.extend(op.deps)
        self.deps = (C.c_int32 * max(1, len(deps)))(*deps)
        self.c = capi.FlatPlan(int(plan.variant), int(plan.split_batch), int(plan.has_recompute),
                               len(plan.forward_ops), len(ops), len(deps), self.ops, self.deps)


def unique_id() -> bytes:
    buf = (C.c_char * 128)()
    check(capi.lib().oases_get_unique_id(buf))
    return bytes(buf)


def rank_layout(cfg: "ModelConfig", world: int, rank: int, degrees=None) -> list:
    """Rank `rank`'s share of every block of a stack on `world` ranks (host-only,
    no device): one dict per block with the oases_block_layout fields -- the
    data-parallel group and its token slice, the rank inside the tensor-parallel
    group and the local weight widths (include/oases.h, csrc/runtime/layout.h).
    degrees: per-block TMP degrees (None: all at `world`)."""
    nb = cfg.layers * (2 if cfg.attention else 1)
    out = (capi.BlockLayout * max(nb, 1))()
    deg = None if degrees is None else (C.c_int32 * len(degrees))(*[int(x) for x in degrees])
    d = cfg.desc()
    check(capi.lib().oases_rank_layout(C.byref(d), int(world), deg, nb if deg is None else len(degrees), int(rank),
                                       out))
    return [{k: getattr(out[b], k) for k, _ in capi.BlockLayout._fields_} for b in range(nb)]


class Context:
    def __init__(self, tp=1, rank=0, device=0, local_workers=1, unique_id: bytes | None = None, nccl_max_ctas=0,
                 gemm_max_ctas=0, comm_disabled=False):
        self._uid = (C.c_char * 128).from_buffer_copy(unique_id) if unique_id else None
        d = capi.CtxDesc(tp, rank, device, local_workers, C.cast(self._uid, C.c_void_p) if self._uid else None,
                         nccl_max_ctas, gemm_max_ctas, int(comm_disabled))
        self._h = C.c_void_p()
        check(capi.lib().oases_ctx_create(C.byref(d), C.byref(self._h)))
        self.tp, self.rank, self.local_workers = tp, rank, local_workers

    def close(self):
        if self._h:
            check(capi.lib().oases_ctx_destroy(self._h))
            self._h = C.c_void_p()

    def __del__(self):
        if _SHUTTING_DOWN[0]:
            return
        try:
            self.close()
        except Exception:
            pass


@dataclass
class StepResult:
    makespan: float
    compute_busy_fraction: float
    comm_exposed: float
    peak_memory: float
    loss: float
    events: list = field(default_factory=list)  # (op_id, stream, start, end)

    def sim_result(self):
        r = t.SimResult()
        r.makespan, r.compute_busy_fraction = self.makespan, self.compute_busy_fraction
        r.comm_exposed, r.peak_memory = self.comm_exposed, self.peak_memory
        tr = []
        for op_id, stream, s0, s1 in self.events:
            e = t.TraceEvent()
            e.op_id, e.stream, e.start, e.end = op_id, t.Stream.Comm if stream else t.Stream.Compute, s0, s1
            tr.append(e)
        r.trace = tr
        return r


class LayerStack:
    """The TMP layer stack of one process (one rank, or all ranks in-process)."""

    def __init__(self, ctx: Context, cfg: ModelConfig, degrees=None):
        """degrees: per-block TMP degree (each dividing ctx.tp, the world size) for a
        planner-chosen mixed strategy (tmpsim Strategy.degrees); None = every block at
        ctx.tp. A degree-d block runs data-parallel on tp/d groups of d ranks; the
        executor inserts the resharding AllGathers and sums the data-parallel gradients."""
        self.ctx, self.cfg = ctx, cfg
        self._h = C.c_void_p()
        d = cfg.desc()
        if degrees is None:
            check(capi.lib().oases_stack_create(ctx._h, C.byref(d), C.byref(self._h)))
        else:
            deg = (C.c_int32 * len(degrees))(*[int(x) for x in degrees])
            check(capi.lib().oases_stack_create_mixed(ctx._h, C.byref(d), deg, len(degrees), C.byref(self._h)))
        self.num_blocks = capi.lib().oases_stack_num_blocks(self._h)
        self.degrees = [capi.lib().oases_stack_block_degree(self._h, b) for b in range(self.num_blocks)]
        self.num_workers = capi.lib().oases_stack_num_workers(self._h)
        self._plan = None

    def close(self):
        if self._h:
            check(capi.lib().oases_stack_destroy(self._h))
            self._h = C.c_void_p()

    def __del__(self):
        if _SHUTTING_DOWN[0]:
            return
        try:
            self.close()
        except Exception:
            pass

    def param_numel(self, block, p):
        return capi.lib().oases_stack_param_numel(self._h, block, p)

    def set_param(self, worker, block, p, host: np.ndarray):
        a = np.ascontiguousarray(host, dtype=np.float64)
        if a.size != self.param_numel(block, p):
            raise ValueError(f"param ({block},{p}) expects {self.param_numel(block, p)} values, got {a.size}")
        check(capi.lib().oases_stack_set_param(self._h, worker, block, p, a.ctypes.data_as(C.c_void_p)))

    def grad(self, worker, block, p) -> np.ndarray:
        out = np.empty(self.param_numel(block, p), dtype=np.float64)
        check(capi.lib().oases_stack_get_grad(self._h, worker, block, p, out.ctypes.data_as(C.c_void_p)))
        return out

    def init_random(self, seed=1234):
        check(capi.lib().oases_stack_init_random(self._h, seed))

    def set_input(self, x):
        """x: host array [batch*seq, hidden]; float64 converted, or a contiguous buffer of the activation dtype."""
        if isinstance(x, np.ndarray) and x.dtype == np.float64:
            a = np.ascontiguousarray(x)
            self._check_numel(a.size)
            check(capi.lib().oases_stack_set_input(self._h, a.ctypes.data_as(C.c_void_p), 2))
        else:
            check(capi.lib().oases_stack_set_input(self._h, C.c_void_p(self._host_ptr(x)), self._dt()))

    def _check_numel(self, n):
        want = self.cfg.batch * self.cfg.seq * self.cfg.hidden
        if n != want:
            raise ValueError(f"input must hold batch*seq*hidden = {want} elements, got {n}")

    def _host_ptr(self, x) -> int:
        """Pointer of a contiguous HOST buffer in the stack's activation dtype holding exactly
        batch*seq*hidden elements (the C-ABI copies 2*T_sub*hidden elements from it)."""
        want = self.cfg.dtype
        try:
            import torch

            if isinstance(x, torch.Tensor):
                if x.is_cuda:
                    raise ValueError("step input must be a host buffer")
                if not x.is_contiguous():
                    raise ValueError("input tensor must be contiguous")
                got = {torch.bfloat16: "bf16", torch.float32: "f32", torch.float64: "f64"}.get(x.dtype)
                if got != want:
                    raise TypeError(f"input dtype {x.dtype} does not match the stack's {want} activations")
                self._check_numel(x.numel())
                return x.data_ptr()
        except ImportError:
            pass
        if isinstance(x, np.ndarray):
            if not x.flags["C_CONTIGUOUS"]:
                raise ValueError("input array must be C-contiguous")
            got = {"float32": "f32", "float64": "f64", "uint16": "bf16", "bfloat16": "bf16"}.get(x.dtype.name,
                                                                                                x.dtype.name)
            if got != want:
                raise TypeError(f"input dtype {x.dtype} does not match the stack's {want} activations "
                                "(pass float64 to convert, or bf16 bits as uint16)")
            self._check_numel(x.size)
            return x.ctypes.data
        raise TypeError("unsupported input buffer")

    def _dt(self):
        return {"bf16": capi.BF16, "f32": capi.F32, "f64": 2}[self.cfg.dtype]

    def bind(self, plan):
        self._flat = _FlatPlan(plan)
        check(capi.lib().oases_plan_bind(self._h, C.byref(self._flat.c)))
        self._plan = plan

    def capture_graph(self):
        check(capi.lib().oases_stack_capture_graph(self._h))

    def step(self, input=None, trace=True) -> StepResult:
        r = capi.StepResult()
        ptr, dt = None, 0
        if input is not None:
            if isinstance(input, np.ndarray) and input.dtype == np.float64:
                self._in = np.ascontiguousarray(input)
                self._check_numel(self._in.size)
                ptr, dt = self._in.ctypes.data_as(C.c_void_p), 2
            else:
                ptr, dt = C.c_void_p(self._host_ptr(input)), self._dt()
        check(capi.lib().oases_step(self._h, ptr, dt, int(trace), C.byref(r)))
        ev = [(r.events[i].op_id, r.events[i].stream, r.events[i].start, r.events[i].end) for i in range(r.n_events)]
        return StepResult(r.makespan, r.compute_busy_fraction, r.comm_exposed, r.peak_memory, r.loss, ev)

    def input_grad(self) -> np.ndarray:
        out = np.empty((self.cfg.batch * self.cfg.seq, self.cfg.hidden), dtype=np.float64)
        check(capi.lib().oases_stack_get_input_grad(self._h, out.ctypes.data_as(C.c_void_p)))
        return out

    def activation(self, worker, block, sb) -> np.ndarray:
        """x_block rows of sub-batch sb of the worker's group of that block (the last
        block's for block == num_blocks): T_sub rows, or T_sub * degree / world with mixed degrees."""
        b = min(block, self.num_blocks - 1)
        rows = self.cfg.batch * self.degrees[b] // self.ctx.tp // 2 * self.cfg.seq if self.num_blocks else 0
        out = np.empty((rows, self.cfg.hidden), dtype=np.float64)
        check(capi.lib().oases_stack_get_activation(self._h, worker, block, sb, out.ctypes.data_as(C.c_void_p)))
        return out

    def kernel_launches(self):
        return capi.lib().oases_stack_kernel_launches(self._h)

    def set_kernel_timing(self, on=True):
        check(capi.lib().oases_stack_set_kernel_timing(self._h, int(on)))

    def graph_kernel_stats(self):
        """Linear-GEMM timings measured inside a replay of the captured step (timing
        events as graph nodes of a separately captured copy of the step)."""
        k = capi.KernelStats()
        check(capi.lib().oases_stack_graph_kernel_stats(self._h, C.byref(k)))
        return {"gemm_ms": k.gemm_ms, "gemm_flops": k.gemm_flops, "gemm_launches": k.gemm_launches}

    def kernel_stats(self):
        k = capi.KernelStats()
        check(capi.lib().oases_stack_kernel_stats(self._h, C.byref(k)))
        return {"gemm_ms": k.gemm_ms, "gemm_flops": k.gemm_flops, "gemm_launches": k.gemm_launches}


def shard_parameter(param: int, full: np.ndarray, *, tp: int, rank: int, attention: bool, heads: int = 1,
                    hidden: int = 0) -> np.ndarray:
    """Megatron partition of an unsharded (TMP=1, oracle layout [in, out]) parameter
    for TMP rank `rank` of `tp` (numerics.hpp:39-44 / costs.cpp:134,143-144):
    column-parallel W_COL/B_COL by output columns (attention: per head, within
    each of Q, K, V), row-parallel W_ROW by input rows; LN and B_ROW replicated."""
    full = np.asarray(full)
    if param in (LN_GAMMA, LN_BETA, B_ROW) or tp == 1:
        return full.copy()
    if attention:
        h = hidden or full.shape[0]
        hl, d = heads // tp, h // heads
        lo, hi = rank * hl * d, (rank + 1) * hl * d
        if param in (W_COL, B_COL):
            cols = np.concatenate([np.arange(part * h + lo, part * h + hi) for part in range(3)])
            return full[..., cols].copy()
        if param == W_ROW:
            return full[lo:hi].copy()
    else:
        if param in (W_COL, B_COL):
            n = full.shape[-1] // tp
            return full[..., rank * n:(rank + 1) * n].copy()
        if param == W_ROW:
            n = full.shape[0] // tp
            return full[rank * n:(rank + 1) * n].copy()
    raise ValueError(f"unknown parameter id {param}")
