"""``sparseconv.execution`` on the B200 engine (reference ``execution.py``).

Layer forwards run the engine (``ExecOptions.dataflow``: the staged
gather -> tcgen05 grouped GEMM -> output-stationary scatter by default,
the fused implicit-GEMM kernel with ``"fused"``/``"auto"``); the movement
primitives run their device kernels.  Arrays cross the boundary as numpy.
The reuse-key ``map_cache`` holds engine maps, so an inverse layer replays
its strided layer's map without leaving HBM.
"""

from __future__ import annotations

import numpy as np
import torch

from paper_2204_10319_b200 import execution as _eng

from .core import SparseTensor, _engine_tensor, _wrap_result
from .mapping import GatherScatterPlan, KernelMap

GATHER_ORDERS = _eng.GATHER_ORDERS
SCATTER_ORDERS = _eng.SCATTER_ORDERS
StageTimer = _eng.StageTimer
LayerStrategy = _eng.LayerStrategy
LayerSpec = _eng.LayerSpec
resolve_strategy = _eng.resolve_strategy
CachedMap = _eng.CachedMap
ExecOptions = _eng.ExecOptions
partition_groups = _eng.partition_groups
MatmulGroup = _eng.MatmulGroup
GroupingStrategy = _eng.GroupingStrategy
schedule_for = _eng.schedule_for
build_grouping = _eng.build_grouping


def _host(x: torch.Tensor) -> np.ndarray:
    return x.detach().cpu().numpy()


def _plan(plan):
    return plan._dev if isinstance(plan, GatherScatterPlan) else plan


def gather(features, plan, order: str = "weight_stationary") -> np.ndarray:
    """Offset-partitioned buffer (reference execution.py:159-180) with
    ``scb_gather``; both orders give the same bit-exact buffer."""
    if order not in GATHER_ORDERS:
        raise ValueError(f"unknown gather order {order!r}")
    f = np.asarray(features)
    if f.shape[0] != plan.n_in:
        raise ValueError("plan does not match the feature row count")
    if plan.total == 0:
        return np.empty((0, f.shape[1]), dtype=f.dtype)
    return _host(_eng.gather(f, _plan(plan), order))


def scatter_accumulate(buffer, plan, n_out: int, order: str = "weight_stationary",
                       out_dtype=np.float32) -> np.ndarray:
    """Fold buffer rows into output rows in ascending buffer-row order
    (reference execution.py:183-218) with the output-stationary
    ``scb_scatter`` (f32 accumulation; the reference folds in f64)."""
    if order not in SCATTER_ORDERS:
        raise ValueError(f"unknown scatter order {order!r}")
    b = np.asarray(buffer)
    if b.shape[0] != plan.total:
        raise ValueError("buffer rows do not match the plan")
    if plan.total == 0 or n_out == 0:
        return np.zeros((n_out, b.shape[1]), dtype=out_dtype)
    return _host(_eng.scatter_accumulate(b, _plan(plan), n_out, order, out_dtype))


def execute_groups(buffer, weights, strategy: GroupingStrategy, map_sizes) -> np.ndarray:
    """Grouped multiplies over an offset-partitioned buffer (reference
    execution.py:331-368) on the grouped GEMM kernel; returns the f32
    partial buffer."""
    b = np.asarray(buffer)
    w = np.asarray(weights, dtype=np.float32)
    sizes = np.asarray(map_sizes, dtype=np.int64)
    if sizes.shape[0] != w.shape[0]:
        raise ValueError("map sizes do not match the weight slices")
    strategy.validate(sizes)
    if b.shape[0] != int(sizes.sum()):
        raise ValueError("buffer rows do not match the map sizes")
    if b.shape[0] == 0:
        return np.zeros((0, w.shape[2]), dtype=np.float32)
    return _host(_eng.execute_groups(b, w, strategy, sizes))


def sparse_conv_forward(t: SparseTensor, w, spec: LayerSpec, strategy: LayerStrategy | None = None,
                        map_cache: dict | None = None,
                        options: ExecOptions | None = None) -> SparseTensor:
    """One sparse convolution layer (reference execution.py:450-509)."""
    out = _eng.sparse_conv_forward(_engine_tensor(t), w, spec, strategy, map_cache, options)
    _host_plans(options)
    return _wrap_result(out, t)


def inverse_conv_forward(t: SparseTensor, w, spec: LayerSpec, map_cache: dict,
                         strategy: LayerStrategy | None = None,
                         options: ExecOptions | None = None) -> SparseTensor:
    """Transposed layer replaying a cached strided map (reference
    execution.py:512-551)."""
    out = _eng.inverse_conv_forward(_engine_tensor(t), w, spec, map_cache, strategy, options)
    _host_plans(options)
    return _wrap_result(out)


def pointwise_apply(t: SparseTensor, op: str, *, bias=None, scale=None,
                    shift=None) -> SparseTensor:
    """relu / bias_add / bn_fold (reference execution.py:554-576) with
    ``scb_pointwise``."""
    return _wrap_result(_eng.pointwise_apply(_engine_tensor(t), op, bias=bias, scale=scale,
                                             shift=shift), t)


def _host_plans(options: ExecOptions | None) -> None:
    """Entries the engine appended to ``plan_log`` keep their maps alive
    (the engine plan holds its map weakly)."""
    if options is None or options.plan_log is None:
        return
    for i, (label, p) in enumerate(options.plan_log):
        if not isinstance(p, GatherScatterPlan) and hasattr(p, "kmap"):
            try:
                km = KernelMap._from_engine(p.kmap)
            except RuntimeError:
                continue
            options.plan_log[i] = (label, GatherScatterPlan(p, km))
