"""Naive, Strassen and Strassen-Winograd products on the B200 engine (mirror of
matmulkit/kernels.py).

Entry points keep the reference signatures, validation order, error types and
``OpCounter`` values. The arithmetic runs in libmk_strassen.so:

* ``naive_mul``            -> mk_dgemm (FP64 DMMA kernel; reference kernels.py:350-367)
* ``strassen_mul``         -> mk_strassen(STRASSEN)        (kernels.py:370-375)
* ``winograd_block_mul``   -> mk_strassen(WINOGRAD_BLOCK)  (kernels.py:378-383)
* ``winograd_knuth_mul``   -> mk_strassen(WINOGRAD_KNUTH[_8CALL]) (kernels.py:386-397)
* ``unrolled_base``        -> mk_strassen / mk_dgemm at orders 2, 4, 8 (kernels.py:400-419)

The recursion depth the engine runs comes from the reference's base policy
(``BasePolicy``): naive-cutoff thresholds are honoured exactly; recursion below the
engine's minimum leaf order (the reference's scalar / unrolled micro-kernels, orders
1..8) is clamped. Integer results are identical either way; the modeled counters always
describe the policy's literal recursion, exactly like the reference's micro fast path
(kernels.py:195-199).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import device
from .core import DimensionError, as_view, result_dtype
from .counters import OpCounter
from .tables import (
    C_QUADS,
    INPUT_QUADS,
    STRASSEN_STEPS,
    WINOGRAD_BLOCK_STEPS,
    WINOGRAD_KNUTH_8CALL_STEPS,
    WINOGRAD_KNUTH_STEPS,
)


@dataclass(frozen=True)
class BasePolicy:
    """Where recursion stops (reference kernels.py:26-57).

    "scalar": down to 1x1; "unrolled": straight-line base kernel at ``order`` (1, 2, 4, 8);
    "naive-cutoff": the naive product at order <= ``threshold``.
    """

    kind: str
    order: int = 1
    threshold: int = 12

    def __post_init__(self):
        if self.kind not in ("scalar", "unrolled", "naive-cutoff"):
            raise ValueError(f"unknown base policy kind {self.kind!r}")
        if self.kind == "unrolled" and self.order not in (1, 2, 4, 8):
            raise ValueError(f"unrolled order must be 1, 2, 4, or 8, got {self.order}")
        if self.kind == "naive-cutoff" and self.threshold < 1:
            raise ValueError(f"cutoff threshold must be >= 1, got {self.threshold}")

    @classmethod
    def scalar_only(cls) -> "BasePolicy":
        return cls("scalar")

    @classmethod
    def unrolled_up_to(cls, order: int) -> "BasePolicy":
        return cls("unrolled", order=order)

    @classmethod
    def naive_cutoff(cls, threshold: int = 12) -> "BasePolicy":
        return cls("naive-cutoff", threshold=threshold)


SCALAR_ONLY = BasePolicy.scalar_only()
DEFAULT_MICRO_ORDER = 8


class KernelDef:
    """Derived per-level figures of one step table."""

    def __init__(self, name: str, steps):
        self.name = name
        self.steps = tuple(steps)
        self.adds_per_level = sum(op != "mul" for op, *_ in self.steps)
        self.muls_per_level = sum(op == "mul" for op, *_ in self.steps)
        temps = []
        for _, dst, _, _ in self.steps:
            if dst not in C_QUADS and dst not in INPUT_QUADS and dst not in temps:
                temps.append(dst)
        self.temp_names = tuple(temps)


KERNEL_DEFS = {
    "strassen": KernelDef("strassen", STRASSEN_STEPS),
    "winograd-block": KernelDef("winograd-block", WINOGRAD_BLOCK_STEPS),
    "winograd-knuth": KernelDef("winograd-knuth", WINOGRAD_KNUTH_STEPS),
    "winograd-knuth-8call": KernelDef("winograd-knuth-8call", WINOGRAD_KNUTH_8CALL_STEPS),
}

_COST_CACHE: dict = {}


def _level_peak(steps, hh: int, child_peak: int, is_temp) -> int:
    """High-water mark of one call: temps allocated in table order, a product's subtree
    peak stacked on whatever is live when it runs (reference kernels.py:229-240)."""
    live = peak = 0
    seen = set()
    for op, dst in steps:
        if is_temp(dst) and dst not in seen:
            seen.add(dst)
            live += hh
            peak = max(peak, live)
        if op == "mul":
            peak = max(peak, live + child_peak)
    return peak


def model_cost(kernel: str, policy: BasePolicy, n: int) -> tuple[int, int, int, int]:
    """(mults, adds, buffer events, peak live aux elements) of the literal recursion."""
    return _model_cost(KERNEL_DEFS[kernel], policy, n)


def _model_cost(kdef: KernelDef, policy: BasePolicy, n: int) -> tuple[int, int, int, int]:
    key = (kdef.name, policy, n)
    if key in _COST_CACHE:
        return _COST_CACHE[key]
    if n == 1:
        res = (1, 0, 0, 0)
    elif policy.kind == "naive-cutoff" and n <= policy.threshold:
        res = (n ** 3, n * n * (n - 1), 0, 0)
    elif policy.kind == "unrolled" and n <= policy.order:
        mm, aa, _, _ = _model_cost(kdef, SCALAR_ONLY, n)
        res = (mm, aa, 0, 0)
    else:
        h = n // 2
        cm, ca, cb, cp = _model_cost(kdef, policy, h)
        peak = _level_peak([(op, dst) for op, dst, _, _ in kdef.steps], h * h, cp, lambda d: d not in C_QUADS)
        k = kdef.muls_per_level
        res = (k * cm, k * ca + kdef.adds_per_level * h * h, k * cb + len(kdef.temp_names), peak)
    _COST_CACHE[key] = res
    return res


def naive_counts(m: int, inner: int, k: int) -> tuple[int, int]:
    """(mults, adds) of the direct method (reference kernels.py:265-266)."""
    return m * inner * k, (m * k * (inner - 1) if inner >= 1 else 0)


def _check_square_pow2(a, b, c) -> int:
    n = a.rows
    if not (a.rows == a.cols == b.rows == b.cols == c.rows == c.cols):
        raise DimensionError(
            f"operands must be square of one order, got {a.rows}x{a.cols}, {b.rows}x{b.cols}, {c.rows}x{c.cols}"
        )
    if n & (n - 1):
        raise DimensionError(f"order {n} is not a power of two; pad inputs first")
    return n


def _run_dc(kernel: str, a, b, c, policy, counter, micro_order) -> OpCounter:
    a, b, c = as_view(a), as_view(b), as_view(c)
    n = _check_square_pow2(a, b, c)
    device.check_disjoint(a, b, c)
    policy = SCALAR_ONLY if policy is None else policy
    counter = OpCounter() if counter is None else counter
    # micro_order (reference kernels.py:343-345) only selects a CPU execution detail there;
    # it is accepted and has no effect on the engine.
    _ = max(1, min(DEFAULT_MICRO_ORDER if micro_order is None else micro_order, 8))
    algo = "winograd-block" if kernel == "winograd-block" else kernel
    levels = device.levels_for(n, policy, algo)
    dtype = result_dtype(a, b)
    if levels == 0:
        device.device_gemm(a, b, c, dtype)
    else:
        device.device_square(algo, a, b, c, levels, dtype)
    counter.absorb(*_model_cost(KERNEL_DEFS[kernel], policy, n))
    return counter


def naive_mul(a, b, c, counter: OpCounter | None = None) -> OpCounter:
    """c = a x b by the direct method, on the FP64 DMMA kernel.

    Counts m*n*k multiplications and m*k*(n-1) additions (reference kernels.py:350-367).
    """
    a, b, c = as_view(a), as_view(b), as_view(c)
    if a.cols != b.rows:
        raise DimensionError(f"inner dimensions differ: {a.cols} vs {b.rows}")
    if c.rows != a.rows or c.cols != b.cols:
        raise DimensionError(f"output must be {a.rows}x{b.cols}, got {c.rows}x{c.cols}")
    device.check_disjoint(a, b, c)
    counter = OpCounter() if counter is None else counter
    device.device_gemm(a, b, c, result_dtype(a, b))
    mm, aa = naive_counts(a.rows, a.cols, b.cols)
    counter.mults += mm
    counter.adds += aa
    return counter


def strassen_mul(a, b, c, policy: BasePolicy | None = None, counter: OpCounter | None = None,
                 micro_order: int | None = None) -> OpCounter:
    """c = a x b with seven recursive products and eighteen block additions per level."""
    return _run_dc("strassen", a, b, c, policy, counter, micro_order)


def winograd_block_mul(a, b, c, policy: BasePolicy | None = None, counter: OpCounter | None = None,
                       micro_order: int | None = None) -> OpCounter:
    """c = a x b via the block Winograd form (seven products, fifteen block additions)."""
    return _run_dc("winograd-block", a, b, c, policy, counter, micro_order)


def winograd_knuth_mul(a, b, c, policy: BasePolicy | None = None, counter: OpCounter | None = None,
                       micro_order: int | None = None, recompute_first_product: bool = False) -> OpCounter:
    """c = a x b via Knuth's u/v/w arrangement; ``recompute_first_product`` selects the
    eight-call variant (reference kernels.py:386-397)."""
    kernel = "winograd-knuth-8call" if recompute_first_product else "winograd-knuth"
    return _run_dc(kernel, a, b, c, policy, counter, micro_order)


def unrolled_base(a, b, c, order: int, counter: OpCounter | None = None) -> OpCounter:
    """Block-Winograd product at order 2, 4 or 8 with the straight-line kernel's counts
    (reference kernels.py:400-419)."""
    if order not in (2, 4, 8):
        raise DimensionError(f"unrolled base kernels exist for orders 2, 4, 8; got {order}")
    a, b, c = as_view(a), as_view(b), as_view(c)
    n = _check_square_pow2(a, b, c)
    if n != order:
        raise DimensionError(f"operands are order {n}, expected {order}")
    device.check_disjoint(a, b, c)
    counter = OpCounter() if counter is None else counter
    levels = 1 if order >= 4 else 0  # leaf order >= 2 on the engine
    dtype = result_dtype(a, b)
    if levels == 0:
        device.device_gemm(a, b, c, dtype)
    else:
        device.device_square("winograd-block", a, b, c, levels, dtype)
    mm, aa, _, _ = _model_cost(KERNEL_DEFS["winograd-block"], SCALAR_ONLY, order)
    counter.absorb(mm, aa, 0, 0)
    return counter


__all__ = [
    "BasePolicy", "SCALAR_ONLY", "KERNEL_DEFS", "model_cost", "naive_mul", "strassen_mul",
    "winograd_block_mul", "winograd_knuth_mul", "unrolled_base",
]

_ = np  # numpy is part of the public dtype contract (result types follow np.result_type)
