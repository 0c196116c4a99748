"""Named variants, the naive/recursive cutoff rule and the shape-agnostic driver
(mirror of matmulkit/hybrid.py).

``multiply`` keeps the reference's contract (hybrid.py:105-146): any compatible shapes,
a new ``Matrix`` result, caller operands never mutated, and the counter tallies of the
reference's padded square-power-of-two run. What differs is only how the engine pads:
the reference pads all three extents to next_pow2(max(m, k, n)) (1.34x the naive flops
for m=12000, k=14000, n=10000); the engine pads each extent to the next multiple of
2^(L+1) (2^(L+2) for n) for its L recursion levels, so the padded problem stays within
a fraction of a percent of the original. Results are the
same product; floating-point association differs and is tolerance-checked.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import device
from .core import DimensionError, Matrix, _is_tensor, as_view, next_pow2
from .counters import OpCounter
from .kernels import KERNEL_DEFS, BasePolicy, _model_cost, naive_counts, naive_mul
from .schedules import IN_PLACE, TWO_TEMP, schedule_model_cost

KERNEL_NAMES = ("naive", "strassen", "winograd-knuth", "winograd-block", "two-temp", "in-place")

DEFAULT_CUTOFF = 12
DEFAULT_UNROLL = 8


def cutoff_naive_preferred(m: int, k: int, n: int) -> bool:
    """True when one level of divide-and-conquer costs more arithmetic than the naive
    method: m*k*n <= 4*(m*k + k*n + m*n) (order <= 12 for squares, hybrid.py:35-40)."""
    if m < 1 or k < 1 or n < 1:
        raise ValueError("dimensions must be >= 1")
    return m * k * n <= 4 * (m * k + k * n + m * n)


@dataclass(frozen=True)
class VariantSpec:
    """Kernel choice + base-case policy + padding behaviour (hybrid.py:43-60)."""

    kernel: str
    base: BasePolicy | None = None
    pad: bool = True

    def __post_init__(self):
        if self.kernel not in KERNEL_NAMES:
            raise ValueError(f"unknown kernel {self.kernel!r}")
        if self.kernel == "naive":
            if self.base is not None:
                raise ValueError("naive kernel takes no base policy")
            if self.pad:
                raise ValueError("naive kernel does not pad")
        elif self.base is None:
            raise ValueError(f"kernel {self.kernel!r} needs a base policy")


def variant_catalog(cutoff: int = DEFAULT_CUTOFF, unroll: int = DEFAULT_UNROLL) -> list[tuple[str, VariantSpec]]:
    """The twelve named presets (hybrid.py:63-82): plain ("scalar"), "mod" (unrolled 8x8
    base) and "mod2" (naive below ``cutoff``) forms of each algorithm."""
    scalar = BasePolicy.scalar_only()
    unrolled = BasePolicy.unrolled_up_to(unroll)
    mod2 = BasePolicy.naive_cutoff(cutoff)
    presets = [("naive", VariantSpec("naive", None, pad=False))]
    presets += [(k, VariantSpec(k, scalar)) for k in ("strassen", "winograd-knuth", "winograd-block")]
    presets += [("strassen-mod", VariantSpec("strassen", unrolled)),
                ("winograd-mod", VariantSpec("winograd-block", unrolled)),
                ("strassen-mod2", VariantSpec("strassen", mod2)),
                ("winograd-mod2", VariantSpec("winograd-block", mod2))]
    presets += [(k, VariantSpec(k, scalar)) for k in ("two-temp", "in-place")]
    presets += [("two-temp-mod", VariantSpec("two-temp", mod2)), ("in-place-mod", VariantSpec("in-place", mod2))]
    return presets


def preset_names() -> list[str]:
    return [name for name, _ in variant_catalog()]


def get_variant(name: str, cutoff: int = DEFAULT_CUTOFF) -> VariantSpec:
    for preset, spec in variant_catalog(cutoff=cutoff):
        if preset == name:
            return spec
    raise KeyError(f"unknown preset {name!r}; valid presets: {', '.join(preset_names())}")


def _kernel_fn(kernel: str):
    from .kernels import strassen_mul, winograd_block_mul, winograd_knuth_mul
    from .schedules import in_place_winograd, two_temp_winograd

    return {
        "strassen": strassen_mul,
        "winograd-knuth": winograd_knuth_mul,
        "winograd-block": winograd_block_mul,
        "two-temp": two_temp_winograd,
        "in-place": in_place_winograd,
    }[kernel]


def modeled_cost(kernel: str, policy: BasePolicy, order: int) -> tuple[int, int, int, int]:
    if kernel in KERNEL_DEFS:
        return _model_cost(KERNEL_DEFS[kernel], policy, order)
    return schedule_model_cost(TWO_TEMP if kernel == "two-temp" else IN_PLACE, policy, order)


def _empty_like_operands(av, rows, cols, dtype) -> Matrix:
    if av.on_device:
        import torch

        return Matrix(torch.empty((rows, cols), dtype=getattr(torch, np.dtype(dtype).name), device=av.arr.device))
    return Matrix(np.empty((rows, cols), dtype=dtype))


def multiply(a, b, spec: VariantSpec, counter: OpCounter | None = None, trace=None) -> Matrix:
    """C = A x B for any compatible shapes, per the given variant (hybrid.py:105-146)."""
    av, bv = as_view(a), as_view(b)
    if av.cols != bv.rows:
        raise DimensionError(f"inner dimensions differ: {av.cols} vs {bv.rows}")
    counter = OpCounter() if counter is None else counter
    m, k, n = av.rows, av.cols, bv.cols
    dtype = np.result_type(av.dtype, bv.dtype)
    if spec.kernel == "naive":
        c = _empty_like_operands(av, m, n, dtype)
        naive_mul(av, bv, c, counter)
        return c
    order = max(m, k, n)
    target = next_pow2(order)
    conforming = m == k == n == target
    if not conforming and not spec.pad:
        raise DimensionError(f"shape ({m}, {k}, {n}) needs padding but the variant does not pad")
    if conforming and spec.kernel != "in-place":
        c = _empty_like_operands(av, n, n, dtype)
        kwargs = {"trace": trace} if trace is not None and spec.kernel == "two-temp" else {}
        _kernel_fn(spec.kernel)(av, bv, c, spec.base, counter, **kwargs)
        return c
    if conforming:  # in-place on staged copies: caller operands stay intact (hybrid.py:131-146)
        pa, pb = av.to_matrix(), bv.to_matrix()
        c = _empty_like_operands(av, n, n, dtype)
        kwargs = {"trace": trace} if trace is not None else {}
        _kernel_fn("in-place")(pa, pb, c, spec.base, counter, **kwargs)
        return c
    # non-conforming: the reference pads to a square of order `target`; the engine pads
    # each extent only to what its recursion needs and reports the reference's tallies.
    if trace is not None and spec.kernel in ("two-temp", "in-place"):
        from .schedules import _top_is_base

        sched = TWO_TEMP if spec.kernel == "two-temp" else IN_PLACE
        if not _top_is_base(target, spec.base):
            for s, _, _ in sched.plan:
                trace(s.render())
    levels = device.levels_for(target, spec.base, spec.kernel if spec.kernel in ("two-temp", "in-place")
                               else spec.kernel)
    c = _empty_like_operands(av, m, n, dtype)
    engine_algo = "winograd-block" if spec.kernel in ("two-temp", "in-place") else spec.kernel
    if levels == 0:
        device.device_gemm(av, bv, c.view(), dtype)
    else:
        device.device_rect(engine_algo, av, bv, c.view(), levels, dtype)
    counter.absorb(*modeled_cost(spec.kernel, spec.base, target))
    return c


__all__ = [
    "KERNEL_NAMES", "DEFAULT_CUTOFF", "DEFAULT_UNROLL", "cutoff_naive_preferred", "VariantSpec",
    "variant_catalog", "preset_names", "get_variant", "multiply",
]

_ = (_is_tensor, naive_counts)
