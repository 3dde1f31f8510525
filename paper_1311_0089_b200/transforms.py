"""Host containers and discrete mean inner product.

Mirror of the parts of ``fftcell.transforms`` the solver path uses
(``/root/reference/pkg/src/fftcell/transforms.py:37-61,168-180``).  The
``(d, *N)`` fp64 component-major layout of :class:`GridField` is exactly the
layout of the device vectors (one such block per right-hand side).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .grid import GridSpec


@dataclass(frozen=True)
class GridField:
    """Real d-vector field, component-major ``(d, *N)`` (``transforms.py:37-61``)."""

    spec: GridSpec
    values: np.ndarray

    def __post_init__(self):
        v = np.asarray(self.values, dtype=float)
        expected = (self.spec.dim,) + self.spec.shape
        if v.shape != expected:
            raise ValueError(f"values shape {v.shape} != expected {expected}")
        object.__setattr__(self, "values", v)

    @classmethod
    def zeros(cls, spec):
        return cls(spec, np.zeros((spec.dim,) + spec.shape))

    @classmethod
    def constant(cls, spec, vec):
        vec = np.asarray(vec, dtype=float)
        values = np.broadcast_to(
            vec.reshape((spec.dim,) + (1,) * spec.dim), (spec.dim,) + spec.shape
        ).copy()
        return cls(spec, values)


def l2_inner(u: GridField, v: GridField) -> float:
    """Discrete mean inner product ``(1/|N|) sum <u^k, v^k>`` (``transforms.py:168-176``)."""
    if u.spec != v.spec:
        raise ValueError("grid specs do not match")
    return float(np.sum(u.values * v.values) / u.spec.total)


def l2_norm(u: GridField) -> float:
    """``transforms.py:179-180``."""
    return float(np.sqrt(max(l2_inner(u, u), 0.0)))


def pairwise_sum_runs(values, counts) -> float:
    """numpy's float64 ``np.sum`` of the array ``values[0]`` x ``counts[0]``,
    ``values[1]`` x ``counts[1]``, ... without materialising it.

    Restates numpy's pairwise summation (blocks of <= 128 elements summed with
    eight accumulators, longer ranges split in halves rounded down to a multiple
    of 8), which ``np.sum`` applies to a contiguous array as one flat pass.  Every
    sub-range that lies inside one run is a constant block whose sum depends only
    on (value, length), so the recursion is memoised: O(log n) work per run.
    Used for ``l2_norm(E_N)`` of a constant load (solver.py:258) on grids far
    too large to expand on the host (tests/test_host_api.py checks it against
    np.sum bit for bit)."""
    values = [float(v) for v in values]
    starts = [0]
    for c in counts:
        starts.append(starts[-1] + int(c))
    memo = {}

    def run_at(i):
        lo, hi = 0, len(values) - 1
        while lo < hi:  # last run with start <= i
            mid = (lo + hi + 1) // 2
            if starts[mid] <= i:
                lo = mid
            else:
                hi = mid - 1
        return lo

    def block(get, n):
        if n < 8:
            res = -0.0
            for i in range(n):
                res += get(i)
            return res
        r = [get(j) for j in range(8)]
        i = 8
        while i < n - (n % 8):
            for j in range(8):
                r[j] += get(i + j)
            i += 8
        res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]))
        while i < n:
            res += get(i)
            i += 1
        return res

    def const(c, n):
        key = (c, n)
        if key not in memo:
            if n <= 128:
                memo[key] = block(lambda i: c, n)
            else:
                n2 = n // 2
                n2 -= n2 % 8
                memo[key] = const(c, n2) + const(c, n - n2)
        return memo[key]

    def pw(off, n):
        k = run_at(off)
        if off + n <= starts[k + 1]:
            return const(values[k], n)
        if n <= 128:
            return block(lambda i: values[run_at(off + i)], n)
        n2 = n // 2
        n2 -= n2 % 8
        return pw(off, n2) + pw(off + n2, n - n2)

    total = starts[-1]
    return pw(0, total) if total > 0 else 0.0
