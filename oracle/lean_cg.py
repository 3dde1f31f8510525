"""Memory-lean restatement of the reference CG for full-size anchors (TEST INFRASTRUCTURE ONLY).

Same algorithm as ``fftcell_oracle.solve_cg`` (``solver.py:142-230``), rewritten
so a 729^3 anisotropic solve fits a 196 GB host:

* the coefficient field stays packed ``(d(d+1)/2, *N)`` (``material.py:30-49``);
  the reference expands it to ``(d, d, *N)`` (``material.py:112``) and its
  einsum reads that (``solver.py:174``) -- the same products, summed over b in
  the same order 0..d-1;
* the projection runs on the real-to-complex half spectrum
  (``scipy.fft.rfftn`` / ``irfftn``, pocketfft, multi-threaded) with the
  frequency grid broadcast from per-axis tables; the reference takes the real
  part of a full complex ``ifftn`` (``solver.py:112-116``): the same operator,
  FFT rounding differs (the parity budget of SURVEY 8(c) is ~1e-12 relative on
  histories, far above it);
* inner products use ``np.vdot`` (BLAS) instead of ``np.sum(x * y)``
  (``solver.py:138-139``): same value up to summation-order rounding.

It is pinned against the standard oracle and the reference's own goldens in
``tests/test_oracle_golden.py::test_lean_cg_matches_reference_golden``.
Only ``tests/`` and ``tests/golden/`` scripts import it.
"""

from __future__ import annotations

import os

import numpy as np


def _freq(n, Y):
    """grid.py:131-146: xi = k / Y with k in numpy fftfreq order."""
    return np.fft.fftfreq(n, d=1.0 / n).round() / Y


class LeanOperator:
    """``p -> G (A p)`` (solver.py:173-174 with the orthogonal G, solver.py:112-116)."""

    def __init__(self, shape, Y, packed=None, scalars=None, workers=None):
        self.shape = tuple(int(n) for n in shape)
        self.d = len(self.shape)
        self.total = int(np.prod(self.shape))
        self.packed = packed
        self.scalars = scalars
        self.workers = workers or os.cpu_count()
        d = self.d
        self.xi = [_freq(n, y) for n, y in zip(self.shape, Y)]
        self.xi[-1] = self.xi[-1][: self.shape[-1] // 2 + 1]  # rfft half axis (odd n: k = 0..(n-1)/2)
        self.pairs = [(a, a) for a in range(d)] + [(a, b) for a in range(d) for b in range(a + 1, d)]
        self.pidx = {}
        for m, (a, b) in enumerate(self.pairs):
            self.pidx[(a, b)] = m
            self.pidx[(b, a)] = m

    def _bcast(self, a):
        s = [1] * self.d
        s[a] = -1
        return self.xi[a].reshape(s)

    def apply_A(self, v, out):
        """material.py:182-187 / the einsum of solver.py:174 (sum over b in order)."""
        d = self.d
        if self.scalars is not None:
            for a in range(d):
                np.multiply(self.scalars, v[a], out=out[a])
            return out
        tmp = np.empty(self.shape)
        for a in range(d):
            np.multiply(self.packed[self.pidx[(a, 0)]], v[0], out=out[a])
            for b in range(1, d):
                np.multiply(self.packed[self.pidx[(a, b)]], v[b], out=tmp)
                out[a] += tmp
        return out

    def project(self, y):
        """_project_hat between forward and inverse transforms (solver.py:106-116)."""
        import scipy.fft as sf

        d = self.d
        axes = tuple(range(1, d + 1))
        Yh = sf.rfftn(y, axes=axes, workers=self.workers)
        hshape = Yh.shape[1:]
        # chunk over axis 0 to bound the temporaries
        step = max(1, hshape[0] // 16)
        xs = [self._bcast(a) for a in range(d)]
        for s in range(0, hshape[0], step):
            sl = slice(s, min(s + step, hshape[0]))
            x0 = xs[0][sl]
            dots = x0 * Yh[0, sl]
            for a in range(1, d):
                dots += xs[a] * Yh[a, sl]
            den = x0 * x0
            for a in range(1, d):
                den = den + xs[a] * xs[a]
            if s == 0:
                den = np.array(np.broadcast_to(den, dots.shape))
                den[(0,) * d] = 1.0
            q = dots / den
            if s == 0:
                q[(0,) * d] = 0.0
            Yh[0, sl] = x0 * q
            for a in range(1, d):
                Yh[a, sl] = xs[a] * q
            del dots, q, den
        return sf.irfftn(Yh, s=self.shape, axes=axes, workers=self.workers)

    def __call__(self, v, out):
        self.apply_A(v, out)
        res = self.project(out)
        out[...] = res
        return out

    def inner(self, x, y):
        return float(np.vdot(x.reshape(-1), y.reshape(-1)) / self.total)


def solve_cg(op, E, tol, max_iter, on_iter=None):
    """solver.py:142-230 (zero init, no reference tensor), in place.

    Returns dict(iterations, converged, history, solution)."""
    d = op.d
    E = np.asarray(E, dtype=float)
    # rhs = -operator(E_N) (solver.py:176-178); E_N is constant per component
    e_n = np.empty((d,) + op.shape)
    for a in range(d):
        e_n[a] = E[a]
    r = np.empty_like(e_n)
    op(e_n, r)
    del e_n
    np.negative(r, out=r)
    r0_norm = np.sqrt(op.inner(r, r))
    history = [np.sqrt(op.inner(r, r))]
    x = np.zeros_like(r)
    if r0_norm == 0.0 or history[0] <= tol * r0_norm:
        return dict(iterations=0, converged=True, history=history, solution=x)
    p = r.copy()
    Ap = np.empty_like(r)
    rr = op.inner(r, r)
    converged = False
    iterations = 0
    for i in range(max_iter):
        op(p, Ap)
        pAp = op.inner(p, Ap)
        if pAp <= 0:
            return dict(iterations=iterations, converged=False, history=history, solution=x,
                        message=f"operator lost positive definiteness (pAp={pAp:.3e})")
        alpha = rr / pAp
        for a in range(d):
            x[a] += alpha * p[a]
            r[a] -= alpha * Ap[a]
        rr_new = op.inner(r, r)
        iterations = i + 1
        history.append(np.sqrt(rr_new))
        if on_iter is not None:
            on_iter(iterations, history[-1])
        if np.sqrt(rr_new) <= tol * r0_norm:
            converged = True
            break
        beta = rr_new / rr
        for a in range(d):
            p[a] *= beta
            p[a] += r[a]
        rr = rr_new
    return dict(iterations=iterations, converged=converged, history=history, solution=x)
