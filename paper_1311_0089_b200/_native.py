"""ctypes binding of ``libfftcell_b200.so`` (C ABI: ``include/fftcell_b200.h``).

The shared library is built in-tree by ``__graft_entry__.build()``.  There is
no CPU fallback: if the library or a CUDA device is missing every call raises
``RuntimeError`` (north_star "no CPU fallback").
"""

from __future__ import annotations

import ctypes
import mmap
import os
from pathlib import Path

import numpy as np

# FC_LIB: an alternative build of the same library (A/B measurements of
# experimental builds without touching the in-tree one)
LIB_PATH = Path(os.environ.get("FC_LIB") or Path(__file__).resolve().parent / "libfftcell_b200.so")
MAX_RHS = 8
MAX_PHASES = 4096  # FC_MAX_PHASES

FC_OK, FC_EINVAL, FC_ENOMEM, FC_ECUDA, FC_ENOTSUP = 0, 1, 2, 3, 4
ST_OK, ST_MAXITER, ST_BREAKDOWN, ST_DIVERGENT = 0, 1, 2, 3

_dp = ctypes.POINTER(ctypes.c_double)
_i64p = ctypes.POINTER(ctypes.c_int64)


class Report(ctypes.Structure):
    _fields_ = [
        ("iterations", ctypes.c_int32),
        ("converged", ctypes.c_int32),
        ("status", ctypes.c_int32),
        ("hist_len", ctypes.c_int32),
        ("detail", ctypes.c_double),
    ]


_lib = None

# (name, restype, argtypes) for every symbol declared in include/fftcell_b200.h
SIGNATURES = [
    ("fc_version", ctypes.c_int32, []),
    ("fc_last_error", ctypes.c_char_p, []),
    ("fc_device_count", ctypes.c_int32, [ctypes.POINTER(ctypes.c_int32)]),
    ("fc_set_plan_option", ctypes.c_int32, [ctypes.c_char_p, ctypes.c_int32]),
    ("fc_reset_plan_options", ctypes.c_int32, []),
    ("fc_create", ctypes.c_int32,
     [ctypes.POINTER(ctypes.c_void_p), ctypes.c_int32, _i64p, _dp, ctypes.c_int32]),
    ("fc_create_sharded", ctypes.c_int32,
     [ctypes.POINTER(ctypes.c_void_p), ctypes.c_int32, _i64p, _dp, ctypes.c_int32, ctypes.POINTER(ctypes.c_int32)]),
    ("fc_nccl_unique_id", ctypes.c_int32, [ctypes.c_void_p]),
    ("fc_create_dist", ctypes.c_int32,
     [ctypes.POINTER(ctypes.c_void_p), ctypes.c_int32, _i64p, _dp, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
      ctypes.c_void_p]),
    ("fc_destroy", None, [ctypes.c_void_p]),
    ("fc_set_coefficients", ctypes.c_int32, [ctypes.c_void_p, ctypes.c_int32, _dp, ctypes.c_int64]),
    ("fc_set_coefficients_indexed", ctypes.c_int32,
     [ctypes.c_void_p, ctypes.c_int32, _dp, ctypes.POINTER(ctypes.c_uint16), ctypes.c_int64]),
    ("fc_compress_coefficients", ctypes.c_int32,
     [ctypes.c_void_p, ctypes.c_int32, ctypes.c_int32, ctypes.POINTER(ctypes.c_int32)]),
    ("fc_load_coefficients", ctypes.c_int32, [ctypes.c_void_p, ctypes.c_int32, ctypes.c_char_p]),
    ("fc_coefficient_bounds", ctypes.c_int32, [ctypes.c_void_p, _dp, _dp, _i64p]),
    ("fc_save_solution", ctypes.c_int32, [ctypes.c_void_p, ctypes.c_int32, ctypes.c_char_p]),
    ("fc_apply_A", ctypes.c_int32, [ctypes.c_void_p, _dp, _dp, ctypes.c_int32]),
    ("fc_project", ctypes.c_int32, [ctypes.c_void_p, ctypes.c_int32, _dp, _dp, _dp, ctypes.c_int32]),
    ("fc_apply_system", ctypes.c_int32, [ctypes.c_void_p, _dp, _dp, ctypes.c_int32]),
    ("fc_solve_cg", ctypes.c_int32,
     [ctypes.c_void_p, ctypes.c_int32, _dp, ctypes.c_double, ctypes.c_int32, ctypes.c_double, _dp, _dp,
      ctypes.POINTER(Report), _dp, _dp, ctypes.c_int64, _i64p]),
    ("fc_solve_fixed_point", ctypes.c_int32,
     [ctypes.c_void_p, ctypes.c_int32, _dp, ctypes.c_double, ctypes.c_int32, _dp, _dp, _dp,
      ctypes.POINTER(Report), _dp]),
    ("fc_energy", ctypes.c_int32, [ctypes.c_void_p, ctypes.c_int32, _dp, _dp, _dp]),
    ("fc_generate_voronoi", ctypes.c_int32,
     [ctypes.c_void_p, ctypes.c_int32, _dp, _dp, ctypes.POINTER(ctypes.c_int32)]),
    ("fc_spheres_stamp", ctypes.c_int32,
     [ctypes.c_void_p, ctypes.c_int32, ctypes.POINTER(ctypes.c_int32), ctypes.c_double, _i64p]),
    ("fc_spheres_finish", ctypes.c_int32, [ctypes.c_void_p, ctypes.c_double, ctypes.c_double]),
    ("fc_set_profiling", ctypes.c_int32, [ctypes.c_void_p, ctypes.c_int32]),
    ("fc_profile_count", ctypes.c_int32, [ctypes.c_void_p]),
    ("fc_profile_get", ctypes.c_int32,
     [ctypes.c_void_p, ctypes.c_int32, ctypes.c_char_p, ctypes.c_int32, _i64p, _dp]),
    ("fc_profile_reset", ctypes.c_int32, [ctypes.c_void_p]),
    ("fc_launch_count", ctypes.c_int64, [ctypes.c_void_p]),
    ("fc_plan_info", ctypes.c_int32, [ctypes.c_void_p, ctypes.c_char_p, ctypes.POINTER(ctypes.c_int32)]),
    ("fc_timer_mark", ctypes.c_int32, [ctypes.c_void_p, ctypes.c_int32]),
    ("fc_timer_elapsed", ctypes.c_int32, [ctypes.c_void_p, ctypes.c_int32, ctypes.c_int32, _dp]),
]


def lib():
    """Load the CUDA library (fails loudly when it has not been built)."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise RuntimeError(
                f"CUDA extension {LIB_PATH.name} is not built; run `python -c "
                "'import __graft_entry__ as g; g.build()'` (no CPU fallback exists)"
            )
        handle = ctypes.CDLL(str(LIB_PATH))
        for name, res, args in SIGNATURES:
            fn = getattr(handle, name)
            fn.restype = res
            fn.argtypes = args
        _lib = handle
    return _lib


def _check(rc):
    if rc == FC_OK:
        return
    msg = lib().fc_last_error().decode(errors="replace")
    if rc == FC_EINVAL:
        raise ValueError(msg)
    if rc == FC_ENOTSUP:
        raise NotImplementedError(msg)
    if rc == FC_ENOMEM:
        raise MemoryError(msg)
    raise RuntimeError(f"CUDA error: {msg}")


def _ptr(a):
    return a.ctypes.data_as(_dp) if a is not None else None


def _c64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(lib().fc_nccl_unique_id(buf))
    return buf.raw


class plan_options:
    """Context manager: plan options (fc_set_plan_option) for the contexts created
    inside the block, e.g. ``with plan_options(aniso_fused=0): Context(spec)``.
    Options are frozen into a context at creation; the defaults are restored on exit."""

    def __init__(self, **opts):
        self.opts = opts

    def __enter__(self):
        for k, v in self.opts.items():
            _check(lib().fc_set_plan_option(k.encode(), int(v)))
        return self

    def __exit__(self, *exc):
        _check(lib().fc_reset_plan_options())


def device_count():
    n = ctypes.c_int32(0)
    rc = lib().fc_device_count(ctypes.byref(n))
    return int(n.value) if rc == FC_OK else 0


class Context:
    """One GridSpec bound to one GPU: coefficients, FFT plans and workspace in HBM."""

    @classmethod
    def distributed(cls, spec, nranks, rank, device_id, unique_id: bytes):
        """One slab per process (fc_create_dist); unique_id from nccl_unique_id() on rank 0."""
        self = cls.__new__(cls)
        self.spec, self.device_id, self.d = spec, device_id, spec.dim
        self.shape, self.total = tuple(spec.shape), spec.total
        self._h = ctypes.c_void_p()
        shape = np.array(spec.shape, dtype=np.int64)
        Y = np.array(spec.half_periods, dtype=np.float64)
        uid = ctypes.create_string_buffer(bytes(unique_id), 128)
        _check(lib().fc_create_dist(ctypes.byref(self._h), spec.dim, shape.ctypes.data_as(_i64p), _ptr(Y),
                                    nranks, rank, device_id, uid))
        self.slabs = ("dist", nranks, rank)
        self.isotropic = None
        return self

    def __init__(self, spec, device_id: int = 0, slabs=None):
        """``slabs``: None (one GPU) or a list of device ids, one per axis-0 slab
        (SURVEY 8(e)); repeating a device emulates several ranks on it."""
        self.spec = spec
        self.device_id = device_id
        self.d = spec.dim
        self.shape = tuple(spec.shape)
        self.total = spec.total
        self._h = ctypes.c_void_p()
        shape = np.array(spec.shape, dtype=np.int64)
        Y = np.array(spec.half_periods, dtype=np.float64)
        if slabs is None:
            _check(lib().fc_create(ctypes.byref(self._h), spec.dim, shape.ctypes.data_as(_i64p), _ptr(Y), device_id))
        else:
            dev = np.ascontiguousarray(slabs, dtype=np.int32)
            _check(lib().fc_create_sharded(ctypes.byref(self._h), spec.dim, shape.ctypes.data_as(_i64p), _ptr(Y),
                                           dev.size, dev.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))))
        self.slabs = slabs
        self.isotropic = None
        self.n_phases = 0

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value and _lib is not None:
            _lib.fc_destroy(h)
            self._h = ctypes.c_void_p()

    # -- coefficients ------------------------------------------------------
    def set_coefficients(self, a, compress=True):
        """Upload a CoefficientField.  A field built by ``CoefficientField.from_phases``
        goes up as labels + table (2 bytes per voxel); any other packed field is
        uploaded whole and, with ``compress``, deduplicated on the device
        (``compress_coefficients``).  ``n_phases`` = distinct tensors of the indexed
        form, 0 when the full field is resident."""
        self.n_phases = 0
        phases = getattr(a, "phases", None)
        if phases is not None and compress:
            self.set_coefficients_indexed(phases[0], phases[1])
            return
        if a.isotropic_values is not None:
            host = _c64(a.isotropic_values)
            kind = 0
        else:
            host = _c64(a.components)
            kind = 1
        _check(lib().fc_set_coefficients(self._h, kind, _ptr(host), host.size))
        self.isotropic = kind == 0
        if kind == 1 and compress and self.d >= 2:
            self.compress_coefficients()

    def set_coefficients_indexed(self, labels, table):
        """Piecewise-constant packed field as ``labels`` (uint16, grid shape) and
        ``table`` (``(d(d+1)/2, n_phases)`` packed tensors): voxel v holds
        ``table[:, labels[v]]``."""
        labels = np.ascontiguousarray(labels, dtype=np.uint16)
        table = _c64(table)
        nsym = self.d * (self.d + 1) // 2
        if table.ndim != 2 or table.shape[0] != nsym:
            raise ValueError(f"table shape {table.shape} != ({nsym}, n_phases)")
        _check(lib().fc_set_coefficients_indexed(self._h, table.shape[1], _ptr(table),
                                                 labels.ctypes.data_as(ctypes.POINTER(ctypes.c_uint16)), labels.size))
        self.isotropic = False
        self.n_phases = int(table.shape[1])

    def compress_coefficients(self, max_phases=MAX_PHASES, keep_packed=False):
        """Deduplicate the resident packed field on the device (exact, bitwise);
        returns the number of distinct tensors, 0 if the field stays as it is."""
        n = ctypes.c_int32(0)
        _check(lib().fc_compress_coefficients(self._h, int(max_phases), int(bool(keep_packed)), ctypes.byref(n)))
        self.n_phases = n.value
        return n.value

    def load_coefficients(self, bin_path, kind):
        """Stream a voxel payload (.bin) into HBM: kind 0 isotropic, 1 packed."""
        _check(lib().fc_load_coefficients(self._h, int(kind), os.fsencode(str(bin_path))))
        self.isotropic = kind == 0

    def plan_info(self, key):
        """What the plan selected: "two_field", "fold_fwd", "packed_fused", "n_phases", "slabs"."""
        v = ctypes.c_int32(0)
        _check(lib().fc_plan_info(self._h, key.encode(), ctypes.byref(v)))
        return v.value

    def coefficient_bounds(self):
        """(c_A, C_A, flat index of the first c_A voxel) of the device field."""
        lo, hi, at = ctypes.c_double(), ctypes.c_double(), ctypes.c_int64()
        _check(lib().fc_coefficient_bounds(self._h, ctypes.byref(lo), ctypes.byref(hi), ctypes.byref(at)))
        return lo.value, hi.value, at.value

    def save_solution(self, bin_path, nrhs=1):
        """Stream the last solve's solution (nrhs, d, *N) from HBM into a .bin payload."""
        _check(lib().fc_save_solution(self._h, int(nrhs), os.fsencode(str(bin_path))))

    def generate_voronoi(self, seeds, packed, want_labels=False, compress=True):
        """Device-side cfg4 polycrystal (replaces the coefficient field; kept in the
        phase-indexed form with ``compress``)."""
        seeds = _c64(seeds)
        packed = _c64(packed)
        labels = np.empty(self.shape, dtype=np.int32) if want_labels else None
        lp = labels.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)) if want_labels else None
        _check(lib().fc_generate_voronoi(self._h, seeds.shape[0], _ptr(seeds), _ptr(packed), lp))
        self.isotropic = False
        self.n_phases = 0
        if compress:
            self.compress_coefficients()
        return labels

    def spheres_stamp(self, centres, radius):
        """Mark the balls of integer ``centres`` ((n, 3)); returns covered voxels."""
        cen = np.ascontiguousarray(np.asarray(centres, dtype=np.int32).reshape(-1, 3))
        cov = ctypes.c_int64(0)
        _check(lib().fc_spheres_stamp(self._h, cen.shape[0], cen.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)),
                                      float(radius), ctypes.byref(cov)))
        return cov.value

    def spheres_finish(self, high, low):
        """Coverage bitmap -> isotropic coefficient field (high inside, low outside)."""
        _check(lib().fc_spheres_finish(self._h, float(high), float(low)))
        self.isotropic = True

    # -- batched field operators ------------------------------------------
    def _batched(self, fn, u, *extra):
        u = _c64(u)
        fshape = (self.d,) + self.shape
        single = u.shape == fshape
        ub = u.reshape((-1,) + fshape)
        out = np.empty_like(ub)
        for s in range(0, ub.shape[0], MAX_RHS):
            chunk = np.ascontiguousarray(ub[s:s + MAX_RHS])
            o = np.empty_like(chunk)
            _check(fn(self._h, *extra, _ptr(chunk), _ptr(o), chunk.shape[0]))
            out[s:s + MAX_RHS] = o
        return out.reshape(fshape) if single else out.reshape(u.shape)

    def apply_A(self, u):
        return self._batched(lib().fc_apply_A, u)

    def apply_system(self, u):
        return self._batched(lib().fc_apply_system, u)

    def project(self, which, ref_matrix, u):
        ref = None if ref_matrix is None else _c64(ref_matrix)
        if ref is not None and ref.shape != (self.d, self.d):
            raise ValueError(f"reference matrix must be {self.d} x {self.d}, got shape {ref.shape}")
        return self._batched(lib().fc_project, u, which, _ptr(ref))

    # -- solvers -----------------------------------------------------------
    def solve_cg(self, E, tol, max_iter, lam=None, init=None, want_x=True, record_iterates=False, out=None):
        E = _c64(np.atleast_2d(E))
        R = E.shape[0]
        fshape = (R, self.d) + self.shape
        if out is not None:
            if out.shape != fshape or out.dtype != np.float64 or not out.flags.c_contiguous:
                raise ValueError(f"out must be a C-contiguous float64 array of shape {fshape}")
            x = out
        else:
            x = np.empty(fshape) if want_x else None
        init = None if init is None else _c64(init).reshape(fshape)
        reps = (Report * R)()
        hist = np.zeros((R, max_iter + 1))
        its = None
        n_it = ctypes.c_int64(0)
        its_map = None
        if record_iterates:
            # room for max_iter + 1 iterates, but only the pages of the iterates
            # actually written get committed (anonymous MAP_NORESERVE mapping):
            # host memory scales with the iterations run, like the reference's list
            nbytes = (max_iter + 1) * int(np.prod(fshape)) * 8
            its_map = mmap.mmap(-1, nbytes, flags=mmap.MAP_PRIVATE | mmap.MAP_ANONYMOUS | getattr(mmap, "MAP_NORESERVE", 0x4000))
            its = np.frombuffer(its_map, dtype=np.float64).reshape((max_iter + 1,) + fshape)
        _check(lib().fc_solve_cg(
            self._h, R, _ptr(E), float(tol), int(max_iter), float(lam) if lam is not None else -1.0,
            _ptr(init), _ptr(x), reps, _ptr(hist), _ptr(its), 0 if its is None else its.shape[0],
            ctypes.byref(n_it)))
        out = []
        for r in range(R):
            rp = reps[r]
            out.append(dict(iterations=rp.iterations, converged=bool(rp.converged), status=rp.status,
                            detail=rp.detail, history=hist[r, :rp.hist_len].copy()))
        iterates = None if its is None else its[: n_it.value].copy()
        if its_map is not None:
            del its
            try:
                its_map.close()
            except BufferError:  # a view is still referenced: freed with it
                pass
        return out, x, iterates

    def solve_fixed_point(self, E, tol, max_iter, ref_matrix, scale, want_x=True):
        E = _c64(np.atleast_2d(E))
        R = E.shape[0]
        x = np.empty((R, self.d) + self.shape) if want_x else None
        reps = (Report * R)()
        hist = np.zeros((R, max_iter))
        sc = _c64(np.broadcast_to(np.asarray(scale, dtype=float), (R,)))
        _check(lib().fc_solve_fixed_point(self._h, R, _ptr(E), float(tol), int(max_iter), _ptr(_c64(ref_matrix)),
                                          _ptr(sc), _ptr(x), reps, _ptr(hist)))
        out = []
        for r in range(R):
            rp = reps[r]
            out.append(dict(iterations=rp.iterations, converged=bool(rp.converged), status=rp.status,
                            detail=rp.detail, history=hist[r, :rp.hist_len].copy()))
        return out, x

    def energy(self, E, x=None):
        """``M[a, b] = <A (E_a + x_a), E_b + x_b>`` over the batch (resident solution if x is None)."""
        E = _c64(np.atleast_2d(E))
        R = E.shape[0]
        out = np.empty((R, R))
        xx = None if x is None else _c64(x)
        _check(lib().fc_energy(self._h, R, _ptr(E), _ptr(xx), _ptr(out)))
        return out

    # -- instrumentation ---------------------------------------------------
    def set_profiling(self, on: bool):
        _check(lib().fc_set_profiling(self._h, 1 if on else 0))

    def profile(self):
        out = {}
        buf = ctypes.create_string_buffer(64)
        for i in range(lib().fc_profile_count(self._h)):
            n = ctypes.c_int64()
            ms = ctypes.c_double()
            _check(lib().fc_profile_get(self._h, i, buf, 64, ctypes.byref(n), ctypes.byref(ms)))
            out[buf.value.decode()] = (int(n.value), float(ms.value))
        return out

    def profile_reset(self):
        _check(lib().fc_profile_reset(self._h))

    def launch_count(self):
        return int(lib().fc_launch_count(self._h))

    def timer_mark(self, slot):
        _check(lib().fc_timer_mark(self._h, slot))

    def timer_elapsed(self, a, b):
        ms = ctypes.c_double()
        _check(lib().fc_timer_elapsed(self._h, a, b, ctypes.byref(ms)))
        return float(ms.value)


_spec_contexts: dict = {}


def context_for_spec(spec, device_id: int = 0) -> Context:
    """Coefficient-free context per (spec, device), for the bare projectors."""
    key = (spec, device_id)
    ctx = _spec_contexts.get(key)
    if ctx is None:
        if len(_spec_contexts) >= 16:
            _spec_contexts.pop(next(iter(_spec_contexts)))
        ctx = Context(spec, device_id)
        _spec_contexts[key] = ctx
    return ctx


def default_device() -> int:
    return int(os.environ.get("LOCAL_RANK", "0")) if device_count() > 1 else 0
