// Sweep, vector and reduction kernels of the GaNi operator / CG / fixed point.
//
// Operator application (reference solver.py:112-122,173-174,265-267):
//   y = M(x) u  (pointwise, M = s*A for CG, A - A0 for the fixed point)
//   -> forward FFT over all axes -> per-mode xi (xi . v) / den, 0 at k = 0
//   -> inverse FFT (1/|N|) -> epilogue.
// It is executed as 2d-1 sweeps over HBM (d = 2: 3 sweeps, d = 3: 5 sweeps):
//   row-forward  : pointwise M(x) u fused with a real->half-complex FFT of the
//                  contiguous axis (two real rows per complex FFT), written
//                  transposed so the next axis becomes contiguous;
//   mid-forward  : (d = 3) C2C along axis 1, written transposed (axis 0 contiguous);
//   outer        : C2C along axis 0, Gamma_hat multiply, inverse C2C, in place;
//   mid-inverse  : (d = 3) inverse of mid-forward;
//   row-inverse  : half-complex->real FFT of the contiguous axis fused with the
//                  CG / fixed-point epilogue and per-CTA dot partials.
// Spectral layouts (R right-hand sides, c = d components, h = (n_last+1)/2):
//   d = 3: W1[R][c][n0][h2][n1], W2[R][c][h2][n1][n0]
//   d = 2: W2[R][c][h1][n0]
// Dots are reduced deterministically: per-CTA partials in fixed slots (fixed
// intra-block tree), summed in fixed order by a single-CTA finalize kernel.
#pragma once
#include "fc_fft.cuh"

namespace fc {

constexpr int kThreads = 256;
constexpr int kMaxDim = 3;

// Input modes of the first sweep.
enum InMode : int {
  IN_FIELD = 0,   // y = s * A u
  IN_PNEW = 1,    // p' = r (first) | r + beta p ; store p'; y = s * A p'
  IN_CONST = 2,   // y = s * A E          (rhs = -op(E_N), E_N never materialised)
  IN_FP = 3,      // y = (A - A0) e
  IN_RAW = 4,     // y = s * u            (bare projector)
};
// Epilogues of the last sweep (g = inverse transform / |N| at the voxel).
enum EpMode : int {
  EP_STORE = 0,   // out = g
  EP_RHS = 1,     // out = -g ; partial sum out^2
  EP_AP = 2,      // out = g ; partial sum p g
  EP_FP = 3,      // e' = E - g ; partial sum (e' - e)^2 ; e = e'
};

struct RhsState {
  double rr, r0, pAp, alpha, beta, prev_update, scale, detail;
  int active, iterations, converged, status, growth, first, has_prev, hist_len;
};
enum Status : int { ST_OK = 0, ST_MAXITER = 1, ST_BREAKDOWN = 2, ST_DIVERGENT = 3 };

struct Geo {
  int dim;
  int n[3];       // shape (n[1], n[2] unused below dim)
  int64_t N;      // voxels
  double invN;
  const double* xi[3];  // xi[a][slot] = k(slot) / Y_a
};

// Slab decomposition along axis 0.  Each slab owns planes
// [s0[me], s0[me+1]) of axis 0 and, for the outer sweep, the (k2, k1) pencils
// q in [qs[me], qs[me+1]).  The middle sweep writes its spectrum in a
// destination-blocked layout so the block for slab p is one contiguous chunk:
//   send[doff[p] + ((r*c + a) * Q_p + (q - qs[p])) * n0l + i0_local]
// and the outer sweep reads full axis-0 pencils from the received segments:
//   recv[roff[p] + ((r*c + a) * Q_me + (q - qs[me])) * n0l(p) + (i0 - s0[p])].
// P = 1 reduces both to the single-GPU layout W2[R][c][q][i0].
constexpr int kMaxSlabs = 8;
struct SlabMap {
  int P, me, n0l;
  int s0[kMaxSlabs + 1];
  int qs[kMaxSlabs + 1];
  long long doff[kMaxSlabs];
  long long roff[kMaxSlabs];
  // Fused exchange (in-process slabs with peer access): the forward middle
  // sweep stores block t straight into slab t's receive buffer (fwd[t] = its
  // segment for this sender) and the outer sweep stores segment t straight
  // back into slab t's send buffer (ret[t]), over NVLink for slabs on other
  // GPUs; no copy pass, the transfer overlaps the sweep's arithmetic.
  int fused;
  double2* fwd[kMaxSlabs];
  double2* ret[kMaxSlabs];
};

__device__ __forceinline__ int slab_of(const int* bounds, int P, int x) {
  int p = 0;
#pragma unroll
  for (int t = 1; t < kMaxSlabs; ++t)
    if (t < P && x >= bounds[t]) p = t;
  return p;
}

__device__ __forceinline__ int64_t send_index(const SlabMap& m, int rc, int q, int i0l) {
  const int p = slab_of(m.qs, m.P, q);
  const int Qp = m.qs[p + 1] - m.qs[p];
  return m.doff[p] + ((int64_t)rc * Qp + (q - m.qs[p])) * m.n0l + i0l;
}
// Destination of a forward-middle-sweep store: the local send block, or (fused)
// the destination slab's receive segment for this sender.
__device__ __forceinline__ double2* send_dst(const SlabMap& m, double2* base, int rc, int q, int i0l) {
  const int p = slab_of(m.qs, m.P, q);
  const int Qp = m.qs[p + 1] - m.qs[p];
  const int64_t inner = ((int64_t)rc * Qp + (q - m.qs[p])) * m.n0l + i0l;
  return (m.fused ? m.fwd[p] : base + m.doff[p]) + inner;
}

struct Coef {
  const double* A;   // iso: (N) ; packed: (nsym, N); null while only the phase-indexed form is resident
  int kind;          // 0 isotropic scalar, 1 packed symmetric
  // phase-indexed form of a piecewise-constant packed field (kind 1): voxel v holds
  // tab[m * nph + lab[v]], bit for bit the packed value (fc_set_coefficients_indexed /
  // fc_compress_coefficients).  Read by coef() and the fused packed first sweep;
  // every other consumer takes the expanded field A.
  const uint16_t* lab = nullptr;
  const double* tab = nullptr;
  int nph = 0;
};

struct InArgs {
  int mode;
  double s;                   // CG reference scale lambda (1 otherwise)
  const double* u;            // IN_FIELD / IN_RAW source, IN_FP e, IN_PNEW r
  const double* p_old;        // IN_PNEW
  double* p_new;              // IN_PNEW
  double* xacc;               // IN_PNEW: deferred x += alpha p_old (null: k_cg_update updates x)
  double E[8][kMaxDim];       // per-RHS loads (IN_CONST / IN_FP uses A0 below)
  double A0[kMaxDim][kMaxDim];
};

// Finalize stages run by the last CTA of a reducing kernel (see finish_block).
enum FinMode : int {
  FIN_NONE = 0,
  FIN_INIT = 1,    // rhs norm: r0 (and history[0] / early exit unless a warm start follows)
  FIN_INIT2 = 2,   // warm start: r = rhs - op(x) norm, history[0], early exit
  FIN_ALPHA = 3,   // pAp, breakdown, alpha
  FIN_BETA = 4,    // rr_new, history, stop test, beta
  FIN_FP = 5,      // fixed point update norm, history, stop, divergence streak
};

struct FinArgs {
  int mode;
  int R;
  int nslot;
  double* part;       // [R][nslot]
  RhsState* st;
  double* hist;       // [R][hcap]
  int hcap;
  double tol;
  int max_iter;
  int window;         // fixed-point divergence window (solver.py:27)
  int with_init;      // FIN_INIT: a warm start follows
  double total;       // global voxel count |N| (inner products divide by it, solver.py:138-139)
  int* any_active;
  unsigned* counter;  // arrival counter, reset by the last CTA
  double* lsum;       // slab-local mode: per-RHS sums go here, k_fin_global finishes
};

struct EpArgs {
  int mode;
  double* out;                // EP_STORE/EP_RHS/EP_AP destination, EP_FP: e (in place)
  const double* p;            // EP_AP
  double E[8][kMaxDim];       // EP_FP
  double* part;               // partial sums [R][nslot]
  int nslot;
  FinArgs fin;
};

__device__ __forceinline__ int pidx(int d, int a, int b) {
  if (a == b) return a;
  if (a > b) { int t = a; a = b; b = t; }
  // (0,1),(0,2),(1,2) after the d diagonal entries (material.py:30-34)
  return d + (a == 0 ? b - 1 : (d - 1) + (b - 2));
}

__device__ __forceinline__ double coef(const Coef& C, int d, int a, int b, int64_t v, int64_t N) {
  if (C.kind == 0) return a == b ? C.A[v] : 0.0;
  if (C.lab != nullptr) return __ldg(C.tab + pidx(d, a, b) * C.nph + C.lab[v]);
  return C.A[(int64_t)pidx(d, a, b) * N + v];
}

__device__ __forceinline__ bool rhs_active(const RhsState* st, int r) {
  return st == nullptr || st[r].active;
}

// First-sweep input, prepared once per CTA (RHS scalars hoisted out of the
// voxel loop).  All reads go through the read-only path (__ldg): nothing the
// first sweep reads is written by it (p' goes to the other p buffer), so the
// loads of a thread can be issued back to back.
struct InEval {
  int mode, d, a;
  double s, beta, alpha;
  bool first;
  int64_t N, base;
  const double* u;
  const double* p_old;
  double* xacc;  // deferred x update of the previous iteration (IN_PNEW, not first)
  const double* A;
  int kind;
  double E0, E1, E2, Ea;  // load of this RHS (scalars: no local-memory arrays)
  double R0, R1, R2;      // row a of the reference tensor
  __device__ __forceinline__ static double sel(int b, double x0, double x1, double x2) {
    return b == 0 ? x0 : (b == 1 ? x1 : x2);
  }

  __device__ __forceinline__ double coefv(int b, int64_t v) const {
    if (kind == 0) return a == b ? __ldg(A + v) : 0.0;
    return __ldg(A + (int64_t)pidx(d, a, b) * N + v);
  }
  // value y_a(v); for IN_PNEW also p'_a(v) in .y (the caller stores it)
  __device__ __forceinline__ double2 operator()(int64_t v) const {
    double pn = 0.0;
    const double y = eval(v, pn);
    return make_double2(y, pn);
  }
  // compile-time specialisation (mode / coefficient kind hoisted out of voxel loops)
  template <int MODE, int KIND>
  __device__ __forceinline__ double eval_t(int64_t v, double& pn) const {
    if constexpr (MODE == IN_RAW) {
      const double x = __ldg(u + base + a * N + v);
      return s == 1.0 ? x : __dmul_rn(s, x);
    } else if constexpr (MODE == IN_FIELD || MODE == IN_CONST) {
      double acc = 0.0;
      if constexpr (KIND == 0) {
        const double x = MODE == IN_CONST ? Ea : __ldg(u + base + a * N + v);
        acc = __dmul_rn(__ldg(A + v), x);
      } else {
#pragma unroll
        for (int b = 0; b < kMaxDim; ++b) {
          if (b >= d) break;
          const double x = MODE == IN_CONST ? sel(b, E0, E1, E2) : __ldg(u + base + b * N + v);
          acc = __dadd_rn(acc, __dmul_rn(__ldg(A + (int64_t)pidx(d, a, b) * N + v), x));
        }
      }
      return s == 1.0 ? acc : __dmul_rn(s, acc);
    } else if constexpr (MODE == IN_PNEW) {
      double acc = 0.0;
      if constexpr (KIND == 0) {
        const int64_t e = base + a * N + v;
        const double x = __ldg(u + e);
        const double po = first ? 0.0 : __ldg(p_old + e);
        const double q = first ? x : __dadd_rn(x, __dmul_rn(beta, po));
        if (xacc) xacc[e] = __dadd_rn(xacc[e], __dmul_rn(alpha, po));
        pn = q;
        acc = __dmul_rn(__ldg(A + v), q);
      } else {
#pragma unroll
        for (int b = 0; b < kMaxDim; ++b) {
          if (b >= d) break;
          const int64_t e = base + b * N + v;
          const double x = __ldg(u + e);
          const double po = first ? 0.0 : __ldg(p_old + e);
          const double q = first ? x : __dadd_rn(x, __dmul_rn(beta, po));
          if (b == a) {
            pn = q;
            if (xacc) xacc[e] = __dadd_rn(xacc[e], __dmul_rn(alpha, po));
          }
          acc = __dadd_rn(acc, __dmul_rn(__ldg(A + (int64_t)pidx(d, a, b) * N + v), q));
        }
      }
      return s == 1.0 ? acc : __dmul_rn(s, acc);
    } else {
      double acc = 0.0;
#pragma unroll
      for (int b = 0; b < kMaxDim; ++b) {
        if (b >= d) break;
        const double A_ab = KIND == 0 ? (a == b ? __ldg(A + v) : 0.0) : __ldg(A + (int64_t)pidx(d, a, b) * N + v);
        const double cab = __dsub_rn(A_ab, sel(b, R0, R1, R2));
        acc = __dadd_rn(acc, __dmul_rn(cab, __ldg(u + base + b * N + v)));
      }
      return acc;
    }
  }

  __device__ __forceinline__ double eval(int64_t v, double& pn) const {
    switch (mode) {
      case IN_RAW: {
        const double x = __ldg(u + base + a * N + v);
        return s == 1.0 ? x : __dmul_rn(s, x);
      }
      case IN_FIELD:
      case IN_CONST: {
        double acc = 0.0;
        if (kind == 0) {
          const double x = mode == IN_CONST ? Ea : __ldg(u + base + a * N + v);
          acc = __dmul_rn(__ldg(A + v), x);
        } else {
#pragma unroll
          for (int b = 0; b < kMaxDim; ++b) {
            if (b >= d) break;
            const double x = mode == IN_CONST ? sel(b, E0, E1, E2) : __ldg(u + base + b * N + v);
            acc = __dadd_rn(acc, __dmul_rn(coefv(b, v), x));
          }
        }
        return s == 1.0 ? acc : __dmul_rn(s, acc);
      }
      case IN_PNEW: {
        double acc = 0.0;
        if (kind == 0) {
          const int64_t e = base + a * N + v;
          const double x = __ldg(u + e);
          const double po = first ? 0.0 : __ldg(p_old + e);
          const double q = first ? x : __dadd_rn(x, __dmul_rn(beta, po));
          if (xacc) xacc[e] = __dadd_rn(xacc[e], __dmul_rn(alpha, po));
          pn = q;
          acc = __dmul_rn(__ldg(A + v), q);
        } else {
#pragma unroll
          for (int b = 0; b < kMaxDim; ++b) {
            if (b >= d) break;
            const int64_t e = base + b * N + v;
            const double x = __ldg(u + e);
            const double po = first ? 0.0 : __ldg(p_old + e);
            const double q = first ? x : __dadd_rn(x, __dmul_rn(beta, po));
            if (b == a) {
              pn = q;
              if (xacc) xacc[e] = __dadd_rn(xacc[e], __dmul_rn(alpha, po));
            }
            acc = __dadd_rn(acc, __dmul_rn(coefv(b, v), q));
          }
        }
        return s == 1.0 ? acc : __dmul_rn(s, acc);
      }
      default: {  // IN_FP: contrast = A - A0 (solver.py:253-255)
        double acc = 0.0;
#pragma unroll
        for (int b = 0; b < kMaxDim; ++b) {
          if (b >= d) break;
          const double cab = __dsub_rn(coefv(b, v), sel(b, R0, R1, R2));
          acc = __dadd_rn(acc, __dmul_rn(cab, __ldg(u + base + b * N + v)));
        }
        return acc;
      }
    }
  }
};

// Static-index selection from a kernel-parameter table (dynamic indexing of
// parameters would force a local-memory copy of the whole argument block).
__device__ __forceinline__ double pick(const double (&T)[8][kMaxDim], int i, int j) {
  double v = 0.0;
#pragma unroll
  for (int x = 0; x < 8; ++x)
#pragma unroll
    for (int y = 0; y < kMaxDim; ++y)
      if (x == i && y == j) v = T[x][y];
  return v;
}
__device__ __forceinline__ double pick3(const double (&T)[kMaxDim][kMaxDim], int i, int j) {
  double v = 0.0;
#pragma unroll
  for (int x = 0; x < kMaxDim; ++x)
#pragma unroll
    for (int y = 0; y < kMaxDim; ++y)
      if (x == i && y == j) v = T[x][y];
  return v;
}

__device__ __forceinline__ InEval make_eval(const InArgs& ia, const Geo& g, const Coef& C, const RhsState* st,
                                            int r, int a) {
  InEval ev;
  ev.mode = ia.mode;
  ev.d = g.dim;
  ev.a = a;
  ev.s = ia.s;
  ev.N = g.N;
  ev.base = (int64_t)r * g.dim * g.N;
  ev.u = ia.u;
  ev.p_old = ia.p_old;
  ev.A = C.A;
  ev.kind = C.kind;
  ev.first = ia.mode == IN_PNEW ? st[r].first != 0 : true;
  ev.beta = ia.mode == IN_PNEW ? st[r].beta : 0.0;
  ev.xacc = (ia.mode == IN_PNEW && !ev.first) ? ia.xacc : nullptr;
  ev.alpha = ev.xacc != nullptr ? st[r].alpha : 0.0;
  // loads / reference rows only where the mode uses them (the static-index
  // selections cost ~100 instructions per thread)
  ev.E0 = ev.E1 = ev.E2 = ev.Ea = 0.0;
  ev.R0 = ev.R1 = ev.R2 = 0.0;
  if (ia.mode == IN_CONST) {
    ev.E0 = pick(ia.E, r, 0);
    ev.E1 = pick(ia.E, r, 1);
    ev.E2 = pick(ia.E, r, 2);
    ev.Ea = pick(ia.E, r, a);
  }
  if (ia.mode == IN_FP) {
    ev.R0 = pick3(ia.A0, a, 0);
    ev.R1 = pick3(ia.A0, a, 1);
    ev.R2 = pick3(ia.A0, a, 2);
  }
  return ev;
}

// Epilogue at voxel v; returns the contribution to the CTA's partial sum.
__device__ __forceinline__ double ep_apply(const EpArgs& ea, int d, int64_t N, int r, int a, int64_t v,
                                           double gval, double Ea) {
  const int64_t e = (int64_t)r * d * N + a * N + v;
  switch (ea.mode) {
    case EP_STORE: ea.out[e] = gval; return 0.0;
    case EP_RHS: { double o = -gval; ea.out[e] = o; return __dmul_rn(o, o); }
    case EP_AP: ea.out[e] = gval; return __dmul_rn(ea.p[e], gval);
    default: {
      double en = __dsub_rn(Ea, gval);
      double df = __dsub_rn(en, ea.out[e]);
      ea.out[e] = en;
      return __dmul_rn(df, df);
    }
  }
}

// Epilogue with the input already loaded (q = p for EP_AP, old e for EP_FP).
__device__ __forceinline__ double ep_store(const EpArgs& ea, int64_t e, double gval, double Ea, double q) {
  switch (ea.mode) {
    case EP_STORE: ea.out[e] = gval; return 0.0;
    case EP_RHS: { double o = -gval; ea.out[e] = o; return __dmul_rn(o, o); }
    case EP_AP: ea.out[e] = gval; return __dmul_rn(q, gval);
    default: {
      const double en = __dsub_rn(Ea, gval);
      const double df = __dsub_rn(en, q);
      ea.out[e] = en;
      return __dmul_rn(df, df);
    }
  }
}

// Same epilogue, value returned in o instead of stored (the caller stores it).
template <int MODE>
__device__ __forceinline__ double ep_value_t(double gval, double Ea, double q, double& o) {
  if constexpr (MODE == EP_STORE) {
    o = gval;
    return 0.0;
  } else if constexpr (MODE == EP_RHS) {
    o = -gval;
    return __dmul_rn(o, o);
  } else if constexpr (MODE == EP_AP) {
    o = gval;
    return __dmul_rn(q, gval);
  } else {
    o = __dsub_rn(Ea, gval);
    const double df = __dsub_rn(o, q);
    return __dmul_rn(df, df);
  }
}

template <int MODE>
__device__ __forceinline__ double ep_store_t(double* __restrict__ out, int64_t e, double gval, double Ea, double q) {
  if constexpr (MODE == EP_STORE) {
    out[e] = gval;
    return 0.0;
  } else if constexpr (MODE == EP_RHS) {
    const double o = -gval;
    out[e] = o;
    return __dmul_rn(o, o);
  } else if constexpr (MODE == EP_AP) {
    out[e] = gval;
    return __dmul_rn(q, gval);
  } else {
    const double en = __dsub_rn(Ea, gval);
    const double df = __dsub_rn(en, q);
    out[e] = en;
    return __dmul_rn(df, df);
  }
}

// Run f(integral_constant<MODE>, integral_constant<KIND>) with runtime values
// lifted to compile time (the switch sits outside every voxel loop).
template <int V>
struct IC {
  static constexpr int value = V;
};
template <typename F>
__device__ __forceinline__ void with_in_mode(int mode, int kind, F&& f) {
  if (kind == 0) {
    switch (mode) {
      case IN_FIELD: f(IC<IN_FIELD>{}, IC<0>{}); break;
      case IN_PNEW: f(IC<IN_PNEW>{}, IC<0>{}); break;
      case IN_CONST: f(IC<IN_CONST>{}, IC<0>{}); break;
      case IN_FP: f(IC<IN_FP>{}, IC<0>{}); break;
      default: f(IC<IN_RAW>{}, IC<0>{}); break;
    }
  } else {
    switch (mode) {
      case IN_FIELD: f(IC<IN_FIELD>{}, IC<1>{}); break;
      case IN_PNEW: f(IC<IN_PNEW>{}, IC<1>{}); break;
      case IN_CONST: f(IC<IN_CONST>{}, IC<1>{}); break;
      case IN_FP: f(IC<IN_FP>{}, IC<1>{}); break;
      default: f(IC<IN_RAW>{}, IC<1>{}); break;
    }
  }
}
template <typename F>
__device__ __forceinline__ void with_ep_mode(int mode, F&& f) {
  switch (mode) {
    case EP_STORE: f(IC<EP_STORE>{}); break;
    case EP_RHS: f(IC<EP_RHS>{}); break;
    case EP_AP: f(IC<EP_AP>{}); break;
    default: f(IC<EP_FP>{}); break;
  }
}

// Warp sum over the lanes that exist (the last warp of a 243-thread CTA is
// partial; absent partners contribute nothing).  Fixed xor tree: deterministic.
__device__ __forceinline__ double warp_sum(double v) {
  const int lane = threadIdx.x & 31;
  const int base = threadIdx.x & ~31;
  const int nact = min(32, (int)blockDim.x - base);
  const unsigned mask = nact == 32 ? 0xffffffffu : ((1u << nact) - 1u);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double other = __shfl_xor_sync(mask, v, o);
    if ((lane ^ o) < nact) v += other;
  }
  return v;
}

// Deterministic block sum (fixed shuffle tree + fixed cross-warp order).
__device__ __forceinline__ double block_sum(double v, double* red) {
  v = warp_sum(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x == 0) {
    const int nw = (blockDim.x + 31) >> 5;
    for (int i = 0; i < nw; ++i) s += red[i];
  }
  return s;  // valid in thread 0
}

// Sum of n partial slots in a fixed order (thread-strided, then the fixed
// block tree); L1 is bypassed because other CTAs wrote the slots.
__device__ double reduce_slots(const double* part, int n, double* red) {
  double acc = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) acc += __ldcg(part + i);
  return block_sum(acc, red);  // thread 0
}

// Scalar CG / fixed-point logic for RHS r given the reduced sum q = sum / |N|
// (thread 0 only).  Mirrors solver.py:176-225 and solver.py:264-291.
__device__ void fin_logic(const FinArgs& f, int r, double sum) {
  RhsState& S = f.st[r];
  const double q = __ddiv_rn(sum, f.total);  // float(np.sum(x*y) / total), solver.py:138-139
  switch (f.mode) {
    case FIN_INIT:
    case FIN_INIT2: {
      if (f.mode == FIN_INIT) {
        S.r0 = sqrt(q);
        S.rr = q;
        if (f.with_init) return;
      } else {
        S.rr = q;
      }
      const double h0 = sqrt(S.rr);
      f.hist[(int64_t)r * f.hcap] = h0;
      S.hist_len = 1;
      S.iterations = 0;
      S.first = 1;
      S.status = ST_OK;
      S.beta = 0.0;
      const bool done = S.r0 == 0.0 || h0 <= f.tol * S.r0;  // solver.py:190-194
      S.active = done ? 0 : 1;
      S.converged = done ? 1 : 0;
      return;
    }
    case FIN_ALPHA: {
      S.pAp = q;
      if (q <= 0.0) {  // solver.py:203-212
        S.active = 0;
        S.converged = 0;
        S.status = ST_BREAKDOWN;
        S.detail = q;
      } else {
        S.alpha = S.rr / q;
      }
      return;
    }
    case FIN_BETA: {
      S.iterations += 1;
      const double h = sqrt(q);
      f.hist[(int64_t)r * f.hcap + S.iterations] = h;
      S.hist_len = S.iterations + 1;
      if (h <= f.tol * S.r0) {
        S.converged = 1;
        S.active = 0;
      } else {
        S.beta = q / S.rr;
        S.rr = q;
        S.first = 0;
        if (S.iterations >= f.max_iter) {
          S.active = 0;
          S.status = ST_MAXITER;
        }
      }
      return;
    }
    case FIN_FP: {
      const double update = sqrt(q);
      f.hist[(int64_t)r * f.hcap + S.iterations] = update;
      S.iterations += 1;
      S.hist_len = S.iterations;
      if (update <= f.tol * S.scale) {
        S.converged = 1;
        S.active = 0;
        return;
      }
      if (S.has_prev && update > S.prev_update) {
        S.growth += 1;
        if (S.growth >= f.window) {
          S.active = 0;
          S.status = ST_DIVERGENT;
          return;
        }
      } else {
        S.growth = 0;
      }
      S.prev_update = update;
      S.has_prev = 1;
      if (S.iterations >= f.max_iter) {
        S.active = 0;
        S.status = ST_MAXITER;
      }
      return;
    }
    default:
      return;
  }
}

// Arrival of one CTA of a reducing kernel.  Thread 0 must already have stored
// this CTA's partial.  The last CTA to arrive sums every RHS's slots in fixed
// order and runs the finalize stage, so no separate finalize launch is needed.
// Every CTA of the launch must call it exactly once (inactive RHS included).
// Arrival half of finish_block: returns (uniformly) whether this CTA is the
// last one; no barrier for FIN_NONE.
__device__ bool arrive_block(const FinArgs& f) {
  if (f.mode == FIN_NONE) return false;
  __shared__ int last;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned total = gridDim.x * gridDim.y * gridDim.z;
    const unsigned prev = atomicAdd(f.counter, 1u);
    last = prev == total - 1;
  }
  __syncthreads();
  return last != 0;
}

__device__ void finalize_block(const FinArgs& f, double* red);

__device__ void finish_block(const FinArgs& f, double* red) {
  if (arrive_block(f)) finalize_block(f, red);
}

// Finalize half: the last CTA sums every RHS's slots and runs the scalar logic.
__device__ void finalize_block(const FinArgs& f, double* red) {
  __threadfence();
  const bool init = f.mode == FIN_INIT || f.mode == FIN_INIT2;
  for (int r = 0; r < f.R; ++r) {
    if (!init && !f.st[r].active) continue;
    const double sum = reduce_slots(f.part + (int64_t)r * f.nslot, f.nslot, red);
    if (threadIdx.x == 0) {
      if (f.lsum) f.lsum[r] = sum;  // slab-local: the global finalize runs in k_fin_global
      else fin_logic(f, r, sum);
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    if (!f.lsum) {
      int any = 0;
      for (int r = 0; r < f.R; ++r) any |= f.st[r].active;
      *f.any_active = any;
    }
    *f.counter = 0u;
  }
}

// Sharded finalize: every slab sums the P slab-local sums in slab order (so all
// slabs hold bit-identical scalars) and runs the same scalar logic.
struct SlabSums {
  const double* p[kMaxSlabs];
  int P;
};
__global__ void k_fin_global(FinArgs f, SlabSums ss) {
  if (threadIdx.x != 0) return;
  const bool init = f.mode == FIN_INIT || f.mode == FIN_INIT2;
  for (int r = 0; r < f.R; ++r) {
    if (!init && !f.st[r].active) continue;
    double sum = 0.0;
    for (int q = 0; q < ss.P; ++q) sum += ss.p[q][r];
    fin_logic(f, r, sum);
  }
  int any = 0;
  for (int r = 0; r < f.R; ++r) any |= f.st[r].active;
  *f.any_active = any;
}

// Split finalize for large grids: the reducing kernel only stores its partials
// (FIN_NONE: no per-CTA fence + atomic round trip while the CTA holds its
// shared memory), then this launch sums them in a fixed two-level order -- G
// chunks per right-hand side, each by one CTA (thread-strided, four
// accumulators, the fixed block tree), the chunk sums in chunk order by the
// last CTA to arrive -- and runs the same scalar logic as finalize_block.
__device__ __forceinline__ double fin_chunk_sum(const double* p, int64_t i0, int64_t i1, double* red) {
  double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
  int64_t i = i0 + threadIdx.x;
  for (; i + 768 < i1; i += 1024) {
    a0 += __ldcg(p + i);
    a1 += __ldcg(p + i + 256);
    a2 += __ldcg(p + i + 512);
    a3 += __ldcg(p + i + 768);
  }
  for (; i < i1; i += 256) a0 += __ldcg(p + i);
  return block_sum((a0 + a1) + (a2 + a3), red);  // thread 0
}

__global__ void __launch_bounds__(1024) k_fin_split(FinArgs f, double* part2, int G) {
  __shared__ double red[256 / 32];
  __shared__ int last;
  const bool init = f.mode == FIN_INIT || f.mode == FIN_INIT2;
  if (G == 1) {
    // few partials: one CTA, a group of 256 threads per right-hand side (up to four
    // side by side), no second level, no arrival.  Same sums in the same order as a
    // 256-thread block_sum of the chunk.
    __shared__ double gred[4][8];
    const int grp = threadIdx.x >> 8, ngrp = blockDim.x >> 8, tl = threadIdx.x & 255;
    for (int q = grp; q < f.R; q += ngrp) {
      if (!init && !f.st[q].active) continue;
      const double* p = f.part + (int64_t)q * f.nslot;
      double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
      int64_t i = tl;
      for (; i + 768 < f.nslot; i += 1024) {
        a0 += __ldcg(p + i);
        a1 += __ldcg(p + i + 256);
        a2 += __ldcg(p + i + 512);
        a3 += __ldcg(p + i + 768);
      }
      for (; i < f.nslot; i += 256) a0 += __ldcg(p + i);
      const double w = warp_sum((a0 + a1) + (a2 + a3));
      asm volatile("bar.sync %0, 256;\n" ::"r"(1 + grp) : "memory");
      if ((tl & 31) == 0) gred[grp][tl >> 5] = w;
      asm volatile("bar.sync %0, 256;\n" ::"r"(1 + grp) : "memory");
      if (tl == 0) {
        double sum = 0.0;
        for (int k = 0; k < 8; ++k) sum += gred[grp][k];
        if (f.lsum) f.lsum[q] = sum;
        else fin_logic(f, q, sum);
      }
    }
    __syncthreads();
    if (threadIdx.x == 0 && !f.lsum) {
      int any = 0;
      for (int q = 0; q < f.R; ++q) any |= f.st[q].active;
      *f.any_active = any;
    }
    return;
  }
  const int r = blockIdx.y, gi = blockIdx.x;
  if (init || f.st[r].active) {
    const int64_t chunk = ((int64_t)f.nslot + G - 1) / G;
    const int64_t i0 = gi * chunk, i1 = min((int64_t)f.nslot, i0 + chunk);
    const double sum = fin_chunk_sum(f.part + (int64_t)r * f.nslot, i0, i1, red);
    if (threadIdx.x == 0) part2[r * G + gi] = sum;
  }
  if (threadIdx.x == 0) {
    __threadfence();
    last = atomicAdd(f.counter, 1u) == gridDim.x * gridDim.y - 1;
  }
  __syncthreads();
  if (!last || threadIdx.x != 0) return;
  __threadfence();
  for (int q = 0; q < f.R; ++q) {
    if (!init && !f.st[q].active) continue;
    double sum = 0.0;
    for (int t = 0; t < G; ++t) sum += __ldcg(part2 + q * G + t);
    if (f.lsum) f.lsum[q] = sum;  // slab-local: the global finalize runs in k_fin_global
    else fin_logic(f, q, sum);
  }
  if (!f.lsum) {
    int any = 0;
    for (int q = 0; q < f.R; ++q) any |= f.st[q].active;
    *f.any_active = any;
  }
  *f.counter = 0u;
}

// Row-sweep geometry: rows of length nl along the contiguous axis, grouped in
// blocks of B consecutive rows of the previous axis (length np), for each
// outer index o < no (d = 3: o = i0; d = 2: no = 1).
struct RowGeo {
  int nl, hl, np, no, B, ntiles;
  int tma = 0;      // transposed spectrum moved by TMA boxes {2B doubles, boxK modes} (fc_tma.cuh)
  int boxK = 0, nbox = 0;
  int qoff = 0;     // last sweep: byte offset of the epilogue-input staging area (0: per-thread loads after the FFT)
};

// ---------------------------------------------------------------------------
// First sweep: pointwise M(x) u, R2C along the contiguous axis, transposed store.
__global__ void __launch_bounds__(kThreads) k_row_fwd(Geo g, RowGeo rg, Coef C, InArgs ia, const RhsState* st,
                                                       FftPlan pl, double2* __restrict__ W) {
  extern __shared__ double2 sm[];
  const int c = g.dim;
  int64_t bid = blockIdx.x;
  const int a = bid % c; bid /= c;
  const int tile = bid % rg.ntiles; bid /= rg.ntiles;
  const int o = bid % rg.no;
  const int r = (int)(bid / rg.no);
  if (!rhs_active(st, r)) return;
  const InEval ev = make_eval(ia, g, C, st, r, a);
  const int row0 = tile * rg.B;
  const int nrows = min(rg.B, rg.np - row0);
  const int npairs = (nrows + 1) >> 1;
  const int ld = rg.nl;
  double2* buf0 = sm;
  double2* buf1 = sm + (size_t)npairs * ld;
  // load: two real rows per complex pencil
  for (int idx = threadIdx.x; idx < npairs * 2 * rg.nl; idx += blockDim.x) {
    const int row = idx / rg.nl, i = idx - row * rg.nl;
    double val = 0.0;
    if (row < nrows) {
      const int64_t v = ((int64_t)o * rg.np + row0 + row) * rg.nl + i;
      double pn = 0.0;
      val = ev.eval(v, pn);
      if (ev.mode == IN_PNEW) ia.p_new[ev.base + a * g.N + v] = pn;
    }
    double* dst = reinterpret_cast<double*>(buf0 + (size_t)(row >> 1) * ld + i);
    dst[row & 1] = val;
  }
  __syncthreads();
  double2* res = smem_fft<false>(buf0, buf1, npairs, ld, pl);
  // separate Z = Ya + i Yb and store Y(k), k < hl, transposed (rows contiguous)
  double2* Wb = W + ((int64_t)(r * c + a) * rg.no + o) * rg.hl * rg.np + row0;
  for (int idx = threadIdx.x; idx < rg.hl * nrows; idx += blockDim.x) {
    const int k = idx / nrows, row = idx - k * nrows;
    const double2* z = res + (size_t)(row >> 1) * ld;
    const double2 zk = z[k];
    const double2 zm = z[k == 0 ? 0 : rg.nl - k];  // conj taken below
    double2 y;
    if ((row & 1) == 0) y = make_double2(0.5 * (zk.x + zm.x), 0.5 * (zk.y - zm.y));
    else y = make_double2(0.5 * (zk.y + zm.y), 0.5 * (zm.x - zk.x));
    Wb[(int64_t)k * rg.np + row] = y;
  }
}

// Last sweep: transposed load, C2R along the contiguous axis, epilogue.
__global__ void __launch_bounds__(kThreads) k_row_inv(Geo g, RowGeo rg, EpArgs ea, const RhsState* st,
                                                       FftPlan pl, const double2* __restrict__ W) {
  extern __shared__ double2 sm[];
  __shared__ double red[kThreads / 32];
  const int c = g.dim;
  int64_t bid = blockIdx.x;
  const int a = bid % c; bid /= c;
  const int tile = bid % rg.ntiles; bid /= rg.ntiles;
  const int o = bid % rg.no;
  const int r = (int)(bid / rg.no);
  if (!rhs_active(st, r)) {
    finish_block(ea.fin, red);
    return;
  }
  const int row0 = tile * rg.B;
  const int nrows = min(rg.B, rg.np - row0);
  const int npairs = (nrows + 1) >> 1;
  const int ld = rg.nl;
  double2* buf0 = sm;
  double2* buf1 = sm + (size_t)npairs * ld;
  const double2* Wb = W + ((int64_t)(r * c + a) * rg.no + o) * rg.hl * rg.np + row0;
  // Z(k) = Ye(k) + i Yo(k), Z(n-k) = conj(Ye(k)) + i conj(Yo(k)); k = 0 uses real parts.
  for (int idx = threadIdx.x; idx < rg.hl * npairs; idx += blockDim.x) {
    const int k = idx / npairs, pr = idx - k * npairs;
    const int re = 2 * pr, ro = 2 * pr + 1;
    double2 ye = Wb[(int64_t)k * rg.np + re];
    double2 yo = ro < nrows ? Wb[(int64_t)k * rg.np + ro] : make_double2(0.0, 0.0);
    double2* z = buf0 + (size_t)pr * ld;
    if (k == 0) {
      z[0] = make_double2(ye.x, yo.x);
    } else {
      z[k] = make_double2(ye.x - yo.y, ye.y + yo.x);
      z[rg.nl - k] = make_double2(ye.x + yo.y, yo.x - ye.y);
    }
  }
  __syncthreads();
  double2* res = smem_fft<true>(buf0, buf1, npairs, ld, pl);
  const double Ea = pick(ea.E, r, a);
  double acc = 0.0;
  for (int idx = threadIdx.x; idx < nrows * rg.nl; idx += blockDim.x) {
    const int row = idx / rg.nl, i = idx - row * rg.nl;
    const double2 z = res[(size_t)(row >> 1) * ld + i];
    const double gv = ((row & 1) ? z.y : z.x) * g.invN;
    const int64_t v = ((int64_t)o * rg.np + row0 + row) * rg.nl + i;
    acc += ep_apply(ea, c, g.N, r, a, v, gv, Ea);
  }
  if (ea.part != nullptr) {
    double s = block_sum(acc, red);
    if (threadIdx.x == 0) {
      const int slot = (o * rg.ntiles + tile) * c + a;
      ea.part[(int64_t)r * ea.nslot + slot] = s;
    }
  }
  finish_block(ea.fin, red);
}

// Middle sweep (d = 3): W1[r][a][i0][k2][i1] <-> W2[r][a][k2][k1][i0].
struct MidGeo {
  int n0, n1, h2, B, nib;
  int tma = 0;          // single slab: bulk pencil copies + TMA boxes on the transposed side
  int rows = 0, nbox = 0;  // box {2B doubles, rows modes}, nbox boxes per CTA
  int rebuild = 0;         // inverse sweep: components 1, 2 = xi1 t, xi2 t from t in component 1's planes
  int regA = 0;            // forward fold: elements of the first shared-memory region (pencils / boxes)
};

template <bool INV>
__global__ void __launch_bounds__(kThreads) k_mid(Geo g, MidGeo mg, SlabMap sm_, const RhsState* st, FftPlan pl,
                                                   const double2* __restrict__ src, double2* __restrict__ dst) {
  extern __shared__ double2 sm[];
  const int c = g.dim;
  int64_t bid = blockIdx.x;
  const int ib = bid % mg.nib; bid /= mg.nib;
  const int k2 = bid % mg.h2; bid /= mg.h2;
  const int a = bid % c;
  const int r = (int)(bid / c);
  if (!rhs_active(st, r)) return;
  const int i00 = ib * mg.B;
  const int nr = min(mg.B, mg.n0 - i00);
  const int ld = mg.n1;
  double2* buf0 = sm;
  double2* buf1 = sm + (size_t)nr * ld;
  const int64_t rc = (int64_t)(r * c + a);
  // W1 offset of (i0, k2, i1): ((rc*n0 + i0)*h2 + k2)*n1 + i1
  // W2 offset of (k2, k1, i0): send_index(rc, k2*n1 + k1, i0) (= ((rc*h2 + k2)*n1 + k1)*n0 + i0
  // for one slab; destination-blocked for P slabs, SlabMap)
  if (!INV) {
    for (int idx = threadIdx.x; idx < nr * mg.n1; idx += blockDim.x) {
      const int row = idx / mg.n1, i1 = idx - row * mg.n1;
      buf0[(size_t)row * ld + i1] = src[((rc * mg.n0 + i00 + row) * mg.h2 + k2) * mg.n1 + i1];
    }
  } else {
    for (int idx = threadIdx.x; idx < nr * mg.n1; idx += blockDim.x) {
      const int k1 = idx / nr, row = idx - k1 * nr;
      buf0[(size_t)row * ld + k1] = src[send_index(sm_, (int)rc, k2 * mg.n1 + k1, i00 + row)];
    }
  }
  __syncthreads();
  double2* res = smem_fft<INV>(buf0, buf1, nr, ld, pl);
  if (!INV) {
    for (int idx = threadIdx.x; idx < nr * mg.n1; idx += blockDim.x) {
      const int k1 = idx / nr, row = idx - k1 * nr;
      *send_dst(sm_, dst, (int)rc, k2 * mg.n1 + k1, i00 + row) = res[(size_t)row * ld + k1];
    }
    if (sm_.fused) __threadfence_system();  // peer stores ordered before the exit
  } else {
    for (int idx = threadIdx.x; idx < nr * mg.n1; idx += blockDim.x) {
      const int row = idx / mg.n1, i1 = idx - row * mg.n1;
      dst[((rc * mg.n0 + i00 + row) * mg.h2 + k2) * mg.n1 + i1] = res[(size_t)row * ld + i1];
    }
  }
}

// Outer sweep: C2C along axis 0, Gamma_hat, inverse, in place on W2.
// Gamma_hat(k) v = xi (xi . v) / den, den = |xi|^2 (orth) or xi^T M xi; 0 at k = 0
// (solver.py:98-110, green.py:81-92).
struct OuterGeo {
  int n0, Q, QB, nqb;   // Q pencils per component, QB per CTA
  int tma = 0;          // single slab: bulk (TMA) pencil loads / stores in k_outer_r
  int R;                // right-hand sides (persistent kernel tiles over R x nqb)
  int n1, h_last;       // d = 3: q = k2 * n1 + k1 ; d = 2: q = k1
  int orth;
  double M[kMaxDim][kMaxDim];
};

// Element (a, local pencil ql, i0) of the outer sweep's input: the received
// segment of the slab owning plane i0 (P = 1: W2[r][a][ql][i0]).
__device__ __forceinline__ int64_t outer_index(const SlabMap& m, int Q, int rc, int ql, int i0) {
  const int p = slab_of(m.s0, m.P, i0);
  const int n0p = m.s0[p + 1] - m.s0[p];
  return m.roff[p] + ((int64_t)rc * Q + ql) * n0p + (i0 - m.s0[p]);
}
// Destination of an outer-sweep result: in place, or (fused) the owning slab's
// send block for this slab.
__device__ __forceinline__ double2* outer_dst(const SlabMap& m, double2* W, int Q, int rc, int ql, int i0) {
  if (!m.fused) return W + outer_index(m, Q, rc, ql, i0);
  const int p = slab_of(m.s0, m.P, i0);
  const int n0p = m.s0[p + 1] - m.s0[p];
  return m.ret[p] + ((int64_t)rc * Q + ql) * n0p + (i0 - m.s0[p]);
}

__global__ void __launch_bounds__(kThreads) k_outer(Geo g, OuterGeo og, SlabMap sm_, const RhsState* st, FftPlan pl,
                                                     double2* __restrict__ W) {
  extern __shared__ double2 sm[];
  const int c = g.dim;
  const int qb = blockIdx.x % og.nqb;
  const int r = blockIdx.x / og.nqb;
  if (!rhs_active(st, r)) return;
  const int q0 = qb * og.QB;
  const int nq = min(og.QB, og.Q - q0);
  const int P = c * nq;
  const int ld = og.n0;
  double2* buf0 = sm;
  double2* buf1 = sm + (size_t)P * ld;
  for (int a = 0; a < c; ++a) {
    double2* d = buf0 + (size_t)a * nq * ld;
    for (int idx = threadIdx.x; idx < nq * og.n0; idx += blockDim.x) {
      const int qq = idx / og.n0, i0 = idx - qq * og.n0;
      d[idx] = W[outer_index(sm_, og.Q, r * c + a, q0 + qq, i0)];
    }
  }
  __syncthreads();
  double2* res = smem_fft<false>(buf0, buf1, P, ld, pl);
  double2* other = res == buf0 ? buf1 : buf0;
  for (int idx = threadIdx.x; idx < nq * og.n0; idx += blockDim.x) {
    const int qq = idx / og.n0, i0 = idx - qq * og.n0;
    const int q = sm_.qs[sm_.me] + q0 + qq;  // global (k2, k1) pencil index
    double xi[kMaxDim];
    xi[0] = g.xi[0][i0];
    bool zero_mode = (i0 == 0);
    if (c == 2) {
      xi[1] = g.xi[1][q];
      zero_mode = zero_mode && q == 0;
    } else if (c == 3) {
      const int k2 = q / og.n1, k1 = q - k2 * og.n1;
      xi[1] = g.xi[1][k1];
      xi[2] = g.xi[2][k2];
      zero_mode = zero_mode && q == 0;
    }
    double2 v[kMaxDim];
    for (int a = 0; a < c; ++a) v[a] = res[((size_t)a * nq + qq) * ld + i0];
    double2 out[kMaxDim];
    if (zero_mode) {
      for (int a = 0; a < c; ++a) out[a] = make_double2(0.0, 0.0);
    } else {
      double2 dots = make_double2(0.0, 0.0);
      double den = 0.0;
      for (int a = 0; a < c; ++a) {
        dots.x += xi[a] * v[a].x;
        dots.y += xi[a] * v[a].y;
      }
      if (og.orth) {
        for (int a = 0; a < c; ++a) den += xi[a] * xi[a];
      } else {
        for (int a = 0; a < c; ++a)
          for (int b = 0; b < c; ++b) den += xi[a] * og.M[a][b] * xi[b];
      }
      const double2 qv = make_double2(dots.x / den, dots.y / den);
      for (int a = 0; a < c; ++a) out[a] = make_double2(xi[a] * qv.x, xi[a] * qv.y);
    }
    for (int a = 0; a < c; ++a) other[((size_t)a * nq + qq) * ld + i0] = out[a];
  }
  __syncthreads();
  double2* res2 = smem_fft<true>(other, res, P, ld, pl);
  for (int a = 0; a < c; ++a) {
    const double2* s = res2 + (size_t)a * nq * ld;
    for (int idx = threadIdx.x; idx < nq * og.n0; idx += blockDim.x) {
      const int qq = idx / og.n0, i0 = idx - qq * og.n0;
      *outer_dst(sm_, W, og.Q, r * c + a, q0 + qq, i0) = s[idx];
    }
  }
  if (sm_.fused) __threadfence_system();
}

// d = 1: the whole line in one CTA per RHS (full complex FFT, no pairing).
__global__ void __launch_bounds__(kThreads) k_line(Geo g, Coef C, InArgs ia, EpArgs ea, const RhsState* st,
                                                    FftPlan pl, int orth, double M00) {
  extern __shared__ double2 sm[];
  __shared__ double red[kThreads / 32];
  const int r = blockIdx.x;
  if (!rhs_active(st, r)) {
    finish_block(ea.fin, red);
    return;
  }
  const InEval ev = make_eval(ia, g, C, st, r, 0);
  const int n = g.n[0];
  double2* buf0 = sm;
  double2* buf1 = sm + n;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    double pn = 0.0;
    buf0[i] = make_double2(ev.eval(i, pn), 0.0);
    if (ev.mode == IN_PNEW) ia.p_new[ev.base + i] = pn;
  }
  __syncthreads();
  double2* res = smem_fft<false>(buf0, buf1, 1, n, pl);
  double2* other = res == buf0 ? buf1 : buf0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    if (i == 0) { other[0] = make_double2(0.0, 0.0); continue; }
    const double xi = g.xi[0][i];
    const double den = orth ? xi * xi : xi * M00 * xi;
    const double2 v = res[i];
    const double2 qv = make_double2((xi * v.x) / den, (xi * v.y) / den);
    other[i] = make_double2(xi * qv.x, xi * qv.y);
  }
  __syncthreads();
  double2* res2 = smem_fft<true>(other, res, 1, n, pl);
  double acc = 0.0;
  const double Ea = pick(ea.E, r, 0);
  for (int i = threadIdx.x; i < n; i += blockDim.x) acc += ep_apply(ea, 1, g.N, r, 0, i, res2[i].x * g.invN, Ea);
  if (ea.part != nullptr) {
    double s = block_sum(acc, red);
    if (threadIdx.x == 0) ea.part[(int64_t)r * ea.nslot] = s;
  }
  finish_block(ea.fin, red);
}

// ---------------------------------------------------------------------------
// Elementwise kernels over one RHS block of c*N values; fixed tiling so the
// partial-sum slots do not depend on scheduling.
constexpr int kVecTile = kThreads * 16;

// x += alpha p ; r -= alpha Ap ; partial <r, r>     (solver.py:213-216)
// 16-byte vector accesses when the per-RHS block length is even; the last
// CTA runs the beta / stop-test finalize (FIN_BETA).
__global__ void __launch_bounds__(kThreads) k_cg_update(int64_t len, RhsState* st, double* __restrict__ x,
                                                        double* __restrict__ rr, const double* __restrict__ p,
                                                        const double* __restrict__ Ap, double* part, int nslot,
                                                        FinArgs fin) {
  __shared__ double red[kThreads / 32];
  // tiles run in reverse order: the first ones read the Ap the last sweep
  // wrote last (still in L2), the last ones write the r the next first sweep
  // reads first.  Slot = tile index, so the reduction order is unchanged.
  const int r = gridDim.y - 1 - blockIdx.y;
  const int tile = gridDim.x - 1 - blockIdx.x;
  if (!st[r].active) {
    finish_block(fin, red);
    return;
  }
  const double alpha = st[r].alpha;
  const int64_t base = (int64_t)r * len;
  const int64_t t0 = (int64_t)tile * kVecTile;
  const int64_t t1 = min(len, t0 + kVecTile);
  double acc = 0.0;
  // 16-byte accesses for any length: the buffers are 16-byte aligned and every
  // tile starts at an even offset, so a tile starting at an odd element (odd
  // per-RHS length, r odd) peels one element; an odd tail is done scalar
  auto upd1 = [&](int64_t e) {
    if (x) x[e] = __dadd_rn(x[e], __dmul_rn(alpha, p[e]));
    const double rn = __dsub_rn(rr[e], __dmul_rn(alpha, Ap[e]));
    rr[e] = rn;
    return __dmul_rn(rn, rn);
  };
  const int64_t g0 = base + t0, g1 = base + t1;  // global element range of this tile
  const int64_t v0 = (g0 + 1) & ~(int64_t)1;     // first even element
  const int64_t v1 = g1 & ~(int64_t)1;           // end of the pair range
  if (threadIdx.x == 0 && g0 < v0) acc += upd1(g0);
  {
    double2* x2 = reinterpret_cast<double2*>(x);
    double2* r2 = reinterpret_cast<double2*>(rr);
    const double2* p2 = reinterpret_cast<const double2*>(p);
    const double2* a2 = reinterpret_cast<const double2*>(Ap);
    const int64_t h0 = v0 >> 1, h1 = v1 >> 1;
    if (x) {
#pragma unroll 4
      for (int64_t i = h0 + threadIdx.x; i < h1; i += blockDim.x) {
        const double2 xv = x2[i], rv = r2[i], pv = __ldg(p2 + i), av = __ldg(a2 + i);
        x2[i] = make_double2(__dadd_rn(xv.x, __dmul_rn(alpha, pv.x)), __dadd_rn(xv.y, __dmul_rn(alpha, pv.y)));
        const double2 rn =
            make_double2(__dsub_rn(rv.x, __dmul_rn(alpha, av.x)), __dsub_rn(rv.y, __dmul_rn(alpha, av.y)));
        r2[i] = rn;
        acc += __dmul_rn(rn.x, rn.x);
        acc += __dmul_rn(rn.y, rn.y);
      }
    } else {  // x deferred to the next first sweep (InArgs::xacc): r and Ap only
      // all loads of the tile issued before the first use (same summation order)
      constexpr int U = kVecTile / 2 / kThreads;
      double2 rv[U], av[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t i = h0 + threadIdx.x + (int64_t)u * kThreads;
        if (i < h1) {
          rv[u] = r2[i];
          av[u] = __ldg(a2 + i);
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t i = h0 + threadIdx.x + (int64_t)u * kThreads;
        if (i < h1) {
          const double2 rn = make_double2(__dsub_rn(rv[u].x, __dmul_rn(alpha, av[u].x)),
                                          __dsub_rn(rv[u].y, __dmul_rn(alpha, av[u].y)));
          r2[i] = rn;
          acc += __dmul_rn(rn.x, rn.x);
          acc += __dmul_rn(rn.y, rn.y);
        }
      }
    }
  }
  if (threadIdx.x == blockDim.x - 1 && v1 < g1 && v1 >= v0) acc += upd1(v1);
  double s = block_sum(acc, red);
  if (threadIdx.x == 0) part[(int64_t)r * nslot + tile] = s;
  finish_block(fin, red);
}

// x += alpha p for one RHS: the deferred x update of its last CG iteration
// (the first sweep applies it for every earlier iteration, see InArgs::xacc)
// RHS r = blockIdx.y is flushed when bit r of owe is set, from p1 when bit r
// of use1 is set, else from p0.
__global__ void __launch_bounds__(kThreads) k_x_flush(int64_t len, const RhsState* st, double* __restrict__ x,
                                                      const double* __restrict__ p0, const double* __restrict__ p1,
                                                      unsigned owe, unsigned use1) {
  const int r = blockIdx.y;
  if (!((owe >> r) & 1u)) return;
  const double* p = ((use1 >> r) & 1u) ? p1 : p0;
  const double alpha = st[r].alpha;
  const int64_t base = (int64_t)r * len;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < len; i += (int64_t)gridDim.x * blockDim.x)
    x[base + i] = __dadd_rn(x[base + i], __dmul_rn(alpha, p[base + i]));
}

// Host side of the deferred x update: a RHS whose last k_cg_update stopped it
// (converged or max_iter) still owes alpha_k p_k; one stopped by a breakdown
// (or at r0) owes nothing.  RHS r was active in loop iterations
// 0 .. iterations-1, so p_k is p[(iterations - 1) & 1] (use1 bit set: p[1]).
inline void x_flush_masks(const RhsState* hs, int R, unsigned& owe, unsigned& use1) {
  owe = use1 = 0u;
  for (int r = 0; r < R; ++r) {
    const RhsState& q = hs[r];
    if (q.iterations >= 1 && q.status != ST_BREAKDOWN && (q.converged || q.status == ST_MAXITER)) {
      owe |= 1u << r;
      if ((q.iterations - 1) & 1) use1 |= 1u << r;
    }
  }
}

// out = a - b ; partial <out, out>      (r = rhs - op(x), solver.py:186)
__global__ void __launch_bounds__(kThreads) k_sub_dot(int64_t len, const double* a, const double* b, double* out,
                                                      double* part, int nslot, FinArgs fin) {
  __shared__ double red[kThreads / 32];
  const int r = blockIdx.y;
  const int64_t base = (int64_t)r * len;
  const int64_t t0 = (int64_t)blockIdx.x * kVecTile;
  const int64_t t1 = min(len, t0 + kVecTile);
  double acc = 0.0;
  for (int64_t i = t0 + threadIdx.x; i < t1; i += blockDim.x) {
    const double o = __dsub_rn(a[base + i], b[base + i]);
    out[base + i] = o;
    acc += __dmul_rn(o, o);
  }
  double s = block_sum(acc, red);
  if (threadIdx.x == 0) part[(int64_t)r * nslot + blockIdx.x] = s;
  finish_block(fin, red);
}

// out[r][a][v] = E[r][a] (x == NULL) or x[r][a][v] - E[r][a]   (e = E_N ; solution = e - E_N)
struct Loads { double E[8][kMaxDim]; };
__global__ void k_fill_loads(int64_t N, int d, Loads L, const double* x, double* out) {
  const int r = blockIdx.y;
  const int64_t len = (int64_t)d * N;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < len; i += (int64_t)gridDim.x * blockDim.x) {
    const int a = (int)(i / N);
    const int64_t e = (int64_t)r * len + i;
    out[e] = x == nullptr ? L.E[r][a] : __dsub_rn(x[e], L.E[r][a]);
  }
}

// out = A u pointwise (material.py:182-187)
__global__ void k_apply_A(Geo g, Coef C, const double* u, double* out) {
  const int r = blockIdx.y;
  const int d = g.dim;
  const int64_t base = (int64_t)r * d * g.N;
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < g.N; v += (int64_t)gridDim.x * blockDim.x) {
    for (int a = 0; a < d; ++a) {
      double acc = 0.0;
      for (int b = 0; b < d; ++b) acc = __dadd_rn(acc, __dmul_rn(coef(C, d, a, b, v, g.N), u[base + b * g.N + v]));
      out[base + a * g.N + v] = acc;
    }
  }
}

// Energy / effective-tensor partials: M[al][be] = sum_v sum_a (A t_al)_a (t_be)_a,
// t_al = E_al + x_al  (homogenize.py:59-67).  One slot per CTA, R*R values.
constexpr int kMaxRhs = 8;
__global__ void __launch_bounds__(kThreads) k_energy(Geo g, Coef C, Loads L, int R, const double* x, double* part,
                                                     int64_t chunk) {
  __shared__ double red[kThreads / 32];
  const int d = g.dim;
  const int64_t v0 = (int64_t)blockIdx.x * chunk;
  const int64_t v1 = min(g.N, v0 + chunk);
  double acc[kMaxRhs * kMaxRhs];
  for (int i = 0; i < R * R; ++i) acc[i] = 0.0;
  for (int64_t v = v0 + threadIdx.x; v < v1; v += blockDim.x) {
    double t[kMaxRhs][kMaxDim];
    double f[kMaxRhs][kMaxDim];
    for (int al = 0; al < R; ++al)
      for (int a = 0; a < d; ++a) t[al][a] = __dadd_rn(x[((int64_t)al * d + a) * g.N + v], L.E[al][a]);
    for (int al = 0; al < R; ++al)
      for (int a = 0; a < d; ++a) {
        double s = 0.0;
        for (int b = 0; b < d; ++b) s = __dadd_rn(s, __dmul_rn(coef(C, d, a, b, v, g.N), t[al][b]));
        f[al][a] = s;
      }
    for (int al = 0; al < R; ++al)
      for (int be = 0; be < R; ++be) {
        double s = 0.0;
        for (int a = 0; a < d; ++a) s = __dadd_rn(s, __dmul_rn(f[al][a], t[be][a]));
        acc[al * R + be] += s;
      }
  }
  for (int i = 0; i < R * R; ++i) {
    double s = block_sum(acc[i], red);
    if (threadIdx.x == 0) part[(int64_t)i * gridDim.x + blockIdx.x] = s;
  }
}

// ---------------------------------------------------------------------------
// Energy matrix finalize: out[i] = (sum of slots) / N in fixed order.
__global__ void k_fin_matrix(const double* part, int nslot, int nval, double total, double* out) {
  __shared__ double red[kThreads / 32];
  for (int i = 0; i < nval; ++i) {
    double s = reduce_slots(part + (int64_t)i * nslot, nslot, red);
    if (threadIdx.x == 0) out[i] = __ddiv_rn(s, total);  // np.sum(...) / total (transforms.py:176)
    __syncthreads();
  }
}

}  // namespace fc

namespace fc {

// ---------------------------------------------------------------------------
// Device generators (SURVEY 8(d) contracts; the host generators in
// generators.py are the bit-exact references on small grids).

// cfg4: nearest seed under the periodic minimum image, voxel centres at the
// integer slot indices; squared distance accumulated axis 0, 1, 2 with
// round-to-nearest ops (no FMA) and strict "<" so the first seed wins ties,
// exactly as generators.voronoi_labels.  Writes the packed tensor of the grain.
// cfg5 generator: one CTA per (centre, z offset) slice of the ball; each thread
// marks voxels (y, x offsets) of that slice in the slab's coverage bitmap and
// counts the bits it newly set (atomicOr's old value), warp-aggregated.
__global__ void __launch_bounds__(256) k_stamp_spheres(int n0g, int n1, int n2, int i0_off, int n0l,
                                                        const int* __restrict__ centres, int ncent, int rad,
                                                        double r2, unsigned* __restrict__ bits,
                                                        unsigned long long* __restrict__ count) {
  const int span = 2 * rad + 1;
  const int cz = blockIdx.x / span;
  const int dz = blockIdx.x % span - rad;
  if (cz >= ncent) return;
  const int z = ((centres[3 * cz] + dz) % n0g + n0g) % n0g;
  const int zl = z - i0_off;
  unsigned long long mine = 0;
  if (zl >= 0 && zl < n0l) {
    const int cy = centres[3 * cz + 1], cx = centres[3 * cz + 2];
    for (int t = threadIdx.x; t < span * span; t += blockDim.x) {
      const int dy = t / span - rad, dx = t % span - rad;
      if ((double)(dz * dz + dy * dy + dx * dx) < r2) {
        const int y = ((cy + dy) % n1 + n1) % n1;
        const int x = ((cx + dx) % n2 + n2) % n2;
        const int64_t v = ((int64_t)zl * n1 + y) * n2 + x;
        const unsigned bit = 1u << (v & 31);
        const unsigned old = atomicOr(bits + (v >> 5), bit);
        mine += (old & bit) ? 0 : 1;
      }
    }
  }
  for (int o = 16; o > 0; o >>= 1) mine += __shfl_xor_sync(0xffffffffu, mine, o);
  if ((threadIdx.x & 31) == 0 && mine) atomicAdd(count, mine);
}

__global__ void k_spheres_field(int64_t N, const unsigned* __restrict__ bits, double high, double low,
                                double* __restrict__ A) {
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < N; v += (int64_t)gridDim.x * blockDim.x)
    A[v] = (bits[v >> 5] >> (v & 31)) & 1u ? high : low;
}

__global__ void k_gen_voronoi(int n0, int n1, int n2, int i0_off, int G, const double* __restrict__ seeds,
                              const double* __restrict__ packed, int nsym, int64_t N, double* __restrict__ A,
                              int* __restrict__ labels) {
  extern __shared__ double sseeds[];
  for (int i = threadIdx.x; i < 3 * G; i += blockDim.x) sseeds[i] = seeds[i];
  __syncthreads();
  const double L0 = n0, L1 = n1, L2 = n2;
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < N; v += (int64_t)gridDim.x * blockDim.x) {
    const int i2 = (int)(v % n2);
    const int64_t t = v / n2;
    const int i1 = (int)(t % n1);
    const int i0 = (int)(t / n1) + i0_off;
    const double p0 = i0, p1 = i1, p2 = i2;
    double best = INFINITY;
    int lab = 0;
    for (int g = 0; g < G; ++g) {
      double a0 = fabs(__dsub_rn(p0, sseeds[3 * g + 0]));
      a0 = fmin(a0, __dsub_rn(L0, a0));
      double a1 = fabs(__dsub_rn(p1, sseeds[3 * g + 1]));
      a1 = fmin(a1, __dsub_rn(L1, a1));
      double a2 = fabs(__dsub_rn(p2, sseeds[3 * g + 2]));
      a2 = fmin(a2, __dsub_rn(L2, a2));
      double d2 = __dadd_rn(__dadd_rn(__dadd_rn(0.0, __dmul_rn(a0, a0)), __dmul_rn(a1, a1)), __dmul_rn(a2, a2));
      if (d2 < best) {
        best = d2;
        lab = g;
      }
    }
    for (int c = 0; c < nsym; ++c) A[(int64_t)c * N + v] = packed[(int64_t)lab * nsym + c];
    if (labels) labels[v] = lab;
  }
}

}  // namespace fc

namespace fc {

// Pointwise first-sweep input for packed coefficients (split variant): writes
// y = M(x) u for all components (and p' for IN_PNEW) so the row FFT can read y
// as a plain field (IN_RAW).  Costs 2 c words/voxel more than the fused sweep
// but runs at streaming bandwidth.
__global__ void __launch_bounds__(256) k_pointwise_aniso(Geo g, Coef C, InArgs ia, const RhsState* st, int R,
                                                         double* __restrict__ y) {
  const int d = g.dim;
  const int64_t N = g.N;
  for (int r = 0; r < R; ++r) {
    if (!rhs_active(st, r)) continue;
    const InEval e0 = make_eval(ia, g, C, st, r, 0);
    const int64_t base = (int64_t)r * d * N;
    for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < N; v += (int64_t)gridDim.x * blockDim.x) {
      double x[kMaxDim] = {0.0, 0.0, 0.0};
#pragma unroll
      for (int b = 0; b < kMaxDim; ++b) {
        if (b >= d) break;
        if (e0.mode == IN_CONST) {
          x[b] = InEval::sel(b, e0.E0, e0.E1, e0.E2);
        } else {
          double xb = __ldg(e0.u + base + b * N + v);
          if (e0.mode == IN_PNEW) {
            if (!e0.first) {
              const double po = __ldg(e0.p_old + base + b * N + v);
              xb = __dadd_rn(xb, __dmul_rn(e0.beta, po));
              if (e0.xacc) e0.xacc[base + b * N + v] = __dadd_rn(e0.xacc[base + b * N + v], __dmul_rn(e0.alpha, po));
            }
            ia.p_new[base + b * N + v] = xb;
          }
          x[b] = xb;
        }
      }
      double Av[6];
#pragma unroll
      for (int m = 0; m < 6; ++m) Av[m] = m < d * (d + 1) / 2 ? __ldg(C.A + (int64_t)m * N + v) : 0.0;
#pragma unroll
      for (int a = 0; a < kMaxDim; ++a) {
        if (a >= d) break;
        double acc = 0.0;
#pragma unroll
        for (int b = 0; b < kMaxDim; ++b) {
          if (b >= d) break;
          double Aab = Av[pidx(d, a, b)];
          if (e0.mode == IN_FP) Aab = __dsub_rn(Aab, pick3(ia.A0, a, b));
          acc = __dadd_rn(acc, __dmul_rn(Aab, x[b]));
        }
        if (e0.mode != IN_FP && e0.s != 1.0) acc = __dmul_rn(e0.s, acc);
        y[base + a * N + v] = acc;
      }
    }
  }
}

}  // namespace fc
