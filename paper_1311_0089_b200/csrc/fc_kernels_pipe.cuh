// Persistent, double-buffered first sweep for power-of-three contiguous axes.
//
// The one-shot row kernel (fc_kernels_reg.cuh: k_row_fwd_r) loads a row block,
// transforms it and stores it, so HBM idles whenever both resident CTAs of an
// SM transform at the same time.  Here one CTA per SM walks the row pairs
// (tile t, t + G, t + 2G, ...) and keeps the next pair's inputs in flight while
// the current pair is transformed: the TMA bulk loads of tile t + G land in
// the second shared-memory stage during the FFT of tile t.
//
// Row block = one complex pencil (rows 2q, 2q+1).  Same layouts, modes and
// rounding as the staged path of k_row_fwd_r; the transposed half spectrum is
// written with TMA tensor boxes (RowGeo::tma).
#pragma once
#include "fc_kernels_reg.cuh"

namespace fc {

constexpr int FC_MAX_RHS_DEV = 8;  // = FC_MAX_RHS (include/fftcell_b200.h)

// doubles per staged array of one row pair (even, room for the 16-byte phase shift)
template <int L>
__host__ __device__ constexpr int pipe_stride() { return (2 * L + 3) & ~1; }

struct PipeTile {
  int a, tile, o, r;
};
__device__ __forceinline__ PipeTile pipe_decode(int64_t t, int c, const RowGeo& rg) {
  PipeTile q;
  q.a = (int)(t % c); t /= c;
  q.tile = (int)(t % rg.ntiles); t /= rg.ntiles;
  q.o = (int)(t % rg.no);
  q.r = (int)(t / rg.no);
  return q;
}

// Persistent first sweep, 2 CTAs per SM.  Shared memory: one input stage
// U[stride] P[stride] (r / p_old, or the raw field) and one spectrum buffer Z
// (the FFT exchange, then the split half spectra Y[k][2] written in place).
// A is read straight from global memory (issued before the stage wait).  As
// soon as the pointwise step has moved the inputs into registers the stage is
// refilled with block t + G by TMA, so those loads overlap this block's FFT,
// split and store.
template <int L>
__global__ void __launch_bounds__(256, 2) k_row_fwd_pp(Geo g, RowGeo rg, Coef C, InArgs ia, const RhsState* st,
                                                       const double2* __restrict__ tw, int64_t ntile,
                                                       const __grid_constant__ CUtensorMap tmW) {
  constexpr int TP = RegTP<L>::value;
  constexpr int hl = (L + 1) / 2;
  constexpr int stride = pipe_stride<L>();
  constexpr int zoff = (2 * stride + 15) & ~15;  // doubles: Z starts 128-byte aligned
  extern __shared__ __align__(128) unsigned char smraw[];
  double* S = reinterpret_cast<double*>(smraw);
  double2* Z = reinterpret_cast<double2*>(S + zoff);
  __shared__ uint64_t bar;
  __shared__ double s_beta[FC_MAX_RHS_DEV];
  __shared__ double s_alpha[FC_MAX_RHS_DEV];
  __shared__ int s_flags[FC_MAX_RHS_DEV];  // bit 0 active, bit 1 first
  const int c = g.dim;
  const int j = threadIdx.x;  // one pencil per CTA: thread j = FFT lane
  const int R = (int)(ntile / ((int64_t)c * rg.ntiles * rg.no));
  if (threadIdx.x < R) {
    const int r = threadIdx.x;
    const bool act = rhs_active(st, r);
    const bool first = ia.mode == IN_PNEW ? st[r].first != 0 : true;
    s_flags[r] = (act ? 1 : 0) | (first ? 2 : 0);
    s_beta[r] = ia.mode == IN_PNEW ? st[r].beta : 0.0;
    s_alpha[r] = ia.mode == IN_PNEW ? st[r].alpha : 0.0;
  }
  if (threadIdx.x == 0) mbar_init(&bar, 1);
  __syncthreads();

  struct Src {
    const double *u, *p, *A;
    int n;
  };
  auto sources = [&](const PipeTile& q) {
    Src o;
    const int row0 = q.tile * 2;
    o.n = min(2, rg.np - row0) * L;
    const int64_t vbase = ((int64_t)q.o * rg.np + row0) * L;
    const int64_t ub = (int64_t)q.r * c * g.N + (int64_t)q.a * g.N + vbase;
    o.u = ia.u + ub;
    o.p = (ia.mode == IN_PNEW && !(s_flags[q.r] & 2)) ? ia.p_old + ub : nullptr;
    o.A = ia.mode != IN_RAW ? C.A + vbase : nullptr;
    return o;
  };
  // first active block at or after t (inactive right-hand sides are skipped)
  auto next_active = [&](int64_t t) {
    while (t < ntile && !(s_flags[pipe_decode(t, c, rg).r] & 1)) t += gridDim.x;
    return t;
  };
  auto prefetch = [&](int64_t t) {  // thread 0
    if (t >= ntile) return;
    const Src o = sources(pipe_decode(t, c, rg));
    const int su = bulk_shift(o.u), sp = o.p ? bulk_shift(o.p) : 0;
    mbar_expect_tx(&bar, bulk_bytes(o.n, su) + (o.p ? bulk_bytes(o.n, sp) : 0u));
    bulk_g2s(S, o.u - su, bulk_bytes(o.n, su), &bar);
    if (o.p) bulk_g2s(S + stride, o.p - sp, bulk_bytes(o.n, sp), &bar);
  };
  int64_t t = next_active(blockIdx.x);
  if (threadIdx.x == 0) prefetch(t);
  unsigned phase = 0u;
  for (; t < ntile;) {
    const PipeTile q = pipe_decode(t, c, rg);
    const int a = q.a, r = q.r;
    const Src o = sources(q);
    const int nrows = o.n / L;
    const bool pnew = ia.mode == IN_PNEW;
    const bool first = (s_flags[r] & 2) != 0;
    const double beta = s_beta[r];
    // coefficient values straight from global memory, issued before the wait
    double av[2][9];
#pragma unroll
    for (int s = 0; s < 9; ++s)
#pragma unroll
      for (int h = 0; h < 2; ++h) av[h][s] = (o.A && h < nrows) ? __ldg(o.A + h * L + j + s * TP) : 0.0;
    mbar_wait(&bar, phase);
    phase ^= 1u;
    const double* st_u = S + bulk_shift(o.u);
    const double* st_p = S + stride + (o.p ? bulk_shift(o.p) : 0);
    double* pw = pnew ? ia.p_new + (o.u - ia.u) : nullptr;
    double* xw = (pnew && !first && ia.xacc) ? ia.xacc + (o.u - ia.u) : nullptr;
    const double alpha = s_alpha[r];
    const double A0aa = ia.mode == IN_FP ? pick3(ia.A0, a, a) : 0.0;
    double2 v[1][9];
#pragma unroll
    for (int s = 0; s < 9; ++s) {
      const int i = j + s * TP;
      double y[2] = {0.0, 0.0};
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        if (h < nrows) {
          const int e = h * L + i;
          double x = st_u[e];
          if (pnew) {
            x = first ? x : __dadd_rn(x, __dmul_rn(beta, st_p[e]));
            pw[e] = x;
            if (xw) xw[e] = __dadd_rn(xw[e], __dmul_rn(alpha, st_p[e]));
          }
          double val;
          if (ia.mode == IN_RAW) val = x;
          else if (ia.mode == IN_FP) val = __dmul_rn(__dsub_rn(av[h][s], A0aa), x);
          else val = __dmul_rn(av[h][s], x);
          if (ia.mode != IN_FP && ia.s != 1.0) val = __dmul_rn(ia.s, val);
          y[h] = val;
        }
      }
      v[0][s] = make_double2(y[0], y[1]);
    }
    const int64_t tn = next_active(t + gridDim.x);
    __syncthreads();  // the stage has been read: refill it with the next block
    if (threadIdx.x == 0) {
      bulk_wait_read0();  // the previous block's spectrum store has left Z
      prefetch(tn);
    }
    fft_reg<L, 1, false>(v, Z, L, j, tw);
    __syncthreads();
#pragma unroll
    for (int s = 0; s < 9; ++s) Z[j + s * TP] = v[0][s];
    __syncthreads();
    // split in place: gather (z_k, z_{L-k}) for this thread's modes, then write Y[k][2]
    constexpr int KP = (hl + TP - 1) / TP;
    double2 zk[KP], zm[KP];
#pragma unroll
    for (int m = 0; m < KP; ++m) {
      const int k = j + m * TP;
      if (k < hl) {
        zk[m] = Z[k];
        zm[m] = Z[k == 0 ? 0 : L - k];
      }
    }
    __syncthreads();
#pragma unroll
    for (int m = 0; m < KP; ++m) {
      const int k = j + m * TP;
      if (k < hl) {
        Z[2 * k] = make_double2(0.5 * (zk[m].x + zm[m].x), 0.5 * (zk[m].y - zm[m].y));
        Z[2 * k + 1] = make_double2(0.5 * (zk[m].y + zm[m].y), 0.5 * (zm[m].x - zk[m].x));
      }
    }
    fence_proxy_async();
    __syncthreads();
    if (threadIdx.x == 0) {
      const int c2 = (r * c + a) * rg.no + q.o;
      for (int b = 0; b < rg.nbox; ++b) tma_store_3d(&tmW, 4 * q.tile, b * rg.boxK, c2, Z + (size_t)b * rg.boxK * 2);
      bulk_commit();
    }
    t = tn;
  }
  if (threadIdx.x == 0) bulk_wait_read0();
}

// Persistent, multi-buffered last sweep (nst <= 4 stages): each CTA walks its
// row blocks and keeps the TMA loads of the next nst - 1 blocks' transposed
// half spectra in flight while it transforms the current one; the consumed stage
// doubles as the FFT exchange buffer and is refilled once the block is done.
// Same epilogues, partial-sum slots and finalize as k_row_inv_r (one arrival
// per CTA at the end).
template <int L>
__global__ void __launch_bounds__(256, 2) k_row_inv_pp(Geo g, RowGeo rg, EpArgs ea, const RhsState* st,
                                                       const double2* __restrict__ tw, int64_t ntile, int stage_c, int nst,
                                                       int qbuf,
                                                       const __grid_constant__ CUtensorMap tmW) {
  constexpr int TP = RegTP<L>::value;
  constexpr int hl = (L + 1) / 2;
  extern __shared__ __align__(128) unsigned char smraw[];
  double2* S = reinterpret_cast<double2*>(smraw);
  __shared__ double red[kMaxBlock / 32];
  __shared__ uint64_t bar[4];
  __shared__ uint64_t barq;  // epilogue input (p / e) of the current block, qbuf != 0
  __shared__ int s_act[FC_MAX_RHS_DEV];
  const int c = g.dim;
  const int B = rg.B;
  const int R = (int)(ntile / ((int64_t)c * rg.ntiles * rg.no));
  if (threadIdx.x < R) s_act[threadIdx.x] = rhs_active(st, threadIdx.x) ? 1 : 0;
  if (threadIdx.x == 0) {
    for (int b = 0; b < nst; ++b) mbar_init(&bar[b], 1);
    mbar_init(&barq, 1);
  }
  double* Q = reinterpret_cast<double*>(S + (size_t)nst * stage_c);  // qbuf: one row block of doubles (+2)
  unsigned qphase = 0u;
  __syncthreads();
  auto issue = [&](int64_t t, int b) {
    if (t >= ntile) return;
    const PipeTile q = pipe_decode(t, c, rg);
    if (!s_act[q.r]) return;
    double2* dst = S + (size_t)b * stage_c;
    mbar_expect_tx(&bar[b], (unsigned)(rg.nbox * rg.boxK * B * 16));
    const int c2 = (q.r * c + q.a) * rg.no + q.o;
    for (int bx = 0; bx < rg.nbox; ++bx)
      tma_load_3d(dst + (size_t)bx * rg.boxK * B, &tmW, 2 * q.tile * B, bx * rg.boxK, c2, &bar[b]);
  };
  int64_t t = blockIdx.x;
  if (threadIdx.x == 0)
    for (int b = 0; b < nst; ++b) issue(t + (int64_t)b * gridDim.x, b);
  const int p = threadIdx.x / TP;
  const int j = threadIdx.x - p * TP;
  const int re = 2 * p, ro = 2 * p + 1;
  const bool need_q = ea.mode == EP_AP || ea.mode == EP_FP;
  unsigned phases = 0u;  // bit b: parity of stage b's next completion (no local array)
  int cur = 0;
  for (; t < ntile; t += gridDim.x) {
    const PipeTile q = pipe_decode(t, c, rg);
    if (s_act[q.r]) {
      const int a = q.a, r = q.r, o = q.o, tile = q.tile;
      mbar_wait(&bar[cur], (phases >> cur) & 1u);
      phases ^= 1u << cur;
      double2* base = S + (size_t)cur * stage_c;
      const int row0 = tile * B;
      const int nrows = min(B, rg.np - row0);
      const int64_t vbase = ((int64_t)o * rg.np + row0) * L;
      const int64_t ebase = ((int64_t)r * c + a) * g.N + vbase;
      const bool he = re < nrows, has_o = ro < nrows;
      const double* qsrc = (ea.mode == EP_AP ? ea.p : ea.out) + ebase;
      const bool qb = need_q && qbuf;
      const int qsh = qb ? bulk_shift(qsrc) : 0;
      if (qb && threadIdx.x == 0) {  // lands during the transform
        mbar_expect_tx(&barq, bulk_bytes(nrows * L, qsh));
        bulk_g2s(Q, qsrc - qsh, bulk_bytes(nrows * L, qsh), &barq);
      }
      double2 v[1][9];
#pragma unroll
      for (int s = 0; s < 9; ++s) {
        const int i = j + s * TP;
        const int k = i < hl ? i : L - i;
        const double2 ye = he ? base[k * B + re] : make_double2(0.0, 0.0);
        const double2 yo = has_o ? base[k * B + ro] : make_double2(0.0, 0.0);
        if (i == 0) v[0][s] = make_double2(ye.x, yo.x);
        else if (i < hl) v[0][s] = make_double2(ye.x - yo.y, ye.y + yo.x);
        else v[0][s] = make_double2(ye.x + yo.y, yo.x - ye.y);
      }
      fft_reg<L, 1, true>(v, base + (size_t)p * L, L, j, tw);
      const double Ea = ea.mode == EP_FP ? pick(ea.E, r, a) : 0.0;
      double2 qv[9];
      if (qb) {
        mbar_wait(&barq, qphase);
        qphase ^= 1u;
        const double* sq = Q + qsh;
#pragma unroll
        for (int s = 0; s < 9; ++s) {
          const int i = j + s * TP;
          qv[s].x = he ? sq[re * L + i] : 0.0;
          qv[s].y = has_o ? sq[ro * L + i] : 0.0;
        }
      } else {
#pragma unroll
        for (int s = 0; s < 9; ++s) {
          const int i = j + s * TP;
          qv[s].x = need_q && he ? __ldg(qsrc + re * L + i) : 0.0;
          qv[s].y = need_q && has_o ? __ldg(qsrc + ro * L + i) : 0.0;
        }
      }
      double acc = 0.0;
      with_ep_mode(ea.mode, [&](auto M) {
        constexpr int MODE = decltype(M)::value;
#pragma unroll
        for (int s = 0; s < 9; ++s) {
          if (he) acc += ep_value_t<MODE>(v[0][s].x * g.invN, Ea, qv[s].x, v[0][s].x);
          if (has_o) acc += ep_value_t<MODE>(v[0][s].y * g.invN, Ea, qv[s].y, v[0][s].y);
        }
      });
      if (ea.part != nullptr) {
        const double sum = block_sum(acc, red);
        if (threadIdx.x == 0) ea.part[(int64_t)r * ea.nslot + (o * rg.ntiles + tile) * c + a] = sum;
      }
      double* __restrict__ out = ea.out;
#pragma unroll
      for (int s = 0; s < 9; ++s) {
        const int i = j + s * TP;
        if (he) out[ebase + (int64_t)re * L + i] = v[0][s].x;
        if (has_o) out[ebase + (int64_t)ro * L + i] = v[0][s].y;
      }
      fence_proxy_async();  // the exchange writes precede the refill of this stage
      __syncthreads();
    }
    if (threadIdx.x == 0) issue(t + (int64_t)nst * gridDim.x, cur);
    cur = cur + 1 == nst ? 0 : cur + 1;
  }
  finish_block(ea.fin, red);
}

// Outer sweep, components one after another (single slab, TMA pencils): each
// thread transforms one component pencil at a time (9 complex in registers
// instead of C x 9), parking the spectra in their shared-memory rows, applies
// Gamma_hat from shared memory and transforms back.  Fewer registers, so more
// resident warps than k_outer_r, for one extra shared-memory pass per
// component.  Same arithmetic as k_outer_r.
template <int L, int C>
__global__ void __launch_bounds__(256, (C == 2 ? 3 : 2)) k_outer_seq(Geo g, OuterGeo og, const RhsState* st,
                                                                      const double2* __restrict__ tw,
                                                                      double2* __restrict__ W) {
  constexpr int TP = RegTP<L>::value;
  extern __shared__ __align__(128) unsigned char smraw[];
  double2* sm = reinterpret_cast<double2*>(smraw);
  __shared__ uint64_t bar;
  const int qb = blockIdx.x % og.nqb;
  const int r = blockIdx.x / og.nqb;
  if (!rhs_active(st, r)) return;
  const int qq = threadIdx.x / TP;
  const int j = threadIdx.x - qq * TP;
  const int ql = qb * og.QB + qq;
  const bool live = ql < og.Q;
  const int nq = min(og.QB, og.Q - qb * og.QB);
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    mbar_expect_tx(&bar, (unsigned)(C * nq * L * 16));
#pragma unroll
    for (int a = 0; a < C; ++a)
      bulk_g2s(sm + (size_t)a * og.QB * L, W + ((int64_t)(r * C + a) * og.Q + (int64_t)qb * og.QB) * L,
               (unsigned)(nq * L * 16), &bar);
  }
  __syncthreads();
  mbar_wait(&bar, 0);
  if constexpr (C == 3) {  // four transforms (g3_* in fc_kernels_reg.cuh); same arithmetic as k_outer_r<L, 3>
    const int k2 = ql / og.n1, k1 = ql - k2 * og.n1;
    const double xi1 = g.xi[1][live ? k1 : 0];
    const double xi2 = g.xi[2][live ? k2 : 0];
    double2* row0 = sm + ((size_t)0 * og.QB + qq) * L;
    double2* row1 = sm + ((size_t)1 * og.QB + qq) * L;
    double2* row2 = sm + ((size_t)2 * og.QB + qq) * L;
#pragma unroll 1
    for (int a = 0; a < 2; ++a) {  // F0 v0 -> row0, F0 (xi1 v1 + xi2 v2) -> row1
      double2* row = a == 0 ? row0 : row1;
      double2 v[1][9];
#pragma unroll
      for (int s = 0; s < 9; ++s) {
        const int i = j + s * TP;
        v[0][s] = !live ? make_double2(0.0, 0.0) : a == 0 ? row0[i] : g3_fold(xi1, xi2, row1[i], row2[i]);
      }
      fft_reg<L, 1, false>(v, row, L, j, tw);
      __syncthreads();
#pragma unroll
      for (int s = 0; s < 9; ++s) row[j + s * TP] = v[0][s];
    }
    __syncthreads();
    if (live) {
#pragma unroll
      for (int s = 0; s < 9; ++s) {
        const int i0 = j + s * TP;
        double2 t0 = row0[i0], t1 = row1[i0];
        g3_mode(og, g.xi[0][i0], xi1, xi2, ql == 0 && i0 == 0, t0, t1);
        row0[i0] = t0;
        row1[i0] = t1;
      }
    }
#pragma unroll 1
    for (int a = 0; a < 2; ++a) {  // row0 <- F0^-1(xi0 q); rows 1, 2 <- xi1 / xi2 F0^-1(q)
      double2* row = a == 0 ? row0 : row1;
      double2 v[1][9];
#pragma unroll
      for (int s = 0; s < 9; ++s) v[0][s] = row[j + s * TP];
      fft_reg<L, 1, true>(v, row, L, j, tw);
      __syncthreads();
      if (a == 0) {
#pragma unroll
        for (int s = 0; s < 9; ++s) row0[j + s * TP] = v[0][s];
      } else {
#pragma unroll
        for (int s = 0; s < 9; ++s) {
          row1[j + s * TP] = g3_scale(xi1, v[0][s]);
          row2[j + s * TP] = g3_scale(xi2, v[0][s]);
        }
      }
    }
  } else {
#pragma unroll 1
  for (int a = 0; a < C; ++a) {  // forward transforms, spectra back in place
    double2* row = sm + ((size_t)a * og.QB + qq) * L;
    double2 v[1][9];
#pragma unroll
    for (int s = 0; s < 9; ++s) v[0][s] = live ? row[j + s * TP] : make_double2(0.0, 0.0);
    fft_reg<L, 1, false>(v, row, L, j, tw);
    __syncthreads();
#pragma unroll
    for (int s = 0; s < 9; ++s) row[j + s * TP] = v[0][s];
  }
  __syncthreads();
  if (live) {  // Gamma_hat(k) v = xi (xi . v) / den, 0 at k = 0 (per thread: its own modes)
    const int q = ql;
    double xi1 = 0.0, xi2 = 0.0;
    if (C == 2) {
      xi1 = g.xi[1][q];
    } else {
      const int k2 = q / og.n1, k1 = q - k2 * og.n1;
      xi1 = g.xi[1][k1];
      xi2 = g.xi[2][k2];
    }
#pragma unroll
    for (int s = 0; s < 9; ++s) {
      const int i0 = j + s * TP;
      double2 v[C];
#pragma unroll
      for (int a = 0; a < C; ++a) v[a] = sm[((size_t)a * og.QB + qq) * L + i0];
      const double xi[3] = {g.xi[0][i0], xi1, xi2};
      double2 out[C];
      if (q == 0 && i0 == 0) {
#pragma unroll
        for (int a = 0; a < C; ++a) out[a] = make_double2(0.0, 0.0);
      } else {
        double2 dots = make_double2(0.0, 0.0);
#pragma unroll
        for (int a = 0; a < C; ++a) {
          dots.x += xi[a] * v[a].x;
          dots.y += xi[a] * v[a].y;
        }
        double den = 0.0;
        if (og.orth) {
#pragma unroll
          for (int a = 0; a < C; ++a) den += xi[a] * xi[a];
        } else {
#pragma unroll
          for (int a = 0; a < C; ++a)
#pragma unroll
            for (int b = 0; b < C; ++b) den += xi[a] * og.M[a][b] * xi[b];
        }
        const double inv = 1.0 / den;
        const double2 qv = make_double2(dots.x * inv, dots.y * inv);
#pragma unroll
        for (int a = 0; a < C; ++a) out[a] = make_double2(xi[a] * qv.x, xi[a] * qv.y);
      }
#pragma unroll
      for (int a = 0; a < C; ++a) sm[((size_t)a * og.QB + qq) * L + i0] = out[a];
    }
  }
#pragma unroll 1
  for (int a = 0; a < C; ++a) {  // inverse transforms (each thread reads the modes it wrote)
    double2* row = sm + ((size_t)a * og.QB + qq) * L;
    double2 v[1][9];
#pragma unroll
    for (int s = 0; s < 9; ++s) v[0][s] = row[j + s * TP];
    fft_reg<L, 1, true>(v, row, L, j, tw);
    __syncthreads();
#pragma unroll
    for (int s = 0; s < 9; ++s) row[j + s * TP] = v[0][s];
  }
  }  // C == 2
  fence_proxy_async();
  __syncthreads();
  if (threadIdx.x == 0) {
#pragma unroll
    for (int a = 0; a < C; ++a)
      bulk_s2g(W + ((int64_t)(r * C + a) * og.Q + (int64_t)qb * og.QB) * L, sm + (size_t)a * og.QB * L,
               (unsigned)(nq * L * 16));
    bulk_commit();
    bulk_wait_read0();
  }
}

}  // namespace fc
