// Persistent, double-buffered last sweep (k_row_inv_pp) and the one-component-
// at-a-time outer sweep (k_outer_seq) for register-path axis lengths.
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
// TF (C = 3): two fields leave, F0^-1 (xi0 q) in row 0 and t = F0^-1 q in row 1; the
// inverse middle sweep rebuilds xi1 t and xi2 t (the same g3_scale products) as it
// loads them (MidGeo::rebuild), so row 2 is neither scaled nor stored here.
#ifndef FC_OUTER_TFI_OCC3
#define FC_OUTER_TFI_OCC3 1  // TFI: two shared-memory rows and <= 84 registers, three resident CTAs per SM
#endif
// TFI (C = 3): the forward middle sweep folded components 1 and 2 (mid_tma_fold):
// row 1 holds u = xi1 v1 + xi2 v2 already, row 2 is not loaded.
template <int L, int C, bool TF = false, bool TFI = false>
__global__ void __launch_bounds__(256, (C == 2 || (TFI && FC_OUTER_TFI_OCC3) ? 3 : 2)) k_outer_seq(Geo g, OuterGeo og, const RhsState* st,
                                                                      const double2* __restrict__ tw,
                                                                      double2* __restrict__ W) {
  constexpr int TP = RegTP<L>::value;
  extern __shared__ __align__(128) unsigned char smraw[];
  double2* sm = reinterpret_cast<double2*>(smraw);
  __shared__ uint64_t bar;
  __shared__ int zero;  // TFI: read per transform so ptxas cannot hoist the next transform's twiddle loads
  const int qb = blockIdx.x % og.nqb;
  const int r = blockIdx.x / og.nqb;
  if (!rhs_active(st, r)) return;
  const int qq = threadIdx.x / TP;
  const int j = threadIdx.x - qq * TP;
  const int ql = qb * og.QB + qq;
  const bool live = ql < og.Q;
  const int nq = min(og.QB, og.Q - qb * og.QB);
  trace_stamp(3, 0);
  if (threadIdx.x == 0) {
    zero = 0;
    mbar_init(&bar, 1);
    constexpr int NIN = TFI ? 2 : C;
    mbar_expect_tx(&bar, (unsigned)(NIN * nq * L * 16));
#pragma unroll
    for (int a = 0; a < NIN; ++a)
      bulk_g2s(sm + (size_t)a * og.QB * L, W + ((int64_t)(r * C + a) * og.Q + (int64_t)qb * og.QB) * L,
               (unsigned)(nq * L * 16), &bar);
  }
  __syncthreads();
  mbar_wait(&bar, 0);
  trace_stamp(3, 1);
  if constexpr (C == 3) {  // four transforms (g3_* in fc_kernels_reg.cuh); same arithmetic as k_outer_r<L, 3>
    const int k2 = ql / og.n1, k1 = ql - k2 * og.n1;
    const double xi1 = g.xi[1][live ? k1 : 0];
    const double xi2 = g.xi[2][live ? k2 : 0];
    double2* row0 = sm + ((size_t)0 * og.QB + qq) * L;
    double2* row1 = sm + ((size_t)1 * og.QB + qq) * L;
    double2* row2 = sm + ((size_t)2 * og.QB + qq) * L;
    // F0 v0 -> row0 (parked: every thread its own nine modes), F0 (xi1 v1 + xi2 v2)
    // stays in registers; Gamma_hat there; q is transformed back right away and
    // rows 1, 2 leave while xi0 q (row0) is still being transformed
    double2 v[1][9];
#pragma unroll 1
    for (int a = 0; a < 2; ++a) {
#pragma unroll
      for (int s = 0; s < 9; ++s) {
        const int i = j + s * TP;
        v[0][s] = !live ? make_double2(0.0, 0.0) : a == 0 ? row0[i] : TFI ? row1[i] : g3_fold(xi1, xi2, row1[i], row2[i]);
      }
      fft_reg<L, 1, false>(v, a == 0 ? row0 : row1, L, j, (TFI && FC_OUTER_TFI_OCC3) ? tw + *reinterpret_cast<volatile int*>(&zero) : tw);
      if (a == 0) {
        __syncthreads();
#pragma unroll
        for (int s = 0; s < 9; ++s) row0[j + s * TP] = v[0][s];
      }
    }
    trace_stamp(3, 2);
    if (live) {
#pragma unroll
      for (int s = 0; s < 9; ++s) {
        const int i0 = j + s * TP;
        double2 t0 = row0[i0];
        g3_mode(og, g.xi[0][i0], xi1, xi2, ql == 0 && i0 == 0, t0, v[0][s]);
        row0[i0] = t0;
      }
    }
#pragma unroll 1
    for (int a = 1; a >= 0; --a) {  // rows 1, 2 <- xi1 / xi2 F0^-1(q); row0 <- F0^-1(xi0 q)
      if (a == 0) {
#pragma unroll
        for (int s = 0; s < 9; ++s) v[0][s] = row0[j + s * TP];
      }
      fft_reg<L, 1, true>(v, a == 0 ? row0 : row1, L, j, (TFI && FC_OUTER_TFI_OCC3) ? tw + *reinterpret_cast<volatile int*>(&zero) : tw);
      __syncthreads();
      if (a == 0) {
#pragma unroll
        for (int s = 0; s < 9; ++s) row0[j + s * TP] = v[0][s];
      } else {
#pragma unroll
        for (int s = 0; s < 9; ++s) {
          if constexpr (TF) {
            row1[j + s * TP] = v[0][s];
          } else {
            row1[j + s * TP] = g3_scale(xi1, v[0][s]);
            row2[j + s * TP] = g3_scale(xi2, v[0][s]);
          }
        }
        fence_proxy_async();
        __syncthreads();
        if (threadIdx.x == 0) {
#pragma unroll
          for (int b = 1; b < (TF ? 2 : C); ++b)
            bulk_s2g(W + ((int64_t)(r * C + b) * og.Q + (int64_t)qb * og.QB) * L, sm + (size_t)b * og.QB * L,
                     (unsigned)(nq * L * 16));
          bulk_commit();
        }
      }
    }
    trace_stamp(3, 3);
    fence_proxy_async();
    __syncthreads();
    if (threadIdx.x == 0) {
      bulk_s2g(W + ((int64_t)(r * C) * og.Q + (int64_t)qb * og.QB) * L, sm, (unsigned)(nq * L * 16));
      bulk_commit();
      trace_stamp(3, 4);
      bulk_wait_read0();
      trace_stamp(3, 5);
    }
    return;
  } else {
  // d = 2: F0 v0 parked in its row (every thread its own nine modes), F0 v1 stays in
  // registers; Gamma_hat there (g2_mode, as k_outer_r<L, 2>); xi1 q is transformed back
  // at once, then xi0 q.  One transform body at a time: <= 84 registers, three CTAs
  // per SM (the twiddle table's address is tied to a shared-memory word per transform,
  // or ptxas hoists the next transform's loads and doubles the registers).
  static_assert(C == 2, "d = 3 takes the branch above");
  double2* row0 = sm + ((size_t)0 * og.QB + qq) * L;
  double2* row1 = sm + ((size_t)1 * og.QB + qq) * L;
  double2 v[1][9];
#pragma unroll 1
  for (int a = 0; a < 2; ++a) {
    double2* row = a == 0 ? row0 : row1;
#pragma unroll
    for (int s = 0; s < 9; ++s) v[0][s] = live ? row[j + s * TP] : make_double2(0.0, 0.0);
    fft_reg<L, 1, false>(v, row, L, j, tw + *reinterpret_cast<volatile int*>(&zero));
    if (a == 0) {
      __syncthreads();
#pragma unroll
      for (int s = 0; s < 9; ++s) row0[j + s * TP] = v[0][s];
    }
  }
  {
    const double xi1 = g.xi[1][live ? ql : 0];
    const bool qzero = live && ql == 0;
#pragma unroll
    for (int s = 0; s < 9; ++s) {
      const int i0 = j + s * TP;
      double2 t0 = row0[i0];
      g2_mode(og, g.xi[0][i0], xi1, qzero && i0 == 0, t0, v[0][s]);
      row0[i0] = t0;
    }
  }
#pragma unroll 1
  for (int a = 1; a >= 0; --a) {
    double2* row = a == 0 ? row0 : row1;
    if (a == 0) {
#pragma unroll
      for (int s = 0; s < 9; ++s) v[0][s] = row0[j + s * TP];
    }
    fft_reg<L, 1, true>(v, row, L, j, tw + *reinterpret_cast<volatile int*>(&zero));
    __syncthreads();
#pragma unroll
    for (int s = 0; s < 9; ++s) row[j + s * TP] = v[0][s];
  }
  }  // C == 2
  trace_stamp(3, 3);
  fence_proxy_async();
  __syncthreads();
  if (threadIdx.x == 0) {
#pragma unroll
    for (int a = 0; a < C; ++a)
      bulk_s2g(W + ((int64_t)(r * C + a) * og.Q + (int64_t)qb * og.QB) * L, sm + (size_t)a * og.QB * L,
               (unsigned)(nq * L * 16));
    bulk_commit();
    trace_stamp(3, 4);
    bulk_wait_read0();
    trace_stamp(3, 5);
  }
}

}  // namespace fc
