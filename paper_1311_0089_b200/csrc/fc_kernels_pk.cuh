// First sweep for packed (anisotropic) coefficients, fused: the pointwise step
// y = M(x) p' (solver.py:174 einsum, solver.py:266 for the fixed point) and the
// row FFT of all C components in one CTA, so y never leaves shared memory.
//
// Two thread mappings over the same row block (npk complex pencils = 2 npk rows
// per component):
//  1. pointwise: thread t walks voxels e = t, t + blockDim, ... of the block and
//     evaluates all C components of y at once, so r, p_old, x and the packed
//     tensor are each read from HBM exactly once per voxel (coalesced: adjacent
//     threads, adjacent voxels); p' and the deferred x update are stored
//     straight back.  y lands in shared memory as ys[a][row][i];
//  2. transform: thread (a, p, j) loads rows (2p, 2p+1) of component a as one
//     complex pencil (two-for-one), runs the register FFT (fc_fft_reg.cuh) with
//     the pencil's own rows as exchange buffer, then the spectrum is split into
//     the two half spectra and stored transposed with one TMA box store per
//     component (tensor map with box {2B, boxK}, B = 2 npk rows).
// The arithmetic (products, sums over b in order, explicit roundings, the FFT)
// is that of k_pointwise_aniso followed by k_row_fwd_r on y, so the result is
// bitwise identical to the split variant (tests/test_gpu_variants.py).
#pragma once
#include "fc_kernels_reg.cuh"

namespace fc {

// Shared memory of k_row_fwd_pk: pencils (C npk L complex, 128-byte rounded) +
// split spectrum boxes (C nbox boxK 2 npk complex).
__host__ __device__ inline size_t pk_smem(int L, int C, int npk, int nbox, int boxK) {
  const size_t pen = ((size_t)C * npk * L * 16 + 127) & ~(size_t)127;
  return pen + (size_t)C * nbox * boxK * 2 * npk * 16;
}

#ifndef FC_PK_IDX_SMEM
#define FC_PK_IDX_SMEM 0  // experiment: phase table staged in shared memory (nph * NSYM * 8 <= 32 KB)
#endif
#ifndef FC_PK_IDX_K
#define FC_PK_IDX_K 3  // voxels per thread in flight, indexed variant
#endif
#ifndef FC_PK_IDX_LATE
#define FC_PK_IDX_LATE 0  // experiment: table reads (L1 hits) in the compute loop, not held across the loads
#endif
#ifndef FC_PK_MINB
#define FC_PK_MINB 2  // resident CTAs per SM the packed variant is compiled for
#endif
#ifndef FC_PK_K
#define FC_PK_K 3
#endif
#ifndef FC_PK_IDX_MINB
#define FC_PK_IDX_MINB 2  // resident CTAs per SM the indexed variant is compiled for
#endif
#ifndef FC_PK_IDX_CS
#define FC_PK_IDX_CS 0  // experiment: streaming (evict-first) loads beside the cached table
#endif

template <int L, int C, bool IDX>
__global__ void __launch_bounds__(256, IDX ? FC_PK_IDX_MINB : FC_PK_MINB) k_row_fwd_pk(Geo g, RowGeo rg, Coef Cf, InArgs ia, const RhsState* st,
                                                       const double2* __restrict__ tw, int npk,
                                                       const __grid_constant__ CUtensorMap tmP) {
  constexpr int TP = RegTP<L>::value;
  constexpr int NSYM = C * (C + 1) / 2;
  constexpr int hl = (L + 1) / 2;
  extern __shared__ __align__(128) unsigned char smraw[];
  double2* sm = reinterpret_cast<double2*>(smraw);
  const int B = 2 * npk;
  const int ntiles = (rg.np + B - 1) / B;
  int64_t bid = blockIdx.x;
  const int tile = bid % ntiles; bid /= ntiles;
  const int o = bid % rg.no;
  const int r = (int)(bid / rg.no);
  if (!rhs_active(st, r)) return;
  const int row0 = tile * B;
  const int nrows = min(B, rg.np - row0);
  const int mode = ia.mode;
  const InEval ev = make_eval(ia, g, Cf, st, r, 0);  // per-RHS scalars (first, beta, alpha, xacc, s)
  const int64_t N = g.N;
  const int64_t vbase = ((int64_t)o * rg.np + row0) * L;
  const int64_t rbase = (int64_t)r * C * N;
  double* ys = reinterpret_cast<double*>(sm);  // [C][B][L]
  const int n = nrows * L;

  // ---- 1. pointwise, all components per voxel ------------------------------
  double Ev[C], M0[C][C];
#pragma unroll
  for (int b = 0; b < C; ++b) {
    Ev[b] = mode == IN_CONST ? pick(ia.E, r, b) : 0.0;
#pragma unroll
    for (int a = 0; a < C; ++a) M0[a][b] = mode == IN_FP ? pick3(ia.A0, a, b) : 0.0;
  }
  const bool use_u = mode != IN_CONST;
  const bool use_p = mode == IN_PNEW && !ev.first;
  const double* __restrict__ U = ia.u + rbase + vbase;
  const double* __restrict__ PO = ia.p_old + rbase + vbase;
  const double* __restrict__ A = Cf.A + vbase;
  // phase-indexed coefficients: one 2-byte label per voxel and the phases' packed
  // tensors from a table that stays in L1 (same values, 2 instead of 8 NSYM bytes
  // per voxel from HBM)
  const uint16_t* __restrict__ LB = IDX ? Cf.lab + vbase : nullptr;
  const double* __restrict__ TB = Cf.tab;
  const int nph = Cf.nph;
#if FC_PK_IDX_SMEM
  if (IDX && nph * NSYM * 8 <= 32768) {
    double* TS = reinterpret_cast<double*>(smraw + pk_smem(L, C, npk, rg.nbox, rg.boxK));
    for (int i = threadIdx.x; i < nph * NSYM; i += blockDim.x) TS[i] = __ldg(Cf.tab + i);
    __syncthreads();
    TB = TS;
  }
#endif
  double* __restrict__ PN = ia.p_new + rbase + vbase;
  double* __restrict__ X = ev.xacc != nullptr ? ev.xacc + rbase + vbase : nullptr;
  trace_stamp(1, 0);
  // voxels per thread in flight (all their loads issued first).  Measured at 729^3
  // (profiles/r02z_ab_pk_k.txt): 2 -> 13.73 ms, 3 -> 13.37 ms (a row pair of 729 is
  // exactly two rounds of 243 threads), 6 -> 32.9 ms (spills)
  constexpr int K = IDX ? FC_PK_IDX_K : FC_PK_K;
  for (int e0 = threadIdx.x; e0 < n; e0 += K * blockDim.x) {
    double u[K][C], po[K][C], xo[K][C], am[K][NSYM];
    // indexed: the labels first, so their latency hides behind the field loads and
    // the table reads (L1 hits) find them ready
    int ph[K];
    if constexpr (IDX) {
#pragma unroll
      for (int k = 0; k < K; ++k) {
        const int e = e0 + k * blockDim.x;
        ph[k] = e < n ? (int)__ldg(LB + e) : 0;
      }
    }
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const int e = e0 + k * blockDim.x;
      const bool ok = e < n;
#pragma unroll
      for (int b = 0; b < C; ++b) {
        if constexpr (IDX && FC_PK_IDX_CS) {
          u[k][b] = (ok && use_u) ? __ldcs(U + b * N + e) : Ev[b];
          po[k][b] = (ok && use_p) ? __ldcs(PO + b * N + e) : 0.0;
        } else {
          u[k][b] = (ok && use_u) ? __ldg(U + b * N + e) : Ev[b];
          po[k][b] = (ok && use_p) ? __ldg(PO + b * N + e) : 0.0;
        }
        xo[k][b] = (ok && X != nullptr) ? X[b * N + e] : 0.0;
      }
      if constexpr (!IDX) {
#pragma unroll
        for (int m = 0; m < NSYM; ++m) am[k][m] = ok ? __ldg(A + m * N + e) : 0.0;
      }
    }
    if constexpr (IDX && !FC_PK_IDX_LATE) {
#pragma unroll
      for (int k = 0; k < K; ++k)
#pragma unroll
        for (int m = 0; m < NSYM; ++m) am[k][m] = FC_PK_IDX_SMEM ? TB[m * nph + ph[k]] : __ldg(TB + m * nph + ph[k]);
    }
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const int e = e0 + k * blockDim.x;
      if (e >= n) break;
      if constexpr (IDX && FC_PK_IDX_LATE) {
#pragma unroll
        for (int m = 0; m < NSYM; ++m) am[k][m] = __ldg(TB + m * nph + ph[k]);
      }
      double x[C];
#pragma unroll
      for (int b = 0; b < C; ++b) {
        double xb = u[k][b];
        if (mode == IN_PNEW) {
          if (use_p) {
            xb = __dadd_rn(xb, __dmul_rn(ev.beta, po[k][b]));
            if (X != nullptr) X[b * N + e] = __dadd_rn(xo[k][b], __dmul_rn(ev.alpha, po[k][b]));
          }
          PN[b * N + e] = xb;
        }
        x[b] = xb;
      }
#pragma unroll
      for (int a = 0; a < C; ++a) {
        double acc = 0.0;
#pragma unroll
        for (int b = 0; b < C; ++b) {
          double Aab = am[k][pidx(C, a, b)];
          if (mode == IN_FP) Aab = __dsub_rn(Aab, M0[a][b]);
          acc = __dadd_rn(acc, __dmul_rn(Aab, x[b]));
        }
        if (mode != IN_FP && ev.s != 1.0) acc = __dmul_rn(ev.s, acc);
        ys[a * B * L + e] = acc;
      }
    }
  }
  __syncthreads();
  trace_stamp(1, 1);

  // ---- 2. row FFT of component a, pencil p (rows 2p, 2p+1) -------------------
  const int per_a = npk * TP;
  const int a = threadIdx.x / per_a;
  const int t = threadIdx.x - a * per_a;
  const int p = t / TP;
  const int j = t - p * TP;
  const int re = 2 * p, ro = 2 * p + 1;
  double2 v[1][9];
#pragma unroll
  for (int s = 0; s < 9; ++s) {
    const int i = j + s * TP;
    v[0][s] = make_double2(re < nrows ? ys[(a * B + re) * L + i] : 0.0, ro < nrows ? ys[(a * B + ro) * L + i] : 0.0);
  }
  // the pencil's exchange buffer is its own rows of ys (read above by this
  // pencil's threads only; fft_reg syncs before its first write)
  double2* smp = sm + (size_t)(a * npk + p) * L;
  fft_reg<L, 1, false>(v, smp, L, j, tw);
  trace_stamp(1, 2);
  __syncthreads();
#pragma unroll
  for (int s = 0; s < 9; ++s) smp[j + s * TP] = v[0][s];
  __syncthreads();
  // split Z = Ye + i Yo into Y_a[k][row], then one TMA box store per (component, box)
  const int npairs = (nrows + 1) >> 1;
  double2* Y = sm + ((((size_t)C * npk * L * 16 + 127) & ~(size_t)127) >> 4);
  const int per_c = hl * npairs;
  const int ybox = rg.nbox * rg.boxK * B;
  for (int idx = threadIdx.x; idx < C * per_c; idx += blockDim.x) {
    const int aa = idx / per_c;
    const int rem = idx - aa * per_c;
    const int k = rem / npairs;
    const int pr = rem - k * npairs;
    const double2* z = sm + (size_t)(aa * npk + pr) * L;
    const double2 zk = z[k];
    const double2 zm = z[k == 0 ? 0 : L - k];
    double2* Ya = Y + (size_t)aa * ybox;
    Ya[k * B + 2 * pr] = make_double2(0.5 * (zk.x + zm.x), 0.5 * (zk.y - zm.y));
    Ya[k * B + 2 * pr + 1] = make_double2(0.5 * (zk.y + zm.y), 0.5 * (zm.x - zk.x));
  }
  fence_proxy_async();
  __syncthreads();
  if (threadIdx.x == 0) {
#pragma unroll
    for (int aa = 0; aa < C; ++aa) {
      const int c2 = (r * C + aa) * rg.no + o;
      for (int b = 0; b < rg.nbox; ++b)
        tma_store_3d(&tmP, 2 * row0, b * rg.boxK, c2, Y + (size_t)aa * ybox + (size_t)b * rg.boxK * B);
    }
    bulk_commit();
    trace_stamp(1, 3);
    bulk_wait_read0();
    trace_stamp(1, 4);
    trace_stamp(1, 5);
  }
}

}  // namespace fc
