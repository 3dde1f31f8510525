// Register-resident radix-9 Stockham FFT for L = 3^k (9 <= L <= 2187).
//
// The BASELINE grids (81, 243, 729, 2187) are powers of three.  For these the
// transform is planned at compile time: TP = L/9 threads per pencil, each
// thread holding 9 complex values in registers; passes are radix-9 (3 x 3
// with constant internal twiddles) plus one radix-3 tail pass when k is odd.
// Data enter and leave in natural order with thread j holding elements
// j + s*TP, s = 0..8, so a pencil is loaded from / stored to HBM directly
// (coalesced over j) and the only shared-memory traffic is one exchange
// between consecutive passes (2 for L = 729, 3 for L = 2187), instead of a
// full smem round trip per radix pass.
//
// Pass S (radix 9, Ns = 9^S) reads x[j + r*TP], multiplies element r by
// w_L^{(j mod Ns) r L/(9 Ns)} (S > 0), runs the 9-point DFT and writes
// y[(j - j mod Ns) * 9 + j mod Ns + r * Ns].  The radix-3 tail (Ns = L/3)
// handles butterflies b = j + m*TP and writes back in place.  Inter-pass
// twiddles come from a compact per-length table (tw layout documented in
// fc_engine.cu: reg_twiddles), read coalesced through the read-only path.
#pragma once
#include "fc_fft.cuh"

namespace fc {

__host__ __device__ constexpr int ipow9(int s) { return s == 0 ? 1 : 9 * ipow9(s - 1); }
__host__ __device__ constexpr int ilog3(int L) { return L <= 1 ? 0 : 1 + ilog3(L / 3); }

template <int L>
struct R9 {
  static constexpr int K = ilog3(L);
  static constexpr int NP9 = K / 2;       // radix-9 passes
  static constexpr bool TAIL = (K % 2) == 1;
  static constexpr int TP = L / 9;        // threads per pencil
  static_assert(ipow9(NP9) * (TAIL ? 3 : 1) == L, "L must be a power of 3");
  static_assert(L >= 9, "L >= 9");
  // offset of pass S (S >= 1) twiddle block: sum_{t=1}^{S-1} 8 * 9^t
  __host__ __device__ static constexpr int off9(int S) { return S <= 1 ? 0 : off9(S - 1) + 8 * ipow9(S - 1); }
  static constexpr int offT = off9(NP9);  // tail block: 2 * (L/3) entries
  static constexpr int table = offT + (TAIL ? 2 * (L / 3) : 0);
};

// --- one radix-9 pass on CPT pencils held by this thread ---------------------
template <int L, int CPT, bool INV, int S>
__device__ __forceinline__ void r9_compute(double2 (&v)[CPT][9], int j, const double2* __restrict__ tw) {
  constexpr int Ns = ipow9(S);
  if constexpr (S > 0) {
    const int k = j % Ns;
    double2 w[8];
#pragma unroll
    for (int r = 1; r < 9; ++r) {
      w[r - 1] = __ldg(tw + R9<L>::off9(S) + (r - 1) * Ns + k);
      if (INV) w[r - 1].y = -w[r - 1].y;
    }
#pragma unroll
    for (int c = 0; c < CPT; ++c)
#pragma unroll
      for (int r = 1; r < 9; ++r) v[c][r] = cmul(v[c][r], w[r - 1]);
  }
#pragma unroll
  for (int c = 0; c < CPT; ++c) bfly9<INV>(v[c]);
}

// Exchange after pass S: write Stockham output positions, read natural j + s*TP.
// sm points at this thread's first pencil; pencils of the thread are pstride apart.
template <int L, int CPT, int S>
__device__ __forceinline__ void r9_exchange(double2 (&v)[CPT][9], double2* sm, int pstride, int j) {
  constexpr int Ns = ipow9(S);
  constexpr int TP = R9<L>::TP;
  const int k = j % Ns;
  const int base = (j - k) * 9 + k;
  __syncthreads();
#pragma unroll
  for (int c = 0; c < CPT; ++c)
#pragma unroll
    for (int r = 0; r < 9; ++r) sm[c * pstride + base + r * Ns] = v[c][r];
  __syncthreads();
#pragma unroll
  for (int c = 0; c < CPT; ++c)
#pragma unroll
    for (int s = 0; s < 9; ++s) v[c][s] = sm[c * pstride + j + s * TP];
}

template <int L, int CPT, bool INV>
__device__ __forceinline__ void r3_tail(double2 (&v)[CPT][9], int j, const double2* __restrict__ tw) {
  constexpr int TP = R9<L>::TP;
  constexpr int L3 = L / 3;
#pragma unroll
  for (int m = 0; m < 3; ++m) {
    const int b = j + m * TP;
    double2 w1 = __ldg(tw + R9<L>::offT + b);
    double2 w2 = __ldg(tw + R9<L>::offT + L3 + b);
    if (INV) { w1.y = -w1.y; w2.y = -w2.y; }
#pragma unroll
    for (int c = 0; c < CPT; ++c) {
      if (b != 0) {
        v[c][m + 3] = cmul(v[c][m + 3], w1);
        v[c][m + 6] = cmul(v[c][m + 6], w2);
      }
      bfly3<INV>(v[c][m], v[c][m + 3], v[c][m + 6]);
    }
  }
}

template <int L, int CPT, bool INV, int S>
struct R9Driver {
  __device__ __forceinline__ static void run(double2 (&v)[CPT][9], double2* sm, int pstride, int j,
                                             const double2* __restrict__ tw) {
    r9_compute<L, CPT, INV, S>(v, j, tw);
    if constexpr (S + 1 < R9<L>::NP9 || R9<L>::TAIL) r9_exchange<L, CPT, S>(v, sm, pstride, j);
    if constexpr (S + 1 < R9<L>::NP9) R9Driver<L, CPT, INV, S + 1>::run(v, sm, pstride, j, tw);
  }
};

__host__ __device__ constexpr bool is_pow3(int L) { return L == 1 || (L % 3 == 0 && is_pow3(L / 3)); }
// Register-path lengths: 3^k (9 .. 2187) and 5 * 3^k (45 .. 1215, the cfg5 axis)
__host__ __device__ constexpr bool is_reg_len(int L) {
  return (L >= 9 && L <= 2187 && is_pow3(L)) || (L % 5 == 0 && L / 5 >= 9 && L / 5 <= 243 && is_pow3(L / 5));
}
// threads per pencil: every register-path length holds 9 elements per thread
template <int L>
struct RegTP {
  static_assert(is_reg_len(L), "register FFT length");
  static constexpr int value = L / 9;
};
// twiddle-table entries of length L (3^k: R9 table; 5 M: M's table + 4 M combine twiddles)
template <int L>
__host__ __device__ constexpr int reg_table() {
  if constexpr (is_pow3(L)) return R9<L>::table;
  else return R9<L / 5>::table + 4 * (L / 5);
}

template <int L, int CPT, bool INV>
__device__ __forceinline__ void fft_reg(double2 (&v)[CPT][9], double2* sm, int pstride, int j,
                                        const double2* __restrict__ tw);

// L = 5 M (M = 3^k >= 9), decimation in time.  Thread j's elements j + s TP all
// lie in the sub-sequence r = j mod 5 (TP = L/9 is a multiple of 5), at
// positions j' + s TP/5 with j' = j / 5: the natural register layout of an
// M-point transform.  Stage A: five M-point register FFTs side by side (group r
// uses sm + r M as its exchange buffer).  Stage B, through shared memory in
// place: X[k2 + M k1] = sum_r w5^{r k1} (w_L^{r k2} Y_r[k2]), k2 < M (radix-5
// butterflies; constant input still gives exact zeros: the sub-transforms leave
// only Y_r[0] = M x, and the k2 = 0 butterfly of five equal values is exact).
template <int L, int CPT, bool INV>
__device__ __forceinline__ void fft_reg_5m(double2 (&v)[CPT][9], double2* sm, int pstride, int j,
                                           const double2* __restrict__ tw) {
  constexpr int M = L / 5;
  constexpr int TP = L / 9;
  const int r = j % 5;
  fft_reg<M, CPT, INV>(v, sm + r * M, pstride, j / 5, tw);
  __syncthreads();
#pragma unroll
  for (int c = 0; c < CPT; ++c)
#pragma unroll
    for (int s = 0; s < 9; ++s) sm[c * pstride + r * M + j / 5 + s * (TP / 5)] = v[c][s];
  __syncthreads();
  const double2* twc = tw + R9<M>::table;  // w_L^{r k2} at twc[(r - 1) M + k2]
  for (int k2 = j; k2 < M; k2 += TP) {
    double2 w[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      w[q] = __ldg(twc + q * M + k2);
      if (INV) w[q].y = -w[q].y;
    }
#pragma unroll
    for (int c = 0; c < CPT; ++c) {
      double2* b = sm + c * pstride + k2;
      double2 x0 = b[0], x1 = b[M], x2 = b[2 * M], x3 = b[3 * M], x4 = b[4 * M];
      if (k2 != 0) {
        x1 = cmul(x1, w[0]);
        x2 = cmul(x2, w[1]);
        x3 = cmul(x3, w[2]);
        x4 = cmul(x4, w[3]);
      }
      bfly5<INV>(x0, x1, x2, x3, x4);
      b[0] = x0;
      b[M] = x1;
      b[2 * M] = x2;
      b[3 * M] = x3;
      b[4 * M] = x4;
    }
  }
  __syncthreads();
#pragma unroll
  for (int c = 0; c < CPT; ++c)
#pragma unroll
    for (int s = 0; s < 9; ++s) v[c][s] = sm[c * pstride + j + s * TP];
}

// Full transform of CPT pencils: on entry v[c][s] = x_c[j + s*TP], on exit X_c[j + s*TP].
// All threads of the block must call it (it contains block barriers); its last
// smem access is followed by no barrier, so callers reusing sm must sync first.
template <int L, int CPT, bool INV>
__device__ __forceinline__ void fft_reg(double2 (&v)[CPT][9], double2* sm, int pstride, int j,
                                        const double2* __restrict__ tw) {
  if constexpr (is_pow3(L)) {
    R9Driver<L, CPT, INV, 0>::run(v, sm, pstride, j, tw);
    if constexpr (R9<L>::TAIL) r3_tail<L, CPT, INV>(v, j, tw);
  } else {
    fft_reg_5m<L, CPT, INV>(v, sm, pstride, j, tw);
  }
}

}  // namespace fc
