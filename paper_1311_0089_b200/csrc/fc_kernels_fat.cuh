// Outer sweep on the fat-thread FFT (fc_fft_fat.cuh), single slab.
//
// One warp (L <= 729) or one three-warp group (L = 2187) owns a pencil from the
// global load to the global store.  Loads and stores go straight between HBM
// and registers (27 x 16 B per thread and component, runs of TP x 16 B
// contiguous bytes), shared memory holds only the transform's exchange buffer
// and one parked spectrum per pencil, and the only barriers are those of the
// group: no CTA-wide barrier, no staging pass, about a third of the
// shared-memory traffic of k_outer_seq.
//
// d = 2 and d = 3 share the folded form of fc_kernels_reg.cuh (g3_*): along an
// axis-0 pencil xi_1 (and xi_2) are constants, so with u = xi_1 v_1 (+ xi_2 v_2)
//   q = (xi_0 F0 v_0 + F0 u) / den,  out_0 = F0^-1(xi_0 q),  out_a = xi_a F0^-1(q).
#pragma once
#include "fc_fft_fat.cuh"
#include "fc_kernels_pipe.cuh"

namespace fc {

template <int L>
struct FatGeo {
  static constexpr int TP = R27<L>::TP;
  static constexpr int PPG = TP <= 27 ? 27 / TP : 1;          // pencils per group
  static constexpr int GT = TP <= 27 ? 32 : ((TP + 31) / 32) * 32;  // threads per group
  // per pencil: the parked spectrum (L complex) and the exchange buffer (L doubles: the
  // transform exchanges real and imaginary parts one after the other)
  static constexpr size_t pencil_bytes = (size_t)L * sizeof(double2) + (((size_t)L * sizeof(double) + 15) & ~(size_t)15);
  static constexpr size_t group_bytes = (size_t)PPG * pencil_bytes;
};

constexpr int kFatThreads = 96;  // 3 one-warp groups or 1 three-warp group

__device__ __forceinline__ double2 conj2(double2 a) { return make_double2(a.x, -a.y); }

// The four transforms of a pencil run through ONE copy of the forward transform
// (a loop that is not unrolled; the inverse is conj F conj, bitwise the mirrored
// arithmetic), so the kernel's code stays small enough for the instruction cache
// with every warp at a different place in it.
template <int L, int C>
__global__ void __launch_bounds__(kFatThreads, 4) k_outer_fat(Geo g, OuterGeo og, const RhsState* st,
                                                               const double2* __restrict__ tw,
                                                               double2* __restrict__ W) {
  using F = FatGeo<L>;
  constexpr int TP = F::TP;
  extern __shared__ __align__(16) unsigned char smraw[];
  const int r = blockIdx.y;
  if (!rhs_active(st, r)) return;
  constexpr int NG = kFatThreads / F::GT;  // groups per CTA
  const int grp = threadIdx.x / F::GT;
  const int t = threadIdx.x - grp * F::GT;
  const bool act = t < F::PPG * TP;
  const int pp = act ? t / TP : 0;
  const int j = act ? t - pp * TP : 0;
  const int64_t ql = ((int64_t)blockIdx.x * NG + grp) * F::PPG + pp;
  const bool live = act && ql < og.Q;
  double2* park = reinterpret_cast<double2*>(smraw + ((size_t)grp * F::PPG + pp) * F::pencil_bytes);
  double2* ex = park + L;  // L doubles
  const SyncGroup gsync{1 + grp, F::GT};
  const SyncWarp wsync{};
  const int qi = live ? (int)ql : 0;
  double xi1, xi2 = 0.0;
  if constexpr (C == 3) {
    const int k2 = qi / og.n1, k1 = qi - k2 * og.n1;
    xi1 = g.xi[1][k1];
    xi2 = g.xi[2][k2];
  } else {
    xi1 = g.xi[1][qi];
  }
  double2* p0 = W + ((int64_t)(r * C + 0) * og.Q + qi) * L + j;
  double2* p1 = W + ((int64_t)(r * C + 1) * og.Q + qi) * L + j;
  double2* p2 = W + ((int64_t)(r * C + (C - 1)) * og.Q + qi) * L + j;
  if (live) {  // the pencils of the second transform on their way to L2 during the first
    constexpr int per = 128 / (int)sizeof(double2);  // complex per 128-byte line
    for (int i = j * per; i < L; i += TP * per) {
      prefetch_l2(p1 - j + i);
      if constexpr (C == 3) prefetch_l2(p2 - j + i);
    }
  }
  const double2 zero = make_double2(0.0, 0.0);
  double2 v[27];
#pragma unroll 1
  for (int ph = 0; ph < 4; ++ph) {
    // 0: F0 v_0 -> parked; 1: F0 u, Gamma_hat per mode: (F0 v_0, F0 u) -> (xi_0 q, q);
    // 2: F0^-1 q -> components 1.. scaled by xi_a; 3: F0^-1 (xi_0 q) -> component 0
    if (ph == 0) {
#pragma unroll
      for (int s = 0; s < 27; ++s) v[s] = live ? p0[s * TP] : zero;
    } else if (ph == 1) {
#pragma unroll
      for (int s = 0; s < 27; ++s) {
        if constexpr (C == 3) v[s] = live ? g3_fold(xi1, xi2, p1[s * TP], p2[s * TP]) : zero;
        else v[s] = live ? g3_scale(xi1, p1[s * TP]) : zero;
      }
    } else if (ph == 3) {
      if (live) {
#pragma unroll
        for (int s = 0; s < 27; ++s) v[s] = park[j + s * TP];
      }
    }
    if constexpr (F::GT == 32) fft_fat<L, false, true>(v, ex, j, live, tw, wsync);
    else fft_fat<L, false, true>(v, ex, j, live, tw, gsync);
    if (!live) continue;
    if (ph == 0) {  // every thread parks and later reads its own elements
#pragma unroll
      for (int s = 0; s < 27; ++s) park[j + s * TP] = v[s];
    } else if (ph == 1) {
#pragma unroll
      for (int s = 0; s < 27; ++s) {
        const int i0 = j + s * TP;
        double2 t0 = park[i0];
        g3_mode(og, g.xi[0][i0], xi1, xi2, ql == 0 && i0 == 0, t0, v[s]);
        park[i0] = conj2(t0);
        v[s] = conj2(v[s]);
      }
    } else if (ph == 2) {
#pragma unroll
      for (int s = 0; s < 27; ++s) {
        p1[s * TP] = g3_scale(xi1, conj2(v[s]));
        if constexpr (C == 3) p2[s * TP] = g3_scale(xi2, conj2(v[s]));
      }
    } else {
#pragma unroll
      for (int s = 0; s < 27; ++s) p0[s * TP] = conj2(v[s]);
    }
  }
}

}  // namespace fc
