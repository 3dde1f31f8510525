// "Fat-thread" register FFT for L = 3^k (27 <= L <= 2187): 27 complex values per
// thread, TP = L/27 threads per pencil.
//
// Against the 9-per-thread transform of fc_fft_reg.cuh this halves the
// shared-memory exchanges (one for L = 243 / 729, two for L = 2187) and makes a
// pencil small enough in threads that one warp (L <= 729: 27 of its 32 lanes) or
// one three-warp group (L = 2187: 81 of 96 lanes) owns it: the exchanges then
// need a warp barrier / a named barrier of the group only, never the CTA, so the
// warps of a CTA run as independent pipelines.
//
// Same Stockham scheme and natural-order register layout as fc_fft_reg.cuh
// (thread j holds x[j + s TP], s = 0..26, on entry and X[j + s TP] on exit):
// radix-27 passes (9 x 3 with constant internal twiddles w27^m) and a radix-3 or
// radix-9 tail when k is not a multiple of 3.  Every butterfly is in difference
// form, so a constant input still gives exact zeros in all non-DC modes.
#pragma once
#include "fc_fft_reg.cuh"

namespace fc {

template <int L>
struct R27 {
  static constexpr int K = ilog3(L);
  static constexpr int NP = K / 3;                                      // radix-27 passes
  static constexpr int TAIL = K % 3 == 0 ? 1 : (K % 3 == 1 ? 3 : 9);    // tail radix (1: none)
  static constexpr int TP = L / 27;                                     // threads per pencil
  static_assert(is_pow3(L) && L >= 27 && L <= 2187 * 9, "fat FFT length");
  static_assert(NP == 1 || NP == 2, "one or two radix-27 passes");
  // twiddle table: pass 1 (Ns = 27): w_L^{k r L/729} at [(r - 1) 27 + k], r = 1..26, k < 27;
  // tail (radix T, Ns = L/T): w_L^{b q} at offT + (q - 1) (L/T) + b, q = 1..T-1, b < L/T
  static constexpr int offT = NP >= 2 ? 26 * 27 : 0;
  static constexpr int table = offT + (TAIL > 1 ? (TAIL - 1) * (L / TAIL) : 0);
};

__host__ __device__ constexpr bool is_fat_len(int L) { return is_pow3(L) && L >= 27 && L <= 2187; }

// cos / sin (2 pi m / 27), m = 1..16
__device__ __forceinline__ constexpr double c27(int m) {
  switch (m) {
    case 1: return 0.9730448705798238388329;
    case 2: return 0.8936326403234122481926;
    case 3: return 0.7660444431189780352024;
    case 4: return 0.5971585917027861648519;
    case 5: return 0.396079766039156823696;
    case 6: return 0.1736481776669303488517;
    case 7: return -0.05814482891047582853875;
    case 8: return -0.2868032327110902531033;
    case 9: return -0.5;
    case 10: return -0.6862416378687335857296;
    case 11: return -0.8354878114129364196538;
    case 12: return -0.9396926207859083840541;
    case 13: return -0.9932383577419429885479;
    case 14: return -0.9932383577419429885479;
    case 15: return -0.9396926207859083840541;
    case 16: return -0.8354878114129364196538;
    default: return 1.0;
  }
}
__device__ __forceinline__ constexpr double s27(int m) {
  switch (m) {
    case 1: return 0.2306158707424401784502;
    case 2: return 0.448799180200462172785;
    case 3: return 0.6427876096865393263226;
    case 4: return 0.8021231927550437850833;
    case 5: return 0.918216106880274014759;
    case 6: return 0.9848077530122080593667;
    case 7: return 0.9983081582712682080478;
    case 8: return 0.9579895123154888744374;
    case 9: return 0.8660254037844386467637;
    case 10: return 0.7273736415730486959872;
    case 11: return 0.5495089780708060352628;
    case 12: return 0.3420201433256687330441;
    case 13: return 0.1160929141252302296757;
    case 14: return -0.1160929141252302296757;
    case 15: return -0.3420201433256687330441;
    case 16: return -0.5495089780708060352628;
    default: return 0.0;
  }
}

// 27-point DFT in registers, natural order in and out:
// X[k1 + 9 k2] = sum_{n2<3} w3^{n2 k2} w27^{n2 k1} DFT9_{n1}(x[3 n1 + n2])[k1]
template <bool INV>
__device__ __forceinline__ void bfly27(double2 (&v)[27]) {
  double2 t[3][9];
#pragma unroll
  for (int n2 = 0; n2 < 3; ++n2)
#pragma unroll
    for (int n1 = 0; n1 < 9; ++n1) t[n2][n1] = v[3 * n1 + n2];
  bfly9<INV>(t[0]);
  bfly9<INV>(t[1]);
  bfly9<INV>(t[2]);
  constexpr double sg = INV ? 1.0 : -1.0;
#pragma unroll
  for (int k1 = 1; k1 < 9; ++k1) {
    t[1][k1] = cmul(t[1][k1], make_double2(c27(k1), sg * s27(k1)));
    t[2][k1] = cmul(t[2][k1], make_double2(c27(2 * k1), sg * s27(2 * k1)));
  }
#pragma unroll
  for (int k1 = 0; k1 < 9; ++k1) {
    bfly3<INV>(t[0][k1], t[1][k1], t[2][k1]);
    v[k1] = t[0][k1];
    v[k1 + 9] = t[1][k1];
    v[k1 + 18] = t[2][k1];
  }
}

// Barriers of the thread group that owns a pencil.
struct SyncWarp {
  __device__ __forceinline__ void operator()() const { __syncwarp(); }
};
struct SyncGroup {  // named barrier `id` over n threads (n a multiple of 32)
  int id, n;
  __device__ __forceinline__ void operator()() const { asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(n) : "memory"); }
};

// Exchange through the group's buffer: v[r] -> position wbase + r wstride, then
// v[s] <- position j + s TP.  HALF: real and imaginary parts go through one
// after the other, so the buffer holds L doubles instead of L complex (the
// 8-byte accesses are conflict-free for the same strides).
template <int L, bool HALF, typename Sync>
__device__ __forceinline__ void fat_exchange(double2 (&v)[27], double2* sm, int wbase, int wstride, int j, bool act,
                                             const Sync& sync) {
  constexpr int TP = R27<L>::TP;
  if constexpr (!HALF) {
    sync();  // earlier readers of sm are done
    if (act) {
#pragma unroll
      for (int r = 0; r < 27; ++r) sm[wbase + r * wstride] = v[r];
    }
    sync();
    if (act) {
#pragma unroll
      for (int s = 0; s < 27; ++s) v[s] = sm[j + s * TP];
    }
  } else {
    double* sd = reinterpret_cast<double*>(sm);
    sync();
    if (act) {
#pragma unroll
      for (int r = 0; r < 27; ++r) sd[wbase + r * wstride] = v[r].x;
    }
    sync();
    if (act) {
#pragma unroll
      for (int s = 0; s < 27; ++s) v[s].x = sd[j + s * TP];
    }
    sync();
    if (act) {
#pragma unroll
      for (int r = 0; r < 27; ++r) sd[wbase + r * wstride] = v[r].y;
    }
    sync();
    if (act) {
#pragma unroll
      for (int s = 0; s < 27; ++s) v[s].y = sd[j + s * TP];
    }
  }
}

// Full transform of one pencil.  j: index of the thread within the pencil's group;
// threads with j >= TP (act == false) carry zeros, take part in the barriers and
// touch no memory.  sm: the group's exchange buffer of L complex (HALF: L doubles).  The last
// shared-memory access is not followed by a barrier.
template <int L, bool INV, bool HALF = false, typename Sync>
__device__ __forceinline__ void fft_fat(double2 (&v)[27], double2* sm, int j, bool act, const double2* __restrict__ tw,
                                        const Sync& sync) {
  using P = R27<L>;
  constexpr int TP = P::TP;
  bfly27<INV>(v);  // pass 0 (Ns = 1)
  if constexpr (L == 27) return;
  fat_exchange<L, HALF>(v, sm, 27 * j, 1, j, act, sync);
  if constexpr (P::NP >= 2) {  // pass 1 (Ns = 27)
    const int k = j % 27;
    if (act) {
#pragma unroll
      for (int r = 1; r < 27; ++r) {
        double2 w = __ldg(tw + (r - 1) * 27 + k);
        if (INV) w.y = -w.y;
        v[r] = cmul(v[r], w);
      }
    }
    bfly27<INV>(v);
    if constexpr (P::TAIL > 1) {
      fat_exchange<L, HALF>(v, sm, (j - k) * 27 + k, 27, j, act, sync);
    }
  }
  if constexpr (P::TAIL == 3) {  // butterflies b = j + m TP over elements s = m, m + 9, m + 18
    constexpr int L3 = L / 3;
#pragma unroll
    for (int m = 0; m < 9; ++m) {
      const int b = act ? j + m * TP : 0;
      double2 w1 = __ldg(tw + P::offT + b);
      double2 w2 = __ldg(tw + P::offT + L3 + b);
      if (INV) { w1.y = -w1.y; w2.y = -w2.y; }
      v[m + 9] = cmul(v[m + 9], w1);
      v[m + 18] = cmul(v[m + 18], w2);
      bfly3<INV>(v[m], v[m + 9], v[m + 18]);
    }
  } else if constexpr (P::TAIL == 9) {  // butterflies b = j + m TP over elements s = m + 3 q
    constexpr int L9 = L / 9;
#pragma unroll
    for (int m = 0; m < 3; ++m) {
      const int b = act ? j + m * TP : 0;
      double2 t[9];
      t[0] = v[m];
#pragma unroll
      for (int q = 1; q < 9; ++q) {
        double2 w = __ldg(tw + P::offT + (q - 1) * L9 + b);
        if (INV) w.y = -w.y;
        t[q] = cmul(v[m + 3 * q], w);
      }
      bfly9<INV>(t);
#pragma unroll
      for (int q = 0; q < 9; ++q) v[m + 3 * q] = t[q];
    }
  }
}

}  // namespace fc
