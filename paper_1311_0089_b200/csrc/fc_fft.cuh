// Odd-length fp64 FFT building blocks staged in shared memory (sm_100a).
//
// Replaces the pocketfft C2C transforms the reference reaches through
// np.fft.fftn / ifftn (solver.py:114-122).  Lengths are any odd integer; the
// factor plan uses specialised radix-3/5/9 butterflies and a generic odd
// prime butterfly.  Every butterfly is written in "difference" form
// (X_k = sum_{j>=1} (x_j - x_0) w^{jk} for k != 0), so a constant input gives
// EXACT zeros in every non-DC mode, as pocketfft does; the reference's
// homogeneous-medium acceptance test (test_acceptance.py:32-44: solution
// exactly 0.0) depends on it.
//
// Algorithm: Stockham autosort, decimation in time.  Pass s with radix R and
// Ns = prod(previous radices) reads x[j + r*L/R], multiplies by the twiddle
// w_L^{(j mod Ns) * r * L/(Ns*R)}, runs a length-R DFT and writes
// y[(j - j mod Ns)*R + (j mod Ns) + r*Ns].  Twiddles come from one table of
// the L-th roots of unity computed on the host in extended precision.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace fc {

constexpr int kMaxFactors = 24;

struct FftPlan {
  int L;                    // transform length (odd)
  int nf;                   // number of passes
  int f[kMaxFactors];       // radix of each pass (3, 5, 9 or any odd prime)
  const double2* roots;     // roots[t] = exp(-2 pi i t / L), t in [0, L)
};

__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 cscale(double s, double2 a) { return make_double2(s * a.x, s * a.y); }
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
// i * s * a
__device__ __forceinline__ double2 cimul(double s, double2 a) { return make_double2(-s * a.y, s * a.x); }

// Twiddle w^t for the transform direction (forward: table, inverse: conjugate).
template <bool INV>
__device__ __forceinline__ double2 root(const double2* roots, int t) {
  double2 w = __ldg(roots + t);
  if (INV) w.y = -w.y;
  return w;
}

// ---- radix-3 -------------------------------------------------------------
// X1 = x0 - (x1+x2)/2 + sgn*i*(sqrt3/2)(x1-x2), sgn = -1 forward, +1 inverse.
template <bool INV>
__device__ __forceinline__ void bfly3(double2& x0, double2& x1, double2& x2) {
  const double s = INV ? 0.86602540378443864676 : -0.86602540378443864676;
  double2 t1 = cadd(x1, x2);
  double2 t2 = make_double2(fma(-0.5, t1.x, x0.x), fma(-0.5, t1.y, x0.y));
  double2 d = csub(x1, x2);
  x0 = cadd(x0, t1);
  // t2 +- i s d as fused multiply-adds (constant input: d = 0, t2 = 0 exactly)
  x1 = make_double2(fma(-s, d.y, t2.x), fma(s, d.x, t2.y));
  x2 = make_double2(fma(s, d.y, t2.x), fma(-s, d.x, t2.y));
}

// ---- radix-5 -------------------------------------------------------------
template <bool INV>
__device__ __forceinline__ void bfly5(double2& x0, double2& x1, double2& x2, double2& x3, double2& x4) {
  const double c = 0.55901699437494742410;   // (cos 72 - cos 144) / 2 = sqrt(5)/4
  const double s1 = INV ? 0.95105651629515357212 : -0.95105651629515357212;  // sin 72
  const double s2 = INV ? 0.58778525229247312917 : -0.58778525229247312917;  // sin 144
  double2 a1 = cadd(x1, x4), a2 = cadd(x2, x3);
  double2 b1 = csub(x1, x4), b2 = csub(x2, x3);
  double2 t5 = cadd(a1, a2);
  double2 t6 = make_double2(x0.x - 0.25 * t5.x, x0.y - 0.25 * t5.y);
  double2 t7 = cscale(c, csub(a1, a2));
  double2 p = cadd(t6, t7), q = csub(t6, t7);
  double2 u = make_double2(s1 * b1.x + s2 * b2.x, s1 * b1.y + s2 * b2.y);
  double2 v = make_double2(s2 * b1.x - s1 * b2.x, s2 * b1.y - s1 * b2.y);
  x0 = cadd(x0, t5);
  x1 = cadd(p, make_double2(-u.y, u.x));
  x4 = csub(p, make_double2(-u.y, u.x));
  x2 = cadd(q, make_double2(-v.y, v.x));
  x3 = csub(q, make_double2(-v.y, v.x));
}

// ---- radix-9 = 3 x 3 with internal twiddles -------------------------------
template <bool INV>
__device__ __forceinline__ void bfly9(double2* v) {
  // columns: v[j], v[j+3], v[j+6]
  bfly3<INV>(v[0], v[3], v[6]);
  bfly3<INV>(v[1], v[4], v[7]);
  bfly3<INV>(v[2], v[5], v[8]);
  // twiddles w9^(j*k) on element (j, k) = v[j + 3k], j,k in {1,2}
  const double c1 = 0.76604444311897803520, s1 = 0.64278760968653932632;   // 40 deg
  const double c2 = 0.17364817766693034885, s2 = 0.98480775301220805936;   // 80 deg
  const double c4 = -0.93969262078590838405, s4 = 0.34202014332566873304;  // 160 deg
  const double sg = INV ? 1.0 : -1.0;
  v[4] = cmul(v[4], make_double2(c1, sg * s1));
  v[7] = cmul(v[7], make_double2(c2, sg * s2));
  v[5] = cmul(v[5], make_double2(c2, sg * s2));
  v[8] = cmul(v[8], make_double2(c4, sg * s4));
  // rows: v[3k], v[3k+1], v[3k+2]
  bfly3<INV>(v[0], v[1], v[2]);
  bfly3<INV>(v[3], v[4], v[5]);
  bfly3<INV>(v[6], v[7], v[8]);
  // output index k1 + 3 k2 held at v[3 k1 + k2] -> transpose 3x3
  double2 t;
  t = v[1]; v[1] = v[3]; v[3] = t;
  t = v[2]; v[2] = v[6]; v[6] = t;
  t = v[5]; v[5] = v[7]; v[7] = t;
}

// One Stockham pass with a compile-time radix over P pencils (leading dim ld).
template <int R, bool INV>
__device__ __forceinline__ void pass_fixed(const double2* __restrict__ src, double2* __restrict__ dst,
                                           int P, int ld, int L, int Ns, const double2* roots) {
  const int nb = L / R;
  const int tws = L / (Ns * R);
  const int total = P * nb;
  for (int t = threadIdx.x; t < total; t += blockDim.x) {
    const int p = t / nb;
    const int j = t - p * nb;
    const double2* s = src + (size_t)p * ld;
    double2 v[R];
#pragma unroll
    for (int r = 0; r < R; ++r) v[r] = s[j + r * nb];
    const int k = j % Ns;
    if (k != 0) {
#pragma unroll
      for (int r = 1; r < R; ++r) v[r] = cmul(v[r], root<INV>(roots, k * r * tws));
    }
    if (R == 3) bfly3<INV>(v[0], v[1], v[2]);
    else if (R == 5) bfly5<INV>(v[0], v[1], v[2], v[3], v[4]);
    else if (R == 9) bfly9<INV>(v);
    double2* d = dst + (size_t)p * ld + (j - k) * R + k;
#pragma unroll
    for (int r = 0; r < R; ++r) d[r * Ns] = v[r];
  }
}

// Generic odd radix R (prime): one thread per output element.
template <bool INV>
__device__ void pass_generic(const double2* __restrict__ src, double2* __restrict__ dst,
                             int P, int ld, int L, int Ns, int R, const double2* roots) {
  const int nb = L / R;
  const int tws = L / (Ns * R);
  const int LR = L / R;  // roots stride for w_R
  const int total = P * nb * R;
  const int h = (R - 1) / 2;
  for (int t = threadIdx.x; t < total; t += blockDim.x) {
    const int m = t % R;           // output index within the butterfly
    const int bt = t / R;
    const int p = bt / nb;
    const int j = bt - p * nb;
    const double2* s = src + (size_t)p * ld;
    const int k = j % Ns;
    auto in = [&](int r) -> double2 {
      double2 x = s[j + r * nb];
      if (k != 0 && r != 0) x = cmul(x, root<INV>(roots, k * r * tws));
      return x;
    };
    double2 x0 = in(0);
    double2 acc;
    if (m == 0) {
      acc = x0;
      for (int r = 1; r < R; ++r) acc = cadd(acc, in(r));
    } else {
      acc = make_double2(0.0, 0.0);
      for (int r = 1; r <= h; ++r) {
        double2 a = in(r), b = in(R - r);
        double2 sum = cadd(csub(a, x0), csub(b, x0));
        double2 dif = csub(a, b);
        double2 w = root<INV>(roots, ((r * m) % R) * LR);
        // w^{rm} x_r + w^{-rm} x_{R-r} = Re(w) * sum + i Im(w) * dif
        acc = cadd(acc, make_double2(w.x * sum.x - w.y * dif.y, w.x * sum.y + w.y * dif.x));
      }
    }
    dst[(size_t)p * ld + (j - k) * R + k + m * Ns] = acc;
  }
}

// In-shared-memory FFT of P pencils of length pl.L, data in buf0 (leading dim
// ld), buf1 is scratch of the same size.  Returns the buffer holding the
// result.  Must be called by all threads of the block; ends with a barrier.
template <bool INV>
__device__ double2* smem_fft(double2* buf0, double2* buf1, int P, int ld, const FftPlan& pl) {
  double2* src = buf0;
  double2* dst = buf1;
  int Ns = 1;
  for (int s = 0; s < pl.nf; ++s) {
    const int R = pl.f[s];
    if (R == 3) pass_fixed<3, INV>(src, dst, P, ld, pl.L, Ns, pl.roots);
    else if (R == 5) pass_fixed<5, INV>(src, dst, P, ld, pl.L, Ns, pl.roots);
    else if (R == 9) pass_fixed<9, INV>(src, dst, P, ld, pl.L, Ns, pl.roots);
    else pass_generic<INV>(src, dst, P, ld, pl.L, Ns, R, pl.roots);
    __syncthreads();
    double2* t = src; src = dst; dst = t;
    Ns *= R;
  }
  return src;
}

}  // namespace fc
