// Sweep kernels for power-of-three axis lengths using the register-resident
// FFT of fc_fft_reg.cuh.  Same data layouts, input modes and epilogues as the
// generic kernels in fc_kernels.cuh (see the layout comment there).
#pragma once
#include "fc_fft_reg.cuh"
#include "fc_kernels.cuh"
#include "fc_tma.cuh"

namespace fc {

constexpr int kMaxBlock = 512;   // row / mid sweeps

#ifdef FC_TRACE  // experimental builds only (tools/exp_build.sh): per-CTA phase stamps of the sweeps
// kernel ids: 0 outer (d = 2), 1 row_fwd_pk, 2 mid_fwd, 3 outer_seq, 4 mid_inv, 5 row_inv
__device__ unsigned long long g_trace[6 * 8 * 8192];
__device__ __forceinline__ void trace_stamp(int kid, int slot) {
  if (threadIdx.x == 0 && blockIdx.x < 8192) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_trace[(kid * 8192 + blockIdx.x) * 8 + slot] = t;
    if (slot == 0) {
      unsigned smid;
      asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
      g_trace[(kid * 8192 + blockIdx.x) * 8 + 7] = smid;
    }
  }
}
#else
__device__ __forceinline__ void trace_stamp(int, int) {}
#endif

// 8-byte asynchronous global->shared copies (LDGSTS): loads stay in flight
// without holding registers, so a CTA issues its whole input tile at once.
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
}
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gmem) : "memory");
}
// Copy n contiguous doubles to shared memory, block-strided, 8-byte granules.
__device__ __forceinline__ void stage_doubles(double* dst, const double* src, int n) {
  for (int i = threadIdx.x; i < n; i += blockDim.x) cp_async8(dst + i, src + i);
}
// Same with 16-byte granules.  dst must be 16-byte aligned and have one spare
// double in front and behind; returns the shift (0 or 1) so element i lands at
// dst[i + shift] (the shift matches the source's 16-byte phase).
__device__ __forceinline__ int stage_doubles16(double* dst, const double* src, int n) {
  const int shift = (int)((reinterpret_cast<uintptr_t>(src) >> 3) & 1);
  double* d = dst + shift;
  // head element when src is 8 mod 16, then pairs, then a possible tail
  int i0 = 0;
  if (shift) {
    if (threadIdx.x == 0 && n > 0) cp_async8(d, src);
    i0 = 1;
  }
  const int npair = (n - i0) >> 1;
  for (int q = threadIdx.x; q < npair; q += blockDim.x) cp_async16(d + i0 + 2 * q, src + i0 + 2 * q);
  const int done = i0 + 2 * npair;
  if (done < n && threadIdx.x == 0) cp_async8(d + done, src + done);
  return shift;
}
constexpr int kMaxBlockOuter = 256;

// First sweep: thread (p, j) of the CTA owns complex pencil p = rows (2p, 2p+1)
// of the row block and loads elements j + s*TP of both rows, computing the
// pointwise input on the fly.  After the FFT the spectrum goes through shared
// memory once more to split the two-for-one pairs and to store transposed.
template <int L>
__global__ void __launch_bounds__(256, 2) k_row_fwd_r(Geo g, RowGeo rg, Coef C, InArgs ia, const RhsState* st,
                                                          const double2* __restrict__ tw, double2* __restrict__ W,
                                                          const __grid_constant__ CUtensorMap tmW) {
  constexpr int TP = RegTP<L>::value;
  extern __shared__ __align__(128) unsigned char smraw[];  // TMA boxes need 128-byte alignment
  double2* sm = reinterpret_cast<double2*>(smraw);
  const int c = g.dim;
  int64_t bid = blockIdx.x;
  const int a = bid % c; bid /= c;
  const int tile = bid % rg.ntiles; bid /= rg.ntiles;
  const int o = bid % rg.no;
  const int r = (int)(bid / rg.no);
  if (!rhs_active(st, r)) return;
  const int row0 = tile * rg.B;
  const int nrows = min(rg.B, rg.np - row0);
  const int p = threadIdx.x / TP;
  const int j = threadIdx.x - p * TP;
  const InEval ev = make_eval(ia, g, C, st, r, a);
  double2 v[1][9];
  double2 pn[9];  // p' of the (even, odd) row at element s (IN_PNEW)
  const int re = 2 * p, ro = 2 * p + 1;
  const bool he = re < nrows, ho = ro < nrows;
  const int64_t vbase = ((int64_t)o * rg.np + row0) * L;
  // staged path: isotropic A, and for the fixed point a reference row without
  // off-diagonal entries (then (A - A0) e is diagonal, solver.py:253-255)
  const bool fp_diag = ev.mode != IN_FP ||
                       ((a == 0 || ev.R0 == 0.0) && (a == 1 || ev.R1 == 0.0) && (a == 2 || ev.R2 == 0.0));
  const bool staged = (ev.kind == 0 || ev.mode == IN_RAW) && ev.mode != IN_CONST && fp_diag;
  if (staged) {
    // isotropic: stage u (r / e / field), p_old and A for the whole row block in
    // smem with cp.async, evaluate, store p' at once (no register array lives
    // across the loop); the staging area is reused as the FFT exchange buffer
    const int stride = (rg.B * L + 3) & ~1;  // even, leaves room for the alignment shift
    double* st_u = reinterpret_cast<double*>(sm);
    double* st_p = st_u + stride;
    double* st_a = st_p + stride;
    const int n = nrows * L;
    const int64_t ub = ev.base + (int64_t)a * g.N + vbase;
    // one thread stages the row block with bulk copies (TMA); the CTA waits on bar
    __shared__ uint64_t bar;
    const bool use_p = ev.mode == IN_PNEW && !ev.first;
    const bool use_a = ev.mode != IN_RAW;
    const int su = bulk_shift(ev.u + ub);
    const int sp = use_p ? bulk_shift(ev.p_old + ub) : 0;
    const int sa = use_a ? bulk_shift(ev.A + vbase) : 0;
    if (threadIdx.x == 0) {
      mbar_init(&bar, 1);
      mbar_expect_tx(&bar, bulk_bytes(n, su) + (use_p ? bulk_bytes(n, sp) : 0u) + (use_a ? bulk_bytes(n, sa) : 0u));
      bulk_g2s(st_u, ev.u + ub - su, bulk_bytes(n, su), &bar);
      if (use_p) bulk_g2s(st_p, ev.p_old + ub - sp, bulk_bytes(n, sp), &bar);
      if (use_a) bulk_g2s(st_a, ev.A + vbase - sa, bulk_bytes(n, sa), &bar);
    }
    st_u += su;
    st_p += sp;
    st_a += sa;
    // deferred x += alpha p_old of the previous iteration (solver.py:213): the x
    // loads are issued before the wait so they overlap the bulk copies
    double* xw = ev.xacc ? ev.xacc + ub : nullptr;
    double xv[2][9];
    if (xw) {
#pragma unroll
      for (int s = 0; s < 9; ++s)
#pragma unroll
        for (int h = 0; h < 2; ++h) xv[h][s] = (2 * p + h < nrows) ? xw[(2 * p + h) * L + j + s * TP] : 0.0;
    }
    __syncthreads();  // barrier initialised before anyone polls it
    mbar_wait(&bar, 0);
    double* pw = ia.p_new + ub;
    const double A0aa = InEval::sel(a, ev.R0, ev.R1, ev.R2);
#pragma unroll
    for (int s = 0; s < 9; ++s) {
      const int i = j + s * TP;
      double y[2] = {0.0, 0.0};
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int row = 2 * p + h;
        if (row < nrows) {
          const int e = row * L + i;
          double x = st_u[e];
          if (ev.mode == IN_PNEW) {
            x = ev.first ? x : __dadd_rn(x, __dmul_rn(ev.beta, st_p[e]));
            pw[e] = x;
          }
          double val;
          if (ev.mode == IN_RAW) val = x;
          else if (ev.mode == IN_FP) val = __dmul_rn(__dsub_rn(st_a[e], A0aa), x);
          else val = __dmul_rn(st_a[e], x);
          if (ev.mode != IN_FP && ev.s != 1.0) val = __dmul_rn(ev.s, val);
          y[h] = val;
        }
      }
      v[0][s] = make_double2(y[0], y[1]);
    }
    if (xw) {  // after the pointwise step: the x loads have had the longest time to land
#pragma unroll
      for (int s = 0; s < 9; ++s)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int e = (2 * p + h) * L + j + s * TP;
          if (2 * p + h < nrows) xw[e] = __dadd_rn(xv[h][s], __dmul_rn(ev.alpha, st_p[e]));
        }
    }
  } else {
    with_in_mode(ev.mode, ev.kind, [&](auto M, auto K) {
      constexpr int MODE = decltype(M)::value, KIND = decltype(K)::value;
#pragma unroll
      for (int s = 0; s < 9; ++s) {
        const int i = j + s * TP;
        double pe = 0.0, po = 0.0;
        const double xe = he ? ev.template eval_t<MODE, KIND>(vbase + (int64_t)re * L + i, pe) : 0.0;
        const double xo = ho ? ev.template eval_t<MODE, KIND>(vbase + (int64_t)ro * L + i, po) : 0.0;
        v[0][s] = make_double2(xe, xo);
        pn[s] = make_double2(pe, po);
      }
    });
  }
  if (ev.mode == IN_PNEW && !staged) {  // p' = r + beta p, stored once by the CTA owning component a
    double* pw = ia.p_new + ev.base + (int64_t)a * g.N + vbase;
#pragma unroll
    for (int s = 0; s < 9; ++s) {
      if (he) pw[(int64_t)re * L + j + s * TP] = pn[s].x;
      if (ho) pw[(int64_t)ro * L + j + s * TP] = pn[s].y;
    }
  }
  double2* smp = sm + (size_t)p * L;
  fft_reg<L, 1, false>(v, smp, L, j, tw);
  __syncthreads();
#pragma unroll
  for (int s = 0; s < 9; ++s) smp[j + s * TP] = v[0][s];
  __syncthreads();
  constexpr int hl = (L + 1) / 2;
  double2* Wb = W + ((int64_t)(r * c + a) * rg.no + o) * hl * rg.np + row0;
  const int npairs = (nrows + 1) >> 1;
  if (rg.tma) {
    // split into Y[k][row] (complex) behind the pencils, then TMA-store the boxes
    // (the store clips rows >= np and modes >= hl)
    const int B = rg.B;
    double2* Y = sm + (((size_t)(B / 2) * L + 7) & ~(size_t)7);
    for (int idx = threadIdx.x; idx < hl * npairs; idx += blockDim.x) {
      const int k = idx / npairs;
      const int pr = idx - k * npairs;
      const double2* z = sm + (size_t)pr * L;
      const double2 zk = z[k];
      const double2 zm = z[k == 0 ? 0 : L - k];
      Y[k * B + 2 * pr] = make_double2(0.5 * (zk.x + zm.x), 0.5 * (zk.y - zm.y));
      Y[k * B + 2 * pr + 1] = make_double2(0.5 * (zk.y + zm.y), 0.5 * (zm.x - zk.x));
    }
    fence_proxy_async();
    __syncthreads();
    if (threadIdx.x == 0) {
      const int c2 = (r * c + a) * rg.no + o;
      for (int b = 0; b < rg.nbox; ++b) tma_store_3d(&tmW, 2 * row0, b * rg.boxK, c2, Y + (size_t)b * rg.boxK * B);
      bulk_commit();
      bulk_wait_read0();
    }
    return;
  }
  // split Z = Ye + i Yo into the two half spectra; one thread per (pair, k)
  for (int idx = threadIdx.x; idx < hl * npairs; idx += blockDim.x) {
    const int pr = idx / hl;
    const int k = idx - pr * hl;
    const double2* z = sm + (size_t)pr * L;
    const double2 zk = z[k];
    const double2 zm = z[k == 0 ? 0 : L - k];
    double2* dst = Wb + (int64_t)k * rg.np + 2 * pr;
    dst[0] = make_double2(0.5 * (zk.x + zm.x), 0.5 * (zk.y - zm.y));
    if (2 * pr + 1 < nrows) dst[1] = make_double2(0.5 * (zk.y + zm.y), 0.5 * (zm.x - zk.x));
  }
}

// Last sweep: transposed half-spectrum load into smem, two-for-one assembly
// straight into registers, inverse FFT, epilogue from registers (coalesced).
template <int L, int NT>
__global__ void __launch_bounds__(NT, NT <= 256 ? 3 : (NT <= 384 ? 2 : 1)) k_row_inv_r(Geo g, RowGeo rg, EpArgs ea, const RhsState* st,
                                                          const double2* __restrict__ tw,
                                                          const double2* __restrict__ W,
                                                          const __grid_constant__ CUtensorMap tmW) {
  constexpr int TP = RegTP<L>::value;
  constexpr int hl = (L + 1) / 2;
  extern __shared__ __align__(128) unsigned char smraw[];  // TMA boxes need 128-byte alignment
  double2* sm = reinterpret_cast<double2*>(smraw);
  __shared__ double red[kMaxBlock / 32];
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
  const double2* Wb = W + ((int64_t)(r * c + a) * rg.no + o) * hl * rg.np + row0;
  const int64_t vbase = ((int64_t)o * rg.np + row0) * L;
  const int64_t ebase = ((int64_t)r * c + a) * g.N + vbase;
  // epilogue input (p for EP_AP, e for EP_FP), read in the epilogue
  const bool need_q = ea.mode == EP_AP || ea.mode == EP_FP;
  const double* qsrc = (ea.mode == EP_AP ? ea.p : ea.out) + ebase;
  __shared__ uint64_t bar, barq;
  // Y staged at sm[k * yk + row * yr]: TMA boxes give [k][row], the fallback [row][k]
  const int yk = rg.tma ? rg.B : 1;
  const int yr = rg.tma ? 1 : hl;
  // epilogue input staged by one bulk copy issued with the spectrum loads, so it
  // lands during the transform instead of after it (the rows of a block are contiguous)
  const bool qpre = need_q && rg.tma && rg.qoff > 0;
  const int qsh = qpre ? bulk_shift(qsrc) : 0;
  const double* Q = reinterpret_cast<const double*>(smraw + rg.qoff) + qsh;
  trace_stamp(5, 0);
  if (rg.tma) {
    if (threadIdx.x == 0) {
      mbar_init(&bar, 1);
      if (qpre) mbar_init(&barq, 1);
      mbar_expect_tx(&bar, (unsigned)(rg.nbox * rg.boxK * rg.B * 16));
      const int c2 = (r * c + a) * rg.no + o;
      for (int b = 0; b < rg.nbox; ++b) tma_load_3d(sm + (size_t)b * rg.boxK * rg.B, &tmW, 2 * row0, b * rg.boxK, c2, &bar);
      if (qpre) {
        mbar_expect_tx(&barq, bulk_bytes(nrows * L, qsh));
        bulk_g2s(smraw + rg.qoff, qsrc - qsh, bulk_bytes(nrows * L, qsh), &barq);
      }
    }
    __syncthreads();
    mbar_wait(&bar, 0);
  } else {
    const int npairs = (nrows + 1) >> 1;
    const int total = hl * npairs;
    for (int base = 0; base < total; base += 4 * blockDim.x) {
      double2 t0[4], t1[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int idx = base + u * blockDim.x + threadIdx.x;
        if (idx < total) {
          const int pr = idx / hl, k = idx - pr * hl;
          const double2* src = Wb + (int64_t)k * rg.np + 2 * pr;
          t0[u] = __ldg(src);
          t1[u] = 2 * pr + 1 < nrows ? __ldg(src + 1) : make_double2(0.0, 0.0);
        }
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int idx = base + u * blockDim.x + threadIdx.x;
        if (idx < total) {
          const int pr = idx / hl, k = idx - pr * hl;
          sm[(2 * pr) * hl + k] = t0[u];
          sm[(2 * pr + 1) * hl + k] = t1[u];
        }
      }
    }
  }
  __syncthreads();
  trace_stamp(5, 1);
  const int p = threadIdx.x / TP;
  const int j = threadIdx.x - p * TP;
  const int re = 2 * p, ro = 2 * p + 1;
  const bool has_o = ro < nrows;
  double2 v[1][9];
#pragma unroll
  for (int s = 0; s < 9; ++s) {
    const int i = j + s * TP;
    const int k = i < hl ? i : L - i;
    double2 ye = re < nrows ? sm[k * yk + re * yr] : make_double2(0.0, 0.0);
    double2 yo = has_o ? sm[k * yk + ro * yr] : make_double2(0.0, 0.0);
    if (i == 0) v[0][s] = make_double2(ye.x, yo.x);
    else if (i < hl) v[0][s] = make_double2(ye.x - yo.y, ye.y + yo.x);
    else v[0][s] = make_double2(ye.x + yo.y, yo.x - ye.y);
  }
  // the exchange buffer overlaps the Y staging area: fft_reg syncs before its first write
  double2* smp = sm + (size_t)p * L;
  fft_reg<L, 1, true>(v, smp, L, j, tw);
  trace_stamp(5, 2);
  const double Ea = ea.mode == EP_FP ? pick(ea.E, r, a) : 0.0;
  const bool he = re < nrows;
  double2 q[9];
  if (qpre) {
    mbar_wait(&barq, 0);
#pragma unroll
    for (int s = 0; s < 9; ++s) {
      const int i = j + s * TP;
      q[s].x = he ? Q[re * L + i] : 0.0;
      q[s].y = has_o ? Q[ro * L + i] : 0.0;
    }
  } else if (need_q) {
#pragma unroll
    for (int s = 0; s < 9; ++s) {
      const int i = j + s * TP;
      q[s].x = he ? __ldg(qsrc + re * L + i) : 0.0;
      q[s].y = has_o ? __ldg(qsrc + ro * L + i) : 0.0;
    }
  }
  double acc = 0.0;
  // epilogue values in registers first: the CTA's partial is published (and its
  // arrival counted) before the output stores, so the arrival fence does not
  // wait for them
  with_ep_mode(ea.mode, [&](auto M) {
    constexpr int MODE = decltype(M)::value;
#pragma unroll
    for (int s = 0; s < 9; ++s) {
      if (he) acc += ep_value_t<MODE>(v[0][s].x * g.invN, Ea, q[s].x, v[0][s].x);
      if (has_o) acc += ep_value_t<MODE>(v[0][s].y * g.invN, Ea, q[s].y, v[0][s].y);
    }
  });
  if (ea.part != nullptr) {
    double sum = block_sum(acc, red);
    if (threadIdx.x == 0) {
      const int slot = (o * rg.ntiles + tile) * c + a;
      ea.part[(int64_t)r * ea.nslot + slot] = sum;
    }
  }
  trace_stamp(5, 3);
  const bool last = arrive_block(ea.fin);
  trace_stamp(5, 4);
  {
    double* __restrict__ out = ea.out;
#pragma unroll
    for (int s = 0; s < 9; ++s) {
      const int i = j + s * TP;
      if (he) out[ebase + (int64_t)re * L + i] = v[0][s].x;
      if (has_o) out[ebase + (int64_t)ro * L + i] = v[0][s].y;
    }
  }
  trace_stamp(5, 5);
  if (last) finalize_block(ea.fin, red);
}

__device__ __forceinline__ double2 g3_scale(double xi, double2 v);  // defined below
__device__ __forceinline__ double2 g3_fold(double xi1, double xi2, double2 v1, double2 v2);

// Middle sweep through TMA (one slab).  Pencil side (W1[rc][i0][k2][:], one
// contiguous row of L modes per i0): one bulk copy per pencil.  Transposed side
// (W2[rc][k2][k1][i0]): tensor boxes {2 BP doubles, rows modes} = BP consecutive
// i0 for rows consecutive k1, landing in smem as [k1][p].
// JF: thread mapping of the transform, pencil-fastest (p = t % BP: the
// transposed shared-memory side is conflict-free) or lane-fastest (p = t / TP:
// the exchanges inside the FFT are conflict-free).
template <int L, bool INV, bool JF>
__device__ __forceinline__ void mid_tma(const Geo& g, const MidGeo& mg, const RhsState* st,
                                        const double2* __restrict__ tw, const double2* __restrict__ src,
                                        double2* __restrict__ dst, const CUtensorMap& tmM, double2* sm,
                                        int ib, int k2, int a, int r) {
  constexpr int TP = RegTP<L>::value;
  const int c = g.dim;
  const int BP = mg.B;
  const int p = JF ? threadIdx.x / TP : threadIdx.x % BP;
  const int j = JF ? threadIdx.x - p * TP : threadIdx.x / BP;
  const int i00 = ib * BP;
  const int np_ = min(BP, mg.n0 - i00);  // live pencils
  const int rc = r * c + a;
  // mg.rebuild (inverse sweep behind k_outer_seq<L, 3, true>): the outer sweep left
  // t = F0^-1 q in component 1's planes instead of xi1 t and xi2 t in planes 1 and
  // 2; both components are rebuilt from it on the way into the registers
  const bool reb = INV && mg.rebuild && a >= 1;
  const int cz = (reb ? r * c + 1 : rc) * mg.h2 + k2;  // tensor coordinate of the source plane
  const double2* pen = (INV ? dst : src) + (((int64_t)rc * mg.n0 + i00) * mg.h2 + k2) * L;  // pencil p at + p*h2*L
  const int64_t pstride = (int64_t)mg.h2 * L;
  __shared__ uint64_t bar;
  trace_stamp(INV ? 4 : 2, 0);
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    if (!INV) {
      mbar_expect_tx(&bar, (unsigned)(np_ * L * 16));
      for (int q = 0; q < np_; ++q) bulk_g2s(sm + (size_t)q * L, pen + q * pstride, (unsigned)(L * 16), &bar);
    } else {
      mbar_expect_tx(&bar, (unsigned)(mg.nbox * mg.rows * BP * 16));
      for (int b = 0; b < mg.nbox; ++b)
        tma_load_3d(sm + (size_t)b * mg.rows * BP, &tmM, 2 * i00, b * mg.rows, cz, &bar);
    }
  }
  __syncthreads();
  mbar_wait(&bar, 0);
  trace_stamp(INV ? 4 : 2, 1);
  double2 v[1][9];
#pragma unroll
  for (int s = 0; s < 9; ++s) {
    const int i = j + s * TP;
    v[0][s] = INV ? sm[(size_t)i * BP + p] : sm[(size_t)p * L + i];
    if (reb) v[0][s] = g3_scale(a == 1 ? g.xi[1][i] : g.xi[2][k2], v[0][s]);
  }
  fft_reg<L, 1, INV>(v, sm + (size_t)p * L, L, j, tw);
  trace_stamp(INV ? 4 : 2, 2);
  __syncthreads();
#pragma unroll
  for (int s = 0; s < 9; ++s) {
    const int i = j + s * TP;
    if (INV) sm[(size_t)p * L + i] = v[0][s];
    else sm[(size_t)i * BP + p] = v[0][s];
  }
  fence_proxy_async();
  __syncthreads();
  if (threadIdx.x == 0) {
    if (INV) {
      for (int q = 0; q < np_; ++q) bulk_s2g(const_cast<double2*>(pen) + q * pstride, sm + (size_t)q * L, (unsigned)(L * 16));
    } else {
      for (int b = 0; b < mg.nbox; ++b) tma_store_3d(&tmM, 2 * i00, b * mg.rows, cz, sm + (size_t)b * mg.rows * BP);
    }
    bulk_commit();
    trace_stamp(INV ? 4 : 2, 3);
    bulk_wait_read0();
    trace_stamp(INV ? 4 : 2, 4);
    trace_stamp(INV ? 4 : 2, 5);
  }
}

template <int L, bool INV, bool JF>
__global__ void __launch_bounds__(kMaxBlock) k_mid_tma(Geo g, MidGeo mg, const RhsState* st,
                                                        const double2* __restrict__ tw, const double2* __restrict__ src,
                                                        double2* __restrict__ dst, const __grid_constant__ CUtensorMap tmM) {
  extern __shared__ __align__(128) unsigned char smraw[];
  int64_t bid = blockIdx.x;
  int a = 0;
  if (INV && mg.rebuild) {  // the CTAs of components 1 and 2 read the same planes: side by side (L2)
    a = bid % g.dim; bid /= g.dim;
  }
  const int ib = bid % mg.nib; bid /= mg.nib;
  const int k2 = bid % mg.h2; bid /= mg.h2;
  if (!(INV && mg.rebuild)) {
    a = bid % g.dim; bid /= g.dim;
  }
  const int r = (int)bid;
  if (!rhs_active(st, r)) return;
  mid_tma<L, INV, JF>(g, mg, st, tw, src, dst, tmM, reinterpret_cast<double2*>(smraw), ib, k2, a, r);
}

// Forward middle sweep that folds components 1 and 2 (MidGeo::fold, with
// k_outer_seq<L, 3, *, true>).  Gamma_hat needs xi . v_hat = xi0 v0 + (xi1 v1 + xi2 v2);
// once axes 2 and 1 are transformed xi1 (k1) and xi2 (k2) are known, so this sweep
// stores u = xi1 F1 v1 + xi2 F1 v2 (g3_fold: the products and the sum the outer sweep
// would form after loading both fields) in component 1's planes of W2 and nothing
// in component 2's.  One CTA, components one after the other (nine complex in
// registers at a time, as mid_tma): both pencil sets are fetched at the start, F1 v1
// is parked transposed in shared memory by the thread that will fold it.
template <int L, bool JF>
__device__ __forceinline__ void mid_tma_fold(const Geo& g, const MidGeo& mg, const double2* __restrict__ tw,
                                             const double2* __restrict__ src, const CUtensorMap& tmM, double2* sm,
                                             int ib, int k2, int r) {
  constexpr int TP = RegTP<L>::value;
  const int BP = mg.B;
  const int p = JF ? threadIdx.x / TP : threadIdx.x % BP;
  const int j = JF ? threadIdx.x - p * TP : threadIdx.x / BP;
  const int i00 = ib * BP;
  const int np_ = min(BP, mg.n0 - i00);
  const int rc1 = r * 3 + 1;
  const int cz1 = rc1 * mg.h2 + k2;
  const double2* pen1 = src + (((int64_t)rc1 * mg.n0 + i00) * mg.h2 + k2) * L;
  const double2* pen2 = pen1 + (int64_t)mg.n0 * mg.h2 * L;
  const int64_t pstride = (int64_t)mg.h2 * L;
  double2* smB = sm + mg.regA;  // component 2's pencils, behind the box region
  __shared__ uint64_t bar;
  __shared__ int zero;
  if (threadIdx.x == 0) {
    zero = 0;
    mbar_init(&bar, 1);
    mbar_expect_tx(&bar, (unsigned)(2 * np_ * L * 16));
    for (int q = 0; q < np_; ++q) bulk_g2s(sm + (size_t)q * L, pen1 + q * pstride, (unsigned)(L * 16), &bar);
    for (int q = 0; q < np_; ++q) bulk_g2s(smB + (size_t)q * L, pen2 + q * pstride, (unsigned)(L * 16), &bar);
  }
  __syncthreads();
  mbar_wait(&bar, 0);
  double2 v[1][9];
  const double xi2 = g.xi[2][k2];
#pragma unroll 1
  for (int a = 0; a < 2; ++a) {  // one transform body: registers as mid_tma
    double2* pen = (a == 0 ? sm : smB) + (size_t)p * L;
    // ptxas would hoist the second transform's 16 twiddle loads (64 registers) above
    // the first transform to hide their latency, doubling the registers per thread:
    // tie the table's address to a shared-memory word read in this iteration
    const double2* twa = tw + *reinterpret_cast<volatile int*>(&zero);
#pragma unroll
    for (int s = 0; s < 9; ++s) v[0][s] = pen[j + s * TP];
    fft_reg<L, 1, false>(v, pen, L, j, twa);
    __syncthreads();  // this component's exchange buffers are free
    if (a == 0) {     // park F1 v1 in the pencil's own row (conflict-free, read back by this thread)
#pragma unroll
      for (int s = 0; s < 9; ++s) pen[j + s * TP] = v[0][s];
    } else {          // fold and store transposed into component 2's region
#pragma unroll
      for (int s = 0; s < 9; ++s) {
        const int i = j + s * TP;
        smB[(size_t)i * BP + p] = g3_fold(g.xi[1][i], xi2, sm[(size_t)p * L + i], v[0][s]);
      }
    }
  }
  sm = smB;  // the boxes leave from component 2's region
  fence_proxy_async();
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int b = 0; b < mg.nbox; ++b) tma_store_3d(&tmM, 2 * i00, b * mg.rows, cz1, sm + (size_t)b * mg.rows * BP);
    bulk_commit();
    bulk_wait_read0();
  }
}

// CTA size the folding sweep is compiled for (the planner's defaults: 256 threads for
// pencils <= 243, two pencils above) and the resident CTAs that keep it at <= 84 registers
__host__ __device__ constexpr int fold_threads(int L) { return L / 9 <= 27 ? 256 : (2 * (L / 9) + 31) / 32 * 32; }
__host__ __device__ constexpr int fold_ctas(int L) {
  return 65536 / (84 * fold_threads(L)) < 1 ? 1 : (65536 / (84 * fold_threads(L)) > 4 ? 4 : 65536 / (84 * fold_threads(L)));
}

template <int L, bool JF>
__global__ void __launch_bounds__(fold_threads(L), fold_ctas(L)) k_mid_tma_fold(Geo g, MidGeo mg, const RhsState* st,
                                                             const double2* __restrict__ tw, const double2* __restrict__ src,
                                                             double2* __restrict__ dst, const __grid_constant__ CUtensorMap tmM) {
  extern __shared__ __align__(128) unsigned char smraw[];
  int64_t bid = blockIdx.x;
  const int ib = bid % mg.nib; bid /= mg.nib;
  const int k2 = bid % mg.h2; bid /= mg.h2;
  const int ap = bid % 2;
  const int r = (int)(bid / 2);
  if (!rhs_active(st, r)) return;
  if (ap == 0) mid_tma<L, false, JF>(g, mg, st, tw, src, dst, tmM, reinterpret_cast<double2*>(smraw), ib, k2, 0, r);
  else mid_tma_fold<L, JF>(g, mg, tw, src, tmM, reinterpret_cast<double2*>(smraw), ib, k2, r);
}

// Middle sweep (d = 3), thread mapping pencil-fastest (t = j * BP + p) so the
// transposed side is written / read in chunks of BP consecutive i0.
template <int L, bool INV>
__global__ void __launch_bounds__(kMaxBlock) k_mid_r(Geo g, MidGeo mg, SlabMap sm_, const RhsState* st,
                                                      const double2* __restrict__ tw,
                                                      const double2* __restrict__ src, double2* __restrict__ dst) {
  constexpr int TP = RegTP<L>::value;
  extern __shared__ double2 sm[];
  const int c = g.dim;
  int64_t bid = blockIdx.x;
  const int ib = bid % mg.nib; bid /= mg.nib;
  const int k2 = bid % mg.h2; bid /= mg.h2;
  const int a = bid % c;
  const int r = (int)(bid / c);
  if (!rhs_active(st, r)) return;
  const int BP = mg.B;
  const int p = threadIdx.x % BP;
  const int j = threadIdx.x / BP;
  const int i00 = ib * BP;
  const bool live = i00 + p < mg.n0;   // mg.n0 = local planes of this slab
  const int rc = r * c + a;
  double2 v[1][9];
  if (!INV) {
    const double2* s0 = src + (((int64_t)rc * mg.n0 + i00 + p) * mg.h2 + k2) * L;
#pragma unroll
    for (int s = 0; s < 9; ++s) v[0][s] = live ? s0[j + s * TP] : make_double2(0.0, 0.0);
  } else if (sm_.P == 1) {
    const double2* s0 = src + (((int64_t)rc * mg.h2 + k2) * L) * sm_.n0l + i00 + p;
#pragma unroll
    for (int s = 0; s < 9; ++s) v[0][s] = live ? s0[(int64_t)(j + s * TP) * sm_.n0l] : make_double2(0.0, 0.0);
  } else {
#pragma unroll
    for (int s = 0; s < 9; ++s)
      v[0][s] = live ? src[send_index(sm_, rc, k2 * L + j + s * TP, i00 + p)] : make_double2(0.0, 0.0);
  }
  fft_reg<L, 1, INV>(v, sm + (size_t)p * L, L, j, tw);
  if (!live) return;
  if (!INV && sm_.P == 1) {
    double2* d0 = dst + (((int64_t)rc * mg.h2 + k2) * L) * sm_.n0l + i00 + p;
#pragma unroll
    for (int s = 0; s < 9; ++s) d0[(int64_t)(j + s * TP) * sm_.n0l] = v[0][s];
  } else if (!INV) {
#pragma unroll
    for (int s = 0; s < 9; ++s) *send_dst(sm_, dst, rc, k2 * L + j + s * TP, i00 + p) = v[0][s];
    if (sm_.fused) __threadfence_system();  // peer stores (other processes' buffers) ordered before the exit
  } else {
    double2* d0 = dst + (((int64_t)rc * mg.n0 + i00 + p) * mg.h2 + k2) * L;
#pragma unroll
    for (int s = 0; s < 9; ++s) d0[j + s * TP] = v[0][s];
  }
}

// d = 3 outer sweep with four axis-0 transforms instead of six.  Along an
// axis-0 pencil xi1 and xi2 are constants, so
//   xi . F0(v) = xi0 F0(v0) + F0(xi1 v1 + xi2 v2)
//   F0^-1(xi_a q) = xi_a F0^-1(q)   (a = 1, 2),   q = (xi . v^) / den,
// i.e. one forward transform of v0, one of the folded u = xi1 v1 + xi2 v2, one
// inverse of xi0 q and one of q, whose result is scaled by xi1 / xi2.  Same
// operator up to rounding; the helpers below fix the arithmetic (explicit
// roundings) so every d = 3 outer kernel that uses them agrees bitwise.
__device__ __forceinline__ double2 g3_fold(double xi1, double xi2, double2 v1, double2 v2) {
  return make_double2(__fma_rn(xi2, v2.x, __dmul_rn(xi1, v1.x)), __fma_rn(xi2, v2.y, __dmul_rn(xi1, v1.y)));
}
// (F0 v0, F0 u) at one mode -> (xi0 q, q); both 0 at k = 0
__device__ __forceinline__ void g3_mode(const OuterGeo& og, double xi0, double xi1, double xi2, bool kzero,
                                        double2& t0, double2& t1) {
  if (kzero) {
    t0 = make_double2(0.0, 0.0);
    t1 = make_double2(0.0, 0.0);
    return;
  }
  double den;
  if (og.orth) {
    den = __fma_rn(xi2, xi2, __fma_rn(xi1, xi1, __dmul_rn(xi0, xi0)));
  } else {
    const double xi[3] = {xi0, xi1, xi2};
    den = 0.0;
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
      for (int b = 0; b < 3; ++b) den = __fma_rn(__dmul_rn(xi[a], og.M[a][b]), xi[b], den);
  }
  const double inv = 1.0 / den;
  const double2 qv = make_double2(__dmul_rn(__fma_rn(xi0, t0.x, t1.x), inv), __dmul_rn(__fma_rn(xi0, t0.y, t1.y), inv));
  t0 = make_double2(__dmul_rn(xi0, qv.x), __dmul_rn(xi0, qv.y));
  t1 = qv;
}
__device__ __forceinline__ double2 g3_scale(double xi, double2 v) { return make_double2(__dmul_rn(xi, v.x), __dmul_rn(xi, v.y)); }

// d = 2: (F0 v0, F0 v1) at one mode -> Gamma_hat(k) v = xi (xi . v) / den, 0 at k = 0.
// (xi . v) / den as one reciprocal and two products (the reference divides twice,
// solver.py:108: the results differ by at most 1 ulp).  Explicit roundings, so
// every d = 2 outer kernel that uses it agrees bitwise.
__device__ __forceinline__ void g2_mode(const OuterGeo& og, double xi0, double xi1, bool kzero, double2& t0, double2& t1) {
  if (kzero) {
    t0 = make_double2(0.0, 0.0);
    t1 = make_double2(0.0, 0.0);
    return;
  }
  double den;
  if (og.orth) {
    den = __fma_rn(xi1, xi1, __dmul_rn(xi0, xi0));
  } else {
    const double xi[2] = {xi0, xi1};
    den = 0.0;
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int b = 0; b < 2; ++b) den = __fma_rn(__dmul_rn(xi[a], og.M[a][b]), xi[b], den);
  }
  const double inv = 1.0 / den;
  const double2 qv = make_double2(__dmul_rn(__fma_rn(xi1, t1.x, __dmul_rn(xi0, t0.x)), inv),
                                  __dmul_rn(__fma_rn(xi1, t1.y, __dmul_rn(xi0, t0.y)), inv));
  t0 = make_double2(__dmul_rn(xi0, qv.x), __dmul_rn(xi0, qv.y));
  t1 = make_double2(__dmul_rn(xi1, qv.x), __dmul_rn(xi1, qv.y));
}

// Outer sweep: each thread owns the C component pencils of one q so Gamma_hat
// is applied in registers between the forward and inverse transforms.
template <int L, int C>
__global__ void __launch_bounds__(kMaxBlockOuter, (C == 2 ? 2 : 1)) k_outer_r(Geo g, OuterGeo og, SlabMap sm_,
                                                                              const RhsState* st,
                                                                              const double2* __restrict__ tw,
                                                                              double2* __restrict__ W) {
  constexpr int TP = RegTP<L>::value;
  extern __shared__ __align__(128) unsigned char smraw[];
  double2* sm = reinterpret_cast<double2*>(smraw);
  const int qb = blockIdx.x % og.nqb;
  const int r = blockIdx.x / og.nqb;
  if (!rhs_active(st, r)) return;
  const int qq = threadIdx.x / TP;
  const int j = threadIdx.x - qq * TP;
  const int ql = qb * og.QB + qq;         // pencil index within this slab's share
  const bool live = ql < og.Q;
  // single slab: the CTA's pencils of component a are one contiguous block
  // W[r][a][q0 .. q0+nq)[n0]; bulk-load it to smem as [a][qq][L] (TMA)
  const int nq = min(og.QB, og.Q - qb * og.QB);
  const bool bulk = og.tma && sm_.P == 1;
  __shared__ uint64_t bar;
  if (bulk) {
    if (threadIdx.x == 0) {
      mbar_init(&bar, 1);
      mbar_expect_tx(&bar, (unsigned)(C * nq * L * 16));
#pragma unroll
      for (int a = 0; a < C; ++a)
        bulk_g2s(sm + (size_t)a * og.QB * L, W + ((int64_t)(r * C + a) * og.Q + (int64_t)qb * og.QB) * L,
                 (unsigned)(nq * L * 16), &bar);
    }
    __syncthreads();
  }
  const int q = sm_.qs[sm_.me] + (live ? ql : 0);  // global (k2, k1) pencil index
  // element offset of entry i0 of this pencil's component rc: one contiguous
  // pencil for a single slab (uniform fast path), received segments otherwise.
  // Recomputed at the stores instead of held across the transforms (registers).
  auto eoff = [&](int i0, int rc) -> int64_t {
    if (sm_.P == 1) return ((int64_t)rc * og.Q + ql) * L + i0;
    const int p = slab_of(sm_.s0, sm_.P, i0);
    const int n0p = sm_.s0[p + 1] - sm_.s0[p];
    return sm_.roff[p] + (int64_t)ql * n0p + (i0 - sm_.s0[p]) + (int64_t)rc * og.Q * n0p;
  };
  if constexpr (C == 3) {
    const int k2 = q / og.n1, k1 = q - k2 * og.n1;
    const double xi1 = g.xi[1][live ? k1 : 0];
    const double xi2 = g.xi[2][live ? k2 : 0];
    auto ld = [&](int a, int i0) -> double2 {
      return bulk ? sm[((size_t)a * og.QB + qq) * L + i0] : W[eoff(i0, r * 3 + a)];
    };
    double2 v[2][9];
    if (bulk) mbar_wait(&bar, 0);
#pragma unroll
    for (int s = 0; s < 9; ++s) {
      const int i0 = j + s * TP;
      v[0][s] = live ? ld(0, i0) : make_double2(0.0, 0.0);
      v[1][s] = live ? g3_fold(xi1, xi2, ld(1, i0), ld(2, i0)) : make_double2(0.0, 0.0);
    }
    double2* smp = sm + (size_t)qq * C * L;
    fft_reg<L, 2, false>(v, smp, L, j, tw);
    const bool qzero = live && q == 0;
#pragma unroll
    for (int s = 0; s < 9; ++s) {
      const int i0 = j + s * TP;
      g3_mode(og, g.xi[0][i0], xi1, xi2, qzero && i0 == 0, v[0][s], v[1][s]);
    }
    fft_reg<L, 2, true>(v, smp, L, j, tw);
    if (bulk) {
      __syncthreads();
#pragma unroll
      for (int s = 0; s < 9; ++s) {
        const int i0 = j + s * TP;
        sm[((size_t)0 * og.QB + qq) * L + i0] = v[0][s];
        sm[((size_t)1 * og.QB + qq) * L + i0] = g3_scale(xi1, v[1][s]);
        sm[((size_t)2 * og.QB + qq) * L + i0] = g3_scale(xi2, v[1][s]);
      }
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
      return;
    }
    if (!live) return;
#pragma unroll
    for (int s = 0; s < 9; ++s) {
      const int i0 = j + s * TP;
      const double2 o[3] = {v[0][s], g3_scale(xi1, v[1][s]), g3_scale(xi2, v[1][s])};
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        if (sm_.fused) *outer_dst(sm_, W, og.Q, r * C + a, ql, i0) = o[a];
        else W[eoff(i0, r * C + a)] = o[a];
      }
    }
    if (sm_.fused) __threadfence_system();
    return;
  } else {
  double2 v[C][9];
  trace_stamp(0, 0);
  if (bulk) {
    mbar_wait(&bar, 0);
    trace_stamp(0, 1);
#pragma unroll
    for (int a = 0; a < C; ++a)
#pragma unroll
      for (int s = 0; s < 9; ++s)
        v[a][s] = live ? sm[((size_t)a * og.QB + qq) * L + j + s * TP] : make_double2(0.0, 0.0);
  } else {
#pragma unroll
    for (int a = 0; a < C; ++a) {
#pragma unroll
      for (int s = 0; s < 9; ++s)
        v[a][s] = live ? W[eoff(j + s * TP, r * C + a)] : make_double2(0.0, 0.0);
    }
  }
  double2* smp = sm + (size_t)qq * C * L;
  fft_reg<L, C, false>(v, smp, L, j, tw);
  trace_stamp(0, 2);
  // Gamma_hat(k) v = xi (xi . v) / den ; 0 at k = 0 (this branch is d = 2: g2_mode)
  static_assert(C == 2, "d = 3 takes the folded branch above");
  {
    const double xi1 = g.xi[1][live ? q : 0];
    const bool qzero = live && q == 0;
#pragma unroll
    for (int s = 0; s < 9; ++s) {
      const int i0 = j + s * TP;
      g2_mode(og, g.xi[0][i0], xi1, qzero && i0 == 0, v[0][s], v[1][s]);
    }
  }
  fft_reg<L, C, true>(v, smp, L, j, tw);
  trace_stamp(0, 3);
  if (bulk) {  // back through smem ([a][qq][L]) and one bulk store per component
    __syncthreads();
#pragma unroll
    for (int a = 0; a < C; ++a)
#pragma unroll
      for (int s = 0; s < 9; ++s) sm[((size_t)a * og.QB + qq) * L + j + s * TP] = v[a][s];
    fence_proxy_async();
    __syncthreads();
    if (threadIdx.x == 0) {
#pragma unroll
      for (int a = 0; a < C; ++a)
        bulk_s2g(W + ((int64_t)(r * C + a) * og.Q + (int64_t)qb * og.QB) * L, sm + (size_t)a * og.QB * L,
                 (unsigned)(nq * L * 16));
      bulk_commit();
      trace_stamp(0, 4);
      bulk_wait_read0();
      trace_stamp(0, 5);
    }
    return;
  }
  if (!live) return;
#pragma unroll
  for (int a = 0; a < C; ++a) {
#pragma unroll
    for (int s = 0; s < 9; ++s) {
      if (sm_.fused) *outer_dst(sm_, W, og.Q, r * C + a, ql, j + s * TP) = v[a][s];
      else W[eoff(j + s * TP, r * C + a)] = v[a][s];
    }
  }
  if (sm_.fused) __threadfence_system();
  }  // C == 2
}

}  // namespace fc

