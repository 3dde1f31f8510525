// Host engine and C ABI (include/fftcell_b200.h) of the B200 GaNi solver.
//
// One context = one GridSpec bound to one GPU: the coefficient field, the
// per-axis FFT plans and the solver workspace live in HBM for the lifetime of
// the context; the CG / fixed-point loops run entirely on the device with the
// per-RHS scalars (alpha, beta, stop flags, histories) in device memory.  The
// host only enqueues iterations and polls one pinned flag, one iteration
// behind, so the stream never drains between iterations.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>  // header-only: ranges cost nothing unless a tool is attached

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <map>
#include <string>
#include <vector>

#include "../../include/fftcell_b200.h"
#include "fc_kernels.cuh"
#include "fc_kernels_reg.cuh"
#include "fc_kernels_pipe.cuh"
#include "fc_kernels_pk.cuh"

// Field allocations carry this many spare bytes: 16-byte-aligned bulk copies
// (fc_tma.cuh) of a row block may read up to 8 bytes past its last element.
constexpr size_t kFieldPad = 64;

using namespace fc;

namespace {

thread_local std::string g_err;

int set_err(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

#define CK(call)                                                                          \
  do {                                                                                    \
    cudaError_t e_ = (call);                                                              \
    if (e_ != cudaSuccess)                                                                \
      return set_err(e_ == cudaErrorMemoryAllocation ? FC_ENOMEM : FC_ECUDA, "%s: %s (%s:%d)", #call, \
                     cudaGetErrorString(e_), __FILE__, __LINE__);                         \
  } while (0)

#define TRY(call)              \
  do {                         \
    int rc_ = (call);          \
    if (rc_ != FC_OK) return rc_; \
  } while (0)

// Scratch device buffer freed on every exit path of the C-ABI call that owns it.
template <typename T>
struct DevBuf {
  T* p = nullptr;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  ~DevBuf() {
    if (p) cudaFree(p);
  }
};

struct DevPlan {
  FftPlan plan{};
  double2* roots = nullptr;
  double2* rtw = nullptr;  // register-FFT twiddle table (L = 3^k only)
};

// register-path lengths (fc_fft_reg.cuh): 3^k for 9..2187 and 5 * 3^k for 45..1215
bool is_pow3_reg(int L) { return fc::is_reg_len(L); }

// Twiddle table of fc_fft_reg.cuh for L = 3^k: for radix-9 pass S >= 1 (Ns = 9^S)
// tw[off9(S) + (r-1) Ns + k] = w_L^{k r L/(9 Ns)}, r = 1..8, k < Ns; tail block
// tw[offT + (r-1) L/3 + b] = w_L^{b r}, r = 1, 2, b < L/3.
std::vector<double2> reg_twiddles(int L, const std::vector<double2>& roots) {
  if (!fc::is_pow3(L)) {  // L = 5 M: M's table (roots of M = roots of L at multiples of 5) + w_L^{r k2}
    const int M = L / 5;
    std::vector<double2> rm(M);
    for (int t = 0; t < M; ++t) rm[t] = roots[(int64_t)5 * t];
    std::vector<double2> tw = reg_twiddles(M, rm);
    if (tw.size() == 1 && fc::R9<9>::table == 0 && M == 9) tw.clear();  // M = 9: no inner table
    for (int r = 1; r < 5; ++r)
      for (int k2 = 0; k2 < M; ++k2) tw.push_back(roots[(int64_t)r * k2 % L]);
    return tw;
  }
  int K = 0;
  for (int t = L; t > 1; t /= 3) ++K;
  const int NP9 = K / 2;
  const bool tail = K % 2;
  std::vector<double2> tw;
  for (int S = 1, Ns = 9; S < NP9; ++S, Ns *= 9)
    for (int r = 1; r < 9; ++r)
      for (int k = 0; k < Ns; ++k) tw.push_back(roots[(int64_t)k * r * (L / (9 * Ns)) % L]);
  if (tail)
    for (int r = 1; r < 3; ++r)
      for (int b = 0; b < L / 3; ++b) tw.push_back(roots[(int64_t)b * r % L]);
  if (tw.empty()) tw.push_back(make_double2(1.0, 0.0));
  return tw;
}

// Factor plan for an odd length: radix-9 passes first, then 3, 5, other primes.
bool make_factors(int L, FftPlan& p) {
  p.L = L;
  p.nf = 0;
  int n = L;
  auto push = [&](int f) {
    if (p.nf >= kMaxFactors) return false;
    p.f[p.nf++] = f;
    return true;
  };
  while (n % 9 == 0) { if (!push(9)) return false; n /= 9; }
  while (n % 3 == 0) { if (!push(3)) return false; n /= 3; }
  while (n % 5 == 0) { if (!push(5)) return false; n /= 5; }
  for (int f = 7; n > 1; f += 2) {
    while (n % f == 0) { if (!push(f)) return false; n /= f; }
    if ((long long)f * f > n && n > 1) { if (!push(n)) return false; n = 1; }
  }
  return true;
}

struct Prof {
  std::string name;
  int64_t launches = 0;
  double ms = 0.0;
};

// Plan options: kernel selection and tile geometry, frozen when a context is
// created (copied from the process-wide table set through fc_set_plan_option).
// The defaults are the measured-fastest choices; the alternatives exist for the
// bitwise variant tests (tests/test_gpu_variants.py) and A/B measurements.
struct PlanOpts {
  int force_generic = 0;   // generic shared-memory Stockham FFT on every axis
  int row_threads = 0;     // first sweep CTA size (0: 128 for rows of 243 points, else 256)
  int row_threads_inv = 0; // last sweep CTA size, <= 512 (0: 256): its own row blocks and tensor boxes
  int mid_threads = 0;     // middle sweep CTA size (0: 256 for pencils <= 243, else 512)
  int outer_threads = 0;   // outer sweep CTA size (0: 2 pencils for short 3-D pencils, else 256)
  int row_tma = 1;         // TMA tensor boxes for the transposed half spectrum
  int mid_tma = 1;         // TMA inverse middle sweep
  int outer_tma = 1;       // bulk pencil copies in the outer sweep
  int outer_seq = -1;      // d = 3 outer sweep one component at a time (-1: for pencils >= 243)
  int inv_pipe = -1;       // persistent double-buffered last sweep (-1: for one-pencil row blocks)
  int mid_threads_inv = 0; // inverse middle sweep CTA size (0: 256 for pencils <= 243, else 3 pencils)
  int mid_map = 1;         // middle sweep transform mapping: 1 lane-fastest, 0 pencil-fastest
  int mid_tma_fwd = 1;     // forward middle sweep through TMA boxes (0: per-thread transposed stores)
  int aniso_fused = 1;     // packed coefficients: fused first sweep (0: pointwise kernel + row FFT)
  int two_field = 1;       // d = 3, one slab: two spectrum fields from the outer to the inverse middle sweep
  int fold_fwd = -1;       // ... and from the forward middle sweep to the outer sweep (needs two_field; -1: middle pencils >= 243)
  int inv_qpre = 1;        // last sweep: epilogue input staged by a bulk copy issued with the spectrum loads
  int fin_split = -1;      // reductions finalized by a separate launch (-1: from 1024 partial slots on)
  int defer_x = 1;         // CG x update deferred into the next first sweep
  int fused_exchange = 1;  // in-process slabs: sweeps store straight into the peers' buffers
  int sync_debug = 0;      // synchronize after every launch (error attribution)
};
PlanOpts g_plan_opts;

}  // namespace

struct fc_ctx {
  int device = 0;
  int dim = 0;
  int n[3] = {1, 1, 1};
  double Y[3] = {1, 1, 1};
  int64_t N = 0;
  cudaStream_t stream = nullptr;
  int smem_optin = 0;
  int num_sms = 0;
  PlanOpts opt;                // plan options (fixed at creation)
  bool force_generic = false;  // opt.force_generic: generic smem FFT for every axis

  std::map<int, DevPlan> plans;  // by length
  double* xi = nullptr;          // concatenated per-axis frequency tables
  int xi_off[3] = {0, 0, 0};

  double* A = nullptr;
  int coef_kind = -1;
  int64_t A_count = 0;
  // phase-indexed form of a packed field (fc_coef.inc); A may be null while it is resident
  uint16_t* lab = nullptr;
  double* tab = nullptr;
  int nph = 0;

  // workspace
  int Rcap = 0;
  int hcap = 0;
  double *x = nullptr, *r = nullptr, *p[2] = {nullptr, nullptr}, *Ap = nullptr;
  double2 *W1 = nullptr, *W2 = nullptr;
  double* part = nullptr;
  int64_t part_cap = 0;
  double* part2 = nullptr;  // chunk sums of the split finalize (kFinChunks x FC_MAX_RHS)
  RhsState* st = nullptr;
  double* hist = nullptr;
  int* any_active = nullptr;
  unsigned* counter = nullptr;  // last-CTA arrival counter of the fused finalize
  int* h_flag = nullptr;  // pinned, 4 slots
  int* h_mapped = nullptr;   // zero-copy "any RHS active" flag written by the finalizing CTA
  int* d_mapped = nullptr;   // its device alias
  cudaEvent_t flag_ev[4] = {};
  double* d_mat = nullptr;
  cudaEvent_t timer_ev[8] = {};

  // tiling
  RowGeo rg{};
  RowGeo rgi{};            // last sweep: its own row blocks (wider tensor boxes)
  MidGeo mg{};
  OuterGeo og{};
  size_t smem_row = 0, smem_mid = 0, smem_outer = 0, smem_line = 0;

  // instrumentation
  bool prof_on = false;
  std::vector<Prof> prof;
  std::map<std::string, int> prof_idx;
  std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> pending;
  std::vector<cudaEvent_t> ev_pool;
  int64_t launches = 0;
  const char* prof_tag = "";  // appended to profile names ("_rhs": right-hand-side / warm-start operators)

  Geo geo() const {
    Geo g{};
    g.dim = dim;
    for (int a = 0; a < 3; ++a) g.n[a] = n[a];
    g.N = N;
    g.invN = 1.0 / (double)Ng;
    for (int a = 0; a < dim; ++a) g.xi[a] = xi + xi_off[a];
    return g;
  }
  Coef coef() const { return Coef{A, coef_kind, lab, tab, nph}; }
  const FftPlan& plan(int L) const { return plans.at(L).plan; }
  const double2* rtw(int L) const { return plans.at(L).rtw; }
  // register-path tiling per sweep (0 = generic path)
  int row_npen = 0, mid_bp = 0, outer_qb = 0;
  int row_npen_inv = 0;     // pencils per CTA of the last sweep
  int pk_npen = 0;          // fused packed-coefficient first sweep: pencils per component (0: split)
  size_t smem_pk = 0;
  int outer_seq = 0;        // d = 3 outer sweep one component at a time
  bool two_field = false;   // outer sweep stores t once, inverse middle sweep rebuilds xi1 t, xi2 t (MidGeo::rebuild)
  bool fold_fwd = false;    // forward middle sweep stores u = xi1 v1 + xi2 v2 (mid_tma_fold)
  CUtensorMap tmW{};        // TMA view of the row-sweep spectrum (RowGeo::tma), first sweep's boxes
  CUtensorMap tmWi{};       // the same view with the last sweep's boxes (rgi)
  CUtensorMap tmP{};        // the same for the fused packed first sweep's row blocks (2 pk_npen rows)
  CUtensorMap tmM{};        // TMA view of the middle sweep's transposed side (MidGeo::tma), forward tiles
  CUtensorMap tmMi{};       // the same for the inverse sweep's tiles (mgi)
  MidGeo mgi{};             // inverse middle sweep tiling (its own pencils per CTA)
  int inv_pipe_blocks = 0;  // persistent double-buffered last sweep: CTAs per SM (0: off)
  int inv_pipe_stage = 0;   // its stage size (complex)
  static constexpr int inv_pipe_nst = 2;   // its stages
  size_t smem_row_r = 0, smem_row_inv_r = 0, smem_mid_r = 0, smem_outer_r = 0;

  // slab decomposition along axis 0.  A plain context is the P = 1
  // case.  A sharded context owns P slab contexts in `sub` (one per device; the
  // same device may host several slabs, which emulates P ranks on one GPU).
  int P = 1, me = 0;
  int n0g = 0;             // global axis-0 length
  int64_t Ng = 0;          // global voxel count
  int s0[kMaxSlabs + 1] = {};  // axis-0 partition
  int qs[kMaxSlabs + 1] = {};  // outer-pencil partition
  double2* W2r = nullptr;  // received outer pencils (P > 1)
  double* lsum = nullptr;  // slab-local reduction sums (2 x FC_MAX_RHS)
  std::vector<fc_ctx*> sub;
  cudaEvent_t sev[4] = {};  // phase events of this slab
  // one process per GPU: this process holds slab `me` only; exchanges and sums go
  // through NCCL (fc_create_dist)
  bool dist = false;
  void* comm = nullptr;        // ncclComm_t
  double* gathered = nullptr;  // [P][FC_MAX_RHS] all ranks' local sums (device)
  double* barrier = nullptr;   // [1 + P] nccl_barrier scratch (device)

  SlabMap slabmap(int R) const {
    SlabMap m{};
    m.P = P;
    m.me = me;
    m.n0l = n[0];
    for (int t = 0; t <= P; ++t) {
      m.s0[t] = s0[t];
      m.qs[t] = qs[t];
    }
    const int cdim = dim;
    long long off = 0;
    for (int t = 0; t < P; ++t) {  // send blocks: per destination t
      m.doff[t] = off;
      off += (long long)R * cdim * (qs[t + 1] - qs[t]) * n[0];
    }
    off = 0;
    for (int t = 0; t < P; ++t) {  // receive segments: per source t
      m.roff[t] = off;
      off += (long long)R * cdim * (qs[me + 1] - qs[me]) * (s0[t + 1] - s0[t]);
    }
    if (fused && sibs != nullptr) {  // peer destinations of the fused exchange (SlabMap::fused)
      m.fused = 1;
      for (int t = 0; t < P; ++t) {
        const fc_ctx* o = (*sibs)[t];
        long long rf = 0, rt = 0;
        for (int u = 0; u < me; ++u) {
          rf += (long long)R * cdim * (qs[t + 1] - qs[t]) * (s0[u + 1] - s0[u]);  // o's receive offset of source me
          rt += (long long)R * cdim * (qs[u + 1] - qs[u]) * (s0[t + 1] - s0[t]);  // o's send offset of destination me
        }
        m.fwd[t] = o->W2r + rf;
        m.ret[t] = o->W2 + rt;
      }
    } else if (fused && ipc_rcap > 0) {  // same offsets in the peers' buffers mapped through CUDA IPC
      m.fused = 1;
      for (int t = 0; t < P; ++t) {
        long long rf = 0, rt = 0;
        for (int u = 0; u < me; ++u) {
          rf += (long long)R * cdim * (qs[t + 1] - qs[t]) * (s0[u + 1] - s0[u]);
          rt += (long long)R * cdim * (qs[u + 1] - qs[u]) * (s0[t + 1] - s0[t]);
        }
        double2* w2 = t == me ? W2 : static_cast<double2*>(ipc_peer[t][0]);
        double2* w2r = t == me ? W2r : static_cast<double2*>(ipc_peer[t][1]);
        m.fwd[t] = w2r + rf;
        m.ret[t] = w2 + rt;
      }
    }
    return m;
  }
  // one process per GPU with the fused exchange: the peers' W2 / W2r mapped
  // into this process (CUDA IPC), opened for workspace capacity ipc_rcap
  void* ipc_peer[kMaxSlabs][2] = {};
  int ipc_rcap = 0;
  unsigned* sphere_bits = nullptr;               // cfg5 generator coverage bitmap (fc_spheres_stamp)
  unsigned long long* sphere_count = nullptr;
  int fused = 0;                                 // fused peer-store exchange (in-process slabs)
  const std::vector<fc_ctx*>* sibs = nullptr;    // all slabs of the parent (fused exchange)
};

namespace {

cudaEvent_t take_event(fc_ctx* c) {
  if (!c->ev_pool.empty()) {
    cudaEvent_t e = c->ev_pool.back();
    c->ev_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  cudaEventCreate(&e);
  return e;
}

// Profiling span on the context's stream (no launch counted): bench.py reads
// it like a kernel, e.g. the NCCL / copy-engine exchanges ("exchange").
struct ProfSpan {
  cudaEvent_t e0 = nullptr;
};
ProfSpan prof_begin(fc_ctx* c) {
  nvtxRangePushA("exchange");
  ProfSpan sp;
  if (c->prof_on) {
    sp.e0 = take_event(c);
    cudaEventRecord(sp.e0, c->stream);
  }
  return sp;
}
void prof_end(fc_ctx* c, const char* name, const ProfSpan& sp) {
  nvtxRangePop();
  if (!c->prof_on || sp.e0 == nullptr) return;
  cudaEvent_t e1 = take_event(c);
  cudaEventRecord(e1, c->stream);
  auto it = c->prof_idx.find(name);
  int idx;
  if (it == c->prof_idx.end()) {
    idx = (int)c->prof.size();
    c->prof_idx[name] = idx;
    c->prof.push_back(Prof{name, 0, 0.0});
  } else {
    idx = it->second;
  }
  c->pending.push_back({idx, {sp.e0, e1}});
}

// NVTX range (nsys / ncu timelines): one per sweep launch, exchange and solver call.
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

// Launch wrapper: counts launches and (when profiling) brackets with events.
template <typename F>
int launch(fc_ctx* c, const char* name, F&& f) {
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (c->prof_on) {
    e0 = take_event(c);
    e1 = take_event(c);
    cudaEventRecord(e0, c->stream);
  }
  {
    const NvtxRange range(name);
    f();
  }
  c->launches++;
  cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) return set_err(FC_ECUDA, "launch of %s failed: %s", name, cudaGetErrorString(err));
  if (c->opt.sync_debug) {
    err = cudaStreamSynchronize(c->stream);
    if (err != cudaSuccess) return set_err(FC_ECUDA, "kernel %s failed: %s", name, cudaGetErrorString(err));
  }
  if (c->prof_on) {
    cudaEventRecord(e1, c->stream);
    const std::string key = std::string(name) + c->prof_tag;
    auto it = c->prof_idx.find(key);
    int idx;
    if (it == c->prof_idx.end()) {
      idx = (int)c->prof.size();
      c->prof_idx[key] = idx;
      c->prof.push_back(Prof{key, 0, 0.0});
    } else {
      idx = it->second;
    }
    c->pending.push_back({idx, {e0, e1}});
  }
  return FC_OK;
}

// Profile names of the launches enqueued while alive get `tag` appended (bench.py
// charges the right-hand-side / warm-start operators their own byte counts).
struct ProfTag {
  fc_ctx* c;
  const char* saved;
  ProfTag(fc_ctx* c_, const char* tag) : c(c_), saved(c_->prof_tag) { c->prof_tag = tag; }
  ~ProfTag() { c->prof_tag = saved; }
};

// Accumulate finished profiling intervals (call after a stream sync).
void drain_profile(fc_ctx* c) {
  for (auto& pe : c->pending) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, pe.second.first, pe.second.second);
    c->prof[pe.first].launches += 1;
    c->prof[pe.first].ms += ms;
    c->ev_pool.push_back(pe.second.first);
    c->ev_pool.push_back(pe.second.second);
  }
  c->pending.clear();
}

int ensure_plan(fc_ctx* c, int L) {
  if (c->plans.count(L)) return FC_OK;
  DevPlan dp;
  if (!make_factors(L, dp.plan)) return set_err(FC_ENOTSUP, "cannot factor length %d", L);
  std::vector<double2> roots(L);
  for (int t = 0; t < L; ++t) {
    // exp(-2 pi i t / L) in extended precision, exactly conjugate-symmetric
    int tt = t <= L / 2 ? t : L - t;
    long double ang = 2.0L * 3.141592653589793238462643383279502884L * (long double)tt / (long double)L;
    double cr = (double)cosl(ang), si = (double)sinl(ang);
    roots[t] = make_double2(cr, t <= L / 2 ? -si : si);
  }
  roots[0] = make_double2(1.0, 0.0);
  CK(cudaMalloc(&dp.roots, sizeof(double2) * L));
  CK(cudaMemcpy(dp.roots, roots.data(), sizeof(double2) * L, cudaMemcpyHostToDevice));
  dp.plan.roots = dp.roots;
  if (is_pow3_reg(L) && !c->force_generic) {
    std::vector<double2> tw = reg_twiddles(L, roots);
    CK(cudaMalloc(&dp.rtw, sizeof(double2) * tw.size()));
    CK(cudaMemcpy(dp.rtw, tw.data(), sizeof(double2) * tw.size(), cudaMemcpyHostToDevice));
  }
  c->plans[L] = dp;
  return FC_OK;
}

template <typename K>
int allow_smem(K kernel, int bytes) {
  cudaFuncAttributes fa;
  CK(cudaFuncGetAttributes(&fa, kernel));
  CK(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes - (int)fa.sharedSizeBytes));
  return FC_OK;
}

// Tile selection: smem per CTA <= soft cap (two CTAs per SM) if possible, else opt-in max.
int choose_tiles(fc_ctx* c) {
  const size_t soft = 100 * 1024, hard = (size_t)c->smem_optin - 1024;
  const int d = c->dim;
  if (d == 1) {
    c->smem_line = (size_t)32 * c->n[0];
    if (c->smem_line > hard) return set_err(FC_ENOTSUP, "grid axis of length %d exceeds the shared-memory line limit", c->n[0]);
    return FC_OK;
  }
  RowGeo& rg = c->rg;
  rg.nl = c->n[d - 1];
  rg.hl = (rg.nl + 1) / 2;
  rg.np = c->n[d - 2];
  rg.no = d == 3 ? c->n[0] : 1;
  {
    int best = 0;
    const int npe = (rg.np + 1) & ~1;
    for (int B = 16; B >= 2; B -= 2) {
      if (B > npe && B > 2) continue;
      size_t bytes = (size_t)16 * B * rg.nl;
      if (bytes <= soft) { best = B; break; }
    }
    if (best == 0 && (size_t)32 * rg.nl <= hard) best = 2;
    if (best == 0) return set_err(FC_ENOTSUP, "contiguous axis of length %d exceeds the shared-memory limit", rg.nl);
    rg.B = best;
    rg.ntiles = (rg.np + rg.B - 1) / rg.B;
    c->smem_row = (size_t)16 * rg.B * rg.nl;
  }
  if (d == 3) {
    MidGeo& mg = c->mg;
    mg.n0 = c->n[0];
    mg.n1 = c->n[1];
    mg.h2 = (c->n[2] + 1) / 2;
    int best = 0;
    for (int B = 16; B >= 1; B /= 2) {
      if (B > mg.n0 && B > 1) continue;
      if ((size_t)32 * B * mg.n1 <= soft) { best = B; break; }
    }
    if (best == 0 && (size_t)32 * mg.n1 <= hard) best = 1;
    if (best == 0) return set_err(FC_ENOTSUP, "middle axis of length %d exceeds the shared-memory limit", mg.n1);
    mg.B = best;
    mg.nib = (mg.n0 + best - 1) / best;
    c->smem_mid = (size_t)32 * best * mg.n1;
  }
  {
    OuterGeo& og = c->og;
    og.n0 = c->n0g;
    og.n1 = d == 3 ? c->n[1] : 1;
    og.h_last = (c->n[d - 1] + 1) / 2;
    og.Q = c->qs[c->me + 1] - c->qs[c->me];
    int best = 0;
    for (int QB = 32; QB >= 1; QB /= 2) {
      if (QB > og.Q && QB > 1) continue;
      if ((size_t)32 * d * QB * og.n0 <= soft) { best = QB; break; }
    }
    if (best == 0 && (size_t)32 * d * og.n0 <= hard) best = 1;
    if (best == 0) return set_err(FC_ENOTSUP, "outer axis of length %d exceeds the shared-memory limit for d=%d", og.n0, d);
    og.QB = best;
    og.nqb = (og.Q + best - 1) / best;
    c->smem_outer = (size_t)32 * d * best * og.n0;
  }
  c->rgi = c->rg;
  // register-resident path for power-of-three axes (fc_kernels_reg.cuh)
  const PlanOpts& op = c->opt;
  if (c->force_generic) return FC_OK;
  if (is_pow3_reg(rg.nl)) {
    const int TP = rg.nl / 9;
    // measured at 243^3 (profiles/r02n_ab_row_inv_threads_cfg3.txt): the first sweep runs
    // 10 % faster in 8-row blocks, the last sweep 30 % slower, so each has its own blocks
    const int rtf = op.row_threads > 0 ? op.row_threads : (TP == 27 ? 128 : 256);
    int npen = std::max(1, std::min(16, std::min(rtf, 256) / TP));
    npen = std::min(npen, (rg.np + 1) / 2);
    rg.B = 2 * npen;
    rg.ntiles = (rg.np + rg.B - 1) / rg.B;
    c->row_npen = npen;
    // exchange buffer (16 npen (L+1)) + staging: first sweep u, p_old, A (3 x 2 npen L
    // doubles)
    c->smem_row_r = (size_t)24 * (((size_t)2 * npen * rg.nl + 3) & ~(size_t)1);
    // TMA boxes of the transposed spectrum: nbox boxes of boxK modes x 2 npen rows
    rg.nbox = (rg.hl + 255) / 256;
    rg.boxK = ((rg.hl + rg.nbox - 1) / rg.nbox + 3) & ~3;  // boxes start 128-byte aligned in smem
    const size_t ybytes = (size_t)16 * rg.nbox * rg.boxK * 2 * npen;
    c->smem_row_r = std::max(c->smem_row_r, (size_t)16 * (((size_t)npen * rg.nl + 7) & ~(size_t)7) + ybytes);
    // last sweep: its own row blocks (up to 512 threads): wider rows in the
    // transposed tensor boxes (16 bytes per row and mode)
    {
      const int rti = op.row_threads_inv > 0 ? op.row_threads_inv : 256;
      int npi = std::max(1, std::min(16, std::min(rti, kMaxBlock) / TP));
      npi = std::min(npi, (rg.np + 1) / 2);
      RowGeo& ri = c->rgi;
      ri = rg;
      ri.B = 2 * npi;
      ri.ntiles = (rg.np + ri.B - 1) / ri.B;
      c->row_npen_inv = npi;
      const size_t ybi = (size_t)16 * rg.nbox * rg.boxK * 2 * npi;
      c->smem_row_inv_r = std::max((size_t)16 * npi * (rg.nl + 1), ybi);
      // the epilogue input (p / e of the row block) staged behind the spectrum by
      // a bulk copy, if the CTAs the register budget allows still fit an SM
      ri.qoff = 0;
      if (op.inv_qpre) {
        const int nt = npi * TP;
        const int want = nt <= 256 ? 3 : (nt <= 384 ? 2 : 1);
        const size_t qoff = (c->smem_row_inv_r + 127) & ~(size_t)127;
        const size_t tot = qoff + (size_t)8 * (2 * npi * rg.nl + 2);
        if (want * (tot + 1024) <= (size_t)c->smem_optin + 1024) {
          ri.qoff = (int)qoff;
          c->smem_row_inv_r = tot;
        }
      }
    }
    // packed coefficients: fused first sweep (fc_kernels_pk.cuh), d components of
    // npk pencils per CTA (<= 256 threads), if two CTAs fit an SM
    if (op.aniso_fused && d >= 2) {
      // (a tensor box holds 4 npk doubles per row: at most 256, so npk <= 64)
      const int npk = std::max(1, std::min((rg.np + 1) / 2, std::min(64, 256 / (d * TP))));
      const size_t sm = pk_smem(rg.nl, d, npk, rg.nbox, rg.boxK);
      if (d * TP <= 256 && 2 * (sm + 1024) <= (size_t)c->smem_optin + 1024 && sm <= 110 * 1024) {
        c->pk_npen = npk;
        c->smem_pk = sm;
      }
    }
  }
  if (d == 3 && is_pow3_reg(c->n[1])) {
    const int TP = c->n[1] / 9;
    const int L1 = c->n[1];
    // pencils per CTA: 256 threads for pencils of <= 243 points (cfg3); for 729
    // (cfg4, TMA on both sides, lane-fastest mapping) 2 pencils forward and 3
    // inverse measured best (profiles/r02d_ab_mid_cfg4.txt)
    auto geo = [&](MidGeo& m, int threads) {
      int bp = std::max(1, std::min(16, std::min(threads, kMaxBlock) / TP));
      bp = std::min(bp, c->n[0]);
      m.B = bp;
      m.nib = (m.n0 + bp - 1) / bp;
      // TMA boxes on the transposed side: rows * bp a multiple of 8 (128-byte boxes)
      m.nbox = (L1 + 255) / 256;
      int rows = (L1 + m.nbox - 1) / m.nbox;
      while ((rows * bp) % 8) ++rows;
      if (rows > 256) m.nbox = 0;  // no box shape: per-thread path
      m.rows = rows;
      return (size_t)16 * std::max(bp * L1, m.nbox * rows * bp);
    };
    const int mtf = op.mid_threads > 0 ? op.mid_threads : (TP <= 27 ? 256 : (c->P > 1 ? 512 : 2 * TP));
    const int mti = op.mid_threads_inv > 0 ? op.mid_threads_inv : (TP <= 27 ? 256 : 3 * TP);
    c->mgi = c->mg;
    c->smem_mid_r = std::max(geo(c->mg, mtf), geo(c->mgi, mti));
    c->mid_bp = c->mg.B;
  }
  if (is_pow3_reg(c->n0g)) {
    OuterGeo& og = c->og;
    const int TP = c->n0g / 9;
    // d = 3 holds 3 x 9 complex per thread: short pencils (TP <= 32) run best
    // as small CTAs (measured at 243^3: 2 pencils, 54 threads, -22 %)
    const int ot = op.outer_threads > 0 ? op.outer_threads : ((d == 3 && TP <= 32) ? 2 * TP : 256);
    int qb = std::max(1, std::min(32, std::min(ot, kMaxBlockOuter) / TP));
    qb = std::min(qb, og.Q);
    og.QB = qb;
    og.nqb = (og.Q + qb - 1) / qb;
    c->outer_qb = qb;
    c->smem_outer_r = (size_t)16 * d * qb * c->n0g;
    og.tma = op.outer_tma;
    // d = 3 with long pencils: one component at a time (measured at 729^3: -19 %;
    // slower for the small 243-length CTAs and for d = 2)
    c->outer_seq = d == 3 ? (op.outer_seq >= 0 ? op.outer_seq : TP >= 27) : (d == 2 && op.outer_seq > 0);
  }
  return FC_OK;
}

// ---- compile-time dispatch of the register kernels on the axis length ----------
#define FC_POW3_SWITCH(L, BODY)         \
  switch (L) {                           \
    case 9: { constexpr int LL = 9; BODY; } break;       \
    case 27: { constexpr int LL = 27; BODY; } break;     \
    case 81: { constexpr int LL = 81; BODY; } break;     \
    case 243: { constexpr int LL = 243; BODY; } break;   \
    case 729: { constexpr int LL = 729; BODY; } break;   \
    case 2187: { constexpr int LL = 2187; BODY; } break; \
    case 45: { constexpr int LL = 45; BODY; } break;     \
    case 135: { constexpr int LL = 135; BODY; } break;   \
    case 405: { constexpr int LL = 405; BODY; } break;   \
    case 1215: { constexpr int LL = 1215; BODY; } break; \
    default: break;                      \
  }

int allow_reg_smem(int mx) {
  int rc = FC_OK;
  auto al = [&](auto k) { if (rc == FC_OK) rc = allow_smem(k, mx); };
  for (int L : {9, 27, 81, 243, 729, 2187, 45, 135, 405, 1215}) {
    FC_POW3_SWITCH(L, {
      al(k_row_fwd_pk<LL, 2, false>);
      al(k_row_fwd_pk<LL, 3, false>);
      al(k_row_fwd_pk<LL, 2, true>);
      al(k_row_fwd_pk<LL, 3, true>);
      al(k_row_fwd_r<LL>);
      al(k_row_inv_r<LL, 256>);
      al(k_row_inv_r<LL, 384>);
      al(k_row_inv_r<LL, 512>);
      al(k_mid_r<LL, false>);
      al(k_mid_r<LL, true>);
      al(k_mid_tma<LL, true, false>);
      al(k_mid_tma<LL, true, true>);
      al(k_mid_tma<LL, false, false>);
      al(k_mid_tma<LL, false, true>);
      al(k_outer_r<LL, 2>);
      al(k_outer_r<LL, 3>);
      al(k_outer_seq<LL, 2>);
      al(k_outer_seq<LL, 3>);
      al(k_outer_seq<LL, 3, true>);
      al(k_outer_seq<LL, 3, true, true>);
      al(k_mid_tma_fold<LL, false>);
      al(k_mid_tma_fold<LL, true>);
    });
  }
  return rc;
}

// TMA tensor map over the row-sweep spectrum (d >= 2, register path): doubles
// {2 np, hl, Rcap c no}, box {2B, boxK, 1} (fc_tma.cuh).  The driver entry point
// is resolved through the runtime, so libcuda is not linked.  FC_ROW_TMA=0
// keeps the per-thread transposed loads / stores.
int make_row_tmap(fc_ctx* c) {
  RowGeo& rg = c->rg;
  rg.tma = 0;
  c->rgi.tma = 0;
  if (c->dim < 2 || !c->row_npen || rg.nbox == 0 || !c->opt.row_tma) {
    c->pk_npen = 0;  // the fused packed first sweep stores through its tensor map
    return FC_OK;
  }
  static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  if (encode == nullptr) {
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&encode, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return set_err(FC_ECUDA, "cuTensorMapEncodeTiled is unavailable");
  }
  void* base = c->dim == 3 ? (void*)c->W1 : (void*)c->W2;
  const int B = 2 * c->row_npen;
  cuuint64_t dims[3] = {(cuuint64_t)2 * rg.np, (cuuint64_t)rg.hl, (cuuint64_t)c->Rcap * c->dim * rg.no};
  cuuint64_t strides[2] = {(cuuint64_t)16 * rg.np, (cuuint64_t)16 * rg.np * rg.hl};
  cuuint32_t box[3] = {(cuuint32_t)(2 * B), (cuuint32_t)rg.boxK, 1};
  cuuint32_t es[3] = {1, 1, 1};
  const CUresult rc = encode(&c->tmW, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, base, dims, strides, box, es,
                             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (rc != CUDA_SUCCESS) return set_err(FC_ECUDA, "cuTensorMapEncodeTiled failed (%d)", (int)rc);
  rg.tma = 1;
  {  // same view, the last sweep's boxes
    cuuint32_t boxi[3] = {(cuuint32_t)(2 * c->rgi.B), (cuuint32_t)rg.boxK, 1};
    const CUresult ri = encode(&c->tmWi, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, base, dims, strides, boxi, es,
                               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (ri != CUDA_SUCCESS) return set_err(FC_ECUDA, "cuTensorMapEncodeTiled (last sweep) failed (%d)", (int)ri);
    c->rgi.tma = 1;
  }
  if (c->pk_npen) {  // same view, boxes of the fused packed first sweep's 2 pk_npen rows
    cuuint32_t boxp[3] = {(cuuint32_t)(4 * c->pk_npen), (cuuint32_t)rg.boxK, 1};
    const CUresult rp = encode(&c->tmP, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, base, dims, strides, boxp, es,
                               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                               CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (rp != CUDA_SUCCESS) return set_err(FC_ECUDA, "cuTensorMapEncodeTiled (packed first sweep) failed (%d)", (int)rp);
  }
  // middle sweep (d = 3, one slab): W2[rc][k2][k1][i0] as doubles {2 n0, n1, R c h2}
  c->mg.tma = c->mgi.tma = 0;
  if (c->dim == 3 && c->mid_bp && c->P == 1 && c->mg.nbox > 0 && c->mgi.nbox > 0 && c->opt.mid_tma) {
    for (int k = 0; k < 2; ++k) {
      MidGeo& mg = k == 0 ? c->mg : c->mgi;
      cuuint64_t md[3] = {(cuuint64_t)2 * mg.n0, (cuuint64_t)mg.n1, (cuuint64_t)c->Rcap * c->dim * mg.h2};
      cuuint64_t ms[2] = {(cuuint64_t)16 * mg.n0, (cuuint64_t)16 * mg.n0 * mg.n1};
      cuuint32_t mb[3] = {(cuuint32_t)(2 * mg.B), (cuuint32_t)mg.rows, 1};
      const CUresult rm = encode(k == 0 ? &c->tmM : &c->tmMi, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, c->W2, md, ms, mb,
                                 es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                 CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      if (rm != CUDA_SUCCESS) return set_err(FC_ECUDA, "cuTensorMapEncodeTiled (middle sweep) failed (%d)", (int)rm);
      mg.tma = 1;
    }
  }
  c->two_field = c->dim == 3 && c->P == 1 && c->opt.two_field && c->mgi.tma && c->outer_qb && c->outer_seq && c->og.tma;
  // (middle pencils of 243 and more, measured; shorter ones keep three fields)
  c->fold_fwd = c->two_field && c->mg.tma && c->opt.mid_tma_fwd && c->mg.B * (c->n[1] / 9) <= fold_threads(c->n[1]) &&
                (c->opt.fold_fwd >= 0 ? c->opt.fold_fwd != 0 : c->n[1] / 9 >= 27);
  return FC_OK;
}

int ensure_workspace(fc_ctx* c, int R, int hcap) {
  const int d = c->dim;
  const int64_t field = (int64_t)d * c->N;
  if (R > c->Rcap) {
    for (double* q : {c->x, c->r, c->p[0], c->p[1], c->Ap}) cudaFree(q);
    cudaFree(c->W1);
    cudaFree(c->W2);
    cudaFree(c->st);
    c->x = c->r = c->p[0] = c->p[1] = c->Ap = nullptr;
    c->W1 = c->W2 = nullptr;
    c->st = nullptr;
    c->Rcap = 0;
    const size_t fb = sizeof(double) * field * R;
    CK(cudaMalloc(&c->x, fb + kFieldPad));
    CK(cudaMalloc(&c->r, fb + kFieldPad));
    CK(cudaMalloc(&c->p[0], fb + kFieldPad));
    CK(cudaMalloc(&c->p[1], fb + kFieldPad));
    CK(cudaMalloc(&c->Ap, fb + kFieldPad));
    if (d >= 2) {
      int64_t spec = (int64_t)R * d * c->N / c->n[d - 1] * ((c->n[d - 1] + 1) / 2);
      CK(cudaMalloc(&c->W2, sizeof(double2) * spec));
      if (d == 3) CK(cudaMalloc(&c->W1, sizeof(double2) * spec));
      if (c->P > 1) {
        cudaFree(c->W2r);
        c->W2r = nullptr;
        const int64_t recv = (int64_t)R * d * (c->qs[c->me + 1] - c->qs[c->me]) * c->n0g;
        CK(cudaMalloc(&c->W2r, sizeof(double2) * recv));
      }
    }
    CK(cudaMalloc(&c->st, sizeof(RhsState) * R));
    c->Rcap = R;
    TRY(make_row_tmap(c));
  }
  // partial-sum slots: max over row sweeps, vector tiles, energy chunks
  int64_t nslot_row = d == 1 ? 1 : (int64_t)c->rgi.no * c->rgi.ntiles * d;
  int64_t nslot_vec = (field + kVecTile - 1) / kVecTile;
  int64_t nslot_en = (c->N + 8191) / 8192;
  int64_t need = std::max<int64_t>(std::max(std::max(nslot_row, nslot_vec), nslot_en), 64) * FC_MAX_RHS * FC_MAX_RHS;
  if (need > c->part_cap) {
    cudaFree(c->part);
    c->part = nullptr;
    CK(cudaMalloc(&c->part, sizeof(double) * need));
    c->part_cap = need;
  }
  if (hcap > c->hcap) {  // history rows: FC_MAX_RHS rows of hcap entries
    cudaFree(c->hist);
    c->hist = nullptr;
    CK(cudaMalloc(&c->hist, sizeof(double) * (int64_t)hcap * FC_MAX_RHS));
    c->hcap = hcap;
  }
  return FC_OK;
}

int64_t nslot_row(const fc_ctx* c) { return c->dim == 1 ? 1 : (int64_t)c->rgi.no * c->rgi.ntiles * c->dim; }
int64_t nslot_vec(const fc_ctx* c) { return ((int64_t)c->dim * c->N + kVecTile - 1) / kVecTile; }

// Reducing launches on large grids hand their finalize to k_fin_split: returns
// the FinArgs the reducing kernel should get (FIN_NONE when split).
constexpr int kFinChunks = 128;
bool fin_is_split(const fc_ctx* c, const FinArgs& f) {
  if (f.mode == FIN_NONE || f.part == nullptr) return false;
  return c->opt.fin_split >= 0 ? c->opt.fin_split != 0 : f.nslot >= 1024;
}
FinArgs fin_for_kernel(const fc_ctx* c, const FinArgs& f) {
  FinArgs k = f;
  if (fin_is_split(c, f)) k.mode = FIN_NONE;
  return k;
}
int launch_fin_split(fc_ctx* c, const FinArgs& f) {
  if (!fin_is_split(c, f)) return FC_OK;
  if (c->part2 == nullptr) CK(cudaMalloc(&c->part2, sizeof(double) * kFinChunks * FC_MAX_RHS));
  const int G = std::max(1, std::min(kFinChunks, f.nslot / 2048));
  const dim3 grid = G == 1 ? dim3(1, 1) : dim3(G, f.R);
  const int nt = G == 1 ? 256 * std::min(f.R, 4) : 256;
  return launch(c, "finalize", [&] { k_fin_split<<<grid, nt, 0, c->stream>>>(f, c->part2, G); });
}

#include "fc_coef.inc"

// One operator application over R fields, in three phases so a sharded run can
// exchange spectra between them: 0 = first sweep (+ forward middle sweep),
// 1 = outer sweep (Gamma_hat), 2 = inverse middle sweep + last sweep.
enum Phase { PH_FWD = 1, PH_OUTER = 2, PH_INV = 4, PH_ALL = 7 };
int run_phases(fc_ctx* c, int phases, int R, const InArgs& ia, EpArgs ea, int orth, const double M[3][3],
               const RhsState* st) {
  const Geo g = c->geo();
  const int d = c->dim;
  // indexed coefficients are read by the fused packed first sweep only
  if ((phases & PH_FWD) && c->lab != nullptr && c->A == nullptr && ia.mode != IN_RAW && !(d >= 2 && c->pk_npen))
    TRY(ensure_expanded(c));
  const Coef C = c->coef();
  cudaStream_t s = c->stream;
  if (ea.part != nullptr) ea.nslot = (int)nslot_row(c);
  const SlabMap smap = c->slabmap(R);
  if (d == 1) {
    const FftPlan pl = c->plan(c->n[0]);
    const size_t sm = c->smem_line;
    return launch(c, "line", [&] { k_line<<<R, kThreads, sm, s>>>(g, C, ia, ea, st, pl, orth, M[0][0]); });
  }
  const RowGeo rg = c->rg;
  const int64_t nrow_blocks = (int64_t)R * rg.no * rg.ntiles * d;
  double2* Wrow = d == 3 ? c->W1 : c->W2;
  const MidGeo mg = c->mg;
  const int64_t nmid = (int64_t)R * d * mg.h2 * mg.nib;
  auto mid = [&](bool inv) -> int {
    const double2* src = inv ? c->W2 : c->W1;
    double2* dst = inv ? c->W1 : c->W2;
    if (c->mid_bp) {
      const double2* tw = c->rtw(c->n[1]);
      const bool jf = c->opt.mid_map != 0;
      MidGeo mt = inv ? c->mgi : mg;
      mt.rebuild = inv && c->two_field;
      if (!inv && c->fold_fwd) {
        const int nt = mt.B * (c->n[1] / 9);
        const int64_t nblk = (int64_t)R * 2 * mt.h2 * mt.nib;
        mt.regA = (int)(c->smem_mid_r / 16);
        const size_t smem = 2 * c->smem_mid_r;  // pencils of component 1 | pencils of component 2, then the boxes
        return launch(c, "mid_fwd", [&] {
          if (jf) FC_POW3_SWITCH(c->n[1], (k_mid_tma_fold<LL, true><<<(unsigned)nblk, nt, smem, s>>>(g, mt, st, tw, src, dst, c->tmM)))
          else FC_POW3_SWITCH(c->n[1], (k_mid_tma_fold<LL, false><<<(unsigned)nblk, nt, smem, s>>>(g, mt, st, tw, src, dst, c->tmM)))
        });
      }
      if ((inv || c->opt.mid_tma_fwd) && mt.tma) {
        // TMA on both sides (bulk pencil copies, tensor boxes on the transposed side)
        const int nt = mt.B * (c->n[1] / 9);
        const int64_t nblk = (int64_t)R * d * mt.h2 * mt.nib;
        const CUtensorMap& tm = inv ? c->tmMi : c->tmM;
        return launch(c, inv ? "mid_inv" : "mid_fwd", [&] {
          if (inv && jf) FC_POW3_SWITCH(c->n[1], (k_mid_tma<LL, true, true><<<(unsigned)nblk, nt, c->smem_mid_r, s>>>(g, mt, st, tw, src, dst, tm)))
          else if (inv) FC_POW3_SWITCH(c->n[1], (k_mid_tma<LL, true, false><<<(unsigned)nblk, nt, c->smem_mid_r, s>>>(g, mt, st, tw, src, dst, tm)))
          else if (jf) FC_POW3_SWITCH(c->n[1], (k_mid_tma<LL, false, true><<<(unsigned)nblk, nt, c->smem_mid_r, s>>>(g, mt, st, tw, src, dst, tm)))
          else FC_POW3_SWITCH(c->n[1], (k_mid_tma<LL, false, false><<<(unsigned)nblk, nt, c->smem_mid_r, s>>>(g, mt, st, tw, src, dst, tm)))
        });
      }
      // per-thread transposed side (slab maps of the sharded paths)
      const int nt = c->mid_bp * (c->n[1] / 9);
      return launch(c, inv ? "mid_inv" : "mid_fwd", [&] {
        if (inv) FC_POW3_SWITCH(c->n[1], (k_mid_r<LL, true><<<(unsigned)nmid, nt, c->smem_mid_r, s>>>(g, mg, smap, st, tw, src, dst)))
        else FC_POW3_SWITCH(c->n[1], (k_mid_r<LL, false><<<(unsigned)nmid, nt, c->smem_mid_r, s>>>(g, mg, smap, st, tw, src, dst)))
      });
    }
    const FftPlan pl1 = c->plan(c->n[1]);
    return launch(c, inv ? "mid_inv" : "mid_fwd", [&] {
      if (inv) k_mid<true><<<(unsigned)nmid, kThreads, c->smem_mid, s>>>(g, mg, smap, st, pl1, src, dst);
      else k_mid<false><<<(unsigned)nmid, kThreads, c->smem_mid, s>>>(g, mg, smap, st, pl1, src, dst);
    });
  };
  if (phases & PH_FWD) {
    const double2* twr = c->row_npen ? c->rtw(rg.nl) : nullptr;
    if (C.kind == 1 && c->pk_npen && ia.mode != IN_RAW) {
      // packed coefficients, fused: y = M(x) u in shared memory, row FFT of all d
      // components in the same CTA (fc_kernels_pk.cuh)
      const int npk = c->pk_npen;
      const int64_t nb = (int64_t)R * rg.no * ((rg.np + 2 * npk - 1) / (2 * npk));
      const int nt = d * npk * (rg.nl / 9);
      TRY(launch(c, "row_fwd", [&] {
        if (C.lab != nullptr) {
          size_t smi = c->smem_pk;
#if FC_PK_IDX_SMEM
          if ((size_t)C.nph * (d * (d + 1) / 2) * 8 <= 32768) smi += (size_t)C.nph * (d * (d + 1) / 2) * 8;
#endif
          if (d == 2) FC_POW3_SWITCH(rg.nl, (k_row_fwd_pk<LL, 2, true><<<(unsigned)nb, nt, smi, s>>>(g, rg, C, ia, st, twr, npk, c->tmP)))
          else FC_POW3_SWITCH(rg.nl, (k_row_fwd_pk<LL, 3, true><<<(unsigned)nb, nt, smi, s>>>(g, rg, C, ia, st, twr, npk, c->tmP)))
        } else {
          if (d == 2) FC_POW3_SWITCH(rg.nl, (k_row_fwd_pk<LL, 2, false><<<(unsigned)nb, nt, c->smem_pk, s>>>(g, rg, C, ia, st, twr, npk, c->tmP)))
          else FC_POW3_SWITCH(rg.nl, (k_row_fwd_pk<LL, 3, false><<<(unsigned)nb, nt, c->smem_pk, s>>>(g, rg, C, ia, st, twr, npk, c->tmP)))
        }
      }));
    } else if (C.kind == 1 && c->row_npen && ia.mode != IN_RAW) {
      // packed coefficients, split: pointwise y = M(x) u (+ p') at streaming
      // bandwidth, then the staged row FFT on y.  y lives in the Ap buffer (free
      // until the last sweep).
      double* y = c->Ap;
      const int blocks = c->num_sms * 8;
      TRY(launch(c, "pointwise", [&] { k_pointwise_aniso<<<blocks, 256, 0, s>>>(g, C, ia, st, R, y); }));
      InArgs raw{};
      raw.mode = IN_RAW;
      raw.s = 1.0;
      raw.u = y;
      const int nt = c->row_npen * (rg.nl / 9);
      TRY(launch(c, "row_fwd", [&] {
        FC_POW3_SWITCH(rg.nl, (k_row_fwd_r<LL><<<(unsigned)nrow_blocks, nt, c->smem_row_r, s>>>(g, rg, C, raw, st, twr, Wrow, c->tmW)));
      }));
    } else if (c->row_npen) {
      const int nt = c->row_npen * (rg.nl / 9);
      TRY(launch(c, "row_fwd", [&] {
        FC_POW3_SWITCH(rg.nl, (k_row_fwd_r<LL><<<(unsigned)nrow_blocks, nt, c->smem_row_r, s>>>(g, rg, C, ia, st, twr, Wrow, c->tmW)));
      }));
    } else {
      const FftPlan pl_last = c->plan(rg.nl);
      TRY(launch(c, "row_fwd", [&] {
        k_row_fwd<<<(unsigned)nrow_blocks, kThreads, c->smem_row, s>>>(g, rg, C, ia, st, pl_last, Wrow);
      }));
    }
    if (d == 3) TRY(mid(false));
  }
  if (phases & PH_OUTER) {
    OuterGeo og = c->og;
    og.orth = orth;
    for (int a = 0; a < 3; ++a)
      for (int b = 0; b < 3; ++b) og.M[a][b] = M[a][b];
    double2* Wout = c->P > 1 ? c->W2r : c->W2;
    og.R = R;
    if (c->outer_qb && c->outer_seq && c->P == 1 && og.tma) {
      const int nt = c->outer_qb * (c->n0g / 9);
      const double2* tw = c->rtw(c->n0g);
      TRY(launch(c, "outer", [&] {
        // folded input: rows 0 and 1 only (three CTAs fit an SM)
        const size_t sm2 = FC_OUTER_TFI_OCC3 ? c->smem_outer_r / 3 * 2 : c->smem_outer_r;
        if (d == 2) FC_POW3_SWITCH(c->n0g, (k_outer_seq<LL, 2><<<(unsigned)(R * og.nqb), nt, c->smem_outer_r, s>>>(g, og, st, tw, Wout)))
        else if (c->fold_fwd) FC_POW3_SWITCH(c->n0g, (k_outer_seq<LL, 3, true, true><<<(unsigned)(R * og.nqb), nt, sm2, s>>>(g, og, st, tw, Wout)))
        else if (c->two_field) FC_POW3_SWITCH(c->n0g, (k_outer_seq<LL, 3, true><<<(unsigned)(R * og.nqb), nt, c->smem_outer_r, s>>>(g, og, st, tw, Wout)))
        else FC_POW3_SWITCH(c->n0g, (k_outer_seq<LL, 3><<<(unsigned)(R * og.nqb), nt, c->smem_outer_r, s>>>(g, og, st, tw, Wout)))
      }));
    } else if (c->outer_qb) {
      const int nt = c->outer_qb * (c->n0g / 9);
      const double2* tw = c->rtw(c->n0g);
      TRY(launch(c, "outer", [&] {
        if (d == 2) FC_POW3_SWITCH(c->n0g, (k_outer_r<LL, 2><<<(unsigned)(R * og.nqb), nt, c->smem_outer_r, s>>>(g, og, smap, st, tw, Wout)))
        else FC_POW3_SWITCH(c->n0g, (k_outer_r<LL, 3><<<(unsigned)(R * og.nqb), nt, c->smem_outer_r, s>>>(g, og, smap, st, tw, Wout)))
      }));
    } else {
      const FftPlan pl0 = c->plan(c->n0g);  // outer axis: global length (a slab holds n[0] < n0g planes)
      TRY(launch(c, "outer", [&] {
        k_outer<<<(unsigned)(R * og.nqb), kThreads, c->smem_outer, s>>>(g, og, smap, st, pl0, Wout);
      }));
    }
  }
  if (!(phases & PH_INV)) return FC_OK;
  if (d == 3) TRY(mid(true));
  // large grids: the last sweep only stores its partials, a separate launch finalizes
  const FinArgs fin_full = ea.fin;
  ea.fin = fin_for_kernel(c, fin_full);
  auto last_sweep = [&]() -> int {
  const RowGeo rgi = c->rgi;
  const int64_t ninv_blocks = (int64_t)R * rgi.no * rgi.ntiles * d;
  if (c->row_npen_inv && rgi.tma && c->inv_pipe_blocks > 0) {
    const int nt = c->row_npen_inv * (rgi.nl / 9);
    const double2* tw = c->rtw(rgi.nl);
    const int64_t ntile = ninv_blocks;
    const unsigned grid = (unsigned)std::min<int64_t>(ntile, (int64_t)c->num_sms * c->inv_pipe_blocks);
    const int stage_c = c->inv_pipe_stage;
    const int nst = c->inv_pipe_nst;
    const size_t smem = (size_t)nst * 16 * stage_c + (size_t)8 * (2 * c->row_npen_inv * rgi.nl + 2);
    return launch(c, "row_inv", [&] {
      FC_POW3_SWITCH(rgi.nl, (k_row_inv_pp<LL><<<grid, nt, smem, s>>>(g, rgi, ea, st, tw, ntile, stage_c, nst, 1, c->tmWi)));
    });
  }
  if (c->row_npen_inv) {
    const int nt = c->row_npen_inv * (rgi.nl / 9);
    const double2* tw = c->rtw(rgi.nl);
    return launch(c, "row_inv", [&] {
      if (nt <= 256) FC_POW3_SWITCH(rgi.nl, (k_row_inv_r<LL, 256><<<(unsigned)ninv_blocks, nt, c->smem_row_inv_r, s>>>(g, rgi, ea, st, tw, Wrow, c->tmWi)))
      else if (nt <= 384) FC_POW3_SWITCH(rgi.nl, (k_row_inv_r<LL, 384><<<(unsigned)ninv_blocks, nt, c->smem_row_inv_r, s>>>(g, rgi, ea, st, tw, Wrow, c->tmWi)))
      else FC_POW3_SWITCH(rgi.nl, (k_row_inv_r<LL, 512><<<(unsigned)ninv_blocks, nt, c->smem_row_inv_r, s>>>(g, rgi, ea, st, tw, Wrow, c->tmWi)))
    });
  }
  const FftPlan pl_last = c->plan(rg.nl);
  return launch(c, "row_inv", [&] {
    k_row_inv<<<(unsigned)nrow_blocks, kThreads, c->smem_row, s>>>(g, rg, ea, st, pl_last, Wrow);
  });
  };
  TRY(last_sweep());
  return launch_fin_split(c, fin_full);
}

int run_operator(fc_ctx* c, int R, const InArgs& ia, EpArgs ea, int orth, const double M[3][3], const RhsState* st) {
  return run_phases(c, PH_ALL, R, ia, ea, orth, M, st);
}

int check_ctx(fc_ctx* c, bool need_coef) {
  if (c == nullptr) return set_err(FC_EINVAL, "null context");
  if (!c->sub.empty()) {  // sharded parent: slabs carry the device state
    if (need_coef && c->coef_kind < 0) return set_err(FC_EINVAL, "coefficients not set");
    return FC_OK;
  }
  if (need_coef && c->A == nullptr && c->lab == nullptr) return set_err(FC_EINVAL, "coefficients not set");
  CK(cudaSetDevice(c->device));
  return FC_OK;
}

int check_R(int R) {
  if (R < 1 || R > FC_MAX_RHS) return set_err(FC_EINVAL, "number of right-hand sides must lie in [1, %d], got %d", FC_MAX_RHS, R);
  return FC_OK;
}

const double kIdentity[3][3] = {{1, 0, 0}, {0, 1, 0}, {0, 0, 1}};

int upload_fields(fc_ctx* c, double* dst, const double* host, int R) {
  CK(cudaMemcpyAsync(dst, host, sizeof(double) * (size_t)R * c->dim * c->N, cudaMemcpyHostToDevice, c->stream));
  return FC_OK;
}
int download_fields(fc_ctx* c, double* host, const double* src, int R) {
  CK(cudaMemcpyAsync(host, src, sizeof(double) * (size_t)R * c->dim * c->N, cudaMemcpyDeviceToHost, c->stream));
  return FC_OK;
}

int sync(fc_ctx* c) {
  CK(cudaStreamSynchronize(c->stream));
  if (c->prof_on) drain_profile(c);
  return FC_OK;
}

FinArgs fin_args(fc_ctx* c, int mode, int R, int nslot, double tol, int max_iter, int with_init = 0) {
  FinArgs f{};
  f.mode = mode;
  f.R = R;
  f.nslot = nslot;
  f.part = c->part;
  f.st = c->st;
  f.hist = c->hist;
  f.hcap = c->hcap;
  f.tol = tol;
  f.max_iter = max_iter;
  f.window = 10;  // solver.py:27
  f.with_init = with_init;
  f.total = (double)c->Ng;  // global voxel count (slab-local N differs)
  f.any_active = c->d_mapped;  // zero-copy: the host reads it after the iteration's event
  f.counter = c->counter;
  return f;
}

}  // namespace

#include "fc_nccl.inc"
#include "fc_shard.inc"
#include "fc_io.inc"

// ===========================================================================
// C ABI
extern "C" {

int32_t fc_version(void) { return 1; }
const char* fc_last_error(void) { return g_err.c_str(); }

int32_t fc_device_count(int32_t* count) {
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess) {
    *count = 0;
    return set_err(FC_ECUDA, "cudaGetDeviceCount: %s", cudaGetErrorString(e));
  }
  *count = n;
  return FC_OK;
}

int32_t fc_set_plan_option(const char* key, int32_t value) {
  if (key == nullptr) return set_err(FC_EINVAL, "null option name");
  PlanOpts& o = g_plan_opts;
  const struct { const char* name; int* field; } table[] = {
      {"force_generic", &o.force_generic}, {"row_threads", &o.row_threads}, {"row_threads_inv", &o.row_threads_inv}, {"mid_threads", &o.mid_threads},
      {"outer_threads", &o.outer_threads}, {"row_tma", &o.row_tma}, {"mid_tma", &o.mid_tma},
      {"outer_tma", &o.outer_tma}, {"outer_seq", &o.outer_seq}, {"inv_pipe", &o.inv_pipe}, {"inv_qpre", &o.inv_qpre}, {"fin_split", &o.fin_split},
      {"aniso_fused", &o.aniso_fused}, {"two_field", &o.two_field}, {"fold_fwd", &o.fold_fwd}, {"defer_x", &o.defer_x}, {"fused_exchange", &o.fused_exchange},
      {"sync_debug", &o.sync_debug}, {"mid_threads_inv", &o.mid_threads_inv}, {"mid_map", &o.mid_map},
      {"mid_tma_fwd", &o.mid_tma_fwd}};
  for (const auto& t : table)
    if (std::strcmp(t.name, key) == 0) {
      *t.field = value;
      return FC_OK;
    }
  return set_err(FC_EINVAL, "unknown plan option '%s'", key);
}

#ifdef FC_TRACE
int32_t fc_debug_trace(unsigned long long* out, int32_t n) {
  CK(cudaDeviceSynchronize());
  CK(cudaMemcpyFromSymbol(out, fc::g_trace, sizeof(unsigned long long) * n));
  return FC_OK;
}
#endif

int32_t fc_reset_plan_options(void) {
  g_plan_opts = PlanOpts{};
  return FC_OK;
}

}  // extern "C"

namespace {

// One slab (or the whole grid when P = 1) on one device.  shape is GLOBAL; the
// slab owns axis-0 planes [me n0 / P, (me + 1) n0 / P) and outer pencils
// [me Q / P, (me + 1) Q / P).
int create_slab(fc_ctx** out, int32_t dim, const int64_t* shape, const double* half_periods, int32_t device, int P,
                int me) {
  *out = nullptr;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) return set_err(FC_ECUDA, "no CUDA device available");
  if (device < 0 || device >= ndev) return set_err(FC_EINVAL, "device %d out of range (have %d)", device, ndev);
  fc_ctx* c = new fc_ctx();
  c->device = device;
  c->dim = dim;
  c->P = P;
  c->me = me;
  c->n0g = (int)shape[0];
  c->Ng = 1;
  for (int a = 0; a < dim; ++a) {
    c->n[a] = (int)shape[a];
    c->Y[a] = half_periods[a];
    c->Ng *= shape[a];
  }
  const int Q = dim == 3 ? (int)(shape[1] * ((shape[2] + 1) / 2)) : (dim == 2 ? (int)((shape[1] + 1) / 2) : 1);
  for (int t = 0; t <= P; ++t) {
    c->s0[t] = (int)((int64_t)t * shape[0] / P);
    c->qs[t] = (int)((int64_t)t * Q / P);
  }
  c->n[0] = c->s0[me + 1] - c->s0[me];
  c->N = c->Ng / shape[0] * c->n[0];
  auto fail = [&](int rc) { fc_destroy(c); return rc; };
  if (cudaSetDevice(device) != cudaSuccess) return fail(set_err(FC_ECUDA, "cudaSetDevice(%d) failed", device));
  cudaDeviceProp prop;
  cudaGetDeviceProperties(&prop, device);
  if (prop.major < 10) return fail(set_err(FC_ECUDA, "device %d is sm_%d%d; this build targets sm_100a", device, prop.major, prop.minor));
  c->smem_optin = (int)prop.sharedMemPerBlockOptin;
  c->opt = g_plan_opts;
  c->force_generic = c->opt.force_generic != 0;
  c->num_sms = prop.multiProcessorCount;
  if (cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking) != cudaSuccess)
    return fail(set_err(FC_ECUDA, "stream creation failed"));
  for (auto& e : c->sev) cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
  int rc = ensure_plan(c, c->n0g);
  for (int a = 1; a < dim && rc == FC_OK; ++a) rc = ensure_plan(c, c->n[a]);
  if (rc) return fail(rc);
  // per-axis frequency tables xi = k / Y (grid.py:131-146); axis 0 is global
  std::vector<double> xi;
  for (int a = 0; a < dim; ++a) {
    c->xi_off[a] = (int)xi.size();
    const int na = a == 0 ? c->n0g : c->n[a];
    for (int i = 0; i < na; ++i) {
      long long k = i <= (na - 1) / 2 ? i : (long long)i - na;
      xi.push_back((double)k / c->Y[a]);
    }
  }
  if (cudaMalloc(&c->xi, sizeof(double) * xi.size()) != cudaSuccess) return fail(set_err(FC_ENOMEM, "xi alloc"));
  cudaMemcpy(c->xi, xi.data(), sizeof(double) * xi.size(), cudaMemcpyHostToDevice);
  rc = choose_tiles(c);
  if (rc) return fail(rc);
  if (P > 1 && dim != 3) return fail(set_err(FC_ENOTSUP, "slab decomposition needs d = 3"));
  const int mx = c->smem_optin;
  if ((rc = allow_smem(k_row_fwd, mx)) || (rc = allow_smem(k_row_inv, mx)) || (rc = allow_smem(k_mid<false>, mx)) ||
      (rc = allow_smem(k_mid<true>, mx)) || (rc = allow_smem(k_outer, mx)) || (rc = allow_smem(k_line, mx)) ||
      (rc = allow_reg_smem(mx)))
    return fail(rc);
  // measured: faster for one pencil per block (L = 2187, cfg2), slower for the
  // short rows of cfg3 / cfg4 (L = 243 / 729: many pencils per block)
  if (c->row_npen_inv && (c->opt.inv_pipe >= 0 ? c->opt.inv_pipe != 0 : c->row_npen_inv == 1) &&
      c->row_npen_inv * (c->rgi.nl / 9) <= 256) {
    const RowGeo& rg = c->rgi;
    const int B = 2 * c->row_npen_inv;
    c->inv_pipe_stage = (std::max(rg.nbox * rg.boxK * B, c->row_npen_inv * (rg.nl + 1)) + 7) & ~7;
    const size_t qbytes = (size_t)8 * (2 * c->row_npen_inv * rg.nl + 2);
    const size_t smem = (size_t)c->inv_pipe_nst * 16 * c->inv_pipe_stage + qbytes;
    int nb = 0;
    FC_POW3_SWITCH(rg.nl, (allow_smem(k_row_inv_pp<LL>, mx),
                           cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_row_inv_pp<LL>, c->row_npen_inv * (rg.nl / 9), smem)));
    c->inv_pipe_blocks = nb;
  }
  if (cudaMalloc(&c->any_active, sizeof(int)) != cudaSuccess) return fail(set_err(FC_ENOMEM, "flag alloc"));
  if (cudaMalloc(&c->counter, sizeof(unsigned)) != cudaSuccess) return fail(set_err(FC_ENOMEM, "counter alloc"));
  cudaMemset(c->counter, 0, sizeof(unsigned));
  if (cudaMalloc(&c->lsum, sizeof(double) * 2 * FC_MAX_RHS) != cudaSuccess) return fail(set_err(FC_ENOMEM, "lsum alloc"));
  if (cudaMallocHost(&c->h_flag, 4 * sizeof(int)) != cudaSuccess) return fail(set_err(FC_ENOMEM, "pinned alloc"));
  if (cudaHostAlloc(&c->h_mapped, sizeof(int), cudaHostAllocMapped) != cudaSuccess ||
      cudaHostGetDevicePointer(&c->d_mapped, c->h_mapped, 0) != cudaSuccess)
    return fail(set_err(FC_ENOMEM, "mapped flag alloc"));
  *c->h_mapped = 1;
  for (auto& e : c->flag_ev) cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
  if (cudaMalloc(&c->d_mat, sizeof(double) * FC_MAX_RHS * FC_MAX_RHS) != cudaSuccess)
    return fail(set_err(FC_ENOMEM, "matrix alloc"));
  *out = c;
  return FC_OK;
}

int check_shape(int32_t dim, const int64_t* shape, const double* half_periods) {
  if (dim < 1 || dim > 3) return set_err(FC_ENOTSUP, "dimension %d not supported (1..3)", dim);
  for (int a = 0; a < dim; ++a) {
    if (shape[a] <= 0 || shape[a] % 2 == 0)
      return set_err(FC_EINVAL, "grid shape must consist of positive odd integers");
    if (!(half_periods[a] > 0)) return set_err(FC_EINVAL, "half_periods must be positive");
    if (shape[a] > (1 << 20)) return set_err(FC_ENOTSUP, "axis length %lld too large", (long long)shape[a]);
  }
  return FC_OK;
}

}  // namespace

extern "C" {

int32_t fc_create(fc_ctx** out, int32_t dim, const int64_t* shape, const double* half_periods, int32_t device) {
  if (out == nullptr) return set_err(FC_EINVAL, "null output pointer");
  *out = nullptr;
  TRY(check_shape(dim, shape, half_periods));
  return create_slab(out, dim, shape, half_periods, device, 1, 0);
}

int32_t fc_create_sharded(fc_ctx** out, int32_t dim, const int64_t* shape, const double* half_periods,
                          int32_t nslabs, const int32_t* devices) {
  if (out == nullptr) return set_err(FC_EINVAL, "null output pointer");
  *out = nullptr;
  TRY(check_shape(dim, shape, half_periods));
  if (nslabs < 1 || nslabs > kMaxSlabs) return set_err(FC_EINVAL, "number of slabs must lie in [1, %d]", kMaxSlabs);
  if (dim != 3) return set_err(FC_ENOTSUP, "slab decomposition is implemented for d = 3");
  if (shape[0] < nslabs) return set_err(FC_EINVAL, "more slabs than axis-0 planes");
  fc_ctx* c = new fc_ctx();
  c->device = -1;  // parent: no device resources of its own
  c->dim = dim;
  c->P = nslabs;
  c->n0g = (int)shape[0];
  c->Ng = 1;
  for (int a = 0; a < dim; ++a) {
    c->n[a] = (int)shape[a];
    c->Y[a] = half_periods[a];
    c->Ng *= shape[a];
  }
  c->N = c->Ng;
  for (int t = 0; t < nslabs; ++t) {
    fc_ctx* sl = nullptr;
    const int dev = devices ? devices[t] : 0;
    int rc = create_slab(&sl, dim, shape, half_periods, dev, nslabs, t);
    if (rc) {
      fc_destroy(c);
      return rc;
    }
    c->sub.push_back(sl);
  }
  // peer access between distinct devices (P2P loads of the slab sums, NVLink copies)
  for (fc_ctx* a : c->sub)
    for (fc_ctx* b : c->sub)
      if (a->device != b->device) {
        int ok = 0;
        cudaDeviceCanAccessPeer(&ok, a->device, b->device);
        if (!ok) {
          fc_destroy(c);
          return set_err(FC_ECUDA, "devices %d and %d cannot access each other", a->device, b->device);
        }
        cudaSetDevice(a->device);
        cudaError_t e = cudaDeviceEnablePeerAccess(b->device, 0);
        if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) {
          fc_destroy(c);
          return set_err(FC_ECUDA, "peer access %d -> %d: %s", a->device, b->device, cudaGetErrorString(e));
        }
        cudaGetLastError();
      }
  // fused exchange: the sweeps store into the other slabs' buffers directly
  // (plan option fused_exchange = 0 keeps the copy-engine exchange)
  const bool fuse = nslabs > 1 && c->sub[0]->opt.fused_exchange;
  for (fc_ctx* sl : c->sub) {
    sl->sibs = &c->sub;
    sl->fused = fuse;
  }
  *out = c;
  return FC_OK;
}

int32_t fc_nccl_unique_id(void* out) {
  if (out == nullptr) return set_err(FC_EINVAL, "null output pointer");
  if (!nccl().ok) return set_err(FC_ENOTSUP, "NCCL unavailable: %s", nccl().why.c_str());
  ncclUniqueId id;
  NK(nccl().getUniqueId(&id));
  std::memcpy(out, &id, sizeof(id));
  return FC_OK;
}

int32_t fc_create_dist(fc_ctx** out, int32_t dim, const int64_t* shape, const double* half_periods, int32_t nranks,
                       int32_t rank, int32_t device, const void* unique_id) {
  if (out == nullptr || unique_id == nullptr) return set_err(FC_EINVAL, "null pointer argument");
  *out = nullptr;
  TRY(check_shape(dim, shape, half_periods));
  if (nranks < 1 || nranks > kMaxSlabs || rank < 0 || rank >= nranks)
    return set_err(FC_EINVAL, "rank %d / world %d outside [0, %d)", rank, nranks, kMaxSlabs);
  if (dim != 3) return set_err(FC_ENOTSUP, "slab decomposition is implemented for d = 3");
  if (shape[0] < nranks) return set_err(FC_EINVAL, "more ranks than axis-0 planes");
  if (!nccl().ok) return set_err(FC_ENOTSUP, "NCCL unavailable: %s", nccl().why.c_str());
  fc_ctx* c = new fc_ctx();
  c->device = -1;
  c->dim = dim;
  c->P = nranks;
  c->me = rank;
  c->dist = true;
  c->n0g = (int)shape[0];
  c->Ng = 1;
  for (int a = 0; a < dim; ++a) {
    c->n[a] = (int)shape[a];
    c->Y[a] = half_periods[a];
    c->Ng *= shape[a];
  }
  c->N = c->Ng;
  fc_ctx* sl = nullptr;
  int rc = create_slab(&sl, dim, shape, half_periods, device, nranks, rank);
  if (rc) {
    delete c;
    return rc;
  }
  c->sub.push_back(sl);
  cudaSetDevice(device);
  ncclUniqueId id;
  std::memcpy(&id, unique_id, sizeof(id));
  ncclComm_t comm;
  ncclResult_t nr = nccl().commInitRank(&comm, nranks, id, rank);
  if (nr != ncclSuccess) {
    fc_destroy(c);
    return set_err(FC_ECUDA, "ncclCommInitRank: %s", nccl().errStr(nr));
  }
  c->comm = comm;
  if (cudaMalloc(&c->gathered, sizeof(double) * FC_MAX_RHS * nranks) != cudaSuccess ||
      cudaMalloc(&c->barrier, sizeof(double) * (1 + nranks)) != cudaSuccess) {
    fc_destroy(c);
    return set_err(FC_ENOMEM, "gather buffer");
  }
  cudaMemset(c->barrier, 0, sizeof(double) * (1 + nranks));
  // fused exchange over CUDA IPC mappings of the peers' spectrum buffers (set up
  // with the workspace, dist_ipc_setup); plan option fused_exchange = 0 keeps
  // the NCCL send / receive exchange
  sl->fused = nranks > 1 && sl->opt.fused_exchange;
  *out = c;
  return FC_OK;
}

void fc_destroy(fc_ctx* c) {
  if (c == nullptr) return;
  for (fc_ctx* sl : c->sub) fc_destroy(sl);
  c->sub.clear();
  if (c->device < 0) {  // sharded parent holds no device resources
    if (c->dist && !c->sub.empty()) {
      cudaSetDevice(c->sub[0]->device);
      dist_ipc_close(c);
    }
    if (c->comm) nccl().commDestroy((ncclComm_t)c->comm);
    cudaFree(c->gathered);
    cudaFree(c->barrier);
    delete c;
    return;
  }
  cudaSetDevice(c->device);
  if (c->stream) cudaStreamSynchronize(c->stream);
  for (auto& kv : c->plans) {
    cudaFree(kv.second.roots);
    cudaFree(kv.second.rtw);
  }
  for (double* q : {c->xi, c->A, c->x, c->r, c->p[0], c->p[1], c->Ap, c->part, c->hist, c->d_mat}) cudaFree(q);
  free_indexed(c);
  cudaFree(c->W1);
  cudaFree(c->W2);
  cudaFree(c->st);
  cudaFree(c->any_active);
  cudaFree(c->counter);
  cudaFree(c->part2);
  cudaFree(c->lsum);
  cudaFree(c->W2r);
  cudaFree(c->sphere_bits);
  cudaFree(c->sphere_count);
  for (auto& e : c->sev)
    if (e) cudaEventDestroy(e);
  if (c->h_flag) cudaFreeHost(c->h_flag);
  if (c->h_mapped) cudaFreeHost(c->h_mapped);
  for (auto& e : c->flag_ev)
    if (e) cudaEventDestroy(e);
  for (auto& pe : c->pending) {
    cudaEventDestroy(pe.second.first);
    cudaEventDestroy(pe.second.second);
  }
  for (auto e : c->ev_pool) cudaEventDestroy(e);
  for (auto& e : c->timer_ev)
    if (e) cudaEventDestroy(e);
  if (c->stream) cudaStreamDestroy(c->stream);
  delete c;
}

int32_t fc_set_coefficients(fc_ctx* c, int32_t kind, const double* host, int64_t count) {
  if (c && !c->sub.empty()) return shard_set_coefficients(c, kind, host, count);
  TRY(check_ctx(c, false));
  const int d = c->dim;
  const int64_t nsym = (int64_t)d * (d + 1) / 2;
  int64_t expect = kind == FC_COEF_ISOTROPIC ? c->N : (kind == FC_COEF_PACKED ? nsym * c->N : -1);
  if (expect < 0) return set_err(FC_EINVAL, "unknown coefficient kind %d", kind);
  if (count != expect) return set_err(FC_EINVAL, "coefficient count %lld != expected %lld", (long long)count, (long long)expect);
  free_indexed(c);
  if (c->A == nullptr || c->A_count != count) {
    cudaFree(c->A);
    c->A = nullptr;
    CK(cudaMalloc(&c->A, sizeof(double) * count + kFieldPad));
    c->A_count = count;
  }
  CK(cudaMemcpyAsync(c->A, host, sizeof(double) * count, cudaMemcpyHostToDevice, c->stream));
  c->coef_kind = kind;
  return sync(c);
}

int32_t fc_set_coefficients_indexed(fc_ctx* c, int32_t n_phases, const double* table, const uint16_t* labels,
                                    int64_t count) {
  if (c == nullptr) return set_err(FC_EINVAL, "null context");
  if (table == nullptr || labels == nullptr) return set_err(FC_EINVAL, "null argument");
  if (n_phases < 1 || n_phases > FC_MAX_PHASES)
    return set_err(FC_EINVAL, "n_phases must lie in [1, %d], got %d", FC_MAX_PHASES, n_phases);
  if (c->dim < 2) return set_err(FC_EINVAL, "indexed coefficients need dim >= 2");
  if (count != c->Ng) return set_err(FC_EINVAL, "label count %lld != grid size %lld", (long long)count, (long long)c->Ng);
  if (!c->sub.empty()) {
    const int64_t plane = c->Ng / c->n0g;
    for (fc_ctx* sl : c->sub) TRY(set_indexed_slab(sl, n_phases, table, labels + (int64_t)sl->s0[sl->me] * plane));
    c->coef_kind = FC_COEF_PACKED;
    return FC_OK;
  }
  TRY(check_ctx(c, false));
  return set_indexed_slab(c, n_phases, table, labels);
}

int32_t fc_compress_coefficients(fc_ctx* c, int32_t max_phases, int32_t keep_packed, int32_t* n_phases) {
  if (c == nullptr) return set_err(FC_EINVAL, "null context");
  if (max_phases < 1 || max_phases > FC_MAX_PHASES)
    return set_err(FC_EINVAL, "max_phases must lie in [1, %d], got %d", FC_MAX_PHASES, max_phases);
  if (c->coef_kind < 0) return set_err(FC_EINVAL, "coefficients not set");
  int most = 0;
  if (!c->sub.empty()) {
    for (fc_ctx* sl : c->sub) {
      int nph = 0;
      TRY(compress_slab(sl, max_phases, keep_packed, &nph));
      most = std::max(most, nph);
    }
  } else {
    TRY(check_ctx(c, true));
    TRY(compress_slab(c, max_phases, keep_packed, &most));
  }
  if (n_phases != nullptr) *n_phases = most;
  return FC_OK;
}

int32_t fc_apply_A(fc_ctx* c, const double* u, double* out, int32_t nf) {
  if (c && !c->sub.empty()) {
    TRY(check_R(nf));
    return shard_field_op(c, 0, nullptr, u, out, nf);
  }
  TRY(check_ctx(c, true));
  TRY(check_R(nf));
  TRY(ensure_workspace(c, nf, 2));
  TRY(upload_fields(c, c->p[0], u, nf));
  const Geo g = c->geo();
  const Coef C = c->coef();
  dim3 grid((unsigned)std::min<int64_t>((c->N + kThreads - 1) / kThreads, 148 * 16), nf);
  TRY(launch(c, "apply_A", [&] { k_apply_A<<<grid, kThreads, 0, c->stream>>>(g, C, c->p[0], c->Ap); }));
  TRY(download_fields(c, out, c->Ap, nf));
  return sync(c);
}

int32_t fc_project(fc_ctx* c, int32_t which, const double* ref, const double* u, double* out, int32_t nf) {
  const NvtxRange nvtx_range("fc_project");
  TRY(check_ctx(c, false));
  TRY(check_R(nf));
  if (which != FC_PROJ_ORTHOGONAL && which != FC_PROJ_GAMMA_REF) return set_err(FC_EINVAL, "unknown projector %d", which);
  if (which == FC_PROJ_GAMMA_REF && ref == nullptr) return set_err(FC_EINVAL, "gamma_ref needs a reference matrix");
  if (!c->sub.empty()) return shard_field_op(c, which == FC_PROJ_ORTHOGONAL ? 2 : 3, ref, u, out, nf);
  TRY(ensure_workspace(c, nf, 2));
  TRY(upload_fields(c, c->p[0], u, nf));
  InArgs ia{};
  ia.mode = IN_RAW;
  ia.s = 1.0;
  ia.u = c->p[0];
  EpArgs ea{};
  ea.mode = EP_STORE;
  ea.out = c->Ap;
  double M[3][3] = {};
  if (which == FC_PROJ_GAMMA_REF)
    for (int a = 0; a < c->dim; ++a)
      for (int b = 0; b < c->dim; ++b) M[a][b] = ref[a * c->dim + b];
  TRY(run_operator(c, nf, ia, ea, which == FC_PROJ_ORTHOGONAL, which == FC_PROJ_ORTHOGONAL ? kIdentity : M, nullptr));
  TRY(download_fields(c, out, c->Ap, nf));
  return sync(c);
}

int32_t fc_apply_system(fc_ctx* c, const double* u, double* out, int32_t nf) {
  const NvtxRange nvtx_range("fc_apply_system");
  if (c && !c->sub.empty()) {
    TRY(check_R(nf));
    return shard_field_op(c, 1, nullptr, u, out, nf);
  }
  TRY(check_ctx(c, true));
  TRY(check_R(nf));
  TRY(ensure_workspace(c, nf, 2));
  TRY(upload_fields(c, c->p[0], u, nf));
  InArgs ia{};
  ia.mode = IN_FIELD;
  ia.s = 1.0;
  ia.u = c->p[0];
  EpArgs ea{};
  ea.mode = EP_STORE;
  ea.out = c->Ap;
  TRY(run_operator(c, nf, ia, ea, 1, kIdentity, nullptr));
  TRY(download_fields(c, out, c->Ap, nf));
  return sync(c);
}

int32_t fc_solve_cg(fc_ctx* c, int32_t R, const double* E, double tol, int32_t max_iter, double lam,
                    const double* init, double* x_out, fc_report* rep, double* hist, double* iterates,
                    int64_t iterates_cap, int64_t* n_iterates) {
  const NvtxRange nvtx_range("fc_solve_cg");
  TRY(check_ctx(c, true));
  TRY(check_R(R));
  if (!(tol > 0 && tol < 1)) return set_err(FC_EINVAL, "tol must lie in (0, 1), got %g", tol);
  if (max_iter < 1) return set_err(FC_EINVAL, "max_iter must be positive");
  if (!c->sub.empty()) {
    if (iterates != nullptr) return set_err(FC_ENOTSUP, "record_iterates is not supported on a sharded context");
    if (n_iterates) *n_iterates = 0;
    return shard_solve_cg(c, R, E, tol, max_iter, lam, init, x_out, rep, hist);
  }
  const int d = c->dim;
  TRY(ensure_workspace(c, R, max_iter + 1));
  cudaStream_t s = c->stream;
  const int64_t fieldR = (int64_t)d * c->N * R;
  const double sc = lam > 0 ? lam : 1.0;
  const int orth = lam > 0 ? 0 : 1;
  double M[3][3] = {};
  for (int a = 0; a < d; ++a) M[a][a] = sc;
  CK(cudaMemsetAsync(c->st, 0, sizeof(RhsState) * R, s));
  CK(cudaMemsetAsync(c->x, 0, sizeof(double) * fieldR, s));
  const int nrow = (int)nslot_row(c);
  const int nvec = (int)nslot_vec(c);
  {  // right-hand side and warm start (profiled as "<kernel>_rhs")
  ProfTag rhs_tag(c, "_rhs");
  if (init != nullptr) {
    // x = G init (solver.py:185)
    TRY(upload_fields(c, c->p[0], init, R));
    InArgs ia{};
    ia.mode = IN_RAW;
    ia.s = 1.0;
    ia.u = c->p[0];
    EpArgs ea{};
    ea.mode = EP_STORE;
    ea.out = c->x;
    TRY(run_operator(c, R, ia, ea, 1, kIdentity, nullptr));
  }
  // rhs = -op(E_N) (solver.py:176-178); the last CTA sets r0 (and history[0])
  {
    InArgs ia{};
    ia.mode = IN_CONST;
    ia.s = sc;
    for (int r = 0; r < R; ++r)
      for (int a = 0; a < d; ++a) ia.E[r][a] = E[r * d + a];
    EpArgs ea{};
    ea.mode = EP_RHS;
    ea.out = init != nullptr ? c->p[1] : c->r;  // Ap is the split first sweep's scratch
    ea.part = c->part;
    ea.fin = fin_args(c, FIN_INIT, R, nrow, tol, max_iter, init != nullptr);
    TRY(run_operator(c, R, ia, ea, orth, M, nullptr));
  }
  if (init != nullptr) {
    // r = rhs - op(x) (solver.py:186)
    InArgs ia{};
    ia.mode = IN_FIELD;
    ia.s = sc;
    ia.u = c->x;
    EpArgs ea{};
    ea.mode = EP_STORE;
    ea.out = c->p[0];
    TRY(run_operator(c, R, ia, ea, orth, M, nullptr));
    dim3 grid(nvec, R);
    FinArgs f = fin_args(c, FIN_INIT2, R, nvec, tol, max_iter);
    TRY(launch(c, "sub_dot", [&] {
      k_sub_dot<<<grid, kThreads, 0, s>>>((int64_t)d * c->N, c->p[1], c->p[0], c->r, c->part, nvec, f);
    }));
  }
  }
  std::vector<RhsState> hs(R);
  CK(cudaMemcpyAsync(hs.data(), c->st, sizeof(RhsState) * R, cudaMemcpyDeviceToHost, s));
  TRY(sync(c));
  bool any = false;
  for (auto& q : hs) any |= q.active != 0;
  int64_t nit = 0;
  if (iterates != nullptr && iterates_cap > 0) {
    TRY(download_fields(c, iterates, c->x, R));
    nit = 1;
  }
  const bool record = iterates != nullptr;
  // x += alpha p is deferred into the next iteration's first sweep, which reads
  // p_old anyway (saves the x read of p in k_cg_update: 1 of its 6 words per
  // element); the last update of each RHS is flushed after the loop.  Bitwise
  // identical to the immediate update.  record_iterates needs x every iteration.
  const bool defer = c->opt.defer_x && !record;
  for (int it = 0; any && it < max_iter; ++it) {
    double* pcur = c->p[it & 1];
    double* pold = c->p[(it + 1) & 1];
    InArgs ia{};
    ia.mode = IN_PNEW;
    ia.s = sc;
    ia.u = c->r;
    ia.p_old = pold;
    ia.p_new = pcur;
    ia.xacc = defer ? c->x : nullptr;
    EpArgs ea{};
    ea.mode = EP_AP;
    ea.out = c->Ap;
    ea.p = pcur;
    ea.part = c->part;
    ea.fin = fin_args(c, FIN_ALPHA, R, nrow, tol, max_iter);
    TRY(run_operator(c, R, ia, ea, orth, M, c->st));
    dim3 grid(nvec, R);
    FinArgs fb = fin_args(c, FIN_BETA, R, nvec, tol, max_iter);
    const FinArgs fbk = fin_for_kernel(c, fb);
    TRY(launch(c, "cg_update", [&] {
      k_cg_update<<<grid, kThreads, 0, s>>>((int64_t)d * c->N, c->st, defer ? nullptr : c->x, c->r, pcur, c->Ap,
                                            c->part, nvec, fbk);
    }));
    TRY(launch_fin_split(c, fb));
    // the flag is monotone (an inactive RHS never reactivates), so reading a
    // later iteration's value is always a valid stop decision
    const int slot = it & 3;
    CK(cudaEventRecord(c->flag_ev[slot], s));
    if (record) {
      TRY(sync(c));
      if (nit < iterates_cap) {
        TRY(download_fields(c, iterates + nit * (int64_t)R * d * c->N, c->x, R));
        TRY(sync(c));
        ++nit;
      }
      any = *(volatile int*)c->h_mapped != 0;
    } else if (it >= 1) {
      const int prev = (it - 1) & 3;
      CK(cudaEventSynchronize(c->flag_ev[prev]));
      if (*(volatile int*)c->h_mapped == 0) any = false;
    }
  }
  TRY(sync(c));
  CK(cudaMemcpy(hs.data(), c->st, sizeof(RhsState) * R, cudaMemcpyDeviceToHost));
  if (defer) {
    unsigned owe, use1;
    x_flush_masks(hs.data(), R, owe, use1);
    if (owe != 0u) {
      const dim3 grid((unsigned)std::min<int64_t>(4 * 148, ((int64_t)d * c->N + kThreads - 1) / kThreads), R);
      TRY(launch(c, "x_flush", [&] {
        k_x_flush<<<grid, kThreads, 0, s>>>((int64_t)d * c->N, c->st, c->x, c->p[0], c->p[1], owe, use1);
      }));
    }
  }
  const int hc = c->hcap;
  for (int r = 0; r < R; ++r) {
    rep[r].iterations = hs[r].iterations;
    rep[r].converged = hs[r].converged;
    rep[r].status = hs[r].status;
    rep[r].hist_len = hs[r].hist_len;
    rep[r].detail = hs[r].detail;
    if (hist != nullptr)
      CK(cudaMemcpy(hist + (int64_t)r * (max_iter + 1), c->hist + (int64_t)r * hc, sizeof(double) * hs[r].hist_len,
                    cudaMemcpyDeviceToHost));
  }
  if (n_iterates) *n_iterates = nit;
  if (x_out != nullptr) {
    TRY(download_fields(c, x_out, c->x, R));
    TRY(sync(c));
  }
  return FC_OK;
}

int32_t fc_solve_fixed_point(fc_ctx* c, int32_t R, const double* E, double tol, int32_t max_iter,
                             const double* ref, const double* scale, double* x_out, fc_report* rep, double* hist) {
  const NvtxRange nvtx_range("fc_solve_fixed_point");
  TRY(check_ctx(c, true));
  TRY(check_R(R));
  if (!(tol > 0 && tol < 1)) return set_err(FC_EINVAL, "tol must lie in (0, 1), got %g", tol);
  if (max_iter < 1) return set_err(FC_EINVAL, "max_iter must be positive");
  if (ref == nullptr || scale == nullptr) return set_err(FC_EINVAL, "reference matrix and scales are required");
  if (!c->sub.empty()) return shard_solve_fp(c, R, E, tol, max_iter, ref, scale, x_out, rep, hist);
  const int d = c->dim;
  TRY(ensure_workspace(c, R, max_iter + 1));
  cudaStream_t s = c->stream;
  std::vector<RhsState> hs(R);
  for (int r = 0; r < R; ++r) {
    std::memset(&hs[r], 0, sizeof(RhsState));
    hs[r].active = 1;
    hs[r].scale = scale[r];
  }
  CK(cudaMemcpyAsync(c->st, hs.data(), sizeof(RhsState) * R, cudaMemcpyHostToDevice, s));
  Loads L{};
  for (int r = 0; r < R; ++r)
    for (int a = 0; a < d; ++a) L.E[r][a] = E[r * d + a];
  const int64_t len = (int64_t)d * c->N;
  dim3 fgrid((unsigned)std::min<int64_t>((len + kThreads - 1) / kThreads, 148 * 16), R);
  TRY(launch(c, "fill_loads", [&] { k_fill_loads<<<fgrid, kThreads, 0, s>>>(c->N, d, L, nullptr, c->x); }));
  double M[3][3] = {};
  InArgs ia{};
  ia.mode = IN_FP;
  ia.s = 1.0;
  ia.u = c->x;
  for (int a = 0; a < d; ++a)
    for (int b = 0; b < d; ++b) {
      M[a][b] = ref[a * d + b];
      ia.A0[a][b] = ref[a * d + b];
    }
  EpArgs ea{};
  ea.mode = EP_FP;
  ea.out = c->x;
  ea.part = c->part;
  for (int r = 0; r < R; ++r)
    for (int a = 0; a < d; ++a) ea.E[r][a] = E[r * d + a];
  const int nrow = (int)nslot_row(c);
  ea.fin = fin_args(c, FIN_FP, R, nrow, tol, max_iter);
  bool any = true;
  for (int it = 0; any && it < max_iter; ++it) {
    TRY(run_operator(c, R, ia, ea, 0, M, c->st));
    const int slot = it & 3;
    CK(cudaEventRecord(c->flag_ev[slot], s));
    if (it >= 1) {
      const int prev = (it - 1) & 3;
      CK(cudaEventSynchronize(c->flag_ev[prev]));
      if (*(volatile int*)c->h_mapped == 0) any = false;
    }
  }
  // solution = e - E_N in place (solver.py:293-294)
  TRY(launch(c, "fill_loads", [&] { k_fill_loads<<<fgrid, kThreads, 0, s>>>(c->N, d, L, c->x, c->x); }));
  TRY(sync(c));
  CK(cudaMemcpy(hs.data(), c->st, sizeof(RhsState) * R, cudaMemcpyDeviceToHost));
  const int hc = c->hcap;
  for (int r = 0; r < R; ++r) {
    rep[r].iterations = hs[r].iterations;
    rep[r].converged = hs[r].converged;
    rep[r].status = hs[r].status;
    rep[r].hist_len = hs[r].hist_len;
    rep[r].detail = 0.0;
    if (hist != nullptr && hs[r].hist_len > 0)
      CK(cudaMemcpy(hist + (int64_t)r * max_iter, c->hist + (int64_t)r * hc, sizeof(double) * hs[r].hist_len,
                    cudaMemcpyDeviceToHost));
  }
  if (x_out != nullptr) {
    TRY(download_fields(c, x_out, c->x, R));
    TRY(sync(c));
  }
  return FC_OK;
}

int32_t fc_energy(fc_ctx* c, int32_t R, const double* E, const double* x, double* out) {
  const NvtxRange nvtx_range("fc_energy");
  if (c && !c->sub.empty()) {
    TRY(check_R(R));
    return shard_energy(c, R, E, x, out);
  }
  TRY(check_ctx(c, true));
  TRY(check_R(R));
  if (c->Rcap < R || c->x == nullptr) {
    if (x == nullptr) return set_err(FC_EINVAL, "no resident solution for %d right-hand sides", R);
    TRY(ensure_workspace(c, R, 2));
  }
  if (x != nullptr) TRY(upload_fields(c, c->x, x, R));
  const Geo g = c->geo();
  const Coef C = c->coef();
  Loads L{};
  for (int r = 0; r < R; ++r)
    for (int a = 0; a < c->dim; ++a) L.E[r][a] = E[r * c->dim + a];
  const int64_t chunk = 8192;
  const int nblk = (int)((c->N + chunk - 1) / chunk);
  if ((int64_t)nblk * R * R > c->part_cap) return set_err(FC_ENOTSUP, "partial buffer too small");
  TRY(launch(c, "energy", [&] { k_energy<<<nblk, kThreads, 0, c->stream>>>(g, C, L, R, c->x, c->part, chunk); }));
  TRY(launch(c, "fin_matrix", [&] { k_fin_matrix<<<1, kThreads, 0, c->stream>>>(c->part, nblk, R * R, (double)c->N, c->d_mat); }));
  CK(cudaMemcpyAsync(out, c->d_mat, sizeof(double) * R * R, cudaMemcpyDeviceToHost, c->stream));
  return sync(c);
}

int32_t fc_generate_voronoi(fc_ctx* c, int32_t n_seeds, const double* seeds, const double* packed,
                            int32_t* labels_out) {
  if (c && !c->sub.empty()) {
    if (labels_out != nullptr) return set_err(FC_ENOTSUP, "labels are not gathered on a sharded context");
    for (fc_ctx* sl : c->sub) TRY(fc_generate_voronoi(sl, n_seeds, seeds, packed, nullptr));
    c->coef_kind = FC_COEF_PACKED;
    return FC_OK;
  }
  TRY(check_ctx(c, false));
  if (c->dim != 3) return set_err(FC_EINVAL, "the Voronoi generator is three-dimensional");
  if (n_seeds < 1 || n_seeds > 4096) return set_err(FC_EINVAL, "n_seeds must lie in [1, 4096]");
  const int nsym = 6;
  DevBuf<double> d_seeds, d_packed;
  DevBuf<int> d_lab;
  CK(cudaMalloc(&d_seeds.p, sizeof(double) * 3 * n_seeds));
  CK(cudaMalloc(&d_packed.p, sizeof(double) * nsym * n_seeds));
  CK(cudaMemcpy(d_seeds.p, seeds, sizeof(double) * 3 * n_seeds, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(d_packed.p, packed, sizeof(double) * nsym * n_seeds, cudaMemcpyHostToDevice));
  if (labels_out) CK(cudaMalloc(&d_lab.p, sizeof(int) * c->N));
  const int64_t count = (int64_t)nsym * c->N;
  free_indexed(c);
  if (c->A == nullptr || c->A_count != count) {
    cudaFree(c->A);
    c->A = nullptr;
    CK(cudaMalloc(&c->A, sizeof(double) * count + kFieldPad));
    c->A_count = count;
  }
  c->coef_kind = FC_COEF_PACKED;
  const int blocks = c->num_sms * 8;
  const size_t sm = sizeof(double) * 3 * n_seeds;
  CK(cudaFuncSetAttribute(k_gen_voronoi, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
  TRY(launch(c, "gen_voronoi", [&] {
    k_gen_voronoi<<<blocks, 256, sm, c->stream>>>(c->n0g, c->n[1], c->n[2], c->s0[c->me], n_seeds, d_seeds.p,
                                                  d_packed.p, nsym, c->N, c->A, d_lab.p);
  }));
  if (labels_out) CK(cudaMemcpyAsync(labels_out, d_lab.p, sizeof(int) * c->N, cudaMemcpyDeviceToHost, c->stream));
  TRY(sync(c));
  return FC_OK;
}

int32_t fc_spheres_stamp(fc_ctx* c, int32_t n, const int32_t* centres, double radius, int64_t* covered) {
  if (covered == nullptr || (n > 0 && centres == nullptr)) return set_err(FC_EINVAL, "null argument");
  if (c && !c->sub.empty()) {
    int64_t tot = 0;
    for (fc_ctx* sl : c->sub) {
      int64_t k = 0;
      TRY(fc_spheres_stamp(sl, n, centres, radius, &k));
      tot += k;
    }
    *covered = tot;
    return FC_OK;
  }
  TRY(check_ctx(c, false));
  if (c->dim != 3) return set_err(FC_EINVAL, "the sphere generator is three-dimensional");
  if (!(radius > 0) || radius > 512) return set_err(FC_EINVAL, "radius must lie in (0, 512]");
  if (n < 0) return set_err(FC_EINVAL, "negative number of centres");
  if (c->sphere_bits == nullptr) {
    const size_t words = (size_t)((c->N + 31) / 32);
    CK(cudaMalloc(&c->sphere_bits, sizeof(unsigned) * words));
    CK(cudaMalloc(&c->sphere_count, sizeof(unsigned long long)));
    CK(cudaMemsetAsync(c->sphere_bits, 0, sizeof(unsigned) * words, c->stream));
    CK(cudaMemsetAsync(c->sphere_count, 0, sizeof(unsigned long long), c->stream));
  }
  if (n > 0) {
    DevBuf<int> d_c;
    CK(cudaMalloc(&d_c.p, sizeof(int) * 3 * n));
    CK(cudaMemcpyAsync(d_c.p, centres, sizeof(int) * 3 * n, cudaMemcpyHostToDevice, c->stream));
    const int rad = (int)std::ceil(radius);
    const unsigned grid = (unsigned)((int64_t)n * (2 * rad + 1));
    TRY(launch(c, "stamp_spheres", [&] {
      k_stamp_spheres<<<grid, 256, 0, c->stream>>>(c->n0g, c->n[1], c->n[2], c->s0[c->me], c->n[0], d_c.p, n, rad,
                                                   radius * radius, c->sphere_bits, c->sphere_count);
    }));
    TRY(sync(c));
  }
  unsigned long long k = 0;
  CK(cudaMemcpy(&k, c->sphere_count, sizeof(k), cudaMemcpyDeviceToHost));
  *covered = (int64_t)k;
  return FC_OK;
}

int32_t fc_spheres_finish(fc_ctx* c, double high, double low) {
  if (c && !c->sub.empty()) {
    for (fc_ctx* sl : c->sub) TRY(fc_spheres_finish(sl, high, low));
    c->coef_kind = FC_COEF_ISOTROPIC;
    return FC_OK;
  }
  TRY(check_ctx(c, false));
  if (c->sphere_bits == nullptr) return set_err(FC_EINVAL, "no spheres stamped");
  free_indexed(c);
  if (c->A == nullptr || c->A_count != c->N) {
    cudaFree(c->A);
    c->A = nullptr;
    CK(cudaMalloc(&c->A, sizeof(double) * c->N + kFieldPad));
    c->A_count = c->N;
  }
  c->coef_kind = FC_COEF_ISOTROPIC;
  TRY(launch(c, "spheres_field", [&] {
    k_spheres_field<<<c->num_sms * 8, 256, 0, c->stream>>>(c->N, c->sphere_bits, high, low, c->A);
  }));
  TRY(sync(c));
  cudaFree(c->sphere_bits);
  cudaFree(c->sphere_count);
  c->sphere_bits = nullptr;
  c->sphere_count = nullptr;
  return FC_OK;
}

int32_t fc_set_profiling(fc_ctx* c, int32_t on) {
  if (c == nullptr) return set_err(FC_EINVAL, "null context");
  if (!c->sub.empty()) {
    for (fc_ctx* sl : c->sub) TRY(fc_set_profiling(sl, on));
    return FC_OK;
  }
  if (!on && c->prof_on) {
    cudaStreamSynchronize(c->stream);
    drain_profile(c);
  }
  c->prof_on = on != 0;
  return FC_OK;
}
int32_t fc_profile_count(fc_ctx* c) {
  if (c && !c->sub.empty()) return fc_profile_count(c->sub[0]);
  return c ? (int32_t)c->prof.size() : 0;
}
int32_t fc_profile_get(fc_ctx* c, int32_t i, char* name, int32_t cap, int64_t* launches, double* ms) {
  if (c && !c->sub.empty()) return fc_profile_get(c->sub[0], i, name, cap, launches, ms);
  if (c == nullptr || i < 0 || i >= (int)c->prof.size()) return set_err(FC_EINVAL, "bad profile index");
  std::snprintf(name, cap, "%s", c->prof[i].name.c_str());
  *launches = c->prof[i].launches;
  *ms = c->prof[i].ms;
  return FC_OK;
}
int32_t fc_profile_reset(fc_ctx* c) {
  if (c == nullptr) return set_err(FC_EINVAL, "null context");
  if (!c->sub.empty()) {
    for (fc_ctx* sl : c->sub) TRY(fc_profile_reset(sl));
    return FC_OK;
  }
  cudaStreamSynchronize(c->stream);
  drain_profile(c);
  c->prof.clear();
  c->prof_idx.clear();
  return FC_OK;
}
int32_t fc_plan_info(fc_ctx* c, const char* key, int32_t* value) {
  if (c == nullptr || key == nullptr || value == nullptr) return set_err(FC_EINVAL, "null argument");
  const fc_ctx* p = c->sub.empty() ? c : c->sub[0];
  const std::string k(key);
  if (k == "two_field") *value = p->two_field;
  else if (k == "fold_fwd") *value = p->fold_fwd;
  else if (k == "packed_fused") *value = p->pk_npen > 0;
  else if (k == "n_phases") *value = p->lab != nullptr ? p->nph : 0;
  else if (k == "slabs") *value = c->sub.empty() ? 1 : (int32_t)c->sub.size();
  else return set_err(FC_EINVAL, "unknown plan key %s", key);
  return FC_OK;
}

int64_t fc_launch_count(fc_ctx* c) {
  if (c && !c->sub.empty()) {
    int64_t n = 0;
    for (fc_ctx* sl : c->sub) n += sl->launches;
    return n;
  }
  return c ? c->launches : 0;
}

int32_t fc_timer_mark(fc_ctx* c, int32_t slot) {
  if (c && !c->sub.empty()) return fc_timer_mark(c->sub[0], slot);
  TRY(check_ctx(c, false));
  if (slot < 0 || slot >= 8) return set_err(FC_EINVAL, "timer slot %d out of range", slot);
  if (!c->timer_ev[slot]) CK(cudaEventCreate(&c->timer_ev[slot]));
  CK(cudaEventRecord(c->timer_ev[slot], c->stream));
  return FC_OK;
}

int32_t fc_timer_elapsed(fc_ctx* c, int32_t a, int32_t b, double* ms) {
  if (c && !c->sub.empty()) return fc_timer_elapsed(c->sub[0], a, b, ms);
  TRY(check_ctx(c, false));
  if (a < 0 || a >= 8 || b < 0 || b >= 8 || !c->timer_ev[a] || !c->timer_ev[b])
    return set_err(FC_EINVAL, "timer slots not recorded");
  CK(cudaEventSynchronize(c->timer_ev[b]));
  float f = 0.f;
  CK(cudaEventElapsedTime(&f, c->timer_ev[a], c->timer_ev[b]));
  *ms = f;
  return FC_OK;
}

}  // extern "C"
