// Bulk asynchronous copies (TMA, sm_90+ / sm_100a) with mbarrier completion.
//
// The sweeps stage whole row blocks / pencils in shared memory.  One elected
// thread issues a handful of cp.async.bulk copies (the copy engine generates
// the addresses), instead of every thread looping over 16-byte cp.async
// granules; the CTA waits on one mbarrier phase.
#pragma once
#include <cstdint>

namespace fc {

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned phase) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}

// Generic-proxy writes to smem must be ordered before a later async-proxy
// (bulk copy) write to the same bytes.
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }

// global -> shared, bytes a multiple of 16, both addresses 16-byte aligned
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// Bytes of the 16-byte-aligned window that covers n doubles starting at src;
// element i then sits at dst[i + shift], shift = (src / 8) & 1.  The window may
// extend 8 bytes past the last element: device fields carry kFieldPad bytes of
// padding (fc_engine.cu: dmalloc_field) so the read stays inside the allocation.
__device__ __forceinline__ int bulk_shift(const double* src) {
  return (int)((reinterpret_cast<uintptr_t>(src) >> 3) & 1);
}
__device__ __forceinline__ unsigned bulk_bytes(int n, int shift) { return (unsigned)(((n + shift) * 8 + 15) & ~15); }

// Stage n doubles (called by ONE thread; the CTA waits on bar): returns shift.
__device__ __forceinline__ int bulk_stage_doubles(double* dst, const double* src, int n, uint64_t* bar) {
  const int shift = bulk_shift(src);
  bulk_g2s(dst, src - shift, bulk_bytes(n, shift), bar);
  return shift;
}

}  // namespace fc

// ---- tiled tensor copies (cuTensorMapEncodeTiled maps built on the host) ----
#include <cuda.h>

namespace fc {

// 3-D box load global -> shared (coordinates innermost first), completes on bar
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, int c0, int c1, int c2, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];\n" ::"r"(
          smem_u32(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}
// 3-D box store shared -> global (out-of-range parts of the box are clipped)
__device__ __forceinline__ void tma_store_3d(const CUtensorMap* map, int c0, int c1, int c2, const void* src) {
  asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.tile.bulk_group [%0, {%1, %2, %3}], [%4];\n" ::"l"(map), "r"(c0),
               "r"(c1), "r"(c2), "r"(smem_u32(src))
               : "memory");
}
// shared -> global bulk store (bytes a multiple of 16, 16-byte aligned), bulk_group completion
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, unsigned bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n" ::"l"(dst), "r"(smem_u32(src)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;\n" ::: "memory"); }
// wait until the smem sources of all committed bulk stores have been read
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory"); }

// Row-spectrum view for the tensor maps: the half spectrum of a row sweep is
// stored transposed, W[(r*c + a)*no + o][k][row] (complex), i.e. a 3-D array of
// doubles {2*np, hl, R*c*no}.  A box {4, kBoxK, 1} = rows (row0, row0+1) of
// kBoxK consecutive modes; in shared memory it lands as [k][2] complex.
constexpr int kBoxK = 256;

}  // namespace fc
