// smnn_tma.cuh -- shared low-level helpers of the fused kernels: dynamic
// shared memory, mbarrier + cp.async.bulk (TMA bulk copy) staging, the time
// chunk map.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace smnn {

extern __shared__ __align__(128) unsigned char smnn_dyn_smem[];

// First time point of chunk k when T points are cut into K chunks.
__device__ __forceinline__ int chunk_begin(int k, int T, int K) { return int((int64_t(k) * T) / K); }

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(bar)), "r"(parity) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// A 16-byte aligned superset [lo, hi) of the global elements [src, src + n):
// cp.async.bulk needs 16-byte aligned addresses and sizes.  Reading up to 15
// bytes outside a tensor stays inside its (>= 256-byte aligned) allocation.
template <class T>
struct Span {
  const T* lo;
  uint32_t bytes;
  int pre;  // element offset of src inside the copied span
  __device__ Span(const T* src, int n) {
    const uintptr_t s = reinterpret_cast<uintptr_t>(src);
    const uintptr_t a = s & ~uintptr_t(15);
    const uintptr_t e = (reinterpret_cast<uintptr_t>(src + n) + 15) & ~uintptr_t(15);
    lo = reinterpret_cast<const T*>(a);
    bytes = n > 0 ? uint32_t(e - a) : 0u;
    pre = int((s - a) / sizeof(T));
  }
};

// Store n elements from shared memory to global memory: a TMA bulk store
// (cp.async.bulk.global.shared::cta) of the 16-byte aligned body, plain stores
// for the unaligned head and tail.  All threads of the CTA call it; thread 0
// issues the bulk copy (the caller commits and waits for the bulk group).
template <class Tio>
__device__ __forceinline__ void rf_store_out(Tio* dst, const Tio* src, int n, int tid, int nt) {
  constexpr int E = int(sizeof(Tio));
  const uintptr_t g0 = reinterpret_cast<uintptr_t>(dst);
  const uintptr_t ga = (g0 + 15) & ~uintptr_t(15), gb = (g0 + uintptr_t(n) * E) & ~uintptr_t(15);
  const int head = int((ga - g0) / E);
  const bool bulk = n * E >= 256 && gb > ga && ((smem_u32(src + head) & 15u) == 0u);
  if (!bulk) {
    for (int e = tid; e < n; e += nt) dst[e] = src[e];
    return;
  }
  const int tail = head + int((gb - ga) / E);
  if (tid < head) dst[tid] = src[tid];
  if (tid < n - tail) dst[tail + tid] = src[tail + tid];
  if (tid == 0)
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst + head),
                 "r"(smem_u32(src + head)), "r"(uint32_t(gb - ga))
                 : "memory");
}

}  // namespace smnn
