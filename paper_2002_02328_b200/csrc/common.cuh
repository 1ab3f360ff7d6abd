// Shared device helpers for the BD3MG sm_100a kernels.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#define BD3MG_HD __host__ __device__ __forceinline__
#define BD3MG_D __device__ __forceinline__

namespace bd3mg {

// ---- cp.async (LDGSTS) with hardware zero-fill ----------------------------
// src_bytes = 0 zero-fills the destination without touching global memory.
template <int BYTES>
BD3MG_D void cp_async(void* smem_dst, const void* gmem_src, bool in_bounds) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem_dst));
  const int n = in_bounds ? BYTES : 0;
  if constexpr (BYTES == 16) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem_src), "r"(n));
  } else {
    asm volatile("cp.async.ca.shared.global [%0], [%1], %2, %3;\n" ::"r"(s), "l"(gmem_src), "n"(BYTES),
                 "r"(n));
  }
}
BD3MG_D void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
BD3MG_D void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// ---- IEEE helpers that forbid FMA contraction where the reference rounds
// each operation separately (numpy elementwise arithmetic). ----------------
BD3MG_D double add_rn(double a, double b) { return __dadd_rn(a, b); }
BD3MG_D double sub_rn(double a, double b) { return __dsub_rn(a, b); }
BD3MG_D double mul_rn(double a, double b) { return __dmul_rn(a, b); }
BD3MG_D float add_rn(float a, float b) { return __fadd_rn(a, b); }
BD3MG_D float sub_rn(float a, float b) { return __fsub_rn(a, b); }
BD3MG_D float mul_rn(float a, float b) { return __fmul_rn(a, b); }
BD3MG_D double fma_rn(double a, double b, double c) { return __fma_rn(a, b, c); }
BD3MG_D float fma_rn(float a, float b, float c) { return __fmaf_rn(a, b, c); }

// ---- packed fp32 pairs (FFMA2, sm_100a): two correctly rounded FMAs per
// instruction, bitwise equal to two fmaf_rn; halves the FMA issue slots.
BD3MG_D unsigned long long pk2(float lo, float hi) {
  unsigned long long r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
BD3MG_D float2 unpk2(unsigned long long v) {
  float2 r;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(r.x), "=f"(r.y) : "l"(v));
  return r;
}
// acc + kp * v per half (v broadcast to both halves)
BD3MG_D unsigned long long ffma2_pair(unsigned long long kp, float v, unsigned long long acc) {
  unsigned long long r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(kp), "l"(pk2(v, v)), "l"(acc));
  return r;
}

// acc + k * vp per half (k broadcast)
BD3MG_D unsigned long long ffma2_bcast(float k, unsigned long long vp, unsigned long long acc) {
  unsigned long long r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(vp), "l"(pk2(k, k)), "l"(acc));
  return r;
}

// ---- deterministic CTA reduction of NV doubles --------------------------
// Fixed shuffle tree inside each warp, then warps summed in index order by
// thread 0.  Result valid in thread 0 only.  `scratch` needs NW*NV doubles.
template <int NV, int NT>
BD3MG_D void cta_reduce(double (&v)[NV], double* scratch) {
  constexpr int NW = NT / 32;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < NV; ++k) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v[k] += __shfl_xor_sync(0xffffffffu, v[k], off);
  }
  if (lane == 0) {
#pragma unroll
    for (int k = 0; k < NV; ++k) scratch[warp * NV + k] = v[k];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      double s = scratch[k];
      for (int w = 1; w < NW; ++w) s += scratch[w * NV + k];
      v[k] = s;
    }
  }
}

}  // namespace bd3mg

// ---- TMA (cp.async.bulk.tensor) + mbarrier helpers -------------------------
namespace bd3mg {
BD3MG_D uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

BD3MG_D void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
BD3MG_D void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory"); }
BD3MG_D void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
BD3MG_D void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t a = smem_u32(bar);
  uint32_t done = 0;
  do {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(a), "r"(parity)
        : "memory");
  } while (!done);
}
// 3-D tiled TMA load of box (c0, c1, c2) into smem, completion on `bar`.
BD3MG_D void tma_load_3d(void* smem_dst, const void* tmap, int c0, int c1, int c2, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];\n" ::
          "r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(tmap)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}
// Bulk prefetch of `bytes` (multiple of 16, 16-byte aligned) into L2.
BD3MG_D void prefetch_l2_bulk(const void* gptr, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(reinterpret_cast<uint64_t>(gptr)), "r"(bytes)
               : "memory");
}
BD3MG_D void tma_prefetch_desc(const void* tmap) {
  asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(tmap)) : "memory");
}
}  // namespace bd3mg
