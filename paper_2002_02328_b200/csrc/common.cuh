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
