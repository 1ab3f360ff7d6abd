// Throughput probes used by bench.py to MEASURE the FMA-pipe peak that the
// H/H^T roofline is quoted against (MEASURED_PEAKS.json has no FP64/FP32
// entry).  Each thread runs 8 independent FMA chains; the result is stored
// so the compiler cannot drop the work.
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/bd3mg_b200.h"

namespace {
template <typename T>
__global__ void __launch_bounds__(256) fma_probe_kernel(T* out, int iters, T a, T b) {
  T r[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) r[k] = (T)(threadIdx.x + k);
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
#pragma unroll
      for (int k = 0; k < 8; ++k) r[k] = fma(r[k], a, b);
    }
  }
  T s = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += r[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// Packed fp32 (FFMA2: two FMAs per lane per instruction, sm_100a)
__device__ __forceinline__ unsigned long long ffma2(unsigned long long a, unsigned long long b,
                                                    unsigned long long c) {
  unsigned long long r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}
__global__ void __launch_bounds__(256) ffma2_probe_kernel(float* out, int iters, float a, float b) {
  unsigned long long r[8];
  const float2 av = make_float2(a, a), bv = make_float2(b, b);
  const unsigned long long ar = *reinterpret_cast<const unsigned long long*>(&av);
  const unsigned long long br = *reinterpret_cast<const unsigned long long*>(&bv);
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const float2 v = make_float2((float)(threadIdx.x + k), (float)(threadIdx.x - k));
    r[k] = *reinterpret_cast<const unsigned long long*>(&v);
  }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
#pragma unroll
      for (int k = 0; k < 8; ++k) r[k] = ffma2(r[k], ar, br);
    }
  }
  float s = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const float2 v = *reinterpret_cast<const float2*>(&r[k]);
    s += v.x + v.y;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
}  // namespace

extern "C" int bd3mg_fma_probe(int32_t dtype, int32_t blocks, int32_t iters, void* out, double* flops_out,
                               void* stream) {
  if (blocks < 1 || iters < 1 || !out) return BD3MG_EINVAL;
  const double flops = (dtype == 2 ? 4.0 : 2.0) * 8 * 16 * (double)iters * 256.0 * blocks;
  if (flops_out) *flops_out = flops;
  if (dtype == 2)  // packed fp32 (FFMA2) probe
    ffma2_probe_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>((float*)out, iters, 0.999999f, 1e-7f);
  else if (dtype == BD3MG_F64)
    fma_probe_kernel<double><<<blocks, 256, 0, (cudaStream_t)stream>>>((double*)out, iters, 0.999999, 1e-7);
  else
    fma_probe_kernel<float><<<blocks, 256, 0, (cudaStream_t)stream>>>((float*)out, iters, 0.999999f, 1e-7f);
  return cudaGetLastError() == cudaSuccess ? BD3MG_OK : BD3MG_ECUDA;
}
