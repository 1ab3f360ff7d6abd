// Separable-PSF fast path: when every output
// plane's kernel is rank one, K[zo] = u_zo (x) v_zo (x) w_zo (axis-aligned
// Gaussians, the BASELINE PSF family), the depth-variant correlation
//
//   H x[zo](y, x) = sum_{a,b,c} K[zo,a,b,c] x[zo+a-rz, y+b-ry, x+c-rx]
//                 = sum_b v_zo[b] sum_c w_zo[c] t_zo(y+b-ry, x+c-rx),
//   t_zo = sum_a u_zo[a] x[zo+a-rz]                      (reference _core.pyx:17-53)
//
// costs kz + kx + ky FMAs per voxel instead of kz*ky*kx, and the adjoint
//
//   H^T v[zi] = sum_a u_zo[a] S_zo(v[zo]),  zo = zi+rz-a,
//   S_zo(f)(y, x) = sum_b v_zo[b] sum_c w_zo[c] f(y+ry-b, x+rx-c)  (_core.pyx:56-96)
//
// applies each plane's flipped 2-D filter once and combines in depth.  Both
// are memory-bound (one plane read + one plane written per output plane),
// so they are measured against HBM, never against the FMA roofline.  The
// summation order differs from the dense kernels (rounding-level, <= 1e-12
// relative in fp64); the factors are detected at upload (blur.py side) and
// the dense graded kernel stays the default everywhere.
//
// One CTA owns a 32 x 16 tile and marches a chunk of output planes in depth.
// Forward: a ring of kz+1 halo tiles of x (TMA, mbarrier per slot) feeds the
// depth combination t (tile + halo, smem), then an x pass and a y pass.
// Adjoint: each input plane is filtered once into a ring of kz filtered
// tiles, and every output plane is a kz-term depth combination of the ring.
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "../../include/bd3mg_b200.h"
#include "common.cuh"
#include "errors.h"

namespace bd3mg {
bool encode_tmap(CUtensorMap* map, const void* base, bool f64, long long nx, long long ny, long long nz, int boxw,
                 int boxh);

namespace {

constexpr int kSx = 32, kSy = 16, kSNT = 128;
constexpr int kChunk = 16;  // output planes marched per CTA

constexpr int sgcd(int a, int b) { return b == 0 ? a : sgcd(b, a % b); }

template <typename T, int K>
struct SepGeo {
  static constexpr int VEC = 16 / (int)sizeof(T);
  static constexpr int R = (K - 1) / 2;
  static constexpr int RXA = (R + VEC - 1) / VEC * VEC, OFF = RXA - R;
  // staged plane tile: x in [x0-RXA, x0+32+R), y in [y0-R, y0+16+R)
  static constexpr int BW = (kSx + RXA + R + 2 * VEC - 1) / (2 * VEC) * (2 * VEC);
  static constexpr int ROWQ = 128 / sgcd(BW * (int)sizeof(T), 128);
  static constexpr int TH = kSy + 2 * R, TW = kSx + 2 * R;
  static constexpr int BH = (TH + ROWQ - 1) / ROWQ * ROWQ;
  static constexpr int PL = BW * BH;
};

struct SepArgs {
  const void* src;   // fragment, plane 0 = depth src_z0
  const void* u;     // (nzk, kz) depth factors
  const void* v;     // (nzk, ky)
  const void* w;     // (nzk, kx)
  void* out;         // rows out_lo .. out_hi
  long long plane;
  int nx, ny, nzk, kz, src_z0, src_nz, out_lo, out_hi;
  int use_tma;
};

template <typename T>
BD3MG_D void stage_plane_fallback(T* dst, const T* src, long long plane, int zrel, int x0, int y0, int nx, int ny,
                                  int bw, int bh, int rxa, int r) {
  const T* base = src + (long long)zrel * plane;
  for (int i = threadIdx.x; i < bw * bh; i += kSNT) {
    const int row = i / bw, col = i - row * bw;
    const int gy = y0 - r + row, gx = x0 - rxa + col;
    const bool ok = gy >= 0 && gy < ny && gx >= 0 && gx < nx;
    cp_async<sizeof(T)>(dst + i, ok ? base + (long long)gy * nx + gx : src, ok);
  }
}

// ---------------------------------------------------------------------------
template <typename T, int K>
__global__ void __launch_bounds__(kSNT) sep_forward_kernel(const __grid_constant__ SepArgs p,
                                                           const __grid_constant__ CUtensorMap tm) {
  using G = SepGeo<T, K>;
  constexpr int R = G::R;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  unsigned char* base = smem_raw + ((128u - (smem_u32(smem_raw) & 127u)) & 127u);
  const int ring = p.kz + 1;
  T* rs = reinterpret_cast<T*>(base);                       // [ring][PL]
  T* tb = rs + (size_t)ring * G::PL;                         // [TH][TW]
  T* rb = tb + G::TH * G::TW;                                // [TH][32]
  uint64_t* bars = reinterpret_cast<uint64_t*>(rb + G::TH * kSx + 1);
  bars = reinterpret_cast<uint64_t*>((reinterpret_cast<uintptr_t>(bars) + 7) & ~uintptr_t(7));

  const int x0 = blockIdx.x * kSx, y0 = blockIdx.y * kSy;
  const int zo_a = p.out_lo + blockIdx.z * kChunk, zo_b = min(zo_a + kChunk - 1, p.out_hi);
  const int rz = (p.kz - 1) / 2;
  const T* src = static_cast<const T*>(p.src);
  // input planes of the chunk inside the fragment
  const int zi_a = max(zo_a - rz, p.src_z0), zi_b = min(zo_b + rz, p.src_z0 + p.src_nz - 1);
  const bool tma = p.use_tma != 0;
  if (tma && threadIdx.x == 0) {
    for (int s = 0; s < ring; ++s) mbar_init(&bars[s], 1);
    fence_mbar_init();
  }
  __syncthreads();
  auto slot = [&](int zi) { return (zi - zi_a) % ring; };
  auto phase = [&](int zi) { return (uint32_t)((zi - zi_a) / ring) & 1u; };
  auto issue = [&](int zi) {
    T* dst = rs + (size_t)slot(zi) * G::PL;
    if (tma) {
      if (threadIdx.x == 0) {
        mbar_expect_tx(&bars[slot(zi)], G::PL * sizeof(T));
        tma_load_3d(dst, &tm, x0 - G::RXA, y0 - R, zi - p.src_z0, &bars[slot(zi)]);
      }
    } else {
      stage_plane_fallback<T>(dst, src, p.plane, zi - p.src_z0, x0, y0, p.nx, p.ny, G::BW, G::BH, G::RXA, R);
      cp_async_commit();
    }
  };
  // keep kz planes resident plus one in flight
  int issued = zi_a - 1;
  auto ensure = [&](int upto) {  // planes <= upto issued (ring permitting)
    while (issued < min(upto, zi_b)) issue(++issued);
  };
  ensure(zo_a + rz + 1);
  int waited = zi_a - 1;
  for (int zo = zo_a; zo <= zo_b; ++zo) {
    // the slot of plane zo+rz+1 last held zo-rz-1, released by the previous
    // iteration's closing barrier
    ensure(zo + rz + 1);
    const int need = min(zo + rz, zi_b);
    if (tma) {
      while (waited < need) {
        ++waited;
        mbar_wait(&bars[slot(waited)], phase(waited));
      }
    } else {
      cp_async_wait<0>();
      __syncthreads();
      waited = need;
    }
    const T* uz = static_cast<const T*>(p.u) + (long long)zo * p.kz;
    const T* vz = static_cast<const T*>(p.v) + (long long)zo * K;
    const T* wz = static_cast<const T*>(p.w) + (long long)zo * K;
    // (1) depth combination over the tile + halo
    const int a_lo = max(0, zi_a - zo + rz), a_hi = min(p.kz - 1, zi_b - zo + rz);
    for (int i = threadIdx.x; i < G::TH * G::TW; i += kSNT) {
      const int r = i / G::TW, c = i - r * G::TW;
      const int si = r * G::BW + c + G::OFF;
      T t = T(0);
      for (int a = a_lo; a <= a_hi; ++a) t = fma_rn(__ldg(uz + a), rs[(size_t)slot(zo + a - rz) * G::PL + si], t);
      tb[i] = t;
    }
    __syncthreads();
    // (2) x pass
    T wk[K], vk[K];
#pragma unroll
    for (int c = 0; c < K; ++c) wk[c] = __ldg(wz + c);
#pragma unroll
    for (int b = 0; b < K; ++b) vk[b] = __ldg(vz + b);
    for (int i = threadIdx.x; i < G::TH * kSx; i += kSNT) {
      const int r = i / kSx, c = i - r * kSx;
      T s = T(0);
#pragma unroll
      for (int cc = 0; cc < K; ++cc) s = fma_rn(wk[cc], tb[r * G::TW + c + cc], s);
      rb[i] = s;
    }
    __syncthreads();
    // (3) y pass + store
    T* out = static_cast<T*>(p.out) + (long long)(zo - p.out_lo) * p.plane;
    for (int i = threadIdx.x; i < kSy * kSx; i += kSNT) {
      const int r = i / kSx, c = i - r * kSx;
      const int y = y0 + r, x = x0 + c;
      T s = T(0);
#pragma unroll
      for (int b = 0; b < K; ++b) s = fma_rn(vk[b], rb[(r + b) * kSx + c], s);
      if (y < p.ny && x < p.nx) out[(long long)y * p.nx + x] = s;
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
template <typename T, int K>
__global__ void __launch_bounds__(kSNT) sep_adjoint_kernel(const __grid_constant__ SepArgs p,
                                                           const __grid_constant__ CUtensorMap tm) {
  using G = SepGeo<T, K>;
  constexpr int R = G::R;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  unsigned char* base = smem_raw + ((128u - (smem_u32(smem_raw) & 127u)) & 127u);
  T* fs = reinterpret_cast<T*>(base);                        // [2][PL] staged input planes
  T* ss = fs + 2 * G::PL;                                     // [kz][16*32] filtered planes
  T* rb = ss + (size_t)p.kz * kSy * kSx;                      // [TH][32]
  uint64_t* bars = reinterpret_cast<uint64_t*>(rb + G::TH * kSx + 1);
  bars = reinterpret_cast<uint64_t*>((reinterpret_cast<uintptr_t>(bars) + 7) & ~uintptr_t(7));

  const int x0 = blockIdx.x * kSx, y0 = blockIdx.y * kSy;
  const int zi_a = p.out_lo + blockIdx.z * kChunk, zi_b = min(zi_a + kChunk - 1, p.out_hi);
  const int rz = (p.kz - 1) / 2;
  const T* src = static_cast<const T*>(p.src);
  // planes zo whose filtered tile is needed: [zi_a-rz, zi_b+rz] within [0, nzk) and the fragment
  const int zo_a = max(max(zi_a - rz, 0), p.src_z0);
  const int zo_b = min(min(zi_b + rz, p.nzk - 1), p.src_z0 + p.src_nz - 1);
  const bool tma = p.use_tma != 0;
  if (tma && threadIdx.x == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    fence_mbar_init();
  }
  __syncthreads();
  auto issue = [&](int zo) {
    const int b = (zo - zo_a) & 1;
    T* dst = fs + b * G::PL;
    if (tma) {
      if (threadIdx.x == 0) {
        mbar_expect_tx(&bars[b], G::PL * sizeof(T));
        tma_load_3d(dst, &tm, x0 - G::RXA, y0 - R, zo - p.src_z0, &bars[b]);
      }
    } else {
      stage_plane_fallback<T>(dst, src, p.plane, zo - p.src_z0, x0, y0, p.nx, p.ny, G::BW, G::BH, G::RXA, R);
      cp_async_commit();
    }
  };
  auto sslot = [&](int zo) { return ((zo % p.kz) + p.kz) % p.kz; };
  if (zo_a <= zo_b) issue(zo_a);
  int zi = zi_a;  // next output plane
  for (int zo = zo_a; zo <= zo_b; ++zo) {
    const int b = (zo - zo_a) & 1;
    if (zo < zo_b) issue(zo + 1);
    if (tma) {
      mbar_wait(&bars[b], (uint32_t)((zo - zo_a) >> 1) & 1u);
    } else {
      if (zo < zo_b) cp_async_wait<1>();
      else cp_async_wait<0>();
      __syncthreads();
    }
    const T* vz = static_cast<const T*>(p.v) + (long long)zo * K;
    const T* wz = static_cast<const T*>(p.w) + (long long)zo * K;
    T wk[K], vk[K];
#pragma unroll
    for (int c = 0; c < K; ++c) wk[c] = __ldg(wz + c);
#pragma unroll
    for (int q = 0; q < K; ++q) vk[q] = __ldg(vz + q);
    const T* f = fs + b * G::PL;
    // x pass (flipped taps) over the rows y0-R .. y0+16+R
    for (int i = threadIdx.x; i < G::TH * kSx; i += kSNT) {
      const int r = i / kSx, c = i - r * kSx;
      T s = T(0);
#pragma unroll
      for (int cc = 0; cc < K; ++cc) s = fma_rn(wk[K - 1 - cc], f[r * G::BW + c + cc + G::OFF], s);
      rb[i] = s;
    }
    __syncthreads();
    // y pass (flipped taps) into the ring slot of zo
    T* sd = ss + (size_t)sslot(zo) * kSy * kSx;
    for (int i = threadIdx.x; i < kSy * kSx; i += kSNT) {
      const int r = i / kSx, c = i - r * kSx;
      T s = T(0);
#pragma unroll
      for (int q = 0; q < K; ++q) s = fma_rn(vk[K - 1 - q], rb[(r + q) * kSx + c], s);
      sd[i] = s;
    }
    __syncthreads();
    // every output whose last contributing plane is now filtered
    while (zi <= zi_b && (min(zi + rz, zo_b) <= zo)) {
      const int a_lo = max(0, zi + rz - zo_b), a_hi = min(p.kz - 1, zi + rz - zo_a);
      T* out = static_cast<T*>(p.out) + (long long)(zi - p.out_lo) * p.plane;
      for (int i = threadIdx.x; i < kSy * kSx; i += kSNT) {
        const int r = i / kSx, c = i - r * kSx;
        const int y = y0 + r, x = x0 + c;
        T s = T(0);
        for (int a = a_lo; a <= a_hi; ++a) {
          const int z = zi + rz - a;
          s = fma_rn(__ldg(static_cast<const T*>(p.u) + (long long)z * p.kz + a),
                     ss[(size_t)sslot(z) * kSy * kSx + i], s);
        }
        if (y < p.ny && x < p.nx) out[(long long)y * p.nx + x] = s;
      }
      ++zi;
    }
    __syncthreads();  // staged slot b is refilled two planes later; ring slots reused after kz planes
  }
  // outputs with no contributing plane inside the fragment are zero
  for (; zi <= zi_b; ++zi) {
    T* out = static_cast<T*>(p.out) + (long long)(zi - p.out_lo) * p.plane;
    for (int i = threadIdx.x; i < kSy * kSx; i += kSNT) {
      const int y = y0 + i / kSx, x = x0 + i % kSx;
      if (y < p.ny && x < p.nx) out[(long long)y * p.nx + x] = T(0);
    }
  }
}

int errf(int code, const char* fmt, ...) __attribute__((format(printf, 2, 3)));
int errf(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  return set_error(code, buf);
}

template <typename T, int K>
int launch_sep(SepArgs& a, bool adj, cudaStream_t s) {
  using G = SepGeo<T, K>;
  static const bool no_tma = getenv("BD3MG_NO_TMA") != nullptr;
  CUtensorMap tm;
  memset(&tm, 0, sizeof(tm));
  a.use_tma = !no_tma && encode_tmap(&tm, a.src, sizeof(T) == 8, a.nx, a.ny, a.src_nz, G::BW, G::BH);
  size_t smem;
  if (!adj)
    smem = 128 + ((size_t)(a.kz + 1) * G::PL + G::TH * G::TW + G::TH * kSx + 2) * sizeof(T) + (a.kz + 2) * 8;
  else
    smem = 128 + ((size_t)2 * G::PL + (size_t)a.kz * kSy * kSx + G::TH * kSx + 2) * sizeof(T) + 4 * 8;
  if (smem > 227 * 1024) return errf(BD3MG_EINVAL, "separable path: kz=%d does not fit shared memory", a.kz);
  auto kern = adj ? sep_adjoint_kernel<T, K> : sep_forward_kernel<T, K>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return errf(BD3MG_ECUDA, "CUDA: %s", cudaGetErrorString(e));
  const int nout = a.out_hi - a.out_lo + 1;
  dim3 grid((a.nx + kSx - 1) / kSx, (a.ny + kSy - 1) / kSy, (nout + kChunk - 1) / kChunk);
  kern<<<grid, kSNT, smem, s>>>(a, tm);
  count_launches(1);
  e = cudaGetLastError();
  return e == cudaSuccess ? BD3MG_OK : errf(BD3MG_ECUDA, "CUDA: %s", cudaGetErrorString(e));
}

template <typename T>
int sep_correlate(const T* frag, int64_t nzf, int64_t ny, int64_t nx, const T* u, const T* v, const T* w,
                  int64_t nzk, int64_t kz, int64_t ky, int64_t kx, int64_t frag_z0, int64_t out_lo, int64_t out_hi,
                  T* out, int adjoint, void* stream) {
  if (!frag || !u || !v || !w || !out) return errf(BD3MG_EINVAL, "null argument");
  if (nzf < 1 || ny < 1 || nx < 1 || nzk < 1 || kz < 1 || kz % 2 == 0 || ky != kx || ky % 2 == 0)
    return errf(BD3MG_EINVAL, "separable path: invalid shape (needs odd kz and ky == kx in 3/5/7/9)");
  if (out_lo < 0 || out_hi < out_lo || out_hi >= nzk)
    return errf(BD3MG_EINVAL, "output rows [%lld, %lld] outside the kernel stack of %lld planes", (long long)out_lo,
                (long long)out_hi, (long long)nzk);
  SepArgs a;
  memset(&a, 0, sizeof(a));
  a.src = frag; a.u = u; a.v = v; a.w = w; a.out = out;
  a.plane = ny * nx; a.nx = (int)nx; a.ny = (int)ny; a.nzk = (int)nzk; a.kz = (int)kz;
  a.src_z0 = (int)frag_z0; a.src_nz = (int)nzf; a.out_lo = (int)out_lo; a.out_hi = (int)out_hi;
  cudaStream_t s = (cudaStream_t)stream;
  const bool adj = adjoint != 0;
  switch (ky) {
    case 3: return launch_sep<T, 3>(a, adj, s);
    case 5: return launch_sep<T, 5>(a, adj, s);
    case 7: return launch_sep<T, 7>(a, adj, s);
    case 9: return launch_sep<T, 9>(a, adj, s);
    default: return errf(BD3MG_EINVAL, "separable path: ky = kx = %lld not instantiated (3/5/7/9)", (long long)ky);
  }
}

}  // namespace
}  // namespace bd3mg

using namespace bd3mg;

extern "C" {

int bd3mg_sep_correlate_f64(const double* frag, int64_t nzf, int64_t ny, int64_t nx, const double* u,
                            const double* v, const double* w, int64_t nzk, int64_t kz, int64_t ky, int64_t kx,
                            int64_t frag_z0, int64_t out_lo, int64_t out_hi, double* out, int32_t adjoint,
                            void* stream) {
  return sep_correlate<double>(frag, nzf, ny, nx, u, v, w, nzk, kz, ky, kx, frag_z0, out_lo, out_hi, out, adjoint,
                               stream);
}
int bd3mg_sep_correlate_f32(const float* frag, int64_t nzf, int64_t ny, int64_t nx, const float* u, const float* v,
                            const float* w, int64_t nzk, int64_t kz, int64_t ky, int64_t kx, int64_t frag_z0,
                            int64_t out_lo, int64_t out_hi, float* out, int32_t adjoint, void* stream) {
  return sep_correlate<float>(frag, nzf, ny, nx, u, v, w, nzk, kz, ky, kx, frag_z0, out_lo, out_hi, out, adjoint,
                              stream);
}

}  // extern "C"
