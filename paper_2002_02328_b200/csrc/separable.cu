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
// filters each plane once and combines in depth.  Both are memory-bound, so
// they are measured against HBM, never against the FMA roofline.  The
// summation order differs from the dense kernels (rounding-level, <= 1e-12
// relative in fp64); the factors are detected at upload (separable.py) and
// the dense graded kernel stays the default everywhere.
//
// Two streaming passes through one temporary volume (grow-only scratch):
//   sep_zw_kernel   depth FIR, a register window of source planes per 8- or
//                   16-byte pixel vector and CH consecutive outputs;
//   sep_xyt_kernel  per-plane separable 2-D filter (fp32): a 64 x 64 tile +
//                   halo per TMA box, double-buffered over 4 planes per CTA,
//                   register-blocked x pass then y pass from 16-byte
//                   shared-memory loads (sep_xy2_kernel: the same without
//                   TMA, for rows that are not 16-byte multiples;
//                   sep_xy_kernel: scalar, the fp64 default).
// Forward = z then xy; adjoint = flipped xy then z.  HBM traffic per launch:
// four volume passes (read src, write tmp, read tmp, write out).
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>

#include "../../include/bd3mg_b200.h"
#include "common.cuh"
#include "conv_dispatch.cuh"
#include "errors.h"

namespace bd3mg {
namespace {

constexpr int kZNT = 256;    // depth-FIR threads
constexpr int kZChunk = 16;  // output planes per depth-FIR thread
constexpr int kXx = 64, kXy = 32, kXNT = 256;

template <typename T>
struct Vec16;
template <>
struct Vec16<double> {
  using type = double2;
};
template <>
struct Vec16<float> {
  using type = float4;
};
template <typename T, int VB>
struct VecB;
template <>
struct VecB<double, 16> {
  using type = double2;
};
template <>
struct VecB<double, 8> {
  using type = double;
};
template <>
struct VecB<float, 16> {
  using type = float4;
};
template <>
struct VecB<float, 8> {
  using type = float2;
};

// Depth FIR.  Forward: dst[zo] = sum_a u[zo][a] src[zo+a-rz] over the source
// planes present; adjoint: dst[zi] = sum_a u[zo][a] src[zo], zo = zi+rz-a.
// src plane 0 = depth s_z0 (s_n planes); dst plane 0 = depth d_lo.
struct SepZArgs {
  const void* src;
  void* dst;
  const void* u;
  long long plane;
  int kz, nzk, s_z0, s_n, d_lo, d_hi;
};

// KZ > 0: taps unrolled at compile time (all kz source loads of an output
// issue back to back; absent planes are predicated off); KZ == 0: runtime kz.
template <typename T, bool ADJ, int KZ>
__global__ void __launch_bounds__(kZNT) sep_z_kernel(const __grid_constant__ SepZArgs p) {
  using V = typename Vec16<T>::type;
  constexpr int VEC = 16 / (int)sizeof(T);
  const long long q = ((long long)blockIdx.x * kZNT + threadIdx.x) * VEC;
  if (q >= p.plane) return;
  // 16-byte accesses need every plane to start on a 16-byte boundary
  const bool full = q + VEC <= p.plane && p.plane % VEC == 0;
  const int z_a = p.d_lo + blockIdx.y * kZChunk, z_b = min(z_a + kZChunk - 1, p.d_hi);
  const int kz = KZ > 0 ? KZ : p.kz;
  const int rz = (kz - 1) / 2;
  const T* src = static_cast<const T*>(p.src);
  const T* u = static_cast<const T*>(p.u);
  T* dst = static_cast<T*>(p.dst);
  // source planes present (adjoint: and inside the stack)
  const int s_lo = ADJ ? max(p.s_z0, 0) : p.s_z0;
  const int s_hi = ADJ ? min(p.s_z0 + p.s_n - 1, p.nzk - 1) : p.s_z0 + p.s_n - 1;
  for (int z = z_a; z <= z_b; ++z) {
    T acc[VEC];
#pragma unroll
    for (int i = 0; i < VEC; ++i) acc[i] = T(0);
    auto tap = [&](int a) {
      const int zs = ADJ ? z + rz - a : z + a - rz;
      if (zs < s_lo || zs > s_hi) return;
      const T c = __ldg(u + (long long)(ADJ ? zs : z) * kz + a);
      const T* sp = src + (long long)(zs - p.s_z0) * p.plane + q;
      if (full) {
        const V v = __ldg(reinterpret_cast<const V*>(sp));
        const T* vs = reinterpret_cast<const T*>(&v);
#pragma unroll
        for (int i = 0; i < VEC; ++i) acc[i] = fma_rn(c, vs[i], acc[i]);
      } else {
        for (int i = 0; i < VEC && q + i < p.plane; ++i) acc[i] = fma_rn(c, sp[i], acc[i]);
      }
    };
    if constexpr (KZ > 0) {
#pragma unroll
      for (int a = 0; a < KZ; ++a) tap(a);
    } else {
      for (int a = 0; a < kz; ++a) tap(a);
    }
    T* dp = dst + (long long)(z - p.d_lo) * p.plane + q;
    if (full) {
      *reinterpret_cast<V*>(dp) = *reinterpret_cast<const V*>(acc);
    } else {
      for (int i = 0; i < VEC && q + i < p.plane; ++i) dp[i] = acc[i];
    }
  }
}

// Register-window depth FIR: a thread owns one 16-byte pixel vector and CH
// consecutive outputs; the CH+KZ-1 source planes they need are loaded once,
// back to back, into registers (absent planes read as zero: exact no-ops),
// and the CHxKZ coefficients of the chunk are staged in shared memory.
// (Measured against a depth-marching ring over whole chunks: the window is
// faster -- its loads are independent, the ring's are one per step.)
template <typename T, bool ADJ, int KZ, int CH, int VB, bool ZFAST>
__global__ void __launch_bounds__(kZNT) sep_zw_kernel(const __grid_constant__ SepZArgs p) {
  using V = typename VecB<T, VB>::type;
  constexpr int VEC = VB / (int)sizeof(T);
  const int zblk = ZFAST ? blockIdx.x : blockIdx.y, pblk = ZFAST ? blockIdx.y : blockIdx.x;
  constexpr int RZ = (KZ - 1) / 2, W = CH + KZ - 1;
  __shared__ T cs[W * KZ];  // FWD: [output i][a]; ADJ: [source row j][a]
  const int z_a = p.d_lo + zblk * CH;
  const int s_lo = ADJ ? max(p.s_z0, 0) : p.s_z0;
  const int s_hi = ADJ ? min(p.s_z0 + p.s_n - 1, p.nzk - 1) : p.s_z0 + p.s_n - 1;
  const T* u = static_cast<const T*>(p.u);
  for (int i = threadIdx.x; i < W * KZ; i += kZNT) {
    const int row = i / KZ, a = i - row * KZ;
    T c = T(0);
    if (!ADJ) {
      const int z = z_a + row;
      if (row < CH && z <= p.d_hi) c = u[(long long)z * KZ + a];
    } else {
      const int zs = z_a - RZ + row;  // rows outside the stack have no coefficients
      if (zs >= 0 && zs < p.nzk) c = u[(long long)zs * KZ + a];
    }
    cs[i] = c;
  }
  __syncthreads();
  const long long q = ((long long)pblk * kZNT + threadIdx.x) * VEC;
  if (q >= p.plane) return;
  const T* src = static_cast<const T*>(p.src);
  V win[W];  // window row j <-> source plane z_a - RZ + j
#pragma unroll
  for (int j = 0; j < W; ++j) {
    const int zs = z_a - RZ + j;
    win[j] = (zs >= s_lo && zs <= s_hi) ? __ldg(reinterpret_cast<const V*>(src + (long long)(zs - p.s_z0) * p.plane + q))
                                         : V{};
  }
  T* dst = static_cast<T*>(p.dst);
#pragma unroll
  for (int i = 0; i < CH; ++i) {
    const int z = z_a + i;
    if (z > p.d_hi) break;
    T acc[VEC];
#pragma unroll
    for (int k = 0; k < VEC; ++k) acc[k] = T(0);
#pragma unroll
    for (int a = 0; a < KZ; ++a) {
      // FWD: source z+a-RZ = window row i+a; ADJ: source zo = z+RZ-a = window row i+2RZ-a
      const int j = ADJ ? i + 2 * RZ - a : i + a;
      const T c = ADJ ? cs[j * KZ + a] : cs[i * KZ + a];
      const T* w = reinterpret_cast<const T*>(&win[j]);
#pragma unroll
      for (int k = 0; k < VEC; ++k) acc[k] = fma_rn(c, w[k], acc[k]);
    }
    *reinterpret_cast<V*>(dst + (long long)(z - p.d_lo) * p.plane + q) = *reinterpret_cast<const V*>(acc);
  }
}

// Per-plane separable 2-D filter of rows [r_lo, r_hi] (global depths; src and
// dst plane 0 = depth z0 each).  FLIP: the adjoint's flipped taps.
struct SepXYArgs {
  const void* src;
  void* dst;
  const void* v;
  const void* w;
  long long plane;
  int nx, ny, s_z0, d_z0, r_lo, r_n;
};

template <typename T, int K, bool FLIP>
__global__ void __launch_bounds__(kXNT) sep_xy_kernel(const __grid_constant__ SepXYArgs p) {
  using V = typename Vec16<T>::type;
  constexpr int VEC = 16 / (int)sizeof(T);
  constexpr int R = (K - 1) / 2;
  constexpr int RXA = (R + VEC - 1) / VEC * VEC, OFF = RXA - R;  // 16-byte aligned row segments
  constexpr int TW = kXx + 2 * RXA, TH = kXy + 2 * R;
  __shared__ __align__(16) T ts[TH][TW + VEC];
  __shared__ T rs[TH][kXx + 1];
  const int z = p.r_lo + blockIdx.z;
  const int x0 = blockIdx.x * kXx, y0 = blockIdx.y * kXy;
  const T* src = static_cast<const T*>(p.src) + (long long)(z - p.s_z0) * p.plane;
  T* dst = static_cast<T*>(p.dst) + (long long)(z - p.d_z0) * p.plane;
  if (p.nx % VEC == 0) {  // every 16-byte chunk is wholly inside or outside the row
    constexpr int CPR = TW / VEC;
    for (int i = threadIdx.x; i < TH * CPR; i += kXNT) {
      const int r = i / CPR, c = (i - r * CPR) * VEC;
      const int y = y0 - R + r, x = x0 - RXA + c;
      const V v = (y >= 0 && y < p.ny && x >= 0 && x < p.nx)
                      ? __ldg(reinterpret_cast<const V*>(src + (long long)y * p.nx + x))
                      : V{};
      *reinterpret_cast<V*>(&ts[r][c]) = v;
    }
  } else {
    for (int i = threadIdx.x; i < TH * TW; i += kXNT) {
      const int r = i / TW, c = i - r * TW;
      const int y = y0 - R + r, x = x0 - RXA + c;
      ts[r][c] = (y >= 0 && y < p.ny && x >= 0 && x < p.nx) ? src[(long long)y * p.nx + x] : T(0);
    }
  }
  T wk[K], vk[K];
  const T* wz = static_cast<const T*>(p.w) + (long long)z * K;
  const T* vz = static_cast<const T*>(p.v) + (long long)z * K;
#pragma unroll
  for (int c = 0; c < K; ++c) {
    wk[c] = __ldg(wz + (FLIP ? K - 1 - c : c));
    vk[c] = __ldg(vz + (FLIP ? K - 1 - c : c));
  }
  __syncthreads();
  for (int i = threadIdx.x; i < TH * kXx; i += kXNT) {
    const int r = i / kXx, c = i - r * kXx;
    T s = T(0);
#pragma unroll
    for (int cc = 0; cc < K; ++cc) s = fma_rn(wk[cc], ts[r][c + cc + OFF], s);
    rs[r][c] = s;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < kXy * kXx; i += kXNT) {
    const int r = i / kXx, c = i - r * kXx;
    const int y = y0 + r, x = x0 + c;
    T s = T(0);
#pragma unroll
    for (int b = 0; b < K; ++b) s = fma_rn(vk[b], rs[r + b][c], s);
    if (y < p.ny && x < p.nx) dst[(long long)y * p.nx + x] = s;
  }
}

// Register-blocked variant of sep_xy_kernel (same sums in the same order, so
// bitwise equal): a thread produces 4 consecutive x outputs of the x pass
// from 16-byte shared-memory loads, and a 4 (x) by RY (y) block of the y pass
// from RY + K - 1 16-byte row loads, so shared-memory traffic per voxel drops
// ~3x (the scalar kernel is shared-memory-bound, not HBM-bound).  Output rows
// are stored as 16-byte vectors where the row allows.  PZ > 1: the CTA walks
// PZ planes of its tile and the next plane's tile loads are in flight in
// registers while the current plane is filtered (rows nx % VEC == 0 only).
template <typename T, int K, bool FLIP, int TX, int TY, int RY, int NT, int PZ>
__global__ void __launch_bounds__(NT, PZ > 1 ? 3 : 1) sep_xy2_kernel(const __grid_constant__ SepXYArgs p) {
  using V = typename Vec16<T>::type;
  constexpr int VEC = 16 / (int)sizeof(T);
  constexpr int G = 4;  // x outputs per thread
  constexpr int R = (K - 1) / 2;
  constexpr int RXA = (R + G - 1) / G * G, OFF = RXA - R;
  constexpr int TW = TX + 2 * RXA, TH = TY + 2 * R;
  constexpr int NC = (OFF + K - 1 + G + G - 1) / G;  // 4-element chunks one x-pass item reads
  constexpr int GX = TX / G;
  constexpr int CPR = TW / VEC, NLD = (TH * CPR + NT - 1) / NT;
  static_assert(TX % G == 0 && TY % RY == 0 && (TY / RY) * GX == NT, "one y-pass item per thread");
  __shared__ __align__(16) T ts[TH][TW];
  __shared__ __align__(16) T rs[TH][TX];
  const int x0 = blockIdx.x * TX, y0 = blockIdx.y * TY;
  const int za = p.r_lo + blockIdx.z * PZ, zb = min(za + PZ, p.r_lo + p.r_n);
  const bool vec_rows = p.nx % VEC == 0;
  V pre[NLD];
  auto load_tile = [&](int z) {  // vector rows: into registers
    const T* src = static_cast<const T*>(p.src) + (long long)(z - p.s_z0) * p.plane;
#pragma unroll
    for (int k = 0; k < NLD; ++k) {
      const int i = threadIdx.x + k * NT;
      const int r = i / CPR, c = (i - r * CPR) * VEC;
      const int y = y0 - R + r, x = x0 - RXA + c;
      pre[k] = (i < TH * CPR && y >= 0 && y < p.ny && x >= 0 && x < p.nx)
                   ? __ldg(reinterpret_cast<const V*>(src + (long long)y * p.nx + x))
                   : V{};
    }
  };
  auto stage_tile = [&]() {
#pragma unroll
    for (int k = 0; k < NLD; ++k) {
      const int i = threadIdx.x + k * NT;
      const int r = i / CPR, c = (i - r * CPR) * VEC;
      if (i < TH * CPR) *reinterpret_cast<V*>(&ts[r][c]) = pre[k];
    }
  };
  if (vec_rows) {
    load_tile(za);
    stage_tile();
  }
  for (int z = za; z < zb; ++z) {
    if (!vec_rows) {
      const T* src = static_cast<const T*>(p.src) + (long long)(z - p.s_z0) * p.plane;
      for (int i = threadIdx.x; i < TH * TW; i += NT) {
        const int r = i / TW, c = i - r * TW;
        const int y = y0 - R + r, x = x0 - RXA + c;
        ts[r][c] = (y >= 0 && y < p.ny && x >= 0 && x < p.nx) ? src[(long long)y * p.nx + x] : T(0);
      }
    }
    T wk[K], vk[K];
    const T* wz = static_cast<const T*>(p.w) + (long long)z * K;
    const T* vz = static_cast<const T*>(p.v) + (long long)z * K;
#pragma unroll
    for (int c = 0; c < K; ++c) {
      wk[c] = __ldg(wz + (FLIP ? K - 1 - c : c));
      vk[c] = __ldg(vz + (FLIP ? K - 1 - c : c));
    }
    __syncthreads();  // ts holds plane z; rs free
    const bool more = vec_rows && z + 1 < zb;
    if (more) load_tile(z + 1);
    for (int i = threadIdx.x; i < TH * GX; i += NT) {
      const int r = i / GX, c = (i - r * GX) * G;
      T seg[NC * G];
#pragma unroll
      for (int j = 0; j < NC * G; j += VEC) *reinterpret_cast<V*>(&seg[j]) = *reinterpret_cast<const V*>(&ts[r][c + j]);
      T o[G];
#pragma unroll
      for (int g = 0; g < G; ++g) {
        T s = T(0);
#pragma unroll
        for (int cc = 0; cc < K; ++cc) s = fma_rn(wk[cc], seg[g + cc + OFF], s);
        o[g] = s;
      }
#pragma unroll
      for (int j = 0; j < G; j += VEC) *reinterpret_cast<V*>(&rs[r][c + j]) = *reinterpret_cast<const V*>(&o[j]);
    }
    __syncthreads();  // rs complete; ts free
    const int gx = threadIdx.x % GX, gy = threadIdx.x / GX;
    const int c = gx * G, r0 = gy * RY;
    T acc[RY][G];
#pragma unroll
    for (int i = 0; i < RY; ++i)
#pragma unroll
      for (int g = 0; g < G; ++g) acc[i][g] = T(0);
#pragma unroll
    for (int j = 0; j < RY + K - 1; ++j) {
      T row[G];
#pragma unroll
      for (int g = 0; g < G; g += VEC) *reinterpret_cast<V*>(&row[g]) = *reinterpret_cast<const V*>(&rs[r0 + j][c + g]);
#pragma unroll
      for (int i = 0; i < RY; ++i) {
        const int b = j - i;  // output row r0+i, tap b, in ascending b per output
        if (b >= 0 && b < K) {
#pragma unroll
          for (int g = 0; g < G; ++g) acc[i][g] = fma_rn(vk[b], row[g], acc[i][g]);
        }
      }
    }
    T* dst = static_cast<T*>(p.dst) + (long long)(z - p.d_z0) * p.plane;
    const int x = x0 + c;
#pragma unroll
    for (int i = 0; i < RY; ++i) {
      const int y = y0 + r0 + i;
      if (y >= p.ny) break;
      T* dp = dst + (long long)y * p.nx + x;
      if (vec_rows && x + G <= p.nx) {
#pragma unroll
        for (int g = 0; g < G; g += VEC) *reinterpret_cast<V*>(dp + g) = *reinterpret_cast<const V*>(&acc[i][g]);
      } else {
#pragma unroll
        for (int g = 0; g < G; ++g)
          if (x + g < p.nx) dp[g] = acc[i][g];
      }
    }
    if (more) stage_tile();  // after this plane's x pass: ts is free
    __syncthreads();          // rs reads done before the next x pass
  }
}

// TMA-fed fp32 2-D filter: the CTA walks PZ planes of one 64 x 64 output
// tile; each plane's (64 + 2 RXA) x (64 + 2R) source tile is a single TMA box
// (halo zero-filled by the copy engine), double-buffered so the next plane
// lands while the current one is filtered.  Same x / y passes as
// sep_xy2_kernel (bitwise equal).
struct SepXYTArgs {
  CUtensorMap tm;  // src rows: (nx, ny, planes), box (TW, TH, 1)
  SepXYArgs a;
};

template <int K>
struct XytGeo {
  static constexpr int TX = 64, TY = 64, RY = 4, NT = 256, G = 4;
  static constexpr int R = (K - 1) / 2, RXA = (R + G - 1) / G * G, OFF = RXA - R;
  static constexpr int TW = TX + 2 * RXA, TH = TY + 2 * R;
  static constexpr int BS = (TH * TW + 31) / 32 * 32;  // buffer stride (floats): TMA needs 128-byte aligned boxes
  static constexpr size_t smem() { return (2 * (size_t)BS + (size_t)TH * TX) * sizeof(float) + 16 + 128; }
};

template <int K, bool FLIP, int PZ>
__global__ void __launch_bounds__(256) sep_xyt_kernel(const __grid_constant__ SepXYTArgs P) {
  using Geo = XytGeo<K>;
  constexpr int TX = Geo::TX, TY = Geo::TY, RY = Geo::RY, NT = Geo::NT, G = Geo::G;
  constexpr int R = Geo::R, RXA = Geo::RXA, OFF = Geo::OFF, TW = Geo::TW, TH = Geo::TH;
  constexpr int NC = (OFF + K - 1 + G + G - 1) / G;
  constexpr int GX = TX / G;
  static_assert((TY / RY) * GX == NT, "one y-pass item per thread");
  const SepXYArgs& p = P.a;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  float* base = reinterpret_cast<float*>((reinterpret_cast<uintptr_t>(smem_raw) + 127) & ~uintptr_t(127));
  float (*ts0)[TW] = reinterpret_cast<float (*)[TW]>(base);
  float (*ts1)[TW] = reinterpret_cast<float (*)[TW]>(base + Geo::BS);
  float (*rs)[TX] = reinterpret_cast<float (*)[TX]>(base + 2 * Geo::BS);
  uint64_t* bar = reinterpret_cast<uint64_t*>(base + 2 * Geo::BS + TH * TX);
  const int x0 = blockIdx.x * TX, y0 = blockIdx.y * TY;
  const int za = p.r_lo + blockIdx.z * PZ, zb = min(za + PZ, p.r_lo + p.r_n);
  constexpr uint32_t kBytes = TH * TW * sizeof(float);
  if (threadIdx.x == 0) {
    tma_prefetch_desc(&P.tm);
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    fence_mbar_init();
    mbar_expect_tx(&bar[0], kBytes);
    tma_load_3d(&ts0[0][0], &P.tm, x0 - RXA, y0 - R, za - p.s_z0, &bar[0]);
  }
  __syncthreads();
  for (int z = za, k = 0; z < zb; ++z, ++k) {
    const int buf = k & 1;
    if (threadIdx.x == 0 && z + 1 < zb) {  // buf^1 was last read by plane z-1's x pass (all past its barrier)
      mbar_expect_tx(&bar[buf ^ 1], kBytes);
      tma_load_3d(buf ? &ts0[0][0] : &ts1[0][0], &P.tm, x0 - RXA, y0 - R, z + 1 - p.s_z0, &bar[buf ^ 1]);
    }
    float wk[K], vk[K];
    const float* wz = static_cast<const float*>(p.w) + (long long)z * K;
    const float* vz = static_cast<const float*>(p.v) + (long long)z * K;
#pragma unroll
    for (int c = 0; c < K; ++c) {
      wk[c] = __ldg(wz + (FLIP ? K - 1 - c : c));
      vk[c] = __ldg(vz + (FLIP ? K - 1 - c : c));
    }
    mbar_wait(&bar[buf], (k >> 1) & 1);
    float (*ts)[TW] = buf ? ts1 : ts0;
    for (int i = threadIdx.x; i < TH * GX; i += NT) {
      const int r = i / GX, c = (i - r * GX) * G;
      float seg[NC * G];
#pragma unroll
      for (int j = 0; j < NC * G; j += 4) *reinterpret_cast<float4*>(&seg[j]) = *reinterpret_cast<const float4*>(&ts[r][c + j]);
      float o[G];
#pragma unroll
      for (int g = 0; g < G; ++g) {
        float acc = 0.f;
#pragma unroll
        for (int cc = 0; cc < K; ++cc) acc = fma_rn(wk[cc], seg[g + cc + OFF], acc);
        o[g] = acc;
      }
      *reinterpret_cast<float4*>(&rs[r][c]) = *reinterpret_cast<const float4*>(o);
    }
    __syncthreads();  // rs complete; ts[buf] free
    const int gx = threadIdx.x % GX, gy = threadIdx.x / GX;
    const int c = gx * G, r0 = gy * RY;
    float acc[RY][G];
#pragma unroll
    for (int i = 0; i < RY; ++i)
#pragma unroll
      for (int g = 0; g < G; ++g) acc[i][g] = 0.f;
#pragma unroll
    for (int j = 0; j < RY + K - 1; ++j) {
      const float4 rv = *reinterpret_cast<const float4*>(&rs[r0 + j][c]);
      const float row[G] = {rv.x, rv.y, rv.z, rv.w};
#pragma unroll
      for (int i = 0; i < RY; ++i) {
        const int b = j - i;
        if (b >= 0 && b < K) {
#pragma unroll
          for (int g = 0; g < G; ++g) acc[i][g] = fma_rn(vk[b], row[g], acc[i][g]);
        }
      }
    }
    float* dst = static_cast<float*>(p.dst) + (long long)(z - p.d_z0) * p.plane;
    const int x = x0 + c;
#pragma unroll
    for (int i = 0; i < RY; ++i) {
      const int y = y0 + r0 + i;
      if (y >= p.ny) break;
      float* dp = dst + (long long)y * p.nx + x;
      if (x + G <= p.nx) {
        *reinterpret_cast<float4*>(dp) = *reinterpret_cast<const float4*>(&acc[i][0]);
      } else {
#pragma unroll
        for (int g = 0; g < G; ++g)
          if (x + g < p.nx) dp[g] = acc[i][g];
      }
    }
    __syncthreads();  // rs reads done before the next x pass
  }
}

template <typename T>
struct Xy2Cfg;
template <>
struct Xy2Cfg<float> {
  static constexpr int TX = 64, TY = 64, RY = 4, NT = 256;
};
template <>
struct Xy2Cfg<double> {
  static constexpr int TX = 64, TY = 32, RY = 2, NT = 256;
};

int env_int(const char* name, int dflt) {
  const char* e = getenv(name);
  return e && *e ? atoi(e) : dflt;
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
int launch_xy(SepXYArgs& a, int nrows, bool flip, cudaStream_t s) {
  if (nrows <= 0) return BD3MG_OK;
  // fp32: the TMA-fed, double-buffered register-blocked filter (5; rows
  // that are not 16-byte multiples take the register-blocked one, 2); fp64:
  // the scalar one (1; at C2 every variant is within +-8%)
  const int xyv = env_int("BD3MG_SEP_XY", sizeof(T) == 4 ? 5 : 1);
  a.r_n = nrows;
  if constexpr (sizeof(T) == 4) {
    if (xyv == 5 && a.nx % 4 == 0 && (reinterpret_cast<uintptr_t>(a.src) & 15) == 0) {
      using Geo = XytGeo<K>;
      constexpr int PZ = 4;  // measured: 2 / 8 / 16 planes per CTA are 0-8% slower (profiles/r1_sep_probe.md)
      SepXYTArgs ta;
      ta.a = a;
      if (!encode_tmap(&ta.tm, a.src, false, a.nx, a.ny, a.r_lo - a.s_z0 + nrows, Geo::TW, Geo::TH))
        return errf(BD3MG_EINVAL, "separable: TMA descriptor rejected");
      auto kern = flip ? sep_xyt_kernel<K, true, PZ> : sep_xyt_kernel<K, false, PZ>;
      cudaError_t e = ensure_smem_attr(kern, Geo::smem());
      if (e != cudaSuccess) return errf(BD3MG_ECUDA, "CUDA: %s", cudaGetErrorString(e));
      dim3 grid((a.nx + Geo::TX - 1) / Geo::TX, (a.ny + Geo::TY - 1) / Geo::TY, (nrows + PZ - 1) / PZ);
      kern<<<grid, Geo::NT, Geo::smem(), s>>>(ta);
      count_launches(1);
      e = cudaGetLastError();
      return e == cudaSuccess ? BD3MG_OK : errf(BD3MG_ECUDA, "CUDA: %s", cudaGetErrorString(e));
    }
  }
  if (xyv == 2 || xyv == 3 || xyv == 5) {
    using C = Xy2Cfg<T>;
    constexpr int PZ = 4;
    const int pz = xyv == 3 ? PZ : 1;
    dim3 grid((a.nx + C::TX - 1) / C::TX, (a.ny + C::TY - 1) / C::TY, (nrows + pz - 1) / pz);
    if (xyv == 3) {
      if (flip)
        sep_xy2_kernel<T, K, true, C::TX, C::TY, C::RY, C::NT, PZ><<<grid, C::NT, 0, s>>>(a);
      else
        sep_xy2_kernel<T, K, false, C::TX, C::TY, C::RY, C::NT, PZ><<<grid, C::NT, 0, s>>>(a);
    } else if (flip) {
      sep_xy2_kernel<T, K, true, C::TX, C::TY, C::RY, C::NT, 1><<<grid, C::NT, 0, s>>>(a);
    } else {
      sep_xy2_kernel<T, K, false, C::TX, C::TY, C::RY, C::NT, 1><<<grid, C::NT, 0, s>>>(a);
    }
  } else {
    dim3 grid((a.nx + kXx - 1) / kXx, (a.ny + kXy - 1) / kXy, nrows);
    if (flip)
      sep_xy_kernel<T, K, true><<<grid, kXNT, 0, s>>>(a);
    else
      sep_xy_kernel<T, K, false><<<grid, kXNT, 0, s>>>(a);
  }
  count_launches(1);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? BD3MG_OK : errf(BD3MG_ECUDA, "CUDA: %s", cudaGetErrorString(e));
}

template <typename T, bool ADJ, int KZ, int CH, int VB, bool ZFAST>
int launch_zw(SepZArgs& a, int n, cudaStream_t s) {
  constexpr int VEC = VB / (int)sizeof(T);
  const unsigned pb = (unsigned)(((a.plane + VEC - 1) / VEC + kZNT - 1) / kZNT), zb = (unsigned)((n + CH - 1) / CH);
  const dim3 g = ZFAST ? dim3(zb, pb) : dim3(pb, zb);
  sep_zw_kernel<T, ADJ, KZ, CH, VB, ZFAST><<<g, kZNT, 0, s>>>(a);
  count_launches(1);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? BD3MG_OK : errf(BD3MG_ECUDA, "CUDA: %s", cudaGetErrorString(e));
}

// Register-window variant: BD3MG_SEP_Z = CH * 1000 + VB * 10 + ZFAST (probe
// knob, scripts/sep_probe.py; results are bitwise equal across variants)
template <typename T, bool ADJ, int KZ>
int launch_zw_var(SepZArgs& a, int n, int var, cudaStream_t s) {
  switch (var) {
    case 8160: return launch_zw<T, ADJ, KZ, 8, 16, false>(a, n, s);
    case 8161: return launch_zw<T, ADJ, KZ, 8, 16, true>(a, n, s);
    case 8080: return launch_zw<T, ADJ, KZ, 8, 8, false>(a, n, s);
    case 8081: return launch_zw<T, ADJ, KZ, 8, 8, true>(a, n, s);
    case 16081: return launch_zw<T, ADJ, KZ, 16, 8, true>(a, n, s);
    case 16161: return launch_zw<T, ADJ, KZ, 16, 16, true>(a, n, s);
    default: return -1;
  }
}

template <typename T>
int launch_z(SepZArgs& a, bool adj, cudaStream_t s) {
  const int n = a.d_hi - a.d_lo + 1;
  if (n <= 0) return BD3MG_OK;
  constexpr int VEC = 16 / (int)sizeof(T);
  const long long vecs = (a.plane + VEC - 1) / VEC;
  dim3 grid((unsigned)((vecs + kZNT - 1) / kZNT), (n + kZChunk - 1) / kZChunk);
  if (a.plane % VEC == 0) {  // register-window kernel
    // measured defaults (profiles/r1_sep_probe.md): fp32 16 outputs per
    // thread, 16-byte vectors, depth chunks fastest in the grid so the window
    // overlap of neighbouring chunks is served by L2; fp64 8 outputs
    const int var = env_int("BD3MG_SEP_Z", sizeof(T) == 4 ? 16161 : 8160);
    switch (a.kz) {
#define BD3MG_SEPZW(KZ)                                                                                           \
  case KZ: {                                                                                                      \
    const int rc = adj ? launch_zw_var<T, true, KZ>(a, n, var, s) : launch_zw_var<T, false, KZ>(a, n, var, s); \
    if (rc >= 0) return rc;                                                                                       \
    return errf(BD3MG_EINVAL, "BD3MG_SEP_Z=%d: unknown depth-FIR variant", var);                                   \
  }
      BD3MG_SEPZW(3) BD3MG_SEPZW(5) BD3MG_SEPZW(7) BD3MG_SEPZW(9) BD3MG_SEPZW(11) BD3MG_SEPZW(13)
      BD3MG_SEPZW(15) BD3MG_SEPZW(17) BD3MG_SEPZW(19) BD3MG_SEPZW(21)
#undef BD3MG_SEPZW
      default: break;
    }
  }
  switch (a.kz) {
#define BD3MG_SEPZ(KZ)                                                  \
  case KZ:                                                              \
    if (adj)                                                            \
      sep_z_kernel<T, true, KZ><<<grid, kZNT, 0, s>>>(a);               \
    else                                                                \
      sep_z_kernel<T, false, KZ><<<grid, kZNT, 0, s>>>(a);              \
    break;
    BD3MG_SEPZ(3) BD3MG_SEPZ(5) BD3MG_SEPZ(7) BD3MG_SEPZ(9) BD3MG_SEPZ(11) BD3MG_SEPZ(13) BD3MG_SEPZ(15)
    BD3MG_SEPZ(17) BD3MG_SEPZ(19) BD3MG_SEPZ(21)
#undef BD3MG_SEPZ
    default:
      if (adj)
        sep_z_kernel<T, true, 0><<<grid, kZNT, 0, s>>>(a);
      else
        sep_z_kernel<T, false, 0><<<grid, kZNT, 0, s>>>(a);
  }
  count_launches(1);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? BD3MG_OK : errf(BD3MG_ECUDA, "CUDA: %s", cudaGetErrorString(e));
}

// Scratch volume per (device, stream), grow-only (a cudaMallocAsync per call
// re-maps the pool when its release threshold is 0: measured 10x slower).
int scratch(cudaStream_t s, size_t bytes, void** out) {
  static std::mutex mu;
  static std::map<std::pair<int, cudaStream_t>, std::pair<void*, size_t>> cache;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return errf(BD3MG_ECUDA, "CUDA: %s", cudaGetErrorString(e));
  std::lock_guard<std::mutex> lock(mu);
  auto& ent = cache[{dev, s}];
  if (ent.second < bytes) {
    if (ent.first) {
      cudaStreamSynchronize(s);
      cudaFree(ent.first);
      ent = {nullptr, 0};
    }
    e = cudaMalloc(&ent.first, bytes);
    if (e != cudaSuccess) return errf(BD3MG_ECUDA, "separable scratch (%zu bytes): %s", bytes, cudaGetErrorString(e));
    ent.second = bytes;
  }
  *out = ent.first;
  return BD3MG_OK;
}

template <typename T, int K>
int run_sep(const T* frag, int nzf, int ny, int nx, const T* u, const T* v, const T* w, int nzk, int kz, int frag_z0,
            int out_lo, int out_hi, T* out, bool adj, cudaStream_t s) {
  const long long plane = (long long)ny * nx;
  const int rz = (kz - 1) / 2;
  if (!adj) {
    // t rows = output rows
    const int n = out_hi - out_lo + 1;
    T* t = nullptr;
    int rc = scratch(s, (size_t)n * plane * sizeof(T), (void**)&t);
    if (rc) return rc;
    SepZArgs za{frag, t, u, plane, kz, nzk, frag_z0, nzf, out_lo, out_hi};
    rc = launch_z<T>(za, false, s);
    SepXYArgs xa{t, out, v, w, plane, nx, ny, out_lo, out_lo, out_lo};
    if (!rc) rc = launch_xy<T, K>(xa, n, false, s);
    return rc;
  }
  // adjoint: filtered planes zo in [out_lo-rz, out_hi+rz] within the stack and the fragment
  const int s_lo = std::max(std::max(out_lo - rz, 0), frag_z0);
  const int s_hi = std::min(std::min(out_hi + rz, nzk - 1), frag_z0 + nzf - 1);
  const int ns = s_hi - s_lo + 1;
  if (ns <= 0) {
    cudaError_t e = cudaMemsetAsync(out, 0, (size_t)(out_hi - out_lo + 1) * plane * sizeof(T), s);
    return e == cudaSuccess ? BD3MG_OK : errf(BD3MG_ECUDA, "CUDA: %s", cudaGetErrorString(e));
  }
  T* sb = nullptr;
  int rc = scratch(s, (size_t)ns * plane * sizeof(T), (void**)&sb);
  if (rc) return rc;
  SepXYArgs xa{frag, sb, v, w, plane, nx, ny, frag_z0, s_lo, s_lo};
  rc = launch_xy<T, K>(xa, ns, true, s);
  SepZArgs za{sb, out, u, plane, kz, nzk, s_lo, ns, out_lo, out_hi};
  if (!rc) rc = launch_z<T>(za, true, s);
  return rc;
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
  cudaStream_t s = (cudaStream_t)stream;
  const bool adj = adjoint != 0;
  const int a0 = (int)nzf, a1 = (int)ny, a2 = (int)nx, a3 = (int)nzk, a4 = (int)kz, a5 = (int)frag_z0;
  const int a6 = (int)out_lo, a7 = (int)out_hi;
  switch (ky) {
    case 3: return run_sep<T, 3>(frag, a0, a1, a2, u, v, w, a3, a4, a5, a6, a7, out, adj, s);
    case 5: return run_sep<T, 5>(frag, a0, a1, a2, u, v, w, a3, a4, a5, a6, a7, out, adj, s);
    case 7: return run_sep<T, 7>(frag, a0, a1, a2, u, v, w, a3, a4, a5, a6, a7, out, adj, s);
    case 9: return run_sep<T, 9>(frag, a0, a1, a2, u, v, w, a3, a4, a5, a6, a7, out, adj, s);
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
