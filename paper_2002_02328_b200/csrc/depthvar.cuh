// Depth-variant 3-D correlation H and its adjoint H^T for sm_100a, with the
// fused epilogues of the BD3MG block step.
//
// Operator (reference pkg/src/bd3mg/_core.pyx:17-53):
//   out[zo,y,x] = sum_{a,b,c} K[zo,a,b,c] * frag[zo+a-rz, y+b-ry, x+c-rx]
// zero outside the fragment / plane.  The adjoint (_core.pyx:56-96) is the
// same correlation with the per-output coefficient set
//   Kt[zi,a',b',c'] = K[zi+a'-rz, kz-1-a', ky-1-b', kx-1-c']   (0 if the
//   source depth zi+a'-rz is outside [0,nzk))
// which is gathered once per CTA into shared memory, so H and H^T share one
// FMA loop.
//
// Work decomposition: one CTA computes a TY x TX output tile of one output
// plane.  It walks the kz input planes of that plane; each plane's halo tile
// (TY+ky-1) x (TX+kx-1) is staged by cp.async (zero-filled outside the
// fragment/plane, so the FMA loop has no branches) into a double-buffered
// shared-memory ring.  Each thread owns an RY x RX register tile of
// accumulators; it streams the RY+ky-1 input rows of its window through
// registers (RX+kx-1 values per row) and applies every coefficient row that
// touches them.  Accumulation order per output is a -> b -> c, the reference
// order, for every fragment offset (so slab and full-volume results are
// bitwise identical, reference tests/test_blur.py:139-147).
//
// Shared-memory row layout is de-interleaved by x mod RX: element e of a row
// lives at (e % RX) * Q + e / RX.  Thread tx reads element tx*RX + j, i.e.
// phase j % RX, slot tx + j / RX: consecutive lanes read consecutive words,
// so every LDS is conflict-free.
#pragma once

#include <cuda.h>

#include <type_traits>

#include "common.cuh"

namespace bd3mg {

enum ConvMode : int {
  M_STORE = 0,  // dst0 = acc
  M_RESID = 1,  // dst0 = acc - sub; partial: sum dst0^2
  M_GRAD = 2,   // (adjoint) dst0 = acc + sub (sub = regulariser gradient rows, greg_kernel)
  M_GRAM1 = 3,  // partial: sum acc0^2               (+ optional store dst0 = acc0)
  M_GRAM2 = 4,  // partial: acc0^2, acc0*acc1, acc1^2 (dual input, shared taps)
  M_GRAMC = 5,  // dst0 = acc0 (H E_S g); partial: acc0^2, acc0*c, c^2 with c = sub[o] (cached H E_S d)
  M_GRAM2P = 6, // M_GRAM2 as two single-input passes over one tile ring (input 1, then input 0):
                // the same tile, sums and partials bit for bit, half the staging smem
  M_GRADF = 7,  // (adjoint) dst0 = acc + greg with the regulariser gradient computed in the epilogue from
                // the iterate tile (TMA-staged into the freed ring buffer): greg_tile's arithmetic, omega
                // stored, optionally the recorder terms + snapshot roll (no separate stencil pass)
};

constexpr int kMaxJobs = 32;
constexpr int kRgNV = 12;  // regulariser-Gram sums per partial row (= kRegNV, stencil.cuh)

template <typename T>
struct alignas(64) ConvJob {
  CUtensorMap tmap0;    // TMA descriptors of src0/src1 (filled by conv_launch)
  CUtensorMap tmap1;
  const T* src0;        // fragment base; plane 0 is global depth src_z0
  const T* src1;        // second fragment (M_GRAM2), same geometry
  T* dst0;              // output rows; row 0 is global depth out_lo
  const T* sub;         // M_RESID: rows aligned with dst0
  const T* xg;          // M_GRADF: iterate fragment (plane 0 = depth xg_z0, xg_nz planes; tmap1 maps it)
  T* omega;             // M_GRADF: omega rows aligned with dst0; M_GRAM2 (fp64): omega rows of the block
                        //   (row 0 = src_z0) -- the regulariser Gram terms are then computed by the tiles
                        //   whose output plane lies inside the block (no separate reg_gram pass), or null
  T* snap;              // M_GRADF: recorder snapshot rows aligned with dst0 (rolled), or null
  double* eparts;       // M_GRADF: recorder partial rows (one per CTA, kEvalNV), or null (no recorder);
                        //   M_GRAM2 with omega: regulariser-Gram partial rows, kRgNV per (block plane, tile)
  long long src_z0;
  long long xg_z0;
  int src_nz, xg_nz;
  int out_lo, nout;     // global output rows [out_lo, out_lo+nout)
  int work_begin;       // prefix of nout over jobs (grid.z index of first plane)
  int use_tma;          // 1: stage tiles with TMA; 0: cp.async fallback
  int epi_tma;          // 1: tmap1 maps `sub` (RESID / GRAD, one input): the epilogue operand tile is
                        //    staged by TMA into the free tile buffer during the last tap plane
};

// Geometry / coefficient part of the launch arguments: everything one output
// tile needs besides its own job (conv_tile takes this; the persistent sweep
// kernel, sweep_pk.cuh, embeds one).
template <typename T>
struct ConvGeom {
  const T* K;           // (nzk, kz, ky, kx) coefficient stack
  int nzk, kz, ky, kx;  // runtime kz; ky/kx also template params on fast path
  int ny, nx;
  long long plane;      // ny*nx
  int nz_global;        // global depth (axial far-face rule)
  double two_eta, lam, two_kappa, delta2, x_min, x_max;  // regulariser (M_GRADF epilogue)
};

template <typename T>
struct ConvArgs : ConvGeom<T> {
  int njobs;
  int tiles_x, tiles_y;
  int raster_group;     // tiles per rasterisation group (0: plain x, y, z order); see cta_pos
  double* partials;     // [gridDim.z * tiles_y * tiles_x][NV]
  const double* gate;   // optional: the launch is a no-op while *gate != 0 (device-side loops, krylov.cuh)
  ConvJob<T> jobs[kMaxJobs];
};

// Launch-order rasterisation of the (tile, z) grid.  Plain order walks all
// tiles of one output plane before the next, so on large planes the kz
// input planes of the CTAs in flight outgrow L2 and are re-read from DRAM
// (C5: each input plane ~10x).  With raster_group = G the linear launch
// index walks z inside groups of G tiles, keeping the in-flight working set
// at G tiles x (in-flight planes + kz) -- L2-resident.  `cta` is the logical
// (z, tile) row of the partial sums, so layouts and reductions do not change.
struct CtaPos {
  int tx, ty, z;
  long long cta;
};
// 64-bit form (any grid).  The fp32 two-plane kernels keep it: their 7 x 7 / 9 x 9 bodies sit at the
// edge of the instruction cache, and the extra code of the 32-bit fast path cost C5's H 3% (measured).
BD3MG_D CtaPos cta_pos64(int group) {
  const long long nx = gridDim.x, ny = gridDim.y, nz = gridDim.z, T = nx * ny;
  const long long L = blockIdx.x + nx * (blockIdx.y + ny * (long long)blockIdx.z);
  long long t, z;
  if (group <= 0 || group >= T) {
    t = L % T;
    z = L / T;
  } else {
    const long long g = L / ((long long)group * nz), full = T / group;
    const long long gg = g < full ? group : T - full * group;
    const long long rem = L - g * group * nz;
    z = rem / gg;
    t = g * group + rem % gg;
  }
  return {(int)(t % nx), (int)(t / nx), (int)z, z * T + t};
}
BD3MG_D CtaPos cta_pos(int group) {
  // (32-bit arithmetic where the grid allows: a 64-bit division is a ~100-instruction subroutine, and
  // every thread of every CTA runs these before its first load)
  const unsigned nx = gridDim.x, ny = gridDim.y, nz = gridDim.z, T = nx * ny;
  const unsigned long long total = (unsigned long long)T * nz;
  if (total < (1ull << 31) && (unsigned long long)nx * ny < (1ull << 31)) {
    const unsigned L = blockIdx.x + nx * (blockIdx.y + ny * blockIdx.z);
    unsigned t, z;
    if (group <= 0 || (unsigned)group >= T) {
      t = blockIdx.x + nx * blockIdx.y;
      z = blockIdx.z;
    } else {
      const unsigned G = (unsigned)group, g = L / (G * nz), full = T / G;
      const unsigned gg = g < full ? G : T - full * G;
      const unsigned rem = L - g * G * nz;
      z = rem / gg;
      t = g * G + rem % gg;
    }
    return {(int)(t % nx), (int)(t / nx), (int)z, (long long)z * T + t};
  }
  return cta_pos64(group);
}

template <int MODE>
struct ModeNV {
  static constexpr int value =
      (MODE == M_RESID || MODE == M_GRAM1) ? 1 : ((MODE == M_GRAM2 || MODE == M_GRAMC || MODE == M_GRAM2P) ? 3 : 0);
};

// ---------------------------------------------------------------------------
// Regulariser pieces shared by the gradient epilogue and the oracle-mirroring
// elementwise kernels.  Each mirrors numpy's separate roundings
// (reference objective.py:87-137).
template <typename T>
struct XView {
  const T* p;          // plane 0 is global depth z0
  long long z0;
  int nzv, ny, nx;
  long long plane;
  BD3MG_D T at(int z, int y, int x) const { return p[(long long)(z - z0) * plane + (long long)y * nx + x]; }
};

// forward differences with a zero row at the far face (objective.py:87-98)
template <typename T>
BD3MG_D T fdx(const XView<T>& v, int z, int y, int x) {
  return (x < v.nx - 1) ? sub_rn(v.at(z, y, x + 1), v.at(z, y, x)) : T(0);
}
template <typename T>
BD3MG_D T fdy(const XView<T>& v, int z, int y, int x) {
  return (y < v.ny - 1) ? sub_rn(v.at(z, y + 1, x), v.at(z, y, x)) : T(0);
}
// half-quadratic weight 1/sqrt(dx^2+dy^2+delta^2) (objective.py:130-132).
// rsqrt (<= 1 ulp from the reference's 1/sqrt) instead of an IEEE sqrt and
// divide: this is the dominant instruction cost of the stencil kernels.
template <typename T>
BD3MG_D T omega_of(T dx, T dy, T delta2) {
  const T s = add_rn(add_rn(mul_rn(dx, dx), mul_rn(dy, dy)), delta2);
  return rsqrt(s);
}

// ---------------------------------------------------------------------------
// Tile configuration.  fp64: RX=2 (one 16-byte LDS per 2 window values);
// fp32: RX=4.  Consecutive lanes of a quarter-warp read consecutive 16-byte
// chunks of one dense smem row, so every window load is conflict-free.
constexpr int cgcd(int a, int b) { return b == 0 ? a : cgcd(b, a % b); }


#ifndef BD3MG_FFMA2
#define BD3MG_FFMA2 1  // packed fp32 FMAs (FFMA2) in the fp32 two-plane correlation kernel
#endif
#ifndef BD3MG_RZ2_RY5
#define BD3MG_RZ2_RY5 4  // rows per thread of the two-plane kernel for 3x3 / 5x5 taps (measured: 4 >= 8 with FFMA2)
#endif
#ifndef BD3MG_RY2
#define BD3MG_RY2 8  // rows per thread of the fp64 dual-input (Gram) mode
#endif
#ifndef BD3MG_RY1
#define BD3MG_RY1 16  // rows per thread of the single-input modes
#endif
#ifndef BD3MG_EARLY_ISSUE
#define BD3MG_EARLY_ISSUE 1  // first TMA load of a tile before its coefficient staging (conv_tile)
#endif
#ifndef BD3MG_WY1
#define BD3MG_WY1 4   // warps per CTA of the single-input modes (tile height WY1 * RY1); measured on B200
                      // at C2: 8 warps x 8 rows (same 64 x 64 tile) ran H in 99.5-117 us against 80 us
#endif

template <typename T, int KY_, int KX_, int MODE, int RYO = 0>
struct ConvCfg {
  static constexpr bool DUAL = (MODE == M_GRAM2);
  static constexpr bool TWOPASS = (MODE == M_GRAM2P);
  static constexpr int KY = KY_, KX = KX_;
  static constexpr int VEC = 16 / sizeof(T);        // elements per 16-byte load
  static constexpr int RX = VEC;                    // outputs per thread in x
  // outputs per thread in y; dual-input rows measured on B200: 8 (fp64), 4 (fp32); the two-pass
  // Gram keeps the dual-input tile (same pixels per CTA, so the same partial sums)
  static constexpr int RY = RYO > 0 ? RYO : (DUAL || TWOPASS) ? (sizeof(T) == 8 ? BD3MG_RY2 : 4) : BD3MG_RY1;
  static constexpr int WX = 32;                     // a warp spans one row group
  static constexpr int WY = (DUAL || TWOPASS || RYO > 0) ? 4 : BD3MG_WY1;  // warps per CTA
  static constexpr int NT = WX * WY;
  static constexpr int TX = WX * RX, TY = WY * RY;
  // TMA boxes must start on a 16-byte boundary in x (measured: odd-element
  // starts fault), so the box origin is x0 - RXA with RXA = RXH rounded up to
  // VEC; OFF = RXA - RXH extra leading columns are read and skipped.
  static constexpr int RXH = (KX - 1) / 2, RYH = (KY - 1) / 2;
  static constexpr int RXA = (RXH + VEC - 1) / VEC * VEC, OFF = RXA - RXH;
  static constexpr int TXH = TX + KX - 1 + OFF, TYH = TY + KY - 1;
  // smem row = TMA box width, padded to 32 bytes; box height padded so the
  // box is a whole number of 128-byte lines (boxes with an odd number of
  // 16-byte chunks per row fault on sm_100a -- measured, scripts/tma_probe.py)
  static constexpr int PITCH = (TXH + 2 * VEC - 1) / (2 * VEC) * (2 * VEC);
  static constexpr int ROWQ = 128 / cgcd(PITCH * (int)sizeof(T), 128);
  static constexpr int BOXH = (TYH + ROWQ - 1) / ROWQ * ROWQ;
  static constexpr int WIN = RX + KX - 1;
  static constexpr int WINP = (OFF + WIN + VEC - 1) / VEC * VEC;  // aligned window incl. OFF lead
  static constexpr int NIN = DUAL ? 2 : 1;
  static constexpr int BOX = BOXH * PITCH;          // elements one TMA box delivers
  static constexpr int TILE = (BOX + 128 / (int)sizeof(T) - 1) / (128 / (int)sizeof(T)) * (128 / (int)sizeof(T));
  static constexpr int NV = ModeNV<MODE>::value;
  static constexpr size_t TILE_BYTES = (size_t)TILE * sizeof(T);  // 128-byte aligned buffer stride
  static constexpr size_t BOX_BYTES = (size_t)BOX * sizeof(T);
  // fp64 dual-input Gram: the regulariser Gram terms of the block are computed before the tap walk
  // (rg_center); their omega tile (TX x TY, cp.async-staged) and the reduction scratch follow the
  // barriers.  The dual-input tile runs 2 CTAs per SM (shared-memory bound), so these 17 KB are free.
  static constexpr bool RGF = DUAL && sizeof(T) == 8;
  static constexpr size_t RG_BYTES = RGF ? (size_t)TX * TY * sizeof(T) + (NT / 32) * kRgNV * sizeof(double) : 0;
  BD3MG_HD static size_t coef_bytes(int kz) { return ((size_t)kz * KY * KX * sizeof(T) + 127) & ~size_t(127); }
  // bytes conv_tile uses from its 128-byte aligned base
  static size_t layout_bytes(int kz) {
    return coef_bytes(kz) + 2 * NIN * TILE_BYTES + 2 * sizeof(uint64_t) + 8 * (NT / 32) * sizeof(double) + RG_BYTES;
  }
  static size_t smem_bytes(int kz) { return layout_bytes(kz) + 128; }
};

template <typename T>
BD3MG_D int find_job(const ConvArgs<T>& p, int zidx) {
  int j = 0;
  while (j + 1 < p.njobs && p.jobs[j + 1].work_begin <= zidx) ++j;
  return j;
}

// Stage the coefficient set of output plane `zo` (adjoint: gathered) into smem.
template <typename T, bool ADJ>
BD3MG_D void stage_coefs(const ConvGeom<T>& p, int zo, T* cs, int nt) {
  const int KYX = p.ky * p.kx, n = p.kz * KYX;
  const int rz = (p.kz - 1) / 2;
  for (int i = threadIdx.x; i < n; i += nt) {
    if (!ADJ) {
      cs[i] = p.K[(long long)zo * n + i];
    } else {
      const int a = i / KYX, rem = i - a * KYX;
      const int b = rem / p.kx, c = rem - b * p.kx;
      const int zsrc = zo + a - rz;
      T v = T(0);
      if (zsrc >= 0 && zsrc < p.nzk)
        v = p.K[(long long)zsrc * n + (long long)(p.kz - 1 - a) * KYX + (p.ky - 1 - b) * p.kx + (p.kx - 1 - c)];
      cs[i] = v;
    }
  }
}

// Fallback staging when TMA is not usable (row pitch not a multiple of 16
// bytes): element-wise cp.async with zero fill into the same dense layout.
template <typename Cfg, typename T>
BD3MG_D void stage_tile_fallback(T* dst, const T* src, long long src_z0, int zi, int y0, int x0, int ny, int nx,
                                 long long plane) {
  const T* base = src + (long long)(zi - src_z0) * plane;
  for (int idx = threadIdx.x; idx < Cfg::BOX; idx += Cfg::NT) {
    const int row = idx / Cfg::PITCH, e = idx - row * Cfg::PITCH;
    const int gy = y0 - Cfg::RYH + row, gx = x0 - Cfg::RXA + e;
    const bool ok = (gy >= 0) && (gy < ny) && (gx >= 0) && (gx < nx);
    const T* g = ok ? base + (long long)gy * nx + gx : src;
    cp_async<sizeof(T)>(dst + idx, g, ok);
  }
}

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

// One input of a tile: TMA map (box PITCH x BOXH at z = depth - z0) and the
// same fragment for the cp.async fallback.
template <typename T>
struct TileSrc {
  const CUtensorMap* tm;
  const T* src;  // plane 0 = global depth z0 (cp.async fallback)
  long long z0;  // global depth of the fragment's first plane
  int nz;        // planes in the fragment (taps outside read zero)
  long long tz0; // global depth of the TMA map's z = 0 (<= z0; a map may span more rows than the fragment)
};

// Everything one output tile of one output plane reads and writes.
template <typename T>
struct TileIO {
  TileSrc<T> in0, in1;          // in1: second input (M_GRAM2; M_GRAM2P runs it as the first pass)
  T* dst;                       // output plane (row y at dst + y*nx), or null
  const T* sub;                 // epilogue operand plane, same alignment, or null
  const CUtensorMap* tm_epi;    // epilogue operand TMA (TX x TY box at (x0, y0, epi_z)), or null;
                                //   M_GRADF: the iterate map (correlation box, halo origin)
  int epi_z;
  bool use_tma;
  // M_GRADF: iterate fragment (axial neighbours read through L2), outputs
  const T* xf = nullptr;
  long long xf_z0 = 0;
  int xf_nz = 0;
  T* omega = nullptr;           // omega plane (row y at omega + y*nx); M_GRAM2: the block's omega plane zo
                                //   (the tile then adds the regulariser Gram terms, rg_center), or null
  T* snap = nullptr;            // snapshot plane or null
  double* epart = nullptr;      // recorder partials (kEvalNV) or null; M_GRAM2: the tile's kRgNV sums
  bool rg_has_d = false;        // M_GRAM2 + omega: the block has a memory column (in1 is d, not g again)
};

constexpr int kGradfNV = 5;     // recorder sums of M_GRADF: box, tv, axial, |x-snap|^2, |snap|^2

// M_GRADF epilogue: g = H^T r + greg for the thread's RY x RX outputs, with
// greg computed here from the staged iterate tile xt (plane zo, origin
// (x0 - RXA, y0 - RYH), pitch PITCH) exactly as greg_tile computes it
// (stencil_tma.cuh; reference objective.py:130-137, :175-186): omega, the
// weighted differences, their adjoints (left / upper neighbours by a lane
// shuffle, the warp above through shared memory, the tile edges from the
// halo), the box and axial terms (planes zo -+ 1 through L2).  Optionally the
// recorder terms of eval_f and the snapshot roll.
template <typename T, typename Cfg>
BD3MG_D void gradf_epilogue(const ConvGeom<T>& p, const TileIO<T>& io, int zo, int x0, int y0, const T* xt,
                            T (&acc)[Cfg::RY][Cfg::RX], double* red_s, T* scratch) {
  using V = typename Vec16<T>::type;
  constexpr int RX = Cfg::RX, RY = Cfg::RY, RXA = Cfg::RXA, RYH = Cfg::RYH, PITCH = Cfg::PITCH;
  constexpr int TX = Cfg::TX;
  static_assert(RX == Cfg::VEC, "one 16-byte vector per thread row");
  const int tx = threadIdx.x % Cfg::WX, ty = threadIdx.x / Cfg::WX;
  const int lane = threadIdx.x & 31;
  const int nx = p.nx, ny = p.ny;
  const T d2 = (T)p.delta2, two_eta = (T)p.two_eta, lam = (T)p.lam, two_kappa = (T)p.two_kappa;
  const T xmin = (T)p.x_min, xmax = (T)p.x_max;
  auto X = [&](int ly, int lx) { return xt[(ly + RYH) * PITCH + lx + RXA]; };
  // omega / weighted differences at tile-local (ly, lx); zero outside the volume (greg_tile's halo rule)
  auto wxy = [&](int ly, int lx, T& w, T& px, T& py, T& sq) {
    const int y = y0 + ly, x = x0 + lx;
    const T c = X(ly, lx);
    const T dx = (x < nx - 1) ? sub_rn(X(ly, lx + 1), c) : T(0);
    const T dy = (y < ny - 1) ? sub_rn(X(ly + 1, lx), c) : T(0);
    sq = add_rn(add_rn(mul_rn(dx, dx), mul_rn(dy, dy)), d2);
    w = rsqrt(sq);
    px = mul_rn(w, dx);
    py = mul_rn(w, dy);
  };
  auto in_vol = [&](int ly, int lx) {
    const int y = y0 + ly, x = x0 + lx;
    return y >= 0 && x >= 0 && y < ny && x < nx;
  };
  // py of the row above each warp's first row: the warp above's last row (shared memory) or the halo row
  // (scratch: the other ring buffer, free after the tap walk)
  T (*s_lastpy)[TX] = reinterpret_cast<T (*)[TX]>(scratch);
  {
    const int lyl = ty * RY + RY - 1;
#pragma unroll
    for (int i = 0; i < RX; ++i) {
      T w, px, py, sq;
      wxy(lyl, tx * RX + i, w, px, py, sq);
      s_lastpy[ty][tx * RX + i] = py;
    }
  }
  __syncthreads();
  const long long plane = p.plane;
  const bool has_m = zo >= 1, has_p = zo < p.nz_global - 1;
  const T* xm_p = has_m ? io.xf + (long long)(zo - 1 - io.xf_z0) * plane : nullptr;
  const T* xp_p = has_p ? io.xf + (long long)(zo + 1 - io.xf_z0) * plane : nullptr;
  double ev[kGradfNV] = {0.0, 0.0, 0.0, 0.0, 0.0};
  const bool eval = io.epart != nullptr;
  T pym[RX];
#pragma unroll
  for (int i = 0; i < RX; ++i) {
    const int lx = tx * RX + i;
    if (ty > 0) {
      pym[i] = s_lastpy[ty - 1][lx];
    } else {
      T w, px, py, sq;
      py = T(0);
      if (in_vol(-1, lx)) wxy(-1, lx, w, px, py, sq);
      pym[i] = py;
    }
  }
  const int xt0 = x0 + tx * RX;
  const bool vec_row = (nx % RX) == 0 && xt0 + RX <= nx;
#pragma unroll
  for (int r = 0; r < RY; ++r) {
    const int ly = ty * RY + r, y = y0 + ly;
    T w[RX], px[RX], py[RX], sq[RX];
#pragma unroll
    for (int i = 0; i < RX; ++i) wxy(ly, tx * RX + i, w[i], px[i], py[i], sq[i]);
    // left neighbour's weighted x-difference: lane - 1 (every lane shuffles), lane 0 from the halo
    T pxl = __shfl_up_sync(0xffffffffu, px[RX - 1], 1);
    if (lane == 0) {
      T ww, pxx, pyy, sqq;
      pxx = T(0);
      if (in_vol(ly, tx * RX - 1)) wxy(ly, tx * RX - 1, ww, pxx, pyy, sqq);
      pxl = pxx;
    }
    const long long o = (long long)y * nx + xt0;
    T xm[RX], xp[RX], sn[RX];
    if (y < ny) {
      if (vec_row) {
        if (has_m) { const V v = __ldcg(reinterpret_cast<const V*>(xm_p + o)); const T* q = reinterpret_cast<const T*>(&v);
#pragma unroll
          for (int i = 0; i < RX; ++i) xm[i] = q[i]; }
        if (has_p) { const V v = __ldcg(reinterpret_cast<const V*>(xp_p + o)); const T* q = reinterpret_cast<const T*>(&v);
#pragma unroll
          for (int i = 0; i < RX; ++i) xp[i] = q[i]; }
        if (eval && io.snap) { const V v = __ldcg(reinterpret_cast<const V*>(io.snap + o)); const T* q = reinterpret_cast<const T*>(&v);
#pragma unroll
          for (int i = 0; i < RX; ++i) sn[i] = q[i]; }
      } else {
#pragma unroll
        for (int i = 0; i < RX; ++i) {
          const bool in = xt0 + i < nx;
          xm[i] = (has_m && in) ? __ldcg(xm_p + o + i) : T(0);
          xp[i] = (has_p && in) ? __ldcg(xp_p + o + i) : T(0);
          sn[i] = (eval && io.snap && in) ? __ldcg(io.snap + o + i) : T(0);
        }
      }
    }
    T gout[RX], wout[RX], xout[RX];
#pragma unroll
    for (int i = 0; i < RX; ++i) {
      const int lx = tx * RX + i, x = x0 + lx;
      const T pxm = (i > 0) ? px[i - 1] : pxl;
      const T xc = X(ly, lx);
      const T clipped = xc < xmin ? xmin : (xc > xmax ? xmax : xc);
      const T box = mul_rn(two_eta, sub_rn(xc, clipped));
      const T tvx = (nx == 1) ? T(0) : sub_rn(pxm, px[i]);
      const T tvy = (ny == 1) ? T(0) : sub_rn(pym[i], py[i]);
      const T xzp = has_p ? xp[i] : T(0);
      const T dzm = has_m ? sub_rn(xc, xm[i]) : T(0);
      const T dzp = has_p ? sub_rn(xzp, xc) : T(0);
      const T greg = add_rn(add_rn(box, mul_rn(lam, add_rn(tvx, tvy))), mul_rn(two_kappa, sub_rn(dzm, dzp)));
      gout[i] = add_rn(acc[r][i], greg);
      wout[i] = w[i];
      xout[i] = xc;
      if (eval && y < ny && x < nx) {
        const double e = (double)xc - (double)clipped;
        ev[0] += e * e;
        ev[1] += (double)sq[i] * (double)w[i];
        if (has_p) ev[2] += ((double)xzp - (double)xc) * ((double)xzp - (double)xc);
        if (io.snap) {
          ev[3] += ((double)xc - (double)sn[i]) * ((double)xc - (double)sn[i]);
          ev[4] += (double)sn[i] * (double)sn[i];
        }
      }
      pym[i] = py[i];
    }
    if (y < ny) {
      if (vec_row) {
        *reinterpret_cast<V*>(io.dst + o) = *reinterpret_cast<const V*>(gout);
        *reinterpret_cast<V*>(io.omega + o) = *reinterpret_cast<const V*>(wout);
        if (eval && io.snap) *reinterpret_cast<V*>(io.snap + o) = *reinterpret_cast<const V*>(xout);
      } else {
#pragma unroll
        for (int i = 0; i < RX; ++i)
          if (xt0 + i < nx) {
            io.dst[o + i] = gout[i];
            io.omega[o + i] = wout[i];
            if (eval && io.snap) io.snap[o + i] = xout[i];
          }
      }
    }
  }
  if (eval) {
    cta_reduce<kGradfNV, Cfg::NT>(ev, red_s);
    if (threadIdx.x == 0) {
#pragma unroll
      for (int k = 0; k < kGradfNV; ++k) io.epart[k] = ev[k];
    }
  }
}

// Regulariser Gram terms of one block plane, computed by the dual-input Gram
// tile whose output plane zo lies inside the block [blo, bhi].  Such a tile
// starts its tap walk at the centre tap, so the first two staged planes are
// plane zo (g0, d0) and, when zo < bhi, plane zo + 1 (g1, d1) of g and d: they
// hold every neighbour the forward differences need; omega comes from the
// tile's cp.async-staged copy `ws` (TX x TY).  Term by term this is
// reg_gram_tile (stencil_tma.cuh; reference objective.py:262-274,
// directions.py:80-85) for the columns [-g, d] embedded on the block:
// v[0..2] column norms, [3..5] omega-weighted TV terms, [6..8] axial terms,
// [9] g.d, [10] nonzeros of g, [11] non-finite entries of g; the CTA's sums go
// to part_out (thread 0).  Out-of-volume pixels of the staged tiles and of
// the omega tile are zero, so they add nothing; only the far-face rules of the
// differences need masks.  Every FP64 instruction here competes with the
// correlation for the FP64 pipe, so the flags are counted on the integer pipe.
// The row loop is kept rolled: ptxas budgets the kernel's uniform registers
// over all of its code, and the tap walk needs them for its coefficients (DFMA
// with a uniform operand; with the coefficients in vector registers the walk
// runs 15% slower -- measured).
#ifndef BD3MG_RG_UNROLL
#define BD3MG_RG_UNROLL 1  // rows of rg_center's loop unrolled together (code size vs latency hiding, see below)
#endif
constexpr int kRgUnroll = BD3MG_RG_UNROLL;
template <typename T, typename Cfg>
__device__ __noinline__ void rg_center(int nx, int ny, int nz_global, int zo, int x0, int y0, int blo, int bhi,
                                       bool has_d, const T* g0, const T* d0, const T* g1, const T* d1, const T* ws,
                                       double* red, double* part_out) {
  using V = typename Vec16<T>::type;
  constexpr int RX = Cfg::RX, RY = Cfg::RY, PITCH = Cfg::PITCH;
  static_assert(RX == 2 && sizeof(T) == 8, "fp64 tile: one 16-byte vector per thread row");
  const int tx = threadIdx.x % Cfg::WX, ty = threadIdx.x / Cfg::WX;
  const int xa = x0 + tx * RX;                     // the thread's two columns xa, xa + 1
  const bool mx0 = xa < nx - 1, mx1 = xa + 1 < nx - 1;
  const int q0 = (ty * RY + Cfg::RYH) * PITCH + tx * RX + Cfg::RXA;
  const bool next = zo < bhi, far = !next && bhi < nz_global - 1, first = zo == blo && blo >= 1;
  double v[9];
#pragma unroll
  for (int k = 0; k < 9; ++k) v[k] = 0.0;
  int nnz = 0, nnf = 0;
  // row r of the thread: columns xa, xa + 1 and the right neighbour xa + 2
  T gc[3], dc[3];
  {
    const V a = *reinterpret_cast<const V*>(g0 + q0);
    gc[0] = a.x; gc[1] = a.y; gc[2] = g0[q0 + 2];
    dc[0] = dc[1] = dc[2] = T(0);
    if (has_d) {
      const V b = *reinterpret_cast<const V*>(d0 + q0);
      dc[0] = b.x; dc[1] = b.y; dc[2] = d0[q0 + 2];
    }
  }
#pragma unroll kRgUnroll
  for (int r = 0; r < RY; ++r) {
    const int ly = ty * RY + r, y = y0 + ly;
    const bool my = y < ny - 1;
    const int q = q0 + (r + 1) * PITCH;
    T gn[3], dn[3];  // the row below
    {
      const V a = *reinterpret_cast<const V*>(g0 + q);
      gn[0] = a.x; gn[1] = a.y; gn[2] = g0[q + 2];
      dn[0] = dn[1] = dn[2] = T(0);
      if (has_d) {
        const V b = *reinterpret_cast<const V*>(d0 + q);
        dn[0] = b.x; dn[1] = b.y; dn[2] = d0[q + 2];
      }
    }
    const V wv = *reinterpret_cast<const V*>(ws + ly * Cfg::TX + tx * RX);
    V g1v = {T(0), T(0)}, d1v = {T(0), T(0)};
    if (next) {
      g1v = *reinterpret_cast<const V*>(g1 + q - PITCH);
      if (has_d) d1v = *reinterpret_cast<const V*>(d1 + q - PITCH);
    }
#pragma unroll
    for (int i = 0; i < RX; ++i) {
      const T g = gc[i], d = dc[i];
      const double w = i == 0 ? wv.x : wv.y;
      const bool mx = i == 0 ? mx0 : mx1;
      // columns b0 = -g, b1 = d
      v[0] += g * g;
      v[1] -= g * d;
      v[2] += d * d;
      const double dx0 = mx ? sub_rn(g, gc[i + 1]) : 0.0;   // -(g[x+1] - g)
      const double dy0 = my ? sub_rn(g, gn[i]) : 0.0;
      const double dx1 = mx ? sub_rn(dc[i + 1], d) : 0.0;
      const double dy1 = my ? sub_rn(dn[i], d) : 0.0;
      v[3] += w * (dx0 * dx0 + dy0 * dy0);
      v[4] += w * (dx0 * dx1 + dy0 * dy1);
      v[5] += w * (dx1 * dx1 + dy1 * dy1);
      // axial row zo of the block-embedded vectors
      double z0v = 0.0, z1v = 0.0;
      if (next) {
        z0v = g - (i == 0 ? g1v.x : g1v.y);
        z1v = (i == 0 ? d1v.x : d1v.y) - d;
      } else if (far) {
        z0v = g;      // -b0
        z1v = -d;     // -b1
      }
      v[6] += z0v * z0v;
      v[7] += z0v * z1v;
      v[8] += z1v * z1v;
      // flags on the integer pipe: g != 0 (either zero sign), g non-finite (exponent all ones)
      const unsigned hi = (unsigned)__double2hiint(g) & 0x7fffffffu, lo = (unsigned)__double2loint(g);
      nnz += (hi | lo) != 0u;
      nnf += hi >= 0x7ff00000u;
    }
#pragma unroll
    for (int k = 0; k < 3; ++k) { gc[k] = gn[k]; dc[k] = dn[k]; }
  }
  double o[kRgNV];
#pragma unroll
  for (int k = 0; k < 9; ++k) o[k] = v[k];
  if (first) { o[6] += v[0]; o[7] += v[1]; o[8] += v[2]; }  // the row above the block: (b - 0)^2
  o[9] = -v[1];  // g.d: every product is the exact negation of (-g).d
  o[10] = (double)nnz;
  o[11] = (double)nnf;
  cta_reduce<kRgNV, Cfg::NT>(o, red);
  if (threadIdx.x == 0 && part_out) {
#pragma unroll
    for (int k = 0; k < kRgNV; ++k) part_out[k] = o[k];
  }
}

// One TY x TX output tile of output plane zo: the kz-tap walk over the staged
// input planes (double-buffered TMA ring, mbarrier completion), the register-
// tiled FMA loop, and the mode's epilogue; `part` receives the CTA's NV
// partial sums (thread 0).  `sbase` is the 128-byte aligned shared memory of
// ConvCfg::smem_bytes.  Shared by conv_tiled_kernel (one tile per CTA) and
// the persistent sweep kernel (sweep_pk.cuh: many tiles per CTA), so both
// compute bit-identical values.
template <typename T, int KY, int KX, int MODE, bool ADJ, int RYO = 0>
BD3MG_D void conv_tile(const ConvGeom<T>& p, const TileIO<T>& io, int zo, int x0, int y0, double* part_out,
                       unsigned char* sbase, uint64_t* bars = nullptr) {
  using Cfg = ConvCfg<T, KY, KX, MODE, RYO>;
  using V = typename Vec16<T>::type;
  constexpr int RX = Cfg::RX, RY = Cfg::RY, NIN = Cfg::NIN, VEC = Cfg::VEC;
  constexpr int WINP = Cfg::WINP, OFF = Cfg::OFF;
  constexpr int RYH = Cfg::RYH, RXA = Cfg::RXA;
  constexpr bool TWOPASS = Cfg::TWOPASS;
  // 128-byte aligned carve-out: [tiles][coefs][mbarriers][reduction scratch]
  T* tiles = reinterpret_cast<T*>(sbase);
  T* coef_s = reinterpret_cast<T*>(sbase + 2 * NIN * Cfg::TILE_BYTES);
  uint64_t* mbar_l = reinterpret_cast<uint64_t*>(sbase + 2 * NIN * Cfg::TILE_BYTES + Cfg::coef_bytes(p.kz));
  double* red_s = reinterpret_cast<double*>(mbar_l + 2);
  uint64_t* mbar = bars ? bars : mbar_l;  // persistent kernel: barriers at a fixed location
  // fused regulariser Gram (fp64 dual-input tile whose output plane lies inside the block)
  constexpr bool kRgf = Cfg::RGF && MODE == M_GRAM2;
  const bool rg_here = kRgf && io.omega != nullptr;

  const int tx = threadIdx.x % Cfg::WX, ty = threadIdx.x / Cfg::WX;
  const int rz = (p.kz - 1) / 2;
  const bool tma = io.use_tma;

  // taps a whose input plane zo+a-rz lies inside the fragment
  const long long zlo_in = io.in0.z0, zhi_in = io.in0.z0 + io.in0.nz - 1;
  const int a_lo = (int)max(0LL, zlo_in - zo + rz);
  const int a_hi = (int)min((long long)p.kz - 1, zhi_in - zo + rz);
  const int ntap = a_hi - a_lo + 1;
  // A tile that also computes the regulariser Gram terms walks its taps so that the centre comes last:
  // a_lo .. rz - 1 upwards, then a_hi .. rz downwards.  The two ring buffers then still hold planes
  // zo + 1 and zo of g and d when the walk ends -- every neighbour those terms need -- and the extra work
  // sits behind the walk (rg_center, called from the epilogue), not inside it.  (The order only regroups
  // the roundings of sums that feed the 2 x 2 Gram; every batching of a block uses the same order.)
  const int n_lo = rg_here ? rz - a_lo : ntap;
  auto tap_of = [&](int step) { return step < n_lo ? a_lo + step : a_hi - (step - n_lo); };
  // steps of the walk: the taps (two-pass Gram: the taps over input 1, then over input 0)
  const int nstep = TWOPASS ? 2 * ntap : ntap;

  if (tma && threadIdx.x == 0) {
    tma_prefetch_desc(io.in0.tm);  // the descriptor fetch overlaps the barrier set-up
    if constexpr (NIN == 2 || TWOPASS) tma_prefetch_desc(io.in1.tm);
    mbar_init(&mbar[0], 1);
    mbar_init(&mbar[1], 1);
    fence_mbar_init();
  }

  auto issue = [&](int step, int b) {
    T* dst = tiles + b * NIN * Cfg::TILE;
    const bool second = TWOPASS && step < ntap;  // pass 0 of the two-pass Gram reads input 1
    const int a = kRgf ? tap_of(step) : a_lo + (TWOPASS && step >= ntap ? step - ntap : step);
    const int zi = zo + a - rz;
    const TileSrc<T>& in = second ? io.in1 : io.in0;
    if (tma) {
      if (threadIdx.x == 0) {
        mbar_expect_tx(&mbar[b], (uint32_t)(NIN * Cfg::BOX_BYTES));
        tma_load_3d(dst, in.tm, x0 - RXA, y0 - RYH, (int)(zi - in.tz0), &mbar[b]);
        if constexpr (NIN == 2)
          tma_load_3d(dst + Cfg::TILE, io.in1.tm, x0 - RXA, y0 - RYH, (int)(zi - io.in1.tz0), &mbar[b]);
      }
    } else {
      stage_tile_fallback<Cfg>(dst, in.src, in.z0, zi, y0, x0, p.ny, p.nx, p.plane);
      if constexpr (NIN == 2)
        stage_tile_fallback<Cfg>(dst + Cfg::TILE, io.in1.src, io.in1.z0, zi, y0, x0, p.ny, p.nx, p.plane);
      cp_async_commit();
    }
  };

  // One tile per CTA (no barriers handed in): the first plane's TMA load is issued before the
  // coefficients are staged, so its latency overlaps their global loads and the barrier below.
  // (The persistent kernel's tiles follow one another in a CTA: its previous tile's epilogue may
  // still read the ring, so there the load waits for the barrier.)
  const bool early = BD3MG_EARLY_ISSUE && tma && bars == nullptr && nstep > 0;
  if (early) issue(0, 0);
  stage_coefs<T, ADJ>(p, zo, coef_s, Cfg::NT);
  __syncthreads();

  T acc[NIN][RY][RX];
#pragma unroll
  for (int s = 0; s < NIN; ++s)
#pragma unroll
    for (int r = 0; r < RY; ++r)
#pragma unroll
      for (int i = 0; i < RX; ++i) acc[s][r][i] = T(0);
  T accp[TWOPASS ? RY : 1][RX];  // two-pass Gram: input 1's sums, parked after pass 0
#pragma unroll
  for (int r = 0; r < (TWOPASS ? RY : 1); ++r)
#pragma unroll
    for (int i = 0; i < RX; ++i) accp[r][i] = T(0);

  if constexpr (kRgf) {
    if (rg_here) {  // each thread stages its own omega values (RY rows x 16 bytes)
      T* rg_w = reinterpret_cast<T*>(red_s + 8 * (Cfg::NT / 32));  // omega tile, TX x TY
      const int xw = x0 + tx * RX;
#pragma unroll 1
      for (int r = 0; r < RY; ++r) {
        const int ly = ty * RY + r, y = y0 + ly;
        const bool ok = y < p.ny && xw + RX <= p.nx;
        cp_async<16>(rg_w + ly * Cfg::TX + tx * RX, ok ? io.omega + (long long)y * p.nx + xw : io.omega, ok);
      }
      cp_async_commit();
    }
  }
  if (nstep > 0 && !early) issue(0, 0);
  // the epilogue operand rows of this tile are pulled into L2 two taps before
  // the end, so the epilogue's loads do not wait on DRAM
  constexpr bool kEpiLoad = MODE == M_RESID || MODE == M_GRAD || MODE == M_GRAMC;
  const bool vec_io = (p.nx % VEC) == 0;  // rows are whole 16-byte chunks
  const int s_pf = max(0, nstep - 2);
  // RESID / GRAD: the epilogue operand tile (y rows or the regulariser
  // gradient) is loaded by TMA into the tile buffer the last tap plane frees,
  // while that plane computes; the epilogue then reads it from shared memory
  constexpr bool kEpiTma =
      (MODE == M_RESID || MODE == M_GRAD || MODE == M_GRAMC || MODE == M_GRADF) && NIN == 1 && sizeof(T) == 8;
  const bool epi_tma = kEpiTma && tma && io.tm_epi != nullptr && (nstep > 0 || MODE == M_GRADF);
  if (MODE == M_GRADF && nstep == 0 && epi_tma && threadIdx.x == 0) {  // no tap in range: stage the iterate now
    mbar_expect_tx(&mbar[1], (uint32_t)Cfg::BOX_BYTES);
    tma_load_3d(tiles + 1 * NIN * Cfg::TILE, io.tm_epi, x0 - RXA, y0 - RYH, io.epi_z, &mbar[1]);
  }
  uint32_t phase = 0;  // bit b = parity of buffer b
  int buf = 0;
  for (int st = 0; st < nstep; ++st) {
    if (st < nstep - 1) {
      issue(st + 1, buf ^ 1);
    } else if (epi_tma && threadIdx.x == 0) {
      if constexpr (MODE == M_GRADF) {  // the iterate plane zo with its halo (same box as the taps)
        mbar_expect_tx(&mbar[buf ^ 1], (uint32_t)Cfg::BOX_BYTES);
        tma_load_3d(tiles + (buf ^ 1) * NIN * Cfg::TILE, io.tm_epi, x0 - RXA, y0 - RYH, io.epi_z, &mbar[buf ^ 1]);
      } else {
        mbar_expect_tx(&mbar[buf ^ 1], (uint32_t)(Cfg::TX * Cfg::TY * sizeof(T)));
        tma_load_3d(tiles + (buf ^ 1) * NIN * Cfg::TILE, io.tm_epi, x0, y0, io.epi_z, &mbar[buf ^ 1]);
      }
    }
    if constexpr (kEpiLoad) {
      if (st == s_pf && vec_io && io.sub && threadIdx.x < Cfg::TY) {
        const int y = y0 + threadIdx.x, w = min(Cfg::TX, p.nx - x0);
        if (y < p.ny && w > 0) prefetch_l2_bulk(io.sub + (long long)y * p.nx + x0, (uint32_t)(w * sizeof(T)));
      }
    }
    if constexpr (TWOPASS) {
      if (st == ntap) {  // pass 0 (input 1) done: park its sums, restart for input 0
#pragma unroll
        for (int r = 0; r < RY; ++r)
#pragma unroll
          for (int i = 0; i < RX; ++i) {
            accp[r][i] = acc[0][r][i];
            acc[0][r][i] = T(0);
          }
      }
    }
    if (tma) {
      mbar_wait(&mbar[buf], (phase >> buf) & 1u);
      phase ^= 1u << buf;
    } else {
      if (st < nstep - 1) cp_async_wait<1>();
      else cp_async_wait<0>();
      __syncthreads();
    }
    const int a = kRgf ? tap_of(st) : a_lo + (TWOPASS && st >= ntap ? st - ntap : st);
    const T* cs = coef_s + a * (KY * KX);
    const T* tb = tiles + buf * NIN * Cfg::TILE + (ty * RY) * Cfg::PITCH + tx * RX;
#pragma unroll
    for (int yi = 0; yi < RY + KY - 1; ++yi) {
      T v[NIN][WINP];
#pragma unroll
      for (int s = 0; s < NIN; ++s)
#pragma unroll
        for (int j = 0; j < WINP; j += VEC) {
          const V q = *reinterpret_cast<const V*>(tb + s * Cfg::TILE + yi * Cfg::PITCH + j);
          if constexpr (VEC == 2) {
            v[s][j] = q.x; v[s][j + 1] = q.y;
          } else {
            v[s][j] = q.x; v[s][j + 1] = q.y; v[s][j + 2] = q.z; v[s][j + 3] = q.w;
          }
        }
      // c outer, rows inner: consecutive FMAs update different accumulators
      // (latency hiding); per output the order is still a -> b -> c.
#pragma unroll
      for (int c = 0; c < KX; ++c) {
#pragma unroll
        for (int r = 0; r < RY; ++r) {
          const int b = yi - r;
          if (b < 0 || b >= KY) continue;
          const T k = cs[b * KX + c];
#pragma unroll
          for (int s = 0; s < NIN; ++s)
#pragma unroll
            for (int i = 0; i < RX; ++i) acc[s][r][i] = fma_rn(k, v[s][OFF + i + c], acc[s][r][i]);
        }
      }
    }
    __syncthreads();
    buf ^= 1;
  }

  // ---- epilogue -----------------------------------------------------------
  const T* etile = tiles + buf * NIN * Cfg::TILE;  // the buffer the last plane left free
  if (epi_tma) mbar_wait(&mbar[buf], (phase >> buf) & 1u);
  if constexpr (MODE == M_GRADF) {
    gradf_epilogue<T, Cfg>(p, io, zo, x0, y0, etile, acc[0], red_s, tiles + (buf ^ 1) * NIN * Cfg::TILE);
    return;
  }
  constexpr int NV = Cfg::NV;
  double part[NV > 0 ? NV : 1];
#pragma unroll
  for (int k = 0; k < (NV > 0 ? NV : 1); ++k) part[k] = 0.0;
  const int xt = x0 + tx * RX;
  // 16-byte loads / stores of the thread's RX outputs where the row allows
  constexpr bool kVecEpi = RX == VEC && (MODE == M_STORE || MODE == M_RESID || MODE == M_GRAD || MODE == M_GRAMC);
  const bool vec_here = kVecEpi && vec_io && xt + RX <= p.nx;
  if constexpr (kVecEpi) {
    if (vec_here) {
#pragma unroll
      for (int r = 0; r < RY; ++r) {
        const int y = y0 + ty * RY + r;
        if (y >= p.ny) continue;
        const long long o = (long long)y * p.nx + xt;
        T res[RX];
        if constexpr (MODE == M_STORE) {
#pragma unroll
          for (int i = 0; i < RX; ++i) res[i] = acc[0][r][i];
        } else {
          const V q = epi_tma ? *reinterpret_cast<const V*>(etile + (ty * RY + r) * Cfg::TX + tx * RX)
                              : *reinterpret_cast<const V*>(io.sub + o);
          const T* qs = reinterpret_cast<const T*>(&q);
#pragma unroll
          for (int i = 0; i < RX; ++i) {
            if constexpr (MODE == M_RESID) {
              res[i] = sub_rn(acc[0][r][i], qs[i]);
              part[0] += (double)res[i] * (double)res[i];
            } else if constexpr (MODE == M_GRAMC) {  // H E_S g out; Gram with the cached H E_S d
              const double a0 = (double)acc[0][r][i], c0 = (double)qs[i];
              res[i] = acc[0][r][i];
              part[0] += a0 * a0;
              part[1] += a0 * c0;
              part[2] += c0 * c0;
            } else {
              res[i] = add_rn(acc[0][r][i], qs[i]);
            }
          }
        }
        if (MODE != M_RESID || io.dst) *reinterpret_cast<V*>(io.dst + o) = *reinterpret_cast<const V*>(res);
      }
    }
  }
  if (!vec_here) {
#pragma unroll
  for (int r = 0; r < RY; ++r) {
    const int y = y0 + ty * RY + r;
    if (y >= p.ny) continue;
#pragma unroll
    for (int i = 0; i < RX; ++i) {
      const int x = x0 + tx * RX + i;
      if (x >= p.nx) continue;
      const long long o = (long long)y * p.nx + x;
      const T a0 = acc[0][r][i];
      if constexpr (MODE == M_STORE) {
        io.dst[o] = a0;
      } else if constexpr (MODE == M_RESID) {
        const T res = sub_rn(a0, io.sub[o]);
        if (io.dst) io.dst[o] = res;
        part[0] += (double)res * (double)res;
      } else if constexpr (MODE == M_GRAD) {
        io.dst[o] = add_rn(a0, io.sub[o]);
      } else if constexpr (MODE == M_GRAM1) {
        if (io.dst) io.dst[o] = a0;
        part[0] += (double)a0 * (double)a0;
      } else if constexpr (MODE == M_GRAM2 || MODE == M_GRAM2P) {
        const T a1 = TWOPASS ? accp[TWOPASS ? r : 0][i] : acc[NIN - 1][r][i];
        part[0] += (double)a0 * (double)a0;
        part[1] += (double)a0 * (double)a1;
        part[2] += (double)a1 * (double)a1;
      } else if constexpr (MODE == M_GRAMC) {
        const double c0 = (double)io.sub[o];
        io.dst[o] = a0;
        part[0] += (double)a0 * (double)a0;
        part[1] += (double)a0 * c0;
        part[2] += c0 * c0;
      }
    }
  }
  }  // !vec_here
  if constexpr (kRgf) {
    // (after the Gram products above: only the three partial sums stay live across the call)
    if (rg_here) {
      const T* t0 = tiles + (buf ^ 1) * NIN * Cfg::TILE;  // the last step: the centre plane zo
      const T* t1 = tiles + buf * NIN * Cfg::TILE;        // the step before: plane zo + 1 (when zo < bhi)
      cp_async_wait<0>();                                 // the omega tile
      T* rg_w = reinterpret_cast<T*>(red_s + 8 * (Cfg::NT / 32));
#ifndef BD3MG_EXP_RGF_NOCALL
      rg_center<T, Cfg>(p.nx, p.ny, p.nz_global, zo, x0, y0, (int)zlo_in, (int)zhi_in, io.rg_has_d, t0,
                        t0 + Cfg::TILE, t1, t1 + Cfg::TILE, rg_w, reinterpret_cast<double*>(rg_w + Cfg::TX * Cfg::TY),
                        io.epart);
#endif
    }
  }
  if constexpr (NV > 0) {
    cta_reduce<NV, Cfg::NT>(part, red_s);
    if (threadIdx.x == 0 && part_out) {
#pragma unroll
      for (int k = 0; k < NV; ++k) part_out[k] = part[k];
    }
  }
}

template <typename T, int KY, int KX, int MODE, bool ADJ>
__global__ void __launch_bounds__(ConvCfg<T, KY, KX, MODE>::NT)
    conv_tiled_kernel(const __grid_constant__ ConvArgs<T> p) {
  using Cfg = ConvCfg<T, KY, KX, MODE>;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  unsigned char* sbase = smem_raw + ((128u - (smem_u32(smem_raw) & 127u)) & 127u);  // stays in .shared
  if (p.gate && *p.gate != 0.0) return;
  const CtaPos pos = cta_pos(p.raster_group);
  const int zidx = pos.z;
  const ConvJob<T>& job = p.jobs[find_job(p, zidx)];
  const int zo = job.out_lo + (zidx - job.work_begin);
  const long long orow = (long long)(zo - job.out_lo) * p.plane;
  TileIO<T> io;
  io.in0 = {&job.tmap0, job.src0, job.src_z0, job.src_nz, job.src_z0};
  io.in1 = {&job.tmap1, job.src1, job.src_z0, job.src_nz, job.src_z0};
  io.dst = job.dst0 ? job.dst0 + orow : nullptr;
  io.sub = job.sub ? job.sub + orow : nullptr;
  io.tm_epi = job.epi_tma ? &job.tmap1 : nullptr;
  io.epi_z = zo - job.out_lo;
  io.use_tma = job.use_tma != 0;
  io.xf = nullptr; io.xf_z0 = 0; io.xf_nz = 0; io.omega = nullptr; io.snap = nullptr; io.epart = nullptr;
  if constexpr (MODE == M_GRADF) {
    io.epi_z = (int)(zo - job.xg_z0);  // the iterate map (tmap1) spans the fragment xg
    io.xf = job.xg; io.xf_z0 = job.xg_z0; io.xf_nz = job.xg_nz;
    io.omega = job.omega + orow;
    io.snap = job.snap ? job.snap + orow : nullptr;
    io.epart = job.eparts ? job.eparts + pos.cta * kGradfNV : nullptr;
  }
  if constexpr (MODE == M_GRAM2 && Cfg::RGF) {
    // the block's regulariser Gram terms ride on the tiles whose output plane lies inside the block
    if (job.omega && zo >= job.src_z0 && zo < job.src_z0 + job.src_nz) {
      const long long brow = zo - job.src_z0;
      io.omega = job.omega + brow * p.plane;
      io.epart = job.eparts + (brow * ((long long)gridDim.x * gridDim.y) + (long long)pos.ty * gridDim.x + pos.tx) * kRgNV;
      io.rg_has_d = job.src1 != job.src0;
    }
  }
  constexpr int NV = Cfg::NV;
  conv_tile<T, KY, KX, MODE, ADJ>(p, io, zo, pos.tx * Cfg::TX, pos.ty * Cfg::TY,
                                  NV > 0 ? p.partials + pos.cta * NV : nullptr, sbase);
}


// ---------------------------------------------------------------------------
// Two output planes per CTA (single-input modes).  Each staged input plane
// zi feeds output zo0 with tap a0 = zi-zo0+rz and output zo0+1 with tap
// a0-1, so every TMA tile / barrier serves two outputs and each thread keeps
// 2 x RY x RX independent accumulators.  Per output the taps are still
// visited in ascending a (then b, c): results are bitwise those of the
// one-plane kernel.  The two coefficient slices of the current plane are
// double-buffered in smem next to the tiles (zero where a tap is invalid).
template <typename T, int KY_, int KX_, int MODE>
struct Rz2Cfg {
  static constexpr int KY = KY_, KX = KX_;
  static constexpr int VEC = 16 / sizeof(T);
  // rows per thread: measured on B200 (scripts/prof_h_cfg.py, scripts/cmp_h.sh)
  // -- 4 (BD3MG_RZ2_RY5) for 3x3 / 5x5 taps, 4 for 7x7 / 9x9
  static constexpr int RX = VEC, RY = (KY <= 5) ? BD3MG_RZ2_RY5 : 4, RZ = 2;
  static constexpr int WX = 32, WY = 4, NT = WX * WY;
  static constexpr int TX = WX * RX, TY = WY * RY;
  static constexpr int RXH = (KX - 1) / 2, RYH = (KY - 1) / 2;
  static constexpr int RXA = (RXH + VEC - 1) / VEC * VEC, OFF = RXA - RXH;
  static constexpr int TXH = TX + KX - 1 + OFF, TYH = TY + KY - 1;
  static constexpr int PITCH = (TXH + 2 * VEC - 1) / (2 * VEC) * (2 * VEC);
  static constexpr int ROWQ = 128 / cgcd(PITCH * (int)sizeof(T), 128);
  static constexpr int BOXH = (TYH + ROWQ - 1) / ROWQ * ROWQ;
  static constexpr int WIN = RX + KX - 1;
  static constexpr int WINP = (OFF + WIN + VEC - 1) / VEC * VEC;
  static constexpr int BOX = BOXH * PITCH;
  static constexpr int TILE = (BOX + 128 / (int)sizeof(T) - 1) / (128 / (int)sizeof(T)) * (128 / (int)sizeof(T));
  static constexpr size_t TILE_BYTES = (size_t)TILE * sizeof(T), BOX_BYTES = (size_t)BOX * sizeof(T);
  static constexpr int NIN = (MODE == M_GRAM2) ? 2 : 1;  // dual input: fp32 packed path only
  static constexpr int NV = ModeNV<MODE>::value;
  static constexpr int KS = KY * KX;                       // one tap slice
  static constexpr size_t SLICE_BYTES = ((size_t)2 * 2 * KS * sizeof(T) + 127) & ~size_t(127);
  // RESID / GRAD / GRAMC: the epilogue operand tiles of both output planes
  // (2 x TX x TY) are TMA-staged into the ring buffer the last input plane
  // frees, so each buffer holds at least that much
  static constexpr bool EPI_T = (MODE == M_RESID || MODE == M_GRAD || MODE == M_GRAMC) && NIN == 1;
  static constexpr int EPI = 2 * TX * TY;
  static constexpr int BUF = (EPI_T && EPI > NIN * TILE) ? EPI : NIN * TILE;  // elements per ring buffer
  static constexpr size_t BUF_BYTES = (size_t)BUF * sizeof(T);
  static size_t smem_bytes(int) {
    return 2 * BUF_BYTES + SLICE_BYTES + 2 * sizeof(uint64_t) + 8 * (NT / 32) * sizeof(double) + 128;
  }
};

template <typename T>
BD3MG_D bool tap_ok(const ConvGeom<T>& p, bool adj, int zo, int a) {
  if (a < 0 || a >= p.kz) return false;
  if (!adj) return true;
  const int zsrc = zo + a - (p.kz - 1) / 2;
  return zsrc >= 0 && zsrc < p.nzk;
}

// coefficient (b, c) of tap a for output plane zo (adjoint: gathered, flipped)
template <typename T, bool ADJ>
BD3MG_D T coef_of(const ConvGeom<T>& p, int zo, int a, int b, int c) {
  const int KYX = p.ky * p.kx, K3 = p.kz * KYX;
  if (!ADJ) return p.K[(long long)zo * K3 + a * KYX + b * p.kx + c];
  const int zsrc = zo + a - (p.kz - 1) / 2;
  return p.K[(long long)zsrc * K3 + (p.kz - 1 - a) * KYX + (p.ky - 1 - b) * p.kx + (p.kx - 1 - c)];
}

template <typename Cfg, typename T, bool D0, bool D1>
BD3MG_D void rz2_plane(const T* tb, const T* cs0, const T* cs1, T (&acc)[2][Cfg::RY][Cfg::RX]) {
  using V = typename Vec16<T>::type;
  constexpr int RX = Cfg::RX, RY = Cfg::RY, VEC = Cfg::VEC, KX = Cfg::KX, KY = Cfg::KY;
#pragma unroll
  for (int yi = 0; yi < RY + KY - 1; ++yi) {
    T v[Cfg::WINP];
#pragma unroll
    for (int j = 0; j < Cfg::WINP; j += VEC) {
      const V q = *reinterpret_cast<const V*>(tb + yi * Cfg::PITCH + j);
      if constexpr (VEC == 2) {
        v[j] = q.x; v[j + 1] = q.y;
      } else {
        v[j] = q.x; v[j + 1] = q.y; v[j + 2] = q.z; v[j + 3] = q.w;
      }
    }
#pragma unroll
    for (int c = 0; c < KX; ++c) {
#pragma unroll
      for (int r = 0; r < RY; ++r) {
        const int b = yi - r;
        if (b < 0 || b >= KY) continue;
        if constexpr (D0) {
          const T k = cs0[b * KX + c];
#pragma unroll
          for (int i = 0; i < RX; ++i) acc[0][r][i] = fma_rn(k, v[Cfg::OFF + i + c], acc[0][r][i]);
        }
        if constexpr (D1) {
          const T k = cs1[b * KX + c];
#pragma unroll
          for (int i = 0; i < RX; ++i) acc[1][r][i] = fma_rn(k, v[Cfg::OFF + i + c], acc[1][r][i]);
        }
      }
    }
  }
}

// fp32 twin of rz2_plane with the two output planes packed into one FFMA2
// lane pair: acc[r][i] = (plane zo0, plane zo0+1) of output (r, i).  The
// input value is broadcast to both lanes and the coefficient pair (k0, k1) is
// one aligned 64-bit load from the interleaved slices, so no register moves
// are needed; each lane is the fmaf_rn of rz2_plane, bit for bit.
// With two inputs (Gram mode) both share the coefficient pair:
// acc[s][r][i] is input s's (plane zo0, plane zo0+1) pair.
template <typename Cfg>
BD3MG_D void rz2_plane_pp(const float* tb, const unsigned long long* cp,
                          unsigned long long (&acc)[Cfg::NIN][Cfg::RY][Cfg::RX]) {
  constexpr int RX = Cfg::RX, RY = Cfg::RY, KX = Cfg::KX, KY = Cfg::KY, NIN = Cfg::NIN;
#pragma unroll
  for (int yi = 0; yi < RY + KY - 1; ++yi) {
    float v[NIN][Cfg::WINP];
#pragma unroll
    for (int s = 0; s < NIN; ++s)
#pragma unroll
      for (int j = 0; j < Cfg::WINP; j += 4) {
        const float4 q = *reinterpret_cast<const float4*>(tb + s * Cfg::TILE + yi * Cfg::PITCH + j);
        v[s][j] = q.x; v[s][j + 1] = q.y; v[s][j + 2] = q.z; v[s][j + 3] = q.w;
      }
#pragma unroll
    for (int c = 0; c < KX; ++c) {
#pragma unroll
      for (int r = 0; r < RY; ++r) {
        const int b = yi - r;
        if (b < 0 || b >= KY) continue;
        const unsigned long long kp = cp[b * KX + c];
#pragma unroll
        for (int s = 0; s < NIN; ++s)
#pragma unroll
          for (int i = 0; i < RX; ++i) acc[s][r][i] = ffma2_pair(kp, v[s][Cfg::OFF + i + c], acc[s][r][i]);
      }
    }
  }
}

template <typename T, int KY, int KX, int MODE, bool ADJ>
__global__ void __launch_bounds__(Rz2Cfg<T, KY, KX, MODE>::NT)
    conv_rz2_kernel(const __grid_constant__ ConvArgs<T> p) {
  using Cfg = Rz2Cfg<T, KY, KX, MODE>;
  using V = typename Vec16<T>::type;
  constexpr int RX = Cfg::RX, RY = Cfg::RY, KS = Cfg::KS, VEC = Cfg::VEC, NIN = Cfg::NIN;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  unsigned char* sbase = smem_raw + ((128u - (smem_u32(smem_raw) & 127u)) & 127u);
  T* tiles = reinterpret_cast<T*>(sbase);  // [buf][input][TILE]
  T* slices = reinterpret_cast<T*>(sbase + 2 * Cfg::BUF_BYTES);  // [buf][out][KS]
  uint64_t* mbar = reinterpret_cast<uint64_t*>(sbase + 2 * Cfg::BUF_BYTES + Cfg::SLICE_BYTES);
  double* red_s = reinterpret_cast<double*>(mbar + 2);
  if (p.gate && *p.gate != 0.0) return;

  const CtaPos pos = cta_pos64(p.raster_group);
  const int zidx = pos.z;
  const int jid = find_job(p, zidx);
  const ConvJob<T>& job = p.jobs[jid];
  const int zo0 = job.out_lo + 2 * (zidx - job.work_begin);
  const bool has1 = zo0 + 1 < job.out_lo + job.nout;
  const int x0 = pos.tx * Cfg::TX, y0 = pos.ty * Cfg::TY;
  const int tx = threadIdx.x % Cfg::WX, ty = threadIdx.x / Cfg::WX;
  const int rz = (p.kz - 1) / 2;
  const bool tma = job.use_tma != 0;
  // input planes feeding either output, inside the fragment
  const int zi_lo = (int)max((long long)(zo0 - rz), job.src_z0);
  const int zi_hi = (int)min((long long)(zo0 + (has1 ? 1 : 0) + rz), job.src_z0 + job.src_nz - 1);

  constexpr bool kPacked = sizeof(T) == 4 && BD3MG_FFMA2;  // FFMA2 over the plane pair
  static_assert(NIN == 1 || kPacked, "dual-input two-plane kernel is the fp32 packed path");
  auto stage_slices = [&](int zi, int b) {  // coefficient slices of input plane zi
    T* dst = slices + b * 2 * KS;
    for (int t = threadIdx.x; t < 2 * KS; t += Cfg::NT) {
      const int o = t / KS, e = t - o * KS;
      const int zo = zo0 + o, a = zi - zo + rz;
      T v = T(0);
      if ((o == 0 || has1) && tap_ok(p, ADJ, zo, a)) v = coef_of<T, ADJ>(p, zo, a, e / KX, e % KX);
      dst[kPacked ? 2 * e + o : t] = v;  // packed: (k0, k1) pairs
    }
  };
  auto issue = [&](int zi, int b) {
    T* dst = tiles + b * Cfg::BUF;
    if (tma) {
      if (threadIdx.x == 0) {
        mbar_expect_tx(&mbar[b], (uint32_t)(NIN * Cfg::BOX_BYTES));
        tma_load_3d(dst, &job.tmap0, x0 - Cfg::RXA, y0 - Cfg::RYH, (int)(zi - job.src_z0), &mbar[b]);
        if constexpr (NIN == 2)
          tma_load_3d(dst + Cfg::TILE, &job.tmap1, x0 - Cfg::RXA, y0 - Cfg::RYH, (int)(zi - job.src_z0), &mbar[b]);
      }
    } else {
      stage_tile_fallback<Cfg>(dst, job.src0, job.src_z0, zi, y0, x0, p.ny, p.nx, p.plane);
      if constexpr (NIN == 2)
        stage_tile_fallback<Cfg>(dst + Cfg::TILE, job.src1, job.src_z0, zi, y0, x0, p.ny, p.nx, p.plane);
      cp_async_commit();
    }
  };

  if (tma && threadIdx.x == 0) {
    mbar_init(&mbar[0], 1);
    mbar_init(&mbar[1], 1);
    fence_mbar_init();
  }
  if (zi_lo <= zi_hi) stage_slices(zi_lo, 0);
  __syncthreads();

  T acc[2][RY][RX];
#pragma unroll
  for (int o = 0; o < 2; ++o)
#pragma unroll
    for (int r = 0; r < RY; ++r)
#pragma unroll
      for (int i = 0; i < RX; ++i) acc[o][r][i] = T(0);
  T acc1[2][RY][RX];                     // input 1 (Gram mode), filled from the packed pairs
  unsigned long long accp[NIN][RY][RX];  // packed (plane 0, plane 1) accumulators per input
#pragma unroll
  for (int s2 = 0; s2 < NIN; ++s2)
#pragma unroll
    for (int r = 0; r < RY; ++r)
#pragma unroll
      for (int i = 0; i < RX; ++i) accp[s2][r][i] = 0ull;

  if (zi_lo <= zi_hi) issue(zi_lo, 0);
  // epilogue operand rows of both output planes pulled into L2 two planes early
  constexpr bool kEpiLoad = MODE == M_RESID || MODE == M_GRAD || MODE == M_GRAMC;
  const bool vec_io = (p.nx % VEC) == 0;
  const int zi_pf = max(zi_lo, zi_hi - 1);
  uint32_t phase = 0;
  int buf = 0;
  constexpr bool kEpiTma = Cfg::EPI_T;
  const bool epi_tma = kEpiTma && tma && job.epi_tma && zi_lo <= zi_hi;
  for (int zi = zi_lo; zi <= zi_hi; ++zi) {
    if (zi < zi_hi) {
      issue(zi + 1, buf ^ 1);
      stage_slices(zi + 1, buf ^ 1);  // visible after this iteration's closing barrier
    } else if (epi_tma && threadIdx.x == 0) {  // both planes' operand tiles into the freed buffer
      mbar_expect_tx(&mbar[buf ^ 1], (uint32_t)(Cfg::EPI * sizeof(T)));
      tma_load_3d(tiles + (buf ^ 1) * Cfg::BUF, &job.tmap1, x0, y0, zo0 - job.out_lo, &mbar[buf ^ 1]);
    }
    if constexpr (kEpiLoad) {
      if (zi == zi_pf && vec_io && job.sub && threadIdx.x < 2 * Cfg::TY) {
        const int o = threadIdx.x / Cfg::TY, y = y0 + threadIdx.x % Cfg::TY, w = min(Cfg::TX, p.nx - x0);
        if ((o == 0 || has1) && y < p.ny && w > 0)
          prefetch_l2_bulk(job.sub + (long long)(zo0 + o - job.out_lo) * p.plane + (long long)y * p.nx + x0,
                           (uint32_t)(w * sizeof(T)));
      }
    }
    if (tma) {
      mbar_wait(&mbar[buf], (phase >> buf) & 1u);
      phase ^= 1u << buf;
    } else {
      if (zi < zi_hi) cp_async_wait<1>();
      else cp_async_wait<0>();
      __syncthreads();
    }
    // one code body for both outputs (invalid taps have zero coefficients:
    // exact no-ops for finite inputs); three specialised bodies overflow
    // the instruction cache for the 7x7 / 9x9 instantiations (measured)
    const T* tb = tiles + buf * Cfg::BUF + (ty * RY) * Cfg::PITCH + tx * RX;
    const T* cs0 = slices + buf * 2 * KS;
    if constexpr (kPacked)
      rz2_plane_pp<Cfg>(reinterpret_cast<const float*>(tb), reinterpret_cast<const unsigned long long*>(cs0), accp);
    else
      rz2_plane<Cfg, T, true, true>(tb, cs0, cs0 + KS, acc);
    __syncthreads();
    buf ^= 1;
  }
  if constexpr (kPacked) {
#pragma unroll
    for (int r = 0; r < RY; ++r)
#pragma unroll
      for (int i = 0; i < RX; ++i) {
        const float2 f = unpk2(accp[0][r][i]);
        acc[0][r][i] = (T)f.x;
        acc[1][r][i] = (T)f.y;
        if constexpr (NIN == 2) {
          const float2 h = unpk2(accp[NIN - 1][r][i]);
          acc1[0][r][i] = (T)h.x;
          acc1[1][r][i] = (T)h.y;
        }
      }
  }

  // ---- epilogue (both output planes) --------------------------------------
  const T* etile = tiles + buf * Cfg::BUF;  // the buffer the last plane left free
  if (epi_tma) mbar_wait(&mbar[buf], (phase >> buf) & 1u);
  constexpr int NV = Cfg::NV;
  double part[NV > 0 ? NV : 1];
#pragma unroll
  for (int k = 0; k < (NV > 0 ? NV : 1); ++k) part[k] = 0.0;
  const int xt = x0 + tx * RX;
  constexpr bool kVecEpi = MODE == M_STORE || MODE == M_RESID || MODE == M_GRAD || MODE == M_GRAMC;
  const bool vec_here = kVecEpi && vec_io && xt + RX <= p.nx;  // RX == VEC: one 16-byte access per row
#pragma unroll
  for (int o = 0; o < 2; ++o) {
    if (o == 1 && !has1) break;
    const long long orow = (long long)(zo0 + o - job.out_lo) * p.plane;
    if constexpr (kVecEpi) {
      if (vec_here) {
#pragma unroll
        for (int r = 0; r < RY; ++r) {
          const int y = y0 + ty * RY + r;
          if (y >= p.ny) continue;
          const long long q = orow + (long long)y * p.nx + xt;
          T res[RX];
          if constexpr (MODE == M_STORE) {
#pragma unroll
            for (int i = 0; i < RX; ++i) res[i] = acc[o][r][i];
          } else {
            const V v = epi_tma ? *reinterpret_cast<const V*>(etile + (o * Cfg::TY + ty * RY + r) * Cfg::TX + tx * RX)
                                : *reinterpret_cast<const V*>(job.sub + q);
            const T* vs = reinterpret_cast<const T*>(&v);
#pragma unroll
            for (int i = 0; i < RX; ++i) {
              if constexpr (MODE == M_RESID) {
                res[i] = sub_rn(acc[o][r][i], vs[i]);
                part[0] += (double)res[i] * (double)res[i];
              } else if constexpr (MODE == M_GRAMC) {  // H E_S g out; Gram with the cached H E_S d
                const double a0 = (double)acc[o][r][i], c0 = (double)vs[i];
                res[i] = acc[o][r][i];
                part[0] += a0 * a0;
                part[1] += a0 * c0;
                part[2] += c0 * c0;
              } else {
                res[i] = add_rn(acc[o][r][i], vs[i]);
              }
            }
          }
          if (MODE != M_RESID || job.dst0) *reinterpret_cast<V*>(job.dst0 + q) = *reinterpret_cast<const V*>(res);
        }
        continue;
      }
    }
#pragma unroll
    for (int r = 0; r < RY; ++r) {
      const int y = y0 + ty * RY + r;
      if (y >= p.ny) continue;
#pragma unroll
      for (int i = 0; i < RX; ++i) {
        const int x = x0 + tx * RX + i;
        if (x >= p.nx) continue;
        const long long q = orow + (long long)y * p.nx + x;
        const T a0 = acc[o][r][i];
        if constexpr (MODE == M_STORE) {
          job.dst0[q] = a0;
        } else if constexpr (MODE == M_RESID) {
          const T res = sub_rn(a0, job.sub[q]);
          if (job.dst0) job.dst0[q] = res;
          part[0] += (double)res * (double)res;
        } else if constexpr (MODE == M_GRAD) {
          job.dst0[q] = add_rn(a0, job.sub[q]);
        } else if constexpr (MODE == M_GRAM1) {
          if (job.dst0) job.dst0[q] = a0;
          part[0] += (double)a0 * (double)a0;
        } else if constexpr (MODE == M_GRAM2) {
          const T a1 = acc1[o][r][i];
          part[0] += (double)a0 * (double)a0;
          part[1] += (double)a0 * (double)a1;
          part[2] += (double)a1 * (double)a1;
        } else if constexpr (MODE == M_GRAMC) {
          const double c0 = (double)job.sub[q];
          job.dst0[q] = a0;
          part[0] += (double)a0 * (double)a0;
          part[1] += (double)a0 * c0;
          part[2] += c0 * c0;
        }
      }
    }
  }
  if constexpr (NV > 0) {
    cta_reduce<NV, Cfg::NT>(part, red_s);
    if (threadIdx.x == 0) {
      const long long cta = pos.cta;
#pragma unroll
      for (int k = 0; k < NV; ++k) p.partials[cta * NV + k] = part[k];
    }
  }
}

// ---------------------------------------------------------------------------
// Generic path for kernel widths without a tuned instantiation: one output
// voxel per thread, runtime ky/kx, same a->b->c order and same epilogues.
constexpr int kGenericNT = 128;
constexpr int kGenericTX = 32, kGenericTY = 4;

template <typename T, int MODE, bool ADJ>
__global__ void __launch_bounds__(kGenericNT) conv_generic_kernel(const __grid_constant__ ConvArgs<T> p) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  T* coef_s = reinterpret_cast<T*>(smem_raw);
  size_t coef_bytes = ((size_t)p.kz * p.ky * p.kx * sizeof(T) + 15) & ~size_t(15);
  double* red_s = reinterpret_cast<double*>(smem_raw + coef_bytes);
  if (p.gate && *p.gate != 0.0) return;
  const CtaPos pos = cta_pos(p.raster_group);
  const int zidx = pos.z;
  const int jid = find_job(p, zidx);
  const ConvJob<T>& job = p.jobs[jid];
  const int zo = job.out_lo + (zidx - job.work_begin);
  stage_coefs<T, ADJ>(p, zo, coef_s, kGenericNT);
  __syncthreads();
  const int x = pos.tx * kGenericTX + (threadIdx.x % kGenericTX);
  const int y = pos.ty * kGenericTY + (threadIdx.x / kGenericTX);
  const int rz = (p.kz - 1) / 2, ry = (p.ky - 1) / 2, rx = (p.kx - 1) / 2;
  constexpr int NV = ModeNV<MODE>::value;
  double part[NV > 0 ? NV : 1];
  for (int k = 0; k < (NV > 0 ? NV : 1); ++k) part[k] = 0.0;
  if (y < p.ny && x < p.nx) {
    T acc0 = T(0), acc1 = T(0);
    for (int a = 0; a < p.kz; ++a) {
      const long long zi = (long long)zo + a - rz;
      if (zi < job.src_z0 || zi >= job.src_z0 + job.src_nz) continue;
      const long long pbase = (zi - job.src_z0) * p.plane;
      for (int b = 0; b < p.ky; ++b) {
        const int yy = y + b - ry;
        if (yy < 0 || yy >= p.ny) continue;
        for (int c = 0; c < p.kx; ++c) {
          const int xx = x + c - rx;
          if (xx < 0 || xx >= p.nx) continue;
          const T k = coef_s[(a * p.ky + b) * p.kx + c];
          const long long off = pbase + (long long)yy * p.nx + xx;
          acc0 = fma_rn(k, job.src0[off], acc0);
          if constexpr (MODE == M_GRAM2) acc1 = fma_rn(k, job.src1[off], acc1);
        }
      }
    }
    const long long o = (long long)(zo - job.out_lo) * p.plane + (long long)y * p.nx + x;
    if constexpr (MODE == M_STORE) {
      job.dst0[o] = acc0;
    } else if constexpr (MODE == M_RESID) {
      const T res = sub_rn(acc0, job.sub[o]);
      if (job.dst0) job.dst0[o] = res;
      part[0] = (double)res * (double)res;
    } else if constexpr (MODE == M_GRAD) {
      job.dst0[o] = add_rn(acc0, job.sub[o]);
    } else if constexpr (MODE == M_GRAM1) {
      if (job.dst0) job.dst0[o] = acc0;
      part[0] = (double)acc0 * (double)acc0;
    } else if constexpr (MODE == M_GRAM2) {
      part[0] = (double)acc0 * (double)acc0;
      part[1] = (double)acc0 * (double)acc1;
      part[2] = (double)acc1 * (double)acc1;
    } else if constexpr (MODE == M_GRAMC) {
      const double c0 = (double)job.sub[o];
      job.dst0[o] = acc0;
      part[0] = (double)acc0 * (double)acc0;
      part[1] = (double)acc0 * c0;
      part[2] = c0 * c0;
    }
  }
  if constexpr (NV > 0) {
    cta_reduce<NV, kGenericNT>(part, red_s);
    if (threadIdx.x == 0) {
      const long long cta = pos.cta;
      for (int k = 0; k < NV; ++k) p.partials[cta * NV + k] = part[k];
    }
  }
}

}  // namespace bd3mg
