// TMA-staged z-marching stencils (used when a row is a whole number of
// 16-byte chunks, i.e. nx * sizeof(T) % 16 == 0; stencil.cuh keeps the
// cp.async kernels for the other shapes).
//
// One CTA owns a 32 x 16 pixel tile of all rows of a job and walks them in
// depth.  Plane tiles (with the halo the stencil needs) arrive by one
// cp.async.bulk.tensor per plane into a ring of mbarrier-tracked slots, so
// the load path costs one instruction per plane instead of an address
// computation and a predicate per element; out-of-volume halo entries are
// zero-filled by the TMA unit.  Each thread owns 4 pixels of a column and
// keeps their values in registers between the two passes of a plane.
//
//   greg_t_kernel      = greg_z_kernel   (regulariser gradient, omega, recorder terms)
//   reg_gram_t_kernel  = reg_gram_z_kernel (regulariser Gram terms, rhs, flags)
//
// Arithmetic is operation-for-operation that of the cp.async kernels
// (reference objective.py:130-137, :175-186, :262-274; directions.py:80-85).
#pragma once

#include <cuda.h>

#include "stencil.cuh"

namespace bd3mg {

constexpr int kTmX = 32;                   // tile width  (one warp row)
constexpr int kTmY = 16;                   // tile height
constexpr int kTmNT = 128;                 // 4 warps
constexpr int kTmR = kTmY / (kTmNT / 32);  // pixels (rows) per thread

template <typename T>
struct StTma {
  CUtensorMap a[kMaxJobs];  // greg: x fragment; reg_gram: g rows
  CUtensorMap b[kMaxJobs];  // reg_gram: d rows
};

// Box geometry: width padded to an even number of 16-byte chunks, height so
// the box is a whole number of 128-byte lines (scripts/tma_probe.py).
template <typename T>
struct GregGeo {
  static constexpr int VEC = 16 / (int)sizeof(T);
  // x from x0 - VEC to x0 + 32 (pixel x0-1 needs its right neighbour x0 .. ;
  // pixel x0+31 needs x0+32); rows y0-1 .. y0+16
  static constexpr int BW = (kTmX + 1 + VEC + 2 * VEC - 1) / (2 * VEC) * (2 * VEC);
  static constexpr int ROWQ = 128 / cgcd(BW * (int)sizeof(T), 128);
  static constexpr int BH = (kTmY + 2 + ROWQ - 1) / ROWQ * ROWQ;
  static constexpr int PL = BW * BH;
  static constexpr int RING = 4;  // z-1, z, z+1 resident, z+2 in flight
  // w*dx / w*dy exchange: the left neighbour's px comes from lane-1 (shuffle),
  // the upper neighbour's py from the thread's previous row; shared memory
  // only holds the halo row (py, y0-1), the halo column (px, x0-1) and each
  // warp's last row (py), so 7 CTAs fit an SM (one wave at 256 x 256 x 64)
  static constexpr int NW = kTmNT / 32;
  static constexpr int HALO = kTmX + kTmY + NW * kTmX;
  static constexpr size_t smem() {
    return 128 + (size_t)RING * PL * sizeof(T) + (size_t)HALO * sizeof(T) + (kTmNT / 32) * kEvalNV * 8 + RING * 8;
  }
};

template <typename T>
struct RgGeo {
  static constexpr int VEC = 16 / (int)sizeof(T);
  // x from x0 to x0 + 32, rows y0 .. y0 + 16
  static constexpr int BW = (kTmX + 1 + 2 * VEC - 1) / (2 * VEC) * (2 * VEC);
  static constexpr int ROWQ = 128 / cgcd(BW * (int)sizeof(T), 128);
  static constexpr int BH = (kTmY + 1 + ROWQ - 1) / ROWQ * ROWQ;
  static constexpr int PL = BW * BH;
  static constexpr int RING = 3;  // z, z+1 resident, z+2 in flight
  static constexpr size_t smem() {
    return 128 + 2 * (size_t)RING * PL * sizeof(T) + (kTmNT / 32) * kRegNV * 8 + RING * 8;
  }
};

// Partial rows are job-major like the cp.async kernels, on this tiling.
inline long long tm_tiles(long long ny, long long nx) {
  return ((nx + kTmX - 1) / kTmX) * ((ny + kTmY - 1) / kTmY);
}

// ---------------------------------------------------------------------------
// Regulariser gradient, omega (+ recorder terms, snapshot roll when EVAL) of
// the 32 x 16 pixel column (bx, by) over every row of job J.  `tma_a` maps
// J.a with the GregGeo box; `base` is 128-byte aligned smem of GregGeo::smem.
template <typename T, bool EVAL>
BD3MG_D void greg_tile(const StGeom<T>& p, const StJob<T>& J, const CUtensorMap* tma_a, int bx, int by,
                       double* part_out, unsigned char* base, uint64_t* bars_ext = nullptr) {
  using G = GregGeo<T>;
  constexpr int VEC = G::VEC;
  T (*xs)[G::PL] = reinterpret_cast<T (*)[G::PL]>(base);
  T* hpy = reinterpret_cast<T*>(base + G::RING * G::PL * sizeof(T));  // py of row y0-1, cols x0..x0+31
  T* hpx = hpy + kTmX;                                                // px of col x0-1, rows y0..y0+15
  T* lastpy = hpx + kTmY;                                             // [warp][lane]: py of the warp's last row
  double* red = reinterpret_cast<double*>(lastpy + G::NW * kTmX);
  uint64_t* bars = bars_ext ? bars_ext : reinterpret_cast<uint64_t*>(red + (kTmNT / 32) * kEvalNV);

  const int x0 = bx * kTmX, y0 = by * kTmY;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int zfirst = max(J.lo - 1, 0), zlast = min(J.hi + 1, p.nz - 1);
  const int nx = p.nx, ny = p.ny;
  if (threadIdx.x == 0) {
    for (int s = 0; s < G::RING; ++s) mbar_init(&bars[s], 1);
    fence_mbar_init();
  }
  __syncthreads();
  auto slot = [&](int z) { return (z - zfirst) % G::RING; };
  auto phase = [&](int z) { return (uint32_t)((z - zfirst) / G::RING) & 1u; };
  auto issue = [&](int z) {  // thread 0
    const int s = slot(z);
    mbar_expect_tx(&bars[s], G::PL * sizeof(T));
    tma_load_3d(xs[s], tma_a, x0 - VEC, y0 - 1, (int)(z - J.a_z0), &bars[s]);
  };
  if (threadIdx.x == 0) {
    tma_prefetch_desc(tma_a);
    for (int z = zfirst; z <= min(J.lo + 1, zlast); ++z) issue(z);
  }
  for (int z = zfirst; z <= J.lo; ++z) mbar_wait(&bars[slot(z)], phase(z));

  const T d2 = (T)p.delta2;
  const T two_eta = (T)p.two_eta, lam = (T)p.lam, two_kappa = (T)p.two_kappa;
  const T xmin = (T)p.x_min, xmax = (T)p.x_max;
  const int x = x0 + lane;
  double ev[kEvalNV] = {0.0, 0.0, 0.0, 0.0, 0.0};
  // halo item of this thread: threads 0..31 the py of (y0-1, x0+t), threads
  // 32..47 the px of (y0+t-32, x0-1)
  constexpr int NEXTRA = kTmX + kTmY;
  const int er = threadIdx.x < kTmX ? 0 : threadIdx.x - kTmX + 1;   // region row (0 = y0-1)
  const int ec = threadIdx.x < kTmX ? threadIdx.x + 1 : 0;          // region col (0 = x0-1)
  const int ey = y0 - 1 + er, ex = x0 - 1 + ec;

  for (int z = J.lo; z <= J.hi; ++z) {
    const long long orow = (long long)(z - J.lo) * p.plane;
    T sn[kTmR];
    if constexpr (EVAL) {
#pragma unroll
      for (int j = 0; j < kTmR; ++j) {
        const int y = y0 + warp * kTmR + j;
        sn[j] = (J.b && y < ny && x < nx) ? J.b[orow + (long long)y * nx + x] : T(0);
      }
    }
    if (threadIdx.x == 0 && z + 2 <= zlast) issue(z + 2);
    if (z + 1 <= zlast) mbar_wait(&bars[slot(z + 1)], phase(z + 1));
    const T* xc_t = xs[slot(z)];
    // pass 1: omega, w*dx, w*dy of the own pixels (kept in registers) and of
    // the row-above / column-left halo (shared with the neighbours)
    T xc[kTmR], px[kTmR], py[kTmR];
#pragma unroll
    for (int j = 0; j < kTmR; ++j) {
      const int ly = warp * kTmR + j, y = y0 + ly;
      const int si = (ly + 1) * G::BW + lane + VEC;
      xc[j] = xc_t[si];
      const T dx = (x < nx - 1) ? sub_rn(xc_t[si + 1], xc[j]) : T(0);
      const T dy = (y < ny - 1) ? sub_rn(xc_t[si + G::BW], xc[j]) : T(0);
      const T sq = add_rn(add_rn(mul_rn(dx, dx), mul_rn(dy, dy)), d2);
      const T w = rsqrt(sq);
      px[j] = mul_rn(w, dx);
      py[j] = mul_rn(w, dy);
      if (y < ny && x < nx) {
        J.out1[orow + (long long)y * nx + x] = w;
        if constexpr (EVAL) ev[1] += (double)sq * (double)w;
      }
    }
    lastpy[warp * kTmX + lane] = py[kTmR - 1];
    if (threadIdx.x < NEXTRA) {
      T ex_px = T(0), ex_py = T(0);
      if (ey >= 0 && ex >= 0 && ey < ny && ex < nx) {
        const int si = er * G::BW + ec - 1 + VEC;
        const T c = xc_t[si];
        const T dx = (ex < nx - 1) ? sub_rn(xc_t[si + 1], c) : T(0);
        const T dy = (ey < ny - 1) ? sub_rn(xc_t[si + G::BW], c) : T(0);
        const T w = rsqrt(add_rn(add_rn(mul_rn(dx, dx), mul_rn(dy, dy)), d2));
        ex_px = mul_rn(w, dx);
        ex_py = mul_rn(w, dy);
      }
      if (threadIdx.x < kTmX) hpy[threadIdx.x] = ex_py;
      else hpx[er - 1] = ex_px;
    }
    // left neighbours' px: lane - 1 (all lanes shuffle before any predication)
    T pxl[kTmR];
#pragma unroll
    for (int j = 0; j < kTmR; ++j) pxl[j] = __shfl_up_sync(0xffffffffu, px[j], 1);
    __syncthreads();
    // pass 2: box + TV divergence + axial terms
    const T* xm_t = xs[slot(max(z - 1, zfirst))];
    const T* xp_t = xs[slot(min(z + 1, zlast))];
    const bool has_m = z >= 1, has_p = z < p.nz - 1;
#pragma unroll
    for (int j = 0; j < kTmR; ++j) {
      const int ly = warp * kTmR + j, y = y0 + ly;
      if (y >= ny || x >= nx) continue;
      const int si = (ly + 1) * G::BW + lane + VEC;
      const T clipped = xc[j] < xmin ? xmin : (xc[j] > xmax ? xmax : xc[j]);
      const T box = mul_rn(two_eta, sub_rn(xc[j], clipped));
      const T pxm = lane > 0 ? pxl[j] : hpx[ly];
      const T pym = j > 0 ? py[j - 1] : (warp > 0 ? lastpy[(warp - 1) * kTmX + lane] : hpy[lane]);
      const T tvx = (nx == 1) ? T(0) : sub_rn(pxm, px[j]);
      const T tvy = (ny == 1) ? T(0) : sub_rn(pym, py[j]);
      const T xzp = has_p ? xp_t[si] : T(0);
      const T dzm = has_m ? sub_rn(xc[j], xm_t[si]) : T(0);
      const T dzp = has_p ? sub_rn(xzp, xc[j]) : T(0);
      J.out0[orow + (long long)y * nx + x] =
          add_rn(add_rn(box, mul_rn(lam, add_rn(tvx, tvy))), mul_rn(two_kappa, sub_rn(dzm, dzp)));
      if constexpr (EVAL) {
        const double e = (double)xc[j] - (double)clipped;
        ev[0] += e * e;
        if (has_p) ev[2] += ((double)xzp - (double)xc[j]) * ((double)xzp - (double)xc[j]);
        if (J.b) {
          ev[3] += ((double)xc[j] - (double)sn[j]) * ((double)xc[j] - (double)sn[j]);
          ev[4] += (double)sn[j] * (double)sn[j];
        }
        if (J.snap_out) J.snap_out[orow + (long long)y * nx + x] = xc[j];
      }
    }
    __syncthreads();  // halo px/py rewritten and the slot of z-1 refilled next iteration
  }
  if constexpr (EVAL) {
    cta_reduce<kEvalNV, kTmNT>(ev, red);
    if (threadIdx.x == 0 && part_out) {
#pragma unroll
      for (int k = 0; k < kEvalNV; ++k) part_out[k] = ev[k];
    }
  }
}

template <typename T, bool EVAL>
__global__ void __launch_bounds__(kTmNT) greg_t_kernel(const __grid_constant__ StArgs<T> p,
                                                       const __grid_constant__ StTma<T> tm) {
  extern __shared__ __align__(128) unsigned char st_smem[];
  unsigned char* base = st_smem + ((128 - (smem_u32(st_smem) & 127)) & 127);
  const long long cta = ((long long)blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
  greg_tile<T, EVAL>(p, p.jobs[blockIdx.z], &tm.a[blockIdx.z], blockIdx.x, blockIdx.y,
                     EVAL ? p.partials + cta * kEvalNV : nullptr, base);
}

// ---------------------------------------------------------------------------
// Regulariser Gram terms, rhs and flags of the 32 x 16 column (bx, by) over
// the rows of job J (g = J.a via tma_a, d = J.b via tma_b, omega = J.w).
// `ldcg`: omega is read through L2 only (written by another CTA of the same
// persistent kernel).
template <typename T, bool LDCG = false>
BD3MG_D void reg_gram_tile(const StGeom<T>& p, const StJob<T>& J, const CUtensorMap* tma_a, const CUtensorMap* tma_b,
                           int bx, int by, double* part_out, unsigned char* base, uint64_t* bars_ext = nullptr) {
  using G = RgGeo<T>;
  T (*gs)[G::PL] = reinterpret_cast<T (*)[G::PL]>(base);
  T (*dss)[G::PL] = reinterpret_cast<T (*)[G::PL]>(base + G::RING * G::PL * sizeof(T));
  double* red = reinterpret_cast<double*>(base + 2 * G::RING * G::PL * sizeof(T));
  uint64_t* bars = bars_ext ? bars_ext : reinterpret_cast<uint64_t*>(red + (kTmNT / 32) * kRegNV);

  const int x0 = bx * kTmX, y0 = by * kTmY;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const bool has_d = J.b != nullptr;
  const int nx = p.nx, ny = p.ny;
  // z-chunk of a block (small grids): the block's own rows decide the
  // embedding rules; the chunk also stages the plane after its last row
  const bool chunk = J.chunk != 0;
  const int blo = chunk ? J.blo : J.lo, bhi = chunk ? J.bhi : J.hi;
  const int zend = J.hi < bhi ? J.hi + 1 : J.hi;  // last plane staged
  if (threadIdx.x == 0) {
    for (int s = 0; s < G::RING; ++s) mbar_init(&bars[s], 1);
    fence_mbar_init();
  }
  __syncthreads();
  auto slot = [&](int z) { return (z - J.lo) % G::RING; };
  auto phase = [&](int z) { return (uint32_t)((z - J.lo) / G::RING) & 1u; };
  auto issue = [&](int z) {  // thread 0
    const int s = slot(z);
    mbar_expect_tx(&bars[s], (has_d ? 2 : 1) * G::PL * sizeof(T));
    tma_load_3d(gs[s], tma_a, x0, y0, z - J.lo + J.tz_off, &bars[s]);
    if (has_d) tma_load_3d(dss[s], tma_b, x0, y0, z - J.lo + J.tz_off_b, &bars[s]);
  };
  if (threadIdx.x == 0) {
    tma_prefetch_desc(tma_a);
    if (has_d) tma_prefetch_desc(tma_b);
    issue(J.lo);
    if (J.lo + 1 <= zend) issue(J.lo + 1);
  }
  mbar_wait(&bars[slot(J.lo)], phase(J.lo));

  double v[kRegNV];
#pragma unroll
  for (int k = 0; k < kRegNV; ++k) v[k] = 0.0;
  const int x = x0 + lane;
  for (int z = J.lo; z <= J.hi; ++z) {
    const long long orow = (long long)(z - J.lo) * p.plane;
    T wv[kTmR];
#pragma unroll
    for (int j = 0; j < kTmR; ++j) {
      const int y = y0 + warp * kTmR + j;
      if constexpr (LDCG) wv[j] = (y < ny && x < nx) ? __ldcg(J.w + orow + (long long)y * nx + x) : T(0);
      else wv[j] = (y < ny && x < nx) ? J.w[orow + (long long)y * nx + x] : T(0);
    }
    if (threadIdx.x == 0 && z + 2 <= zend) issue(z + 2);
    if (z + 1 <= zend) mbar_wait(&bars[slot(z + 1)], phase(z + 1));
    const T* g0 = gs[slot(z)];
    const T* d0 = dss[slot(z)];
    const T* g1 = gs[slot(min(z + 1, zend))];
    const T* d1 = dss[slot(min(z + 1, zend))];
#pragma unroll
    for (int j = 0; j < kTmR; ++j) {
      const int ly = warp * kTmR + j, y = y0 + ly;
      if (y >= ny || x >= nx) continue;
      const int q = ly * G::BW + lane;
      const T g = g0[q];
      const T d = has_d ? d0[q] : T(0);
      const double b0 = -(double)g, b1 = (double)d;
      v[0] += b0 * b0;
      v[1] += b0 * b1;
      v[2] += b1 * b1;
      const double w = (double)wv[j];
      const double dx0 = (x < nx - 1) ? -(double)sub_rn(g0[q + 1], g) : 0.0;
      const double dy0 = (y < ny - 1) ? -(double)sub_rn(g0[q + G::BW], g) : 0.0;
      const double dx1 = (has_d && x < nx - 1) ? (double)sub_rn(d0[q + 1], d) : 0.0;
      const double dy1 = (has_d && y < ny - 1) ? (double)sub_rn(d0[q + G::BW], d) : 0.0;
      v[3] += w * (dx0 * dx0 + dy0 * dy0);
      v[4] += w * (dx0 * dx1 + dy0 * dy1);
      v[5] += w * (dx1 * dx1 + dy1 * dy1);
      double z0v, z1v;  // axial row z of the block-embedded vectors
      if (z < bhi) {
        z0v = -((double)g1[q] - (double)g);
        z1v = has_d ? (double)d1[q] - (double)d : 0.0;
      } else if (bhi < p.nz - 1) {
        z0v = -b0;
        z1v = -b1;
      } else {
        z0v = 0.0;
        z1v = 0.0;
      }
      v[6] += z0v * z0v;
      v[7] += z0v * z1v;
      v[8] += z1v * z1v;
      if (z == blo && blo >= 1) {
        v[6] += b0 * b0;
        v[7] += b0 * b1;
        v[8] += b1 * b1;
      }
      v[9] += (double)g * (double)d;
      v[10] += (g != T(0)) ? 1.0 : 0.0;
      v[11] += isfinite((double)g) ? 0.0 : 1.0;
    }
    __syncthreads();  // slot of z is refilled next iteration
  }
  cta_reduce<kRegNV, kTmNT>(v, red);
  if (threadIdx.x == 0 && part_out) {
#pragma unroll
    for (int k = 0; k < kRegNV; ++k) part_out[k] = v[k];
  }
}

template <typename T>
__global__ void __launch_bounds__(kTmNT) reg_gram_t_kernel(const __grid_constant__ StArgs<T> p,
                                                           const __grid_constant__ StTma<T> tm) {
  extern __shared__ __align__(128) unsigned char st_smem[];
  unsigned char* base = st_smem + ((128 - (smem_u32(st_smem) & 127)) & 127);
  const long long cta = ((long long)blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
  reg_gram_tile<T>(p, p.jobs[blockIdx.z], &tm.a[blockIdx.z], &tm.b[blockIdx.z], blockIdx.x, blockIdx.y,
                   p.partials + cta * kRegNV, base);
}

}  // namespace bd3mg
