// HBM-bound stencil kernels of the block step, 2-D shared-memory tiled:
// every field is read from DRAM once (neighbours come from the staged tile,
// the +-1 plane values from L2), every half-quadratic weight is computed once
// per pixel.
//
//   greg_z_kernel      regulariser gradient 2eta*box + lam*TV + 2kappa*axial
//                      and the weights omega (reference objective.py:130-137,
//                      :175-186), optionally fused with the recorder terms;
//                      the H^T epilogue adds it to H^T r.
//   reg_gram_z_kernel  regulariser part of the forward-only Gram for
//                      D = [-g, d] plus rhs / flags (directions.py:80-85 with
//                      A from objective.py:262-274).
//   eval_kernel        box / TV / axial terms of f and the stop-rule norms
//                      (objective.py:148-152, scheduler.py:218-219).
#pragma once

#include "depthvar.cuh"

namespace bd3mg {

constexpr int kTS = 32;                 // tile edge (pixels)
constexpr int kStNT = 256;              // threads: 32 (x) x 8 (y); 4 rows per thread
constexpr int kStRows = kTS / (kStNT / kTS);
constexpr int kRegNV = 12;              // sums produced per block by reg_gram
static_assert(kRegNV == kRgNV, "the fused regulariser Gram (depthvar.cuh, rg_center) writes the same rows");
constexpr int kEvalNV = 5;              // box, tv, axial, |x-snap|^2, |snap|^2

template <typename T>
struct StJob {
  const T* a;      // primary field, plane 0 = depth a_z0 (x for greg/eval, g for reg_gram)
  const T* b;      // reg_gram: d (plane 0 = depth lo) or null; eval: snapshot rows (row 0 = lo) or null
  const T* w;      // reg_gram: omega rows (row 0 = lo)
  T* out0;         // greg: regulariser gradient rows (row 0 = lo)
  T* out1;         // greg: omega rows (row 0 = lo)
  long long a_z0;
  int lo, hi;      // rows of the job
  int work_begin;  // first grid.z index of the job
  int chunk;       // reg_gram (TMA path): [lo, hi] is a z-chunk of the block [blo, bhi]
  int blo, bhi;
  T* snap_out;     // greg with recorder terms: snapshot roll, snap_out row z-lo = x row z after it is read (or null)
  int tz_off, tz_off_b;  // reg_gram TMA: z coordinate of row lo in the maps of a / b (0: maps start at row lo)
};

// geometry and regulariser weights of a stencil launch (the tile functions
// of stencil_tma.cuh take this; the persistent sweep kernel embeds one)
template <typename T>
struct StGeom {
  int nz, ny, nx;
  long long plane;
  double two_eta, lam, two_kappa, delta2, x_min, x_max;
};

template <typename T>
struct StArgs : StGeom<T> {
  int njobs, tiles_x, tiles_y;
  double* partials;  // reg_gram / eval: [grid.z * tiles][NV]
  StJob<T> jobs[kMaxJobs];
};

template <typename T>
BD3MG_D int st_find_job(const StArgs<T>& p, int zidx) {
  int j = 0;
  while (j + 1 < p.njobs && p.jobs[j + 1].work_begin <= zidx) ++j;
  return j;
}

// Load plane rows [y0+oy, y0+oy+H) x cols [x0+ox, x0+ox+W) into s (pitch P);
// out-of-volume entries are 0 (never used: the far-face rules mask them).
template <typename T, int H, int W, int P>
BD3MG_D void st_load(T* s, const T* plane, int y0, int x0, int oy, int ox, int ny, int nx) {
#pragma unroll
  for (int i = threadIdx.x; i < H * W; i += kStNT) {
    const int r = i / W, c = i - r * W;
    const int y = y0 + oy + r, x = x0 + ox + c;
    s[r * P + c] = (y >= 0 && y < ny && x >= 0 && x < nx) ? plane[(long long)y * nx + x] : T(0);
  }
}

// ---------------------------------------------------------------------------
// ---------------------------------------------------------------------------
template <typename T>
__global__ void __launch_bounds__(kStNT) eval_kernel(const __grid_constant__ StArgs<T> p) {
  constexpr int SP = kTS + 1;
  __shared__ T xs[SP * SP];
  __shared__ double red[(kStNT / 32) * kEvalNV];
  const StJob<T>& J = p.jobs[st_find_job(p, blockIdx.z)];
  const int z = J.lo + (blockIdx.z - J.work_begin);
  const int x0 = blockIdx.x * kTS, y0 = blockIdx.y * kTS;
  const T* xp = J.a + (long long)(z - J.a_z0) * p.plane;
  st_load<T, SP, SP, SP>(xs, xp, y0, x0, 0, 0, p.ny, p.nx);
  const int tx = threadIdx.x % kTS, ty = threadIdx.x / kTS;
  T xz[kStRows], sn[kStRows];  // x(z+1), snapshot: in flight during the tile load
#pragma unroll
  for (int j = 0; j < kStRows; ++j) {
    const int y = y0 + ty + j * (kStNT / kTS), x = x0 + tx;
    const bool in = y < p.ny && x < p.nx;
    const long long q = (long long)y * p.nx + x;
    xz[j] = (in && z < p.nz - 1) ? xp[q + p.plane] : T(0);
    sn[j] = (in && J.b) ? J.b[(long long)(z - J.lo) * p.plane + q] : T(0);
  }
  __syncthreads();
  double v[kEvalNV] = {0.0, 0.0, 0.0, 0.0, 0.0};
#pragma unroll
  for (int j = 0; j < kStRows; ++j) {
    const int ly = ty + j * (kStNT / kTS);
    const int y = y0 + ly, x = x0 + tx;
    if (y >= p.ny || x >= p.nx) continue;
    const long long q = (long long)y * p.nx + x;
    const double xc = (double)xs[ly * SP + tx];
    const double cl = xc < p.x_min ? p.x_min : (xc > p.x_max ? p.x_max : xc);
    v[0] += (xc - cl) * (xc - cl);
    const double dx = (x < p.nx - 1) ? (double)xs[ly * SP + tx + 1] - xc : 0.0;
    const double dy = (y < p.ny - 1) ? (double)xs[(ly + 1) * SP + tx] - xc : 0.0;
    const double s2 = dx * dx + dy * dy + p.delta2;
    v[1] += s2 * rsqrt(s2);
    if (z < p.nz - 1) {
      const double dz = (double)xz[j] - xc;
      v[2] += dz * dz;
    }
    if (J.b) {
      const double s = (double)sn[j];
      v[3] += (xc - s) * (xc - s);
      v[4] += s * s;
    }
  }
  cta_reduce<kEvalNV, kStNT>(v, red);
  if (threadIdx.x == 0) {
    const long long cta = ((long long)blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
#pragma unroll
    for (int k = 0; k < kEvalNV; ++k) p.partials[cta * kEvalNV + k] = v[k];
  }
}

// ---------------------------------------------------------------------------
// z-marching variants: one CTA owns a 32x32 tile of ALL rows of a job and
// walks them in depth through a cp.async ring of halo tiles, so every plane
// is read once per CTA and the block reduction runs once per CTA.
// Partial rows are job-major: row = (job * tiles_y + by) * tiles_x + bx.

template <typename T, int H, int W, int P>
BD3MG_D void st_load_async(T* s, const T* plane, int y0, int x0, int oy, int ox, int ny, int nx) {
#pragma unroll
  for (int i = threadIdx.x; i < H * W; i += kStNT) {
    const int r = i / W, c = i - r * W;
    const int y = y0 + oy + r, x = x0 + ox + c;
    const bool ok = y >= 0 && y < ny && x >= 0 && x < nx;
    cp_async<sizeof(T)>(s + r * P + c, ok ? plane + (long long)y * nx + x : plane, ok);
  }
}

template <typename T>
__global__ void __launch_bounds__(kStNT) reg_gram_z_kernel(const __grid_constant__ StArgs<T> p) {
  constexpr int SP = kTS + 1;        // rows/cols y0 .. y0+32
  constexpr int PL = SP * SP;
  constexpr int RING = 3;            // planes z, z+1 resident, z+2 in flight
  extern __shared__ __align__(128) unsigned char st_smem[];
  T (*gs)[PL] = reinterpret_cast<T (*)[PL]>(st_smem);
  T (*dss)[PL] = reinterpret_cast<T (*)[PL]>(st_smem + RING * PL * sizeof(T));
  double* red = reinterpret_cast<double*>(st_smem + 2 * RING * PL * sizeof(T));
  const StJob<T>& J = p.jobs[blockIdx.z];
  const int x0 = blockIdx.x * kTS, y0 = blockIdx.y * kTS;
  const bool has_d = J.b != nullptr;
  const int tx = threadIdx.x % kTS, ty = threadIdx.x / kTS;
  auto load = [&](int z, int slot) {
    const long long off = (long long)(z - J.lo) * p.plane;
    st_load_async<T, SP, SP, SP>(gs[slot], J.a + off, y0, x0, 0, 0, p.ny, p.nx);
    if (has_d) st_load_async<T, SP, SP, SP>(dss[slot], J.b + off, y0, x0, 0, 0, p.ny, p.nx);
    cp_async_commit();
  };
  double v[kRegNV];
#pragma unroll
  for (int k = 0; k < kRegNV; ++k) v[k] = 0.0;
  load(J.lo, 0);
  if (J.lo + 1 <= J.hi) load(J.lo + 1, 1);
  for (int z = J.lo; z <= J.hi; ++z) {
    const int cur = (z - J.lo) % RING, nxt = (z + 1 - J.lo) % RING;
    T wv[kStRows];  // omega of this plane's pixels
#pragma unroll
    for (int j = 0; j < kStRows; ++j) {
      const int y = y0 + ty + j * (kStNT / kTS), x = x0 + tx;
      wv[j] = (y < p.ny && x < p.nx) ? J.w[(long long)(z - J.lo) * p.plane + (long long)y * p.nx + x] : T(0);
    }
    if (z + 2 <= J.hi) load(z + 2, (z + 2 - J.lo) % RING);
    // planes z (and z+1 if inside the job) have landed
    if (z + 2 <= J.hi) cp_async_wait<1>();
    else cp_async_wait<0>();
    __syncthreads();
    const T* g0 = gs[cur];
    const T* d0 = dss[cur];
    const T* g1 = gs[nxt];
    const T* d1 = dss[nxt];
#pragma unroll
    for (int j = 0; j < kStRows; ++j) {
      const int ly = ty + j * (kStNT / kTS);
      const int y = y0 + ly, x = x0 + tx;
      if (y >= p.ny || x >= p.nx) continue;
      const int q = ly * SP + tx;
      const T g = g0[q];
      const T d = has_d ? d0[q] : T(0);
      const double b0 = -(double)g, b1 = (double)d;
      v[0] += b0 * b0;
      v[1] += b0 * b1;
      v[2] += b1 * b1;
      const double w = (double)wv[j];
      const double dx0 = (x < p.nx - 1) ? -(double)sub_rn(g0[q + 1], g) : 0.0;
      const double dy0 = (y < p.ny - 1) ? -(double)sub_rn(g0[q + SP], g) : 0.0;
      const double dx1 = (has_d && x < p.nx - 1) ? (double)sub_rn(d0[q + 1], d) : 0.0;
      const double dy1 = (has_d && y < p.ny - 1) ? (double)sub_rn(d0[q + SP], d) : 0.0;
      v[3] += w * (dx0 * dx0 + dy0 * dy0);
      v[4] += w * (dx0 * dx1 + dy0 * dy1);
      v[5] += w * (dx1 * dx1 + dy1 * dy1);
      double z0v, z1v;  // axial row z of the block-embedded vectors
      if (z < J.hi) {
        z0v = -((double)g1[q] - (double)g);
        z1v = has_d ? (double)d1[q] - (double)d : 0.0;
      } else if (J.hi < p.nz - 1) {
        z0v = -b0;
        z1v = -b1;
      } else {
        z0v = 0.0;
        z1v = 0.0;
      }
      v[6] += z0v * z0v;
      v[7] += z0v * z1v;
      v[8] += z1v * z1v;
      if (z == J.lo && J.lo >= 1) {
        v[6] += b0 * b0;
        v[7] += b0 * b1;
        v[8] += b1 * b1;
      }
      v[9] += (double)g * (double)d;
      v[10] += (g != T(0)) ? 1.0 : 0.0;
      v[11] += isfinite((double)g) ? 0.0 : 1.0;
    }
    __syncthreads();  // slot `cur` is refilled next iteration
  }
  cta_reduce<kRegNV, kStNT>(v, red);
  if (threadIdx.x == 0) {
    const long long cta = ((long long)blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
#pragma unroll
    for (int k = 0; k < kRegNV; ++k) p.partials[cta * kRegNV + k] = v[k];
  }
}

template <typename T>
constexpr size_t reg_gram_z_smem() { return 2 * 3 * (kTS + 1) * (kTS + 1) * sizeof(T) + (kStNT / 32) * kRegNV * 8; }
template <typename T>
constexpr size_t greg_z_smem() {
  return (kStNT / 32) * kEvalNV * 8 + 4 * (kTS + 2) * (kTS + 2) * sizeof(T) + 2 * (kTS + 1) * (kTS + 1) * sizeof(T);
}

// Regulariser gradient + omega (+ recorder terms when EVAL) for all rows of
// a job; x planes z-1, z, z+1 resident, z+2 in flight.
template <typename T, bool EVAL>
__global__ void __launch_bounds__(kStNT) greg_z_kernel(const __grid_constant__ StArgs<T> p) {
  constexpr int XP = kTS + 2;        // rows/cols y0-1 .. y0+32
  constexpr int PL = XP * XP;
  constexpr int RING = 4;
  constexpr int PP = kTS + 1;        // px/py rows/cols y0-1 .. y0+31
  extern __shared__ __align__(128) unsigned char st_smem[];
  double* red = reinterpret_cast<double*>(st_smem);  // (kStNT/32)*kEvalNV doubles
  T (*xs)[PL] = reinterpret_cast<T (*)[PL]>(st_smem + (kStNT / 32) * kEvalNV * 8);
  T* pxs = reinterpret_cast<T*>(st_smem + (kStNT / 32) * kEvalNV * 8 + RING * PL * sizeof(T));
  T* pys = pxs + PP * PP;
  const StJob<T>& J = p.jobs[blockIdx.z];
  const int x0 = blockIdx.x * kTS, y0 = blockIdx.y * kTS;
  const int tx = threadIdx.x % kTS, ty = threadIdx.x / kTS;
  const T d2 = (T)p.delta2;
  const T two_eta = (T)p.two_eta, lam = (T)p.lam, two_kappa = (T)p.two_kappa;
  const T xmin = (T)p.x_min, xmax = (T)p.x_max;
  // ring slot of depth z (planes lo-1 .. hi+1 may be loaded)
  auto slot = [&](int z) { return (z - J.lo + 1) % RING; };
  auto load = [&](int z) {
    st_load_async<T, XP, XP, XP>(xs[slot(z)], J.a + (long long)(z - J.a_z0) * p.plane, y0, x0, -1, -1, p.ny, p.nx);
    cp_async_commit();
  };
  const int zfirst = max(J.lo - 1, 0), zlast = min(J.hi + 1, p.nz - 1);
  int loaded = zfirst - 1;  // highest depth issued
  while (loaded < min(J.lo + 1, zlast)) load(++loaded);
  double ev[kEvalNV] = {0.0, 0.0, 0.0, 0.0, 0.0};
  for (int z = J.lo; z <= J.hi; ++z) {
    T sn[kStRows];
    if constexpr (EVAL) {
#pragma unroll
      for (int j = 0; j < kStRows; ++j) {
        const int y = y0 + ty + j * (kStNT / kTS), x = x0 + tx;
        sn[j] = (J.b && y < p.ny && x < p.nx) ? J.b[(long long)(z - J.lo) * p.plane + (long long)y * p.nx + x] : T(0);
      }
    }
    if (loaded < zlast && loaded < z + 2) load(++loaded);  // prefetch z+2
    if (loaded > z + 1) cp_async_wait<1>();
    else cp_async_wait<0>();
    __syncthreads();
    const T* xc_t = xs[slot(z)];
    const long long orow = (long long)(z - J.lo) * p.plane;
    for (int i = threadIdx.x; i < PP * PP; i += kStNT) {
      const int r = i / PP, c = i - r * PP;
      const int y = y0 - 1 + r, x = x0 - 1 + c;
      T px = T(0), py = T(0);
      if (y >= 0 && y < p.ny && x >= 0 && x < p.nx) {
        const T xc = xc_t[r * XP + c];
        const T dx = (x < p.nx - 1) ? sub_rn(xc_t[r * XP + c + 1], xc) : T(0);
        const T dy = (y < p.ny - 1) ? sub_rn(xc_t[(r + 1) * XP + c], xc) : T(0);
        const T sq = add_rn(add_rn(mul_rn(dx, dx), mul_rn(dy, dy)), d2);
        const T w = rsqrt(sq);  // = omega_of(dx, dy, d2)
        px = mul_rn(w, dx);
        py = mul_rn(w, dy);
        if (r >= 1 && c >= 1) {
          J.out1[orow + (long long)y * p.nx + x] = w;
          if (EVAL) ev[1] += (double)sq * (double)w;
        }
      }
      pxs[i] = px;
      pys[i] = py;
    }
    __syncthreads();
    const T* xm_t = xs[slot(z - 1)];
    const T* xp_t = xs[slot(z + 1)];
#pragma unroll
    for (int j = 0; j < kStRows; ++j) {
      const int ly = ty + j * (kStNT / kTS);
      const int y = y0 + ly, x = x0 + tx;
      if (y >= p.ny || x >= p.nx) continue;
      const int r = ly + 1, c = tx + 1;
      const T xc = xc_t[r * XP + c];
      const T clipped = xc < xmin ? xmin : (xc > xmax ? xmax : xc);
      const T box = mul_rn(two_eta, sub_rn(xc, clipped));
      const T px0 = pxs[r * PP + c], pxm = pxs[r * PP + c - 1];
      const T py0 = pys[r * PP + c], pym = pys[(r - 1) * PP + c];
      const T tvx = (p.nx == 1) ? T(0) : (x == 0) ? -px0 : (x == p.nx - 1) ? pxm : sub_rn(pxm, px0);
      const T tvy = (p.ny == 1) ? T(0) : (y == 0) ? -py0 : (y == p.ny - 1) ? pym : sub_rn(pym, py0);
      const T xzp = (z < p.nz - 1) ? xp_t[r * XP + c] : T(0);
      const T dzm = (z - 1 >= 0 && z - 1 < p.nz - 1) ? sub_rn(xc, xm_t[r * XP + c]) : T(0);
      const T dzp = (z < p.nz - 1) ? sub_rn(xzp, xc) : T(0);
      J.out0[orow + (long long)y * p.nx + x] =
          add_rn(add_rn(box, mul_rn(lam, add_rn(tvx, tvy))), mul_rn(two_kappa, sub_rn(dzm, dzp)));
      if constexpr (EVAL) {
        const double e = (double)xc - (double)clipped;
        ev[0] += e * e;
        if (z < p.nz - 1) ev[2] += ((double)xzp - (double)xc) * ((double)xzp - (double)xc);
        if (J.b) {
          ev[3] += ((double)xc - (double)sn[j]) * ((double)xc - (double)sn[j]);
          ev[4] += (double)sn[j] * (double)sn[j];
        }
        if (J.snap_out) J.snap_out[orow + (long long)y * p.nx + x] = xc;
      }
    }
    __syncthreads();  // ring slot of z-1 is refilled next iteration; px/py rewritten
  }
  if constexpr (EVAL) {
    cta_reduce<kEvalNV, kStNT>(ev, red);
    if (threadIdx.x == 0) {
      const long long cta = ((long long)blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
#pragma unroll
      for (int k = 0; k < kEvalNV; ++k) p.partials[cta * kEvalNV + k] = ev[k];
    }
  }
}

}  // namespace bd3mg
