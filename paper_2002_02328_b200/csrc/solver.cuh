// HBM-bound kernels of the BD3MG block step: regulariser Gram terms, the
// per-block 2x2 memory-gradient solve, the in-place block update, the
// elementwise objective terms, the majorant regulariser epilogue, and the
// deterministic two-level reductions that feed them.
#pragma once

#include "stencil.cuh"

namespace bd3mg {

constexpr int kEwNT = 256;           // threads per CTA, elementwise kernels
constexpr int kInfoNV = 16;          // doubles of StepInfo per block

// ---------------------------------------------------------------------------
// Deterministic final reduction: out[j*nv + k] = sum_{r in [begin_j, end_j)}
// rows[r*nv + k], each thread summing a fixed stride class in order, then a
// fixed tree (cta_sum_rows).  One CTA per job.
struct RowRanges {
  int njobs;
  long long begin[kMaxJobs];
  long long end[kMaxJobs];
};

constexpr int kRedMaxNV = 12;
// Deterministic CTA sum of rows[begin:end, 0:nv]: fixed stride classes per
// thread, a butterfly over the warp (a + b == b + a bitwise, so every lane
// holds the same sum), then the 8 warp sums in warp order.  Result in
// res[0:nv] for every thread (after the barrier).  Latency: 5 shuffles and
// one barrier instead of an 8-level shared-memory tree.
static __device__ __forceinline__ void cta_sum_rows(const double* __restrict__ rows, int nv, long long begin,
                                             long long end, double (*s)[kEwNT / 32], double* res) {
  constexpr int NW = kEwNT / 32;
  double acc[kRedMaxNV];
#pragma unroll
  for (int k = 0; k < kRedMaxNV; ++k) acc[k] = 0.0;
  for (long long r = begin + threadIdx.x; r < end; r += kEwNT) {
#pragma unroll
    for (int k = 0; k < kRedMaxNV; ++k)
      if (k < nv) acc[k] += rows[r * nv + k];
  }
#pragma unroll
  for (int k = 0; k < kRedMaxNV; ++k) {
    if (k < nv) {
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) acc[k] += __shfl_xor_sync(0xffffffffu, acc[k], off);
    }
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) {
#pragma unroll
    for (int k = 0; k < kRedMaxNV; ++k)
      if (k < nv) s[k][warp] = acc[k];
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < kRedMaxNV; ++k) {
    if (k < nv) {
      double t = s[k][0];
#pragma unroll
      for (int w = 1; w < NW; ++w) t += s[k][w];
      res[k] = t;
    }
  }
  __syncthreads();
}

static __global__ void __launch_bounds__(kEwNT) reduce_rows_kernel(const double* __restrict__ rows, int nv,
                                                            const __grid_constant__ RowRanges rr,
                                                            double* __restrict__ out, int out_stride) {
  __shared__ double s[kRedMaxNV][kEwNT / 32];
  double res[kRedMaxNV];
  const int j = blockIdx.x;
  cta_sum_rows(rows, nv, rr.begin[j], rr.end[j], s, res);
  if (threadIdx.x == 0)
    for (int k = 0; k < nv; ++k) out[j * out_stride + k] = res[k];
}

// ---------------------------------------------------------------------------
// 2x2 symmetric pseudo-inverse (reference directions.py:43-54): eigenvalues
// with |lambda| <= 1e-12 * max|lambda| are dropped.  Stable Jacobi rotation.
BD3MG_D void pinv_sym2(double a, double b, double c, double tol_rel, double& pa, double& pb, double& pc) {
  double l1, l2, cs, sn;
  if (b == 0.0) {
    l1 = a; l2 = c; cs = 1.0; sn = 0.0;
  } else {
    const double th = (c - a) / (2.0 * b);
    double t;
    if (fabs(th) > 1e150) t = 0.5 / th;
    else t = (th >= 0.0 ? 1.0 : -1.0) / (fabs(th) + sqrt(1.0 + th * th));
    cs = 1.0 / sqrt(1.0 + t * t);
    sn = t * cs;
    l1 = a - t * b;
    l2 = c + t * b;
  }
  // eigenvectors v1 = (cs, -sn), v2 = (sn, cs)
  const double amax = fmax(fabs(l1), fabs(l2));
  if (amax == 0.0) { pa = pb = pc = 0.0; return; }
  const double i1 = fabs(l1) > tol_rel * amax ? 1.0 / l1 : 0.0;
  const double i2 = fabs(l2) > tol_rel * amax ? 1.0 / l2 : 0.0;
  pa = cs * cs * i1 + sn * sn * i2;
  pb = -cs * sn * i1 + sn * cs * i2;
  pc = sn * sn * i1 + cs * cs * i2;
}

struct SolveArgs {
  int nblocks;
  double two_eta, lam, two_kappa;
  double prune_tol, pinv_tol;
  int has_d[kMaxJobs];
  // fused reduce + solve: partial-row ranges of each block
  int nv_gram;                       // 1 (GRAM1) or 3 values per conv partial row
  long long g_begin[kMaxJobs], g_end[kMaxJobs];
  long long r_begin[kMaxJobs], r_end[kMaxJobs];
};

// info layout per block (kInfoNV doubles):
// 0-2 gram (00,01,11 of the kept columns; 1 column -> [0]), 3-4 rhs,
// 5-6 coeffs, 7 ncols, 8 status (0 ok, 1 non-finite g, 2 non-finite increment), 9 |g|, 10 c_g
// (coefficient of -g), 11 c_d (coefficient of d), 12 column mask (1:-g, 2:d)
static __device__ void solve_one(const SolveArgs& p, int j, const double* D, const double* R, double* o) {
  for (int k = 0; k < kInfoNV; ++k) o[k] = 0.0;
  const double gg = R[0], dd = R[2], gd = R[9];
  const double gn = sqrt(gg);
  o[9] = gn;
  if (R[11] > 0.0) { o[8] = 1.0; return; }      // non-finite gradient
  if (R[10] == 0.0) return;                      // g == 0: zero step
  const double tol = p.prune_tol * (1.0 + gn);
  const bool k0 = gn > tol;
  const bool k1 = p.has_d[j] && sqrt(dd) > tol;
  const int ncols = (int)k0 + (int)k1;
  o[7] = ncols;
  o[12] = (k0 ? 1 : 0) + (k1 ? 2 : 0);
  if (ncols == 0) return;
  // full 2x2 for columns [-g, d]; data part <H b_i, H b_j> (H(-g) = -Hg)
  const double G00 = D[0] + p.two_eta * R[0] + p.lam * R[3] + p.two_kappa * R[6];
  const double G01 = -D[1] + p.two_eta * R[1] + p.lam * R[4] + p.two_kappa * R[7];
  const double G11 = D[2] + p.two_eta * R[2] + p.lam * R[5] + p.two_kappa * R[8];
  const double r0 = -gg, r1 = gd;
  double cg = 0.0, cd = 0.0;
  if (ncols == 2) {
    double pa, pb, pc;
    pinv_sym2(G00, G01, G11, p.pinv_tol, pa, pb, pc);
    cg = -(pa * r0 + pb * r1);
    cd = -(pb * r0 + pc * r1);
    o[0] = G00; o[1] = G01; o[2] = G11; o[3] = r0; o[4] = r1; o[5] = cg; o[6] = cd;
  } else {
    const double G = k0 ? G00 : G11, r = k0 ? r0 : r1;
    const double pinv = (G != 0.0 && fabs(G) > p.pinv_tol * fabs(G)) ? 1.0 / G : 0.0;
    const double cf = -(pinv * r);
    if (k0) cg = cf; else cd = cf;
    o[0] = G; o[3] = r; o[5] = cf;
  }
  o[10] = cg;
  o[11] = cd;
  // a finite gradient whose solve overflowed: the increment would be
  // non-finite (the reference master refuses it, scheduler.py:147-148);
  // status 2, nothing applied
  if (!isfinite(cg) || !isfinite(cd)) o[8] = 2.0;
}

// One CTA per block: reduce its conv and regulariser partial rows (same
// deterministic order per value as reduce_rows_kernel: fixed stride classes
// per thread, warp butterfly, warps in order), then the 2x2 solve.  Both row
// sets are summed in ONE pass -- their loads are issued together and all 15
// values share the butterfly and the barrier -- because this launch sits on
// the critical path of every block step and is pure latency.
static __global__ void __launch_bounds__(kEwNT) reduce_solve_kernel(const __grid_constant__ SolveArgs p,
                                                             const double* __restrict__ gram_rows,
                                                             const double* __restrict__ reg_rows,
                                                             double* __restrict__ info) {
  constexpr int NW = kEwNT / 32, NG = 3, NR = kRegNV;
  __shared__ double s[NG + NR][NW];
  const int j = blockIdx.x;
  const int nvg = p.nv_gram;
  double aD[NG], aR[NR];
#pragma unroll
  for (int k = 0; k < NG; ++k) aD[k] = 0.0;
#pragma unroll
  for (int k = 0; k < NR; ++k) aR[k] = 0.0;
  long long rg = p.g_begin[j] + threadIdx.x, rr = p.r_begin[j] + threadIdx.x;
  const long long eg = p.g_end[j], er = p.r_end[j];
  while (rg < eg || rr < er) {
    double vD[NG], vR[NR];
    const bool hg = rg < eg, hr = rr < er;
#pragma unroll
    for (int k = 0; k < NG; ++k) vD[k] = (hg && k < nvg) ? gram_rows[rg * nvg + k] : 0.0;
#pragma unroll
    for (int k = 0; k < NR; ++k) vR[k] = hr ? reg_rows[rr * NR + k] : 0.0;
    if (hg) {
#pragma unroll
      for (int k = 0; k < NG; ++k)
        if (k < nvg) aD[k] += vD[k];
    }
    if (hr) {
#pragma unroll
      for (int k = 0; k < NR; ++k) aR[k] += vR[k];
    }
    rg += kEwNT;
    rr += kEwNT;
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
#pragma unroll
    for (int k = 0; k < NG; ++k) aD[k] += __shfl_xor_sync(0xffffffffu, aD[k], off);
#pragma unroll
    for (int k = 0; k < NR; ++k) aR[k] += __shfl_xor_sync(0xffffffffu, aR[k], off);
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) {
#pragma unroll
    for (int k = 0; k < NG; ++k) s[k][warp] = aD[k];
#pragma unroll
    for (int k = 0; k < NR; ++k) s[NG + k][warp] = aR[k];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double D[kRedMaxNV], R[kRedMaxNV];
#pragma unroll
    for (int k = 0; k < NG; ++k) {
      double t = s[k][0];
#pragma unroll
      for (int w = 1; w < NW; ++w) t += s[k][w];
      D[k] = k < nvg ? t : 0.0;
    }
#pragma unroll
    for (int k = 0; k < NR; ++k) {
      double t = s[NG + k][0];
#pragma unroll
      for (int w = 1; w < NW; ++w) t += s[NG + k][w];
      R[k] = t;
    }
    solve_one(p, j, D, R, info + j * kInfoNV);
  }
}

// ---------------------------------------------------------------------------
// increment = c_g * (-g) + c_d * d  (reference directions.py:86), optionally
// applied in place: x_S += inc; d_mem_S = inc (scheduler.py:151-153).
template <typename T>
struct UpdBlock {
  const T* g;
  const T* d;      // may be null
  T* inc_out;      // may be null
  T* x;            // block rows of the iterate, may be null
  T* dmem;         // block rows of the memory store, may be null
  long long n;
  int ctas;
};
template <typename T>
struct UpdArgs {
  int nblocks;
  // the sweep's recorder terms (eval_finalize_kernel), folded into this launch
  const double* fin_sums;  // [data sum, ew5...] or null
  double* fin_terms;
  double fin_eta, fin_lam, fin_kappa;
  UpdBlock<T> blk[kMaxJobs];
};

// Mirrored rows of the updated iterate: elements [a, b) of block `blk` are
// also stored to dst[i - a] -- a peer GPU's halo inbox mapped over NVLink
// (cudaIpc), so the halo exchange of the sharded sweep rides on the update's
// own stores instead of a separate collective.
template <typename T>
struct MirSeg {
  T* dst;
  long long a, b;
  int blk;
};
constexpr int kMaxMirSegs = 64;
template <typename T, int NSEG>
struct MirArgs {
  int n;
  MirSeg<T> s[NSEG > 0 ? NSEG : 1];
};

template <typename T, int NSEG>
__device__ __forceinline__ void mirror_store(const MirArgs<T, NSEG>& m, long long i, T v) {
  if constexpr (NSEG > 0) {
    for (int j = 0; j < m.n; ++j) {
      const MirSeg<T>& s = m.s[j];
      if (s.blk == (int)blockIdx.y && i >= s.a && i < s.b) s.dst[i - s.a] = v;
    }
  }
}

template <typename T, int NSEG>
__global__ void __launch_bounds__(kEwNT) update_kernel(const __grid_constant__ UpdArgs<T> p,
                                                        const __grid_constant__ MirArgs<T, NSEG> m,
                                                        const double* __restrict__ info) {
  if (p.fin_terms && blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) {
    const double* sums = p.fin_sums;
    const double data = 0.5 * sums[0], box = p.fin_eta * sums[1], tv = p.fin_lam * sums[2], ax = p.fin_kappa * sums[3];
    double* t = p.fin_terms;
    t[0] = data; t[1] = box; t[2] = tv; t[3] = ax;
    t[4] = data + box + tv + ax;
    t[5] = sums[4]; t[6] = sums[5];
  }
  const UpdBlock<T>& B = p.blk[blockIdx.y];
  if ((int)blockIdx.x >= B.ctas) return;
  const double* o = info + blockIdx.y * kInfoNV;
  const long long i0 = (long long)blockIdx.x * kEwNT + threadIdx.x, di = (long long)B.ctas * kEwNT;
  if (o[8] != 0.0) {  // non-finite gradient: host raises, nothing applied (mirrors keep x current)
    if constexpr (NSEG > 0)
      if (B.x)
        for (long long i = i0; i < B.n; i += di) mirror_store(m, i, B.x[i]);
    return;
  }
  const T cg = (T)o[10], cd = (T)o[11];
  const bool has_d = B.d != nullptr;
  for (long long i = i0; i < B.n; i += di) {
    T inc = mul_rn(-B.g[i], cg);
    if (has_d) inc = add_rn(inc, mul_rn(B.d[i], cd));
    if (B.inc_out) B.inc_out[i] = inc;
    if (B.x) {
      const T xn = add_rn(B.x[i], inc);
      B.x[i] = xn;
      mirror_store(m, i, xn);
    }
    if (B.dmem) B.dmem[i] = inc;
  }
  if constexpr (NSEG > 0) __threadfence_system();  // peer stores ordered before the stream's next work
}

// terms: [data, box, tv, axial, f, |x-snap|^2, |snap|^2]
static __global__ void eval_finalize_kernel(const double* __restrict__ data1, const double* __restrict__ ew5,
                                     double eta, double lam, double kappa, double* __restrict__ terms) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  const double data = 0.5 * data1[0];
  const double box = eta * ew5[0];
  const double tv = lam * ew5[1];
  const double ax = kappa * ew5[2];
  terms[0] = data; terms[1] = box; terms[2] = tv; terms[3] = ax;
  terms[4] = data + box + tv + ax;
  terms[5] = ew5[3]; terms[6] = ew5[4];
}

// ---------------------------------------------------------------------------
// MajorantOperator.apply regulariser epilogue (objective.py:262-274), in place
// on out = (H^T H)_SS v:  out += 2eta v; out += lam(DxT(w Dx v)+DyT(w Dy v));
// out += 2kappa (dz[:-1]-dz[1:]) of the block-embedded v.
template <typename T>
struct MajArgs {
  const T* v;
  const T* omega;
  T* out;
  int lo, hi, nz, ny, nx;
  long long plane, n;
  double two_eta, lam, two_kappa;
  const double* gate;  // optional: no-op while *gate != 0 (krylov.cuh)
};

template <typename T>
__global__ void __launch_bounds__(kEwNT) majorant_reg_kernel(const __grid_constant__ MajArgs<T> p) {
  const long long i = (long long)blockIdx.x * kEwNT + threadIdx.x;
  if (i >= p.n || (p.gate && *p.gate != 0.0)) return;
  const int h = p.hi - p.lo + 1;
  const int t = (int)(i / p.plane);  // local plane
  const long long rem = i % p.plane;
  const int y = (int)(rem / p.nx), x = (int)(rem % p.nx);
  const XView<T> vv{p.v, 0, h, p.ny, p.nx, p.plane};
  const XView<T> wv{p.omega, 0, h, p.ny, p.nx, p.plane};
  const T vc = vv.at(t, y, x);
  T o = add_rn(p.out[i], mul_rn((T)p.two_eta, vc));
  const T px0 = mul_rn(wv.at(t, y, x), fdx(vv, t, y, x));
  const T py0 = mul_rn(wv.at(t, y, x), fdy(vv, t, y, x));
  T tvx, tvy;
  if (p.nx == 1) tvx = T(0);
  else if (x == 0) tvx = -px0;
  else {
    const T pxm = mul_rn(wv.at(t, y, x - 1), fdx(vv, t, y, x - 1));
    tvx = (x == p.nx - 1) ? pxm : sub_rn(pxm, px0);
  }
  if (p.ny == 1) tvy = T(0);
  else if (y == 0) tvy = -py0;
  else {
    const T pym = mul_rn(wv.at(t, y - 1, x), fdy(vv, t, y - 1, x));
    tvy = (y == p.ny - 1) ? pym : sub_rn(pym, py0);
  }
  o = add_rn(o, mul_rn((T)p.lam, add_rn(tvx, tvy)));
  // dz over global rows [lo-1, hi] of the embedded vector (objective.py:267-273)
  T dzm, dzp;
  if (t == 0) dzm = (p.lo - 1 >= 0) ? vc : T(0);
  else dzm = sub_rn(vc, vv.at(t - 1, y, x));
  if (t == h - 1) dzp = (p.hi < p.nz - 1) ? -vc : T(0);
  else dzp = sub_rn(vv.at(t + 1, y, x), vc);
  o = add_rn(o, mul_rn((T)p.two_kappa, sub_rn(dzm, dzp)));
  p.out[i] = o;
}

// Cached H E_S d_mem for the next visit: H E_S inc = c_g * H E_S(-g) + c_d * H E_S d
// (linearity), over the block's output rows.  hd: rows [olo, ohi] per block.
template <typename T>
struct HdBlock {
  const T* hg;  // H E_S g rows
  T* hd;        // cache rows (in: H E_S d_mem, out: H E_S increment)
  long long n;
  int ctas;
};
template <typename T>
struct HdArgs {
  int nblocks;
  HdBlock<T> blk[kMaxJobs];
};
template <typename T>
__global__ void __launch_bounds__(kEwNT) hd_update_kernel(const __grid_constant__ HdArgs<T> p,
                                                           const double* __restrict__ info) {
  const HdBlock<T>& B = p.blk[blockIdx.y];
  if ((int)blockIdx.x >= B.ctas) return;
  const double* o = info + blockIdx.y * kInfoNV;
  if (o[8] != 0.0) return;
  const T cg = (T)o[10], cd = (T)o[11];
  for (long long i = (long long)blockIdx.x * kEwNT + threadIdx.x; i < B.n; i += (long long)B.ctas * kEwNT)
    B.hd[i] = add_rn(mul_rn(-B.hg[i], cg), mul_rn(B.hd[i], cd));
}

// Variant "hd-incremental": the residual r = H x - y of the anchor is kept
// across sweeps by linearity, r += sum_b H E_b inc_b, from the hd-cache rows
// the step has just updated (hd_b = H E_b inc_b over rows [olo_b, ohi_b]);
// contributions of overlapping blocks are added in block order.  A block
// whose gradient was non-finite applied nothing and adds nothing.
template <typename T>
struct RIncArgs {
  T* r;  // plane 0 = depth r_z0
  long long plane;
  int r_z0, u_lo, u_hi, nblocks;
  const T* hd[kMaxJobs];
  int olo[kMaxJobs], ohi[kMaxJobs];
};
template <typename T>
__global__ void __launch_bounds__(kEwNT) resid_inc_kernel(const __grid_constant__ RIncArgs<T> p,
                                                           const double* __restrict__ info) {
  const long long n = (long long)(p.u_hi - p.u_lo + 1) * p.plane;
  for (long long i = (long long)blockIdx.x * kEwNT + threadIdx.x; i < n; i += (long long)gridDim.x * kEwNT) {
    const int z = p.u_lo + (int)(i / p.plane);
    const long long q = i - (long long)(z - p.u_lo) * p.plane;
    T* rp = p.r + (long long)(z - p.r_z0) * p.plane + q;
    T v = *rp;
    for (int b = 0; b < p.nblocks; ++b)
      if (z >= p.olo[b] && z <= p.ohi[b] && info[b * kInfoNV + 8] == 0.0)
        v = add_rn(v, p.hd[b][(long long)(z - p.olo[b]) * p.plane + q]);
    *rp = v;
  }
}

// Sum of squares of n elements, one partial per CTA (fixed grid, fixed
// per-thread order, warp butterfly: deterministic).
template <typename T>
__global__ void __launch_bounds__(kEwNT) sumsq_kernel(const T* __restrict__ a, long long n,
                                                       double* __restrict__ partials) {
  __shared__ double s[kEwNT / 32];
  double acc = 0.0;
  for (long long i = (long long)blockIdx.x * kEwNT + threadIdx.x; i < n; i += (long long)gridDim.x * kEwNT) {
    const double v = (double)a[i];
    acc += v * v;
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
  if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = s[0];
    for (int w = 1; w < kEwNT / 32; ++w) t += s[w];
    partials[blockIdx.x] = t;
  }
}

// receive_update's block write (scheduler.py:151-153): x += inc; d_mem = inc.
template <typename T>
__global__ void __launch_bounds__(kEwNT) apply_increment_kernel(T* __restrict__ x, T* __restrict__ dmem,
                                                                 const T* __restrict__ inc, long long n) {
  for (long long i = (long long)blockIdx.x * kEwNT + threadIdx.x; i < n; i += (long long)gridDim.x * kEwNT) {
    const T v = inc[i];
    x[i] = add_rn(x[i], v);
    if (dmem) dmem[i] = v;
  }
}

// Half-quadratic weights of rows [lo, lo+n/plane) of a fragment
// (objective.py:130-132, cached by MajorantOperator.__init__ :233-235).
template <typename T>
__global__ void __launch_bounds__(kEwNT) omega_kernel(const __grid_constant__ XView<T> xv, int lo, long long n,
                                                       T delta2, T* __restrict__ out) {
  const long long i = (long long)blockIdx.x * kEwNT + threadIdx.x;
  if (i >= n) return;
  const int z = lo + (int)(i / xv.plane);
  const long long rem = i % xv.plane;
  const int y = (int)(rem / xv.nx), x = (int)(rem % xv.nx);
  out[i] = omega_of(fdx(xv, z, y, x), fdy(xv, z, y, x), delta2);
}

}  // namespace bd3mg
