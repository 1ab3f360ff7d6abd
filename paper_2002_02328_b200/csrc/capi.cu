// C ABI of the B200-native BD3MG hot path (declarations: include/bd3mg_b200.h).
//
// Orchestrates the kernels of depthvar.cuh / solver.cuh into the reference
// operators: H/H^T rows (_core.pyx), _grad_rows / eval_f /
// MajorantOperator.apply (objective.py), mg_direction (directions.py) and the
// block update of receive_update (scheduler.py).
#include <algorithm>
#include <climits>
#include <atomic>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <functional>
#include <mutex>
#include <queue>
#include <type_traits>
#include <string>
#include <vector>

#include <cudaTypedefs.h>

#include "../../include/bd3mg_b200.h"
#include "conv_dispatch.cuh"
#include "errors.h"
#include "krylov.cuh"
#include "sweep_pk.cuh"
#include "solver.cuh"
#include "stencil_tma.cuh"

using namespace bd3mg;

namespace {

thread_local std::string g_err;
std::atomic<long long> g_launches{0};  // kernels launched by this library
inline void launched(int n = 1) { g_launches.fetch_add(n, std::memory_order_relaxed); }

int fail(int code, const char* fmt, ...) __attribute__((format(printf, 2, 3)));
int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

#define CU(expr)                                                                              \
  do {                                                                                        \
    cudaError_t e__ = (expr);                                                                 \
    if (e__ != cudaSuccess) return fail(BD3MG_ECUDA, "%s: %s", #expr, cudaGetErrorString(e__)); \
  } while (0)

constexpr double kPruneTol = 1e-14;  // directions.py:19
constexpr int kSumsqCtas = 4 * 148;  // fixed grid of the recorder's sum of squares (deterministic)
constexpr double kPinvTol = 1e-12;   // directions.py:22

// Bump allocator over a caller workspace; measure mode sizes it.
struct Ws {
  char* base = nullptr;
  size_t cap = 0, off = 0;
  bool measure = true;
  template <typename U>
  U* take(size_t n) {
    off = (off + 255) & ~size_t(255);
    // measure mode hands out non-null placeholders: callers branch on
    // pointers (e.g. the recorder's residual sum), so sizing must see the
    // same pointers as the real call; they are never dereferenced
    U* p = measure ? reinterpret_cast<U*>(uintptr_t(4096) + off) : reinterpret_cast<U*>(base + off);
    off += n * sizeof(U);
    return p;
  }
  bool ok() const { return measure || off <= cap; }
};

// Ordered flag stores for the asynchronous halo rings: each store is
// preceded by a system-scope fence, so a host (or peer) that sees flag i
// also sees every earlier store of this stream -- the ring data the update
// kernel wrote over NVLink and the flags before i.
struct PubArgs {
  int n;
  volatile long long* word[BD3MG_MAX_FLAGS];
  long long value[BD3MG_MAX_FLAGS];
};
__global__ void publish_kernel(const __grid_constant__ PubArgs a) {
  for (int i = 0; i < a.n; ++i) {
    __threadfence_system();
    *a.word[i] = a.value[i];
  }
  __threadfence_system();
}

int ws_fail(const Ws& ws) {
  return fail(BD3MG_EWORKSPACE, "workspace too small: %zu bytes needed, %zu given", ws.off, ws.cap);
}

bool odd_pos(int64_t k) { return k >= 1 && (k % 2) == 1; }

int check_geom(const bd3mg_geom_t* g) {
  if (!g) return fail(BD3MG_EINVAL, "null geometry");
  if (g->nx < 1 || g->ny < 1 || g->nz < 1) return fail(BD3MG_EINVAL, "dimensions must be >= 1");
  if (!odd_pos(g->kx) || !odd_pos(g->ky) || !odd_pos(g->kz)) return fail(BD3MG_EINVAL, "kernel dims must be odd and >= 1");
  if (g->dtype != BD3MG_F64 && g->dtype != BD3MG_F32) return fail(BD3MG_EINVAL, "unknown dtype %d", g->dtype);
  if (g->nx * g->ny > (int64_t)1 << 31) return fail(BD3MG_EINVAL, "plane too large");
  return BD3MG_OK;
}

template <typename T>
ConvArgs<T> base_args(const bd3mg_geom_t* g, const bd3mg_reg_t* r, const T* K) {
  ConvArgs<T> a;
  memset(&a, 0, sizeof(a));
  a.K = K;
  a.nzk = (int)g->nz;
  a.kz = g->kz; a.ky = g->ky; a.kx = g->kx;
  a.ny = (int)g->ny; a.nx = (int)g->nx;
  a.plane = g->ny * g->nx;
  a.nz_global = (int)g->nz;
  if (r) {
    a.two_eta = 2.0 * r->eta;
    a.lam = r->lam;
    a.two_kappa = 2.0 * r->kappa;
    a.delta2 = r->delta * r->delta;
    a.x_min = r->x_min;
    a.x_max = r->x_max;
  }
  return a;
}

template <typename T>
StArgs<T> st_args(const bd3mg_geom_t* g, const bd3mg_reg_t* r) {
  StArgs<T> a;
  memset(&a, 0, sizeof(a));
  a.nz = (int)g->nz; a.ny = (int)g->ny; a.nx = (int)g->nx; a.plane = g->ny * g->nx;
  a.tiles_x = (int)((g->nx + kTS - 1) / kTS);
  a.tiles_y = (int)((g->ny + kTS - 1) / kTS);
  if (r) {
    a.two_eta = 2.0 * r->eta; a.lam = r->lam; a.two_kappa = 2.0 * r->kappa;
    a.delta2 = r->delta * r->delta; a.x_min = r->x_min; a.x_max = r->x_max;
  }
  return a;
}
inline long long st_tiles(const bd3mg_geom_t* g) { return ((g->nx + kTS - 1) / kTS) * ((g->ny + kTS - 1) / kTS); }

// One CTA column per job (z-marching kernels): grid.z = njobs.
template <typename T, typename Kern>
cudaError_t st_launch_z(Kern kern, StArgs<T>& a, size_t smem, cudaStream_t s) {
  if (a.njobs == 0) return cudaSuccess;
  cudaError_t e = ensure_smem_attr(kern, smem);
  if (e != cudaSuccess) return e;
  kern<<<dim3(a.tiles_x, a.tiles_y, a.njobs), kStNT, smem, s>>>(a);
  launched();
  return cudaGetLastError();
}

// TMA-staged stencils when every row is a whole number of 16-byte chunks.
template <typename T>
bool st_use_tma(long long nx) {
  static const bool off = getenv("BD3MG_NO_TMA") != nullptr;
  return !off && (nx * (long long)sizeof(T)) % 16 == 0;
}
// partial rows per job of the z-marching stencils (greg / reg_gram)
template <typename T>
long long z_tiles(const bd3mg_geom_t* g) {
  return st_use_tma<T>(g->nx) ? tm_tiles(g->ny, g->nx) : st_tiles(g);
}

// Regulariser gradient (+ omega, + recorder terms when `eval`) of every job.
constexpr size_t kGregPad = 8192;  // see launch_greg
template <typename T>
int launch_greg(StArgs<T>& a, bool eval, cudaStream_t s, size_t pad_hint = 0) {
  if (a.njobs == 0) return BD3MG_OK;
  if (!st_use_tma<T>(a.nx)) {
    CU(st_launch_z<T>(eval ? greg_z_kernel<T, true> : greg_z_kernel<T, false>, a, greg_z_smem<T>(), s));
    return BD3MG_OK;
  }
  using G = GregGeo<T>;
  static StTma<T> tm;  // host staging of the descriptors (copied into the launch)
  static std::mutex mu;
  std::lock_guard<std::mutex> lock(mu);
  for (int j = 0; j < a.njobs; ++j) {
    const StJob<T>& J = a.jobs[j];
    const long long zl = std::min<long long>(J.hi + 1, a.nz - 1);
    if (!encode_tmap(&tm.a[j], J.a, sizeof(T) == 8, a.nx, a.ny, zl - J.a_z0 + 1, G::BW, G::BH))
      return fail(BD3MG_EINVAL, "greg: TMA descriptor rejected (job %d)", j);
  }
  auto kern = eval ? greg_t_kernel<T, true> : greg_t_kernel<T, false>;
  // pad_hint: extra dynamic shared memory per CTA of the sweep's recorder stencil (when it runs next to a
  // residual correlation: the sweep passes kGregPad).  In fp64, 8 KB more make it 33 KB,
  // so at most four of its CTAs (not five or six) share an SM with a 76.7 KB correlation CTA of the
  // residual correlation's last wave, in which this stencil runs.  Measured at C2: 395.5 -> 390.0 us per
  // sweep (4 KB: 396, 14 KB: 398, 24 KB: 398-399, 50 KB: 402).  BD3MG_ST_PAD=<bytes> overrides.
  static const long pad_env = getenv("BD3MG_ST_PAD") ? atol(getenv("BD3MG_ST_PAD")) : -1;
  const size_t pad = pad_env >= 0 ? (size_t)pad_env : pad_hint;
  CU(ensure_smem_attr(kern, G::smem() + pad + 49 * 1024));
  kern<<<dim3((a.nx + kTmX - 1) / kTmX, (a.ny + kTmY - 1) / kTmY, a.njobs), kTmNT, G::smem() + pad, s>>>(a, tm);
  launched();
  CU(cudaGetLastError());
  return BD3MG_OK;
}

// Regulariser Gram terms of every job (a = g rows, b = d rows, w = omega rows).
template <typename T>
int launch_reg_gram(StArgs<T>& a, cudaStream_t s) {
  if (a.njobs == 0) return BD3MG_OK;
  if (!st_use_tma<T>(a.nx)) {
    CU(st_launch_z<T>(reg_gram_z_kernel<T>, a, reg_gram_z_smem<T>(), s));
    return BD3MG_OK;
  }
  using G = RgGeo<T>;
  static StTma<T> tm;
  static std::mutex mu;
  std::lock_guard<std::mutex> lock(mu);
  for (int j = 0; j < a.njobs; ++j) {
    const StJob<T>& J = a.jobs[j];
    const long long h = (J.chunk && J.hi < J.bhi ? J.hi + 1 : J.hi) - J.lo + 1;  // chunks stage one plane more
    if (!encode_tmap(&tm.a[j], J.a, sizeof(T) == 8, a.nx, a.ny, h, G::BW, G::BH) ||
        (J.b && !encode_tmap(&tm.b[j], J.b, sizeof(T) == 8, a.nx, a.ny, h, G::BW, G::BH)))
      return fail(BD3MG_EINVAL, "reg_gram: TMA descriptor rejected (job %d)", j);
  }
  // extra dynamic shared memory per CTA, as for the recorder stencil (launch_greg): measured for the fp32
  // sweeps, where this stencil runs next to the Gram correlation (C2 fp32 278.8 -> 277.6 us, C3 3769 ->
  // 3753 us at +8 KB; +16 KB and more are slower).  BD3MG_RG_PAD=<bytes> overrides.
  static const long pad_env = getenv("BD3MG_RG_PAD") ? atol(getenv("BD3MG_RG_PAD")) : -1;
  const size_t pad = pad_env >= 0 ? (size_t)pad_env : (sizeof(T) == 4 ? kGregPad : 0);
  CU(ensure_smem_attr(reg_gram_t_kernel<T>, G::smem() + pad + 49 * 1024));
  reg_gram_t_kernel<T><<<dim3((a.nx + kTmX - 1) / kTmX, (a.ny + kTmY - 1) / kTmY, a.njobs), kTmNT, G::smem() + pad, s>>>(a, tm);
  launched();
  CU(cudaGetLastError());
  return BD3MG_OK;
}

// Lay jobs out along grid.z (one plane per z index) and launch `kern`.
template <typename T, typename Kern>
cudaError_t st_launch(Kern kern, StArgs<T>& a, cudaStream_t s) {
  int wb = 0;
  for (int j = 0; j < a.njobs; ++j) {
    a.jobs[j].work_begin = wb;
    wb += a.jobs[j].hi - a.jobs[j].lo + 1;
  }
  if (wb == 0) return cudaSuccess;
  kern<<<dim3(a.tiles_x, a.tiles_y, wb), kStNT, 0, s>>>(a);
  launched();
  return cudaGetLastError();
}

// partial rows (one per CTA) of a conv launch over one job of `nout` planes
template <typename T>
long long conv_tiles(const bd3mg_geom_t* g, int mode) {
  const ConvGrid cg = conv_grid<T>(g->ky, g->kx, mode, (int)g->ny, (int)g->nx);
  return (long long)cg.tiles_x * cg.tiles_y;
}
template <typename T>
long long conv_rows(const bd3mg_geom_t* g, int mode, long long nout) {
  return conv_zunits<T>(g->ky, g->kx, mode, nout) * conv_tiles<T>(g, mode);
}

cudaError_t reduce(const double* rows, int nv, const std::vector<std::pair<long long, long long>>& ranges,
                   double* out, int out_stride, cudaStream_t s) {
  for (size_t b0 = 0; b0 < ranges.size(); b0 += kMaxJobs) {
    RowRanges rr;
    memset(&rr, 0, sizeof(rr));
    rr.njobs = (int)std::min<size_t>(kMaxJobs, ranges.size() - b0);
    for (int j = 0; j < rr.njobs; ++j) {
      rr.begin[j] = ranges[b0 + j].first;
      rr.end[j] = ranges[b0 + j].second;
    }
    reduce_rows_kernel<<<rr.njobs, kEwNT, 0, s>>>(rows, nv, rr, out + b0 * out_stride, out_stride);
    launched();
  }
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
template <typename T>
int correlate_rows(const T* frag, int64_t nzf, int64_t ny, int64_t nx, const T* K, int64_t nzk, int64_t kz,
                   int64_t ky, int64_t kx, int64_t frag_z0, int64_t out_lo, int64_t out_hi, T* out, bool adj,
                   cudaStream_t s) {
  if (!odd_pos(kz) || !odd_pos(ky) || !odd_pos(kx)) return fail(BD3MG_EINVAL, "kernel dims must be odd and >= 1");
  if (ny < 1 || nx < 1 || nzf < 1 || nzk < 1) return fail(BD3MG_EINVAL, "empty fragment or kernel stack");
  const int64_t nout = out_hi - out_lo + 1;
  if (nout < 0) return fail(BD3MG_EINVAL, "out_hi < out_lo - 1");
  if (nout == 0) return BD3MG_OK;
  if (out_lo < 0) return fail(BD3MG_EINVAL, "out_lo < 0");
  if (!adj && out_hi >= nzk) return fail(BD3MG_EINVAL, "output row %lld outside the kernel stack (nz=%lld)",
                                         (long long)out_hi, (long long)nzk);
  bd3mg_geom_t g{nx, ny, nzk, (int32_t)kx, (int32_t)ky, (int32_t)kz, 0};
  ConvArgs<T> a = base_args<T>(&g, nullptr, K);
  a.njobs = 1;
  ConvJob<T>& j = a.jobs[0];
  j.src0 = frag; j.src_z0 = frag_z0; j.src_nz = (int)nzf;
  j.dst0 = out; j.out_lo = (int)out_lo; j.nout = (int)nout; j.work_begin = 0;
  CU(conv_launch<T>(M_STORE, adj, a, (int)nout, s));
  launched();
  return BD3MG_OK;
}

// ---------------------------------------------------------------------------
template <typename T>
int grad_rows_impl(const bd3mg_geom_t* g, const bd3mg_reg_t* r, const T* K, const T* y, const T* frag,
                   int64_t frag_z0, int64_t nzf, int64_t lo, int64_t hi, T* g_out, T* omega_out, Ws& ws,
                   cudaStream_t s) {
  const int64_t nz = g->nz, plane = g->ny * g->nx, rz = (g->kz - 1) / 2;
  if (lo < 0 || hi < lo || hi >= nz) return fail(BD3MG_EINVAL, "invalid rows [%lld, %lld]", (long long)lo, (long long)hi);
  const int64_t need_lo = std::max<int64_t>(0, lo - 1), need_hi = std::min<int64_t>(nz - 1, hi + 1);
  if (frag_z0 > need_lo || frag_z0 + nzf - 1 < need_hi)
    return fail(BD3MG_EINVAL, "fragment [%lld, %lld] does not cover the stencil rows [%lld, %lld]",
                (long long)frag_z0, (long long)(frag_z0 + nzf - 1), (long long)need_lo, (long long)need_hi);
  const int64_t o_lo = std::max<int64_t>(0, lo - rz), o_hi = std::min<int64_t>(nz - 1, hi + rz);
  const int64_t nr = o_hi - o_lo + 1, h = hi - lo + 1;
  T* rbuf = ws.take<T>(nr * plane);
  T* greg = ws.take<T>(h * plane);
  double* parts = ws.take<double>(conv_rows<T>(g, M_RESID, nr));
  if (ws.measure) return BD3MG_OK;
  if (!ws.ok()) return ws_fail(ws);
  {
    StArgs<T> sa = st_args<T>(g, r);
    sa.njobs = 1;
    sa.jobs[0].a = frag; sa.jobs[0].a_z0 = frag_z0; sa.jobs[0].lo = (int)lo; sa.jobs[0].hi = (int)hi;
    sa.jobs[0].out0 = greg; sa.jobs[0].out1 = omega_out;
    int rc = launch_greg<T>(sa, false, s);
    if (rc) return rc;
  }
  ConvArgs<T> a = base_args<T>(g, r, K);
  a.njobs = 1;
  a.partials = parts;
  a.jobs[0].src0 = frag; a.jobs[0].src_z0 = frag_z0; a.jobs[0].src_nz = (int)nzf;
  a.jobs[0].dst0 = rbuf; a.jobs[0].sub = y + o_lo * plane;
  a.jobs[0].out_lo = (int)o_lo; a.jobs[0].nout = (int)nr;
  CU(conv_launch<T>(M_RESID, false, a, (int)nr, s));
  launched();
  ConvArgs<T> b = base_args<T>(g, r, K);
  b.njobs = 1;
  ConvJob<T>& j = b.jobs[0];
  j.src0 = rbuf; j.src_z0 = o_lo; j.src_nz = (int)nr;
  j.dst0 = g_out; j.sub = greg;
  j.out_lo = (int)lo; j.nout = (int)h;
  CU(conv_launch<T>(M_GRAD, true, b, (int)h, s));
  launched();
  return BD3MG_OK;
}

// Objective terms over rows [lo, hi] from a fragment covering [lo-2rz, hi+2rz]
// (clamped): data term of H rows minus y rows, box / TV / axial over the rows.
template <typename T>
int eval_rows_impl(const bd3mg_geom_t* g, const bd3mg_reg_t* r, const T* K, const T* y_rows, const T* frag,
                   int64_t frag_z0, int64_t nzf, int64_t lo, int64_t hi, const T* snap_rows, double* terms, Ws& ws,
                   cudaStream_t s, const T* resid_rows = nullptr) {
  const int64_t nz = g->nz, plane = g->ny * g->nx;
  if (lo < 0 || hi < lo || hi >= nz) return fail(BD3MG_EINVAL, "invalid rows [%lld, %lld]", (long long)lo, (long long)hi);
  const int64_t need_hi = std::min<int64_t>(nz - 1, hi + 1);
  if (frag_z0 > lo || frag_z0 + nzf - 1 < need_hi)
    return fail(BD3MG_EINVAL, "fragment does not cover rows [%lld, %lld]", (long long)lo, (long long)need_hi);
  const int64_t nr = hi - lo + 1, n = nr * plane;
  const long long crow = conv_rows<T>(g, M_RESID, nr);
  double* parts = ws.take<double>(std::max<long long>(crow, kSumsqCtas));
  const long long erows = nr * st_tiles(g);
  double* eparts = ws.take<double>((size_t)erows * kEvalNV);
  double* sums = ws.take<double>(8);
  if (ws.measure) return BD3MG_OK;
  if (!ws.ok()) return ws_fail(ws);
  if (resid_rows) {  // data term from a kept residual (variant "hd-incremental")
    sumsq_kernel<T><<<kSumsqCtas, kEwNT, 0, s>>>(resid_rows, n, parts);
    launched();
    CU(cudaGetLastError());
    CU(reduce(parts, 1, {{0, kSumsqCtas}}, sums, 1, s));
  } else {
    ConvArgs<T> a = base_args<T>(g, r, K);
    a.njobs = 1;
    a.partials = parts;
    a.jobs[0].src0 = frag; a.jobs[0].src_z0 = frag_z0; a.jobs[0].src_nz = (int)nzf;
    a.jobs[0].dst0 = nullptr; a.jobs[0].sub = y_rows;
    a.jobs[0].out_lo = (int)lo; a.jobs[0].nout = (int)nr;
    CU(conv_launch<T>(M_RESID, false, a, (int)nr, s));
    launched();
    CU(reduce(parts, 1, {{0, crow}}, sums, 1, s));
  }
  StArgs<T> e = st_args<T>(g, r);
  e.njobs = 1;
  e.jobs[0].a = frag; e.jobs[0].a_z0 = frag_z0; e.jobs[0].b = snap_rows; e.jobs[0].lo = (int)lo; e.jobs[0].hi = (int)hi;
  e.partials = eparts;
  CU(st_launch<T>(eval_kernel<T>, e, s));
  CU(reduce(eparts, kEvalNV, {{0, erows}}, sums + 1, kEvalNV, s));
  eval_finalize_kernel<<<1, 1, 0, s>>>(sums, sums + 1, r->eta, r->lam, r->kappa, terms); launched();
  CU(cudaGetLastError());
  return BD3MG_OK;
}

template <typename T>
int eval_f_impl(const bd3mg_geom_t* g, const bd3mg_reg_t* r, const T* K, const T* y, const T* x, const T* snap,
                double* terms, Ws& ws, cudaStream_t s) {
  return eval_rows_impl<T>(g, r, K, y, x, 0, g->nz, 0, g->nz - 1, snap, terms, ws, s);
}

template <typename T>
int majorant_impl(const bd3mg_geom_t* g, const bd3mg_reg_t* r, const T* K, const T* omega, const T* v, int64_t lo,
                  int64_t hi, T* out, Ws& ws, cudaStream_t s, const double* gate = nullptr) {
  const int64_t nz = g->nz, plane = g->ny * g->nx, rz = (g->kz - 1) / 2;
  if (lo < 0 || hi < lo || hi >= nz) return fail(BD3MG_EINVAL, "invalid block [%lld, %lld]", (long long)lo, (long long)hi);
  const int64_t o_lo = std::max<int64_t>(0, lo - rz), o_hi = std::min<int64_t>(nz - 1, hi + rz);
  const int64_t nr = o_hi - o_lo + 1, h = hi - lo + 1;
  T* hv = ws.take<T>(nr * plane);
  if (ws.measure) return BD3MG_OK;
  if (!ws.ok()) return ws_fail(ws);
  ConvArgs<T> a = base_args<T>(g, r, K);
  a.njobs = 1;
  a.gate = gate;
  a.jobs[0].src0 = v; a.jobs[0].src_z0 = lo; a.jobs[0].src_nz = (int)h;
  a.jobs[0].dst0 = hv; a.jobs[0].out_lo = (int)o_lo; a.jobs[0].nout = (int)nr;
  CU(conv_launch<T>(M_STORE, false, a, (int)nr, s));
  launched();
  ConvArgs<T> b = base_args<T>(g, r, K);
  b.njobs = 1;
  b.gate = gate;
  b.jobs[0].src0 = hv; b.jobs[0].src_z0 = o_lo; b.jobs[0].src_nz = (int)nr;
  b.jobs[0].dst0 = out; b.jobs[0].out_lo = (int)lo; b.jobs[0].nout = (int)h;
  CU(conv_launch<T>(M_STORE, true, b, (int)h, s));
  launched();
  MajArgs<T> m;
  m.v = v; m.omega = omega; m.out = out; m.lo = (int)lo; m.hi = (int)hi; m.nz = (int)nz;
  m.ny = (int)g->ny; m.nx = (int)g->nx; m.plane = plane; m.n = h * plane;
  m.two_eta = 2.0 * r->eta; m.lam = r->lam; m.two_kappa = 2.0 * r->kappa;
  m.gate = gate;
  majorant_reg_kernel<T><<<(unsigned)((m.n + kEwNT - 1) / kEwNT), kEwNT, 0, s>>>(m); launched();
  CU(cudaGetLastError());
  return BD3MG_OK;
}

template <typename T>
int omega_impl(const bd3mg_geom_t* g, const bd3mg_reg_t* r, const T* frag, int64_t frag_z0, int64_t nzf, int64_t lo,
               int64_t hi, T* out, cudaStream_t s) {
  if (lo < 0 || hi < lo || hi >= g->nz) return fail(BD3MG_EINVAL, "invalid rows [%lld, %lld]", (long long)lo, (long long)hi);
  if (frag_z0 > lo || frag_z0 + nzf - 1 < hi) return fail(BD3MG_EINVAL, "fragment does not cover the rows");
  const int64_t plane = g->ny * g->nx, n = (hi - lo + 1) * plane;
  XView<T> xv{frag, frag_z0, (int)nzf, (int)g->ny, (int)g->nx, plane};
  omega_kernel<T><<<(unsigned)((n + kEwNT - 1) / kEwNT), kEwNT, 0, s>>>(xv, (int)lo, n, (T)(r->delta * r->delta), out); launched();
  CU(cudaGetLastError());
  return BD3MG_OK;
}

// ---------------------------------------------------------------------------
// Device CG on the block majorant (reference directions.py:117-149) and the
// power iteration of rho(H^T H) (objective.py:345-370): see krylov.cuh.
// The host enqueues iterations without waiting on them; it only reads a
// host-mapped mirror of the iteration counter to stay at most kCgAhead
// iterations ahead of the device (and to stop enqueueing once the solve has
// stopped).  Inside a graph capture every iteration is enqueued (gated).
constexpr int kCgAhead = 3;

struct HostMirror {
  volatile double* h = nullptr;
  double* d = nullptr;
  int device = -1;
};
cudaError_t host_mirror(HostMirror** out) {
  thread_local HostMirror m;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (m.device != dev) {
    void* hp = nullptr;
    e = cudaHostAlloc(&hp, 64, cudaHostAllocMapped | cudaHostAllocPortable);
    if (e != cudaSuccess) return e;
    void* dp = nullptr;
    e = cudaHostGetDevicePointer(&dp, hp, 0);
    if (e != cudaSuccess) return e;
    m.h = (volatile double*)hp;
    m.d = (double*)dp;
    m.device = dev;
  }
  *out = &m;
  return cudaSuccess;
}

template <typename T>
int cg_solve_impl(const bd3mg_geom_t* g, const bd3mg_reg_t* r, const T* K, const T* omega, const T* b, int64_t lo,
                  int64_t hi, double tol, int maxit, T* x_out, double* state_out, Ws& ws, cudaStream_t s) {
  if (lo < 0 || hi < lo || hi >= g->nz) return fail(BD3MG_EINVAL, "invalid block [%lld, %lld]", (long long)lo, (long long)hi);
  if (maxit < 0) return fail(BD3MG_EINVAL, "negative iteration budget");
  const long long n = (hi - lo + 1) * g->ny * g->nx;
  CgVecs<T> v;
  v.n = n;
  v.b = b;
  v.x = ws.take<T>(n); v.r = ws.take<T>(n); v.p = ws.take<T>(n); v.ap = ws.take<T>(n); v.best = ws.take<T>(n);
  double* parts = ws.take<double>(kKryCtas);
  double* st = ws.take<double>(CG_NV);
  const size_t off_maj = ws.off;  // the majorant's own scratch follows, reused every iteration
  int rc = majorant_impl<T>(g, r, K, omega, v.p, lo, hi, v.ap, ws, s, st + CG_STATUS);
  if (rc || ws.measure) return rc;
  if (!ws.ok()) return ws_fail(ws);
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  CU(cudaStreamIsCapturing(s, &cap));
  HostMirror* hm = nullptr;
  if (cap == cudaStreamCaptureStatusNone) CU(host_mirror(&hm));
  volatile double* hmir = hm ? hm->h : nullptr;
  double* dmir = hm ? hm->d : nullptr;
  if (hmir) { hmir[0] = -1.0; hmir[1] = 0.0; }
  cg_init_kernel<T><<<kKryCtas, kEwNT, 0, s>>>(v, parts); launched();
  cg_init_state_kernel<<<1, kEwNT, 0, s>>>(parts, st, dmir); launched();
  CU(cudaGetLastError());
  for (int it = 1; it <= maxit; ++it) {
    Ws mw = ws;
    mw.off = off_maj;
    rc = majorant_impl<T>(g, r, K, omega, v.p, lo, hi, v.ap, mw, s, st + CG_STATUS);
    if (rc) return rc;
    cg_pap_kernel<T><<<kKryCtas, kEwNT, 0, s>>>(v, st, parts); launched();
    cg_alpha_kernel<<<1, kEwNT, 0, s>>>(parts, st); launched();
    cg_xr_kernel<T><<<kKryCtas, kEwNT, 0, s>>>(v, st, parts); launched();
    cg_check_kernel<<<1, kEwNT, 0, s>>>(parts, st, tol, maxit, dmir); launched();
    cg_p_kernel<T><<<kKryCtas, kEwNT, 0, s>>>(v, st); launched();
    CU(cudaGetLastError());
    if (hmir) {
      // stay at most kCgAhead iterations ahead; stop enqueueing once stopped
      while (hmir[1] == 0.0 && hmir[0] < (double)(it - kCgAhead)) {
        const cudaError_t q = cudaStreamQuery(s);
        if (q == cudaSuccess) break;  // drained: the mirror is final
        if (q != cudaErrorNotReady) return fail(BD3MG_ECUDA, "cg: %s", cudaGetErrorString(q));
      }
      if (hmir[1] != 0.0) break;
    }
  }
  cg_result_kernel<T><<<kKryCtas, kEwNT, 0, s>>>(v, st, x_out); launched();
  if (state_out) CU(cudaMemcpyAsync(state_out, st, CG_NV * sizeof(double), cudaMemcpyDeviceToDevice, s));
  CU(cudaGetLastError());
  return BD3MG_OK;
}

template <typename T>
int power_hth_impl(const bd3mg_geom_t* g, const T* K, T* v, int iters, double* norms, double* state_out, Ws& ws,
                   cudaStream_t s) {
  if (iters < 0) return fail(BD3MG_EINVAL, "negative iteration count");
  const long long n = g->nz * g->ny * g->nx;
  T* hv = ws.take<T>(n);
  T* w = ws.take<T>(n);
  double* parts = ws.take<double>(kKryCtas);
  double* st = ws.take<double>(2);
  if (ws.measure) return BD3MG_OK;
  if (!ws.ok()) return ws_fail(ws);
  CU(cudaMemsetAsync(st, 0, 2 * sizeof(double), s));
  for (int it = 0; it < iters; ++it) {
    ConvArgs<T> a = base_args<T>(g, nullptr, K);
    a.gate = st;
    a.njobs = 1;
    a.jobs[0].src0 = v; a.jobs[0].src_z0 = 0; a.jobs[0].src_nz = (int)g->nz;
    a.jobs[0].dst0 = hv; a.jobs[0].out_lo = 0; a.jobs[0].nout = (int)g->nz;
    CU(conv_launch<T>(M_STORE, false, a, (int)g->nz, s));
    launched();
    ConvArgs<T> b2 = base_args<T>(g, nullptr, K);
    b2.gate = st;
    b2.njobs = 1;
    b2.jobs[0].src0 = hv; b2.jobs[0].src_z0 = 0; b2.jobs[0].src_nz = (int)g->nz;
    b2.jobs[0].dst0 = w; b2.jobs[0].out_lo = 0; b2.jobs[0].nout = (int)g->nz;
    CU(conv_launch<T>(M_STORE, true, b2, (int)g->nz, s));
    launched();
    pw_norm_kernel<T><<<kKryCtas, kEwNT, 0, s>>>(w, n, st, parts); launched();
    pw_finish_kernel<<<1, kEwNT, 0, s>>>(parts, st, norms, it); launched();
    pw_scale_kernel<T><<<kKryCtas, kEwNT, 0, s>>>(w, v, n, st); launched();
    CU(cudaGetLastError());
  }
  if (state_out) CU(cudaMemcpyAsync(state_out, st, 2 * sizeof(double), cudaMemcpyDeviceToDevice, s));
  return BD3MG_OK;
}

// ---------------------------------------------------------------------------
// Batched mg_direction (+ optional in-place receive_update).
// A side stream (+ fork/join events) per (device, main stream): the sweep
// runs its HBM-bound stencils next to the FMA-bound correlations.  Event
// record / wait is legal inside CUDA-graph capture (the side stream joins the
// capture and is joined back before the sweep returns).
constexpr int kMaxParts = 4;  // GRAD -> GRAM -> solve -> update chains of a batched step
struct SideStream {
  // The block scheduler dispatches concurrent kernels of equal priority in launch order: a later
  // kernel's CTAs start only when the earlier kernel has none left to dispatch, i.e. in its last wave
  // (measured with scripts/sweep_timeline.py), so the streams overlap tails, not whole kernels.
  // BD3MG_SIDE_PRIO=hi gives the stencil stream a higher priority: eager launches then run the stencils
  // right after their producers, but torch's graph instantiation ignores node priorities and the sweep is
  // work-conserving either way (measured: +-1%), so equal priorities stay the default.
  cudaStream_t side = nullptr;             // stencils, recorder reductions
  cudaStream_t chain[kMaxParts - 1] = {};  // streams of the chains after the first (which stays on the caller's)
  cudaEvent_t ev[8 + 6 * kMaxParts] = {};
  // events 8..: per chain p  fork (8+5p), regulariser-Gram fork (9+5p), its join (10+5p), chain join (11+5p),
  // tail fork (12+5p); then kMaxParts "chain's regulariser gradient ready" events
};
cudaError_t side_stream(cudaStream_t main, SideStream** out) {
  static std::mutex mu;
  static std::map<std::pair<int, cudaStream_t>, SideStream> cache;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lock(mu);
  SideStream& ss = cache[{dev, main}];
  if (!ss.side) {
    int least = 0, greatest = 0;
    (void)cudaDeviceGetStreamPriorityRange(&least, &greatest);
    const char* pr = getenv("BD3MG_SIDE_PRIO");
    const int prio = (pr && pr[0] == 'h') ? greatest : 0;
    e = cudaStreamCreateWithPriority(&ss.side, cudaStreamNonBlocking, prio);
    for (int i = 0; i < kMaxParts - 1 && e == cudaSuccess; ++i)
      e = cudaStreamCreateWithFlags(&ss.chain[i], cudaStreamNonBlocking);
    for (int i = 0; i < 8 + 6 * kMaxParts && e == cudaSuccess; ++i)
      e = cudaEventCreateWithFlags(&ss.ev[i], cudaEventDisableTiming);
    if (e != cudaSuccess) return e;
  }
  *out = &ss;
  return cudaSuccess;
}
inline cudaError_t hop(cudaStream_t from, cudaStream_t to, cudaEvent_t ev) {
  cudaError_t e = cudaEventRecord(ev, from);
  return e == cudaSuccess ? cudaStreamWaitEvent(to, ev, 0) : e;
}

// Number of GRAD -> Gram -> solve -> update chains of a batched step of nt blocks (mg_steps_chunk);
// chain p covers blocks [nt * p / parts, nt * (p + 1) / parts).
// fp32: chains where the launches are short enough for their tails to matter -- measured with the
// per-chain residual and stencils: C2 fp32 +9.4%, C3 +0.8%, C4 +0.7%, C5 (2^29 voxels) -0.4% -- so up to
// 2^27 voxels per step.  `voxels`: rows x plane of the step's blocks.
template <typename T>
int chain_parts(bool side_stream, int nt, long long voxels) {
  const char* pe = getenv("BD3MG_PARTS");  // (read per call: the tests switch it)
  const int parts_env = pe ? atoi(pe) : 0;
  const bool dtype_ok = sizeof(T) == 8 || (voxels > 0 && voxels <= (1LL << 27) && !getenv("BD3MG_NO_CHAINS_F32"));
  int parts = (side_stream && nt >= 4 && dtype_ok && !getenv("BD3MG_NO_SPLIT")) ? 2 : 1;
  if (parts > 1 && parts_env > 0) parts = std::min(std::min(parts_env, kMaxParts), nt);
  return parts;
}

// Options of the batched step used by the sweep driver.
template <typename T>
struct StepOpts {
  double* resid_sq = nullptr;  // device: sum of residual^2 over rows [rec_lo, rec_hi] (shared anchor)
  int64_t rec_lo = 0, rec_hi = -1;
  T* const* hd = nullptr;      // per task: cached H E_S d_mem over rows [olo, ohi] (updated in place)
  T* const* greg = nullptr;    // per task: precomputed regulariser gradient rows (skip the greg launch)
  T* const* omega = nullptr;   // per task: precomputed omega rows
  SideStream* ss = nullptr;    // run reg_gram next to the Gram correlation
  const bd3mg_mirror_t* mirrors = nullptr;  // rows of the updated iterate also stored to (peer) buffers
  int nmirrors = 0;
  const double* fin_sums = nullptr;  // the sweep's recorder sums: finalised by the update launch
  double* fin_terms = nullptr;
  T* r_full = nullptr;         // variant "hd-incremental": r = Hx - y kept across calls (plane 0 = r_full_z0)
  int64_t r_full_z0 = 0;
  bool r_refresh = false;      // recompute r_full exactly in this call
  // recorder terms fused into the gradient correlation (M_GRADF): snapshot rows [rec_lo, rec_hi] (rolled)
  // and the stencil sums written to rec_sums[0..4] (the sweep's sums + 1)
  bool rec_gradf = false;
  T* rec_snap = nullptr;
  double* rec_sums = nullptr;
  bool side_forked = false;    // the caller forked the side stream (ss->ev[0]) before this call
  // side-stream work of the caller, enqueued right after the residual launch(es): phase -1 = all of it;
  // with the residual launched per chain (below), phase k = chain k's share (after launch k; the last
  // phase also closes the recorder's reduction)
  std::function<int(int)> after_resid;
  // per-chain regulariser gradient: chain p's gradient correlation waits for chain_ready[p] only (events the
  // caller records on the side stream after that chain's stencil), not for the whole side stream
  const cudaEvent_t* chain_ready = nullptr;
};

// The gradient correlation with the regulariser gradient fused into its
// epilogue (M_GRADF: no separate stencil pass) where it exists: fp64, square
// 3 / 5 / 7 / 9 taps, TMA-staged rows.
template <typename T>
bool gradf_ok(const bd3mg_geom_t* g) {
  // opt-in (BD3MG_GRADF=1): correct and bitwise, but measured slower at C2 (445 vs 424 us per sweep): the
  // epilogue's stencil math and L2 round trips sit on the correlation's critical path, while the separate
  // stencil mostly overlaps the residual correlation on the side stream
  const char* on = getenv("BD3MG_GRADF");
  const bool off = getenv("BD3MG_NO_GRADF") != nullptr || !on || on[0] == '0';
  return !off && sizeof(T) == 8 && g->kx == g->ky && (g->kx == 3 || g->kx == 5 || g->kx == 7 || g->kx == 9) &&
         st_use_tma<T>(g->nx);
}

// The regulariser Gram terms computed by the dual-input Gram correlation in
// front of its tap walk (rg_center, depthvar.cuh) instead of a separate
// reg_gram stencil pass: fp64, square 3 / 5 / 7 / 9 taps, rows of whole
// 16-byte chunks.  BD3MG_NO_RGF=1 keeps the separate pass (the persistent
// sweep's bitwise twin).
template <typename T>
bool rgf_ok(const bd3mg_geom_t* g, int gmode) {
  const bool off = getenv("BD3MG_NO_RGF") != nullptr;
  return !off && sizeof(T) == 8 && gmode == M_GRAM2 && conv_tiled_shape(g->ky, g->kx) &&
         !conv_rz2<T>(g->ky, g->kx, M_GRAM2) && (g->nx * (long long)sizeof(T)) % 16 == 0;
}

// Small stencil grids (one block of a cyclic / asynchronous step): each
// block's z-march is cut into chunks of c planes so a block alone fills ~2
// CTAs per SM (the march is a serial chain of TMA round trips per CTA).  c
// depends on the block and the plane only -- never on how many blocks share
// a launch -- so a block's regulariser-Gram partial sums are grouped the same
// way in every batching (sharded, pipelined and single-launch sweeps stay
// bitwise equal).  TMA path only; returns h for an unchunked block.
template <typename T>
int64_t stencil_chunk(const bd3mg_geom_t* g, int64_t h) {
  static const int sms = [] {
    int d = 0, n = 148;
    if (cudaGetDevice(&d) != cudaSuccess || cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, d) != cudaSuccess)
      n = 148;
    return n;
  }();
  static const bool off = getenv("BD3MG_NO_ST_CHUNK") != nullptr;
  if (off || !st_use_tma<T>(g->nx) || h < 2) return h;
  const long long tiles = tm_tiles(g->ny, g->nx), want = 2LL * sms;
  if (tiles >= want) return h;
  const long long k = std::min<long long>((want + tiles - 1) / tiles, h);
  return (h + k - 1) / k;
}

// Launch a stencil over `jobs` in groups of at most kMaxJobs (partials
// job-major, continuing across the groups).
template <typename T, typename F>
int launch_jobs(const StArgs<T>& proto, const std::vector<StJob<T>>& jobs, size_t partial_doubles_per_job,
                F&& launch) {
  for (size_t j0 = 0; j0 < jobs.size(); j0 += kMaxJobs) {
    StArgs<T> a = proto;
    a.njobs = (int)std::min<size_t>(kMaxJobs, jobs.size() - j0);
    for (int j = 0; j < a.njobs; ++j) a.jobs[j] = jobs[j0 + j];
    if (proto.partials) a.partials = proto.partials + j0 * partial_doubles_per_job;
    int rc = launch(a);
    if (rc) return rc;
  }
  return BD3MG_OK;
}

template <typename T>
int mg_steps_chunk(const bd3mg_geom_t* g, const bd3mg_reg_t* r, const T* K, const T* y, const bd3mg_task_t* tasks,
                   int nt, double* info_out, Ws& ws, cudaStream_t s, const StepOpts<T>& opt = StepOpts<T>()) {
  const int64_t nz = g->nz, plane = g->ny * g->nx, rz = (g->kz - 1) / 2;
  std::vector<int64_t> olo(nt), ohi(nt), h(nt);
  bool shared = true, any_d = false;
  for (int t = 0; t < nt; ++t) {
    const bd3mg_task_t& k = tasks[t];
    if (k.z_lo < 0 || k.z_hi < k.z_lo || k.z_hi >= nz)
      return fail(BD3MG_EINVAL, "invalid block [%lld, %lld]", (long long)k.z_lo, (long long)k.z_hi);
    const int64_t s_lo = std::max<int64_t>(0, k.z_lo - g->kz), s_hi = std::min<int64_t>(nz - 1, k.z_hi + g->kz);
    if (k.frag_z0 > s_lo || k.frag_z0 + k.nzf - 1 < s_hi)
      return fail(BD3MG_EINVAL, "slab [%lld, %lld] does not cover the required support [%lld, %lld] of block [%lld, %lld]",
                  (long long)k.frag_z0, (long long)(k.frag_z0 + k.nzf - 1), (long long)s_lo, (long long)s_hi,
                  (long long)k.z_lo, (long long)k.z_hi);
    olo[t] = std::max<int64_t>(0, k.z_lo - rz);
    ohi[t] = std::min<int64_t>(nz - 1, k.z_hi + rz);
    h[t] = k.z_hi - k.z_lo + 1;
    if (k.frag != tasks[0].frag || k.frag_z0 != tasks[0].frag_z0 || k.nzf != tasks[0].nzf) shared = false;
    if (k.d_mem) any_d = true;
  }
  // residual rows: union (shared anchor) or per task
  std::vector<T*> rb(nt);
  std::vector<int64_t> r_z0(nt), r_n(nt);
  long long resid_work = 0;
  int64_t u_lo = 0, u_hi = -1;
  if (shared) {
    u_lo = *std::min_element(olo.begin(), olo.end());
    u_hi = *std::max_element(ohi.begin(), ohi.end());
    T* ru = opt.r_full ? opt.r_full + (u_lo - opt.r_full_z0) * plane : ws.take<T>((u_hi - u_lo + 1) * plane);
    for (int t = 0; t < nt; ++t) { rb[t] = ru; r_z0[t] = u_lo; r_n[t] = u_hi - u_lo + 1; }
    resid_work = u_hi - u_lo + 1;
  } else {
    for (int t = 0; t < nt; ++t) {
      rb[t] = ws.take<T>((ohi[t] - olo[t] + 1) * plane);
      r_z0[t] = olo[t]; r_n[t] = ohi[t] - olo[t] + 1;
      resid_work += r_n[t];
    }
  }
  std::vector<T*> gb(nt), wb(nt), grb(nt);
  const bool pre = opt.greg != nullptr;
  const bool gradf = gradf_ok<T>(g);  // regulariser gradient in the gradient correlation's epilogue
  if (opt.rec_gradf && !gradf) return fail(BD3MG_EINVAL, "fused recorder needs the fused gradient");
  for (int t = 0; t < nt; ++t) {
    gb[t] = ws.take<T>(h[t] * plane);
    wb[t] = (pre && opt.omega) ? opt.omega[t] : ws.take<T>(h[t] * plane);
    grb[t] = pre ? opt.greg[t] : (gradf ? nullptr : ws.take<T>(h[t] * plane));
  }
  long long gram_work = 0;
  for (int t = 0; t < nt; ++t) gram_work += ohi[t] - olo[t] + 1;
  const bool cached = opt.hd != nullptr;
  const int gmode = cached ? M_GRAMC : (any_d ? M_GRAM2 : M_GRAM1);
  std::vector<T*> hgb(nt, nullptr);
  if (cached)
    for (int t = 0; t < nt; ++t) hgb[t] = ws.take<T>((ohi[t] - olo[t] + 1) * plane);
  if (opt.resid_sq && !shared) return fail(BD3MG_EINVAL, "recorder residual needs a shared anchor");
  if (opt.resid_sq && opt.rec_hi >= opt.rec_lo && (opt.rec_lo < u_lo || opt.rec_hi > u_hi))
    return fail(BD3MG_EINVAL, "recorder rows outside the residual rows");
  // recorder rows split the shared residual job so its partial rows align
  std::vector<std::pair<int64_t, int64_t>> rjobs;  // (out_lo, nout) of the residual jobs
  int rec_job = -1;
  if (shared) {
    if (opt.resid_sq && opt.rec_hi >= opt.rec_lo) {
      if (opt.rec_lo > u_lo) rjobs.push_back({u_lo, opt.rec_lo - u_lo});
      rec_job = (int)rjobs.size();
      rjobs.push_back({opt.rec_lo, opt.rec_hi - opt.rec_lo + 1});
      if (opt.rec_hi < u_hi) rjobs.push_back({opt.rec_hi + 1, u_hi - opt.rec_hi});
    } else {
      rjobs.push_back({u_lo, u_hi - u_lo + 1});
    }
  } else {
    for (int t = 0; t < nt; ++t) rjobs.push_back({olo[t], r_n[t]});
  }
  long long resid_rows = 0, gram_rows = 0;
  for (auto& rj : rjobs) resid_rows += conv_rows<T>(g, M_RESID, rj.second);
  for (int t = 0; t < nt; ++t) gram_rows += conv_rows<T>(g, gmode, ohi[t] - olo[t] + 1);
  (void)resid_work;
  (void)gram_work;
  const long long conv_part_rows = std::max<long long>(std::max(resid_rows, gram_rows), kSumsqCtas);
  double* cparts = ws.take<double>((size_t)conv_part_rows * 3);
  // (sized whether or not a side stream is used: workspace sizing runs without one)
  // (+ one plane pair of rows per extra launch when the residual goes out per chain in fp32)
  double* rsq_parts = opt.resid_sq ? ws.take<double>((size_t)std::max<long long>(
                                         resid_rows + kMaxParts * conv_tiles<T>(g, M_RESID), 1))
                                   : nullptr;
  bool rsq_forked = false;  // the residual's reduction goes to the side stream
  bool resid_split = false;  // the residual went out per chain: the first chain runs on a chain stream
  std::pair<long long, long long> rsq_range{0, 0};
  long long grad_rows = 0;  // recorder partial rows of the fused gradient (one per GRADF CTA)
  for (int t = 0; t < nt; ++t) grad_rows += conv_rows<T>(g, M_GRAD, h[t]);
  double* eparts_g = opt.rec_gradf ? ws.take<double>((size_t)grad_rows * kGradfNV) : nullptr;
  long long hsum = 0;
  for (int t = 0; t < nt; ++t) hsum += h[t];
  // one partial row per (job, tile); a z-chunked block is several jobs
  long long rg_total = 0;
  for (int t = 0; t < nt; ++t) {
    const int64_t c = stencil_chunk<T>(g, h[t]);
    rg_total += (h[t] + c - 1) / c;
  }
  // fused into the Gram correlation: one partial row per (block plane, Gram tile)
  // (only with TMA staging: every d_mem block must be 16-byte aligned like the workspace rows)
  bool rgf = rgf_ok<T>(g, gmode) && !getenv("BD3MG_NO_TMA");
  for (int t = 0; t < nt && rgf; ++t)
    if (tasks[t].d_mem && (reinterpret_cast<uintptr_t>(tasks[t].d_mem) & 15)) rgf = false;
  const long long rgf_tiles = rgf ? conv_tiles<T>(g, M_GRAM2) : 0;
  // (sized for either path: the choice may differ between the sizing call and the launch)
  const long long reg_rows = std::max<long long>(rgf_ok<T>(g, gmode) ? hsum * conv_tiles<T>(g, M_GRAM2) : 0,
                                                 rg_total * z_tiles<T>(g));
  double* rparts = ws.take<double>((size_t)reg_rows * kRegNV);
  if (ws.measure) return BD3MG_OK;
  if (!ws.ok()) return ws_fail(ws);

  // regulariser gradient of every block (whole blocks, or z-chunks of them)
  auto greg_launch = [&](cudaStream_t st) -> int {
    std::vector<StJob<T>> jobs;
    for (int t = 0; t < nt; ++t) {
      const int64_t c = stencil_chunk<T>(g, h[t]);
      for (int64_t lo = tasks[t].z_lo; lo <= tasks[t].z_hi; lo += c) {
        StJob<T> J;
        memset(&J, 0, sizeof(J));
        J.a = (const T*)tasks[t].frag; J.a_z0 = tasks[t].frag_z0;
        J.lo = (int)lo; J.hi = (int)std::min<int64_t>(lo + c - 1, tasks[t].z_hi);
        J.out0 = grb[t] + (lo - tasks[t].z_lo) * plane; J.out1 = wb[t] + (lo - tasks[t].z_lo) * plane;
        jobs.push_back(J);
      }
    }
    return launch_jobs<T>(st_args<T>(g, r), jobs, 0, [&](StArgs<T>& a) { return launch_greg<T>(a, false, st); });
  };
  // (0) block steps with a side stream (mg_steps): the regulariser gradient
  // needs x only, so it runs next to the residual correlation
  const bool greg_side = opt.ss && !pre && !gradf;
  if (greg_side) {
    CU(hop(s, opt.ss->side, opt.ss->ev[0]));
    int rc = greg_launch(opt.ss->side);
    if (rc) return rc;
  }
  // (1) r = H x - y (variant "hd-incremental": kept from the previous call
  // unless refreshed; the recorder's data term is then a sum of squares)
  if (opt.r_full && !opt.r_refresh) {
    if (opt.resid_sq) {
      if (opt.rec_hi >= opt.rec_lo) {
        sumsq_kernel<T><<<kSumsqCtas, kEwNT, 0, s>>>(rb[0] + (opt.rec_lo - u_lo) * plane,
                                                     (opt.rec_hi - opt.rec_lo + 1) * plane, cparts);
        launched();
        CU(cudaGetLastError());
        CU(reduce(cparts, 1, {{0, kSumsqCtas}}, opt.resid_sq, 1, s));
      } else {
        CU(cudaMemsetAsync(opt.resid_sq, 0, sizeof(double), s));
      }
    }
  } else {
    ConvArgs<T> a = base_args<T>(g, r, K);
    a.partials = cparts;
    a.njobs = (int)rjobs.size();
    for (int t = 0; t < a.njobs; ++t) {
      const bd3mg_task_t& k = tasks[shared ? 0 : t];
      ConvJob<T>& j = a.jobs[t];
      j.src0 = (const T*)k.frag; j.src_z0 = k.frag_z0; j.src_nz = (int)k.nzf;
      j.out_lo = (int)rjobs[t].first; j.nout = (int)rjobs[t].second;
      j.dst0 = (shared ? rb[0] : rb[t]) + (rjobs[t].first - (shared ? u_lo : olo[t])) * plane;
      j.sub = y + rjobs[t].first * plane;
    }
    // with a side stream the residual's partial rows get their own buffer and the recorder's reduction of
    // them runs on the side stream, off the correlations' critical path (joined before the solve)
    const bool rsq_side = opt.resid_sq && opt.ss && rec_job >= 0;
    if (rsq_side) a.partials = rsq_parts;
    // Two chains with per-chain stencils (the fp64 Jacobi sweep): the residual is launched per chain as
    // well -- first the rows the first chain's gradient needs, [u_lo, ohi of its last block], then the
    // rest -- with the first chain's stencil enqueued between the two.  The first chain's gradient
    // correlation then starts when ITS rows and ITS stencil are done, under the second launch, instead of
    // after the whole residual and the stencil's run in its last wave.  Partial rows keep the order of the
    // single launch (plane-major), so the recorder's sum has the same bits.
    // (any number of chains: launch k covers the rows up to chain k's last gradient row that the earlier
    // launches have not produced; the last chain stays on the caller's stream)
    std::vector<int> zend;  // last residual row of each launch
    const int nchains = chain_parts<T>(opt.ss != nullptr, nt, hsum * plane);
    if (opt.chain_ready && opt.after_resid && shared && rjobs.size() == 1 && nchains >= 2 && nchains <= 4 &&
        !getenv("BD3MG_NO_RESID_SPLIT")) {
      int prev = (int)u_lo - 1;
      for (int k = 0; k < nchains; ++k) {
        const int tl_ = (int)((long long)nt * (k + 1) / nchains) - 1;  // last block of chain k
        const int e = k == nchains - 1 ? (int)u_hi : (int)std::min<int64_t>(ohi[tl_], u_hi);
        if (e <= prev) { zend.clear(); break; }
        zend.push_back(e);
        prev = e;
      }
      if (!zend.empty() && zend.back() != (int)u_hi) zend.clear();
    }
    long long resid_b0 = 0;  // first partial row of the recorder job
    long long resid_nrows = rec_job >= 0 ? conv_rows<T>(g, M_RESID, rjobs[rec_job].second) : 0;  // and their number
    if (!zend.empty()) {
      cudaEvent_t evr[3] = {opt.ss->ev[2], opt.ss->ev[4], opt.ss->ev[5]};
      int z0 = (int)rjobs[0].first;
      size_t prow = 0;
      for (int k = 0; k < nchains; ++k) {
        ConvArgs<T> ak = a;
        ak.jobs[0].out_lo = z0;
        ak.jobs[0].nout = zend[k] - z0 + 1;
        ak.jobs[0].dst0 = a.jobs[0].dst0 + (long long)(z0 - (int)rjobs[0].first) * plane;
        ak.jobs[0].sub = a.jobs[0].sub + (long long)(z0 - (int)rjobs[0].first) * plane;
        ak.partials = a.partials + prow;
        CU(conv_launch<T>(M_RESID, false, ak, 0, s));
        launched();
        if (k < nchains - 1) CU(cudaEventRecord(evr[k], s));  // chain k's residual rows are done
        const int rc = opt.after_resid(k);
        if (rc) return rc;
        prow += (size_t)conv_rows<T>(g, M_RESID, ak.jobs[0].nout);
        z0 = zend[k] + 1;
      }
      resid_nrows = (long long)prow;  // (the two-plane kernels round every launch up to whole plane pairs)
    } else {
      CU(conv_launch<T>(M_RESID, false, a, 0, s));
      launched();
      if (opt.after_resid) {
        const int rc = opt.after_resid(-1);
        if (rc) return rc;
      }
      if (rec_job >= 0) resid_b0 = (long long)a.jobs[rec_job].work_begin * conv_tiles<T>(g, M_RESID);
    }
    resid_split = !zend.empty();
    if (opt.resid_sq) {  // recorder data term of the anchor, before cparts is reused
      if (rec_job >= 0) {
        const long long b0 = resid_b0;
        if (rsq_side) {  // enqueued below, after the side stream's stencil is joined
          rsq_range = {b0, b0 + resid_nrows};
          rsq_forked = true;
        } else {
          CU(reduce(cparts, 1, {{b0, b0 + resid_nrows}}, opt.resid_sq, 1, s));
        }
      } else {
        CU(cudaMemsetAsync(opt.resid_sq, 0, sizeof(double), s));
      }
    }
  }
  // join the recorder / regulariser-gradient stencil of the side stream (when one was forked: by the
  // sweep before this call, or above)
  if (opt.ss && (greg_side || opt.side_forked) && !opt.chain_ready) CU(hop(opt.ss->side, s, opt.ss->ev[1]));
  if (rsq_forked) {  // the recorder's data term next to the gradient correlation
    CU(hop(s, opt.ss->side, opt.ss->ev[7]));
    CU(reduce(rsq_parts, 1, {rsq_range}, opt.resid_sq, 1, opt.ss->side));
  }
  // (2) regulariser gradient + omega (tiled stencil), then g = H^T r + it
  if (!pre && !greg_side && !gradf) {
    int rc = greg_launch(s);
    if (rc) return rc;
  }
  // (2b)-(7) The blocks are cut into `parts` groups, each a chain GRAD -> (regulariser Gram on the side
  // stream | data Gram) -> solve -> update on its own stream.  The correlations of one chain fill the last
  // waves of another's instead of idling SMs, and an earlier chain's HBM-bound solve + update run under a
  // later chain's FMA-bound Gram correlation instead of after it (fp32 steps up to 2^27 voxels as well,
  // see chain_parts).  A block's update touches only its own
  // rows of x and d_mem, and no later kernel of another chain reads those (the Gram inputs are the
  // chain's own g and d rows), so the chains are independent once the residual is formed.
  // BD3MG_PARTS=n overrides (1: one chain, the pre-split layout).
  const int parts = chain_parts<T>(opt.ss != nullptr, nt, hsum * plane);
  // the fused-gradient recorder (opt-in) reduces its sums over all chains before the update: one tail
  const bool chain_tails = parts > 1 && !opt.rec_gradf;
  std::vector<std::pair<long long, long long>> granges(nt);
  long long gram_row0 = 0;  // first partial row of the current part's Gram launch
  const long long tl_reg = z_tiles<T>(g);
  std::vector<int> rg_begin(nt), rg_end(nt);  // regulariser-Gram jobs of each block
  int rg_jobs = 0;
  long long grad_row0 = 0;  // first recorder row of the current part's fused-gradient launch
  // mirrors: every row must be updated by this call (checked over all blocks before any chain launches)
  for (int j = 0; j < opt.nmirrors; ++j) {
    const bd3mg_mirror_t& M = opt.mirrors[j];
    int64_t covered = 0;
    for (int t = 0; t < nt; ++t) {
      const int64_t lo = std::max<int64_t>(M.z_lo, tasks[t].z_lo), hi = std::min<int64_t>(M.z_hi, tasks[t].z_hi);
      if (lo > hi) continue;
      if (!tasks[t].x_rows) return fail(BD3MG_EINVAL, "mirrored rows need an in-place update");
      covered += hi - lo + 1;
    }
    if (covered != M.z_hi - M.z_lo + 1)
      return fail(BD3MG_EINVAL, "mirror rows [%lld, %lld] are not all updated by this call", (long long)M.z_lo,
                  (long long)M.z_hi);
  }
  // (5)+(6) per-block reductions and the 2x2 solves of blocks [t0, t1), one CTA per block
  auto launch_solve = [&](int t0, int t1, cudaStream_t st) -> int {
    SolveArgs sa;
    memset(&sa, 0, sizeof(sa));
    sa.nblocks = t1 - t0;
    sa.two_eta = 2.0 * r->eta; sa.lam = r->lam; sa.two_kappa = 2.0 * r->kappa;
    sa.prune_tol = kPruneTol; sa.pinv_tol = kPinvTol;
    sa.nv_gram = gmode == M_GRAM1 ? 1 : 3;
    const long long tl = z_tiles<T>(g);
    for (int t = t0; t < t1; ++t) {
      sa.has_d[t - t0] = tasks[t].d_mem != nullptr;
      sa.g_begin[t - t0] = granges[t].first; sa.g_end[t - t0] = granges[t].second;
      sa.r_begin[t - t0] = rgf ? rg_begin[t] : rg_begin[t] * tl;
      sa.r_end[t - t0] = rgf ? rg_end[t] : rg_end[t] * tl;
    }
    reduce_solve_kernel<<<t1 - t0, kEwNT, 0, st>>>(sa, cparts, rparts, info_out + (size_t)t0 * kInfoNV); launched();
    CU(cudaGetLastError());
    return BD3MG_OK;
  };
  // (7) increments / in-place update of blocks [t0, t1); `fin`: this launch also writes the recorder terms
  auto launch_update = [&](int t0, int t1, bool fin, cudaStream_t st) -> int {
#ifndef BD3MG_EXP_SKIP_UPDATE
    UpdArgs<T> ua;
    memset(&ua, 0, sizeof(ua));
    ua.nblocks = t1 - t0;
    if (fin) { ua.fin_sums = opt.fin_sums; ua.fin_terms = opt.fin_terms; }
    ua.fin_eta = r->eta; ua.fin_lam = r->lam; ua.fin_kappa = r->kappa;
    int mc = 1;
    for (int t = t0; t < t1; ++t) {
      UpdBlock<T>& B = ua.blk[t - t0];
      B.g = gb[t]; B.d = (const T*)tasks[t].d_mem; B.inc_out = (T*)tasks[t].inc_out;
      B.x = (T*)tasks[t].x_rows; B.dmem = (T*)tasks[t].dmem_rows;
      B.n = h[t] * plane;
      B.ctas = (int)std::max<int64_t>(1, std::min<int64_t>((B.n + 4 * kEwNT - 1) / (4 * kEwNT), 1024));
      mc = std::max(mc, B.ctas);
    }
    double* info_p = info_out + (size_t)t0 * kInfoNV;
    // split each mirror into per-block element ranges of the in-place update
    MirArgs<T, kMaxMirSegs> ma;
    memset(&ma, 0, sizeof(ma));
    for (int j = 0; j < opt.nmirrors; ++j) {
      const bd3mg_mirror_t& M = opt.mirrors[j];
      for (int t = t0; t < t1; ++t) {
        const int64_t lo = std::max<int64_t>(M.z_lo, tasks[t].z_lo), hi = std::min<int64_t>(M.z_hi, tasks[t].z_hi);
        if (lo > hi) continue;
        if (ma.n == kMaxMirSegs) return fail(BD3MG_EINVAL, "more than %d mirror segments", kMaxMirSegs);
        MirSeg<T>& S = ma.s[ma.n++];
        S.blk = t - t0;
        S.a = (lo - tasks[t].z_lo) * plane;
        S.b = (hi - tasks[t].z_lo + 1) * plane;
        S.dst = (T*)M.dst + (lo - M.z_lo) * plane;
      }
    }
    if (ma.n == 0) {
      update_kernel<T, 0><<<dim3(mc, t1 - t0), kEwNT, 0, st>>>(ua, MirArgs<T, 0>{0, {}}, info_p); launched();
    } else {
      update_kernel<T, kMaxMirSegs><<<dim3(mc, t1 - t0), kEwNT, 0, st>>>(ua, ma, info_p); launched();
    }
    CU(cudaGetLastError());
#else
    (void)t0; (void)t1; (void)fin; (void)st;
#endif
    return BD3MG_OK;
  };
  // stream of a chain: the first stays on the caller's stream -- except with the per-chain residual,
  // where the caller's stream still carries the second residual launch: then the first chain moves to a
  // chain stream (it waits for its residual rows only) and the second stays on the caller's
  auto stream_of = [&](int part) -> cudaStream_t {
    if (resid_split) return part < parts - 1 ? opt.ss->chain[part] : s;
    return part == 0 ? s : opt.ss->chain[part - 1];
  };
  if (resid_split) {
    cudaEvent_t evr[3] = {opt.ss->ev[2], opt.ss->ev[4], opt.ss->ev[5]};
    for (int part = 0; part < parts - 1; ++part) CU(cudaStreamWaitEvent(opt.ss->chain[part], evr[part], 0));
  } else {
    for (int part = 1; part < parts; ++part)  // fork after RESID / greg
      CU(hop(s, opt.ss->chain[part - 1], opt.ss->ev[8 + 5 * part]));
  }
  if (opt.chain_ready)  // each chain waits for its own blocks' regulariser gradient
    for (int part = 0; part < parts; ++part) CU(cudaStreamWaitEvent(stream_of(part), opt.chain_ready[part], 0));
  for (int part = 0; part < parts; ++part) {
    const int t0 = (int)((long long)nt * part / parts), t1 = (int)((long long)nt * (part + 1) / parts);
    const int np = t1 - t0;
    cudaStream_t sp = stream_of(part);
    {
      ConvArgs<T> a = base_args<T>(g, r, K);
      a.njobs = np;
      for (int t = t0; t < t1; ++t) {
        ConvJob<T>& j = a.jobs[t - t0];
        j.src0 = rb[t]; j.src_z0 = r_z0[t]; j.src_nz = (int)r_n[t];
        j.dst0 = gb[t]; j.sub = grb[t];
        j.out_lo = (int)tasks[t].z_lo; j.nout = (int)h[t];
        if (gradf) {  // regulariser gradient (+ recorder terms) from the iterate tile in the epilogue
          j.xg = (const T*)tasks[t].frag; j.xg_z0 = tasks[t].frag_z0; j.xg_nz = (int)tasks[t].nzf;
          j.omega = wb[t];
          j.snap = (opt.rec_gradf && opt.rec_snap) ? opt.rec_snap + (tasks[t].z_lo - opt.rec_lo) * plane : nullptr;
          j.eparts = opt.rec_gradf ? eparts_g + (size_t)grad_row0 * kGradfNV : nullptr;  // rows: this launch's CTAs
        }
      }
      CU(conv_launch<T>(gradf ? M_GRADF : M_GRAD, true, a, 0, sp));
      launched();
      for (int t = t0; t < t1; ++t) grad_row0 += conv_rows<T>(g, M_GRAD, h[t]);
    }
    // regulariser Gram terms on the side stream, concurrent with the Gram correlation
    // (or inside the Gram correlation itself: rgf)
    cudaStream_t s3 = sp;
    if (rgf) {
      for (int t = t0; t < t1; ++t) {
        rg_begin[t] = rg_jobs;  // in partial rows, not jobs
        rg_jobs += (int)(h[t] * rgf_tiles);
        rg_end[t] = rg_jobs;
      }
    } else if (opt.ss) {
      CU(hop(sp, opt.ss->side, opt.ss->ev[9 + 5 * part]));
      s3 = opt.ss->side;
    }
    if (!rgf) {
      StArgs<T> sa = st_args<T>(g, r);
      sa.partials = rparts + (size_t)rg_jobs * tl_reg * kRegNV;  // job-major rows after the earlier parts
      std::vector<StJob<T>> jobs;
      for (int t = t0; t < t1; ++t) {
        const int64_t c = stencil_chunk<T>(g, h[t]);
        rg_begin[t] = rg_jobs + (int)jobs.size();
        for (int64_t lo = tasks[t].z_lo; lo <= tasks[t].z_hi; lo += c) {
          const int64_t o = (lo - tasks[t].z_lo) * plane;
          StJob<T> J;
          memset(&J, 0, sizeof(J));
          J.a = gb[t] + o; J.a_z0 = lo; J.b = tasks[t].d_mem ? (const T*)tasks[t].d_mem + o : nullptr;
          J.w = wb[t] + o;
          J.lo = (int)lo; J.hi = (int)std::min<int64_t>(lo + c - 1, tasks[t].z_hi);
          if (c < h[t]) { J.chunk = 1; J.blo = (int)tasks[t].z_lo; J.bhi = (int)tasks[t].z_hi; }
          jobs.push_back(J);
        }
        rg_end[t] = rg_jobs + (int)jobs.size();
      }
      rg_jobs += (int)jobs.size();
#ifndef BD3MG_EXP_SKIP_REGGRAM
      int rc = launch_jobs<T>(sa, jobs, (size_t)tl_reg * kRegNV,
                              [&](StArgs<T>& a) { return launch_reg_gram<T>(a, s3); });
      if (rc) return rc;
#endif
    }
    // (4) data Gram <H b_i, H b_j> (forward only, both columns share the taps)
    {
      ConvArgs<T> a = base_args<T>(g, r, K);
      a.njobs = np;
      a.partials = cparts + (size_t)gram_row0 * 3;
      for (int t = t0; t < t1; ++t) {
        ConvJob<T>& j = a.jobs[t - t0];
        j.src0 = gb[t];
        j.src1 = tasks[t].d_mem ? (const T*)tasks[t].d_mem : gb[t];
        if (cached) { j.sub = opt.hd[t]; j.dst0 = hgb[t]; }
        if (rgf) { j.omega = wb[t]; j.eparts = rparts + (size_t)rg_begin[t] * kRegNV; }
        j.src_z0 = tasks[t].z_lo; j.src_nz = (int)h[t];
        j.out_lo = (int)olo[t]; j.nout = (int)(ohi[t] - olo[t] + 1);
      }
      CU(conv_launch<T>(gmode, false, a, 0, sp));
      launched();
      const long long tiles = conv_tiles<T>(g, gmode);  // partial rows per grid.z unit
      long long rows = 0;
      for (int t = t0; t < t1; ++t) {
        const long long b0 = (long long)a.jobs[t - t0].work_begin * tiles;
        const long long nr = conv_rows<T>(g, gmode, a.jobs[t - t0].nout);
        granges[t] = {gram_row0 + b0, gram_row0 + b0 + nr};
        rows = std::max(rows, b0 + nr);
      }
      gram_row0 += rows;
    }
    if (chain_tails) {
      // this chain's solve + update as soon as its own sums are in: the side stream has run the
      // recorder's reductions and this chain's regulariser Gram by the event recorded here
      CU(hop(opt.ss->side, sp, opt.ss->ev[10 + 5 * part]));
      int rc = launch_solve(t0, t1, sp);
      if (rc) return rc;
      rc = launch_update(t0, t1, part == 0, sp);
      if (rc) return rc;
    }
  }
  for (int part = 0; part < parts; ++part)  // join the chains that ran on chain streams
    if (stream_of(part) != s) CU(hop(stream_of(part), s, opt.ss->ev[11 + 5 * part]));
  if (opt.ss) CU(hop(opt.ss->side, s, opt.ss->ev[3]));  // join the side stream
  if (opt.rec_gradf)  // the recorder's stencil sums from the fused gradient's partial rows
    CU(reduce(eparts_g, kGradfNV, {{0, grad_rows}}, opt.rec_sums, kGradfNV, s));
  if (!chain_tails) {
    int rc = launch_solve(0, nt, s);
    if (rc) return rc;
    rc = launch_update(0, nt, true, s);
    if (rc) return rc;
  }
  // (8) cached H E_S d_mem for the next visit (variant "hd-cache"), and the
  // maintained residual (variant "hd-incremental")
  if (cached) {
    HdArgs<T> ha;
    memset(&ha, 0, sizeof(ha));
    ha.nblocks = nt;
    int mc = 1;
    for (int t = 0; t < nt; ++t) {
      HdBlock<T>& B = ha.blk[t];
      B.hg = hgb[t]; B.hd = opt.hd[t]; B.n = (ohi[t] - olo[t] + 1) * plane;
      B.ctas = (int)std::max<int64_t>(1, std::min<int64_t>((B.n + 4 * kEwNT - 1) / (4 * kEwNT), 1024));
      mc = std::max(mc, B.ctas);
    }
    hd_update_kernel<T><<<dim3(mc, nt), kEwNT, 0, s>>>(ha, info_out); launched();
    CU(cudaGetLastError());
    if (opt.r_full) {
      RIncArgs<T> ra;
      memset(&ra, 0, sizeof(ra));
      ra.r = opt.r_full; ra.plane = plane; ra.r_z0 = (int)opt.r_full_z0;
      ra.u_lo = (int)u_lo; ra.u_hi = (int)u_hi; ra.nblocks = nt;
      for (int t = 0; t < nt; ++t) { ra.hd[t] = opt.hd[t]; ra.olo[t] = (int)olo[t]; ra.ohi[t] = (int)ohi[t]; }
      const long long n = (u_hi - u_lo + 1) * plane;
      const int ctas = (int)std::max<long long>(1, std::min<long long>((n + 4 * kEwNT - 1) / (4 * kEwNT), 8 * 148));
      resid_inc_kernel<T><<<ctas, kEwNT, 0, s>>>(ra, info_out); launched();
      CU(cudaGetLastError());
    }
  }
  return BD3MG_OK;
}

template <typename T>
int mg_steps_impl(const bd3mg_geom_t* g, const bd3mg_reg_t* r, const T* K, const T* y, const bd3mg_task_t* tasks,
                  int ntasks, double* info_out, Ws& ws, cudaStream_t s, const bd3mg_mirror_t* mirrors = nullptr,
                  int nmirrors = 0, T* const* hd = nullptr, T* resid = nullptr) {
  if (ntasks < 0) return fail(BD3MG_EINVAL, "negative task count");
  if (resid) {  // variant "hd-incremental" for block steps: one launch, in place, whole-volume anchor
    if (!hd || ntasks > kMaxJobs) return fail(BD3MG_EINVAL, "incremental steps need the hd cache and <= %d tasks", kMaxJobs);
    for (int t = 0; t < ntasks; ++t)
      if (!hd[t] || !tasks[t].x_rows || tasks[t].frag_z0 != 0 || tasks[t].nzf != g->nz || tasks[t].frag != tasks[0].frag)
        return fail(BD3MG_EINVAL, "incremental steps need in-place tasks on one whole-volume anchor (task %d)", t);
  }
  if (nmirrors < 0 || (nmirrors > 0 && (!mirrors || ntasks > kMaxJobs)))
    return fail(BD3MG_EINVAL, "invalid mirror list (mirrored calls are one launch of <= %d tasks)", kMaxJobs);
  for (int j = 0; j < nmirrors; ++j)
    if (!mirrors[j].dst || mirrors[j].z_hi < mirrors[j].z_lo) return fail(BD3MG_EINVAL, "invalid mirror %d", j);
  StepOpts<T> opt;
  opt.mirrors = mirrors;
  opt.nmirrors = nmirrors;
  opt.hd = hd;
  opt.r_full = resid;
  opt.r_full_z0 = 0;
  // eager block steps overlap the stencils on a side stream (measured: async
  // mode at C2 8040 -> 8880 block-it/s); inside a graph capture the extra
  // branch costs more than it hides for one-block steps (cyclic sweep 7985 ->
  // 7597), so captured calls stay on one stream
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  if (!ws.measure) CU(cudaStreamIsCapturing(s, &cap));
  if (!ws.measure && cap == cudaStreamCaptureStatusNone && !getenv("BD3MG_NO_SIDE_STREAM")) {
    SideStream* ss = nullptr;
    CU(side_stream(s, &ss));
    opt.ss = ss;
  }
  // tasks run in launches of kMaxJobs; an in-place update of one launch would
  // move the anchor of the next, so in-place calls are limited to one launch
  if (ntasks > kMaxJobs)
    for (int t = 0; t < ntasks; ++t)
      if (tasks[t].x_rows)
        return fail(BD3MG_EINVAL, "in-place updates (x_rows) need at most %d tasks per call", kMaxJobs);
  size_t peak = 0;
  for (int t0 = 0; t0 < ntasks; t0 += kMaxJobs) {
    const int nt = std::min(kMaxJobs, ntasks - t0);
    Ws sub = ws;
    sub.off = 0;
    if (!ws.measure) { sub.base = ws.base; sub.cap = ws.cap; }
    int rc = mg_steps_chunk<T>(g, r, K, y, tasks + t0, nt, info_out ? info_out + (size_t)t0 * kInfoNV : nullptr,
                               sub, s, opt);
    if (rc != BD3MG_OK) return rc;
    peak = std::max(peak, sub.off);
  }
  ws.off = std::max(ws.off, peak);
  return BD3MG_OK;
}

// ---------------------------------------------------------------------------
// Persistent sweep (sweep_pk.cuh): plan + launch.  The queue order comes from
// a list-scheduling simulation of the sweep's items on the kernel's resident
// slots (item costs from the tap counts and staged bytes, priority = longest
// path to the end of the sweep), so consumers are queued about when their
// inputs are expected to be ready; correctness never depends on the model
// (every item waits on its counters, and every dependency is earlier in the
// order).
constexpr int kPkIneligible = 1000;

// BD3MG_PK_TRACE=1: per-item timestamps of the last persistent sweep
// (diagnostics; bd3mg_pk_trace copies them out)
struct PkTrace {
  std::mutex mu;
  unsigned long long* buf = nullptr;
  size_t cap = 0, n = 0;
};
PkTrace& pk_trace() {
  static PkTrace t;
  return t;
}
std::atomic<long long> g_pk_launches{0};  // persistent sweeps launched (bd3mg_pk_launches)

struct PkGroup {
  int type, b, z, aux;
  int n;         // items
  double cost;   // per item (model microseconds on a slot of its class)
  int aff;       // the earliest block whose update depends on the group (pipelining bias)
  std::vector<int> succ;
  int npred = 0;
  double bl = 0, prio = 0;
  int started = 0, finished = 0;
};

// FMA-bound correlation tiles vs memory-bound items (stencils, solve,
// update, reductions).  The simulation gives every SM one memory slot and
// the rest to correlations (an idle slot takes the other class when its own
// has nothing ready), so the order interleaves the HBM-bound items with the
// correlations at the rate the SMs can overlap them.
inline bool pk_is_conv(int type) { return type == PK_RESID || type == PK_GRAD || type == PK_GRAM; }

// returns false when the order does not fit kPkMaxSeg segments
static bool pk_schedule(std::vector<PkGroup>& G, int slots, int sms, int nb, std::vector<PkSeg>& segs,
                        uint32_t& total) {
  const int ng = (int)G.size();
  for (int i = ng - 1; i >= 0; --i) {  // groups are created in a topological order
    double m = 0;
    for (int j : G[i].succ) m = std::max(m, G[j].bl);
    G[i].bl = G[i].cost + m;
    // longest path first; among comparable paths the earlier block (its
    // update then overlaps the later blocks' correlations)
    G[i].prio = G[i].bl + 4.0 * (nb - G[i].aff);
  }
  for (auto& g : G)
    for (int j : g.succ) G[j].npred++;
  auto cmp = [&](int a, int b) { return G[a].prio != G[b].prio ? G[a].prio < G[b].prio : a > b; };
  using PQ = std::priority_queue<int, std::vector<int>, decltype(cmp)>;
  PQ ready[2] = {PQ(cmp), PQ(cmp)};  // [0] correlation items, [1] memory-bound items
  for (int i = 0; i < ng; ++i)
    if (G[i].npred == 0 && G[i].n > 0) ready[pk_is_conv(G[i].type) ? 0 : 1].push(i);
  struct Ev {
    double t;
    int g, cls;
    bool operator>(const Ev& o) const { return t > o.t; }
  };
  std::priority_queue<Ev, std::vector<Ev>, std::greater<Ev>> running;
  const int mem_slots = std::max(1, std::min(slots / 2, sms));  // one memory-bound item per SM
  int free_slots[2] = {slots - mem_slots, mem_slots};
  double t = 0;
  segs.clear();
  total = 0;
  int last_group = -1;
  auto start = [&](int cls, int q) {
    const int gi = ready[q].top();
    PkGroup& g = G[gi];
    if (last_group != gi) {  // a new segment (a group's items are taken in order)
      PkSeg sg;
      sg.first = total;
      sg.type = (uint8_t)g.type;
      sg.b = (uint8_t)g.b;
      if (pk_is_conv(g.type)) { sg.z = (uint16_t)g.z; sg.aux = (uint16_t)g.started; }
      else if (g.type == PK_RG) { sg.z = (uint16_t)g.started; sg.aux = (uint16_t)g.aux; }
      else if (g.type == PK_RED) { sg.z = (uint16_t)g.z; sg.aux = 0; }
      else { sg.z = (uint16_t)g.started; sg.aux = 0; }  // GREG: first tile, UPD: first chunk, SOLVE: 0
      segs.push_back(sg);
      last_group = gi;
    }
    ++total;
    ++g.started;
    --free_slots[cls];
    running.push({t + g.cost, gi, cls});
    if (g.started == g.n) ready[q].pop();
  };
  while (true) {
    bool progress = true;
    while (progress) {
      progress = false;
      for (int cls = 0; cls < 2; ++cls) {
        if (free_slots[cls] == 0) continue;
        if (!ready[cls].empty()) { start(cls, cls); progress = true; }
        else if (!ready[1 - cls].empty()) { start(cls, 1 - cls); progress = true; }
      }
      if ((int)segs.size() > kPkMaxSeg) return false;
    }
    if (running.empty()) break;
    const Ev e = running.top();
    running.pop();
    t = e.t;
    ++free_slots[e.cls];
    PkGroup& g = G[e.g];
    if (++g.finished == g.n)
      for (int j : g.succ)
        if (--G[j].npred == 0) ready[pk_is_conv(G[j].type) ? 0 : 1].push(j);
  }
  for (auto& g : G)
    if (g.started != g.n) return false;  // unreachable group: malformed plan
  return true;
}

template <int K>
static bool pk_maps(PkArgs<double>& a, const bd3mg_geom_t* g, const double* x, int64_t nzf, const double* y_rows,
                    const double* r, int64_t nres, const double* gb, const double* greg, int64_t hsum,
                    const double* dm) {
  using CR = ConvCfg<double, K, K, M_RESID, kPkRY>;
  using CM = ConvCfg<double, K, K, M_GRAM2P>;
  using GG = GregGeo<double>;
  using RG = RgGeo<double>;
  const long long nx = g->nx, ny = g->ny;
  return encode_tmap(&a.tm_x, x, true, nx, ny, nzf, CR::PITCH, CR::BOXH) &&
         encode_tmap(&a.tm_y, y_rows, true, nx, ny, nres, CR::TX, CR::TY) &&
         encode_tmap(&a.tm_r, r, true, nx, ny, nres, CR::PITCH, CR::BOXH) &&
         encode_tmap(&a.tm_greg, greg, true, nx, ny, hsum, CR::TX, CR::TY) &&
         encode_tmap(&a.tm_g, gb, true, nx, ny, hsum, CM::PITCH, CM::BOXH) &&
         encode_tmap(&a.tm_d, dm, true, nx, ny, nzf, CM::PITCH, CM::BOXH) &&
         encode_tmap(&a.tm_xs, x, true, nx, ny, nzf, GG::BW, GG::BH) &&
         encode_tmap(&a.tm_gs, gb, true, nx, ny, hsum, RG::BW, RG::BH) &&
         encode_tmap(&a.tm_ds, dm, true, nx, ny, nzf, RG::BW, RG::BH);
}

template <int K>
static int pk_bar_off(int kz) { return (int)PkCfg<double, K>::data_bytes(kz); }

// The whole fused sweep as one persistent launch (fp64, square 3/5/7/9 taps,
// TMA-able rows, recorder fused, memory store present, no hd variants).
// Returns kPkIneligible when it does not apply (the multi-kernel path runs).
template <typename T>
int pk_sweep(const bd3mg_geom_t* g, const bd3mg_reg_t* r, const T* K, const T* y, const bd3mg_sweep_t* sw,
             double* terms, double* info, Ws& ws, cudaStream_t s, const bd3mg_mirror_t* mirrors, int nmirrors) {
  if constexpr (!std::is_same<T, double>::value) {
    return kPkIneligible;
  } else {
    // opt-in (BD3MG_PK=1): measured slower than the multi-kernel sweep at C2 so far (535 vs 424 us, see
    // DESIGN.md); read per call so tests can compare both paths
    const char* pk_env = getenv("BD3MG_PK");
    const bool off = getenv("BD3MG_NO_PK") != nullptr || !pk_env || pk_env[0] == '0';
    const int Kk = g->kx;
    if (off || g->kx != g->ky || !(Kk == 3 || Kk == 5 || Kk == 7 || Kk == 9) || !st_use_tma<T>(g->nx) || !sw->dmem ||
        sw->hd_cache || nmirrors > kMaxMirSegs)
      return kPkIneligible;
    const int64_t nz = g->nz, plane = g->ny * g->nx, rz = (g->kz - 1) / 2;
    const int nb = sw->nblocks;
    const int64_t rec_lo = sw->rec_lo, rec_hi = sw->rec_hi, hsum = rec_hi - rec_lo + 1;
    const int64_t u_lo = std::max<int64_t>(0, rec_lo - rz), u_hi = std::min<int64_t>(nz - 1, rec_hi + rz);
    if (u_lo < sw->frag_z0 || u_hi > sw->frag_z0 + sw->nzf - 1 + rz) return kPkIneligible;
    const int64_t P = u_hi - u_lo + 1;
    using CR = ConvCfg<double, 5, 5, M_RESID, kPkRY>;
    using CM = ConvCfg<double, 5, 5, M_GRAM2P>;
    const int conv_tx = (int)((g->nx + CR::TX - 1) / CR::TX), conv_ty = (int)((g->ny + CR::TY - 1) / CR::TY);
    const int gram_tx = (int)((g->nx + CM::TX - 1) / CM::TX), gram_ty = (int)((g->ny + CM::TY - 1) / CM::TY);
    const int st_tx = (int)((g->nx + kTmX - 1) / kTmX), st_ty = (int)((g->ny + kTmY - 1) / kTmY);
    const int conv_tiles = conv_tx * conv_ty, gram_tiles = gram_tx * gram_ty, st_tiles = st_tx * st_ty;
    std::vector<int> lo(nb), hi(nb), olo(nb), ohi(nb), rgc(nb), nch(nb);
    long long grows = 0, rrows = 0;
    std::vector<long long> g_row0(nb), rg_row0(nb);
    for (int b = 0; b < nb; ++b) {
      lo[b] = (int)sw->blocks[2 * b];
      hi[b] = (int)sw->blocks[2 * b + 1];
      olo[b] = (int)std::max<int64_t>(0, lo[b] - rz);
      ohi[b] = (int)std::min<int64_t>(nz - 1, hi[b] + rz);
      const int h = hi[b] - lo[b] + 1;
      rgc[b] = (int)stencil_chunk<T>(g, h);
      nch[b] = (h + rgc[b] - 1) / rgc[b];
      g_row0[b] = grows;
      grows += (long long)(ohi[b] - olo[b] + 1) * gram_tiles;
      rg_row0[b] = rrows;
      rrows += (long long)nch[b] * st_tiles;
    }
    T* rbuf = ws.take<T>(P * plane);
    T* gbuf = ws.take<T>(hsum * plane);
    T* grbuf = ws.take<T>(hsum * plane);
    T* wbuf = ws.take<T>(hsum * plane);
    double* eparts = ws.take<double>((size_t)nb * st_tiles * kEvalNV);
    double* cparts = ws.take<double>((size_t)P * conv_tiles);
    double* gparts = ws.take<double>((size_t)grows * 3);
    double* rparts = ws.take<double>((size_t)rrows * kRegNV);
    double* sums = ws.take<double>(8);
    int* ctr = ws.take<int>(pk_ctr_count((int)P));
    if (ws.measure) return BD3MG_OK;
    if (!ws.ok()) return ws_fail(ws);

    static thread_local PkArgs<double> a;
    memset(&a, 0, sizeof(a));
    const double* x = (const double*)sw->x;
    double* dm = (double*)sw->dmem;
    bool maps = false;
    switch (Kk) {
      case 3: maps = pk_maps<3>(a, g, x, sw->nzf, (const double*)y + u_lo * plane, rbuf, P, gbuf, grbuf, hsum, dm); a.bar_off = pk_bar_off<3>(g->kz); break;
      case 5: maps = pk_maps<5>(a, g, x, sw->nzf, (const double*)y + u_lo * plane, rbuf, P, gbuf, grbuf, hsum, dm); a.bar_off = pk_bar_off<5>(g->kz); break;
      case 7: maps = pk_maps<7>(a, g, x, sw->nzf, (const double*)y + u_lo * plane, rbuf, P, gbuf, grbuf, hsum, dm); a.bar_off = pk_bar_off<7>(g->kz); break;
      default: maps = pk_maps<9>(a, g, x, sw->nzf, (const double*)y + u_lo * plane, rbuf, P, gbuf, grbuf, hsum, dm); a.bar_off = pk_bar_off<9>(g->kz); break;
    }
    if (!maps) return kPkIneligible;
    a.cg.K = (const double*)K;
    a.cg.nzk = (int)nz; a.cg.kz = g->kz; a.cg.ky = g->ky; a.cg.kx = g->kx;
    a.cg.ny = (int)g->ny; a.cg.nx = (int)g->nx; a.cg.plane = plane; a.cg.nz_global = (int)nz;
    a.sg.nz = (int)nz; a.sg.ny = (int)g->ny; a.sg.nx = (int)g->nx; a.sg.plane = plane;
    a.sg.two_eta = 2.0 * r->eta; a.sg.lam = r->lam; a.sg.two_kappa = 2.0 * r->kappa;
    a.sg.delta2 = r->delta * r->delta; a.sg.x_min = r->x_min; a.sg.x_max = r->x_max;
    a.x = x; a.xw = (double*)sw->x; a.frag_z0 = sw->frag_z0; a.nzf = (int)sw->nzf;
    a.y = (const double*)y; a.r = rbuf; a.u_lo = (int)u_lo; a.u_hi = (int)u_hi;
    a.g = gbuf; a.greg = grbuf; a.omega = wbuf; a.rec_lo = (int)rec_lo; a.rec_hi = (int)rec_hi;
    a.dmem = dm; a.snap = (double*)sw->snap;
    a.eparts = eparts; a.cparts = cparts; a.gparts = gparts; a.rparts = rparts;
    a.sums = sums; a.terms = terms; a.info = info; a.ctr = ctr;
    a.nb = nb;
    for (int b = 0; b < nb; ++b) {
      a.lo[b] = lo[b]; a.hi[b] = hi[b]; a.olo[b] = olo[b]; a.rg_c[b] = rgc[b];
      a.g_row0[b] = g_row0[b]; a.rg_row0[b] = rg_row0[b];
    }
    a.conv_tx = conv_tx; a.conv_tiles = conv_tiles; a.gram_tx = gram_tx; a.gram_tiles = gram_tiles;
    a.st_tx = st_tx; a.st_tiles = st_tiles;
    a.upd_chunk = 4096;
    a.fin_eta = r->eta; a.fin_lam = r->lam; a.fin_kappa = r->kappa;
    SolveArgs& so = a.solve;
    so.nblocks = nb;
    so.two_eta = 2.0 * r->eta; so.lam = r->lam; so.two_kappa = 2.0 * r->kappa;
    so.prune_tol = kPruneTol; so.pinv_tol = kPinvTol;
    so.nv_gram = 3;
    for (int b = 0; b < nb; ++b) so.has_d[b] = 1;
    // mirrors: per-block element ranges of the in-place update (as mg_steps_chunk)
    for (int j = 0; j < nmirrors; ++j) {
      const bd3mg_mirror_t& M = mirrors[j];
      int64_t covered = 0;
      for (int b = 0; b < nb; ++b) {
        const int64_t l = std::max<int64_t>(M.z_lo, lo[b]), h = std::min<int64_t>(M.z_hi, hi[b]);
        if (l > h) continue;
        if (a.mir.n == kMaxMirSegs) return kPkIneligible;
        MirSeg<double>& S = a.mir.s[a.mir.n++];
        S.blk = b;
        S.a = (l - lo[b]) * plane;
        S.b = (h - lo[b] + 1) * plane;
        S.dst = (double*)M.dst + (l - M.z_lo) * plane;
        covered += h - l + 1;
      }
      if (covered != M.z_hi - M.z_lo + 1)
        return fail(BD3MG_EINVAL, "mirror rows [%lld, %lld] are not all updated by this call", (long long)M.z_lo,
                    (long long)M.z_hi);
    }
    // ---- the plan: groups, costs, dependencies ----
    int slots = 0;
    a.total = 0;
    CU(pk_launch(a, Kk, s, &slots));  // resident slots (no launch with an empty queue)
    static thread_local std::vector<PkSeg> segs;
    static thread_local std::vector<PkGroup> G;
    G.clear();
    const double c_tap = 2.0 * (Kk * Kk) / 25.0 * kPkRY / 8.0;  // one tap over a 64 x (4 kPkRY) tile at a slot's FMA share
    const double c_plane = 1.5;                     // one z-march plane of a 32 x 16 stencil column
    auto add = [&](int type, int b, int z, int aux, int n, double cost, int aff) {
      PkGroup q;
      q.type = type; q.b = b; q.z = z; q.aux = aux; q.n = n; q.cost = cost; q.aff = aff;
      G.push_back(q);
      return (int)G.size() - 1;
    };
    auto block_of = [&](int64_t z) {  // block containing row z (clamped to the recorder rows)
      z = std::min<int64_t>(std::max<int64_t>(z, rec_lo), rec_hi);
      int bb = 0;
      while (bb + 1 < nb && lo[bb + 1] <= z) ++bb;
      return bb;
    };
    std::vector<int> gid_resid(P), gid_greg(nb), gid_solve(nb);
    std::vector<std::vector<int>> gid_grad(nb), gid_rg(nb), gid_gram(nb);
    for (int64_t z = u_lo; z <= u_hi; ++z) {
      int taps = 0;
      for (int a2 = 0; a2 < g->kz; ++a2) {
        const int64_t zi = z + a2 - rz;
        taps += (zi >= sw->frag_z0 && zi < sw->frag_z0 + sw->nzf) ? 1 : 0;
      }
      gid_resid[z - u_lo] = add(PK_RESID, 0, (int)z, 0, conv_tiles, taps * c_tap, block_of(z - rz));
    }
    for (int b = 0; b < nb; ++b)
      gid_greg[b] = add(PK_GREG, b, 0, 0, st_tiles, (hi[b] - lo[b] + 3) * c_plane, std::max(0, b - 1));
    for (int b = 0; b < nb; ++b)
      for (int zi = lo[b]; zi <= hi[b]; ++zi) {
        int taps = 0;
        for (int a2 = 0; a2 < g->kz; ++a2) {
          const int64_t zs = zi + a2 - rz;
          taps += (zs >= u_lo && zs <= u_hi && zs < nz) ? 1 : 0;
        }
        const int id = add(PK_GRAD, b, zi, 0, conv_tiles, taps * c_tap, b);
        gid_grad[b].push_back(id);
        for (int64_t z = std::max<int64_t>(u_lo, zi - rz); z <= std::min<int64_t>(u_hi, zi + rz); ++z)
          G[gid_resid[z - u_lo]].succ.push_back(id);
        G[gid_greg[b]].succ.push_back(id);
      }
    for (int b = 0; b < nb; ++b) {
      for (int c = 0; c < nch[b]; ++c) {
        const int clo = lo[b] + c * rgc[b], chi = std::min(hi[b], clo + rgc[b] - 1);
        const int id = add(PK_RG, b, 0, c, st_tiles, 2 * (chi - clo + 2) * c_plane, b);
        gid_rg[b].push_back(id);
        for (int q : gid_grad[b]) G[q].succ.push_back(id);
        G[gid_greg[b]].succ.push_back(id);
      }
      for (int zo = olo[b]; zo <= ohi[b]; ++zo) {
        const int taps = std::min(hi[b], zo + (int)rz) - std::max(lo[b], zo - (int)rz) + 1;
        const int id = add(PK_GRAM, b, zo, 0, gram_tiles, taps * c_tap, b);  // two passes over half-height tiles
        gid_gram[b].push_back(id);
        for (int q : gid_grad[b]) G[q].succ.push_back(id);
      }
    }
    for (int b = 0; b < nb; ++b) {
      gid_solve[b] = add(PK_SOLVE, b, 0, 0, 1, 5.0, b);
      for (int q : gid_gram[b]) G[q].succ.push_back(gid_solve[b]);
      for (int q : gid_rg[b]) G[q].succ.push_back(gid_solve[b]);
    }
    for (int b = 0; b < nb; ++b) {
      const long long n = (long long)(hi[b] - lo[b] + 1) * plane;
      const int chunks = (int)((n + a.upd_chunk - 1) / a.upd_chunk);
      const int id = add(PK_UPD, b, 0, 0, chunks, 6.0, b);
      G[gid_solve[b]].succ.push_back(id);
      for (int64_t z = std::max<int64_t>(u_lo, lo[b] - rz); z <= std::min<int64_t>(u_hi, hi[b] + rz); ++z)
        G[gid_resid[z - u_lo]].succ.push_back(id);
      for (int bb = std::max(0, b - 1); bb <= std::min(nb - 1, b + 1); ++bb) G[gid_greg[bb]].succ.push_back(id);
    }
    {
      const int id0 = add(PK_RED, 0, 0, 0, 1, 3.0, nb);
      for (int b = 0; b < nb; ++b) G[gid_greg[b]].succ.push_back(id0);
      const int id1 = add(PK_RED, 0, 1, 0, 1, 3.0, nb);
      for (int64_t z = rec_lo; z <= rec_hi; ++z) G[gid_resid[z - u_lo]].succ.push_back(id1);
    }
    uint32_t total = 0;
    int sms = 148;
    {
      int dev = 0;
      if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    }
    if (!pk_schedule(G, slots, sms, nb, segs, total)) return kPkIneligible;
    a.nseg = (int)segs.size();
    for (int i = 0; i < a.nseg; ++i) a.seg[i] = segs[i];
    a.total = total;
    if (getenv("BD3MG_PK_DEBUG"))
      fprintf(stderr, "pk: %d slots, %u items, %d segments, %zu groups, params %zu B\n", slots, total, a.nseg,
              G.size(), sizeof(PkArgs<double>));
    a.trace = nullptr;
    if (getenv("BD3MG_PK_TRACE")) {
      PkTrace& tr = pk_trace();
      std::lock_guard<std::mutex> lock(tr.mu);
      if (tr.cap < total) {
        if (tr.buf) cudaFree(tr.buf);
        tr.buf = nullptr;
        tr.cap = 0;
        CU(cudaMalloc(&tr.buf, (size_t)total * 32));
        tr.cap = total;
      }
      tr.n = total;
      a.trace = tr.buf;
    }
    CU(cudaMemsetAsync(ctr, 0, sizeof(int) * pk_ctr_count((int)P), s));
    CU(pk_launch(a, Kk, s, nullptr));
    launched();
    g_pk_launches.fetch_add(1);
    return BD3MG_OK;
  }
}

// One block-Jacobi sweep (see bd3mg_jacobi_sweep in the header).  When the
// blocks tile the recorder rows exactly (single GPU, or a rank's owned rows)
// the recorder pass is fused into the regulariser-gradient stencil (same x
// tiles); otherwise a separate eval stencil runs first.  Scratch layout:
// [eval partials][sums][greg, omega per block][step scratch].
template <typename T>
int jacobi_sweep_impl(const bd3mg_geom_t* g, const bd3mg_reg_t* r, const T* K, const T* y, const bd3mg_sweep_t* sw,
                      double* terms, double* info, Ws& ws, cudaStream_t s, const bd3mg_mirror_t* mirrors = nullptr,
                      int nmirrors = 0, T* r_full = nullptr, bool r_refresh = false) {
  if (!sw || sw->nblocks < 1 || sw->nblocks > kMaxJobs)
    return fail(BD3MG_EINVAL, "jacobi sweep needs 1..%d blocks", kMaxJobs);
  const int64_t plane = g->ny * g->nx, rz = (g->kz - 1) / 2;
  T* x = (T*)sw->x;
  T* dm = (T*)sw->dmem;
  const int nb = sw->nblocks;
  std::vector<bd3mg_task_t> tasks(nb);
  std::vector<T*> hd(nb), grb(nb), wb(nb);
  int64_t hd_off = 0, hsum = 0, bmin = INT64_MAX, bmax = -1;
  for (int b = 0; b < nb; ++b) {
    const int64_t lo = sw->blocks[2 * b], hi = sw->blocks[2 * b + 1];
    if (lo < sw->frag_z0 || hi >= sw->frag_z0 + sw->nzf || hi < lo) return fail(BD3MG_EINVAL, "block outside the fragment");
    bd3mg_task_t& t = tasks[b];
    t.frag = x; t.frag_z0 = sw->frag_z0; t.nzf = sw->nzf; t.z_lo = lo; t.z_hi = hi;
    t.d_mem = dm ? dm + (lo - sw->frag_z0) * plane : nullptr;
    t.inc_out = nullptr;
    t.x_rows = x ? x + (lo - sw->frag_z0) * plane : nullptr;
    t.dmem_rows = dm ? dm + (lo - sw->frag_z0) * plane : nullptr;
    const int64_t olo = std::max<int64_t>(0, lo - rz), ohi = std::min<int64_t>(g->nz - 1, hi + rz);
    hd[b] = sw->hd_cache ? (T*)sw->hd_cache + hd_off : nullptr;
    hd_off += (ohi - olo + 1) * plane;
    hsum += hi - lo + 1;
    bmin = std::min(bmin, lo);
    bmax = std::max(bmax, hi);
  }
  const bool rec = sw->rec_hi >= sw->rec_lo;
  const int64_t nrec = rec ? sw->rec_hi - sw->rec_lo + 1 : 0;
  bool contiguous = true;  // blocks in order, back to back
  for (int b = 1; b < nb; ++b) contiguous &= sw->blocks[2 * b] == sw->blocks[2 * b - 1] + 1;
  const bool fused = rec && contiguous && bmin == sw->rec_lo && bmax == sw->rec_hi && hsum == nrec;
  if (rec && (sw->rec_lo < sw->frag_z0 || sw->rec_hi >= sw->frag_z0 + sw->nzf))
    return fail(BD3MG_EINVAL, "recorder rows outside the fragment");
  // the persistent one-launch sweep where it applies (bitwise the same results)
  size_t pk_need = 0;
  if (fused && !r_full) {
    Ws wp = ws;
    const int rc = pk_sweep<T>(g, r, K, y, sw, terms, info, wp, s, mirrors, nmirrors);
    if (ws.measure) {
      if (rc == BD3MG_OK) pk_need = wp.off;
    } else if (rc != kPkIneligible) {
      ws.off = wp.off;
      return rc;
    }
  }
  const long long erows = std::max<long long>(1, std::max<long long>(nrec * st_tiles(g), nb * z_tiles<T>(g)));
  double* eparts = ws.take<double>((size_t)erows * kEvalNV);
  double* sums = ws.take<double>(8);
  if (fused)
    for (int b = 0; b < nb; ++b) {
      const int64_t hb = sw->blocks[2 * b + 1] - sw->blocks[2 * b] + 1;
      grb[b] = ws.take<T>(hb * plane);
      wb[b] = ws.take<T>(hb * plane);
    }
  StepOpts<T> opt;
  opt.resid_sq = sums;
  opt.rec_lo = sw->rec_lo;
  opt.rec_hi = sw->rec_hi;
  opt.hd = sw->hd_cache ? hd.data() : nullptr;
  if (nmirrors < 0 || (nmirrors > 0 && !mirrors)) return fail(BD3MG_EINVAL, "invalid mirror list");
  for (int j = 0; j < nmirrors; ++j)
    if (!mirrors[j].dst || mirrors[j].z_hi < mirrors[j].z_lo) return fail(BD3MG_EINVAL, "invalid mirror %d", j);
  opt.mirrors = mirrors;
  opt.nmirrors = nmirrors;
  if (r_full) {
    // every residual row must be one this device's blocks update
    if (!sw->hd_cache) return fail(BD3MG_EINVAL, "the incremental residual needs the hd cache");
    if (sw->frag_z0 != 0 || sw->nzf != g->nz || !contiguous || bmin != 0 || bmax != g->nz - 1)
      return fail(BD3MG_EINVAL, "the incremental residual needs blocks tiling the whole volume on one device");
    opt.r_full = r_full;
    opt.r_full_z0 = 0;
    opt.r_refresh = r_refresh;
  }
  if (fused) { opt.greg = grb.data(); opt.omega = wb.data(); }
#ifndef BD3MG_EXP_SKIP_UPDATE
  opt.fin_sums = sums;  // the update launch writes the recorder terms
  opt.fin_terms = terms;
#endif
  // recorder terms + snapshot roll fused into the gradient correlation (no stencil pass)
  const bool rec_gradf = fused && gradf_ok<T>(g);
  if (rec_gradf) {
    opt.greg = nullptr;
    opt.omega = nullptr;
    opt.rec_gradf = true;
    opt.rec_snap = (T*)sw->snap;
    opt.rec_sums = sums + 1;
  }
  SideStream* ss = nullptr;
  cudaStream_t s1 = s;  // stream of the recorder / regulariser-gradient stencil
  // (function scope: the step below may run the stencil launches through opt.after_resid)
  const cudaEvent_t* chain_events = nullptr;
  std::function<int(int)> side_work;
  if (!ws.measure && rec_gradf) {
    if (!ws.ok()) return ws_fail(ws);
    if (!getenv("BD3MG_NO_SIDE_STREAM")) {
      CU(side_stream(s, &ss));
      opt.ss = ss;
    }
  } else if (!ws.measure) {
    if (!ws.ok()) return ws_fail(ws);
    if (fused && !getenv("BD3MG_NO_SIDE_STREAM")) {
      CU(side_stream(s, &ss));
      opt.ss = ss;
      CU(hop(s, ss->side, ss->ev[0]));  // fork: the stencil runs next to the residual correlation
      opt.side_forked = true;
      s1 = ss->side;
    }
    // (1) recorder pass of the anchor (+ regulariser gradient when fused), snapshot roll
    side_work = [&, s1](int phase) -> int {
    if (!rec) {
      if (phase >= 0 && phase < chain_parts<T>(true, nb, hsum * plane) - 1) return BD3MG_OK;
      CU(cudaMemsetAsync(sums + 1, 0, kEvalNV * sizeof(double), s1));
    } else {
      StArgs<T> e = st_args<T>(g, r);
      e.partials = eparts;
      if (fused) {
        e.njobs = nb;
        for (int b = 0; b < nb; ++b) {
          StJob<T>& J = e.jobs[b];
          J.a = x; J.a_z0 = sw->frag_z0; J.lo = (int)sw->blocks[2 * b]; J.hi = (int)sw->blocks[2 * b + 1];
          J.b = sw->snap ? (const T*)sw->snap + (J.lo - sw->rec_lo) * plane : nullptr;
          J.snap_out = sw->snap ? (T*)sw->snap + (J.lo - sw->rec_lo) * plane : nullptr;  // snapshot roll
          J.out0 = grb[b]; J.out1 = wb[b];
        }
#ifndef BD3MG_EXP_SKIP_GREG
        if (chain_events) {
          // one stencil launch per chain of the block step (partial rows stay job-major), an event after each
          const int parts = chain_parts<T>(true, nb, hsum * plane);
          for (int part = 0; part < parts; ++part) {
            if (phase >= 0 && part != phase) continue;
            const int b0 = (int)((long long)nb * part / parts), b1 = (int)((long long)nb * (part + 1) / parts);
            StArgs<T> ep = e;
            ep.njobs = b1 - b0;
            for (int b = b0; b < b1; ++b) ep.jobs[b - b0] = e.jobs[b];
            ep.partials = eparts + (size_t)b0 * z_tiles<T>(g) * kEvalNV;
            int rc = launch_greg<T>(ep, true, s1, kGregPad);
            if (rc) return rc;
            CU(cudaEventRecord(chain_events[part], s1));
          }
        } else {
          // (next to the residual correlation on the side stream: the same residency bound, measured at
          // fp32 too -- C2 fp32 282.9 -> 279.1 us, C3 3784 -> 3770 us)
          const bool beside_resid = s1 != s && !(r_full && !r_refresh);
          int rc = launch_greg<T>(e, true, s1, beside_resid ? kGregPad : 0);
          if (rc) return rc;
        }
#endif
      } else {
        e.njobs = 1;
        e.jobs[0].a = x; e.jobs[0].a_z0 = sw->frag_z0; e.jobs[0].b = (const T*)sw->snap;
        e.jobs[0].lo = (int)sw->rec_lo; e.jobs[0].hi = (int)sw->rec_hi;
        CU(st_launch<T>(eval_kernel<T>, e, s1));
      }
      if (phase >= 0 && phase < chain_parts<T>(true, nb, hsum * plane) - 1) return BD3MG_OK;  // (the reduction follows the last stencil launch)
      CU(reduce(eparts, kEvalNV, {{0, fused ? nb * z_tiles<T>(g) : nrec * st_tiles(g)}}, sums + 1, kEvalNV, s1));
      if (sw->snap && !fused)  // fused: the stencil rolled the snapshot as it read it
        CU(cudaMemcpyAsync(sw->snap, x + (sw->rec_lo - sw->frag_z0) * plane, (size_t)nrec * plane * sizeof(T),
                           cudaMemcpyDeviceToDevice, s1));
    }
      return BD3MG_OK;
    };
    // The stencil is enqueued right AFTER the residual correlation's launch: the block scheduler serves
    // equal-priority kernels in launch order, so the correlation's CTAs go first and the stencil fills its
    // last wave instead of holding every SM for the sweep's first 27 us; and it is launched once per chain
    // of the block step, so the first chain's gradient correlation starts as soon as its own blocks'
    // regulariser gradient is there (C2 fp64: 409 -> 406 us; fp32, one chain: 1% slower at C2, neutral at
    // C3, so fp64 only).  BD3MG_GREG_AFTER=0: the stencil first.
    const char* ga = getenv("BD3MG_GREG_AFTER");  // (read per call: the tests switch it)
    const bool greg_after = ga ? ga[0] != '0' : true;
    if (greg_after && chain_parts<T>(true, nb, hsum * plane) > 1 && opt.side_forked && !(r_full && !r_refresh)) {
      opt.after_resid = side_work;
      if (fused && rec && chain_parts<T>(true, nb, hsum * plane) > 1 && !getenv("BD3MG_NO_CHAIN_GREG")) {
        chain_events = ss->ev + 8 + 5 * kMaxParts;  // kMaxParts events after the chain events
        opt.chain_ready = chain_events;
      }
    } else {
      const int rc0 = side_work(-1);
      if (rc0) return rc0;
    }
  }
  // (2) the fused block steps at the anchor (x, dmem updated in place)
  Ws sub = ws;
  int rc = mg_steps_chunk<T>(g, r, K, y, tasks.data(), nb, info, sub, s, opt);
  ws.off = std::max(sub.off, pk_need);
  if (rc != BD3MG_OK || ws.measure) return rc;
  if (!ws.ok()) return ws_fail(ws);
#ifdef BD3MG_EXP_SKIP_UPDATE
  eval_finalize_kernel<<<1, 1, 0, s>>>(sums, sums + 1, r->eta, r->lam, r->kappa, terms); launched();
  CU(cudaGetLastError());
#endif
  return BD3MG_OK;
}

template <typename F>
size_t measure(F&& f) {
  Ws ws;
  ws.measure = true;
  if (f(ws) != BD3MG_OK) return (size_t)-1;
  return ws.off + 256;
}

Ws make_ws(void* p, size_t n) {
  Ws ws;
  ws.base = (char*)p;
  ws.cap = n;
  ws.measure = false;
  return ws;
}

}  // namespace

// ---------------------------------------------------------------------------
namespace bd3mg {
int set_error(int code, const char* msg) { return fail(code, "%s", msg); }
void count_launches(int n) { launched(n); }

bool encode_tmap(CUtensorMap* map, const void* base, bool f64, long long nx, long long ny, long long nz, int boxw,
                 int boxh, int boxd) {
  static const PFN_cuTensorMapEncodeTiled_v12000 fn = []() -> PFN_cuTensorMapEncodeTiled_v12000 {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
    return nullptr;
  }();  // thread-safe one-time lookup
  const size_t es = f64 ? 8 : 4;
  if (!fn || !base || (reinterpret_cast<uintptr_t>(base) & 15) || ((size_t)nx * es) % 16 || boxw > 256 ||
      boxh > 256 || boxd < 1 || boxd > 256 || ((size_t)boxw * es) % 16)
    return false;
  const cuuint64_t dims[3] = {(cuuint64_t)nx, (cuuint64_t)ny, (cuuint64_t)nz};
  const cuuint64_t strides[2] = {(cuuint64_t)(nx * es), (cuuint64_t)(nx * ny * es)};
  const cuuint32_t box[3] = {(cuuint32_t)boxw, (cuuint32_t)boxh, (cuuint32_t)boxd};
  const cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = fn(map, f64 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3,
                  const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}
}  // namespace bd3mg

// ===========================================================================
extern "C" {

const char* bd3mg_last_error(void) { return g_err.c_str(); }
const char* bd3mg_version(void) { return "bd3mg_b200 0.1 sm_100a"; }

// This library links its own (static) CUDA runtime: its notion of the
// calling thread's current device is bound explicitly to the device of the
// caller's stream (one process per GPU: rank r on device r).
int bd3mg_set_device(int device) {
  CU(cudaSetDevice(device));
  return BD3MG_OK;
}
int bd3mg_get_device(int* device) {
  if (!device) return fail(BD3MG_EINVAL, "null argument");
  CU(cudaGetDevice(device));
  return BD3MG_OK;
}
long long bd3mg_launch_count(void) { return g_launches.load(); }

int bd3mg_depthvar_correlate_f64(const double* frag, int64_t nzf, int64_t ny, int64_t nx, const double* kernels,
                                 int64_t nzk, int64_t kz, int64_t ky, int64_t kx, int64_t frag_z0, int64_t out_lo,
                                 int64_t out_hi, double* out, void* stream) {
  return correlate_rows<double>(frag, nzf, ny, nx, kernels, nzk, kz, ky, kx, frag_z0, out_lo, out_hi, out, false,
                                (cudaStream_t)stream);
}
int bd3mg_depthvar_correlate_adjoint_f64(const double* frag, int64_t nzf, int64_t ny, int64_t nx,
                                         const double* kernels, int64_t nzk, int64_t kz, int64_t ky, int64_t kx,
                                         int64_t frag_z0, int64_t out_lo, int64_t out_hi, double* out,
                                         void* stream) {
  return correlate_rows<double>(frag, nzf, ny, nx, kernels, nzk, kz, ky, kx, frag_z0, out_lo, out_hi, out, true,
                                (cudaStream_t)stream);
}
int bd3mg_depthvar_correlate_f32(const float* frag, int64_t nzf, int64_t ny, int64_t nx, const float* kernels,
                                 int64_t nzk, int64_t kz, int64_t ky, int64_t kx, int64_t frag_z0, int64_t out_lo,
                                 int64_t out_hi, float* out, void* stream) {
  return correlate_rows<float>(frag, nzf, ny, nx, kernels, nzk, kz, ky, kx, frag_z0, out_lo, out_hi, out, false,
                               (cudaStream_t)stream);
}
int bd3mg_depthvar_correlate_adjoint_f32(const float* frag, int64_t nzf, int64_t ny, int64_t nx,
                                         const float* kernels, int64_t nzk, int64_t kz, int64_t ky, int64_t kx,
                                         int64_t frag_z0, int64_t out_lo, int64_t out_hi, float* out,
                                         void* stream) {
  return correlate_rows<float>(frag, nzf, ny, nx, kernels, nzk, kz, ky, kx, frag_z0, out_lo, out_hi, out, true,
                               (cudaStream_t)stream);
}

static int correlate_host(const double* frag, int64_t nzf, int64_t ny, int64_t nx, const double* kernels,
                          int64_t nzk, int64_t kz, int64_t ky, int64_t kx, int64_t frag_z0, int64_t out_lo,
                          int64_t out_hi, double* out, bool adj) {
  const int64_t nout = out_hi - out_lo + 1;
  if (nout <= 0 || nzf < 1 || ny < 1 || nx < 1 || nzk < 1) {
    return correlate_rows<double>(nullptr, nzf, ny, nx, nullptr, nzk, kz, ky, kx, frag_z0, out_lo, out_hi, nullptr,
                                  adj, 0);
  }
  const size_t nf = (size_t)nzf * ny * nx, nk = (size_t)nzk * kz * ky * kx, no = (size_t)nout * ny * nx;
  double *df = nullptr, *dk = nullptr, *dout = nullptr;
  cudaStream_t s;
  CU(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  int rc = BD3MG_OK;
  do {
    if (cudaMallocAsync(&df, nf * 8, s) != cudaSuccess || cudaMallocAsync(&dk, nk * 8, s) != cudaSuccess ||
        cudaMallocAsync(&dout, no * 8, s) != cudaSuccess) {
      rc = fail(BD3MG_ECUDA, "device allocation failed");
      break;
    }
    if (cudaMemcpyAsync(df, frag, nf * 8, cudaMemcpyHostToDevice, s) != cudaSuccess ||
        cudaMemcpyAsync(dk, kernels, nk * 8, cudaMemcpyHostToDevice, s) != cudaSuccess) {
      rc = fail(BD3MG_ECUDA, "host-to-device copy failed");
      break;
    }
    rc = correlate_rows<double>(df, nzf, ny, nx, dk, nzk, kz, ky, kx, frag_z0, out_lo, out_hi, dout, adj, s);
    if (rc != BD3MG_OK) break;
    if (cudaMemcpyAsync(out, dout, no * 8, cudaMemcpyDeviceToHost, s) != cudaSuccess) {
      rc = fail(BD3MG_ECUDA, "device-to-host copy failed");
      break;
    }
  } while (0);
  if (df) cudaFreeAsync(df, s);
  if (dk) cudaFreeAsync(dk, s);
  if (dout) cudaFreeAsync(dout, s);
  cudaError_t e = cudaStreamSynchronize(s);
  cudaStreamDestroy(s);
  if (rc == BD3MG_OK && e != cudaSuccess) rc = fail(BD3MG_ECUDA, "%s", cudaGetErrorString(e));
  return rc;
}

int bd3mg_depthvar_correlate_host_f64(const double* frag, int64_t nzf, int64_t ny, int64_t nx,
                                      const double* kernels, int64_t nzk, int64_t kz, int64_t ky, int64_t kx,
                                      int64_t frag_z0, int64_t out_lo, int64_t out_hi, double* out) {
  return correlate_host(frag, nzf, ny, nx, kernels, nzk, kz, ky, kx, frag_z0, out_lo, out_hi, out, false);
}
int bd3mg_depthvar_correlate_adjoint_host_f64(const double* frag, int64_t nzf, int64_t ny, int64_t nx,
                                              const double* kernels, int64_t nzk, int64_t kz, int64_t ky,
                                              int64_t kx, int64_t frag_z0, int64_t out_lo, int64_t out_hi,
                                              double* out) {
  return correlate_host(frag, nzf, ny, nx, kernels, nzk, kz, ky, kx, frag_z0, out_lo, out_hi, out, true);
}

// ---- fused operators ------------------------------------------------------
#define DISPATCH_T(g, CALL_F64, CALL_F32) ((g)->dtype == BD3MG_F64 ? (CALL_F64) : (CALL_F32))

size_t bd3mg_grad_rows_ws_bytes(const bd3mg_geom_t* g, int64_t lo, int64_t hi) {
  if (check_geom(g) != BD3MG_OK) return (size_t)-1;
  return measure([&](Ws& ws) {
    return DISPATCH_T(g,
                      grad_rows_impl<double>(g, nullptr, nullptr, nullptr, nullptr, 0, g->nz, lo, hi, nullptr,
                                             nullptr, ws, 0),
                      grad_rows_impl<float>(g, nullptr, nullptr, nullptr, nullptr, 0, g->nz, lo, hi, nullptr,
                                            nullptr, ws, 0));
  });
}

int bd3mg_grad_rows(const bd3mg_geom_t* g, const bd3mg_reg_t* r, const void* kernels, const void* y,
                    const void* frag, int64_t frag_z0, int64_t nzf, int64_t lo, int64_t hi, void* g_out,
                    void* omega_out, void* wsp, size_t ws_bytes, void* stream) {
  int rc = check_geom(g);
  if (rc) return rc;
  if (!r) return fail(BD3MG_EINVAL, "null regulariser");
  Ws ws = make_ws(wsp, ws_bytes);
  return DISPATCH_T(g,
                    grad_rows_impl<double>(g, r, (const double*)kernels, (const double*)y, (const double*)frag,
                                           frag_z0, nzf, lo, hi, (double*)g_out, (double*)omega_out, ws,
                                           (cudaStream_t)stream),
                    grad_rows_impl<float>(g, r, (const float*)kernels, (const float*)y, (const float*)frag, frag_z0,
                                          nzf, lo, hi, (float*)g_out, (float*)omega_out, ws,
                                          (cudaStream_t)stream));
}

size_t bd3mg_eval_f_ws_bytes(const bd3mg_geom_t* g) {
  if (check_geom(g) != BD3MG_OK) return (size_t)-1;
  bd3mg_reg_t r{1, 1, 1, 1, 0, 1};
  return measure([&](Ws& ws) {
    return DISPATCH_T(g, eval_f_impl<double>(g, &r, nullptr, nullptr, nullptr, nullptr, nullptr, ws, 0),
                      eval_f_impl<float>(g, &r, nullptr, nullptr, nullptr, nullptr, nullptr, ws, 0));
  });
}

int bd3mg_eval_f(const bd3mg_geom_t* g, const bd3mg_reg_t* r, const void* kernels, const void* y, const void* x,
                 const void* snap, double* terms_out, void* wsp, size_t ws_bytes, void* stream) {
  int rc = check_geom(g);
  if (rc) return rc;
  if (!r) return fail(BD3MG_EINVAL, "null regulariser");
  Ws ws = make_ws(wsp, ws_bytes);
  return DISPATCH_T(g,
                    eval_f_impl<double>(g, r, (const double*)kernels, (const double*)y, (const double*)x,
                                        (const double*)snap, terms_out, ws, (cudaStream_t)stream),
                    eval_f_impl<float>(g, r, (const float*)kernels, (const float*)y, (const float*)x,
                                       (const float*)snap, terms_out, ws, (cudaStream_t)stream));
}

size_t bd3mg_eval_rows_ws_bytes(const bd3mg_geom_t* g, int64_t lo, int64_t hi) {
  if (check_geom(g) != BD3MG_OK) return (size_t)-1;
  bd3mg_reg_t r{1, 1, 1, 1, 0, 1};
  return measure([&](Ws& ws) {
    return DISPATCH_T(g, eval_rows_impl<double>(g, &r, nullptr, nullptr, nullptr, 0, g->nz, lo, hi, nullptr, nullptr,
                                                ws, 0),
                      eval_rows_impl<float>(g, &r, nullptr, nullptr, nullptr, 0, g->nz, lo, hi, nullptr, nullptr,
                                            ws, 0));
  });
}

int bd3mg_eval_rows(const bd3mg_geom_t* g, const bd3mg_reg_t* r, const void* kernels, const void* y_rows,
                    const void* frag, int64_t frag_z0, int64_t nzf, int64_t lo, int64_t hi, const void* snap_rows,
                    double* terms_out, void* wsp, size_t ws_bytes, void* stream) {
  int rc = check_geom(g);
  if (rc) return rc;
  if (!r) return fail(BD3MG_EINVAL, "null regulariser");
  Ws ws = make_ws(wsp, ws_bytes);
  return DISPATCH_T(g,
                    eval_rows_impl<double>(g, r, (const double*)kernels, (const double*)y_rows, (const double*)frag,
                                           frag_z0, nzf, lo, hi, (const double*)snap_rows, terms_out, ws,
                                           (cudaStream_t)stream),
                    eval_rows_impl<float>(g, r, (const float*)kernels, (const float*)y_rows, (const float*)frag,
                                          frag_z0, nzf, lo, hi, (const float*)snap_rows, terms_out, ws,
                                          (cudaStream_t)stream));
}

int bd3mg_omega_rows(const bd3mg_geom_t* g, const bd3mg_reg_t* r, const void* frag, int64_t frag_z0, int64_t nzf,
                     int64_t lo, int64_t hi, void* omega_out, void* stream) {
  int rc = check_geom(g);
  if (rc) return rc;
  if (!r) return fail(BD3MG_EINVAL, "null regulariser");
  return DISPATCH_T(g,
                    omega_impl<double>(g, r, (const double*)frag, frag_z0, nzf, lo, hi, (double*)omega_out,
                                       (cudaStream_t)stream),
                    omega_impl<float>(g, r, (const float*)frag, frag_z0, nzf, lo, hi, (float*)omega_out,
                                      (cudaStream_t)stream));
}

int bd3mg_apply_increment(int32_t dtype, void* x_rows, void* dmem_rows, const void* inc, int64_t n, void* stream) {
  if (n < 0 || !x_rows || !inc) return fail(BD3MG_EINVAL, "invalid increment arguments");
  if (n == 0) return BD3MG_OK;
  const unsigned grid = (unsigned)std::min<int64_t>((n + kEwNT - 1) / kEwNT, 4 * 148);
  if (dtype == BD3MG_F64)
    apply_increment_kernel<double><<<grid, kEwNT, 0, (cudaStream_t)stream>>>((double*)x_rows, (double*)dmem_rows,
                                                                            (const double*)inc, n);
  else if (dtype == BD3MG_F32)
    apply_increment_kernel<float><<<grid, kEwNT, 0, (cudaStream_t)stream>>>((float*)x_rows, (float*)dmem_rows,
                                                                           (const float*)inc, n);
  else
    return fail(BD3MG_EINVAL, "unknown dtype %d", dtype);
  launched();
  CU(cudaGetLastError());
  return BD3MG_OK;
}

size_t bd3mg_majorant_apply_ws_bytes(const bd3mg_geom_t* g, int64_t lo, int64_t hi) {
  if (check_geom(g) != BD3MG_OK) return (size_t)-1;
  bd3mg_reg_t r{1, 1, 1, 1, 0, 1};
  return measure([&](Ws& ws) {
    return DISPATCH_T(g, majorant_impl<double>(g, &r, nullptr, nullptr, nullptr, lo, hi, nullptr, ws, 0),
                      majorant_impl<float>(g, &r, nullptr, nullptr, nullptr, lo, hi, nullptr, ws, 0));
  });
}

int bd3mg_majorant_apply(const bd3mg_geom_t* g, const bd3mg_reg_t* r, const void* kernels, const void* omega,
                         const void* v, int64_t lo, int64_t hi, void* out, void* wsp, size_t ws_bytes,
                         void* stream) {
  int rc = check_geom(g);
  if (rc) return rc;
  if (!r) return fail(BD3MG_EINVAL, "null regulariser");
  Ws ws = make_ws(wsp, ws_bytes);
  return DISPATCH_T(g,
                    majorant_impl<double>(g, r, (const double*)kernels, (const double*)omega, (const double*)v, lo,
                                          hi, (double*)out, ws, (cudaStream_t)stream),
                    majorant_impl<float>(g, r, (const float*)kernels, (const float*)omega, (const float*)v, lo, hi,
                                         (float*)out, ws, (cudaStream_t)stream));
}

size_t bd3mg_cg_solve_ws_bytes(const bd3mg_geom_t* g, int64_t lo, int64_t hi) {
  if (check_geom(g) != BD3MG_OK) return (size_t)-1;
  bd3mg_reg_t r{1, 1, 1, 1, 0, 1};
  return measure([&](Ws& ws) {
    return DISPATCH_T(g, cg_solve_impl<double>(g, &r, nullptr, nullptr, nullptr, lo, hi, 1.0, 1, nullptr, nullptr, ws, 0),
                      cg_solve_impl<float>(g, &r, nullptr, nullptr, nullptr, lo, hi, 1.0, 1, nullptr, nullptr, ws, 0));
  });
}

int bd3mg_cg_solve(const bd3mg_geom_t* g, const bd3mg_reg_t* r, const void* kernels, const void* omega, const void* b,
                   int64_t lo, int64_t hi, double tol, int32_t maxit, void* x_out, double* state_out, void* wsp,
                   size_t ws_bytes, void* stream) {
  int rc = check_geom(g);
  if (rc) return rc;
  if (!r || !kernels || !omega || !b || !x_out) return fail(BD3MG_EINVAL, "null argument");
  Ws ws = make_ws(wsp, ws_bytes);
  return DISPATCH_T(g,
                    cg_solve_impl<double>(g, r, (const double*)kernels, (const double*)omega, (const double*)b, lo, hi,
                                          tol, maxit, (double*)x_out, state_out, ws, (cudaStream_t)stream),
                    cg_solve_impl<float>(g, r, (const float*)kernels, (const float*)omega, (const float*)b, lo, hi,
                                         tol, maxit, (float*)x_out, state_out, ws, (cudaStream_t)stream));
}

size_t bd3mg_power_hth_ws_bytes(const bd3mg_geom_t* g) {
  if (check_geom(g) != BD3MG_OK) return (size_t)-1;
  return measure([&](Ws& ws) {
    return DISPATCH_T(g, power_hth_impl<double>(g, nullptr, nullptr, 1, nullptr, nullptr, ws, 0),
                      power_hth_impl<float>(g, nullptr, nullptr, 1, nullptr, nullptr, ws, 0));
  });
}

int bd3mg_power_hth(const bd3mg_geom_t* g, const void* kernels, void* v, int32_t iters, double* norms_out,
                    double* state_out, void* wsp, size_t ws_bytes, void* stream) {
  int rc = check_geom(g);
  if (rc) return rc;
  if (!kernels || !v || (iters > 0 && !norms_out)) return fail(BD3MG_EINVAL, "null argument");
  Ws ws = make_ws(wsp, ws_bytes);
  return DISPATCH_T(g,
                    power_hth_impl<double>(g, (const double*)kernels, (double*)v, iters, norms_out, state_out, ws,
                                           (cudaStream_t)stream),
                    power_hth_impl<float>(g, (const float*)kernels, (float*)v, iters, norms_out, state_out, ws,
                                          (cudaStream_t)stream));
}

long long bd3mg_pk_launches(void) { return g_pk_launches.load(); }

int bd3mg_pk_trace(void* host, int64_t max_items, int64_t* n_out) {
  PkTrace& tr = pk_trace();
  std::lock_guard<std::mutex> lock(tr.mu);
  CU(cudaDeviceSynchronize());
  const int64_t n = std::min<int64_t>((int64_t)tr.n, max_items);
  if (n_out) *n_out = (int64_t)tr.n;
  if (host && n > 0) CU(cudaMemcpy(host, tr.buf, (size_t)n * 32, cudaMemcpyDeviceToHost));
  return BD3MG_OK;
}

size_t bd3mg_jacobi_sweep_ws_bytes(const bd3mg_geom_t* g, const bd3mg_sweep_t* sw) {
  if (check_geom(g) != BD3MG_OK) return (size_t)-1;
  bd3mg_reg_t r{1, 1, 1, 1, 0, 1};
  return measure([&](Ws& ws) {
    return DISPATCH_T(g, jacobi_sweep_impl<double>(g, &r, nullptr, nullptr, sw, nullptr, nullptr, ws, 0),
                      jacobi_sweep_impl<float>(g, &r, nullptr, nullptr, sw, nullptr, nullptr, ws, 0));
  });
}

int64_t bd3mg_jacobi_cache_elems(const bd3mg_geom_t* g, const bd3mg_sweep_t* sw) {
  if (check_geom(g) != BD3MG_OK || !sw) return -1;
  const int64_t plane = g->ny * g->nx, rz = (g->kz - 1) / 2;
  int64_t n = 0;
  for (int b = 0; b < sw->nblocks; ++b) {
    const int64_t lo = sw->blocks[2 * b], hi = sw->blocks[2 * b + 1];
    n += (std::min<int64_t>(g->nz - 1, hi + rz) - std::max<int64_t>(0, lo - rz) + 1) * plane;
  }
  return n;
}

int bd3mg_jacobi_sweep(const bd3mg_geom_t* g, const bd3mg_reg_t* r, const void* kernels, const void* y,
                       const bd3mg_sweep_t* sw, double* terms_out, double* info_out, void* wsp, size_t ws_bytes,
                       void* stream) {
  int rc = check_geom(g);
  if (rc) return rc;
  if (!r || !sw || !info_out || !terms_out) return fail(BD3MG_EINVAL, "null argument");
  Ws ws = make_ws(wsp, ws_bytes);
  cudaStream_t s = (cudaStream_t)stream;
  return DISPATCH_T(g,
                    jacobi_sweep_impl<double>(g, r, (const double*)kernels, (const double*)y, sw, terms_out, info_out,
                                              ws, s),
                    jacobi_sweep_impl<float>(g, r, (const float*)kernels, (const float*)y, sw, terms_out, info_out, ws,
                                             s));
}

int bd3mg_jacobi_sweep_mirrored(const bd3mg_geom_t* g, const bd3mg_reg_t* r, const void* kernels, const void* y,
                                const bd3mg_sweep_t* sw, const bd3mg_mirror_t* mirrors, int nmirrors,
                                double* terms_out, double* info_out, void* wsp, size_t ws_bytes, void* stream) {
  int rc = check_geom(g);
  if (rc) return rc;
  if (!r || !sw || !info_out || !terms_out) return fail(BD3MG_EINVAL, "null argument");
  Ws ws = make_ws(wsp, ws_bytes);
  cudaStream_t s = (cudaStream_t)stream;
  return DISPATCH_T(g,
                    jacobi_sweep_impl<double>(g, r, (const double*)kernels, (const double*)y, sw, terms_out, info_out,
                                              ws, s, mirrors, nmirrors),
                    jacobi_sweep_impl<float>(g, r, (const float*)kernels, (const float*)y, sw, terms_out, info_out, ws,
                                             s, mirrors, nmirrors));
}

int bd3mg_jacobi_sweep_incremental(const bd3mg_geom_t* g, const bd3mg_reg_t* r, const void* kernels, const void* y,
                                   const bd3mg_sweep_t* sw, void* resid, int refresh, double* terms_out,
                                   double* info_out, void* wsp, size_t ws_bytes, void* stream) {
  int rc = check_geom(g);
  if (rc) return rc;
  if (!r || !sw || !info_out || !terms_out || !resid) return fail(BD3MG_EINVAL, "null argument");
  Ws ws = make_ws(wsp, ws_bytes);
  cudaStream_t s = (cudaStream_t)stream;
  return DISPATCH_T(g,
                    jacobi_sweep_impl<double>(g, r, (const double*)kernels, (const double*)y, sw, terms_out, info_out,
                                              ws, s, nullptr, 0, (double*)resid, refresh != 0),
                    jacobi_sweep_impl<float>(g, r, (const float*)kernels, (const float*)y, sw, terms_out, info_out, ws,
                                             s, nullptr, 0, (float*)resid, refresh != 0));
}

size_t bd3mg_mg_steps_incremental_ws_bytes(const bd3mg_geom_t* g, const bd3mg_task_t* tasks, int ntasks) {
  if (check_geom(g) != BD3MG_OK || ntasks < 1 || ntasks > kMaxJobs) return (size_t)-1;
  bd3mg_reg_t r{1, 1, 1, 1, 0, 1};
  std::vector<void*> hd(ntasks, reinterpret_cast<void*>(uintptr_t(4096)));  // placeholders: sizing only
  void* resid = reinterpret_cast<void*>(uintptr_t(4096));
  return measure([&](Ws& ws) {
    return DISPATCH_T(g,
                      mg_steps_impl<double>(g, &r, nullptr, nullptr, tasks, ntasks, nullptr, ws, 0, nullptr, 0,
                                            (double* const*)hd.data(), (double*)resid),
                      mg_steps_impl<float>(g, &r, nullptr, nullptr, tasks, ntasks, nullptr, ws, 0, nullptr, 0,
                                           (float* const*)hd.data(), (float*)resid));
  });
}

int bd3mg_mg_steps_incremental(const bd3mg_geom_t* g, const bd3mg_reg_t* r, const void* kernels, const void* y,
                               const bd3mg_task_t* tasks, int ntasks, void* const* hd, void* resid,
                               double* info_out, void* wsp, size_t ws_bytes, void* stream) {
  int rc = check_geom(g);
  if (rc) return rc;
  if (!r || !info_out || !hd || !resid) return fail(BD3MG_EINVAL, "null argument");
  Ws ws = make_ws(wsp, ws_bytes);
  return DISPATCH_T(g,
                    mg_steps_impl<double>(g, r, (const double*)kernels, (const double*)y, tasks, ntasks, info_out, ws,
                                          (cudaStream_t)stream, nullptr, 0, (double* const*)hd, (double*)resid),
                    mg_steps_impl<float>(g, r, (const float*)kernels, (const float*)y, tasks, ntasks, info_out, ws,
                                         (cudaStream_t)stream, nullptr, 0, (float* const*)hd, (float*)resid));
}

int bd3mg_eval_f_resid(const bd3mg_geom_t* g, const bd3mg_reg_t* r, const void* resid, const void* x,
                       const void* snap, double* terms_out, void* wsp, size_t ws_bytes, void* stream) {
  int rc = check_geom(g);
  if (rc) return rc;
  if (!r || !resid || !x || !terms_out) return fail(BD3MG_EINVAL, "null argument");
  Ws ws = make_ws(wsp, ws_bytes);
  cudaStream_t s = (cudaStream_t)stream;
  return DISPATCH_T(g,
                    eval_rows_impl<double>(g, r, nullptr, nullptr, (const double*)x, 0, g->nz, 0, g->nz - 1,
                                           (const double*)snap, terms_out, ws, s, (const double*)resid),
                    eval_rows_impl<float>(g, r, nullptr, nullptr, (const float*)x, 0, g->nz, 0, g->nz - 1,
                                          (const float*)snap, terms_out, ws, s, (const float*)resid));
}

/* ---- peer (NVLink) memory: halo inboxes written by other ranks' kernels ---- */
int bd3mg_peer_alloc(size_t bytes, void** dev_out, void* ipc_handle_out) {
  if (!dev_out || !ipc_handle_out || bytes == 0) return fail(BD3MG_EINVAL, "invalid peer allocation");
  void* p = nullptr;
  CU(cudaMalloc(&p, bytes));
  cudaError_t e = cudaMemset(p, 0, bytes);
  cudaIpcMemHandle_t h;
  if (e == cudaSuccess) e = cudaIpcGetMemHandle(&h, p);
  if (e != cudaSuccess) {
    cudaFree(p);
    return fail(BD3MG_ECUDA, "peer allocation: %s", cudaGetErrorString(e));
  }
  memcpy(ipc_handle_out, &h, sizeof(h));
  *dev_out = p;
  return BD3MG_OK;
}

int bd3mg_peer_open(const void* ipc_handle, void** dev_out) {
  if (!ipc_handle || !dev_out) return fail(BD3MG_EINVAL, "null argument");
  cudaIpcMemHandle_t h;
  memcpy(&h, ipc_handle, sizeof(h));
  CU(cudaIpcOpenMemHandle(dev_out, h, cudaIpcMemLazyEnablePeerAccess));
  return BD3MG_OK;
}

int bd3mg_mg_steps_mirrored(const bd3mg_geom_t* g, const bd3mg_reg_t* r, const void* kernels, const void* y,
                            const bd3mg_task_t* tasks, int ntasks, const bd3mg_mirror_t* mirrors, int nmirrors,
                            double* info_out, void* wsp, size_t ws_bytes, void* stream) {
  int rc = check_geom(g);
  if (rc) return rc;
  if (!r) return fail(BD3MG_EINVAL, "null regulariser");
  if (!info_out) return fail(BD3MG_EINVAL, "info_out is required");
  Ws ws = make_ws(wsp, ws_bytes);
  return DISPATCH_T(g,
                    mg_steps_impl<double>(g, r, (const double*)kernels, (const double*)y, tasks, ntasks, info_out,
                                          ws, (cudaStream_t)stream, mirrors, nmirrors),
                    mg_steps_impl<float>(g, r, (const float*)kernels, (const float*)y, tasks, ntasks, info_out, ws,
                                         (cudaStream_t)stream, mirrors, nmirrors));
}

int bd3mg_host_register(void* host, size_t bytes, void** dev_out) {
  if (!host || !dev_out || bytes == 0) return fail(BD3MG_EINVAL, "invalid host range");
  CU(cudaHostRegister(host, bytes, cudaHostRegisterMapped | cudaHostRegisterPortable));
  cudaError_t e = cudaHostGetDevicePointer(dev_out, host, 0);
  if (e != cudaSuccess) {
    cudaHostUnregister(host);
    return fail(BD3MG_ECUDA, "cudaHostGetDevicePointer: %s", cudaGetErrorString(e));
  }
  return BD3MG_OK;
}

int bd3mg_host_unregister(void* host) {
  if (host) CU(cudaHostUnregister(host));
  return BD3MG_OK;
}

int bd3mg_publish(const bd3mg_flag_t* flags, int nflags, void* stream) {
  if (nflags < 0 || nflags > BD3MG_MAX_FLAGS || (nflags > 0 && !flags))
    return fail(BD3MG_EINVAL, "1..%d flags per publish", BD3MG_MAX_FLAGS);
  if (nflags == 0) return BD3MG_OK;
  PubArgs a;
  a.n = nflags;
  for (int i = 0; i < nflags; ++i) {
    if (!flags[i].word) return fail(BD3MG_EINVAL, "null flag word %d", i);
    a.word[i] = (volatile long long*)flags[i].word;
    a.value[i] = flags[i].value;
  }
  publish_kernel<<<1, 1, 0, (cudaStream_t)stream>>>(a); launched();
  CU(cudaGetLastError());
  return BD3MG_OK;
}

int bd3mg_peer_close(void* dev) {
  if (dev) CU(cudaIpcCloseMemHandle(dev));
  return BD3MG_OK;
}

int bd3mg_peer_free(void* dev) {
  if (dev) CU(cudaFree(dev));
  return BD3MG_OK;
}

size_t bd3mg_mg_steps_ws_bytes(const bd3mg_geom_t* g, const bd3mg_task_t* tasks, int ntasks) {
  if (check_geom(g) != BD3MG_OK) return (size_t)-1;
  bd3mg_reg_t r{1, 1, 1, 1, 0, 1};
  return measure([&](Ws& ws) {
    return DISPATCH_T(g, mg_steps_impl<double>(g, &r, nullptr, nullptr, tasks, ntasks, nullptr, ws, 0),
                      mg_steps_impl<float>(g, &r, nullptr, nullptr, tasks, ntasks, nullptr, ws, 0));
  });
}

int bd3mg_mg_steps(const bd3mg_geom_t* g, const bd3mg_reg_t* r, const void* kernels, const void* y,
                   const bd3mg_task_t* tasks, int ntasks, double* info_out, void* wsp, size_t ws_bytes,
                   void* stream) {
  int rc = check_geom(g);
  if (rc) return rc;
  if (!r) return fail(BD3MG_EINVAL, "null regulariser");
  if (!info_out) return fail(BD3MG_EINVAL, "info_out is required");
  Ws ws = make_ws(wsp, ws_bytes);
  return DISPATCH_T(g,
                    mg_steps_impl<double>(g, r, (const double*)kernels, (const double*)y, tasks, ntasks, info_out,
                                          ws, (cudaStream_t)stream),
                    mg_steps_impl<float>(g, r, (const float*)kernels, (const float*)y, tasks, ntasks, info_out, ws,
                                         (cudaStream_t)stream));
}

}  // extern "C"

// ---- host-buffer problem handle --------------------------------------------
namespace {
__global__ void cvt_kernel_f64_to_f32(const double* __restrict__ a, float* __restrict__ b, long long n) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    b[i] = (float)a[i];
}
__global__ void cvt_kernel_f32_to_f64(const float* __restrict__ a, double* __restrict__ b, long long n) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    b[i] = (double)a[i];
}
struct DevBuf {
  void* p = nullptr;
  size_t n = 0;
  cudaError_t reserve(size_t bytes) {
    if (bytes <= n) return cudaSuccess;
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
    cudaError_t e = cudaMalloc(&p, bytes);
    if (e == cudaSuccess) n = bytes;
    return e;
  }
  ~DevBuf() { if (p) cudaFree(p); }
};
}  // namespace

constexpr int kPipeMax = 8;     // groups of the pipelined host sweep (upper bound)
constexpr int kPipeGroups = 4;  // default, measured: e2e 5970 (2), 6260 (3), 6266 (4) block-it/s at C2

struct bd3mg_problem {
  bd3mg_geom_t g;
  bd3mg_reg_t r;
  int device;
  cudaStream_t s;
  DevBuf K, y, stage, slab, dmem, inc, info, ws, terms;
  DevBuf dmem_res;          // device-resident memory store (sweep with dmem == NULL)
  int64_t dmem_res_z0 = -1, dmem_res_n = 0;
  // pipelined host sweep: copy streams, per-group fragments / workspaces, events
  cudaStream_t s_in = nullptr, s_out = nullptr;
  cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
  cudaEvent_t ev_piece[kPipeMax] = {};
  DevBuf frag[kPipeMax], gws[kPipeMax];
  double* info_h = nullptr;   // pinned: per-block records of the last pipelined sweep
  double* terms_h = nullptr;  // pinned: per-group recorder terms
  cudaGraphExec_t graph = nullptr;
  std::vector<int64_t> graph_key;
  int graph_groups = 0;
  // calls on one handle share its stream, staging buffers and workspace:
  // they serialise here (the reference's live engine calls its core from
  // several worker threads at once; give each thread its own handle for
  // concurrent work)
  std::mutex mu;
};

static int download_f64(bd3mg_problem* p, const DevBuf& src, size_t n, double* host) {
  if (p->g.dtype == BD3MG_F64) {
    CU(cudaMemcpyAsync(host, src.p, n * 8, cudaMemcpyDeviceToHost, p->s));
  } else {
    CU(p->stage.reserve(n * 8));
    cvt_kernel_f32_to_f64<<<592, 256, 0, p->s>>>((const float*)src.p, (double*)p->stage.p, (long long)n);
    launched();
    CU(cudaGetLastError());
    CU(cudaMemcpyAsync(host, p->stage.p, n * 8, cudaMemcpyDeviceToHost, p->s));
  }
  return BD3MG_OK;
}

static int upload_f64(bd3mg_problem* p, const double* host, size_t n, DevBuf& dst) {
  const size_t esz = p->g.dtype == BD3MG_F64 ? 8 : 4;
  CU(dst.reserve(n * esz));
  if (p->g.dtype == BD3MG_F64) {
    CU(cudaMemcpyAsync(dst.p, host, n * 8, cudaMemcpyHostToDevice, p->s));
  } else {
    CU(p->stage.reserve(n * 8));
    CU(cudaMemcpyAsync(p->stage.p, host, n * 8, cudaMemcpyHostToDevice, p->s));
    cvt_kernel_f64_to_f32<<<592, 256, 0, p->s>>>((const double*)p->stage.p, (float*)dst.p, (long long)n);
    CU(cudaGetLastError());
  }
  return BD3MG_OK;
}

extern "C" {

int bd3mg_problem_create(const bd3mg_geom_t* g, const bd3mg_reg_t* r, const double* kernels_host,
                         const double* y_host, int device, bd3mg_problem** out) {
  int rc = check_geom(g);
  if (rc) return rc;
  if (!r || !kernels_host || !y_host || !out) return fail(BD3MG_EINVAL, "null argument");
  CU(cudaSetDevice(device));
  bd3mg_problem* p = new bd3mg_problem();
  p->g = *g;
  p->r = *r;
  p->device = device;
  if (cudaStreamCreateWithFlags(&p->s, cudaStreamNonBlocking) != cudaSuccess) {
    delete p;
    return fail(BD3MG_ECUDA, "stream creation failed");
  }
  const size_t nk = (size_t)g->nz * g->kz * g->ky * g->kx, nv = (size_t)g->nz * g->ny * g->nx;
  rc = upload_f64(p, kernels_host, nk, p->K);
  if (!rc) rc = upload_f64(p, y_host, nv, p->y);
  if (!rc && cudaStreamSynchronize(p->s) != cudaSuccess) rc = fail(BD3MG_ECUDA, "upload failed");
  if (rc) {
    bd3mg_problem_destroy(p);
    return rc;
  }
  *out = p;
  return BD3MG_OK;
}

int bd3mg_problem_destroy(bd3mg_problem* p) {
  if (!p) return BD3MG_OK;
  cudaSetDevice(p->device);
  cudaStreamSynchronize(p->s);
  for (cudaStream_t t : {p->s_in, p->s_out})
    if (t) {
      cudaStreamSynchronize(t);
      cudaStreamDestroy(t);
    }
  for (cudaEvent_t e : p->ev)
    if (e) cudaEventDestroy(e);
  for (cudaEvent_t e : p->ev_piece)
    if (e) cudaEventDestroy(e);
  if (p->graph) cudaGraphExecDestroy(p->graph);
  if (p->info_h) cudaFreeHost(p->info_h);
  if (p->terms_h) cudaFreeHost(p->terms_h);
  cudaStreamDestroy(p->s);
  delete p;
  return BD3MG_OK;
}

int bd3mg_problem_mg_direction_host(bd3mg_problem* p, const double* x_slab, int64_t slab_z0, int64_t nzs,
                                    int64_t z_lo, int64_t z_hi, const double* d_mem, double* inc_out,
                                    double* info_out) {
  if (!p || !x_slab || !inc_out) return fail(BD3MG_EINVAL, "null argument");
  std::lock_guard<std::mutex> lock(p->mu);
  CU(cudaSetDevice(p->device));
  const bd3mg_geom_t* g = &p->g;
  const int64_t plane = g->ny * g->nx, h = z_hi - z_lo + 1;
  if (h < 1) return fail(BD3MG_EINVAL, "empty block");
  const size_t esz = g->dtype == BD3MG_F64 ? 8 : 4;
  int rc = upload_f64(p, x_slab, (size_t)nzs * plane, p->slab);
  if (rc) return rc;
  if (d_mem) {
    rc = upload_f64(p, d_mem, (size_t)h * plane, p->dmem);
    if (rc) return rc;
  }
  CU(p->inc.reserve((size_t)h * plane * esz));
  CU(p->info.reserve(BD3MG_INFO_DOUBLES * sizeof(double)));
  bd3mg_task_t t;
  memset(&t, 0, sizeof(t));
  t.frag = p->slab.p; t.frag_z0 = slab_z0; t.nzf = nzs; t.z_lo = z_lo; t.z_hi = z_hi;
  t.d_mem = d_mem ? p->dmem.p : nullptr;
  t.inc_out = p->inc.p;
  const size_t wsb = bd3mg_mg_steps_ws_bytes(g, &t, 1);
  if (wsb == (size_t)-1) return BD3MG_EINVAL;
  CU(p->ws.reserve(wsb));
  rc = bd3mg_mg_steps(g, &p->r, p->K.p, p->y.p, &t, 1, (double*)p->info.p, p->ws.p, wsb, p->s);
  if (rc) return rc;
  double info[BD3MG_INFO_DOUBLES];
  if (g->dtype == BD3MG_F64) {
    CU(cudaMemcpyAsync(inc_out, p->inc.p, (size_t)h * plane * 8, cudaMemcpyDeviceToHost, p->s));
  } else {
    CU(p->stage.reserve((size_t)h * plane * 8));
    cvt_kernel_f32_to_f64<<<592, 256, 0, p->s>>>((const float*)p->inc.p, (double*)p->stage.p, (long long)h * plane);
    CU(cudaGetLastError());
    CU(cudaMemcpyAsync(inc_out, p->stage.p, (size_t)h * plane * 8, cudaMemcpyDeviceToHost, p->s));
  }
  CU(cudaMemcpyAsync(info, p->info.p, sizeof(info), cudaMemcpyDeviceToHost, p->s));
  CU(cudaStreamSynchronize(p->s));
  if (info_out) memcpy(info_out, info, sizeof(info));
  if (info[8] != 0.0)
    return fail(BD3MG_ENONFINITE, info[8] == 2.0 ? "non-finite increment" : "non-finite gradient");
  return BD3MG_OK;
}

// Session-mode sweep of the whole volume with the PCIe transfers overlapped.
// The blocks split into G depth-contiguous groups.  x arrives piece by piece
// on a copy stream (group g's support first); group g's fragment takes the
// planes it shares with group g-1 by a D2D copy from g-1's fragment before
// g-1 updates them.  Group g's sweep runs while later pieces are in flight,
// and each group's updated rows go back to the host (second copy stream)
// while the next groups compute.  Every group is a bd3mg_jacobi_sweep over
// the same anchor, so the iterate is bitwise that of one sweep over all
// blocks; the recorder terms are the sums of the groups' (every term, f
// included, is a sum over rows).
static int pipeline_enqueue(bd3mg_problem* p, double* x, const int64_t* blocks, int nblocks, int* groups_out) {
  const bd3mg_geom_t* g = &p->g;
  const int64_t nz = g->nz, plane = g->ny * g->nx, kz = g->kz;
  const bool f32 = g->dtype == BD3MG_F32;
  const size_t esz = f32 ? 4 : 8;
  static const int env_groups = [] {
    const char* e = getenv("BD3MG_PIPELINE_GROUPS");
    return e ? atoi(e) : 0;
  }();
  const int G = std::max(2, std::min(env_groups > 0 ? env_groups : kPipeGroups, std::min(nblocks, kPipeMax)));
  int first[kPipeMax + 1];
  for (int q = 0; q <= G; ++q) first[q] = (int)((long long)nblocks * q / G);
  int64_t lo[kPipeMax], hi[kPipeMax], z0[kPipeMax], need[kPipeMax];
  for (int q = 0; q < G; ++q) {
    lo[q] = blocks[2 * first[q]];
    hi[q] = blocks[2 * first[q + 1] - 1];
    z0[q] = std::max<int64_t>(0, lo[q] - kz);
    need[q] = std::min(nz - 1, hi[q] + kz);
  }
  if (!p->s_in) {
    CU(cudaStreamCreateWithFlags(&p->s_in, cudaStreamNonBlocking));
    CU(cudaStreamCreateWithFlags(&p->s_out, cudaStreamNonBlocking));
    for (auto& e : p->ev) CU(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    for (auto& e : p->ev_piece) CU(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  }
  if (p->dmem_res_z0 != 0 || p->dmem_res_n != nz) {
    CU(p->dmem_res.reserve((size_t)nz * plane * esz));
    CU(cudaMemsetAsync(p->dmem_res.p, 0, (size_t)nz * plane * esz, p->s));
    p->dmem_res_z0 = 0;
    p->dmem_res_n = nz;
  }
  for (int q = 0; q < G; ++q) {
    CU(p->frag[q].reserve((size_t)(need[q] - z0[q] + 1) * plane * esz));
    CU(p->gws[q].reserve(0));
  }
  CU(p->info.reserve((size_t)nblocks * BD3MG_INFO_DOUBLES * sizeof(double)));
  CU(p->terms.reserve((size_t)G * BD3MG_EVAL_DOUBLES * sizeof(double)));
  // fp32 problems: x crosses PCIe as float64 through a staging volume and is
  // narrowed / widened on the device next to the copies
  if (f32) CU(p->stage.reserve((size_t)nz * plane * 8));
  double* stage = (double*)p->stage.p;
  auto fr = [&](int q) { return (char*)p->frag[q].p; };  // byte pointer; element size esz
  auto rows = [&](int q, int64_t z) { return fr(q) + (size_t)(z - z0[q]) * plane * esz; };
  // (1) pieces of x, each into the first group that needs them
  CU(cudaEventRecord(p->ev[3], p->s));  // the previous call's use of the buffers is ordered on s
  CU(cudaStreamWaitEvent(p->s_in, p->ev[3], 0));
  int64_t have = -1;  // last plane shipped
  for (int q = 0; q < G; ++q) {
    if (need[q] > have) {
      const size_t n = (size_t)(need[q] - have) * plane;
      if (!f32) {
        CU(cudaMemcpyAsync(rows(q, have + 1), x + (have + 1) * plane, n * 8, cudaMemcpyHostToDevice, p->s_in));
      } else {
        CU(cudaMemcpyAsync(stage + (have + 1) * plane, x + (have + 1) * plane, n * 8, cudaMemcpyHostToDevice,
                           p->s_in));
        cvt_kernel_f64_to_f32<<<592, 256, 0, p->s_in>>>(stage + (have + 1) * plane, (float*)rows(q, have + 1),
                                                        (long long)n);
        launched();
        CU(cudaGetLastError());
      }
      have = need[q];
    }
    CU(cudaEventRecord(p->ev_piece[q], p->s_in));
  }
  auto sweep = [&](int q) -> int {
    bd3mg_sweep_t sw;
    memset(&sw, 0, sizeof(sw));
    sw.x = fr(q); sw.dmem = (char*)p->dmem_res.p + (size_t)z0[q] * plane * esz; sw.frag_z0 = z0[q]; sw.nzf = need[q] - z0[q] + 1;
    sw.blocks = blocks + 2 * first[q]; sw.nblocks = first[q + 1] - first[q];
    sw.rec_lo = lo[q]; sw.rec_hi = hi[q]; sw.snap = nullptr;
    const size_t wsb = bd3mg_jacobi_sweep_ws_bytes(g, &sw);
    if (wsb == (size_t)-1) return BD3MG_EINVAL;
    CU(p->gws[q].reserve(wsb));
    return bd3mg_jacobi_sweep(g, &p->r, p->K.p, p->y.p, &sw, (double*)p->terms.p + q * BD3MG_EVAL_DOUBLES,
                              (double*)p->info.p + (size_t)first[q] * BD3MG_INFO_DOUBLES, p->gws[q].p, wsb, p->s);
  };
  for (int q = 0; q < G; ++q) {
    CU(cudaStreamWaitEvent(p->s, p->ev_piece[q], 0));
    // planes group q+1 shares with q, before q's sweep updates them
    if (q + 1 < G) {
      const int64_t a = z0[q + 1], b = std::min(need[q], need[q + 1]);
      if (b >= a)
        CU(cudaMemcpyAsync(fr(q + 1), rows(q, a), (size_t)(b - a + 1) * plane * esz, cudaMemcpyDeviceToDevice,
                           p->s));
    }
    int rc = sweep(q);
    if (rc) return rc;
    // group q's rows back to the host while the later groups compute
    const size_t nq = (size_t)(hi[q] - lo[q] + 1) * plane;
    if (!f32) {
      CU(cudaEventRecord(p->ev[2], p->s));
      CU(cudaStreamWaitEvent(p->s_out, p->ev[2], 0));
      CU(cudaMemcpyAsync(x + lo[q] * plane, rows(q, lo[q]), nq * 8, cudaMemcpyDeviceToHost, p->s_out));
    } else {
      cvt_kernel_f32_to_f64<<<592, 256, 0, p->s>>>((const float*)rows(q, lo[q]), stage + lo[q] * plane, (long long)nq);
      launched();
      CU(cudaGetLastError());
      CU(cudaEventRecord(p->ev[2], p->s));
      CU(cudaStreamWaitEvent(p->s_out, p->ev[2], 0));
      CU(cudaMemcpyAsync(x + lo[q] * plane, stage + lo[q] * plane, nq * 8, cudaMemcpyDeviceToHost, p->s_out));
    }
  }
  // per-group records into pinned host memory; join the copy streams back into s
  CU(cudaMemcpyAsync(p->info_h, p->info.p, (size_t)nblocks * BD3MG_INFO_DOUBLES * sizeof(double),
                     cudaMemcpyDeviceToHost, p->s));
  CU(cudaMemcpyAsync(p->terms_h, p->terms.p, (size_t)G * BD3MG_EVAL_DOUBLES * sizeof(double), cudaMemcpyDeviceToHost,
                     p->s));
  CU(cudaEventRecord(p->ev[0], p->s_in));
  CU(cudaStreamWaitEvent(p->s, p->ev[0], 0));
  CU(cudaEventRecord(p->ev[1], p->s_out));
  CU(cudaStreamWaitEvent(p->s, p->ev[1], 0));
  *groups_out = G;
  return BD3MG_OK;
}

// The enqueued work of one call is captured once per (host x, blocks) key and
// replayed as one CUDA graph: the ~20 launches per group and the copies cost
// one cudaGraphLaunch (measured: the host launch cost was exposed between the
// overlapped copies).  Capture needs page-locked x (pageable copies are not
// capturable); other calls run the same work eagerly.
static int pipelined_session_sweep(bd3mg_problem* p, double* x, const int64_t* blocks, int nblocks,
                                   double* terms_out, double* info_out) {
  if (!p->info_h) {
    CU(cudaHostAlloc((void**)&p->info_h, (size_t)kMaxJobs * BD3MG_INFO_DOUBLES * sizeof(double),
                     cudaHostAllocDefault));
    CU(cudaHostAlloc((void**)&p->terms_h, (size_t)kPipeMax * BD3MG_EVAL_DOUBLES * sizeof(double),
                     cudaHostAllocDefault));
  }
  if (nblocks > kMaxJobs) return fail(BD3MG_EINVAL, "at most %d blocks per sweep", kMaxJobs);
  std::vector<int64_t> key(blocks, blocks + 2 * nblocks);
  key.push_back((int64_t)(uintptr_t)x);
  int G = 0;
  if (p->graph && key == p->graph_key) {
    CU(cudaGraphLaunch(p->graph, p->s));
    G = p->graph_groups;
  } else {
    int rc = pipeline_enqueue(p, x, blocks, nblocks, &G);
    if (rc) return rc;
    CU(cudaStreamSynchronize(p->s));
    cudaPointerAttributes attr;
    const bool pinned = cudaPointerGetAttributes(&attr, x) == cudaSuccess && attr.type == cudaMemoryTypeHost;
    if (pinned && getenv("BD3MG_NO_GRAPH") == nullptr) {  // capture for the next calls with this key
      if (p->graph) {
        cudaGraphExecDestroy(p->graph);
        p->graph = nullptr;
      }
      cudaGraph_t gr = nullptr;
      CU(cudaStreamBeginCapture(p->s, cudaStreamCaptureModeThreadLocal));
      int g2 = 0;
      rc = pipeline_enqueue(p, x, blocks, nblocks, &g2);
      cudaError_t e = cudaStreamEndCapture(p->s, &gr);
      if (rc) return rc;
      CU(e);
      e = cudaGraphInstantiate(&p->graph, gr, 0);
      cudaGraphDestroy(gr);
      CU(e);
      p->graph_key = key;
      p->graph_groups = g2;
    }
  }
  CU(cudaStreamSynchronize(p->s));
  const double* info = p->info_h;
  if (terms_out)
    for (int i = 0; i < BD3MG_EVAL_DOUBLES; ++i) {
      double t = 0.0;
      for (int q = 0; q < G; ++q) t += p->terms_h[(size_t)q * BD3MG_EVAL_DOUBLES + i];
      terms_out[i] = t;
    }
  if (info_out) memcpy(info_out, info, (size_t)nblocks * BD3MG_INFO_DOUBLES * sizeof(double));
  for (int b = 0; b < nblocks; ++b)
    if (info[(size_t)b * BD3MG_INFO_DOUBLES + 8] != 0.0)
      return fail(BD3MG_ENONFINITE, info[(size_t)b * BD3MG_INFO_DOUBLES + 8] == 2.0 ? "non-finite increment"
                                                                                   : "non-finite gradient");
  return BD3MG_OK;
}

int bd3mg_problem_jacobi_sweep_host(bd3mg_problem* p, double* x, double* dmem, int64_t frag_z0, int64_t nzf,
                                    const int64_t* blocks, int nblocks, double* terms_out, double* info_out) {
  if (!p || !x || !blocks || nblocks < 1) return fail(BD3MG_EINVAL, "null argument");
  std::lock_guard<std::mutex> lock(p->mu);
  CU(cudaSetDevice(p->device));
  const bd3mg_geom_t* g = &p->g;
  if (frag_z0 < 0 || nzf < 1 || frag_z0 + nzf > g->nz) return fail(BD3MG_EINVAL, "invalid fragment");
  {
    // pipelined path: session mode, fp64, whole volume, >= 4 depth-ordered back-to-back blocks
    bool ok = !dmem && frag_z0 == 0 && nzf == g->nz && nblocks >= 4 &&
              getenv("BD3MG_NO_PIPELINE") == nullptr && blocks[0] >= 0 && blocks[2 * nblocks - 1] < g->nz;
    for (int b = 0; ok && b < nblocks; ++b) {
      ok = blocks[2 * b] <= blocks[2 * b + 1];
      if (b > 0) ok = ok && blocks[2 * b] == blocks[2 * b - 1] + 1;
    }
    if (ok) return pipelined_session_sweep(p, x, blocks, nblocks, terms_out, info_out);
  }
  if (p->graph) {  // this path may reallocate buffers the captured pipeline refers to
    CU(cudaStreamSynchronize(p->s));
    cudaGraphExecDestroy(p->graph);
    p->graph = nullptr;
    p->graph_key.clear();
  }
  const size_t n = (size_t)nzf * g->ny * g->nx;
  const size_t esz = g->dtype == BD3MG_F64 ? 8 : 4;
  int64_t rec_lo = blocks[0], rec_hi = blocks[1];
  for (int b = 1; b < nblocks; ++b) {
    rec_lo = std::min(rec_lo, blocks[2 * b]);
    rec_hi = std::max(rec_hi, blocks[2 * b + 1]);
  }
  int rc = upload_f64(p, x, n, p->slab);
  if (!rc && dmem) rc = upload_f64(p, dmem, n, p->dmem);
  if (rc) return rc;
  DevBuf* dm = &p->dmem;
  if (!dmem) {  // session mode: memory store stays on the device between calls
    if (p->dmem_res_z0 != frag_z0 || p->dmem_res_n != nzf) {
      CU(p->dmem_res.reserve(n * esz));
      CU(cudaMemsetAsync(p->dmem_res.p, 0, n * esz, p->s));
      p->dmem_res_z0 = frag_z0;
      p->dmem_res_n = nzf;
    }
    dm = &p->dmem_res;
  }
  CU(p->info.reserve((size_t)nblocks * BD3MG_INFO_DOUBLES * sizeof(double)));
  CU(p->terms.reserve(BD3MG_EVAL_DOUBLES * sizeof(double)));
  bd3mg_sweep_t sw;
  memset(&sw, 0, sizeof(sw));
  sw.x = p->slab.p; sw.dmem = dm->p; sw.frag_z0 = frag_z0; sw.nzf = nzf;
  sw.blocks = blocks; sw.nblocks = nblocks; sw.rec_lo = rec_lo; sw.rec_hi = rec_hi; sw.snap = nullptr;
  const size_t wsb = bd3mg_jacobi_sweep_ws_bytes(g, &sw);
  if (wsb == (size_t)-1) return BD3MG_EINVAL;
  CU(p->ws.reserve(wsb));
  rc = bd3mg_jacobi_sweep(g, &p->r, p->K.p, p->y.p, &sw, (double*)p->terms.p, (double*)p->info.p, p->ws.p, wsb, p->s);
  if (rc) return rc;
  rc = download_f64(p, p->slab, n, x);
  if (!rc && dmem) rc = download_f64(p, p->dmem, n, dmem);
  if (rc) return rc;
  std::vector<double> info((size_t)nblocks * BD3MG_INFO_DOUBLES);
  CU(cudaMemcpyAsync(info.data(), p->info.p, info.size() * sizeof(double), cudaMemcpyDeviceToHost, p->s));
  if (terms_out)
    CU(cudaMemcpyAsync(terms_out, p->terms.p, BD3MG_EVAL_DOUBLES * sizeof(double), cudaMemcpyDeviceToHost, p->s));
  CU(cudaStreamSynchronize(p->s));
  if (info_out) memcpy(info_out, info.data(), info.size() * sizeof(double));
  for (int b = 0; b < nblocks; ++b)
    if (info[(size_t)b * BD3MG_INFO_DOUBLES + 8] != 0.0)
      return fail(BD3MG_ENONFINITE, info[(size_t)b * BD3MG_INFO_DOUBLES + 8] == 2.0 ? "non-finite increment"
                                                                                   : "non-finite gradient");
  return BD3MG_OK;
}

}  // extern "C"
