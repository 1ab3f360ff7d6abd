// Device-resident Krylov loops of the ablation path:
// conjugate gradients on the block majorant (reference directions.py:117-149,
// driven by mm_direction :152-168) and the power iteration of
// rho(H^T H) (objective.py:345-370).
//
// Every scalar of the recursion (|b|, r.r, p.Ap, alpha, beta, the best
// iterate's residual, the stop state) lives in a small device state vector;
// each iteration is a fixed sequence of launches whose kernels read the
// state and exit at once when the solve has stopped, so the host enqueues
// iterations without waiting on any of them (it only watches a host-mapped
// copy of the iteration counter to stay at most a few iterations ahead).
// Dot products use fixed grids and fixed reduction trees: deterministic.
#pragma once

#include "solver.cuh"

namespace bd3mg {

constexpr int kKryCtas = 592;  // 4 x 148 SMs: fixed partial-sum grid of the dot products

// state layout (doubles)
enum CgState : int {
  CG_BNORM = 0,    // |b|
  CG_RS = 1,       // r.r of the current residual
  CG_BEST = 2,     // residual norm of the best iterate so far
  CG_ALPHA = 3,
  CG_BETA = 4,
  CG_STATUS = 5,   // 0 running, 1 converged (x is the result), 2 stopped (best is the result)
  CG_IT = 6,       // iterations performed
  CG_RELRES = 7,   // relative residual of the returned iterate
  CG_COPYBEST = 8, // this iteration's x is the new best iterate
  CG_NV = 16
};

template <typename T>
struct CgVecs {
  T* x;
  T* r;
  T* p;
  T* ap;
  T* best;
  const T* b;
  long long n;
};

// a.b partials over a fixed grid (one row per CTA)
template <typename T>
BD3MG_D double dot_partial(const T* __restrict__ a, const T* __restrict__ b, long long n, double* s) {
  double acc = 0.0;
  for (long long i = (long long)blockIdx.x * kEwNT + threadIdx.x; i < n; i += (long long)gridDim.x * kEwNT)
    acc += (double)a[i] * (double)b[i];
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
  if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = acc;
  __syncthreads();
  double t = 0.0;
  if (threadIdx.x == 0) {
    t = s[0];
    for (int w = 1; w < kEwNT / 32; ++w) t += s[w];
  }
  return t;
}

// one CTA: sum of `rows` partials (fixed stride classes + warp butterfly)
BD3MG_D double sum_partials(const double* __restrict__ parts, int rows, double* s) {
  double acc = 0.0;
  for (int i = threadIdx.x; i < rows; i += kEwNT) acc += parts[i];
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
  if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = acc;
  __syncthreads();
  double t = s[0];
  for (int w = 1; w < kEwNT / 32; ++w) t += s[w];
  return t;
}

// x = 0, r = p = b, partials of b.b
template <typename T>
__global__ void __launch_bounds__(kEwNT) cg_init_kernel(CgVecs<T> v, double* __restrict__ parts) {
  __shared__ double s[kEwNT / 32];
  for (long long i = (long long)blockIdx.x * kEwNT + threadIdx.x; i < v.n; i += (long long)gridDim.x * kEwNT) {
    const T bi = v.b[i];
    v.x[i] = T(0);
    v.r[i] = bi;
    v.p[i] = bi;
    v.best[i] = T(0);
  }
  const double t = dot_partial(v.b, v.b, v.n, s);
  if (threadIdx.x == 0) parts[blockIdx.x] = t;
}

__global__ void __launch_bounds__(kEwNT) cg_init_state_kernel(const double* __restrict__ parts, double* st,
                                                               volatile double* host_it) {
  __shared__ double s[kEwNT / 32];
  const double bb = sum_partials(parts, kKryCtas, s);
  if (threadIdx.x == 0) {
    for (int k = 0; k < CG_NV; ++k) st[k] = 0.0;
    const double bn = sqrt(bb);
    st[CG_BNORM] = bn;
    st[CG_RS] = bb;
    st[CG_BEST] = bn;
    if (bn == 0.0) st[CG_STATUS] = 1.0;  // x = 0, converged, 0 iterations, relres 0
    if (host_it) { host_it[0] = 0.0; host_it[1] = st[CG_STATUS]; }
  }
}

// p.Ap partials (Ap from the majorant apply of this iteration)
template <typename T>
__global__ void __launch_bounds__(kEwNT) cg_pap_kernel(CgVecs<T> v, const double* __restrict__ st,
                                                        double* __restrict__ parts) {
  __shared__ double s[kEwNT / 32];
  if (st[CG_STATUS] != 0.0) return;
  const double t = dot_partial(v.p, v.ap, v.n, s);
  if (threadIdx.x == 0) parts[blockIdx.x] = t;
}

// alpha = rs / p.Ap, or stop at the best iterate on loss of definiteness
__global__ void __launch_bounds__(kEwNT) cg_alpha_kernel(const double* __restrict__ parts, double* st) {
  __shared__ double s[kEwNT / 32];
  if (st[CG_STATUS] != 0.0) return;
  const double pap = sum_partials(parts, kKryCtas, s);
  if (threadIdx.x == 0) {
    st[CG_IT] += 1.0;
    if (!(pap > 0.0)) {  // directions.py:133-134 (p_ap <= 0: break)
      st[CG_STATUS] = 2.0;
      st[CG_RELRES] = st[CG_BEST] / st[CG_BNORM];
    } else {
      st[CG_ALPHA] = st[CG_RS] / pap;
    }
  }
}

// x += alpha p; r -= alpha Ap; partials of r.r
template <typename T>
__global__ void __launch_bounds__(kEwNT) cg_xr_kernel(CgVecs<T> v, const double* __restrict__ st,
                                                       double* __restrict__ parts) {
  __shared__ double s[kEwNT / 32];
  if (st[CG_STATUS] != 0.0) return;
  const T alpha = (T)st[CG_ALPHA];
  for (long long i = (long long)blockIdx.x * kEwNT + threadIdx.x; i < v.n; i += (long long)gridDim.x * kEwNT) {
    v.x[i] = add_rn(v.x[i], mul_rn(alpha, v.p[i]));
    v.r[i] = sub_rn(v.r[i], mul_rn(alpha, v.ap[i]));
  }
  const double t = dot_partial(v.r, v.r, v.n, s);
  if (threadIdx.x == 0) parts[blockIdx.x] = t;
}

// residual bookkeeping: best iterate, convergence, budget, beta
__global__ void __launch_bounds__(kEwNT) cg_check_kernel(const double* __restrict__ parts, double* st, double tol,
                                                          int maxit, volatile double* host_it) {
  __shared__ double s[kEwNT / 32];
  if (st[CG_STATUS] != 0.0) return;
  const double rs_new = sum_partials(parts, kKryCtas, s);
  if (threadIdx.x == 0) {
    const double res = sqrt(rs_new);
    st[CG_COPYBEST] = 0.0;
    if (res < st[CG_BEST]) {
      st[CG_BEST] = res;
      st[CG_COPYBEST] = 1.0;
    }
    if (res <= tol * st[CG_BNORM]) {  // directions.py:144-145
      st[CG_STATUS] = 1.0;
      st[CG_RELRES] = res / st[CG_BNORM];
      st[CG_COPYBEST] = 0.0;
    } else if (st[CG_IT] >= (double)maxit) {  // budget: the best iterate
      st[CG_STATUS] = 2.0;
      st[CG_RELRES] = st[CG_BEST] / st[CG_BNORM];
    } else {
      st[CG_BETA] = rs_new / st[CG_RS];
      st[CG_RS] = rs_new;
    }
    if (host_it) { host_it[0] = st[CG_IT]; host_it[1] = st[CG_STATUS]; }
  }
}

// best = x where this iteration improved it; p = r + beta p while running
template <typename T>
__global__ void __launch_bounds__(kEwNT) cg_p_kernel(CgVecs<T> v, const double* __restrict__ st) {
  const bool copy = st[CG_COPYBEST] != 0.0, run = st[CG_STATUS] == 0.0;
  if (!copy && !run) return;
  const T beta = (T)st[CG_BETA];
  for (long long i = (long long)blockIdx.x * kEwNT + threadIdx.x; i < v.n; i += (long long)gridDim.x * kEwNT) {
    if (copy) v.best[i] = v.x[i];
    if (run) v.p[i] = add_rn(v.r[i], mul_rn(beta, v.p[i]));
  }
}

// result: x if converged, else the best iterate
template <typename T>
__global__ void __launch_bounds__(kEwNT) cg_result_kernel(CgVecs<T> v, const double* __restrict__ st, T* out) {
  const bool conv = st[CG_STATUS] == 1.0;
  for (long long i = (long long)blockIdx.x * kEwNT + threadIdx.x; i < v.n; i += (long long)gridDim.x * kEwNT)
    out[i] = conv ? v.x[i] : v.best[i];
}

// ---------------------------------------------------------------------------
// power iteration: |w| partials, then v = w / |w| (objective.py:359-366)
template <typename T>
__global__ void __launch_bounds__(kEwNT) pw_norm_kernel(const T* __restrict__ w, long long n,
                                                         const double* __restrict__ st, double* __restrict__ parts) {
  __shared__ double s[kEwNT / 32];
  if (st[0] != 0.0) return;
  const double t = dot_partial(w, w, n, s);
  if (threadIdx.x == 0) parts[blockIdx.x] = t;
}

__global__ void __launch_bounds__(kEwNT) pw_finish_kernel(const double* __restrict__ parts, double* st,
                                                           double* __restrict__ norms, int it) {
  __shared__ double s[kEwNT / 32];
  if (st[0] != 0.0) return;
  const double nrm = sqrt(sum_partials(parts, kKryCtas, s));
  if (threadIdx.x == 0) {
    norms[it] = nrm;
    st[1] = nrm;
    if (nrm == 0.0) st[0] = 1.0;  // H annihilated the iterate: the host restarts from the RNG
  }
}

template <typename T>
__global__ void __launch_bounds__(kEwNT) pw_scale_kernel(const T* __restrict__ w, T* __restrict__ v, long long n,
                                                          const double* __restrict__ st) {
  if (st[0] != 0.0) return;
  const T nrm = (T)st[1];
  for (long long i = (long long)blockIdx.x * kEwNT + threadIdx.x; i < n; i += (long long)gridDim.x * kEwNT)
    v[i] = w[i] / nrm;
}

}  // namespace bd3mg
