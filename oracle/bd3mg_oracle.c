/*
 * TEST INFRASTRUCTURE ONLY -- the CPU oracle of the BD3MG hot path.
 * Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg may
 * load this library; the product path never does.
 *
 * Plain-C restatement of the reference's native core
 * /root/reference/pkg/src/bd3mg/_core.pyx:
 *   oracle_correlate          <- depthvar_correlate         (_core.pyx:17-53)
 *   oracle_correlate_adjoint  <- depthvar_correlate_adjoint (_core.pyx:56-96)
 * Same loop order (rows, y, x, then taps a -> b -> c), same skip rules for
 * out-of-fragment / out-of-plane taps, separate multiply and add (built with
 * -ffp-contract=off, like the reference's -O3 x86-64 build without FMA).
 * Output rows are independent, so rows are spread over `threads` OpenMP
 * threads (1 = the reference's single-threaded loop).
 */
#include <stdint.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef int64_t idx_t;

static void correlate_row(const double* frag, idx_t nzf, idx_t ny, idx_t nx, const double* ker, idx_t kz,
                          idx_t ky, idx_t kx, idx_t frag_z0, idx_t zo, double* out_plane) {
  const idx_t rz = (kz - 1) / 2, ry = (ky - 1) / 2, rx = (kx - 1) / 2;
  const double* kp = ker + zo * kz * ky * kx;
  for (idx_t y = 0; y < ny; ++y) {
    for (idx_t x = 0; x < nx; ++x) {
      double acc = 0.0;
      for (idx_t a = 0; a < kz; ++a) {
        const idx_t zf = zo + a - rz - frag_z0;
        if (zf < 0 || zf >= nzf) continue;
        for (idx_t b = 0; b < ky; ++b) {
          const idx_t yy = y + b - ry;
          if (yy < 0 || yy >= ny) continue;
          for (idx_t c = 0; c < kx; ++c) {
            const idx_t xx = x + c - rx;
            if (xx < 0 || xx >= nx) continue;
            acc += kp[(a * ky + b) * kx + c] * frag[(zf * ny + yy) * nx + xx];
          }
        }
      }
      out_plane[y * nx + x] = acc;
    }
  }
}

static void correlate_adjoint_row(const double* frag, idx_t nzf, idx_t ny, idx_t nx, const double* ker,
                                  idx_t nzk, idx_t kz, idx_t ky, idx_t kx, idx_t frag_z0, idx_t zi,
                                  double* out_plane) {
  const idx_t rz = (kz - 1) / 2, ry = (ky - 1) / 2, rx = (kx - 1) / 2;
  for (idx_t y = 0; y < ny; ++y) {
    for (idx_t x = 0; x < nx; ++x) {
      double acc = 0.0;
      for (idx_t a = 0; a < kz; ++a) {
        const idx_t zo = zi + rz - a;
        if (zo < 0 || zo >= nzk) continue;
        const idx_t zf = zo - frag_z0;
        if (zf < 0 || zf >= nzf) continue;
        const double* kp = ker + zo * kz * ky * kx;
        for (idx_t b = 0; b < ky; ++b) {
          const idx_t yy = y + ry - b;
          if (yy < 0 || yy >= ny) continue;
          for (idx_t c = 0; c < kx; ++c) {
            const idx_t xx = x + rx - c;
            if (xx < 0 || xx >= nx) continue;
            acc += kp[(a * ky + b) * kx + c] * frag[(zf * ny + yy) * nx + xx];
          }
        }
      }
      out_plane[y * nx + x] = acc;
    }
  }
}

int oracle_correlate(const double* frag, idx_t nzf, idx_t ny, idx_t nx, const double* ker, idx_t nzk, idx_t kz,
                     idx_t ky, idx_t kx, idx_t frag_z0, idx_t out_lo, idx_t out_hi, double* out, int threads) {
  const idx_t nout = out_hi - out_lo + 1;
  if (nout < 0 || out_lo < 0 || (nout > 0 && out_hi >= nzk)) return 1;
#pragma omp parallel for schedule(static) num_threads(threads > 0 ? threads : 1)
  for (idx_t i = 0; i < nout; ++i)
    correlate_row(frag, nzf, ny, nx, ker, kz, ky, kx, frag_z0, out_lo + i, out + i * ny * nx);
  return 0;
}

int oracle_correlate_adjoint(const double* frag, idx_t nzf, idx_t ny, idx_t nx, const double* ker, idx_t nzk,
                             idx_t kz, idx_t ky, idx_t kx, idx_t frag_z0, idx_t out_lo, idx_t out_hi, double* out,
                             int threads) {
  const idx_t nout = out_hi - out_lo + 1;
  if (nout < 0 || out_lo < 0) return 1;
#pragma omp parallel for schedule(static) num_threads(threads > 0 ? threads : 1)
  for (idx_t i = 0; i < nout; ++i)
    correlate_adjoint_row(frag, nzf, ny, nx, ker, nzk, kz, ky, kx, frag_z0, out_lo + i, out + i * ny * nx);
  return 0;
}
