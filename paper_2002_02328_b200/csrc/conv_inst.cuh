// Explicit instantiation body of conv_launch<T>; included once per dtype TU
// so the large unrolled kernels compile in parallel.
#pragma once

#include "conv_dispatch.cuh"

namespace bd3mg {

template <typename T>
cudaError_t conv_launch(int mode, bool adj, ConvArgs<T>& p, int total_work, cudaStream_t s) {
  // grid.z units: planes, or plane pairs for the two-plane kernel; the
  // callers' work_begin / total_work are recomputed here
  (void)total_work;
  long long wb = 0;
  for (int j = 0; j < p.njobs; ++j) {
    p.jobs[j].work_begin = (int)wb;
    wb += conv_zunits<T>(p.ky, p.kx, mode, p.jobs[j].nout);
  }
  total_work = (int)wb;
  if (total_work <= 0) return cudaSuccess;
  const ConvGrid g = conv_grid<T>(p.ky, p.kx, mode, p.ny, p.nx);
  p.tiles_x = g.tiles_x;
  p.tiles_y = g.tiles_y;
  // BD3MG_RASTER_GROUP=G walks z inside groups of G tiles (cta_pos).  At C5
  // it cuts the correlations' DRAM reads ~5-9x (21 -> 4.4 GB for RESID: the
  // input planes stay L2-resident) but runs 0.8-1.8% slower (measured with G
  // = 32 / 64 / 128 / 256): the kernels are FMA-bound and the plain order's
  // re-reads are free, so the plain order is the default
  static const int group_env = [] {
    const char* e = getenv("BD3MG_RASTER_GROUP");
    return e ? atoi(e) : 0;
  }();
  p.raster_group = group_env;
  if (!adj) {
    switch (mode) {
      case M_STORE: return launch_mode<T, M_STORE, false>(p, total_work, s);
      case M_RESID: return launch_mode<T, M_RESID, false>(p, total_work, s);
      case M_GRAM1: return launch_mode<T, M_GRAM1, false>(p, total_work, s);
      case M_GRAM2: return launch_mode<T, M_GRAM2, false>(p, total_work, s);
      case M_GRAMC: return launch_mode<T, M_GRAMC, false>(p, total_work, s);
      default: return cudaErrorInvalidValue;
    }
  }
  switch (mode) {
    case M_STORE: return launch_mode<T, M_STORE, true>(p, total_work, s);
    case M_GRAD: return launch_mode<T, M_GRAD, true>(p, total_work, s);
    case M_GRADF:  // fp64 tiled shapes only (the caller checks conv_gradf_ok)
      if constexpr (sizeof(T) == 8) {
        switch (p.ky == p.kx ? p.ky : 0) {
          case 3: return launch_tiled<T, 3, M_GRADF, true>(p, total_work, s);
          case 5: return launch_tiled<T, 5, M_GRADF, true>(p, total_work, s);
          case 7: return launch_tiled<T, 7, M_GRADF, true>(p, total_work, s);
          case 9: return launch_tiled<T, 9, M_GRADF, true>(p, total_work, s);
          default: return cudaErrorInvalidValue;
        }
      }
      return cudaErrorInvalidValue;
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace bd3mg
