// Host-side dispatch of the depth-variant correlation kernels: picks the
// register-tiled instantiation for square ky = kx in {3,5,7,9}, else the
// generic one-voxel-per-thread kernel.
#pragma once

#include <cstdio>
#include <cstdlib>
#include <map>
#include <mutex>

#include "depthvar.cuh"

namespace bd3mg {

struct ConvGrid {
  int tiles_x, tiles_y;
};

inline bool conv_tiled_shape(int ky, int kx) {
  return ky == kx && (ky == 3 || ky == 5 || ky == 7 || ky == 9);
}

// Two output planes per CTA (conv_rz2_kernel) for single-input modes on
// tiled shapes: used where measured faster -- fp32 (FFMA has the register
// headroom); in fp64 the second coefficient set does not fit the uniform
// registers and the one-plane kernel wins.  BD3MG_RZ2=0/1 overrides.
template <typename T>
inline bool conv_rz2(int ky, int kx, int mode) {
  static const int env = [] {
    const char* e = getenv("BD3MG_RZ2");
    return e ? atoi(e) : -1;
  }();
  const bool want = env < 0 ? (sizeof(T) == 4) : env != 0;
  // the dual-input (Gram) variant exists as the fp32 packed-pair kernel only
  return want && conv_tiled_shape(ky, kx) && (mode != M_GRAM2 || (sizeof(T) == 4 && BD3MG_FFMA2));
}

// grid.z units of a job with `nout` output planes
template <typename T>
inline long long conv_zunits(int ky, int kx, int mode, long long nout) {
  return conv_rz2<T>(ky, kx, mode) ? (nout + 1) / 2 : nout;
}

template <typename T>
ConvGrid conv_grid(int ky, int kx, int mode, int ny, int nx) {
  if (!conv_tiled_shape(ky, kx))
    return {(nx + kGenericTX - 1) / kGenericTX, (ny + kGenericTY - 1) / kGenericTY};
  if (conv_rz2<T>(ky, kx, mode)) {
    constexpr int TX = Rz2Cfg<T, 3, 3, M_STORE>::TX;
    const int TY = ky <= 5 ? Rz2Cfg<T, 3, 3, M_STORE>::TY : Rz2Cfg<T, 7, 7, M_STORE>::TY;
    return {(nx + TX - 1) / TX, (ny + TY - 1) / TY};
  }
  constexpr int TX = ConvCfg<T, 3, 3, M_STORE>::TX;
  const int TY = (mode == M_GRAM2) ? ConvCfg<T, 3, 3, M_GRAM2>::TY : ConvCfg<T, 3, 3, M_STORE>::TY;
  return {(nx + TX - 1) / TX, (ny + TY - 1) / TY};
}

// Raise a kernel's dynamic-smem limit once per (kernel, device); keyed by the
// kernel's address (kernels sharing a signature must not share the entry).
inline cudaError_t ensure_smem_attr_ptr(const void* kern, size_t bytes) {
  if (bytes <= 48 * 1024) return cudaSuccess;
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, size_t> granted;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lock(mu);
  size_t& g = granted[{kern, dev}];
  if (g >= bytes) return cudaSuccess;
  e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  if (e == cudaSuccess) g = 227 * 1024;
  return e;
}
template <typename Kern>
inline cudaError_t ensure_smem_attr(Kern kern, size_t bytes) {
  return ensure_smem_attr_ptr(reinterpret_cast<const void*>(kern), bytes);
}

// TMA descriptor of a fragment (nx, ny, nz) with a (boxw, boxh, 1) box;
// out-of-bounds elements are zero-filled by the copy engine.  Returns false
// when the layout is not TMA-legal (row pitch / base not 16-byte aligned).
bool encode_tmap(CUtensorMap* map, const void* base, bool f64, long long nx, long long ny, long long nz, int boxw,
                 int boxh, int boxd = 1);

template <typename T, int K, int MODE, bool ADJ>
cudaError_t launch_tiled(ConvArgs<T>& p, int total_work, cudaStream_t s) {
  using Cfg = ConvCfg<T, K, K, MODE>;
  static const bool no_tma = getenv("BD3MG_NO_TMA") != nullptr;  // diagnostics: force cp.async staging
  for (int j = 0; j < p.njobs; ++j) {
    ConvJob<T>& jb = p.jobs[j];
    const bool f64 = sizeof(T) == 8;
    bool ok = encode_tmap(&jb.tmap0, jb.src0, f64, p.nx, p.ny, jb.src_nz, Cfg::PITCH, Cfg::BOXH);
    if (ok && Cfg::NIN == 2) ok = encode_tmap(&jb.tmap1, jb.src1, f64, p.nx, p.ny, jb.src_nz, Cfg::PITCH, Cfg::BOXH);
    jb.use_tma = (ok && !no_tma) ? 1 : 0;
    jb.epi_tma = 0;
    if constexpr (MODE == M_GRADF) {  // the iterate tile with its halo: same box as the taps
      if (!jb.use_tma || !jb.xg || !encode_tmap(&jb.tmap1, jb.xg, f64, p.nx, p.ny, jb.xg_nz, Cfg::PITCH, Cfg::BOXH))
        return cudaErrorInvalidValue;  // the fused regulariser gradient needs TMA staging
      jb.epi_tma = 1;
    }
    if constexpr ((MODE == M_RESID || MODE == M_GRAD || MODE == M_GRAMC) && Cfg::NIN == 1 && sizeof(T) == 8) {
      static const bool no_epi = getenv("BD3MG_NO_EPI_TMA") != nullptr;
      if (jb.use_tma && jb.sub && !no_epi)
        jb.epi_tma = encode_tmap(&jb.tmap1, jb.sub, f64, p.nx, p.ny, jb.nout, Cfg::TX, Cfg::TY) ? 1 : 0;
    }
    if (getenv("BD3MG_DEBUG_TMA")) fprintf(stderr, "conv K=%d mode=%d job=%d tma=%d box=%dx%d\n", K, MODE, j, (int)jb.use_tma, Cfg::PITCH, Cfg::BOXH);
  }
  const size_t sm = Cfg::smem_bytes(p.kz);
  auto kern = conv_tiled_kernel<T, K, K, MODE, ADJ>;
  cudaError_t e = ensure_smem_attr(kern, sm);
  if (e != cudaSuccess) return e;
  dim3 grid(p.tiles_x, p.tiles_y, total_work);
  kern<<<grid, Cfg::NT, sm, s>>>(p);
  return cudaGetLastError();
}

template <typename T, int K, int MODE, bool ADJ>
cudaError_t launch_rz2(ConvArgs<T>& p, int total_work, cudaStream_t s) {
  using Cfg = Rz2Cfg<T, K, K, MODE>;
  for (int j = 0; j < p.njobs; ++j) {
    ConvJob<T>& jb = p.jobs[j];
    jb.use_tma = encode_tmap(&jb.tmap0, jb.src0, sizeof(T) == 8, p.nx, p.ny, jb.src_nz, Cfg::PITCH, Cfg::BOXH) &&
                 getenv("BD3MG_NO_TMA") == nullptr;
  }
  for (int j = 0; j < p.njobs; ++j) {  // epilogue operand tiles of both output planes (RESID / GRAD / GRAMC)
    ConvJob<T>& jb = p.jobs[j];
    jb.epi_tma = 0;
    if constexpr (Cfg::EPI_T) {
      static const bool no_epi = getenv("BD3MG_NO_EPI_TMA") != nullptr;
      if (jb.use_tma && jb.sub && !no_epi)
        jb.epi_tma = encode_tmap(&jb.tmap1, jb.sub, sizeof(T) == 8, p.nx, p.ny, jb.nout, Cfg::TX, Cfg::TY, 2) ? 1 : 0;
    }
  }
  const size_t sm = Cfg::smem_bytes(p.kz);
  if constexpr (Cfg::NIN == 2) {
    for (int j = 0; j < p.njobs; ++j) {
      ConvJob<T>& jb = p.jobs[j];
      jb.use_tma = jb.use_tma &&
                   encode_tmap(&jb.tmap1, jb.src1, sizeof(T) == 8, p.nx, p.ny, jb.src_nz, Cfg::PITCH, Cfg::BOXH);
    }
  }
  auto kern = conv_rz2_kernel<T, K, K, MODE, ADJ>;
  cudaError_t e = ensure_smem_attr(kern, sm);
  if (e != cudaSuccess) return e;
  dim3 grid(p.tiles_x, p.tiles_y, total_work);
  kern<<<grid, Cfg::NT, sm, s>>>(p);
  return cudaGetLastError();
}

template <typename T, int MODE, bool ADJ>
cudaError_t launch_generic(ConvArgs<T>& p, int total_work, cudaStream_t s) {
  size_t coef = ((size_t)p.kz * p.ky * p.kx * sizeof(T) + 15) & ~size_t(15);
  const size_t sm = coef + 8 * (kGenericNT / 32) * sizeof(double);
  auto kern = conv_generic_kernel<T, MODE, ADJ>;
  cudaError_t e = ensure_smem_attr(kern, sm);
  if (e != cudaSuccess) return e;
  dim3 grid(p.tiles_x, p.tiles_y, total_work);
  kern<<<grid, kGenericNT, sm, s>>>(p);
  return cudaGetLastError();
}

template <typename T, int MODE, bool ADJ>
cudaError_t launch_mode(ConvArgs<T>& p, int total_work, cudaStream_t s) {
  if (p.ky == p.kx) {
    if constexpr (MODE == M_GRAM2) {
      if constexpr (sizeof(T) == 4 && BD3MG_FFMA2) {
        if (conv_rz2<T>(p.ky, p.kx, MODE)) {
          switch (p.ky) {
            case 3: return launch_rz2<T, 3, MODE, ADJ>(p, total_work, s);
            case 5: return launch_rz2<T, 5, MODE, ADJ>(p, total_work, s);
            case 7: return launch_rz2<T, 7, MODE, ADJ>(p, total_work, s);
            case 9: return launch_rz2<T, 9, MODE, ADJ>(p, total_work, s);
            default: break;
          }
        }
      }
      switch (p.ky) {
        case 3: return launch_tiled<T, 3, MODE, ADJ>(p, total_work, s);
        case 5: return launch_tiled<T, 5, MODE, ADJ>(p, total_work, s);
        case 7: return launch_tiled<T, 7, MODE, ADJ>(p, total_work, s);
        case 9: return launch_tiled<T, 9, MODE, ADJ>(p, total_work, s);
        default: break;
      }
    } else if (conv_rz2<T>(p.ky, p.kx, MODE)) {
      switch (p.ky) {
        case 3: return launch_rz2<T, 3, MODE, ADJ>(p, total_work, s);
        case 5: return launch_rz2<T, 5, MODE, ADJ>(p, total_work, s);
        case 7: return launch_rz2<T, 7, MODE, ADJ>(p, total_work, s);
        case 9: return launch_rz2<T, 9, MODE, ADJ>(p, total_work, s);
        default: break;
      }
    } else {
      switch (p.ky) {
        case 3: return launch_tiled<T, 3, MODE, ADJ>(p, total_work, s);
        case 5: return launch_tiled<T, 5, MODE, ADJ>(p, total_work, s);
        case 7: return launch_tiled<T, 7, MODE, ADJ>(p, total_work, s);
        case 9: return launch_tiled<T, 9, MODE, ADJ>(p, total_work, s);
        default: break;
      }
    }
  }
  return launch_generic<T, MODE, ADJ>(p, total_work, s);
}

// Fill tiles_{x,y} and launch `mode` over `total_work` output planes.
template <typename T>
cudaError_t conv_launch(int mode, bool adj, ConvArgs<T>& p, int total_work, cudaStream_t s);

}  // namespace bd3mg
