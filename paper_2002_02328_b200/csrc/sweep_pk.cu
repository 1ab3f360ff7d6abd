// Instantiations and launcher of the persistent block-Jacobi sweep
// (sweep_pk.cuh); the plan (tensor maps, counters, item order) is built by
// jacobi_sweep_impl in capi.cu.
#include <map>
#include <mutex>

#include "conv_dispatch.cuh"
#include "sweep_pk.cuh"

namespace bd3mg {

template <typename T, int K>
static cudaError_t pk_launch_k(const PkArgs<T>& a, cudaStream_t s, int* slots) {
  auto kern = sweep_pk_kernel<T, K>;
  const size_t sm = PkCfg<T, K>::smem_bytes(a.cg.kz);
  cudaError_t e = ensure_smem_attr(kern, sm);
  if (e != cudaSuccess) return e;
  static std::mutex mu;
  static std::map<std::pair<int, size_t>, int> grid_of;  // (device, smem) -> resident CTAs
  int dev = 0;
  e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  int grid = 0;
  {
    std::lock_guard<std::mutex> lock(mu);
    auto it = grid_of.find({dev, sm});
    if (it == grid_of.end()) {
      int occ = 0, sms = 0;
      e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, 128, sm);
      if (e == cudaSuccess) e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      if (e != cudaSuccess) return e;
      if (occ < 1) return cudaErrorInvalidConfiguration;
      it = grid_of.emplace(std::make_pair(dev, sm), occ * sms).first;
    }
    grid = it->second;
  }
  if (slots) *slots = grid;
  if (!a.total) return cudaSuccess;
  kern<<<grid, 128, sm, s>>>(a);
  return cudaGetLastError();
}

cudaError_t pk_launch(const PkArgs<double>& a, int K, cudaStream_t s, int* slots) {
  switch (K) {
    case 3: return pk_launch_k<double, 3>(a, s, slots);
    case 5: return pk_launch_k<double, 5>(a, s, slots);
    case 7: return pk_launch_k<double, 7>(a, s, slots);
    case 9: return pk_launch_k<double, 9>(a, s, slots);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace bd3mg
