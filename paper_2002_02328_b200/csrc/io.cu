// BD3MGVOL / BD3MGPSF payloads streamed between files and device memory.
//
// The reference containers (volume.py:104-145, blur.py:201-236) are a small
// little-endian header followed by a float64 payload.  The header is parsed
// by the Python host (paper_2002_02328_b200/volume.py, blur.py) so that its
// error messages match the reference word for word; these entry points move
// the payload, which is what scales (2.1 GB for a C5 field):
//
//   file --read()--> pinned chunk (x2) --H2D--> device [--cvt--> fp32]
//
// Two pinned chunks alternate, so the read of chunk i+1 overlaps the copy of
// chunk i.  The finiteness check of read_volume (volume.py:142-143) and of
// check_volume on write (volume.py:87-94) runs on the device, on the float64
// values, before any narrowing to fp32.
#include <cuda_runtime.h>
#include <fcntl.h>
#include <stdint.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <cerrno>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>

#include "../../include/bd3mg_b200.h"
#include "errors.h"

namespace bd3mg {
namespace {

constexpr size_t kChunkBytes = size_t(16) << 20;  // 16 MiB per pinned chunk
constexpr int kCvtBlocks = 592, kCvtThreads = 256;

// Non-finite flag: integer OR, so the result does not depend on ordering.
__global__ void finite_f64_kernel(const double* __restrict__ a, long long n, int* bad) {
  int local = 0;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    local |= !isfinite(a[i]);
  if (__syncthreads_or(local) && threadIdx.x == 0) atomicOr(bad, 1);
}
__global__ void finite_f32_kernel(const float* __restrict__ a, long long n, int* bad) {
  int local = 0;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    local |= !isfinite(a[i]);
  if (__syncthreads_or(local) && threadIdx.x == 0) atomicOr(bad, 1);
}
// f64 chunk -> f32 field, checking the float64 values
__global__ void narrow_check_kernel(const double* __restrict__ a, float* __restrict__ b, long long n, int* bad) {
  int local = 0;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const double v = a[i];
    local |= !isfinite(v);
    b[i] = (float)v;
  }
  if (__syncthreads_or(local) && threadIdx.x == 0) atomicOr(bad, 1);
}
__global__ void widen_kernel(const float* __restrict__ a, double* __restrict__ b, long long n) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    b[i] = (double)a[i];
}

int errf(int code, const char* fmt, ...) __attribute__((format(printf, 2, 3)));
int errf(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  return set_error(code, buf);
}
int cuda_err(cudaError_t e) { return errf(BD3MG_ECUDA, "CUDA: %s", cudaGetErrorString(e)); }

// Staging resources of one call (pinned chunks, events, device scratch).
struct Stage {
  void* host[2] = {nullptr, nullptr};
  cudaEvent_t ev[2] = {nullptr, nullptr};
  double* dev = nullptr;  // f64 chunk for the fp32 paths
  int* flag = nullptr;
  int* flag_host = nullptr;
  cudaStream_t stream = nullptr;
  bool live = false;
  ~Stage() {
    if (live) cudaStreamSynchronize(stream);  // no copy may still target the chunks
    for (int i = 0; i < 2; ++i) {
      if (host[i]) cudaFreeHost(host[i]);
      if (ev[i]) cudaEventDestroy(ev[i]);
    }
    if (dev) cudaFree(dev);
    if (flag) cudaFree(flag);
    if (flag_host) cudaFreeHost(flag_host);
  }
  cudaError_t init(bool need_dev, cudaStream_t s) {
    stream = s;
    live = true;
    cudaError_t e = cudaSuccess;
    for (int i = 0; i < 2 && e == cudaSuccess; ++i) {
      e = cudaHostAlloc(&host[i], kChunkBytes, cudaHostAllocDefault);
      if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming);
    }
    if (e == cudaSuccess && need_dev) e = cudaMalloc(&dev, kChunkBytes);
    if (e == cudaSuccess) e = cudaMalloc(&flag, sizeof(int));
    if (e == cudaSuccess) e = cudaHostAlloc(&flag_host, sizeof(int), cudaHostAllocDefault);
    if (e == cudaSuccess) e = cudaMemsetAsync(flag, 0, sizeof(int), s);
    return e;
  }
};

struct Fd {
  int fd = -1;
  ~Fd() {
    if (fd >= 0) close(fd);
  }
};

// read exactly n bytes at offset off (pread loop); returns bytes read
long long read_at(int fd, void* buf, size_t n, long long off) {
  size_t got = 0;
  while (got < n) {
    const ssize_t r = pread(fd, (char*)buf + got, n - got, (off_t)(off + (long long)got));
    if (r < 0) {
      if (errno == EINTR) continue;
      return -1;
    }
    if (r == 0) break;
    got += (size_t)r;
  }
  return (long long)got;
}

bool write_all(int fd, const void* buf, size_t n) {
  size_t put = 0;
  while (put < n) {
    const ssize_t r = write(fd, (const char*)buf + put, n - put);
    if (r < 0) {
      if (errno == EINTR) continue;
      return false;
    }
    put += (size_t)r;
  }
  return true;
}

}  // namespace
}  // namespace bd3mg

using namespace bd3mg;

extern "C" {

int bd3mg_payload_read_device(const char* path, int64_t offset, int64_t n, void* dev_out, int32_t dtype,
                              void* stream) {
  if (!path || !dev_out || n < 0 || offset < 0 || (dtype != BD3MG_F64 && dtype != BD3MG_F32))
    return errf(BD3MG_EINVAL, "payload_read: invalid argument");
  cudaStream_t s = (cudaStream_t)stream;
  Fd f;
  f.fd = open(path, O_RDONLY | O_CLOEXEC);
  if (f.fd < 0) return errf(BD3MG_EIO, "cannot open %s: %s", path, strerror(errno));
  struct stat st;
  if (fstat(f.fd, &st) != 0) return errf(BD3MG_EIO, "stat %s: %s", path, strerror(errno));
  const long long bytes = n * 8;
  if ((long long)st.st_size < offset + bytes)
    return errf(BD3MG_EFORMAT, "truncated payload: expected %lld bytes, got %lld", bytes,
                std::max<long long>(0, (long long)st.st_size - offset));
  if (n == 0) return BD3MG_OK;
  Stage sg;
  cudaError_t e = sg.init(dtype == BD3MG_F32, s);
  if (e != cudaSuccess) return cuda_err(e);
  const long long per = (long long)(kChunkBytes / 8);
  long long done = 0;
  int i = 0;
  int launches = 0;
  while (done < n) {
    const long long m = std::min(per, n - done);
    const int b = i & 1;
    if (i >= 2 && (e = cudaEventSynchronize(sg.ev[b])) != cudaSuccess) return cuda_err(e);
    if (read_at(f.fd, sg.host[b], (size_t)m * 8, offset + done * 8) != m * 8)
      return errf(BD3MG_EIO, "short read of %s", path);
    if (dtype == BD3MG_F64) {
      double* dst = (double*)dev_out + done;
      e = cudaMemcpyAsync(dst, sg.host[b], (size_t)m * 8, cudaMemcpyHostToDevice, s);
      if (e == cudaSuccess) e = cudaEventRecord(sg.ev[b], s);
      if (e == cudaSuccess) {
        finite_f64_kernel<<<kCvtBlocks, kCvtThreads, 0, s>>>(dst, m, sg.flag);
        e = cudaGetLastError();
      }
    } else {
      e = cudaMemcpyAsync(sg.dev, sg.host[b], (size_t)m * 8, cudaMemcpyHostToDevice, s);
      if (e == cudaSuccess) e = cudaEventRecord(sg.ev[b], s);
      if (e == cudaSuccess) {
        narrow_check_kernel<<<kCvtBlocks, kCvtThreads, 0, s>>>(sg.dev, (float*)dev_out + done, m, sg.flag);
        e = cudaGetLastError();
      }
    }
    if (e != cudaSuccess) return cuda_err(e);
    ++launches;
    done += m;
    ++i;
  }
  count_launches(launches);
  e = cudaMemcpyAsync(sg.flag_host, sg.flag, sizeof(int), cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return cuda_err(e);
  if (*sg.flag_host) return set_error(BD3MG_EFORMAT, "non-finite payload");
  return BD3MG_OK;
}

int bd3mg_field_nonfinite(const void* dev, int64_t n, int32_t dtype, int32_t* bad_out, void* stream) {
  if ((!dev && n > 0) || n < 0 || !bad_out || (dtype != BD3MG_F64 && dtype != BD3MG_F32))
    return errf(BD3MG_EINVAL, "field_nonfinite: invalid argument");
  cudaStream_t s = (cudaStream_t)stream;
  int* flag = nullptr;
  int host = 0;
  cudaError_t e = cudaMallocAsync((void**)&flag, sizeof(int), s);
  if (e == cudaSuccess) e = cudaMemsetAsync(flag, 0, sizeof(int), s);
  if (e == cudaSuccess && n > 0) {
    if (dtype == BD3MG_F64)
      finite_f64_kernel<<<kCvtBlocks, kCvtThreads, 0, s>>>((const double*)dev, n, flag);
    else
      finite_f32_kernel<<<kCvtBlocks, kCvtThreads, 0, s>>>((const float*)dev, n, flag);
    e = cudaGetLastError();
    count_launches(1);
  }
  if (e == cudaSuccess) e = cudaMemcpyAsync(&host, flag, sizeof(int), cudaMemcpyDeviceToHost, s);
  if (flag) cudaFreeAsync(flag, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return cuda_err(e);
  *bad_out = host;
  return BD3MG_OK;
}

int bd3mg_payload_write_device(const char* path, const void* dev_in, int64_t n, int32_t dtype, void* stream) {
  if (!path || (!dev_in && n > 0) || n < 0 || (dtype != BD3MG_F64 && dtype != BD3MG_F32))
    return errf(BD3MG_EINVAL, "payload_write: invalid argument");
  cudaStream_t s = (cudaStream_t)stream;
  Fd f;
  f.fd = open(path, O_WRONLY | O_APPEND | O_CLOEXEC);
  if (f.fd < 0) return errf(BD3MG_EIO, "cannot open %s: %s", path, strerror(errno));
  if (n == 0) return BD3MG_OK;
  Stage sg;
  cudaError_t e = sg.init(dtype == BD3MG_F32, s);
  if (e != cudaSuccess) return cuda_err(e);
  const long long per = (long long)(kChunkBytes / 8);
  const long long nchunks = (n + per - 1) / per;
  int launches = 0;
  // chunk i is staged into host[i & 1] on the stream; the host writes chunk
  // i-1 to the file while chunk i is in flight
  auto stage = [&](long long i) -> cudaError_t {
    const long long at = i * per, m = std::min(per, n - at);
    const int b = (int)(i & 1);
    const void* src = (const double*)dev_in + at;
    if (dtype == BD3MG_F32) {
      widen_kernel<<<kCvtBlocks, kCvtThreads, 0, s>>>((const float*)dev_in + at, sg.dev, m);
      ++launches;
      src = sg.dev;
    }
    cudaError_t r = cudaMemcpyAsync(sg.host[b], src, (size_t)m * 8, cudaMemcpyDeviceToHost, s);
    return r == cudaSuccess ? cudaEventRecord(sg.ev[b], s) : r;
  };
  if ((e = stage(0)) != cudaSuccess) return cuda_err(e);
  for (long long i = 0; i < nchunks; ++i) {
    const int b = (int)(i & 1);
    if ((e = cudaEventSynchronize(sg.ev[b])) != cudaSuccess) return cuda_err(e);
    if (i + 1 < nchunks && (e = stage(i + 1)) != cudaSuccess) return cuda_err(e);
    const long long m = std::min(per, n - i * per);
    if (!write_all(f.fd, sg.host[b], (size_t)m * 8)) return errf(BD3MG_EIO, "write to %s failed: %s", path, strerror(errno));
  }
  count_launches(launches);
  return BD3MG_OK;
}

}  // extern "C"
