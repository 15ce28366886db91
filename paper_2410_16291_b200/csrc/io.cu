// satsweep-b200: file front door.
//
// Moves raster payloads between files and device memory without a numpy
// round trip: the reference reads a whole file into a Python bytes object and
// converts it (pkg/src/satsweep/imgio.py:72-103 read_pgm, :160-174 read_raw);
// here the payload streams through two pinned staging chunks -- several
// threads pread chunk k+1 while chunk k is in flight over PCIe -- straight
// into the destination tensor.  Big-endian 16-bit PGM samples are swapped on
// the device after the copy (the reference's astype(">u2" -> native)).
// Header parsing and the reference's error messages stay in the Python facade
// (imgio.py), which calls these entry points with the payload offset and size.
#include <fcntl.h>
#include <sys/stat.h>
#include <unistd.h>

#include <cerrno>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "ssb_common.cuh"
#include "../../include/satsweep_b200.h"

namespace ssb {
int io_fail(int code, const char* fmt, ...);  // capi.cu (thread-local last error)
}

namespace {
using namespace ssb;

constexpr int64_t kChunk = 16ll << 20;  // staging chunk (measured: 16 MB x 8 readers best)
constexpr int kMaxReaders = 16;

int64_t chunk_bytes() {  // tuning: SSB_IO_CHUNK_MB
  static const int64_t c = [] {
    const char* e = getenv("SSB_IO_CHUNK_MB");
    return e && atoi(e) > 0 ? (int64_t)atoi(e) << 20 : kChunk;
  }();
  return c;
}
int readers() {  // tuning: SSB_IO_READERS (parallel preads per chunk)
  static const int r = [] {
    const char* e = getenv("SSB_IO_READERS");
    const int v = e ? atoi(e) : 8;
    return v < 1 ? 1 : v > kMaxReaders ? kMaxReaders : v;
  }();
  return r;
}

// in-place byte swap of 16-bit samples: 8 samples per thread via 128-bit words
__global__ void swap16_kernel(uint16_t* __restrict__ p, int64_t n) {
  const int64_t n8 = n / 8;
  uint4* q = reinterpret_cast<uint4*>(p);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n8; i += (int64_t)gridDim.x * blockDim.x) {
    uint4 v = q[i];
    v.x = __byte_perm(v.x, 0, 0x2301);
    v.y = __byte_perm(v.y, 0, 0x2301);
    v.z = __byte_perm(v.z, 0, 0x2301);
    v.w = __byte_perm(v.w, 0, 0x2301);
    q[i] = v;
  }
  const int64_t t = n8 * 8 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (blockIdx.x == 0 && t < n) p[t] = (uint16_t)((p[t] >> 8) | (p[t] << 8));
}

// out-of-place variant for the write path (source stays untouched)
__global__ void swap16_copy_kernel(const uint16_t* __restrict__ s, uint16_t* __restrict__ d, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const uint16_t v = s[i];
    d[i] = (uint16_t)((v >> 8) | (v << 8));
  }
}

// any NaN/Inf among n floats -> *flag = 1 (the device half of grid.py:82-83)
__global__ void nonfinite_kernel(const float* __restrict__ x, int64_t n, int* __restrict__ flag) {
  bool bad = false;
  const bool vec = (reinterpret_cast<uintptr_t>(x) & 15) == 0;
  const int64_t n4 = vec ? n / 4 : 0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (int64_t i = t0; i < n4; i += stride) {
    const float4 v = reinterpret_cast<const float4*>(x)[i];
    bad |= !isfinite(v.x) | !isfinite(v.y) | !isfinite(v.z) | !isfinite(v.w);
  }
  for (int64_t i = n4 * 4 + t0; i < n; i += stride) bad |= !isfinite(x[i]);
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(flag, 1);
}

cudaError_t launch_swap16(void* p, int64_t n, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  int64_t blocks = (n / 8 + kThreads - 1) / kThreads;
  if (blocks < 1) blocks = 1;
  if (blocks > (int64_t)kNumSMs * 8) blocks = (int64_t)kNumSMs * 8;
  swap16_kernel<<<(int)blocks, kThreads, 0, st>>>(reinterpret_cast<uint16_t*>(p), n);
  note_launch(1);
  return cudaGetLastError();
}

// pread exactly len bytes at off (parallel slices); false on error / short read
bool pread_full(int fd, char* dst, int64_t len, int64_t off) {
  auto one = [fd](char* d, int64_t n, int64_t o) -> bool {
    while (n > 0) {
      const ssize_t r = pread(fd, d, (size_t)n, (off_t)o);
      if (r < 0 && errno == EINTR) continue;
      if (r <= 0) return false;
      d += r; n -= r; o += r;
    }
    return true;
  };
  const int nr = readers();
  if (len < (4ll << 20) || nr == 1) return one(dst, len, off);
  const int64_t slice = ((len + nr - 1) / nr + 4095) & ~int64_t(4095);
  bool ok[kMaxReaders];
  std::vector<std::thread> th;
  for (int t = 0; t < nr; ++t) {
    const int64_t a = t * slice, b = (t + 1) * slice < len ? (t + 1) * slice : len;
    ok[t] = true;
    if (a >= b) continue;
    th.emplace_back([&, t, a, b] { ok[t] = one(dst + a, b - a, off + a); });
  }
  for (auto& x : th) x.join();
  for (int t = 0; t < nr; ++t)
    if (!ok[t]) return false;
  return true;
}

bool pwrite_full(int fd, const char* src, int64_t len, int64_t off) {
  while (len > 0) {
    const ssize_t r = pwrite(fd, src, (size_t)len, (off_t)off);
    if (r < 0 && errno == EINTR) continue;
    if (r <= 0) return false;
    src += r; len -= r; off += r;
  }
  return true;
}

struct Staging {
  char* buf[2] = {nullptr, nullptr};
  cudaEvent_t ev[2] = {nullptr, nullptr};
  int64_t size = 0;
  cudaError_t init(int64_t n) {
    size = n < chunk_bytes() ? n : chunk_bytes();
    for (int i = 0; i < 2; ++i) {
      cudaError_t e = cudaHostAlloc(reinterpret_cast<void**>(&buf[i]), (size_t)size, cudaHostAllocDefault);
      if (e != cudaSuccess) return e;
      e = cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming);
      if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
  }
  ~Staging() {
    for (int i = 0; i < 2; ++i) {
      if (ev[i]) { cudaEventSynchronize(ev[i]); cudaEventDestroy(ev[i]); }
      if (buf[i]) cudaFreeHost(buf[i]);
    }
  }
};

int cuda_err(cudaError_t e, const char* where) {
  return io_fail(e == cudaErrorMemoryAllocation ? SSB_ENOMEM : SSB_ECUDA, "%s: %s", where, cudaGetErrorString(e));
}

struct Fd {
  int fd = -1;
  ~Fd() { if (fd >= 0) close(fd); }
};
}  // namespace

extern "C" {

int ssb_file_to_device(const char* path, int64_t offset, int64_t nbytes, void* dst, int swap16, void* stream) {
  if (!path || offset < 0 || nbytes < 0 || (nbytes > 0 && !dst)) return io_fail(SSB_EINVAL, "bad file_to_device arguments");
  if (swap16 && ((nbytes & 1) || (reinterpret_cast<uintptr_t>(dst) & 15)))
    return io_fail(SSB_EINVAL, "swap16 needs an even byte count and a 16-byte aligned destination");
  Fd f;
  f.fd = open(path, O_RDONLY | O_CLOEXEC);
  if (f.fd < 0) return io_fail(SSB_EINVAL, "cannot open %s: %s", path, strerror(errno));
  struct stat sb;
  if (fstat(f.fd, &sb) != 0 || (int64_t)sb.st_size < offset + nbytes)
    return io_fail(SSB_EINVAL, "%s holds %lld bytes, fewer than offset %lld + %lld", path, (long long)sb.st_size,
                   (long long)offset, (long long)nbytes);
  if (nbytes == 0) return SSB_OK;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  Staging sg;
  cudaError_t e = sg.init(nbytes);
  if (e != cudaSuccess) return cuda_err(e, "pinned staging");
  char* d = reinterpret_cast<char*>(dst);
  int64_t k = 0;
  for (int64_t pos = 0; pos < nbytes; pos += sg.size, ++k) {
    const int b = (int)(k & 1);
    const int64_t len = nbytes - pos < sg.size ? nbytes - pos : sg.size;
    if (k >= 2 && (e = cudaEventSynchronize(sg.ev[b])) != cudaSuccess) return cuda_err(e, "staging reuse");
    if (!pread_full(f.fd, sg.buf[b], len, offset + pos))
      return io_fail(SSB_EINVAL, "short read from %s at byte %lld", path, (long long)(offset + pos));
    if ((e = cudaMemcpyAsync(d + pos, sg.buf[b], (size_t)len, cudaMemcpyHostToDevice, st)) != cudaSuccess)
      return cuda_err(e, "H2D copy");
    if ((e = cudaEventRecord(sg.ev[b], st)) != cudaSuccess) return cuda_err(e, "event");
  }
  if (swap16 && (e = launch_swap16(dst, nbytes / 2, st)) != cudaSuccess) return cuda_err(e, "swap16");
  if ((e = cudaStreamSynchronize(st)) != cudaSuccess) return cuda_err(e, "file_to_device");
  return SSB_OK;
}

int ssb_f32_nonfinite(const void* x, int64_t n, int* flag, void* stream) {
  if (n < 0 || (n > 0 && (!x || !flag))) return io_fail(SSB_EINVAL, "bad f32_nonfinite arguments");
  if (n == 0) return SSB_OK;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  int64_t blocks = (n / 4 + kThreads - 1) / kThreads;
  if (blocks < 1) blocks = 1;
  if (blocks > (int64_t)kNumSMs * 8) blocks = (int64_t)kNumSMs * 8;
  nonfinite_kernel<<<(int)blocks, kThreads, 0, st>>>(reinterpret_cast<const float*>(x), n, flag);
  note_launch(1);
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? SSB_OK : cuda_err(e, "f32_nonfinite");
}

int ssb_device_to_file(const char* path, int64_t offset, const void* src, int64_t nbytes, int swap16, void* stream) {
  if (!path || offset < 0 || nbytes < 0 || (nbytes > 0 && !src)) return io_fail(SSB_EINVAL, "bad device_to_file arguments");
  if (swap16 && (nbytes & 1)) return io_fail(SSB_EINVAL, "swap16 needs an even byte count");
  Fd f;
  f.fd = open(path, O_WRONLY | O_CREAT | O_CLOEXEC, 0644);
  if (f.fd < 0) return io_fail(SSB_EINVAL, "cannot open %s for writing: %s", path, strerror(errno));
  if (ftruncate(f.fd, (off_t)(offset + nbytes)) != 0)
    return io_fail(SSB_EINVAL, "cannot size %s: %s", path, strerror(errno));
  if (nbytes == 0) return SSB_OK;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  Staging sg;
  cudaError_t e = sg.init(nbytes);
  if (e != cudaSuccess) return cuda_err(e, "pinned staging");
  void* tmp = nullptr;  // device chunk for swapped samples
  if (swap16 && (e = cudaMallocAsync(&tmp, (size_t)sg.size, st)) != cudaSuccess) return cuda_err(e, "swap staging");
  const char* s = reinterpret_cast<const char*>(src);
  int64_t pend_pos[2] = {-1, -1}, pend_len[2] = {0, 0};
  int rc = SSB_OK;
  auto drain = [&](int b) -> bool {
    if (pend_pos[b] < 0) return true;
    if ((e = cudaEventSynchronize(sg.ev[b])) != cudaSuccess) { rc = cuda_err(e, "D2H copy"); return false; }
    if (!pwrite_full(f.fd, sg.buf[b], pend_len[b], offset + pend_pos[b])) {
      rc = io_fail(SSB_EINVAL, "short write to %s: %s", path, strerror(errno));
      return false;
    }
    pend_pos[b] = -1;
    return true;
  };
  int64_t k = 0;
  for (int64_t pos = 0; pos < nbytes && rc == SSB_OK; pos += sg.size, ++k) {
    const int b = (int)(k & 1);
    const int64_t len = nbytes - pos < sg.size ? nbytes - pos : sg.size;
    if (!drain(b)) break;
    const void* from = s + pos;
    if (swap16) {
      const int64_t n = len / 2;
      int64_t blocks = (n + kThreads - 1) / kThreads;
      if (blocks > (int64_t)kNumSMs * 8) blocks = (int64_t)kNumSMs * 8;
      swap16_copy_kernel<<<(int)blocks, kThreads, 0, st>>>(reinterpret_cast<const uint16_t*>(from),
                                                             reinterpret_cast<uint16_t*>(tmp), n);
      note_launch(1);
      from = tmp;
    }
    if ((e = cudaMemcpyAsync(sg.buf[b], from, (size_t)len, cudaMemcpyDeviceToHost, st)) != cudaSuccess) {
      rc = cuda_err(e, "D2H copy");
      break;
    }
    if ((e = cudaEventRecord(sg.ev[b], st)) != cudaSuccess) { rc = cuda_err(e, "event"); break; }
    pend_pos[b] = pos;
    pend_len[b] = len;
    if (swap16) {  // tmp is reused by the next chunk: finish this one first
      if (!drain(b)) break;
    }
  }
  if (rc == SSB_OK) drain((int)(k & 1));        // chunk k-2 (older)
  if (rc == SSB_OK) drain((int)((k + 1) & 1));  // chunk k-1
  if (tmp) cudaFreeAsync(tmp, st);
  cudaStreamSynchronize(st);
  return rc;
}

}  // extern "C"
