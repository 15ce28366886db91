// satsweep-b200: the extern "C" boundary (include/satsweep_b200.h).
//
// Validation mirrors the reference's error contract so the Python facade can
// map status codes onto the same exception types:
//   window/stride geometry  -> SSB_EINVAL  (InvalidWindowError, grid.py:133-143)
//   allocation failure      -> SSB_ENOMEM  (ResourceLimitError, integral.py:76-83)
//   non-finite F32 pixels   -> SSB_ENONFINITE (GridValidationError, grid.py:82-83)
#include <atomic>
#include <chrono>
#include <memory>
#include <thread>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <mutex>
#include <string>
#include <vector>

#include "ssb_common.cuh"
#include "../../include/satsweep_b200.h"

namespace ssb {
void widen_u32_to_u64(const uint32_t* src, uint64_t* dst, size_t n);  // host_widen.cpp
void widen_u16_to_u64(const uint16_t* src, uint64_t* dst, size_t n);
void copy_u64_stream(const uint64_t* src, uint64_t* dst, size_t n);
}

#ifndef SSB_ENONFINITE
#define SSB_ENONFINITE 5
#endif

namespace ssb {
cudaError_t launch_sat_prepare(int dtype, const void* in, int64_t R, int64_t C, int64_t in_ld, bool sq, void* ws,
                               void* totals, void* totals_sq, int* nonfinite, cudaStream_t st);
cudaError_t launch_sat_finish(int dtype, const void* in, int64_t R, int64_t C, int64_t in_ld, void* sat, void* sat_sq,
                              int64_t sat_ld, const void* carry, const void* carry_sq, void* ws, cudaStream_t st);
int64_t sat_workspace_bytes(int dtype, int64_t R, int64_t C, bool sq);
cudaError_t launch_sat_onepass(int dtype, const void* in, int64_t R, int64_t C, int64_t in_ld, void* sat, void* sat_sq,
                               int64_t sat_ld, const void* carry, const void* carry_sq, void* ws, cudaStream_t st);
bool onepass_supported(int dtype, bool sq);
int64_t sat_onepass_workspace_bytes(int dtype, int64_t R, int64_t C, bool sq);
cudaError_t launch_sat_build(int dtype, const void* in, int64_t R, int64_t C, int64_t in_ld, void* sat, void* sat_sq,
                             int64_t sat_ld, const void* carry, const void* carry_sq, void* ws, int* nonfinite,
                             cudaStream_t st);
void sat_plan_info(int dtype, int64_t R, int64_t C, bool sq, int64_t* info);
cudaError_t launch_window_eval(const void* sat, const void* sat_sq, bool is_float, int in_dtype, int64_t R, int64_t C,
                               int64_t sat_ld, int64_t w, int64_t s, int mask, WinOut o, cudaStream_t st);
cudaError_t launch_window_fused(const void* in, int dtype, int64_t R, int64_t C, int64_t in_ld, int64_t w, int mask,
                                WinOut o, int* nonfinite, int nK, cudaStream_t st);
cudaError_t launch_window_eval_multi(const void* sat, const void* sat_sq, bool is_float, int in_dtype, int64_t R,
                                     int64_t C, int64_t sat_ld, int nwin, const int64_t* ws, int mask, const WinOut* outs,
                                     cudaStream_t st);
bool sat_sweep_supported(int dtype, int64_t w, int mask);
int64_t sat_sweep_workspace_bytes(int dtype, int64_t R, int64_t C);
void sat_sweep_plan_info(int dtype, int64_t R, int64_t C, int64_t w, int64_t* info);
cudaError_t launch_sat_sweep(int dtype, const void* in, int64_t R, int64_t C, int64_t in_ld, void* sat, int64_t sat_ld,
                             int64_t w, int mask, WinOut o, void* ws, cudaStream_t st, bool onepass);
constexpr int64_t kFusedMaxWindow = 3072;

static std::atomic<long long> g_launches{0};
void note_launch(int n) { g_launches.fetch_add(n, std::memory_order_relaxed); }
int io_fail(int code, const char* fmt, ...);
int shard_fail(int code, const char* fmt, ...);
int shard_cuda_fail(cudaError_t e, const char* where);
}  // namespace ssb

using namespace ssb;

namespace {
thread_local std::string t_err;

int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  t_err = buf;
  return code;
}

int cuda_fail(cudaError_t e, const char* where) {
  if (e == cudaErrorMemoryAllocation) return fail(SSB_ENOMEM, "%s: %s", where, cudaGetErrorString(e));
  return fail(SSB_ECUDA, "%s: %s", where, cudaGetErrorString(e));
}

bool valid_dtype(int d) { return d == SSB_U8 || d == SSB_U16 || d == SSB_I32 || d == SSB_F32; }
int elem_size(int d) { return d == SSB_U8 ? 1 : d == SSB_U16 ? 2 : 4; }

int check_image(int dtype, int64_t rows, int64_t cols, int64_t in_ld) {
  if (!valid_dtype(dtype)) return fail(SSB_EUNSUPPORTED, "unsupported element dtype code %d", dtype);
  if (rows < 1 || cols < 1) return fail(SSB_EINVAL, "grid dims must be >= 1, got %lldx%lld", (long long)rows, (long long)cols);
  if (in_ld < cols) return fail(SSB_EINVAL, "in_ld %lld < cols %lld", (long long)in_ld, (long long)cols);
  return SSB_OK;
}

// Table writers store rows with 256-bit st.global.v4.b64 (sat_tiles.cuh,
// sat_sweep.cu), so every table row must start on a 32-byte boundary: the
// table base 32-byte aligned and the pitch a multiple of 4 elements.
int check_table_out(const void* sat, const void* sat_sq, int64_t sat_ld, int64_t cols) {
  if (sat_ld < cols + 1 || (sat_ld & 3))
    return fail(SSB_EINVAL, "sat_ld must be a multiple of 4 and >= cols+1 (got %lld for %lld cols)", (long long)sat_ld,
                (long long)cols);
  if ((reinterpret_cast<uintptr_t>(sat) & 31) || (reinterpret_cast<uintptr_t>(sat_sq) & 31))
    return fail(SSB_EINVAL, "tables must be 32-byte aligned");
  return SSB_OK;
}

int check_aligned(const void* p, const char* what) {
  if (reinterpret_cast<uintptr_t>(p) & 15) return fail(SSB_EINVAL, "%s must be 16-byte aligned", what);
  return SSB_OK;
}

int check_window(int64_t rows, int64_t cols, int64_t w, int64_t stride) {
  if (w < 1) return fail(SSB_EINVAL, "window size must be >= 1, got %lld", (long long)w);
  if (stride < 1) return fail(SSB_EINVAL, "stride must be >= 1, got %lld", (long long)stride);
  if (w > rows || w > cols)
    return fail(SSB_EINVAL, "window size %lld exceeds grid dims %lldx%lld; windows must fit fully inside the grid",
                (long long)w, (long long)rows, (long long)cols);
  return SSB_OK;
}

int check_stats(int dtype, int mask) {
  if (mask == 0 || (mask & ~(SSB_SUM | SSB_MEAN | SSB_STD)) != 0) return fail(SSB_EINVAL, "bad stat mask %d", mask);
  if (dtype == SSB_I32 && (mask & SSB_STD))
    return fail(SSB_EUNSUPPORTED, "std is not supported for int32 input (squared sums exceed 64 bits)");
  return SSB_OK;
}

cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// Launches go to the caller's stream, which may belong to a device other than
// the calling thread's current one: make the stream's device current for the
// call and restore the caller's device afterwards.
struct DeviceGuard {
  int prev = -1;
  cudaError_t err = cudaSuccess;
  explicit DeviceGuard(void* stream) {
    int d = 0;
    if ((err = cudaStreamGetDevice(as_stream(stream), &d)) != cudaSuccess) return;
    if ((err = cudaGetDevice(&prev)) != cudaSuccess) return;
    if (d != prev) err = cudaSetDevice(d);
    else prev = -1;
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};
#define SSB_DEVICE_GUARD(stream)                                  \
  DeviceGuard device_guard_(stream);                              \
  if (device_guard_.err != cudaSuccess) return cuda_fail(device_guard_.err, "stream device")
}  // namespace

// the calling thread's write census (ssb_census_enable); kernels launched by
// this thread while it is set count their stores into it
namespace {
thread_local Census t_census;
}
Census ssb::census_sink() { return t_census; }

// shard.cu and io.cu report through the same thread-local message
int ssb::shard_fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  t_err = buf;
  return code;
}

int ssb::shard_cuda_fail(cudaError_t e, const char* where) { return cuda_fail(e, where); }

int ssb::io_fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  t_err = buf;
  return code;
}

extern "C" {

int ssb_abi_version(void) { return SSB_ABI_VERSION; }

int ssb_census_enable(unsigned long long* table_rows, int64_t n_table_rows, unsigned long long* table_cols,
                      int64_t n_table_cols, unsigned long long* out_rows, int64_t n_out_rows) {
  if ((table_rows && n_table_rows < 1) || (table_cols && n_table_cols < 1) || (out_rows && n_out_rows < 1) ||
      (!table_rows != !table_cols))
    return fail(SSB_EINVAL, "bad census buffers");
  t_census = Census{table_rows, table_cols, out_rows, table_rows ? n_table_rows : 0, table_cols ? n_table_cols : 0,
                    out_rows ? n_out_rows : 0};
  return SSB_OK;
}

int ssb_census_disable(void) {
  t_census = Census{};
  return SSB_OK;
}
const char* ssb_last_error(void) { return t_err.c_str(); }
int64_t ssb_launch_count(void) { return (int64_t)g_launches.load(); }
int64_t ssb_window_fused_max_w(void) { return kFusedMaxWindow; }

int64_t ssb_sat_workspace_bytes(int in_dtype, int64_t rows, int64_t cols, int with_squares) {
  if (!valid_dtype(in_dtype) || rows < 1 || cols < 1) return -1;
  return sat_workspace_bytes(in_dtype, rows, cols, with_squares != 0);
}

int64_t ssb_sat_lookback_workspace_bytes(int in_dtype, int64_t rows, int64_t cols, int with_squares) {
  if (!valid_dtype(in_dtype) || rows < 1 || cols < 1 || !onepass_supported(in_dtype, with_squares != 0)) return -1;
  return sat_onepass_workspace_bytes(in_dtype, rows, cols, with_squares != 0);
}

int ssb_sat_plan(int in_dtype, int64_t rows, int64_t cols, int with_squares, int64_t* info4) {
  if (!valid_dtype(in_dtype) || rows < 1 || cols < 1 || !info4) return fail(SSB_EINVAL, "bad plan request");
  sat_plan_info(in_dtype, rows, cols, with_squares != 0, info4);
  return SSB_OK;
}

int ssb_sat_prepare(const void* in, int in_dtype, int64_t rows, int64_t cols, int64_t in_ld, int with_squares,
                    void* ws, int64_t ws_bytes, void* band_totals, void* band_totals_sq, int* nonfinite_flag,
                    void* stream) {
  int rc = check_image(in_dtype, rows, cols, in_ld);
  if (rc) return rc;
  if (in_dtype == SSB_I32 && with_squares) return fail(SSB_EUNSUPPORTED, "squared tables are not supported for int32 input");
  if ((rc = check_aligned(in, "input raster"))) return rc;
  const int64_t need = sat_workspace_bytes(in_dtype, rows, cols, with_squares != 0);
  if (!ws || ws_bytes < need) return fail(SSB_EINVAL, "workspace too small: need %lld bytes", (long long)need);
  SSB_DEVICE_GUARD(stream);
  cudaError_t e = launch_sat_prepare(in_dtype, in, rows, cols, in_ld, with_squares != 0, ws, band_totals,
                                     band_totals_sq, nonfinite_flag, as_stream(stream));
  return e == cudaSuccess ? SSB_OK : cuda_fail(e, "ssb_sat_prepare");
}

int ssb_sat_finish(const void* in, int in_dtype, int64_t rows, int64_t cols, int64_t in_ld, void* sat, void* sat_sq,
                   int64_t sat_ld, const void* carry, const void* carry_sq, void* ws, int64_t ws_bytes, void* stream) {
  int rc = check_image(in_dtype, rows, cols, in_ld);
  if (rc) return rc;
  if (!sat && !sat_sq) return fail(SSB_EINVAL, "no table to write");
  if ((rc = check_aligned(in, "input raster"))) return rc;
  if ((rc = check_table_out(sat, sat_sq, sat_ld, cols))) return rc;
  const int64_t need = sat_workspace_bytes(in_dtype, rows, cols, sat_sq != nullptr);
  if (!ws || ws_bytes < need) return fail(SSB_EINVAL, "workspace too small: need %lld bytes", (long long)need);
  SSB_DEVICE_GUARD(stream);
  cudaError_t e = launch_sat_finish(in_dtype, in, rows, cols, in_ld, sat, sat_sq, sat_ld, carry, carry_sq, ws,
                                    as_stream(stream));
  return e == cudaSuccess ? SSB_OK : cuda_fail(e, "ssb_sat_finish");
}

int ssb_sat_build(const void* in, int in_dtype, int64_t rows, int64_t cols, int64_t in_ld, void* sat, void* sat_sq,
                  int64_t sat_ld, const void* carry, const void* carry_sq, void* ws, int64_t ws_bytes,
                  int* nonfinite_flag, void* stream) {
  int rc = check_image(in_dtype, rows, cols, in_ld);
  if (rc) return rc;
  if (in_dtype == SSB_I32 && sat_sq) return fail(SSB_EUNSUPPORTED, "squared tables are not supported for int32 input");
  if (!sat && !sat_sq) return fail(SSB_EINVAL, "no table to write");
  if ((rc = check_aligned(in, "input raster"))) return rc;
  if ((rc = check_table_out(sat, sat_sq, sat_ld, cols))) return rc;
  const int64_t need = sat_workspace_bytes(in_dtype, rows, cols, sat_sq != nullptr);
  if (!ws || ws_bytes < need) return fail(SSB_EINVAL, "workspace too small: need %lld bytes", (long long)need);
  SSB_DEVICE_GUARD(stream);
  cudaError_t e = launch_sat_build(in_dtype, in, rows, cols, in_ld, sat, sat_sq, sat_ld, carry, carry_sq, ws,
                                   nonfinite_flag, as_stream(stream));
  return e == cudaSuccess ? SSB_OK : cuda_fail(e, "ssb_sat_build");
}

int ssb_sat_build_lookback(const void* in, int in_dtype, int64_t rows, int64_t cols, int64_t in_ld, void* sat,
                           void* sat_sq, int64_t sat_ld, const void* carry, const void* carry_sq, void* ws,
                           int64_t ws_bytes, void* stream) {
  int rc = check_image(in_dtype, rows, cols, in_ld);
  if (rc) return rc;
  if (!onepass_supported(in_dtype, sat_sq != nullptr))
    return fail(SSB_EUNSUPPORTED, "the single-pass build takes integer input (no squares for int32)");
  if (!sat && !sat_sq) return fail(SSB_EINVAL, "no table to write");
  if ((rc = check_aligned(in, "input raster"))) return rc;
  if ((rc = check_table_out(sat, sat_sq, sat_ld, cols))) return rc;
  const int64_t need = sat_onepass_workspace_bytes(in_dtype, rows, cols, sat_sq != nullptr);
  if (!ws || ws_bytes < need) return fail(SSB_EINVAL, "workspace too small: need %lld bytes", (long long)need);
  SSB_DEVICE_GUARD(stream);
  cudaError_t e = launch_sat_onepass(in_dtype, in, rows, cols, in_ld, sat, sat_sq, sat_ld, carry, carry_sq, ws,
                                     as_stream(stream));
  return e == cudaSuccess ? SSB_OK : cuda_fail(e, "ssb_sat_build_lookback");
}

int ssb_window_eval(const void* sat, const void* sat_sq, int in_dtype, int64_t rows, int64_t cols, int64_t sat_ld,
                    int64_t w, int64_t stride, int stat_mask, void* out_sum, double* out_mean, double* out_std,
                    int64_t out_ld, void* stream) {
  int rc = check_image(in_dtype, rows, cols, cols);
  if (rc) return rc;
  if ((rc = check_window(rows, cols, w, stride))) return rc;
  if ((rc = check_stats(in_dtype, stat_mask))) return rc;
  if (!sat || sat_ld < cols + 1) return fail(SSB_EINVAL, "bad table");
  if ((stat_mask & SSB_STD) && !sat_sq) return fail(SSB_EINVAL, "squared sums required for std dev");
  if (((stat_mask & SSB_SUM) && !out_sum) || ((stat_mask & SSB_MEAN) && !out_mean) || ((stat_mask & SSB_STD) && !out_std))
    return fail(SSB_EINVAL, "missing output buffer");
  const int64_t out_c = (cols - w) / stride + 1;
  if (out_ld < out_c) return fail(SSB_EINVAL, "out_ld < output cols");
  WinOut o{out_sum, out_mean, out_std, out_ld};
  SSB_DEVICE_GUARD(stream);
  cudaError_t e = launch_window_eval(sat, sat_sq, in_dtype == SSB_F32, in_dtype, rows, cols, sat_ld, w, stride,
                                     stat_mask, o, as_stream(stream));
  return e == cudaSuccess ? SSB_OK : cuda_fail(e, "ssb_window_eval");
}

int ssb_sat_swa_supported(int in_dtype, int64_t w, int stat_mask) {
  return valid_dtype(in_dtype) && sat_sweep_supported(in_dtype, w, stat_mask) ? 1 : 0;
}

int64_t ssb_sat_swa_workspace_bytes(int in_dtype, int64_t rows, int64_t cols) {
  if (!valid_dtype(in_dtype) || in_dtype == SSB_F32 || rows < 1 || cols < 1) return -1;
  return sat_sweep_workspace_bytes(in_dtype, rows, cols);
}

int ssb_sat_swa_plan(int in_dtype, int64_t rows, int64_t cols, int64_t w, int64_t* info4) {
  if (!valid_dtype(in_dtype) || in_dtype == SSB_F32 || rows < 1 || cols < 1 || w < 1 || !info4)
    return fail(SSB_EINVAL, "bad plan request");
  sat_sweep_plan_info(in_dtype, rows, cols, w, info4);
  return SSB_OK;
}

}  // extern "C"

static int sat_build_swa_impl(bool onepass, const void* in, int in_dtype, int64_t rows, int64_t cols, int64_t in_ld, void* sat,
                      int64_t sat_ld, int64_t w, int stat_mask, void* out_sum, double* out_mean, int64_t out_ld,
                      void* ws, int64_t ws_bytes, void* stream) {
  int rc = check_image(in_dtype, rows, cols, in_ld);
  if (rc) return rc;
  if ((rc = check_window(rows, cols, w, 1))) return rc;
  if ((rc = check_stats(in_dtype, stat_mask))) return rc;
  if (!sat_sweep_supported(in_dtype, w, stat_mask))
    return fail(SSB_EUNSUPPORTED, "table+sweep pass takes integer input, sum/mean and w <= 257 (dtype %d, w %lld)",
                in_dtype, (long long)w);
  if ((rc = check_aligned(in, "input raster"))) return rc;
  if (!sat) return fail(SSB_EINVAL, "no table to write");
  if ((rc = check_table_out(sat, nullptr, sat_ld, cols))) return rc;
  if (((stat_mask & SSB_SUM) && !out_sum) || ((stat_mask & SSB_MEAN) && !out_mean))
    return fail(SSB_EINVAL, "missing output buffer");
  if (out_ld < cols - w + 1) return fail(SSB_EINVAL, "out_ld < output cols");
  const int64_t need = sat_sweep_workspace_bytes(in_dtype, rows, cols);
  if (!ws || ws_bytes < need) return fail(SSB_EINVAL, "workspace too small: need %lld bytes", (long long)need);
  WinOut o{out_sum, out_mean, nullptr, out_ld};
  SSB_DEVICE_GUARD(stream);
  cudaError_t e = launch_sat_sweep(in_dtype, in, rows, cols, in_ld, sat, sat_ld, w, stat_mask, o, ws,
                                   as_stream(stream), onepass);
  return e == cudaSuccess ? SSB_OK : cuda_fail(e, "ssb_sat_build_swa");
}

namespace {
// buffer sets in flight for ssb_swa_host (SSB_HOST_SETS overrides; read once)
int host_sets() {
  static const int n = [] {
    const char* e = getenv("SSB_HOST_SETS");
    const int v = e ? atoi(e) : 3;
    return v < 1 ? 1 : v > 8 ? 8 : v;
  }();
  return n;
}

// one private pool per device for ssb_swa_host's band buffers, created on
// first use; it keeps the last call's buffers reserved (never the caller's
// default pool or torch's allocator) until ssb_host_release()
std::mutex g_pool_mu;
cudaMemPool_t g_pools[64] = {};
cudaError_t host_pool(int device, cudaMemPool_t* out) {
  std::mutex& mu = g_pool_mu;
  cudaMemPool_t* pools = g_pools;
  if (device < 0 || device >= 64) return cudaErrorInvalidDevice;
  std::lock_guard<std::mutex> lk(mu);
  if (!pools[device]) {
    cudaMemPoolProps props = {};
    props.allocType = cudaMemAllocationTypePinned;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = device;
    cudaError_t e = cudaMemPoolCreate(&pools[device], &props);
    if (e != cudaSuccess) return e;
    uint64_t thr = UINT64_MAX;  // keep blocks for reuse across the bands of one call
    cudaMemPoolSetAttribute(pools[device], cudaMemPoolAttrReleaseThreshold, &thr);
  }
  *out = pools[device];
  return cudaSuccess;
}

// ---- narrow wire format of ssb_swa_host (uint32 sums over PCIe, widened on the host) ----
std::atomic<int> g_host_threads{0};  // widening threads per call (0: automatic)
std::atomic<int> g_host_wire{0};  // 0: automatic (32 bits when every sum provably fits), 64: always full width
std::atomic<int64_t> t_host_h2d{0}, t_host_d2h{0};  // bytes copied by the process's latest ssb_swa_host call

// pinned staging ring, one per device, kept between calls (pinning ~2 GB takes
// longer than a C5 call); released by ssb_host_release().  A concurrent call on
// the same device gets its own temporary ring.
struct StageCache {
  void* p = nullptr;
  size_t bytes = 0;
  bool busy = false;
};
StageCache g_stage[64];

// 4 sums per thread: two 16-byte loads, one 16-byte store; a band's outputs are
// contiguous.  *band_max receives the band's largest sum (one atomic per warp):
// a band whose sums all fit 16 bits leaves as uint16 instead.
__global__ void __launch_bounds__(256) narrow_u64_u32_kernel(const uint64_t* __restrict__ src, uint32_t* __restrict__ dst,
                                                             int64_t n, uint32_t* __restrict__ band_max) {
  const int64_t n4 = n >> 2;
  uint32_t mx = 0u;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
    const ulonglong2 a = __ldcs(reinterpret_cast<const ulonglong2*>(src) + 2 * i);
    const ulonglong2 b = __ldcs(reinterpret_cast<const ulonglong2*>(src) + 2 * i + 1);
    const uint4 v = make_uint4((uint32_t)a.x, (uint32_t)a.y, (uint32_t)b.x, (uint32_t)b.y);
    mx = max(max(mx, max(v.x, v.y)), max(v.z, v.w));
    __stcs(reinterpret_cast<uint4*>(dst) + i, v);
  }
  if (blockIdx.x == 0 && threadIdx.x < (n & 3)) {
    const uint32_t v = (uint32_t)src[(n4 << 2) + threadIdx.x];
    dst[(n4 << 2) + threadIdx.x] = v;
    mx = max(mx, v);
  }
  mx = __reduce_max_sync(0xffffffffu, mx);
  if ((threadIdx.x & 31) == 0 && mx) atomicMax(band_max, mx);
}

// 8 sums per thread (32-byte load, 16-byte store); only for bands whose largest sum fits 16 bits
__global__ void __launch_bounds__(256) narrow_u32_u16_kernel(const uint32_t* __restrict__ src, uint16_t* __restrict__ dst,
                                                             int64_t n) {
  const int64_t n8 = n >> 3;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n8; i += (int64_t)gridDim.x * blockDim.x) {
    const uint4 a = __ldcs(reinterpret_cast<const uint4*>(src) + 2 * i);
    const uint4 b = __ldcs(reinterpret_cast<const uint4*>(src) + 2 * i + 1);
    __stcs(reinterpret_cast<uint4*>(dst) + i,
           make_uint4(a.x | (a.y << 16), a.z | (a.w << 16), b.x | (b.y << 16), b.z | (b.w << 16)));
  }
  if (blockIdx.x == 0 && threadIdx.x < (n & 7)) dst[(n8 << 3) + threadIdx.x] = (uint16_t)src[(n8 << 3) + threadIdx.x];
}

// Host side of the narrow wire.  A band's uint32 sums leave the device in
// chunks of whole output rows (a few MB, SSB_HOST_CHUNK_KB) through a small
// pinned ring, so a chunk is widened while it is still in the host's last-level
// cache; a coordinator waits for each chunk's copy to land, worker t widens
// chunks t, t + T, ... into the caller's array, and the issuing thread reuses a
// ring slot only after the chunk that held it has been widened.
struct WirePipe {
  struct Desc {           // what a ring slot holds; written before `issued`, read after `landed`
    uint64_t* dst = nullptr;  // first output row of the chunk in the caller's array
    int64_t rows = 0;
    int esz = 4;              // bytes per element on the wire: 2 / 4 (widened to uint64) or 8 (copied)
  };
  int device = 0, T = 1, NS = 1;  // workers, ring slots
  int64_t out_c = 0, out_ld = 0;
  int64_t rpc = 1;                // output rows per uint32 chunk (other widths take the rows that fill the same bytes)
  uint32_t* stage = nullptr;
  size_t slot_elems = 0;          // uint32 elements per slot (a slot holds at least one 8-byte row)
  std::vector<Desc> desc;         // per slot
  int64_t copied_bytes = 0;       // device->host bytes of the narrow chunks (issuing thread)
  std::vector<cudaEvent_t> copied;  // per slot: the chunk's device->host copy has completed
  std::atomic<int64_t> issued{0}, landed{0};
  std::atomic<int64_t> total{-1};   // chunks in all, published once the last one is issued
  std::atomic<bool> abort{false};
  std::unique_ptr<std::atomic<int64_t>[]> prog;  // 1 + the last chunk each worker finished
  std::vector<std::thread> threads;
  cudaError_t coord_err = cudaSuccess;
  std::unique_ptr<double[]> busy;  // seconds each worker spent widening (SSB_HOST_PROF)
  double slot_wait_s = 0.0;       // seconds the issuing thread waited for a free slot

  static void nap() { std::this_thread::sleep_for(std::chrono::microseconds(5)); }

  void plan(int64_t chunk_elems, int64_t band_rows) {
    rpc = chunk_elems / out_c;
    if (rpc < 1) rpc = 1;
    if (rpc > band_rows) rpc = band_rows;
    if (rpc < 2) rpc = 2;  // room for one row of 8-byte elements
    slot_elems = (size_t)rpc * out_c;
  }
  int64_t rows_per_chunk(int esz) const { const int64_t r = rpc * 4 / esz; return r < 1 ? 1 : r; }
  // waits until chunk g has reached `stage` (true) or no chunk g will come (false)
  bool wait_for(const std::atomic<int64_t>& stage_count, int64_t g) {
    for (;;) {
      if (stage_count.load(std::memory_order_acquire) > g) return true;
      const int64_t n = total.load(std::memory_order_acquire);
      if ((n >= 0 && g >= n) || abort.load()) return false;
      nap();
    }
  }

  void start() {
    prog.reset(new std::atomic<int64_t>[T]);
    for (int t = 0; t < T; ++t) prog[t].store(0);
    busy.reset(new double[T]());
    threads.emplace_back([this] {
      cudaSetDevice(device);
      for (int64_t g = 0; wait_for(issued, g); ++g) {
        const cudaError_t e = cudaEventSynchronize(copied[g % NS]);
        if (e != cudaSuccess) { coord_err = e; abort.store(true); return; }
        landed.store(g + 1, std::memory_order_release);
      }
    });
    for (int t = 0; t < T; ++t)
      threads.emplace_back([this, t] {
        for (int64_t g = t; wait_for(landed, g); g += T) {
          const Desc d = desc[g % NS];
          const uint32_t* src = stage + (size_t)(g % NS) * slot_elems;
          const auto t0 = std::chrono::steady_clock::now();
          auto put = [&](size_t off, uint64_t* dst, size_t n) {  // n elements from element offset `off` of the slot
            if (d.esz == 2) widen_u16_to_u64(reinterpret_cast<const uint16_t*>(src) + off, dst, n);
            else if (d.esz == 4) widen_u32_to_u64(src + off, dst, n);
            else copy_u64_stream(reinterpret_cast<const uint64_t*>(src) + off, dst, n);
          };
          if (out_ld == out_c) {
            put(0, d.dst, (size_t)d.rows * out_c);
          } else {
            for (int64_t r = 0; r < d.rows; ++r) put((size_t)r * out_c, d.dst + (size_t)r * out_ld, (size_t)out_c);
          }
          busy[t] += std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
          prog[t].store(g + 1, std::memory_order_release);
        }
      });
  }
  // the slot of chunk g is free once chunk g - NS has been widened
  bool wait_slot(int64_t g) {
    if (g < NS) return true;
    const int64_t prev = g - NS;
    std::atomic<int64_t>& p = prog[prev % T];
    if (p.load(std::memory_order_acquire) > prev) return true;
    const auto t0 = std::chrono::steady_clock::now();
    while (p.load(std::memory_order_acquire) <= prev) {
      if (abort.load()) return false;
      nap();
    }
    slot_wait_s += std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    return true;
  }
  // Enqueue one band's results (nb rows of esz-byte elements at band_src) on the copy stream, chunk by
  // chunk into the ring (a slot is free once the chunk that held it is widened); each chunk is handed to
  // the host threads when its copy lands.  dst: the band's first row in the caller's array.
  // Returns cudaSuccess, a CUDA error, or cudaErrorUnknown when the host side stopped.
  cudaError_t issue_band(cudaStream_t d2h_st, const char* band_src, int esz, int64_t nb, uint64_t* dst) {
    const int64_t step = rows_per_chunk(esz);  // about the same bytes per chunk in every format
    for (int64_t r0 = 0; r0 < nb; r0 += step) {
      const int64_t g = issued.load(std::memory_order_relaxed), nr = r0 + step < nb ? step : nb - r0;
      if (!wait_slot(g)) return cudaErrorUnknown;
      const int slot = (int)(g % NS);
      desc[slot] = Desc{dst + (size_t)r0 * out_ld, nr, esz};
      copied_bytes += nr * out_c * esz;
      cudaError_t e = cudaMemcpyAsync(stage + (size_t)slot * slot_elems, band_src + (size_t)r0 * out_c * esz,
                                      (size_t)nr * out_c * esz, cudaMemcpyDeviceToHost, d2h_st);
      if (e == cudaSuccess) e = cudaEventRecord(copied[slot], d2h_st);
      if (e != cudaSuccess) return e;
      issued.store(g + 1, std::memory_order_release);
    }
    return cudaSuccess;
  }
  // threads from the call's settings; ring from the device's cache (or a temporary one); events; start
  int threads_for_call() const {
    static const int env_t = [] { const char* v = getenv("SSB_HOST_THREADS"); return v ? atoi(v) : 0; }();
    static const int env_lws = [] { const char* v = getenv("LOCAL_WORLD_SIZE"); const int n = v ? atoi(v) : 1; return n < 1 ? 1 : n; }();
    const int hw = (int)std::thread::hardware_concurrency() / env_lws;
    const int set_t = g_host_threads.load();
    const int t = set_t > 0 ? set_t : env_t > 0 ? env_t : (hw > 3 ? hw - 2 : 1);
    return t > 64 ? 64 : t;
  }
  // no more chunks: the threads leave once the issued ones are widened
  void finish(bool ok) {
    if (!ok) abort.store(true);
    total.store(issued.load(), std::memory_order_release);
    for (auto& th : threads) th.join();
    threads.clear();
  }
};
}  // namespace

extern "C" {

int ssb_sat_build_swa(const void* in, int in_dtype, int64_t rows, int64_t cols, int64_t in_ld, void* sat,
                      int64_t sat_ld, int64_t w, int stat_mask, void* out_sum, double* out_mean, int64_t out_ld,
                      void* ws, int64_t ws_bytes, void* stream) {
  return sat_build_swa_impl(false, in, in_dtype, rows, cols, in_ld, sat, sat_ld, w, stat_mask, out_sum, out_mean,
                            out_ld, ws, ws_bytes, stream);
}

int ssb_sat_build_swa_onepass(const void* in, int in_dtype, int64_t rows, int64_t cols, int64_t in_ld, void* sat,
                              int64_t sat_ld, int64_t w, int stat_mask, void* out_sum, double* out_mean,
                              int64_t out_ld, void* ws, int64_t ws_bytes, void* stream) {
  return sat_build_swa_impl(true, in, in_dtype, rows, cols, in_ld, sat, sat_ld, w, stat_mask, out_sum, out_mean,
                            out_ld, ws, ws_bytes, stream);
}

int ssb_window_eval_multi(const void* sat, const void* sat_sq, int in_dtype, int64_t rows, int64_t cols,
                          int64_t sat_ld, int n_windows, const int64_t* windows, int stat_mask,
                          void* const* out_sums, double* const* out_means, double* const* out_stds,
                          const int64_t* out_lds, void* stream) {
  if (n_windows < 1 || !windows) return fail(SSB_EINVAL, "windows list must be non-empty");
  for (int k = 0; k < n_windows; ++k) {  // validate all before any work (integral.py:205-208)
    int rc = check_window(rows, cols, windows[k], 1);
    if (rc) return rc;
  }
  int rc = check_stats(in_dtype, stat_mask);
  if (rc) return rc;
  if (!sat || sat_ld < cols + 1) return fail(SSB_EINVAL, "bad table");
  if ((stat_mask & SSB_STD) && !sat_sq) return fail(SSB_EINVAL, "squared sums required for std dev");
  SSB_DEVICE_GUARD(stream);
  // groups of up to 8 windows share one pass over the table
  for (int k0 = 0; k0 < n_windows; k0 += 8) {
    const int nk = n_windows - k0 < 8 ? n_windows - k0 : 8;
    WinOut outs[8];
    bool ok = true;
    for (int k = 0; k < nk; ++k) {
      const int kk = k0 + k;
      outs[k] = WinOut{out_sums ? out_sums[kk] : nullptr, out_means ? out_means[kk] : nullptr,
                       out_stds ? out_stds[kk] : nullptr, out_lds[kk]};
      if (((stat_mask & SSB_SUM) && !outs[k].sum) || ((stat_mask & SSB_MEAN) && !outs[k].mean) ||
          ((stat_mask & SSB_STD) && !outs[k].std_))
        return fail(SSB_EINVAL, "missing output buffer");
      if (out_lds[kk] < cols - windows[kk] + 1) return fail(SSB_EINVAL, "out_ld < output cols");
    }
    cudaError_t e = launch_window_eval_multi(sat, sat_sq, in_dtype == SSB_F32, in_dtype, rows, cols, sat_ld, nk,
                                             windows + k0, stat_mask, outs, as_stream(stream));
    if (e == cudaErrorNotSupported) {
      cudaGetLastError();
      ok = false;
    } else if (e != cudaSuccess) {
      return cuda_fail(e, "ssb_window_eval_multi");
    }
    if (!ok) {
      for (int k = 0; k < nk; ++k) {
        const int kk = k0 + k;
        rc = ssb_window_eval(sat, sat_sq, in_dtype, rows, cols, sat_ld, windows[kk], 1, stat_mask, outs[k].sum,
                             outs[k].mean, outs[k].std_, out_lds[kk], stream);
        if (rc) return rc;
      }
    }
  }
  return SSB_OK;
}

int ssb_window_fused(const void* in, int in_dtype, int64_t rows, int64_t cols, int64_t in_ld, int64_t w,
                     int stat_mask, void* out_sum, double* out_mean, double* out_std, int64_t out_ld,
                     int* nonfinite_flag, int segments, void* stream) {
  int rc = check_image(in_dtype, rows, cols, in_ld);
  if (rc) return rc;
  if ((rc = check_window(rows, cols, w, 1))) return rc;
  if ((rc = check_stats(in_dtype, stat_mask))) return rc;
  if (w > kFusedMaxWindow) return fail(SSB_EUNSUPPORTED, "fused path supports w <= %lld", (long long)kFusedMaxWindow);
  if ((rc = check_aligned(in, "input raster"))) return rc;
  if (((stat_mask & SSB_SUM) && !out_sum) || ((stat_mask & SSB_MEAN) && !out_mean) || ((stat_mask & SSB_STD) && !out_std))
    return fail(SSB_EINVAL, "missing output buffer");
  if (out_ld < cols - w + 1) return fail(SSB_EINVAL, "out_ld < output cols");
  WinOut o{out_sum, out_mean, out_std, out_ld};
  SSB_DEVICE_GUARD(stream);
  cudaError_t e = launch_window_fused(in, in_dtype, rows, cols, in_ld, w, stat_mask, o, nonfinite_flag, segments,
                                      as_stream(stream));
  return e == cudaSuccess ? SSB_OK : cuda_fail(e, "ssb_window_fused");
}

int ssb_window_sum_at(const void* sat, int is_float_table, int64_t rows, int64_t cols, int64_t sat_ld, int64_t top,
                      int64_t left, int64_t w, void* out_value, void* stream) {
  if (w < 1 || top < 0 || left < 0 || top + w > rows || left + w > cols)  // integral.py:122-125
    return fail(SSB_EINVAL, "%lldx%lld region at (%lld, %lld) does not lie within the %lldx%lld source", (long long)w,
                (long long)w, (long long)top, (long long)left, (long long)rows, (long long)cols);
  const uint64_t* t = reinterpret_cast<const uint64_t*>(sat);
  uint64_t c[4];
  const int64_t idx[4] = {(top + w) * sat_ld + left + w, top * sat_ld + left + w, (top + w) * sat_ld + left,
                          top * sat_ld + left};
  SSB_DEVICE_GUARD(stream);
  cudaStream_t st = as_stream(stream);
  for (int k = 0; k < 4; ++k) {
    cudaError_t e = cudaMemcpyAsync(&c[k], t + idx[k], 8, cudaMemcpyDeviceToHost, st);
    if (e != cudaSuccess) return cuda_fail(e, "ssb_window_sum_at");
  }
  cudaError_t e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return cuda_fail(e, "ssb_window_sum_at");
  if (is_float_table) {
    double d[4];
    memcpy(d, c, sizeof(d));
    const double v = (d[0] - d[1]) - (d[2] - d[3]);
    memcpy(out_value, &v, 8);
  } else {
    const uint64_t v = (c[0] - c[1]) - (c[2] - c[3]);
    memcpy(out_value, &v, 8);
  }
  return SSB_OK;
}

// ---------------------------------------------------------------------------
// host-buffer end-to-end path (helpers host_sets / host_pool above)
int ssb_host_release(void) {
  std::lock_guard<std::mutex> lk(g_pool_mu);
  for (auto& p : g_pools)
    if (p) {
      cudaError_t e = cudaMemPoolTrimTo(p, 0);
      if (e != cudaSuccess) return cuda_fail(e, "ssb_host_release");
    }
  for (auto& c : g_stage)
    if (c.p && !c.busy) {
      cudaFreeHost(c.p);
      c = StageCache{};
    }
  return SSB_OK;
}

int ssb_host_wire(int bits) {
  const int prev = g_host_wire.load();
  if (bits == 0 || bits == 32 || bits == 64) g_host_wire.store(bits);
  return prev;
}

int ssb_host_widen(const void* src, int src_bits, void* dst_u64, int64_t n) {
  if (!src || !dst_u64 || n < 0) return fail(SSB_EINVAL, "ssb_host_widen: bad arguments");
  if (src_bits == 32) widen_u32_to_u64(reinterpret_cast<const uint32_t*>(src), reinterpret_cast<uint64_t*>(dst_u64), (size_t)n);
  else if (src_bits == 16) widen_u16_to_u64(reinterpret_cast<const uint16_t*>(src), reinterpret_cast<uint64_t*>(dst_u64), (size_t)n);
  else return fail(SSB_EINVAL, "ssb_host_widen: src_bits must be 16 or 32");
  return SSB_OK;
}

int ssb_host_threads(int n) {
  const int prev = g_host_threads.load();
  if (n >= 0) g_host_threads.store(n > 64 ? 64 : n);
  return prev;
}

void ssb_host_last_copy_bytes(int64_t* h2d_bytes, int64_t* d2h_bytes) {
  if (h2d_bytes) *h2d_bytes = t_host_h2d.load();
  if (d2h_bytes) *d2h_bytes = t_host_d2h.load();
}


int ssb_swa_host(const void* in_host, int in_dtype, int64_t rows, int64_t cols, int64_t in_ld, int64_t w,
                 int64_t stride, int stat_mask, void* out_sum_host, double* out_mean_host, double* out_std_host,
                 int64_t out_ld, int pipeline, int device, int64_t band_rows) {
  int rc = check_image(in_dtype, rows, cols, in_ld);
  if (rc) return rc;
  if ((rc = check_window(rows, cols, w, stride))) return rc;
  if ((rc = check_stats(in_dtype, stat_mask))) return rc;
  if (pipeline == SSB_PIPE_FUSED && (stride != 1 || w > kFusedMaxWindow)) pipeline = SSB_PIPE_TABLE;
  const bool sweep_ok = stride == 1 && sat_sweep_supported(in_dtype, w, stat_mask);
  const bool sq = (stat_mask & SSB_STD) != 0;
  const int es = elem_size(in_dtype);
  const int64_t out_r = (rows - w) / stride + 1, out_c = (cols - w) / stride + 1;
  if (out_ld < out_c) return fail(SSB_EINVAL, "out_ld < output cols");
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) return cuda_fail(e, "cudaSetDevice");
  // the bands' kernels see band-local rows: the write census covers the
  // device entry points only, so it is suspended for this call
  struct CensusPause {
    Census saved = t_census;
    CensusPause() { t_census = Census{}; }
    ~CensusPause() { t_census = saved; }
  } census_pause;

  // band geometry: output rows [o0, o1) need input rows [o0*s, (o1-1)*s + w)
  const int64_t sat_ld = ((cols + 1) + 3) & ~int64_t(3);  // 32-byte aligned rows
  const int nstats = ((stat_mask & SSB_SUM) ? 1 : 0) + ((stat_mask & SSB_MEAN) ? 1 : 0) + ((stat_mask & SSB_STD) ? 1 : 0);
  auto in_rows_for = [&](int64_t nb) { return (nb - 1) * stride + w; };
  if (band_rows <= 0) {
    // ~3 GB of device buffers per band set (C5: ~2,000-row bands; 1k-8k-row
    // bands measured within box-to-box noise, 0.85-1.0 s, D2H at 90-97 % of
    // the pinned PCIe ceiling), at least 4 bands when the image is large
    const double per_out_row = (double)stride * ((double)cols * es +
                               (pipeline == SSB_PIPE_TABLE ? 8.0 * sat_ld * (sq ? 2 : 1) : 0.0)) +
                               8.0 * (double)out_c * nstats;
    band_rows = (int64_t)(3.0e9 / per_out_row);
    const int64_t quarter = (out_r + 3) / 4;
    if (band_rows > quarter && out_r > 4096) band_rows = quarter;
    if (band_rows >= 2048) band_rows &= ~int64_t(1023);  // C5: 2,048-row bands (0.91 vs 0.95 s at 2,080)
    if (band_rows < 1) band_rows = 1;
  }
  if (band_rows > out_r) band_rows = out_r;
  const int64_t n_bands = (out_r + band_rows - 1) / band_rows;
  // buffer sets in flight (one stream each): the D2H of the results is the
  // critical path, so a set's H2D + compute overlaps the other sets' D2H
  const int n_sets = (int)(n_bands < host_sets() ? n_bands : host_sets());
  const int64_t max_in_rows = in_rows_for(band_rows);

  const size_t in_bytes = (size_t)max_in_rows * cols * es;
  const size_t sat_bytes = pipeline == SSB_PIPE_TABLE ? (size_t)(max_in_rows + 1) * sat_ld * 8 : 0;
  const size_t ws_bytes = pipeline == SSB_PIPE_TABLE ? (size_t)sat_workspace_bytes(in_dtype, max_in_rows, cols, sq) : 0;
  const size_t out_bytes = (size_t)band_rows * out_c * 8;
  // narrow wire: unsigned sums that provably fit 32 bits cross PCIe as uint32
  // and are widened into the caller's uint64 array by host threads
  // (host_widen.cpp); small results are not worth the threads
  const double maxv = in_dtype == SSB_U8 ? 255.0 : in_dtype == SSB_U16 ? 65535.0 : 0.0;
  const bool narrow = g_host_wire.load() != 64 && (stat_mask & SSB_SUM) && out_sum_host && maxv > 0.0 &&
                      (double)w * (double)w * maxv < 4294967296.0 && out_r * out_c >= (int64_t(1) << 22);
  const bool allow16 = g_host_wire.load() != 32;
  uint32_t* h_max = nullptr;  // pinned: the bands' largest sums, one word per buffer set (tail of the ring)
  // 64-bit results bound for pageable memory take the ring too (8-byte chunks, copied by the same
  // threads): a DMA into pageable memory is staged by the driver at a fraction of the PCIe rate
  auto pageable = [](const void* q) {
    if (!q) return false;
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, q) != cudaSuccess) { cudaGetLastError(); return true; }
    return a.type == cudaMemoryTypeUnregistered;
  };
  const bool stage_ok = g_host_wire.load() != 64 && out_r * out_c >= (int64_t(1) << 22);
  const bool stage_sum = stage_ok && !narrow && (stat_mask & SSB_SUM) && pageable(out_sum_host);
  const bool stage_mean = stage_ok && (stat_mask & SSB_MEAN) && pageable(out_mean_host);
  const bool stage_std = stage_ok && (stat_mask & SSB_STD) && pageable(out_std_host);
  const bool piped = narrow || stage_sum || stage_mean || stage_std;  // the ring and its threads are in use
  int64_t d2h_direct = 0;  // bytes copied straight into the caller's arrays
  int64_t h2d_bytes = 0;  // uploaded: every band's input rows (consecutive bands share w - stride rows)

  struct Set {
    cudaStream_t st = nullptr;         // H2D + compute of this set's bands
    cudaEvent_t ready = nullptr;       // band results complete (recorded on st)
    cudaEvent_t drained = nullptr;     // band results copied out (recorded on the D2H stream)
    void *in = nullptr, *sat = nullptr, *sq = nullptr, *ws = nullptr, *o_sum = nullptr, *o_mean = nullptr,
         *o_std = nullptr, *o_n32 = nullptr;
    uint32_t* d_max = nullptr;  // the band's largest sum (narrow wire)
  };
  std::vector<Set> sets(n_sets);
  // every D2H goes through ONE stream in band order: the result copy is the
  // critical path, and a single in-order copy stream keeps one copy engine
  // streaming at the PCIe ceiling while the sets' H2D + compute run beside it
  cudaStream_t d2h_st = nullptr;
  int* d_flag = nullptr;
  int status = SSB_OK;
  // band buffers come from a library-private stream-ordered pool, trimmed
  // back to zero before returning: the caller's default pool (and torch's
  // allocator) never see a changed release threshold or memory kept reserved
  cudaMemPool_t pool = nullptr;
  if ((e = host_pool(device, &pool)) != cudaSuccess) return cuda_fail(e, "memory pool");
  auto alloc = [&](void** p, size_t n, cudaStream_t st) -> bool {
    if (n == 0) return true;
    cudaError_t ae = cudaMallocFromPoolAsync(p, n, pool, st);
    if (ae != cudaSuccess) { status = cuda_fail(ae, "device allocation"); return false; }
    return true;
  };
  if ((e = cudaStreamCreateWithFlags(&d2h_st, cudaStreamNonBlocking)) != cudaSuccess) status = cuda_fail(e, "stream");
  for (auto& s : sets) {
    if (status != SSB_OK) break;
    if ((e = cudaStreamCreateWithFlags(&s.st, cudaStreamNonBlocking)) != cudaSuccess ||
        (e = cudaEventCreateWithFlags(&s.ready, cudaEventDisableTiming)) != cudaSuccess ||
        (e = cudaEventCreateWithFlags(&s.drained, cudaEventDisableTiming)) != cudaSuccess) {
      status = cuda_fail(e, "stream");
      break;
    }
    if (!alloc(&s.in, in_bytes, s.st) || !alloc(&s.sat, sat_bytes, s.st) || !alloc(&s.sq, sq ? sat_bytes : 0, s.st) ||
        !alloc(&s.ws, ws_bytes, s.st) || !alloc(&s.o_sum, (stat_mask & SSB_SUM) ? out_bytes : 0, s.st) ||
        !alloc(&s.o_mean, (stat_mask & SSB_MEAN) ? out_bytes : 0, s.st) ||
        !alloc(&s.o_std, (stat_mask & SSB_STD) ? out_bytes : 0, s.st) || !alloc(&s.o_n32, narrow ? out_bytes / 2 : 0, s.st) ||
        !alloc(reinterpret_cast<void**>(&s.d_max), narrow ? 256 : 0, s.st))
      break;
  }
  WirePipe pipe;
  StageCache* cache = nullptr;  // the device's cached ring when this call holds it
  void* own_stage = nullptr;    // a temporary ring otherwise
  if (piped && status == SSB_OK) {
    // widening threads: ssb_host_threads(), else SSB_HOST_THREADS, else this process's share of the
    // cores (one process per GPU under torchrun: LOCAL_WORLD_SIZE) minus the issuing thread and the coordinator
    pipe.device = device;
    pipe.T = pipe.threads_for_call();
    pipe.out_c = out_c; pipe.out_ld = out_ld;
    static const int env_kb = [] { const char* v = getenv("SSB_HOST_CHUNK_KB"); return v ? atoi(v) : 0; }();
    pipe.plan((int64_t)(env_kb > 0 ? env_kb : 2048) * 256, band_rows);  // uint32 elements per chunk
    pipe.NS = pipe.T + 4;
    const size_t need = pipe.slot_elems * 4 * pipe.NS + 256;  // + the bands' maxima (one word per buffer set)
    {
      std::lock_guard<std::mutex> lk(g_pool_mu);
      StageCache& c = g_stage[device];
      if (!c.busy) {
        if (c.bytes < need) {
          if (c.p) cudaFreeHost(c.p);
          c = StageCache{};
          if ((e = cudaHostAlloc(&c.p, need, cudaHostAllocDefault)) == cudaSuccess) c.bytes = need;
          else { c.p = nullptr; status = cuda_fail(e, "pinned staging"); }
        }
        if (c.p) { c.busy = true; cache = &c; pipe.stage = reinterpret_cast<uint32_t*>(c.p); }
      }
    }
    if (!cache && status == SSB_OK) {
      if ((e = cudaHostAlloc(&own_stage, need, cudaHostAllocDefault)) != cudaSuccess) status = cuda_fail(e, "pinned staging");
      pipe.stage = reinterpret_cast<uint32_t*>(own_stage);
    }
    if (pipe.stage) h_max = pipe.stage + pipe.slot_elems * pipe.NS;
    pipe.desc.assign(pipe.NS, WirePipe::Desc{});
    pipe.copied.assign(pipe.NS, nullptr);
    for (auto& ev : pipe.copied)
      if (status == SSB_OK && (e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming)) != cudaSuccess)
        status = cuda_fail(e, "event");
    if (status == SSB_OK) {
      try {
        pipe.start();
      } catch (const std::exception& ex) {  // thread creation failed: stop the ones that started
        pipe.finish(false);
        status = fail(SSB_ECUDA, "host widening threads: %s", ex.what());
      }
    }
  }
  if (status == SSB_OK && (e = cudaMalloc(&d_flag, sizeof(int))) != cudaSuccess) status = cuda_fail(e, "flag");
  if (status == SSB_OK && (e = cudaMemset(d_flag, 0, sizeof(int))) != cudaSuccess) status = cuda_fail(e, "flag");

  // one band's host->device copy and kernels on its set's stream
  auto compute_band = [&](int64_t b) -> bool {
    Set& s = sets[b % n_sets];
    const int64_t o0 = b * band_rows, o1 = (o0 + band_rows < out_r) ? o0 + band_rows : out_r;
    const int64_t nb = o1 - o0, r0 = o0 * stride, nr = in_rows_for(nb);
    const char* src = reinterpret_cast<const char*>(in_host) + (size_t)r0 * in_ld * es;
    // the set's outputs may be overwritten once its previous band is copied out
    if (b >= n_sets && (e = cudaStreamWaitEvent(s.st, s.drained, 0)) != cudaSuccess) { status = cuda_fail(e, "wait"); return false; }
    const void* band_in = s.in;
    // contiguous rows: one linear copy (no per-row DMA descriptors)
    e = in_ld == cols ? cudaMemcpyAsync(s.in, src, (size_t)nr * cols * es, cudaMemcpyHostToDevice, s.st)
                      : cudaMemcpy2DAsync(s.in, (size_t)cols * es, src, (size_t)in_ld * es, (size_t)cols * es,
                                          (size_t)nr, cudaMemcpyHostToDevice, s.st);
    if (e != cudaSuccess) { status = cuda_fail(e, "H2D"); return false; }
    h2d_bytes += nr * cols * es;
    WinOut o{s.o_sum, reinterpret_cast<double*>(s.o_mean), reinterpret_cast<double*>(s.o_std), out_c};
    if (pipeline == SSB_PIPE_TABLE && sweep_ok) {  // table + windows without reading the table back
      e = launch_sat_sweep(in_dtype, band_in, nr, cols, cols, s.sat, sat_ld, w, stat_mask, o, s.ws, s.st, false);
    } else if (pipeline == SSB_PIPE_TABLE) {
      e = launch_sat_build(in_dtype, band_in, nr, cols, cols, s.sat, s.sq, sat_ld, nullptr, nullptr, s.ws, d_flag, s.st);
      if (e == cudaSuccess)
        e = launch_window_eval(s.sat, s.sq, in_dtype == SSB_F32, in_dtype, nr, cols, sat_ld, w, stride, stat_mask, o, s.st);
    } else {
      e = launch_window_fused(band_in, in_dtype, nr, cols, cols, w, stat_mask, o, d_flag, 0, s.st);
    }
    if (e != cudaSuccess) { status = cuda_fail(e, "band compute"); return false; }
    if (narrow) {
      if ((e = cudaMemsetAsync(s.d_max, 0, 4, s.st)) != cudaSuccess) { status = cuda_fail(e, "narrow"); return false; }
      narrow_u64_u32_kernel<<<kNumSMs * 8, 256, 0, s.st>>>(reinterpret_cast<const uint64_t*>(s.o_sum),
                                                           reinterpret_cast<uint32_t*>(s.o_n32), nb * out_c, s.d_max);
      note_launch(1);
      if ((e = cudaGetLastError()) != cudaSuccess ||
          (e = cudaMemcpyAsync(h_max + (b % n_sets), s.d_max, 4, cudaMemcpyDeviceToHost, s.st)) != cudaSuccess) {
        status = cuda_fail(e, "narrow");
        return false;
      }
    }
    if ((e = cudaEventRecord(s.ready, s.st)) != cudaSuccess) { status = cuda_fail(e, "event"); return false; }
    return true;
  };
  // the band's results to the host on the one copy stream
  auto drain_band = [&](int64_t b) -> bool {
    Set& s = sets[b % n_sets];
    const int64_t o0 = b * band_rows, o1 = (o0 + band_rows < out_r) ? o0 + band_rows : out_r;
    const int64_t nb = o1 - o0;
    if ((e = cudaStreamWaitEvent(d2h_st, s.ready, 0)) != cudaSuccess) { status = cuda_fail(e, "event"); return false; }
    auto d2h = [&](void* host, void* dev) -> bool {
      if (!host) return true;
      char* dst = reinterpret_cast<char*>(host) + (size_t)o0 * out_ld * 8;
      cudaError_t ce = out_ld == out_c
                           ? cudaMemcpyAsync(dst, dev, (size_t)nb * out_c * 8, cudaMemcpyDeviceToHost, d2h_st)
                           : cudaMemcpy2DAsync(dst, (size_t)out_ld * 8, dev, (size_t)out_c * 8, (size_t)out_c * 8,
                                               (size_t)nb, cudaMemcpyDeviceToHost, d2h_st);
      if (ce != cudaSuccess) { status = cuda_fail(ce, "D2H"); return false; }
      d2h_direct += nb * out_c * 8;
      return true;
    };
    // 64-bit results: straight into pinned arrays, through the ring into pageable ones
    auto out64 = [&](bool staged, void* host, void* dev) -> bool {
      if (!host || !staged) return d2h(host, dev);
      e = pipe.issue_band(d2h_st, reinterpret_cast<const char*>(dev), 8, nb, reinterpret_cast<uint64_t*>(host) + (size_t)o0 * out_ld);
      if (e != cudaSuccess) {
        status = e == cudaErrorUnknown ? fail(SSB_ECUDA, "host widening stopped") : cuda_fail(e, "D2H");
        return false;
      }
      return true;
    };
    if (narrow) {
      // a band whose largest sum fits 16 bits leaves as uint16 (decided from the band's maximum, which
      // the narrowing kernel computed; the issuing thread runs ahead of the device, so this wait is short)
      if ((e = cudaEventSynchronize(s.ready)) != cudaSuccess) { status = cuda_fail(e, "event"); return false; }
      const bool half = allow16 && h_max[b % n_sets] < 65536u;
      if (half) {  // the uint64 sums are dead once narrowed: their buffer takes the uint16 copy
        narrow_u32_u16_kernel<<<kNumSMs * 8, 256, 0, d2h_st>>>(reinterpret_cast<const uint32_t*>(s.o_n32),
                                                               reinterpret_cast<uint16_t*>(s.o_sum), nb * out_c);
        note_launch(1);
        if ((e = cudaGetLastError()) != cudaSuccess) { status = cuda_fail(e, "narrow"); return false; }
      }
      const char* band_src = reinterpret_cast<const char*>(half ? s.o_sum : s.o_n32);
      e = pipe.issue_band(d2h_st, band_src, half ? 2 : 4, nb, reinterpret_cast<uint64_t*>(out_sum_host) + (size_t)o0 * out_ld);
      if (e != cudaSuccess) {
        status = e == cudaErrorUnknown ? fail(SSB_ECUDA, "host widening stopped") : cuda_fail(e, "D2H");
        return false;
      }
    }
    if (!out64(stage_sum, (stat_mask & SSB_SUM) && !narrow ? out_sum_host : nullptr, s.o_sum) ||
        !out64(stage_mean, (stat_mask & SSB_MEAN) ? out_mean_host : nullptr, s.o_mean) ||
        !out64(stage_std, (stat_mask & SSB_STD) ? out_std_host : nullptr, s.o_std))
      return false;
    if ((e = cudaEventRecord(s.drained, d2h_st)) != cudaSuccess) { status = cuda_fail(e, "event"); return false; }
    return true;
  };
  // A drain through the ring blocks the issuing thread on ring slots for about
  // as long as the band's copy takes, so the next band's upload and kernels
  // are enqueued first; the straight copy never blocks.
  for (int64_t b = 0; status == SSB_OK && b < n_bands; ++b) {
    if (!compute_band(b)) break;
    if (piped ? (b >= 1 && !drain_band(b - 1)) : !drain_band(b)) break;
  }
  if (piped && status == SSB_OK) drain_band(n_bands - 1);
  t_host_h2d = h2d_bytes;
  if (d2h_st) {
    cudaError_t se = cudaStreamSynchronize(d2h_st);
    if (se != cudaSuccess && status == SSB_OK) status = cuda_fail(se, "stream sync");
  }
  for (auto& s : sets) {
    if (!s.st) continue;
    cudaError_t se = cudaStreamSynchronize(s.st);
    if (se != cudaSuccess && status == SSB_OK) status = cuda_fail(se, "stream sync");
    void* ptrs[] = {s.in, s.sat, s.sq, s.ws, s.o_sum, s.o_mean, s.o_std, s.o_n32, s.d_max};
    for (void* p : ptrs) if (p) cudaFreeAsync(p, s.st);
    cudaStreamSynchronize(s.st);
    if (s.ready) cudaEventDestroy(s.ready);
    if (s.drained) cudaEventDestroy(s.drained);
    cudaStreamDestroy(s.st);
  }
  if (d2h_st) cudaStreamDestroy(d2h_st);
  t_host_d2h = d2h_direct + pipe.copied_bytes;
  if (piped) {
    if (!pipe.threads.empty()) pipe.finish(status == SSB_OK);  // joins after the last band is widened
    if (pipe.coord_err != cudaSuccess && status == SSB_OK) status = cuda_fail(pipe.coord_err, "D2H wait");
    static const bool prof = getenv("SSB_HOST_PROF") != nullptr;  // tuning: where the host side spends its time
    if (prof && pipe.busy) {
      double mx = 0, sum = 0;
      for (int t = 0; t < pipe.T; ++t) { sum += pipe.busy[t]; if (pipe.busy[t] > mx) mx = pipe.busy[t]; }
      fprintf(stderr, "ssb_swa_host wire: T=%d slots=%d chunks=%lld x %lld rows (x2 as uint16), widen busy max %.3f s mean %.3f s, slot wait %.3f s\n",
              pipe.T, pipe.NS, (long long)pipe.issued.load(), (long long)pipe.rpc, mx, sum / pipe.T, pipe.slot_wait_s);
    }
    for (auto ev : pipe.copied) if (ev) cudaEventDestroy(ev);
    if (own_stage) cudaFreeHost(own_stage);
    if (cache) { std::lock_guard<std::mutex> lk(g_pool_mu); cache->busy = false; }
  }
  // the freed band buffers stay reserved in the library's pool for the next
  // call (mapping ~9 GB of fresh device memory costs ~0.1 s per C5 call);
  // ssb_host_release() returns them.  Errors trim it right away.
  if (status != SSB_OK) cudaMemPoolTrimTo(pool, 0);
  if (d_flag) {
    int h = 0;
    if (status == SSB_OK) {
      cudaError_t fe = cudaMemcpy(&h, d_flag, sizeof(int), cudaMemcpyDeviceToHost);
      if (fe != cudaSuccess) status = cuda_fail(fe, "flag D2H");
    }
    cudaFree(d_flag);
    if (status == SSB_OK && h) status = fail(SSB_ENONFINITE, "F32 grid contains NaN or Inf; only finite values are admitted");
  }
  return status;
}

// Device-resident uint64 sums -> the caller's host array through the narrow
// wire of ssb_swa_host (multi_window and the other paths that evaluate on the
// device and return host arrays, api.py:58-67): rows x cols contiguous on the
// device, bands of ~32 M sums double-buffered through two narrowing buffers.
int ssb_sums_to_host(const void* dev_sums, int64_t rows, int64_t cols, uint64_t max_sum, void* host_out, int64_t out_ld,
                     void* stream) {
  if (!dev_sums || !host_out || rows < 1 || cols < 1 || out_ld < cols) return fail(SSB_EINVAL, "ssb_sums_to_host: bad arguments");
  SSB_DEVICE_GUARD(stream);
  cudaStream_t src_st = as_stream(stream);
  int device = 0;
  cudaError_t e = cudaGetDevice(&device);
  if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
  const bool stage_ok = g_host_wire.load() != 64 && rows * cols >= (int64_t(1) << 22);
  const bool narrow = stage_ok && max_sum > 0 && max_sum < 4294967296ull && (reinterpret_cast<uintptr_t>(dev_sums) & 15) == 0;
  const bool allow16 = g_host_wire.load() != 32;
  const uint64_t* src = reinterpret_cast<const uint64_t*>(dev_sums);
  // 8-byte values without a 32-bit bound (float64 results, wide sums) bound for pageable memory: through the
  // ring as they are, copied out by the host threads
  bool staged64 = false;
  if (stage_ok && !narrow) {
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, host_out) != cudaSuccess) { cudaGetLastError(); staged64 = true; }
    else staged64 = a.type == cudaMemoryTypeUnregistered;
  }
  if (!narrow && !staged64) {  // the straight 64-bit copy
    e = out_ld == cols ? cudaMemcpyAsync(host_out, src, (size_t)rows * cols * 8, cudaMemcpyDeviceToHost, src_st)
                       : cudaMemcpy2DAsync(host_out, (size_t)out_ld * 8, src, (size_t)cols * 8, (size_t)cols * 8, (size_t)rows,
                                           cudaMemcpyDeviceToHost, src_st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(src_st);
    t_host_h2d = 0;
    t_host_d2h = rows * cols * 8;
    return e == cudaSuccess ? SSB_OK : cuda_fail(e, "ssb_sums_to_host");
  }
  // bands of whole rows whose first sum is 16-byte aligned (the narrowing kernels use 16-byte accesses)
  int64_t band_rows = (int64_t(1) << 25) / cols;
  if (band_rows < 2) band_rows = 2;
  band_rows &= ~int64_t(1);
  if (band_rows > rows || !narrow) band_rows = rows;
  const int64_t n_bands = (rows + band_rows - 1) / band_rows;
  const int n_sets = !narrow ? 0 : n_bands < 2 ? 1 : 2;
  struct Set {
    void *n32 = nullptr, *n16 = nullptr;
    uint32_t* d_max = nullptr;
    cudaEvent_t ready = nullptr, drained = nullptr;
  } sets[2];
  int status = SSB_OK;
  cudaStream_t work = nullptr, d2h_st = nullptr;
  cudaEvent_t produced = nullptr;
  cudaMemPool_t pool = nullptr;
  if ((e = host_pool(device, &pool)) != cudaSuccess) return cuda_fail(e, "memory pool");
  if ((e = cudaStreamCreateWithFlags(&work, cudaStreamNonBlocking)) != cudaSuccess ||
      (e = cudaStreamCreateWithFlags(&d2h_st, cudaStreamNonBlocking)) != cudaSuccess ||
      (e = cudaEventCreateWithFlags(&produced, cudaEventDisableTiming)) != cudaSuccess ||
      (e = cudaEventRecord(produced, src_st)) != cudaSuccess || (e = cudaStreamWaitEvent(work, produced, 0)) != cudaSuccess ||
      (e = cudaStreamWaitEvent(d2h_st, produced, 0)) != cudaSuccess)
    status = cuda_fail(e, "stream");
  const size_t band_elems = (size_t)band_rows * cols;
  for (int k = 0; k < n_sets && status == SSB_OK; ++k) {
    Set& st = sets[k];
    if ((e = cudaMallocFromPoolAsync(&st.n32, band_elems * 4, pool, work)) != cudaSuccess ||
        (e = cudaMallocFromPoolAsync(&st.n16, band_elems * 2, pool, work)) != cudaSuccess ||
        (e = cudaMallocFromPoolAsync(reinterpret_cast<void**>(&st.d_max), 256, pool, work)) != cudaSuccess ||
        (e = cudaEventCreateWithFlags(&st.ready, cudaEventDisableTiming)) != cudaSuccess ||
        (e = cudaEventCreateWithFlags(&st.drained, cudaEventDisableTiming)) != cudaSuccess)
      status = cuda_fail(e, "device allocation");
  }
  WirePipe pipe;
  StageCache* cache = nullptr;
  void* own_stage = nullptr;
  uint32_t* h_max = nullptr;
  if (status == SSB_OK) {
    pipe.device = device;
    pipe.T = pipe.threads_for_call();
    pipe.out_c = cols; pipe.out_ld = out_ld;
    static const int env_kb = [] { const char* v = getenv("SSB_HOST_CHUNK_KB"); return v ? atoi(v) : 0; }();
    pipe.plan((int64_t)(env_kb > 0 ? env_kb : 2048) * 256, band_rows);
    pipe.NS = pipe.T + 4;
    const size_t need = pipe.slot_elems * 4 * pipe.NS + 256;
    {
      std::lock_guard<std::mutex> lk(g_pool_mu);
      StageCache& c = g_stage[device];
      if (!c.busy) {
        if (c.bytes < need) {
          if (c.p) cudaFreeHost(c.p);
          c = StageCache{};
          if ((e = cudaHostAlloc(&c.p, need, cudaHostAllocDefault)) == cudaSuccess) c.bytes = need;
          else { c.p = nullptr; status = cuda_fail(e, "pinned staging"); }
        }
        if (c.p) { c.busy = true; cache = &c; pipe.stage = reinterpret_cast<uint32_t*>(c.p); }
      }
    }
    if (!cache && status == SSB_OK) {
      if ((e = cudaHostAlloc(&own_stage, need, cudaHostAllocDefault)) != cudaSuccess) status = cuda_fail(e, "pinned staging");
      pipe.stage = reinterpret_cast<uint32_t*>(own_stage);
    }
    if (pipe.stage) h_max = pipe.stage + pipe.slot_elems * pipe.NS;
    pipe.desc.assign(pipe.NS, WirePipe::Desc{});
    pipe.copied.assign(pipe.NS, nullptr);
    for (auto& ev : pipe.copied)
      if (status == SSB_OK && (e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming)) != cudaSuccess)
        status = cuda_fail(e, "event");
    if (status == SSB_OK) {
      try {
        pipe.start();
      } catch (const std::exception& ex) {
        pipe.finish(false);
        status = fail(SSB_ECUDA, "host widening threads: %s", ex.what());
      }
    }
  }
  auto narrow_band = [&](int64_t b) -> bool {  // uint64 -> uint32 + the band's largest sum, on the work stream
    Set& st = sets[b % n_sets];
    const int64_t r0 = b * band_rows, nb = (r0 + band_rows < rows ? r0 + band_rows : rows) - r0;
    if ((b >= n_sets && (e = cudaStreamWaitEvent(work, st.drained, 0)) != cudaSuccess) ||
        (e = cudaMemsetAsync(st.d_max, 0, 4, work)) != cudaSuccess) {
      status = cuda_fail(e, "narrow");
      return false;
    }
    narrow_u64_u32_kernel<<<kNumSMs * 8, 256, 0, work>>>(src + (size_t)r0 * cols, reinterpret_cast<uint32_t*>(st.n32), nb * cols, st.d_max);
    note_launch(1);
    if ((e = cudaGetLastError()) != cudaSuccess ||
        (e = cudaMemcpyAsync(h_max + (b % n_sets), st.d_max, 4, cudaMemcpyDeviceToHost, work)) != cudaSuccess ||
        (e = cudaEventRecord(st.ready, work)) != cudaSuccess) {
      status = cuda_fail(e, "narrow");
      return false;
    }
    return true;
  };
  auto drain_band = [&](int64_t b) -> bool {
    Set& st = sets[b % n_sets];
    const int64_t r0 = b * band_rows, nb = (r0 + band_rows < rows ? r0 + band_rows : rows) - r0;
    if ((e = cudaStreamWaitEvent(d2h_st, st.ready, 0)) != cudaSuccess || (e = cudaEventSynchronize(st.ready)) != cudaSuccess) {
      status = cuda_fail(e, "event");
      return false;
    }
    const bool half = allow16 && h_max[b % n_sets] < 65536u;
    if (half) {
      narrow_u32_u16_kernel<<<kNumSMs * 8, 256, 0, d2h_st>>>(reinterpret_cast<const uint32_t*>(st.n32),
                                                             reinterpret_cast<uint16_t*>(st.n16), nb * cols);
      note_launch(1);
      if ((e = cudaGetLastError()) != cudaSuccess) { status = cuda_fail(e, "narrow"); return false; }
    }
    e = pipe.issue_band(d2h_st, reinterpret_cast<const char*>(half ? st.n16 : st.n32), half ? 2 : 4, nb,
                        reinterpret_cast<uint64_t*>(host_out) + (size_t)r0 * out_ld);
    if (e == cudaSuccess) e = cudaEventRecord(st.drained, d2h_st);
    if (e != cudaSuccess) {
      status = e == cudaErrorUnknown ? fail(SSB_ECUDA, "host widening stopped") : cuda_fail(e, "D2H");
      return false;
    }
    return true;
  };
  if (narrow) {
    for (int64_t b = 0; status == SSB_OK && b < n_bands; ++b) {
      if (!narrow_band(b)) break;
      if (b >= 1 && !drain_band(b - 1)) break;
    }
    if (status == SSB_OK) drain_band(n_bands - 1);
  } else if (status == SSB_OK) {  // staged64: the array as it is
    e = pipe.issue_band(d2h_st, reinterpret_cast<const char*>(src), 8, rows, reinterpret_cast<uint64_t*>(host_out));
    if (e != cudaSuccess) status = e == cudaErrorUnknown ? fail(SSB_ECUDA, "host copy stopped") : cuda_fail(e, "D2H");
  }
  if (d2h_st) { cudaStreamSynchronize(d2h_st); }
  if (work) {
    cudaStreamSynchronize(work);
    for (auto& st : sets) {
      void* ptrs[] = {st.n32, st.n16, st.d_max};
      for (void* q : ptrs) if (q) cudaFreeAsync(q, work);
      if (st.ready) cudaEventDestroy(st.ready);
      if (st.drained) cudaEventDestroy(st.drained);
    }
    cudaStreamSynchronize(work);
    cudaStreamDestroy(work);
  }
  if (d2h_st) cudaStreamDestroy(d2h_st);
  if (produced) cudaEventDestroy(produced);
  if (!pipe.threads.empty()) pipe.finish(status == SSB_OK);
  if (pipe.coord_err != cudaSuccess && status == SSB_OK) status = cuda_fail(pipe.coord_err, "D2H wait");
  for (auto ev : pipe.copied) if (ev) cudaEventDestroy(ev);
  if (own_stage) cudaFreeHost(own_stage);
  if (cache) { std::lock_guard<std::mutex> lk(g_pool_mu); cache->busy = false; }
  t_host_h2d = 0;
  t_host_d2h = pipe.copied_bytes;
  return status;
}


}  // extern "C"
