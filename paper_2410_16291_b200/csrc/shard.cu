// satsweep-b200: row-band sharding across the GPUs of one process
// (ssb_sharded_*).
//
// The reference splits one image over CPU workers of one process
// (pkg/src/satsweep/parallel.py:80-134, `swa(method="parallel")` with
// workers = os.cpu_count(), api.py:51-52 / parallel.py:71-72).  Here the
// workers are GPUs: device g owns a contiguous band of image rows (the
// reference's `partition` rule over OUTPUT rows, parallel.py:80-90) and
//
//   * receives the (w-1)-row halo below its band from the following devices
//     by peer copies over NVLink (cudaMemcpyPeerAsync), then evaluates its
//     output rows with the fused window kernel -- table offsets of the rows
//     above the band cancel in the four-corner difference, so nothing else
//     is exchanged for the window statistics;
//   * for the global integral image, reduces its band's column totals
//     (ssb_sat_prepare's band_totals), gathers the totals of the devices
//     above it (peer copies of (cols+1)-long vectors), sums them in a fixed
//     order (band_carry_kernel: the exclusive scan over bands) and writes
//     its global table rows with that carry row (ssb_sat_finish) -- no extra
//     pass over any table.
//
// Multi-process callers (one rank per GPU, torch.distributed/NCCL) use the
// same kernels: ssb_sat_prepare -> all-gather of the totals ->
// ssb_band_carry -> ssb_sat_finish (paper_2410_16291_b200/shard.py).
#include <cstdint>
#include <vector>

#include "ssb_common.cuh"
#include "../../include/satsweep_b200.h"

namespace ssb {
cudaError_t launch_sat_prepare(int dtype, const void* in, int64_t R, int64_t C, int64_t in_ld, bool sq, void* ws,
                               void* totals, void* totals_sq, int* nonfinite, cudaStream_t st);
cudaError_t launch_sat_finish(int dtype, const void* in, int64_t R, int64_t C, int64_t in_ld, void* sat, void* sat_sq,
                              int64_t sat_ld, const void* carry, const void* carry_sq, void* ws, cudaStream_t st);
int64_t sat_workspace_bytes(int dtype, int64_t R, int64_t C, bool sq);
cudaError_t launch_window_fused(const void* in, int dtype, int64_t R, int64_t C, int64_t in_ld, int64_t w, int mask,
                                WinOut o, int* nonfinite, int nK, cudaStream_t st);
void note_launch(int n);
int shard_fail(int code, const char* fmt, ...);
int shard_cuda_fail(cudaError_t e, const char* where);

// carry[c] = sum over g < band of parts[g * ld + c], in g order (exact modulo
// 2^64 for integer tables; a fixed order for float64 ones)
template <typename T>
__global__ void __launch_bounds__(kThreads) band_carry_kernel(const T* __restrict__ parts, int band, int64_t len,
                                                              int64_t ld, T* __restrict__ carry) {
  for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < len; c += (int64_t)gridDim.x * blockDim.x) {
    T acc = T(0);
    for (int g = 0; g < band; ++g) acc += parts[(int64_t)g * ld + c];
    carry[c] = acc;
  }
}

cudaError_t launch_band_carry(const void* parts, int band, int64_t len, int64_t ld, bool is_float, void* carry,
                              cudaStream_t st) {
  const int64_t want = (len + kThreads - 1) / kThreads;
  const int blocks = (int)(want < 4 * kNumSMs ? (want < 1 ? 1 : want) : 4 * kNumSMs);
  if (is_float)
    band_carry_kernel<double><<<blocks, kThreads, 0, st>>>(reinterpret_cast<const double*>(parts), band, len, ld,
                                                           reinterpret_cast<double*>(carry));
  else
    band_carry_kernel<uint64_t><<<blocks, kThreads, 0, st>>>(reinterpret_cast<const uint64_t*>(parts), band, len, ld,
                                                             reinterpret_cast<uint64_t*>(carry));
  note_launch(1);
  return cudaGetLastError();
}

// ---- geometry (mirrors paper_2410_16291_b200/shard.py, stride 1) ----------
struct BandGeom {
  int64_t own_lo, own_hi, need_lo, need_hi, out_lo, out_hi, cap_rows;
};

// parallel.py:80-90: at most p balanced contiguous blocks, the first n % p one larger
static void partition_rows(int64_t n, int p, std::vector<std::pair<int64_t, int64_t>>& out) {
  out.clear();
  const int q = (int)(n < p ? n : p) < 1 ? 1 : (int)(n < p ? n : p);
  const int64_t base = n / q, rem = n % q;
  int64_t lo = 0;
  for (int k = 0; k < q; ++k) {
    const int64_t hi = lo + base + (k < rem ? 1 : 0);
    out.emplace_back(lo, hi);
    lo = hi;
  }
  while ((int)out.size() < p) out.emplace_back(n, n);
}

static void band_plan(int64_t R, int64_t w, int n, std::vector<BandGeom>& g) {
  const int64_t out_r = R - w + 1;
  std::vector<std::pair<int64_t, int64_t>> parts;
  partition_rows(out_r, n, parts);
  g.assign(n, BandGeom{});
  int64_t cur = 0;
  for (int k = 0; k < n; ++k) {
    int64_t a = parts[k].first;
    int64_t b = k + 1 < n ? parts[k + 1].first : R;
    if (a > R) a = R;
    if (b > R) b = R;
    if (b < a) b = a;
    if (a < cur) a = cur;  // ownership is a partition of [0, R)
    if (b < a) b = a;
    cur = b;
    g[k].own_lo = a;
    g[k].own_hi = b;
    g[k].out_lo = parts[k].first;
    g[k].out_hi = parts[k].second;
    if (g[k].out_hi > g[k].out_lo) {
      g[k].need_lo = g[k].out_lo;
      g[k].need_hi = g[k].out_hi - 1 + w;
    } else {
      g[k].need_lo = g[k].need_hi = 0;
    }
  }
  g[n - 1].own_hi = R;
  for (int k = 0; k < n; ++k) {
    // band buffer: row 0 = global row own_lo; own rows then the halo rows
    const int64_t top = g[k].need_hi > g[k].own_hi ? g[k].need_hi : g[k].own_hi;
    g[k].cap_rows = top - g[k].own_lo;
  }
}

static int64_t sharded_ws_bytes(int dtype, int64_t own_rows, int64_t C, int n, bool table) {
  if (!table) return 0;
  const int64_t sat_ws = own_rows > 0 ? sat_workspace_bytes(dtype, own_rows, C, false) : 0;
  const int64_t len = C + 1;
  // [sat workspace][gathered totals: n x len][carry: len], 8-byte elements, 256-byte aligned parts
  auto up = [](int64_t b) { return (b + 255) & ~int64_t(255); };
  return up(sat_ws) + up((int64_t)n * len * 8) + up(len * 8);
}

}  // namespace ssb

using namespace ssb;

namespace {
struct DevScope {  // make a device current, restore the caller's afterwards
  int prev = -1;
  cudaError_t err = cudaSuccess;
  explicit DevScope(int d) {
    if ((err = cudaGetDevice(&prev)) == cudaSuccess && prev != d) err = cudaSetDevice(d);
  }
  ~DevScope() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};
}  // namespace

extern "C" {

int ssb_band_carry(const void* parts, int band, int64_t len, int64_t parts_ld, int is_float, void* carry,
                   void* stream) {
  if (band < 0 || len < 1 || parts_ld < len || !carry || (band > 0 && !parts))
    return shard_fail(SSB_EINVAL, "bad band-carry request");
  int d = 0;
  cudaError_t e = cudaStreamGetDevice(reinterpret_cast<cudaStream_t>(stream), &d);
  if (e != cudaSuccess) return shard_cuda_fail(e, "stream device");
  DevScope ds(d);
  if (ds.err != cudaSuccess) return shard_cuda_fail(ds.err, "cudaSetDevice");
  e = launch_band_carry(parts, band, len, parts_ld, is_float != 0, carry, reinterpret_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? SSB_OK : shard_cuda_fail(e, "ssb_band_carry");
}

int ssb_sharded_plan(int64_t rows, int64_t cols, int64_t w, int ndev, int64_t* plan7) {
  if (rows < 1 || cols < 1 || w < 1 || w > rows || w > cols || ndev < 1 || !plan7)
    return shard_fail(SSB_EINVAL, "bad sharding request (%lldx%lld, w %lld, %d devices)", (long long)rows,
                      (long long)cols, (long long)w, ndev);
  std::vector<BandGeom> g;
  band_plan(rows, w, ndev, g);
  for (int k = 0; k < ndev; ++k) {
    const int64_t v[7] = {g[k].own_lo, g[k].own_hi, g[k].need_lo, g[k].need_hi, g[k].out_lo, g[k].out_hi, g[k].cap_rows};
    for (int j = 0; j < 7; ++j) plan7[7 * k + j] = v[j];
  }
  return SSB_OK;
}

int64_t ssb_sharded_workspace_bytes(int in_dtype, int64_t rows, int64_t cols, int64_t w, int ndev, int band,
                                    int with_table) {
  if (in_dtype < SSB_U8 || in_dtype > SSB_F32 || rows < 1 || cols < 1 || w < 1 || w > rows || w > cols || ndev < 1 ||
      band < 0 || band >= ndev)
    return -1;
  std::vector<BandGeom> g;
  band_plan(rows, w, ndev, g);
  const int64_t b = sharded_ws_bytes(in_dtype, g[band].own_hi - g[band].own_lo, cols, ndev, with_table != 0);
  return b > 0 ? b : 8;
}

int ssb_sharded_swa(int ndev, const int* devs, int in_dtype, int64_t rows, int64_t cols, int64_t w, int stat_mask,
                    void* const* bands, void* const* sats, int64_t sat_ld, void* const* out_sum,
                    double* const* out_mean, double* const* out_std, int64_t out_ld, void* const* ws,
                    const int64_t* ws_bytes, void* const* streams) {
  if (ndev < 1 || !devs || !bands || !streams) return shard_fail(SSB_EINVAL, "bad device list");
  if (in_dtype < SSB_U8 || in_dtype > SSB_F32) return shard_fail(SSB_EUNSUPPORTED, "unsupported element dtype code %d", in_dtype);
  if (rows < 1 || cols < 1) return shard_fail(SSB_EINVAL, "grid dims must be >= 1");
  if (w < 1 || w > rows || w > cols)
    return shard_fail(SSB_EINVAL, "window size %lld exceeds grid dims %lldx%lld; windows must fit fully inside the grid",
                      (long long)w, (long long)rows, (long long)cols);
  if (w > ssb_window_fused_max_w())
    return shard_fail(SSB_EUNSUPPORTED, "sharded windows support w <= %lld", (long long)ssb_window_fused_max_w());
  if (stat_mask & ~(SSB_SUM | SSB_MEAN | SSB_STD)) return shard_fail(SSB_EINVAL, "bad stat mask %d", stat_mask);
  if (in_dtype == SSB_I32 && (stat_mask & SSB_STD))
    return shard_fail(SSB_EUNSUPPORTED, "std is not supported for int32 input (squared sums exceed 64 bits)");
  const bool table = sats != nullptr;
  if (!table && stat_mask == 0) return shard_fail(SSB_EINVAL, "nothing to compute");
  if (table && (sat_ld < cols + 1 || (sat_ld & 3))) return shard_fail(SSB_EINVAL, "sat_ld must be a multiple of 4 and >= cols+1");
  if (out_ld < cols - w + 1) return shard_fail(SSB_EINVAL, "out_ld < output cols");
  std::vector<BandGeom> g;
  band_plan(rows, w, ndev, g);
  const int es = in_dtype == SSB_U8 ? 1 : in_dtype == SSB_U16 ? 2 : 4;
  const int64_t len = cols + 1;
  const bool is_float = in_dtype == SSB_F32;
  for (int k = 0; k < ndev; ++k) {
    if (!bands[k] && g[k].cap_rows > 0) return shard_fail(SSB_EINVAL, "band %d has no buffer", k);
    if (reinterpret_cast<uintptr_t>(bands[k]) & 15) return shard_fail(SSB_EINVAL, "band %d must be 16-byte aligned", k);
    if (g[k].out_hi > g[k].out_lo) {
      if (((stat_mask & SSB_SUM) && !(out_sum && out_sum[k])) || ((stat_mask & SSB_MEAN) && !(out_mean && out_mean[k])) ||
          ((stat_mask & SSB_STD) && !(out_std && out_std[k])))
        return shard_fail(SSB_EINVAL, "missing output buffer for band %d", k);
    }
    if (table) {
      if (!sats[k] || (reinterpret_cast<uintptr_t>(sats[k]) & 31)) return shard_fail(SSB_EINVAL, "band %d table must be 32-byte aligned", k);
      const int64_t need = sharded_ws_bytes(in_dtype, g[k].own_hi - g[k].own_lo, cols, ndev, true);
      if (!ws || !ws[k] || !ws_bytes || ws_bytes[k] < need)
        return shard_fail(SSB_EINVAL, "band %d workspace too small: need %lld bytes", k, (long long)need);
    }
  }
  auto S = [&](int k) { return reinterpret_cast<cudaStream_t>(streams[k]); };
  auto band_row = [&](int k, int64_t global_row) {
    return reinterpret_cast<char*>(bands[k]) + (size_t)(global_row - g[k].own_lo) * cols * es;
  };
  auto up = [](int64_t b) { return (b + 255) & ~int64_t(255); };
  auto gathered = [&](int k) {
    const int64_t sat_ws = g[k].own_hi > g[k].own_lo ? sat_workspace_bytes(in_dtype, g[k].own_hi - g[k].own_lo, cols, false) : 0;
    return reinterpret_cast<char*>(ws[k]) + up(sat_ws);
  };
  auto carry_of = [&](int k) { return gathered(k) + up((int64_t)ndev * len * 8); };

  int prev = 0;
  cudaError_t e = cudaGetDevice(&prev);
  if (e != cudaSuccess) return shard_cuda_fail(e, "cudaGetDevice");
  if (census_sink().trow || census_sink().orow)  // bands write band-local rows
    return shard_fail(SSB_EUNSUPPORTED, "the write census covers single-device entry points only");
  std::vector<cudaEvent_t> ev_in(ndev, nullptr), ev_tot(ndev, nullptr), ev_done(ndev, nullptr);
  int status = SSB_OK;
  auto cf = [&](cudaError_t ce, const char* where) {
    if (ce != cudaSuccess && status == SSB_OK) status = shard_cuda_fail(ce, where);
    return ce == cudaSuccess && status == SSB_OK;
  };
  // 1. events on each device; "own rows ready" = everything the caller queued so far
  for (int k = 0; k < ndev && status == SSB_OK; ++k) {
    if (!cf(cudaSetDevice(devs[k]), "cudaSetDevice")) break;
    if (!cf(cudaEventCreateWithFlags(&ev_in[k], cudaEventDisableTiming), "event") ||
        !cf(cudaEventCreateWithFlags(&ev_tot[k], cudaEventDisableTiming), "event") ||
        !cf(cudaEventCreateWithFlags(&ev_done[k], cudaEventDisableTiming), "event"))
      break;
    cf(cudaEventRecord(ev_in[k], S(k)), "event record");
  }
  // 2. windows on a side stream forked per device (they do not wait for the
  //    table's phases): halo rows from the following devices by peer copies,
  //    then this band's output rows by the fused window kernel
  std::vector<SideHandle> side(ndev);
  for (int k = 0; k < ndev && status == SSB_OK; ++k) {
    if (!cf(cudaSetDevice(devs[k]), "cudaSetDevice")) break;
    if (!cf(side_fork(S(k), &side[k]), "side stream")) break;
    if (g[k].out_hi <= g[k].out_lo) continue;
    for (int j = 0; j < ndev && status == SSB_OK; ++j) {
      if (j == k) continue;
      const int64_t lo = g[j].own_lo > g[k].need_lo ? g[j].own_lo : g[k].need_lo;
      const int64_t hi = g[j].own_hi < g[k].need_hi ? g[j].own_hi : g[k].need_hi;
      if (hi <= lo) continue;
      if (!cf(cudaStreamWaitEvent(side[k].s, ev_in[j], 0), "wait")) break;
      cf(cudaMemcpyPeerAsync(band_row(k, lo), devs[k], band_row(j, lo), devs[j], (size_t)(hi - lo) * cols * es,
                             side[k].s),
         "halo peer copy");
    }
    if (stat_mask == 0 || status != SSB_OK) continue;
    WinOut o{out_sum ? out_sum[k] : nullptr, out_mean ? out_mean[k] : nullptr, out_std ? out_std[k] : nullptr, out_ld};
    cf(launch_window_fused(band_row(k, g[k].need_lo), in_dtype, g[k].need_hi - g[k].need_lo, cols, cols, w, stat_mask,
                           o, nullptr, 0, side[k].s),
       "sharded windows");
  }
  // 3. table phase 1 on the caller's streams: band column totals into this
  //    device's slot of its gather buffer
  for (int k = 0; table && k < ndev && status == SSB_OK; ++k) {
    if (!cf(cudaSetDevice(devs[k]), "cudaSetDevice")) break;
    char* mine = gathered(k) + (size_t)k * len * 8;
    const int64_t nown = g[k].own_hi - g[k].own_lo;
    if (nown > 0)
      cf(launch_sat_prepare(in_dtype, bands[k], nown, cols, cols, false, ws[k], mine, nullptr, nullptr, S(k)), "ssb_sat_prepare");
    else
      cf(cudaMemsetAsync(mine, 0, len * 8, S(k)), "memset");
    cf(cudaEventRecord(ev_tot[k], S(k)), "event record");
  }
  // 4. table phase 2: gather the totals of the bands above, exclusive scan, write with the carry
  for (int k = 0; table && k < ndev && status == SSB_OK; ++k) {
    if (!cf(cudaSetDevice(devs[k]), "cudaSetDevice")) break;
    for (int j = 0; j < k && status == SSB_OK; ++j) {
      if (!cf(cudaStreamWaitEvent(S(k), ev_tot[j], 0), "wait")) break;
      cf(cudaMemcpyPeerAsync(gathered(k) + (size_t)j * len * 8, devs[k], gathered(j) + (size_t)j * len * 8, devs[j],
                             (size_t)len * 8, S(k)),
         "totals peer copy");
    }
    if (status != SSB_OK) break;
    const void* carry = nullptr;
    if (k > 0) {
      cf(launch_band_carry(gathered(k), k, len, len, is_float, carry_of(k), S(k)), "band carry");
      carry = carry_of(k);
    }
    const int64_t nown = g[k].own_hi - g[k].own_lo;
    if (nown > 0) {
      cf(launch_sat_finish(in_dtype, bands[k], nown, cols, cols, sats[k], nullptr, sat_ld, carry, nullptr, ws[k], S(k)),
         "ssb_sat_finish");
    } else if (carry) {  // an empty band's table is its carry row
      cf(cudaMemcpyAsync(sats[k], carry, (size_t)len * 8, cudaMemcpyDeviceToDevice, S(k)), "carry row");
    } else {
      cf(cudaMemsetAsync(sats[k], 0, (size_t)len * 8, S(k)), "carry row");
    }
  }
  // 5. join: the side streams back into the callers' streams, then no stream
  //    finishes before the peer copies that read its band (or its totals) have
  //    run, so the caller may reuse every buffer in stream order
  for (int k = 0; k < ndev; ++k) {
    if (!ev_done[k]) continue;
    cudaSetDevice(devs[k]);
    if (side[k].s) cf(side_join(S(k), side[k]), "side join");
    cf(cudaEventRecord(ev_done[k], S(k)), "event record");
  }
  for (int k = 0; k < ndev; ++k) {
    if (!ev_done[k]) continue;
    cudaSetDevice(devs[k]);
    for (int j = 0; j < ndev; ++j)
      if (j != k && ev_done[j]) cf(cudaStreamWaitEvent(S(k), ev_done[j], 0), "join");
  }
  for (int k = 0; k < ndev; ++k) {
    if (ev_in[k] || ev_tot[k] || ev_done[k]) cudaSetDevice(devs[k]);
    if (ev_in[k]) cudaEventDestroy(ev_in[k]);
    if (ev_tot[k]) cudaEventDestroy(ev_tot[k]);
    if (ev_done[k]) cudaEventDestroy(ev_done[k]);
  }
  cudaSetDevice(prev);
  return status;
}

}  // extern "C"
