// satsweep-b200: device self-tests of arithmetic identities the kernels rely on.
//
// ssb_selftest_division: the finalisation divides window sums by n = w*w
// (stats.py:55-74) with div_n (ssb_common.cuh): a multiply by RN(1/n) and one
// FMA correction instead of the iterative IEEE division.  This kernel checks,
// bit for bit, div_n(x, n, RN(1/n)) == __ddiv_rn(x, n) over caller-supplied x.
#include "ssb_common.cuh"
#include "../../include/satsweep_b200.h"

namespace ssb {
void note_launch(int n);
int shard_fail(int code, const char* fmt, ...);
int shard_cuda_fail(cudaError_t e, const char* where);

__global__ void __launch_bounds__(kThreads) division_check_kernel(const double* __restrict__ x, int64_t n, double d,
                                                                   double inv, unsigned long long* __restrict__ bad) {
  unsigned long long local = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double a = div_n(x[i], d, inv);
    const double b = __ddiv_rn(x[i], d);
    local += __double_as_longlong(a) != __double_as_longlong(b);
  }
  local = warp_sum(local);
  if ((threadIdx.x & 31) == 0 && local) atomicAdd(bad, local);
}
}  // namespace ssb

extern "C" int ssb_selftest_division(const double* x, int64_t n, double divisor, unsigned long long* mismatches,
                                     void* stream) {
  using namespace ssb;
  if (!x || n < 1 || !mismatches || !(divisor > 0.0)) return shard_fail(SSB_EINVAL, "bad self-test request");
  const int blocks = (int)((n + kThreads - 1) / kThreads < 4 * kNumSMs ? (n + kThreads - 1) / kThreads : 4 * kNumSMs);
  division_check_kernel<<<blocks, kThreads, 0, reinterpret_cast<cudaStream_t>(stream)>>>(x, n, divisor,
                                                                                        1.0 / divisor, mismatches);
  note_launch(1);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? SSB_OK : shard_cuda_fail(e, "ssb_selftest_division");
}
