// HBM write ceilings, part 3 (tuning probe): the fused window kernel's output
// pattern at C5 (69,745 x 84,745 u64, ld 84,745; warps own 1,793-output strips
// x row segments, 4 warps per CTA in strip-major tile order) with 16-byte vs
// 32-byte lane stores, and segment counts 42 / 85 / 170 / 340.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o wr_probe3 wr_probe3.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void win_wr(uint64_t* out, int64_t OR, int64_t OC, int two, int nJ, int nK, int64_t sro, int mode) {
  const int lane = threadIdx.x & 31;
  const int t = blockIdx.x * 4 + (threadIdx.x >> 5);
  if (t >= nJ * nK) return;
  const int J = t % nJ, K = t / nJ;
  const int64_t oc0 = (int64_t)J * two;
  const int nout = (int)(OC - oc0 < two ? OC - oc0 : two);
  const int64_t r0 = (int64_t)K * sro, r1 = r0 + sro < OR ? r0 + sro : OR;
  uint64_t v = t;
  for (int64_t i = r0; i < r1; ++i) {
    uint64_t* row = out + i * OC + oc0;
    const int d = (int)((reinterpret_cast<uintptr_t>(row) >> 3) & 1);
    v += 7;
    if (mode == 0 || mode == 3 || mode == 4) {  // 16-byte pairs, lane-consecutive
      for (int j = d + 2 * lane; j + 1 < nout; j += 64) {
        uint64_t* p = row + j;
        if (mode == 0) { ulonglong2 q; q.x = v; q.y = v + 1; __stcs(reinterpret_cast<ulonglong2*>(p), q); }
        else if (mode == 3) asm volatile("st.global.L1::no_allocate.v2.u64 [%0], {%1, %2};" ::"l"(p), "l"(v), "l"(v) : "memory");
        else asm volatile("st.global.v2.u64 [%0], {%1, %2};" ::"l"(p), "l"(v), "l"(v) : "memory");
      }
    } else if (mode == 1 || mode == 5) {  // 8-byte, lane-consecutive
      for (int j = lane; j < nout; j += 32) {
        if (mode == 1) __stcs(reinterpret_cast<unsigned long long*>(row + j), (unsigned long long)v);
        else row[j] = v;
      }
    } else {  // 32-byte (4 outputs) per lane where 32-byte aligned
      const int d4 = (int)((4 - ((reinterpret_cast<uintptr_t>(row) >> 3) & 3)) & 3);
      for (int j = d4 + 4 * lane; j + 3 < nout; j += 128) {
        uint64_t* p = row + j;
        if (mode == 2) asm volatile("st.global.L1::no_allocate.v4.b64 [%0], {%1, %2, %3, %4};" ::"l"(p), "l"(v), "l"(v), "l"(v), "l"(v) : "memory");
        else if (mode == 6) asm volatile("st.global.cs.v4.b64 [%0], {%1, %2, %3, %4};" ::"l"(p), "l"(v), "l"(v), "l"(v), "l"(v) : "memory");
        else asm volatile("st.global.v4.b64 [%0], {%1, %2, %3, %4};" ::"l"(p), "l"(v), "l"(v), "l"(v), "l"(v) : "memory");
      }
    }
  }
}

int main() {
  const int64_t OR = 69745, OC = 84745;
  uint64_t* out;
  cudaMalloc(&out, (size_t)OR * OC * 8 + 4096);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int two = 1793, nJ = (int)((OC + two - 1) / two);
  const double gb = (double)OR * OC * 8 / 1e9;
  for (int mode = 0; mode < 8; ++mode)
    for (int nK : {85, 1360}) {
      const int64_t sro = (OR + nK - 1) / nK;
      const int blocks = (nJ * nK + 3) / 4;
      auto fn = [&] { win_wr<<<blocks, 128>>>(out, OR, OC, two, nJ, nK, sro, mode); };
      for (int i = 0; i < 2; ++i) fn();
      cudaEventRecord(e0);
      for (int i = 0; i < 5; ++i) fn();
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      ms /= 5;
      printf("{\"probe\": \"win_wr\", \"mode\": %d, \"nK\": %d, \"GB\": %.2f, \"ms\": %.3f, \"GBs\": %.1f, \"err\": \"%s\"}\n",
             mode, nK, gb, ms, gb / (ms * 1e-3), cudaGetErrorString(cudaGetLastError()));
      fflush(stdout);
    }
  return 0;
}
