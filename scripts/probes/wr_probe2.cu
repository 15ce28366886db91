// HBM write ceilings, part 2 (tuning probe): which write *patterns* reach the
// 6.9-7.4 TB/s that wr_probe.cu saw for wr32 at 16 CTAs/SM and memset, vs the
// 6.0-6.3 TB/s of the same stores at 4-8 CTAs/SM?  Grid-stride 256-bit stores
// over a sweep of grid sizes / block sizes, and the C5 table's own tile
// pattern (warp = 512 table columns x SR rows, 8-byte elements, pitch 85,004)
// with lane-strided (lane owns 128 B) vs lane-contiguous (32 B per lane per
// instruction) row stores, CTAs over adjacent strips vs adjacent segments.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o wr_probe2 wr_probe2.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ void st256(void* p, uint64_t a, uint64_t b, uint64_t c, uint64_t d) {
  asm volatile("st.global.L1::no_allocate.v4.b64 [%0], {%1, %2, %3, %4};" ::"l"(p), "l"(a), "l"(b), "l"(c), "l"(d)
               : "memory");
}
__global__ void wr32(char* p, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    st256(p + 32 * i, i, 1, 2, 3);
}
// table tiles: PR rows x PC cols (8 B), strips of 512 cols, segments of SR rows.
// mode bit0: lane-contiguous stores; bit1: warps of a CTA over adjacent segments
// (else adjacent strips).  One warp per tile, grid covers all tiles.
__global__ void tile_wr(uint64_t* t, int64_t PR, int64_t PC, int64_t ld, int SR, int nJ, int nK, int mode) {
  const int wpc = blockDim.x >> 5;
  const int lane = threadIdx.x & 31;
  const int64_t tw = (int64_t)blockIdx.x * wpc + (threadIdx.x >> 5);
  int J, K;
  if (mode & 2) {  // CTA = wpc adjacent segments of one strip
    const int64_t grp = tw / wpc;
    J = (int)(grp % nJ);
    K = (int)((grp / nJ) * wpc + (tw % wpc));
  } else {
    J = (int)(tw % nJ);
    K = (int)(tw / nJ);
  }
  if (K >= nK) return;
  const int64_t r0 = (int64_t)K * SR, r1 = r0 + SR < PR ? r0 + SR : PR;
  const int64_t c0 = (int64_t)J * 512;
  if (c0 + 512 > ld) return;
  uint64_t v = tw;
  for (int64_t r = r0; r < r1; ++r) {
    uint64_t* row = t + r * ld + c0;
    v += 3;
    if (mode & 1) {
#pragma unroll
      for (int k = 0; k < 4; ++k) st256(row + 4 * (lane + 32 * k), v, v + 1, v + 2, v + 3);
    } else {
#pragma unroll
      for (int k = 0; k < 4; ++k) st256(row + 16 * lane + 4 * k, v, v + 1, v + 2, v + 3);
    }
  }
}

int main() {
  const size_t bytes = (size_t)48 << 30;
  char* b;
  cudaMalloc(&b, bytes + 4096);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto run = [&](const char* name, int c1, int c2, double gb, auto fn) {
    for (int i = 0; i < 2; ++i) fn();
    cudaEventRecord(e0);
    for (int i = 0; i < 5; ++i) fn();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    ms /= 5;
    cudaError_t e = cudaGetLastError();
    printf("{\"probe\": \"%s\", \"a\": %d, \"b\": %d, \"GB\": %.2f, \"ms\": %.3f, \"GBs\": %.1f, \"err\": \"%s\"}\n", name,
           c1, c2, gb, ms, gb / (ms * 1e-3), cudaGetErrorString(e));
    fflush(stdout);
  };
  const double gb = bytes / 1e9;
  for (int th : {128, 256, 512, 1024})
    for (int occ : {8, 16, 32, 64, 256}) {
      const int blocks = 148 * occ * 256 / th;
      run("wr32", th, occ, gb, [&] { wr32<<<blocks, th>>>(b, bytes / 32); });
    }
  run("memset0", 0, 0, gb, [&] { cudaMemsetAsync(b, 0, bytes); });
  run("memset1", 1, 0, gb, [&] { cudaMemsetAsync(b, 1, bytes); });
  // C5 table geometry: 70,001 x 85,001 (pitch 85,004), 47.6 GB
  const int64_t PR = 70001, PC = 85001, ld = 85004;
  const int nJ = (int)(PC / 512);  // full strips only
  const double tgb = (double)PR * nJ * 512 * 8 / 1e9;
  for (int SR : {128, 512, 2048})
    for (int mode = 0; mode < 4; ++mode)
      for (int wpc : {4, 8}) {
        const int nK = (int)((PR + SR - 1) / SR);
        const int64_t tiles = (int64_t)nJ * nK;
        const int blocks = (int)((tiles + wpc - 1) / wpc);
        run(mode & 2 ? (mode & 1 ? "tile_seg_contig" : "tile_seg_strided") : (mode & 1 ? "tile_strip_contig" : "tile_strip_strided"),
            SR, wpc, tgb, [&] { tile_wr<<<blocks, 32 * wpc>>>((uint64_t*)b, PR, PC, ld, SR, nJ, nK, mode); });
      }
  return 0;
}
