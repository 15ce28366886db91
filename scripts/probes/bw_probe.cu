// HBM ceilings by access mix on this B200: write-only, read-only, copy (1:1),
// and a 1:8 read:write mix (the C5 step's shape: 1 B/px read, 8+8 B/px write).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o bw_probe bw_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void wr(uint4* p, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    __stcs(p + i, make_uint4(i, 1, 2, 3));
}
__global__ void rd(const uint4* p, size_t n, unsigned* sink) {
  unsigned acc = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    uint4 v = __ldcs(p + i);
    acc ^= v.x ^ v.y ^ v.z ^ v.w;
  }
  if (acc == 0x12345678u) *sink = acc;
}
__global__ void cp(const uint4* a, uint4* b, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    __stcs(b + i, __ldcs(a + i));
}
// read 1 uint4, write 8 uint4 (to a buffer 8x larger)
__global__ void mix18(const uint4* a, uint4* b, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    uint4 v = __ldcs(a + i);
    const size_t base = (i / 32) * 256 + (i % 32);
#pragma unroll
    for (int k = 0; k < 8; ++k) __stcs(b + base + 32 * k, v);
  }
}

int main() {
  const size_t bytes = (size_t)48 << 30;
  uint4 *a, *b;
  unsigned* sink;
  cudaMalloc(&a, bytes / 8 + 4096);
  cudaMalloc(&b, bytes + 4096);
  cudaMalloc(&sink, 4);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  int blocks = 148 * 8, th = 256;
  auto run = [&](const char* name, double gb, auto fn) {
    for (int i = 0; i < 2; ++i) fn();
    cudaEventRecord(e0);
    for (int i = 0; i < 5; ++i) fn();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    ms /= 5;
    printf("{\"probe\": \"%s\", \"GB\": %.2f, \"ms\": %.3f, \"GBs\": %.1f}\n", name, gb, ms, gb / (ms * 1e-3));
  };
  const size_t n = bytes / 16;
  run("write_only", bytes / 1e9, [&] { wr<<<blocks, th>>>(b, n); });
  run("read_only", bytes / 1e9, [&] { rd<<<blocks, th>>>(b, n, sink); });
  run("copy_1to1", bytes / 1e9, [&] { cp<<<blocks, th>>>(b, b + n / 2, n / 2); });
  run("read1_write8", (bytes / 8 + bytes) / 1e9, [&] { mix18<<<blocks, th>>>(a, b, n / 8); });
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) printf("error %s\n", cudaGetErrorString(e));
  return 0;
}
