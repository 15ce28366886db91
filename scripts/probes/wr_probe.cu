// HBM write ceilings by store flavour on this B200 (tuning probe, not product):
// is the 6.13 TB/s write-only figure of bw_probe.cu a property of the DRAM or
// of 16-byte grid-stride streaming stores?  Variants: 16-byte .cs / plain /
// 256-bit stores, grid-stride vs blocked ownership, occupancy, TMA bulk stores
// (cp.async.bulk.global.shared::cta) from shared memory, cudaMemsetAsync, and
// the 1:16 read:write mix of the C5 step with the best flavour.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o wr_probe wr_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ void st256(void* p, uint64_t a, uint64_t b, uint64_t c, uint64_t d) {
  asm volatile("st.global.L1::no_allocate.v4.b64 [%0], {%1, %2, %3, %4};" ::"l"(p), "l"(a), "l"(b), "l"(c), "l"(d)
               : "memory");
}
__device__ __forceinline__ void st256cs(void* p, uint64_t a, uint64_t b, uint64_t c, uint64_t d) {
  asm volatile("st.global.cs.v4.b64 [%0], {%1, %2, %3, %4};" ::"l"(p), "l"(a), "l"(b), "l"(c), "l"(d) : "memory");
}

__global__ void wr16cs(uint4* p, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    __stcs(p + i, make_uint4(i, 1, 2, 3));
}
__global__ void wr16(uint4* p, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    p[i] = make_uint4(i, 1, 2, 3);
}
// n in 32-byte units
__global__ void wr32(char* p, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    st256(p + 32 * i, i, 1, 2, 3);
}
__global__ void wr32cs(char* p, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    st256cs(p + 32 * i, i, 1, 2, 3);
}
// blocked: each warp owns a contiguous chunk of `chunk` 32-byte units
__global__ void wr32blk(char* p, size_t n, size_t chunk) {
  const size_t gw = (blockIdx.x * (size_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const size_t nw = ((size_t)gridDim.x * blockDim.x) >> 5;
  for (size_t c = gw; c * chunk < n; c += nw) {
    const size_t b = c * chunk, e = b + chunk < n ? b + chunk : n;
    for (size_t i = b + lane; i < e; i += 32) st256(p + 32 * i, i, 1, 2, 3);
  }
}
// 8-byte stores (the window kernels' output width)
__global__ void wr8(uint64_t* p, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    __stcs(p + i, (uint64_t)i);
}
// TMA bulk store: each CTA fills a smem tile once, then streams it out in
// `tile` byte bulk copies, keeping up to 8 groups in flight
template <int TILE>
__global__ void wrtma(char* p, size_t bytes) {
  extern __shared__ __align__(128) unsigned char sm[];
  for (int i = threadIdx.x; i < TILE / 16; i += blockDim.x) reinterpret_cast<uint4*>(sm)[i] = make_uint4(i, 1, 2, 3);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  if (threadIdx.x != 0) return;
  const size_t ntiles = bytes / TILE;
  const uint32_t s = (uint32_t)__cvta_generic_to_shared(sm);
  int k = 0;
  for (size_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(p + t * TILE), "r"(s), "n"(TILE)
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    if (++k >= 8) asm volatile("cp.async.bulk.wait_group.read 7;" ::: "memory");
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}
// C5 mix: read 1 x 16 B, write 16 x 16 B, 256-bit stores
__global__ void mix116(const uint4* a, char* b, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    uint4 v = __ldcs(a + i);
    const size_t base = (i / 32) * 256 + (i % 32);  // 32-byte units
#pragma unroll
    for (int k = 0; k < 8; ++k) st256(b + 32 * (base + 32 * k), v.x, v.y, v.z, k);
  }
}

int main() {
  const size_t bytes = (size_t)48 << 30;
  char *a, *b;
  cudaMalloc(&a, bytes / 16 + 4096);
  cudaMalloc(&b, bytes + 4096);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto run = [&](const char* name, int cfg, double gb, auto fn) {
    for (int i = 0; i < 2; ++i) fn();
    cudaEventRecord(e0);
    for (int i = 0; i < 5; ++i) fn();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    ms /= 5;
    cudaError_t e = cudaGetLastError();
    printf("{\"probe\": \"%s\", \"cfg\": %d, \"GB\": %.2f, \"ms\": %.3f, \"GBs\": %.1f, \"err\": \"%s\"}\n", name, cfg, gb,
           ms, gb / (ms * 1e-3), cudaGetErrorString(e));
    fflush(stdout);
  };
  const double gb = bytes / 1e9;
  for (int occ : {4, 8, 16}) {
    int blocks = 148 * occ, th = 256;
    run("wr16cs", occ, gb, [&] { wr16cs<<<blocks, th>>>((uint4*)b, bytes / 16); });
    run("wr16", occ, gb, [&] { wr16<<<blocks, th>>>((uint4*)b, bytes / 16); });
    run("wr32", occ, gb, [&] { wr32<<<blocks, th>>>(b, bytes / 32); });
    run("wr32cs", occ, gb, [&] { wr32cs<<<blocks, th>>>(b, bytes / 32); });
    run("wr8", occ, gb, [&] { wr8<<<blocks, th>>>((uint64_t*)b, bytes / 8); });
  }
  for (size_t chunk : {128, 1024, 8192})
    run("wr32blk", (int)chunk, gb, [&] { wr32blk<<<148 * 8, 256>>>(b, bytes / 32, chunk); });
  cudaFuncSetAttribute(wrtma<16384>, cudaFuncAttributeMaxDynamicSharedMemorySize, 16384);
  cudaFuncSetAttribute(wrtma<32768>, cudaFuncAttributeMaxDynamicSharedMemorySize, 32768);
  for (int occ : {1, 2, 4, 8}) {
    run("tma16k", occ, gb, [&] { wrtma<16384><<<148 * occ, 32, 16384>>>(b, bytes); });
    run("tma32k", occ, gb, [&] { wrtma<32768><<<148 * occ, 32, 32768>>>(b, bytes); });
  }
  run("memset", 0, gb, [&] { cudaMemsetAsync(b, 1, bytes); });
  run("mix116_wr32", 8, (bytes / 16 + bytes) / 1e9, [&] { mix116<<<148 * 8, 256>>>((const uint4*)a, b, bytes / 256); });
  return 0;
}
