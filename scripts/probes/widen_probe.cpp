// Host-side u32 -> u64 widening copy bandwidth (tuning probe for the e2e wire format):
// T threads, each widening a contiguous slice of a pinned-like buffer with AVX2 + streaming stores.
// g++ -O3 -pthread -o widen_probe widen_probe.cpp
#include <immintrin.h>
#include <sys/mman.h>

#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>

__attribute__((target("avx2"))) static void widen_avx2(const uint32_t* s, uint64_t* d, size_t n, bool nt) {
  size_t i = 0;
  for (; i < n && (reinterpret_cast<uintptr_t>(d + i) & 31); ++i) d[i] = s[i];
  if (nt) {
    for (; i + 8 <= n; i += 8) {
      const __m128i a = _mm_loadu_si128(reinterpret_cast<const __m128i*>(s + i));
      const __m128i b = _mm_loadu_si128(reinterpret_cast<const __m128i*>(s + i + 4));
      _mm256_stream_si256(reinterpret_cast<__m256i*>(d + i), _mm256_cvtepu32_epi64(a));
      _mm256_stream_si256(reinterpret_cast<__m256i*>(d + i + 4), _mm256_cvtepu32_epi64(b));
    }
    _mm_sfence();
  } else {
    for (; i + 8 <= n; i += 8) {
      const __m128i a = _mm_loadu_si128(reinterpret_cast<const __m128i*>(s + i));
      const __m128i b = _mm_loadu_si128(reinterpret_cast<const __m128i*>(s + i + 4));
      _mm256_storeu_si256(reinterpret_cast<__m256i*>(d + i), _mm256_cvtepu32_epi64(a));
      _mm256_storeu_si256(reinterpret_cast<__m256i*>(d + i + 4), _mm256_cvtepu32_epi64(b));
    }
  }
  for (; i < n; ++i) d[i] = s[i];
}

int main(int argc, char** argv) {
  const size_t n = (size_t)(argc > 1 ? atof(argv[1]) : 1e9);  // elements
  uint32_t* src = static_cast<uint32_t*>(mmap(nullptr, n * 4, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0));
  uint64_t* dst = static_cast<uint64_t*>(mmap(nullptr, n * 8, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0));
  const int hw = (int)std::thread::hardware_concurrency();
  {  // first touch in parallel
    std::vector<std::thread> th;
    for (int t = 0; t < hw; ++t)
      th.emplace_back([=] {
        const size_t a = n * t / hw, b = n * (t + 1) / hw;
        for (size_t i = a; i < b; ++i) src[i] = (uint32_t)i;
        memset(dst + a, 0, (b - a) * 8);
      });
    for (auto& x : th) x.join();
  }
  for (int nt = 1; nt >= 0; --nt)
    for (int T : {1, 2, 4, 8, 12, 16, 32}) {
      if (T > 2 * hw) continue;
      double best = 1e9;
      for (int rep = 0; rep < 3; ++rep) {
        const auto t0 = std::chrono::steady_clock::now();
        std::vector<std::thread> th;
        for (int t = 0; t < T; ++t)
          th.emplace_back([=] { const size_t a = n * t / T, b = n * (t + 1) / T; widen_avx2(src + a, dst + a, b - a, nt); });
        for (auto& x : th) x.join();
        const double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        if (s < best) best = s;
      }
      printf("{\"probe\": \"widen\", \"nt_stores\": %d, \"threads\": %d, \"elems\": %zu, \"s\": %.4f, \"out_GBs\": %.1f, \"Gelem_s\": %.2f}\n", nt, T, n,
             best, n * 8 / best / 1e9, n / best / 1e9);
      fflush(stdout);
    }
  uint64_t chk = 0;
  for (size_t i = 0; i < n; i += n / 1000 + 1) chk += dst[i] - i;
  printf("check %llu\n", (unsigned long long)chk);
  return 0;
}
