// satsweep-b200: host half of ssb_swa_host's narrow wire format.
//
// When every window sum provably fits 32 bits (w^2 * max pixel < 2^32), the
// device narrows the uint64 sums to uint32 -- or, for a band whose largest sum
// fits 16 bits, to uint16 -- before the device->host copy (the result copy is
// the end-to-end critical path), and the library's host threads widen each
// landed chunk into the caller's uint64 array (api.py:28-55 returns uint64).  This file is only that widening copy:
// zero-extension with streaming stores, no arithmetic of the path runs here.
#include <immintrin.h>

#include <cstddef>
#include <cstdint>

namespace ssb {

namespace {
__attribute__((target("avx2"))) void widen_avx2(const uint32_t* s, uint64_t* d, size_t n) {
  size_t i = 0;
  for (; i < n && (reinterpret_cast<uintptr_t>(d + i) & 31); ++i) d[i] = s[i];
  for (; i + 8 <= n; i += 8) {
    const __m128i a = _mm_loadu_si128(reinterpret_cast<const __m128i*>(s + i));
    const __m128i b = _mm_loadu_si128(reinterpret_cast<const __m128i*>(s + i + 4));
    _mm256_stream_si256(reinterpret_cast<__m256i*>(d + i), _mm256_cvtepu32_epi64(a));
    _mm256_stream_si256(reinterpret_cast<__m256i*>(d + i + 4), _mm256_cvtepu32_epi64(b));
  }
  _mm_sfence();
  for (; i < n; ++i) d[i] = s[i];
}

__attribute__((target("avx2"))) void widen16_avx2(const uint16_t* s, uint64_t* d, size_t n) {
  size_t i = 0;
  for (; i < n && (reinterpret_cast<uintptr_t>(d + i) & 31); ++i) d[i] = s[i];
  for (; i + 8 <= n; i += 8) {
    const __m128i a = _mm_loadu_si128(reinterpret_cast<const __m128i*>(s + i));  // 8 x uint16
    _mm256_stream_si256(reinterpret_cast<__m256i*>(d + i), _mm256_cvtepu16_epi64(a));
    _mm256_stream_si256(reinterpret_cast<__m256i*>(d + i + 4), _mm256_cvtepu16_epi64(_mm_srli_si128(a, 8)));
  }
  _mm_sfence();
  for (; i < n; ++i) d[i] = s[i];
}

__attribute__((target("avx2"))) void copy64_avx2(const uint64_t* s, uint64_t* d, size_t n) {
  size_t i = 0;
  for (; i < n && (reinterpret_cast<uintptr_t>(d + i) & 31); ++i) d[i] = s[i];
  for (; i + 8 <= n; i += 8) {
    const __m256i a = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(s + i));
    const __m256i b = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(s + i + 4));
    _mm256_stream_si256(reinterpret_cast<__m256i*>(d + i), a);
    _mm256_stream_si256(reinterpret_cast<__m256i*>(d + i + 4), b);
  }
  _mm_sfence();
  for (; i < n; ++i) d[i] = s[i];
}

template <typename T>
void widen_plain(const T* s, uint64_t* d, size_t n) {
  for (size_t i = 0; i < n; ++i) d[i] = s[i];
}
}  // namespace

// dst[i] = src[i] for i < n (zero-extended); dst only 8-byte aligned
void widen_u32_to_u64(const uint32_t* src, uint64_t* dst, size_t n) {
  static const bool avx2 = __builtin_cpu_supports("avx2");
  if (avx2) widen_avx2(src, dst, n);
  else widen_plain(src, dst, n);
}

void widen_u16_to_u64(const uint16_t* src, uint64_t* dst, size_t n) {
  static const bool avx2 = __builtin_cpu_supports("avx2");
  if (avx2) widen16_avx2(src, dst, n);
  else widen_plain(src, dst, n);
}

}  // namespace ssb

// 8-byte results (float64 mean / std, wide sums) from the pinned ring into pageable memory
namespace ssb {
void copy_u64_stream(const uint64_t* src, uint64_t* dst, size_t n) {
  static const bool avx2 = __builtin_cpu_supports("avx2");
  if (avx2) copy64_avx2(src, dst, n);
  else widen_plain(src, dst, n);
}
}  // namespace ssb
