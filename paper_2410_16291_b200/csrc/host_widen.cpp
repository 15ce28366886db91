// satsweep-b200: host half of ssb_swa_host's narrow wire format.
//
// When every window sum provably fits 32 bits (w^2 * max pixel < 2^32), the
// device narrows the uint64 sums to uint32 before the device->host copy (half
// the PCIe bytes; the result copy is the end-to-end critical path), and the
// library's host threads widen each landed band into the caller's uint64
// array (api.py:28-55 returns uint64).  This file is only that widening copy:
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

void widen_plain(const uint32_t* s, uint64_t* d, size_t n) {
  for (size_t i = 0; i < n; ++i) d[i] = s[i];
}
}  // namespace

// dst[i] = src[i] for i < n (zero-extended); dst only 8-byte aligned
void widen_u32_to_u64(const uint32_t* src, uint64_t* dst, size_t n) {
  static const bool avx2 = __builtin_cpu_supports("avx2");
  if (avx2) widen_avx2(src, dst, n);
  else widen_plain(src, dst, n);
}

}  // namespace ssb
