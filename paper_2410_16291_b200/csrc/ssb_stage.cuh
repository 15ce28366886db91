// satsweep-b200: TMA row staging shared by the table build and the fused path.
//
// A warp stages up to 32 raster rows (lane q -> row q) into shared memory with
// 1-D bulk copies (cp.async.bulk) completing on one mbarrier.  Each row is
// copied as the 16-byte-aligned span covering image columns [c_lo, c_hi); the
// row buffer is [16-byte pad][span], and `off` records where image column 0 of
// that row would sit, so column c is at byte 16 + off + c * ES of the buffer.
// Bytes past the end of the raster are never read: a trailing partial chunk is
// copied by the lane with ordinary loads before the barrier is armed.
// Readers extract a lane's LB consecutive bytes at any byte position with
// warp-uniform funnel shifts (lanes differ by multiples of 16 bytes).
#pragma once

#include <climits>
#include <cstdint>
#include <cstring>

#include "ssb_async.cuh"

namespace ssb {

constexpr int kNoRow = INT_MIN;

struct RowSpan {
  const char* a = nullptr;  // aligned start (copy source)
  const char* b = nullptr;  // aligned end of the bulk part
  int off = kNoRow;
};

// Compute (and tail-fill) the span of one row; `rowp` = address of image column 0.
__device__ __forceinline__ RowSpan row_span(const char* rowp, int64_t c_lo, int64_t c_hi, int es,
                                            const char* end_valid, unsigned char* dst_row) {
  RowSpan sp;
  const char* lo = rowp + c_lo * es;
  const char* hi = rowp + c_hi * es;
  sp.a = reinterpret_cast<const char*>(reinterpret_cast<uintptr_t>(lo) & ~uintptr_t(15));
  sp.b = reinterpret_cast<const char*>((reinterpret_cast<uintptr_t>(hi) + 15) & ~uintptr_t(15));
  if (sp.b > end_valid) {  // never read past the raster: copy the tail bytes by hand
    sp.b = reinterpret_cast<const char*>(reinterpret_cast<uintptr_t>(end_valid) & ~uintptr_t(15));
    if (sp.b < sp.a) sp.b = sp.a;
    unsigned char* dst = dst_row + 16;
    for (const char* p = sp.b; p < hi; ++p) dst[p - sp.a] = (unsigned char)__ldg(p);
  }
  sp.off = (int)(rowp - sp.a);
  return sp;
}

// Warp-collective: arm `bar` with the total bytes of all lanes' spans, then
// issue each lane's bulk copy into its row buffer.  Lanes without a row pass
// has = false.  Must be called by all 32 lanes.
__device__ __forceinline__ void warp_issue(const RowSpan& sp, bool has, unsigned char* dst_row, uint64_t* bar,
                                           int lane) {
  uint32_t bytes = (has && sp.b > sp.a) ? (uint32_t)(sp.b - sp.a) : 0u;
#pragma unroll
  for (int d = 16; d >= 1; d >>= 1) bytes += __shfl_xor_sync(0xffffffffu, bytes, d);
  fence_proxy_async();
  __syncwarp();
  if (lane == 0) mbar_arrive_expect_tx(bar, bytes);
  __syncwarp();
  if (has && sp.b > sp.a) bulk_g2s(dst_row + 16, sp.a, (uint32_t)(sp.b - sp.a), bar);
}

// Per-lane arming: the mbarrier is initialised with one arrival per issuing
// lane (lanes [0, nl)); each of them arms its own byte count and issues its
// copy, so no warp-wide byte reduction or extra __syncwarp is needed (lanes
// without a row arrive with 0 bytes).  Lanes >= nl do nothing.
__device__ __forceinline__ void lane_issue(const RowSpan& sp, bool has, unsigned char* dst_row, uint64_t* bar, int lane,
                                           int nl) {
  if (lane >= nl) return;
  const uint32_t bytes = (has && sp.b > sp.a) ? (uint32_t)(sp.b - sp.a) : 0u;
  fence_proxy_async();
  mbar_arrive_expect_tx(bar, bytes);
  if (bytes) bulk_g2s(dst_row + 16, sp.a, bytes, bar);
}

// warp_issue with an L2 cache policy on the bulk copies (createpolicy operand)
__device__ __forceinline__ void warp_issue_hint(const RowSpan& sp, bool has, unsigned char* dst_row, uint64_t* bar,
                                                int lane, uint64_t pol) {
  uint32_t bytes = (has && sp.b > sp.a) ? (uint32_t)(sp.b - sp.a) : 0u;
#pragma unroll
  for (int d = 16; d >= 1; d >>= 1) bytes += __shfl_xor_sync(0xffffffffu, bytes, d);
  fence_proxy_async();
  __syncwarp();
  if (lane == 0) mbar_arrive_expect_tx(bar, bytes);
  __syncwarp();
  if (has && sp.b > sp.a) bulk_g2s_hint(dst_row + 16, sp.a, (uint32_t)(sp.b - sp.a), bar, pol);
}

template <int NO, int SW>
__device__ __forceinline__ void shift_words(const uint32_t* w, uint32_t* o, int sb) {
#pragma unroll
  for (int k = 0; k < NO; ++k) o[k] = __funnelshift_r(w[k + SW], w[k + SW + 1], sb);
}

// LB (multiple of 4) consecutive bytes starting at byte Q of a row buffer.
template <int LB>
__device__ __forceinline__ void lane_bytes(const unsigned char* rowbuf, int Q, uint32_t (&o)[LB / 4]) {
  constexpr int NC = (LB + 15) / 16 + 1, NO = LB / 4;  // chunks covering LB bytes at any 16-byte phase
  const uint4* p = reinterpret_cast<const uint4*>(rowbuf + (Q & ~15));
  uint32_t w[NC * 4];
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    const uint4 v = p[c];
    w[4 * c] = v.x; w[4 * c + 1] = v.y; w[4 * c + 2] = v.z; w[4 * c + 3] = v.w;
  }
  const int s = Q & 15, sb = (s & 3) * 8;
  switch (s >> 2) {  // warp-uniform
    case 0: shift_words<NO, 0>(w, o, sb); break;
    case 1: shift_words<NO, 1>(w, o, sb); break;
    case 2: shift_words<NO, 2>(w, o, sb); break;
    default: shift_words<NO, 3>(w, o, sb); break;
  }
}

// element k of packed words
template <typename InT>
__device__ __forceinline__ InT elem(const uint32_t* o, int k) {
  if constexpr (sizeof(InT) == 1) return (InT)(o[k >> 2] >> (8 * (k & 3)));
  else if constexpr (sizeof(InT) == 2) return (InT)(o[k >> 1] >> (16 * (k & 1)));
  else { InT v; memcpy(&v, &o[k], 4); return v; }
}

template <typename InT>
__device__ __forceinline__ void clear_elem(uint32_t* o, int k) {
  if constexpr (sizeof(InT) == 1) o[k >> 2] &= ~(0xFFu << (8 * (k & 3)));
  else if constexpr (sizeof(InT) == 2) o[k >> 1] &= ~(0xFFFFu << (16 * (k & 1)));
  else o[k] = 0u;
}

// Lane's E elements starting at image column c0 of a staged row (0 outside [0, C)
// and for rows without data).
// MAYBE_EMPTY = false: the caller guarantees the row has data (no select of zeros).
template <typename InT, int E, bool MAYBE_EMPTY = true>
__device__ __forceinline__ void lane_elems_packed(const unsigned char* rowbuf, int off, int64_t c0, int64_t C,
                                                  uint32_t (&o)[E * sizeof(InT) / 4]) {
  constexpr int NO = E * (int)sizeof(InT) / 4;
  if (MAYBE_EMPTY && off == kNoRow) {
#pragma unroll
    for (int k = 0; k < NO; ++k) o[k] = 0u;
    return;
  }
  lane_bytes<E * (int)sizeof(InT)>(rowbuf, 16 + off + (int)(c0 * (int64_t)sizeof(InT)), o);
  if (c0 < 0 || c0 + E > C) {
#pragma unroll
    for (int k = 0; k < E; ++k)
      if (c0 + k < 0 || c0 + k >= C) clear_elem<InT>(o, k);
  }
}

// The lane's valid elements [klo, khi) of E columns starting at image column
// c0 (columns outside [0, C) read as 0).  Computed once per sweep, so the
// per-row extraction needs no 64-bit per-element bounds tests: interior lanes
// (full) take no clearing at all.
struct LaneRange {
  int klo, khi;
  bool full;
};
template <int E>
__device__ __forceinline__ LaneRange lane_range(int64_t c0, int64_t C) {
  LaneRange r;
  r.klo = c0 < 0 ? (int)min64(-c0, E) : 0;
  r.khi = (int)max64(0, min64(E, C - c0));
  r.full = r.klo == 0 && r.khi == E;
  return r;
}

// lane_elems_packed with a precomputed LaneRange and a shift-free path for
// lanes whose data starts on a 16-byte boundary of the row buffer.
template <typename InT, int E, bool MAYBE_EMPTY = true>
__device__ __forceinline__ void lane_elems_ranged(const unsigned char* rowbuf, int off, int64_t c0, const LaneRange& lr,
                                                  uint32_t (&o)[E * sizeof(InT) / 4]) {
  constexpr int NO = E * (int)sizeof(InT) / 4;
  if (MAYBE_EMPTY && off == kNoRow) {
#pragma unroll
    for (int k = 0; k < NO; ++k) o[k] = 0u;
    return;
  }
  const int Q = 16 + off + (int)(c0 * (int64_t)sizeof(InT));
  if ((Q & 15) == 0) {  // 16-byte aligned lane data (warp-uniform): plain vector loads
    const uint4* p = reinterpret_cast<const uint4*>(rowbuf + Q);
    if constexpr (NO % 4 == 0) {
#pragma unroll
      for (int c = 0; c < NO / 4; ++c) {
        const uint4 v = p[c];
        o[4 * c] = v.x; o[4 * c + 1] = v.y; o[4 * c + 2] = v.z; o[4 * c + 3] = v.w;
      }
    } else {
      lane_bytes<E * (int)sizeof(InT)>(rowbuf, Q, o);
    }
  } else {
    lane_bytes<E * (int)sizeof(InT)>(rowbuf, Q, o);
  }
  if (!lr.full) {
#pragma unroll
    for (int k = 0; k < E; ++k)
      if (k < lr.klo || k >= lr.khi) clear_elem<InT>(o, k);
  }
}

}  // namespace ssb
