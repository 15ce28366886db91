// satsweep-b200: warp-tile helpers shared by the table-build kernels
// (sat_build.cu: reduce-then-scan; sat_onepass.cu: single pass with
// decoupled look-back).
#pragma once

#include <climits>
#include <cstdint>
#include <cstring>

#include "ssb_async.cuh"
#include "ssb_common.cuh"
#include "ssb_stage.cuh"

namespace ssb {

// ---- tile geometry -----------------------------------------------------------
template <typename InT>
struct Geo {
  using Tr = Elem<InT>;
  static constexpr int TW = Tr::kTW;                 // table columns per strip
  static constexpr int ES = (int)sizeof(InT);        // element bytes
  static constexpr int E = TW / 32;                  // elements per lane in a row
  static constexpr int LB = E * ES;                  // bytes per lane (16 or 32)
  static constexpr int ROWB = TW * ES + 48;          // staged row: 16 B pad + aligned span (<= TW*ES + 32)
  static constexpr int CPT = TW / kThreads;          // columns per thread in column passes
};


// ---- TMA row staging ----------------------------------------------------------
// Warp 0 stages table rows [r0, r0+nr) x table cols [j0, j0+TW) of the padded
// image, lane r handling row r (RB <= 32).  offs[r] = byte offset such that
// image column c of row r sits at stage + r*ROWB + 16 + offs[r] + c*ES
// (kNoRow: the row has no image data).
template <typename InT, int RB>
__device__ __forceinline__ void stage_issue(unsigned char* stage, int* offs, uint64_t* bar, const InT* in, int64_t R,
                                            int64_t C, int64_t in_ld, int64_t r0, int nr, int64_t j0, int lane) {
  static_assert(RB <= 32, "one lane per staged row");
  using G = Geo<InT>;
  const char* base = reinterpret_cast<const char*>(in);
  const char* end_valid = base + ((R - 1) * in_ld + C) * G::ES;
  const int64_t c_lo = j0 > 0 ? j0 - 1 : 0;
  const int64_t c_hi = (j0 - 1 + G::TW) < C ? (j0 - 1 + G::TW) : C;
  const int64_t ir = r0 + lane - 1;
  const bool has = lane < nr && ir >= 0 && ir < R && c_hi > c_lo;
  RowSpan sp;
  unsigned char* dst = stage + lane * G::ROWB;
  if (has) sp = row_span(base + ir * in_ld * G::ES, c_lo, c_hi, G::ES, end_valid, dst);
  if (lane < RB) offs[lane] = has ? sp.off : kNoRow;
  warp_issue(sp, has, dst, bar, lane);
}

// Lane's E consecutive elements starting at image column c0 of staged row r,
// as LB/4 packed 32-bit words.  Columns outside [0, C) and rows without data
// read as 0.
template <typename InT> struct Pack {
  static constexpr int NW = Geo<InT>::LB / 4;  // words per lane
};

template <typename InT>
__device__ __forceinline__ void lane_words(const unsigned char* stage, const int* offs, int r, int64_t c0, int64_t C,
                                           uint32_t (&o)[Pack<InT>::NW]) {
  using G = Geo<InT>;
  lane_elems_packed<InT, G::E>(stage + r * G::ROWB, offs[r], c0, C, o);
}

// sum of the lane's elements in Loc / of their squares in LocSq
// pairwise (tree) sum of E values: log2(E) dependent adds instead of E
template <int N, typename T>
__device__ __forceinline__ T tree_sum(T (&v)[N]) {
#pragma unroll
  for (int h = N / 2; h >= 1; h /= 2) {
#pragma unroll
    for (int k = 0; k < h; ++k) v[k] = add(v[k], v[k + h]);
  }
  return v[0];
}

template <typename InT>
__device__ __forceinline__ typename Elem<InT>::Loc lane_total(const uint32_t* o) {
  using Loc = typename Elem<InT>::Loc;
  Loc t = Loc(0);
  if constexpr (sizeof(InT) == 1) {
#pragma unroll
    for (int i = 0; i < Pack<InT>::NW; ++i) t = __dp4a(o[i], 0x01010101u, t);
  } else if constexpr (Elem<InT>::kFloat) {
    Loc v[Geo<InT>::E];
#pragma unroll
    for (int k = 0; k < Geo<InT>::E; ++k) v[k] = conv<Loc>(elem<InT>(o, k));
    t = tree_sum(v);
  } else {
#pragma unroll
    for (int k = 0; k < Geo<InT>::E; ++k) t = add(t, conv<Loc>(elem<InT>(o, k)));
  }
  return t;
}
template <typename InT>
__device__ __forceinline__ typename Elem<InT>::LocSq lane_total_sq(const uint32_t* o) {
  using LocSq = typename Elem<InT>::LocSq;
  LocSq t = LocSq(0);
  if constexpr (sizeof(InT) == 1) {
#pragma unroll
    for (int i = 0; i < Pack<InT>::NW; ++i) t = __dp4a(o[i], o[i], t);
  } else if constexpr (Elem<InT>::kFloat) {
    LocSq v[Geo<InT>::E];
#pragma unroll
    for (int k = 0; k < Geo<InT>::E; ++k) v[k] = convsq<LocSq>(elem<InT>(o, k));
    t = tree_sum(v);
  } else {
#pragma unroll
    for (int k = 0; k < Geo<InT>::E; ++k) t = add(t, convsq<LocSq>(elem<InT>(o, k)));
  }
  return t;
}

template <typename InT>
__device__ __forceinline__ bool any_nonfinite(const uint32_t* o) {
  if constexpr (Elem<InT>::kFloat) {
    bool bad = false;
#pragma unroll
    for (int k = 0; k < Geo<InT>::E; ++k) bad |= !isfinite(elem<InT>(o, k));
    return bad;
  } else {
    return false;
  }
}

// ---------------------------------------------------------------------------
// Warp tiles.  Phases 1 and 3 give every warp its own (strip J, segment K)
// tile and its own 2-deep TMA row pipeline: the warp sweeps the segment top to
// bottom, lane l owning E consecutive table columns.  A row's strip-local
// prefix is a lane-serial prefix plus one warp shuffle scan, and the vertical
// accumulation happens in the same lane's registers -- no shared-memory
// transpose and no CTA-wide barrier anywhere in the sweep.
constexpr int kWarpsPerCta = kThreads / 32;

template <typename InT, int RB_ = 0, int NSTG_ = 2>
struct WarpStage {
  using G = Geo<InT>;
  static constexpr int RBW = RB_ > 0 ? RB_ : (G::ES == 1 ? 8 : 4);  // rows per stage (<= 32)
  static constexpr int NSTG = NSTG_;                               // ring depth
  alignas(16) unsigned char buf[NSTG][RBW * G::ROWB];
  int offs[NSTG][RBW];
  uint64_t bar[NSTG];
};

template <int WPC = kWarpsPerCta>
__device__ __forceinline__ void warp_tile(int nJ, int nK, int& J, int& K) {
  const int t = blockIdx.x * WPC + (threadIdx.x >> 5);
  J = t % nJ;
  K = t / nJ;
  if (K >= nK) K = -1;
}

template <typename WS>
__device__ __forceinline__ void warp_stage_init(WS& ws, int lane) {
  if (lane == 0) {
    for (int i = 0; i < WS::NSTG; ++i) mbar_init(&ws.bar[i], 1);
    fence_mbar_init();
  }
  __syncwarp();
}

template <int N, int OFF, typename T>
__device__ __forceinline__ T warp_reduce_scatter_step(T (&v)[N], int lane) {
  if constexpr (N == 1) {
    T x = v[0];
#pragma unroll
    for (int d = OFF; d >= 1; d >>= 1) x = add(x, shfl_xor(x, d));
    return x;
  } else {
    constexpr int H = N / 2;
    const bool upper = (lane & OFF) != 0;
    T w[H];
#pragma unroll
    for (int k = 0; k < H; ++k) {
      const T mine = upper ? v[k + H] : v[k];
      const T other = upper ? v[k] : v[k + H];
      w[k] = add(mine, shfl_xor(other, OFF));
    }
    return warp_reduce_scatter_step<H, OFF / 2>(w, lane);
  }
}

// Reduce-scatter of N per-lane values across the warp (N a power of two <= 32):
// returns the 32-lane total of value index lane / (32 / N) -- N + 5 - log2(N)
// shuffles instead of 5N for N separate warp sums.
template <int N, typename T>
__device__ __forceinline__ T warp_reduce_scatter(T (&v)[N], int lane) {
  static_assert(N >= 1 && N <= 32 && (N & (N - 1)) == 0, "power of two");
  if constexpr (N == 1) {
    return warp_sum(v[0]);
  } else {
    // halving steps: offsets 16, 8, ... while more than one value remains
    constexpr int H = N / 2;
    const bool upper = (lane & 16) != 0;
    T w[H];
#pragma unroll
    for (int k = 0; k < H; ++k) {
      const T mine = upper ? v[k + H] : v[k];
      const T other = upper ? v[k] : v[k + H];
      w[k] = add(mine, shfl_xor(other, 16));
    }
    return warp_reduce_scatter_step<H, 8>(w, lane);
  }
}


#ifndef SSB_SCAN_STHINT
#define SSB_SCAN_STHINT 0
#endif
template <typename Acc, int E>
__device__ __forceinline__ void store_lane_cols(Acc* __restrict__ dst, const Acc (&v)[E], int64_t col, int64_t PC) {
  if (col + E <= PC) {
#if SSB_SCAN_STHINT
    const uint64_t pol = SSB_SCAN_STHINT == 1 ? policy_evict_first() : policy_evict_last();
#endif
#pragma unroll
    for (int k = 0; k < E; k += 4) {
      U64x4 q;
      memcpy(&q, &v[k], 32);
#if SSB_SCAN_STHINT
      st256_hint(dst + k, q, pol);
#else
      st256(dst + k, q);
#endif
    }
  } else {
#pragma unroll
    for (int k = 0; k < E; ++k)
      if (col + k < PC) st_cs(dst + k, v[k]);
  }
}

}  // namespace ssb
