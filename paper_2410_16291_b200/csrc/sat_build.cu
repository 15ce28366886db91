// satsweep-b200: summed-area table construction on sm_100a.
//
// Replaces the reference's fill -> row cumsum -> column cumsum pipeline
// (pkg/src/satsweep/integral.py:86-116, parallel.py:106-121) with a
// reduce-then-scan design that writes every table entry exactly once:
//
//   phase 1  sat_reduce   per (strip J, segment K) tile: the total of every
//                         table row inside the strip and the strip-local
//                         prefix of the segment's column totals.  Reads the
//                         image once; writes ~8/TW + 8/SR bytes per pixel.
//   phase 2  sat_rowcarry exclusive scan of row totals across strips
//                         (the left carry of every row in every strip),
//            sat_segsum   per-(segment, strip) sum of those left carries,
//            sat_topcarry exclusive scan down the segments of the segment
//                         column totals (the table row above each segment).
//   phase 3  sat_scan     per tile: warp row scans, transpose through
//                         swizzled smem, column accumulation in registers,
//                         128-bit coalesced streaming stores.
//
// Both image-reading phases stage RB image rows per step into shared memory
// with TMA bulk copies (cp.async.bulk, UBLKCP) on a 2-deep mbarrier pipeline,
// so the global loads of step b+1 are in flight while step b is computed.
// Rows are copied as the 16-byte-aligned span covering the strip; each lane
// re-aligns its elements with funnel shifts (the shift is warp-uniform).
//
// Table entry for table row i inside segment K and column j inside strip J:
//   S[i][j] = Top[K][j] + sum_{k0 <= i' <= i} ( RL[J][i'] + RPloc[i'][j] )
// where RPloc is the strip-local row prefix.  Integer tables are exact modulo
// 2^64; f32 input accumulates in double with a deterministic order.
#include <climits>
#include <cstdlib>

#include "ssb_async.cuh"
#include "ssb_common.cuh"
#include "ssb_stage.cuh"

#ifndef SSB_SCAN_MINB
#define SSB_SCAN_MINB 2
#endif

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
template <typename InT>
__device__ __forceinline__ typename Elem<InT>::Loc lane_total(const uint32_t* o) {
  using Loc = typename Elem<InT>::Loc;
  Loc t = Loc(0);
  if constexpr (sizeof(InT) == 1) {
#pragma unroll
    for (int i = 0; i < Pack<InT>::NW; ++i) t = __dp4a(o[i], 0x01010101u, t);
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

template <typename InT, int RB_ = 0>
struct WarpStage {
  using G = Geo<InT>;
  static constexpr int RBW = RB_ > 0 ? RB_ : (G::ES == 1 ? 8 : 4);  // rows per stage (<= 32)
  alignas(16) unsigned char buf[2][RBW * G::ROWB];
  int offs[2][RBW];
  uint64_t bar[2];
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
    mbar_init(&ws.bar[0], 1);
    mbar_init(&ws.bar[1], 1);
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

// ---------------------------------------------------------------------------
// phase 1
template <typename InT, bool SQ, int RBR, int WPC>
__global__ void __launch_bounds__(32 * WPC)
sat_reduce_kernel(const InT* __restrict__ in, int64_t R, int64_t C, int64_t in_ld,
                  typename Elem<InT>::Acc* __restrict__ rowtot, typename Elem<InT>::Acc* __restrict__ rowtot_sq,
                  typename Elem<InT>::Acc* __restrict__ colp, typename Elem<InT>::Acc* __restrict__ colp_sq,
                  int64_t SR, int nJ, int nK, int* __restrict__ nonfinite) {
  using Tr = Elem<InT>;
  using Loc = typename Tr::Loc;
  using LocSq = typename Tr::LocSq;
  using Acc = typename Tr::Acc;
  using G = Geo<InT>;
  using WS = WarpStage<InT, RBR>;
  constexpr int TW = G::TW, E = G::E, RB = WS::RBW;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  WS* stages = reinterpret_cast<WS*>(smem_raw);
  const int lane = threadIdx.x & 31;
  WS& ws = stages[threadIdx.x >> 5];
  int J, K;
  warp_tile<WPC>(nJ, nK, J, K);
  if (K < 0) return;
  const int64_t PR = R + 1, PC = C + 1;
  const int64_t j0 = (int64_t)J * TW, k0 = (int64_t)K * SR;
  const int64_t k1 = min(k0 + SR, PR);
  const int nblk = (int)((k1 - k0 + RB - 1) / RB);
  const int64_t c0 = j0 + lane * E - 1;
  bool nf = false;
  warp_stage_init(ws, lane);
  stage_issue<InT, RB>(ws.buf[0], ws.offs[0], &ws.bar[0], in, R, C, in_ld, k0, (int)min64(RB, k1 - k0), j0, lane);

  Loc cs[E];  // column partials over the segment (<= SR rows: no overflow in Loc / LocSq)
  LocSq csq[E];
#pragma unroll
  for (int k = 0; k < E; ++k) { cs[k] = Loc(0); csq[k] = LocSq(0); }
  // u8: bytes are summed two per 32-bit register (16-bit halves, exact for
  // <= 257 rows) and flushed into cs every 256 rows
  constexpr bool kPacked = sizeof(InT) == 1;
  constexpr int NWD = Pack<InT>::NW;
  uint32_t pk_lo[kPacked ? NWD : 1], pk_hi[kPacked ? NWD : 1];
#pragma unroll
  for (int i = 0; i < (kPacked ? NWD : 1); ++i) { pk_lo[i] = 0u; pk_hi[i] = 0u; }
  int since_flush = 0;
  const bool lane_inside = c0 >= 0 && c0 + E <= C;
  const int qbase = 16 + (int)(c0 * G::ES);
  auto flush = [&]() {
    if constexpr (kPacked) {
#pragma unroll
      for (int i = 0; i < NWD; ++i) {
        cs[4 * i + 0] = add(cs[4 * i + 0], (Loc)(pk_lo[i] & 0xFFFFu));
        cs[4 * i + 2] = add(cs[4 * i + 2], (Loc)(pk_lo[i] >> 16));
        cs[4 * i + 1] = add(cs[4 * i + 1], (Loc)(pk_hi[i] & 0xFFFFu));
        cs[4 * i + 3] = add(cs[4 * i + 3], (Loc)(pk_hi[i] >> 16));
        pk_lo[i] = 0u;
        pk_hi[i] = 0u;
      }
    }
    since_flush = 0;
  };

  for (int b = 0; b < nblk; ++b) {
    const int s = b & 1;
    const int64_t r0 = k0 + (int64_t)b * RB;
    const int nr = (int)min64(RB, k1 - r0);
    if (b + 1 < nblk) {
      const int64_t rn = r0 + RB;
      stage_issue<InT, RB>(ws.buf[s ^ 1], ws.offs[s ^ 1], &ws.bar[s ^ 1], in, R, C, in_ld, rn,
                           (int)min64(RB, k1 - rn), j0, lane);
    }
    mbar_wait(&ws.bar[s], (uint32_t)((b >> 1) & 1));
    Loc part[RB];      // lane partial of each staged row
    LocSq part_sq[RB];
    // interior blocks (all RB rows are image rows) on interior lanes (all E
    // columns inside the image) take a check-free path
    const bool fast = lane_inside && nr == RB && r0 >= 1 && r0 + RB - 1 <= R;
#pragma unroll
    for (int r = 0; r < RB; ++r) {
      part[r] = Loc(0);
      part_sq[r] = LocSq(0);
      if (fast || r < nr) {
        uint32_t o[NWD];
        if (fast) lane_bytes<G::LB>(ws.buf[s] + r * G::ROWB, qbase + ws.offs[s][r], o);
        else lane_words<InT>(ws.buf[s], ws.offs[s], r, c0, C, o);
        part[r] = lane_total<InT>(o);
        if constexpr (kPacked) {
#pragma unroll
          for (int i = 0; i < NWD; ++i) {
            pk_lo[i] += o[i] & 0x00FF00FFu;
            pk_hi[i] += (o[i] >> 8) & 0x00FF00FFu;
          }
        } else {
#pragma unroll
          for (int k = 0; k < E; ++k) cs[k] = add(cs[k], conv<Loc>(elem<InT>(o, k)));
        }
        if constexpr (SQ) {
          part_sq[r] = lane_total_sq<InT>(o);
#pragma unroll
          for (int k = 0; k < E; ++k) csq[k] = add(csq[k], convsq<LocSq>(elem<InT>(o, k)));
        }
        nf |= any_nonfinite<InT>(o);
      }
    }
    since_flush += RB;
    if (since_flush >= 256) flush();
    // row totals: lane l ends with the total of row l / (32 / RB)
    const Loc rs = warp_reduce_scatter<RB>(part, lane);
    const int myrow = lane / (32 / RB);
    const bool writer = (lane % (32 / RB)) == 0 && myrow < nr;
    if (writer) rowtot[(r0 + myrow) * nJ + J] = (Acc)rs;
    if constexpr (SQ) {
      const LocSq rq = warp_reduce_scatter<RB>(part_sq, lane);
      if (writer) rowtot_sq[(r0 + myrow) * nJ + J] = (Acc)rq;
    }
    __syncwarp();  // stage s fully read before it is refilled
  }
  flush();

  // strip-local prefix of the segment's column totals
  Acc run = Acc(0), runq = Acc(0);
  Acc col[E], colq[E];
#pragma unroll
  for (int k = 0; k < E; ++k) {
    run = add(run, (Acc)cs[k]); col[k] = run;
    if constexpr (SQ) { runq = add(runq, (Acc)csq[k]); colq[k] = runq; }
  }
  const Acc off = sub(warp_incl_scan(run, lane), run);
  Acc offq = Acc(0);
  if constexpr (SQ) offq = sub(warp_incl_scan(runq, lane), runq);
  const int64_t cbase = j0 + lane * E;
#pragma unroll
  for (int k = 0; k < E; ++k) {
    if (cbase + k < PC) {
      colp[(int64_t)K * PC + cbase + k] = add(off, col[k]);
      if constexpr (SQ) colp_sq[(int64_t)K * PC + cbase + k] = add(offq, colq[k]);
    }
  }
  if (nf && nonfinite) atomicOr(nonfinite, 1);
}

// ---------------------------------------------------------------------------
// phase 2a: left carries (exclusive scan across strips), in place, one warp
// per table row over the row-major [PR][nJ] row-total layout.
template <typename Acc>
__global__ void __launch_bounds__(kThreads)
sat_rowcarry_kernel(Acc* __restrict__ rowtot, int nJ, int64_t PR) {
  const int64_t i = (int64_t)blockIdx.x * (kThreads / 32) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (i >= PR) return;
  constexpr int MAXM = 16;  // strips per lane per pass
  int mm = (nJ + 31) / 32;
  if (mm > MAXM) mm = MAXM;
  Acc* row = rowtot + i * nJ;
  Acc carry = Acc(0);
  for (int base = 0; base < nJ; base += 32 * mm) {
    Acc v[MAXM];
    Acc run = Acc(0);
#pragma unroll
    for (int k = 0; k < MAXM; ++k) {
      const int J = base + lane * mm + k;
      v[k] = (k < mm && J < nJ) ? row[J] : Acc(0);
      run = add(run, v[k]);
    }
    const Acc incl = warp_incl_scan(run, lane);
    Acc acc = add(carry, sub(incl, run));
#pragma unroll
    for (int k = 0; k < MAXM; ++k) {
      const int J = base + lane * mm + k;
      if (k < mm && J < nJ) { row[J] = acc; acc = add(acc, v[k]); }
    }
    carry = add(carry, __shfl_sync(0xffffffffu, incl, 31));
  }
}

// phase 2a': per (segment, strip) sum of left carries: CTA (K, 32-strip group),
// warp w sums rows k0+w, k0+w+8, ... with lanes over strips (coalesced), then a
// fixed-order combine of the 8 warp partials.
template <typename Acc>
__global__ void __launch_bounds__(kThreads)
sat_segsum_kernel(const Acc* __restrict__ rl, Acc* __restrict__ srl, int nJ, int64_t PR, int64_t SR) {
  __shared__ Acc part[kThreads / 32][32];
  const int K = blockIdx.x;
  const int J = blockIdx.y * 32 + (threadIdx.x & 31);
  const int warp = threadIdx.x >> 5;
  const int64_t k0 = (int64_t)K * SR, k1 = min(k0 + SR, PR);
  Acc sacc = Acc(0);
  if (J < nJ) {
    constexpr int B = 8;
    for (int64_t i0 = k0 + warp; i0 < k1; i0 += (int64_t)(kThreads / 32) * B) {
      Acc v[B];
#pragma unroll
      for (int u = 0; u < B; ++u) {
        const int64_t i = i0 + (int64_t)u * (kThreads / 32);
        v[u] = i < k1 ? rl[i * nJ + J] : Acc(0);
      }
#pragma unroll
      for (int u = 0; u < B; ++u) sacc = add(sacc, v[u]);
    }
  }
  part[warp][threadIdx.x & 31] = sacc;
  __syncthreads();
  if (warp == 0 && J < nJ) {
    Acc t = Acc(0);
    for (int w = 0; w < kThreads / 32; ++w) t = add(t, part[w][threadIdx.x]);
    srl[(int64_t)K * nJ + J] = t;
  }
}

// phase 2b: table row above every segment (without any band carry), in place
// over the column prefixes.  The final running value is the image's last table
// row -- the band column totals used by row-band shards.
template <typename Acc>
__global__ void sat_topcarry_kernel(Acc* __restrict__ colp, const Acc* __restrict__ srl, Acc* __restrict__ totals,
                                    int nK, int nJ, int64_t PC, int TW) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= PC) return;
  const int J = (int)(j / TW);
  constexpr int B = 8;
  Acc run = Acc(0);
  for (int K0 = 0; K0 < nK; K0 += B) {
    Acc v[B], sr[B];
#pragma unroll
    for (int k = 0; k < B; ++k) {
      v[k] = (K0 + k < nK) ? colp[(int64_t)(K0 + k) * PC + j] : Acc(0);
      sr[k] = (K0 + k < nK) ? srl[(int64_t)(K0 + k) * nJ + J] : Acc(0);
    }
#pragma unroll
    for (int k = 0; k < B; ++k) {
      if (K0 + k < nK) colp[(int64_t)(K0 + k) * PC + j] = run;
      run = add(run, add(v[k], sr[k]));
    }
  }
  if (totals) totals[j] = run;
}

// adds a carry row to every segment's top row (row-band shards)
template <typename Acc>
__global__ void sat_apply_carry_kernel(Acc* __restrict__ colp, const Acc* __restrict__ carry, int nK, int64_t PC) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= PC) return;
  const Acc c = carry[j];
  for (int K = 0; K < nK; ++K) colp[(int64_t)K * PC + j] = add(colp[(int64_t)K * PC + j], c);
}

// ---------------------------------------------------------------------------
// phase 3
template <typename Acc, int E>
__device__ __forceinline__ void store_lane_cols(Acc* __restrict__ dst, const Acc (&v)[E], int64_t col, int64_t PC) {
  if (col + E <= PC) {
#pragma unroll
    for (int k = 0; k < E; k += 4) {
      U64x4 q;
      memcpy(&q, &v[k], 32);
      st256(dst + k, q);
    }
  } else {
#pragma unroll
    for (int k = 0; k < E; ++k)
      if (col + k < PC) st_cs(dst + k, v[k]);
  }
}

template <typename InT, bool SQ>
__global__ void __launch_bounds__(kThreads, SQ ? 2 : SSB_SCAN_MINB)
sat_scan_kernel(const InT* __restrict__ in, int64_t R, int64_t C, int64_t in_ld,
                typename Elem<InT>::Acc* __restrict__ sat, typename Elem<InT>::Acc* __restrict__ sat_sq, int64_t sat_ld,
                const typename Elem<InT>::Acc* __restrict__ rl, const typename Elem<InT>::Acc* __restrict__ rl_sq,
                const typename Elem<InT>::Acc* __restrict__ top, const typename Elem<InT>::Acc* __restrict__ top_sq,
                int64_t SR, int nJ, int nK) {
  using Tr = Elem<InT>;
  using Loc = typename Tr::Loc;
  using LocSq = typename Tr::LocSq;
  using Acc = typename Tr::Acc;
  using G = Geo<InT>;
  using WS = WarpStage<InT>;
  constexpr int TW = G::TW, E = G::E, RB = WS::RBW;
  static_assert(E % 4 == 0, "256-bit stores");
  extern __shared__ __align__(16) unsigned char smem_raw[];
  WS* stages = reinterpret_cast<WS*>(smem_raw);
  const int lane = threadIdx.x & 31;
  WS& ws = stages[threadIdx.x >> 5];
  int J, K;
  warp_tile(nJ, nK, J, K);
  if (K < 0) return;
  const int64_t PR = R + 1, PC = C + 1;
  const int64_t j0 = (int64_t)J * TW, k0 = (int64_t)K * SR;
  const int64_t k1 = min(k0 + SR, PR);
  const int nblk = (int)((k1 - k0 + RB - 1) / RB);
  const int64_t cbase = j0 + lane * E;  // table column of the lane's first element
  const int64_t c0 = cbase - 1;         // matching image column
  warp_stage_init(ws, lane);
  stage_issue<InT, RB>(ws.buf[0], ws.offs[0], &ws.bar[0], in, R, C, in_ld, k0, (int)min64(RB, k1 - k0), j0, lane);

  Acc acc[E], accq[E];
#pragma unroll
  for (int k = 0; k < E; ++k) {
    acc[k] = cbase + k < PC ? top[(int64_t)K * PC + cbase + k] : Acc(0);
    if constexpr (SQ) accq[k] = cbase + k < PC ? top_sq[(int64_t)K * PC + cbase + k] : Acc(0);
  }
  const bool writes_plain = sat != nullptr;

  for (int b = 0; b < nblk; ++b) {
    const int s = b & 1;
    const int64_t r0 = k0 + (int64_t)b * RB;
    const int nr = (int)min64(RB, k1 - r0);
    if (b + 1 < nblk) {
      const int64_t rn = r0 + RB;
      stage_issue<InT, RB>(ws.buf[s ^ 1], ws.offs[s ^ 1], &ws.bar[s ^ 1], in, R, C, in_ld, rn,
                           (int)min64(RB, k1 - rn), j0, lane);
    }
    Acc rlv = Acc(0), rlqv = Acc(0);  // lane r: left carry of row r
    if (lane < nr) {
      rlv = rl[(r0 + lane) * nJ + J];
      if constexpr (SQ) rlqv = rl_sq[(r0 + lane) * nJ + J];
    }
    mbar_wait(&ws.bar[s], (uint32_t)((b >> 1) & 1));
    for (int r = 0; r < nr; ++r) {
      uint32_t o[Pack<InT>::NW];
      lane_words<InT>(ws.buf[s], ws.offs[s], r, c0, C, o);
      const int64_t row = r0 + r;
      {
        const Loc t = lane_total<InT>(o);
        Loc run = sub(warp_incl_scan(t, lane), t);  // exclusive: prefix of the lanes to the left
        const Acc left = __shfl_sync(0xffffffffu, rlv, r);
#pragma unroll
        for (int k = 0; k < E; ++k) {
          run = add(run, conv<Loc>(elem<InT>(o, k)));
          acc[k] = add(acc[k], add(left, (Acc)run));
        }
        if (writes_plain) store_lane_cols<Acc, E>(sat + row * sat_ld + cbase, acc, cbase, PC);
      }
      if constexpr (SQ) {
        const LocSq t = lane_total_sq<InT>(o);
        LocSq run = sub(warp_incl_scan(t, lane), t);
        const Acc left = __shfl_sync(0xffffffffu, rlqv, r);
#pragma unroll
        for (int k = 0; k < E; ++k) {
          run = add(run, convsq<LocSq>(elem<InT>(o, k)));
          accq[k] = add(accq[k], add(left, (Acc)run));
        }
        store_lane_cols<Acc, E>(sat_sq + row * sat_ld + cbase, accq, cbase, PC);
      }
    }
    __syncwarp();  // stage s fully read before it is refilled
  }
}

// ---------------------------------------------------------------------------
// host-side launch
struct SatPlan {
  int TW, nJ, nK;
  int64_t SR, PR, PC;
  // workspace offsets in elements of 8 bytes
  int64_t off_rowtot, off_rowtot_sq, off_colp, off_colp_sq, off_srl, off_srl_sq, total;
};

inline int tw_for(int dtype) { return (dtype == IN_U8 || dtype == IN_U16) ? 512 : 256; }

inline SatPlan make_sat_plan(int dtype, int64_t R, int64_t C, bool sq) {
  SatPlan p{};
  p.TW = tw_for(dtype);
  p.PR = R + 1; p.PC = C + 1;
  p.nJ = (int)((p.PC + p.TW - 1) / p.TW);
  const int RB = 8;  // segment height is a multiple of every kernel's row block
  const int64_t target_tiles = 64LL * kNumSMs;  // warp tiles: ~4 waves of 16 warps per SM
  int64_t wantK = (target_tiles + p.nJ - 1) / p.nJ;
  int64_t SR = (p.PR + wantK - 1) / wantK;
  SR = ((SR + RB - 1) / RB) * RB;
  if (SR > 1024) SR = 1024;
  if (SR < RB) SR = RB;
  p.SR = SR;
  p.nK = (int)((p.PR + SR - 1) / SR);
  int64_t o = 0;
  p.off_rowtot = o; o += (int64_t)p.nJ * p.PR;
  p.off_rowtot_sq = o; if (sq) o += (int64_t)p.nJ * p.PR;
  p.off_colp = o; o += (int64_t)p.nK * p.PC;
  p.off_colp_sq = o; if (sq) o += (int64_t)p.nK * p.PC;
  p.off_srl = o; o += (int64_t)p.nK * p.nJ;
  p.off_srl_sq = o; if (sq) o += (int64_t)p.nK * p.nJ;
  p.total = o;
  return p;
}


template <typename InT, bool SQ, int RBR, int WPC>
cudaError_t launch_reduce_rw(const InT* x, int64_t R, int64_t C, int64_t in_ld, typename Elem<InT>::Acc* rowtot,
                             typename Elem<InT>::Acc* rowtot_sq, typename Elem<InT>::Acc* colp,
                             typename Elem<InT>::Acc* colp_sq, int* nonfinite, cudaStream_t st, const SatPlan& p) {
  const int tb = (int)(((int64_t)p.nJ * p.nK + WPC - 1) / WPC);
  const int smem = (int)(sizeof(WarpStage<InT, RBR>) * WPC);
  auto kfn = sat_reduce_kernel<InT, SQ, RBR, WPC>;
  cudaError_t e = cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  kfn<<<tb, 32 * WPC, smem, st>>>(x, R, C, in_ld, rowtot, rowtot_sq, colp, colp_sq, p.SR, p.nJ, p.nK, nonfinite);
  return cudaGetLastError();
}

// Reduce kernel shape: 8-row stages, 8 warps per CTA (measured best among
// 4/8/16/32-row stages x 4/8 warps at C5).
template <typename InT, bool SQ>
cudaError_t launch_reduce_cfg(const InT* x, int64_t R, int64_t C, int64_t in_ld, typename Elem<InT>::Acc* rowtot,
                              typename Elem<InT>::Acc* rowtot_sq, typename Elem<InT>::Acc* colp,
                              typename Elem<InT>::Acc* colp_sq, int* nonfinite, cudaStream_t st, const SatPlan& p) {
  return launch_reduce_rw<InT, SQ, 0, kWarpsPerCta>(x, R, C, in_ld, rowtot, rowtot_sq, colp, colp_sq, nonfinite, st, p);
}

template <typename InT, bool SQ>
cudaError_t launch_sat_prepare_t(const void* in, int64_t R, int64_t C, int64_t in_ld, void* ws, void* totals,
                                 void* totals_sq, int* nonfinite, cudaStream_t st, const SatPlan& p) {
  using Acc = typename Elem<InT>::Acc;
  Acc* w = reinterpret_cast<Acc*>(ws);
  Acc* rowtot = w + p.off_rowtot;
  Acc* rowtot_sq = SQ ? w + p.off_rowtot_sq : nullptr;
  Acc* colp = w + p.off_colp;
  Acc* colp_sq = SQ ? w + p.off_colp_sq : nullptr;
  Acc* srl = w + p.off_srl;
  Acc* srl_sq = SQ ? w + p.off_srl_sq : nullptr;
  const InT* x = reinterpret_cast<const InT*>(in);
  cudaError_t e = launch_reduce_cfg<InT, SQ>(x, R, C, in_ld, rowtot, rowtot_sq, colp, colp_sq, nonfinite, st, p);
  if (e != cudaSuccess) return e;
  const int nb_rows = (int)((p.PR + kThreads / 32 - 1) / (kThreads / 32));
  sat_rowcarry_kernel<Acc><<<nb_rows, kThreads, 0, st>>>(rowtot, p.nJ, p.PR);
  if (SQ) sat_rowcarry_kernel<Acc><<<nb_rows, kThreads, 0, st>>>(rowtot_sq, p.nJ, p.PR);
  const dim3 sgrid(p.nK, (p.nJ + 31) / 32);
  sat_segsum_kernel<Acc><<<sgrid, kThreads, 0, st>>>(rowtot, srl, p.nJ, p.PR, p.SR);
  if (SQ) sat_segsum_kernel<Acc><<<sgrid, kThreads, 0, st>>>(rowtot_sq, srl_sq, p.nJ, p.PR, p.SR);
  const int nb_cols = (int)((p.PC + kThreads - 1) / kThreads);
  sat_topcarry_kernel<Acc><<<nb_cols, kThreads, 0, st>>>(colp, srl, reinterpret_cast<Acc*>(totals), p.nK, p.nJ, p.PC, p.TW);
  if (SQ) sat_topcarry_kernel<Acc><<<nb_cols, kThreads, 0, st>>>(colp_sq, srl_sq, reinterpret_cast<Acc*>(totals_sq), p.nK, p.nJ, p.PC, p.TW);
  note_launch(SQ ? 7 : 4);
  return cudaGetLastError();
}

template <typename InT, bool SQ>
cudaError_t launch_sat_finish_t(const void* in, int64_t R, int64_t C, int64_t in_ld, void* sat, void* sat_sq,
                                int64_t sat_ld, const void* carry, const void* carry_sq, void* ws, cudaStream_t st,
                                const SatPlan& p) {
  using Acc = typename Elem<InT>::Acc;
  Acc* w = reinterpret_cast<Acc*>(ws);
  Acc* rowtot = w + p.off_rowtot;
  Acc* rowtot_sq = SQ ? w + p.off_rowtot_sq : nullptr;
  Acc* colp = w + p.off_colp;
  Acc* colp_sq = SQ ? w + p.off_colp_sq : nullptr;
  const int nb_cols = (int)((p.PC + kThreads - 1) / kThreads);
  if (carry) { sat_apply_carry_kernel<Acc><<<nb_cols, kThreads, 0, st>>>(colp, reinterpret_cast<const Acc*>(carry), p.nK, p.PC); note_launch(1); }
  if (SQ && carry_sq) { sat_apply_carry_kernel<Acc><<<nb_cols, kThreads, 0, st>>>(colp_sq, reinterpret_cast<const Acc*>(carry_sq), p.nK, p.PC); note_launch(1); }
  const int tb = (int)(((int64_t)p.nJ * p.nK + kWarpsPerCta - 1) / kWarpsPerCta);
  const int smem = (int)(sizeof(WarpStage<InT>) * kWarpsPerCta);
  cudaError_t e = cudaFuncSetAttribute(sat_scan_kernel<InT, SQ>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  sat_scan_kernel<InT, SQ><<<tb, kThreads, smem, st>>>(reinterpret_cast<const InT*>(in), R, C, in_ld,
                                                    reinterpret_cast<Acc*>(sat), reinterpret_cast<Acc*>(sat_sq),
                                                    sat_ld, rowtot, rowtot_sq, colp, colp_sq, p.SR, p.nJ, p.nK);
  note_launch(1);
  return cudaGetLastError();
}

#define SSB_SAT_DISPATCH(CALL_T)                                                \
  switch (dtype) {                                                              \
    case IN_U8: return sq ? CALL_T(uint8_t, true) : CALL_T(uint8_t, false);     \
    case IN_U16: return sq ? CALL_T(uint16_t, true) : CALL_T(uint16_t, false);  \
    case IN_I32: return sq ? CALL_T(int32_t, true) : CALL_T(int32_t, false);    \
    case IN_F32: return sq ? CALL_T(float, true) : CALL_T(float, false);        \
    default: return cudaErrorInvalidValue;                                      \
  }

cudaError_t launch_sat_prepare(int dtype, const void* in, int64_t R, int64_t C, int64_t in_ld, bool sq, void* ws,
                               void* totals, void* totals_sq, int* nonfinite, cudaStream_t st) {
  const SatPlan p = make_sat_plan(dtype, R, C, sq);
#define CALL_T(T, S) launch_sat_prepare_t<T, S>(in, R, C, in_ld, ws, totals, totals_sq, nonfinite, st, p)
  SSB_SAT_DISPATCH(CALL_T)
#undef CALL_T
}

cudaError_t launch_sat_finish(int dtype, const void* in, int64_t R, int64_t C, int64_t in_ld, void* sat, void* sat_sq,
                              int64_t sat_ld, const void* carry, const void* carry_sq, void* ws, cudaStream_t st) {
  const bool sq = sat_sq != nullptr;
  const SatPlan p = make_sat_plan(dtype, R, C, sq);
#define CALL_T(T, S) launch_sat_finish_t<T, S>(in, R, C, in_ld, sat, sat_sq, sat_ld, carry, carry_sq, ws, st, p)
  SSB_SAT_DISPATCH(CALL_T)
#undef CALL_T
}
#undef SSB_SAT_DISPATCH

void sat_plan_info(int dtype, int64_t R, int64_t C, bool sq, int64_t* info) {
  const SatPlan p = make_sat_plan(dtype, R, C, sq);
  info[0] = p.TW; info[1] = p.SR; info[2] = p.nJ; info[3] = p.nK;
}

int64_t sat_workspace_bytes(int dtype, int64_t R, int64_t C, bool sq) {
  return make_sat_plan(dtype, R, C, sq).total * 8;
}

}  // namespace ssb
