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
#define SSB_SCAN_MINB 1
#endif
#ifndef SSB_SCAN_STAGES
#define SSB_SCAN_STAGES 2
#endif
#ifndef SSB_SCAN_MINB_SQ
#define SSB_SCAN_MINB_SQ 2
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

// ---------------------------------------------------------------------------
// phase 1
#ifndef SSB_REDUCE_MINB
#define SSB_REDUCE_MINB 3
#endif
#ifndef SSB_REDUCE_MINB_SQ
#define SSB_REDUCE_MINB_SQ 2
#endif
template <typename InT, bool SQ, int RBR, int WPC>
__global__ void __launch_bounds__(32 * WPC, SQ ? SSB_REDUCE_MINB_SQ : SSB_REDUCE_MINB)
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
    if constexpr (kPacked && !SQ && (RB % 2) == 0) {
      if (fast) {
        // two rows at a time: byte pairs unpacked with LOP3 / PRMT, both rows
        // folded into the 16-bit column partials by one 3-input add each
#pragma unroll
        for (int r = 0; r < RB; r += 2) {
          uint32_t o1[NWD], o2[NWD];
          lane_bytes<G::LB>(ws.buf[s] + r * G::ROWB, qbase + ws.offs[s][r], o1);
          lane_bytes<G::LB>(ws.buf[s] + (r + 1) * G::ROWB, qbase + ws.offs[s][r + 1], o2);
          part[r] = lane_total<InT>(o1);
          part[r + 1] = lane_total<InT>(o2);
#pragma unroll
          for (int i = 0; i < NWD; ++i) {
            pk_lo[i] += (o1[i] & 0x00FF00FFu) + (o2[i] & 0x00FF00FFu);
            pk_hi[i] += __byte_perm(o1[i], 0u, 0x4341) + __byte_perm(o2[i], 0u, 0x4341);
          }
          part_sq[r] = part_sq[r + 1] = LocSq(0);
        }
      }
    }
#pragma unroll
    for (int r = 0; r < RB; ++r) {
      if constexpr (kPacked && !SQ && (RB % 2) == 0) {
        if (fast) continue;
      }
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
// one thread per column, serial down the segments (few segments: one pass over colp)
template <typename Acc>
__global__ void sat_topcarry_serial_kernel(Acc* __restrict__ colp, const Acc* __restrict__ srl, Acc* __restrict__ totals,
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

// many segments: 32 columns x kTopChunks segment chunks per CTA: each thread sums its chunk,
// an exclusive scan over the chunks gives its offset, then it rewrites its
// chunk -- kTopChunks-way parallel down the segments instead of one serial walk.
constexpr int kTopChunks = 8;
template <typename Acc>
__global__ void __launch_bounds__(32 * kTopChunks)
sat_topcarry_kernel(Acc* __restrict__ colp, const Acc* __restrict__ srl, Acc* __restrict__ totals, int nK, int nJ,
                    int64_t PC, int TW) {
  __shared__ Acc part[kTopChunks][32];
  const int c = threadIdx.x & 31, q = threadIdx.x >> 5;
  const int64_t j = (int64_t)blockIdx.x * 32 + c;
  const bool live = j < PC;
  const int J = live ? (int)(j / TW) : 0;
  const int ch = (nK + kTopChunks - 1) / kTopChunks;
  const int ka = q * ch, kb = min(nK, ka + ch);
  Acc sum = Acc(0);
  if (live) {
    for (int K = ka; K < kb; ++K) sum = add(sum, add(colp[(int64_t)K * PC + j], srl[(int64_t)K * nJ + J]));
  }
  part[q][c] = sum;
  __syncthreads();
  Acc run = Acc(0);
  for (int p = 0; p < q; ++p) run = add(run, part[p][c]);
  if (live) {
    for (int K = ka; K < kb; ++K) {
      const Acc v = add(colp[(int64_t)K * PC + j], srl[(int64_t)K * nJ + J]);
      colp[(int64_t)K * PC + j] = run;
      run = add(run, v);
    }
    if (totals && q == kTopChunks - 1) totals[j] = run;
  }
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

template <typename InT, bool SQ>
__global__ void __launch_bounds__(kThreads, SQ ? SSB_SCAN_MINB_SQ : SSB_SCAN_MINB)
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
  using WS = WarpStage<InT, 0, SSB_SCAN_STAGES>;
  constexpr int TW = G::TW, E = G::E, RB = WS::RBW, NSTG = WS::NSTG;
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
#pragma unroll
  for (int pb = 0; pb < NSTG - 1; ++pb) {
    if (pb < nblk) {
      const int64_t rp = k0 + (int64_t)pb * RB;
      stage_issue<InT, RB>(ws.buf[pb], ws.offs[pb], &ws.bar[pb], in, R, C, in_ld, rp, (int)min64(RB, k1 - rp), j0,
                           lane);
    }
  }

  Acc acc[E], accq[E];
#pragma unroll
  for (int k = 0; k < E; ++k) {
    acc[k] = cbase + k < PC ? top[(int64_t)K * PC + cbase + k] : Acc(0);
    if constexpr (SQ) accq[k] = cbase + k < PC ? top_sq[(int64_t)K * PC + cbase + k] : Acc(0);
  }
  const bool writes_plain = sat != nullptr;

  for (int b = 0; b < nblk; ++b) {
    const int s = b % NSTG;
    const int64_t r0 = k0 + (int64_t)b * RB;
    const int nr = (int)min64(RB, k1 - r0);
    if (b + NSTG - 1 < nblk) {  // refill the stage consumed in iteration b - 1
      const int sn = (b + NSTG - 1) % NSTG;
      const int64_t rn = r0 + (int64_t)(NSTG - 1) * RB;
      stage_issue<InT, RB>(ws.buf[sn], ws.offs[sn], &ws.bar[sn], in, R, C, in_ld, rn, (int)min64(RB, k1 - rn), j0,
                           lane);
    }
    Acc rlv = Acc(0), rlqv = Acc(0);  // lane r: left carry of row r
    if (lane < nr) {
      rlv = rl[(r0 + lane) * nJ + J];
      if constexpr (SQ) rlqv = rl_sq[(r0 + lane) * nJ + J];
    }
    mbar_wait(&ws.bar[s], (uint32_t)((b / NSTG) & 1));
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
// Single pass (integer kinds): one kernel reads every pixel once and writes
// every table entry once, with decoupled look-back carries across CTA tiles
// (north_star subsystem 1).
//
// Tile (J, K) = SR table rows x TW table columns, handed out by an atomic
// ticket in (K, J) order, so a tile only ever waits on tiles with smaller
// tickets, which are already resident: no deadlock for any grid size.
//   1. TMA-stage the tile's SR image rows into shared memory (kept for step 5).
//   2. Per warp (RPW rows): row totals and column sums (packed for u8).
//      Publish the row totals (horizontal aggregate, flag 1).
//   3. Horizontal look-back over strips J-1, J-2, ...: add aggregates until a
//      published inclusive prefix (flag 2) -> left carry RL of each row.
//      Publish RL + row totals (flag 2).
//   4. Vertical aggregate V[j] = sum_rows RL + strip-local prefix of the
//      tile's column sums; publish (flag 1).  Vertical look-back over
//      segments K-1, K-2, ... -> Top[j] (table row above the tile).  Publish
//      Top + V (= the tile's bottom table row, flag 2) before writing.
//   5. Per warp: scan the staged rows, accumulating down the columns in
//      registers, 256-bit streaming stores of every table row.
// Integer tables are exact modulo 2^64, so the look-back's summation order
// (which depends on timing) cannot change a single bit.  F32 input keeps the
// reduce-then-scan pipeline, whose fp64 summation order is fixed.
// CTA = 8 worker warps (staging, pass 1, pass 2: the table stores) + 1 control
// warp that owns every published value, flag and look-back.  The control warp
// never issues table stores, so its release fences do not wait for the
// streaming writes of the workers to drain.
#ifndef SSB_ONE_WORKERS
#define SSB_ONE_WORKERS 8
#endif
constexpr int kOneWorkers = SSB_ONE_WORKERS;
constexpr int kOneThreads = 32 * (kOneWorkers + 1);

template <typename InT>
struct OneGeo {
  using G = Geo<InT>;
  static constexpr int TW = G::TW;
  static constexpr int E = G::E;                       // columns per lane
  static constexpr int SR = (G::ES == 1 ? 16 : 8) * kOneWorkers;  // tile rows (16 / 8 per worker warp)
  static constexpr int NW = kOneWorkers;               // worker warps
  static constexpr int RPW = SR / NW;                  // rows per worker warp
  static constexpr int HPL = SR / 32;                  // row values per lane (horizontal look-back)
  static constexpr int CPT = TW / (32 * NW);           // columns per worker thread (column scan)
};

struct OneWs {
  unsigned int* ticket;
  unsigned int* flag_h;
  unsigned int* flag_v;
  uint64_t* h_agg;  // [nT][SR]
  uint64_t* h_inc;
  uint64_t* v_agg;  // [nT][TW]
  uint64_t* v_inc;
  uint64_t* hq_agg;
  uint64_t* hq_inc;
  uint64_t* vq_agg;
  uint64_t* vq_inc;
};

#ifdef SSB_ONEPASS_PROF
// tuning build only: per-phase time of the single-pass kernel (ns, summed over tiles)
__device__ unsigned long long g_onepass_prof[8];
__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define ONEPASS_MARK(i) do { if (tid == 0) { const unsigned long long _n = gtime(); atomicAdd(&g_onepass_prof[i], _n - _pt); _pt = _n; } } while (0)
#define CTRL_T0() unsigned long long _c0 = gtime()
#define CTRL_MARK(i) do { if (lane == 0) { const unsigned long long _n = gtime(); atomicAdd(&g_onepass_prof[i], _n - _c0); _c0 = _n; } } while (0)
#else
#define ONEPASS_MARK(i) do { } while (0)
#define CTRL_T0() do { } while (0)
#define CTRL_MARK(i) do { } while (0)
#endif

__device__ __forceinline__ unsigned int ld_acquire_u32(const unsigned int* p) {
  unsigned int v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_u32(unsigned int* p, unsigned int v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

template <typename InT, bool SQ>
struct OneSmem {
  using Tr = Elem<InT>;
  using O = OneGeo<InT>;
  using G = Geo<InT>;
  alignas(16) unsigned char stage[O::SR * G::ROWB];
  typename Tr::Loc cs[O::NW][O::TW];                 // per-warp column sums -> exclusive over warps
  typename Tr::LocSq csq[SQ ? O::NW : 1][SQ ? O::TW : 1];
  typename Tr::Loc tot[O::TW];                        // tile column totals
  typename Tr::LocSq totq[SQ ? O::TW : 1];
  uint64_t rt[O::SR], rtq[SQ ? O::SR : 1];            // row totals
  uint64_t rl[O::SR], rlq[SQ ? O::SR : 1];            // row left carries
  uint64_t top[O::TW], topq[SQ ? O::TW : 1];          // table row above the tile
  uint64_t rlb[O::NW + 1], rlbq[O::NW + 1];           // sum of RL over the rows before each warp
  int offs[O::SR];
  uint64_t bar[O::NW];
  int ticket;
};

// lane-serial + warp exclusive scan of E per-lane values (strip-local prefix)
template <int E, typename T>
__device__ __forceinline__ void strip_prefix(const T (&v)[E], uint64_t (&o)[E], int lane) {
  uint64_t run = 0;
#pragma unroll
  for (int k = 0; k < E; ++k) { run += (uint64_t)v[k]; o[k] = run; }
  const uint64_t ex = warp_incl_scan(run, lane) - run;
#pragma unroll
  for (int k = 0; k < E; ++k) o[k] += ex;
}

template <int E>
__device__ __forceinline__ void ld_lane_vec(const uint64_t* p, uint64_t (&v)[E]) {
#pragma unroll
  for (int k = 0; k < E; k += 2) {
    const ulonglong2 x = __ldcg(reinterpret_cast<const ulonglong2*>(p + k));
    v[k] = x.x;
    v[k + 1] = x.y;
  }
}
template <int E>
__device__ __forceinline__ void st_lane_vec(uint64_t* p, const uint64_t (&v)[E]) {
#pragma unroll
  for (int k = 0; k < E; k += 2) __stcg(reinterpret_cast<ulonglong2*>(p + k), make_ulonglong2(v[k], v[k + 1]));
}

template <typename InT, bool SQ>
__global__ void __launch_bounds__(kOneThreads, SQ ? 1 : (kOneWorkers <= 4 ? 4 : 2))
sat_onepass_kernel(const InT* __restrict__ in, int64_t R, int64_t C, int64_t in_ld, uint64_t* __restrict__ sat,
                   uint64_t* __restrict__ sat_sq, int64_t sat_ld, const uint64_t* __restrict__ carry,
                   const uint64_t* __restrict__ carry_sq, OneWs ws, int nJ, int nK) {
  using Tr = Elem<InT>;
  using Loc = typename Tr::Loc;
  using LocSq = typename Tr::LocSq;
  using O = OneGeo<InT>;
  using G = Geo<InT>;
  constexpr int TW = O::TW, E = O::E, SR = O::SR, RPW = O::RPW, NW = O::NW;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  OneSmem<InT, SQ>& sm = *reinterpret_cast<OneSmem<InT, SQ>*>(smem_raw);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const bool control = warp == NW;
  const int64_t PR = R + 1, PC = C + 1;
  const int nT = nJ * nK;
  if (!control && lane == 0) mbar_init(&sm.bar[warp], 1);
  fence_mbar_init();
  __syncthreads();
  uint32_t phase = 0;
  const bool writes_plain = sat != nullptr;
#ifdef SSB_ONEPASS_PROF
  unsigned long long _pt = gtime();
#endif
  for (;; phase ^= 1u) {
    if (tid == 0) sm.ticket = (int)atomicAdd(ws.ticket, 1u);
    __syncthreads();  // S0 (also: every warp is done with the previous tile)
    const int t = sm.ticket;
    if (t >= nT) break;
    const int K = t / nJ, J = t - K * nJ;
    const int64_t j0 = (int64_t)J * TW, k0 = (int64_t)K * SR;
    const int nr = (int)min64(SR, PR - k0);
    const int rw0 = warp * RPW;  // first tile row of this (worker) warp
    const int64_t cbase = j0 + lane * E;  // table column of the lane's first element
    const int64_t c0 = cbase - 1;
    ONEPASS_MARK(0);
    if (!control) {
      // 1. each worker stages its own RPW rows (lane q -> row rw0 + q)
      stage_issue<InT, RPW>(sm.stage + rw0 * G::ROWB, sm.offs + rw0, &sm.bar[warp], in, R, C, in_ld, k0 + rw0,
                            max(0, min(RPW, nr - rw0)), j0, lane);
      mbar_wait(&sm.bar[warp], phase);
      ONEPASS_MARK(1);
      // 2. row totals + column sums of the warp's rows
      Loc part[RPW];
      LocSq partq[RPW];
      Loc cs[E];
      LocSq csq[E];
#pragma unroll
      for (int k = 0; k < E; ++k) { cs[k] = Loc(0); csq[k] = LocSq(0); }
      constexpr bool kPacked = sizeof(InT) == 1;
      constexpr int NWD = Pack<InT>::NW;
      uint32_t pk_lo[kPacked ? NWD : 1], pk_hi[kPacked ? NWD : 1];
#pragma unroll
      for (int i = 0; i < (kPacked ? NWD : 1); ++i) { pk_lo[i] = 0u; pk_hi[i] = 0u; }
#pragma unroll
      for (int r = 0; r < RPW; ++r) {
        part[r] = Loc(0);
        partq[r] = LocSq(0);
        if (rw0 + r < nr) {
          uint32_t o[NWD];
          lane_words<InT>(sm.stage, sm.offs, rw0 + r, c0, C, o);
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
            partq[r] = lane_total_sq<InT>(o);
#pragma unroll
            for (int k = 0; k < E; ++k) csq[k] = add(csq[k], convsq<LocSq>(elem<InT>(o, k)));
          }
        }
      }
      if constexpr (kPacked) {
#pragma unroll
        for (int i = 0; i < NWD; ++i) {
          cs[4 * i + 0] = pk_lo[i] & 0xFFFFu;
          cs[4 * i + 2] = pk_lo[i] >> 16;
          cs[4 * i + 1] = pk_hi[i] & 0xFFFFu;
          cs[4 * i + 3] = pk_hi[i] >> 16;
        }
      }
      const Loc rs = warp_reduce_scatter<RPW>(part, lane);
      const int myrow = lane / (32 / RPW);
      const bool writer = (lane % (32 / RPW)) == 0;
      if (writer) sm.rt[rw0 + myrow] = (uint64_t)rs;
      if constexpr (SQ) {
        const LocSq rq = warp_reduce_scatter<RPW>(partq, lane);
        if (writer) sm.rtq[rw0 + myrow] = (uint64_t)rq;
      }
#pragma unroll
      for (int k = 0; k < E; ++k) {
        sm.cs[warp][lane * E + k] = cs[k];
        if constexpr (SQ) sm.csq[warp][lane * E + k] = csq[k];
      }
    }
    __syncthreads();  // S1
    ONEPASS_MARK(2);
    if (control) {
      CTRL_T0();
      // publish the horizontal aggregate (row totals)
#pragma unroll
      for (int q = 0; q < O::HPL; ++q) {
        const int r = lane + 32 * q;
        __stcg(ws.h_agg + (int64_t)t * SR + r, sm.rt[r]);
        if constexpr (SQ) __stcg(ws.hq_agg + (int64_t)t * SR + r, sm.rtq[r]);
      }
      __threadfence();
      __syncwarp();
      if (lane == 0) st_release_u32(ws.flag_h + t, 1u);
      CTRL_MARK(4);
      // 3. warp-wide horizontal look-back: lane i examines strip jj - i, so one
      // round sees 32 predecessors; the aggregates up to the nearest inclusive
      // prefix are then summed with independent loads
      uint64_t hl[O::HPL], hq[O::HPL];
#pragma unroll
      for (int q = 0; q < O::HPL; ++q) { hl[q] = 0; hq[q] = 0; }
      for (int jj = J - 1; jj >= 0;) {
        const int my = jj - lane;
        const unsigned int f = my >= 0 ? ld_acquire_u32(ws.flag_h + K * nJ + my) : 2u;  // strip -1: carry 0
        const unsigned int pre = __ballot_sync(0xffffffffu, f == 2u);
        const unsigned int wait = __ballot_sync(0xffffffffu, f == 0u);
        const int p = pre ? __ffs(pre) - 1 : 32;    // nearest inclusive prefix
        const int q = wait ? __ffs(wait) - 1 : 32;  // nearest strip not yet published
        const int use = p < q ? p : q;               // strips jj .. jj-use+1 contribute aggregates
        __syncwarp();
        for (int i = 0; i < use; ++i) {
          const int64_t idx = (int64_t)(K * nJ + jj - i) * SR;
#pragma unroll
          for (int qq = 0; qq < O::HPL; ++qq) {
            hl[qq] += __ldcg(ws.h_agg + idx + lane + 32 * qq);
            if constexpr (SQ) hq[qq] += __ldcg(ws.hq_agg + idx + lane + 32 * qq);
          }
        }
        if (p < q) {
          if (jj - p >= 0) {
            const int64_t idx = (int64_t)(K * nJ + jj - p) * SR;
#pragma unroll
            for (int qq = 0; qq < O::HPL; ++qq) {
              hl[qq] += __ldcg(ws.h_inc + idx + lane + 32 * qq);
              if constexpr (SQ) hq[qq] += __ldcg(ws.hq_inc + idx + lane + 32 * qq);
            }
          }
          break;
        }
        jj -= use;
        if (use == 0) __nanosleep(32);
      }
      CTRL_MARK(7);
#pragma unroll
      for (int q = 0; q < O::HPL; ++q) {
        const int r = lane + 32 * q;
        sm.rl[r] = hl[q];
        __stcg(ws.h_inc + (int64_t)t * SR + r, hl[q] + sm.rt[r]);
        if constexpr (SQ) {
          sm.rlq[r] = hq[q];
          __stcg(ws.hq_inc + (int64_t)t * SR + r, hq[q] + sm.rtq[r]);
        }
      }
      __threadfence();
      __syncwarp();
      if (lane == 0) st_release_u32(ws.flag_h + t, 2u);
      // RL summed over the rows before each worker warp (rows past the tile carry 0)
      uint64_t bsum = 0, bsq = 0;
      if (lane < NW) {
        for (int r = 0; r < RPW; ++r) {
          const int rr = lane * RPW + r;
          if (rr < nr) { bsum += sm.rl[rr]; if constexpr (SQ) bsq += sm.rlq[rr]; }
        }
      }
      const uint64_t ib = warp_incl_scan(bsum, lane), ibq = warp_incl_scan(bsq, lane);
      if (lane <= NW) {
        sm.rlb[lane] = ib - bsum;
        if constexpr (SQ) sm.rlbq[lane] = ibq - bsq;
      }
    } else {
      // exclusive scan of the column sums over the worker warps; tile totals
#pragma unroll
      for (int q = 0; q < O::CPT; ++q) {
        const int col = tid + 32 * NW * q;
        Loc run = Loc(0);
        LocSq runq = LocSq(0);
#pragma unroll
        for (int w = 0; w < NW; ++w) {
          const Loc v = sm.cs[w][col];
          sm.cs[w][col] = run;
          run = add(run, v);
          if constexpr (SQ) {
            const LocSq vq = sm.csq[w][col];
            sm.csq[w][col] = runq;
            runq = add(runq, vq);
          }
        }
        sm.tot[col] = run;
        if constexpr (SQ) sm.totq[col] = runq;
      }
    }
    __syncthreads();  // S2
    ONEPASS_MARK(3);
    if (control) {
      // 4. vertical aggregate V = strip-local prefix of the column totals + sum of RL;
      // lane l owns table columns [l*E, l*E + E) of the strip
      uint64_t vag[E], vagq[E], tp[E], tpq[E];
      {
        Loc v[E];
#pragma unroll
        for (int k = 0; k < E; ++k) v[k] = sm.tot[lane * E + k];
        strip_prefix<E>(v, vag, lane);
        const uint64_t rl_all = sm.rlb[NW];
#pragma unroll
        for (int k = 0; k < E; ++k) { vag[k] += rl_all; tp[k] = 0; tpq[k] = 0; }
        st_lane_vec<E>(ws.v_agg + (int64_t)t * TW + lane * E, vag);
        if constexpr (SQ) {
          LocSq vq[E];
#pragma unroll
          for (int k = 0; k < E; ++k) vq[k] = sm.totq[lane * E + k];
          strip_prefix<E>(vq, vagq, lane);
          const uint64_t rlq_all = sm.rlbq[NW];
#pragma unroll
          for (int k = 0; k < E; ++k) vagq[k] += rlq_all;
          st_lane_vec<E>(ws.vq_agg + (int64_t)t * TW + lane * E, vagq);
        }
      }
      __threadfence();
      __syncwarp();
      if (lane == 0) st_release_u32(ws.flag_v + t, 1u);
      int kk = K - 1;
      for (; kk >= 0; --kk) {
        const int idx = kk * nJ + J;
        unsigned int f = 0;
        if (lane == 0) {
          while ((f = ld_acquire_u32(ws.flag_v + idx)) == 0u) __nanosleep(32);
        }
        __syncwarp();
        f = __shfl_sync(0xffffffffu, f, 0);
        uint64_t v[E];
        ld_lane_vec<E>((f == 2u ? ws.v_inc : ws.v_agg) + (int64_t)idx * TW + lane * E, v);
#pragma unroll
        for (int k = 0; k < E; ++k) tp[k] += v[k];
        if constexpr (SQ) {
          ld_lane_vec<E>((f == 2u ? ws.vq_inc : ws.vq_agg) + (int64_t)idx * TW + lane * E, v);
#pragma unroll
          for (int k = 0; k < E; ++k) tpq[k] += v[k];
        }
        if (f == 2u) break;
      }
      if (kk < 0 && carry) {
#pragma unroll
        for (int k = 0; k < E; ++k) {
          if (cbase + k < PC) {
            tp[k] += carry[cbase + k];
            if constexpr (SQ) if (carry_sq) tpq[k] += carry_sq[cbase + k];
          }
        }
      }
      uint64_t inc[E];
#pragma unroll
      for (int k = 0; k < E; ++k) { sm.top[lane * E + k] = tp[k]; inc[k] = tp[k] + vag[k]; }
      st_lane_vec<E>(ws.v_inc + (int64_t)t * TW + lane * E, inc);
      if constexpr (SQ) {
#pragma unroll
        for (int k = 0; k < E; ++k) { sm.topq[lane * E + k] = tpq[k]; inc[k] = tpq[k] + vagq[k]; }
        st_lane_vec<E>(ws.vq_inc + (int64_t)t * TW + lane * E, inc);
      }
      __threadfence();
      __syncwarp();
      if (lane == 0) st_release_u32(ws.flag_v + t, 2u);
    }
    __syncthreads();  // S3
    ONEPASS_MARK(5);
    if (!control) {
      // 5. scan the warp's rows and write them
      uint64_t acc[E], accq[E];
      {
        Loc v[E];
        uint64_t cp[E];
#pragma unroll
        for (int k = 0; k < E; ++k) v[k] = sm.cs[warp][lane * E + k];
        strip_prefix<E>(v, cp, lane);
        const uint64_t before = sm.rlb[warp];
#pragma unroll
        for (int k = 0; k < E; ++k) acc[k] = sm.top[lane * E + k] + before + cp[k];
        if constexpr (SQ) {
          LocSq vq[E];
#pragma unroll
          for (int k = 0; k < E; ++k) vq[k] = sm.csq[warp][lane * E + k];
          strip_prefix<E>(vq, cp, lane);
          const uint64_t bq = sm.rlbq[warp];
#pragma unroll
          for (int k = 0; k < E; ++k) accq[k] = sm.topq[lane * E + k] + bq + cp[k];
        }
      }
      for (int r = 0; r < RPW; ++r) {
        const int rr = rw0 + r;
        if (rr >= nr) break;
        uint32_t o[Pack<InT>::NW];
        lane_words<InT>(sm.stage, sm.offs, rr, c0, C, o);
        const int64_t row = k0 + rr;
        {
          const Loc tt = lane_total<InT>(o);
          Loc run = sub(warp_incl_scan(tt, lane), tt);
          const uint64_t left = sm.rl[rr];
#pragma unroll
          for (int k = 0; k < E; ++k) {
            run = add(run, conv<Loc>(elem<InT>(o, k)));
            acc[k] += left + (uint64_t)run;
          }
          if (writes_plain) store_lane_cols<uint64_t, E>(sat + row * sat_ld + cbase, acc, cbase, PC);
        }
        if constexpr (SQ) {
          const LocSq tt = lane_total_sq<InT>(o);
          LocSq run = sub(warp_incl_scan(tt, lane), tt);
          const uint64_t left = sm.rlq[rr];
#pragma unroll
          for (int k = 0; k < E; ++k) {
            run = add(run, convsq<LocSq>(elem<InT>(o, k)));
            accq[k] += left + (uint64_t)run;
          }
          store_lane_cols<uint64_t, E>(sat_sq + row * sat_ld + cbase, accq, cbase, PC);
        }
      }
    }
    ONEPASS_MARK(6);
  }
}

struct OnePlan {
  int TW, SR, nJ, nK;
  int64_t nT;
  int64_t bytes;  // workspace
};

inline OnePlan make_one_plan(int dtype, int64_t R, int64_t C, bool sq) {
  OnePlan p{};
  p.TW = (dtype == IN_U8 || dtype == IN_U16) ? 512 : 256;
  p.SR = (dtype == IN_U8 ? 16 : 8) * kOneWorkers;
  p.nJ = (int)((C + 1 + p.TW - 1) / p.TW);
  p.nK = (int)((R + 1 + p.SR - 1) / p.SR);
  p.nT = (int64_t)p.nJ * p.nK;
  const int64_t flags = 16 + ((2 * p.nT * 4 + 15) / 16) * 16;
  p.bytes = flags + (int64_t)(sq ? 2 : 1) * p.nT * (2 * p.SR + 2 * p.TW) * 8;
  return p;
}

template <typename InT, bool SQ>
cudaError_t launch_sat_onepass_t(const void* in, int64_t R, int64_t C, int64_t in_ld, void* sat, void* sat_sq,
                                 int64_t sat_ld, const void* carry, const void* carry_sq, void* wsp, cudaStream_t st,
                                 const OnePlan& p) {
  if (p.nT >= (int64_t)INT_MAX / 2) return cudaErrorNotSupported;
  char* base = reinterpret_cast<char*>(wsp);
  OneWs ws{};
  ws.ticket = reinterpret_cast<unsigned int*>(base);
  ws.flag_h = reinterpret_cast<unsigned int*>(base + 16);
  ws.flag_v = ws.flag_h + p.nT;
  const int64_t flags = 16 + ((2 * p.nT * 4 + 15) / 16) * 16;
  uint64_t* d = reinterpret_cast<uint64_t*>(base + flags);
  ws.h_agg = d; d += p.nT * p.SR;
  ws.h_inc = d; d += p.nT * p.SR;
  ws.v_agg = d; d += p.nT * p.TW;
  ws.v_inc = d; d += p.nT * p.TW;
  if (SQ) {
    ws.hq_agg = d; d += p.nT * p.SR;
    ws.hq_inc = d; d += p.nT * p.SR;
    ws.vq_agg = d; d += p.nT * p.TW;
    ws.vq_inc = d; d += p.nT * p.TW;
  }
  cudaError_t e = cudaMemsetAsync(base, 0, (size_t)flags, st);
  if (e != cudaSuccess) return e;
  const int smem = (int)sizeof(OneSmem<InT, SQ>);
  auto kfn = sat_onepass_kernel<InT, SQ>;
  e = cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  int per_sm = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kfn, kOneThreads, smem);
  if (e != cudaSuccess || per_sm < 1) per_sm = 1;
  int64_t blocks = (int64_t)kNumSMs * per_sm;
  if (blocks > p.nT) blocks = p.nT;
  kfn<<<(int)blocks, kOneThreads, smem, st>>>(reinterpret_cast<const InT*>(in), R, C, in_ld,
                                             reinterpret_cast<uint64_t*>(sat), reinterpret_cast<uint64_t*>(sat_sq),
                                             sat_ld, reinterpret_cast<const uint64_t*>(carry),
                                             reinterpret_cast<const uint64_t*>(carry_sq), ws, p.nJ, p.nK);
  note_launch(1);
  return cudaGetLastError();
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
#ifndef SSB_TILES_PER_SM
#define SSB_TILES_PER_SM 64
#endif
  const int64_t target_tiles = (int64_t)SSB_TILES_PER_SM * kNumSMs;  // warp tiles: ~4 waves of 16 warps per SM
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
#ifndef SSB_REDUCE_WPC
#define SSB_REDUCE_WPC 8
#endif
#ifndef SSB_REDUCE_RB
#define SSB_REDUCE_RB 0
#endif
  return launch_reduce_rw<InT, SQ, SSB_REDUCE_RB, SSB_REDUCE_WPC>(x, R, C, in_ld, rowtot, rowtot_sq, colp, colp_sq,
                                                                  nonfinite, st, p);
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
  // measured: serial walk for <= 128 segments (C5: 49 vs 69 us), chunked above (C2: 46 -> 30 us)
  if (p.nK <= 128) {
    const int nb = (int)((p.PC + kThreads - 1) / kThreads);
    sat_topcarry_serial_kernel<Acc><<<nb, kThreads, 0, st>>>(colp, srl, reinterpret_cast<Acc*>(totals), p.nK, p.nJ, p.PC, p.TW);
    if (SQ) sat_topcarry_serial_kernel<Acc><<<nb, kThreads, 0, st>>>(colp_sq, srl_sq, reinterpret_cast<Acc*>(totals_sq), p.nK, p.nJ, p.PC, p.TW);
  } else {
    const int nb_top = (int)((p.PC + 31) / 32);
    sat_topcarry_kernel<Acc><<<nb_top, 32 * kTopChunks, 0, st>>>(colp, srl, reinterpret_cast<Acc*>(totals), p.nK, p.nJ, p.PC, p.TW);
    if (SQ) sat_topcarry_kernel<Acc><<<nb_top, 32 * kTopChunks, 0, st>>>(colp_sq, srl_sq, reinterpret_cast<Acc*>(totals_sq), p.nK, p.nJ, p.PC, p.TW);
  }
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
  const int smem = (int)(sizeof(WarpStage<InT, 0, SSB_SCAN_STAGES>) * kWarpsPerCta);
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

// single-pass build for integer kinds (cudaErrorNotSupported for F32 / i32 squares)
cudaError_t launch_sat_onepass(int dtype, const void* in, int64_t R, int64_t C, int64_t in_ld, void* sat, void* sat_sq,
                               int64_t sat_ld, const void* carry, const void* carry_sq, void* ws, cudaStream_t st) {
  const bool sq = sat_sq != nullptr;
  const OnePlan p = make_one_plan(dtype, R, C, sq);
  switch (dtype) {
    case IN_U8:
      return sq ? launch_sat_onepass_t<uint8_t, true>(in, R, C, in_ld, sat, sat_sq, sat_ld, carry, carry_sq, ws, st, p)
                : launch_sat_onepass_t<uint8_t, false>(in, R, C, in_ld, sat, sat_sq, sat_ld, carry, carry_sq, ws, st, p);
    case IN_U16:
      return sq ? launch_sat_onepass_t<uint16_t, true>(in, R, C, in_ld, sat, sat_sq, sat_ld, carry, carry_sq, ws, st, p)
                : launch_sat_onepass_t<uint16_t, false>(in, R, C, in_ld, sat, sat_sq, sat_ld, carry, carry_sq, ws, st, p);
    case IN_I32:
      if (sq) return cudaErrorNotSupported;
      return launch_sat_onepass_t<int32_t, false>(in, R, C, in_ld, sat, sat_sq, sat_ld, carry, carry_sq, ws, st, p);
    default:
      return cudaErrorNotSupported;
  }
}

int64_t sat_onepass_workspace_bytes(int dtype, int64_t R, int64_t C, bool sq) {
  return make_one_plan(dtype, R, C, sq).bytes;
}

bool onepass_supported(int dtype, bool sq) { return dtype == IN_U8 || dtype == IN_U16 || (dtype == IN_I32 && !sq); }

// Default: reduce-then-scan (measured faster at C5: 10.5 ms vs 12.8 ms, see
// DESIGN.md section 3); SSB_SAT_PATH=one routes ssb_sat_build through the
// single-pass look-back kernel for A/B runs.
static bool onepass_enabled(int dtype, bool sq) {
  static const bool want_one = [] {
    const char* e = getenv("SSB_SAT_PATH");
    return e && e[0] == 'o';
  }();
  return want_one && onepass_supported(dtype, sq);
}

// whole-table build (ssb_sat_build): single pass for integer kinds, reduce-then-scan otherwise
cudaError_t launch_sat_build(int dtype, const void* in, int64_t R, int64_t C, int64_t in_ld, void* sat, void* sat_sq,
                             int64_t sat_ld, const void* carry, const void* carry_sq, void* ws, int* nonfinite,
                             cudaStream_t st) {
  const bool sq = sat_sq != nullptr;
  if (onepass_enabled(dtype, sq))
    return launch_sat_onepass(dtype, in, R, C, in_ld, sat, sat_sq, sat_ld, carry, carry_sq, ws, st);
  cudaError_t e = launch_sat_prepare(dtype, in, R, C, in_ld, sq, ws, nullptr, nullptr, nonfinite, st);
  if (e != cudaSuccess) return e;
  return launch_sat_finish(dtype, in, R, C, in_ld, sat, sat_sq, sat_ld, carry, carry_sq, ws, st);
}

#ifdef SSB_ONEPASS_PROF
extern "C" int ssb_debug_onepass_prof(unsigned long long* out8, int reset) {
  cudaMemcpyFromSymbol(out8, g_onepass_prof, sizeof(unsigned long long) * 8);
  if (reset) {
    unsigned long long z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    cudaMemcpyToSymbol(g_onepass_prof, z, sizeof(z));
  }
  return 0;
}
#endif

void sat_plan_info(int dtype, int64_t R, int64_t C, bool sq, int64_t* info) {
  const SatPlan p = make_sat_plan(dtype, R, C, sq);
  info[0] = p.TW; info[1] = p.SR; info[2] = p.nJ; info[3] = p.nK;
}

// prepare/finish and ssb_sat_build (plus the single-pass needs when SSB_SAT_PATH=one routes there)
int64_t sat_workspace_bytes(int dtype, int64_t R, int64_t C, bool sq) {
  const int64_t two = make_sat_plan(dtype, R, C, sq).total * 8;
  const int64_t one = onepass_enabled(dtype, sq) ? make_one_plan(dtype, R, C, sq).bytes : 0;
  return two > one ? two : one;
}

}  // namespace ssb
