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
//   phase 3  sat_scan     per warp tile: lane-serial row prefix + one warp
//                         shuffle scan per row, the column accumulation in
//                         the lane's registers (no smem transpose, no CTA
//                         barrier), 256-bit streaming stores
//                         (st.global.v4.b64; table rows 32-byte aligned).
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
#include "sat_tiles.cuh"
#include "sat_plan.cuh"

#ifndef SSB_SCAN_MINB
#define SSB_SCAN_MINB 1
#endif
#ifndef SSB_SCAN_STAGES
#define SSB_SCAN_STAGES 2
#endif
#ifndef SSB_SCAN_RB
#define SSB_SCAN_RB 0  // rows per TMA stage in the scan (0: 8 for 1-byte, 4 for wider pixels)
#endif
#ifndef SSB_SCAN_MINB_SQ
#define SSB_SCAN_MINB_SQ 2
#endif

namespace ssb {

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
#ifdef SSB_REDUCE_LOADONLY
    // tuning probe: staging only (measures the read pattern's bandwidth)
    if (lane == 0) rowtot[r0 * nJ + J] += ws.buf[s][16];
    __syncwarp();
    continue;
#endif
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
#ifndef SSB_SCAN_WPC
#define SSB_SCAN_WPC 8
#endif
constexpr int kScanWarps = SSB_SCAN_WPC;
template <typename InT, bool SQ>
__global__ void __launch_bounds__(32 * kScanWarps, SQ ? SSB_SCAN_MINB_SQ : SSB_SCAN_MINB)
sat_scan_kernel(const InT* __restrict__ in, int64_t R, int64_t C, int64_t in_ld,
                typename Elem<InT>::Acc* __restrict__ sat, typename Elem<InT>::Acc* __restrict__ sat_sq, int64_t sat_ld,
                const typename Elem<InT>::Acc* __restrict__ rl, const typename Elem<InT>::Acc* __restrict__ rl_sq,
                const typename Elem<InT>::Acc* __restrict__ top, const typename Elem<InT>::Acc* __restrict__ top_sq,
                int64_t SR, int nJ, int nK, Census cz) {
  using Tr = Elem<InT>;
  using Loc = typename Tr::Loc;
  using LocSq = typename Tr::LocSq;
  using Acc = typename Tr::Acc;
  using G = Geo<InT>;
  using WS = WarpStage<InT, SSB_SCAN_RB, SSB_SCAN_STAGES>;
  constexpr int TW = G::TW, E = G::E, RB = WS::RBW, NSTG = WS::NSTG;
  static_assert(E % 4 == 0, "256-bit stores");
  extern __shared__ __align__(16) unsigned char smem_raw[];
  WS* stages = reinterpret_cast<WS*>(smem_raw);
  const int lane = threadIdx.x & 31;
  WS& ws = stages[threadIdx.x >> 5];
  int J, K;
  warp_tile<kScanWarps>(nJ, nK, J, K);
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
#ifdef SSB_SCAN_STOREONLY
    // tuning probe: the table stores without the row arithmetic
    for (int r = 0; r < nr; ++r) {
#pragma unroll
      for (int k = 0; k < E; ++k) acc[k] = add(acc[k], (Acc)rlv);
      if (writes_plain) store_lane_cols<Acc, E>(sat + (r0 + r) * sat_ld + cbase, acc, cbase, PC);
    }
    __syncwarp();
    continue;
#endif
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
      if (cz.trow != nullptr) {  // census: table positions (row, col) this lane stored
#pragma unroll
        for (int k = 0; k < E; ++k) {
          if (cbase + k < PC) {
            census_add(cz.trow, cz.ntr, row);
            census_add(cz.tcol, cz.ntc, cbase + k);
          }
        }
      }
    }
    __syncwarp();  // stage s fully read before it is refilled
  }
}

// ---------------------------------------------------------------------------
// host-side launch (SatPlan / make_sat_plan: sat_plan.cuh)

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
  const int tb = (int)(((int64_t)p.nJ * p.nK + kScanWarps - 1) / kScanWarps);
  const int smem = (int)(sizeof(WarpStage<InT, SSB_SCAN_RB, SSB_SCAN_STAGES>) * kScanWarps);
  auto kfn = sat_scan_kernel<InT, SQ>;
  cudaError_t e = cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  kfn<<<tb, 32 * kScanWarps, smem, st>>>(reinterpret_cast<const InT*>(in), R, C, in_ld,
                                                    reinterpret_cast<Acc*>(sat), reinterpret_cast<Acc*>(sat_sq),
                                                    sat_ld, rowtot, rowtot_sq, colp, colp_sq, p.SR, p.nJ, p.nK,
                                                    census_sink());
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

// phases 1-2 on an explicit plan (the table+sweep pipeline uses taller segments)
cudaError_t launch_sat_prepare_plan(int dtype, const void* in, int64_t R, int64_t C, int64_t in_ld, bool sq, void* ws,
                                    int* nonfinite, cudaStream_t st, const SatPlan& p) {
#define CALL_T(T, S) launch_sat_prepare_t<T, S>(in, R, C, in_ld, ws, nullptr, nullptr, nonfinite, st, p)
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


// single-pass look-back build (sat_onepass.cu)
cudaError_t launch_sat_onepass(int dtype, const void* in, int64_t R, int64_t C, int64_t in_ld, void* sat, void* sat_sq,
                               int64_t sat_ld, const void* carry, const void* carry_sq, void* ws, cudaStream_t st);
int64_t sat_onepass_workspace_bytes(int dtype, int64_t R, int64_t C, bool sq);
bool onepass_supported(int dtype, bool sq);

// Default: reduce-then-scan (measured faster at C5: 10.5 ms vs 12.8 ms, see
// DESIGN.md section 3); SSB_SAT_PATH=one routes ssb_sat_build through the
// single-pass look-back kernel for A/B runs.
static bool onepass_enabled(int dtype, bool sq) {
  static const bool want_one = env_char("SSB_SAT_PATH") == 'o';
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


void sat_plan_info(int dtype, int64_t R, int64_t C, bool sq, int64_t* info) {
  const SatPlan p = make_sat_plan(dtype, R, C, sq);
  info[0] = p.TW; info[1] = p.SR; info[2] = p.nJ; info[3] = p.nK;
}

// prepare/finish and ssb_sat_build (plus the single-pass needs when SSB_SAT_PATH=one routes there)
int64_t sat_workspace_bytes(int dtype, int64_t R, int64_t C, bool sq) {
  const int64_t two = make_sat_plan(dtype, R, C, sq).total * 8;
  const int64_t one = onepass_enabled(dtype, sq) ? sat_onepass_workspace_bytes(dtype, R, C, sq) : 0;
  return two > one ? two : one;
}

}  // namespace ssb
