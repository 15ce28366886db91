// satsweep-b200: summed-area table construction on sm_100a.
//
// Replaces the reference's fill -> row cumsum -> column cumsum pipeline
// (pkg/src/satsweep/integral.py:86-116, parallel.py:106-121) with a
// reduce-then-scan design that writes every table entry exactly once:
//
//   phase 1  sat_reduce   per (strip J, segment K) tile: row totals of every
//                         table row inside the strip and the strip-local
//                         prefix of the segment's column totals.  Reads the
//                         image once; writes ~8/TW + 8/SR bytes per pixel.
//   phase 2  sat_rowcarry exclusive scan of row totals across strips
//                         (the left carry of every row in every strip),
//            sat_segsum   per-(segment, strip) sum of those left carries,
//            sat_topcarry exclusive scan down the segments of the segment
//                         column totals (the table row above each segment).
//   phase 3  sat_scan     per tile: stage RB image rows in shared memory, warp
//                         row scans, transpose through swizzled smem, column
//                         accumulation in registers, 128-bit coalesced stores.
//
// Table entry for table row i inside segment K and column j inside strip J:
//   S[i][j] = Top[K][j] + sum_{k0 <= i' <= i} ( RL[J][i'] + RPloc[i'][j] )
// where RPloc is the strip-local row prefix.  Integer tables are exact modulo
// 2^64; f32 input accumulates in double with a deterministic order.
#include "ssb_common.cuh"

namespace ssb {

// ---- shared memory layout helpers -------------------------------------------
// Row-scan lanes own E consecutive elements; the transpose buffer uses an XOR
// swizzle of 16-byte chunks so both the per-lane row writes and the
// per-thread column reads are bank-conflict free.
template <int CPL>
__device__ __forceinline__ int swz_chunk(int c) {
  if constexpr (CPL <= 1) {
    return c;
  } else {
    const int l = c / CPL, q = c % CPL;
    const int f = (CPL >= 8) ? (l & 7) : ((l / (8 / CPL)) & (CPL - 1));
    return l * CPL + (q ^ f);
  }
}

template <typename T, int TW>
struct SwzRow {
  static constexpr int kPerChunk = 16 / sizeof(T);
  static constexpr int kE = TW / 32;                      // elements per lane
  static constexpr int kCPL = kE * (int)sizeof(T) / 16;  // 16-byte chunks per lane
  __device__ static __forceinline__ int idx(int e) {
    const int c = e / kPerChunk;
    return swz_chunk<kCPL>(c) * kPerChunk + (e % kPerChunk);
  }
};

// Stage table rows [r0, r0+nr) x table cols [j0, j0+TW) of the padded image
// into smem (raw element type).  Element (r, e) <- X'[r0+r][j0+e].
template <typename InT, int TW, int RB>
__device__ __forceinline__ void stage_rows(InT (*sin)[TW], const InT* __restrict__ in, int64_t R, int64_t C,
                                           int64_t in_ld, int64_t r0, int nr, int64_t j0, int tid,
                                           int* nonfinite_local) {
  constexpr int kPer = TW / kThreads;
#pragma unroll 4
  for (int r = 0; r < nr; ++r) {
    const int64_t ir = r0 + r - 1;  // image row
    const bool row_ok = ir >= 0 && ir < R;
    const InT* rowp = in + ir * in_ld;
#pragma unroll
    for (int k = 0; k < kPer; ++k) {
      const int e = tid + k * kThreads;
      const int64_t ic = j0 + e - 1;  // image col
      InT v = InT(0);
      if (row_ok && ic >= 0 && ic < C) {
        v = __ldg(rowp + ic);
        if (is_nonfinite(v)) *nonfinite_local = 1;
      }
      sin[r][e] = v;
    }
  }
}

// ---------------------------------------------------------------------------
// phase 1
template <typename InT, bool SQ>
__global__ void __launch_bounds__(kThreads, 2)
sat_reduce_kernel(const InT* __restrict__ in, int64_t R, int64_t C, int64_t in_ld,
                  typename Elem<InT>::Acc* __restrict__ rowtot, typename Elem<InT>::Acc* __restrict__ rowtot_sq,
                  typename Elem<InT>::Acc* __restrict__ colp, typename Elem<InT>::Acc* __restrict__ colp_sq,
                  int64_t SR, int* __restrict__ nonfinite) {
  using Tr = Elem<InT>;
  using Loc = typename Tr::Loc;
  using LocSq = typename Tr::LocSq;
  using Acc = typename Tr::Acc;
  constexpr int TW = Tr::kTW;
  constexpr int RB = SQ ? 16 : 32;
  constexpr int E = TW / 32;
  constexpr int CPT = TW / kThreads;
  constexpr int NW = kThreads / 32;

  __shared__ __align__(16) InT sin[RB][TW];
  __shared__ Acc swarp[2][NW];
  __shared__ int s_nonfinite;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t PR = R + 1, PC = C + 1;
  const int J = blockIdx.x, K = blockIdx.y;
  const int64_t j0 = (int64_t)J * TW, k0 = (int64_t)K * SR;
  const int64_t k1 = min(k0 + SR, PR);
  if (tid == 0) s_nonfinite = 0;
  int nf = 0;

  Acc cs[CPT], csq[CPT];
#pragma unroll
  for (int c = 0; c < CPT; ++c) { cs[c] = Acc(0); csq[c] = Acc(0); }

  for (int64_t r0 = k0; r0 < k1; r0 += RB) {
    const int nr = (int)((k1 - r0) < RB ? (k1 - r0) : RB);
    stage_rows<InT, TW, RB>(sin, in, R, C, in_ld, r0, nr, j0, tid, &nf);
    __syncthreads();
    // column totals (thread owns columns tid*CPT ..)
    for (int r = 0; r < nr; ++r) {
#pragma unroll
      for (int c = 0; c < CPT; ++c) {
        const InT x = sin[r][tid * CPT + c];
        cs[c] = add(cs[c], conv<Acc>(x));
        if constexpr (SQ) csq[c] = add(csq[c], convsq<Acc>(x));
      }
    }
    // row totals (warp per row, lane owns E consecutive elements)
    for (int r = warp; r < nr; r += NW) {
      Loc s = Loc(0);
      LocSq q = LocSq(0);
#pragma unroll
      for (int k = 0; k < E; ++k) {
        const InT x = sin[r][lane * E + k];
        s = add(s, conv<Loc>(x));
        if constexpr (SQ) q = add(q, convsq<LocSq>(x));
      }
      s = warp_sum(s);
      if constexpr (SQ) q = warp_sum(q);
      if (lane == 0) {
        rowtot[(int64_t)J * PR + r0 + r] = (Acc)s;
        if constexpr (SQ) rowtot_sq[(int64_t)J * PR + r0 + r] = (Acc)q;
      }
    }
    __syncthreads();
  }

  // block inclusive scan of the column totals across the strip
  {
    Acc run = Acc(0), runq = Acc(0);
#pragma unroll
    for (int c = 0; c < CPT; ++c) {
      run = add(run, cs[c]); cs[c] = run;
      if constexpr (SQ) { runq = add(runq, csq[c]); csq[c] = runq; }
    }
    Acc inc = warp_incl_scan(run, lane);
    Acc incq = Acc(0);
    if constexpr (SQ) incq = warp_incl_scan(runq, lane);
    if (lane == 31) { swarp[0][warp] = inc; if constexpr (SQ) swarp[1][warp] = incq; }
    __syncthreads();
    Acc off = sub(inc, run), offq = Acc(0);
    if constexpr (SQ) offq = sub(incq, runq);
    for (int w2 = 0; w2 < warp; ++w2) {
      off = add(off, swarp[0][w2]);
      if constexpr (SQ) offq = add(offq, swarp[1][w2]);
    }
#pragma unroll
    for (int c = 0; c < CPT; ++c) {
      const int64_t col = j0 + tid * CPT + c;
      if (col < PC) {
        colp[(int64_t)K * PC + col] = add(off, cs[c]);
        if constexpr (SQ) colp_sq[(int64_t)K * PC + col] = add(offq, csq[c]);
      }
    }
  }
  if (nf) s_nonfinite = 1;
  __syncthreads();
  if (tid == 0 && s_nonfinite && nonfinite) atomicOr(nonfinite, 1);
}

// ---------------------------------------------------------------------------
// phase 2a: left carries (exclusive scan across strips), in place.
template <typename Acc>
__global__ void sat_rowcarry_kernel(Acc* __restrict__ rowtot, int nJ, int64_t PR) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= PR) return;
  Acc run = Acc(0);
  for (int J = 0; J < nJ; ++J) {
    const Acc v = rowtot[(int64_t)J * PR + i];
    rowtot[(int64_t)J * PR + i] = run;
    run = add(run, v);
  }
}

// phase 2a': per (segment, strip) sum of left carries, deterministic tree.
template <typename Acc>
__global__ void __launch_bounds__(kThreads)
sat_segsum_kernel(const Acc* __restrict__ rl, Acc* __restrict__ srl, int nJ, int64_t PR, int64_t SR) {
  __shared__ Acc sw[kThreads / 32];
  const int J = blockIdx.x, K = blockIdx.y;
  const int64_t k0 = (int64_t)K * SR, k1 = min(k0 + SR, PR);
  Acc s = Acc(0);
  for (int64_t i = k0 + threadIdx.x; i < k1; i += kThreads) s = add(s, rl[(int64_t)J * PR + i]);
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) sw[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    Acc t = Acc(0);
    for (int w = 0; w < kThreads / 32; ++w) t = add(t, sw[w]);
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
  Acc run = Acc(0);
  for (int K = 0; K < nK; ++K) {
    const Acc v = colp[(int64_t)K * PC + j];
    colp[(int64_t)K * PC + j] = run;
    run = add(run, add(v, srl[(int64_t)K * nJ + J]));
  }
  if (totals) totals[j] = run;
}

// ---------------------------------------------------------------------------
// phase 3
template <typename InT, bool SQ>
struct ScanSmem {
  using Tr = Elem<InT>;
  static constexpr int TW = Tr::kTW;
  static constexpr int RB = SQ ? 16 : 32;
  InT sin[RB][TW];
  typename Tr::Loc rp[RB][TW];
  typename Tr::LocSq rq[SQ ? RB : 1][SQ ? TW : 1];
  typename Tr::Acc rl[RB];
  typename Tr::Acc rlq[RB];
};

template <typename Acc, int CPT>
__device__ __forceinline__ void store_cols(Acc* __restrict__ dst, const Acc (&v)[CPT], int64_t col, int64_t PC) {
  if constexpr (CPT == 2) {
    if (col + 1 < PC) { st_cs2(dst, v[0], v[1]); return; }
    if (col < PC) st_cs(dst, v[0]);
  } else {
    if (col < PC) st_cs(dst, v[0]);
  }
}

template <typename InT, bool SQ>
__global__ void __launch_bounds__(kThreads, 2)
sat_scan_kernel(const InT* __restrict__ in, int64_t R, int64_t C, int64_t in_ld,
                typename Elem<InT>::Acc* __restrict__ sat, typename Elem<InT>::Acc* __restrict__ sat_sq, int64_t sat_ld,
                const typename Elem<InT>::Acc* __restrict__ rl, const typename Elem<InT>::Acc* __restrict__ rl_sq,
                const typename Elem<InT>::Acc* __restrict__ top, const typename Elem<InT>::Acc* __restrict__ top_sq,
                int64_t SR) {
  using Tr = Elem<InT>;
  using Loc = typename Tr::Loc;
  using LocSq = typename Tr::LocSq;
  using Acc = typename Tr::Acc;
  using SM = ScanSmem<InT, SQ>;
  constexpr int TW = SM::TW, RB = SM::RB, E = TW / 32, CPT = TW / kThreads, NW = kThreads / 32;
  using SwP = SwzRow<Loc, TW>;
  using SwQ = SwzRow<LocSq, TW>;

  extern __shared__ __align__(16) unsigned char smem_raw[];
  SM& sm = *reinterpret_cast<SM*>(smem_raw);

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t PR = R + 1, PC = C + 1;
  const int J = blockIdx.x, K = blockIdx.y;
  const int64_t j0 = (int64_t)J * TW, k0 = (int64_t)K * SR;
  const int64_t k1 = min(k0 + SR, PR);
  const int64_t mycol = j0 + tid * CPT;
  int nf = 0;

  Acc acc[CPT], accq[CPT];
#pragma unroll
  for (int c = 0; c < CPT; ++c) {
    const int64_t col = mycol + c;
    acc[c] = col < PC ? top[(int64_t)K * PC + col] : Acc(0);
    if constexpr (SQ) accq[c] = col < PC ? top_sq[(int64_t)K * PC + col] : Acc(0);
  }

  for (int64_t r0 = k0; r0 < k1; r0 += RB) {
    const int nr = (int)((k1 - r0) < RB ? (k1 - r0) : RB);
    stage_rows<InT, TW, RB>(sm.sin, in, R, C, in_ld, r0, nr, j0, tid, &nf);
    if (tid < nr) {
      sm.rl[tid] = rl[(int64_t)J * PR + r0 + tid];
      if constexpr (SQ) sm.rlq[tid] = rl_sq[(int64_t)J * PR + r0 + tid];
    }
    __syncthreads();

    // strip-local row prefixes, one warp per row
    for (int r = warp; r < nr; r += NW) {
      Loc p[E];
      LocSq q[E];
      Loc s = Loc(0);
      LocSq sq = LocSq(0);
#pragma unroll
      for (int k = 0; k < E; ++k) {
        const InT x = sm.sin[r][lane * E + k];
        s = add(s, conv<Loc>(x)); p[k] = s;
        if constexpr (SQ) { sq = add(sq, convsq<LocSq>(x)); q[k] = sq; }
      }
      const Loc off = sub(warp_incl_scan(s, lane), s);
      LocSq offq = LocSq(0);
      if constexpr (SQ) offq = sub(warp_incl_scan(sq, lane), sq);
#pragma unroll
      for (int k = 0; k < E; ++k) {
        sm.rp[r][SwP::idx(lane * E + k)] = add(off, p[k]);
        if constexpr (SQ) sm.rq[r][SwQ::idx(lane * E + k)] = add(offq, q[k]);
      }
    }
    __syncthreads();

    // column accumulation + stores
    for (int r = 0; r < nr; ++r) {
      const Acc rlv = sm.rl[r];
      Acc rlqv = Acc(0);
      if constexpr (SQ) rlqv = sm.rlq[r];
#pragma unroll
      for (int c = 0; c < CPT; ++c) {
        const int e = tid * CPT + c;
        acc[c] = add(acc[c], add(rlv, (Acc)sm.rp[r][SwP::idx(e)]));
        if constexpr (SQ) accq[c] = add(accq[c], add(rlqv, (Acc)sm.rq[r][SwQ::idx(e)]));
      }
      const int64_t row = r0 + r;
      if (sat != nullptr) store_cols<Acc, CPT>(sat + row * sat_ld + mycol, acc, mycol, PC);
      if constexpr (SQ) store_cols<Acc, CPT>(sat_sq + row * sat_ld + mycol, accq, mycol, PC);
    }
    __syncthreads();
  }
  (void)nf;
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
  const int RB = sq ? 16 : 32;
  const int64_t target_tiles = 4 * kNumSMs;
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

// adds a carry row to every segment's top row (row-band shards)
template <typename Acc>
__global__ void sat_apply_carry_kernel(Acc* __restrict__ colp, const Acc* __restrict__ carry, int nK, int64_t PC) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= PC) return;
  const Acc c = carry[j];
  for (int K = 0; K < nK; ++K) colp[(int64_t)K * PC + j] = add(colp[(int64_t)K * PC + j], c);
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
  dim3 grid(p.nJ, p.nK);
  sat_reduce_kernel<InT, SQ><<<grid, kThreads, 0, st>>>(x, R, C, in_ld, rowtot, rowtot_sq, colp, colp_sq, p.SR, nonfinite);
  const int nb_rows = (int)((p.PR + kThreads - 1) / kThreads);
  sat_rowcarry_kernel<Acc><<<nb_rows, kThreads, 0, st>>>(rowtot, p.nJ, p.PR);
  if (SQ) sat_rowcarry_kernel<Acc><<<nb_rows, kThreads, 0, st>>>(rowtot_sq, p.nJ, p.PR);
  sat_segsum_kernel<Acc><<<grid, kThreads, 0, st>>>(rowtot, srl, p.nJ, p.PR, p.SR);
  if (SQ) sat_segsum_kernel<Acc><<<grid, kThreads, 0, st>>>(rowtot_sq, srl_sq, p.nJ, p.PR, p.SR);
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
  const size_t smem = sizeof(ScanSmem<InT, SQ>);
  auto kfn = sat_scan_kernel<InT, SQ>;
  cudaError_t e = cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  dim3 grid(p.nJ, p.nK);
  kfn<<<grid, kThreads, smem, st>>>(reinterpret_cast<const InT*>(in), R, C, in_ld, reinterpret_cast<Acc*>(sat),
                                    reinterpret_cast<Acc*>(sat_sq), sat_ld, rowtot, rowtot_sq, colp, colp_sq, p.SR);
  note_launch(1);
  return cudaGetLastError();
}

#define SSB_SAT_DISPATCH(CALL_T)                                  \
  switch (dtype) {                                                \
    case IN_U8: return sq ? CALL_T(uint8_t, true) : CALL_T(uint8_t, false);     \
    case IN_U16: return sq ? CALL_T(uint16_t, true) : CALL_T(uint16_t, false);  \
    case IN_I32: return sq ? CALL_T(int32_t, true) : CALL_T(int32_t, false);    \
    case IN_F32: return sq ? CALL_T(float, true) : CALL_T(float, false);        \
    default: return cudaErrorInvalidValue;                        \
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
