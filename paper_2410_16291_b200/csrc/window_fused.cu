// satsweep-b200: fused window statistics that never materialise the table.
//
// Same outputs as build_sat + sweep_window_sums + finalize
// (pkg/src/satsweep/integral.py:109-116, :141-163; stats.py:35-74) for stride 1,
// computed from the image directly.  The four-corner identity needs only
// *local* prefix sums: a per-column offset added to every table row cancels in
// (br - tr) and a per-row offset cancels in (bl - tl).  Each CTA
// owns a strip of output columns and a segment of output rows and keeps, per
// image column of the strip (+ w-1 halo columns), the vertical running sum of
// the last w rows in registers:
//     V[c] += x[r][c] - x[r-w][c]
// Each finished row is prefix-summed across the strip (warp shuffles + one
// cross-warp step) and out[j] = P[j+w] - P[j].  Row x[r-w] is re-read from L2.
//
// Integer sums use modular arithmetic of the narrowest width that holds the
// final window sum (u32 for u8 while w^2*255 < 2^32), so intermediate prefix
// sums may wrap without affecting the result.  f32 input uses double.
#include <cstdlib>

#include "ssb_common.cuh"
#include "ssb_stage.cuh"
#include "ssb_packed.cuh"

#ifndef SSB_FUSED_PACK_E
#define SSB_FUSED_PACK_E 2048  // uint8 packed strips: image columns per warp
#endif
#ifndef SSB_FUSED_STAGES
#define SSB_FUSED_STAGES 2
#endif
#ifndef SSB_FUSED_OUT_UNROLL
#define SSB_FUSED_OUT_UNROLL 4
#endif
#ifndef SSB_FUSED_MINB
#define SSB_FUSED_MINB 3
#endif

namespace ssb {

constexpr int kFusedOutUnroll = SSB_FUSED_OUT_UNROLL;  // outputs in flight per lane in the store loop

template <typename InT, int E>
__device__ __forceinline__ void load_cols(const InT* __restrict__ p, int64_t c0, int64_t C, bool vec_ok, InT (&x)[E]) {
  constexpr int kBytes = E * (int)sizeof(InT);
  if (vec_ok && c0 + E <= C) {
    if constexpr (kBytes == 4) {
      const uint32_t v = __ldg(reinterpret_cast<const unsigned int*>(p + c0));
      memcpy(x, &v, 4);
    } else if constexpr (kBytes == 8) {
      const uint2 v = __ldg(reinterpret_cast<const uint2*>(p + c0));
      memcpy(x, &v, 8);
    } else {
      static_assert(kBytes % 16 == 0, "vector width");
#pragma unroll
      for (int k = 0; k < kBytes / 16; ++k) {
        const uint4 v = __ldg(reinterpret_cast<const uint4*>(p + c0) + k);
        memcpy(reinterpret_cast<char*>(x) + 16 * k, &v, 16);
      }
    }
  } else {
#pragma unroll
    for (int k = 0; k < E; ++k) x[k] = (c0 + k < C) ? __ldg(p + c0 + k) : InT(0);
  }
}

template <typename VT> __device__ __forceinline__ VT tv(uint8_t x) { return (VT)x; }
template <typename VT> __device__ __forceinline__ VT tv(uint16_t x) { return (VT)x; }
template <typename VT> __device__ __forceinline__ VT tv(int32_t x) { return (VT)(int64_t)x; }
template <typename VT> __device__ __forceinline__ VT tv(float x) { return (VT)x; }

struct FusedGeom {
  int64_t R, C, in_ld, out_r, out_c;
  int w;
  int two;      // output columns per strip
  int64_t sro;  // output rows per segment
  int mask;
  int vec_ok;
  Census cz;
};

template <typename InT, typename VT, typename VQ, bool SQ, int E, int G>
struct FusedSmem {
  static constexpr int NV = kThreads * E;
  VT p[G][NV + 1];
  VQ pq[SQ ? G : 1][SQ ? NV + 1 : 1];
  VT sw[G][kThreads / 32];
  VQ swq[G][kThreads / 32];
};

template <typename InT, typename VT, typename VQ, bool SQ, int E, int G>
__global__ void __launch_bounds__(kThreads)
window_fused_kernel(const InT* __restrict__ in, FusedGeom g, WinOut o, FinalizeInt fi, int* __restrict__ nonfinite) {
  using SM = FusedSmem<InT, VT, VQ, SQ, E, G>;
  constexpr bool kFloat = Elem<InT>::kFloat;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  SM& sm = *reinterpret_cast<SM*>(smem_raw);

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t oc0 = (int64_t)blockIdx.x * g.two;
  const int64_t or0 = (int64_t)blockIdx.y * g.sro;
  const int64_t or1 = min(or0 + g.sro, g.out_r);
  const int nout = (int)((g.out_c - oc0) < g.two ? (g.out_c - oc0) : g.two);
  if (or0 >= or1 || nout <= 0) return;
  const int w = g.w;
  const int64_t c0 = oc0 + (int64_t)tid * E;  // first image column owned
  const int64_t r_end = or1 + w - 1;          // one past last input row
  int nf = 0;

  VT V[E];
  VQ Vq[E];
#pragma unroll
  for (int k = 0; k < E; ++k) { V[k] = VT(0); Vq[k] = VQ(0); }

  for (int64_t rb = or0; rb < r_end; rb += G) {
    VT S[G][E];
    VQ Q[G][E];
    // ---- vertical sliding update for G rows
#pragma unroll
    for (int gg = 0; gg < G; ++gg) {
      const int64_t r = rb + gg;
      if (r < r_end) {
        InT xn[E];
        load_cols<InT, E>(in + r * g.in_ld, c0, g.C, g.vec_ok, xn);
        if (r - w >= or0) {
          InT xo[E];
          load_cols<InT, E>(in + (r - w) * g.in_ld, c0, g.C, g.vec_ok, xo);
#pragma unroll
          for (int k = 0; k < E; ++k) {
            V[k] = sub(add(V[k], tv<VT>(xn[k])), tv<VT>(xo[k]));
            if constexpr (SQ) {
              if constexpr (kFloat) Vq[k] = sub(add(Vq[k], __dmul_rn((double)xn[k], (double)xn[k])), __dmul_rn((double)xo[k], (double)xo[k]));
              else Vq[k] = sub(add(Vq[k], tv<VQ>(xn[k]) * tv<VQ>(xn[k])), tv<VQ>(xo[k]) * tv<VQ>(xo[k]));
            }
          }
        } else {
#pragma unroll
          for (int k = 0; k < E; ++k) {
            V[k] = add(V[k], tv<VT>(xn[k]));
            if constexpr (SQ) {
              if constexpr (kFloat) Vq[k] = add(Vq[k], __dmul_rn((double)xn[k], (double)xn[k]));
              else Vq[k] = add(Vq[k], tv<VQ>(xn[k]) * tv<VQ>(xn[k]));
            }
          }
        }
        if constexpr (kFloat) {
#pragma unroll
          for (int k = 0; k < E; ++k) if (is_nonfinite(xn[k])) nf = 1;
        }
      }
      // inclusive prefix inside the thread's E columns
      VT run = VT(0);
      VQ runq = VQ(0);
#pragma unroll
      for (int k = 0; k < E; ++k) {
        run = add(run, V[k]); S[gg][k] = run;
        if constexpr (SQ) { runq = add(runq, Vq[k]); Q[gg][k] = runq; }
      }
      // warp scan of thread totals
      const VT inc = warp_incl_scan(run, lane);
      const VT exc = sub(inc, run);
#pragma unroll
      for (int k = 0; k < E; ++k) S[gg][k] = add(S[gg][k], exc);
      if (lane == 31) sm.sw[gg][warp] = inc;
      if constexpr (SQ) {
        const VQ incq = warp_incl_scan(runq, lane);
        const VQ excq = sub(incq, runq);
#pragma unroll
        for (int k = 0; k < E; ++k) Q[gg][k] = add(Q[gg][k], excq);
        if (lane == 31) sm.swq[gg][warp] = incq;
      }
    }
    __syncthreads();
    // ---- cross-warp offsets, publish P rows: P[m] = sum_{c<m} V[c]
#pragma unroll
    for (int gg = 0; gg < G; ++gg) {
      VT off = VT(0);
      VQ offq = VQ(0);
      for (int w2 = 0; w2 < warp; ++w2) {
        off = add(off, sm.sw[gg][w2]);
        if constexpr (SQ) offq = add(offq, sm.swq[gg][w2]);
      }
#pragma unroll
      for (int k = 0; k < E; ++k) {
        sm.p[gg][tid * E + k + 1] = add(off, S[gg][k]);
        if constexpr (SQ) sm.pq[gg][tid * E + k + 1] = add(offq, Q[gg][k]);
      }
      if (tid == 0) {
        sm.p[gg][0] = VT(0);
        if constexpr (SQ) sm.pq[gg][0] = VQ(0);
      }
    }
    __syncthreads();
    // ---- outputs for the rows of this group that complete a window
#pragma unroll
    for (int gg = 0; gg < G; ++gg) {
      const int64_t r = rb + gg;
      const int64_t i = r - (w - 1);
      if (r < r_end && i >= or0) {
        const int64_t base = i * o.ld + oc0;
        for (int j = tid; j < nout; j += kThreads) {
          const VT sv = sub(sm.p[gg][j + w], sm.p[gg][j]);
          VQ qv = VQ(0);
          if constexpr (SQ) qv = sub(sm.pq[gg][j + w], sm.pq[gg][j]);
          if constexpr (kFloat) {
            if (g.mask & ST_SUM) st_cs(reinterpret_cast<double*>(o.sum) + base + j, (double)sv);
            if (g.mask & ST_MEAN) st_cs(o.mean + base + j, fin_mean_f((double)sv, fi.dn, fi.inv_n));
            if (g.mask & ST_STD) st_cs(o.std_ + base + j, fin_std_f((double)sv, (double)qv, fi.dn, fi.inv_n));
          } else {
            // widen modular result: unsigned for u8/u16, sign-extended for i32
            uint64_t s64;
            if constexpr (sizeof(VT) == 4) s64 = (uint64_t)(uint32_t)sv;
            else s64 = (uint64_t)sv;
            uint64_t q64 = 0;
            if constexpr (SQ) {
              if constexpr (sizeof(VQ) == 4) q64 = (uint64_t)(uint32_t)qv;
              else q64 = (uint64_t)qv;
            }
            if (g.mask & ST_SUM) st_cs(reinterpret_cast<uint64_t*>(o.sum) + base + j, s64);
            if (g.mask & ST_MEAN) st_cs(o.mean + base + j, fin_mean_int(s64, fi));
            if (g.mask & ST_STD) st_cs(o.std_ + base + j, fin_std_int(s64, q64, fi));
          }
          census_add(g.cz.orow, g.cz.nor, i);
        }
      }
    }
    // the next group's first __syncthreads protects sm.p / sm.sw reuse
  }
  if (nf && nonfinite) atomicOr(nonfinite, 1);
}

template <typename InT, typename VT, typename VQ, bool SQ, int E, int G>
cudaError_t launch_fused_t(const void* in, FusedGeom g, WinOut o, FinalizeInt fi, int* nonfinite, int nK_override,
                           cudaStream_t st) {
  using SM = FusedSmem<InT, VT, VQ, SQ, E, G>;
  constexpr int NV = SM::NV;
  int two = NV - g.w + 1;
  two = (two / 16) * 16;
  if (two < 16) return cudaErrorInvalidValue;
  g.two = two;
  const int64_t nJ = (g.out_c + two - 1) / two;
  int64_t nK = nK_override > 0 ? nK_override : (2 * kNumSMs + nJ - 1) / nJ;
  if (nK > g.out_r) nK = g.out_r;
  if (nK < 1) nK = 1;
  g.sro = (g.out_r + nK - 1) / nK;
  nK = (g.out_r + g.sro - 1) / g.sro;
  auto kfn = window_fused_kernel<InT, VT, VQ, SQ, E, G>;
  const size_t smem = sizeof(SM);
  cudaError_t e = cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  dim3 grid((unsigned)nJ, (unsigned)nK);
  kfn<<<grid, kThreads, smem, st>>>(reinterpret_cast<const InT*>(in), g, o, fi, nonfinite);
  note_launch(1);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Strip kernel (default).  Every warp owns one output-column strip of TWo = NV
// - w + 1 columns (NV = 32 E image columns incl. the w-1 halo) and one segment
// of output rows, and sweeps it top to bottom on its own 2-deep TMA ring
// (rows r and r-w staged per step, ssb_stage.cuh).  Lane l keeps the vertical
// sums V of image columns [l E, l E + E) in registers -- for uint8 with
// w <= 256 two columns per register as 16-bit halves (V <= 65280).  Per
// finished row the lane-serial prefix + one warp scan give P, written to a
// per-warp smem buffer with one pad word per 32 (P[u] at word u + u / 32:
// lane-consecutive reads are conflict-free and advance by a constant 33 words
// per 32 outputs; the lane-contiguous writes see at most 2-way conflicts), so
// out[j] = P[j+w] - P[j] is read and stored by consecutive lanes (coalesced
// 8-byte stores).  No CTA barrier anywhere.
constexpr int kStripWarps = 4;  // warps per CTA

template <typename InT, int E, int RB, typename VT, typename VQ, bool SQ>
struct StripSmem {
  static constexpr int NV = 32 * E;
  static constexpr int ROWB = NV * (int)sizeof(InT) + 48;
  static constexpr int NSTG = SSB_FUSED_STAGES;  // ring depth (row pairs in flight + 1)
  alignas(16) unsigned char stage[NSTG][2 * RB][ROWB];
  int offs[NSTG][2 * RB];
  uint64_t bar[NSTG];
  VT p[NV + 72];                  // P[u] = sum of columns < u, at word u + u / 32 (packed path: pp())
  VQ pq[SQ ? NV + 64 : 1];
};

template <typename InT, int E, int RB, typename VT, typename VQ, bool SQ, bool PACK, int MASKT>
__global__ void __launch_bounds__(32 * kStripWarps, SSB_FUSED_MINB)
fused_strip_kernel(const InT* __restrict__ in, FusedGeom g, WinOut o, FinalizeInt fi, int nJ, int nK,
                   int* __restrict__ nonfinite) {
  using SM = StripSmem<InT, E, RB, VT, VQ, SQ>;
  constexpr int NV = SM::NV, ES = (int)sizeof(InT), NW = E * ES / 4;
  constexpr bool kFloat = Elem<InT>::kFloat;
  static_assert(!PACK || (ES == 1 && sizeof(VT) == 4), "packed vertical sums are for uint8");
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  SM& sm = reinterpret_cast<SM*>(smem_raw)[warp];
  const int t = blockIdx.x * kStripWarps + warp;
  if (t >= nJ * nK) return;
  const int J = t % nJ, K = t / nJ;
  const int w = g.w;
  const int64_t oc0 = (int64_t)J * g.two;
  const int nout = (int)min64(g.two, g.out_c - oc0);
  const int64_t or0 = (int64_t)K * g.sro, or1 = min64(or0 + g.sro, g.out_r);
  if (nout <= 0 || or0 >= or1) return;
  const int64_t r_beg = or0, r_end = or1 + w - 1;  // input rows of this segment
  const int nblk = (int)((r_end - r_beg + RB - 1) / RB);
  const int64_t c_lo = oc0, c_hi = min64(oc0 + NV, g.C);
  const int64_t c0 = oc0 + lane * E;
  const char* base = reinterpret_cast<const char*>(in);
  const char* end_valid = base + ((g.R - 1) * g.in_ld + g.C) * ES;
  if (lane == 0) {
    for (int i = 0; i < SM::NSTG; ++i) mbar_init(&sm.bar[i], 2 * RB);  // one arrival per staging lane
    fence_mbar_init();
  }
  __syncwarp();
  // lane q < RB stages new row rb+q; lane RB+q stages old row rb+q-w
  auto issue = [&](int b, int s) {
    const int64_t rb = r_beg + (int64_t)b * RB;
    const int q = lane % RB;
    const bool old = lane >= RB;
#ifdef SSB_FUSED_PROBE_OLD  // tuning probe: leaving rows read from the entering row (wrong sums; traffic as with an on-chip history)
    const int64_t r = rb + q;
#else
    const int64_t r = rb + q - (old ? w : 0);
#endif
    const bool has = lane < 2 * RB && rb + q < r_end && (!old || rb + q - w >= r_beg);
    unsigned char* dst = sm.stage[s][lane < 2 * RB ? lane : 0];
    RowSpan sp;
    if (has) sp = row_span(base + r * g.in_ld * ES, c_lo, c_hi, ES, end_valid, dst);
    if (lane < 2 * RB) sm.offs[s][lane] = has ? sp.off : kNoRow;
    lane_issue(sp, has, dst, &sm.bar[s], lane, 2 * RB);
  };
  for (int b = 0; b < SM::NSTG - 1; ++b)
    if (b < nblk) issue(b, b);

  constexpr int NVR = PACK ? E / 2 : E;  // registers holding V
  VT V[NVR];
  VQ Vq[E];
#pragma unroll
  for (int k = 0; k < NVR; ++k) V[k] = VT(0);
#pragma unroll
  for (int k = 0; k < E; ++k) Vq[k] = VQ(0);
  bool nf = false;
  const LaneRange lr = lane_range<E>(c0, g.C);
  // every row read below has data (new rows < R; leaving rows only from the
  // segment's w-th row on), so no empty-row selects.
  // 4-byte pixels: bounds from the precomputed range, shift-free aligned loads
  // (C4 2.91 -> 2.75 ms, C2 0.61 -> 0.56 ms at the time); uint8 keeps the per-row test
  // (measured 0.1 ms slower at C5 with the range)
  auto row_elems = [&](const unsigned char* rowbuf, int off, uint32_t (&x)[NW]) {
    if constexpr (ES == 4) lane_elems_ranged<InT, E, false>(rowbuf, off, c0, lr, x);
    else lane_elems_packed<InT, E, false>(rowbuf, off, c0, g.C, x);
  };
  const int ubase = lane * E + 1;                        // first P index this lane writes
  const int addr_a = lane;                               // word of P[lane]
  const int addr_b = lane + w + ((lane + w) >> 5);       // word of P[lane + w]

  for (int b = 0; b < nblk; ++b) {
    const int s = b % SM::NSTG;
    if (b + SM::NSTG - 1 < nblk) issue(b + SM::NSTG - 1, (b + SM::NSTG - 1) % SM::NSTG);
    mbar_wait(&sm.bar[s], (uint32_t)((b / SM::NSTG) & 1));
    const int64_t rb = r_beg + (int64_t)b * RB;
#pragma unroll
    for (int q = 0; q < RB; ++q) {
      const int64_t r = rb + q;
      if (r >= r_end) break;
      if (r >= r_beg + w) {  // row r-w leaves the window first (staged from the segment's w-th row on)
        uint32_t oo[NW];
        row_elems(sm.stage[s][RB + q], sm.offs[s][RB + q], oo);
        if constexpr (PACK) {
          // V[2i] holds columns 4i, 4i+2 and V[2i+1] columns 4i+1, 4i+3 (16-bit halves;
          // V >= the leaving row per column, so no borrow crosses a half)
#pragma unroll
          for (int i = 0; i < NW; ++i) {
            V[2 * i] -= (oo[i] & 0x00FF00FFu);
            V[2 * i + 1] -= ((oo[i] >> 8) & 0x00FF00FFu);
          }
        } else {
#pragma unroll
          for (int k = 0; k < E; ++k) V[k] = sub(V[k], tv<VT>(elem<InT>(oo, k)));
        }
        if constexpr (SQ) {
#pragma unroll
          for (int k = 0; k < E; ++k) {
            const InT xo = elem<InT>(oo, k);
            // x^2 of a float is exact in double, so the FMA rounds once, like mul + add
            if constexpr (kFloat) Vq[k] = __fma_rn(-(double)xo, (double)xo, Vq[k]);
            else Vq[k] = sub(Vq[k], tv<VQ>(xo) * tv<VQ>(xo));
          }
        }
      }
      {
        uint32_t on[NW];
        row_elems(sm.stage[s][q], sm.offs[s][q], on);
        if constexpr (PACK) {
#pragma unroll
          for (int i = 0; i < NW; ++i) {
            V[2 * i] += (on[i] & 0x00FF00FFu);
            V[2 * i + 1] += ((on[i] >> 8) & 0x00FF00FFu);
          }
        } else {
#pragma unroll
          for (int k = 0; k < E; ++k) {
            const InT xn = elem<InT>(on, k);
            V[k] = add(V[k], tv<VT>(xn));
            if constexpr (kFloat) nf |= is_nonfinite(xn);
          }
        }
        if constexpr (SQ) {
#pragma unroll
          for (int k = 0; k < E; ++k) {
            const InT xn = elem<InT>(on, k);
            if constexpr (kFloat) Vq[k] = __fma_rn((double)xn, (double)xn, Vq[k]);
            else Vq[k] = add(Vq[k], tv<VQ>(xn) * tv<VQ>(xn));
          }
        }
      }
      if (r < r_beg + w - 1) continue;  // window not yet complete
      const int64_t i = r - (w - 1);
      if constexpr (PACK) {
        if (g.mask == ST_SUM) {  // uint8 sums: packed prefix + paired outputs
          packed_sums_row<E>(V, sm.p, i * o.ld + oc0, reinterpret_cast<uint64_t*>(o.sum), nout, w, lane, g.cz, i);
          continue;
        }
      }
      // P[u] = sum_{c < u} V[c] at word u + u / 32; lane writes u = lane E + k + 1
      {
        auto vcol = [&](int k) -> VT {
          if constexpr (PACK) {
            const uint32_t pair = V[2 * (k >> 2) + (k & 1)];
            return (VT)((k & 2) ? (pair >> 16) : (pair & 0xFFFFu));
          } else {
            return V[k];
          }
        };
        // lane total by a pairwise tree (one short dependency chain), the
        // lanes to the left by an exclusive warp scan, then the running prefix
        VT run = warp_excl_scan(tree_sum<E, VT>(vcol), lane);
#pragma unroll
        for (int k = 0; k < E; ++k) {
          run = add(run, vcol(k));
          const int u = ubase + k;
          sm.p[u + (u >> 5)] = run;
        }
        if (lane == 0) sm.p[0] = VT(0);
      }
      if constexpr (SQ) {
        VQ run = warp_excl_scan(tree_sum<E, VQ>([&](int k) { return Vq[k]; }), lane);
#pragma unroll
        for (int k = 0; k < E; ++k) {
          run = add(run, Vq[k]);
          const int u = ubase + k;
          sm.pq[u + (u >> 5)] = run;
        }
        if (lane == 0) sm.pq[0] = VQ(0);
      }
      __syncwarp();
      // out[j] = P[j + w] - P[j], j = lane + 32 q: both words advance by 33 per q
      const int64_t obase = i * o.ld + oc0 + lane;
      const int nq = (nout - lane + 31) >> 5;
      if (!kFloat && !SQ && g.mask == ST_SUM) {
        uint64_t* dst = reinterpret_cast<uint64_t*>(o.sum) + obase;
        int a = addr_a, bw = addr_b;
#pragma unroll kFusedOutUnroll
        for (int qq = 0; qq < nq; ++qq, a += 33, bw += 33, dst += 32) {
          const VT sv = sub(sm.p[bw], sm.p[a]);
          if constexpr (sizeof(VT) == 4) st_cs(dst, (uint64_t)(uint32_t)sv);
          else st_cs(dst, (uint64_t)sv);
        }
        census_add(g.cz.orow, g.cz.nor, i, (unsigned long long)nq);  // this lane's stores of row i
      } else {
        // MASKT != 0: the stat set is a compile-time constant (no per-output tests)
        const int mk = MASKT != 0 ? MASKT : g.mask;
        int a = addr_a, bw = addr_b;
        // output pointers advance by 32 per step (no 64-bit index arithmetic
        // per output); a stat that is not requested is never dereferenced
        uint64_t* p_sum = reinterpret_cast<uint64_t*>(o.sum) + obase;
        double* p_mean = o.mean + obase;
        double* p_std = o.std_ + obase;
        for (int qq = 0; qq < nq; ++qq, a += 33, bw += 33, p_sum += 32, p_mean += 32, p_std += 32) {
          const VT sv = sub(sm.p[bw], sm.p[a]);
          VQ qv = VQ(0);
          if constexpr (SQ) qv = sub(sm.pq[bw], sm.pq[a]);
          if constexpr (kFloat) {
            if (mk & ST_SUM) st_cs(reinterpret_cast<double*>(p_sum), (double)sv);
            if (mk & ST_MEAN) st_cs(p_mean, fin_mean_f((double)sv, fi.dn, fi.inv_n));
            if (mk & ST_STD) st_cs(p_std, fin_std_f((double)sv, (double)qv, fi.dn, fi.inv_n));
          } else {
            uint64_t s64, q64 = 0;
            if constexpr (sizeof(VT) == 4) s64 = (uint64_t)(uint32_t)sv; else s64 = (uint64_t)sv;
            if constexpr (SQ) { if constexpr (sizeof(VQ) == 4) q64 = (uint64_t)(uint32_t)qv; else q64 = (uint64_t)qv; }
            if (mk & ST_SUM) st_cs(p_sum, s64);
            if (mk & ST_MEAN) st_cs(p_mean, fin_mean_int(s64, fi));
            if (mk & ST_STD) st_cs(p_std, fin_std_int(s64, q64, fi));
          }
        }
        census_add(g.cz.orow, g.cz.nor, i, (unsigned long long)nq);  // this lane's stores of row i
      }
      __syncwarp();
    }
    __syncwarp();  // stage s fully read before it is refilled
  }
  if (nf && nonfinite) atomicOr(nonfinite, 1);
}

template <typename InT, int E, typename VT, typename VQ, bool SQ, bool PACK, int MASKT = 0>
cudaError_t launch_strip_t(const void* in, FusedGeom g, WinOut o, FinalizeInt fi, int* nonfinite, int nK_override,
                           cudaStream_t st) {
  constexpr int ROWB = 32 * E * (int)sizeof(InT) + 48;
  constexpr int RB = ROWB <= 1100 ? 2 : 1;
  using SM = StripSmem<InT, E, RB, VT, VQ, SQ>;
  g.two = SM::NV - g.w + 1;
  // 4-byte pixels: strips start on 16-byte column boundaries, so rows whose
  // start is 16-byte aligned stage every lane's data 16-byte aligned
  if constexpr (sizeof(InT) == 4) g.two = g.two >= 8 ? g.two & ~3 : g.two;
  const int nJ = (int)((g.out_c + g.two - 1) / g.two);
  static const int env_k = env_int("SSB_FUSED_SEGMENTS", 0);  // tuning: row segments per strip
  if (nK_override <= 0 && env_k > 0) nK_override = env_k;
  int64_t nK = nK_override > 0 ? nK_override : (int64_t)(2 * kNumSMs * 12 + nJ - 1) / nJ;
  if (nK > g.out_r) nK = g.out_r;
  if (nK < 1) nK = 1;
  g.sro = (g.out_r + nK - 1) / nK;
  nK = (g.out_r + g.sro - 1) / g.sro;
  auto kfn = fused_strip_kernel<InT, E, RB, VT, VQ, SQ, PACK, MASKT>;
  size_t smem = sizeof(SM) * kStripWarps;
  {  // tuning: SSB_FUSED_SMEM_KB pads the CTA's shared memory to cap CTAs per SM
     // (room for a concurrent kernel's CTAs on the same SMs)
    static const long pad_kb = env_int("SSB_FUSED_SMEM_KB", 0);
    if ((size_t)pad_kb * 1024 > smem) smem = (size_t)pad_kb * 1024;
  }
  cudaError_t e = cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  const int64_t warps = (int64_t)nJ * nK;
  const int blocks = (int)((warps + kStripWarps - 1) / kStripWarps);
  kfn<<<blocks, 32 * kStripWarps, smem, st>>>(reinterpret_cast<const InT*>(in), g, o, fi, nJ, (int)nK, nonfinite);
  note_launch(1);
  return cudaGetLastError();
}

template <typename T> constexpr bool kFloat_v = Elem<T>::kFloat;

// uint8 with packed vertical sums (w <= 256, no squares): 64 bytes of raster
// per lane and row (2048-column strips); otherwise 32 bytes per lane.  Falls
// back to the CTA kernel below when fewer than 64 outputs per strip remain.
template <typename InT, typename VT, typename VQ, bool SQ>
bool launch_strip(const void* in, FusedGeom g, WinOut o, FinalizeInt fi, int* nonfinite, int nK, cudaStream_t st,
                  cudaError_t& err) {
  constexpr int E1 = 32 / (int)sizeof(InT);
  if constexpr (sizeof(InT) == 1 && sizeof(VT) == 4 && !SQ) {
    if (g.w <= 256 && SSB_FUSED_PACK_E - 256 + 1 >= 64) {
      err = launch_strip_t<InT, SSB_FUSED_PACK_E / 32, VT, VQ, SQ, true>(in, g, o, fi, nonfinite, nK, st);
      return true;
    }
  }
  // 4-byte elements with wide windows: 512-column strips (16 per lane), so the
  // w-1 halo columns cost less than with 256 (C2: w=100, C4: w=64)
  if constexpr (sizeof(InT) == 4) {
    static const bool wide = env_int("SSB_FUSED_WIDE", 1) != 0;  // tuning: 0 keeps 256-column strips
    if (wide && g.w > 48 && 32 * 2 * E1 - g.w + 1 >= 64) {
      // the BASELINE stat sets get a compile-time mask: C4 mean + std, C2 sum + mean
      if (kFloat_v<InT> && SQ && g.mask == (ST_MEAN | ST_STD))
        err = launch_strip_t<InT, 2 * E1, VT, VQ, SQ, false, ST_MEAN | ST_STD>(in, g, o, fi, nonfinite, nK, st);
      else if (!SQ && g.mask == (ST_SUM | ST_MEAN))
        err = launch_strip_t<InT, 2 * E1, VT, VQ, SQ, false, ST_SUM | ST_MEAN>(in, g, o, fi, nonfinite, nK, st);
      else
        err = launch_strip_t<InT, 2 * E1, VT, VQ, SQ, false>(in, g, o, fi, nonfinite, nK, st);
      return true;
    }
  }
  if (32 * E1 - g.w + 1 < 64) return false;
  err = launch_strip_t<InT, E1, VT, VQ, SQ, false>(in, g, o, fi, nonfinite, nK, st);
  return true;
}

// rows per group: keep the G x E snapshot registers at <= 64 32-bit registers
template <typename VT, typename VQ, bool SQ, int E>
constexpr int fused_group() {
  constexpr int words = E * ((int)sizeof(VT) + (SQ ? (int)sizeof(VQ) : 0)) / 4;
  constexpr int g = 64 / words;
  return g >= 8 ? 8 : g >= 4 ? 4 : g >= 2 ? 2 : 1;
}

template <typename InT, typename VT, typename VQ, bool SQ>
cudaError_t launch_fused_e(const void* in, FusedGeom g, WinOut o, FinalizeInt fi, int* nonfinite, int nK, cudaStream_t st) {
  static const bool cta = env_char("SSB_FUSED_PATH") == 'c';  // tuning: "cta" forces the CTA kernel
  if (!cta) {
    cudaError_t err = cudaSuccess;
    if (launch_strip<InT, VT, VQ, SQ>(in, g, o, fi, nonfinite, nK, st, err)) return err;
  }
  if (g.w <= 256) return launch_fused_t<InT, VT, VQ, SQ, 4, fused_group<VT, VQ, SQ, 4>()>(in, g, o, fi, nonfinite, nK, st);
  if (g.w <= 1024) return launch_fused_t<InT, VT, VQ, SQ, 8, fused_group<VT, VQ, SQ, 8>()>(in, g, o, fi, nonfinite, nK, st);
  return launch_fused_t<InT, VT, VQ, SQ, 16, fused_group<VT, VQ, SQ, 16>()>(in, g, o, fi, nonfinite, nK, st);
}

// Largest window the fused path accepts (wider windows go through the table).
constexpr int kFusedMaxW = 3072;

cudaError_t launch_window_fused(const void* in, int dtype, int64_t R, int64_t C, int64_t in_ld, int64_t w, int mask,
                                WinOut o, int* nonfinite, int nK, cudaStream_t st) {
  if (w < 1 || w > kFusedMaxW) return cudaErrorInvalidValue;
  FusedGeom g{};
  g.R = R; g.C = C; g.in_ld = in_ld; g.w = (int)w; g.mask = mask;
  g.cz = census_sink();
  g.out_r = R - w + 1; g.out_c = C - w + 1;
  const int es = dtype == IN_U8 ? 1 : dtype == IN_U16 ? 2 : 4;
  const int E = w <= 256 ? 4 : w <= 1024 ? 8 : 16;
  int vb = E * es; if (vb > 16) vb = 16;
  g.vec_ok = ((reinterpret_cast<uintptr_t>(in) % vb) == 0) && (((in_ld * es) % vb) == 0);
  const bool sq = (mask & ST_STD) != 0;
  FinalizeInt fi{};
  fi.n = (uint64_t)(w * w);
  fi.dn = (double)(w * w);
  fi.inv_n = 1.0 / fi.dn;
  const double maxv = dtype == IN_U8 ? 255.0 : dtype == IN_U16 ? 65535.0 : 2147483648.0;
  fi.u64_ok = ((unsigned __int128)(uint64_t)(w * w) * (uint64_t)maxv) <= (unsigned __int128)0xFFFFFFFFull;
  fi.is_signed = dtype == IN_I32;
  const unsigned __int128 ww = (unsigned __int128)(uint64_t)(w * w);
  switch (dtype) {
    case IN_U8: {
      const bool s32 = ww * 255u < ((unsigned __int128)1 << 32);
      const bool q32 = ww * 65025u < ((unsigned __int128)1 << 32);
      if (!sq) return s32 ? launch_fused_e<uint8_t, uint32_t, uint32_t, false>(in, g, o, fi, nonfinite, nK, st)
                          : launch_fused_e<uint8_t, uint64_t, uint64_t, false>(in, g, o, fi, nonfinite, nK, st);
      if (s32 && q32) return launch_fused_e<uint8_t, uint32_t, uint32_t, true>(in, g, o, fi, nonfinite, nK, st);
      if (s32) return launch_fused_e<uint8_t, uint32_t, uint64_t, true>(in, g, o, fi, nonfinite, nK, st);
      return launch_fused_e<uint8_t, uint64_t, uint64_t, true>(in, g, o, fi, nonfinite, nK, st);
    }
    case IN_U16: {
      const bool s32 = ww * 65535u < ((unsigned __int128)1 << 32);
      if (!sq) return s32 ? launch_fused_e<uint16_t, uint32_t, uint64_t, false>(in, g, o, fi, nonfinite, nK, st)
                          : launch_fused_e<uint16_t, uint64_t, uint64_t, false>(in, g, o, fi, nonfinite, nK, st);
      return s32 ? launch_fused_e<uint16_t, uint32_t, uint64_t, true>(in, g, o, fi, nonfinite, nK, st)
                 : launch_fused_e<uint16_t, uint64_t, uint64_t, true>(in, g, o, fi, nonfinite, nK, st);
    }
    case IN_I32:
      if (sq) return cudaErrorInvalidValue;
      return launch_fused_e<int32_t, uint64_t, uint64_t, false>(in, g, o, fi, nonfinite, nK, st);
    case IN_F32:
      return sq ? launch_fused_e<float, double, double, true>(in, g, o, fi, nonfinite, nK, st)
                : launch_fused_e<float, double, double, false>(in, g, o, fi, nonfinite, nK, st);
    default:
      return cudaErrorInvalidValue;
  }
}

}  // namespace ssb
