// satsweep-b200: single-pass summed-area table build with decoupled look-back
// (ssb_sat_build_lookback; north_star subsystem 1).
// for the measured comparison with the default reduce-then-scan build
// (sat_build.cu), which shares the warp-tile helpers in sat_tiles.cuh.
#include <climits>
#include <cstdlib>
#include <type_traits>

#include "ssb_async.cuh"
#include "ssb_common.cuh"
#include "ssb_stage.cuh"
#include "sat_tiles.cuh"

namespace ssb {

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

}  // namespace ssb
