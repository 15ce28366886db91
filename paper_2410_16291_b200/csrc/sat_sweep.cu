// satsweep-b200: the integral image AND its window statistics
// (ssb_sat_build_swa / ssb_sat_build_swa_onepass).
//
// The reference builds the table (integral.py:109-116 / parallel.py:106-121)
// and then sweeps it with four-corner lookups (integral.py:141-163): 25 B/px
// at C5 (1 in + 8 table write + 8 table read + 8 out).  The window sums do not
// need the table -- a per-column offset cancels in (br - tr) and a per-row
// offset in (bl - tl) -- so both pipelines here write the table once and never
// read it back (17 B/px):
//
//   * default (launch_sat_sweep, bottom of the file): the reduce-then-scan
//     build (sat_build.cu) on the caller's stream and, concurrently on a
//     forked side stream, the fused window kernel (window_fused.cu) over the
//     raster; the fastest on B200 (C5 19.8 ms);
//   * one-pass kernel (sat_sweep_kernel): the warp that writes a table row
//     also emits the windows whose bottom corner row it is (C5 20.1 ms,
//     latency-bound).
//
// One-pass kernel.  Phase 3 of the reduce-then-scan build gives every warp a
// (strip J, segment K) tile of TWW table columns x SR table rows; the warp
// sweeps it top to bottom, lane l owning E table columns, with the vertical
// table accumulation in registers.  For the window sums the same warp keeps,
// per image column of its strip plus a halo of HW >= w - 1 columns to the
// left, the vertical sum of the last w image rows,
//     V[c] = sum_{r' in [row-w, row)} x[r'][c]   (updated by +x[row-1] - x[row-1-w]),
// so the window with bottom-right table corner (row, j+w) is
//     out[row-w][j] = (S[row][j+w] - S[row-w][j+w]) - (S[row][j] - S[row-w][j])
//                   = sum_{c in [j, j+w)} V[c]                          (any left/top carry cancels)
// = P[j+w] - P[j] over the warp-local prefix P of V (smem, one pad word per 32).
// A warp owns the outputs whose right corner column lies in its strip.  Its
// first w rows are a warm-up (V only) unless the segment starts at the top.
// Rows are staged by TMA bulk copies: per step RB new rows (row - 1) and RB
// leaving rows (row - 1 - w) over image columns [j0 - 1 - HW, j0 - 1 + TWW).
//
// Integer window sums are exact in the narrowest modular width holding the
// final sum (u32 for u8/u16 at w <= 256); the table is uint64 modulo 2^64 and
// bit-identical to sat_build.cu's.  Stats: SUM and MEAN (no squared table).
#include <cstdlib>
#include <type_traits>

#include "ssb_async.cuh"
#include "ssb_common.cuh"
#include "ssb_stage.cuh"
#include "sat_plan.cuh"
#include "sat_tiles.cuh"

#ifndef SSB_SWEEP_SPW_U8
#define SSB_SWEEP_SPW_U8 2  // uint8: build strips (512 table columns) per warp
#endif
#ifndef SSB_SWEEP_RB_U8
#define SSB_SWEEP_RB_U8 1  // uint8: rows staged per TMA step (new + leaving rows each)
#endif
#ifndef SSB_SWEEP_STAGES_U8
#define SSB_SWEEP_STAGES_U8 6  // uint8: TMA ring depth (6 x 1 row measured 1.5 % faster than 2 x 2 at C5)
#endif
#ifndef SSB_SWEEP_WPC
#define SSB_SWEEP_WPC 4
#endif
#ifndef SSB_SWEEP_MINB
#define SSB_SWEEP_MINB 2
#endif

namespace ssb {

cudaError_t launch_sat_prepare_plan(int dtype, const void* in, int64_t R, int64_t C, int64_t in_ld, bool sq, void* ws,
                                    int* nonfinite, cudaStream_t st, const SatPlan& p);

constexpr int kSweepWarps = SSB_SWEEP_WPC;
constexpr int kSweepHalo = 256;  // halo columns: windows up to 257

template <typename InT> struct SweepCfg;
// SPW = build strips per warp (the warp's table columns TWW = SPW * TW),
// RB = rows staged per step, NST = TMA ring depth, VT = modular type of the vertical sums,
// PACK = two 16-bit vertical sums per register (uint8, w <= 257)
template <> struct SweepCfg<uint8_t> {
  static constexpr int SPW = SSB_SWEEP_SPW_U8, RB = SSB_SWEEP_RB_U8, NST = SSB_SWEEP_STAGES_U8;
  using VT = uint32_t;
  static constexpr bool PACK = true;
};
template <> struct SweepCfg<uint16_t> {
  static constexpr int SPW = 1, RB = 2, NST = 2;
  using VT = uint32_t;
  static constexpr bool PACK = false;
};
template <> struct SweepCfg<int32_t> {
  static constexpr int SPW = 1, RB = 2, NST = 2;
  using VT = uint64_t;
  static constexpr bool PACK = false;
};

template <typename InT, int HW>
struct SweepGeo {
  using Cfg = SweepCfg<InT>;
  static constexpr int TWW = Geo<InT>::TW * Cfg::SPW;   // table columns per warp
  static constexpr int E = TWW / 32, EH = HW / 32;       // main / halo elements per lane
  static constexpr int ES = (int)sizeof(InT), NV = HW + TWW;
  static constexpr int ROWB = NV * ES + 48;
};

template <typename InT, int HW>
struct SweepSmem {
  using Cfg = SweepCfg<InT>;
  using VT = typename Cfg::VT;
  using SG = SweepGeo<InT, HW>;
  static constexpr int RB = Cfg::RB;
  alignas(16) unsigned char guard[64];  // a halo lane left of column 0 may read a few bytes before its row
  static constexpr int NST = Cfg::NST;  // TMA ring depth
  alignas(16) unsigned char stage[NST][2 * RB][SG::ROWB];
  int offs[NST][2 * RB];
  uint64_t bar[NST];
  VT p[SG::NV + SG::NV / 32 + 8];  // P[u] = sum_{v < u} V[v] at word u + u / 32 (packed path: pp(u + d))
};

// V +/-= one staged row's elements (NW packed words per lane).  Packed (uint8):
// V[2i] holds columns 4i, 4i+2 and V[2i+1] columns 4i+1, 4i+3 as 16-bit halves.
template <typename InT, bool PACK, bool ADD, typename VT, int NV, int NW>
__device__ __forceinline__ void vupdate(VT (&V)[NV], const uint32_t (&x)[NW]) {
  if constexpr (PACK) {
    static_assert(NV == 2 * NW, "two registers per packed word");
#pragma unroll
    for (int i = 0; i < NW; ++i) {
      const uint32_t lo = x[i] & 0x00FF00FFu, hi = (x[i] >> 8) & 0x00FF00FFu;
      if constexpr (ADD) { V[2 * i] += lo; V[2 * i + 1] += hi; }
      else { V[2 * i] -= lo; V[2 * i + 1] -= hi; }
    }
  } else {
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      const VT v = conv<VT>(elem<InT>(x, k));
      V[k] = ADD ? add(V[k], v) : sub(V[k], v);
    }
  }
}

__device__ __forceinline__ unsigned long long get4(const U64x4& v, int i) {
  return i == 0 ? v.x : i == 1 ? v.y : i == 2 ? v.z : v.w;
}
__device__ __forceinline__ void set4(U64x4& v, int i, unsigned long long x) {
  if (i == 0) v.x = x; else if (i == 1) v.y = x; else if (i == 2) v.z = x; else v.w = x;
}

// word index of P entry v: two pad words per 64 keep even v 8-byte aligned
__device__ __forceinline__ int opp(int v) { return v + 2 * (v >> 6); }

// One output row of the one-pass kernel for uint8 sums from packed vertical
// sums (Vh: the lane's EH halo columns, Vm: its E strip columns; V[2g] holds
// columns 4g, 4g+2 and V[2g+1] columns 4g+1, 4g+3 as 16-bit halves).  P index
// u (halo u = lane EH + k + 1, strip u = HW + lane E + k + 1) is stored at word
// opp(u + d), d chosen so that every output pair (j, j+1) that is 16-byte
// aligned in global memory reads its operands with 64-bit shared loads; the
// running prefix takes one DP2A per column.  orow = output of column j_lo,
// u0 = its P index.
template <int E, int EH, int HW>
__device__ __forceinline__ void onepass_packed_row(const uint32_t (&Vm)[E / 2], const uint32_t (&Vh)[EH / 2],
                                                   uint32_t* P, uint64_t* __restrict__ orow, int u0, int nout, int w,
                                                   int lane) {
  const int e = (int)((reinterpret_cast<uintptr_t>(orow) >> 3) & 1);  // first output not 16-byte aligned
  const int d = (u0 + e) & 1;
  uint32_t th = 0u, tm = 0u;
#pragma unroll
  for (int i = 0; i < EH / 2; ++i) th = __dp2a_lo(Vh[i], 0x0101u, th);
#pragma unroll
  for (int i = 0; i < E / 2; ++i) tm = __dp2a_lo(Vm[i], 0x0101u, tm);
  const uint32_t ih = warp_incl_scan(th, lane);
  const uint32_t hall = __shfl_sync(0xffffffffu, ih, 31);
  const uint32_t im = warp_incl_scan(tm, lane);
  auto write4 = [&](const uint32_t (&V)[2], uint32_t& run, int u) {
    const uint32_t r0 = __dp2a_lo(V[0], 0x0001u, run);
    const uint32_t r1 = __dp2a_lo(V[1], 0x0001u, r0);
    const uint32_t r2 = __dp2a_lo(V[0], 0x0100u, r1);
    const uint32_t r3 = __dp2a_lo(V[1], 0x0100u, r2);
    P[opp(u + d)] = r0;
    P[opp(u + 1 + d)] = r1;
    P[opp(u + 2 + d)] = r2;
    P[opp(u + 3 + d)] = r3;
    run = r3;
  };
  uint32_t run = ih - th;
#pragma unroll
  for (int q = 0; q < EH / 4; ++q) {
    const uint32_t v2[2] = {Vh[2 * q], Vh[2 * q + 1]};
    write4(v2, run, lane * EH + 4 * q + 1);
  }
  run = hall + (im - tm);
#pragma unroll
  for (int q = 0; q < E / 4; ++q) {
    const uint32_t v2[2] = {Vm[2 * q], Vm[2 * q + 1]};
    write4(v2, run, HW + lane * E + 4 * q + 1);
  }
  if (lane == 0) P[opp(d)] = 0u;
  __syncwarp();
  if (lane == 0) {
    if (e) orow[0] = (uint64_t)(P[opp(u0 + w + d)] - P[opp(u0 + d)]);
    if ((nout - e) & 1) orow[nout - 1] = (uint64_t)(P[opp(u0 + nout - 1 + w + d)] - P[opp(u0 + nout - 1 + d)]);
  }
  const int npair = (nout - e) >> 1;
  const int va = u0 + e + d + 2 * lane;  // even
  const uint32_t* pa = P + opp(va);
  uint64_t* dst = orow + e + 2 * lane;
  const int nq = (npair - lane + 31) >> 5;
  if ((w & 1) == 0) {
    const uint32_t* pb = P + opp(va + w);
#pragma unroll 4
    for (int qq = 0; qq < nq; ++qq) {
      const uint2 A = *reinterpret_cast<const uint2*>(pa + 66 * qq);
      const uint2 B = *reinterpret_cast<const uint2*>(pb + 66 * qq);
      st_cs2(dst + 64 * qq, (uint64_t)(B.x - A.x), (uint64_t)(B.y - A.y));
    }
  } else {
    const uint32_t* pb0 = P + opp(va + w);
    const uint32_t* pb1 = P + opp(va + w + 1);
#pragma unroll 4
    for (int qq = 0; qq < nq; ++qq) {
      const uint2 A = *reinterpret_cast<const uint2*>(pa + 66 * qq);
      st_cs2(dst + 64 * qq, (uint64_t)(pb0[66 * qq] - A.x), (uint64_t)(pb1[66 * qq] - A.y));
    }
  }
  __syncwarp();  // P is rewritten by the next row
}

// sum of a lane's E elements in the table's local type
template <typename InT, int E>
__device__ __forceinline__ typename Elem<InT>::Loc lane_sum(const uint32_t (&x)[E * sizeof(InT) / 4]) {
  using Loc = typename Elem<InT>::Loc;
  Loc t = Loc(0);
  if constexpr (sizeof(InT) == 1) {
#pragma unroll
    for (int i = 0; i < E / 4; ++i) t = __dp4a(x[i], 0x01010101u, t);
  } else {
#pragma unroll
    for (int k = 0; k < E; ++k) t = add(t, conv<Loc>(elem<InT>(x, k)));
  }
  return t;
}

// vertical sum of the lane's k-th column
template <bool PACK, typename VT, int NV>
__device__ __forceinline__ VT vcol(const VT (&V)[NV], int k) {
  if constexpr (PACK) {
    const uint32_t pair = V[2 * (k >> 2) + (k & 1)];
    return (VT)((k & 2) ? (pair >> 16) : (pair & 0xFFFFu));
  } else {
    return V[k];
  }
}

template <typename InT, int HW>
__global__ void __launch_bounds__(32 * kSweepWarps, SSB_SWEEP_MINB)
sat_sweep_kernel(const InT* __restrict__ in, int64_t R, int64_t C, int64_t in_ld,
                 typename Elem<InT>::Acc* __restrict__ sat, int64_t sat_ld,
                 const typename Elem<InT>::Acc* __restrict__ rl, const typename Elem<InT>::Acc* __restrict__ top,
                 int64_t top_stride, int64_t SR, int nJ, int nJw, int nK, int w, WinOut o, int mask, FinalizeInt fi) {
  using Cfg = SweepCfg<InT>;
  using VT = typename Cfg::VT;
  using Loc = typename Elem<InT>::Loc;
  using Acc = typename Elem<InT>::Acc;
  using SM = SweepSmem<InT, HW>;
  using SG = SweepGeo<InT, HW>;
  constexpr int TW = SG::TWW, E = SG::E, ES = SG::ES, RB = Cfg::RB, EH = SG::EH, SPW = Cfg::SPW;
  constexpr bool PACK = Cfg::PACK;
  constexpr int NWM = E * ES / 4, NWH = EH * ES / 4;  // packed words per lane: main / halo
  static_assert(HW % 32 == 0 && EH * ES >= 4, "halo lanes");
  static_assert(!PACK || ES == 1, "packed vertical sums are for uint8");
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  SM& sm = reinterpret_cast<SM*>(smem_raw)[warp];
  int J, K;  // J: warp strip (SPW build strips), K: sweep segment
  warp_tile<kSweepWarps>(nJw, nK, J, K);
  if (K < 0) return;
  const int64_t PR = R + 1, PC = C + 1;
  const int64_t j0 = (int64_t)J * TW, k0 = (int64_t)K * SR;
  const int64_t k1 = min64(k0 + SR, PR);
  const int64_t cb = j0 - 1 - HW;  // image column of V index 0
  const int64_t c_lo = max64(cb, 0), c_hi = min64(j0 - 1 + TW, C);
  // table rows swept: [ra, k1); rows below k0 only warm the vertical sums up
  const int64_t ra = K == 0 ? 0 : max64(1, k0 - w);
  const int64_t rsub = max64(ra, 1) + w;  // from here on the leaving row is subtracted
  const int nblk = (int)((k1 - ra + RB - 1) / RB);
  const int64_t cbase = j0 + lane * E;    // table column of the lane's first element
  const int64_t cm0 = cbase - 1;          // matching image column
  const int64_t ch0 = cb + (int64_t)lane * EH;  // first halo image column of the lane
  const bool halo_lane = ch0 + EH > 0 && ch0 < C;
  const char* base = reinterpret_cast<const char*>(in);
  const char* end_valid = base + ((R - 1) * in_ld + C) * ES;
  const int64_t out_c = C - w + 1;
  const int64_t j_lo = max64(j0 - w, 0), j_hi = min64(j0 - w + TW, out_c);
  const int nout = (int)(j_hi - j_lo);

  if (lane == 0) {
    for (int i = 0; i < SM::NST; ++i) mbar_init(&sm.bar[i], 1);
    fence_mbar_init();
  }
  __syncwarp();
  // lane q < RB stages image row (row - 1), lane RB + q the leaving row (row - 1 - w), row = rb + q
  auto issue = [&](int b, int s) {
    const int64_t rb = ra + (int64_t)b * RB;
    const int q = lane % RB;
    const bool old = lane >= RB;
    const int64_t row = rb + q;
    const int64_t ir = row - 1 - (old ? w : 0);
    const bool has = lane < 2 * RB && row < k1 && row >= 1 && (!old || row >= rsub) && c_hi > c_lo;
    unsigned char* dst = sm.stage[s][lane < 2 * RB ? lane : 0];
    RowSpan sp;
    if (has) sp = row_span(base + ir * in_ld * ES, c_lo, c_hi, ES, end_valid, dst);
    if (lane < 2 * RB) sm.offs[s][lane] = has ? sp.off : kNoRow;
    warp_issue(sp, has, dst, &sm.bar[s], lane);
  };
  for (int b = 0; b < SM::NST - 1; ++b)
    if (b < nblk) issue(b, b);

  // table accumulators as 4-element vectors: one 256-bit store each without
  // register re-packing (a plain Acc[E] array cost 8 moves per store)
  U64x4 acc4[E / 4];
#pragma unroll
  for (int k = 0; k < E; ++k)
    set4(acc4[k / 4], k % 4, (unsigned long long)(cbase + k < PC ? top[(int64_t)K * top_stride + cbase + k] : Acc(0)));
  constexpr int NVM = PACK ? E / 2 : E, NVH = PACK ? EH / 2 : EH;
  VT Vm[NVM], Vh[NVH];
#pragma unroll
  for (int k = 0; k < NVM; ++k) Vm[k] = VT(0);
#pragma unroll
  for (int k = 0; k < NVH; ++k) Vh[k] = VT(0);
  const int u_a = (int)(j_lo - cb) + lane;  // P index of out column j_lo + lane (left edge)
  const int addr_a = u_a + (u_a >> 5);
  const int addr_b = (u_a + w) + ((u_a + w) >> 5);

  auto load_main = [&](int s, int slot, uint32_t (&x)[NWM]) {
    lane_elems_packed<InT, E>(sm.stage[s][slot], sm.offs[s][slot], cm0, C, x);
  };
  auto load_halo = [&](int s, int slot, uint32_t (&x)[NWH]) {
    if (halo_lane) {
      lane_elems_packed<InT, EH>(sm.stage[s][slot], sm.offs[s][slot], ch0, C, x);
    } else {
#pragma unroll
      for (int i = 0; i < NWH; ++i) x[i] = 0u;
    }
  };
  for (int b = 0; b < nblk; ++b) {
    const int s = b % SM::NST;
    if (b + SM::NST - 1 < nblk) issue(b + SM::NST - 1, (b + SM::NST - 1) % SM::NST);
    const int64_t rb = ra + (int64_t)b * RB;
    Acc rlv = Acc(0);  // lane q: left carry of table row rb + q
    if (lane < RB && rb + lane >= k0 && rb + lane < k1) rlv = rl[(rb + lane) * nJ + J * SPW];
    mbar_wait(&sm.bar[s], (uint32_t)((b / SM::NST) & 1));
#pragma unroll
    for (int q = 0; q < RB; ++q) {
      const int64_t row = rb + q;
      if (row >= k1) break;
      uint32_t xm[NWM], xh[NWH];
      if (row >= rsub) {  // the leaving row first: V >= it per column, so packed halves never borrow
        load_main(s, RB + q, xm);
        load_halo(s, RB + q, xh);
        vupdate<InT, PACK, false>(Vm, xm);
        vupdate<InT, PACK, false>(Vh, xh);
      }
      load_main(s, q, xm);
      load_halo(s, q, xh);
      vupdate<InT, PACK, true>(Vm, xm);
      vupdate<InT, PACK, true>(Vh, xh);
      if (row < k0) continue;  // warm-up row
      {  // table row: strip-local prefix + left carry, accumulated down the column
        const Loc t = lane_sum<InT, E>(xm);
        // element k's row value = left carry + lanes to the left + lane-local prefix
        const Acc base = add(__shfl_sync(0xffffffffu, rlv, q), (Acc)sub(warp_incl_scan(t, lane), t));
        if constexpr (sizeof(InT) == 1) {
          // lane-local prefix by DP4A: bytes 0..m of word i in one step from the group base
          uint32_t g = 0u;
#pragma unroll
          for (int i = 0; i < NWM; ++i) {
            const uint32_t p0 = __dp4a(xm[i], 0x00000001u, g), p1 = __dp4a(xm[i], 0x00000101u, g);
            const uint32_t p2 = __dp4a(xm[i], 0x00010101u, g), p3 = __dp4a(xm[i], 0x01010101u, g);
            acc4[i].x += base + p0;
            acc4[i].y += base + p1;
            acc4[i].z += base + p2;
            acc4[i].w += base + p3;
            g = p3;
          }
        } else {
          Loc pre = Loc(0);
#pragma unroll
          for (int k = 0; k < E; ++k) {
            pre = add(pre, conv<Loc>(elem<InT>(xm, k)));
            set4(acc4[k / 4], k % 4, get4(acc4[k / 4], k % 4) + (unsigned long long)add(base, (Acc)pre));
          }
        }
        Acc* dst = sat + row * sat_ld + cbase;
        if (cbase + E <= PC) {
#pragma unroll
          for (int i = 0; i < E / 4; ++i) st256(dst + 4 * i, acc4[i]);
        } else {
#pragma unroll
          for (int k = 0; k < E; ++k)
            if (cbase + k < PC) st_cs(dst + k, (Acc)get4(acc4[k / 4], k % 4));
        }
      }
      if (row < w || nout <= 0) continue;  // no window ends on this row
      if constexpr (PACK) {
        if (mask == ST_SUM) {  // uint8 sums: DP2A prefix, paired 16-byte output stores
          onepass_packed_row<E, EH, HW>(Vm, Vh, sm.p, reinterpret_cast<uint64_t*>(o.sum) + (row - w) * o.ld + j_lo,
                                       (int)(j_lo - cb), nout, w, lane);
          continue;
        }
      }
      {  // P = prefix of V over [halo | strip]
        VT th = VT(0), tm = VT(0);
#pragma unroll
        for (int k = 0; k < EH; ++k) th = add(th, vcol<PACK>(Vh, k));
#pragma unroll
        for (int k = 0; k < E; ++k) tm = add(tm, vcol<PACK>(Vm, k));
        const VT ih = warp_incl_scan(th, lane);
        const VT hall = __shfl_sync(0xffffffffu, ih, 31);
        const VT im = warp_incl_scan(tm, lane);
        VT run = sub(ih, th);
#pragma unroll
        for (int k = 0; k < EH; ++k) {
          run = add(run, vcol<PACK>(Vh, k));
          const int u = lane * EH + k + 1;
          sm.p[u + (u >> 5)] = run;
        }
        run = add(hall, sub(im, tm));
#pragma unroll
        for (int k = 0; k < E; ++k) {
          run = add(run, vcol<PACK>(Vm, k));
          const int u = HW + lane * E + k + 1;
          sm.p[u + (u >> 5)] = run;
        }
        if (lane == 0) sm.p[0] = VT(0);
      }
      __syncwarp();
      {  // out[j] = P[j + w] - P[j], consecutive lanes -> consecutive columns
        const int64_t obase = (row - w) * o.ld + j_lo + lane;
        const int nq = (nout - lane + 31) >> 5;
        int a = addr_a, bw = addr_b;
        if (mask == ST_SUM && nout == TW) {
          uint64_t* dst = reinterpret_cast<uint64_t*>(o.sum) + obase;
#pragma unroll
          for (int qq = 0; qq < TW / 32; ++qq) st_cs(dst + 32 * qq, (uint64_t)sub(sm.p[bw + 33 * qq], sm.p[a + 33 * qq]));
        } else if (mask == ST_SUM) {
          uint64_t* dst = reinterpret_cast<uint64_t*>(o.sum) + obase;
#pragma unroll 4
          for (int qq = 0; qq < nq; ++qq, a += 33, bw += 33, dst += 32) {
            const VT sv = sub(sm.p[bw], sm.p[a]);
            st_cs(dst, (uint64_t)sv);
          }
        } else {
          for (int qq = 0; qq < nq; ++qq, a += 33, bw += 33) {
            const int64_t at = obase + 32 * qq;
            const uint64_t s64 = (uint64_t)sub(sm.p[bw], sm.p[a]);
            if (mask & ST_SUM) st_cs(reinterpret_cast<uint64_t*>(o.sum) + at, s64);
            if (mask & ST_MEAN) st_cs(o.mean + at, fin_mean_int(s64, fi));
          }
        }
      }
      __syncwarp();  // P is rewritten by the next row
    }
    __syncwarp();  // stage s fully read before it is refilled
  }
}

// ---------------------------------------------------------------------------
// host side
//
// The reduce phase keeps the build's plan (SR rows per segment, TW-wide
// strips): left carries are per table row, so only the segment height of the
// sweep matters, and it is a multiple m of SR (the top carry of sweep segment
// K is the build's top carry of segment m K).  m minimises
// waves(m) * (m SR + w): whole waves of resident warps, each sweeping one
// segment plus its w warm-up rows.
struct SweepPlan {
  SatPlan p;
  int nJw, nKs;
  int64_t SRs, m;
};

template <typename InT>
SweepPlan make_sweep_plan_t(int dtype, int64_t R, int64_t C, int64_t w) {
  constexpr int SPW = SweepCfg<InT>::SPW;
  SweepPlan sp{};
  sp.p = make_sat_plan(dtype, R, C, false);
  sp.nJw = (sp.p.nJ + SPW - 1) / SPW;
  const int64_t resident = (int64_t)kNumSMs * kSweepWarps * SSB_SWEEP_MINB;
  static const int fixed_m = env_int("SSB_SWEEP_M", 0);  // tuning: fixed segment multiple
  int64_t best_m = 1;
  double best = 1e300;
  for (int64_t m = 1; m <= sp.p.nK; ++m) {
    const int64_t nks = (sp.p.nK + m - 1) / m;
    if (m > 1 && (sp.p.nK + m - 2) / (m - 1) == nks) continue;  // same segment count as a smaller m
    const int64_t tiles = nks * sp.nJw;
    const double cost = (double)((tiles + resident - 1) / resident) * (double)(min64(m * sp.p.SR, sp.p.PR) + w);
    if (cost < best) { best = cost; best_m = m; }
  }
  if (fixed_m > 0) best_m = fixed_m;
  sp.m = best_m;
  sp.SRs = best_m * sp.p.SR;
  sp.nKs = (int)((sp.p.PR + sp.SRs - 1) / sp.SRs);
  return sp;
}

inline SweepPlan make_sweep_plan(int dtype, int64_t R, int64_t C, int64_t w) {
  switch (dtype) {
    case IN_U8: return make_sweep_plan_t<uint8_t>(dtype, R, C, w);
    case IN_U16: return make_sweep_plan_t<uint16_t>(dtype, R, C, w);
    default: return make_sweep_plan_t<int32_t>(dtype, R, C, w);
  }
}

bool sat_sweep_supported(int dtype, int64_t w, int mask) {
  if (w < 1 || w > kSweepHalo + 1) return false;
  if (mask == 0 || (mask & ~(ST_SUM | ST_MEAN)) != 0) return false;
  const unsigned __int128 ww = (unsigned __int128)(uint64_t)(w * w);
  switch (dtype) {
    case IN_U8: return true;                                          // w^2 * 255 < 2^32, V <= 65535
    case IN_U16: return ww * 65535u < ((unsigned __int128)1 << 32);   // u32 window sums
    case IN_I32: return true;                                         // u64 (signed) sums
    default: return false;
  }
}

int64_t sat_workspace_bytes(int dtype, int64_t R, int64_t C, bool sq);

int64_t sat_sweep_workspace_bytes(int dtype, int64_t R, int64_t C) {
  const int64_t one = make_sat_plan(dtype, R, C, false).total * 8;
  const int64_t two = sat_workspace_bytes(dtype, R, C, false);  // includes the look-back build's needs
  return one > two ? one : two;
}

void sat_sweep_plan_info(int dtype, int64_t R, int64_t C, int64_t w, int64_t* info) {
  const SweepPlan sp = make_sweep_plan(dtype, R, C, w);
  info[0] = sp.nJw; info[1] = sp.SRs; info[2] = sp.nKs; info[3] = sp.m;
}

template <typename InT>
cudaError_t launch_sweep_t(const void* in, int64_t R, int64_t C, int64_t in_ld, void* sat, int64_t sat_ld, int w,
                           int mask, WinOut o, void* ws, cudaStream_t st, const SweepPlan& sp) {
  using Acc = typename Elem<InT>::Acc;
  constexpr int HW = kSweepHalo;
  using SM = SweepSmem<InT, HW>;
  const SatPlan& p = sp.p;
  Acc* wsa = reinterpret_cast<Acc*>(ws);
  FinalizeInt fi{};
  fi.n = (uint64_t)w * (uint64_t)w;
  fi.dn = (double)fi.n;
  fi.inv_n = 1.0 / fi.dn;
  fi.u64_ok = true;
  fi.is_signed = std::is_same<InT, int32_t>::value;
  auto kfn = sat_sweep_kernel<InT, HW>;
  const int smem = (int)(sizeof(SM) * kSweepWarps);
  cudaError_t e = cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  const int tb = (int)(((int64_t)sp.nJw * sp.nKs + kSweepWarps - 1) / kSweepWarps);
  kfn<<<tb, 32 * kSweepWarps, smem, st>>>(reinterpret_cast<const InT*>(in), R, C, in_ld, reinterpret_cast<Acc*>(sat),
                                          sat_ld, wsa + p.off_rowtot, wsa + p.off_colp, sp.m * p.PC, sp.SRs, p.nJ,
                                          sp.nJw, sp.nKs, w, o, mask, fi);
  note_launch(1);
  return cudaGetLastError();
}

cudaError_t launch_sat_build(int dtype, const void* in, int64_t R, int64_t C, int64_t in_ld, void* sat, void* sat_sq,
                             int64_t sat_ld, const void* carry, const void* carry_sq, void* ws, int* nonfinite,
                             cudaStream_t st);
cudaError_t launch_window_fused(const void* in, int dtype, int64_t R, int64_t C, int64_t in_ld, int64_t w, int mask,
                                WinOut o, int* nonfinite, int nK, cudaStream_t st);
cudaError_t launch_window_eval(const void* sat, const void* sat_sq, bool is_float, int in_dtype, int64_t R, int64_t C,
                               int64_t sat_ld, int64_t w, int64_t s, int mask, WinOut o, cudaStream_t st);

// Default: the table build (reduce-then-scan, sat_build.cu) and the fused
// window kernel (window_fused.cu), which evaluates the windows from the
// raster instead of reading the table back.  The two are independent, so the
// windows run on a side stream forked from and joined back into the caller's
// stream: measured at C5 (B200) 19.8 ms concurrent vs 21.0 ms back to back,
// 20.1 ms for the one-pass kernel above and 25.1 ms for build + corner sweep.
// ssb_sat_build_swa_onepass (or SSB_SWA_PATH=onepass) runs the one-pass kernel.
static bool swa_onepass_env() {
  static const bool one = env_char("SSB_SWA_PATH") == 'o';
  return one;
}


// The fused kernel outruns the corner sweep for uint8 (w <= 256) and uint16
// (w <= 128) rasters of at least 2^24 pixels (measured, scripts/pipe_probe.py,
// scripts/bench_configs.py); elsewhere the table is read back by the corner
// sweep (C2 int32: 0.74 vs 1.47 ms; C1 2048^2: launch-bound, 0.11 vs 0.17 ms).
bool sweep_uses_fused(int dtype, int64_t R, int64_t C, int64_t w) {
  return R * C >= ((int64_t)1 << 24) && ((dtype == IN_U8 && w <= 256) || (dtype == IN_U16 && w <= 128));
}

// Side streams for the fork/join of ssb_sat_build_swa: a small thread-local
// pool keyed by the caller's stream (so two caller streams never wait on each
// other's fork points), each entry on the caller stream's device.  Entries are
// created whole (stream and both events) before they are published and
// destroyed with the thread.
struct SideStream {
  cudaStream_t caller = nullptr;
  int dev = -1;
  cudaStream_t s = nullptr;
  cudaEvent_t fork = nullptr, join = nullptr;
  unsigned long long last_use = 0;
};

struct SidePool {
  static constexpr int kMax = 16;
  SideStream e[kMax];
  unsigned long long tick = 0;
  static void release(SideStream& c) {
    if (c.fork) cudaEventDestroy(c.fork);
    if (c.join) cudaEventDestroy(c.join);
    if (c.s) cudaStreamDestroy(c.s);
    c = SideStream{};
  }
  ~SidePool() {
    for (auto& c : e) release(c);
  }
};
static thread_local SidePool t_side;

static cudaError_t side_stream(cudaStream_t caller, SideStream*& out) {
  int dev = 0;
  cudaError_t e = cudaStreamGetDevice(caller, &dev);
  if (e != cudaSuccess) return e;
  SidePool& pool = t_side;
  SideStream* victim = &pool.e[0];
  for (auto& c : pool.e) {
    if (c.s && c.caller == caller && c.dev == dev) {
      c.last_use = ++pool.tick;
      out = &c;
      return cudaSuccess;
    }
    if (!c.s || (victim->s && c.last_use < victim->last_use)) victim = &c;
  }
  // the least recently used entry (its pending work keeps running; a reused
  // stream only orders new work after it)
  SideStream fresh;
  fresh.caller = caller;
  fresh.dev = dev;
  if ((e = cudaStreamCreateWithFlags(&fresh.s, cudaStreamNonBlocking)) == cudaSuccess &&
      (e = cudaEventCreateWithFlags(&fresh.fork, cudaEventDisableTiming)) == cudaSuccess &&
      (e = cudaEventCreateWithFlags(&fresh.join, cudaEventDisableTiming)) == cudaSuccess) {
    SidePool::release(*victim);
    *victim = fresh;
    victim->last_use = ++pool.tick;
    out = victim;
    return cudaSuccess;
  }
  SidePool::release(fresh);
  return e;
}

// Fork a side stream off `st` (it waits for st's work so far) / join it back
// (st waits for the side stream's work so far).
cudaError_t side_fork(cudaStream_t st, SideHandle* h) {
  SideStream* side = nullptr;
  cudaError_t e = side_stream(st, side);
  if (e != cudaSuccess) return e;
  if ((e = cudaEventRecord(side->fork, st)) != cudaSuccess) return e;
  if ((e = cudaStreamWaitEvent(side->s, side->fork, 0)) != cudaSuccess) return e;
  h->s = side->s;
  h->join = side->join;
  return cudaSuccess;
}

cudaError_t side_join(cudaStream_t st, const SideHandle& h) {
  cudaError_t e = cudaEventRecord(h.join, h.s);
  return e == cudaSuccess ? cudaStreamWaitEvent(st, h.join, 0) : e;
}

// table + window statistics: the table build on the caller's stream with the
// fused window kernel on a forked side stream, or reduce + carries then the
// one-pass table+sweep kernel
cudaError_t launch_sat_sweep(int dtype, const void* in, int64_t R, int64_t C, int64_t in_ld, void* sat, int64_t sat_ld,
                             int64_t w, int mask, WinOut o, void* ws, cudaStream_t st, bool onepass) {
  if (!onepass && !swa_onepass_env()) {
    if (!sweep_uses_fused(dtype, R, C, w)) {
      cudaError_t e = launch_sat_build(dtype, in, R, C, in_ld, sat, nullptr, sat_ld, nullptr, nullptr, ws, nullptr, st);
      if (e != cudaSuccess) return e;
      return launch_window_eval(sat, nullptr, false, dtype, R, C, sat_ld, w, 1, mask, o, st);
    }
    SideHandle side;
    cudaError_t e = side_fork(st, &side);
    if (e != cudaSuccess) return e;
    e = launch_sat_build(dtype, in, R, C, in_ld, sat, nullptr, sat_ld, nullptr, nullptr, ws, nullptr, st);
    const cudaError_t ef = launch_window_fused(in, dtype, R, C, in_ld, w, mask, o, nullptr, 0, side.s);
    // always join, so the caller's stream never runs ahead of the side stream
    const cudaError_t ew = side_join(st, side);
    return e != cudaSuccess ? e : ef != cudaSuccess ? ef : ew;
  }
  const SweepPlan sp = make_sweep_plan(dtype, R, C, w);
  cudaError_t e = launch_sat_prepare_plan(dtype, in, R, C, in_ld, false, ws, nullptr, st, sp.p);
  if (e != cudaSuccess) return e;
  switch (dtype) {
    case IN_U8: return launch_sweep_t<uint8_t>(in, R, C, in_ld, sat, sat_ld, (int)w, mask, o, ws, st, sp);
    case IN_U16: return launch_sweep_t<uint16_t>(in, R, C, in_ld, sat, sat_ld, (int)w, mask, o, ws, st, sp);
    case IN_I32: return launch_sweep_t<int32_t>(in, R, C, in_ld, sat, sat_ld, (int)w, mask, o, ws, st, sp);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace ssb
