// satsweep-b200: the integral image AND its window sums in one persistent
// column-strip sweep (uint8 rasters, w <= 256): the headline step of
// ssb_sat_build_swa.
//
// Same products as build_sat + sweep_window_sums (pkg/src/satsweep/integral.py
// :109-116, :141-163): the (R+1) x (C+1) uint64 table and the window sums, bit
// for bit.  Why a new kernel: the concurrent pair (reduce-then-scan build ||
// fused windows, sat_sweep.cu) moves 121.7 GB for the 100.8 GB the step needs
// -- the raster is read by the reduce, the scan, and twice by the window kernel
// (rows r and r-w), because ~1,800 warps each sweep their own short segment,
// so the w-row history behind them is ~1 GB, far beyond L2.
//
// Here each CTA owns one 576-column strip of the table (+ 320 halo columns for
// the windows) and sweeps ALL rows top to bottom, 16 rows per step:
//   * the history behind the CTAs is 148 strips x w rows x 896 bytes = 32 MB,
//     so the leaving rows (r - w) come back from L2 (raster rows are fetched
//     with an evict_last policy, leaving rows with evict_first, the 95 GB of
//     table and window stores stream past as evict-first);
//   * no top carries: a column's running table value stays in the thread that
//     owns it for the whole height;
//   * left carries (the row's total left of the strip) come from a small
//     pre-pass (strip_carry_kernel: one read of the raster, 41 MB of u32
//     carries at C5), so no CTA ever waits on another.
// Per step: phase 1 (7 warps) updates the vertical window sums V of the 896
// columns (two columns per 32-bit word as 16-bit halves, as in window_fused.cu)
// and the 4-column byte sums of the table row segment; phase 2 (16 warps, one
// row each) scans those sums across the strip and turns V into window sums
// (packed_sums_row); phase 3 (144 threads, 4 table columns each) adds carry +
// prefix to the column accumulators and stores the 16 table rows with 256-bit
// stores.  Integer sums are exact modulo 2^64 in the same ring as the
// reference's U64 table.
#include <cstdint>

#include "ssb_async.cuh"
#include "ssb_common.cuh"
#include "ssb_stage.cuh"
#include "ssb_packed.cuh"

#ifndef SSB_STRIP_PROBE
#define SSB_STRIP_PROBE 0  // tuning probes (wrong results): 1 no window outputs, 2 no table stores
#endif

namespace ssb {
void note_launch(int n);

constexpr int kStripCols = 576;                 // table columns per CTA
constexpr int kStripSpan = 896;                 // raster columns per CTA (576 + halo, 28 per lane)
constexpr int kStripRows = 16;                  // rows per step
constexpr int kStripVThreads = kStripSpan / 4;  // group A: 224 threads own 4 columns each of V
constexpr int kStripTThreads = kStripCols / 4;  // group C: 144 threads own 4 table columns each
constexpr int kStripPWords = 960;               // per-warp prefix buffer (packed_sums_row, pp() layout)
// warp roles: A (V update) 0..6, B (window rows, 2 per warp) 7..14, C (table) 15..19
constexpr int kWarpsA = kStripVThreads / 32, kWarpsB = kStripRows / 2, kWarpsC = 5;
constexpr int kWarpB0 = kWarpsA, kWarpC0 = kWarpsA + kWarpsB;
constexpr int kStripThreads = 32 * (kWarpsA + kWarpsB + kWarpsC);  // 640

struct StripSmem {
  uint64_t vfull[2];  // V rows of a step written (group A, one arrival per warp)
  uint64_t vfree[2];  // V rows of a step consumed (group B)
  uint32_t vs[2][kStripRows][2 * kStripVThreads];  // V of each row of the step (packed words), by step parity
  uint32_t wt[2][kStripRows][kWarpsC];             // group C: per-warp totals of each row's byte sums
  uint32_t lx[2][kStripRows];                      // left carries of the step's rows
  uint32_t pw[kWarpsB][kStripPWords];
};

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// 4 raster bytes [c, c + 4) of a row through L2 with a cache policy; bytes at
// or past column C read as 0 (never loaded past the row)
__device__ __forceinline__ uint32_t ld_word(const uint8_t* row, int64_t c, int64_t C, uint64_t pol) {
  if (c + 4 <= C) {
    uint32_t v;
    asm volatile("ld.global.nc.L2::cache_hint.b32 %0, [%1], %2;" : "=r"(v) : "l"(row + c), "l"(pol));
    return v;
  }
  uint32_t v = 0u;
  for (int k = 0; k < 4; ++k)
    if (c + k < C) v |= (uint32_t)__ldg(row + c + k) << (8 * k);
  return v;
}

// ---- pre-pass: left carry of every (row, strip) -------------------------------
// Lx[r][s] = sum of x[r][c] for c < 576 s (u32: at most 576 * 255 * strips).
// One warp per row: lane l sums strips l, l + 32, ... with 8-byte loads
// (in_ld % 8 == 0), then an exclusive scan across the strips.
__global__ void __launch_bounds__(256) strip_carry_kernel(const uint8_t* __restrict__ in, int64_t R, int64_t C,
                                                           int64_t in_ld, int nS, uint32_t* __restrict__ lx) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t r = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); r < R; r += warps) {
    const uint8_t* row = in + r * in_ld;
    uint32_t carry = 0;
    for (int s0 = 0; s0 < nS; s0 += 32) {
      const int s = s0 + lane;
      uint32_t tot = 0;
      if (s < nS) {
        const int64_t c0 = (int64_t)s * kStripCols;
        const int64_t c1 = c0 + kStripCols < C ? c0 + kStripCols : C;
        if (c1 - c0 == kStripCols) {
          const uint2* p = reinterpret_cast<const uint2*>(row + c0);
#pragma unroll 8
          for (int k = 0; k < kStripCols / 8; ++k) {
            const uint2 v = __ldcs(p + k);
            tot = __dp4a(v.x, 0x01010101u, tot);
            tot = __dp4a(v.y, 0x01010101u, tot);
          }
        } else {
          for (int64_t c = c0; c < c1; ++c) tot += row[c];
        }
      }
      const uint32_t inc = warp_incl_scan(tot, lane);
      if (s < nS) lx[r * nS + s] = carry + inc - tot;
      carry += __shfl_sync(0xffffffffu, inc, 31);
    }
  }
}

__global__ void __launch_bounds__(kStripThreads, 1)
sat_strip_kernel(const uint8_t* __restrict__ in, int64_t R, int64_t C, int64_t in_ld, uint64_t* __restrict__ sat,
                 int64_t sat_ld, uint64_t* __restrict__ out, int64_t out_ld, int64_t out_c, int w,
                 const uint32_t* __restrict__ lx, int nS, Census cz) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  StripSmem& sm = *reinterpret_cast<StripSmem*>(smem_raw);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int s = blockIdx.x;
  const int64_t c0 = (int64_t)s * kStripCols;  // first table column = first raster column of the span
  const int64_t PC = C + 1;
  const int nsteps = (int)((R + kStripRows - 1) / kStripRows);
  if (tid == 0) {
    for (int i = 0; i < 2; ++i) {
      mbar_init(&sm.vfull[i], kWarpsA);
      mbar_init(&sm.vfree[i], kWarpsB);
    }
    fence_mbar_init();
  }
  __syncthreads();

  if (warp < kWarpB0) {
    // ---- group A: vertical window sums of the 896 span columns, 4 per thread.
    // Raster words come straight from global memory (coalesced 128-byte warp
    // loads): entering rows with an evict_last policy (they are read again w
    // rows later, as leaving rows, from L2), leaving rows with evict_first.
    // The next step's words are loaded while this step is computed.
    const int64_t cc = c0 + 4 * tid;
    const uint64_t keep = policy_evict_last(), drop = policy_evict_first();
    uint32_t nw[kStripRows], ow[kStripRows];
    auto load = [&](int b) {
#pragma unroll
      for (int g = 0; g < kStripRows; ++g) {
        const int64_t r = (int64_t)b * kStripRows + g, ro = r - w;
        nw[g] = r < R && cc < C ? ld_word(in + r * in_ld, cc, C, keep) : 0u;
        ow[g] = r < R && ro >= 0 && cc < C ? ld_word(in + ro * in_ld, cc, C, drop) : 0u;
      }
    };
    load(0);
    uint32_t V0 = 0u, V1 = 0u;
    for (int b = 0; b < nsteps; ++b) {
      const int vb = b & 1;
      uint32_t cn[kStripRows], co[kStripRows];
#pragma unroll
      for (int g = 0; g < kStripRows; ++g) { cn[g] = nw[g]; co[g] = ow[g]; }
      if (b + 1 < nsteps) load(b + 1);
      if (b >= 2) mbar_wait(&sm.vfree[vb], (uint32_t)(((b - 2) >> 1) & 1));
#pragma unroll
      for (int g = 0; g < kStripRows; ++g) {
        // V >= the leaving row in every column, so no borrow crosses a 16-bit half
        V0 = V0 - (co[g] & 0x00FF00FFu) + (cn[g] & 0x00FF00FFu);
        V1 = V1 - ((co[g] >> 8) & 0x00FF00FFu) + ((cn[g] >> 8) & 0x00FF00FFu);
        sm.vs[vb][g][2 * tid] = V0;
        sm.vs[vb][g][2 * tid + 1] = V1;
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&sm.vfull[vb]);
    }
  } else if (warp < kWarpC0) {
    // ---- group B: window sums of 2 rows per warp per step from V
    const int bw = warp - kWarpB0;
    const int64_t out_r = R - w + 1;
    const int nout = (int)(out_c - c0 < kStripCols ? out_c - c0 : kStripCols);
    for (int b = 0; b < nsteps; ++b) {
      const int vb = b & 1;
      mbar_wait(&sm.vfull[vb], (uint32_t)((b >> 1) & 1));
#pragma unroll
      for (int rr = 0; rr < 2; ++rr) {
        const int g = 2 * bw + rr;
        const int64_t r = (int64_t)b * kStripRows + g;
        const int64_t i = r - (w - 1);  // the output row whose bottom row is r
        if (!(SSB_STRIP_PROBE & 1) && r < R && i >= 0 && i < out_r && nout > 0) {
          uint32_t Vl[14];
#pragma unroll
          for (int k = 0; k < 14; ++k) Vl[k] = sm.vs[vb][g][14 * lane + k];
          packed_sums_row<28>(Vl, sm.pw[bw], i * out_ld + c0, out, nout, w, lane, cz, i);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&sm.vfree[vb]);
    }
  } else {
    // ---- group C: the table, 4 columns per thread (the same raster words as
    // group A's first 144 threads, mostly L1/L2 hits)
    const int ct = tid - 32 * kWarpC0, cw = warp - kWarpC0;
    const int64_t tc = c0 + 4 * ct;  // table column of this thread's first accumulator
    const bool tab = ct < kStripTThreads && tc < PC;
    const int64_t cc = tc;           // its raster columns (table col c <- image cols < c)
    const bool ldr = ct < kStripTThreads && cc < C;
    const uint64_t pol = policy_evict_last();
    uint32_t nw[kStripRows];
    auto load = [&](int b) {
#pragma unroll
      for (int g = 0; g < kStripRows; ++g) {
        const int64_t r = (int64_t)b * kStripRows + g;
        nw[g] = ldr && r < R ? ld_word(in + r * in_ld, cc, C, pol) : 0u;
      }
    };
    load(0);
    uint64_t acc[4] = {0ull, 0ull, 0ull, 0ull};
    if (tab) {  // table row 0: the zero border
      const U64x4 z{0ull, 0ull, 0ull, 0ull};
      if (tc + 4 <= PC) st256(sat + tc, z);
      else for (int k = 0; k < 4; ++k) if (tc + k < PC) st_cs(sat + tc + k, (uint64_t)0);
      if (cz.trow != nullptr)
        for (int k = 0; k < 4; ++k)
          if (tc + k < PC) { census_add(cz.trow, cz.ntr, 0); census_add(cz.tcol, cz.ntc, tc + k); }
    }
    for (int b = 0; b < nsteps; ++b) {
      const int pb = b & 1;
      const int64_t r0 = (int64_t)b * kStripRows;
      if (ct < kStripRows) sm.lx[pb][ct] = r0 + ct < R ? lx[(r0 + ct) * nS + s] : 0u;
      uint32_t xw[kStripRows], inc[kStripRows];
#pragma unroll
      for (int g = 0; g < kStripRows; ++g) xw[g] = nw[g];
      if (b + 1 < nsteps) load(b + 1);
#pragma unroll
      for (int g = 0; g < kStripRows; ++g) {
        const uint32_t t4 = __dp4a(xw[g], 0x01010101u, 0u);
        inc[g] = warp_incl_scan(t4, lane) - t4;  // exclusive prefix within the warp
        if (lane == 31) sm.wt[pb][g][cw] = inc[g] + t4;
      }
      asm volatile("bar.sync 1, %0;" ::"n"(32 * kWarpsC) : "memory");  // group C only
      if (tab) {
#pragma unroll
        for (int g = 0; g < kStripRows; ++g) {
          const int64_t r = r0 + g;
          if (r >= R) break;
          uint32_t left32 = inc[g];
          for (int k = 0; k < cw; ++k) left32 += sm.wt[pb][g][k];
          const uint32_t x = xw[g];
          const uint32_t b0 = x & 0xFFu, b1 = (x >> 8) & 0xFFu, b2 = (x >> 16) & 0xFFu;
          const uint64_t left = (uint64_t)sm.lx[pb][g] + (uint64_t)left32;
          acc[0] += left;
          acc[1] += left + b0;
          acc[2] += left + b0 + b1;
          acc[3] += left + b0 + b1 + b2;
          uint64_t* dst = sat + (r + 1) * sat_ld + tc;
          if (SSB_STRIP_PROBE & 2) {
            if (acc[0] == 0x123456789ull) st_cs(dst, acc[1]);  // keep the arithmetic alive
          } else if (tc + 4 <= PC) {
            const U64x4 v{acc[0], acc[1], acc[2], acc[3]};
            st256(dst, v);
          } else {
            for (int k = 0; k < 4; ++k)
              if (tc + k < PC) st_cs(dst + k, acc[k]);
          }
          if (cz.trow != nullptr)
            for (int k = 0; k < 4; ++k)
              if (tc + k < PC) { census_add(cz.trow, cz.ntr, r + 1); census_add(cz.tcol, cz.ntc, tc + k); }
        }
      }
    }
  }
}

bool sat_strip_supported(const void* in, int dtype, int64_t R, int64_t C, int64_t in_ld, int64_t w, int mask,
                         int64_t sat_ld) {
  // uint8 sums, w <= 256 (16-bit V halves), rasters wide enough to give every
  // SM a strip, 8-byte aligned rows for the carry pre-pass
  return dtype == IN_U8 && mask == ST_SUM && w <= 256 && C >= (int64_t)kNumSMs * kStripCols / 2 && R >= w &&
         (in_ld % 8) == 0 && (reinterpret_cast<uintptr_t>(in) % 8) == 0 && (sat_ld % 4) == 0 &&
         C * 255 < ((int64_t)1 << 32);
}

int64_t sat_strip_workspace_bytes(int64_t R, int64_t C) {
  const int64_t nS = (C + 1 + kStripCols - 1) / kStripCols;
  return R * nS * 4 + 256;
}

cudaError_t launch_sat_strip(const void* in, int64_t R, int64_t C, int64_t in_ld, void* sat, int64_t sat_ld, int64_t w,
                             WinOut o, void* ws, cudaStream_t st) {
  const int nS = (int)((C + 1 + kStripCols - 1) / kStripCols);
  uint32_t* lx = reinterpret_cast<uint32_t*>(ws);
  const int cblocks = (int)((R + 7) / 8 < 16 * kNumSMs ? (R + 7) / 8 : 16 * kNumSMs);
  strip_carry_kernel<<<cblocks, 256, 0, st>>>(reinterpret_cast<const uint8_t*>(in), R, C, in_ld, nS, lx);
  note_launch(1);
  const size_t smem = sizeof(StripSmem);
  cudaError_t e = cudaFuncSetAttribute(sat_strip_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  sat_strip_kernel<<<nS, kStripThreads, smem, st>>>(reinterpret_cast<const uint8_t*>(in), R, C, in_ld,
                                                    reinterpret_cast<uint64_t*>(sat), sat_ld,
                                                    reinterpret_cast<uint64_t*>(o.sum), o.ld, C - w + 1, (int)w, lx,
                                                    nS, census_sink());
  note_launch(1);
  return cudaGetLastError();
}

}  // namespace ssb
