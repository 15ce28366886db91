// satsweep-b200: uint8 window sums of one row from packed vertical sums
// (shared by window_fused.cu's strip kernel and sat_strip.cu).
#pragma once

#include <cstdint>

#include "ssb_common.cuh"

namespace ssb {

// uint8 sums from packed vertical sums (V[2g] = columns 4g, 4g+2 and V[2g+1] =
// columns 4g+1, 4g+3 as 16-bit halves).  One output row of a strip:
//   * the lane total and the running prefix take one DP2A per column
//     (a.lo16 * b.byte0 + a.hi16 * b.byte1 + c extracts and adds in one step);
//   * P[u] is stored at word pp(u + d), pp(v) = v + 2 (v >> 6): even v are
//     8-byte aligned, and d = 1 when the row's first output is not 16-byte
//     aligned in global memory, so every output pair (j, j + 1) that is 16-byte aligned in global memory
//     reads its two P words with one 64-bit shared load per operand;
//   * pairs leave as one 16-byte streaming store.
__device__ __forceinline__ int pp(int v) { return v + 2 * (v >> 6); }

#ifndef SSB_FUSED_ST
#define SSB_FUSED_ST 0
#endif
// 16-byte output store: streaming (evict-first) by default; tuning variants
__device__ __forceinline__ void st_pair(uint64_t* p, uint64_t a, uint64_t b) {
#if SSB_FUSED_ST == 0
  st_cs2(p, a, b);
#elif SSB_FUSED_ST == 1
  asm volatile("st.global.L1::no_allocate.v2.u64 [%0], {%1, %2};" ::"l"(p), "l"(a), "l"(b) : "memory");
#else
  asm volatile("st.global.v2.u64 [%0], {%1, %2};" ::"l"(p), "l"(a), "l"(b) : "memory");
#endif
}

template <int E>
__device__ __forceinline__ void packed_sums_row(const uint32_t (&V)[E / 2], uint32_t* P, int64_t gb,
                                                uint64_t* __restrict__ out, int nout, int w, int lane,
                                                const Census& cz, int64_t i) {
  const int d = (int)((reinterpret_cast<uintptr_t>(out + gb) >> 3) & 1);  // 16-byte phase of output 0
  uint32_t tot = 0u;
#pragma unroll
  for (int i = 0; i < E / 2; ++i) tot = __dp2a_lo(V[i], 0x0101u, tot);
  uint32_t run = warp_incl_scan(tot, lane) - tot;
  const int ub = lane * E + 1 + d;  // pp argument of this lane's first P entry
#pragma unroll
  for (int q = 0; q < E / 4; ++q) {
    const uint32_t r0 = __dp2a_lo(V[2 * q], 0x0001u, run);
    const uint32_t r1 = __dp2a_lo(V[2 * q + 1], 0x0001u, r0);
    const uint32_t r2 = __dp2a_lo(V[2 * q], 0x0100u, r1);
    const uint32_t r3 = __dp2a_lo(V[2 * q + 1], 0x0100u, r2);
    P[pp(ub + 4 * q)] = r0;
    P[pp(ub + 4 * q + 1)] = r1;
    P[pp(ub + 4 * q + 2)] = r2;
    P[pp(ub + 4 * q + 3)] = r3;
    run = r3;
  }
  if (lane == 0) P[pp(d)] = 0u;
  __syncwarp();
  uint64_t* orow = out + gb;
  if (lane == 0) {
    if (d) { orow[0] = (uint64_t)(P[pp(w + 1)] - P[pp(1)]); census_add(cz.orow, cz.nor, i); }  // leading single
    if ((nout - d) & 1) {                                                                       // trailing
      orow[nout - 1] = (uint64_t)(P[pp(nout - 1 + w + d)] - P[pp(nout - 1 + d)]);
      census_add(cz.orow, cz.nor, i);
    }
  }
  const int npair = (nout - d) >> 1;
  // pair m: outputs j = d + 2m, d + 2m + 1; P words at pp(j + d) (even) and pp(j + w + d)
  const int va = 2 * lane + 2 * d, vb = va + w;
  const uint32_t* pa = P + pp(va);
  uint64_t* dst = orow + d + 2 * lane;
  const int nq = (npair - lane + 31) >> 5;
  if ((w & 1) == 0) {
    const uint32_t* pb = P + pp(vb);
#pragma unroll 4
    for (int qq = 0; qq < nq; ++qq) {
      const uint2 A = *reinterpret_cast<const uint2*>(pa + 66 * qq);
      const uint2 B = *reinterpret_cast<const uint2*>(pb + 66 * qq);
      st_pair(dst + 64 * qq, (uint64_t)(B.x - A.x), (uint64_t)(B.y - A.y));
    }
  } else {
    const uint32_t* pb0 = P + pp(vb);
    const uint32_t* pb1 = P + pp(vb + 1);
#pragma unroll 4
    for (int qq = 0; qq < nq; ++qq) {
      const uint2 A = *reinterpret_cast<const uint2*>(pa + 66 * qq);
      st_pair(dst + 64 * qq, (uint64_t)(pb0[66 * qq] - A.x), (uint64_t)(pb1[66 * qq] - A.y));
    }
  }
  census_add(cz.orow, cz.nor, i, 2ull * (unsigned long long)nq);  // this lane's pairs of row i
  __syncwarp();  // P is rewritten by the next row
}

}  // namespace ssb
