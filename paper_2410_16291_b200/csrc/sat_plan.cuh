// satsweep-b200: tiling plan of the reduce-then-scan table build, shared by
// sat_build.cu (table only) and sat_sweep.cu (table + window sums in one pass).
// A plan cuts the padded (R+1) x (C+1) table into strips of TW table columns
// and segments of SR table rows; the workspace holds the per-(row, strip) row
// totals -> left carries, the per-(segment, column) column prefixes -> top
// carries, and the per-(segment, strip) sums of left carries.
#pragma once

#include <cstdint>

#include "ssb_common.cuh"

namespace ssb {

struct SatPlan {
  int TW, nJ, nK;
  int64_t SR, PR, PC;
  // workspace offsets in elements of 8 bytes
  int64_t off_rowtot, off_rowtot_sq, off_colp, off_colp_sq, off_srl, off_srl_sq, total;
};

inline int tw_for(int dtype) { return (dtype == IN_U8 || dtype == IN_U16) ? 512 : 256; }

// sr_fixed > 0 forces the segment height (rounded up to a multiple of 8):
// the table+sweep kernel (sat_sweep.cu) wants taller segments than the build.
inline SatPlan make_sat_plan(int dtype, int64_t R, int64_t C, bool sq, int64_t sr_fixed = 0) {
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
#ifndef SSB_SR_CAP
#define SSB_SR_CAP 512
#endif
  if (SR > SSB_SR_CAP) SR = SSB_SR_CAP;
  if (sr_fixed > 0) SR = ((sr_fixed + RB - 1) / RB) * RB;
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

}  // namespace ssb
