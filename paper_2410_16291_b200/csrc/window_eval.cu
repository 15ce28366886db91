// satsweep-b200: four-corner window evaluation over a device-resident table.
//
// Reference: sweep_window_sums / corner_view (pkg/src/satsweep/integral.py:133-163)
// followed by stats.finalize (pkg/src/satsweep/stats.py:35-74).  One kernel reads
// the sum table (and the squared table for std) and writes any subset of
// {sum, mean, std} in a single pass, in the reference's evaluation order
//   (br - tr) - (bl - tl).
//
// Traversal: outputs are grouped into column panels whose width is chosen so
// that w table rows of one panel stay resident in L2; inside a panel work items
// are (output row, 512-column chunk) in row-major order and a persistent grid
// strides over them.  A table row is first read as the bottom corner row of
// output row i-w and re-read from L2 as the top corner row of output row i, so
// HBM sees each table byte about once.
#include "ssb_common.cuh"

namespace ssb {

struct EvalGeom {
  int64_t out_r, out_c, w, s, sat_ld;
  int64_t pw;        // panel width in output columns (multiple of kChunk)
  int64_t n_panels, cpp, cpl;  // chunks per full panel / in the last panel
  int64_t n_items;
  int mask;
};

constexpr int kChunk = 2 * kThreads;  // 512 output columns per work item

template <typename Acc> struct Fin;
template <> struct Fin<uint64_t> {
  FinalizeInt f;
  __device__ __forceinline__ double mean(uint64_t s) const { return fin_mean_int(s, f); }
  __device__ __forceinline__ double std_(uint64_t s, uint64_t q) const { return fin_std_int(s, q, f); }
};
template <> struct Fin<double> {
  double dn;
  __device__ __forceinline__ double mean(double s) const { return fin_mean_f(s, dn); }
  __device__ __forceinline__ double std_(double s, double q) const { return fin_std_f(s, q, dn); }
};

__device__ __forceinline__ void decode_item(const EvalGeom& g, int64_t it, int64_t& row, int64_t& cb) {
  const int64_t per_full = g.out_r * g.cpp;
  const int64_t p = it / per_full;
  const int64_t rem = it - p * per_full;
  const int64_t cpp = (p == g.n_panels - 1) ? g.cpl : g.cpp;
  row = rem / cpp;
  cb = p * g.pw + (rem - row * cpp) * kChunk;
}

template <typename Acc>
__device__ __forceinline__ Acc corner4(Acc br, Acc tr, Acc bl, Acc tl) { return sub(sub(br, tr), sub(bl, tl)); }

template <typename Acc>
__device__ __forceinline__ void emit_pair(const EvalGeom& g, const WinOut& o, const Fin<Acc>& fin, int64_t i, int64_t j,
                                          Acc s0, Acc s1, Acc q0, Acc q1, bool two, bool vec_out) {
  const int64_t base = i * o.ld + j;
  if (g.mask & ST_SUM) {
    Acc* p = reinterpret_cast<Acc*>(o.sum) + base;
    if (two && vec_out) st_cs2(p, s0, s1);
    else { st_cs(p, s0); if (two) st_cs(p + 1, s1); }
  }
  if (g.mask & ST_MEAN) {
    double* p = o.mean + base;
    const double a = fin.mean(s0);
    if (two) { const double b = fin.mean(s1); if (vec_out) st_cs2(p, a, b); else { st_cs(p, a); st_cs(p + 1, b); } }
    else st_cs(p, a);
  }
  if (g.mask & ST_STD) {
    double* p = o.std_ + base;
    const double a = fin.std_(s0, q0);
    if (two) { const double b = fin.std_(s1, q1); if (vec_out) st_cs2(p, a, b); else { st_cs(p, a); st_cs(p + 1, b); } }
    else st_cs(p, a);
  }
}

template <typename Acc> struct Pair;
template <> struct Pair<uint64_t> { using V = ulonglong2; };
template <> struct Pair<double> { using V = double2; };

// Vector path: stride 1, even window, even sat_ld -> all four corner pairs are
// 16-byte aligned.
template <typename Acc, bool SQ>
__global__ void __launch_bounds__(kThreads)
window_eval_vec_kernel(const Acc* __restrict__ sat, const Acc* __restrict__ sq, EvalGeom g, WinOut o, Fin<Acc> fin) {
  using V = typename Pair<Acc>::V;
  const bool vec_out = ((o.ld & 1) == 0);
  for (int64_t it = blockIdx.x; it < g.n_items; it += gridDim.x) {
    int64_t i, cb;
    decode_item(g, it, i, cb);
    const int64_t j = cb + 2 * threadIdx.x;
    if (j >= g.out_c) continue;
    const bool two = (j + 1) < g.out_c;
    const int64_t top = i * g.sat_ld, bot = (i + g.w) * g.sat_ld;
    Acc s0, s1, q0 = Acc(0), q1 = Acc(0);
    if (two) {
      const V tl = __ldg(reinterpret_cast<const V*>(sat + top + j));
      const V tr = __ldg(reinterpret_cast<const V*>(sat + top + j + g.w));
      const V bl = __ldg(reinterpret_cast<const V*>(sat + bot + j));
      const V br = __ldg(reinterpret_cast<const V*>(sat + bot + j + g.w));
      s0 = corner4<Acc>(br.x, tr.x, bl.x, tl.x);
      s1 = corner4<Acc>(br.y, tr.y, bl.y, tl.y);
      if constexpr (SQ) {
        const V qtl = __ldg(reinterpret_cast<const V*>(sq + top + j));
        const V qtr = __ldg(reinterpret_cast<const V*>(sq + top + j + g.w));
        const V qbl = __ldg(reinterpret_cast<const V*>(sq + bot + j));
        const V qbr = __ldg(reinterpret_cast<const V*>(sq + bot + j + g.w));
        q0 = corner4<Acc>(qbr.x, qtr.x, qbl.x, qtl.x);
        q1 = corner4<Acc>(qbr.y, qtr.y, qbl.y, qtl.y);
      }
    } else {
      s0 = corner4(__ldg(sat + bot + j + g.w), __ldg(sat + top + j + g.w), __ldg(sat + bot + j), __ldg(sat + top + j));
      s1 = s0;
      if constexpr (SQ) {
        q0 = corner4(__ldg(sq + bot + j + g.w), __ldg(sq + top + j + g.w), __ldg(sq + bot + j), __ldg(sq + top + j));
        q1 = q0;
      }
    }
    emit_pair<Acc>(g, o, fin, i, j, s0, s1, q0, q1, two, vec_out);
  }
}

// General path: any stride / odd window; two outputs per thread, strided.
template <typename Acc, bool SQ>
__global__ void __launch_bounds__(kThreads)
window_eval_gen_kernel(const Acc* __restrict__ sat, const Acc* __restrict__ sq, EvalGeom g, WinOut o, Fin<Acc> fin) {
  for (int64_t it = blockIdx.x; it < g.n_items; it += gridDim.x) {
    int64_t i, cb;
    decode_item(g, it, i, cb);
    const int64_t top = i * g.s * g.sat_ld, bot = (i * g.s + g.w) * g.sat_ld;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int64_t j = cb + threadIdx.x + h * kThreads;
      if (j >= g.out_c) continue;
      const int64_t l = j * g.s, r = j * g.s + g.w;
      const Acc s0 = corner4(__ldg(sat + bot + r), __ldg(sat + top + r), __ldg(sat + bot + l), __ldg(sat + top + l));
      Acc q0 = Acc(0);
      if constexpr (SQ) q0 = corner4(__ldg(sq + bot + r), __ldg(sq + top + r), __ldg(sq + bot + l), __ldg(sq + top + l));
      emit_pair<Acc>(g, o, fin, i, j, s0, s0, q0, q0, false, false);
    }
  }
}

inline EvalGeom make_eval_geom(int64_t R, int64_t C, int64_t w, int64_t s, int64_t sat_ld, int mask, bool sq) {
  EvalGeom g{};
  g.out_r = (R - w) / s + 1;
  g.out_c = (C - w) / s + 1;
  g.w = w; g.s = s; g.sat_ld = sat_ld; g.mask = mask;
  // panel: keep (w*s + 1) table rows of the panel (both tables) in ~48 MB of L2
  const double budget = 48.0 * 1024 * 1024;
  const double row_bytes = 8.0 * (sq ? 2 : 1) * (double)(w + 1);
  int64_t pw = (int64_t)(budget / row_bytes / (double)s);
  pw = (pw / kChunk) * kChunk;
  if (pw < kChunk) pw = kChunk;
  const int64_t full = ((g.out_c + kChunk - 1) / kChunk) * kChunk;
  if (pw > full) pw = full;
  g.pw = pw;
  g.n_panels = (g.out_c + pw - 1) / pw;
  g.cpp = pw / kChunk;
  const int64_t last_w = g.out_c - (g.n_panels - 1) * pw;
  g.cpl = (last_w + kChunk - 1) / kChunk;
  g.n_items = g.out_r * (g.cpp * (g.n_panels - 1) + g.cpl);
  return g;
}

cudaError_t launch_window_eval(const void* sat, const void* sat_sq, bool is_float, int in_dtype, int64_t R, int64_t C,
                               int64_t sat_ld, int64_t w, int64_t s, int mask, WinOut o, cudaStream_t st) {
  const bool sq = (mask & ST_STD) != 0;
  const EvalGeom g = make_eval_geom(R, C, w, s, sat_ld, mask, sq);
  if (g.n_items <= 0) return cudaSuccess;
  const bool vec = (s == 1) && ((w & 1) == 0) && ((sat_ld & 1) == 0) &&
                   ((reinterpret_cast<uintptr_t>(sat) & 15) == 0) &&
                   (!sq || (reinterpret_cast<uintptr_t>(sat_sq) & 15) == 0);
  const int64_t max_blocks = (int64_t)kNumSMs * 8;
  const int blocks = (int)(g.n_items < max_blocks ? g.n_items : max_blocks);
  const double dn = (double)(w * w);
  if (is_float) {
    Fin<double> fin{dn};
    const double* a = reinterpret_cast<const double*>(sat);
    const double* b = reinterpret_cast<const double*>(sat_sq);
    if (vec) { if (sq) window_eval_vec_kernel<double, true><<<blocks, kThreads, 0, st>>>(a, b, g, o, fin);
               else window_eval_vec_kernel<double, false><<<blocks, kThreads, 0, st>>>(a, b, g, o, fin); }
    else { if (sq) window_eval_gen_kernel<double, true><<<blocks, kThreads, 0, st>>>(a, b, g, o, fin);
           else window_eval_gen_kernel<double, false><<<blocks, kThreads, 0, st>>>(a, b, g, o, fin); }
  } else {
    Fin<uint64_t> fin{};
    fin.f.n = (uint64_t)(w * w);
    fin.f.dn = dn;
    const double maxv = in_dtype == IN_U8 ? 255.0 : in_dtype == IN_U16 ? 65535.0 : 2147483648.0;
    // w^4 * max^2 <= 2^64 - 1, evaluated exactly in 128-bit integers
    {
      unsigned __int128 ww = (unsigned __int128)(uint64_t)w * (uint64_t)w;
      unsigned __int128 m = (unsigned __int128)(uint64_t)maxv;
      bool ok = true;
      // (ww*m)^2 <= lim  <=>  ww*m <= floor(sqrt(lim)) = 2^32 - 1 (exact since lim = 2^64-1)
      unsigned __int128 a = ww * m;
      if (a > (unsigned __int128)0xFFFFFFFFull) ok = false;
      fin.f.u64_ok = ok;
    }
    fin.f.is_signed = (in_dtype == IN_I32);
    const uint64_t* a = reinterpret_cast<const uint64_t*>(sat);
    const uint64_t* b = reinterpret_cast<const uint64_t*>(sat_sq);
    if (vec) { if (sq) window_eval_vec_kernel<uint64_t, true><<<blocks, kThreads, 0, st>>>(a, b, g, o, fin);
               else window_eval_vec_kernel<uint64_t, false><<<blocks, kThreads, 0, st>>>(a, b, g, o, fin); }
    else { if (sq) window_eval_gen_kernel<uint64_t, true><<<blocks, kThreads, 0, st>>>(a, b, g, o, fin);
           else window_eval_gen_kernel<uint64_t, false><<<blocks, kThreads, 0, st>>>(a, b, g, o, fin); }
  }
  note_launch(1);
  return cudaGetLastError();
}

}  // namespace ssb
