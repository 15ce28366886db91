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
#include <atomic>
#include <cstdlib>

#include "ssb_async.cuh"
#include "ssb_common.cuh"

namespace ssb {

struct EvalGeom {
  int64_t out_r, out_c, w, s, sat_ld;
  int64_t pw;        // panel width in output columns (multiple of kChunk)
  int64_t n_panels, cpp, cpl;  // chunks per full panel / in the last panel
  int64_t n_items;
  int mask;
  int vec_out;  // output rows aligned for VW-wide stores
  int hints;    // L2 policy: 0 none, 1 bottom evict_last + top evict_first, 2 top evict_first only
  Census cz;
};

constexpr int kChunk = 2 * kThreads;  // 512 output columns per work item

template <typename Acc> struct Fin;
template <> struct Fin<uint64_t> {
  FinalizeInt f;
  __device__ __forceinline__ double mean(uint64_t s) const { return fin_mean_int(s, f); }
  __device__ __forceinline__ double std_(uint64_t s, uint64_t q) const { return fin_std_int(s, q, f); }
};
template <> struct Fin<double> {
  double dn, inv;
  __device__ __forceinline__ double mean(double s) const { return fin_mean_f(s, dn, inv); }
  __device__ __forceinline__ double std_(double s, double q) const { return fin_std_f(s, q, dn, inv); }
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
      census_add(g.cz.orow, g.cz.nor, i);
    }
  }
}

// Row-sweep path (stride 1).  CTA b owns chunk (b % cpp) of every panel and
// visits output rows q, q+k, q+2k, ... (q = b / cpp, k = gridDim / cpp); all
// CTAs are resident at once, so the rows in flight form a narrow band of one
// panel and the top corner row of output row i (loaded as a bottom row w rows
// earlier) is served from L2.  Lane l of warp v evaluates outputs
// j = chunk + 128 v + l + 32 u (u < 4): every corner load and every store is a
// fully coalesced 256-byte warp access, whatever the alignment of the output
// rows (a contiguous 69,745 x 84,745 result has 8-byte-aligned rows), and each
// thread keeps 16 independent loads in flight.  No integer division in the loop.
constexpr int kOutPerThread = 4;
constexpr int kRowChunk = kThreads * kOutPerThread;  // 1024 outputs per CTA row step

__device__ __forceinline__ uint64_t ldg_hint(const uint64_t* p, uint64_t pol) {
  uint64_t v;
  asm volatile("ld.global.nc.L2::cache_hint.b64 %0, [%1], %2;" : "=l"(v) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ double ldg_hint(const double* p, uint64_t pol) {
  return __longlong_as_double((long long)ldg_hint(reinterpret_cast<const uint64_t*>(p), pol));
}

template <typename Acc, bool SQ>
__global__ void __launch_bounds__(kThreads)
window_eval_rows_kernel(const Acc* __restrict__ sat, const Acc* __restrict__ sq, EvalGeom g, WinOut o, Fin<Acc> fin) {
  constexpr int U = kOutPerThread;
  const int cpp = (int)g.cpp;
  const int c = blockIdx.x % cpp;
  const int q = blockIdx.x / cpp;
  const int k = gridDim.x / cpp;
  if (q >= k) return;
  const uint64_t keep = g.hints == 1 ? policy_evict_last() : policy_evict_normal();
  const uint64_t drop = g.hints == 0 ? policy_evict_normal() : policy_evict_first();
  const int64_t w = g.w, ld = g.sat_ld;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int64_t p = 0; p < g.n_panels; ++p) {
    const int64_t chunks = (p == g.n_panels - 1) ? g.cpl : g.cpp;
    if (c >= chunks) continue;
    const int64_t jb = p * g.pw + (int64_t)c * kRowChunk + warp * (32 * U) + lane;
    if (jb >= g.out_c) continue;
    const bool full = jb + 32 * (U - 1) < g.out_c;
#pragma unroll 2
    for (int64_t i = q; i < g.out_r; i += k) {
      const Acc* top = sat + i * ld + jb;
      const Acc* bot = top + w * ld;
      Acc s[U], qq[U];
      if (full) {
        Acc tl[U], tr[U], bl[U], br[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          tl[u] = ldg_hint(top + 32 * u, drop);
          tr[u] = ldg_hint(top + 32 * u + w, drop);
          bl[u] = ldg_hint(bot + 32 * u, keep);
          br[u] = ldg_hint(bot + 32 * u + w, keep);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) s[u] = corner4<Acc>(br[u], tr[u], bl[u], tl[u]);
        if constexpr (SQ) {
          const Acc* qt = sq + i * ld + jb;
          const Acc* qb = qt + w * ld;
#pragma unroll
          for (int u = 0; u < U; ++u) {
            tl[u] = ldg_hint(qt + 32 * u, drop);
            tr[u] = ldg_hint(qt + 32 * u + w, drop);
            bl[u] = ldg_hint(qb + 32 * u, keep);
            br[u] = ldg_hint(qb + 32 * u + w, keep);
          }
#pragma unroll
          for (int u = 0; u < U; ++u) qq[u] = corner4<Acc>(br[u], tr[u], bl[u], tl[u]);
        }
      } else {
#pragma unroll
        for (int u = 0; u < U; ++u) {
          if (jb + 32 * u < g.out_c) {
            const int64_t d = 32 * u;
            s[u] = corner4<Acc>(__ldg(bot + d + w), __ldg(top + d + w), __ldg(bot + d), __ldg(top + d));
            if constexpr (SQ) {
              const Acc* qt = sq + i * ld + jb;
              const Acc* qb = qt + w * ld;
              qq[u] = corner4<Acc>(__ldg(qb + d + w), __ldg(qt + d + w), __ldg(qb + d), __ldg(qt + d));
            }
          }
        }
      }
      const int64_t base = i * o.ld + jb;
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (!full && jb + 32 * u >= g.out_c) break;
        const int64_t at = base + 32 * u;
        if (g.mask & ST_SUM) st_cs(reinterpret_cast<Acc*>(o.sum) + at, s[u]);
        if (g.mask & ST_MEAN) st_cs(o.mean + at, fin.mean(s[u]));
        if constexpr (SQ) if (g.mask & ST_STD) st_cs(o.std_ + at, fin.std_(s[u], qq[u]));
        census_add(g.cz.orow, g.cz.nor, i);
      }
    }
  }
}

// panel width (output columns, multiple of `chunk`) that keeps the w+1 table
// rows a panel touches (both tables) within ~`budget` bytes of L2
inline int64_t panel_width(int64_t out_c, int64_t w, int64_t s, bool sq, int64_t chunk, double budget) {
  const double row_bytes = 8.0 * (sq ? 2 : 1) * (double)(w * s + 1);
  int64_t pw = (int64_t)(budget / row_bytes);
  pw = (pw / chunk) * chunk;
  if (pw < chunk) pw = chunk;
  const int64_t full = ((out_c + chunk - 1) / chunk) * chunk;
  return pw > full ? full : pw;
}

// TMA path (stride 1, moderate w): per row step the CTA bulk-copies the top and
// bottom table row segments [j0, j0 + CW + w) into shared memory (cp.async.bulk,
// 4-stage full/empty mbarrier ring driven by one producer thread), then every
// thread evaluates outputs j0 + t + 256 u from shared memory and streams them
// out with coalesced stores.  Each table byte crosses L2->SM about
// (CW + w) / CW times per row instead of twice, and the copy engine keeps tens
// of KB per SM in flight without occupying load slots.
constexpr int kTmaMaxNS = 8;  // pipeline depth (runtime, <= 8)

// Work items are handed out in order by an atomic ticket, so the items in
// flight are always a contiguous range of the global order: the rows being
// evaluated stay a narrow band of one panel and a table row fetched as a bottom
// corner row is still in L2 when it is needed as a top corner row w rows later
// (a static assignment lets CTAs drift apart and doubled the table reads).
//
// Item = (panel p, bottom table row rb, chunk c).  The stage holds the bottom
// row segment once and one top row segment per window whose output row
// rb - w_k exists, so with several windows (multi_window,
// integral.py:199-210) the shared bottom row crosses L2->SM once instead of
// once per window.  The sweep is bound by L2 throughput (~12 TB/s for hits,
// misses and the output stream together), so bytes moved into shared memory
// are what this layout minimises; every table byte comes from HBM about once
// for the whole window set.
__device__ unsigned long long g_eval_tickets[256];

constexpr int kMaxWin = 8;
struct MultiEval {
  int nwin;
  int mask;
  int is_signed;
  int64_t wmin, wmax, R, sat_ld;
  int64_t pw, n_panels, cpp, cpl;       // panels of output columns (chunks of CW)
  int64_t w[kMaxWin], out_r[kMaxWin], out_c[kMaxWin];
  WinOut o[kMaxWin];
  uint64_t n[kMaxWin];
  double dn[kMaxWin], inv[kMaxWin];
  unsigned char u64_ok[kMaxWin];
  // stage layout (elements, per table): bottom segment at 0, top segment of
  // window k at off[k]; a stage is NT * stage_elems elements
  int off[kMaxWin];
  int stage_elems;
  Census cz;
  int64_t census_off[kMaxWin];  // first census row of window k
};

template <typename Acc> struct FinK;
template <> struct FinK<uint64_t> {
  __device__ static Fin<uint64_t> make(const MultiEval& m, int k) {
    Fin<uint64_t> f{};
    f.f.n = m.n[k]; f.f.dn = m.dn[k]; f.f.inv_n = m.inv[k]; f.f.u64_ok = m.u64_ok[k] != 0;
    f.f.is_signed = m.is_signed != 0;
    return f;
  }
};
template <> struct FinK<double> {
  __device__ static Fin<double> make(const MultiEval& m, int k) { return Fin<double>{m.dn[k], m.inv[k]}; }
};

// even number of elements covering [j0, j0 + CW + w) (reads reach index CW - 1 + w)
__host__ __device__ __forceinline__ int64_t seg_need(int64_t cw, int64_t w) { return (cw + w + 1) & ~int64_t(1); }

template <typename Acc, bool SQ, int U, bool MULTI, bool HINTS>
__global__ void __launch_bounds__(kThreads + 32)
window_eval_tma_kernel(const Acc* __restrict__ sat, const Acc* __restrict__ sq, const __grid_constant__ MultiEval g,
                       unsigned long long* __restrict__ ticket, int NS, int batch) {
  constexpr int NT = SQ ? 2 : 1;
  constexpr int kTmaCW = kThreads * U;  // output columns per item
  extern __shared__ __align__(16) unsigned char smem_raw[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw);
  uint64_t* empty = full + kTmaMaxNS;
  // per stage: bottom table row (-1 done, -2 skip), first column j0, window mask
  int64_t* meta = reinterpret_cast<int64_t*>(empty + kTmaMaxNS);
  int64_t* meta_j0 = meta + kTmaMaxNS;
  int* meta_mask = reinterpret_cast<int*>(meta_j0 + kTmaMaxNS);
  Acc* buf = reinterpret_cast<Acc*>(smem_raw + 384);              // [NS][NT][stage_elems]
  const int tid = threadIdx.x, lane = tid & 31;
  const int64_t ld = g.sat_ld;
  const int nwin = MULTI ? g.nwin : 1;
  const int64_t stage_stride = (int64_t)NT * g.stage_elems;
  const int64_t nrb = g.R + 1 - g.wmin;  // bottom rows wmin..R
  const int64_t per_panel = nrb * g.cpp;
  const int64_t total = per_panel * (g.n_panels - 1) + nrb * g.cpl;
  if (tid == 0) {
    for (int i = 0; i < NS; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], kThreads / 32);
    }
    fence_mbar_init();
  }
  __syncthreads();
  // warp 8 is the producer (one elected lane); warps 0-7 consume
  if (tid >= kThreads) {
    if (lane != 0) return;
    int64_t cur = 0, cur_end = 0;
    int64_t next_b = (int64_t)atomicAdd(ticket, (unsigned long long)batch);
    // decoded position of `cur`: full decode at the start of a ticket batch,
    // then a carry-propagating increment (no divisions on the issue path).
    // 32-bit arithmetic: item counts stay far below 2^31.
    const uint32_t ppan = (uint32_t)per_panel, cppf = (uint32_t)g.cpp, cppl = (uint32_t)g.cpl;
    const uint32_t nrb32 = (uint32_t)nrb;
    uint32_t dp = 0, drb = 0, dc = 0, dcpp = 0;
    auto decode = [&](int64_t it64) {
      const uint32_t it = (uint32_t)it64;
      dp = it / ppan;
      const uint32_t rem = it - dp * ppan;
      dcpp = ((int64_t)dp == g.n_panels - 1) ? cppl : cppf;
      drb = rem / dcpp;
      dc = rem - drb * dcpp;
    };
    auto advance = [&]() {
      if (++dc < dcpp) return;
      dc = 0;
      if (++drb < nrb32) return;
      drb = 0;
      ++dp;
      dcpp = ((int64_t)dp == g.n_panels - 1) ? cppl : cppf;
    };
    uint64_t pol_keep = 0, pol_drop = 0;
    if constexpr (HINTS) { pol_keep = policy_evict_last(); pol_drop = policy_evict_first(); }
    uint32_t s = 0, phase = 0;
    for (int64_t m = 0;; ++m) {
      if (m >= NS) mbar_wait(&empty[s], phase ^ 1u);
      if (cur == cur_end) {  // tickets come in batches; the next batch is requested ahead
        cur = next_b;
        cur_end = next_b + batch;
        if (cur < total) next_b = (int64_t)atomicAdd(ticket, (unsigned long long)batch);
        if (cur < total) decode(cur);
      } else {
        advance();
      }
      const int64_t it = cur++;
      if (it >= total) {
        meta[s] = -1;
        mbar_arrive_expect_tx(&full[s], 0);
        return;
      }
      const int64_t rb = (int64_t)drb + g.wmin;
      const int64_t j0 = (int64_t)dp * g.pw + (int64_t)dc * kTmaCW;
      const int64_t avail = ld - j0;
      int mask = 0;
      int64_t wv = 0;
      uint32_t bytes = 0;
      for (int k = 0; k < nwin; ++k) {
        if (rb >= g.w[k] && j0 < g.out_c[k]) {  // output row rb - w_k exists, chunk inside its columns
          mask |= 1 << k;
          wv = g.w[k] > wv ? g.w[k] : wv;
          const int64_t len = seg_need(kTmaCW, g.w[k]);
          bytes += (uint32_t)((len < avail ? len : avail) * 8);
        }
      }
      if (mask == 0) {
        meta[s] = -2;
        mbar_arrive_expect_tx(&full[s], 0);
      } else {
        meta[s] = rb;
        meta_j0[s] = j0;
        meta_mask[s] = mask;
        const int64_t lb = seg_need(kTmaCW, wv);
        const uint32_t bb = (uint32_t)((lb < avail ? lb : avail) * 8);
        fence_proxy_async();
        mbar_arrive_expect_tx(&full[s], (bytes + bb) * NT);
        Acc* b = buf + (int64_t)s * stage_stride;
        if constexpr (HINTS) {
          // bottom rows come back as top rows w rows later: keep them in L2;
          // a top row of the largest window is read for the last time
          bulk_g2s_hint(b, sat + rb * ld + j0, bb, &full[s], pol_keep);
          if constexpr (SQ) bulk_g2s_hint(b + g.stage_elems, sq + rb * ld + j0, bb, &full[s], pol_keep);
        } else {
          bulk_g2s(b, sat + rb * ld + j0, bb, &full[s]);
          if constexpr (SQ) bulk_g2s(b + g.stage_elems, sq + rb * ld + j0, bb, &full[s]);
        }
        for (int k = 0; k < nwin; ++k) {
          if (!((mask >> k) & 1)) continue;
          const int64_t len = seg_need(kTmaCW, g.w[k]);
          const uint32_t tb = (uint32_t)((len < avail ? len : avail) * 8);
          const int64_t top = (rb - g.w[k]) * ld + j0;
          if constexpr (HINTS) {
            const uint64_t pol = g.w[k] == g.wmax ? pol_drop : pol_keep;
            bulk_g2s_hint(b + g.off[k], sat + top, tb, &full[s], pol);
            if constexpr (SQ) bulk_g2s_hint(b + g.stage_elems + g.off[k], sq + top, tb, &full[s], pol);
          } else {
            bulk_g2s(b + g.off[k], sat + top, tb, &full[s]);
            if constexpr (SQ) bulk_g2s(b + g.stage_elems + g.off[k], sq + top, tb, &full[s]);
          }
        }
      }
      if (++s == (uint32_t)NS) { s = 0; phase ^= 1u; }
    }
  }
  uint32_t s = 0, phase = 0;
  for (;;) {
    mbar_wait(&full[s], phase);
    const int64_t rb = meta[s];
    if (rb == -1) break;
    if (rb != -2) {
      const int64_t j0 = meta_j0[s];
      const int mask = meta_mask[s];
      const Acc* B = buf + (int64_t)s * stage_stride;
      // bottom-left corners are shared by every window
      Acc bl[U], blq[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        bl[u] = B[tid + kThreads * u];
        if constexpr (SQ) blq[u] = B[g.stage_elems + tid + kThreads * u];
      }
      auto window = [&](int k) {
        const int w = (int)g.w[k];
        const Acc* T = B + g.off[k];
        Acc sv[U], qv[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int jj = tid + kThreads * u;
          sv[u] = corner4<Acc>(B[jj + w], T[jj + w], bl[u], T[jj]);
          if constexpr (SQ) {
            const Acc* BQ = B + g.stage_elems;
            const Acc* TQ = T + g.stage_elems;
            qv[u] = corner4<Acc>(BQ[jj + w], TQ[jj + w], blq[u], TQ[jj]);
          }
        }
        const WinOut& o = g.o[k];
        const Fin<Acc> fin = FinK<Acc>::make(g, k);
        const int64_t base = (rb - w) * o.ld + j0;
        const int64_t oc = g.out_c[k] - j0;
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int jj = tid + kThreads * u;
          if (jj >= oc) break;
          const int64_t at = base + jj;
          if (g.mask & ST_SUM) st_cs(reinterpret_cast<Acc*>(o.sum) + at, sv[u]);
          if (g.mask & ST_MEAN) st_cs(o.mean + at, fin.mean(sv[u]));
          if constexpr (SQ) if (g.mask & ST_STD) st_cs(o.std_ + at, fin.std_(sv[u], qv[u]));
          census_add(g.cz.orow, g.cz.nor, g.census_off[k] + (rb - w));
        }
      };
      if constexpr (MULTI) {
        // a rolled loop: the 8-slot unrolled form ran slower (instruction
        // cache pressure) despite fewer instructions
#pragma unroll 1
        for (int k = 0; k < nwin; ++k)
          if ((mask >> k) & 1) window(k);
      } else {
        window(0);
      }
    }
    __syncwarp();
    if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&empty[s])) : "memory");
    if (++s == (uint32_t)NS) { s = 0; phase ^= 1u; }
  }
}

// panel width (output columns, multiple of `chunk`) that keeps the w+1 table
// rows a panel touches (both tables) within ~`budget` bytes of L2
inline int64_t panel_width_max(int64_t out_c, int64_t wmax, bool sq, int64_t chunk, double budget) {
  const double row_bytes = 8.0 * (sq ? 2 : 1) * (double)(wmax + 1);
  int64_t pw = (int64_t)(budget / row_bytes);
  pw = (pw / chunk) * chunk;
  if (pw < chunk) pw = chunk;
  const int64_t full = ((out_c + chunk - 1) / chunk) * chunk;
  return pw > full ? full : pw;
}

template <typename Acc, bool SQ, int U>
cudaError_t launch_tma_multi_u(const void* sat, const void* sat_sq, MultiEval m, cudaStream_t st, bool& used) {
  used = false;
  constexpr int NT = SQ ? 2 : 1;
  constexpr int64_t kTmaCW = kThreads * U;
  static const int batch = env_int("SSB_EVAL_BATCH", 4);
  static const int env_ns = env_int("SSB_EVAL_STAGES", 0);
  // multi-window stages are large (a top segment per window): 2 stages keep
  // 3 CTAs per SM resident (C3 sweep 9.2 -> 8.5 ms); single window: 3 stages
  int NS = env_ns > 0 ? env_ns : (m.nwin > 1 ? 2 : 3);
  if (NS < 2) NS = 2;
  if (NS > kTmaMaxNS) NS = kTmaMaxNS;
  // stage layout: bottom segment (covers the widest window), then one top
  // segment per window; every segment an even element count (16-byte aligned)
  int64_t el = seg_need(kTmaCW, m.wmax);
  for (int k = 0; k < m.nwin; ++k) {
    m.off[k] = (int)el;
    el += seg_need(kTmaCW, m.w[k]);
  }
  m.stage_elems = (int)el;
  const size_t smem = 384 + (size_t)NS * NT * el * sizeof(Acc);
  if (smem > 220 * 1024 || (reinterpret_cast<uintptr_t>(sat) & 15) ||
      (SQ && (reinterpret_cast<uintptr_t>(sat_sq) & 15)) || (m.sat_ld & 1))
    return cudaSuccess;
  static const double env_mb = env_double("SSB_EVAL_L2_MB", 0.0);
  int64_t out_c_max = 0;
  for (int k = 0; k < m.nwin; ++k) out_c_max = m.out_c[k] > out_c_max ? m.out_c[k] : out_c_max;
  // the panel's wmax + 1 most recent table rows stay hot in L2.  Single
  // window: 16 MB panels with evict_last on bottom rows / evict_first on top
  // rows (C5 sweep 15.14 -> 14.81 ms); the multi-window set measured best
  // without policies at 8 MB.
  const double mb = env_mb > 0 ? env_mb : (m.nwin == 1 ? 16.0 : 8.0);
  m.pw = panel_width_max(out_c_max, m.wmax, SQ, kTmaCW, mb * 1024 * 1024);
  m.n_panels = (out_c_max + m.pw - 1) / m.pw;
  m.cpp = m.pw / kTmaCW;
  m.cpl = (out_c_max - (m.n_panels - 1) * m.pw + kTmaCW - 1) / kTmaCW;
  const bool multi = m.nwin > 1;
  static const int env_h = env_int("SSB_EVAL_TMA_HINTS", -1);  // tuning: L2 policies on the table row copies
  const bool hints = env_h >= 0 ? env_h != 0 : !multi;
  auto kfn = multi ? (hints ? window_eval_tma_kernel<Acc, SQ, U, true, true> : window_eval_tma_kernel<Acc, SQ, U, true, false>)
                   : (hints ? window_eval_tma_kernel<Acc, SQ, U, false, true> : window_eval_tma_kernel<Acc, SQ, U, false, false>);
  cudaError_t e = cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int per_sm = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kfn, kThreads + 32, smem);
  if (e != cudaSuccess || per_sm < 1) per_sm = 1;
  const int blocks = kNumSMs * per_sm;
  // one ticket counter per launch, from a small ring (concurrent launches on
  // different streams get different slots)
  static std::atomic<unsigned> slot{0};
  unsigned long long* tickets = nullptr;
  e = cudaGetSymbolAddress(reinterpret_cast<void**>(&tickets), g_eval_tickets);
  if (e != cudaSuccess) return e;
  unsigned long long* ticket = tickets + (slot.fetch_add(1) % 256);
  e = cudaMemsetAsync(ticket, 0, sizeof(unsigned long long), st);
  if (e != cudaSuccess) return e;
  kfn<<<blocks, kThreads + 32, smem, st>>>(reinterpret_cast<const Acc*>(sat), reinterpret_cast<const Acc*>(sat_sq),
                                           m, ticket, NS, batch);
  used = true;
  return cudaGetLastError();
}

template <typename Acc, bool SQ>
cudaError_t launch_tma_multi(const void* sat, const void* sat_sq, const MultiEval& m, cudaStream_t st, bool& used) {
  // multi-window stages hold one top segment per window: narrower chunks keep
  // two CTAs per SM resident (tuning: SSB_EVAL_U=2|4)
  static const int env_u = env_int("SSB_EVAL_U", 0);
  const int u = env_u > 0 ? env_u : (m.nwin > 2 ? 2 : 4);
  if (u == 1) return launch_tma_multi_u<Acc, SQ, 1>(sat, sat_sq, m, st, used);
  if (u == 2) return launch_tma_multi_u<Acc, SQ, 2>(sat, sat_sq, m, st, used);
  return launch_tma_multi_u<Acc, SQ, 4>(sat, sat_sq, m, st, used);
}

inline void fill_fin(MultiEval& m, int k, int in_dtype) {
  const uint64_t w = (uint64_t)m.w[k];
  m.n[k] = w * w;
  m.dn[k] = (double)(w * w);
  m.inv[k] = 1.0 / m.dn[k];
  const uint64_t maxv = in_dtype == IN_U8 ? 255u : in_dtype == IN_U16 ? 65535u : 2147483648u;
  // stats.py:28-32: w^4 * max^2 <= 2^64 - 1  <=>  w^2 * max <= 2^32 - 1
  m.u64_ok[k] = ((unsigned __int128)(w * w) * maxv) <= (unsigned __int128)0xFFFFFFFFull ? 1 : 0;
}

// single-window wrapper over the multi-window TMA kernel
template <typename Acc, bool SQ>
cudaError_t launch_tma(const void* sat, const void* sat_sq, EvalGeom g, WinOut o, int in_dtype, cudaStream_t st,
                       bool& used) {
  MultiEval m{};
  m.nwin = 1;
  m.mask = g.mask;
  m.is_signed = in_dtype == IN_I32;
  m.wmin = m.wmax = g.w;
  m.R = g.out_r + g.w - 1;
  m.sat_ld = g.sat_ld;
  m.w[0] = g.w; m.out_r[0] = g.out_r; m.out_c[0] = g.out_c; m.o[0] = o;
  m.cz = g.cz;
  m.census_off[0] = 0;
  fill_fin(m, 0, in_dtype);
  return launch_tma_multi<Acc, SQ>(sat, sat_sq, m, st, used);
}

inline EvalGeom make_eval_geom(int64_t R, int64_t C, int64_t w, int64_t s, int64_t sat_ld, int mask, bool sq) {
  EvalGeom g{};
  g.out_r = (R - w) / s + 1;
  g.out_c = (C - w) / s + 1;
  g.w = w; g.s = s; g.sat_ld = sat_ld; g.mask = mask;
  g.cz = census_sink();
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

inline int env_int_cached_hints() {
  static const int h = env_int("SSB_EVAL_HINTS", 2);
  return h;
}

template <typename Acc, bool SQ>
cudaError_t launch_rows(const void* sat, const void* sat_sq, EvalGeom g, WinOut o, Fin<Acc> fin, cudaStream_t st) {
  constexpr int64_t CH = kRowChunk;
  static const double env_mb = env_double("SSB_EVAL_L2_MB", 24.0);
  static const int env_k = env_int("SSB_EVAL_ROWS_IN_FLIGHT", 0);
  g.hints = env_int_cached_hints();
  g.pw = panel_width(g.out_c, g.w, 1, SQ, CH, env_mb * 1024 * 1024);
  g.n_panels = (g.out_c + g.pw - 1) / g.pw;
  g.cpp = g.pw / CH;
  g.cpl = (g.out_c - (g.n_panels - 1) * g.pw + CH - 1) / CH;
  // persistent grid: every CTA resident at once, so the rows in flight stay a
  // narrow band and the panel's w table rows stay in L2
  int per_sm = 0;
  cudaError_t oe = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, window_eval_rows_kernel<Acc, SQ>,
                                                                 kThreads, 0);
  if (oe != cudaSuccess || per_sm < 1) per_sm = 1;
  int64_t k = (int64_t)kNumSMs * per_sm / g.cpp;
  if (env_k > 0 && env_k < k) k = env_k;
  if (k < 1) k = 1;
  if (k > g.out_r) k = g.out_r;
  const int blocks = (int)(k * g.cpp);
  window_eval_rows_kernel<Acc, SQ><<<blocks, kThreads, 0, st>>>(reinterpret_cast<const Acc*>(sat),
                                                               reinterpret_cast<const Acc*>(sat_sq), g, o, fin);
  return cudaGetLastError();
}

template <typename Acc>
cudaError_t launch_eval_t(const void* sat, const void* sat_sq, EvalGeom g, WinOut o, Fin<Acc> fin, bool sq, int in_dtype,
                          cudaStream_t st) {
  if (g.s == 1) {
    static const bool ldg = env_char("SSB_EVAL_PATH") == 'l';  // tuning: "ldg" forces the load-based sweep
    if (!ldg) {
      bool used = false;
      cudaError_t e = sq ? launch_tma<Acc, true>(sat, sat_sq, g, o, in_dtype, st, used)
                         : launch_tma<Acc, false>(sat, sat_sq, g, o, in_dtype, st, used);
      if (e != cudaSuccess || used) return e;
    }
    return sq ? launch_rows<Acc, true>(sat, sat_sq, g, o, fin, st) : launch_rows<Acc, false>(sat, sat_sq, g, o, fin, st);
  }
  const int64_t max_blocks = (int64_t)kNumSMs * 8;
  const int blocks = (int)(g.n_items < max_blocks ? g.n_items : max_blocks);
  const Acc* x = reinterpret_cast<const Acc*>(sat);
  const Acc* y = reinterpret_cast<const Acc*>(sat_sq);
  if (sq) window_eval_gen_kernel<Acc, true><<<blocks, kThreads, 0, st>>>(x, y, g, o, fin);
  else window_eval_gen_kernel<Acc, false><<<blocks, kThreads, 0, st>>>(x, y, g, o, fin);
  return cudaGetLastError();
}

cudaError_t launch_window_eval(const void* sat, const void* sat_sq, bool is_float, int in_dtype, int64_t R, int64_t C,
                               int64_t sat_ld, int64_t w, int64_t s, int mask, WinOut o, cudaStream_t st) {
  const bool sq = (mask & ST_STD) != 0;
  const EvalGeom g = make_eval_geom(R, C, w, s, sat_ld, mask, sq);
  if (g.n_items <= 0) return cudaSuccess;
  cudaError_t e;
  if (is_float) {
    Fin<double> fin{(double)(w * w), 1.0 / (double)(w * w)};
    e = launch_eval_t<double>(sat, sat_sq, g, o, fin, sq, in_dtype, st);
  } else {
    Fin<uint64_t> fin{};
    fin.f.n = (uint64_t)(w * w);
    fin.f.dn = (double)(w * w);
    fin.f.inv_n = 1.0 / fin.f.dn;
    const uint64_t maxv = in_dtype == IN_U8 ? 255u : in_dtype == IN_U16 ? 65535u : 2147483648u;
    // stats.py:28-32: w^4 * max^2 <= 2^64 - 1  <=>  w^2 * max <= 2^32 - 1
    fin.f.u64_ok = ((unsigned __int128)(uint64_t)(w * w) * maxv) <= (unsigned __int128)0xFFFFFFFFull;
    fin.f.is_signed = (in_dtype == IN_I32);
    e = launch_eval_t<uint64_t>(sat, sat_sq, g, o, fin, sq, in_dtype, st);
  }
  note_launch(1);
  return e;
}

// Several stride-1 windows from one table pass (single kernel); returns
// cudaErrorNotSupported if the TMA path cannot take this request.
cudaError_t launch_window_eval_multi(const void* sat, const void* sat_sq, bool is_float, int in_dtype, int64_t R,
                                     int64_t C, int64_t sat_ld, int nwin, const int64_t* ws, int mask, const WinOut* outs,
                                     cudaStream_t st) {
  if (nwin < 1 || nwin > kMaxWin) return cudaErrorNotSupported;
  MultiEval m{};
  m.nwin = nwin;
  m.mask = mask;
  m.cz = census_sink();
  m.is_signed = in_dtype == IN_I32;
  m.R = R;
  m.sat_ld = sat_ld;
  m.wmin = ws[0];
  m.wmax = ws[0];
  for (int k = 0; k < nwin; ++k) {
    m.w[k] = ws[k];
    m.out_r[k] = R - ws[k] + 1;
    m.out_c[k] = C - ws[k] + 1;
    m.o[k] = outs[k];
    m.census_off[k] = k == 0 ? 0 : m.census_off[k - 1] + m.out_r[k - 1];
    m.wmin = ws[k] < m.wmin ? ws[k] : m.wmin;
    m.wmax = ws[k] > m.wmax ? ws[k] : m.wmax;
    fill_fin(m, k, in_dtype);
  }
  const bool sq = (mask & ST_STD) != 0;
  bool used = false;
  cudaError_t e;
  if (is_float) e = sq ? launch_tma_multi<double, true>(sat, sat_sq, m, st, used) : launch_tma_multi<double, false>(sat, sat_sq, m, st, used);
  else e = sq ? launch_tma_multi<uint64_t, true>(sat, sat_sq, m, st, used) : launch_tma_multi<uint64_t, false>(sat, sat_sq, m, st, used);
  if (e != cudaSuccess) return e;
  if (!used) return cudaErrorNotSupported;
  note_launch(1);
  return cudaSuccess;
}

}  // namespace ssb
