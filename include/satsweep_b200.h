/*
 * satsweep_b200.h -- C ABI of the B200-native integral-image / sliding-window
 * engine (libsatsweep_b200.so).
 *
 * The reference (`satsweep`, /root/reference/pkg) is a pure-Python package
 * with no native ABI; its hot path is reached through these Python call
 * sites, each of which one entry point below replaces:
 *
 *   ssb_sat_build        build_sat / build_sat_parallel
 *                        (pkg/src/satsweep/integral.py:109-116, parallel.py:106-121)
 *   ssb_sat_prepare +    the same, split so a row-band shard can exchange its
 *   ssb_sat_finish       column totals before writing
 *   ssb_window_eval      sweep_window_sums + finalize
 *                        (integral.py:141-163, :178-189; stats.py:35-74)
 *   ssb_window_eval_multi swa_multi_window (integral.py:199-210)
 *   ssb_sat_build_swa    build_sat + sweep_window_sums + finalize in one pass
 *                        (integral.py:166-189: the builder and sweep seams fused)
 *   ssb_window_fused     swa_integral / swa_parallel for stride 1 without a
 *                        materialised table (integral.py:192-196, parallel.py:137-149)
 *   ssb_window_sum_at    window_sum (integral.py:119-130)
 *   ssb_swa_host         api.swa with host buffers (api.py:28-55): host->device
 *                        copies, compute, device->host copies, streamed by bands
 *   ssb_file_to_device   the payload read of read_pgm / read_raw
 *                        (imgio.py:72-103, :160-174) straight into device memory
 *   ssb_device_to_file   the payload write of write_pgm / write_raw
 *                        (imgio.py:106-116, :127-139) straight from device memory
 *
 * Conventions
 *   - Device rasters must be 16-byte aligned (rows are staged with TMA bulk
 *     copies).  Tables that the library WRITES must be 32-byte aligned with
 *     a pitch that is a multiple of 4 elements (rows are stored with 256-bit
 *     stores; SSB_EINVAL otherwise); tables it only READS need 16-byte
 *     alignment and an even pitch for the TMA corner sweep.
 *   - Every device pointer is caller-allocated device memory.  The one
 *     allocation the library keeps is ssb_swa_host's band buffers, held in a
 *     library-private memory pool between calls (never the default pool or
 *     the caller's allocator) until ssb_host_release().
 *   - `stream` is a cudaStream_t (NULL = legacy default stream).  Device entry
 *     points are asynchronous on that stream.
 *   - Tables are (rows+1) x (cols+1) with a zero border row/column and row
 *     pitch `sat_ld` elements (see the alignment rule above).  Integer
 *     tables are uint64 modulo 2^64, float tables double.
 *   - Returns SSB_OK or an error code; ssb_last_error() gives a thread-local
 *     message.  No entry point falls back to a CPU implementation.
 */
#ifndef SATSWEEP_B200_H
#define SATSWEEP_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SSB_ABI_VERSION 1

/* status codes */
#define SSB_OK 0
#define SSB_EINVAL 1       /* bad argument (InvalidWindowError / ValueError side) */
#define SSB_ECUDA 2        /* CUDA runtime error */
#define SSB_ENOMEM 3       /* device or pinned allocation failed (ResourceLimitError) */
#define SSB_EUNSUPPORTED 4 /* valid request this build does not implement (TypeError side) */
#define SSB_ENONFINITE 5   /* F32 input holds NaN/Inf (GridValidationError, grid.py:82-83) */

/* element kinds (grid.py:17-46 ElemKind; I32 is an extension for BASELINE C2) */
#define SSB_U8 0
#define SSB_U16 1
#define SSB_I32 2
#define SSB_F32 3

/* statistic bits (grid.py:49-61 StatKind); several may be requested at once */
#define SSB_SUM 1
#define SSB_MEAN 2
#define SSB_STD 4

/* pipelines for ssb_swa_host */
#define SSB_PIPE_TABLE 0 /* build table(s) in HBM, then evaluate corners */
#define SSB_PIPE_FUSED 1 /* never materialise the table (stride 1 only) */

int ssb_abi_version(void);
const char* ssb_last_error(void);

/* Scratch bytes needed by ssb_sat_prepare/finish/build (carry vectors). */
int64_t ssb_sat_workspace_bytes(int in_dtype, int64_t rows, int64_t cols, int with_squares);

/* Tiling of the table build: info4 = {strip width (table cols), segment
 * height (table rows), number of strips, number of segments}.  Used for the
 * WriteCensus analogue (parallel.py:35-51). */
int ssb_sat_plan(int in_dtype, int64_t rows, int64_t cols, int with_squares, int64_t* info4);

/* Phase 1+2: reads the image once, fills the workspace.  If `band_totals`
 * (cols+1 entries, device) is non-NULL it receives the last table row of this
 * image *without* any carry -- the per-band column-total vector exchanged
 * between row-band shards.  `nonfinite_flag` (device int, nullable) is OR-ed
 * with 1 if an F32 pixel is NaN/Inf (grid.py:82-83). */
int ssb_sat_prepare(const void* in, int in_dtype, int64_t rows, int64_t cols, int64_t in_ld, int with_squares,
                    void* ws, int64_t ws_bytes, void* band_totals, void* band_totals_sq, int* nonfinite_flag,
                    void* stream);

/* Phase 3: writes the table(s); `sat` may be NULL when only the squared
 * table is wanted (build_sat(img, squared=True)).  `carry`/`carry_sq` (cols+1 entries, nullable)
 * are added to every table row: row 0 becomes `carry`, i.e. the global table
 * row above this band. */
int ssb_sat_finish(const void* in, int in_dtype, int64_t rows, int64_t cols, int64_t in_ld, void* sat,
                   void* sat_sq, int64_t sat_ld, const void* carry, const void* carry_sq, void* ws,
                   int64_t ws_bytes, void* stream);

/* prepare + finish. */
int ssb_sat_build(const void* in, int in_dtype, int64_t rows, int64_t cols, int64_t in_ld, void* sat, void* sat_sq,
                  int64_t sat_ld, const void* carry, const void* carry_sq, void* ws, int64_t ws_bytes,
                  int* nonfinite_flag, void* stream);

/* Window statistics from table(s) of a rows x cols image.  `sat_sq` is needed
 * iff SSB_STD is requested.  Output dtypes: sum = uint64 for U8/U16, int64 for
 * I32, double for F32; mean/std = double.  `out_ld` is the output row pitch
 * in elements.  Output dims: ((rows-w)/stride+1) x ((cols-w)/stride+1). */
int ssb_window_eval(const void* sat, const void* sat_sq, int in_dtype, int64_t rows, int64_t cols, int64_t sat_ld,
                    int64_t w, int64_t stride, int stat_mask, void* out_sum, double* out_mean, double* out_std,
                    int64_t out_ld, void* stream);

/* Same contract and bit-identical result as ssb_sat_build, computed by the
 * single-pass kernel: each pixel read once, each entry written once, carries
 * between tiles by decoupled look-back (north_star subsystem 1).  Integer
 * input only (u8, u16, i32 without squares; SSB_EUNSUPPORTED otherwise).
 * Slower than the default reduce-then-scan build at BASELINE C5 on B200
 * (DESIGN.md section 3), so ssb_sat_build does not route here unless the
 * environment variable SSB_SAT_PATH=one is set.  Its workspace (tile flags and
 * published aggregates) is sized by ssb_sat_lookback_workspace_bytes (-1 for
 * unsupported requests). */
int64_t ssb_sat_lookback_workspace_bytes(int in_dtype, int64_t rows, int64_t cols, int with_squares);
int ssb_sat_build_lookback(const void* in, int in_dtype, int64_t rows, int64_t cols, int64_t in_ld, void* sat,
                           void* sat_sq, int64_t sat_ld, const void* carry, const void* carry_sq, void* ws,
                           int64_t ws_bytes, void* stream);

/* Integral image AND its stride-1 window statistics (build_sat +
 * sweep_window_sums + finalize, integral.py:109-116, :141-189, fused at the
 * builder/sweep seams integral.py:166-189): writes the same table as
 * ssb_sat_build (no carry, no squares) and the same outputs as
 * ssb_window_eval on it, without reading the table back.  Integer input only;
 * stats SUM and/or MEAN; w <= 257 (u16: w <= 256).  ssb_sat_swa_supported
 * reports whether a request qualifies (1) or not (0); the workspace is
 * ssb_sat_swa_workspace_bytes.  ssb_sat_build_swa runs the faster pipeline
 * measured on B200: for uint8 (w <= 256) and uint16 (w <= 128) the table
 * build and, concurrently on a forked stream joined back into `stream`, the
 * windows from the raster by the fused kernel; otherwise the table build and
 * the corner sweep.  ssb_sat_build_swa_onepass runs the one-pass kernel,
 * whose table writer also emits the windows (same results; A/B, DESIGN.md
 * section 4). */
int ssb_sat_swa_supported(int in_dtype, int64_t w, int stat_mask);
int64_t ssb_sat_swa_workspace_bytes(int in_dtype, int64_t rows, int64_t cols);
/* Tiling of ssb_sat_build_swa: info4 = {warp strips, sweep segment height
 * (table rows), sweep segments, segment multiple of the build plan}. */
int ssb_sat_swa_plan(int in_dtype, int64_t rows, int64_t cols, int64_t w, int64_t* info4);
int ssb_sat_build_swa(const void* in, int in_dtype, int64_t rows, int64_t cols, int64_t in_ld, void* sat,
                      int64_t sat_ld, int64_t w, int stat_mask, void* out_sum, double* out_mean, int64_t out_ld,
                      void* ws, int64_t ws_bytes, void* stream);
int ssb_sat_build_swa_onepass(const void* in, int in_dtype, int64_t rows, int64_t cols, int64_t in_ld, void* sat,
                              int64_t sat_ld, int64_t w, int stat_mask, void* out_sum, double* out_mean,
                              int64_t out_ld, void* ws, int64_t ws_bytes, void* stream);

/* Several window sizes (stride 1) from one set of tables. */
int ssb_window_eval_multi(const void* sat, const void* sat_sq, int in_dtype, int64_t rows, int64_t cols,
                          int64_t sat_ld, int n_windows, const int64_t* windows, int stat_mask,
                          void* const* out_sums, double* const* out_means, double* const* out_stds,
                          const int64_t* out_lds, void* stream);

/* Stride-1 window statistics straight from the image.  `segments` = number of
 * row segments (0 = automatic). */
int ssb_window_fused(const void* in, int in_dtype, int64_t rows, int64_t cols, int64_t in_ld, int64_t w,
                     int stat_mask, void* out_sum, double* out_mean, double* out_std, int64_t out_ld,
                     int* nonfinite_flag, int segments, void* stream);

/* Largest window ssb_window_fused accepts. */
int64_t ssb_window_fused_max_w(void);

/* One four-corner lookup (window_sum); `out_value` is HOST memory receiving a
 * uint64 (integer table) or double (float table).  Synchronises `stream`. */
int ssb_window_sum_at(const void* sat, int is_float_table, int64_t rows, int64_t cols, int64_t sat_ld, int64_t top,
                      int64_t left, int64_t w, void* out_value, void* stream);

/* End-to-end with HOST buffers: input rows x cols at pitch in_ld (elements),
 * outputs at pitch out_ld.  Streams output-row bands through the device
 * (each band builds its own local table; offsets cancel) with
 * copies overlapped on their own streams.  Pinned host buffers give full PCIe
 * bandwidth; pageable ones work but are slower.  SUM results that provably
 * fit 32 bits cross PCIe as uint32 (see ssb_host_wire).  `band_rows` = output rows per
 * band (0 = automatic). */
int ssb_swa_host(const void* in_host, int in_dtype, int64_t rows, int64_t cols, int64_t in_ld, int64_t w,
                 int64_t stride, int stat_mask, void* out_sum_host, double* out_mean_host, double* out_std_host,
                 int64_t out_ld, int pipeline, int device, int64_t band_rows);

/* ---- row-band sharding over several GPUs ----------
 * Replaces the reference's worker fan-out of one process
 * (swa(method="parallel"), api.py:51-52 -> swa_parallel / build_sat_parallel /
 * parallel_sweep, parallel.py:80-149): device g owns a contiguous band of
 * image rows by the reference's partition rule over OUTPUT rows
 * (parallel.py:80-90).
 *
 * ssb_sharded_plan: plan7[7*g .. 7*g+6] = {own_lo, own_hi, need_lo, need_hi,
 * out_lo, out_hi, cap_rows}: image rows [own_lo, own_hi) are OWNED by device g
 * (a partition of [0, rows)); its output rows [out_lo, out_hi) need image rows
 * [need_lo, need_hi) (own rows + the (w-1)-row halo below); its band buffer
 * holds cap_rows rows starting at global row own_lo.  Pure host function. */
int ssb_sharded_plan(int64_t rows, int64_t cols, int64_t w, int ndev, int64_t* plan7);

/* Scratch for band `band` of ssb_sharded_swa (with_table: the global-table
 * workspace + the gathered column totals; 8 bytes when no table is built). */
int64_t ssb_sharded_workspace_bytes(int in_dtype, int64_t rows, int64_t cols, int64_t w, int ndev, int band,
                                    int with_table);

/* Window statistics (stride 1) and, with `sats`, the GLOBAL integral image
 * of a rows x cols image sharded over ndev devices of this process.  Per
 * device g (every array indexed by g; devs[g] may repeat a device):
 *   bands[g]   device buffer of cap_rows x cols on devs[g]; the caller fills the
 *              own rows (row 0 = global row own_lo) and the library writes the
 *              halo rows after them, copied from the following devices' own
 *              rows by peer copies (NVLink P2P) -- the halo exchange;
 *   sats[g]    (nullable array) (own_hi - own_lo + 1) x sat_ld table, 32-byte
 *              aligned, sat_ld a multiple of 4: global table rows
 *              [own_lo, own_hi] (row 0 is the carry row = the table row above
 *              the band).  Built from the band's column totals, gathered from
 *              the devices above by peer copies and summed in band order
 *              (the exclusive scan of per-band column-total vectors);
 *   out_*[g]   the band's output rows [out_lo, out_hi) at pitch out_ld;
 *   ws[g]      ssb_sharded_workspace_bytes(..., g, sats != NULL) bytes;
 *   streams[g] a stream on devs[g]; all work is asynchronous on it, and every
 *              stream is joined with every other before the call returns, so
 *              the caller may reuse any buffer in stream order.
 * stat_mask may be 0 (table only).  F32 finiteness is not checked here (use
 * ssb_f32_nonfinite on each band).  w <= ssb_window_fused_max_w(). */
int ssb_sharded_swa(int ndev, const int* devs, int in_dtype, int64_t rows, int64_t cols, int64_t w, int stat_mask,
                    void* const* bands, void* const* sats, int64_t sat_ld, void* const* out_sum,
                    double* const* out_mean, double* const* out_std, int64_t out_ld, void* const* ws,
                    const int64_t* ws_bytes, void* const* streams);

/* carry[c] = sum_{g < band} parts[g * parts_ld + c] for c < len (uint64
 * modulo 2^64, or double when is_float), summed in g order: the exclusive
 * scan over row bands of their column-total vectors, for multi-process
 * callers that gathered the totals themselves (e.g. an NCCL all-gather of
 * ssb_sat_prepare's band_totals); the result is ssb_sat_finish's carry. */
int ssb_band_carry(const void* parts, int band, int64_t len, int64_t parts_ld, int is_float, void* carry,
                   void* stream);

/* Self-test: adds to *mismatches (device counter) the number of x[i] (device,
 * n doubles) for which the finalisation's division by `divisor` (multiply by
 * RN(1/divisor) + one FMA correction) differs in any bit from the IEEE
 * division __ddiv_rn.  Asynchronous on `stream`. */
int ssb_selftest_division(const double* x, int64_t n, double divisor, unsigned long long* mismatches, void* stream);

/* Write census (the device side of the reference's WriteCensus,
 * parallel.py:35-51; tests/debug only).  While enabled on the calling thread,
 * every table entry (r, c) a table build stores adds 1 to table_rows[r] and
 * table_cols[c], and every output position a window kernel stores adds 1 to
 * out_rows[i] (with several windows in one call, window k's rows follow those
 * of windows 0..k-1).  Counters are caller-zeroed device uint64 arrays; NULL
 * disables a kind (table_rows and table_cols go together).  Exactly-once
 * coverage means table_rows[r] == cols+1, table_cols[c] == rows+1 and
 * out_rows[i] == output cols.  One atomic per store: slow, never on by
 * default.  ssb_swa_host (band-local rows) suspends it; ssb_sharded_swa
 * refuses it. */
int ssb_census_enable(unsigned long long* table_rows, int64_t n_table_rows, unsigned long long* table_cols,
                      int64_t n_table_cols, unsigned long long* out_rows, int64_t n_out_rows);
int ssb_census_disable(void);

/* Return the band buffers ssb_swa_host keeps reserved between calls (its
 * private pool on every device) to the device, and free its pinned staging
 * rings. */
int ssb_host_release(void);

/* Wire format of ssb_swa_host's SUM results (api.py:28-55 returns uint64 on
 * the host; the device->host copy of the results is the end-to-end critical
 * path).  0 (default): when every sum provably fits 32 bits (unsigned pixels,
 * w^2 * max pixel < 2^32) the device narrows the sums before the copy -- to
 * uint32, or to uint16 for a band whose largest sum (computed on the device)
 * is below 2^16 -- and the library's host threads zero-extend each landed
 * chunk into the caller's uint64 array: a half or a quarter of the PCIe
 * bytes, the same values; every other case copies 64-bit results straight
 * into the caller's array.  32: never narrower than uint32.  64: always the
 * straight copy.  Returns the previous setting; other values only query.
 * (At 0 and 32, 64-bit results bound for PAGEABLE host arrays also travel
 * through the library's pinned ring, copied by the same host threads.) */
int ssb_host_wire(int bits);

/* Device-resident uint64 sums (rows x cols, contiguous, DEVICE pointer, e.g.
 * the outputs of ssb_window_eval_multi / ssb_window_fused) into the caller's
 * HOST uint64 array at pitch out_ld, through the narrow wire described at
 * ssb_host_wire when max_sum -- an upper bound on every sum, e.g.
 * w * w * max pixel; 0 = unknown -- is below 2^32 (multi_window and the other
 * host-returning paths of api.py:58-67).  Any other contiguous 8-byte results
 * (max_sum = 0: float64 mean / std, wide sums) bound for a pageable array are
 * copied through the same ring as they are.  Waits for the work already
 * queued on `stream`; returns when host_out is complete. */
int ssb_sums_to_host(const void* dev_sums, int64_t rows, int64_t cols, uint64_t max_sum, void* host_out, int64_t out_ld,
                     void* stream);

/* The host half of the narrow wire on its own: dst_u64[i] = src[i] for i < n,
 * zero-extended from src_bits = 16 or 32 (HOST pointers, any element
 * alignment; AVX2 streaming stores where the CPU has them).  No device work. */
int ssb_host_widen(const void* src, int src_bits, void* dst_u64, int64_t n);

/* Host threads each ssb_swa_host call uses to widen narrow-wire results
 * (0 = automatic: the process's share of the cores minus two; n > 0 fixes it,
 * e.g. cores / devices when one process drives several GPUs at once).  Returns
 * the previous setting; negative values only query. */
int ssb_host_threads(int n);

/* Bytes the process's latest ssb_swa_host call copied host->device and
 * device->host (what crossed PCIe, after the wire format above). */
void ssb_host_last_copy_bytes(int64_t* h2d_bytes, int64_t* d2h_bytes);

/* Count of kernel launches the library issued since load (diagnostics). */
int64_t ssb_launch_count(void);

/* File front door.  Copy `nbytes` at byte `offset` of the
 * file at `path` into device memory `dst`, streamed through pinned staging
 * with parallel reads overlapped with the host->device copies.  swap16 != 0
 * byte-swaps 16-bit samples on the device afterwards (big-endian PGM); it
 * needs an even `nbytes` and a 16-byte aligned `dst`.  The file must hold at
 * least offset + nbytes bytes (SSB_EINVAL otherwise).  Synchronises `stream`.
 * Replaces the payload half of imgio.read_pgm / read_raw (imgio.py:93-103,
 * :169-174); header parsing and its error messages stay in the facade. */
int ssb_file_to_device(const char* path, int64_t offset, int64_t nbytes, void* dst, int swap16, void* stream);

/* Sets *flag (device int, caller-zeroed) to 1 if any of the n floats at `x`
 * is NaN or +-Inf: the finiteness rule of ImageGrid (grid.py:82-83) for rasters
 * that arrive on the device without a host copy.  Asynchronous on `stream`. */
int ssb_f32_nonfinite(const void* x, int64_t n, int* flag, void* stream);

/* Write `nbytes` of device memory `src` into the file at `path` starting at
 * byte `offset` (created if absent, sized to offset + nbytes; bytes before
 * `offset`, e.g. a PGM header, are kept).  swap16 != 0 writes 16-bit samples
 * big-endian (the source is not modified).  Synchronises `stream`.  Replaces
 * the payload half of imgio.write_pgm / write_raw (imgio.py:106-116, :127-139). */
int ssb_device_to_file(const char* path, int64_t offset, const void* src, int64_t nbytes, int swap16, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* SATSWEEP_B200_H */
