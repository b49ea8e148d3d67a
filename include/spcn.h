/*
 * spcn.h — C ABI of libspcn.so, the B200 (sm_100a) hot path of
 * structure-preserving color normalization (SPCN).
 *
 * Every entry point replaces one function of the reference package
 * `slidenorm` (/root/reference/pkg/src/slidenorm, cited as src/<file>:<line>).
 * The ABI is plain C: device pointers + sizes, a cudaStream_t passed as
 * `void*`, no C++ or torch types.  Calls are stream-ordered and do not
 * synchronize the host unless stated; they are reentrant across host threads
 * and streams (no global mutable state except a thread-local error string).
 *
 * Return codes map 1:1 onto the reference exception taxonomy
 * (src/errors.py:1-36; ValueError for argument checks).
 */
#ifndef SPCN_H_
#define SPCN_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes ------------------------------------------------------ */
#define SPCN_OK 0
#define SPCN_EINVAL 1            /* ValueError (argument / invariant check)   */
#define SPCN_EBLANK 2            /* BlankSlideError        src/errors.py:24   */
#define SPCN_EINSUFFICIENT 3     /* InsufficientPixelsError src/errors.py:28  */
#define SPCN_ESTAIN_ABSENT 4     /* StainAbsentError       src/errors.py:32   */
#define SPCN_EDEGENERATE 5       /* DegenerateStainError   src/errors.py:36   */
#define SPCN_ECUDA 6             /* CUDA runtime error                          */
#define SPCN_ENCCL 7             /* collective error (multi-GPU stats)          */

/* ---- precision of the per-pixel transform ------------------------------ */
#define SPCN_PREC_EXACT 0   /* fp32 fast path + certified rounding; pixels whose
                               rounding is not certified are recomputed in fp64
                               in the reference's operation order: output is
                               byte-identical to src/pipeline.py:260-272      */
#define SPCN_PREC_FAST 1    /* fp32 only (±1 LSB vs the reference)            */
#define SPCN_PREC_STRICT 2  /* fp64 for every pixel, reference operation order */

/* Parameters of one source→target recoloring (src/pipeline.py:260
 * `_process_strip(pixels, src_i0, src_basis, code_lam, factors, tgt_basis,
 * tgt_i0)`).  Bases are row-major 3x2 (basis[c*2+j], channel c, stain j). */
/* spcn_xform_params.cert_alpha: 0 = analytic per-pixel bound; (0, 1e-3) =
 * a calibrated bound from spcn_xform_calibrate; SPCN_CALIBRATE_INLINE =
 * calibrate on the device inside spcn_xform_rgb8 (no host round trip).     */
#define SPCN_CALIBRATE_INLINE (-1.0)
/* SPCN_CALIBRATE_DEVICE: the bound is already in the workspace's calibration
 * word — multi-GPU: every rank runs spcn_xform_calibrate_part on its share
 * of the colours, then the words are all-reduced with max (uint32: the bits
 * of a non-negative float order like the float).                           */
#define SPCN_CALIBRATE_DEVICE (-2.0)

typedef struct spcn_xform_params {
  double src_i0[3];
  double src_basis[6];
  double code_lam;          /* >= 0; reference default 0.0 (src/pipeline.py:277) */
  double factors[2];        /* tgt_p99 / src_p99 (src/normalize.py:103-112)      */
  double tgt_basis[6];
  double tgt_i0[3];
  const double* od_table;   /* optional host pointer to the (3,256) fp64 OD table
                               ln(i0_c/clip(i,1,i0_c)) for i=0..255 computed by the
                               caller with the reference's own expression
                               (src/optics.py:89-94); NULL = computed with libm  */
  int32_t precision;        /* SPCN_PREC_*                                       */
  int32_t max_sweeps;       /* CD sweep cap, reference 2000 (src/stain_sep.py:168) */
  double cert_alpha;        /* EXACT only: relative certification bound from
                               spcn_xform_calibrate (> 0), or <= 0 for the
                               analytic per-pixel bound                          */
} spcn_xform_params;

/* Exhaustive calibration of the EXACT certification bound for one parameter
 * set: runs the fp32 path and the fp64 reference-order path on all 2^24 RGB
 * colours and returns alpha = 1.5 * max relative error + 2^-22 (or -1 when
 * the fast path is not applicable).  Valid by exhaustion for every input.
 * Synchronizes `stream`; ~0.5 ms on a B200.  workspace >= 16 bytes.        */
int spcn_xform_calibrate(const spcn_xform_params* p, void* workspace,
                         size_t workspace_bytes, double* alpha_out, void* stream);

/* Device workspace (bytes) needed by spcn_xform_rgb8 for `npix` pixels.     */
size_t spcn_xform_workspace_bytes(int64_t npix);

/* Recolor `npix` packed RGB8 pixels: src → dst (both device pointers, may be
 * the same buffer).  Replaces `_process_strip` src/pipeline.py:260-272
 * (= beer_lambert src/optics.py:71 + code_densities src/stain_sep.py:168 +
 * normalize_block src/normalize.py:115).  Host-side checks mirror
 * validate_basis (src/stain_sep.py:89-101), the normalize_block factor check
 * (src/normalize.py:141-142) and beer_lambert's i0 check (src/optics.py:90). */
int spcn_xform_rgb8(const uint8_t* src, uint8_t* dst, int64_t npix,
                    const spcn_xform_params* p, void* workspace,
                    size_t workspace_bytes, void* stream);

/* Number of pixels the last EXACT-mode call on `workspace` sent to the fp64
 * repair path (synchronizes `stream`; diagnostics only).                    */
int spcn_xform_repair_count(const void* workspace, void* stream, int64_t* count);

/* Per-pixel density coding: od (3,n) fp64 device, h (2,n) fp64 device.
 * Replaces code_densities src/stain_sep.py:168-201 (bit-identical: same
 * operation order, same bitwise CD fixed point, same sweep cap).            */
int spcn_code_densities(const double* od, double* h, int64_t n,
                        const double* basis, double lam, int32_t max_sweeps,
                        void* stream);

/* Recombination + inverse Beer-Lambert: h (2,n) fp64 device → out (n,3) u8.
 * Replaces normalize_block src/normalize.py:115-151.                        */
int spcn_normalize_block(const double* h, uint8_t* out, int64_t n,
                         const double* factors, const double* tgt_basis,
                         const double* tgt_i0, void* stream);

/* Beer-Lambert OD of packed RGB8 pixels: px (n,3) u8 → od (3,n) fp64
 * (channel-major, the layout code_densities consumes).  Replaces
 * beer_lambert src/optics.py:71-94 via the same 256-entry table.           */
int spcn_beer_lambert(const uint8_t* px, double* od, int64_t n,
                      const double* i0, const double* od_table, void* stream);

/* Inverse Beer-Lambert: od (n,3) fp64 device → out (n,3) u8,
 * floor(i0_c*exp(-v)+0.5) clipped to [0,255].  Replaces inverse_beer_lambert
 * src/optics.py:97-110.                                                     */
int spcn_inverse_beer_lambert(const double* od, uint8_t* out, int64_t n,
                              const double* i0, void* stream);

/* ---- fit: pixel sampling (src/pipeline.py:128-200) -------------------- */
#define SPCN_SAMPLE_CHUNK 4096   /* raster-order pixels per counting chunk  */

/* A rectangular region of an RGB8 image in device memory: pixel (row, col)
 * of the patch is at byte 3*(base + row*row_stride + col) of `img`.        */
typedef struct spcn_patch {
  int64_t base;        /* pixel offset of the top-left pixel                 */
  int32_t width, height;
  int64_t row_stride;  /* pixels between consecutive rows                    */
} spcn_patch;

/* What the visit loop decided to take from one visited patch.               */
typedef struct spcn_patch_take {
  int64_t take_nonwhite;   /* first N non-white pixels in raster order        */
  int64_t out_base;        /* where they go in the output sample (pixels)     */
  int32_t take_bright[3];  /* first N values > thr per channel (bright pools) */
  int32_t problem;         /* which fit problem's bright histogram to feed     */
} spcn_patch_take;

/* Per-chunk counts for `npatches` patches (device array of spcn_patch):
 * counts[(p*max_chunks + k)*4 + {0,1,2,3}] = #non-white, #R>thr, #G>thr,
 * #B>thr among raster pixels [k*CHUNK, (k+1)*CHUNK) of patch p.  Non-white
 * means "not all channels > thr" (src/pipeline.py:176).                     */
int spcn_sample_count(const uint8_t* img, const spcn_patch* patches, int32_t npatches,
                      int32_t max_chunks, int32_t white_threshold, int32_t* counts,
                      void* stream);

/* One-patch items (every item's candidate grid is one patch, e.g. a batch of
 * 512^2 tiles with patch_size 1000): the visit rules of src/pipeline.py:
 * 156-184 per item from the chunk counts of spcn_sample_count — non-white
 * take = min(total, target) if total >= used_min (the background cutoff
 * times the patch area) else 0, bright takes = min(total, cap) — and the
 * sample offsets as an exclusive scan of the takes: the take rows
 * spcn_sample_compact reads, and take_nw[i] (device) for the read-back.   */
int spcn_visit_single(const int32_t* counts, int32_t n, int32_t chunks, double used_min,
                      int64_t target, int64_t cap, spcn_patch_take* takes, int64_t* take_nw,
                      void* stream);

/* Ordered compaction of the decided takes: the first take_nonwhite non-white
 * pixels of each patch (raster order) → out_px[out_base ...] (RGB8), and the
 * first take_bright[c] values > thr of channel c → bright_hist[problem][c][v]
 * (+=, caller zeroes).  Reproduces the raster-order prefixes of
 * src/pipeline.py:167-181 exactly.                                          */
int spcn_sample_compact(const uint8_t* img, const spcn_patch* patches, int32_t npatches,
                        int32_t max_chunks, int32_t white_threshold, const int32_t* counts,
                        const spcn_patch_take* takes, uint8_t* out_px, int32_t* bright_hist,
                        void* stream);

/* The reference's patch visit loop (src/pipeline.py:156-184) on the device,
 * for candidates [k0, k0 + n) of the visit order (one thread, sequential like
 * the reference), continuing `state` across calls:
 *   state (int64[8], zero before the first call): collected, visited, used,
 *   bright_n[3], stopped, need_more (set when the batch ran out before a stop
 *   rule fired and more candidates exist: call again with the next batch).
 * counts: spcn_sample_count output for the n candidates; dims[k] = {w, h} of
 * candidate k0+k; takes[k] receives its decision (take 0 when not visited);
 * offsets[1] = collected (the sample's end offset).                        */
typedef struct spcn_visit_plan {
  int64_t target_pixels, sample_cap;
  int32_t max_patches, ncand;   /* ncand = candidates in the visit order (<= 10*max_patches) */
  double background_cutoff;     /* SamplePlan.background_fraction_cutoff */
} spcn_visit_plan;
int spcn_sample_visit(const int32_t* counts, int32_t n, int32_t max_chunks, int32_t k0,
                      const int32_t* dims, const spcn_visit_plan* plan, int64_t* state,
                      spcn_patch_take* takes, int64_t* offsets, void* stream);

/* Background i0 per problem and channel: exact 80th percentile of the bright
 * pool given as 256-bin counts (estimate_max_intensity src/optics.py:35-68).
 * Empty pools give 255 and empty[p*3+c] = 1 (the reference's warning case). */
int spcn_i0_from_hist(const int32_t* hist, int32_t nprob, double* i0, int32_t* empty,
                      void* stream);

/* Per-problem OD tables lut[p][c][i] = ln(i0[p][c] / clip(i,1,i0[p][c])).   */
int spcn_od_tables(const double* i0, int32_t nprob, double* lut, void* stream);

/* ---- fit: sparse-NMF basis, density coding, p99 ------------------------ */
typedef struct spcn_snmf_cfg {
  double lam;            /* SnmfConfig.lam (src/stain_sep.py:50), 0.1 default  */
  double rel_tol;        /* SnmfConfig.rel_tol, 1e-6                          */
  double w_init[6];      /* initial basis (row-major 3x2): reference_basis() +
                            default_rng(seed).uniform(0, 0.05), clamped and
                            column-normalised (src/stain_sep.py:271-274)      */
  int32_t max_outer;     /* SnmfConfig.max_outer_iters, 200                   */
  int32_t cluster;       /* CTAs per problem (1 = batched, 8 = single slide)  */
} spcn_snmf_cfg;

/* Batched fit_basis (src/stain_sep.py:239-336).  Problem p's sample is the
 * RGB8 pixels [offsets[p], offsets[p+1]) of `samples`, coded to OD through
 * luts[p] (3x256 fp64) (or, when `od` is non-NULL, the fp64 OD columns
 * od[c*total + i], c = 0..2, in which case `samples`/`luts` are ignored).
 * Writes the ordered basis (nprob x 6, row-major), the objective history
 * (nprob x (max_outer+1)) and info (nprob x 4: iterations, converged, warning
 * flags bit0=no-convergence bit1=one-stain, history length).  hscratch
 * (optional, >= total + nprob/2 + 1 fp64 words) holds a per-problem table of
 * distinct sample colours with pixel counts, so each SNMF pass visits every
 * colour once with its weight, and the work-queue ticket; NULL = one visit
 * per sample.  Device pointers.                                            */
int spcn_snmf_batched(const uint8_t* samples, const double* od, const int64_t* offsets,
                      int32_t nprob,
                      const double* luts, const spcn_snmf_cfg* cfg, double* hscratch,
                      int64_t total, double* basis_out, double* history_out,
                      int32_t* info_out, void* stream);

/* Batched code_densities of the fit samples (src/pipeline.py:226): h[j*total
 * + i] for the pixels of every problem with its own table and basis.        */
int spcn_code_samples(const uint8_t* samples, const int64_t* offsets, int32_t nprob,
                      int64_t max_m, const double* luts, const double* bases, double lam,
                      int32_t max_sweeps, double* h, int64_t total, void* stream);

/* Per-segment, per-stain percentile p of densities h (2 x total, fp64):
 * stain_stats src/normalize.py:83-100 with percentile src/order_stats.py:11-36
 * computed by exact radix select.  out[s*2+j]; absent[s*2+j] = 1 when the
 * segment is empty or its max is <= 0 (StainAbsentError).  Scratch: qbuf of
 * 6*nseg*32 bytes, selbuf of 6*nseg doubles (device).                      */
int spcn_percentile_segments(const double* h, int64_t total, const int64_t* seg_offsets,
                             int32_t nseg, double p, void* qbuf, double* selbuf, double* out,
                             int32_t* absent, void* stream);

/* The same two steps over the colour table spcn_snmf_batched left in
 * hscratch (problem p: ucount[p] (rgb, pixel count) entries at offsets[p]):
 * spcn_code_table codes each distinct colour once (h at the entry's index);
 * spcn_percentile_table gives the per-problem percentile of the expanded
 * multiset (weighted exact radix select) — identical to spcn_code_samples +
 * spcn_percentile_segments on the samples.                                 */
int spcn_code_table(const void* hscratch, const int64_t* offsets, int32_t nprob, int64_t max_m,
                    const double* luts, const double* bases, double lam, int32_t max_sweeps,
                    double* h, int64_t total, void* stream);
int spcn_percentile_table(const double* h, int64_t total, const void* hscratch,
                          const int64_t* seg_offsets, int32_t nseg, double p, double* out,
                          int32_t* absent, void* stream);

/* Generic exact k-th smallest (0-based) of values[begin, end) for nq queries
 * given as device arrays; out[q] (device).                                  */
int spcn_select_kth(const double* values, const int64_t* begin, const int64_t* end,
                    const int64_t* k, int32_t nq, void* qbuf, double* out, void* stream);

/* ---- batched recolouring (many items, own source params, one target) --- */
/* One batch = N independent `_normalize_one` (src/cli.py:220-244) transforms:
 * item i's pixels are [off[i], off[i+1]) of the concatenated src/dst.       */
typedef struct spcn_batch_target {
  double i0[3];
  double basis[6];          /* row-major 3x2 */
  double p99[2];
} spcn_batch_target;

/* Byte sizes of the opaque per-item blocks spcn_batch_params writes.        */
int spcn_batch_sizes(size_t* fast_scalar_bytes, size_t* strict_param_bytes);

/* Build per-item parameter blocks ON THE DEVICE from batched fit results
 * (i0 nx3, luts nx3x256 fp64, bases nx6, p99 nx2; all device): factors
 * tgt_p99/src_p99 with the reference's degeneracy checks
 * (src/normalize.py:103-112, src/pipeline.py:291-297).  status (device, in:
 * 0 = fit ok / <0 = fit error code; out: 0 = fast path, 1 = strict path
 * only, -SPCN_EDEGENERATE = degenerate stain).                              */
int spcn_batch_params(int32_t nitems, const double* i0, const double* luts, const double* bases,
                      const double* p99, const spcn_batch_target* tgt, double code_lam,
                      int32_t max_sweeps, int32_t precision, void* fast_scalars, float* flut,
                      void* strict_params, int32_t* status, void* stream);

/* Recolour every item (status 0 via the fast kernel, status 1 via the fp64
 * kernel, errors skipped).  off_host/off_dev: n+1 pixel offsets (multiples of
 * 16); fast_scalars/flut/strict_params: the device blocks spcn_batch_params
 * wrote; status_host: host copy of its status output.  EXACT needs a
 * workspace of spcn_xform_workspace_bytes(total pixels).                     */
int spcn_xform_batch(const uint8_t* src, uint8_t* dst, int32_t nitems, const int64_t* off_host,
                     const int64_t* off_dev, const void* fast_scalars,
                     const int32_t* status_host, const int32_t* status_dev, const float* flut,
                     const void* strict_params, int32_t precision, void* workspace,
                     size_t workspace_bytes, void* stream);

/* ---- whole-slide ("global") percentile mode --
 * Extension of stain_stats (src/normalize.py:58-100): the p99 of the
 * densities of EVERY non-white pixel (not all channels > white_threshold,
 * src/pipeline.py:176), coded like code_densities (src/stain_sep.py:168-201)
 * with p->src_i0 / src_basis / code_lam / max_sweeps (target fields unused).
 * spcn_stats_hist: fp32 densities binned into hist[j*nbins + bin], bin =
 * (float_bits(h_j) - base[j]) >> shift[j], shift <= 23 (keys below base are
 * counted in counts[1+j]; counts[0] += non-white pixels; h = 0 counts into
 * bin 0 when base[j] == 0).  Approximate: it only places the refine window.
 * spcn_stats_refine: exact classification against [lo[j], hi[j]): densities
 * that may lie in the window are recomputed in fp64 in the reference's order
 * (once per colour per CTA); counts[j] += exact count below lo[j],
 * counts[2+j] += pixels in the window, listed as counts[5+j] (value, pixel
 * count) pairs cand[j*cap + i] / cand_count[j*cap + i] (the first `cap`),
 * counts[4] += fp64 evaluations.  All buffers device; hist/counts accumulate
 * (caller zeroes; counts has 7 entries); src 16-byte aligned.  Multi-GPU: sum
 * hist/counts across ranks, gather the (value, count) lists.                */
int spcn_stats_hist(const uint8_t* src, int64_t npix, const spcn_xform_params* p,
                    int32_t white_threshold, const uint32_t* base, const uint32_t* shift,
                    int32_t nbins, unsigned long long* hist, unsigned long long* counts,
                    void* stream);
int spcn_stats_refine(const uint8_t* src, int64_t npix, const spcn_xform_params* p,
                      int32_t white_threshold, const double* lo, const double* hi,
                      unsigned long long* counts, double* cand, unsigned long long* cand_count,
                      unsigned long long cap, void* stream);
/* One-pass exact mode.  spcn_stats_table: every non-white pixel whose
 * density is not surely below lo[j] (fp32 bound, as in the refine) for some
 * stain j is counted in table[rgb] (2^24 u64 counters, r | g<<8 | b<<16;
 * accumulates; caller zeroes); counts[0] += non-white pixels.  Pixels off the
 * table have exact densities < lo[j] in both stains.  Multi-GPU: sum the
 * tables and counts across ranks.
 * spcn_stats_table_scan: for every colour with table[rgb] > 0, the exact
 * fp64 densities in the reference's order (x[2i], x[2i+1]) and its count w[i]
 * (the first `cap`, in no particular order); n_out[0] += present colours,
 * n_out[1] += their pixels, n_out[2 + j] = max(n_out[2 + j], bits of the
 * largest x_j) (4 entries, caller zeroes).  The p-th percentile follows from
 * a weighted select over the entries with x >= lo (see global_stats.py).
 * spcn_stats_cube_classes + spcn_stats_table_cube: the same table pass with a
 * class table in front, built from the same params/white/lo into `classes`
 * (SPCN_CUBE_CLASS_BYTES: 32 KiB of cell classes, one byte per 8x8x8 RGB
 * cell, then the 2 MiB bitmap of candidate colours): most pixels are decided
 * by one shared-memory byte.  Same table/counts contract as spcn_stats_table. */
#define SPCN_CUBE_CLASS_BYTES ((32u << 10) + (2u << 20))
int spcn_stats_cube_classes(const spcn_xform_params* p, int32_t white_threshold,
                            const double* lo, uint8_t* classes, void* stream);
int spcn_stats_table_cube(const uint8_t* src, int64_t npix, const spcn_xform_params* p,
                          int32_t white_threshold, const double* lo, const uint8_t* classes,
                          unsigned long long* table, unsigned long long* counts, void* stream);
/* Exact selection over table entries without sorting them: hist[j*nbins + b]
 * += w[i] for the entries with x[2i+j] >= lo[j] in bin b = min(nbins-1,
 * floor((x - lo[j]) * scale[j])) (caller zeroes; sum across ranks), then
 * spcn_table_entries_collect lists the entries of bins [bins[2j], bins[2j+1]]
 * of stain j as (vals[j*cap + k], wts[j*cap + k]), nsel[j] += their number
 * (entries past cap are counted, not stored).                             */
int spcn_table_entries_hist(const double* x, const unsigned long long* w, int64_t m,
                            const double* lo, const double* scale, int32_t nbins,
                            unsigned long long* hist, void* stream);
int spcn_table_entries_collect(const double* x, const unsigned long long* w, int64_t m,
                               const double* lo, const double* scale, int32_t nbins,
                               const int32_t* bins, double* vals, unsigned long long* wts,
                               unsigned long long cap, unsigned long long* nsel, void* stream);
int spcn_stats_table(const uint8_t* src, int64_t npix, const spcn_xform_params* p,
                     int32_t white_threshold, const double* lo, unsigned long long* table,
                     unsigned long long* counts, void* stream);
int spcn_stats_table_scan(const spcn_xform_params* p, const unsigned long long* table,
                          double* x, unsigned long long* w, unsigned long long cap,
                          unsigned long long* n_out, void* stream);

/* ---- measurement input: synthetic H&E slides --------------------------- */
typedef struct spcn_synth_params {
  float i0[3];             /* background intensity per channel              */
  float basis[6];          /* mixing basis, row-major 3x2 (reference H&E)   */
  float tissue_fraction;
  int32_t layout;          /* 0 = scatter, 1 = block (src/synthetic.py:75-89) */
  int32_t dense;           /* 0 = sparse_densities, 1 = dense_densities     */
} spcn_synth_params;

/* Render rows [row0, row0+rows) of a width x height synthetic slide into
 * `out` (packed RGB8, 16-byte aligned).  Model of src/synthetic.py:26-121
 * with a counter-based RNG (pixel content depends only on seed and the
 * pixel's absolute position).  Not part of the reference's API: it is the
 * input generator for 400-Mpx..10-Gpx measurements.                        */
int spcn_render_synthetic(uint8_t* out, int64_t width, int64_t row0, int64_t rows,
                          int64_t height, uint64_t seed, const spcn_synth_params* p,
                          void* stream);

/* Copy `bytes` of device memory into pinned host memory with a small kernel
 * (stores through the host mapping) rather than a copy engine, stream-ordered;
 * for small read-backs that must not wait behind large transfers queued on
 * the copy engine by other streams.  Falls back to cudaMemcpyAsync when the
 * buffer is not mapped or not 4-byte aligned.                               */
int spcn_readback(const void* src, void* host_pinned, int64_t bytes, void* stream);

/* Wait for `stream` (after a spcn_readback, before reading the pinned bytes). */
int spcn_stream_sync(void* stream);

/* ---- one-slide fit in two stream-ordered steps (launch-bound path) ------
 * The fit of one resident slide is ~0.2 ms of kernels; these two entry
 * points issue each of its device phases with one call (the same kernels as
 * the individual entries above) so the host pays one call per phase.
 * Arena A (SPCN_FIT_ARENA_A bytes, device): state i64[8] @0 (collected,
 * visited, used, bright counts x3, stopped, need-more-candidates), offsets
 * i64[2] @64, i0 f64[3] @80, empty-pool flags i32[3] @104, bright histogram
 * i32[3][256] @128.  Arena B (SPCN_FIT_ARENA_B bytes): ordered basis f64[6]
 * @0, p99 f64[2] @48, SNMF info i32[4] @64, stain-absent flags i32[2] @80.
 *
 * spcn_fit_sample_step: one candidate batch of the visit loop (zeroing the
 * arena first when zero_arena != 0): sample_count -> sample_visit ->
 * sample_compact -> i0_from_hist, then the first readback_bytes of arena A
 * into pinned host memory (caller syncs the stream before reading).
 * spcn_fit_basis_step: the host OD table (pinned, 3x256 f64, the reference's
 * own np.log values) -> device, SNMF basis, densities (code_lam), the pooled
 * p99 when want_p99 != 0, then the first readback_bytes of arena B into
 * pinned memory.  The pinned table must stay untouched until the stream has
 * passed this call.                                                        */
#define SPCN_FIT_ARENA_A 3200
#define SPCN_FIT_ARENA_B 88
int spcn_fit_sample_step(const uint8_t* img, const spcn_patch* patches, int32_t n,
                         int32_t max_chunks, int32_t k0, const int32_t* dims,
                         const spcn_visit_plan* plan, int32_t white_threshold, int32_t zero_arena,
                         void* arena_a, int32_t* counts, spcn_patch_take* takes,
                         uint8_t* sample_out, void* readback_pinned, int64_t readback_bytes,
                         void* stream);
int spcn_fit_basis_step(const uint8_t* sample, int64_t m, const int64_t* offsets,
                        const double* lut_pinned, double* lut_dev, const spcn_snmf_cfg* cfg,
                        double* hscratch, double* history, void* arena_b, double code_lam,
                        int32_t max_sweeps, double* h, void* qbuf, double* selbuf,
                        int32_t want_p99, void* readback_pinned, int64_t readback_bytes,
                        void* stream);

/* Exhaustive calibration of part `part` of `nparts` of the 2^24 colours into
 * the workspace's calibration word (zeroed first; stream-ordered).  With
 * every part's word max-reduced, cert_alpha = SPCN_CALIBRATE_DEVICE makes the
 * transform use it — the same bound as one full calibration.               */
int spcn_xform_calibrate_part(const spcn_xform_params* p, int32_t part, int32_t nparts,
                              void* workspace, int64_t workspace_bytes, void* stream);

/* Fit -> transform with no host round trip (the device-built recolouring).
 * The source half of the recolouring is read on the device from a fit that
 * is still in flight on `stream`: the OD table spcn_fit_basis_step uploaded
 * (lut_dev) and its arena B (basis | p99 | info | absent).  One call builds
 * the parameters (1 CTA, the same params.cuh code as spcn_xform_rgb8), runs
 * the exhaustive calibration, the EXACT recolour and the fp64 repairs —
 * byte-identical to spcn_xform_rgb8 with the host-built parameters and
 * SPCN_CALIBRATE_INLINE.  Replaces the host half of src/pipeline.py:275-296
 * (scale_factors + the per-strip constants) for a resident slide.
 * status_pinned (optional, pinned host int32) receives the build status, and
 * the call then returns once it has landed — with everything enqueued on the
 * stream before the call (e.g. the fit's arena read-back) also in host
 * memory, while the recolour itself is still running (stream-ordered, like
 * spcn_xform_rgb8).  Status 0 = recolouring; otherwise (stain absent,
 * degenerate p99, an invalid or ill-conditioned basis: the strict-only case)
 * dst is left untouched and the caller runs spcn_xform_rgb8 with host
 * parameters, which raises the reference's error or takes the strict path.
 * src and dst must share their 16-byte alignment phase; workspace as for
 * spcn_xform_rgb8 (spcn_xform_workspace_bytes(npix)).                       */
typedef struct spcn_xform_fitted {
  const double* src_od_table;   /* device: 3 x 256 f64 source OD table         */
  const void* src_fit;          /* device: SPCN_FIT_ARENA_B bytes (arena B)    */
  double tgt_basis[6];
  double tgt_p99[2];            /* > 0 (scale_factors' numerators)             */
  double tgt_i0[3];
  double code_lam;
  int32_t max_sweeps;
  int32_t flags;                /* SPCN_FITTED_* (0: calibrated bound)          */
  /* optional: a target fitted on the device in the same stream — its arena B
   * (basis | p99 | info | absent) and its i0 (3 f64); tgt_basis / tgt_p99 /
   * tgt_i0 above are then ignored and the target's checks (absent stain, p99
   * > 0, valid basis) join the device-side decline conditions              */
  const void* tgt_fit;
  const double* tgt_i0_dev;
} spcn_xform_fitted;
/* flags: the analytic per-pixel certification bound instead of the
 * exhaustive calibration (images below ~2^24 px, where the 0.3 ms
 * calibration does not pay) — the same bytes either way.                    */
#define SPCN_FITTED_ANALYTIC 1
int spcn_xform_rgb8_fitted(const uint8_t* src, uint8_t* dst, int64_t npix,
                           const spcn_xform_fitted* p, void* workspace, size_t workspace_bytes,
                           int32_t* status_pinned, void* stream);

/* The same recolouring in two calls, for a row-band group: prepare builds
 * the parameters into a slot (*slot_out) and runs part `part` of `nparts` of
 * the exhaustive calibration into the workspace's calibration word (with
 * status_pinned it returns once the status is in host memory); the caller
 * max-reduces that word across the ranks (one int32 all-reduce,
 * stream-ordered) and then calls run, which recolours with the reduced bound
 * and releases the slot.  Every prepare must be followed by a run on the
 * same stream (npix 0 only releases the slot; a run that fails its argument
 * checks releases it too).  There are SPCN_FITTED_SLOTS slots per device: a
 * prepare while every slot is prepared-but-not-run (other threads) blocks
 * until one of them runs.                                                   */
#define SPCN_FITTED_SLOTS 2
int spcn_xform_fitted_prepare(const spcn_xform_fitted* p, int32_t part, int32_t nparts,
                              void* workspace, size_t workspace_bytes, int32_t* status_pinned,
                              int32_t* slot_out, void* stream);
int spcn_xform_fitted_run(const uint8_t* src, uint8_t* dst, int64_t npix, int32_t slot,
                          void* workspace, size_t workspace_bytes, void* stream);

/* Thread-local description of the last error ("" if none).                 */
const char* spcn_last_error(void);

/* Library version string.                                                   */
const char* spcn_version(void);

/* Number of kernels libspcn has launched in this process (diagnostics).     */
uint64_t spcn_launch_count(void);

/* Launch shape of the recolor kernel on the current device (diagnostics).   */
const char* spcn_xform_shape(void);

/* Per-launch timing of the main recolor kernel (measurement): while enabled,
 * spcn_xform_rgb8 records a CUDA event pair on its stream around each
 * k_xform_warp launch.  spcn_xform_timing synchronizes on the recorded events
 * and returns the number of timed launches and their summed duration (ms),
 * then clears the record.                                                  */
int spcn_xform_timing_enable(int32_t on);
int spcn_xform_timing(int64_t* launches, double* total_ms);

#ifdef __cplusplus
}
#endif
#endif /* SPCN_H_ */
