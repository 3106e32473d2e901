/*
 * mwb.h — C ABI of the B200 (sm_100a) confocal DAS/DMAS imaging path.
 *
 * This is the drop-in boundary below the reference's Python imaging entry
 * points (package `mwbeam`, /root/reference/pkg/src/mwbeam).  Every entry
 * point takes plain device pointers, sizes and a cudaStream_t passed as
 * `void*`; nothing here allocates on the hot path and no torch type appears
 * in a signature.  All functions return 0 on success and a negative code on
 * error; `mwb_last_error()` returns a thread-local message for the last
 * failure on the calling thread.
 *
 * Replaced reference interfaces (file:line relative to /root/reference):
 *   mwb_delay_table        <- pkg/src/mwbeam/beamform.py:182-190  delays / i0 / frac
 *   mwb_energies           <- pkg/src/mwbeam/beamform.py:169-212  _multistatic_energies
 *                             (also das_energy / dmas_energy, beamform.py:242-253,
 *                              and the 64-point batching of image(), beamform.py:325-336)
 *   mwb_enumerate_lattice  <- pkg/src/mwbeam/beamform.py:268-280  _region_cells
 *                             + the skip filter of image(), beamform.py:309-315
 *                             + cell centres, beamform.py:321-323
 *   mwb_select_roi         <- pkg/src/mwbeam/coarse2fine.py:169-256 select_roi
 *   mwb_enumerate_volume, mwb_select_roi_volume: the same for 3-D voxel grids
 *                             (BASELINE configs[4]; no reference counterpart)
 *   mwb_argmax_dense       <- pkg/src/mwbeam/beamform.py:101-104  EnergyMap.argmax_cell
 *   mwb_simulate           <- pkg/src/mwbeam/simulate.py:111-162 simulate (input producer)
 *   mwb_compact_payload    <- pkg/src/mwbeam/io.py:65-86 load_dataset (device staging of the
 *                             .mwb series in the layout the energy entry points take)
 *   mwb_render_pgm         <- pkg/src/mwbeam/io.py:122-137 export_energy_map's raster
 *                             over EnergyMap.dense, beamform.py:116-128
 *                             (also fused into mwb_energies through `argmax_key`)
 */
#ifndef MWB_H
#define MWB_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* beamformer kind (reference BeamformerKind, beamform.py:41-50) */
#define MWB_DAS 0
#define MWB_DMAS 1

/* interpolation (reference _check_interpolation, beamform.py:131-133) */
#define MWB_INTERP_LINEAR 0
#define MWB_INTERP_NEAREST 1

/* status codes */
#define MWB_OK 0
#define MWB_EINVAL (-1)
#define MWB_ECUDA (-2)
#define MWB_ERANGE (-3)

/* select_roi termination codes (reference MetricTrace.termination strings) */
#define MWB_TERM_NONE 0
#define MWB_TERM_DEGENERATE 1       /* "degenerate"       coarse2fine.py:189-192 */
#define MWB_TERM_REGION_FLOOR 2     /* "region-floor"     coarse2fine.py:202-205 */
#define MWB_TERM_N_MIN 3            /* "n-min"            coarse2fine.py:227-229 */
#define MWB_TERM_DISTANCE 4         /* "distance-metrics" coarse2fine.py:250-252 */
#define MWB_TERM_EMPTY (-1)         /* ValueError         coarse2fine.py:187-188 */
#define MWB_TERM_OVERFLOW (-2)      /* more than MWB_MAX_ITERS iterations */

#define MWB_MAX_ITERS 64
#define MWB_MAX_CHILDREN 8

/* Regions are inclusive cell boxes {x0, y0, z0, x1, y1, z1} (z0 = z1 = 0 for
 * 2-D grids).  Dense slots are (ix * ny + iy) * nz + iz (ix * ny + iy in 2-D). */

/* one select_roi iteration (reference IterationRecord, coarse2fine.py:127-152).
 * n_children is 4 (2-D quadrants, reference order) or 8 (3-D octants, index =
 * xhigh + 2*yhigh + 4*zhigh).  has_stats: 0 = None (empty child), 1 =
 * {"mu","var"} (first iteration), 2 = full metric parts. */
typedef struct mwb_iter_record {
  int32_t iteration;
  int32_t n_children;
  int32_t counts[MWB_MAX_CHILDREN];
  int32_t selected;
  int32_t satisfied;
  int32_t has_stats[MWB_MAX_CHILDREN];
  int32_t clamped[MWB_MAX_CHILDREN];
  int32_t selected_region[6];
  int32_t expanded_region[6];
  double scores[MWB_MAX_CHILDREN];
  double mu[MWB_MAX_CHILDREN];
  double var[MWB_MAX_CHILDREN];
  double delta_raw[MWB_MAX_CHILDREN];
  double delta[MWB_MAX_CHILDREN];
  double w;
  double b;
} mwb_iter_record_t;

/* select_roi trace (reference MetricTrace, coarse2fine.py:155-166) */
typedef struct mwb_trace {
  int32_t termination;
  int32_t n_records;
  int32_t final_region[6];
  mwb_iter_record_t records[MWB_MAX_ITERS];
} mwb_trace_t;

/* BASELINE configs[2] segmentation trace (no reference counterpart). */
#define MWB_SEG_MAX_ITERS 32
typedef struct mwb_seg_record {
  int32_t iteration;
  int32_t selected;        /* quadrant index, reference order */
  int32_t parent[6];       /* region that was split */
  int32_t selected_region[6];
  double shift;            /* subtracted before max/mean (DMAS: iteration minimum) */
  double score[4];         /* max / mean of the shifted sub-grid energies */
  double emax[4];
  double emean[4];
} mwb_seg_record_t;

typedef struct mwb_seg_trace {
  int32_t n_records;
  int32_t stopped;         /* 1 when the stop size was reached */
  int32_t final_region[6];
  mwb_seg_record_t records[MWB_SEG_MAX_ITERS];
} mwb_seg_trace_t;

const char* mwb_last_error(void);
int mwb_version(void);
/* sizeof(mwb_trace_t), for binding-layout checks */
int64_t mwb_trace_bytes(void);

/*
 * Per-point delay table (computed once per focal-point list and geometry, then
 * reused by every scan / kind / window).  For each tile of 256 consecutive
 * points and each channel it stores the exact range {lo, hi} of the integer
 * delays and, per point, (i0 - lo) << 23 | frac23 where i0 = floor(n),
 * frac23 = floor((n - i0) * 2^23) and n = (|p - a_tx| + |p - a_rx|) / (v dt)
 * in fp64 (beamform.py:182-190).  The interpolation weights are then
 * f1 = frac23 * 2^-23 and f0 = 1 - f1, identical for a point in every call.
 * `table` must hold mwb_delay_table_bytes(n_pts, n_chan) bytes.
 */
int64_t mwb_delay_table_bytes(int n_pts, int n_chan);
int mwb_delay_table(const double* pts_xyz, int n_pts, const int32_t* d_count,
                    const int32_t* chan_txrx, int n_chan, const double* ant_xyz, int n_ant,
                    double inv_scale, int interp, void* table, void* stream);

/*
 * Synthesized DAS and/or DMAS energies of a list of focal points over S scans
 * that share one antenna geometry (replaces beamform.py:169-212).  Both kinds
 * share the per-sample channel sum s = Σ_c a_c, so requesting both costs one
 * pass over the samples: DAS = Σ_k s_k^2, DMAS = ½ Σ_k (s_k^2 − Σ_c a_c,k^2).
 *
 *   sig        device fp32 [S][n_chan][ld]; populated channels only (all-zero
 *              channels contribute exactly 0 in the reference and are dropped);
 *              samples n_samples..ld-1 must be zero; ld % 4 == 0.
 *   scan_stride  floats between scans (multiple of 4).
 *   chan_txrx  device int32 [n_chan][2] transmitter/receiver antenna index.
 *   ant_xyz    device fp64 [n_ant][3] antenna positions (m).
 *   inv_scale  1 / (propagation_speed * sample_interval)  (samples per metre).
 *   pts_xyz    device fp64 [n_pts][3] focal points (z = 0 for the 2-D slice).
 *   out_idx    device int32 [n_pts] output slot of each point (NULL = identity).
 *   d_count    device int32 scalar overriding n_pts (<= n_pts) or NULL; lets a
 *              device-side enumerator feed this launch without a host sync.
 *   table      the mwb_delay_table of the same points / channels / interp.
 *   k0, window energy is summed over aligned samples k in [k0, k0+window);
 *              the reference's full-record sum is k0 = 0, window = n_samples.
 *   out_das, out_dmas  device fp32 outputs (either may be NULL = kind not
 *              wanted), out[s*out_stride + out_idx[p]].
 *   key_das, key_dmas  device uint64 [S] or NULL: atomicMax of
 *              (ordered(value) << 32 | ~slot) = max energy, ties to the lowest slot.
 *   flags      device int32 or NULL: bit 0 set when a non-finite energy occurs.
 *   mode       0 = shared-memory staged (TMA bulk copies), 1 = L1/L2 gather.
 */
int mwb_energies(const float* sig, int n_scans, int64_t scan_stride, int n_chan, int ld,
                 int n_samples, const int32_t* chan_txrx, const double* ant_xyz, int n_ant,
                 double inv_scale, const double* pts_xyz, const int32_t* out_idx, int n_pts,
                 const int32_t* d_count, const void* table, int interp, int k0, int window,
                 float* out_das, float* out_dmas, int64_t out_stride, uint64_t* key_das,
                 uint64_t* key_dmas, int32_t* flags, int mode, void* stream);

/*
 * mwb_energies with a partials workspace: when the launch has few tiles and
 * the window spans several 32-sample chunks (the reference's full-record
 * energies, beamform.py:211-212), the chunks are spread over more CTAs and a
 * second kernel sums each point's chunk partials in chunk order, so every
 * energy is bit-identical to mwb_energies.  workspace_bytes >=
 * mwb_energies_split_bytes(n_pts, n_scans, window) enables the split; with a
 * smaller (or NULL) workspace the call is exactly mwb_energies.
 */
int64_t mwb_energies_split_bytes(int n_pts, int n_scans, int window);
int mwb_energies_split(const float* sig, int n_scans, int64_t scan_stride, int n_chan, int ld,
                       int n_samples, const int32_t* chan_txrx, const double* ant_xyz, int n_ant,
                       double inv_scale, const double* pts_xyz, const int32_t* out_idx, int n_pts,
                       const int32_t* d_count, const void* table, int interp, int k0, int window,
                       float* out_das, float* out_dmas, int64_t out_stride, uint64_t* key_das,
                       uint64_t* key_dmas, int32_t* flags, int mode, void* workspace,
                       int64_t workspace_bytes, void* stream);

/*
 * Packed multi-scan point lists: tile_info[t] = {scan, valid points} (int32
 * pairs) for every 256-point tile t of pts_xyz; each tile belongs to one scan.
 * The table is built per tile; the energy launch evaluates tile t on scan
 * tile_info[t].x only (one launch for per-scan point lists, e.g. every scan's
 * fine pass of a framework batch).  Other arguments as above.
 */
int mwb_delay_table_tiles(const double* pts_xyz, int n_pts, const int32_t* tile_info,
                          const int32_t* chan_txrx, int n_chan, const double* ant_xyz, int n_ant,
                          double inv_scale, int interp, void* table, void* stream);
int mwb_energies_tiles(const float* sig, int n_scans, int64_t scan_stride, int n_chan, int ld,
                       int n_samples, const int32_t* chan_txrx, const double* ant_xyz, int n_ant,
                       double inv_scale, const double* pts_xyz, const int32_t* out_idx, int n_pts,
                       const int32_t* tile_info, const void* table, int interp, int k0, int window,
                       float* out_das, float* out_dmas, int64_t out_stride, uint64_t* key_das,
                       uint64_t* key_dmas, int32_t* flags, int mode, void* stream);

/*
 * Batched fine-pass enumeration: the stride-1 cells of each scan's device
 * region d_regions[s] (int32[6]) that pass `mask` and are not on the
 * skip_stride lattice.  _count writes {padded points, tiles} to d_totals
 * (device int32[2]) and leaves each scan's cell count in the first n_scans
 * int32 of the workspace; after reading the totals, _write fills pts_xyz /
 * out_idx (slot ix*ny+iy) / tile_info.  Each scan starts on a 256-point tile
 * boundary.
 */
int64_t mwb_regions_workspace_bytes(int n_scans);
int mwb_enumerate_regions_count(int nx, int ny, const int32_t* d_regions, int n_scans,
                                const uint8_t* mask, int skip_stride, int32_t* d_totals,
                                void* workspace, void* stream);
int mwb_enumerate_regions_write(double ox, double oy, double res, int nx, int ny,
                                const int32_t* d_regions, int n_scans,
                                const uint8_t* mask, int skip_stride, double* pts_xyz,
                                int32_t* out_idx, int32_t* tile_info, void* workspace, void* stream);

/* Workspace (bytes) for mwb_enumerate_lattice / mwb_enumerate_volume. */
int64_t mwb_lattice_workspace_bytes(int nx, int ny, int stride);
int64_t mwb_volume_workspace_bytes(int nx, int ny, int nz, int stride);

/*
 * Enumerate the stride-`stride` lattice cells of region {x0,y0,x1,y1} (or of
 * the device region d_region, int32[6], when non-NULL), keep cells with
 * mask[slot] (mask may be NULL) and drop cells whose indices are all
 * multiples of skip_stride (> 0).  Writes fp64 cell centres origin +
 * (i + 0.5) * res (pts_xyz, z = 0), the dense slot (out_idx), the count
 * (d_count) and sets valid[slot] = 1.  Points come out in 16x16 lattice tiles.
 */
int mwb_enumerate_lattice(double ox, double oy, double res, int nx, int ny, int x0, int y0,
                          int x1, int y1, const int32_t* d_region, int stride,
                          const uint8_t* mask, int skip_stride, double* pts_xyz,
                          int32_t* out_idx, int32_t* d_count, uint8_t* valid, void* workspace,
                          void* stream);

/* 3-D voxel variant: box is a HOST int32[6]; points in 8x8x4 voxel tiles;
 * centres origin + (i + 0.5) * res on all three axes. */
int mwb_enumerate_volume(double ox, double oy, double oz, double res, int nx, int ny, int nz,
                         const int32_t* box, const int32_t* d_region, int stride,
                         const uint8_t* mask, int skip_stride, double* pts_xyz,
                         int32_t* out_idx, int32_t* d_count, uint8_t* valid, void* workspace,
                         void* stream);

/*
 * Device-resident iterative quadrant selection on a dense nx x ny energy map
 * whose valid cells lie on multiples of `lattice`.  Region {x0,y0,x1,y1} is
 * the breast region.  Writes the final region to d_region_out (int32[6]) and
 * the full trace to d_trace (mwb_trace_t).  One CTA, no host sync.
 */
int mwb_select_roi(const float* dense, const uint8_t* valid, int nx, int ny, int lattice,
                   int x0, int y0, int x1, int y1, double frame_fraction, int n_min,
                   int32_t* d_region_out, mwb_trace_t* d_trace, void* stream);

/* One select_roi per scan of a batch: CTA s reads dense + s * dense_stride
 * (the valid mask is shared) and writes d_regions_out[s] / d_traces[s]. */
int mwb_select_roi_batch(const float* dense, int64_t dense_stride, const uint8_t* valid, int nx,
                         int ny, int lattice, int x0, int y0, int x1, int y1,
                         double frame_fraction, int n_min, int n_scans, int32_t* d_regions_out,
                         mwb_trace_t* d_traces, void* stream);

/* 3-D octant selection on an nx x ny x nz map (box: HOST int32[6]). */
int mwb_select_roi_volume(const float* dense, const uint8_t* valid, int nx, int ny, int nz,
                          int lattice, const int32_t* box, double frame_fraction, int n_min,
                          int32_t* d_region_out, mwb_trace_t* d_trace, void* stream);

/*
 * BASELINE configs[2] segmentation: starting from region {x0,y0,x1,y1} of an
 * nx x ny grid (origin, res), split into the 4 reference quadrants, image each
 * on an n_sub x n_sub sub-grid spanning it (centres corner + (i + 0.5) * side /
 * n_sub), score each by max/mean of its energies (DMAS energies are shifted by
 * the iteration minimum so the ratio is defined), keep the argmax (ties to the
 * lowest index) and repeat until the kept segment's larger side is <=
 * stop_cells; at most max_iters iterations are enqueued (finished searches
 * turn the remaining launches into no-ops, so nothing syncs with the host).
 * The final segment goes to d_region_out (int32[6]); the first iteration's
 * sub-grids form the (2 n_sub)^2 low-resolution image `lowres` (may be NULL).
 */
int64_t mwb_segment_workspace_bytes(int n_sub, int n_chan);
int mwb_segment(const float* sig, int n_chan, int ld, int n_samples, const int32_t* chan_txrx,
                const double* ant_xyz, int n_ant, double inv_scale, int interp, int k0, int window,
                int kind, double ox, double oy, double res, int nx, int ny, int x0, int y0, int x1,
                int y1, int n_sub, int stop_cells, int max_iters, int32_t* d_region_out,
                float* lowres, mwb_seg_trace_t* d_trace, void* workspace, void* stream);

/*
 * mwb_segment for S scans [S][n_chan][ld] (scan_stride floats apart) that
 * share the antenna geometry, grid and start region: each scan runs its own
 * quadrant search, all scans advancing together (four launches per iteration
 * for the whole batch; finished scans add no work).  Outputs per scan s:
 * d_regions_out[6 s..], d_traces[s] and, if lowres != NULL, the (2 n_sub)^2
 * low-resolution image at lowres + s (2 n_sub)^2.  Every value equals what
 * mwb_segment returns for that scan alone (same routines, same order).
 * Replaces a per-scan loop over mwb_segment (no reference counterpart; see
 * mwb_segment).
 */
int64_t mwb_segment_batch_workspace_bytes(int n_scans, int n_sub, int n_chan);
int mwb_segment_batch(const float* sig, int n_scans, int64_t scan_stride, int n_chan, int ld,
                      int n_samples, const int32_t* chan_txrx, const double* ant_xyz, int n_ant,
                      double inv_scale, int interp, int k0, int window, int kind, double ox,
                      double oy, double res, int nx, int ny, int x0, int y0, int x1, int y1,
                      int n_sub, int stop_cells, int max_iters, int32_t* d_regions_out,
                      float* lowres, mwb_seg_trace_t* d_traces, void* workspace, void* stream);

/*
 * Batched segmentation over a precomputed region tree.  The regions a search
 * can visit depend only on the start region {x0,y0,x1,y1}, stop_cells and
 * max_iters, so a plan holds, for one geometry, grid and mask, the sub-grid
 * points and delay tables of every region that gets split and the fine-pass
 * cells (region & mask, stride 1) and tables of every region a search can end
 * in.  A run then costs two launches per iteration for the whole batch and two
 * for the fine pass, with no host synchronisation (CUDA-graph capturable).
 *
 * mwb_segment_plan_info: info[0] = plan bytes, info[1] = regions split,
 *   info[2] = terminal regions, info[3] = fine tiles per scan (workspace
 *   sizing).  MWB_ERANGE when the tree exceeds 16384 regions (use
 *   mwb_segment_batch then).
 * mwb_segment_plan_prepare: fills the plan (synchronises `stream` once: the
 *   node list is copied from the host).
 * mwb_segment_run_workspace_bytes: includes, for small batches with windows
 *   of several chunks (the full record), room for window-split partials.
 * mwb_segment_run: the search for S scans as in mwb_segment_batch, then every
 *   scan's fine pass into out_fine + s * out_stride (slot ix * ny + iy of the
 *   final region's cells; other slots untouched), argmax keys keys[s] (as
 *   mwb_energies; zero them first), fine-cell counts fine_counts[s] (may be
 *   NULL) and the non-finite flag.  Per scan, identical to mwb_segment + a
 *   lattice pass over its final region.
 */
int mwb_segment_plan_info(int nx, int ny, int x0, int y0, int x1, int y1, int n_sub, int stop_cells,
                          int max_iters, int n_chan, int64_t* info);
int mwb_segment_plan_prepare(const int32_t* chan_txrx, int n_chan, const double* ant_xyz, int n_ant,
                             double inv_scale, int interp, double ox, double oy, double res, int nx,
                             int ny, int x0, int y0, int x1, int y1, const uint8_t* mask, int n_sub,
                             int stop_cells, int max_iters, void* plan, void* stream);
int64_t mwb_segment_run_workspace_bytes(int n_scans, int n_sub, int fine_tiles_per_scan, int window);
int mwb_segment_run(const void* plan, const float* sig, int n_scans, int64_t scan_stride, int n_chan,
                    int ld, int n_samples, const int32_t* chan_txrx, const double* ant_xyz, int n_ant,
                    double inv_scale, int interp, int k0, int window, int kind, int nx, int ny, int x0,
                    int y0, int x1, int y1, int n_sub, int stop_cells, int max_iters,
                    int32_t* d_regions_out, float* lowres, mwb_seg_trace_t* d_traces, float* out_fine,
                    int64_t out_stride, uint64_t* keys, int32_t* fine_counts, int32_t* flags,
                    void* workspace, void* stream);

/*
 * Device-side scan synthesis (the input producer of the path): writes S scans
 * [S][n_chan][ld] fp32 (samples >= n_samples zero) for point scatterers
 * scatterers[S][n_scat][4] = {x, y, z, amplitude}.  model 0 = the reference
 * simulator's cosine-modulated Gaussian (a = fc, b = envelope width,
 * c = duration; simulate.py:53-73, 141-156), model 1 = BASELINE's
 * differentiated Gaussian (a = tau, b = centre t_c).  noise_mode 0 = none,
 * 1 = absolute sigma (sigma_param[s]), 2 = SNR in dB against the scan's peak
 * |clean| (sigma_param[s] = SNR, peak_ws = uint32[S] workspace).  Noise is
 * Philox-4x32-10 (seed, scan, channel, sample) + Box-Muller, reproducible but
 * not numpy's PCG64 stream.
 */
int mwb_simulate(float* out, int n_scans, int n_chan, int n_samples, int ld, const int32_t* chan_txrx,
                 const double* ant_xyz, int n_ant, const double* scatterers, int n_scat, double v, double dt,
                 double t0, int model, double a, double b, double c, const double* sigma_param, int noise_mode,
                 uint64_t seed, uint32_t* peak_ws, void* stream);

/*
 * Tensor-core (tcgen05) variant of mwb_energies for many scans of one
 * geometry (tile_info: NULL, or the padded layout's per-tile {0, count}): per
 * channel the tile's interpolation weights
 * [256 x 16] multiply the Hankel windows of 8 scans [16 x 256] in fp16 hi/lo
 * split (about fp32 accuracy), accumulated over channels in TMEM; DMAS's
 * channel self-terms come from windowed Gram entries.  Requirements: window
 * == 32 and every tile's per-channel delay spread <= 14 samples (check once
 * per table with mwb_table_max_span); otherwise use mwb_energies.  A tile
 * found to violate the spread limit sets bit 1 (value 2) of *flags; a span
 * start outside [j_lo, j_lo + j_count - 16] sets bit 2 (value 4).  The DMAS
 * self-terms come from windowed Gram entries precomputed per (scan,
 * channel, window offset j in [j_lo, j_lo + j_count)) by a pre-pass that also
 * takes each scan's max |y| (the per-scan fp16 scale).
 * Workspace: mwb_energies_tc_workspace_bytes(n_scans, n_chan, j_count, n_pts).
 */
int64_t mwb_energies_tc_workspace_bytes(int n_scans, int n_chan, int j_count, int n_pts);
/* Windows of any multiple of 32 samples (the reference's full-record energy,
 * beamform.py:211-212, included) on the tensor cores: one W = 32
 * mwb_energies_tc call per 32-sample chunk of the window [k0, k0 + window),
 * the chunk energies summed in fp64 and rounded once; writes the cells
 * `valid` marks (n_cells = nx * ny = the output stride) of each scan's maps,
 * their argmax keys and the flags of every chunk call (both kinds in one
 * fused pass per chunk).  Replaces, for batches of
 * one geometry, the per-dataset image() of beamform.py:283-342 with its
 * default full-record window. */
int64_t mwb_energies_tc_record_workspace_bytes(int n_scans, int n_chan, int j_count, int n_pts, int n_cells);
int mwb_energies_tc_record(const float* sig, int n_scans, int64_t scan_stride, int n_chan, int ld, int n_samples,
                           const int32_t* chan_txrx, const double* ant_xyz, int n_ant, double inv_scale,
                           const double* pts_xyz, const int32_t* out_idx, int n_pts, const int32_t* tile_info,
                           const void* table, int interp, int k0, int window, const uint8_t* valid, int n_cells,
                           float* out_das, float* out_dmas, uint64_t* key_das, uint64_t* key_dmas, int32_t* flags,
                           int j_lo, int j_count, void* workspace, void* stream);
int mwb_table_max_span(const void* table, int n_pts, int n_chan, int32_t* d_out, void* stream);
/* smallest / largest per-channel span start lo over the table's non-empty
 * tiles -> d_out[0], d_out[1]; the window-offset range of mwb_energies_tc is
 * j_lo = d_out[0], j_count = d_out[1] + 16 - d_out[0]. */
int mwb_table_lo_range(const void* table, int n_pts, int n_chan, const int32_t* tile_info, int32_t* d_out,
                       void* stream);
int mwb_energies_tc(const float* sig, int n_scans, int64_t scan_stride, int n_chan, int ld, int n_samples,
                    const int32_t* chan_txrx, const double* ant_xyz, int n_ant, double inv_scale,
                    const double* pts_xyz, const int32_t* out_idx, int n_pts, const int32_t* d_count,
                    const int32_t* tile_info, const void* table, int interp, int k0, int window, float* out_das,
                    float* out_dmas, int64_t out_stride, uint64_t* key_das, uint64_t* key_dmas, int32_t* flags,
                    int j_lo, int j_count, void* workspace, void* stream);

/*
 * Padded lattice enumeration (for mwb_energies_tc on masked or ragged grids):
 * like mwb_enumerate_lattice, but lattice tile t's points occupy slots
 * [256 t, 256 t + count_t) of pts_xyz / out_idx (the list has
 * 256 * mwb_lattice_tile_count(nx, ny, stride) slots) and tile_info[t] =
 * {0, count_t} (int32 pairs), the per-tile record mwb_delay_table_tiles and
 * mwb_energies_tc take.  Table tiles then coincide with 16 x 16 lattice
 * tiles, whose delay spread is small.  d_count receives the total count.
 */
int64_t mwb_lattice_tile_count(int nx, int ny, int stride);
int mwb_enumerate_lattice_padded(double ox, double oy, double res, int nx, int ny, int x0, int y0, int x1, int y1,
                                 int stride, const uint8_t* mask, int skip_stride, double* pts_xyz,
                                 int32_t* out_idx, int32_t* tile_info, int32_t* d_count, uint8_t* valid,
                                 void* workspace, void* stream);

/*
 * One-call lattice image: the reference's image(ds, kind, grid, region,
 * stride, mask, skip=stride-lattice) (mwbeam/beamform.py:283-342) as
 * enumerate -> delay table -> one fused DAS/DMAS launch, all stream-ordered,
 * no host sync.  Region {x0,y0,x1,y1} of an nx x ny grid (origin ox, oy;
 * cell centres origin + (i + 0.5) * res).  Energies of the evaluated cells go
 * to out_das / out_dmas (nx * ny dense, either may be NULL) at slot
 * ix * ny + iy, and valid[slot] = 1; untouched cells keep their contents.
 * d_count receives the number of evaluated cells.  key_das / key_dmas /
 * flags are as in mwb_energies and must be zeroed by the caller, like valid.
 * Workspace: mwb_image_lattice_workspace_bytes(nx, ny, stride, n_chan).
 */
int64_t mwb_image_lattice_workspace_bytes(int nx, int ny, int stride, int n_chan);
int mwb_image_lattice(const float* sig, int n_chan, int ld, int n_samples, const int32_t* chan_txrx,
                      const double* ant_xyz, int n_ant, double inv_scale, int interp, int k0, int window,
                      double ox, double oy, double res, int nx, int ny, int x0, int y0, int x1, int y1,
                      int stride, const uint8_t* mask, int skip_stride, float* out_das, float* out_dmas,
                      uint8_t* valid, int32_t* d_count, uint64_t* key_das, uint64_t* key_dmas, int32_t* flags,
                      void* workspace, void* stream);

/* argmax over a dense map (valid cells only); key as in mwb_energies. */
int mwb_argmax_dense(const float* dense, const uint8_t* valid, int n, uint64_t* key,
                     void* stream);

/*
 * The coarse-to-fine framework's fine pass (coarse2fine.py:321-323) on a
 * precomputed whole-grid point list in the padded 16 x 16 tile layout
 * (mwb_enumerate_lattice_padded + mwb_delay_table_tiles, tile_info {0, count}):
 * only cells inside the device box region {x0, y0, z0, x1, y1, z1} (the select
 * kernel's output) that are not coarse-lattice cells (ix % skip_stride == 0 &&
 * iy % skip_stride == 0; skip_stride 0 = none) are evaluated and written; each is
 * marked in valid and counted into *count (device, atomically added).  Tiles
 * with no such cell exit at once, so the launch costs about what the ROI
 * costs, with no host sync and no per-call enumeration or delay table.
 * Other arguments as mwb_energies / mwb_energies_split (one scan).
 */
int mwb_energies_region(const float* sig, int n_chan, int ld, int n_samples, const int32_t* chan_txrx,
                        const double* ant_xyz, int n_ant, double inv_scale, const double* pts_xyz,
                        const int32_t* out_idx, int n_pts, const int32_t* tile_info, const void* table, int interp,
                        int k0, int window, float* out_das, float* out_dmas, uint64_t* key_das, uint64_t* key_dmas,
                        int32_t* flags, const int32_t* region, int ny, int skip_stride, uint8_t* valid,
                        int32_t* count, int mode, void* workspace, int64_t workspace_bytes, void* stream);

/*
 * Device staging of a .mwb container's series.  payload: the file's (m*m, n)
 * fp64 little-endian series already in device memory (one H2D of the bytes).
 * Writes the populated channels (any sample != 0; NaN counts as nonzero) in
 * row-major (i, j) order as fp32 rows of ld >= n floats with a zero tail to
 * out (capacity m*m rows), their (tx, rx) pairs to pairs (capacity m*m x 2
 * int32) and the count to *count (device).  An all-zero record keeps channel
 * (0, 0).  ws: m*m int32 of device workspace.  m in [1, 256].
 */
int mwb_compact_payload(const double* payload, int m, int n, int ld, float* out, int32_t* pairs, int32_t* count,
                        int32_t* ws, void* stream);

/*
 * 8-bit PGM rasters of n_maps energy maps (export_energy_map's rendering):
 * values (value_bits 32: float, 64: double) and valid (bytes) are
 * [n_maps][map_stride] with cell (ix, iy) at ix * ny + iy.  Writes vrange
 * (2 doubles per map: min and max over the valid cells) and raster
 * [n_maps][ny][nx] (row r = iy, column c = ix), each byte
 * rint(255 * clip((v - min) / (max - min), 0, 1)) in IEEE fp64, where v is the
 * cell's value, else (stride > 1) the value of the stride lattice cell whose
 * block holds it, else 0; a constant map renders as zeros.
 */
int mwb_render_pgm(const void* values, int value_bits, const uint8_t* valid, int n_maps, int nx, int ny,
                   int64_t map_stride, int stride, double* vrange, uint8_t* raster, void* stream);

/* Compact readback of a framework composite: out[i] = dense[coarse_slots[i]]
 * for i < n_coarse, then the device box region {x0, y0, z0, x1, y1, z1}'s
 * cells in (ix, iy, iz) order (dense is [nx][ny][nz], nz = 1 in 2-D), at most
 * cap values in all. */
int mwb_gather_composite(const float* dense, int ny, int nz, const int32_t* coarse_slots, int n_coarse,
                         const int32_t* region, float* out, int64_t cap, void* stream);

/* Stream-ordered copy of `bytes` between any two CUDA-visible addresses
 * (cudaMemcpyDefault): the drop-in's per-call signal-slot refill and result
 * readback without a framework op per copy. */
int mwb_memcpy_async(void* dst, const void* src, int64_t bytes, void* stream);

/* Blocks the calling host thread until `stream` has drained
 * (cudaStreamSynchronize): the one wait of a drop-in call before it decodes
 * the readback (pkg/src/mwbeam/coarse2fine.py:301-350 returns host values). */
int mwb_stream_synchronize(void* stream);

/* Stream-ordered 2-D copy (cudaMemcpy2DAsync, cudaMemcpyDefault): `height`
 * rows of `width` bytes, row pitches in bytes. */
int mwb_memcpy2d_async(void* dst, int64_t dpitch, const void* src, int64_t spitch, int64_t width, int64_t height,
                       void* stream);

/* The samples mwb_energies_tc reads from each channel row for a window start
 * k0 and a window-offset range (j_lo, j_count), rows of ld samples: out[0] =
 * the first sample, out[1] = the count (the Gram and fp16-plane pre-passes
 * read exactly [out[0], out[0] + out[1]); samples past ld read as zeros).  A
 * host-to-device pipeline may ship only that range of each row. */
/* K-packing statistics of the last mwb_energies_tc call (window 32) that used
 * `workspace` with these sizes: the MMA steps of all (table tile, M-block)
 * items of one scan-group pair (synchronous; for roofline accounting -- each
 * step is 6 tcgen05.mma M128 x N256 x K16 per pair of 8-scan groups). */
int mwb_tc_plan_steps(const void* workspace, int n_scans, int n_chan, int j_count, int n_pts, int window,
                      int64_t* out_steps);
int mwb_tc_sample_range(int k0, int j_lo, int j_count, int ld, int32_t* out);

/* Elapsed milliseconds between consecutive recorded events: out_ms[i] =
 * events[i] -> events[i + 1] for i < n_events - 1 (the framework report's
 * phase timings in one call). */
/* Host-side compaction of an (rows, n) fp64 record into fp32 rows of ld
 * floats (zero tail) for the rows holding a nonzero sample (x != 0.0),
 * their indices in keep; an all-zero record keeps row 0.  Returns the row
 * count (>= 1) or a negative status.  The drop-in's upload of a new dataset
 * (pkg/src/mwbeam/simulate.py:76-108 BackscatterDataset.signals). */
int mwb_compact_rows_host(const double* src, int rows, int n, int ld, float* dst, int32_t* keep);
int mwb_elapsed_ms(void* const* events, int n_events, float* out_ms);

/*
 * Roofline microbenchmarks run on the device: which = 0 shared-memory LDS.32
 * bandwidth (bytes), 1 FFMA2 (flops), 2 scalar FFMA (flops).  Writes the work
 * done by one launch to *work and the elapsed milliseconds to *ms.
 */
int mwb_microbench(int which, double* work, float* ms, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* MWB_H */
