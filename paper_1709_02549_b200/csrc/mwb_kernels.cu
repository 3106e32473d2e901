// mwb_kernels.cu — sm_100a kernels + C ABI for confocal DAS/DMAS imaging and
// the coarse-to-fine segment selection of arXiv 1709.02549.
//
// Reference (CPU, numpy) being replaced, paths relative to /root/reference:
//   energy kernel      pkg/src/mwbeam/beamform.py:169-212 (_multistatic_energies)
//   lattice + skip     pkg/src/mwbeam/beamform.py:268-280, 309-323 (_region_cells, image)
//   segment selection  pkg/src/mwbeam/coarse2fine.py:169-256 (select_roi), 67-109
//   argmax tie-break   pkg/src/mwbeam/beamform.py:101-104 (EnergyMap.argmax_cell)
//
// Design:
//   * one CTA = a tile of 256 focal points (128 threads x 2 points; the two
//     points of a thread are packed into float2 lanes of FFMA2/FADD2/FMUL2);
//   * per tile, each channel's needed sample span [k0+lo_c, k0+hi_c+CH] is
//     staged into shared memory with cp.async.bulk (TMA 1-D) into a 3-deep
//     full/empty mbarrier ring across (scan, window-chunk, channel-group)
//     steps;
//   * per-point per-antenna distances are fp64 (exactly the reference's
//     expression, no FMA contraction), the per-channel delay is
//     (d_tx + d_rx) * inv_scale in fp64, split into i0 = floor and an fp32
//     fraction — computed per point only, so a point's energy is bit-identical
//     whichever tile or call evaluates it;
//   * 32 (or 48) window samples per point live in registers (float2 s[CH]);
//     the per-point accumulation order over channels and samples is fixed;
//   * many scans of one geometry (configs[3]) go to the tensor-core kernel
//     in mwb_tc.cuh instead (mwb_energies_tc).
//
// Layout: this file holds the C ABI (include/mwb.h); the device code is in
// headers included into one translation unit, inside an anonymous namespace:
//   mwb_common.cuh     constants, PTX helpers, shared numerics, EnergyParams
//   mwb_energy.cuh     K0 delay table, K1 energy kernel, window-split reduce
//   mwb_lattice.cuh    lattice / voxel / per-scan region enumeration
//   mwb_select.cuh     K2 / K2w select_roi (quadrants, octants)
//   mwb_simulate.cuh   K5 device scan synthesis
//   mwb_segment.cuh    K4 BASELINE segmentation (single, batched, region tree)
//   mwb_microbench.cuh roofline microbenchmarks
//   mwb_tc.cuh         K1-TC tensor-core multi-scan kernel
#include <cuda.h>  // CUtensorMap (types only; the encoder comes through cudaGetDriverEntryPoint)
#include <cuda_runtime.h>
#include <vector>
#include <cuda_fp16.h>
#include <algorithm>
#include <stdint.h>
#include <stdio.h>
#include <stdarg.h>
#include <string.h>
#include <math.h>
#include <stdlib.h>

#include "../../include/mwb.h"

namespace {

#include "mwb_common.cuh"
#include "mwb_energy.cuh"
#include "mwb_lattice.cuh"
#include "mwb_select.cuh"
#include "mwb_simulate.cuh"
#include "mwb_segment.cuh"
#include "mwb_microbench.cuh"
#include "mwb_tc.cuh"
#include "mwb_tch.cuh"
#include "mwb_io.cuh"

}  // namespace

// ============================================================================
// C ABI
// ============================================================================
extern "C" {

const char* mwb_last_error(void) { return g_err; }

int mwb_version(void) { return 1; }

int64_t mwb_trace_bytes(void) { return (int64_t)sizeof(mwb_trace_t); }

int64_t mwb_delay_table_bytes(int n_pts, int n_chan) {
  if (n_pts < 0 || n_chan < 1) return -1;
  const long long tiles = (n_pts + TILE - 1) / TILE;
  return (int64_t)table_layout(tiles > 0 ? tiles : 1, n_chan).total;
}

static int delay_table_impl(const double* pts_xyz, int n_pts, const int32_t* d_count, const int32_t* tile_info,
                            const int32_t* chan_txrx, int n_chan, const double* ant_xyz, int n_ant,
                            double inv_scale, int interp, void* table, void* stream) {
  if (n_pts < 0 || n_chan < 1 || n_ant < 1) return set_err(MWB_EINVAL, "mwb_delay_table: bad sizes");
  if (n_pts == 0) return MWB_OK;
  if (n_ant > MAX_ANT) return set_err(MWB_ERANGE, "mwb_delay_table: too many antennas (%d)", n_ant);
  if (n_chan > MAX_CHAN) return set_err(MWB_ERANGE, "mwb_delay_table: too many channels (%d)", n_chan);
  if (interp != MWB_INTERP_LINEAR && interp != MWB_INTERP_NEAREST)
    return set_err(MWB_EINVAL, "mwb_delay_table: bad interpolation");
  if (!pts_xyz || !chan_txrx || !ant_xyz || !table) return set_err(MWB_EINVAL, "mwb_delay_table: null pointer");
  if (!(inv_scale > 0.0) || !isfinite(inv_scale)) return set_err(MWB_EINVAL, "mwb_delay_table: inv_scale must be > 0");
  const long long tiles = (n_pts + TILE - 1) / TILE;
  const TableLayout T = table_layout(tiles, n_chan);
  TableParams p;
  p.pts = pts_xyz;
  p.P = n_pts;
  p.d_count = d_count;
  p.chan = chan_txrx;
  p.C = n_chan;
  p.ant = ant_xyz;
  p.M = n_ant;
  p.inv_scale = inv_scale;
  p.interp = interp;
  p.tile_info = reinterpret_cast<const int2*>(tile_info);
  unsigned char* base = reinterpret_cast<unsigned char*>(table);
  p.words = reinterpret_cast<uint32_t*>(base + T.words);
  p.span = reinterpret_cast<int2*>(base + T.span);
  p.wide = reinterpret_cast<int*>(base + T.wide);
  const size_t sm = sizeof(double) * ((size_t)n_ant * TILE + 2 * (size_t)n_ant) + sizeof(int) * (2 * (size_t)n_chan + 2) +
                    sizeof(int2) * (size_t)n_chan;
  if (sm > 227 * 1024) return set_err(MWB_ERANGE, "mwb_delay_table: shared memory %lld bytes", (long long)sm);
  cudaError_t e = cudaFuncSetAttribute(delay_table_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  if (e != cudaSuccess) return set_err(MWB_ECUDA, "cudaFuncSetAttribute: %s", cudaGetErrorString(e));
  delay_table_kernel<<<(unsigned)tiles, TPB, sm, reinterpret_cast<cudaStream_t>(stream)>>>(p);
  return check_launch("delay_table_kernel");
}

int mwb_delay_table(const double* pts_xyz, int n_pts, const int32_t* d_count, const int32_t* chan_txrx,
                    int n_chan, const double* ant_xyz, int n_ant, double inv_scale, int interp,
                    void* table, void* stream) {
  return delay_table_impl(pts_xyz, n_pts, d_count, nullptr, chan_txrx, n_chan, ant_xyz, n_ant, inv_scale, interp,
                          table, stream);
}

int mwb_delay_table_tiles(const double* pts_xyz, int n_pts, const int32_t* tile_info, const int32_t* chan_txrx,
                          int n_chan, const double* ant_xyz, int n_ant, double inv_scale, int interp,
                          void* table, void* stream) {
  if (!tile_info) return set_err(MWB_EINVAL, "mwb_delay_table_tiles: null tile_info");
  return delay_table_impl(pts_xyz, n_pts, nullptr, tile_info, chan_txrx, n_chan, ant_xyz, n_ant, inv_scale, interp,
                          table, stream);
}

// Argument checks and EnergyParams of mwb_energies / mwb_energies_tiles /
// mwb_energies_tc.  Returns MWB_OK with *empty set when there is no work.
static int energy_params(const float* sig, int n_scans, int64_t scan_stride, int n_chan, int ld, int n_samples,
                         const int32_t* chan_txrx, const double* ant_xyz, int n_ant, double inv_scale,
                         const double* pts_xyz, const int32_t* out_idx, int n_pts, const int32_t* d_count,
                         const int32_t* tile_info, const void* table, int interp, int k0, int window,
                         float* out_das, float* out_dmas, int64_t out_stride, uint64_t* key_das,
                         uint64_t* key_dmas, int32_t* flags, int mode, EnergyParams& p, bool& empty) {
  empty = false;
  if (n_pts < 0 || n_scans < 0 || n_chan < 0 || n_ant < 1 || window < 0 || k0 < 0)
    return set_err(MWB_EINVAL, "mwb_energies: negative size");
  if (n_pts == 0 || n_scans == 0) {
    empty = true;
    return MWB_OK;
  }
  if (n_chan == 0 || window == 0)
    return set_err(MWB_EINVAL, "mwb_energies: no channels or empty window");
  if (!out_das && !out_dmas) return set_err(MWB_EINVAL, "mwb_energies: no output (kind) requested");
  if (interp != MWB_INTERP_LINEAR && interp != MWB_INTERP_NEAREST)
    return set_err(MWB_EINVAL, "mwb_energies: bad interpolation");
  if (n_ant > MAX_ANT) return set_err(MWB_ERANGE, "mwb_energies: too many antennas (%d)", n_ant);
  if (n_chan > MAX_CHAN) return set_err(MWB_ERANGE, "mwb_energies: too many channels (%d)", n_chan);
  if (ld % 4 != 0 || scan_stride % 4 != 0 || ld < n_samples)
    return set_err(MWB_EINVAL, "mwb_energies: ld and scan_stride must be multiples of 4, ld >= n_samples");
  if (!sig || !chan_txrx || !ant_xyz || !pts_xyz || !table)
    return set_err(MWB_EINVAL, "mwb_energies: null pointer");
  if (((uintptr_t)sig & 15) != 0) return set_err(MWB_EINVAL, "mwb_energies: sig must be 16-byte aligned");
  if (!(inv_scale > 0.0) || !isfinite(inv_scale)) return set_err(MWB_EINVAL, "mwb_energies: inv_scale must be > 0");

  const long long tiles = (n_pts + TILE - 1) / TILE;
  const TableLayout T = table_layout(tiles, n_chan);
  const unsigned char* base = reinterpret_cast<const unsigned char*>(table);
  p.sig = sig;
  p.scan_stride = scan_stride;
  p.n_scans = n_scans;
  p.C = n_chan;
  p.ld = ld;
  p.N = n_samples;
  p.chan = chan_txrx;
  p.ant = ant_xyz;
  p.M = n_ant;
  p.inv_scale = inv_scale;
  p.pts = pts_xyz;
  p.out_idx = out_idx;
  p.P = n_pts;
  p.d_count = d_count;
  p.tile_info = reinterpret_cast<const int2*>(tile_info);
  p.tile_src = nullptr;
  p.src_tiles = 0;
  p.tab_words = reinterpret_cast<const uint32_t*>(base + T.words);
  p.tab_span = reinterpret_cast<const int2*>(base + T.span);
  p.tab_wide = reinterpret_cast<const int*>(base + T.wide);
  p.interp = interp;
  p.k0 = k0;
  p.W = window;
  p.out_das = out_das;
  p.out_dmas = out_dmas;
  p.out_stride = out_stride;
  p.key_das = reinterpret_cast<unsigned long long*>(key_das);
  p.key_dmas = reinterpret_cast<unsigned long long*>(key_dmas);
  p.flags = flags;
  p.mode = mode;
  p.scans_per_cta = 1;
  p.cap = 0;
  p.part = nullptr;
  p.chunks_per_cta = 0;
  p.filt_region = nullptr;
  p.filt_ny = 1;
  p.filt_skip = 0;
  p.filt_valid = nullptr;
  p.filt_count = nullptr;
  return MWB_OK;
}

struct RegionFilter {
  const int32_t* region;
  int ny, skip;
  uint8_t* valid;
  int32_t* count;
};

static int energies_impl(const float* sig, int n_scans, int64_t scan_stride, int n_chan, int ld,
                         int n_samples, const int32_t* chan_txrx, const double* ant_xyz, int n_ant,
                         double inv_scale, const double* pts_xyz, const int32_t* out_idx, int n_pts,
                         const int32_t* d_count, const int32_t* tile_info, const void* table, int interp, int k0,
                         int window, float* out_das, float* out_dmas, int64_t out_stride, uint64_t* key_das,
                         uint64_t* key_dmas, int32_t* flags, int mode, void* stream,
                         const int32_t* tile_src = nullptr, int n_src_pts = 0, void* part_ws = nullptr,
                         int64_t part_bytes = 0, const RegionFilter* filt = nullptr) {
  // tile_src (with tile_info): launched tile t evaluates source tile tile_src[t]
  // of a shared point list / table of n_src_pts points; n_pts counts the
  // launched (packed output) positions
  EnergyParams p;
  bool empty;
  const int rc = energy_params(sig, n_scans, scan_stride, n_chan, ld, n_samples, chan_txrx, ant_xyz, n_ant,
                               inv_scale, pts_xyz, out_idx, tile_src ? n_src_pts : n_pts, d_count, tile_info, table,
                               interp, k0, window, out_das, out_dmas, out_stride, key_das, key_dmas, flags, mode, p,
                               empty);
  if (rc || empty) return rc;
  if (tile_src) {
    p.tile_src = tile_src;
    p.src_tiles = (n_src_pts + TILE - 1) / TILE;
    p.P = n_pts;
  }
  if (filt) {
    p.filt_region = filt->region;
    p.filt_ny = filt->ny;
    p.filt_skip = filt->skip;
    p.filt_valid = filt->valid;
    p.filt_count = filt->count;
  }
  const long long tiles = (n_pts + TILE - 1) / TILE;
  // register chunk: 48 samples for windows that are a multiple of 48 (the
  // configs[4] W = 48 would waste a third of a 2 x 32 split), else 32
  const int ch = (window % 48 == 0 && window % 32 != 0) ? MWB_W48_CH : MWB_W32_CH;
  const int resident = ch == 48 ? MWB_W48_MINB : MWB_W32_MINB;  // CTAs per SM the register budget allows
  // stage capacity: every channel's span for a compact tile, capped at 32 KB
  // and at what leaves `resident` CTAs room in the SM's 228 KB
  long long cap = (long long)n_chan * (ch + 24);
  cap = (cap + 3) & ~3LL;
  if (cap > CAP_MAX) cap = CAP_MAX;
  {
    const long long fixed = (long long)smem_layout(n_chan, 0).total + 1024;  // + per-CTA reserve
    const long long fit = ((228LL * 1024 / resident - fixed) / (4LL * NSTAGE)) & ~3LL;
    if (cap > fit) cap = fit;
  }
  if (cap < 256) cap = 256;
  p.cap = (int)cap;
  p.scans_per_cta = tile_info ? 1 : choose_scans_per_cta((int)tiles, n_scans);
  const SmemLayout L = smem_layout(n_chan, p.cap);
  if (L.total > 227 * 1024)
    return set_err(MWB_ERANGE, "mwb_energies: shared memory %lld bytes exceeds 227 KB", (long long)L.total);
  dim3 grid((unsigned)tiles, tile_info ? 1 : (n_scans + p.scans_per_cta - 1) / p.scans_per_cta);
  // Window split: a launch with few tiles and a long window (the reference's
  // full-record energies) leaves most SMs idle, so the window's chunks are
  // spread over grid.z when the caller passed a partials workspace.  Launches
  // over a device count (lattice passes) may hold far fewer points than their
  // tile bound, so they are treated as small.
  const int n_chunks = (window + ch - 1) / ch;
  if (part_ws && n_chunks > 1) {
    // launches over a device count or an ROI filter may do far less work than their tile bound
    const long long work_ctas = (long long)((d_count || filt) ? std::min<long long>(tiles, 16) : tiles) * grid.y;
    const long long target = 148LL * resident * 4;
    long long groups = std::min<long long>(n_chunks, (target + work_ctas - 1) / work_ctas);
    const long long rows = tile_info ? (long long)n_pts : (long long)n_scans * n_pts;
    const long long need = rows * n_chunks * (long long)sizeof(float2);
    if (groups > 1 && need <= part_bytes && grid.y * groups <= 65535) {
      p.chunks_per_cta = (int)((n_chunks + groups - 1) / groups);
      grid.z = (unsigned)((n_chunks + p.chunks_per_cta - 1) / p.chunks_per_cta);
      p.part = reinterpret_cast<float2*>(part_ws);
    }
  }
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const int kind = out_das && out_dmas ? KIND_BOTH : (out_das ? KIND_DAS : KIND_DMAS);
  // MWB_MINB=4 selects the 4-CTA/SM (<=128 registers) build of the 32-sample kernel
  static const int minb = [] {
    const char* e = getenv("MWB_MINB");
    return (e && atoi(e) == 4) ? 4 : 3;
  }();
  void (*fn)(EnergyParams);
  if (ch == 48)
    fn = kind == KIND_DAS ? energy_kernel<KIND_DAS, MWB_W48_MINB, 48>
         : (kind == KIND_DMAS ? energy_kernel<KIND_DMAS, MWB_W48_MINB, 48> : energy_kernel<KIND_BOTH, MWB_W48_MINB, 48>);
#if MWB_W48_CH == 24
  else if (ch == 24)
    fn = kind == KIND_DAS ? energy_kernel<KIND_DAS, 3, 24>
         : (kind == KIND_DMAS ? energy_kernel<KIND_DMAS, 3, 24> : energy_kernel<KIND_BOTH, 3, 24>);
#endif
  else if (minb == 4)
    fn = kind == KIND_DAS ? energy_kernel<KIND_DAS, 4, 32>
         : (kind == KIND_DMAS ? energy_kernel<KIND_DMAS, 4, 32> : energy_kernel<KIND_BOTH, 4, 32>);
  else
    fn = kind == KIND_DAS ? energy_kernel<KIND_DAS, MWB_W32_MINB, MWB_W32_CH>
         : (kind == KIND_DMAS ? energy_kernel<KIND_DMAS, MWB_W32_MINB, MWB_W32_CH>
                              : energy_kernel<KIND_BOTH, MWB_W32_MINB, MWB_W32_CH>);
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L.total);
  if (e != cudaSuccess) return set_err(MWB_ECUDA, "cudaFuncSetAttribute: %s", cudaGetErrorString(e));
  fn<<<grid, TPB, L.total, st>>>(p);
  if (!p.part) return check_launch("energy_kernel");
  if (const int lrc = check_launch("energy_kernel")) return lrc;
  void (*rk)(EnergyParams, int) = kind == KIND_DAS ? energy_reduce_kernel<KIND_DAS>
                                  : (kind == KIND_DMAS ? energy_reduce_kernel<KIND_DMAS> : energy_reduce_kernel<KIND_BOTH>);
  rk<<<dim3((unsigned)((n_pts + 255) / 256), tile_info ? 1u : (unsigned)n_scans), 256, 0, st>>>(p, n_chunks);
  return check_launch("energy_reduce_kernel");
}

int mwb_energies(const float* sig, int n_scans, int64_t scan_stride, int n_chan, int ld,
                 int n_samples, const int32_t* chan_txrx, const double* ant_xyz, int n_ant,
                 double inv_scale, const double* pts_xyz, const int32_t* out_idx, int n_pts,
                 const int32_t* d_count, const void* table, int interp, int k0, int window,
                 float* out_das, float* out_dmas, int64_t out_stride, uint64_t* key_das,
                 uint64_t* key_dmas, int32_t* flags, int mode, void* stream) {
  return energies_impl(sig, n_scans, scan_stride, n_chan, ld, n_samples, chan_txrx, ant_xyz, n_ant, inv_scale,
                       pts_xyz, out_idx, n_pts, d_count, nullptr, table, interp, k0, window, out_das, out_dmas,
                       out_stride, key_das, key_dmas, flags, mode, stream);
}

int64_t mwb_energies_split_bytes(int n_pts, int n_scans, int window) {
  if (n_pts < 0 || n_scans < 0 || window < 0) return -1;
  const int ch = (window % 48 == 0 && window % 32 != 0) ? MWB_W48_CH : MWB_W32_CH;
  return (int64_t)n_pts * n_scans * ((window + ch - 1) / ch) * (int64_t)sizeof(float2);
}

int mwb_energies_split(const float* sig, int n_scans, int64_t scan_stride, int n_chan, int ld,
                       int n_samples, const int32_t* chan_txrx, const double* ant_xyz, int n_ant,
                       double inv_scale, const double* pts_xyz, const int32_t* out_idx, int n_pts,
                       const int32_t* d_count, const void* table, int interp, int k0, int window,
                       float* out_das, float* out_dmas, int64_t out_stride, uint64_t* key_das,
                       uint64_t* key_dmas, int32_t* flags, int mode, void* workspace, int64_t workspace_bytes,
                       void* stream) {
  return energies_impl(sig, n_scans, scan_stride, n_chan, ld, n_samples, chan_txrx, ant_xyz, n_ant, inv_scale,
                       pts_xyz, out_idx, n_pts, d_count, nullptr, table, interp, k0, window, out_das, out_dmas,
                       out_stride, key_das, key_dmas, flags, mode, stream, nullptr, 0, workspace, workspace_bytes);
}

int mwb_energies_tiles(const float* sig, int n_scans, int64_t scan_stride, int n_chan, int ld, int n_samples,
                       const int32_t* chan_txrx, const double* ant_xyz, int n_ant, double inv_scale,
                       const double* pts_xyz, const int32_t* out_idx, int n_pts, const int32_t* tile_info,
                       const void* table, int interp, int k0, int window, float* out_das, float* out_dmas,
                       int64_t out_stride, uint64_t* key_das, uint64_t* key_dmas, int32_t* flags, int mode,
                       void* stream) {
  if (!tile_info) return set_err(MWB_EINVAL, "mwb_energies_tiles: null tile_info");
  return energies_impl(sig, n_scans, scan_stride, n_chan, ld, n_samples, chan_txrx, ant_xyz, n_ant, inv_scale,
                       pts_xyz, out_idx, n_pts, nullptr, tile_info, table, interp, k0, window, out_das, out_dmas,
                       out_stride, key_das, key_dmas, flags, mode, stream);
}

int mwb_energies_region(const float* sig, int n_chan, int ld, int n_samples, const int32_t* chan_txrx,
                        const double* ant_xyz, int n_ant, double inv_scale, const double* pts_xyz,
                        const int32_t* out_idx, int n_pts, const int32_t* tile_info, const void* table, int interp,
                        int k0, int window, float* out_das, float* out_dmas, uint64_t* key_das, uint64_t* key_dmas,
                        int32_t* flags, const int32_t* region, int ny, int skip_stride, uint8_t* valid,
                        int32_t* count, int mode, void* workspace, int64_t workspace_bytes, void* stream) {
  if (!tile_info || !region || !valid || !count || !out_idx || ny < 1)
    return set_err(MWB_EINVAL, "mwb_energies_region: null pointer or bad ny");
  const RegionFilter f{region, ny, skip_stride, valid, count};
  return energies_impl(sig, 1, 0, n_chan, ld, n_samples, chan_txrx, ant_xyz, n_ant, inv_scale, pts_xyz, out_idx,
                       n_pts, nullptr, tile_info, table, interp, k0, window, out_das, out_dmas, 0, key_das, key_dmas,
                       flags, mode, stream, nullptr, 0, workspace, workspace_bytes, &f);
}

// ---- tensor-core path (mwb_tc.cuh) ----------------------------------------
// cuTensorMapEncodeTiled through the runtime's driver entry point (no libcuda link)
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_tiled() {
  static EncodeTiledFn fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      f = nullptr;
    return reinterpret_cast<EncodeTiledFn>(f);
  }();
  return fn;
}

// 3-D tensor map {d0, d1, d2} (elements; d0 contiguous), row strides in
// bytes, box {b0, b1, b2}; out-of-bounds elements load as zeros
static int encode_3d(CUtensorMap* m, const void* base, uint64_t d0, uint64_t d1, uint64_t d2, uint64_t stride1,
                     uint64_t stride2, uint32_t b0, uint32_t b1, uint32_t b2, CUtensorMapDataType type) {
  EncodeTiledFn fn = encode_tiled();
  if (!fn) return set_err(MWB_ECUDA, "cuTensorMapEncodeTiled unavailable");
  const cuuint64_t dims[3] = {d0, d1, d2};
  const cuuint64_t strides[2] = {stride1, stride2};
  const cuuint32_t box[3] = {b0, b1, b2};
  const cuuint32_t estr[3] = {1, 1, 1};
  const CUresult r = fn(m, type, 3, const_cast<void*>(base), dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return set_err(MWB_ECUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return MWB_OK;
}

// rank-R tensor map (R <= 5): dims[0] contiguous, byte strides of dims 1..R-1
static int encode_nd(CUtensorMap* m, const void* base, int rank, const uint64_t* dims, const uint64_t* strides,
                     const uint32_t* box, CUtensorMapDataType type) {
  EncodeTiledFn fn = encode_tiled();
  if (!fn) return set_err(MWB_ECUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t d[5], st[4];
  cuuint32_t b[5], e[5];
  for (int i = 0; i < rank; ++i) {
    d[i] = dims[i];
    b[i] = box[i];
    e[i] = 1;
    if (i) st[i - 1] = strides[i - 1];
  }
  const CUresult r = fn(m, type, (cuuint32_t)rank, const_cast<void*>(base), d, st, b, e, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return set_err(MWB_ECUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return MWB_OK;
}

// workspace: [absmax u32 x S | gram {E, X} float4 pairs x quads*C*J | fp16 planes S*C*2*Lp]
static size_t tc_ws_absmax(int n_scans) { return align_up(sizeof(uint32_t) * (size_t)(n_scans > 0 ? n_scans : 1), 256); }
static size_t tc_ws_gram(int n_scans, int n_chan, int j_count) {
  return 2 * sizeof(float4) * (size_t)((n_scans + 3) / 4) * (size_t)n_chan * (size_t)j_count;
}
// plane length: the staged box [x0, x0 + SPANH) with x0 <= J - 16, 16-byte rows
static int tc_plane_len(int j_count) { return (j_count - 16 + tc::SPANH_MAX + 7) & ~7; }
static size_t tc_ws_planes(int n_scans, int n_chan, int j_count) {
  return sizeof(__half) * 2 * (size_t)n_scans * (size_t)n_chan * (size_t)tc_plane_len(j_count);
}

// W = 32 (mwb_tch.cuh): 8-scan interleaved planes [G][C][2][Lp][8] and the step plan
static size_t tc_ws_planes8(int n_scans, int n_chan, int j_count) {  // whole pairs of 8-scan groups
  return sizeof(__half) * 2 * 16 * (size_t)((n_scans + 15) / 16) * (size_t)n_chan * (size_t)tc_plane_len(j_count);
}
// per (tile, M-block): steps | step records | last steps per channel | A operands (<= C steps of 8 KB)
static size_t tc_ws_plan(int n_pts, int n_chan) {
  const size_t blocks = 2 * (size_t)(n_pts > 0 ? (n_pts + TILE - 1) / TILE : 1);
  return align_up(sizeof(int) * blocks, 256) + align_up(sizeof(uint4) * (size_t)n_chan * blocks, 256) +
         align_up(sizeof(int) * (size_t)n_chan * blocks, 256) + (size_t)tch::OP_B * (size_t)n_chan * blocks;
}

int64_t mwb_energies_tc_workspace_bytes(int n_scans, int n_chan, int j_count, int n_pts) {
  if (n_scans < 0 || n_chan < 1 || j_count < 16 || n_pts < 0) return -1;
  const size_t planes = std::max(tc_ws_planes(n_scans, n_chan, j_count), tc_ws_planes8(n_scans, n_chan, j_count));
  return (int64_t)(tc_ws_absmax(n_scans) + align_up(tc_ws_gram(n_scans, n_chan, j_count), 256) +
                   align_up(planes, 256) + align_up(tc_ws_plan(n_pts, n_chan), 256));
}

int mwb_table_lo_range(const void* table, int n_pts, int n_chan, const int32_t* tile_info, int32_t* d_out,
                       void* stream) {
  if (!table || !d_out || n_pts < 0 || n_chan < 1) return set_err(MWB_EINVAL, "mwb_table_lo_range: bad arguments");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  cudaError_t e = cudaMemsetAsync(d_out, 0x7F, sizeof(int32_t), st);
  if (e == cudaSuccess) e = cudaMemsetAsync(d_out + 1, 0xFF, sizeof(int32_t), st);
  if (e != cudaSuccess) return set_err(MWB_ECUDA, "cudaMemsetAsync: %s", cudaGetErrorString(e));
  if (n_pts == 0) return MWB_OK;
  const long long tiles = (n_pts + TILE - 1) / TILE;
  const TableLayout T = table_layout(tiles, n_chan);
  const unsigned char* base = reinterpret_cast<const unsigned char*>(table);
  long long blocks = (tiles * n_chan + 255) / 256;
  if (blocks > 148 * 4) blocks = 148 * 4;
  tc::table_lo_range_kernel<<<(unsigned)blocks, 256, 0, st>>>(reinterpret_cast<const int2*>(base + T.span),
                                                              reinterpret_cast<const int2*>(tile_info), tiles,
                                                              n_chan, d_out);
  return check_launch("table_lo_range_kernel");
}

int mwb_table_max_span(const void* table, int n_pts, int n_chan, int32_t* d_out, void* stream) {
  if (!table || !d_out || n_pts < 0 || n_chan < 1) return set_err(MWB_EINVAL, "mwb_table_max_span: bad arguments");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  cudaError_t e = cudaMemsetAsync(d_out, 0, sizeof(int32_t), st);
  if (e != cudaSuccess) return set_err(MWB_ECUDA, "cudaMemsetAsync: %s", cudaGetErrorString(e));
  if (n_pts == 0) return MWB_OK;
  const long long tiles = (n_pts + TILE - 1) / TILE;
  const TableLayout T = table_layout(tiles, n_chan);
  const unsigned char* base = reinterpret_cast<const unsigned char*>(table);
  long long blocks = (tiles * n_chan + 255) / 256;
  if (blocks > 148 * 4) blocks = 148 * 4;
  tc::table_max_span_kernel<<<(unsigned)blocks, 256, 0, st>>>(reinterpret_cast<const int2*>(base + T.span),
                                                              reinterpret_cast<const int*>(base + T.wide), tiles,
                                                              n_chan, d_out);
  return check_launch("table_max_span_kernel");
}

// one configuration of the tensor-core kernel: tensor maps, smem, persistent grid
extern "C++" {
template <class C>
static int launch_tc(const EnergyParams& e, int kind, int n_pts, int n_scans, int n_chan, int j_lo, int j_count,
                     int Lp, const uint32_t* absmax, const float4* gx, const __half* planes, cudaStream_t st) {
  int rc;
  tc::Params P;
  P.e = e;
  P.absmax = absmax;
  P.j_lo = j_lo;
  P.J = j_count;
  P.Lp = Lp;
  P.n_tiles = (n_pts + TILE - 1) / TILE;
  P.n_groups = (n_scans + C::SPG - 1) / C::SPG;
  const int quads = (n_scans + 3) / 4;
  if ((rc = encode_3d(&P.tm_planes, planes, (uint64_t)Lp, (uint64_t)2 * n_chan, (uint64_t)n_scans, (uint64_t)Lp * 2,
                      (uint64_t)Lp * 2 * 2 * n_chan, C::SPANH, 2, C::SPG, CU_TENSOR_MAP_DATA_TYPE_FLOAT16)))
    return rc;
  if ((rc = encode_3d(&P.tm_gram, gx, (uint64_t)8 * j_count, (uint64_t)n_chan, (uint64_t)quads,
                      (uint64_t)32 * j_count, (uint64_t)32 * j_count * n_chan, 128, 1, C::QUADS,
                      CU_TENSOR_MAP_DATA_TYPE_FLOAT32)))
    return rc;
  const tc::Layout L = tc::layout<C>();
  void (*fn)(tc::Params) = kind == KIND_DAS    ? tc::energy_tc_kernel<KIND_DAS, C>
                           : kind == KIND_DMAS ? tc::energy_tc_kernel<KIND_DMAS, C>
                                               : tc::energy_tc_kernel<KIND_BOTH, C>;
  cudaError_t ce = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L.total);
  if (ce != cudaSuccess) return set_err(MWB_ECUDA, "cudaFuncSetAttribute: %s", cudaGetErrorString(ce));
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const long long items = (long long)P.n_tiles * P.n_groups;
  const unsigned grid = (unsigned)std::min<long long>(items, sms > 0 ? sms : 148);
  fn<<<grid, tc::THREADS, L.total, st>>>(P);
  return check_launch("energy_tc_kernel");
}

// W = 32: the Hankel-in-place kernel (mwb_tch.cuh)
static int launch_tch(const EnergyParams& e, int kind, int n_pts, int n_scans, int n_chan, int j_lo, int j_count,
                      int Lp, const uint32_t* absmax, const float4* gx, const __half* planes8, const int* plan_n,
                      const uint4* plan, const int* plan_last, const unsigned char* a_ops, cudaStream_t st) {
  int rc;
  tch::Params P;
  P.e = e;
  P.absmax = absmax;
  P.plan_n = plan_n;
  P.plan = plan;
  P.plan_last = plan_last;
  P.a_ops = a_ops;
  P.j_lo = j_lo;
  P.J = j_count;
  P.Lp = Lp;
  P.n_tiles = (n_pts + TILE - 1) / TILE;
  P.n_pairs = (n_scans + tch::NGRP * tch::SPG - 1) / (tch::NGRP * tch::SPG);
  const int quads = (n_scans + 3) / 4;
  {
    // planes [2 n_pairs][C][hi | lo][Lp][8] fp16, viewed as 32-bit words so that a plane's rows
    // off + [0, ROWS) are one 896 B box row: one box = both groups' hi and lo spans of a channel
    const uint64_t prow = 16 * (uint64_t)Lp;  // bytes per plane
    const uint64_t dims[4] = {4 * (uint64_t)Lp, 2, (uint64_t)n_chan, 2 * (uint64_t)P.n_pairs};
    const uint64_t strides[3] = {prow, prow * 2, prow * 2 * n_chan};
    const uint32_t box[4] = {4 * tch::ROWS, 2, 1, tch::NGRP};
    if ((rc = encode_nd(&P.tm_planes, planes8, 4, dims, strides, box, CU_TENSOR_MAP_DATA_TYPE_UINT32))) return rc;
  }
  if ((rc = encode_3d(&P.tm_gram, gx, (uint64_t)8 * j_count, (uint64_t)n_chan, (uint64_t)quads,
                      (uint64_t)32 * j_count, (uint64_t)32 * j_count * n_chan, 128, 1, tch::QUADS,
                      CU_TENSOR_MAP_DATA_TYPE_FLOAT32)))
    return rc;
  const tch::Layout L = tch::layout();
  void (*fn)(tch::Params) = kind == KIND_DAS    ? tch::energy_tch_kernel<KIND_DAS>
                            : kind == KIND_DMAS ? tch::energy_tch_kernel<KIND_DMAS>
                                                : tch::energy_tch_kernel<KIND_BOTH>;
  cudaError_t ce = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L.total);
  if (ce != cudaSuccess) return set_err(MWB_ECUDA, "cudaFuncSetAttribute: %s", cudaGetErrorString(ce));
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const long long items = 2LL * P.n_tiles * P.n_pairs;
  const unsigned grid = (unsigned)std::min<long long>(items, sms > 0 ? sms : 148);
#ifdef MWB_TCH_PROF
  {
    unsigned long long z[16] = {0};
    cudaMemcpyToSymbol(tch::tch_prof, z, sizeof(z));
  }
#endif
#ifdef MWB_TCH_TRACE
  {
    unsigned int z0 = 0;
    cudaMemcpyToSymbol(tch::tch_trace_n, &z0, sizeof(z0));
  }
#endif
  fn<<<grid, tch::THREADS, L.total, st>>>(P);
#ifdef MWB_TCH_TRACE
  {
    cudaDeviceSynchronize();
    unsigned int nev = 0;
    cudaMemcpyFromSymbol(&nev, tch::tch_trace_n, sizeof(nev));
    nev = std::min(nev, 8192u);
    std::vector<unsigned long long> ev(2 * (size_t)nev);
    cudaMemcpyFromSymbol(ev.data(), tch::tch_trace, sizeof(unsigned long long) * 2 * nev);
    FILE* f = fopen(getenv("MWB_TCH_TRACE_FILE") ? getenv("MWB_TCH_TRACE_FILE") : "/tmp/tch_trace.txt", "w");
    for (unsigned int k = 0; k < nev; ++k)
      fprintf(f, "%llu %llu %llu\n", ev[2 * k], ev[2 * k + 1] >> 32, ev[2 * k + 1] & 0xFFFFFFFFull);
    fclose(f);
  }
#endif
#ifdef MWB_TCH_PROF
  {
    cudaDeviceSynchronize();
    unsigned long long z[16];
    cudaMemcpyFromSymbol(z, tch::tch_prof, sizeof(z));
    const double n = (double)grid;
    fprintf(stderr, "tch prof per CTA (Mclk): issuer total %.2f wait o_full %.2f wait acc_empty %.2f | builder0 "
            "total %.2f o_empty %.2f s_full %.2f acc_full %.2f epilogue %.2f | producer s_empty %.2f | items %.1f "
            "steps %.1f | producer issue %.2f total %.2f | A producer waits %.2f\n",
            z[2] / n / 1e6, z[0] / n / 1e6, z[1] / n / 1e6, z[10] / n / 1e6, z[3] / n / 1e6, z[4] / n / 1e6,
            z[5] / n / 1e6, z[6] / n / 1e6, z[7] / n / 1e6, z[8] / n, z[9] / n, z[11] / n / 1e6, z[12] / n / 1e6,
            z[15] / n / 1e6);
    fprintf(stderr, "tch prof issuer o_full waits (Mclk): item first step %.2f, steps 1-2 %.2f\n", z[15] / n / 1e6,
            z[14] / n / 1e6);
  }
#endif
  return check_launch("energy_tch_kernel");
}
}  // extern "C++"

int mwb_energies_tc(const float* sig, int n_scans, int64_t scan_stride, int n_chan, int ld, int n_samples,
                    const int32_t* chan_txrx, const double* ant_xyz, int n_ant, double inv_scale,
                    const double* pts_xyz, const int32_t* out_idx, int n_pts, const int32_t* d_count,
                    const int32_t* tile_info, const void* table, int interp, int k0, int window, float* out_das,
                    float* out_dmas, int64_t out_stride, uint64_t* key_das, uint64_t* key_dmas, int32_t* flags,
                    int j_lo, int j_count, void* workspace, void* stream) {
  EnergyParams e;
  bool empty;
  int rc = energy_params(sig, n_scans, scan_stride, n_chan, ld, n_samples, chan_txrx, ant_xyz, n_ant, inv_scale,
                         pts_xyz, out_idx, n_pts, d_count, tile_info, table, interp, k0, window, out_das, out_dmas,
                         out_stride, key_das, key_dmas, flags, 0, e, empty);
  if (rc || empty) return rc;
  if (window != 32 && window != 48)
    return set_err(MWB_EINVAL, "mwb_energies_tc: window must be 32 or 48 (got %d)", window);
  if (!workspace) return set_err(MWB_EINVAL, "mwb_energies_tc: null workspace");
  if (j_lo < 0 || j_count < 16) return set_err(MWB_EINVAL, "mwb_energies_tc: bad window-offset range");
  if (n_chan > 0xFFFF) return set_err(MWB_ERANGE, "mwb_energies_tc: %d channels (at most 65535)", n_chan);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  unsigned char* ws = reinterpret_cast<unsigned char*>(workspace);
  uint32_t* absmax = reinterpret_cast<uint32_t*>(ws);
  float4* gx = reinterpret_cast<float4*>(ws + tc_ws_absmax(n_scans));
  __half* planes = reinterpret_cast<__half*>(ws + tc_ws_absmax(n_scans) +
                                             align_up(tc_ws_gram(n_scans, n_chan, j_count), 256));
  const int Lp = tc_plane_len(j_count);
  cudaError_t ce = cudaMemsetAsync(absmax, 0, sizeof(uint32_t) * (size_t)n_scans, st);
  if (ce != cudaSuccess) return set_err(MWB_ECUDA, "cudaMemsetAsync: %s", cudaGetErrorString(ce));
  const size_t sm = sizeof(float) * 4 * (size_t)Lp;
  if (sm > 48 * 1024) return set_err(MWB_ERANGE, "mwb_energies_tc: window-offset range %d too wide", j_count);
  tc::gram_kernel<<<dim3((unsigned)n_chan, (unsigned)((n_scans + 3) / 4)), 128, sm, st>>>(
      sig, scan_stride, n_scans, n_chan, ld, k0, window, j_lo, j_count, Lp, gx, absmax);
  if ((rc = check_launch("gram_kernel"))) return rc;
  const int kind = out_das && out_dmas ? KIND_BOTH : (out_das ? KIND_DAS : KIND_DMAS);
  if (window == 32) {
    // 8-scan interleaved planes, the per-tile step plan, the Hankel-in-place kernel
    const int groups = 2 * ((n_scans + 15) / 16);  // whole pairs (the last pair's missing group is zeros)
    const long long tiles = (n_pts + TILE - 1) / TILE;
    unsigned char* pl = ws + tc_ws_absmax(n_scans) + align_up(tc_ws_gram(n_scans, n_chan, j_count), 256) +
                        align_up(std::max(tc_ws_planes(n_scans, n_chan, j_count),
                                          tc_ws_planes8(n_scans, n_chan, j_count)), 256);
    int* plan_n = reinterpret_cast<int*>(pl);
    uint4* plan = reinterpret_cast<uint4*>(pl + align_up(sizeof(int) * 2 * (size_t)tiles, 256));
    int* plan_last = reinterpret_cast<int*>(reinterpret_cast<unsigned char*>(plan) +
                                            align_up(sizeof(uint4) * (size_t)n_chan * 2 * tiles, 256));
    unsigned char* a_ops =
        reinterpret_cast<unsigned char*>(plan_last) + align_up(sizeof(int) * (size_t)n_chan * 2 * tiles, 256);
    tch::planes8_kernel<<<dim3((unsigned)n_chan, (unsigned)groups), 256, 0, st>>>(
        sig, scan_stride, n_scans, n_chan, ld, k0, j_lo, Lp, absmax, planes);
    if ((rc = check_launch("planes8_kernel"))) return rc;
    const TableLayout T = table_layout(tiles, n_chan);
    const unsigned char* tb = reinterpret_cast<const unsigned char*>(table);
    tch::plan_kernel<<<(unsigned)(2 * tiles), 256, sizeof(int) * 5 * (size_t)n_chan, st>>>(
        reinterpret_cast<const uint32_t*>(tb + T.words), reinterpret_cast<const int2*>(tile_info), n_pts, n_chan,
        plan_n, plan, plan_last);
    if ((rc = check_launch("plan_kernel"))) return rc;
    tch::abuild_kernel<<<(unsigned)(2 * tiles), 256, 0, st>>>(reinterpret_cast<const uint32_t*>(tb + T.words), n_chan,
                                                             plan_n, plan, a_ops);
    if ((rc = check_launch("abuild_kernel"))) return rc;
    return launch_tch(e, kind, n_pts, n_scans, n_chan, j_lo, j_count, Lp, absmax, gx, planes, plan_n, plan,
                      plan_last, a_ops, st);
  }
  tc::planes_kernel<<<dim3((unsigned)n_chan, (unsigned)n_scans), 128, 0, st>>>(sig, scan_stride, n_chan, ld, k0,
                                                                                j_lo, Lp, absmax, planes);
  if ((rc = check_launch("planes_kernel"))) return rc;
  if (n_scans >= 4) return launch_tc<tc::Cfg48x4>(e, kind, n_pts, n_scans, n_chan, j_lo, j_count, Lp, absmax, gx, planes, st);
  return launch_tc<tc::Cfg48x1>(e, kind, n_pts, n_scans, n_chan, j_lo, j_count, Lp, absmax, gx, planes, st);
}


// ---------------------------------------------------------------------------
// Long windows on the tensor cores: the window's 32-sample chunks one W = 32
// call each, the chunk energies summed in fp64 (DAS: sum of the chunks' sum of
// S^2; DMAS: of their (S^2 - Q) / 2 -- both additive over the window), then
// rounded to fp32 once, with the argmax keys and the non-finite flag of the
// final maps.
// ---------------------------------------------------------------------------
namespace {
__global__ void __launch_bounds__(256) record_accum_kernel(const float* __restrict__ tmp, double* __restrict__ acc,
                                                           long long n) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    acc[i] += (double)tmp[i];
}

__global__ void __launch_bounds__(256) record_finish_kernel(const double* __restrict__ acc, int n_cells,
                                                            const uint8_t* __restrict__ valid, float* out,
                                                            long long out_stride, unsigned long long* keys,
                                                            int32_t* flags) {
  const int s = blockIdx.y;
  const double* a = acc + (size_t)s * n_cells;
  float* o = out + (size_t)s * (size_t)out_stride;
  unsigned long long key = 0ull;
  bool bad = false;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n_cells; i += gridDim.x * blockDim.x) {
    if (!valid[i]) continue;
    const float v = __double2float_rn(a[i]);
    o[i] = v;
    if (isfinite(v)) key = max(key, (unsigned long long)argmax_key(v, i)); else bad = true;
  }
  if (keys) {
    const uint32_t hi = __reduce_max_sync(0xffffffffu, (uint32_t)(key >> 32));
    const uint32_t lo = __reduce_max_sync(0xffffffffu, (uint32_t)(key >> 32) == hi ? (uint32_t)key : 0u);
    key = ((unsigned long long)hi << 32) | lo;
    if ((threadIdx.x & 31) == 0 && key != 0ull) atomicMax(keys + s, key);
  }
  if (bad && flags) atomicOr(flags, 1);
}
}  // namespace

// [tmp DAS | tmp DMAS] fp32 chunk maps, then [acc DAS | acc DMAS] fp64
static size_t record_tmp_bytes(int n_scans, int n_cells) {
  return align_up(2 * (size_t)n_scans * n_cells * sizeof(float), 256);
}
static size_t record_maps_bytes(int n_scans, int n_cells) {
  return record_tmp_bytes(n_scans, n_cells) + 2 * (size_t)n_scans * n_cells * sizeof(double);
}

int64_t mwb_energies_tc_record_workspace_bytes(int n_scans, int n_chan, int j_count, int n_pts, int n_cells) {
  const int64_t tc_bytes = mwb_energies_tc_workspace_bytes(n_scans, n_chan, j_count, n_pts);
  if (tc_bytes < 0 || n_cells < 1) return -1;
  return (int64_t)align_up((size_t)tc_bytes, 256) + (int64_t)record_maps_bytes(n_scans, n_cells);
}

int mwb_energies_tc_record(const float* sig, int n_scans, int64_t scan_stride, int n_chan, int ld, int n_samples,
                           const int32_t* chan_txrx, const double* ant_xyz, int n_ant, double inv_scale,
                           const double* pts_xyz, const int32_t* out_idx, int n_pts, const int32_t* tile_info,
                           const void* table, int interp, int k0, int window, const uint8_t* valid, int n_cells,
                           float* out_das, float* out_dmas, uint64_t* key_das, uint64_t* key_dmas, int32_t* flags,
                           int j_lo, int j_count, void* workspace, void* stream) {
  if (window < 32 || window % 32) return set_err(MWB_EINVAL, "mwb_energies_tc_record: window %d is not a multiple of 32", window);
  if (!workspace || !valid || n_cells < 1 || n_scans < 0) return set_err(MWB_EINVAL, "mwb_energies_tc_record: bad arguments");
  if (!out_das && !out_dmas) return set_err(MWB_EINVAL, "mwb_energies_tc_record: no output");
  if (n_scans == 0 || n_pts == 0) return MWB_OK;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  unsigned char* ws = reinterpret_cast<unsigned char*>(workspace);
  const int64_t tc_bytes = mwb_energies_tc_workspace_bytes(n_scans, n_chan, j_count, n_pts);
  if (tc_bytes < 0) return set_err(MWB_EINVAL, "mwb_energies_tc_record: bad sizes");
  float* tmp = reinterpret_cast<float*>(ws + align_up((size_t)tc_bytes, 256));
  double* acc = reinterpret_cast<double*>(reinterpret_cast<unsigned char*>(tmp) + record_tmp_bytes(n_scans, n_cells));
  const long long n = (long long)n_scans * n_cells;
  float* tmp_k[2] = {out_das ? tmp : nullptr, out_dmas ? tmp + n : nullptr};
  int rc;
  cudaError_t ce = cudaMemsetAsync(acc, 0, 2 * sizeof(double) * (size_t)n, st);
  if (ce == cudaSuccess) ce = cudaMemsetAsync(tmp, 0, 2 * sizeof(float) * (size_t)n, st);  // cells no point writes
  if (ce != cudaSuccess) return set_err(MWB_ECUDA, "cudaMemsetAsync: %s", cudaGetErrorString(ce));
  for (int q = 0; q < window / 32; ++q) {  // both kinds in one fused W = 32 pass per chunk
    if ((rc = mwb_energies_tc(sig, n_scans, scan_stride, n_chan, ld, n_samples, chan_txrx, ant_xyz, n_ant, inv_scale,
                              pts_xyz, out_idx, n_pts, nullptr, tile_info, table, interp, k0 + 32 * q, 32, tmp_k[0],
                              tmp_k[1], n_cells, nullptr, nullptr, flags, j_lo, j_count, workspace, stream)))
      return rc;
    for (int kk = 0; kk < 2; ++kk) {
      if (!tmp_k[kk]) continue;
      record_accum_kernel<<<4 * 148, 256, 0, st>>>(tmp_k[kk], acc + (size_t)kk * n, n);
      if ((rc = check_launch("record_accum_kernel"))) return rc;
    }
  }
  for (int kk = 0; kk < 2; ++kk) {
    float* out = kk == 0 ? out_das : out_dmas;
    if (!out) continue;
    const unsigned bx = (unsigned)std::min(64, (n_cells + 255) / 256);
    record_finish_kernel<<<dim3(bx, (unsigned)n_scans), 256, 0, st>>>(
        acc + (size_t)kk * n, n_cells, valid, out, n_cells,
        reinterpret_cast<unsigned long long*>(kk == 0 ? key_das : key_dmas), flags);
    if ((rc = check_launch("record_finish_kernel"))) return rc;
  }
  return MWB_OK;
}

static long long lattice_tiles(int nx, int ny, int nz, int stride, int tx, int ty, int tz) {
  const long long Lx = (nx + stride - 1) / stride, Ly = (ny + stride - 1) / stride,
                  Lz = (nz + stride - 1) / stride;
  return ((Lx + tx - 1) / tx) * ((Ly + ty - 1) / ty) * ((Lz + tz - 1) / tz);
}

int64_t mwb_lattice_workspace_bytes(int nx, int ny, int stride) {
  if (nx < 1 || ny < 1 || stride < 1) return -1;
  return 2 * lattice_tiles(nx, ny, 1, stride, 16, 16, 1) * (long long)sizeof(int) + 256;
}

int64_t mwb_volume_workspace_bytes(int nx, int ny, int nz, int stride) {
  if (nx < 1 || ny < 1 || nz < 1 || stride < 1) return -1;
  return 2 * lattice_tiles(nx, ny, nz, stride, 8, 8, 4) * (long long)sizeof(int) + 256;
}

static int enumerate_common(LatticeParams& p, int tx, int ty, int tz, void* workspace, void* stream) {
  const long long tiles = lattice_tiles(p.nx, p.ny, p.nz, p.stride, tx, ty, tz);
  p.tx = tx;
  p.ty = ty;
  p.tz = tz;
  p.n_tiles_max = (int)tiles;
  p.tile_counts = reinterpret_cast<int*>(workspace);
  p.tile_offsets = p.tile_counts + tiles;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  lattice_count_kernel<<<(unsigned)tiles, 256, 0, st>>>(p);
  lattice_scan_kernel<<<1, 1024, 0, st>>>(p);
  lattice_write_kernel<<<(unsigned)tiles, 256, 0, st>>>(p);
  return check_launch("enumerate_lattice");
}

int mwb_enumerate_lattice(double ox, double oy, double res, int nx, int ny, int x0, int y0,
                          int x1, int y1, const int32_t* d_region, int stride,
                          const uint8_t* mask, int skip_stride, double* pts_xyz,
                          int32_t* out_idx, int32_t* d_count, uint8_t* valid, void* workspace,
                          void* stream) {
  if (nx < 1 || ny < 1 || stride < 1) return set_err(MWB_EINVAL, "mwb_enumerate_lattice: bad grid/stride");
  if (!d_region && (x0 < 0 || y0 < 0 || x1 >= nx || y1 >= ny || x0 > x1 || y0 > y1))
    return set_err(MWB_EINVAL, "mwb_enumerate_lattice: region outside the grid");
  if (!pts_xyz || !out_idx || !d_count || !valid || !workspace)
    return set_err(MWB_EINVAL, "mwb_enumerate_lattice: null pointer");
  LatticeParams p;
  p.pad_info = nullptr;
  p.ox = ox; p.oy = oy; p.oz = 0.0; p.res = res;
  p.nx = nx; p.ny = ny; p.nz = 1;
  p.planar = 1;
  p.r[0] = x0; p.r[1] = y0; p.r[2] = 0; p.r[3] = x1; p.r[4] = y1; p.r[5] = 0;
  p.d_region = d_region;
  p.stride = stride;
  p.mask = mask;
  p.skip = skip_stride;
  p.pts = pts_xyz;
  p.out_idx = out_idx;
  p.d_count = d_count;
  p.valid = valid;
  return enumerate_common(p, 16, 16, 1, workspace, stream);
}

int64_t mwb_lattice_tile_count(int nx, int ny, int stride) {
  if (nx < 1 || ny < 1 || stride < 1) return -1;
  return lattice_tiles(nx, ny, 1, stride, 16, 16, 1);
}

int mwb_enumerate_lattice_padded(double ox, double oy, double res, int nx, int ny, int x0, int y0, int x1, int y1,
                                 int stride, const uint8_t* mask, int skip_stride, double* pts_xyz,
                                 int32_t* out_idx, int32_t* tile_info, int32_t* d_count, uint8_t* valid,
                                 void* workspace, void* stream) {
  if (nx < 1 || ny < 1 || stride < 1) return set_err(MWB_EINVAL, "mwb_enumerate_lattice_padded: bad grid/stride");
  if (x0 < 0 || y0 < 0 || x1 >= nx || y1 >= ny || x0 > x1 || y0 > y1)
    return set_err(MWB_EINVAL, "mwb_enumerate_lattice_padded: region outside the grid");
  if (!pts_xyz || !out_idx || !tile_info || !d_count || !valid || !workspace)
    return set_err(MWB_EINVAL, "mwb_enumerate_lattice_padded: null pointer");
  LatticeParams p;
  p.pad_info = reinterpret_cast<int2*>(tile_info);
  p.ox = ox; p.oy = oy; p.oz = 0.0; p.res = res;
  p.nx = nx; p.ny = ny; p.nz = 1;
  p.planar = 1;
  p.r[0] = x0; p.r[1] = y0; p.r[2] = 0; p.r[3] = x1; p.r[4] = y1; p.r[5] = 0;
  p.d_region = nullptr;
  p.stride = stride;
  p.mask = mask;
  p.skip = skip_stride;
  p.pts = pts_xyz;
  p.out_idx = out_idx;
  p.d_count = d_count;
  p.valid = valid;
  return enumerate_common(p, 16, 16, 1, workspace, stream);
}

int mwb_enumerate_volume(double ox, double oy, double oz, double res, int nx, int ny, int nz,
                         const int32_t* box, const int32_t* d_region, int stride,
                         const uint8_t* mask, int skip_stride, double* pts_xyz,
                         int32_t* out_idx, int32_t* d_count, uint8_t* valid, void* workspace,
                         void* stream) {
  if (nx < 1 || ny < 1 || nz < 1 || stride < 1) return set_err(MWB_EINVAL, "mwb_enumerate_volume: bad grid/stride");
  if ((long long)nx * ny * nz > 0x7FFFFFFFLL) return set_err(MWB_ERANGE, "mwb_enumerate_volume: grid too large");
  if (!box) return set_err(MWB_EINVAL, "mwb_enumerate_volume: null box");
  const int dims[3] = {nx, ny, nz};
  for (int a = 0; a < 3; ++a)
    if (!d_region && (box[a] < 0 || box[3 + a] >= dims[a] || box[a] > box[3 + a]))
      return set_err(MWB_EINVAL, "mwb_enumerate_volume: box outside the grid");
  if (!pts_xyz || !out_idx || !d_count || !valid || !workspace)
    return set_err(MWB_EINVAL, "mwb_enumerate_volume: null pointer");
  LatticeParams p;
  p.pad_info = nullptr;
  p.ox = ox; p.oy = oy; p.oz = oz; p.res = res;
  p.nx = nx; p.ny = ny; p.nz = nz;
  p.planar = 0;
  for (int i = 0; i < 6; ++i) p.r[i] = box[i];
  p.d_region = d_region;
  p.stride = stride;
  p.mask = mask;
  p.skip = skip_stride;
  p.pts = pts_xyz;
  p.out_idx = out_idx;
  p.d_count = d_count;
  p.valid = valid;
  return enumerate_common(p, 8, 8, 4, workspace, stream);
}

static RegionBatch region_batch(void* workspace, int n_scans) {
  RegionBatch b;
  b.n_scans = n_scans;
  int* w = reinterpret_cast<int*>(workspace);
  b.scan_counts = w;
  b.scan_offsets = w + n_scans;
  b.totals = w + 2 * n_scans;
  return b;
}

int64_t mwb_regions_workspace_bytes(int n_scans) {
  if (n_scans < 0) return -1;
  return (long long)sizeof(int) * (2LL * n_scans + 2) + 256;
}

static LatticeParams region_params(double ox, double oy, double res, int nx, int ny, const int32_t* d_regions,
                                   const uint8_t* mask, int skip_stride) {
  LatticeParams p;
  p.pad_info = nullptr;
  memset(&p, 0, sizeof(p));
  p.ox = ox; p.oy = oy; p.oz = 0.0; p.res = res;
  p.nx = nx; p.ny = ny; p.nz = 1;
  p.planar = 1;
  p.d_region = d_regions;
  p.stride = 1;
  p.mask = mask;
  p.skip = skip_stride;
  p.tx = 16; p.ty = 16; p.tz = 1;
  return p;
}

int mwb_enumerate_regions_count(int nx, int ny, const int32_t* d_regions, int n_scans, const uint8_t* mask,
                                int skip_stride, int32_t* d_totals, void* workspace, void* stream) {
  if (nx < 1 || ny < 1 || n_scans < 1 || n_scans > 65535)
    return set_err(MWB_EINVAL, "mwb_enumerate_regions_count: bad sizes");
  if (!d_regions || !d_totals || !workspace) return set_err(MWB_EINVAL, "mwb_enumerate_regions_count: null pointer");
  RegionBatch b = region_batch(workspace, n_scans);
  LatticeParams p = region_params(0.0, 0.0, 1.0, nx, ny, d_regions, mask, skip_stride);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  region_count_kernel<<<n_scans, 256, 0, st>>>(p, b);
  region_offsets_kernel<<<1, 1024, 0, st>>>(b);
  cudaMemcpyAsync(d_totals, b.totals, 2 * sizeof(int), cudaMemcpyDeviceToDevice, st);
  return check_launch("enumerate_regions_count");
}

int mwb_enumerate_regions_write(double ox, double oy, double res, int nx, int ny, const int32_t* d_regions,
                                int n_scans, const uint8_t* mask, int skip_stride, double* pts_xyz,
                                int32_t* out_idx, int32_t* tile_info, void* workspace, void* stream) {
  if (nx < 1 || ny < 1 || n_scans < 1 || n_scans > 65535)
    return set_err(MWB_EINVAL, "mwb_enumerate_regions_write: bad sizes");
  if (!d_regions || !pts_xyz || !out_idx || !tile_info || !workspace)
    return set_err(MWB_EINVAL, "mwb_enumerate_regions_write: null pointer");
  RegionBatch b = region_batch(workspace, n_scans);
  LatticeParams p = region_params(ox, oy, res, nx, ny, d_regions, mask, skip_stride);
  p.pts = pts_xyz;
  p.out_idx = out_idx;
  region_write_kernel<<<n_scans, 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(p, b,
                                                                                 reinterpret_cast<int2*>(tile_info));
  return check_launch("enumerate_regions_write");
}

static int select_common(SelectParams& p, void* stream, int n_scans = 1) {
  long long n = 1;
  for (int a = 0; a < 3; ++a) {
    p.sl0[a] = (p.breast.lo[a] + p.D - 1) / p.D;
    const int l1 = p.breast.hi[a] / p.D;
    p.sL[a] = l1 >= p.sl0[a] ? l1 - p.sl0[a] + 1 : 0;
    n *= p.sL[a];
  }
  p.staged = n > 0 && n <= SEL_STAGE_MAX;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (p.dims == 2 && n > 0 && n <= SAT_MAX_CELLS) {  // K2s: summed-area tables, one CTA per scan
    const size_t sm = sat_smem_bytes(p.sL[0], p.sL[1]);
    cudaError_t e = cudaFuncSetAttribute(select_roi_sat_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)sat_smem_bytes(SAT_MAX_CELLS, 1) > (int)sm ? (int)sat_smem_bytes(SAT_MAX_CELLS, 1) : (int)sm);
    if (e != cudaSuccess) return set_err(MWB_ECUDA, "cudaFuncSetAttribute: %s", cudaGetErrorString(e));
    select_roi_sat_kernel<<<n_scans, SAT_TPB, sm, st>>>(p);
    return check_launch("select_roi_sat_kernel");
  }
  const size_t sm = p.staged ? sizeof(float) * (size_t)n : 0;
  void (*fn)(SelectParams) = p.dims == 3 ? select_roi_kernel<8> : select_roi_kernel<4>;
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)(sizeof(float) * SEL_STAGE_MAX));
  if (e != cudaSuccess) return set_err(MWB_ECUDA, "cudaFuncSetAttribute: %s", cudaGetErrorString(e));
  fn<<<n_scans, SEL_TPB, sm, st>>>(p);
  return check_launch("select_roi_kernel");
}

int mwb_select_roi(const float* dense, const uint8_t* valid, int nx, int ny, int lattice,
                   int x0, int y0, int x1, int y1, double frame_fraction, int n_min,
                   int32_t* d_region_out, mwb_trace_t* d_trace, void* stream) {
  if (nx < 1 || ny < 1 || lattice < 1) return set_err(MWB_EINVAL, "mwb_select_roi: bad grid");
  if (x0 < 0 || y0 < 0 || x1 >= nx || y1 >= ny || x0 > x1 || y0 > y1)
    return set_err(MWB_EINVAL, "mwb_select_roi: region outside the grid");
  if (!(frame_fraction >= 0.0 && frame_fraction < 1.0) || n_min < 1)
    return set_err(MWB_EINVAL, "mwb_select_roi: bad frame_fraction / n_min");
  if (!dense || !valid || !d_region_out || !d_trace) return set_err(MWB_EINVAL, "mwb_select_roi: null pointer");
  SelectParams p;
  p.dense = dense;
  p.valid = valid;
  p.nx = nx;
  p.ny = ny;
  p.nz = 1;
  p.D = lattice;
  p.dims = 2;
  p.breast = Box{{x0, y0, 0}, {x1, y1, 0}};
  p.frac = frame_fraction;
  p.n_min = n_min;
  p.region_out = d_region_out;
  p.trace = d_trace;
  p.dense_stride = 0;
  return select_common(p, stream);
}

int mwb_select_roi_batch(const float* dense, int64_t dense_stride, const uint8_t* valid, int nx, int ny,
                         int lattice, int x0, int y0, int x1, int y1, double frame_fraction, int n_min, int n_scans,
                         int32_t* d_regions_out, mwb_trace_t* d_traces, void* stream) {
  if (n_scans < 0 || dense_stride < (int64_t)nx * ny) return set_err(MWB_EINVAL, "mwb_select_roi_batch: bad batch");
  if (n_scans == 0) return MWB_OK;
  if (nx < 1 || ny < 1 || lattice < 1) return set_err(MWB_EINVAL, "mwb_select_roi_batch: bad grid");
  if (x0 < 0 || y0 < 0 || x1 >= nx || y1 >= ny || x0 > x1 || y0 > y1)
    return set_err(MWB_EINVAL, "mwb_select_roi_batch: region outside the grid");
  if (!(frame_fraction >= 0.0 && frame_fraction < 1.0) || n_min < 1)
    return set_err(MWB_EINVAL, "mwb_select_roi_batch: bad frame_fraction / n_min");
  if (!dense || !valid || !d_regions_out || !d_traces) return set_err(MWB_EINVAL, "mwb_select_roi_batch: null pointer");
  SelectParams p;
  p.dense = dense;
  p.valid = valid;
  p.nx = nx;
  p.ny = ny;
  p.nz = 1;
  p.D = lattice;
  p.dims = 2;
  p.breast = Box{{x0, y0, 0}, {x1, y1, 0}};
  p.frac = frame_fraction;
  p.n_min = n_min;
  p.region_out = d_regions_out;
  p.trace = d_traces;
  p.dense_stride = dense_stride;
  return select_common(p, stream, n_scans);
}

int mwb_select_roi_volume(const float* dense, const uint8_t* valid, int nx, int ny, int nz,
                          int lattice, const int32_t* box, double frame_fraction, int n_min,
                          int32_t* d_region_out, mwb_trace_t* d_trace, void* stream) {
  if (nx < 1 || ny < 1 || nz < 1 || lattice < 1 || !box) return set_err(MWB_EINVAL, "mwb_select_roi_volume: bad grid");
  const int dims[3] = {nx, ny, nz};
  for (int a = 0; a < 3; ++a)
    if (box[a] < 0 || box[3 + a] >= dims[a] || box[a] > box[3 + a])
      return set_err(MWB_EINVAL, "mwb_select_roi_volume: box outside the grid");
  if (!(frame_fraction >= 0.0 && frame_fraction < 1.0) || n_min < 1)
    return set_err(MWB_EINVAL, "mwb_select_roi_volume: bad frame_fraction / n_min");
  if (!dense || !valid || !d_region_out || !d_trace) return set_err(MWB_EINVAL, "mwb_select_roi_volume: null pointer");
  SelectParams p;
  p.dense = dense;
  p.valid = valid;
  p.nx = nx;
  p.ny = ny;
  p.nz = nz;
  p.D = lattice;
  p.dims = 3;
  p.breast = Box{{box[0], box[1], box[2]}, {box[3], box[4], box[5]}};
  p.frac = frame_fraction;
  p.n_min = n_min;
  p.region_out = d_region_out;
  p.trace = d_trace;
  p.dense_stride = 0;
  return select_common(p, stream);
}

int mwb_simulate(float* out, int n_scans, int n_chan, int n_samples, int ld, const int32_t* chan_txrx,
                 const double* ant_xyz, int n_ant, const double* scatterers, int n_scat, double v, double dt,
                 double t0, int model, double a, double b, double c, const double* sigma_param, int noise_mode,
                 uint64_t seed, uint32_t* peak_ws, void* stream) {
  if (n_scans < 0 || n_chan < 1 || n_samples < 1 || ld < n_samples || n_ant < 2 || n_scat < 0)
    return set_err(MWB_EINVAL, "mwb_simulate: bad sizes");
  if (model != 0 && model != 1) return set_err(MWB_EINVAL, "mwb_simulate: bad model");
  if (noise_mode < 0 || noise_mode > 2 || (noise_mode && !sigma_param) || (noise_mode == 2 && !peak_ws))
    return set_err(MWB_EINVAL, "mwb_simulate: bad noise arguments");
  if (!(v > 0) || !(dt > 0)) return set_err(MWB_EINVAL, "mwb_simulate: v and dt must be > 0");
  if (!out || !chan_txrx || !ant_xyz || (n_scat && !scatterers)) return set_err(MWB_EINVAL, "mwb_simulate: null pointer");
  if (n_scans == 0) return MWB_OK;
  if (n_chan > 65535 || n_scans > 65535) return set_err(MWB_ERANGE, "mwb_simulate: grid too large");
  SimParams p;
  p.out = out; p.S = n_scans; p.C = n_chan; p.N = n_samples; p.ld = ld;
  p.chan = chan_txrx; p.ant = ant_xyz; p.scat = scatterers; p.K = n_scat;
  p.v = v; p.dt = dt; p.t0 = t0; p.model = model; p.a = a; p.b = b; p.c = c;
  p.peak = reinterpret_cast<unsigned int*>(peak_ws); p.sigma_param = sigma_param; p.noise_mode = noise_mode;
  p.seed = seed;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (noise_mode == 2) cudaMemsetAsync(peak_ws, 0, sizeof(uint32_t) * n_scans, st);
  dim3 g1((ld + 255) / 256, n_chan, n_scans);
  sim_clean_kernel<<<g1, 256, 0, st>>>(p);
  int rc = check_launch("sim_clean_kernel");
  if (rc || !noise_mode) return rc;
  dim3 g2((n_samples / 4 + 1 + 127) / 128, n_chan, n_scans);
  sim_noise_kernel<<<g2, 128, 0, st>>>(p);
  return check_launch("sim_noise_kernel");
}

int64_t mwb_segment_workspace_bytes(int n_sub, int n_chan) {
  if (n_sub < 1 || n_sub > 64 || n_chan < 1) return -1;
  const long long n = 4LL * n_sub * n_sub;
  const long long tiles = (n + TILE - 1) / TILE;
  return (long long)align_up(sizeof(SegState), 256) + (long long)align_up(24 * n, 256) +
         (long long)align_up(4 * n, 256) + (long long)table_layout(tiles, n_chan).total;
}

int mwb_segment(const float* sig, int n_chan, int ld, int n_samples, const int32_t* chan_txrx,
                const double* ant_xyz, int n_ant, double inv_scale, int interp, int k0, int window,
                int kind, double ox, double oy, double res, int nx, int ny, int x0, int y0, int x1,
                int y1, int n_sub, int stop_cells, int max_iters, int32_t* d_region_out,
                float* lowres, mwb_seg_trace_t* d_trace, void* workspace, void* stream) {
  if (n_sub < 1 || n_sub > 64 || stop_cells < 1 || max_iters < 0 || max_iters > MWB_SEG_MAX_ITERS)
    return set_err(MWB_EINVAL, "mwb_segment: bad n_sub / stop_cells / max_iters");
  if (nx < 1 || ny < 1 || x0 < 0 || y0 < 0 || x1 >= nx || y1 >= ny || x0 > x1 || y0 > y1)
    return set_err(MWB_EINVAL, "mwb_segment: region outside the grid");
  if (kind != MWB_DAS && kind != MWB_DMAS) return set_err(MWB_EINVAL, "mwb_segment: bad kind");
  if (!d_region_out || !d_trace || !workspace) return set_err(MWB_EINVAL, "mwb_segment: null pointer");
  const int n = 4 * n_sub * n_sub;
  unsigned char* ws = reinterpret_cast<unsigned char*>(workspace);
  SegState* st = reinterpret_cast<SegState*>(ws);
  ws += align_up(sizeof(SegState), 256);
  double* pts = reinterpret_cast<double*>(ws);
  ws += align_up(24 * (size_t)n, 256);
  float* e = reinterpret_cast<float*>(ws);
  ws += align_up(4 * (size_t)n, 256);
  void* table = ws;
  cudaStream_t cs = reinterpret_cast<cudaStream_t>(stream);
  seg_init_kernel<<<1, 1, 0, cs>>>(st, x0, y0, x1, y1, stop_cells, d_trace);
  int rc = check_launch("seg_init_kernel");
  if (rc) return rc;
  for (int it = 0; it < max_iters; ++it) {
    // the done flag turns every launch of a finished search into a no-op
    seg_points_kernel<<<(n + 255) / 256, 256, 0, cs>>>(st, ox, oy, res, n_sub, pts);
    if ((rc = check_launch("seg_points_kernel"))) return rc;
    if ((rc = mwb_delay_table(pts, n, nullptr, chan_txrx, n_chan, ant_xyz, n_ant, inv_scale, interp, table, stream)))
      return rc;
    if ((rc = mwb_energies(sig, 1, 0, n_chan, ld, n_samples, chan_txrx, ant_xyz, n_ant, inv_scale, pts, nullptr,
                           n, nullptr, table, interp, k0, window, kind == MWB_DAS ? e : nullptr,
                           kind == MWB_DMAS ? e : nullptr, 0, nullptr, nullptr, nullptr, 0, stream)))
      return rc;
    seg_score_kernel<<<1, 256, 0, cs>>>(st, e, n_sub, kind == MWB_DMAS, stop_cells, lowres, d_trace);
    if ((rc = check_launch("seg_score_kernel"))) return rc;
  }
  seg_region_kernel<<<1, 1, 0, cs>>>(st, d_region_out);
  return check_launch("seg_region_kernel");
}

// Batched configs[2] search: S scans of one geometry, grid and start region,
// each with its own quadrant sequence.  Every iteration is four launches for
// the whole batch (points + tile list, delay table, energies, scores); a scan
// that has finished contributes empty tiles.  Per scan, every value equals
// mwb_segment's (same point placement, table words, energy routine and
// scoring body).
static long long seg_batch_per_scan(int n_sub) {
  const long long n = 4LL * n_sub * n_sub;
  return (n + TILE - 1) / TILE * TILE;
}

int64_t mwb_segment_batch_workspace_bytes(int n_scans, int n_sub, int n_chan) {
  if (n_scans < 1 || n_scans > 65535 || n_sub < 1 || n_sub > 64 || n_chan < 1) return -1;
  const long long per = seg_batch_per_scan(n_sub), n = per * n_scans;
  return (long long)align_up(sizeof(SegState) * (size_t)n_scans, 256) + (long long)align_up(24 * n, 256) +
         (long long)align_up(4 * n, 256) + (long long)align_up(8 * (n / TILE), 256) +
         (long long)table_layout(n / TILE, n_chan).total;
}

int mwb_segment_batch(const float* sig, int n_scans, int64_t scan_stride, int n_chan, int ld, int n_samples,
                      const int32_t* chan_txrx, const double* ant_xyz, int n_ant, double inv_scale, int interp,
                      int k0, int window, int kind, double ox, double oy, double res, int nx, int ny, int x0,
                      int y0, int x1, int y1, int n_sub, int stop_cells, int max_iters, int32_t* d_regions_out,
                      float* lowres, mwb_seg_trace_t* d_traces, void* workspace, void* stream) {
  if (n_scans < 1 || n_scans > 65535) return set_err(MWB_EINVAL, "mwb_segment_batch: n_scans must be in [1, 65535]");
  if (n_sub < 1 || n_sub > 64 || stop_cells < 1 || max_iters < 0 || max_iters > MWB_SEG_MAX_ITERS)
    return set_err(MWB_EINVAL, "mwb_segment_batch: bad n_sub / stop_cells / max_iters");
  if (nx < 1 || ny < 1 || x0 < 0 || y0 < 0 || x1 >= nx || y1 >= ny || x0 > x1 || y0 > y1)
    return set_err(MWB_EINVAL, "mwb_segment_batch: region outside the grid");
  if (kind != MWB_DAS && kind != MWB_DMAS) return set_err(MWB_EINVAL, "mwb_segment_batch: bad kind");
  if (!d_regions_out || !d_traces || !workspace) return set_err(MWB_EINVAL, "mwb_segment_batch: null pointer");
  const long long per = seg_batch_per_scan(n_sub), n = per * n_scans;
  if (n > 0x7FFFFFFFLL) return set_err(MWB_ERANGE, "mwb_segment_batch: %lld points exceed int32", n);
  unsigned char* ws = reinterpret_cast<unsigned char*>(workspace);
  SegState* st = reinterpret_cast<SegState*>(ws);
  ws += align_up(sizeof(SegState) * (size_t)n_scans, 256);
  double* pts = reinterpret_cast<double*>(ws);
  ws += align_up(24 * n, 256);
  float* e = reinterpret_cast<float*>(ws);
  ws += align_up(4 * n, 256);
  int2* tile_info = reinterpret_cast<int2*>(ws);
  ws += align_up(8 * (n / TILE), 256);
  void* table = ws;
  const int32_t* ti = reinterpret_cast<const int32_t*>(tile_info);
  cudaStream_t cs = reinterpret_cast<cudaStream_t>(stream);
  seg_init_batch_kernel<<<(n_scans + 255) / 256, 256, 0, cs>>>(st, n_scans, x0, y0, x1, y1, stop_cells, d_traces);
  int rc = check_launch("seg_init_batch_kernel");
  if (rc) return rc;
  for (int it = 0; it < max_iters; ++it) {
    seg_points_batch_kernel<<<dim3((unsigned)(per / TILE), (unsigned)n_scans), TILE, 0, cs>>>(
        st, (int)per, ox, oy, res, n_sub, pts, tile_info);
    if ((rc = check_launch("seg_points_batch_kernel"))) return rc;
    if ((rc = mwb_delay_table_tiles(pts, (int)n, ti, chan_txrx, n_chan, ant_xyz, n_ant, inv_scale, interp, table,
                                    stream)))
      return rc;
    if ((rc = mwb_energies_tiles(sig, n_scans, scan_stride, n_chan, ld, n_samples, chan_txrx, ant_xyz, n_ant,
                                 inv_scale, pts, nullptr, (int)n, ti, table, interp, k0, window,
                                 kind == MWB_DAS ? e : nullptr, kind == MWB_DMAS ? e : nullptr, 0, nullptr, nullptr,
                                 nullptr, 0, stream)))
      return rc;
    seg_score_batch_kernel<<<n_scans, 256, 0, cs>>>(st, e, (int)per, n_sub, kind == MWB_DMAS, stop_cells, lowres,
                                                    d_traces);
    if ((rc = check_launch("seg_score_batch_kernel"))) return rc;
  }
  seg_region_batch_kernel<<<(n_scans + 255) / 256, 256, 0, cs>>>(st, n_scans, d_regions_out);
  return check_launch("seg_region_batch_kernel");
}

// ---- batched search over a precomputed region tree -------------------------
// The regions a search can visit depend only on the start region, the stop
// size and the iteration bound, so for a fixed grid the sub-grid points and
// delay tables of every search node, and the fine-pass cells and tables of
// every terminal node, are built once (mwb_segment_plan_prepare) and shared
// by every scan of every batch.  A run is then 2 launches per iteration
// (energies of each scan's node tiles through tile_src; score + next map)
// plus 2 for the fine pass, with no host synchronisation.
struct SegTree {
  std::vector<SegNode> nodes;
  std::vector<int> search, term;
  long long fine_bound = 0;  // padded fine-pass points over terminal nodes
  int fine_tps = 0;          // most tiles of one terminal node
};

constexpr int SEG_TREE_MAX_NODES = 1 << 14;

static int build_seg_tree(int x0, int y0, int x1, int y1, int stop_cells, int max_iters, SegTree& T) {
  T = SegTree();
  std::vector<int> depth;
  SegNode root;
  memset(&root, 0, sizeof(root));
  root.region[0] = x0; root.region[1] = y0; root.region[3] = x1; root.region[4] = y1;
  T.nodes.push_back(root);
  depth.push_back(0);
  for (size_t i = 0; i < T.nodes.size(); ++i) {
    SegNode& nd = T.nodes[i];
    const int w = nd.region[3] - nd.region[0] + 1, h = nd.region[4] - nd.region[1] + 1;
    const bool done = max(w, h) <= stop_cells || w < 2 || h < 2;
    for (int k = 0; k < 4; ++k) nd.child[k] = -1;
    nd.search = nd.term = -1;
    if (done || depth[i] >= max_iters) {
      nd.term = (int)T.term.size();
      T.term.push_back((int)i);
      const long long tiles = ((long long)w * h + TILE - 1) / TILE;
      T.fine_bound += tiles * TILE;
      T.fine_tps = max(T.fine_tps, (int)tiles);
      continue;
    }
    nd.search = (int)T.search.size();
    T.search.push_back((int)i);
    Box r, q[MAXCH];
    for (int a = 0; a < 3; ++a) {
      r.lo[a] = nd.region[a];
      r.hi[a] = nd.region[3 + a];
    }
    split_box(r, 2, q);  // w, h >= 2: four quadrants
    const int d = depth[i];
    for (int k = 0; k < 4; ++k) {
      if (T.nodes.size() >= (size_t)SEG_TREE_MAX_NODES) return set_err(MWB_ERANGE, "segment tree: too many regions");
      T.nodes[i].child[k] = (int)T.nodes.size();
      SegNode c;
      memset(&c, 0, sizeof(c));
      for (int a = 0; a < 3; ++a) {
        c.region[a] = q[k].lo[a];
        c.region[3 + a] = q[k].hi[a];
      }
      T.nodes.push_back(c);  // invalidates nd
      depth.push_back(d + 1);
    }
  }
  return MWB_OK;
}

struct SegPlanLayout {
  size_t nodes, term_regions, search_ids, s_pts, s_info, s_table, r_ws, f_pts, f_idx, f_info, f_table, total;
};

static SegPlanLayout seg_plan_layout(const SegTree& T, int per_node, int n_chan) {
  SegPlanLayout L;
  const long long ns = (long long)T.search.size(), nt = (long long)T.term.size();
  const long long s_pts = ns * per_node;
  size_t o = 0;
  L.nodes = o;        o = align_up(o + sizeof(SegNode) * T.nodes.size(), 256);
  L.term_regions = o; o = align_up(o + sizeof(int) * 6 * (size_t)nt, 256);
  L.search_ids = o;   o = align_up(o + sizeof(int) * (size_t)ns, 256);
  L.s_pts = o;        o = align_up(o + 24 * (size_t)s_pts, 256);
  L.s_info = o;       o = align_up(o + 8 * (size_t)(s_pts / TILE), 256);
  L.s_table = o;      o += table_layout(s_pts / TILE, n_chan).total;
  L.r_ws = o;         o = align_up(o + (size_t)mwb_regions_workspace_bytes((int)nt), 256);
  L.f_pts = o;        o = align_up(o + 24 * (size_t)T.fine_bound, 256);
  L.f_idx = o;        o = align_up(o + 4 * (size_t)T.fine_bound, 256);
  L.f_info = o;       o = align_up(o + 8 * (size_t)(T.fine_bound / TILE), 256);
  L.f_table = o;      o += table_layout(T.fine_bound / TILE, n_chan).total;
  L.total = o;
  return L;
}

static int seg_tree_args(int nx, int ny, int x0, int y0, int x1, int y1, int n_sub, int stop_cells, int max_iters,
                         const char* who) {
  if (n_sub < 1 || n_sub > 64 || stop_cells < 1 || max_iters < 0 || max_iters > MWB_SEG_MAX_ITERS)
    return set_err(MWB_EINVAL, "%s: bad n_sub / stop_cells / max_iters", who);
  if (nx < 1 || ny < 1 || x0 < 0 || y0 < 0 || x1 >= nx || y1 >= ny || x0 > x1 || y0 > y1)
    return set_err(MWB_EINVAL, "%s: region outside the grid", who);
  return MWB_OK;
}

int mwb_segment_plan_info(int nx, int ny, int x0, int y0, int x1, int y1, int n_sub, int stop_cells,
                          int max_iters, int n_chan, int64_t* info) {
  int rc = seg_tree_args(nx, ny, x0, y0, x1, y1, n_sub, stop_cells, max_iters, "mwb_segment_plan_info");
  if (rc) return rc;
  if (n_chan < 1 || !info) return set_err(MWB_EINVAL, "mwb_segment_plan_info: bad n_chan / null info");
  SegTree T;
  if ((rc = build_seg_tree(x0, y0, x1, y1, stop_cells, max_iters, T))) return rc;
  const int per = (int)seg_batch_per_scan(n_sub);
  info[0] = (int64_t)seg_plan_layout(T, per, n_chan).total;
  info[1] = (int64_t)T.search.size();
  info[2] = (int64_t)T.term.size();
  info[3] = (int64_t)T.fine_tps;
  return MWB_OK;
}

int mwb_segment_plan_prepare(const int32_t* chan_txrx, int n_chan, const double* ant_xyz, int n_ant,
                             double inv_scale, int interp, double ox, double oy, double res, int nx, int ny,
                             int x0, int y0, int x1, int y1, const uint8_t* mask, int n_sub, int stop_cells,
                             int max_iters, void* plan, void* stream) {
  int rc = seg_tree_args(nx, ny, x0, y0, x1, y1, n_sub, stop_cells, max_iters, "mwb_segment_plan_prepare");
  if (rc) return rc;
  if (!chan_txrx || !ant_xyz || !plan || n_chan < 1) return set_err(MWB_EINVAL, "mwb_segment_plan_prepare: null pointer");
  SegTree T;
  if ((rc = build_seg_tree(x0, y0, x1, y1, stop_cells, max_iters, T))) return rc;
  const int per = (int)seg_batch_per_scan(n_sub);
  const SegPlanLayout L = seg_plan_layout(T, per, n_chan);
  unsigned char* base = reinterpret_cast<unsigned char*>(plan);
  cudaStream_t cs = reinterpret_cast<cudaStream_t>(stream);
  // nodes, search-node ids and terminal regions: one host->device copy
  std::vector<unsigned char> blob(L.s_pts);
  memcpy(blob.data() + L.nodes, T.nodes.data(), sizeof(SegNode) * T.nodes.size());
  int* treg = reinterpret_cast<int*>(blob.data() + L.term_regions);
  for (size_t k = 0; k < T.term.size(); ++k)
    for (int a = 0; a < 6; ++a) treg[6 * k + a] = T.nodes[T.term[k]].region[a];
  if (!T.search.empty()) memcpy(blob.data() + L.search_ids, T.search.data(), sizeof(int) * T.search.size());
  const int* d_search_ids = reinterpret_cast<const int*>(base + L.search_ids);
  cudaError_t e = cudaMemcpyAsync(base, blob.data(), blob.size(), cudaMemcpyHostToDevice, cs);
  if (e != cudaSuccess) return set_err(MWB_ECUDA, "mwb_segment_plan_prepare: %s", cudaGetErrorString(e));
  const SegNode* nodes = reinterpret_cast<const SegNode*>(base + L.nodes);
  // search nodes: sub-grid points + delay table
  const long long s_pts = (long long)T.search.size() * per;
  if (s_pts > 0) {
    int2* s_info = reinterpret_cast<int2*>(base + L.s_info);
    seg_tree_points_kernel<<<dim3((unsigned)(per / TILE), (unsigned)T.search.size()), TILE, 0, cs>>>(
        nodes, d_search_ids, per, ox, oy, res, n_sub, reinterpret_cast<double*>(base + L.s_pts), s_info);
    if ((rc = check_launch("seg_tree_points_kernel"))) return rc;
    if ((rc = mwb_delay_table_tiles(reinterpret_cast<double*>(base + L.s_pts), (int)s_pts,
                                    reinterpret_cast<const int32_t*>(s_info), chan_txrx, n_chan, ant_xyz, n_ant,
                                    inv_scale, interp, base + L.s_table, stream)))
      return rc;
  }
  // terminal nodes: fine-pass cells (region & mask) + delay table
  const int nt = (int)T.term.size();
  const int32_t* d_treg = reinterpret_cast<const int32_t*>(base + L.term_regions);
  cudaMemsetAsync(base + L.f_info, 0, 8 * (size_t)(T.fine_bound / TILE), cs);
  RegionBatch b = region_batch(base + L.r_ws, nt);
  LatticeParams lp = region_params(ox, oy, res, nx, ny, d_treg, mask, 0);
  region_count_kernel<<<nt, 256, 0, cs>>>(lp, b);
  region_offsets_kernel<<<1, 1024, 0, cs>>>(b);
  lp.pts = reinterpret_cast<double*>(base + L.f_pts);
  lp.out_idx = reinterpret_cast<int*>(base + L.f_idx);
  region_write_kernel<<<nt, 256, 0, cs>>>(lp, b, reinterpret_cast<int2*>(base + L.f_info));
  if ((rc = check_launch("segment plan: terminal cells"))) return rc;
  if ((rc = mwb_delay_table_tiles(reinterpret_cast<double*>(base + L.f_pts), (int)T.fine_bound,
                                  reinterpret_cast<const int32_t*>(base + L.f_info), chan_txrx, n_chan, ant_xyz,
                                  n_ant, inv_scale, interp, base + L.f_table, stream)))
    return rc;
  // the host blob must outlive its async copy
  e = cudaStreamSynchronize(cs);
  if (e != cudaSuccess) return set_err(MWB_ECUDA, "mwb_segment_plan_prepare: %s", cudaGetErrorString(e));
  return MWB_OK;
}

// Chunk partials for window-split launches of a small batch (long windows,
// e.g. the full record): sized for the larger of the search and fine lists,
// and only while that stays small (large batches fill the GPU unsplit).
static long long seg_run_part_bytes(int n_scans, int n_sub, int fine_tps, int window) {
  const int ch = (window % 48 == 0 && window % 32 != 0) ? MWB_W48_CH : MWB_W32_CH;
  const long long n_chunks = (window + ch - 1) / ch;
  const long long rows = (long long)n_scans * std::max<long long>(seg_batch_per_scan(n_sub), (long long)fine_tps * TILE);
  const long long bytes = rows * n_chunks * (long long)sizeof(float2);
  return (n_chunks > 1 && bytes <= (64LL << 20)) ? bytes : 0;
}

static long long seg_run_base_bytes(int n_scans, int n_sub, int fine_tps) {
  const long long per = seg_batch_per_scan(n_sub), n = per * n_scans;
  const long long ft = (long long)n_scans * fine_tps;
  return (long long)align_up(sizeof(SegState) * (size_t)n_scans, 256) + (long long)align_up(4 * n, 256) +
         (long long)align_up(4 * (n / TILE), 256) + (long long)align_up(8 * (n / TILE), 256) +
         (long long)align_up(4 * ft, 256) + (long long)align_up(8 * ft, 256);
}

int64_t mwb_segment_run_workspace_bytes(int n_scans, int n_sub, int fine_tps, int window) {
  if (n_scans < 1 || n_scans > 65535 || n_sub < 1 || n_sub > 64 || fine_tps < 0 || window < 0) return -1;
  return seg_run_base_bytes(n_scans, n_sub, fine_tps) + seg_run_part_bytes(n_scans, n_sub, fine_tps, window);
}

int mwb_segment_run(const void* plan, const float* sig, int n_scans, int64_t scan_stride, int n_chan, int ld,
                    int n_samples, const int32_t* chan_txrx, const double* ant_xyz, int n_ant, double inv_scale,
                    int interp, int k0, int window, int kind, int nx, int ny, int x0, int y0, int x1, int y1,
                    int n_sub, int stop_cells, int max_iters, int32_t* d_regions_out, float* lowres,
                    mwb_seg_trace_t* d_traces, float* out_fine, int64_t out_stride, uint64_t* keys,
                    int32_t* fine_counts, int32_t* flags, void* workspace, void* stream) {
  int rc = seg_tree_args(nx, ny, x0, y0, x1, y1, n_sub, stop_cells, max_iters, "mwb_segment_run");
  if (rc) return rc;
  if (n_scans < 1 || n_scans > 65535) return set_err(MWB_EINVAL, "mwb_segment_run: n_scans must be in [1, 65535]");
  if (kind != MWB_DAS && kind != MWB_DMAS) return set_err(MWB_EINVAL, "mwb_segment_run: bad kind");
  if (!plan || !d_regions_out || !d_traces || !out_fine || !workspace)
    return set_err(MWB_EINVAL, "mwb_segment_run: null pointer");
  if (out_stride < (int64_t)nx * ny) return set_err(MWB_EINVAL, "mwb_segment_run: out_stride < nx * ny");
  SegTree T;
  if ((rc = build_seg_tree(x0, y0, x1, y1, stop_cells, max_iters, T))) return rc;
  const long long per = seg_batch_per_scan(n_sub), n = per * n_scans;
  const int tps = (int)(per / TILE), lw = 4 * n_sub * n_sub;
  const long long ft = (long long)n_scans * T.fine_tps;
  if (n > 0x7FFFFFFFLL || ft * TILE > 0x7FFFFFFFLL) return set_err(MWB_ERANGE, "mwb_segment_run: batch too large");
  const SegPlanLayout L = seg_plan_layout(T, (int)per, n_chan);
  const unsigned char* pb = reinterpret_cast<const unsigned char*>(plan);
  const SegNode* nodes = reinterpret_cast<const SegNode*>(pb + L.nodes);
  unsigned char* ws = reinterpret_cast<unsigned char*>(workspace);
  SegState* st = reinterpret_cast<SegState*>(ws);
  ws += align_up(sizeof(SegState) * (size_t)n_scans, 256);
  float* e = reinterpret_cast<float*>(ws);
  ws += align_up(4 * n, 256);
  int* s_src = reinterpret_cast<int*>(ws);
  ws += align_up(4 * (n / TILE), 256);
  int2* s_info = reinterpret_cast<int2*>(ws);
  ws += align_up(8 * (n / TILE), 256);
  int* f_src = reinterpret_cast<int*>(ws);
  ws += align_up(4 * ft, 256);
  int2* f_info = reinterpret_cast<int2*>(ws);
  void* part = reinterpret_cast<unsigned char*>(workspace) + seg_run_base_bytes(n_scans, n_sub, T.fine_tps);
  const long long part_bytes = seg_run_part_bytes(n_scans, n_sub, T.fine_tps, window);
  cudaStream_t cs = reinterpret_cast<cudaStream_t>(stream);
  seg_tree_init_kernel<<<(n_scans + 255) / 256, 256, 0, cs>>>(st, n_scans, x0, y0, x1, y1, stop_cells, d_traces,
                                                               nodes, tps, lw, s_src, s_info);
  if ((rc = check_launch("seg_tree_init_kernel"))) return rc;
  const long long s_pts = (long long)T.search.size() * per;
  for (int it = 0; it < max_iters && s_pts > 0; ++it) {
    if ((rc = energies_impl(sig, n_scans, scan_stride, n_chan, ld, n_samples, chan_txrx, ant_xyz, n_ant, inv_scale,
                            reinterpret_cast<const double*>(pb + L.s_pts), nullptr, (int)n, nullptr,
                            reinterpret_cast<const int32_t*>(s_info), pb + L.s_table, interp, k0, window,
                            kind == MWB_DAS ? e : nullptr, kind == MWB_DMAS ? e : nullptr, 0, nullptr, nullptr,
                            nullptr, 0, stream, s_src, (int)s_pts, part_bytes ? part : nullptr, part_bytes)))
      return rc;
    seg_tree_score_kernel<<<n_scans, 256, 0, cs>>>(st, e, (int)per, n_sub, kind == MWB_DMAS, stop_cells, lowres,
                                                   d_traces, nodes, s_src, s_info);
    if ((rc = check_launch("seg_tree_score_kernel"))) return rc;
  }
  const RegionBatch b = region_batch(const_cast<unsigned char*>(pb) + L.r_ws, (int)T.term.size());
  seg_tree_fine_map_kernel<<<(unsigned)((ft + 255) / 256 + (ft == 0)), 256, 0, cs>>>(
      st, n_scans, nodes, b.scan_counts, b.scan_offsets, T.fine_tps, f_src, f_info, d_regions_out, fine_counts);
  if ((rc = check_launch("seg_tree_fine_map_kernel"))) return rc;
  if (ft == 0 || T.fine_bound == 0) return MWB_OK;
  return energies_impl(sig, n_scans, scan_stride, n_chan, ld, n_samples, chan_txrx, ant_xyz, n_ant, inv_scale,
                       reinterpret_cast<const double*>(pb + L.f_pts), reinterpret_cast<const int32_t*>(pb + L.f_idx),
                       (int)(ft * TILE), nullptr, reinterpret_cast<const int32_t*>(f_info), pb + L.f_table, interp,
                       k0, window, kind == MWB_DAS ? out_fine : nullptr, kind == MWB_DMAS ? out_fine : nullptr,
                       out_stride, kind == MWB_DAS ? keys : nullptr, kind == MWB_DMAS ? keys : nullptr, flags, 0,
                       stream, f_src, (int)T.fine_bound, part_bytes ? part : nullptr, part_bytes);
}

// One-call lattice image (beamform.py:283-342 as a single C entry point): the
// enumeration, delay table and fused energy launch of the Python `image()`
// path, with every buffer supplied by the caller.  Workspace layout:
// [points fp64 x3 | slots int32 | enumeration scratch | delay table].
static size_t lattice_points_max(int nx, int ny, int stride) {
  return (size_t)((nx + stride - 1) / stride) * (size_t)((ny + stride - 1) / stride);
}

int64_t mwb_image_lattice_workspace_bytes(int nx, int ny, int stride, int n_chan) {
  if (nx < 1 || ny < 1 || stride < 1 || n_chan < 1) return -1;
  const size_t pm = lattice_points_max(nx, ny, stride);
  if (pm > 0x7FFFFFFFu) return -1;
  const int64_t tb = mwb_delay_table_bytes((int)pm, n_chan);
  if (tb < 0) return -1;
  return (int64_t)(align_up(24 * pm, 256) + align_up(4 * pm, 256) +
                   align_up((size_t)mwb_lattice_workspace_bytes(nx, ny, stride), 256) + (size_t)tb);
}

int mwb_image_lattice(const float* sig, int n_chan, int ld, int n_samples, const int32_t* chan_txrx,
                      const double* ant_xyz, int n_ant, double inv_scale, int interp, int k0, int window,
                      double ox, double oy, double res, int nx, int ny, int x0, int y0, int x1, int y1,
                      int stride, const uint8_t* mask, int skip_stride, float* out_das, float* out_dmas,
                      uint8_t* valid, int32_t* d_count, uint64_t* key_das, uint64_t* key_dmas, int32_t* flags,
                      void* workspace, void* stream) {
  if (!out_das && !out_dmas) return set_err(MWB_EINVAL, "mwb_image_lattice: no output map");
  const int64_t need = mwb_image_lattice_workspace_bytes(nx, ny, stride, n_chan);
  if (need < 0) return set_err(MWB_EINVAL, "mwb_image_lattice: bad grid / stride / channels");
  if (!workspace) return set_err(MWB_EINVAL, "mwb_image_lattice: null workspace");
  const size_t pm = lattice_points_max(nx, ny, stride);
  unsigned char* ws = reinterpret_cast<unsigned char*>(workspace);
  double* pts = reinterpret_cast<double*>(ws);
  ws += align_up(24 * pm, 256);
  int32_t* slots = reinterpret_cast<int32_t*>(ws);
  ws += align_up(4 * pm, 256);
  void* scratch = ws;
  ws += align_up((size_t)mwb_lattice_workspace_bytes(nx, ny, stride), 256);
  void* table = ws;
  int rc = mwb_enumerate_lattice(ox, oy, res, nx, ny, x0, y0, x1, y1, nullptr, stride, mask, skip_stride, pts, slots,
                                 d_count, valid, scratch, stream);
  if (rc) return rc;
  if ((rc = mwb_delay_table(pts, (int)pm, d_count, chan_txrx, n_chan, ant_xyz, n_ant, inv_scale, interp, table,
                            stream)))
    return rc;
  return mwb_energies(sig, 1, 0, n_chan, ld, n_samples, chan_txrx, ant_xyz, n_ant, inv_scale, pts, slots, (int)pm,
                      d_count, table, interp, k0, window, out_das, out_dmas, 0, key_das, key_dmas, flags, 0, stream);
}

int mwb_argmax_dense(const float* dense, const uint8_t* valid, int n, uint64_t* key, void* stream) {
  if (n < 0 || !dense || !valid || !key) return set_err(MWB_EINVAL, "mwb_argmax_dense: bad arguments");
  if (n == 0) return MWB_OK;
  int blocks = (n + 255) / 256;
  if (blocks > 148 * 8) blocks = 148 * 8;
  argmax_dense_kernel<<<blocks, 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      dense, valid, n, reinterpret_cast<unsigned long long*>(key));
  return check_launch("argmax_dense_kernel");
}

int mwb_compact_payload(const double* payload, int m, int n, int ld, float* out, int32_t* pairs, int32_t* count,
                        int32_t* ws, void* stream) {
  if (m < 1 || m > 256 || n < 1 || ld < n) return set_err(MWB_EINVAL, "mwb_compact_payload: bad sizes");
  if (!payload || !out || !pairs || !count || !ws) return set_err(MWB_EINVAL, "mwb_compact_payload: null pointer");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  payload_flag_kernel<<<m * m, IO_THREADS, 0, st>>>(payload, n, ws);
  int rc = check_launch("payload_flag_kernel");
  if (rc) return rc;
  payload_rows_kernel<<<1, IO_THREADS, 0, st>>>(ws, m, pairs, count);
  if ((rc = check_launch("payload_rows_kernel"))) return rc;
  dim3 g((ld + IO_THREADS - 1) / IO_THREADS < 8 ? (ld + IO_THREADS - 1) / IO_THREADS : 8, m * m);
  payload_convert_kernel<<<g, IO_THREADS, 0, st>>>(payload, n, ld, ws, out);
  return check_launch("payload_convert_kernel");
}

int mwb_render_pgm(const void* values, int value_bits, const uint8_t* valid, int n_maps, int nx, int ny,
                   int64_t map_stride, int stride, double* vrange, uint8_t* raster, void* stream) {
  if (n_maps < 0 || nx < 1 || ny < 1 || stride < 1 || map_stride < (int64_t)nx * ny)
    return set_err(MWB_EINVAL, "mwb_render_pgm: bad sizes");
  if (value_bits != 32 && value_bits != 64) return set_err(MWB_EINVAL, "mwb_render_pgm: value_bits must be 32 or 64");
  if (!values || !valid || !vrange || !raster) return set_err(MWB_EINVAL, "mwb_render_pgm: null pointer");
  if (n_maps == 0) return MWB_OK;
  if (n_maps > 65535) return set_err(MWB_ERANGE, "mwb_render_pgm: too many maps");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const long long cells = (long long)nx * ny;
  long long blocks = (cells + IO_THREADS - 1) / IO_THREADS;
  dim3 g((unsigned)(blocks < 1024 ? blocks : 1024), n_maps);
  if (value_bits == 32) {
    render_range_kernel<float><<<n_maps, IO_THREADS, 0, st>>>(static_cast<const float*>(values), valid, cells,
                                                              map_stride, vrange);
    int rc = check_launch("render_range_kernel");
    if (rc) return rc;
    render_pgm_kernel<float><<<g, IO_THREADS, 0, st>>>(static_cast<const float*>(values), valid, nx, ny, map_stride,
                                                       stride, vrange, raster);
  } else {
    render_range_kernel<double><<<n_maps, IO_THREADS, 0, st>>>(static_cast<const double*>(values), valid, cells,
                                                               map_stride, vrange);
    int rc = check_launch("render_range_kernel");
    if (rc) return rc;
    render_pgm_kernel<double><<<g, IO_THREADS, 0, st>>>(static_cast<const double*>(values), valid, nx, ny,
                                                        map_stride, stride, vrange, raster);
  }
  return check_launch("render_pgm_kernel");
}

int mwb_gather_composite(const float* dense, int ny, int nz, const int32_t* coarse_slots, int n_coarse,
                         const int32_t* region, float* out, int64_t cap, void* stream) {
  if (!dense || ny < 1 || nz < 1 || n_coarse < 0 || (n_coarse && !coarse_slots) || !region || !out || cap < 0)
    return set_err(MWB_EINVAL, "mwb_gather_composite: bad arguments");
  gather_composite_kernel<<<64, IO_THREADS, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      dense, ny, nz, coarse_slots, n_coarse, region, out, cap);
  return check_launch("gather_composite_kernel");
}

int mwb_memcpy_async(void* dst, const void* src, int64_t bytes, void* stream) {
  if (bytes < 0 || (bytes && (!dst || !src))) return set_err(MWB_EINVAL, "mwb_memcpy_async: bad arguments");
  if (bytes == 0) return MWB_OK;
  const cudaError_t e = cudaMemcpyAsync(dst, src, (size_t)bytes, cudaMemcpyDefault,
                                        reinterpret_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? MWB_OK : set_err(MWB_ECUDA, "cudaMemcpyAsync: %s", cudaGetErrorString(e));
}

int mwb_stream_synchronize(void* stream) {
  const cudaError_t e = cudaStreamSynchronize(reinterpret_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? MWB_OK : set_err(MWB_ECUDA, "cudaStreamSynchronize: %s", cudaGetErrorString(e));
}

int mwb_memcpy2d_async(void* dst, int64_t dpitch, const void* src, int64_t spitch, int64_t width, int64_t height,
                       void* stream) {
  if (width < 0 || height < 0 || dpitch < width || spitch < width || ((width && height) && (!dst || !src)))
    return set_err(MWB_EINVAL, "mwb_memcpy2d_async: bad arguments");
  if (!width || !height) return MWB_OK;
  const cudaError_t e = cudaMemcpy2DAsync(dst, (size_t)dpitch, src, (size_t)spitch, (size_t)width, (size_t)height,
                                          cudaMemcpyDefault, reinterpret_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? MWB_OK : set_err(MWB_ECUDA, "cudaMemcpy2DAsync: %s", cudaGetErrorString(e));
}

int mwb_tc_plan_steps(const void* workspace, int n_scans, int n_chan, int j_count, int n_pts, int window,
                      int64_t* out_steps) {
  if (!workspace || !out_steps || n_scans < 1 || n_chan < 1 || j_count < 16 || n_pts < 1)
    return set_err(MWB_EINVAL, "mwb_tc_plan_steps: bad arguments");
  if (window != 32) return set_err(MWB_EINVAL, "mwb_tc_plan_steps: the step plan exists for window 32 only");
  const long long blocks = 2LL * ((n_pts + TILE - 1) / TILE);
  const unsigned char* pl = reinterpret_cast<const unsigned char*>(workspace) + tc_ws_absmax(n_scans) +
                            align_up(tc_ws_gram(n_scans, n_chan, j_count), 256) +
                            align_up(std::max(tc_ws_planes(n_scans, n_chan, j_count),
                                              tc_ws_planes8(n_scans, n_chan, j_count)), 256);
  std::vector<int> n((size_t)blocks);
  const cudaError_t e = cudaMemcpy(n.data(), pl, sizeof(int) * (size_t)blocks, cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) return set_err(MWB_ECUDA, "cudaMemcpy: %s", cudaGetErrorString(e));
  int64_t total = 0;
  for (int v : n) total += v;
  *out_steps = total;
  return MWB_OK;
}

int mwb_tc_sample_range(int k0, int j_lo, int j_count, int ld, int32_t* out) {
  if (!out || k0 < 0 || j_lo < 0 || j_count < 16 || ld < 1) return set_err(MWB_EINVAL, "mwb_tc_sample_range: bad arguments");
  const long long first = (long long)k0 + j_lo, len = tc_plane_len(j_count);
  out[0] = (int32_t)std::min<long long>(first, ld);
  out[1] = (int32_t)std::max<long long>(0, std::min<long long>(len, ld - first));
  return MWB_OK;
}

// Host-side compaction of a reference record (the drop-in's upload of a new
// dataset): the rows of an (rows, n) fp64 array that hold a nonzero sample
// (x != 0.0: -0.0 counts as zero, NaN as nonzero -- numpy's flat != 0.0 of
// _device.compact_channels), converted to fp32 rows of ld floats with a zero
// tail.  A row's scan stops at its first nonzero word; an all-zero record
// keeps row 0 (zeros).  Returns the row count, or a negative status.
int mwb_compact_rows_host(const double* src, int rows, int n, int ld, float* dst, int32_t* keep) {
  if (!src || !dst || !keep || rows < 1 || n < 0 || ld < n) return set_err(MWB_EINVAL, "mwb_compact_rows_host: bad arguments");
  int count = 0;
  for (int r = 0; r < rows; ++r) {
    const uint64_t* w = reinterpret_cast<const uint64_t*>(src + (size_t)r * n);
    bool nz = false;
    for (int i = 0; i < n && !nz; i += 64) {
      uint64_t acc = 0;
      const int e = std::min(n, i + 64);
      for (int k = i; k < e; ++k) acc |= w[k] << 1;  // drop the sign: -0.0 is zero
      nz = acc != 0;
    }
    if (!nz) continue;
    const double* x = src + (size_t)r * n;
    float* o = dst + (size_t)count * ld;
    for (int k = 0; k < n; ++k) o[k] = (float)x[k];
    for (int k = n; k < ld; ++k) o[k] = 0.f;
    keep[count++] = r;
  }
  if (count == 0) {
    for (int k = 0; k < ld; ++k) dst[k] = 0.f;
    keep[0] = 0;
    count = 1;
  }
  return count;
}

int mwb_elapsed_ms(void* const* events, int n_events, float* out_ms) {
  if (n_events < 2 || !events || !out_ms) return set_err(MWB_EINVAL, "mwb_elapsed_ms: bad arguments");
  for (int i = 0; i + 1 < n_events; ++i) {
    const cudaError_t e = cudaEventElapsedTime(out_ms + i, reinterpret_cast<cudaEvent_t>(events[i]),
                                               reinterpret_cast<cudaEvent_t>(events[i + 1]));
    if (e != cudaSuccess) return set_err(MWB_ECUDA, "cudaEventElapsedTime: %s", cudaGetErrorString(e));
  }
  return MWB_OK;
}

int mwb_microbench(int which, double* work, float* ms, void* stream) {
  if (!work || !ms) return set_err(MWB_EINVAL, "mwb_microbench: null pointer");
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  float* sink = nullptr;
  if (cudaMalloc(&sink, 1024 * sizeof(float)) != cudaSuccess) return set_err(MWB_ECUDA, "cudaMalloc failed");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int blocks = sms * 2, threads = 1024;
  for (int rep = 0; rep < 2; ++rep) {  // first launch warms up
    cudaEventRecord(a, st);
    if (which == 0) mb_lds_kernel<<<blocks, threads, 0, st>>>(sink, 7);
    else if (which == 1) mb_ffma2_kernel<<<blocks, threads, 0, st>>>(sink, 0.5f);
    else if (which == 2) mb_ffma_kernel<<<blocks, threads, 0, st>>>(sink, 0.5f);
    else if (which >= 100 && which < 110) mb_lds_pattern_kernel<1><<<blocks, threads, 0, st>>>(sink, which - 100);
    else if (which >= 110 && which < 120) mb_lds_pattern_kernel<2><<<blocks, threads, 0, st>>>(sink, which - 110);
    else mb_lds_pattern_kernel<4><<<blocks, threads, 0, st>>>(sink, which - 120);
    cudaEventRecord(b, st);
  }
  cudaEventSynchronize(b);
  cudaEventElapsedTime(ms, a, b);
  const double thr = (double)blocks * threads * MB_ITERS;
  if (which == 0) *work = thr * 32 * 4.0;           // bytes loaded from shared memory
  else if (which == 1) *work = thr * 8 * 2 * 2.0;   // 8 FFMA2 = 16 FMA = 32 flop
  else if (which == 2) *work = thr * 16 * 2.0;
  else {  // bytes delivered to registers by the pattern probe
    const int words = which < 110 ? 1 : (which < 120 ? 2 : 4);
    *work = (double)blocks * threads * (MB_ITERS / 4) * 16 * 4.0 * words;
  }
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  cudaFree(sink);
  return check_launch("microbench");
}

}  // extern "C"
