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

constexpr int TPB = 128;          // threads per energy CTA
constexpr int TILE = 2 * TPB;     // focal points per CTA
#ifndef MWB_W48_MINB
#define MWB_W48_MINB 3  // CTAs per SM of the W = 48 kernel: 3 (<= 168 registers, one channel in flight) beat 2
                        // (255 registers, two channels): 7.9 vs 8.4 ms on the configs[4] volume
#endif
#ifndef MWB_W48_CH
#define MWB_W48_CH 48  // register chunk for W % 48 == 0 windows (experiment knob: 24)
#endif
constexpr int MAX_ANT = 64;
constexpr int MAX_CHAN = 4096;
constexpr int CAP_MAX = 8192;     // floats per stage buffer (32 KB)
constexpr int NSTAGE = 3;         // stage-buffer ring depth (full/empty mbarrier pairs)

// Debug builds (-DMWB_DEBUG_BOUNDS, libmwb_debug.so) trap on any shared-memory
// staging index outside its buffer; compute-sanitizer is not available on the
// GPU pool, so this is the bounds check the parity suite runs against.
#ifdef MWB_DEBUG_BOUNDS
#define MWB_CHECK(cond) \
  do {                  \
    if (!(cond)) __trap(); \
  } while (0)
#else
#define MWB_CHECK(cond) \
  do {                  \
  } while (0)
#endif

thread_local char g_err[512] = "";

int set_err(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return code;
}

int check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    snprintf(g_err, sizeof(g_err), "%s: %s", what, cudaGetErrorString(e));
    return MWB_ECUDA;
  }
  return MWB_OK;
}

// ----------------------------------------------------------------------------
// small PTX helpers (mbarrier + 1-D bulk copy)
// ----------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
}

__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t done = 0;
  const uint32_t addr = smem_u32(bar);
  while (!done) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(addr), "r"(parity)
        : "memory");
  }
}

// Bulk prefetch of [src, src + bytes) into L2 (16-byte aligned, multiple of 16).
__device__ __forceinline__ void bulk_prefetch_l2(const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// ----------------------------------------------------------------------------
// numerics shared by every path (lattice, point list, batched, 3-D)
// ----------------------------------------------------------------------------

// |p - a| exactly as numpy evaluates sqrt(dx*dx + dy*dy + dz*dz)
// (beamform.py:182-185): no FMA contraction, IEEE sqrt.
__device__ __forceinline__ double antenna_distance(double px, double py, double pz, double ax,
                                                   double ay, double az) {
  const double dx = __dsub_rn(px, ax);
  const double dy = __dsub_rn(py, ay);
  const double dz = __dsub_rn(pz, az);
  const double s = __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
  return __dsqrt_rn(s);
}

// Split a fractional delay (samples) into i0 = floor(n) and a 23-bit fixed-point
// fraction (beamform.py:186-190; nearest -> rint, 187-188).  The weights used by
// every path are f1 = q * 2^-23, f0 = 1 - f1 (both exact in fp32, f0 + f1 == 1),
// a function of the point alone, so a point's energy never depends on the tile.
//
// One conversion does both: n * 2^23 is exact (power-of-two scaling, n <= 2^30),
// so v = floor(n * 2^23) = floor(n) * 2^23 + trunc((n - floor n) * 2^23), i.e.
// i0 = v >> 23 and fq = v & (2^23 - 1), bit-identical to the two-step split.
// (The delay-table kernel evaluates ~10^9 of these per 128^3 volume; this form
// drops its FRND, one F2I and a DADD per word.)
__device__ __forceinline__ void split_delay_q(double n, int interp, int& i0, uint32_t& fq) {
  if (interp == MWB_INTERP_NEAREST) n = rint(n);
  // clamp to [0, 2^30] with NaN -> 0 (a failed compare selects the bound):
  // the same result as fmin(fmax(n, 0), 2^30) without fmax's NaN fix-up code
  n = n >= 0.0 ? n : 0.0;
  n = n <= 1073741824.0 ? n : 1073741824.0;
  const long long v = __double2ll_rd(__dmul_rn(n, 8388608.0));
  i0 = static_cast<int>(v >> 23);
  fq = static_cast<uint32_t>(v) & 0x7FFFFFu;
}

__device__ __forceinline__ float weight_f1(uint32_t fq) {
  return __fsub_rn(__uint_as_float(0x3F800000u | (fq & 0x7FFFFFu)), 1.0f);
}

// per-point per-channel delay in samples: (d_tx + d_rx) / (v dt)  (beamform.py:186)
__device__ __forceinline__ double pair_delay(double dtx, double drx, double inv_scale) {
  return __dmul_rn(__dadd_rn(dtx, drx), inv_scale);
}

__device__ __forceinline__ uint32_t ordered_f32(float v) {
  uint32_t u = __float_as_uint(v);
  if (v == 0.0f) u = 0u;  // -0.0 == +0.0 (Python compares values)
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

__device__ __forceinline__ uint64_t argmax_key(float v, int slot) {
  return (static_cast<uint64_t>(ordered_f32(v)) << 32) |
         static_cast<uint64_t>(0xFFFFFFFFu - static_cast<uint32_t>(slot));
}

constexpr int KIND_DAS = 0, KIND_DMAS = 1, KIND_BOTH = 2;

// Accumulate one channel into the register window of two points (float2 lanes):
//   a = f0*y[k] + f1*y[k+1];  s += a            (beamform.py:207-208; DAS 203-205)
//   q += a*a                                    (DMAS only, beamform.py:209)
// DAS and DMAS share s, so one pass yields both energies.
template <int KIND, bool TAIL, int CH, class Load>
__device__ __forceinline__ void accumulate_channel(float2 (&s)[CH], float2& qe, float2& qo,
                                                   const float2 f0, const float2 f1,
                                                   const Load& load, const int valid) {
  static_assert(CH % 4 == 0, "chunk starts must keep the 16-byte span alignment phase");
  float2 prev = load(0);
#pragma unroll
  for (int k = 0; k < CH; ++k) {
    const float2 nxt = load(k + 1);
    float2 a = __fmul2_rn(f0, prev);
    a = __ffma2_rn(f1, nxt, a);
    s[k] = __fadd2_rn(s[k], a);
    if (KIND != KIND_DAS && (!TAIL || k < valid)) {
#ifdef MWB_ONE_Q
      qe = __ffma2_rn(a, a, qe);
#else
      if (k & 1)
        qo = __ffma2_rn(a, a, qo);
      else
        qe = __ffma2_rn(a, a, qe);
#endif
    }
    prev = nxt;
  }
}

// Chunk epilogue: S = Σ_k s_k^2 (fp32, fixed order) and Q = Σ q (DMAS);
// DAS energy = Σ S, DMAS energy = ½ Σ (S − Q), summed over chunks in fp64
// (beamform.py:210-212).
template <int CH>
__device__ __forceinline__ float2 chunk_sumsq(const float2 (&s)[CH], const int valid) {
  float2 acc = make_float2(0.f, 0.f);
#pragma unroll
  for (int k = 0; k < CH; ++k)
    if (k < valid) acc = __ffma2_rn(s[k], s[k], acc);
  return acc;
}

struct EnergyParams {
  const float* sig;
  long long scan_stride;
  int n_scans;
  int C;
  int ld;
  int N;
  const int* chan;
  const double* ant;
  int M;
  double inv_scale;
  const double* pts;
  const int* out_idx;
  int P;
  const int* d_count;
  const int2* tile_info;      // packed multi-scan lists: {scan, valid points} per tile, or NULL
  const int* tile_src;        // with tile_info: source tile of the point list / table per launched tile, or NULL
  const uint32_t* tab_words;  // [tiles][C][TILE]
  const int2* tab_span;       // [tiles][C] {lo, hi}
  const int* tab_wide;        // [tiles]
  int interp;
  int k0;
  int W;
  float* out_das;
  float* out_dmas;
  long long out_stride;
  unsigned long long* key_das;
  unsigned long long* key_dmas;
  int* flags;
  int mode;
  int scans_per_cta;
  int cap;  // floats per stage buffer
  // window split across CTAs (blockIdx.z takes chunks [z*chunks_per_cta, ...)):
  // each chunk's per-point {S, Q} go to part[(s * P + point) * n_chunks + q]
  // and energy_reduce_kernel sums them in chunk order, as the unsplit kernel does
  float2* part;
  int chunks_per_cta;
};

struct SmemLayout {
  size_t lo, alloc, off, sb, misc, mbar, stage, total;
};

__host__ __device__ inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

__host__ __device__ inline SmemLayout smem_layout(int C, int cap) {
  SmemLayout L;
  size_t o = 0;
  L.lo = o;      o += sizeof(int) * (size_t)C;
  L.alloc = o;   o += sizeof(int) * (size_t)C;
  L.off = o;     o += sizeof(int) * (size_t)C;
  L.sb = o;      o += sizeof(int) * (size_t)C;
  L.misc = o;    o += sizeof(int) * 16;
  o = align_up(o, 16);
  L.mbar = o;    o += sizeof(uint64_t) * 2 * NSTAGE;
  o = align_up(o, 128);
  L.stage = o;   o += sizeof(float) * NSTAGE * (size_t)cap;
  L.total = o;
  return L;
}

// table layout inside one workspace buffer
struct TableLayout {
  size_t words, span, wide, total;
};

__host__ __device__ inline TableLayout table_layout(long long tiles, int C) {
  TableLayout T;
  size_t o = 0;
  T.words = o; o += sizeof(uint32_t) * (size_t)tiles * C * TILE;
  o = align_up(o, 16);
  T.span = o;  o += sizeof(int2) * (size_t)tiles * C;
  o = align_up(o, 16);
  T.wide = o;  o += sizeof(int) * (size_t)tiles;
  T.total = align_up(o, 256);
  return T;
}

constexpr int SPAN_BITS = 9;                       // i0 - lo_c stored in 9 bits
constexpr int SPAN_MAX = (1 << SPAN_BITS) - 1;

// ----------------------------------------------------------------------------
// K0: per point-list delay table (computed once, reused by every scan)
//   word(p, c) = (i0 - lo_c) << 23 | frac23,  span(c) = {lo_c, hi_c} per tile
// ----------------------------------------------------------------------------
struct TableParams {
  const double* pts;
  int P;
  const int* d_count;
  const int* chan;
  int C;
  const double* ant;
  int M;
  double inv_scale;
  int interp;
  uint32_t* words;
  int2* span;
  int* wide;
  const int2* tile_info;  // packed multi-scan lists: {scan, valid points} per tile, or NULL
};

// Word loop of delay_table_kernel for one thread's two points (da, da + TPB).
// ~10^9 words per 128^3 volume and the loop is issue-bound, so: channel
// offsets come pre-scaled to bytes from shared memory, the output pointer
// advances one tile row per channel (no per-word index arithmetic), the
// interpolation mode is a template parameter (no if-converted rint on the
// linear path), and four channels per thread in flight hide fp64 latency.
//
// Linear words skip split_delay_q's [0, 2^30] clamp: this loop only runs for
// non-wide tiles, where every finite point's i0 lies in the tile's span
// [lo, hi] (within [0, 2^30]); a NaN point converts to 0 or INT64_MIN, either
// way i0 = 0, fq = 0, as after the clamp.  q = floor(n 2^23) comes from one
// DMUL by inv_scale * 2^23 (power-of-two scaling commutes with rounding).
template <bool NEAREST>
__device__ __forceinline__ void table_words(uint32_t* wp, const unsigned char* da, const int2* coff, const int* lo,
                                            int C, double inv_scale) {
  const int interp = NEAREST ? MWB_INTERP_NEAREST : MWB_INTERP_LINEAR;
  if (!NEAREST) {
    const double inv23 = __dmul_rn(inv_scale, 8388608.0);
#pragma unroll 4
    for (int c = 0; c < C; ++c, wp += TILE) {
      const int2 o = coff[c];
      const double* ta = reinterpret_cast<const double*>(da + o.x);
      const double* ra = reinterpret_cast<const double*>(da + o.y);
      const long long va = __double2ll_rd(__dmul_rn(__dadd_rn(ta[0], ra[0]), inv23));
      const long long vb = __double2ll_rd(__dmul_rn(__dadd_rn(ta[TPB], ra[TPB]), inv23));
      const int l = lo[c];
      const int ia = static_cast<int>(va >> 23), ib = static_cast<int>(vb >> 23);
      wp[0] = ((uint32_t)min(max(ia - l, 0), SPAN_MAX) << 23) | (static_cast<uint32_t>(va) & 0x7FFFFFu);
      wp[TPB] = ((uint32_t)min(max(ib - l, 0), SPAN_MAX) << 23) | (static_cast<uint32_t>(vb) & 0x7FFFFFu);
    }
    return;
  }
#pragma unroll 4
  for (int c = 0; c < C; ++c, wp += TILE) {
    const int2 o = coff[c];
    const double* ta = reinterpret_cast<const double*>(da + o.x);
    const double* ra = reinterpret_cast<const double*>(da + o.y);
    int ia, ib;
    uint32_t qa, qb;
    split_delay_q(pair_delay(ta[0], ra[0], inv_scale), interp, ia, qa);
    split_delay_q(pair_delay(ta[TPB], ra[TPB], inv_scale), interp, ib, qb);
    const int l = lo[c];
    wp[0] = ((uint32_t)min(max(ia - l, 0), SPAN_MAX) << 23) | qa;
    wp[TPB] = ((uint32_t)min(max(ib - l, 0), SPAN_MAX) << 23) | qb;
  }
}

__global__ void __launch_bounds__(TPB) delay_table_kernel(const TableParams p) {
  extern __shared__ __align__(128) unsigned char smem[];
  double* dist = reinterpret_cast<double*>(smem);                 // [M][TILE]
  double* amin = dist + (size_t)p.M * TILE;                      // [M]
  double* amax = amin + p.M;                                     // [M]
  int* lo = reinterpret_cast<int*>(amax + p.M);                  // [C]
  int* hi = lo + p.C;                                            // [C]
  int* wide = hi + p.C;
  int2* coff = reinterpret_cast<int2*>(wide + 2);                // [C] {tx, rx} row offsets in bytes
  const int tid = threadIdx.x;
  const int n_pts = p.d_count ? min(*p.d_count, p.P) : p.P;
  const int tile0 = blockIdx.x * TILE;
  if (tile0 >= n_pts) return;
  const int n_in = p.tile_info ? p.tile_info[blockIdx.x].y : min(TILE, n_pts - tile0);
  if (n_in <= 0) {  // empty padded tile: a zero span, no words
    for (int c = tid; c < p.C; c += TPB) p.span[(size_t)blockIdx.x * p.C + c] = make_int2(0, 0);
    if (tid == 0) p.wide[blockIdx.x] = 0;
    return;
  }
  const int la = tid, lb = tid + TPB;
  const int ga = tile0 + (la < n_in ? la : 0), gb = tile0 + (lb < n_in ? lb : 0);
  const double pax = p.pts[3 * (size_t)ga], pay = p.pts[3 * (size_t)ga + 1], paz = p.pts[3 * (size_t)ga + 2];
  const double pbx = p.pts[3 * (size_t)gb], pby = p.pts[3 * (size_t)gb + 1], pbz = p.pts[3 * (size_t)gb + 2];
  for (int i = 0; i < p.M; ++i) {
    const double ax = __ldg(p.ant + 3 * i), ay = __ldg(p.ant + 3 * i + 1), az = __ldg(p.ant + 3 * i + 2);
    dist[i * TILE + la] = antenna_distance(pax, pay, paz, ax, ay, az);
    dist[i * TILE + lb] = antenna_distance(pbx, pby, pbz, ax, ay, az);
  }
  for (int c = tid; c < p.C; c += TPB) {
    lo[c] = 0x7FFFFFFF;
    hi[c] = -1;
    coff[c] = make_int2(__ldg(p.chan + 2 * c) * TILE * (int)sizeof(double),
                        __ldg(p.chan + 2 * c + 1) * TILE * (int)sizeof(double));
  }
  if (tid == 0) *wide = 0;
  __syncthreads();
  // per-channel i0 range from per-antenna distance bounds over the tile's
  // points: fl(+), fl(*), floor and rint are monotone, so every point's i0 for
  // channel (tx, rx) lies in [i0(dmin_tx + dmin_rx), i0(dmax_tx + dmax_rx)]
  const int lane = tid & 31, warp = tid >> 5;
  for (int i = warp; i < p.M; i += TPB / 32) {
    double mn = INFINITY, mx = -INFINITY;
    for (int j = lane; j < n_in; j += 32) {
      const double d = dist[i * TILE + j];
      mn = fmin(mn, d);
      mx = fmax(mx, d);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
      mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    }
    if (lane == 0) {
      amin[i] = mn;
      amax[i] = mx;
    }
  }
  __syncthreads();
  for (int c = tid; c < p.C; c += TPB) {
    const int tx = __ldg(p.chan + 2 * c), rx = __ldg(p.chan + 2 * c + 1);
    uint32_t q;
    split_delay_q(pair_delay(amin[tx], amin[rx], p.inv_scale), p.interp, lo[c], q);
    split_delay_q(pair_delay(amax[tx], amax[rx], p.inv_scale), p.interp, hi[c], q);
  }
  __syncthreads();
  const size_t tile = blockIdx.x;
  for (int c = tid; c < p.C; c += TPB) {
    p.span[tile * p.C + c] = make_int2(lo[c], hi[c]);
    if (hi[c] - lo[c] > SPAN_MAX) atomicOr(wide, 1);
  }
  __syncthreads();
  if (tid == 0) p.wide[tile] = *wide;
  if (*wide) return;  // wide tiles are evaluated from the points directly
  uint32_t* wp = p.words + tile * (size_t)p.C * TILE + la;
  if (p.interp == MWB_INTERP_NEAREST)
    table_words<true>(wp, reinterpret_cast<const unsigned char*>(dist + la), coff, lo, p.C, p.inv_scale);
  else
    table_words<false>(wp, reinterpret_cast<const unsigned char*>(dist + la), coff, lo, p.C, p.inv_scale);
}

#ifndef MWB_CH_UNROLL
#define MWB_CH_UNROLL 2  // two channels in flight per warp: +3.4% on configs[3] (scripts/variants.sh)
#endif
constexpr int kChannelUnroll = MWB_CH_UNROLL;  // channel-loop unroll (experiment knob)

// (1 + f1) as fp32 bits in one LOP3: (w & 0x7FFFFF) | 0x3F800000
__device__ __forceinline__ float one_plus_f1(uint32_t w) {
  uint32_t r;
  asm("lop3.b32 %0, %1, 0x7FFFFF, %2, 0xEA;" : "=r"(r) : "r"(w), "r"(0x3F800000u));
  return __uint_as_float(r);
}

// Channels [c_begin, c_end) of one step on the smem-staged samples.  The delay
// words of the next channel are fetched while the current one is processed.
template <int KIND, bool TAIL, int CH>
__device__ __forceinline__ void channel_loop(float2 (&sacc)[CH], float2& qe, float2& qo,
                                             const uint32_t* __restrict__ tw, const int* sb,
                                             const float* buf, int c_begin, int c_end, int la, int lb,
                                             int valid, int cap) {
  const uint32_t* wp = tw + (size_t)c_begin * TILE;
  uint32_t wa = __ldg(wp + la), wb = __ldg(wp + lb);
#ifdef MWB_PREFETCH2
  uint32_t wa2 = 0, wb2 = 0;
  if (c_begin + 1 < c_end) {
    wa2 = __ldg(wp + TILE + la);
    wb2 = __ldg(wp + TILE + lb);
  }
#endif
  // two channels in flight for 32-sample chunks; one for 48 (keeps the W = 48
  // kernel within the 168 registers of 3 CTAs per SM)
  constexpr int kUnroll = CH == 48 ? 1 : kChannelUnroll;
#pragma unroll kUnroll
  for (int c = c_begin; c < c_end; ++c) {
    const uint32_t ca = wa, cw = wb;
    wp += TILE;
#ifdef MWB_PREFETCH2
    wa = wa2;
    wb = wb2;
    if (c + 2 < c_end) {
      wa2 = __ldg(wp + TILE + la);
      wb2 = __ldg(wp + TILE + lb);
    }
#else
    if (c + 1 < c_end) {
      wa = __ldg(wp + la);
      wb = __ldg(wp + lb);
    }
#endif
    const float2 f1 = __fadd2_rn(make_float2(one_plus_f1(ca), one_plus_f1(cw)), make_float2(-1.f, -1.f));
    const float2 f0 = __ffma2_rn(f1, make_float2(-1.f, -1.f), make_float2(1.f, 1.f));
    const float* base = buf + sb[c];
    MWB_CHECK(sb[c] >= 0 && sb[c] + (int)(ca >> 23) + CH < cap && sb[c] + (int)(cw >> 23) + CH < cap);
    const float* ya = base + (ca >> 23);
    const float* yb = base + (cw >> 23);
    auto load = [&](int k) { return make_float2(ya[k], yb[k]); };
    accumulate_channel<KIND, TAIL, CH>(sacc, qe, qo, f0, f1, load, valid);
  }
}

// ----------------------------------------------------------------------------
// K1: staged fractional gather + fused DAS/DMAS window accumulation
// ----------------------------------------------------------------------------
template <int KIND, int MINB, int CH>
__global__ void __launch_bounds__(TPB, MINB) energy_kernel(const EnergyParams p) {
  extern __shared__ __align__(128) unsigned char smem[];
  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int warp = tid >> 5;

  const int n_pts = p.d_count ? min(*p.d_count, p.P) : p.P;
  const int tile0 = blockIdx.x * TILE;
  if (tile0 >= n_pts) return;
  int n_in_tile = min(TILE, n_pts - tile0);
  int scan_begin = blockIdx.y * p.scans_per_cta;
  int n_my_scans = min(p.scans_per_cta, p.n_scans - scan_begin);
  if (p.tile_info) {  // each tile belongs to one scan (per-scan point lists, packed)
    const int2 ti = p.tile_info[blockIdx.x];
    scan_begin = ti.x;
    n_in_tile = ti.y;
    n_my_scans = 1;
    if (n_in_tile <= 0 || scan_begin < 0) return;
  }
  if (scan_begin >= p.n_scans) return;

  const SmemLayout L = smem_layout(p.C, p.cap);
  int* clo = reinterpret_cast<int*>(smem + L.lo);
  int* calloc_ = reinterpret_cast<int*>(smem + L.alloc);
  int* coff = reinterpret_cast<int*>(smem + L.off);
  int* sb = reinterpret_cast<int*>(smem + L.sb);
  int* misc = reinterpret_cast<int*>(smem + L.misc);
  uint64_t* mbar = reinterpret_cast<uint64_t*>(smem + L.mbar);
  float* stage = reinterpret_cast<float*>(smem + L.stage);

  // source tile of the points / table (a shared, precomputed list) and the
  // packed output position; the same tile unless tile_src remaps it
  const size_t tile = p.tile_src ? (size_t)__ldg(p.tile_src + blockIdx.x) : (size_t)blockIdx.x;
  const bool wide = __ldg(p.tab_wide + tile) != 0;
  const uint32_t* tw = p.tab_words + tile * (size_t)p.C * TILE;
  const int2* tsp = p.tab_span + tile * (size_t)p.C;

  const int la = tid, lb = tid + TPB;
  const bool va = la < n_in_tile, vb = lb < n_in_tile;
  // (source point indices are re-derived in the gather path below: keeping
  // them live across the sample loop costs the register-capped kernels spills)
  const int oa = va ? (p.out_idx ? __ldg(p.out_idx + (int)tile * TILE + la) : tile0 + la) : -1;
  const int ob = vb ? (p.out_idx ? __ldg(p.out_idx + (int)tile * TILE + lb) : tile0 + lb) : -1;

  // ---- per-channel spans and stage-buffer groups --------------------------
  for (int c = tid; c < p.C; c += TPB) {
    const int2 sp = __ldg(tsp + c);
    clo[c] = sp.x;
    // samples k0+q*CH + [lo, hi+CH] plus up to 3 of alignment slack
    calloc_[c] = (sp.y - sp.x + CH + 8 + 3) & ~3;
  }
  if (tid == 0) {
    for (int b = 0; b < NSTAGE; ++b) {
      mbar_init(&mbar[b], 32);                  // full: the 32 lanes of the producer warp
      mbar_init(&mbar[NSTAGE + b], TPB / 32);   // empty: one arrival per consumer warp
    }
    fence_mbar_init();
  }
  __syncthreads();
  if (warp == 0) {
    // largest span -> channels per stage group; then per-group offsets from a
    // warp-wide exclusive prefix sum of the spans (32 channels per round)
    int mx = 0;
    for (int c = lane; c < p.C; c += 32) mx = max(mx, calloc_[c]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    int G = (!wide && p.mode == 0 && mx <= p.cap) ? p.cap / mx : 0;
    if (G > p.C) G = p.C;
    int carry = 0;
    for (int base = 0; base < p.C; base += 32) {
      const int c = base + lane;
      const int v = c < p.C ? calloc_[c] : 0;
      int x = v;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
      }
      if (c < p.C) coff[c] = carry + x - v;  // global exclusive prefix
      carry += __shfl_sync(0xffffffffu, x, 31);
    }
    __syncwarp();
    if (G > 0)
      for (int c = lane; c < p.C; c += 32) sb[c] = coff[(c / G) * G];
    __syncwarp();
    if (G > 0)
      for (int c = lane; c < p.C; c += 32) coff[c] -= sb[c];  // offset within the group
    if (lane == 0) {
      misc[0] = G;
      misc[1] = G > 0 ? (p.C + G - 1) / G : 0;
    }
  }
  __syncthreads();
  // smem slot of sample (k0 + q*CH + lo_c) in channel c's span: the same for
  // every chunk q because CH % 4 == 0
  for (int c = tid; c < p.C; c += TPB) sb[c] = coff[c] + ((p.k0 + clo[c]) & 3);
  __syncthreads();
  const int G = misc[0];
  const int n_groups = misc[1];
  const int n_chunks = (p.W + CH - 1) / CH;
  const int q_begin = p.part ? (int)blockIdx.z * p.chunks_per_cta : 0;
  const int n_local = p.part ? min(p.chunks_per_cta, n_chunks - q_begin) : n_chunks;

  // Producer (warp 0, all lanes): stage step t into ring slot t % NSTAGE once
  // the consumers released the slot's previous use.  Zero-fills (spans past
  // the record) are written before the lanes' arrivals on the full barrier,
  // whose release/acquire makes them visible with the TMA bytes.
  auto issue = [&](int t) {
    const int b = t % NSTAGE, use = t / NSTAGE;
    if (use > 0) mbar_wait(&mbar[NSTAGE + b], (use - 1) & 1);
    const int g = t % n_groups;
    const int r = t / n_groups;
    const int q = q_begin + r % n_local;
    const int s = scan_begin + r / n_local;
    const int c_begin = g * G, c_end = min(p.C, c_begin + G);
    float* buf = stage + b * p.cap;
    const float* scan_sig = p.sig + (size_t)s * (size_t)p.scan_stride;
    const int cb = p.k0 + q * CH;
    uint32_t bytes_lane = 0;
    for (int c = c_begin + lane; c < c_end; c += 32) {
      const long long start4 = ((long long)cb + clo[c]) & ~3LL;
      const int alloc = calloc_[c];
      const long long n = min((long long)alloc, max((long long)p.ld - start4, 0LL));
      bytes_lane += (uint32_t)(n * 4);
      float* dst = buf + coff[c];
      MWB_CHECK(coff[c] >= 0 && coff[c] + alloc <= p.cap);
      for (long long j = max(n, 0LL); j < alloc; ++j) dst[j] = 0.f;  // past the record: zeros
    }
    uint32_t bytes = bytes_lane;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) bytes += __shfl_xor_sync(0xffffffffu, bytes, o);
    if (lane == 0)
      mbar_arrive_expect_tx(&mbar[b], bytes);
    else
      mbar_arrive(&mbar[b]);
    __syncwarp();
    for (int c = c_begin + lane; c < c_end; c += 32) {
      const long long start4 = ((long long)cb + clo[c]) & ~3LL;
      const long long n = min((long long)calloc_[c], max((long long)p.ld - start4, 0LL));
      if (n > 0)
        bulk_g2s(buf + coff[c], scan_sig + (size_t)c * p.ld + start4, (uint32_t)(n * 4), &mbar[b]);
    }
    // The group's delay words ([c_begin, c_end) x TILE, contiguous) are read
    // by every consumer thread NSTAGE - 1 steps from now.  A table larger than
    // L2 (a 128^3 volume: 4.2 GB) would put DRAM latency on each channel's
    // word load, so each chunk's first use of a group pulls its block into L2
    // here (later scans of a multi-scan CTA find it there).
    if (r < n_local && lane == 0) bulk_prefetch_l2(tw + (size_t)c_begin * TILE, (uint32_t)(c_end - c_begin) * TILE * 4u);
  };

  const int nsteps = (n_groups > 0 ? n_groups : 1) * n_local * n_my_scans;

  float2 sacc[CH];
  float2 qe = make_float2(0.f, 0.f), qo = make_float2(0.f, 0.f);
  double eS_a = 0.0, eS_b = 0.0, eQ_a = 0.0, eQ_b = 0.0;

  if (G > 0 && warp == 0)
    for (int t = 0; t < NSTAGE - 1 && t < nsteps; ++t) issue(t);

  for (int t = 0; t < nsteps; ++t) {
    const int g = G > 0 ? t % n_groups : 0;
    const int r = G > 0 ? t / n_groups : t;
    const int q = q_begin + r % n_local;
    const int s = scan_begin + r / n_local;
    const int valid = min(CH, p.W - q * CH);
    const int cb = p.k0 + q * CH;

    if (G > 0) mbar_wait(&mbar[t % NSTAGE], (t / NSTAGE) & 1);
    if (g == 0) {
#pragma unroll
      for (int k = 0; k < CH; ++k) sacc[k] = make_float2(0.f, 0.f);
      qe = make_float2(0.f, 0.f);
      qo = make_float2(0.f, 0.f);
    }
    const int c_begin = G > 0 ? g * G : 0;
    const int c_end = G > 0 ? min(p.C, c_begin + G) : p.C;
    const float* buf = stage + (t % NSTAGE) * p.cap;
    const float* scan_sig = p.sig + (size_t)s * (size_t)p.scan_stride;

    if (G > 0) {
      // fast path: packed delay words (L2-resident table), samples from smem
      if (valid == CH)
        channel_loop<KIND, false, CH>(sacc, qe, qo, tw, sb, buf, c_begin, c_end, la, lb, valid, p.cap);
      else
        channel_loop<KIND, true, CH>(sacc, qe, qo, tw, sb, buf, c_begin, c_end, la, lb, valid, p.cap);
    } else {
      // L1/L2 gather path (mode 1 or a tile whose delay spread exceeds the table):
      // same weights, loads straight from global with a zero tail.
      const int src0 = (p.tile_src ? __ldg(p.tile_src + blockIdx.x) : (int)blockIdx.x) * TILE;
      const int ga = src0 + (va ? la : 0), gb = src0 + (vb ? lb : 0);
      const double pax = p.pts[3 * (size_t)ga], pay = p.pts[3 * (size_t)ga + 1], paz = p.pts[3 * (size_t)ga + 2];
      const double pbx = p.pts[3 * (size_t)gb], pby = p.pts[3 * (size_t)gb + 1], pbz = p.pts[3 * (size_t)gb + 2];
      for (int c = 0; c < p.C; ++c) {
        int ia, ib;
        uint32_t qa, qb;
        if (!wide) {
          const uint32_t wa = __ldg(tw + (size_t)c * TILE + la), wb = __ldg(tw + (size_t)c * TILE + lb);
          const int l = clo[c];
          ia = l + (int)(wa >> 23);
          ib = l + (int)(wb >> 23);
          qa = wa;
          qb = wb;
        } else {
          const int tx = __ldg(p.chan + 2 * c), rx = __ldg(p.chan + 2 * c + 1);
          const double* at = p.ant + 3 * tx;
          const double* ar = p.ant + 3 * rx;
          split_delay_q(pair_delay(antenna_distance(pax, pay, paz, at[0], at[1], at[2]),
                                   antenna_distance(pax, pay, paz, ar[0], ar[1], ar[2]), p.inv_scale),
                        p.interp, ia, qa);
          split_delay_q(pair_delay(antenna_distance(pbx, pby, pbz, at[0], at[1], at[2]),
                                   antenna_distance(pbx, pby, pbz, ar[0], ar[1], ar[2]), p.inv_scale),
                        p.interp, ib, qb);
        }
        const float2 f1 = make_float2(weight_f1(qa), weight_f1(qb));
        const float2 f0 = __ffma2_rn(f1, make_float2(-1.f, -1.f), make_float2(1.f, 1.f));
        const float* yc = scan_sig + (size_t)c * p.ld;
        const long long ma = (long long)cb + ia, mb = (long long)cb + ib;
        const int ldv = p.ld;
        auto load = [&](int k) {
          const long long xa = ma + k, xb = mb + k;
          return make_float2(xa < ldv ? __ldg(yc + xa) : 0.f, xb < ldv ? __ldg(yc + xb) : 0.f);
        };
        if (valid == CH)
          accumulate_channel<KIND, false, CH>(sacc, qe, qo, f0, f1, load, valid);
        else
          accumulate_channel<KIND, true, CH>(sacc, qe, qo, f0, f1, load, valid);
      }
    }

    if (g == (G > 0 ? n_groups - 1 : 0) && p.part) {
      // window split: this chunk's sums go to the reduce pass
      const float2 S = chunk_sumsq<CH>(sacc, valid);
      const float2 Q = KIND != KIND_DAS ? __fadd2_rn(qe, qo) : make_float2(0.f, 0.f);
      // rows: (scan, point) for shared point lists, the launched position for packed per-scan lists
      float2* pp = p.part + ((p.tile_info ? (size_t)0 : (size_t)s * p.P) + tile0) * n_chunks + q;
      if (va) pp[(size_t)la * n_chunks] = make_float2(S.x, Q.x);
      if (vb) pp[(size_t)lb * n_chunks] = make_float2(S.y, Q.y);
    } else if (g == (G > 0 ? n_groups - 1 : 0)) {
      const float2 S = chunk_sumsq<CH>(sacc, valid);
      eS_a += (double)S.x;
      eS_b += (double)S.y;
      if (KIND != KIND_DAS) {
        const float2 Q = __fadd2_rn(qe, qo);
        eQ_a += (double)Q.x;
        eQ_b += (double)Q.y;
      }
      if (q == n_chunks - 1) {
        bool bad = false;
#pragma unroll
        for (int kk = 0; kk < 2; ++kk) {
          const bool want = kk == 0 ? KIND != KIND_DMAS : KIND != KIND_DAS;
          if (!want) continue;
          float ea, eb;
          if (kk == 0) {
            ea = __double2float_rn(eS_a);
            eb = __double2float_rn(eS_b);
          } else {
            ea = __double2float_rn(0.5 * (eS_a - eQ_a));
            eb = __double2float_rn(0.5 * (eS_b - eQ_b));
          }
          float* out = (kk == 0 ? p.out_das : p.out_dmas) + (size_t)s * (size_t)p.out_stride;
          unsigned long long* keys = kk == 0 ? p.key_das : p.key_dmas;
          unsigned long long key = 0ull;
          if (va) {
            out[oa] = ea;
            if (isfinite(ea)) key = argmax_key(ea, oa); else bad = true;
          }
          if (vb) {
            out[ob] = eb;
            if (isfinite(eb)) key = max(key, (unsigned long long)argmax_key(eb, ob)); else bad = true;
          }
          if (keys) {
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) key = max(key, __shfl_xor_sync(0xffffffffu, key, o));
            if (lane == 0 && key != 0ull) atomicMax(keys + s, key);
          }
        }
        if (bad && p.flags) atomicOr(p.flags, 1);
        eS_a = eS_b = eQ_a = eQ_b = 0.0;
      }
    }
    if (G > 0) {
      __syncwarp();
      if (lane == 0) mbar_arrive(&mbar[NSTAGE + t % NSTAGE]);  // this warp is done with the slot
      if (warp == 0 && t + NSTAGE - 1 < nsteps) issue(t + NSTAGE - 1);
    }
  }
}
// ----------------------------------------------------------------------------
// lattice enumeration (beamform.py:268-280 + skip filter 309-315 + centres
// 321-323), generalised to 3-D voxel grids (nz > 1).  Regions on the device
// are int32[6] {x0, y0, z0, x1, y1, z1}; the dense slot of a cell is
// (ix * ny + iy) * nz + iz (= ix * ny + iy in 2-D).
// ----------------------------------------------------------------------------
struct LatticeParams {
  double ox, oy, oz, res;
  int nx, ny, nz;
  int planar;  // 1: 2-D slice, point z = 0 exactly
  int r[6];
  const int* d_region;
  int stride;
  const uint8_t* mask;
  int skip;
  double* pts;
  int* out_idx;
  int* d_count;
  uint8_t* valid;
  int* tile_counts;
  int* tile_offsets;
  int n_tiles_max;
  int tx, ty, tz;  // tile shape (tx*ty*tz == 256)
  int2* pad_info;  // padded layout: lattice tile t -> points [256 t, 256 t + count), {0, count} here; or NULL
};

struct LatticeGeom {
  int s[3], L[3], T[3];
};

__device__ __forceinline__ LatticeGeom lattice_geom(const LatticeParams& p) {
  int r[6];
#pragma unroll
  for (int i = 0; i < 6; ++i) r[i] = p.d_region ? p.d_region[i] : p.r[i];
  const int D = p.stride;
  const int tdim[3] = {p.tx, p.ty, p.tz};
  LatticeGeom g;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    g.s[a] = (r[a] + D - 1) / D * D;
    g.L[a] = g.s[a] <= r[3 + a] ? (r[3 + a] - g.s[a]) / D + 1 : 0;
    g.T[a] = (g.L[a] + tdim[a] - 1) / tdim[a];
  }
  return g;
}

__device__ __forceinline__ bool lattice_cell(const LatticeParams& p, const LatticeGeom& g, int tile,
                                             int t, int& ix, int& iy, int& iz) {
  if (tile >= g.T[0] * g.T[1] * g.T[2]) return false;
  const int tzi = tile % g.T[2], tyi = (tile / g.T[2]) % g.T[1], txi = tile / (g.T[2] * g.T[1]);
  const int lz = tzi * p.tz + t % p.tz;
  const int ly = tyi * p.ty + (t / p.tz) % p.ty;
  const int lx = txi * p.tx + t / (p.tz * p.ty);
  if (lx >= g.L[0] || ly >= g.L[1] || lz >= g.L[2]) return false;
  ix = g.s[0] + lx * p.stride;
  iy = g.s[1] + ly * p.stride;
  iz = g.s[2] + lz * p.stride;
  const size_t slot = ((size_t)ix * p.ny + iy) * p.nz + iz;
  if (p.mask && !p.mask[slot]) return false;
  if (p.skip > 0 && ix % p.skip == 0 && iy % p.skip == 0 && iz % p.skip == 0) return false;
  return true;
}

__global__ void __launch_bounds__(256) lattice_count_kernel(const LatticeParams p) {
  const LatticeGeom g = lattice_geom(p);
  int ix, iy, iz;
  const bool ok = lattice_cell(p, g, blockIdx.x, threadIdx.x, ix, iy, iz);
  const int n = __syncthreads_count(ok);
  if (threadIdx.x == 0) p.tile_counts[blockIdx.x] = n;
}

// exclusive prefix sum of counts[0..n) into offsets (one 1024-thread CTA); total -> *total
__device__ void block_exclusive_scan(const int* counts, int* offsets, int n, int* total) {
  __shared__ int warp_sums[32];
  __shared__ int carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int base = 0; base < n; base += 1024) {
    const int i = base + threadIdx.x;
    const int v = i < n ? counts[i] : 0;
    int x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) warp_sums[warp] = x;
    __syncthreads();
    if (warp == 0) {
      int w = warp_sums[lane];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, w, o);
        if (lane >= o) w += y;
      }
      warp_sums[lane] = w;
    }
    __syncthreads();
    const int excl = carry + (warp > 0 ? warp_sums[warp - 1] : 0) + x - v;
    if (i < n) offsets[i] = excl;
    __syncthreads();
    if (threadIdx.x == 0) carry += warp_sums[31];
    __syncthreads();
  }
  if (threadIdx.x == 0) *total = carry;
}

__global__ void __launch_bounds__(1024) lattice_scan_kernel(const LatticeParams p) {
  block_exclusive_scan(p.tile_counts, p.tile_offsets, p.n_tiles_max, p.d_count);
}

__global__ void __launch_bounds__(256) lattice_write_kernel(const LatticeParams p) {
  __shared__ int wsum[8];
  const LatticeGeom g = lattice_geom(p);
  int ix = 0, iy = 0, iz = 0;
  const bool ok = lattice_cell(p, g, blockIdx.x, threadIdx.x, ix, iy, iz);
  const unsigned bal = __ballot_sync(0xffffffffu, ok);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) wsum[warp] = __popc(bal);
  __syncthreads();
  int before = 0;
  for (int w = 0; w < warp; ++w) before += wsum[w];
  if (p.pad_info && threadIdx.x == 0) {
    int total = 0;
    for (int w = 0; w < 8; ++w) total += wsum[w];
    p.pad_info[blockIdx.x] = make_int2(0, total);
  }
  if (!ok) return;
  const int rank = before + __popc(bal & ((1u << lane) - 1u));
  const int pos = p.pad_info ? (int)blockIdx.x * 256 + rank : p.tile_offsets[blockIdx.x] + rank;
  const size_t slot = ((size_t)ix * p.ny + iy) * p.nz + iz;
  // cell centre origin + (i + 0.5) * res, no FMA contraction (beamform.py:321-322)
  p.pts[3 * (size_t)pos] = __dadd_rn(p.ox, __dmul_rn((double)ix + 0.5, p.res));
  p.pts[3 * (size_t)pos + 1] = __dadd_rn(p.oy, __dmul_rn((double)iy + 0.5, p.res));
  p.pts[3 * (size_t)pos + 2] = p.planar ? 0.0 : __dadd_rn(p.oz, __dmul_rn((double)iz + 0.5, p.res));
  p.out_idx[pos] = (int)slot;
  p.valid[slot] = 1;
}

// ----------------------------------------------------------------------------
// Batched enumeration of per-scan regions (stride 1, 2-D): every scan's cells
// go to one packed point list in which each scan starts on a 256-point tile
// boundary; tile_info[t] = {scan, valid points} drives the table and energy
// kernels, so one launch serves every scan's fine pass.  One CTA per scan
// walks its region's 16x16 enumeration tiles in order (a fine-pass region is
// a handful of tiles: a CTA per (scan, tile) spends its time being scheduled).
// ----------------------------------------------------------------------------
struct RegionBatch {
  int n_scans;
  int* scan_counts;   // [S] valid cells of each scan's region
  int* scan_offsets;  // [S] first point of each scan (multiple of TILE)
  int* totals;        // [2] padded points, tiles
};

__global__ void __launch_bounds__(256) region_count_kernel(LatticeParams p, const RegionBatch b) {
  const int s = blockIdx.x;
  p.d_region += 6 * s;
  const LatticeGeom g = lattice_geom(p);
  const int nt = g.T[0] * g.T[1] * g.T[2];
  int total = 0;
  for (int t = 0; t < nt; ++t) {
    int ix, iy, iz;
    total += __syncthreads_count(lattice_cell(p, g, t, threadIdx.x, ix, iy, iz));
  }
  if (threadIdx.x == 0) b.scan_counts[s] = total;
}

// padded per-scan sizes -> scan offsets (points); totals = (points, tiles)
__global__ void __launch_bounds__(1024) region_offsets_kernel(const RegionBatch b) {
  __shared__ int warp_sums[32];
  __shared__ int carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int base = 0; base < b.n_scans; base += 1024) {
    const int i = base + threadIdx.x;
    const int v = i < b.n_scans ? (b.scan_counts[i] + TILE - 1) / TILE * TILE : 0;
    int x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) warp_sums[warp] = x;
    __syncthreads();
    if (warp == 0) {
      int w = warp_sums[lane];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, w, o);
        if (lane >= o) w += y;
      }
      warp_sums[lane] = w;
    }
    __syncthreads();
    if (i < b.n_scans) b.scan_offsets[i] = carry + (warp > 0 ? warp_sums[warp - 1] : 0) + x - v;
    __syncthreads();
    if (threadIdx.x == 0) carry += warp_sums[31];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    b.totals[0] = carry;
    b.totals[1] = carry / TILE;
  }
}

__global__ void __launch_bounds__(256) region_write_kernel(LatticeParams p, const RegionBatch b, int2* tile_info) {
  __shared__ int wsum[2][8];
  const int s = blockIdx.x;
  p.d_region += 6 * s;
  const LatticeGeom g = lattice_geom(p);
  const int nt = g.T[0] * g.T[1] * g.T[2];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int base = b.scan_offsets[s];
  int carry = 0;
  for (int t = 0; t < nt; ++t) {
    int ix = 0, iy = 0, iz = 0;
    const bool ok = lattice_cell(p, g, t, threadIdx.x, ix, iy, iz);
    const unsigned bal = __ballot_sync(0xffffffffu, ok);
    int* ws = wsum[t & 1];  // double-buffered: one barrier per tile
    if (lane == 0) ws[warp] = __popc(bal);
    __syncthreads();
    int before = 0, all = 0;
#pragma unroll
    for (int w = 0; w < 8; ++w) {
      before += w < warp ? ws[w] : 0;
      all += ws[w];
    }
    if (ok) {
      const int pos = base + carry + before + __popc(bal & ((1u << lane) - 1u));
      p.pts[3 * (size_t)pos] = __dadd_rn(p.ox, __dmul_rn((double)ix + 0.5, p.res));
      p.pts[3 * (size_t)pos + 1] = __dadd_rn(p.oy, __dmul_rn((double)iy + 0.5, p.res));
      p.pts[3 * (size_t)pos + 2] = 0.0;
      p.out_idx[pos] = ix * p.ny + iy;
    }
    carry += all;
  }
  const int t0 = base / TILE;
  for (int j = threadIdx.x; j * TILE < carry; j += blockDim.x)
    tile_info[t0 + j] = make_int2(s, min(TILE, carry - j * TILE));
}

// ----------------------------------------------------------------------------
// K2: device-resident select_roi (coarse2fine.py:169-256), one CTA.
// 2-D grids split into the reference's 4 quadrants (geometry.py:225-242);
// 3-D grids (nz > 1) into 8 octants with the same rules per axis.
// ----------------------------------------------------------------------------
constexpr int SEL_TPB = 256;
constexpr int MAXCH = MWB_MAX_CHILDREN;

struct Box {
  int lo[3], hi[3];
};

__device__ __forceinline__ bool box_contains(const Box& r, int ix, int iy, int iz) {
  return r.lo[0] <= ix && ix <= r.hi[0] && r.lo[1] <= iy && iy <= r.hi[1] && r.lo[2] <= iz &&
         iz <= r.hi[2];
}

// children in the reference quadrant order: index = xh + 2*yh (+ 4*zh)
__host__ __device__ __forceinline__ int split_box(const Box& r, int dims, Box q[MAXCH]) {
  int mid[3];
  for (int a = 0; a < dims; ++a) {
    const int w = r.hi[a] - r.lo[a] + 1;
    if (w < 2) return 0;
    mid[a] = r.lo[a] + (w + 1) / 2 - 1;  // last cell of the low half
  }
  const int n = 1 << dims;
  for (int k = 0; k < n; ++k) {
    for (int a = 0; a < 3; ++a) {
      if (a >= dims) {
        q[k].lo[a] = r.lo[a];
        q[k].hi[a] = r.hi[a];
      } else if ((k >> a) & 1) {
        q[k].lo[a] = mid[a] + 1;
        q[k].hi[a] = r.hi[a];
      } else {
        q[k].lo[a] = r.lo[a];
        q[k].hi[a] = mid[a];
      }
    }
  }
  return n;
}

// Region.expand (geometry.py:244-257): grow by ceil(f*side), clipped
__device__ __forceinline__ Box expand_box(const Box& r, double f, const Box& clip, int dims) {
  Box e = r;
  for (int a = 0; a < dims; ++a) {
    const int g = (int)ceil(__dmul_rn(f, (double)(r.hi[a] - r.lo[a] + 1)));
    e.lo[a] = max(r.lo[a] - g, clip.lo[a]);
    e.hi[a] = min(r.hi[a] + g, clip.hi[a]);
  }
  return e;
}

template <int K>
__device__ void block_sum(double (&v)[K], double* red /* [8][K] */, double* outv /* [K] */) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < K; ++k) {
    double x = v[k];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    if (lane == 0) red[warp * K + k] = x;
  }
  __syncthreads();
  if (threadIdx.x < K) {
    double x = 0.0;
    for (int w = 0; w < SEL_TPB / 32; ++w) x += red[w * K + threadIdx.x];  // fixed order
    outv[threadIdx.x] = x;
  }
  __syncthreads();
}

struct SelectParams {
  const float* dense;
  const uint8_t* valid;
  int nx, ny, nz, D, dims;
  Box breast;
  double frac;
  int n_min;
  int* region_out;
  mwb_trace_t* trace;
  long long dense_stride;  // batched selection: floats between consecutive scans' maps
  int staged;       // 1: the breast box's lattice is staged in shared memory
  int sl0[3], sL[3];  // staged lattice origin / extent (lattice units)
};

constexpr int SEL_STAGE_MAX = 24576;  // lattice cells staged in shared memory (96 KB)

// visit valid lattice cells of box r (from the shared-memory copy when staged;
// entries without a value are NaN there, as energies are always finite)
template <class F>
__device__ __forceinline__ void for_cells(const SelectParams& p, const float* sv, const Box& r, F&& f) {
  const int D = p.D;
  int l0[3], L[3];
  for (int a = 0; a < 3; ++a) {
    l0[a] = (r.lo[a] + D - 1) / D;
    const int l1 = r.hi[a] / D;
    if (l1 < l0[a]) return;
    L[a] = l1 - l0[a] + 1;
  }
  const int n = L[0] * L[1] * L[2];
  for (int i = threadIdx.x; i < n; i += SEL_TPB) {
    const int lz = i % L[2], ly = (i / L[2]) % L[1], lx = i / (L[2] * L[1]);
    const int ix = (l0[0] + lx) * D, iy = (l0[1] + ly) * D, iz = (l0[2] + lz) * D;
    if (p.staged) {
      const int si = ((l0[0] + lx - p.sl0[0]) * p.sL[1] + (l0[1] + ly - p.sl0[1])) * p.sL[2] + (l0[2] + lz - p.sl0[2]);
      const float v = sv[si];
      if (v == v) f(ix, iy, iz, (double)v);
    } else {
      const size_t slot = ((size_t)ix * p.ny + iy) * p.nz + iz;
      if (p.valid[slot]) f(ix, iy, iz, (double)p.dense[slot]);
    }
  }
}

__device__ __forceinline__ void put_box(int32_t* dst, const Box& b) {
  dst[0] = b.lo[0]; dst[1] = b.lo[1]; dst[2] = b.lo[2];
  dst[3] = b.hi[0]; dst[4] = b.hi[1]; dst[5] = b.hi[2];
}

// One select_roi decision (coarse2fine.py:207-252) from the children's and
// expansions' statistics: scores (variance on the first iteration, Eq. (5)
// after), np.argmax, the n_min stop, W/B of the previous vs the new selection
// and the record.  Called by all 32 lanes of one warp: lane k scores child k
// and writes its record fields, the argmax is a shuffle reduction, lane 0
// does W/B.  Returns the termination code (every lane); lane 0 writes, when
// the loop goes on, nxt = {W, B, n, sum, m2} of the new selection and next_sel.
template <int NK>
__device__ int select_score(const SelectParams& p, mwb_trace_t* tr, int iteration, int nk, const Box* rg,
                            const double* cnt, const double* sums, const double* mean, const double* m2,
                            double n_sel, double sum_sel, double m2_sel, double sigma_prev_sq, bool have_prev,
                            double prev_w, double prev_b, double* nxt, Box* next_sel) {
  const int lane = threadIdx.x & 31;
  const int rec_i = iteration;
  mwb_iter_record_t* rec = rec_i < MWB_MAX_ITERS ? &tr->records[rec_i] : nullptr;
  // the record's fields go straight to global memory; entries past
  // n_children and unset delta fields are zero
  const int k = lane;
  int has = 0, clamped = 0, count = 0;
  double mu = 0.0, var = 0.0, dr = 0.0, dl = 0.0, sc = -INFINITY;
  if (k < nk) {
    count = (int)cnt[k];
    if (cnt[k] != 0.0) {  // else an empty child: -inf (coarse2fine.py:215-217)
      mu = mean[k];
      var = m2[k] / cnt[k];
      if (iteration == 0) {  // first iteration scores by variance (218-220)
        sc = var;
        has = 1;
      } else {  // Eq. (5) (_metric_parts, 67-91)
        has = 2;
        if (var == 0.0) {
          sc = mu;
        } else {
          dr = __ddiv_rn(__dsub_rn(var, sigma_prev_sq), var);
          dl = fmin(fmax(dr, 0.0), 1.0);
          sc = __dadd_rn(__dmul_rn(__dsub_rn(1.0, dl), mu), __dmul_rn(dl, var));
          clamped = dl != dr;
        }
      }
    }
  }
  if (rec && k < MWB_MAX_CHILDREN) {
    rec->counts[k] = count;
    rec->has_stats[k] = has;
    rec->clamped[k] = clamped;
    rec->scores[k] = k < nk ? sc : 0.0;
    rec->mu[k] = mu;
    rec->var[k] = var;
    rec->delta_raw[k] = dr;
    rec->delta[k] = dl;
  }
  // np.argmax (first maximum): the larger score wins, ties go to the lower index
  double best = sc;
  int selq = k < nk ? k : 0x7FFF, selc = count;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double ob = __shfl_xor_sync(0xffffffffu, best, o);
    const int oq = __shfl_xor_sync(0xffffffffu, selq, o), oc = __shfl_xor_sync(0xffffffffu, selc, o);
    if (ob > best || (ob == best && oq < selq)) {
      best = ob;
      selq = oq;
      selc = oc;
    }
  }
  if (selq >= nk) selq = 0;  // every score -inf: argmax returns 0
  if ((selq == 0 ? (int)cnt[0] : selc) < p.n_min) return MWB_TERM_N_MIN;
  const int e = nk + selq;
  const double n_e = cnt[e], sum_e = sums[e], m2_e = m2[e];
  // W, B of the previous vs the new selection (class_distances, 94-109)
  const double w = __dadd_rn(m2_sel, m2_e);
  const double ma = sum_sel / n_sel, mb = sum_e / n_e;
  const double grand = __ddiv_rn(__dadd_rn(sum_sel, sum_e), __dadd_rn(n_sel, n_e));
  const double da = __dsub_rn(ma, grand), db = __dsub_rn(mb, grand);
  const double b = __dadd_rn(__dmul_rn(n_sel, __dmul_rn(da, da)), __dmul_rn(n_e, __dmul_rn(db, db)));
  const bool satisfied = !have_prev || (b > prev_b || w < prev_w);  // OR (235)
  if (lane == 0) {
    if (rec) {
      rec->iteration = iteration + 1;
      rec->n_children = nk;
      rec->selected = selq;
      rec->satisfied = satisfied;
      put_box(rec->selected_region, rg[selq]);
      put_box(rec->expanded_region, rg[e]);
      rec->w = w;
      rec->b = b;
    }
    nxt[0] = w;
    nxt[1] = b;
    nxt[2] = n_e;
    nxt[3] = sum_e;
    nxt[4] = m2_e;
    *next_sel = rg[e];
  }
  return rec_i >= MWB_MAX_ITERS ? MWB_TERM_OVERFLOW : (satisfied ? MWB_TERM_NONE : MWB_TERM_DISTANCE);
}

template <int NK>  // 4 children (2-D quadrants) or 8 (3-D octants)
__global__ void __launch_bounds__(SEL_TPB) select_roi_kernel(const SelectParams p0) {
  // CTA b handles scan b of a batch (maps dense_stride floats apart)
  SelectParams p = p0;
  p.dense += (size_t)blockIdx.x * p0.dense_stride;
  p.region_out += 6 * blockIdx.x;
  p.trace += blockIdx.x;
  __shared__ double red[8 * 2 * 2 * NK];
  __shared__ double res[2 * 2 * NK];
  __shared__ int ctl[2];
  __shared__ Box next_sel;
  extern __shared__ float sv[];
  mwb_trace_t* tr = p.trace;
  if (p.staged) {  // one pass over global memory; every later pass reads shared memory
    const int n = p.sL[0] * p.sL[1] * p.sL[2];
    for (int i = threadIdx.x; i < n; i += SEL_TPB) {
      const int lz = i % p.sL[2], ly = (i / p.sL[2]) % p.sL[1], lx = i / (p.sL[2] * p.sL[1]);
      const size_t slot = ((size_t)(p.sl0[0] + lx) * p.D * p.ny + (size_t)(p.sl0[1] + ly) * p.D) * p.nz +
                          (size_t)(p.sl0[2] + lz) * p.D;
      sv[i] = p.valid[slot] ? p.dense[slot] : __int_as_float(0x7fc00000);
    }
    __syncthreads();
  }

  // breast-region stats: count, sum, min, max (coarse2fine.py:186-199)
  double n_sel, sum_sel, m2_sel;
  {
    double acc[2] = {0.0, 0.0};
    double mn = INFINITY, mx = -INFINITY;
    for_cells(p, sv, p.breast, [&](int, int, int, double v) {
      acc[0] += 1.0;
      acc[1] += v;
      mn = fmin(mn, v);
      mx = fmax(mx, v);
    });
    block_sum<2>(acc, red, res);
    n_sel = res[0];
    sum_sel = res[1];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
      mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    }
    if (lane == 0) {
      red[warp] = mn;
      red[8 + warp] = mx;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int w = 1; w < SEL_TPB / 32; ++w) {
        red[0] = fmin(red[0], red[w]);
        red[8] = fmax(red[8], red[8 + w]);
      }
    }
    __syncthreads();
    mn = red[0];
    mx = red[8];
    __syncthreads();
    if (n_sel == 0.0 || mx == mn) {
      if (threadIdx.x == 0) {
        tr->termination = n_sel == 0.0 ? MWB_TERM_EMPTY : MWB_TERM_DEGENERATE;
        tr->n_records = 0;
        put_box(tr->final_region, p.breast);
        put_box(p.region_out, p.breast);
      }
      return;
    }
    const double mean = sum_sel / n_sel;
    double d2[1] = {0.0};
    for_cells(p, sv, p.breast, [&](int, int, int, double v) {
      const double d = v - mean;
      d2[0] += d * d;
    });
    block_sum<1>(d2, red, res);
    m2_sel = res[0];
  }

  Box sel = p.breast;
  double sigma_prev_sq = m2_sel / n_sel;
  double prev_w = 0.0, prev_b = 0.0;
  bool have_prev = false;
  int iteration = 0;
  int term = MWB_TERM_NONE;

  while (term == MWB_TERM_NONE) {
    Box rg[2 * MAXCH];
    const int nk = split_box(sel, NK == 8 ? 3 : 2, rg);
    if (nk == 0) {
      term = MWB_TERM_REGION_FLOOR;
      break;
    }
    for (int k = 0; k < nk; ++k) rg[nk + k] = expand_box(rg[k], p.frac, sel, p.dims);

    // pass 1: count and sum of every child and of every child's expansion
    // children are disjoint: a cell's child index follows from the split point
    // of each axis (children k have lo = mid+1 on axis a iff bit a of k)
    int mid[3];
    for (int a = 0; a < 3; ++a) mid[a] = rg[0].hi[a];
    double a1[4 * NK];
#pragma unroll
    for (int k = 0; k < 4 * NK; ++k) a1[k] = 0.0;
    for_cells(p, sv, sel, [&](int ix, int iy, int iz, double v) {
      const int kc = (ix > mid[0]) | ((iy > mid[1]) << 1) | (NK == 8 ? ((iz > mid[2]) << 2) : 0);
#pragma unroll
      for (int k = 0; k < NK; ++k)
        if (k == kc) {
          a1[2 * k] += 1.0;
          a1[2 * k + 1] += v;
        }
#pragma unroll
      for (int k = NK; k < 2 * NK; ++k)
        if (box_contains(rg[k], ix, iy, iz)) {
          a1[2 * k] += 1.0;
          a1[2 * k + 1] += v;
        }
    });
    block_sum<4 * NK>(a1, red, res);
    double cnt[2 * NK], mean[2 * NK], sums[2 * NK];
#pragma unroll
    for (int k = 0; k < 2 * NK; ++k) {
      cnt[k] = res[2 * k];
      sums[k] = res[2 * k + 1];
      mean[k] = cnt[k] > 0.0 ? sums[k] / cnt[k] : 0.0;
    }
    __syncthreads();
    // pass 2: Σ (x - mean)^2 (two-pass variance, as numpy's var)
    double a2[2 * NK];
#pragma unroll
    for (int k = 0; k < 2 * NK; ++k) a2[k] = 0.0;
    for_cells(p, sv, sel, [&](int ix, int iy, int iz, double v) {
      const int kc = (ix > mid[0]) | ((iy > mid[1]) << 1) | (NK == 8 ? ((iz > mid[2]) << 2) : 0);
#pragma unroll
      for (int k = 0; k < NK; ++k)
        if (k == kc) {
          const double d = v - mean[k];
          a2[k] += d * d;
        }
#pragma unroll
      for (int k = NK; k < 2 * NK; ++k)
        if (box_contains(rg[k], ix, iy, iz)) {
          const double d = v - mean[k];
          a2[k] += d * d;
        }
    });
    block_sum<2 * NK>(a2, red, res);
    double m2[2 * NK];
#pragma unroll
    for (int k = 0; k < 2 * NK; ++k) m2[k] = res[k];
    __syncthreads();

    if (threadIdx.x < 32) {
      const int t = select_score<NK>(p, tr, iteration, nk, rg, cnt, sums, mean, m2, n_sel, sum_sel, m2_sel,
                                     sigma_prev_sq, have_prev, prev_w, prev_b, red, &next_sel);
      if (threadIdx.x == 0) ctl[0] = t;
    }
    __syncthreads();
    term = ctl[0];
    if (term == MWB_TERM_N_MIN) break;
    iteration += 1;
    if (term != MWB_TERM_NONE) break;
    prev_w = red[0];
    prev_b = red[1];
    have_prev = true;
    n_sel = red[2];
    sum_sel = red[3];
    m2_sel = red[4];
    sigma_prev_sq = m2_sel / n_sel;
    sel = next_sel;
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    tr->termination = term;
    tr->n_records = min(iteration, MWB_MAX_ITERS);
    put_box(tr->final_region, sel);
    put_box(p.region_out, sel);
  }
}
// ----------------------------------------------------------------------------
// K2w: warp-per-scan select_roi for 2-D lattices whose breast box stages in
// SEL_WARP_STAGE cells (the framework's 16..64-cell-wide low-res lattices).
// A 256-thread CTA spends most of its time in barriers and 16-double block
// reductions when every thread visits only ~5 cells per pass; a warp visits
// ~36 per lane, reduces with shuffles only, and SEL_WPB scans share a CTA.
// Cells are walked in lattice coordinates (no div/mod per cell) and each
// cell's child / expansion membership is four range tests per axis (the
// expansions are per-axis: expand_box grows each axis independently).
// Same decisions as select_roi_kernel<4>; the summation order is the warp's,
// so single-scan and batched selection both dispatch here for such lattices
// and stay bit-identical to each other.
// ----------------------------------------------------------------------------
constexpr int SEL_WPB = 4;
constexpr int SEL_WARP_STAGE = 4096;
constexpr int SEL_SPLIT_MAX_SCANS = 148;  // below a wave of scans, a CTA of 8 warps per scan

struct SelWarpCtl {
  double nxt[5];
  Box next;
  int term;
};

__device__ __forceinline__ double warp_sum_d(double x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  return x;
}
__device__ __forceinline__ int warp_sum_i(int x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  return x;
}

// f(lx, ly, v) for every valid cell of box r; lattice cells are i = lane + 32k
// of the r-lattice in row-major order, advanced incrementally.  Each lane
// loads its next SEL_U cells before visiting them in order, so the shared-
// memory latency overlaps while every accumulator sees the same sequence.
constexpr int SEL_U = 4;
template <class F>
__device__ __forceinline__ void warp_cells(const float* sv, int sLy, int sl0x, int sl0y, int D, const Box& r,
                                           F&& f) {
  const int l0x = (r.lo[0] + D - 1) / D, l1x = r.hi[0] / D;
  const int l0y = (r.lo[1] + D - 1) / D, l1y = r.hi[1] / D;
  if (l1x < l0x || l1y < l0y) return;
  const int Ly = l1y - l0y + 1, n = (l1x - l0x + 1) * Ly;
  const int lane = threadIdx.x & 31;
  const int q = 32 / Ly, rr = 32 - q * Ly;
  int lx = lane / Ly, ly = lane - lx * Ly;
  const float* base = sv + (l0x - sl0x) * sLy + (l0y - sl0y);
  for (int i0 = lane; i0 < n; i0 += 32 * SEL_U) {
    float v[SEL_U];
    int cx[SEL_U], cy[SEL_U];
#pragma unroll
    for (int u = 0; u < SEL_U; ++u) {
      cx[u] = lx;
      cy[u] = ly;
      const bool in = i0 + 32 * u < n;
      const float x = base[in ? lx * sLy + ly : 0];  // unconditional load: no branch per cell
      v[u] = in ? x : __int_as_float(0x7fc00000);
      lx += q;
      ly += rr;
      if (ly >= Ly) {
        ly -= Ly;
        ++lx;
      }
    }
#pragma unroll
    for (int u = 0; u < SEL_U; ++u)
      if (v[u] == v[u]) f(l0x + cx[u], l0y + cy[u], v[u]);
  }
}

// SPLIT = false: SEL_WPB scans per CTA, one warp each (batches).
// SPLIT = true:  one scan per CTA of SEL_SPLIT_WARPS warps (single scans: a
//   lone warp is latency bound).  Every warp walks the same cells in the same
//   lane order, but in the iteration passes warp k accumulates only box k, so
//   each box's sum sees exactly the additions of the one-warp kernel and the
//   two modes agree bit for bit.
constexpr int SEL_SPLIT_WARPS = 8;

template <bool SPLIT>
__global__ void __launch_bounds__(SPLIT ? SEL_SPLIT_WARPS * 32 : SEL_WPB * 32)
    select_roi_warp_kernel(const SelectParams p, int n_scans) {
  constexpr int NT = SPLIT ? SEL_SPLIT_WARPS * 32 : 32;  // threads sharing one scan
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int s = SPLIT ? (int)blockIdx.x : (int)blockIdx.x * SEL_WPB + warp;
  if (s >= n_scans) return;
  extern __shared__ float smem_sel[];
  __shared__ SelWarpCtl wctl[SEL_WPB];
  __shared__ double box_stat[2][8];  // SPLIT: per-box sums / m2 from the owning warp
  __shared__ int box_cnt[8];
  SelWarpCtl& wc = wctl[SPLIT ? 0 : warp];
  const int D = p.D, sLx = p.sL[0], sLy = p.sL[1], sl0x = p.sl0[0], sl0y = p.sl0[1];
  const int nst = sLx * sLy;
  float* sv = smem_sel + (SPLIT ? 0 : warp * nst);
  const float* dense = p.dense + (size_t)s * p.dense_stride;
  int32_t* region_out = p.region_out + 6 * s;
  mwb_trace_t* tr = p.trace + s;
  const int tid = SPLIT ? (int)threadIdx.x : lane;
  const bool leader = tid == 0;

  {  // stage the breast box's lattice: both loads independent, 8 in flight per thread
    int lx = tid / sLy, ly = tid - lx * sLy;
    const int q = NT / sLy, rr = NT - q * sLy;
#pragma unroll 8
    for (int i = tid; i < nst; i += NT) {
      const size_t slot = (size_t)(sl0x + lx) * D * p.ny + (size_t)(sl0y + ly) * D;
      const float v = __ldg(dense + slot);
      const uint8_t ok = __ldg(p.valid + slot);
      sv[i] = ok ? v : __int_as_float(0x7fc00000);
      lx += q;
      ly += rr;
      if (ly >= sLy) {
        ly -= sLy;
        ++lx;
      }
    }
  }
  if (SPLIT)
    __syncthreads();
  else
    __syncwarp();

  // breast-region stats: count, sum, min, max, then the two-pass m2
  // (coarse2fine.py:186-199); SPLIT warps all compute them (identically)
  double n_sel, sum_sel, m2_sel;
  {
    int c = 0;
    double sm = 0.0;
    float mn = INFINITY, mx = -INFINITY;  // exact in fp32: the values are fp32
    warp_cells(sv, sLy, sl0x, sl0y, D, p.breast, [&](int, int, float v) {
      ++c;
      sm += (double)v;
      mn = fminf(mn, v);
      mx = fmaxf(mx, v);
    });
    n_sel = (double)warp_sum_i(c);
    sum_sel = warp_sum_d(sm);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      mn = fminf(mn, __shfl_xor_sync(0xffffffffu, mn, o));
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    }
    if (n_sel == 0.0 || mx == mn) {
      if (leader) {
        tr->termination = n_sel == 0.0 ? MWB_TERM_EMPTY : MWB_TERM_DEGENERATE;
        tr->n_records = 0;
        put_box(tr->final_region, p.breast);
        put_box(region_out, p.breast);
      }
      return;
    }
    const double mean = sum_sel / n_sel;
    double d2 = 0.0;
    warp_cells(sv, sLy, sl0x, sl0y, D, p.breast, [&](int, int, float v) {
      const double d = (double)v - mean;
      d2 = __fma_rn(d, d, d2);
    });
    m2_sel = warp_sum_d(d2);
  }

  Box sel = p.breast;
  double sigma_prev_sq = m2_sel / n_sel;
  double prev_w = 0.0, prev_b = 0.0;
  bool have_prev = false;
  int iteration = 0;
  int term = MWB_TERM_NONE;

  while (true) {
    Box rg[8];
    const int nk = split_box(sel, 2, rg);
    if (nk == 0) {
      term = MWB_TERM_REGION_FLOOR;
      break;
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) rg[4 + k] = expand_box(rg[k], p.frac, sel, 2);
    // lattice thresholds: a cell is in a high-half child iff l * D > mid;
    // expansion ranges per axis: x from rg[4] (low) / rg[5] (high), y from rg[4] / rg[6]
    const int mxl = rg[0].hi[0] / D, myl = rg[0].hi[1] / D;
    const int ex0l = (rg[4].lo[0] + D - 1) / D, ex0h = rg[4].hi[0] / D;
    const int ex1l = (rg[5].lo[0] + D - 1) / D, ex1h = rg[5].hi[0] / D;
    const int ey0l = (rg[4].lo[1] + D - 1) / D, ey0h = rg[4].hi[1] / D;
    const int ey1l = (rg[6].lo[1] + D - 1) / D, ey1h = rg[6].hi[1] / D;
    double cnt[8], sums[8], mean[8], m2[8];

    if constexpr (SPLIT) {
      // warp k owns box k: the same membership tests as below, as one rectangle
      const int k = warp;
      const bool xhi = k < 4 ? (k & 1) : false, yhi = k < 4 ? (k >> 1) & 1 : false;
      const int rx0 = k < 4 ? (xhi ? mxl + 1 : INT_MIN) : ((k - 4) & 1 ? ex1l : ex0l);
      const int rx1 = k < 4 ? (xhi ? INT_MAX : mxl) : ((k - 4) & 1 ? ex1h : ex0h);
      const int ry0 = k < 4 ? (yhi ? myl + 1 : INT_MIN) : ((k - 4) >> 1 ? ey1l : ey0l);
      const int ry1 = k < 4 ? (yhi ? INT_MAX : myl) : ((k - 4) >> 1 ? ey1h : ey0h);
      int ci = 0;
      double a1 = 0.0;
      warp_cells(sv, sLy, sl0x, sl0y, D, sel, [&](int lx, int ly, float fv) {
        const double v = fv;
        if (rx0 <= lx && lx <= rx1 && ry0 <= ly && ly <= ry1) {
          ++ci;
          a1 += v;
        }
      });
      ci = warp_sum_i(ci);
      a1 = warp_sum_d(a1);
      if (lane == 0) {
        box_cnt[k] = ci;
        box_stat[0][k] = a1;
      }
      __syncthreads();
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        cnt[j] = (double)box_cnt[j];
        sums[j] = box_stat[0][j];
        mean[j] = cnt[j] > 0.0 ? sums[j] / cnt[j] : 0.0;
      }
      double a2 = 0.0;
      const double mu = mean[k];
      warp_cells(sv, sLy, sl0x, sl0y, D, sel, [&](int lx, int ly, float fv) {
        const double v = fv;
        if (rx0 <= lx && lx <= rx1 && ry0 <= ly && ly <= ry1) {
          const double d = v - mu;
          a2 = __fma_rn(d, d, a2);  // explicit: both modes round alike
        }
      });
      a2 = warp_sum_d(a2);
      if (lane == 0) box_stat[1][k] = a2;
      __syncthreads();
#pragma unroll
      for (int j = 0; j < 8; ++j) m2[j] = box_stat[1][j];
    } else {
      // pass 1: count and sum of every child and of every child's expansion
      int ci[8];
      double a1[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        ci[k] = 0;
        a1[k] = 0.0;
      }
      warp_cells(sv, sLy, sl0x, sl0y, D, sel, [&](int lx, int ly, float fv) {
        const double v = fv;
        const int kc = (lx > mxl) | ((ly > myl) << 1);
        const bool x0 = ex0l <= lx && lx <= ex0h, x1 = ex1l <= lx && lx <= ex1h;
        const bool y0 = ey0l <= ly && ly <= ey0h, y1 = ey1l <= ly && ly <= ey1h;
        const bool in[8] = {kc == 0, kc == 1, kc == 2, kc == 3, x0 && y0, x1 && y0, x0 && y1, x1 && y1};
#pragma unroll
        for (int k = 0; k < 8; ++k)
          if (in[k]) {
            ++ci[k];
            a1[k] += v;
          }
      });
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        cnt[k] = (double)warp_sum_i(ci[k]);
        sums[k] = warp_sum_d(a1[k]);
        mean[k] = cnt[k] > 0.0 ? sums[k] / cnt[k] : 0.0;
      }
      // pass 2: sum of (x - mean)^2 (two-pass variance, as numpy's var)
      double a2[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) a2[k] = 0.0;
      warp_cells(sv, sLy, sl0x, sl0y, D, sel, [&](int lx, int ly, float fv) {
        const double v = fv;
        const int kc = (lx > mxl) | ((ly > myl) << 1);
        const bool x0 = ex0l <= lx && lx <= ex0h, x1 = ex1l <= lx && lx <= ex1h;
        const bool y0 = ey0l <= ly && ly <= ey0h, y1 = ey1l <= ly && ly <= ey1h;
        const bool in[8] = {kc == 0, kc == 1, kc == 2, kc == 3, x0 && y0, x1 && y0, x0 && y1, x1 && y1};
#pragma unroll
        for (int k = 0; k < 8; ++k)
          if (in[k]) {
            const double d = v - mean[k];
            a2[k] = __fma_rn(d, d, a2[k]);
          }
      });
#pragma unroll
      for (int k = 0; k < 8; ++k) m2[k] = warp_sum_d(a2[k]);
    }

    if (!SPLIT || warp == 0) {
      const int t = select_score<4>(p, tr, iteration, nk, rg, cnt, sums, mean, m2, n_sel, sum_sel, m2_sel,
                                    sigma_prev_sq, have_prev, prev_w, prev_b, wc.nxt, &wc.next);
      if (lane == 0) wc.term = t;
    }
    if (SPLIT)
      __syncthreads();
    else
      __syncwarp();
    term = wc.term;
    if (term == MWB_TERM_N_MIN) break;
    iteration += 1;
    if (term != MWB_TERM_NONE) break;
    prev_w = wc.nxt[0];
    prev_b = wc.nxt[1];
    have_prev = true;
    n_sel = wc.nxt[2];
    sum_sel = wc.nxt[3];
    m2_sel = wc.nxt[4];
    sigma_prev_sq = m2_sel / n_sel;
    sel = wc.next;
    if (SPLIT)
      __syncthreads();
    else
      __syncwarp();
  }
  if (leader) {
    tr->termination = term;
    tr->n_records = min(iteration, MWB_MAX_ITERS);
    put_box(tr->final_region, sel);
    put_box(region_out, sel);
  }
}

// ----------------------------------------------------------------------------
// K5: device-side scan synthesis (the step before the path)
//   model 0: the reference simulator (simulate.py:53-73, 141-156): cosine-
//            modulated Gaussian p(t) = exp(-u^2 / 2w^2) cos(2 pi fc u),
//            u = t - duration/2, amplitude contrast / max(d_i d_j, 1e-9)
//   model 1: BASELINE's differentiated Gaussian -(u/tau) e^{1/2 - u^2/2tau^2},
//            u = t - t_c, amplitude / (d_i d_j)
// Both evaluate the pulse only within +-12 envelope widths of the channel's
// delay (|p| < 1e-29 beyond; the host generator uses the same support).  The
// signal is fp64, stored fp32.  Noise: Philox-4x32-10 keyed by (seed, scan),
// counter (channel, sample / 4), Box-Muller; sigma per scan either absolute or
// peak|clean| / 10^(SNR/20).
// ----------------------------------------------------------------------------
struct SimParams {
  float* out;
  int S, C, N, ld;
  const int* chan;
  const double* ant;
  const double* scat;  // [S][K][4] x, y, z, amplitude
  int K;
  double v, dt, t0;
  int model;
  double a, b, c;      // model 0: fc, width, duration; model 1: tau, t_c, unused
  unsigned int* peak;  // [S] float bits of max |clean|
  const double* sigma_param;  // [S]: absolute sigma (noise_mode 1) or SNR dB (2)
  int noise_mode;      // 0 none, 1 absolute, 2 SNR vs peak
  unsigned long long seed;
};

__device__ __forceinline__ double sim_pulse(const SimParams& p, double t) {
  if (p.model == 0) {
    const double u = t - p.c / 2.0;
    return exp(-(u * u) / (2.0 * p.b * p.b)) * cos(2.0 * M_PI * p.a * u);
  }
  const double x = (t - p.b) / p.a;
  return -x * exp(0.5 - 0.5 * x * x);
}

__global__ void sim_clean_kernel(const SimParams p) {
  const int c = blockIdx.y, s = blockIdx.z;
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  float* row = p.out + ((size_t)s * p.C + c) * p.ld;
  double acc = 0.0;
  if (k < p.N) {
    const int tx = p.chan[2 * c], rx = p.chan[2 * c + 1];
    const double t = p.t0 + p.dt * (double)k;
    const double half = 12.0 * (p.model == 0 ? p.b : p.a);
    for (int j = 0; j < p.K; ++j) {
      const double* q = p.scat + ((size_t)s * p.K + j) * 4;
      const double di = antenna_distance(p.ant[3 * tx], p.ant[3 * tx + 1], p.ant[3 * tx + 2], q[0], q[1], q[2]);
      const double dj = antenna_distance(p.ant[3 * rx], p.ant[3 * rx + 1], p.ant[3 * rx + 2], q[0], q[1], q[2]);
      const double tau = (di + dj) / p.v;
      const double centre = p.model == 0 ? tau + p.c / 2.0 : tau + p.b;
      if (fabs(t - centre) > half) continue;
      const double spread = p.model == 0 ? fmax(di * dj, 1e-9) : di * dj;
      acc += q[3] / spread * sim_pulse(p, t - tau);
    }
  }
  const float v = (float)acc;
  if (k < p.ld) row[k] = k < p.N ? v : 0.f;
  if (p.noise_mode == 2) {  // per-scan peak of |clean| (positive floats order as uints)
    unsigned int u = __float_as_uint(fabsf(v));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) u = max(u, __shfl_xor_sync(0xffffffffu, u, o));
    if ((threadIdx.x & 31) == 0 && u) atomicMax(p.peak + s, u);
  }
}

__device__ __forceinline__ uint4 philox4x32_10(uint4 ctr, uint2 key) {
  const uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u, W0 = 0x9E3779B9u, W1 = 0xBB67AE85u;
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint32_t hi0 = __umulhi(M0, ctr.x), lo0 = M0 * ctr.x;
    const uint32_t hi1 = __umulhi(M1, ctr.z), lo1 = M1 * ctr.z;
    ctr = make_uint4(hi1 ^ ctr.y ^ key.x, lo1, hi0 ^ ctr.w ^ key.y, lo0);
    key.x += W0;
    key.y += W1;
  }
  return ctr;
}

__global__ void sim_noise_kernel(const SimParams p) {
  const int c = blockIdx.y, s = blockIdx.z;
  const int k4 = (blockIdx.x * blockDim.x + threadIdx.x) * 4;
  if (k4 >= p.N) return;
  double sigma = p.sigma_param[s];
  if (p.noise_mode == 2) sigma = (double)__uint_as_float(p.peak[s]) / pow(10.0, sigma / 20.0);
  const uint4 r = philox4x32_10(make_uint4((uint32_t)c, (uint32_t)(k4 >> 2), (uint32_t)s, 0x6D77u),
                                make_uint2((uint32_t)p.seed, (uint32_t)(p.seed >> 32)));
  const double inv = 1.0 / 4294967296.0;
  const double u1 = ((double)r.x + 1.0) * inv, u2 = (double)r.y * inv;  // u1 in (0, 1]
  const double u3 = ((double)r.z + 1.0) * inv, u4 = (double)r.w * inv;
  const double r1 = sqrt(-2.0 * log(u1)), r2 = sqrt(-2.0 * log(u3));
  double z[4];
  sincospi(2.0 * u2, &z[1], &z[0]);
  sincospi(2.0 * u4, &z[3], &z[2]);
  z[0] *= r1; z[1] *= r1; z[2] *= r2; z[3] *= r2;
  float* row = p.out + ((size_t)s * p.C + c) * p.ld;
  for (int i = 0; i < 4 && k4 + i < p.N; ++i) row[k4 + i] = (float)((double)row[k4 + i] + sigma * z[i]);
}

// ----------------------------------------------------------------------------
// K4: BASELINE configs[2] segmentation (quadrants scored on an n_sub x n_sub
// sub-grid with max/mean, argmax kept, stop at a given segment size).  No
// reference counterpart; the control flow is restated from BASELINE.json and
// follows Region.quadrants (geometry.py:225-242) for the split.
// ----------------------------------------------------------------------------
struct SegState {
  int region[6];
  int done;
  int iter;
  int node;  // batched tree search: index of the current region in the SegNode tree
};

// Batched search over a precomputed tree: every region a search can reach
// (the start region, its quadrants, theirs, ... down to the stop size) is a
// node; search nodes own the 4 n_sub^2 sub-grid points (and delay-table
// tiles) used to choose among their children, terminal nodes own their
// full-resolution fine-pass cells.
struct SegNode {
  int region[6];
  int search;    // slot in the search-node list, or -1
  int term;      // slot in the terminal-node list, or -1
  int child[4];  // node index of each quadrant (search nodes), else -1
};

// point t of the 4 sub-grids of the current region (fp64 centres):
// x = ox + x0*res + (i + 0.5) * (w*res / n_sub), likewise y.  Shared by the
// single-scan and batched searches, so both place every point bit-identically.
__device__ __forceinline__ void seg_point(const SegState* st, double ox, double oy, double res, int n_sub, int t,
                                          double* pts) {
  const int per = n_sub * n_sub;
  Box r;
  for (int a = 0; a < 3; ++a) {
    r.lo[a] = st->region[a];
    r.hi[a] = st->region[3 + a];
  }
  Box q[MAXCH];
  if (split_box(r, 2, q) == 0) return;
  const int k = t / per, i = (t % per) / n_sub, j = t % n_sub;
  const double wx = __dmul_rn((double)(q[k].hi[0] - q[k].lo[0] + 1), res);
  const double wy = __dmul_rn((double)(q[k].hi[1] - q[k].lo[1] + 1), res);
  const double cx = __dadd_rn(ox, __dmul_rn((double)q[k].lo[0], res));
  const double cy = __dadd_rn(oy, __dmul_rn((double)q[k].lo[1], res));
  pts[3 * (size_t)t] = __dadd_rn(cx, __dmul_rn((double)i + 0.5, __ddiv_rn(wx, (double)n_sub)));
  pts[3 * (size_t)t + 1] = __dadd_rn(cy, __dmul_rn((double)j + 0.5, __ddiv_rn(wy, (double)n_sub)));
  pts[3 * (size_t)t + 2] = 0.0;
}

__global__ void seg_points_kernel(SegState* st, double ox, double oy, double res, int n_sub, double* pts) {
  if (st->done) return;
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= 4 * n_sub * n_sub) return;
  seg_point(st, ox, oy, res, n_sub, t, pts);
}

// Batched search: scan s owns points [s * per_scan, (s + 1) * per_scan) of the
// packed list (per_scan = 4 n_sub^2 rounded up to whole 256-point tiles).
// tile_info[t] = {s, valid points}; a finished scan's tiles get 0 valid points,
// so the table and energy launches skip them.  grid = (tiles per scan, S).
__global__ void __launch_bounds__(256) seg_points_batch_kernel(const SegState* st, int per_scan, double ox, double oy,
                                                               double res, int n_sub, double* pts, int2* tile_info) {
  const int s = blockIdx.y;
  const int n = 4 * n_sub * n_sub;
  const int t = blockIdx.x * TILE + threadIdx.x;
  const bool done = st[s].done != 0;
  if (threadIdx.x == 0)
    tile_info[(size_t)s * (per_scan / TILE) + blockIdx.x] = make_int2(s, done ? 0 : min(TILE, n - (int)blockIdx.x * TILE));
  if (done || t >= n) return;
  seg_point(st + s, ox, oy, res, n_sub, t, pts + 3 * (size_t)s * per_scan);
}

// score the 4 quadrants (max/mean, DMAS shifted by the iteration minimum),
// keep the argmax (ties -> lowest index), shrink the region, record the trace
// (one 256-thread CTA per search; the batched kernel runs this same body per
// scan, so its decisions and trace are bit-identical to the single-scan search)
__device__ __forceinline__ void seg_score(SegState* st, const float* e, int n_sub, int shift_min, int stop_cells,
                                          float* lowres, mwb_seg_trace_t* tr, const SegNode* nodes = nullptr) {
  __shared__ double red[8][12];
  __shared__ double fin[12];
  if (st->done) return;
  const int it0 = st->iter;  // read before thread 0 advances the state
  const int per = n_sub * n_sub;
  Box r;
  for (int a = 0; a < 3; ++a) {
    r.lo[a] = st->region[a];
    r.hi[a] = st->region[3 + a];
  }
  Box q[MAXCH];
  const int nk = split_box(r, 2, q);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // pass 1: global min (for the DMAS shift) and per-quadrant max
  double mn = INFINITY, mxq[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
  for (int t = threadIdx.x; t < 4 * per; t += blockDim.x) {
    const double v = (double)e[t];
    mn = fmin(mn, v);
    mxq[t / per] = fmax(mxq[t / per], v);
  }
  for (int o = 16; o > 0; o >>= 1) {
    mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
    for (int k = 0; k < 4; ++k) mxq[k] = fmax(mxq[k], __shfl_xor_sync(0xffffffffu, mxq[k], o));
  }
  if (lane == 0) {
    red[warp][0] = mn;
    for (int k = 0; k < 4; ++k) red[warp][1 + k] = mxq[k];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int k = 0; k < 5; ++k) {
      double x = red[0][k];
      for (int w = 1; w < (int)(blockDim.x / 32); ++w) x = k == 0 ? fmin(x, red[w][k]) : fmax(x, red[w][k]);
      fin[k] = x;
    }
  }
  __syncthreads();
  const double shift = shift_min ? fin[0] : 0.0;
  // pass 2: per-quadrant sums of the shifted energies (fixed order)
  double sq[4] = {0.0, 0.0, 0.0, 0.0};
  for (int t = threadIdx.x; t < 4 * per; t += blockDim.x) sq[t / per] += (double)e[t] - shift;
  for (int o = 16; o > 0; o >>= 1)
    for (int k = 0; k < 4; ++k) sq[k] += __shfl_xor_sync(0xffffffffu, sq[k], o);
  __syncthreads();
  if (lane == 0)
    for (int k = 0; k < 4; ++k) red[warp][k] = sq[k];
  __syncthreads();
  if (threadIdx.x == 0) {
    const int it = st->iter;
    mwb_seg_record_t rec;
    memset(&rec, 0, sizeof(rec));
    rec.iteration = it + 1;
    rec.shift = shift;
    for (int a = 0; a < 6; ++a) rec.parent[a] = st->region[a];
    double best = -INFINITY;
    int sel = 0;
    for (int k = 0; k < 4; ++k) {
      double s = 0.0;
      for (int w = 0; w < (int)(blockDim.x / 32); ++w) s += red[w][k];
      const double mean = s / (double)per;
      const double mx = fin[1 + k] - shift;
      const double score = mean > 0.0 ? mx / mean : 0.0;
      rec.emax[k] = mx;
      rec.emean[k] = mean;
      rec.score[k] = score;
      if (score > best) {
        best = score;
        sel = k;
      }
    }
    rec.selected = sel;
    put_box(rec.selected_region, q[sel]);
    if (it < MWB_SEG_MAX_ITERS) tr->records[it] = rec;
    for (int a = 0; a < 3; ++a) {
      st->region[a] = q[sel].lo[a];
      st->region[3 + a] = q[sel].hi[a];
    }
    st->iter = it + 1;
    if (nodes) st->node = nodes[st->node].child[sel];
    tr->n_records = min(it + 1, MWB_SEG_MAX_ITERS);
    const int w = q[sel].hi[0] - q[sel].lo[0] + 1, h = q[sel].hi[1] - q[sel].lo[1] + 1;
    if (max(w, h) <= stop_cells || w < 2 || h < 2) st->done = 1;
    put_box(tr->final_region, q[sel]);
    tr->stopped = st->done;
  }
  // the first iteration's sub-grids are the low-resolution background:
  // a (2 n_sub) x (2 n_sub) image of the starting region, row = x index
  if (lowres && it0 == 0 && nk == 4) {
    for (int t = threadIdx.x; t < 4 * per; t += blockDim.x) {
      const int k = t / per, i = (t % per) / n_sub, j = t % n_sub;
      const int gx = (k & 1) * n_sub + i, gy = (k >> 1) * n_sub + j;
      lowres[gx * 2 * n_sub + gy] = e[t];
    }
  }
}

__global__ void __launch_bounds__(256) seg_score_kernel(SegState* st, const float* e, int n_sub, int shift_min,
                                                         int stop_cells, float* lowres, mwb_seg_trace_t* tr) {
  seg_score(st, e, n_sub, shift_min, stop_cells, lowres, tr);
}

// one CTA per scan; e holds per_scan energies per scan
__global__ void __launch_bounds__(256) seg_score_batch_kernel(SegState* st, const float* e, int per_scan, int n_sub,
                                                               int shift_min, int stop_cells, float* lowres,
                                                               mwb_seg_trace_t* tr) {
  const int s = blockIdx.x;
  const int lw = 4 * n_sub * n_sub;
  seg_score(st + s, e + (size_t)s * per_scan, n_sub, shift_min, stop_cells, lowres ? lowres + (size_t)s * lw : nullptr,
            tr + s);
}

__device__ __forceinline__ void seg_init(SegState* st, int x0, int y0, int x1, int y1, int stop_cells,
                                         mwb_seg_trace_t* tr) {
  st->region[0] = x0; st->region[1] = y0; st->region[2] = 0;
  st->region[3] = x1; st->region[4] = y1; st->region[5] = 0;
  st->iter = 0;
  st->node = 0;
  const int w = x1 - x0 + 1, h = y1 - y0 + 1;
  st->done = (max(w, h) <= stop_cells || w < 2 || h < 2) ? 1 : 0;
  tr->n_records = 0;
  tr->stopped = st->done;
  for (int a = 0; a < 6; ++a) tr->final_region[a] = st->region[a];
}

__global__ void seg_init_kernel(SegState* st, int x0, int y0, int x1, int y1, int stop_cells, mwb_seg_trace_t* tr) {
  seg_init(st, x0, y0, x1, y1, stop_cells, tr);
}

__global__ void seg_region_kernel(const SegState* st, int32_t* region_out) {
  for (int a = 0; a < 6; ++a) region_out[a] = st->region[a];
}

__global__ void seg_init_batch_kernel(SegState* st, int n_scans, int x0, int y0, int x1, int y1, int stop_cells,
                                      mwb_seg_trace_t* tr) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s < n_scans) seg_init(st + s, x0, y0, x1, y1, stop_cells, tr + s);
}

__global__ void seg_region_batch_kernel(const SegState* st, int n_scans, int32_t* region_out) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s < n_scans)
    for (int a = 0; a < 6; ++a) region_out[6 * (size_t)s + a] = st[s].region[a];
}

// ---- tree search (precomputed per-node points and delay tables) ----------
// sub-grid points of every search node (grid = (tiles per node, search nodes))
__global__ void __launch_bounds__(256) seg_tree_points_kernel(const SegNode* nodes, const int* search_ids,
                                                              int per_node, double ox, double oy, double res,
                                                              int n_sub, double* pts, int2* tile_info) {
  const int k = blockIdx.y;
  const int n = 4 * n_sub * n_sub;
  const int t = blockIdx.x * TILE + threadIdx.x;
  if (threadIdx.x == 0)
    tile_info[(size_t)k * (per_node / TILE) + blockIdx.x] = make_int2(k, min(TILE, n - (int)blockIdx.x * TILE));
  if (t >= n) return;
  SegState st;
  const SegNode& nd = nodes[search_ids[k]];
  for (int a = 0; a < 6; ++a) st.region[a] = nd.region[a];
  st.done = 0;
  seg_point(&st, ox, oy, res, n_sub, t, pts + 3 * (size_t)k * per_node);
}

// launched tile (s, j) of the next search step -> tile j of scan s's node
__device__ __forceinline__ void seg_tree_map(const SegState& st, const SegNode* nodes, int s, int j, int tps, int n,
                                             int* tile_src, int2* tile_info) {
  const int k = st.done ? -1 : nodes[st.node].search;
  const size_t t = (size_t)s * tps + j;
  tile_src[t] = k < 0 ? 0 : k * tps + j;
  tile_info[t] = make_int2(s, k < 0 ? 0 : min(TILE, n - j * TILE));
}

__global__ void seg_tree_init_kernel(SegState* st, int n_scans, int x0, int y0, int x1, int y1, int stop_cells,
                                     mwb_seg_trace_t* tr, const SegNode* nodes, int tps, int n, int* tile_src,
                                     int2* tile_info) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= n_scans) return;
  seg_init(st + s, x0, y0, x1, y1, stop_cells, tr + s);
  for (int j = 0; j < tps; ++j) seg_tree_map(st[s], nodes, s, j, tps, n, tile_src, tile_info);
}

// score + move to the chosen child + map the next step's tiles (one CTA per scan)
__global__ void __launch_bounds__(256) seg_tree_score_kernel(SegState* st, const float* e, int per_scan, int n_sub,
                                                              int shift_min, int stop_cells, float* lowres,
                                                              mwb_seg_trace_t* tr, const SegNode* nodes,
                                                              int* tile_src, int2* tile_info) {
  const int s = blockIdx.x;
  const int lw = 4 * n_sub * n_sub;
  seg_score(st + s, e + (size_t)s * per_scan, n_sub, shift_min, stop_cells,
            lowres ? lowres + (size_t)s * lw : nullptr, tr + s, nodes);
  __syncthreads();
  const int tps = per_scan / TILE;
  for (int j = threadIdx.x; j < tps; j += blockDim.x) seg_tree_map(st[s], nodes, s, j, tps, lw, tile_src, tile_info);
}

// fine pass: launched tile (s, j) -> tile j of the cell list of scan s's final
// (terminal) node; regions and fine-cell counts per scan
__global__ void seg_tree_fine_map_kernel(const SegState* st, int n_scans, const SegNode* nodes,
                                         const int* term_counts, const int* term_offsets, int fine_tps,
                                         int* tile_src, int2* tile_info, int32_t* region_out, int32_t* fine_counts) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (long long)n_scans * fine_tps) return;
  const int s = (int)(i / fine_tps), j = (int)(i % fine_tps);
  const int k = nodes[st[s].node].term;
  const int cnt = k < 0 ? 0 : term_counts[k];
  const bool on = j * TILE < cnt;
  tile_src[i] = on ? term_offsets[k] / TILE + j : 0;
  tile_info[i] = make_int2(s, on ? min(TILE, cnt - j * TILE) : 0);
  if (j == 0) {
    for (int a = 0; a < 6; ++a) region_out[6 * (size_t)s + a] = st[s].region[a];
    if (fine_counts) fine_counts[s] = cnt;
  }
}

__global__ void argmax_dense_kernel(const float* dense, const uint8_t* valid, int n,
                                    unsigned long long* key) {
  unsigned long long best = 0ull;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    if (valid[i] && isfinite(dense[i])) best = max(best, (unsigned long long)argmax_key(dense[i], i));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) best = max(best, __shfl_xor_sync(0xffffffffu, best, o));
  if ((threadIdx.x & 31) == 0 && best) atomicMax(key, best);
}

// ----------------------------------------------------------------------------
// roofline microbenchmarks
// ----------------------------------------------------------------------------
constexpr int MB_ITERS = 4096;

__global__ void __launch_bounds__(1024) mb_lds_kernel(float* sink, int salt) {
  __shared__ float buf[2048];
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) buf[i] = (float)(i ^ salt);
  __syncthreads();
  float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
  int base = threadIdx.x & 31;
  for (int it = 0; it < MB_ITERS; ++it) {
    const float* b = buf + ((base + it * 37) & 1023);
#pragma unroll
    for (int k = 0; k < 32; k += 4) {
      a0 += b[k];
      a1 += b[k + 1];
      a2 += b[k + 2];
      a3 += b[k + 3];
    }
  }
  const float r = a0 + a1 + a2 + a3;
  if (r == 1234.5f) sink[threadIdx.x] = r;
}

__global__ void __launch_bounds__(1024) mb_ffma2_kernel(float* sink, float seed) {
  float2 acc[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) acc[j] = make_float2(seed + j, seed - j);
  const float2 m = make_float2(1.0000001f, 0.9999999f), a = make_float2(1e-7f, -1e-7f);
  for (int it = 0; it < MB_ITERS; ++it) {
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[j] = __ffma2_rn(acc[j], m, a);
  }
  float r = 0.f;
#pragma unroll
  for (int j = 0; j < 8; ++j) r += acc[j].x + acc[j].y;
  if (r == 1234.5f) sink[threadIdx.x] = r;
}

__global__ void __launch_bounds__(1024) mb_ffma_kernel(float* sink, float seed) {
  float acc[16];
#pragma unroll
  for (int j = 0; j < 16; ++j) acc[j] = seed + j;
  float m = 1.0000001f + seed * 1e-9f, a = 1e-7f;
  for (int it = 0; it < MB_ITERS; ++it) {
#pragma unroll
    for (int j = 0; j < 16; ++j) acc[j] = fmaf(acc[j], m, a);
  }
  float r = 0.f;
#pragma unroll
  for (int j = 0; j < 16; ++j) r += acc[j];
  if (r == 1234.5f) sink[threadIdx.x] = r;
}

// shared-memory load-width / broadcast pattern probe: WORDS = 1, 2, 4 (LDS.32/64/128);
// lane address (in units of WORDS words): 0 consecutive, 1 all-same, 2 lane/2,
// 3 lane/4, 4 lane/8, 5 (lane*3)/8 (a delay-like monotone spread)
template <int WORDS>
__global__ void __launch_bounds__(1024) mb_lds_pattern_kernel(float* sink, int pattern) {
  __shared__ __align__(16) float buf[8192];
  for (int i = threadIdx.x; i < 8192; i += blockDim.x) buf[i] = (float)(i & 1023);
  __syncthreads();
  const int lane = threadIdx.x & 31;
  int a;
  switch (pattern) {
    case 0: a = lane; break;
    case 1: a = 0; break;
    case 2: a = lane >> 1; break;
    case 3: a = lane >> 2; break;
    case 4: a = lane >> 3; break;
    default: a = (lane * 3) >> 3; break;
  }
  float acc[4] = {0.f, 0.f, 0.f, 0.f};
  for (int it = 0; it < MB_ITERS / 4; ++it) {
    const int base = ((it * 37) & 63) * 32;  // stays 16-byte aligned per WORDS
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      const float* b = buf + (base + (a + k * 8) * WORDS) % 8192;
      if (WORDS == 1) {
        acc[k & 3] += b[0];
      } else if (WORDS == 2) {
        const float2 v = *reinterpret_cast<const float2*>(b);
        acc[k & 3] += v.x + v.y;
      } else {
        const float4 v = *reinterpret_cast<const float4*>(b);
        acc[k & 3] += (v.x + v.y) + (v.z + v.w);
      }
    }
  }
  const float r = acc[0] + acc[1] + acc[2] + acc[3];
  if (r == 1234.5f) sink[threadIdx.x] = r;
}

// Second pass of a window-split launch: per (scan, point), the chunk sums in
// chunk order (fp64), then exactly the unsplit kernel's epilogue.
template <int KIND>
__global__ void __launch_bounds__(256) energy_reduce_kernel(const EnergyParams p, int n_chunks) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  int s = blockIdx.y, src = i;
  bool v;
  size_t row;
  if (p.tile_info) {  // packed per-scan lists: launched position i, its tile's scan and source point
    const int2 ti = p.tile_info[i / TILE];
    s = ti.x;
    v = i < p.P && (i % TILE) < ti.y && s >= 0;
    if (p.tile_src) src = __ldg(p.tile_src + i / TILE) * TILE + i % TILE;
    row = (size_t)i;
  } else {
    const int n_pts = p.d_count ? min(*p.d_count, p.P) : p.P;
    v = i < n_pts;
    row = (size_t)s * p.P + i;
  }
  double eS = 0.0, eQ = 0.0;
  if (v) {
    const float2* pp = p.part + row * n_chunks;
    for (int q = 0; q < n_chunks; ++q) {
      const float2 sq = pp[q];
      eS += (double)sq.x;
      if (KIND != KIND_DAS) eQ += (double)sq.y;
    }
  }
  const int o = v ? (p.out_idx ? __ldg(p.out_idx + src) : i) : -1;
  const int lane = threadIdx.x & 31;
  bool bad = false;
#pragma unroll
  for (int kk = 0; kk < 2; ++kk) {
    const bool want = kk == 0 ? KIND != KIND_DMAS : KIND != KIND_DAS;
    if (!want) continue;
    const float e = kk == 0 ? __double2float_rn(eS) : __double2float_rn(0.5 * (eS - eQ));
    float* out = (kk == 0 ? p.out_das : p.out_dmas) + (size_t)s * (size_t)p.out_stride;
    unsigned long long* keys = kk == 0 ? p.key_das : p.key_dmas;
    unsigned long long key = 0ull;
    if (v) {
      out[o] = e;
      if (isfinite(e)) key = argmax_key(e, o); else bad = true;
    }
    if (keys) {  // a warp's positions lie in one 256-point tile, hence one scan
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) key = max(key, __shfl_xor_sync(0xffffffffu, key, off));
      if (lane == 0 && key != 0ull) atomicMax(keys + s, key);
    }
  }
  if (bad && p.flags) atomicOr(p.flags, 1);
}

int choose_scans_per_cta(int tiles, int n_scans) {
  const long long target = 148LL * 3 * 8;  // >= 8 waves of 3 CTAs/SM
  long long spc = (long long)tiles * n_scans / target;
  spc = spc < 1 ? 1 : (spc > 16 ? 16 : spc);
  while ((n_scans + spc - 1) / spc > 65535) spc *= 2;
  return (int)spc;
}

#include "mwb_tc.cuh"

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
  return MWB_OK;
}

static int energies_impl(const float* sig, int n_scans, int64_t scan_stride, int n_chan, int ld,
                         int n_samples, const int32_t* chan_txrx, const double* ant_xyz, int n_ant,
                         double inv_scale, const double* pts_xyz, const int32_t* out_idx, int n_pts,
                         const int32_t* d_count, const int32_t* tile_info, const void* table, int interp, int k0,
                         int window, float* out_das, float* out_dmas, int64_t out_stride, uint64_t* key_das,
                         uint64_t* key_dmas, int32_t* flags, int mode, void* stream,
                         const int32_t* tile_src = nullptr, int n_src_pts = 0, void* part_ws = nullptr,
                         int64_t part_bytes = 0) {
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
    p.P = n_pts;
  }
  const long long tiles = (n_pts + TILE - 1) / TILE;
  // register chunk: 48 samples for windows that are a multiple of 48 (the
  // configs[4] W = 48 would waste a third of a 2 x 32 split), else 32
  const int ch = (window % 48 == 0 && window % 32 != 0) ? MWB_W48_CH : 32;
  const int resident = ch == 48 ? MWB_W48_MINB : 3;  // CTAs per SM the register budget allows
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
    const long long work_ctas = (long long)(d_count ? std::min<long long>(tiles, 16) : tiles) * grid.y;
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
    fn = kind == KIND_DAS ? energy_kernel<KIND_DAS, 3, 32>
         : (kind == KIND_DMAS ? energy_kernel<KIND_DMAS, 3, 32> : energy_kernel<KIND_BOTH, 3, 32>);
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
  const int ch = (window % 48 == 0 && window % 32 != 0) ? MWB_W48_CH : 32;
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

int64_t mwb_energies_tc_workspace_bytes(int n_scans, int n_chan, int j_count) {
  if (n_scans < 0 || n_chan < 1 || j_count < 16) return -1;
  return (int64_t)(tc_ws_absmax(n_scans) + align_up(tc_ws_gram(n_scans, n_chan, j_count), 256) +
                   align_up(tc_ws_planes(n_scans, n_chan, j_count), 256));
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
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  unsigned char* ws = reinterpret_cast<unsigned char*>(workspace);
  uint32_t* absmax = reinterpret_cast<uint32_t*>(ws);
  float4* gx = reinterpret_cast<float4*>(ws + tc_ws_absmax(n_scans));
  __half* planes = reinterpret_cast<__half*>(ws + tc_ws_absmax(n_scans) +
                                             align_up(tc_ws_gram(n_scans, n_chan, j_count), 256));
  const int Lp = tc_plane_len(j_count);
  cudaError_t ce = cudaMemsetAsync(absmax, 0, sizeof(uint32_t) * (size_t)n_scans, st);
  if (ce != cudaSuccess) return set_err(MWB_ECUDA, "cudaMemsetAsync: %s", cudaGetErrorString(ce));
  {
    const size_t sm = sizeof(float) * 4 * (size_t)Lp;
    if (sm > 48 * 1024) return set_err(MWB_ERANGE, "mwb_energies_tc: window-offset range %d too wide", j_count);
    tc::gram_kernel<<<dim3((unsigned)n_chan, (unsigned)((n_scans + 3) / 4)), 128, sm, st>>>(
        sig, scan_stride, n_scans, n_chan, ld, k0, window, j_lo, j_count, Lp, gx, absmax);
    if ((rc = check_launch("gram_kernel"))) return rc;
    tc::planes_kernel<<<dim3((unsigned)n_chan, (unsigned)n_scans), 128, 0, st>>>(sig, scan_stride, n_chan, ld, k0,
                                                                                  j_lo, Lp, absmax, planes);
    if ((rc = check_launch("planes_kernel"))) return rc;
  }
  const int kind = out_das && out_dmas ? KIND_BOTH : (out_das ? KIND_DAS : KIND_DMAS);
  if (window == 32) return launch_tc<tc::Cfg32x8>(e, kind, n_pts, n_scans, n_chan, j_lo, j_count, Lp, absmax, gx, planes, st);
  if (n_scans >= 4) return launch_tc<tc::Cfg48x4>(e, kind, n_pts, n_scans, n_chan, j_lo, j_count, Lp, absmax, gx, planes, st);
  return launch_tc<tc::Cfg48x1>(e, kind, n_pts, n_scans, n_chan, j_lo, j_count, Lp, absmax, gx, planes, st);
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
  if (p.dims == 2 && n > 0 && n <= SEL_WARP_STAGE) {  // K2w: warp per scan, or one warp per box
    const bool split = n_scans < SEL_SPLIT_MAX_SCANS;
    void (*wk)(SelectParams, int) = split ? select_roi_warp_kernel<true> : select_roi_warp_kernel<false>;
    const size_t smw = sizeof(float) * (size_t)n * (split ? 1 : SEL_WPB);
    cudaError_t e = cudaFuncSetAttribute(wk, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)(sizeof(float) * SEL_WARP_STAGE * SEL_WPB));
    if (e != cudaSuccess) return set_err(MWB_ECUDA, "cudaFuncSetAttribute: %s", cudaGetErrorString(e));
    if (split)
      wk<<<n_scans, SEL_SPLIT_WARPS * 32, smw, st>>>(p, n_scans);
    else
      wk<<<(n_scans + SEL_WPB - 1) / SEL_WPB, SEL_WPB * 32, smw, st>>>(p, n_scans);
    return check_launch("select_roi_warp_kernel");
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
  const int ch = (window % 48 == 0 && window % 32 != 0) ? MWB_W48_CH : 32;
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
