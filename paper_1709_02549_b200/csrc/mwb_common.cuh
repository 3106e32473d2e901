// mwb_common.cuh — constants, PTX helpers (mbarrier, 1-D bulk copy) and the numerics shared by every path
// (included by mwb_kernels.cu inside its anonymous namespace; one translation unit)
#pragma once


constexpr int TPB = 128;          // threads per energy CTA
constexpr int TILE = 2 * TPB;     // focal points per CTA
#ifndef MWB_W48_MINB
#define MWB_W48_MINB 3  // CTAs per SM of the W = 48 kernel: 3 (<= 168 registers, one channel in flight) beat 2
                        // (255 registers, two channels): 7.9 vs 8.4 ms on the configs[4] volume
#endif
#ifndef MWB_W32_CH
#define MWB_W32_CH 32  // register chunk of every other window (experiment knob: 16, with MWB_W32_MINB CTAs per SM)
#endif
#ifndef MWB_W32_MINB
#define MWB_W32_MINB 3
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
#ifdef MWB_RATIO_FORM
  // a = f0 * a',  a' = y[k] + r*y[k+1],  r = f1/f0  (f0 = 1 - f1 >= 2^-23):
  //   s += f0*a' is one FFMA, and sum_k a^2 = f0^2 * sum_k a'^2, so the
  //   channel costs 3 FFMA per sample (2 for DAS) instead of 4 (3).
  const float2 r = make_float2(__fdividef(f1.x, f0.x), __fdividef(f1.y, f0.y));
  float2 qce = make_float2(0.f, 0.f);
#ifdef MWB_RATIO_Q2
  float2 qco = make_float2(0.f, 0.f);
#endif
#pragma unroll
  for (int k = 0; k < CH; ++k) {
    const float2 nxt = load(k + 1);
    const float2 ap = __ffma2_rn(r, nxt, prev);
    s[k] = __ffma2_rn(f0, ap, s[k]);
    if (KIND != KIND_DAS && (!TAIL || k < valid)) {
#ifdef MWB_RATIO_Q2
      if (k & 1)
        qco = __ffma2_rn(ap, ap, qco);
      else
#endif
        qce = __ffma2_rn(ap, ap, qce);
    }
    prev = nxt;
  }
  if (KIND != KIND_DAS) {
    const float2 g = __fmul2_rn(f0, f0);
    qe = __ffma2_rn(g, qce, qe);
#ifdef MWB_RATIO_Q2
    qo = __ffma2_rn(g, qco, qo);
#endif
  }
  return;
#endif
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
  int src_tiles;              // tiles of that source list (bounds checks of the debug build)
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
  // ROI filter (the framework's fine pass over a precomputed whole-grid
  // table): only points whose output cell (ix, iy) = (o / filt_ny, o % filt_ny)
  // lies in the device box filt_region {x0, y0, z0, x1, y1, z1} and is not a
  // coarse-lattice cell (ix % filt_skip == 0 && iy % filt_skip == 0; 0 = none;
  // skip 1 = every cell is coarse, the Manual(1) framework)
  // are written; each written cell is marked in filt_valid and counted in
  // *filt_count.  CTAs with no such point exit before staging anything.
  const int* filt_region;
  int filt_ny;
  int filt_skip;
  uint8_t* filt_valid;
  int* filt_count;
};

__device__ __forceinline__ bool filter_keep(const EnergyParams& p, int o) {
  const int ix = o / p.filt_ny, iy = o - ix * p.filt_ny;
  const bool in = p.filt_region[0] <= ix && ix <= p.filt_region[3] && p.filt_region[1] <= iy &&
                  iy <= p.filt_region[4];
  const bool coarse = p.filt_skip > 0 && ix % p.filt_skip == 0 && iy % p.filt_skip == 0;
  return in && !coarse;
}

// mark and count the cells a filtered launch writes (one atomic per warp)
__device__ __forceinline__ void filter_mark(const EnergyParams& p, bool wa, int oa, bool wb, int ob) {
  if (wa) p.filt_valid[oa] = 1;
  if (wb) p.filt_valid[ob] = 1;
  const int n = __popc(__ballot_sync(0xffffffffu, wa)) + __popc(__ballot_sync(0xffffffffu, wb));
  if ((threadIdx.x & 31) == 0 && n) atomicAdd(p.filt_count, n);
}

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
