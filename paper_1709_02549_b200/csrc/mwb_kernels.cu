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
//   * per tile, each channel's needed sample span [k0+lo_c, k0+hi_c+WCH] is
//     staged into shared memory with cp.async.bulk (TMA 1-D) against an
//     mbarrier, double-buffered across (scan, window-chunk, channel-group)
//     steps;
//   * per-point per-antenna distances are fp64 (exactly the reference's
//     expression, no FMA contraction), the per-channel delay is
//     (d_tx + d_rx) * inv_scale in fp64, split into i0 = floor and an fp32
//     fraction — computed per point only, so a point's energy is bit-identical
//     whichever tile or call evaluates it;
//   * 32 window samples per point live in registers (float2 s[32]); the
//     per-point accumulation order over channels and samples is fixed.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdarg.h>
#include <string.h>
#include <math.h>

#include "../../include/mwb.h"

namespace {

constexpr int TPB = 128;          // threads per energy CTA
constexpr int TILE = 2 * TPB;     // focal points per CTA
constexpr int WCH = 32;           // window samples per register chunk
constexpr int MAX_ANT = 64;
constexpr int MAX_CHAN = 4096;
constexpr int CAP_MAX = 8192;     // floats per stage buffer (32 KB)

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

// Split a fractional delay (samples) into i0 = floor(n) and the interpolation
// weights (beamform.py:186-190; nearest -> rint, 187-188).
__device__ __forceinline__ void split_delay(double n, int interp, int& i0, float& f0, float& f1) {
  if (interp == MWB_INTERP_NEAREST) n = rint(n);
  n = fmin(fmax(n, 0.0), 1073741824.0);
  const double fl = floor(n);
  const double fr = __dsub_rn(n, fl);
  i0 = static_cast<int>(fl);
  f1 = __double2float_rn(fr);
  f0 = __double2float_rn(__dsub_rn(1.0, fr));
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

// Accumulate one channel into the register window of two points.
//   DAS : s += f0*y[k] ; s += f1*y[k+1]                (beamform.py:203-205)
//   DMAS: a = f0*y[k] + f1*y[k+1]; s += a; q += a*a    (beamform.py:207-209)
template <int KIND, bool TAIL, class Load>
__device__ __forceinline__ void accumulate_channel(float2 (&s)[WCH], float2& qe, float2& qo,
                                                   const float2 f0, const float2 f1,
                                                   const Load& load, const int valid) {
  float2 prev = load(0);
#pragma unroll
  for (int k = 0; k < WCH; ++k) {
    const float2 nxt = load(k + 1);
    if (KIND == MWB_DAS) {
      s[k] = __ffma2_rn(f0, prev, s[k]);
      s[k] = __ffma2_rn(f1, nxt, s[k]);
    } else {
      float2 a = __fmul2_rn(f0, prev);
      a = __ffma2_rn(f1, nxt, a);
      s[k] = __fadd2_rn(s[k], a);
      if (!TAIL || k < valid) {
        if (k & 1)
          qo = __ffma2_rn(a, a, qo);
        else
          qe = __ffma2_rn(a, a, qe);
      }
    }
    prev = nxt;
  }
}

// Chunk epilogue: Σ_k s_k^2 (DAS, beamform.py:211) or ½Σ_k(s_k^2 − q_k) (DMAS, 212),
// fp32 within the chunk, fp64 across chunks; fixed summation order.
template <int KIND>
__device__ __forceinline__ void chunk_energy(const float2 (&s)[WCH], const float2 qe,
                                             const float2 qo, const int valid, double& ea,
                                             double& eb) {
  float2 acc = make_float2(0.f, 0.f);
#pragma unroll
  for (int k = 0; k < WCH; ++k)
    if (k < valid) acc = __ffma2_rn(s[k], s[k], acc);
  if (KIND == MWB_DAS) {
    ea += static_cast<double>(acc.x);
    eb += static_cast<double>(acc.y);
  } else {
    const float2 q = __fadd2_rn(qe, qo);
    ea += 0.5 * (static_cast<double>(acc.x) - static_cast<double>(q.x));
    eb += 0.5 * (static_cast<double>(acc.y) - static_cast<double>(q.y));
  }
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
  int interp;
  int k0;
  int W;
  float* out;
  long long out_stride;
  unsigned long long* argmax;
  int* flags;
  int mode;
  int scans_per_cta;
  int cap;  // floats per stage buffer
};

struct SmemLayout {
  size_t dist, chan, lo, alloc, off, ant_min, ant_max, misc, mbar, stage, total;
};

__host__ __device__ inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

__host__ __device__ inline SmemLayout smem_layout(int M, int C, int cap) {
  SmemLayout L;
  size_t o = 0;
  L.dist = o;    o += sizeof(double) * (size_t)M * TILE;
  L.chan = o;    o += sizeof(int2) * (size_t)C;
  L.lo = o;      o += sizeof(int) * (size_t)C;
  L.alloc = o;   o += sizeof(int) * (size_t)C;
  L.off = o;     o += sizeof(int) * (size_t)C;
  o = align_up(o, 8);
  L.ant_min = o; o += sizeof(double) * (size_t)M;
  L.ant_max = o; o += sizeof(double) * (size_t)M;
  L.misc = o;    o += sizeof(int) * 16;
  o = align_up(o, 16);
  L.mbar = o;    o += sizeof(uint64_t) * 2;
  o = align_up(o, 128);
  L.stage = o;   o += sizeof(float) * 2 * (size_t)cap;
  L.total = o;
  return L;
}

// ----------------------------------------------------------------------------
// K1: fused delay + staged fractional gather + DAS/DMAS window accumulation
// ----------------------------------------------------------------------------
template <int KIND>
__global__ void __launch_bounds__(TPB, 3) energy_kernel(const EnergyParams p) {
  extern __shared__ __align__(128) unsigned char smem[];
  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int warp = tid >> 5;

  const int n_pts = p.d_count ? min(*p.d_count, p.P) : p.P;
  const int tile0 = blockIdx.x * TILE;
  if (tile0 >= n_pts) return;
  const int n_in_tile = min(TILE, n_pts - tile0);
  const int scan_begin = blockIdx.y * p.scans_per_cta;
  if (scan_begin >= p.n_scans) return;
  const int n_my_scans = min(p.scans_per_cta, p.n_scans - scan_begin);

  const SmemLayout L = smem_layout(p.M, p.C, p.cap);
  double* dist = reinterpret_cast<double*>(smem + L.dist);
  int2* chs = reinterpret_cast<int2*>(smem + L.chan);
  int* clo = reinterpret_cast<int*>(smem + L.lo);
  int* calloc_ = reinterpret_cast<int*>(smem + L.alloc);
  int* coff = reinterpret_cast<int*>(smem + L.off);
  double* amin = reinterpret_cast<double*>(smem + L.ant_min);
  double* amax = reinterpret_cast<double*>(smem + L.ant_max);
  int* misc = reinterpret_cast<int*>(smem + L.misc);
  uint64_t* mbar = reinterpret_cast<uint64_t*>(smem + L.mbar);
  float* stage = reinterpret_cast<float*>(smem + L.stage);

  // ---- phase A: points, distances, per-channel spans ----------------------
  const int la = tid, lb = tid + TPB;
  const bool va = la < n_in_tile, vb = lb < n_in_tile;
  const int ga = tile0 + (va ? la : 0), gb = tile0 + (vb ? lb : 0);
  const double pax = p.pts[3 * (size_t)ga], pay = p.pts[3 * (size_t)ga + 1],
               paz = p.pts[3 * (size_t)ga + 2];
  const double pbx = p.pts[3 * (size_t)gb], pby = p.pts[3 * (size_t)gb + 1],
               pbz = p.pts[3 * (size_t)gb + 2];
  for (int i = 0; i < p.M; ++i) {
    const double ax = __ldg(p.ant + 3 * i), ay = __ldg(p.ant + 3 * i + 1),
                 az = __ldg(p.ant + 3 * i + 2);
    dist[i * TILE + la] = antenna_distance(pax, pay, paz, ax, ay, az);
    dist[i * TILE + lb] = antenna_distance(pbx, pby, pbz, ax, ay, az);
  }
  for (int c = tid; c < p.C; c += TPB) chs[c] = make_int2(__ldg(p.chan + 2 * c), __ldg(p.chan + 2 * c + 1));
  if (tid == 0) {
    mbar_init(&mbar[0], 1);
    mbar_init(&mbar[1], 1);
    fence_mbar_init();
  }
  __syncthreads();

  // exact per-antenna min/max distance over the tile's valid points
  for (int i = warp; i < p.M; i += TPB / 32) {
    double mn = INFINITY, mx = -INFINITY;
    for (int j = lane; j < n_in_tile; j += 32) {
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

  // channel spans: every point's i0 for channel c lies in [lo_c, hi_c] because
  // fl(+) and fl(*) are monotone (no margin needed; nearest adds one sample).
  for (int c = tid; c < p.C; c += TPB) {
    const int2 tr = chs[c];
    int lo, hi;
    float f0, f1;
    split_delay(__dmul_rn(__dadd_rn(amin[tr.x], amin[tr.y]), p.inv_scale), MWB_INTERP_LINEAR, lo,
                f0, f1);
    split_delay(__dmul_rn(__dadd_rn(amax[tr.x], amax[tr.y]), p.inv_scale), MWB_INTERP_LINEAR, hi,
                f0, f1);
    if (p.interp == MWB_INTERP_NEAREST) hi += 1;
    clo[c] = lo;
    // samples k0+q*WCH + [lo, hi+WCH] plus up to 3 of alignment slack each side
    long long a = (long long)(hi - lo) + WCH + 8;
    a = (a + 3) & ~3LL;
    calloc_[c] = (int)min(a, (long long)1 << 30);
  }
  __syncthreads();
  if (tid == 0) {
    int mx = 0;
    for (int c = 0; c < p.C; ++c) mx = max(mx, calloc_[c]);
    int G = (p.mode == 0 && mx <= p.cap) ? p.cap / mx : 0;
    if (G > p.C) G = p.C;
    int run = 0;
    for (int c = 0; c < p.C; ++c) {
      if (G > 0 && c % G == 0) run = 0;
      coff[c] = run;
      run += calloc_[c];
    }
    misc[0] = G;
    misc[1] = G > 0 ? (p.C + G - 1) / G : 0;
  }
  __syncthreads();
  const int G = misc[0];
  const int n_groups = misc[1];
  const int n_chunks = (p.W + WCH - 1) / WCH;

  const int oa = va ? (p.out_idx ? __ldg(p.out_idx + ga) : ga) : -1;
  const int ob = vb ? (p.out_idx ? __ldg(p.out_idx + gb) : gb) : -1;

  // per-step bookkeeping
  auto chunk_base = [&](int q) { return p.k0 + q * WCH; };

  // Issue the bulk copies of step t into buffer (t & 1).  Warp 0 only.
  auto issue = [&](int t) {
    const int g = t % n_groups;
    const int r = t / n_groups;
    const int q = r % n_chunks;
    const int s = scan_begin + r / n_chunks;
    const int c_begin = g * G, c_end = min(p.C, c_begin + G);
    float* buf = stage + (t & 1) * p.cap;
    const float* scan_sig = p.sig + (size_t)s * (size_t)p.scan_stride;
    uint32_t bytes_lane = 0;
    for (int c = c_begin + lane; c < c_end; c += 32) {
      const long long start = (long long)chunk_base(q) + clo[c];
      const long long start4 = start & ~3LL;
      const long long avail = (long long)p.ld - start4;
      const long long n = min((long long)calloc_[c], max(avail, 0LL));
      bytes_lane += (uint32_t)(n * 4);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) bytes_lane += __shfl_xor_sync(0xffffffffu, bytes_lane, o);
    if (lane == 0) mbar_arrive_expect_tx(&mbar[t & 1], bytes_lane);
    __syncwarp();
    for (int c = c_begin + lane; c < c_end; c += 32) {
      const long long start = (long long)chunk_base(q) + clo[c];
      const long long start4 = start & ~3LL;
      const long long avail = (long long)p.ld - start4;
      const int alloc = calloc_[c];
      const long long n = min((long long)alloc, max(avail, 0LL));
      float* dst = buf + coff[c];
      if (n > 0) bulk_g2s(dst, scan_sig + (size_t)c * p.ld + start4, (uint32_t)(n * 4), &mbar[t & 1]);
      for (long long j = max(n, 0LL); j < alloc; ++j) dst[j] = 0.f;  // past the record: zeros
    }
  };

  const double isc = p.inv_scale;
  const int nsteps = (n_groups > 0 ? n_groups : 1) * n_chunks * n_my_scans;

  float2 sacc[WCH];
  float2 qe = make_float2(0.f, 0.f), qo = make_float2(0.f, 0.f);
  double ea = 0.0, eb = 0.0;

  if (G > 0 && warp == 0) issue(0);

  for (int t = 0; t < nsteps; ++t) {
    const int g = G > 0 ? t % n_groups : 0;
    const int r = G > 0 ? t / n_groups : t;
    const int q = r % n_chunks;
    const int si = r / n_chunks;
    const int s = scan_begin + si;
    const int valid = min(WCH, p.W - q * WCH);

    if (G > 0) {
      if (warp == 0 && t + 1 < nsteps) issue(t + 1);
      mbar_wait(&mbar[t & 1], (t >> 1) & 1);
    }
    if (g == 0) {
#pragma unroll
      for (int k = 0; k < WCH; ++k) sacc[k] = make_float2(0.f, 0.f);
      qe = make_float2(0.f, 0.f);
      qo = make_float2(0.f, 0.f);
    }

    const int c_begin = G > 0 ? g * G : 0;
    const int c_end = G > 0 ? min(p.C, c_begin + G) : p.C;
    const int cb = chunk_base(q);
    const float* buf = stage + (t & 1) * p.cap;
    const float* scan_sig = p.sig + (size_t)s * (size_t)p.scan_stride;

    for (int c = c_begin; c < c_end; ++c) {
      const int2 tr = chs[c];
      const double na = __dmul_rn(__dadd_rn(dist[tr.x * TILE + la], dist[tr.y * TILE + la]), isc);
      const double nb = __dmul_rn(__dadd_rn(dist[tr.x * TILE + lb], dist[tr.y * TILE + lb]), isc);
      int ia, ib;
      float2 f0, f1;
      split_delay(na, p.interp, ia, f0.x, f1.x);
      split_delay(nb, p.interp, ib, f0.y, f1.y);
      if (G > 0) {
        const int sbase = coff[c] - ((cb + clo[c]) & ~3) + cb;
        const float* ya = buf + sbase + ia;
        const float* yb = buf + sbase + ib;
        auto load = [&](int k) { return make_float2(ya[k], yb[k]); };
        if (valid == WCH)
          accumulate_channel<KIND, false>(sacc, qe, qo, f0, f1, load, valid);
        else
          accumulate_channel<KIND, true>(sacc, qe, qo, f0, f1, load, valid);
      } else {
        // L1/L2 gather path: same arithmetic, loads straight from global.
        const float* yc = scan_sig + (size_t)c * p.ld;
        const long long ma = (long long)cb + ia, mb = (long long)cb + ib;
        const int ldv = p.ld;
        auto load = [&](int k) {
          const long long xa = ma + k, xb = mb + k;
          return make_float2(xa < ldv ? __ldg(yc + xa) : 0.f, xb < ldv ? __ldg(yc + xb) : 0.f);
        };
        if (valid == WCH)
          accumulate_channel<KIND, false>(sacc, qe, qo, f0, f1, load, valid);
        else
          accumulate_channel<KIND, true>(sacc, qe, qo, f0, f1, load, valid);
      }
    }

    if (g == (G > 0 ? n_groups - 1 : 0)) {
      chunk_energy<KIND>(sacc, qe, qo, valid, ea, eb);
      if (q == n_chunks - 1) {
        const float eaf = __double2float_rn(ea), ebf = __double2float_rn(eb);
        float* out = p.out + (size_t)s * (size_t)p.out_stride;
        unsigned long long key = 0ull;
        bool bad = false;
        if (va) {
          out[oa] = eaf;
          if (isfinite(eaf)) key = argmax_key(eaf, oa); else bad = true;
        }
        if (vb) {
          out[ob] = ebf;
          if (isfinite(ebf)) key = max(key, (unsigned long long)argmax_key(ebf, ob)); else bad = true;
        }
        if (p.argmax) {
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) key = max(key, __shfl_xor_sync(0xffffffffu, key, o));
          if (lane == 0 && key != 0ull) atomicMax(p.argmax + s, key);
        }
        if (bad && p.flags) atomicOr(p.flags, 1);
        ea = 0.0;
        eb = 0.0;
      }
    }
    if (G > 0) __syncthreads();
  }
}

// ----------------------------------------------------------------------------
// lattice enumeration (beamform.py:268-280 + skip filter 309-315 + centres 321-323)
// ----------------------------------------------------------------------------
struct LatticeParams {
  double ox, oy, res;
  int nx, ny;
  int x0, y0, x1, y1;
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
};

struct LatticeGeom {
  int sx, sy, Lx, Ly, TX, TY;
};

__device__ __forceinline__ LatticeGeom lattice_geom(const LatticeParams& p) {
  int x0 = p.x0, y0 = p.y0, x1 = p.x1, y1 = p.y1;
  if (p.d_region) {
    x0 = p.d_region[0]; y0 = p.d_region[1]; x1 = p.d_region[2]; y1 = p.d_region[3];
  }
  const int D = p.stride;
  LatticeGeom g;
  g.sx = (x0 + D - 1) / D * D;
  g.sy = (y0 + D - 1) / D * D;
  g.Lx = g.sx <= x1 ? (x1 - g.sx) / D + 1 : 0;
  g.Ly = g.sy <= y1 ? (y1 - g.sy) / D + 1 : 0;
  g.TX = (g.Lx + 15) / 16;
  g.TY = (g.Ly + 15) / 16;
  return g;
}

__device__ __forceinline__ bool lattice_cell(const LatticeParams& p, const LatticeGeom& g, int tile,
                                             int t, int& ix, int& iy) {
  if (tile >= g.TX * g.TY) return false;
  const int tx = tile / g.TY, ty = tile % g.TY;
  const int lx = tx * 16 + (t >> 4), ly = ty * 16 + (t & 15);
  if (lx >= g.Lx || ly >= g.Ly) return false;
  ix = g.sx + lx * p.stride;
  iy = g.sy + ly * p.stride;
  if (p.mask && !p.mask[(size_t)ix * p.ny + iy]) return false;
  if (p.skip > 0 && ix % p.skip == 0 && iy % p.skip == 0) return false;
  return true;
}

__global__ void __launch_bounds__(256) lattice_count_kernel(const LatticeParams p) {
  const LatticeGeom g = lattice_geom(p);
  int ix, iy;
  const bool ok = lattice_cell(p, g, blockIdx.x, threadIdx.x, ix, iy);
  const int n = __syncthreads_count(ok);
  if (threadIdx.x == 0) p.tile_counts[blockIdx.x] = n;
}

__global__ void __launch_bounds__(1024) lattice_scan_kernel(const LatticeParams p) {
  __shared__ int warp_sums[32];
  __shared__ int carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int base = 0; base < p.n_tiles_max; base += 1024) {
    const int i = base + threadIdx.x;
    const int v = i < p.n_tiles_max ? p.tile_counts[i] : 0;
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
    if (i < p.n_tiles_max) p.tile_offsets[i] = excl;
    __syncthreads();
    if (threadIdx.x == 0) carry += warp_sums[31];
    __syncthreads();
  }
  if (threadIdx.x == 0) *p.d_count = carry;
}

__global__ void __launch_bounds__(256) lattice_write_kernel(const LatticeParams p) {
  __shared__ int wsum[8];
  const LatticeGeom g = lattice_geom(p);
  int ix = 0, iy = 0;
  const bool ok = lattice_cell(p, g, blockIdx.x, threadIdx.x, ix, iy);
  const unsigned bal = __ballot_sync(0xffffffffu, ok);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) wsum[warp] = __popc(bal);
  __syncthreads();
  int before = 0;
  for (int w = 0; w < warp; ++w) before += wsum[w];
  if (!ok) return;
  const int rank = before + __popc(bal & ((1u << lane) - 1u));
  const int pos = p.tile_offsets[blockIdx.x] + rank;
  const int slot = ix * p.ny + iy;
  p.pts[3 * (size_t)pos] = __dadd_rn(p.ox, __dmul_rn((double)ix + 0.5, p.res));
  p.pts[3 * (size_t)pos + 1] = __dadd_rn(p.oy, __dmul_rn((double)iy + 0.5, p.res));
  p.pts[3 * (size_t)pos + 2] = 0.0;
  p.out_idx[pos] = slot;
  p.valid[slot] = 1;
}

// ----------------------------------------------------------------------------
// K2: device-resident select_roi (coarse2fine.py:169-256), one CTA
// ----------------------------------------------------------------------------
constexpr int SEL_TPB = 256;

struct Reg {
  int x0, y0, x1, y1;
};

__device__ __forceinline__ bool reg_contains(const Reg& r, int ix, int iy) {
  return r.x0 <= ix && ix <= r.x1 && r.y0 <= iy && iy <= r.y1;
}

// Region.quadrants (geometry.py:225-242): low half gets the odd cell
__device__ __forceinline__ bool quadrants(const Reg& r, Reg q[4]) {
  const int w = r.x1 - r.x0 + 1, h = r.y1 - r.y0 + 1;
  if (w < 2 || h < 2) return false;
  const int xm = r.x0 + (w + 1) / 2 - 1;
  const int ym = r.y0 + (h + 1) / 2 - 1;
  q[0] = {r.x0, r.y0, xm, ym};
  q[1] = {xm + 1, r.y0, r.x1, ym};
  q[2] = {r.x0, ym + 1, xm, r.y1};
  q[3] = {xm + 1, ym + 1, r.x1, r.y1};
  return true;
}

// Region.expand (geometry.py:244-257): grow by ceil(f*side), clipped
__device__ __forceinline__ Reg expand(const Reg& r, double f, const Reg& clip) {
  const int px = (int)ceil(__dmul_rn(f, (double)(r.x1 - r.x0 + 1)));
  const int py = (int)ceil(__dmul_rn(f, (double)(r.y1 - r.y0 + 1)));
  return {max(r.x0 - px, clip.x0), max(r.y0 - py, clip.y0), min(r.x1 + px, clip.x1),
          min(r.y1 + py, clip.y1)};
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
    for (int w = 0; w < SEL_TPB / 32; ++w) x += red[w * K + threadIdx.x];
    outv[threadIdx.x] = x;
  }
  __syncthreads();
}

struct SelectParams {
  const float* dense;
  const uint8_t* valid;
  int nx, ny, D;
  Reg breast;
  double frac;
  int n_min;
  int* region_out;
  mwb_trace_t* trace;
};

// visit valid lattice cells of region r
template <class F>
__device__ __forceinline__ void for_cells(const SelectParams& p, const Reg& r, F&& f) {
  const int D = p.D;
  const int lx0 = (r.x0 + D - 1) / D, ly0 = (r.y0 + D - 1) / D;
  const int lx1 = r.x1 / D, ly1 = r.y1 / D;
  if (lx1 < lx0 || ly1 < ly0) return;
  const int Lx = lx1 - lx0 + 1, Ly = ly1 - ly0 + 1;
  const long long n = (long long)Lx * Ly;
  for (long long i = threadIdx.x; i < n; i += SEL_TPB) {
    const int ix = (lx0 + (int)(i / Ly)) * D, iy = (ly0 + (int)(i % Ly)) * D;
    const size_t slot = (size_t)ix * p.ny + iy;
    if (p.valid[slot]) f(ix, iy, (double)p.dense[slot]);
  }
}

__global__ void __launch_bounds__(SEL_TPB) select_roi_kernel(const SelectParams p) {
  __shared__ double red[8 * 16];
  __shared__ double res[16];
  __shared__ int ctl[8];
  __shared__ Reg shared_regs[8];
  mwb_trace_t* tr = p.trace;

  // breast-region stats: count, sum, min, max
  double n_sel, sum_sel, m2_sel;
  {
    double acc[2] = {0.0, 0.0};
    double mn = INFINITY, mx = -INFINITY;
    for_cells(p, p.breast, [&](int, int, double v) {
      acc[0] += 1.0;
      acc[1] += v;
      mn = fmin(mn, v);
      mx = fmax(mx, v);
    });
    block_sum<2>(acc, red, res);
    n_sel = res[0];
    sum_sel = res[1];
    // min/max via the same scratch
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
        tr->final_region[0] = p.region_out[0] = p.breast.x0;
        tr->final_region[1] = p.region_out[1] = p.breast.y0;
        tr->final_region[2] = p.region_out[2] = p.breast.x1;
        tr->final_region[3] = p.region_out[3] = p.breast.y1;
      }
      return;
    }
    const double mean = sum_sel / n_sel;
    double d2[1] = {0.0};
    for_cells(p, p.breast, [&](int, int, double v) {
      const double d = v - mean;
      d2[0] += d * d;
    });
    block_sum<1>(d2, red, res);
    m2_sel = res[0];
  }

  Reg sel = p.breast;
  double sigma_prev_sq = m2_sel / n_sel;
  double prev_w = 0.0, prev_b = 0.0;
  bool have_prev = false;
  int iteration = 0;
  int term = MWB_TERM_NONE;

  while (term == MWB_TERM_NONE) {
    Reg rg[8];
    if (!quadrants(sel, rg)) {
      term = MWB_TERM_REGION_FLOOR;
      break;
    }
    for (int k = 0; k < 4; ++k) rg[4 + k] = expand(rg[k], p.frac, sel);

    // pass 1: count and sum for 4 quadrants + their 4 expansions
    double a1[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) a1[k] = 0.0;
    for_cells(p, sel, [&](int ix, int iy, double v) {
#pragma unroll
      for (int k = 0; k < 8; ++k)
        if (reg_contains(rg[k], ix, iy)) {
          a1[2 * k] += 1.0;
          a1[2 * k + 1] += v;
        }
    });
    block_sum<16>(a1, red, res);
    double cnt[8], mean[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      cnt[k] = res[2 * k];
      mean[k] = cnt[k] > 0.0 ? res[2 * k + 1] / cnt[k] : 0.0;
    }
    double sums[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) sums[k] = res[2 * k + 1];
    __syncthreads();
    // pass 2: Σ (x - mean)^2 (two-pass variance, as numpy's var)
    double a2[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) a2[k] = 0.0;
    for_cells(p, sel, [&](int ix, int iy, double v) {
#pragma unroll
      for (int k = 0; k < 8; ++k)
        if (reg_contains(rg[k], ix, iy)) {
          const double d = v - mean[k];
          a2[k] += d * d;
        }
    });
    block_sum<8>(a2, red, res);
    double m2[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) m2[k] = res[k];
    __syncthreads();

    if (threadIdx.x == 0) {
      const int rec_i = iteration;  // record index if accepted
      mwb_iter_record_t rec;
      memset(&rec, 0, sizeof(rec));
      double scores[4];
      for (int k = 0; k < 4; ++k) {
        rec.quadrant_counts[k] = (int)cnt[k];
        if (cnt[k] == 0.0) {
          scores[k] = -INFINITY;
          rec.has_stats[k] = 0;
        } else {
          const double mu = mean[k], var = m2[k] / cnt[k];
          rec.mu[k] = mu;
          rec.var[k] = var;
          if (iteration == 0) {
            scores[k] = var;
            rec.has_stats[k] = 1;
          } else {
            rec.has_stats[k] = 2;
            if (var == 0.0) {
              scores[k] = mu;
              rec.delta_raw[k] = 0.0;
              rec.delta[k] = 0.0;
              rec.clamped[k] = 0;
            } else {
              const double dr = __ddiv_rn(__dsub_rn(var, sigma_prev_sq), var);
              const double dl = fmin(fmax(dr, 0.0), 1.0);
              scores[k] = __dadd_rn(__dmul_rn(__dsub_rn(1.0, dl), mu), __dmul_rn(dl, var));
              rec.delta_raw[k] = dr;
              rec.delta[k] = dl;
              rec.clamped[k] = dl != dr;
            }
          }
        }
        rec.scores[k] = scores[k];
      }
      int selq = 0;
      for (int k = 1; k < 4; ++k)
        if (scores[k] > scores[selq]) selq = k;
      if (rec.quadrant_counts[selq] < p.n_min) {
        ctl[0] = MWB_TERM_N_MIN;
      } else {
        const int e = 4 + selq;
        const double n_e = cnt[e], sum_e = sums[e], m2_e = m2[e];
        const double w = __dadd_rn(m2_sel, m2_e);
        const double ma = sum_sel / n_sel, mb = sum_e / n_e;
        const double grand = __ddiv_rn(__dadd_rn(sum_sel, sum_e), __dadd_rn(n_sel, n_e));
        const double da = __dsub_rn(ma, grand), db = __dsub_rn(mb, grand);
        const double b = __dadd_rn(__dmul_rn(n_sel, __dmul_rn(da, da)), __dmul_rn(n_e, __dmul_rn(db, db)));
        const bool satisfied = !have_prev || (b > prev_b || w < prev_w);
        rec.iteration = iteration + 1;
        rec.selected = selq;
        rec.satisfied = satisfied;
        rec.selected_region[0] = rg[selq].x0; rec.selected_region[1] = rg[selq].y0;
        rec.selected_region[2] = rg[selq].x1; rec.selected_region[3] = rg[selq].y1;
        rec.expanded_region[0] = rg[e].x0; rec.expanded_region[1] = rg[e].y0;
        rec.expanded_region[2] = rg[e].x1; rec.expanded_region[3] = rg[e].y1;
        rec.w = w;
        rec.b = b;
        if (rec_i < MWB_MAX_ITERS) tr->records[rec_i] = rec;
        ctl[0] = rec_i >= MWB_MAX_ITERS ? MWB_TERM_OVERFLOW : (satisfied ? MWB_TERM_NONE : MWB_TERM_DISTANCE);
        ctl[1] = selq;
        red[0] = w;
        red[1] = b;
        red[2] = n_e;
        red[3] = sum_e;
        red[4] = m2_e;
        shared_regs[0] = rg[e];
      }
    }
    __syncthreads();
    term = ctl[0];
    if (term == MWB_TERM_N_MIN) break;
    iteration += 1;
    if (term != MWB_TERM_NONE) break;
    // accept the expanded selection
    prev_w = red[0];
    prev_b = red[1];
    have_prev = true;
    n_sel = red[2];
    sum_sel = red[3];
    m2_sel = red[4];
    sigma_prev_sq = m2_sel / n_sel;
    sel = shared_regs[0];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    tr->termination = term;
    tr->n_records = min(iteration, MWB_MAX_ITERS);
    tr->final_region[0] = p.region_out[0] = sel.x0;
    tr->final_region[1] = p.region_out[1] = sel.y0;
    tr->final_region[2] = p.region_out[2] = sel.x1;
    tr->final_region[3] = p.region_out[3] = sel.y1;
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

int choose_scans_per_cta(int tiles, int n_scans) {
  const long long target = 148LL * 3 * 8;  // >= 8 waves of 3 CTAs/SM
  long long spc = (long long)tiles * n_scans / target;
  spc = spc < 1 ? 1 : (spc > 16 ? 16 : spc);
  while ((n_scans + spc - 1) / spc > 65535) spc *= 2;
  return (int)spc;
}

}  // namespace

// ============================================================================
// C ABI
// ============================================================================
extern "C" {

const char* mwb_last_error(void) { return g_err; }

int mwb_version(void) { return 1; }

int64_t mwb_trace_bytes(void) { return (int64_t)sizeof(mwb_trace_t); }

int mwb_energies(const float* sig, int n_scans, int64_t scan_stride, int n_chan, int ld,
                 int n_samples, const int32_t* chan_txrx, const double* ant_xyz, int n_ant,
                 double inv_scale, const double* pts_xyz, const int32_t* out_idx, int n_pts,
                 const int32_t* d_count, int kind, int interp, int k0, int window, float* out,
                 int64_t out_stride, uint64_t* argmax_key, int32_t* flags, int mode,
                 void* stream) {
  if (n_pts < 0 || n_scans < 0 || n_chan < 0 || n_ant < 1 || window < 0 || k0 < 0)
    return set_err(MWB_EINVAL, "mwb_energies: negative size");
  if (n_pts == 0 || n_scans == 0) return MWB_OK;
  if (n_chan == 0 || window == 0)
    return set_err(MWB_EINVAL, "mwb_energies: no channels or empty window");
  if (kind != MWB_DAS && kind != MWB_DMAS) return set_err(MWB_EINVAL, "mwb_energies: bad kind");
  if (interp != MWB_INTERP_LINEAR && interp != MWB_INTERP_NEAREST)
    return set_err(MWB_EINVAL, "mwb_energies: bad interpolation");
  if (n_ant > MAX_ANT) return set_err(MWB_ERANGE, "mwb_energies: too many antennas (%d)", n_ant);
  if (n_chan > MAX_CHAN) return set_err(MWB_ERANGE, "mwb_energies: too many channels (%d)", n_chan);
  if (ld % 4 != 0 || scan_stride % 4 != 0 || ld < n_samples)
    return set_err(MWB_EINVAL, "mwb_energies: ld and scan_stride must be multiples of 4, ld >= n_samples");
  if (!sig || !chan_txrx || !ant_xyz || !pts_xyz || !out)
    return set_err(MWB_EINVAL, "mwb_energies: null pointer");
  if (((uintptr_t)sig & 15) != 0) return set_err(MWB_EINVAL, "mwb_energies: sig must be 16-byte aligned");
  if (inv_scale <= 0.0 || !isfinite(inv_scale)) return set_err(MWB_EINVAL, "mwb_energies: inv_scale must be > 0");

  EnergyParams p;
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
  p.interp = interp;
  p.k0 = k0;
  p.W = window;
  p.out = out;
  p.out_stride = out_stride;
  p.argmax = reinterpret_cast<unsigned long long*>(argmax_key);
  p.flags = flags;
  p.mode = mode;
  // stage capacity: every channel's span for a compact tile, capped at 32 KB
  long long cap = (long long)n_chan * (WCH + 24);
  cap = (cap + 3) & ~3LL;
  if (cap > CAP_MAX) cap = CAP_MAX;
  if (cap < 256) cap = 256;
  p.cap = (int)cap;
  const int tiles = (n_pts + TILE - 1) / TILE;
  p.scans_per_cta = choose_scans_per_cta(tiles, n_scans);
  const SmemLayout L = smem_layout(n_ant, n_chan, p.cap);
  if (L.total > 227 * 1024) return set_err(MWB_ERANGE, "mwb_energies: shared memory %lld bytes exceeds 227 KB", (long long)L.total);
  dim3 grid(tiles, (n_scans + p.scans_per_cta - 1) / p.scans_per_cta);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  cudaError_t e;
  if (kind == MWB_DAS) {
    e = cudaFuncSetAttribute(energy_kernel<MWB_DAS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L.total);
    if (e != cudaSuccess) return set_err(MWB_ECUDA, "cudaFuncSetAttribute: %s", cudaGetErrorString(e));
    energy_kernel<MWB_DAS><<<grid, TPB, L.total, st>>>(p);
  } else {
    e = cudaFuncSetAttribute(energy_kernel<MWB_DMAS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L.total);
    if (e != cudaSuccess) return set_err(MWB_ECUDA, "cudaFuncSetAttribute: %s", cudaGetErrorString(e));
    energy_kernel<MWB_DMAS><<<grid, TPB, L.total, st>>>(p);
  }
  return check_launch("energy_kernel");
}

int64_t mwb_lattice_workspace_bytes(int nx, int ny, int stride) {
  if (nx < 1 || ny < 1 || stride < 1) return -1;
  const long long Lx = (nx + stride - 1) / stride, Ly = (ny + stride - 1) / stride;
  const long long tiles = ((Lx + 15) / 16) * ((Ly + 15) / 16);
  return 2 * tiles * (long long)sizeof(int) + 256;
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
  p.ox = ox; p.oy = oy; p.res = res;
  p.nx = nx; p.ny = ny;
  p.x0 = x0; p.y0 = y0; p.x1 = x1; p.y1 = y1;
  p.d_region = d_region;
  p.stride = stride;
  p.mask = mask;
  p.skip = skip_stride;
  p.pts = pts_xyz;
  p.out_idx = out_idx;
  p.d_count = d_count;
  p.valid = valid;
  // upper bound on tiles: the lattice of the whole grid
  const long long Lx = (nx + stride - 1) / stride, Ly = (ny + stride - 1) / stride;
  const long long tiles = ((Lx + 15) / 16) * ((Ly + 15) / 16);
  p.n_tiles_max = (int)tiles;
  p.tile_counts = reinterpret_cast<int*>(workspace);
  p.tile_offsets = p.tile_counts + tiles;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  lattice_count_kernel<<<(unsigned)tiles, 256, 0, st>>>(p);
  lattice_scan_kernel<<<1, 1024, 0, st>>>(p);
  lattice_write_kernel<<<(unsigned)tiles, 256, 0, st>>>(p);
  return check_launch("enumerate_lattice");
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
  p.D = lattice;
  p.breast = {x0, y0, x1, y1};
  p.frac = frame_fraction;
  p.n_min = n_min;
  p.region_out = d_region_out;
  p.trace = d_trace;
  select_roi_kernel<<<1, SEL_TPB, 0, reinterpret_cast<cudaStream_t>(stream)>>>(p);
  return check_launch("select_roi_kernel");
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
    else mb_ffma_kernel<<<blocks, threads, 0, st>>>(sink, 0.5f);
    cudaEventRecord(b, st);
  }
  cudaEventSynchronize(b);
  cudaEventElapsedTime(ms, a, b);
  const double thr = (double)blocks * threads * MB_ITERS;
  if (which == 0) *work = thr * 32 * 4.0;           // bytes loaded from shared memory
  else if (which == 1) *work = thr * 8 * 2 * 2.0;   // 8 FFMA2 = 16 FMA = 32 flop
  else *work = thr * 16 * 2.0;
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  cudaFree(sink);
  return check_launch("microbench");
}

}  // extern "C"
