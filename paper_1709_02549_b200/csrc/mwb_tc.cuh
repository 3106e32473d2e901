// Tensor-core (tcgen05 / TMEM / TMA) path of the multi-scan energy kernel.
// Included by mwb_kernels.cu after the PTX helpers, EnergyParams and the
// delay-table layout.
//
// Restatement of _multistatic_energies (mwbeam/beamform.py:169-212) for a
// 256-point table tile and a group of SPG scans of one geometry, with the
// per-sample channel sum on the tensor cores:
//
//   S[p, (s, k)] = sum_c sum_m A_c[p, m] * H_{c,s}[m, k]
//
//   A_c[p, m]     = f0(p,c) at m = d, f1(p,c) at m = d + 1, else 0, where
//                   d = i0(p,c) - lo_c is the delay word's offset in the
//                   tile's span (scan-independent: built once per channel and
//                   reused by all SPG scans of the group),
//   H_{c,s}[m, k] = y_{c,s}[k0 + lo_c + m + k]  (Hankel of the staged window).
//
// So S is a [256 x 16] x [16 x (SPG * W)] product per channel, accumulated
// over the channels in TMEM (fp32).  DAS = sum_k S^2 (beamform.py:211).
// DMAS = 1/2 (sum_k S^2 - Q) (beamform.py:212) with
//   Q[p, s] = sum_c sum_k a^2 = sum_c f0^2 E(j) + 2 f0 f1 X(j) + f1^2 E(j+1),
// j = lo_c + d, E(j) = sum_k y[k0+j+k]^2, X(j) = sum_k y[k0+j+k] y[k0+j+k+1]:
// windowed Gram entries that depend on the absolute window start only, so a
// pre-pass (gram_kernel) computes them once per (scan, channel, j) and every
// tile gathers them per point on the CUDA cores.
//
// Precision: operands are split hi + lo in fp16 (y scaled per scan by a power
// of two so |y| < 2^15; planes_kernel writes the scaled hi / lo planes), and
// S = A_hi H_hi + A_hi H_lo + A_lo H_hi (the dropped A_lo H_lo term is ~2^-22
// relative), i.e. about fp32 accuracy.
//
// Per launch: gram_kernel (Gram entries + per-scan max |y|), planes_kernel
// (scaled fp16 planes of the sample range the windows touch), then
// energy_tc_kernel.  Roles of energy_tc_kernel (8 NG + 2 warps, one CTA per
// SM, persistent over (tile, group) items):
//   warps 0..8NG-1  builders in NG groups of 8 taking interleaved channel
//                   steps: thread pt of a group owns point pt (its A row and
//                   Q partial), warp w8 owns scan w8 (its 32 Hankel rows,
//                   read from the staged planes); at an item's end every
//                   group publishes its Q partials and takes part in the
//                   TMEM epilogue (scans s = g, g + NG, ...)
//   warp 8NG        producer: per channel step one tensor-map TMA copy of the
//                   group's planes and one of the two quads' Gram slices
//   warp 8NG+1      MMA issuer: one thread, 6 tcgen05.mma per channel step
// Rings: staging (NS deep, full by TMA complete_tx, empty by the builders),
// operands (NO deep, full by the builders, empty by tcgen05.commit),
// accumulator (full by commit, empty by the builders after the epilogue's
// tcgen05.ld).  Measured alternatives (dedicated epilogue warps, A in TMEM,
// deeper or shallower rings) are recorded in DESIGN.md.

namespace tc {

constexpr int K = 16;                      // taps per channel: d + 1 <= K - 1
constexpr int NS = 16;                     // staging ring depth
constexpr int NO = 4;                      // operand ring depth
#ifndef MWB_TC_GROUPS
#define MWB_TC_GROUPS 3
#endif
constexpr int NG = MWB_TC_GROUPS;          // builder groups (step t -> group t % NG)
constexpr int GW = 8;                      // warps per builder group
constexpr int NBW = NG * GW;               // builder warps
constexpr int NBT = NBW * 32;              // builder threads
constexpr int THREADS = NBT + 64;          // + producer warp + MMA warp
constexpr int A_BYTES = TILE * K * 2;      // one of hi/lo, both M-blocks: 8 KB
constexpr int MB_BYTES = 128 * K * 2;      // one M-block: 4 KB
constexpr uint32_t LBO = 128, SBO = 256;   // core-matrix strides (bytes)
constexpr size_t SMEM_MIN = 120 * 1024;    // > half the SM: one CTA per SM (TMEM is sized for one)
constexpr int SPANH_MAX = 72;              // largest staged span (W = 48): the planes' length uses it

// Window W and scans per group SPG: everything the kernel derives from them.
template <int WIN, int SPG_>
struct Cfg {
  static constexpr int W = WIN;
  static constexpr int SPG = SPG_;
  static constexpr int N = W * SPG;                       // MMA N (scans x window samples)
  static constexpr int QUADS = (SPG + 3) / 4;             // Gram entries interleave 4 scans per float4
  static constexpr int SPANH = (W + 22 + 7) & ~7;         // staged halves per (scan, plane): (off & 7) + W + K - 1 + 1
  static constexpr int H_BYTES = N * K * 2;               // one of hi/lo
  static constexpr int OP_BYTES = 2 * A_BYTES + 2 * H_BYTES;
  static constexpr int STAGE_BYTES = (SPG * 2 * SPANH * 2 + 127) & ~127;  // [scan][hi | lo][SPANH] fp16; TMA
                                                                          // destinations are 128-byte aligned
  static constexpr int GQ_FLOAT4 = QUADS * 2 * 16;        // per stage: [quad][d = 0..15][e, x] float4
  static constexpr int D_COLS = 2 * N;                    // two M-blocks x N fp32 accumulator columns
  static constexpr int TMEM_COLS = D_COLS <= 32 ? 32 : D_COLS <= 64 ? 64 : D_COLS <= 128 ? 128
                                   : D_COLS <= 256 ? 256 : 512;
  // kind::f16 instruction descriptor: f16 x f16 -> f32, both K-major, M = 128
  static constexpr uint32_t IDESC = (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
  static_assert(W % 16 == 0 && N % 16 == 0 && N <= 256 && D_COLS <= 512, "tcgen05 shape");
  static_assert(SPG % 4 == 0 || 4 % SPG == 0, "a group tiles the 4-scan Gram quads");
  static_assert(SPANH <= SPANH_MAX, "plane length");
  static_assert(OP_BYTES % 128 == 0 && (GQ_FLOAT4 * 16) % 128 == 0, "128-byte aligned ring slots");
};
using Cfg48x4 = Cfg<48, 4>;  // W = 48 batches (N = 192)
using Cfg48x1 = Cfg<48, 1>;  // configs[4]: one scan, W = 48 (N = 48)

struct Layout {
  size_t ops, stage, g, qx, bar, tmem, total;
};

template <class C>
__host__ __device__ inline Layout layout() {
  Layout L;
  size_t o = 0;
  L.ops = o;   o += (size_t)NO * C::OP_BYTES;
  L.stage = o; o += (size_t)NS * C::STAGE_BYTES;
  L.g = o;     o += (size_t)NS * C::GQ_FLOAT4 * sizeof(float4);  // staged Gram slices, one per sample stage
  L.qx = o;    o += NG * (size_t)C::SPG * TILE * sizeof(float);  // every group's Q partial sums
  o = align_up(o, 8);
  L.bar = o;   o += sizeof(uint64_t) * (2 * NS + 2 * NO + 2);
  L.tmem = o;  o += 16;
  L.total = o < SMEM_MIN ? SMEM_MIN : align_up(o, 128);
  return L;
}

// byte offset of (row r, tap m) in a K-major, no-swizzle operand of 8 x 16 B
// core matrices: the two 8-tap halves LBO apart, 8-row groups SBO apart
__device__ __forceinline__ uint32_t kmajor_off(int r, int half) {
  return (uint32_t)(r >> 3) * SBO + (uint32_t)half * LBO + (uint32_t)(r & 7) * 16u;
}

__device__ __forceinline__ uint64_t smem_desc(uint32_t addr) {
  return (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)((LBO >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((SBO >> 4) & 0x3FFF) << 32) | ((uint64_t)1 << 46);  // version 1, no swizzle
}

__device__ __forceinline__ void mma(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, int x, int y, int z, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
      "[%5];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void builders_sync() { asm volatile("bar.sync 1, %0;" ::"n"(NBT) : "memory"); }

// 32 consecutive fp32 TMEM columns of this thread's lane
__device__ __forceinline__ void tmem_ld32(uint32_t addr, float (&v)[32]) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(addr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

// 16 consecutive fp32 TMEM columns of this thread's lane
__device__ __forceinline__ void tmem_ld16(uint32_t addr, float (&v)[16]) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(addr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

// hi/lo fp16 split of two values, packed as half2 words
__device__ __forceinline__ void split2(float a, float b, uint32_t& hi, uint32_t& lo) {
  const __half2 h = __floats2half2_rn(a, b);
  const float2 back = __half22float2(h);
  const __half2 l = __floats2half2_rn(a - back.x, b - back.y);
  hi = *reinterpret_cast<const uint32_t*>(&h);
  lo = *reinterpret_cast<const uint32_t*>(&l);
}

// power-of-two scale putting a scan's max |y| in [2^14, 2^15); 1 for an
// all-zero or non-finite scan (non-finite energies are flagged downstream)
__device__ __forceinline__ int scale_exp(uint32_t absmax_bits) {
  if (absmax_bits == 0u || absmax_bits >= 0x7F800000u) return 0;
  const int e = (int)(absmax_bits >> 23) - 127;  // floor(log2 max) (subnormals: -127)
  return max(-100, min(100, 14 - e));
}
__device__ __forceinline__ float pow2f(int e) { return __int_as_float((e + 127) << 23); }


// points of table tile `tile`: the padded layout's {scan, count} record, or
// the compact list's remainder; <= 0 means nothing to do (every role skips it)
__device__ __forceinline__ int tile_points(const EnergyParams& p, int tile, int n_pts) {
  if (p.tile_info) return min(TILE, __ldg(&p.tile_info[tile].y));
  return min(TILE, n_pts - tile * TILE);
}

struct alignas(64) Params {
  CUtensorMap tm_planes;  // 3-D {Lp, 2 C, S} fp16 (scaled hi | lo planes): box {SPANH, 2, SPG}
  CUtensorMap tm_gram;    // 3-D {8 J, C, quads} fp32 (interleaved {E, X} float4 pairs): box {128, 1, QUADS}
  EnergyParams e;
  const uint32_t* absmax;  // [n_scans] bits of max |y| per scan (over the samples any window touches)

  int j_lo, J;             // positions j = lo_c + d, j in [j_lo, j_lo + J)
  int Lp;                  // plane length: samples k0 + j_lo + [0, Lp)
  int n_tiles;
  int n_groups;
};

template <int KIND, class C>
__global__ void __launch_bounds__(THREADS, 1) energy_tc_kernel(const __grid_constant__ Params P) {
  constexpr int W = C::W, SPG = C::SPG, N = C::N, QUADS = C::QUADS, SPANH = C::SPANH;
  constexpr int H_BYTES = C::H_BYTES, OP_BYTES = C::OP_BYTES, STAGE_BYTES = C::STAGE_BYTES;
  constexpr int GQ_FLOAT4 = C::GQ_FLOAT4, TMEM_COLS = C::TMEM_COLS;
  constexpr uint32_t IDESC = C::IDESC;
  extern __shared__ __align__(1024) unsigned char smem[];
  const EnergyParams& p = P.e;
  const Layout L = layout<C>();
  unsigned char* ops = smem + L.ops;
  unsigned char* stage_bytes = smem + L.stage;
  float* gstage = reinterpret_cast<float*>(smem + L.g);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + L.bar);
  uint64_t* s_full = bar;
  uint64_t* s_empty = bar + NS;
  uint64_t* o_full = bar + 2 * NS;
  uint64_t* o_empty = bar + 2 * NS + NO;
  uint64_t* acc_full = bar + 2 * NS + 2 * NO;
  uint64_t* acc_empty = acc_full + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + L.tmem);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int n_pts = p.d_count ? min(*p.d_count, p.P) : p.P;
  const int n_items = P.n_tiles * P.n_groups;

  if (tid == 0) {
    for (int i = 0; i < NS; ++i) {
      mbar_init(&s_full[i], 1);
      mbar_init(&s_empty[i], GW);
    }
    for (int i = 0; i < NO; ++i) {
      mbar_init(&o_full[i], GW);
      mbar_init(&o_empty[i], 1);
    }
    mbar_init(acc_full, 1);
    mbar_init(acc_empty, NBW);
    fence_mbar_init();
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == NBW) {
    // ===== producer: stage channel c's window span of every scan in the group
    int t = 0;
    for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
      const int tile = item % P.n_tiles, group = item / P.n_tiles;
      if (tile_points(p, tile, n_pts) <= 0) continue;
      const int2* tsp = p.tab_span + (size_t)tile * p.C;
      int lo32 = 0;  // lane i holds lo of channel (c & ~31) + i
      for (int c = 0; c < p.C; ++c, ++t) {
        const int slot = t % NS, use = t / NS;
        if ((c & 31) == 0) lo32 = c + lane < p.C ? __ldg(&tsp[c + lane].x) : 0;
        const int lo_c = __shfl_sync(0xffffffffu, lo32, c & 31);
        if (use > 0) mbar_wait(&s_empty[slot], (use - 1) & 1);
        // one tensor copy stages the group's spans (zeros past the record and
        // past the last scan), one more the two quads' Gram slices
        if (lane == 0) {
          const int off = min(max(lo_c - P.j_lo, 0), P.J - 16);  // in range by construction (j_lo, J from the table)
          if (off != lo_c - P.j_lo && p.flags) atomicOr(p.flags, 4);
          mbar_arrive_expect_tx(&s_full[slot], (uint32_t)(SPG * 2 * SPANH * 2 + GQ_FLOAT4 * 16));
          tma_load_3d(stage_bytes + slot * STAGE_BYTES, &P.tm_planes, off & ~7, 2 * c, group * SPG, &s_full[slot]);
          // Gram quads hold scans 4q .. 4q + 3: the group's first scan's quad
          tma_load_3d(reinterpret_cast<float4*>(gstage) + slot * GQ_FLOAT4, &P.tm_gram, 8 * off, c,
                      (group * SPG) / 4, &s_full[slot]);
        }
        __syncwarp();
      }
    }
  } else if (warp == NBW + 1) {
    // ===== MMA issuer (one thread)
    if (lane == 0) {
      int t = 0, it = 0;
      for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
        const int tile = item % P.n_tiles;
        if (tile_points(p, tile, n_pts) <= 0) continue;
        if (it > 0) mbar_wait(acc_empty, (it - 1) & 1);
        fence_after();
        for (int c = 0; c < p.C; ++c, ++t) {
          const int slot = t % NO;
          mbar_wait(&o_full[slot], (t / NO) & 1);
          fence_after();
          const uint32_t base = smem_u32(ops + (size_t)slot * OP_BYTES);
          const uint64_t b_hi = smem_desc(base + 2 * A_BYTES), b_lo = smem_desc(base + 2 * A_BYTES + H_BYTES);
#pragma unroll
          for (int mb = 0; mb < 2; ++mb) {
            const uint64_t a_hi = smem_desc(base + mb * MB_BYTES), a_lo = smem_desc(base + A_BYTES + mb * MB_BYTES);
            const uint32_t d = tmem + (uint32_t)(mb * N);
            mma(d, a_hi, b_hi, IDESC, c > 0 ? 1u : 0u);
            mma(d, a_hi, b_lo, IDESC, 1u);
            mma(d, a_lo, b_hi, IDESC, 1u);
          }
          commit(&o_empty[slot]);
        }
        commit(acc_full);
        ++it;
      }
    }
    __syncwarp();
  } else {
    // ===== builders + epilogue: NG groups of 8 warps take interleaved
    // pipeline steps (gp = warp >> 3: steps t with t % NG == gp), so NG
    // channels' operand chains are in flight at once.  Within a group thread
    // pt (0..255) owns point pt (A row, Q) and warp w8 = warp & 7 owns scan w8
    // of the group (its 32 Hankel rows and Gram entries).  Group 0 also runs
    // the epilogue (TMEM lane quarter w8 & 3 of M-block w8 >> 2).
    const int gp = warp >> 3, w8 = warp & 7;
    const int pt = w8 * 32 + lane;
    const int mb = pt >> 7, row = pt & 127;
    int t = 0, it = 0, my = 0;  // my: this group's step count (Gram buffer parity)
    for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
      const int tile = item % P.n_tiles, group = item / P.n_tiles;
      const int tile0 = tile * TILE;
      const int n_in = tile_points(p, tile, n_pts);
      if (n_in <= 0) continue;
      const int nsg = min(SPG, p.n_scans - group * SPG);
      const uint32_t* tw = p.tab_words + (size_t)tile * p.C * TILE;
      const int2* tsp = p.tab_span + (size_t)tile * p.C;
      float q[SPG < 4 ? 4 : SPG];
#pragma unroll
      for (int s = 0; s < SPG; ++s) q[s] = 0.f;
      bool bad = false, bad_span = false;
      // first channel of this item handled by this group
      int c = (gp - t % NG + NG) % NG;
      t += c;
      uint32_t w_next = c < p.C ? __ldg(tw + (size_t)c * TILE + pt) : 0u;
      int lo_next = c < p.C ? __ldg(&tsp[c].x) : 0;
      for (; c < p.C; c += NG, t += NG, ++my) {
        const int slot = t % NS, oslot = t % NO;
        const uint32_t w = w_next;
        const int lo_c = lo_next;
        if (c + NG < p.C) {
          w_next = __ldg(tw + (size_t)(c + NG) * TILE + pt);
          lo_next = __ldg(&tsp[c + NG].x);
        }
        int d = (int)(w >> 23);
        if (d > K - 2) {  // tile span beyond the K taps (the host checks mwb_table_max_span first)
          bad_span = true;
          d = K - 2;
        }
        const float f1 = weight_f1(w);
        const float f0 = 1.0f - f1;
        MWB_CHECK(d >= 0 && d + 1 < K);
        // ---- A row (weights), once the MMA released this operand slot
        if (t >= NO) mbar_wait(&o_empty[oslot], (t / NO - 1) & 1);
        unsigned char* op = ops + (size_t)oslot * OP_BYTES;
        {
          uint32_t f0h, f0l;
          split2(f0, f1, f0h, f0l);  // low half f0, high half f1
          const uint32_t f1h = f0h >> 16, f1l = f0l >> 16;
          f0h &= 0xFFFFu;
          f0l &= 0xFFFFu;
          // word j holds taps 2j (low) and 2j + 1 (high)
          const int j0 = d >> 1;
          const bool odd = d & 1;
          const uint32_t ph = odd ? (f0h << 16) : (f0h | (f1h << 16));
          const uint32_t pl = odd ? (f0l << 16) : (f0l | (f1l << 16));
          const uint32_t nh = odd ? f1h : 0u, nl = odd ? f1l : 0u;
          uint32_t hi[8], lo[8];
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            hi[j] = j == j0 ? ph : (j == j0 + 1 ? nh : 0u);
            lo[j] = j == j0 ? pl : (j == j0 + 1 ? nl : 0u);
          }
          unsigned char* ah = op + mb * MB_BYTES;
          unsigned char* al = op + A_BYTES + mb * MB_BYTES;
          *reinterpret_cast<uint4*>(ah + kmajor_off(row, 0)) = make_uint4(hi[0], hi[1], hi[2], hi[3]);
          *reinterpret_cast<uint4*>(ah + kmajor_off(row, 1)) = make_uint4(hi[4], hi[5], hi[6], hi[7]);
          *reinterpret_cast<uint4*>(al + kmajor_off(row, 0)) = make_uint4(lo[0], lo[1], lo[2], lo[3]);
          *reinterpret_cast<uint4*>(al + kmajor_off(row, 1)) = make_uint4(lo[4], lo[5], lo[6], lo[7]);
        }
        // ---- Hankel rows and Gram entries of scan w8, once staged
        mbar_wait(&s_full[slot], (t / NS) & 1);
        const int n_row = w8 * 32 + lane;  // H row (s, k) = (n / W, n % W)
        if (w8 * 32 < N && n_row < N) {
          // Hankel row k of scan s: taps m -> plane element o + m with
          // o = (lo_c - j_lo) % 8 + k; 9 aligned words per plane, shifted by
          // one half for odd o
          const int hs = n_row / W, k = n_row - hs * W;
          const int off = min(max(lo_c - P.j_lo, 0), P.J - 16);
          const int o = (off & 7) + k;
          const uint32_t* hw = reinterpret_cast<const uint32_t*>(stage_bytes + slot * STAGE_BYTES) +
                               hs * SPANH + (o >> 1);  // [scan][hi | lo][SPANH halves] = SPANH words per scan
          const bool odd = o & 1;
          MWB_CHECK(hs < SPG && (o >> 1) + 8 < SPANH / 2 && off + 16 <= P.J);  // 9 words inside each plane
          uint32_t hi[8], lo[8];
          {
            uint32_t u[9];
#pragma unroll
            for (int j = 0; j < 9; ++j) u[j] = hw[j];
#pragma unroll
            for (int j = 0; j < 8; ++j) hi[j] = odd ? __funnelshift_r(u[j], u[j + 1], 16) : u[j];
#pragma unroll
            for (int j = 0; j < 9; ++j) u[j] = hw[SPANH / 2 + j];
#pragma unroll
            for (int j = 0; j < 8; ++j) lo[j] = odd ? __funnelshift_r(u[j], u[j + 1], 16) : u[j];
          }
          unsigned char* hh = op + 2 * A_BYTES;
          unsigned char* hl = hh + H_BYTES;
          *reinterpret_cast<uint4*>(hh + kmajor_off(n_row, 0)) = make_uint4(hi[0], hi[1], hi[2], hi[3]);
          *reinterpret_cast<uint4*>(hh + kmajor_off(n_row, 1)) = make_uint4(hi[4], hi[5], hi[6], hi[7]);
          *reinterpret_cast<uint4*>(hl + kmajor_off(n_row, 0)) = make_uint4(lo[0], lo[1], lo[2], lo[3]);
          *reinterpret_cast<uint4*>(hl + kmajor_off(n_row, 1)) = make_uint4(lo[4], lo[5], lo[6], lo[7]);
        }
        fence_async_smem();  // A / H generic writes -> visible to the tensor core
        __syncwarp();
        if (lane == 0) mbar_arrive(&o_full[oslot]);
        {
          // Q += f0^2 e(d) + 2 f0 f1 x(d) + f1^2 e(d + 1), 4 scans per LDS.128
          const float w0 = f0 * f0, w1 = 2.f * f0 * f1, w2 = f1 * f1;
          const float4* gsl = reinterpret_cast<const float4*>(gstage) + slot * GQ_FLOAT4;
          MWB_CHECK(d >= 0 && d <= K - 2 && (QUADS - 1) * 32 + 2 * d + 2 < GQ_FLOAT4);
          if constexpr (SPG < 4) {
            // groups smaller than a quad: this group's scans start at component (group * SPG) % 4
            const int comp0 = (group * SPG) & 3;
            const float4 E = gsl[2 * d], X = gsl[2 * d + 1], E1 = gsl[2 * d + 2];
#pragma unroll
            for (int s = 0; s < SPG; ++s) {
              const int cp = comp0 + s;
              const float e = cp == 0 ? E.x : cp == 1 ? E.y : cp == 2 ? E.z : E.w;
              const float x = cp == 0 ? X.x : cp == 1 ? X.y : cp == 2 ? X.z : X.w;
              const float e1 = cp == 0 ? E1.x : cp == 1 ? E1.y : cp == 2 ? E1.z : E1.w;
              q[s] = fmaf(w0, e, fmaf(w1, x, fmaf(w2, e1, q[s])));
            }
          } else
#pragma unroll
          for (int qd = 0; qd < QUADS; ++qd) {
            const float4 E = gsl[qd * 32 + 2 * d], X = gsl[qd * 32 + 2 * d + 1], E1 = gsl[qd * 32 + 2 * d + 2];
            if (4 * qd + 0 < SPG) q[4 * qd + 0] = fmaf(w0, E.x, fmaf(w1, X.x, fmaf(w2, E1.x, q[4 * qd + 0])));
            if (4 * qd + 1 < SPG) q[4 * qd + 1] = fmaf(w0, E.y, fmaf(w1, X.y, fmaf(w2, E1.y, q[4 * qd + 1])));
            if (4 * qd + 2 < SPG) q[4 * qd + 2] = fmaf(w0, E.z, fmaf(w1, X.z, fmaf(w2, E1.z, q[4 * qd + 2])));
            if (4 * qd + 3 < SPG) q[4 * qd + 3] = fmaf(w0, E.w, fmaf(w1, X.w, fmaf(w2, E1.w, q[4 * qd + 3])));
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&s_empty[slot]);  // samples and Gram slices consumed
      }
      t -= (c - p.C);  // c overshot C by 0..NG-1: t is now the first step of the next item
      // ---- every group publishes its Q partial sums; group g then runs the
      // epilogue for the group's scans s = g, g + NG, ... (TMEM lane quarter
      // w8 & 3 of M-block w8 >> 2 is the same point in every group)
      float* qx = reinterpret_cast<float*>(smem + L.qx);
#pragma unroll
      for (int s = 0; s < SPG; ++s) qx[(gp * SPG + s) * TILE + pt] = q[s];
      builders_sync();
      mbar_wait(acc_full, it & 1);
      fence_after();
      const bool valid = pt < n_in;
      const int g = tile0 + (valid ? pt : 0);
      const int slot_out = valid ? (p.out_idx ? __ldg(p.out_idx + g) : g) : -1;
      const uint32_t lane_base = (uint32_t)((w8 & 3) * 32) << 16;
      for (int s = gp; s < nsg; s += NG) {  // warp-uniform
        float qs = 0.f;
#pragma unroll
        for (int g2 = 0; g2 < NG; ++g2) qs += qx[(g2 * SPG + s) * TILE + pt];
        float e0 = 0.f, e1 = 0.f;
#pragma unroll
        for (int kc = 0; kc < W; kc += 16) {
          float v[16];
          tmem_ld16(tmem + lane_base + (uint32_t)(mb * N + s * W + kc), v);
#pragma unroll
          for (int k = 0; k < 16; k += 2) {
            e0 = fmaf(v[k], v[k], e0);
            e1 = fmaf(v[k + 1], v[k + 1], e1);
          }
        }
        const int scan = group * SPG + s;
        const float inv = pow2f(-scale_exp(__ldg(P.absmax + scan)));
        const double E = ((double)e0 + (double)e1) * (double)inv * (double)inv;  // S was in scaled units
#pragma unroll
        for (int kk = 0; kk < 2; ++kk) {
          const bool want = kk == 0 ? KIND != KIND_DMAS : KIND != KIND_DAS;
          if (!want) continue;
          const float raw = kk == 0 ? __double2float_rn(E) : __double2float_rn(0.5 * (E - (double)qs));
          const float en = raw;
          float* out = (kk == 0 ? p.out_das : p.out_dmas) + (size_t)scan * (size_t)p.out_stride;
          unsigned long long* keys = kk == 0 ? p.key_das : p.key_dmas;
          unsigned long long key = 0ull;
          if (valid) {
            out[slot_out] = en;
            if (isfinite(en)) key = argmax_key(en, slot_out); else bad = true;
          }
          if (keys) {
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) key = max(key, __shfl_xor_sync(0xffffffffu, key, o));
            if (lane == 0 && key != 0ull) atomicMax(keys + scan, key);
          }
        }
      }
      builders_sync();  // every group has read qx before the next item overwrites it
      if (p.flags && (bad || bad_span)) atomicOr(p.flags, (bad ? 1 : 0) | (bad_span ? 2 : 0));
      fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(acc_empty);
      ++it;
    }
  }
  fence_before();
  __syncthreads();
  fence_after();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS));
}

// Windowed Gram entries of every (scan quad, channel) at window offsets
// j in [j_lo, j_lo + J) past k0: E(j) = sum_{k<W} y[k0+j+k]^2 and
// X(j) = sum_{k<W} y[k0+j+k] y[k0+j+k+1] (zeros past the record), the 4
// scans of the quad interleaved per float4, stored as {E, X} pairs.  They depend on the absolute
// window start only, so every tile's DMAS self-terms gather from them.  The
// same pass takes each scan's max |y| over the samples any window touches
// (bits; non-negative floats order like their bits), the input of the
// per-scan power-of-two scale.
__global__ void __launch_bounds__(128) gram_kernel(const float* sig, long long scan_stride, int n_scans, int C,
                                                   int ld, int k0, int win, int j_lo, int J, int R, float4* gx,
                                                   uint32_t* absmax) {
  extern __shared__ float yq[];  // [4][R], R >= J + win + 1: the planes' range (the |y| max covers it)
  __shared__ uint32_t wmax[4][4];
  const int c = blockIdx.x, quad = blockIdx.y, tid = threadIdx.x;
  const long long base = (long long)k0 + j_lo;
  uint32_t m[4];
#pragma unroll
  for (int sq = 0; sq < 4; ++sq) {
    m[sq] = 0u;
    const int s = quad * 4 + sq;
    const float* row = sig + (size_t)s * (size_t)scan_stride + (size_t)c * ld;
    for (int r = tid; r < R; r += blockDim.x) {
      const long long idx = base + r;
      const float v = (s < n_scans && idx < ld) ? __ldg(row + idx) : 0.f;
      yq[sq * R + r] = v;
      m[sq] = max(m[sq], __float_as_uint(fabsf(v)));
    }
  }
#pragma unroll
  for (int sq = 0; sq < 4; ++sq) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m[sq] = max(m[sq], __shfl_xor_sync(0xffffffffu, m[sq], o));
    if ((tid & 31) == 0) wmax[sq][tid >> 5] = m[sq];
  }
  __syncthreads();
  if (tid < 4) {
    const uint32_t v = max(max(wmax[tid][0], wmax[tid][1]), max(wmax[tid][2], wmax[tid][3]));
    if (quad * 4 + tid < n_scans && v) atomicMax(absmax + quad * 4 + tid, v);
  }
  const size_t row_out = ((size_t)quad * C + c) * J;
  for (int jj = tid; jj < J; jj += blockDim.x) {
    float e[4], x[4];
#pragma unroll
    for (int sq = 0; sq < 4; ++sq) {
      const float* y = yq + sq * R + jj;
      float a = 0.f, b = 0.f;
#pragma unroll 8
      for (int k = 0; k < win; ++k) {
        a = fmaf(y[k], y[k], a);
        b = fmaf(y[k], y[k + 1], b);
      }
      e[sq] = a;
      x[sq] = b;
    }
    gx[2 * (row_out + jj)] = make_float4(e[0], e[1], e[2], e[3]);
    gx[2 * (row_out + jj) + 1] = make_float4(x[0], x[1], x[2], x[3]);
  }
}

// Scaled fp16 hi / lo planes of each (scan, channel) over the samples the
// windows touch, k0 + j_lo + [0, Lp): v = y * 2^e_s (the scan's power-of-two
// scale), hi = fp16(v), lo = fp16(v - hi); zeros past the record.  Layout
// [S][C][hi | lo][Lp], the tensor-core kernel's staging source.
__global__ void __launch_bounds__(128) planes_kernel(const float* sig, long long scan_stride, int C, int ld, int k0,
                                                     int j_lo, int Lp, const uint32_t* absmax, __half* planes) {
  const int c = blockIdx.x, s = blockIdx.y;
  const float sc = pow2f(scale_exp(__ldg(absmax + s)));
  const float* row = sig + (size_t)s * (size_t)scan_stride + (size_t)c * ld;
  __half* hi = planes + ((size_t)s * C + c) * 2 * (size_t)Lp;
  __half* lo = hi + Lp;
  for (int i = threadIdx.x; i < Lp; i += blockDim.x) {
    const long long idx = (long long)k0 + j_lo + i;
    const float v = idx < ld ? __ldg(row + idx) * sc : 0.f;
    const __half h = __float2half_rn(v);
    hi[i] = h;
    lo[i] = __float2half_rn(v - __half2float(h));
  }
}

// smallest and largest per-channel span start lo over the table's non-empty
// tiles (out[0] atomicMin, out[1] atomicMax; the caller presets them)
__global__ void table_lo_range_kernel(const int2* span, const int2* tile_info, long long tiles, int C, int* out) {
  int mn = 0x7FFFFFFF, mx = -1;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < tiles * C;
       i += (long long)gridDim.x * blockDim.x) {
    const long long tile = i / C;
    if (tile_info && tile_info[tile].y <= 0) continue;
    const int lo = span[i].x;
    mn = min(mn, lo);
    mx = max(mx, lo);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, o));
    mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMin(out, mn);
    atomicMax(out + 1, mx);
  }
}

// largest per-channel delay spread (hi - lo) over the table's tiles; wide
// tiles report 1 << 30
__global__ void table_max_span_kernel(const int2* span, const int* wide, long long tiles, int C, int* out) {
  int m = 0;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < tiles * C;
       i += (long long)gridDim.x * blockDim.x) {
    const long long tile = i / C;
    const int2 sp = span[i];
    m = max(m, wide[tile] ? (1 << 30) : sp.y - sp.x);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) atomicMax(out, m);
}

}  // namespace tc
