// Tensor-core path for W = 32 batches (configs[3]) with the Hankel operand
// read in place.  Included by mwb_kernels.cu after mwb_tc.cuh, whose helpers
// (MMA / commit / fences, TMEM loads, the hi/lo split, the per-scan scale,
// the Gram pre-pass) it shares.
//
// Same product as mwb_tc.cuh (restating beamform.py:169-212):
//   S[p, (s, k)] = sum over K positions m of A[p, m] * B[m, (s, k)]
// with the operand layouts chosen so that B needs no building at all:
//   * the fp16 planes are time-major with the 8 scans of a group interleaved,
//     Y[t][s] (16 bytes per time row, planes8_kernel);
//   * B[m, n = 8k + s] = Y[b + m + k][s] is then an MN-major no-swizzle
//     operand whose core matrices (8 scans x 8 consecutive rows) start 16
//     bytes apart along N (SBO = 16, overlapping) and 8 rows apart along K
//     (LBO): the tensor core reads the Hankel windows straight out of the
//     TMA-staged planes (scripts/tc_hankel_probe.cu checks this bit-exactly,
//     and at the K-major operand's 128 clk per M128 x N256 x K16 MMA);
//   * the two 8-tap K halves of one MMA may come from two different channels'
//     staged spans: LBO is set per step to their address difference.  The
//     halves of a step are consecutive (one channel, or the next one); a
//     channel staged in ring slot 0 is also copied to a mirror slot past the
//     ring's end, so the second half always lies above the first (LBO > 0).
// K is therefore packed in 8-tap halves.  A work item is one M-block (128
// points of a table tile) and a pair of 8-scan groups.  Per (M-block, channel)
// the points' exact delay-offset range [dmin, dmax] (from the table words)
// needs one half when dmax - dmin <= 6 (taps dmin + [0, 8) hold every f0, f1
// pair) and two halves otherwise (<= 14, the tensor-core path's
// precondition).  Halves are laid out channel after channel and cut into
// K = 16 steps (plan_kernel), so an item costs ceil(halves / 2) MMA steps
// instead of one per channel (configs[3]: about 40 instead of 66).
//
// The A rows (interpolation weights, hi/lo, 8 KB per step) depend on the table
// and the plan only, so abuild_kernel writes them once per call for every
// (M-block, step), and an operand-producer warp copies step t's rows into
// operand slot t % NO (one bulk copy) once the MMAs of step t - NO completed.
// The MMAs of both scan groups read them (A_hi once for its four products,
// A_lo once for its two: the A collector buffer).  Three groups of 8 warps
// take interleaved steps: warp 0 of the step's group waits for the two staged
// channels and writes the B descriptor, and every thread (row, kh) adds the
// DMAS self-terms Q of the channels whose first half is in the step (Gram
// entries, as in mwb_tc.cuh) for its scan group kh; the step's o_full
// completes with the A copy and the group's 8 arrivals.  The issuer's one
// commit per step (done[t % DR]) frees the step's operand slot and, at a
// channel's last step, its staging slot.  Work items run in chunks of BCH
// M-blocks over all scan-group pairs, so the chunk's A rows stay in L2.
// TMEM: lane = row, column = 256 g + 8 k + s for scan s of group g.

namespace tch {

using tc::K;
constexpr int W = 32, SPG = 8, N = W * SPG;   // N = 256 per scan group: 8 scans x 32 window samples
constexpr int NGRP = 2;                       // scan groups per item (A reused by both)
constexpr int ROWS_M = 128;                   // points per item (one M-block)
#ifndef MWB_TCH_NS
#define MWB_TCH_NS 24
#endif
#ifndef MWB_TCH_NO
#define MWB_TCH_NO 4
#endif
constexpr int NS = MWB_TCH_NS;                // staging ring (one channel per slot)
constexpr int NO = MWB_TCH_NO;                // operand ring (A rows of one step)
constexpr int DR = 32;                        // step-completion barriers
static_assert(NS <= DR && NO <= DR && NS <= 32, "ring depths: a staged channel's release step is < DR steps old");
#ifndef MWB_TCH_PCH
#define MWB_TCH_PCH 8
#endif
constexpr int PCH = MWB_TCH_PCH;              // channels the producer stages per round (one per lane)
static_assert(32 % PCH == 0 && PCH <= NS, "producer rounds");
#ifndef MWB_TCH_GROUPS
#define MWB_TCH_GROUPS 3
#endif
constexpr int NG = MWB_TCH_GROUPS;            // builder groups (step t -> builder group t % NG)
constexpr int GW = 8;
constexpr int NBW = NG * GW, NBT = NBW * 32;
constexpr int THREADS = NBT + 96;             // + staging producer, MMA issuer, operand producer
constexpr int ROWS = 56;                      // staged rows per plane: r + m + k <= 22 + 7 + 31 (wide) / 14 + 7 + 31
constexpr int PLANE_B = ROWS * 16;            // 896 B per plane
constexpr int GPL_B = 2 * PLANE_B;            // hi | lo of one scan group
constexpr int STAGE_B = NGRP * GPL_B;         // both groups
constexpr int A_B = ROWS_M * K * 2;           // one of hi / lo: 4 KB
constexpr int OP_B = 2 * A_B;
constexpr int QUADS = NGRP * SPG / 4;         // Gram quads per item
constexpr int GQ_FLOAT4 = QUADS * 2 * 16;     // quads x 16 positions x {E, X}
constexpr int TMEM_COLS = 512;
// kind::f16, f32 accumulate, A K-major, B MN-major (bit 16), N = 256, M = 128
constexpr uint32_t IDESC = (1u << 4) | (1u << 16) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
constexpr size_t SMEM_MIN = 120 * 1024;

struct Layout {
  size_t ops, stage, g, qx, ex, meta, bar, tmem, total;
};
__host__ __device__ inline Layout layout() {
  Layout L;
  size_t o = 0;
  L.ops = o;   o += (size_t)NO * OP_B;
  L.stage = o; o += (size_t)(NS + 1) * STAGE_B;              // + the mirror of slot 0 (see the producer)
  L.g = o;     o += (size_t)NS * GQ_FLOAT4 * 16;
  L.qx = o;    o += (size_t)NG * NGRP * SPG * ROWS_M * 4;  // Q partials per builder group
  L.ex = o;    o += (size_t)NG * NGRP * SPG * ROWS_M * 4;  // DAS partial sums per builder group
  o = align_up(o, 8);
  L.meta = o;  o += sizeof(uint64_t) * NO;                 // per operand slot: the step's B descriptor
  L.bar = o;   o += sizeof(uint64_t) * (NS + DR + NO + 2);
  L.tmem = o;  o += 16;
  L.total = o < SMEM_MIN ? SMEM_MIN : align_up(o, 128);
  return L;
}

// plan half word: bit 31 valid, bit 30 the channel's first half, bit 27
// (c / NS) & 1 and bits 22..26 c % NS (the channel's staging-ring position
// relative to the item's first channel), bits 16..21 the half's first row r
// (offset past lo_c), bits 0..15 the channel c
__device__ __forceinline__ bool hv_valid(uint32_t h) { return h >> 31; }
__device__ __forceinline__ bool hv_first(uint32_t h) { return (h >> 30) & 1u; }
__device__ __forceinline__ int hv_row(uint32_t h) { return (int)((h >> 16) & 63u); }
__device__ __forceinline__ int hv_chan(uint32_t h) { return (int)(h & 0xFFFFu); }
__host__ __device__ constexpr uint32_t hv_ring_bits(int c) {
  return ((uint32_t)(c % NS) << 22) | ((uint32_t)((c / NS) & 1) << 27);
}
// Staging slot of a half's channel and the parity of its fill: the item's
// channels start at ring position tcb (tr = tcb % NS, tq = (tcb / NS) & 1), so
// channel c sits at (tcb + c) % NS, filled in phase ((tcb + c) / NS) & 1
__device__ __forceinline__ int hv_slot(uint32_t h, int tr, int tq, uint32_t& parity) {
  int s = tr + (int)((h >> 22) & 31u);
  const int carry = s >= NS ? 1 : 0;
  s -= carry * NS;
  parity = (uint32_t)(tq ^ (int)((h >> 27) & 1u) ^ carry);
  return s;
}

__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile("{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.u32 %0, 1, 0, P;\n\t}" : "=r"(pred));
  return pred != 0;
}

__device__ __forceinline__ void tma_load_4d(void* dst, const CUtensorMap* map, int x0, int x1, int x2, int x3,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], "
      "[%6];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x0), "r"(x1), "r"(x2), "r"(x3), "r"(smem_u32(bar))
      : "memory");
}

#ifndef MWB_TCH_COLLECTOR
#define MWB_TCH_COLLECTOR 1
#endif
// tcgen05.mma with an A-collector usage: FILL reads A from shared memory and
// keeps it, USE / LASTUSE take the kept A (LASTUSE then frees it); the MMAs of
// one fill..lastuse run are issued back to back with the same A descriptor
enum { CA_FILL, CA_USE, CA_LASTUSE };
template <int U>
__device__ __forceinline__ void mma_ca(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc, uint32_t accumulate) {
  if constexpr (U == CA_FILL)
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16.collector::a::fill [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
        "l"(a), "l"(b), "r"(idesc), "r"(accumulate));
  else if constexpr (U == CA_USE)
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16.collector::a::use [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
        "l"(a), "l"(b), "r"(idesc), "r"(accumulate));
  else
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16.collector::a::lastuse [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
        "l"(a), "l"(b), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void builders_sync_tch() { asm volatile("bar.sync 1, %0;" ::"n"(NBT) : "memory"); }

__device__ __forceinline__ uint64_t desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | ((uint64_t)1 << 46);
}

struct alignas(64) Params {
  CUtensorMap tm_planes;  // 4-D {4 Lp words, hi | lo, C, 2 n_pairs} (planes as 32-bit words): box {4 ROWS, 2, 1, NGRP}
  CUtensorMap tm_gram;    // as tc::Params::tm_gram, box {128, 1, QUADS}
  EnergyParams e;
  const uint32_t* absmax;
  const int* plan_n;       // [tiles * 2] steps per M-block
  const uint4* plan;       // [tiles * 2][C] step records {half 0, half 1, 0, 0}
  const int* plan_last;    // [tiles * 2][C] the last step reading each channel
  const unsigned char* a_ops;  // [tiles * 2][C][OP_B]: every step's A rows (abuild_kernel)
  int j_lo, J, Lp, n_tiles, n_pairs;
};

// Work items in chunks of BCH M-blocks: every pair of scan groups of a chunk,
// M-block fastest, so that the CTAs share one chunk's A operands (BCH x ~40
// steps x 8 KB) and one or two pairs' planes and Gram slices in L2.
#ifndef MWB_TCH_BCH
#define MWB_TCH_BCH 64
#endif
constexpr int BCH = MWB_TCH_BCH;
__device__ __forceinline__ void item_coords(int it, int n_blocks, int n_pairs, int& blk, int& pair) {
  const int per = BCH * n_pairs;
  const int ch = it / per, rem = it - ch * per;
  const int bbc = min(BCH, n_blocks - ch * BCH);
  pair = rem / bbc;
  blk = ch * BCH + (rem - pair * bbc);
}


// points of M-block mb of table tile `tile` (<= 0: nothing to do)
__device__ __forceinline__ int block_points(const EnergyParams& p, int tile, int mb, int n_pts) {
  return min(ROWS_M, tc::tile_points(p, tile, n_pts) - mb * ROWS_M);
}

#ifdef MWB_TCH_TRACE
// event log of CTA 0 (development aid): {clock64, code << 32 | arg}
__device__ unsigned long long tch_trace[2 * 8192];
__device__ unsigned int tch_trace_n;
__device__ __forceinline__ void trace_ev(int code, int arg) {
  if (blockIdx.x != 0) return;
  const unsigned int k = atomicAdd(&tch_trace_n, 1u);
  if (k < 8192) {
    tch_trace[2 * k] = (unsigned long long)clock64();
    tch_trace[2 * k + 1] = ((unsigned long long)code << 32) | (unsigned int)arg;
  }
}
#define TRACE(code, arg) trace_ev(code, arg)
#else
#define TRACE(code, arg)
#endif

#ifdef MWB_TCH_PROF
__device__ unsigned long long tch_prof[16];
#define PROF_T(k, stmt)                  \
  do {                                   \
    const long long _t0 = clock64();     \
    stmt;                                \
    prof[k] += clock64() - _t0;          \
  } while (0)
#else
#define PROF_T(k, stmt) stmt
#endif

template <int KIND>
__global__ void __launch_bounds__(THREADS, 1) energy_tch_kernel(const __grid_constant__ Params P) {
  extern __shared__ __align__(1024) unsigned char smem[];
  const EnergyParams& p = P.e;
  const Layout L = layout();
  unsigned char* ops = smem + L.ops;
  unsigned char* stage = smem + L.stage;
  const float4* gstage = reinterpret_cast<const float4*>(smem + L.g);
  uint64_t* meta = reinterpret_cast<uint64_t*>(smem + L.meta);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + L.bar);
  uint64_t* s_full = bar;
  uint64_t* done = bar + NS;  // done[t % DR]: the MMAs of step t completed (tcgen05.commit)
  uint64_t* o_full = bar + NS + DR;
  uint64_t* acc_full = bar + NS + DR + NO;
  uint64_t* acc_empty = acc_full + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + L.tmem);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int n_pts = p.d_count ? min(*p.d_count, p.P) : p.P;
  const int n_blocks = 2 * P.n_tiles;
  const int n_items = n_blocks * P.n_pairs;  // item -> (tile, M-block) fastest, then the scan-group pair

  if (tid == 0) {
    for (int i = 0; i < NS; ++i) mbar_init(&s_full[i], 1);
    for (int i = 0; i < DR; ++i) mbar_init(&done[i], 1);
    for (int i = 0; i < NO; ++i) mbar_init(&o_full[i], 1 + GW);  // the A copy's expect_tx + the step's Q warps
    mbar_init(acc_full, 1);
    mbar_init(acc_empty, NBW);
    fence_mbar_init();
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = *tmem_slot;
#ifdef MWB_TCH_PROF
  long long prof[16] = {0};
  const long long t_start = clock64();
#endif

  if (warp == NBW) {
    // ===== producer: per channel, both scan groups' planes of the span and
    // the four quads' Gram slices, PCH channels at a time (lane j issues
    // channel c0 + j).  A ring slot is reused once the MMAs of the last step
    // reading its previous channel completed (done[]; that step is < NS <= DR
    // steps before the MMA frontier, since the steps in between need at most
    // NS - 1 channels); releases come in channel order, so the chunk waits
    // for its last slot only.
    int t = 0, steps = 0;
    int rel = -1;  // lane s: the global step that releases ring slot s (NS <= 32)
    for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
      int blk, pair;
      item_coords(item, n_blocks, P.n_pairs, blk, pair);
      const int tile = blk >> 1, mb = blk & 1;
      if (block_points(p, tile, mb, n_pts) <= 0) continue;
      const int2* tsp = p.tab_span + (size_t)tile * p.C;
      const int* last = P.plan_last + (size_t)blk * p.C;
      int lo32 = 0, last32 = 0;
      for (int c0 = 0; c0 < p.C; c0 += PCH) {
        if ((c0 & 31) == 0) {
          lo32 = c0 + lane < p.C ? __ldg(&tsp[c0 + lane].x) : 0;
          last32 = c0 + lane < p.C ? __ldg(&last[c0 + lane]) : 0;
        }
        const int n = min(PCH, p.C - c0);
        const int src = (c0 & 31) + (lane < n ? lane : 0);
        const int lo_c = __shfl_sync(0xffffffffu, lo32, src);
        const int last_c = __shfl_sync(0xffffffffu, last32, src);
        const int prev = __shfl_sync(0xffffffffu, rel, (t + n - 1) % NS);
        if (prev >= 0) PROF_T(7, mbar_wait(&done[prev % DR], (prev / DR) & 1));
        const int j = (lane - t % NS + NS) % NS;  // the chunk channel whose slot is lane's
        const int last_j = __shfl_sync(0xffffffffu, last_c, j & 31);
        if (lane < NS && j < n) rel = steps + last_j;
#ifdef MWB_TCH_PROF
        const long long _pi = clock64();
#endif
        if (lane < n) {
          const int c = c0 + lane, slot = (t + lane) % NS;
          const int off = min(max(lo_c - P.j_lo, 0), P.J - 16);
          if (off != lo_c - P.j_lo && p.flags) atomicOr(p.flags, 4);
          // a channel in slot 0 also lands in the mirror slot NS: a step whose
          // second half (the next channel) wraps around the ring reads it there,
          // above its first half, so that the two halves' LBO is positive
          mbar_arrive_expect_tx(&s_full[slot], (uint32_t)((slot == 0 ? 2 : 1) * STAGE_B + GQ_FLOAT4 * 16));
          tma_load_4d(stage + slot * STAGE_B, &P.tm_planes, 4 * off, 0, c, NGRP * pair, &s_full[slot]);
          if (slot == 0) tma_load_4d(stage + NS * STAGE_B, &P.tm_planes, 4 * off, 0, c, NGRP * pair, &s_full[0]);
          tc::tma_load_3d(const_cast<float4*>(gstage) + slot * GQ_FLOAT4, &P.tm_gram, 8 * off, c, QUADS * pair,
                          &s_full[slot]);
        }
        __syncwarp();
#ifdef MWB_TCH_PROF
        prof[11] += clock64() - _pi;
#endif
        t += n;
      }
      steps += __ldg(P.plan_n + blk);
    }
  } else if (warp == NBW + 2) {
    // ===== operand producer: step t's A rows (hi | lo, 8 KB, built per
    // (M-block, step) by abuild_kernel: they depend on the table only) into
    // operand slot t % NO once the MMAs of step t - NO completed
    int t = 0;
    for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
      int blk, pair;
      item_coords(item, n_blocks, P.n_pairs, blk, pair);
      if (block_points(p, blk >> 1, blk & 1, n_pts) <= 0) continue;
      const int nst = __ldg(P.plan_n + blk);
      const unsigned char* src = P.a_ops + (size_t)blk * p.C * OP_B;
      for (int i = 0; i < nst; ++i, ++t) {
        const int slot = t % NO;
        if (t >= NO) PROF_T(14, mbar_wait(&done[(t - NO) % DR], ((t - NO) / DR) & 1));
        if (lane == 0) {
          mbar_arrive_expect_tx(&o_full[slot], (uint32_t)OP_B);
          bulk_g2s(ops + (size_t)slot * OP_B, src + (size_t)i * OP_B, (uint32_t)OP_B, &o_full[slot]);
          TRACE(9, t);
        }
        __syncwarp();
      }
    }
  } else if (warp == NBW + 1) {
    // ===== MMA issuer: the whole warp runs the loop (warp-uniform values),
    // one elected lane issues.  Per step 6 MMAs (2 scan groups x 3 split
    // products; the B descriptor from the step's builders) and one commit to
    // done[t % DR]
    int t = 0, it = 0;
    for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
      int blk, pair;
      item_coords(item, n_blocks, P.n_pairs, blk, pair);
      if (block_points(p, blk >> 1, blk & 1, n_pts) <= 0) continue;
      const int nst = __ldg(P.plan_n + blk);
      if (it > 0) PROF_T(1, mbar_wait(acc_empty, (it - 1) & 1));
      if (lane == 0) TRACE(2, it);
      tc::fence_after();
      for (int i = 0; i < nst; ++i, ++t) {
        const int slot = t % NO;
#ifdef MWB_TCH_PROF
        {
          const long long _t0 = clock64();
          mbar_wait(&o_full[slot], (t / NO) & 1);
          const long long dt = clock64() - _t0;
          prof[0] += dt;
          if (i == 0) prof[15] += dt;        // first step of an item
          else if (i < 3) prof[5] += dt;     // steps 1, 2
        }
#else
        mbar_wait(&o_full[slot], (t / NO) & 1);
#endif
        if (lane == 0) TRACE(1, t);
        tc::fence_after();
        const uint64_t b0 = meta[slot];
        const uint32_t base = smem_u32(ops + (size_t)slot * OP_B);
        const uint64_t a_hi = tc::smem_desc(base), a_lo = tc::smem_desc(base + A_B);
        if (elect_one()) {
#pragma unroll
          for (int g = 0; g < NGRP; ++g) {
            const uint64_t b_hi = b0 + (uint64_t)((g * GPL_B) >> 4);  // start-address field
            const uint64_t b_lo = b_hi + (PLANE_B >> 4);
            const uint32_t d = tmem + (uint32_t)(g * N);
#if MWB_TCH_COLLECTOR
            // A_hi is read from shared memory once for its four products and
            // A_lo once for its two (the A collector buffer), 64 instead of
            // 192 operand wavefronts per step
            if (g == 0) {
              mma_ca<CA_FILL>(d, a_hi, b_hi, IDESC, i > 0 ? 1u : 0u);
              mma_ca<CA_USE>(d, a_hi, b_lo, IDESC, 1u);
            } else {
              mma_ca<CA_USE>(d, a_hi, b_hi, IDESC, i > 0 ? 1u : 0u);
              mma_ca<CA_LASTUSE>(d, a_hi, b_lo, IDESC, 1u);
            }
#else
            tc::mma(d, a_hi, b_hi, IDESC, i > 0 ? 1u : 0u);
            tc::mma(d, a_hi, b_lo, IDESC, 1u);
            tc::mma(d, a_lo, b_hi, IDESC, 1u);
#endif
          }
#if MWB_TCH_COLLECTOR
          mma_ca<CA_FILL>(tmem, a_lo, b0, IDESC, 1u);
          mma_ca<CA_LASTUSE>(tmem + (uint32_t)N, a_lo, b0 + (uint64_t)(GPL_B >> 4), IDESC, 1u);
#endif
          tc::commit(&done[t % DR]);
          if (i + 1 == nst) tc::commit(acc_full);
        }
        __syncwarp();
      }
      ++it;
    }
  } else {
    // ===== Q gatherers + epilogue: NG groups of 8 warps take interleaved
    // steps (item step i -> group i % NG); warp 0 of the step's group waits for
    // its staged channels and writes its B descriptor; thread (row, kh) owns
    // the DMAS self-term partials and the epilogue of point `row` for scan
    // group kh
    const int gp = warp >> 3, w8 = warp & 7;
    const int pt = w8 * 32 + lane;
    const int row = pt & (ROWS_M - 1), kh = pt >> 7;
    int t = 0, tcb = 0, it = 0;
    for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
      int blk, pair;
      item_coords(item, n_blocks, P.n_pairs, blk, pair);
      const int tile = blk >> 1, mb = blk & 1;
      const int n_in = block_points(p, tile, mb, n_pts);
      if (n_in <= 0) continue;
      const int grp = NGRP * pair + kh;  // this thread's scan group
      const int nsg = min(SPG, p.n_scans - grp * SPG);
      const int nst = __ldg(P.plan_n + blk);
      const uint4* rec = P.plan + (size_t)blk * p.C;
      const int tr = tcb % NS, tq = (tcb / NS) & 1;
      float q[SPG];
#pragma unroll
      for (int s = 0; s < SPG; ++s) q[s] = 0.f;
      bool bad = false, bad_span = false;
      // step i of the item goes to builder group i % NG (a fixed assignment,
      // so every Q partial sum has the same operands in the same order
      // whatever the CTA processed before)
      int i = gp;
      // delay words straight from the table (L2), one group step ahead
      const uint32_t* twb = p.tab_words + (size_t)tile * p.C * TILE + mb * ROWS_M + row;
      uint2 rc = make_uint2(0u, 0u), rn = make_uint2(0u, 0u);
      if (i < nst) {
        const uint4 x = __ldg(rec + i);
        rc = make_uint2(x.x, x.y);
      }
      if (i + NG < nst) {
        const uint4 x = __ldg(rec + i + NG);
        rn = make_uint2(x.x, x.y);
      }
      // (the words of the channels whose first half is in the step: the Q gathers')
      auto first_word = [&](uint32_t h) {
        return hv_valid(h) && hv_first(h) ? __ldg(twb + (size_t)hv_chan(h) * TILE) : 0u;
      };
      uint32_t wc0 = first_word(rc.x), wc1 = first_word(rc.y);
      for (; i < nst; i += NG) {
        const uint2 cur = rc;
        const uint32_t wh0 = wc0, wh1 = wc1;
        wc0 = first_word(rn.x);
        wc1 = first_word(rn.y);
        rc = rn;
        rn = make_uint2(0u, 0u);
        if (i + 2 * NG < nst) {
          const uint4 x = __ldg(rec + i + 2 * NG);
          rn = make_uint2(x.x, x.y);
        }
        const int ts = t + i, oslot = ts % NO;
        if (ts >= NO) PROF_T(3, mbar_wait(&done[(ts - NO) % DR], ((ts - NO) / DR) & 1));
        if (w8 == 0 && lane == 0) TRACE(3, (gp << 20) | ts);
#ifdef MWB_TCH_PROF
        const long long _ta = clock64();
#endif
        if (w8 == 0) {
          // the step's B operand (group 0, hi plane): the two halves' rows in
          // address order -- they are consecutive (the same channel, or the
          // next one, whose slot wraps to the mirror slot NS); a missing
          // second half reads the next row (its A half is zero).  This warp
          // waits for both staged channels, so that the step's o_full implies
          // them.
          uint32_t p0, p1 = 0u;
          const int s0 = hv_slot(cur.x, tr, tq, p0);
          int s1 = s0;
          if (hv_valid(cur.y)) {
            s1 = hv_slot(cur.y, tr, tq, p1);
            if (s1 < s0) s1 += NS;
          }
          PROF_T(4, mbar_wait(&s_full[s0], p0));
          if (s1 != s0) PROF_T(4, mbar_wait(&s_full[s1 == NS ? 0 : s1], p1));
          const uint32_t a0 = (uint32_t)(s0 * STAGE_B + hv_row(cur.x) * 16);
          const uint32_t a1 = hv_valid(cur.y) ? (uint32_t)(s1 * STAGE_B + hv_row(cur.y) * 16) : a0 + 16u;
          if (lane == 0) meta[oslot] = desc(smem_u32(stage) + a0, a1 - a0, 16);
        }
#ifdef MWB_TCH_PROF
        const long long _tq = clock64();
        prof[12] += _tq - _ta;
#endif
        // ---- Q of the channels starting in this step, for scan group kh (read
        // before the step's arrival: the step's MMAs may then release a slot):
        // Q += f0^2 e(d) + 2 f0 f1 x(d) + f1^2 e(d + 1), 4 scans per LDS.128
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const uint32_t hw = h ? cur.y : cur.x;
          if (!hv_valid(hw) || !hv_first(hw)) continue;  // warp-uniform
          uint32_t par;
          const int slot = hv_slot(hw, tr, tq, par);
          PROF_T(4, mbar_wait(&s_full[slot], par));
          const uint32_t w = h ? wh1 : wh0;
          const int d = (int)(w >> 23);
          if (d - hv_row(hw) > K - 2 || d > K - 2) bad_span = true;  // beyond the two halves / the Gram slice
          const int dg = min(d, K - 2);
          const float f1 = weight_f1(w), f0 = 1.0f - f1;
          const float w0 = f0 * f0, w1 = 2.f * f0 * f1, w2 = f1 * f1;
          const float4* gsl = gstage + slot * GQ_FLOAT4 + kh * 2 * 16 * 2;
#pragma unroll
          for (int qd = 0; qd < 2; ++qd) {
            const float4* gr = gsl + qd * 32 + 2 * dg;
            const float4 E = gr[0], X = gr[1], E1 = gr[2];
            // FFMA2: two scans per instruction, each lane the scalar
            // fma(w0, E, fma(w1, X, fma(w2, E1, q)))
            const float2 w0v = make_float2(w0, w0), w1v = make_float2(w1, w1), w2v = make_float2(w2, w2);
            const float2 qa = __ffma2_rn(w0v, make_float2(E.x, E.y),
                                         __ffma2_rn(w1v, make_float2(X.x, X.y),
                                                    __ffma2_rn(w2v, make_float2(E1.x, E1.y),
                                                               make_float2(q[4 * qd + 0], q[4 * qd + 1]))));
            const float2 qb = __ffma2_rn(w0v, make_float2(E.z, E.w),
                                         __ffma2_rn(w1v, make_float2(X.z, X.w),
                                                    __ffma2_rn(w2v, make_float2(E1.z, E1.w),
                                                               make_float2(q[4 * qd + 2], q[4 * qd + 3]))));
            q[4 * qd + 0] = qa.x;
            q[4 * qd + 1] = qa.y;
            q[4 * qd + 2] = qb.x;
            q[4 * qd + 3] = qb.y;
          }
        }
#ifdef MWB_TCH_PROF
        prof[13] += clock64() - _tq;
#endif
        __syncwarp();
        if (lane == 0) mbar_arrive(&o_full[oslot]);  // this warp's Gram reads of step ts are done
        if (w8 == 0 && lane == 0) TRACE(4, (gp << 20) | ts);
      }
      t += nst;
      tcb += p.C;
      // ---- epilogue: builder group gp sums S^2 over the column chunks
      // kc = gp, gp + NG, ... (16 columns = 2 window samples x 8 scans) of
      // scan group kh; then it finishes scans s = gp, gp + NG, ... of group kh
      float* qx = reinterpret_cast<float*>(smem + L.qx);
      float* ex = reinterpret_cast<float*>(smem + L.ex);
#pragma unroll
      for (int s = 0; s < SPG; ++s) qx[((gp * NGRP + kh) * SPG + s) * ROWS_M + row] = q[s];
      // the output stage's global inputs, loaded while the last MMAs run: the
      // point's output slot and the inverse scales of this thread's scans
      const bool valid = row < n_in;
      const int g = tile * TILE + mb * ROWS_M + (valid ? row : 0);
      const int slot_out = valid ? (p.out_idx ? __ldg(p.out_idx + g) : g) : -1;
      float inv_s[(SPG + NG - 1) / NG];
#pragma unroll
      for (int k = 0; k < (SPG + NG - 1) / NG; ++k) {
        const int sc = gp + k * NG;
        inv_s[k] = sc < nsg ? tc::pow2f(-tc::scale_exp(__ldg(P.absmax + grp * SPG + sc))) : 0.f;
      }
      PROF_T(5, mbar_wait(acc_full, it & 1));
      if (w8 == 0 && lane == 0) TRACE(5, (gp << 20) | it);
#ifdef MWB_TCH_PROF
      const long long t_epi = clock64();
#endif
      tc::fence_after();
      {
        const uint32_t lane_base = (uint32_t)((w8 & 3) * 32) << 16;
        float e[SPG];
#pragma unroll
        for (int s = 0; s < SPG; ++s) e[s] = 0.f;
        for (int kc = gp; kc < N / 16; kc += NG) {
          float v[16];
          tc::tmem_ld16(tmem + lane_base + (uint32_t)(kh * N + kc * 16), v);
#pragma unroll
          for (int s = 0; s < SPG; s += 2) {  // FFMA2, each lane fma(v8, v8, fma(v, v, e))
            const float2 a = make_float2(v[s], v[s + 1]), b = make_float2(v[s + 8], v[s + 9]);
            const float2 r = __ffma2_rn(b, b, __ffma2_rn(a, a, make_float2(e[s], e[s + 1])));
            e[s] = r.x;
            e[s + 1] = r.y;
          }
        }
        // this warp's TMEM reads are complete (tcgen05.wait::ld): once every
        // builder warp has arrived the next item's MMAs may overwrite TMEM
        tc::fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(acc_empty);
        if (w8 == 0 && lane == 0) TRACE(6, (gp << 20) | it);
#pragma unroll
        for (int s = 0; s < SPG; ++s) ex[((gp * NGRP + kh) * SPG + s) * ROWS_M + row] = e[s];
      }
      builders_sync_tch();
      if (w8 == 0 && lane == 0) TRACE(7, (gp << 20) | it);
#pragma unroll
      for (int k = 0; k < (SPG + NG - 1) / NG; ++k) {
        const int s = gp + k * NG;
        if (s >= nsg) break;  // warp-uniform
        float qs = 0.f;
        double es = 0.0;
#pragma unroll
        for (int g2 = 0; g2 < NG; ++g2) {
          qs += qx[((g2 * NGRP + kh) * SPG + s) * ROWS_M + row];
          es += (double)ex[((g2 * NGRP + kh) * SPG + s) * ROWS_M + row];
        }
        const int scan = grp * SPG + s;
        const float inv = inv_s[k];
        const double E = es * (double)inv * (double)inv;  // S was in scaled units
#pragma unroll
        for (int kk = 0; kk < 2; ++kk) {
          const bool want = kk == 0 ? KIND != KIND_DMAS : KIND != KIND_DAS;
          if (!want) continue;
          const float en = kk == 0 ? __double2float_rn(E) : __double2float_rn(0.5 * (E - (double)qs));
          float* out = (kk == 0 ? p.out_das : p.out_dmas) + (size_t)scan * (size_t)p.out_stride;
          unsigned long long* keys = kk == 0 ? p.key_das : p.key_dmas;
          unsigned long long key = 0ull;
          if (valid) {
            out[slot_out] = en;
            if (isfinite(en)) key = argmax_key(en, slot_out); else bad = true;
          }
          if (keys) {  // warp max of the 64-bit keys: the high words, then the low words among the maxima
            const uint32_t hi = __reduce_max_sync(0xffffffffu, (uint32_t)(key >> 32));
            const uint32_t lo = __reduce_max_sync(0xffffffffu, (uint32_t)(key >> 32) == hi ? (uint32_t)key : 0u);
            key = ((unsigned long long)hi << 32) | lo;
            if (lane == 0 && key != 0ull) atomicMax(keys + scan, key);
          }
        }
      }
      builders_sync_tch();  // every group has read qx / ex before the next item overwrites them
      if (w8 == 0 && lane == 0) TRACE(8, (gp << 20) | it);
      if (p.flags && (bad || bad_span)) atomicOr(p.flags, (bad ? 1 : 0) | (bad_span ? 2 : 0));
#ifdef MWB_TCH_PROF
      prof[6] += clock64() - t_epi;
      prof[8] += 1;
      prof[9] += nst;
#endif
      ++it;
    }
  }
#ifdef MWB_TCH_PROF
  prof[2] = clock64() - t_start;
  // issuer lane 0: 0, 1, 2; builder warp 0 lane 0: 3..6, 8, 9, 10, 12, 13; producer lane 0: 7
  if (warp == NBW + 1 && lane == 0) {
    atomicAdd(&tch_prof[15], prof[15]);
    atomicAdd(&tch_prof[14], prof[5]);
    atomicAdd(&tch_prof[0], prof[0]);
    atomicAdd(&tch_prof[1], prof[1]);
    atomicAdd(&tch_prof[2], prof[2]);
  }
  if (warp == 0 && lane == 0) {
    for (int k = 3; k <= 6; ++k) atomicAdd(&tch_prof[k], prof[k]);
    atomicAdd(&tch_prof[8], prof[8]);
    atomicAdd(&tch_prof[9], prof[9]);
    atomicAdd(&tch_prof[10], prof[2]);
  }
  if (warp == NBW && lane == 0) {
    atomicAdd(&tch_prof[7], prof[7]);
    atomicAdd(&tch_prof[11], prof[11]);
    atomicAdd(&tch_prof[12], prof[2]);
  }
#endif
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS));
}

// The A operands of every (M-block, step), hi | lo in the K-major no-swizzle
// core-matrix layout the MMA reads (tc::kmajor_off): thread (row, kh) writes
// K half kh of row `row` -- the interpolation weights f0 at tap d - r and f1
// at d - r + 1 of the plan half's 8 taps (those inside them).  They depend on
// the table and the plan only, not on the scans.
__global__ void __launch_bounds__(256) abuild_kernel(const uint32_t* __restrict__ words, int C,
                                                     const int* __restrict__ plan_n, const uint4* __restrict__ plan,
                                                     unsigned char* __restrict__ a_ops) {
  const int blk = blockIdx.x, tile = blk >> 1, mb = blk & 1;
  const int row = threadIdx.x & (ROWS_M - 1), kh = threadIdx.x >> 7;
  const int nst = plan_n[blk];
  const uint32_t* tw = words + (size_t)tile * C * TILE + mb * ROWS_M + row;
  for (int i = 0; i < nst; ++i) {
    const uint4 r = __ldg(plan + (size_t)blk * C + i);
    const uint32_t hw = kh ? r.y : r.x;
    uint32_t hi[4] = {0u, 0u, 0u, 0u}, lo[4] = {0u, 0u, 0u, 0u};
    if (hv_valid(hw)) {
      const uint32_t w = __ldg(tw + (size_t)hv_chan(hw) * TILE);
      const int rel = (int)(w >> 23) - hv_row(hw);  // f0 at tap rel of this half, f1 at rel + 1
      const float f1 = weight_f1(w);
      uint32_t f0h, f0l;
      tc::split2(1.0f - f1, f1, f0h, f0l);  // low half f0, high half f1
      const uint32_t f1h = f0h >> 16, f1l = f0l >> 16;
      f0h &= 0xFFFFu;
      f0l &= 0xFFFFu;
      const int j0 = rel >> 1;  // arithmetic: rel may be -1 .. 21
      const bool odd = rel & 1;
      const uint32_t ph = odd ? (f0h << 16) : (f0h | (f1h << 16));
      const uint32_t pl = odd ? (f0l << 16) : (f0l | (f1l << 16));
      const uint32_t nh = odd ? f1h : 0u, nl = odd ? f1l : 0u;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        hi[j] = j == j0 ? ph : (j == j0 + 1 ? nh : 0u);
        lo[j] = j == j0 ? pl : (j == j0 + 1 ? nl : 0u);
      }
    }
    unsigned char* op = a_ops + ((size_t)blk * C + i) * OP_B;
    *reinterpret_cast<uint4*>(op + tc::kmajor_off(row, kh)) = make_uint4(hi[0], hi[1], hi[2], hi[3]);
    *reinterpret_cast<uint4*>(op + A_B + tc::kmajor_off(row, kh)) = make_uint4(lo[0], lo[1], lo[2], lo[3]);
  }
}

// Scaled fp16 hi / lo planes, time-major with the 8 scans of a group
// interleaved: [G][C][hi | lo][Lp][8] over samples k0 + j_lo + [0, Lp); zeros
// past the record and for the missing scans (and groups) of the last pair.
__global__ void __launch_bounds__(256) planes8_kernel(const float* sig, long long scan_stride, int n_scans, int C,
                                                      int ld, int k0, int j_lo, int Lp, const uint32_t* absmax,
                                                      __half* planes) {
  const int c = blockIdx.x, g = blockIdx.y;
  __half* hi = planes + ((size_t)g * C + c) * 2 * (size_t)Lp * 8;
  __half* lo = hi + (size_t)Lp * 8;
  for (int i = threadIdx.x; i < Lp * 8; i += blockDim.x) {
    const int tr = i >> 3, s = i & 7, scan = g * 8 + s;
    const long long idx = (long long)k0 + j_lo + tr;
    float v = 0.f;
    if (scan < n_scans && idx < ld)
      v = __ldg(sig + (size_t)scan * (size_t)scan_stride + (size_t)c * ld + idx) *
          tc::pow2f(tc::scale_exp(__ldg(absmax + scan)));
    const __half h = __float2half_rn(v);
    hi[i] = h;
    lo[i] = __float2half_rn(v - __half2float(h));
  }
}

// The step plan of every (table tile, M-block) (see the header): one CTA per
// M-block; a warp per channel takes the exact delay-offset range of the
// block's words (padded slots repeat the tile's first point), one warp lays
// the halves out, every thread writes step records and last steps.
__global__ void __launch_bounds__(256) plan_kernel(const uint32_t* __restrict__ words,
                                                   const int2* __restrict__ tile_info, int n_pts, int C,
                                                   int* __restrict__ plan_n, uint4* __restrict__ plan,
                                                   int* __restrict__ plan_last) {
  extern __shared__ int sh[];  // [C] first row | [C] halves | [C] first half index | [2 C] half -> channel
  int* r0 = sh;
  int* cnt = sh + C;
  int* h0 = sh + 2 * C;
  int* hch = sh + 3 * C;
  __shared__ int n_half;
  const int blk = blockIdx.x, tile = blk >> 1, mb = blk & 1, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int in_tile = tile_info ? min(TILE, tile_info[tile].y) : min(TILE, n_pts - tile * TILE);
  if (in_tile - mb * ROWS_M <= 0) {
    if (tid == 0) plan_n[blk] = 0;
    return;
  }
  const uint32_t* tw = words + (size_t)tile * C * TILE + mb * ROWS_M;
  for (int c = warp; c < C; c += 8) {
    int mn = 1 << 30, mx = -1;
#pragma unroll
    for (int k = 0; k < ROWS_M / 32; ++k) {
      const int d = (int)(__ldg(tw + (size_t)c * TILE + k * 32 + lane) >> 23);
      mn = min(mn, d);
      mx = max(mx, d);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, o));
      mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    }
    // one half when every f0, f1 pair fits taps mn + [0, 8); else two halves
    // from mn (a spread above 14 is flagged by the kernel)
    if (lane == 0) {
      r0[c] = min(mn, 31);
      cnt[c] = mx - mn <= 6 ? 1 : 2;
    }
  }
  __syncthreads();
  if (warp == 0) {
    int carry = 0;
    for (int cb = 0; cb < C; cb += 32) {
      const int c = cb + lane;
      const int nh = c < C ? cnt[c] : 0;
      int incl = nh;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += v;
      }
      if (c < C) {
        const int first = carry + incl - nh;
        h0[c] = first;
        hch[first] = c;
        if (nh == 2) hch[first + 1] = c | (1 << 16);  // second half
      }
      carry += __shfl_sync(0xffffffffu, incl, 31);
    }
    if (lane == 0) n_half = carry;
  }
  __syncthreads();
  const int nh = n_half, nst = (nh + 1) >> 1;
  uint4* out = plan + (size_t)blk * C;
  for (int s = tid; s < nst; s += blockDim.x) {
    uint32_t hw[2];
    for (int k = 0; k < 2; ++k) {
      const int hi_ = 2 * s + k;
      if (hi_ >= nh) {
        hw[k] = 0u;
        continue;
      }
      const int c = hch[hi_] & 0xFFFF, second = hch[hi_] >> 16;
      hw[k] = (1u << 31) | (second ? 0u : (1u << 30)) | hv_ring_bits(c) | ((uint32_t)(r0[c] + 8 * second) << 16) |
              (uint32_t)c;
    }
    out[s] = make_uint4(hw[0], hw[1], 0u, 0u);
  }
  // the step whose completion releases channel c's staging slot: its last
  // (the Q gathers of its first step precede that step's MMAs: o_full)
  for (int c = tid; c < C; c += blockDim.x)
    plan_last[(size_t)blk * C + c] = (h0[c] + cnt[c] - 1) >> 1;
  if (tid == 0) plan_n[blk] = nst;
}

}  // namespace tch
