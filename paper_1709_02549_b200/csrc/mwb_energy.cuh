// mwb_energy.cuh — K0 delay table, K1 staged-gather energy kernel, window-split reduce (beamform.py:169-212)
// (included by mwb_kernels.cu inside its anonymous namespace; one translation unit)
#pragma once

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
  MWB_CHECK(!p.tile_src || (long long)tile < p.src_tiles);
  const bool wide = __ldg(p.tab_wide + tile) != 0;
  const uint32_t* tw = p.tab_words + tile * (size_t)p.C * TILE;
  const int2* tsp = p.tab_span + tile * (size_t)p.C;

  const int la = tid, lb = tid + TPB;
  const bool va = la < n_in_tile, vb = lb < n_in_tile;
  // (source point indices are re-derived in the gather path below: keeping
  // them live across the sample loop costs the register-capped kernels spills)
  const int oa = va ? (p.out_idx ? __ldg(p.out_idx + (int)tile * TILE + la) : tile0 + la) : -1;
  const int ob = vb ? (p.out_idx ? __ldg(p.out_idx + (int)tile * TILE + lb) : tile0 + lb) : -1;
  // ROI filter: which of this thread's points are written; a CTA with none exits
  const bool wa = va && (!p.filt_region || filter_keep(p, oa));
  const bool wb = vb && (!p.filt_region || filter_keep(p, ob));
  if (p.filt_region && !__syncthreads_or(wa || wb)) return;

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
      MWB_CHECK(q < n_chunks && s < p.n_scans);
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
        if (p.filt_region) filter_mark(p, wa, oa, wb, ob);
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
          if (wa) {
            out[oa] = ea;
            if (isfinite(ea)) key = argmax_key(ea, oa); else bad = true;
          }
          if (wb) {
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
    MWB_CHECK(!p.tile_src || !v || src < p.src_tiles * TILE);
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
  int o = v ? (p.out_idx ? __ldg(p.out_idx + src) : i) : -1;
  if (p.filt_region) {
    v = v && filter_keep(p, o);
    filter_mark(p, v, o, false, 0);
  }
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
