// mwb_select.cuh — K2 / K2w device select_roi (coarse2fine.py:169-256), quadrants and octants
// (included by mwb_kernels.cu inside its anonymous namespace; one translation unit)
#pragma once

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
// K2s: 2-D select_roi on summed-area tables (single scans and batches, one
// CTA per scan).  Every statistic the selection needs is a box statistic of
// the coarse lattice: count, mean and sum of squared deviations of a child
// quadrant, of a child's expansion, of the current selection.  Three
// summed-area tables over the staged breast box — valid count, sum of
// (x - c) and sum of (x - c)^2 in fp64, with c the breast box's mean (a shift
// that keeps the one-pass m2 = Q - S^2 / n free of cancellation) — turn each
// into four lookups, so an iteration costs O(1) instead of two passes over
// the cells.  The tables are built once (row then column prefix sums, all
// threads); warp 0 then runs the iterations: lane k evaluates box k (four
// children, four expansions) and makes select_score's decision (Eq. (5), the
// first-index argmax, the n_min stop, W/B with the OR test) with the same
// arithmetic as the cell-walking K2.  Decisions match the reference's two-pass numpy
// statistics up to fp64 rounding (near-ties are the parity bar's excuse).
// ----------------------------------------------------------------------------
constexpr int SAT_TPB = 256;
constexpr int SAT_MAX_CELLS = 4096;  // staged lattice cells (tables: 20 B per (Lx+1)(Ly+1) entry)

__host__ __device__ inline size_t sat_smem_bytes(int lx, int ly) {
  const size_t e = (size_t)(lx + 1) * (ly + 1);
  return e * (2 * sizeof(double) + sizeof(int));
}

struct SatView {
  const int* c;
  const double* s;
  const double* q;
  int ly1;  // Ly + 1 (row length)
  // box of lattice indices [x0, x1] x [y0, y1] relative to the staged origin
  __device__ __forceinline__ void box(int x0, int y0, int x1, int y1, double& n, double& S, double& Q) const {
    if (x1 < x0 || y1 < y0) {
      n = S = Q = 0.0;
      return;
    }
    const int a = x0 * ly1 + y0, b = x0 * ly1 + y1 + 1, cc = (x1 + 1) * ly1 + y0, d = (x1 + 1) * ly1 + y1 + 1;
    n = (double)(c[d] - c[b] - c[cc] + c[a]);
    S = __dadd_rn(__dsub_rn(__dsub_rn(s[d], s[b]), s[cc]), s[a]);
    Q = __dadd_rn(__dsub_rn(__dsub_rn(q[d], q[b]), q[cc]), q[a]);
  }
};

__global__ void __launch_bounds__(SAT_TPB) select_roi_sat_kernel(const SelectParams p) {
  const int s = blockIdx.x;
  const float* dense = p.dense + (size_t)s * p.dense_stride;
  int32_t* region_out = p.region_out + 6 * s;
  mwb_trace_t* tr = p.trace + s;
  const int D = p.D, Lx = p.sL[0], Ly = p.sL[1], sl0x = p.sl0[0], sl0y = p.sl0[1];
  const int ly1 = Ly + 1, n_cells = Lx * Ly;
  extern __shared__ __align__(16) unsigned char smem_sat[];
  double* ts = reinterpret_cast<double*>(smem_sat);
  double* tq = ts + (size_t)(Lx + 1) * ly1;
  int* tc = reinterpret_cast<int*>(tq + (size_t)(Lx + 1) * ly1);
  __shared__ double red_d[SAT_TPB / 32];
  __shared__ int red_i[SAT_TPB / 32];
  __shared__ float red_f[2][SAT_TPB / 32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

  // stage: each cell's value (NaN when it holds none) into the sum table's
  // interior, then the breast box's count, sum (fixed order) and min / max
  float mn = INFINITY, mx = -INFINITY;
  double sm = 0.0;
  int cnt = 0;
#pragma unroll 4
  for (int i = tid; i < n_cells; i += SAT_TPB) {
    const int lx = i / Ly, ly = i - lx * Ly;
    const size_t slot = (size_t)(sl0x + lx) * D * p.ny + (size_t)(sl0y + ly) * D;
    const uint8_t okb = __ldg(p.valid + slot);  // both loads issued back to back
    const float raw = __ldg(dense + slot);       // (unwritten cells are never used)
    const bool ok = okb != 0;
    const float v = ok ? raw : 0.f;
    ts[(lx + 1) * ly1 + ly + 1] = ok ? (double)v : __longlong_as_double(0x7ff8000000000000LL);
    if (ok) {
      ++cnt;
      sm += (double)v;
      mn = fminf(mn, v);
      mx = fmaxf(mx, v);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    sm += __shfl_xor_sync(0xffffffffu, sm, o);
    cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
    mn = fminf(mn, __shfl_xor_sync(0xffffffffu, mn, o));
    mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  }
  if (lane == 0) {
    red_d[warp] = sm;
    red_i[warp] = cnt;
    red_f[0][warp] = mn;
    red_f[1][warp] = mx;
  }
  __syncthreads();
  double n_all = 0.0, s_all = 0.0;
  mn = INFINITY;
  mx = -INFINITY;
  for (int w = 0; w < SAT_TPB / 32; ++w) {  // every thread, same order
    n_all += (double)red_i[w];
    s_all += red_d[w];
    mn = fminf(mn, red_f[0][w]);
    mx = fmaxf(mx, red_f[1][w]);
  }
  if (n_all == 0.0 || mx == mn) {  // coarse2fine.py:186-192
    if (tid == 0) {
      tr->termination = n_all == 0.0 ? MWB_TERM_EMPTY : MWB_TERM_DEGENERATE;
      tr->n_records = 0;
      put_box(tr->final_region, p.breast);
      put_box(region_out, p.breast);
    }
    return;
  }
  const double c0 = s_all / n_all;  // the shift
  // interior entries -> (count, x - c0, (x - c0)^2); zero borders
  for (int i = tid; i < (Lx + 1) * ly1; i += SAT_TPB) {
    const int x = i / ly1, y = i - x * ly1;
    if (x == 0 || y == 0) {
      ts[i] = 0.0;
      tq[i] = 0.0;
      tc[i] = 0;
    } else {
      const double v = ts[i];
      const bool ok = v == v;
      const double d = ok ? __dsub_rn(v, c0) : 0.0;
      ts[i] = d;
      tq[i] = __dmul_rn(d, d);
      tc[i] = ok ? 1 : 0;
    }
  }
  __syncthreads();
  for (int x = tid + 1; x <= Lx; x += SAT_TPB) {  // prefix along y, one row per thread
    double a = 0.0, b = 0.0;
    int k = 0;
    for (int y = 1; y <= Ly; ++y) {
      const int i = x * ly1 + y;
      a = __dadd_rn(a, ts[i]);
      b = __dadd_rn(b, tq[i]);
      k += tc[i];
      ts[i] = a;
      tq[i] = b;
      tc[i] = k;
    }
  }
  __syncthreads();
  for (int y = tid + 1; y <= Ly; y += SAT_TPB) {  // then along x, one column per thread
    double a = 0.0, b = 0.0;
    int k = 0;
    for (int x = 1; x <= Lx; ++x) {
      const int i = x * ly1 + y;
      a = __dadd_rn(a, ts[i]);
      b = __dadd_rn(b, tq[i]);
      k += tc[i];
      ts[i] = a;
      tq[i] = b;
      tc[i] = k;
    }
  }
  __syncthreads();
  if (warp != 0) return;

  const SatView T{tc, ts, tq, ly1};
  // lattice-index box of a cell box, relative to the staged origin
  auto lat = [&](const Box& r, int& x0, int& y0, int& x1, int& y1) {
    x0 = (r.lo[0] + D - 1) / D - sl0x;
    x1 = r.hi[0] / D - sl0x;
    y0 = (r.lo[1] + D - 1) / D - sl0y;
    y1 = r.hi[1] / D - sl0y;
  };
  // the selection's statistics: n, shifted sum, m2 (one-pass on shifted data)
  double n_sel, sum_sel, m2_sel;
  {
    int x0, y0, x1, y1;
    lat(p.breast, x0, y0, x1, y1);
    double Q;
    T.box(x0, y0, x1, y1, n_sel, sum_sel, Q);
    m2_sel = fmax(__dsub_rn(Q, __dmul_rn(__ddiv_rn(sum_sel, n_sel), sum_sel)), 0.0);
  }
  // Iterations, lane-parallel: lane k < 4 owns child quadrant k, lane 4 + k
  // its expansion (expand_box of child k within the selection); every other
  // quantity is warp-uniform.  The arithmetic is select_score's (Eq. (5),
  // np.argmax ties to the lower index, the n_min stop, W/B with the OR test).
  int sx0 = p.breast.lo[0], sy0 = p.breast.lo[1], sx1 = p.breast.hi[0], sy1 = p.breast.hi[1];
  double sigma_prev_sq = m2_sel / n_sel;
  double prev_w = 0.0, prev_b = 0.0;
  bool have_prev = false;
  int iteration = 0, term = MWB_TERM_NONE;
  const int kq = lane & 3;
  while (true) {
    const int wx = sx1 - sx0 + 1, wy = sy1 - sy0 + 1;
    if (wx < 2 || wy < 2) {  // Region.quadrants() is None (geometry.py:233-234)
      term = MWB_TERM_REGION_FLOOR;
      break;
    }
    const int mxs = sx0 + (wx + 1) / 2 - 1, mys = sy0 + (wy + 1) / 2 - 1;  // last cells of the low halves
    // child kq (index = xhigh + 2 yhigh, geometry.py:235-240)
    int bx0 = (kq & 1) ? mxs + 1 : sx0, bx1 = (kq & 1) ? sx1 : mxs;
    int by0 = (kq & 2) ? mys + 1 : sy0, by1 = (kq & 2) ? sy1 : mys;
    const int cx0 = bx0, cy0 = by0, cx1 = bx1, cy1 = by1;
    if (lane >= 4) {  // its expansion: ceil(f * side) per axis, clipped (geometry.py:244-257)
      const int gx = (int)ceil(__dmul_rn(p.frac, (double)(bx1 - bx0 + 1)));
      const int gy = (int)ceil(__dmul_rn(p.frac, (double)(by1 - by0 + 1)));
      bx0 = max(bx0 - gx, sx0);
      bx1 = min(bx1 + gx, sx1);
      by0 = max(by0 - gy, sy0);
      by1 = min(by1 + gy, sy1);
    }
    double bn = 0.0, bs = 0.0, bm2 = 0.0, bmu = 0.0;
    if (lane < 8) {
      double Q;
      T.box((bx0 + D - 1) / D - sl0x, (by0 + D - 1) / D - sl0y, bx1 / D - sl0x, by1 / D - sl0y, bn, bs, Q);
      if (bn > 0.0) {
        const double ms = __ddiv_rn(bs, bn);  // shifted mean
        bmu = __dadd_rn(c0, ms);
        bm2 = fmax(__dsub_rn(Q, __dmul_rn(ms, bs)), 0.0);  // Q - S^2 / n
      }
    }
    // lanes 0..3: scores (coarse2fine.py:212-224)
    int has = 0, clamped = 0;
    double var = 0.0, dr = 0.0, dl = 0.0, sc = -INFINITY;
    if (lane < 4 && bn > 0.0) {
      var = __ddiv_rn(bm2, bn);
      if (iteration == 0) {
        sc = var;
        has = 1;
      } else {
        has = 2;
        if (var == 0.0) {
          sc = bmu;
        } else {
          dr = __ddiv_rn(__dsub_rn(var, sigma_prev_sq), var);
          dl = fmin(fmax(dr, 0.0), 1.0);
          sc = __dadd_rn(__dmul_rn(__dsub_rn(1.0, dl), bmu), __dmul_rn(dl, var));
          clamped = dl != dr;
        }
      }
    }
    mwb_iter_record_t* rec = iteration < MWB_MAX_ITERS ? &tr->records[iteration] : nullptr;
    if (rec && lane < MWB_MAX_CHILDREN) {
      const bool kid = lane < 4;
      rec->counts[lane] = kid ? (int)bn : 0;
      rec->has_stats[lane] = has;
      rec->clamped[lane] = clamped;
      rec->scores[lane] = kid ? sc : 0.0;
      rec->mu[lane] = kid ? bmu : 0.0;
      rec->var[lane] = var;
      rec->delta_raw[lane] = dr;
      rec->delta[lane] = dl;
    }
    // np.argmax over the 4 scores: larger wins, ties to the lower index
    double best = lane < 4 ? sc : -INFINITY;
    int selq = lane < 4 ? lane : 0x7FFF;
#pragma unroll
    for (int o = 2; o > 0; o >>= 1) {
      const double ob = __shfl_xor_sync(0xffffffffu, best, o);
      const int oq = __shfl_xor_sync(0xffffffffu, selq, o);
      if (ob > best || (ob == best && oq < selq)) {
        best = ob;
        selq = oq;
      }
    }
    selq = __shfl_sync(0xffffffffu, selq, 0);
    if (selq >= 4) selq = 0;  // every score -inf: argmax returns 0
    const double n_q = __shfl_sync(0xffffffffu, bn, selq);
    if (n_q < (double)p.n_min) {  // coarse2fine.py:227-229
      term = MWB_TERM_N_MIN;
      break;
    }
    const int e = 4 + selq;
    const double n_e = __shfl_sync(0xffffffffu, bn, e), sum_e = __shfl_sync(0xffffffffu, bs, e);
    const double m2_e = __shfl_sync(0xffffffffu, bm2, e);
    // W, B of the previous vs the new selection (class_distances, 94-109)
    const double w = __dadd_rn(m2_sel, m2_e);
    const double ma = __ddiv_rn(sum_sel, n_sel), mb = __ddiv_rn(sum_e, n_e);
    const double grand = __ddiv_rn(__dadd_rn(sum_sel, sum_e), __dadd_rn(n_sel, n_e));
    const double da = __dsub_rn(ma, grand), db = __dsub_rn(mb, grand);
    const double b = __dadd_rn(__dmul_rn(n_sel, __dmul_rn(da, da)), __dmul_rn(n_e, __dmul_rn(db, db)));
    const bool satisfied = !have_prev || (b > prev_b || w < prev_w);  // OR (235)
    const int ex0 = __shfl_sync(0xffffffffu, bx0, e), ey0 = __shfl_sync(0xffffffffu, by0, e);
    const int ex1 = __shfl_sync(0xffffffffu, bx1, e), ey1 = __shfl_sync(0xffffffffu, by1, e);
    if (rec && lane == selq) {  // the selected child's lane holds its box
      const Box cb{{cx0, cy0, 0}, {cx1, cy1, 0}};
      put_box(rec->selected_region, cb);
    }
    if (rec && lane == 0) {
      rec->iteration = iteration + 1;
      rec->n_children = 4;
      rec->selected = selq;
      rec->satisfied = satisfied;
      put_box(rec->expanded_region, Box{{ex0, ey0, 0}, {ex1, ey1, 0}});
      rec->w = w;
      rec->b = b;
    }
    if (!rec) {
      term = MWB_TERM_OVERFLOW;
      break;
    }
    iteration += 1;
    if (!satisfied) {
      term = MWB_TERM_DISTANCE;
      break;
    }
    prev_w = w;
    prev_b = b;
    have_prev = true;
    n_sel = n_e;
    sum_sel = sum_e;
    m2_sel = m2_e;
    sigma_prev_sq = m2_sel / n_sel;
    sx0 = ex0;
    sy0 = ey0;
    sx1 = ex1;
    sy1 = ey1;
  }
  const Box sel{{sx0, sy0, 0}, {sx1, sy1, 0}};
  if (lane == 0) {
    tr->termination = term;
    tr->n_records = min(iteration, MWB_MAX_ITERS);
    put_box(tr->final_region, sel);
    put_box(region_out, sel);
  }
}
