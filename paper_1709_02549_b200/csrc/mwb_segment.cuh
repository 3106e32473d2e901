// mwb_segment.cuh — K4 BASELINE configs[2] segmentation, single-scan, batched and region-tree kernels
// (included by mwb_kernels.cu inside its anonymous namespace; one translation unit)
#pragma once

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
