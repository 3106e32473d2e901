// mwb_lattice.cuh — lattice / voxel / per-scan region enumeration (beamform.py:268-280, 309-323)
// (included by mwb_kernels.cu inside its anonymous namespace; one translation unit)
#pragma once

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
