// Wire formats either side of the imaging path.
// Included by mwb_kernels.cu.
//
// (1) .mwb payload staging (reference io.py:65-86 reads the container; the
//     imaging kernels consume populated channels only): the raw fp64 (M*M, N)
//     series, copied to the device as bytes, is compacted to the fp32 [C][ld]
//     layout of every energy kernel.  A channel is populated when any sample
//     is nonzero (all-zero channels add exactly 0 to DAS and DMAS,
//     beamform.py:199-212); the order stays the reference's row-major (i, j).
//
//       payload_flag_kernel     one CTA per channel: any(sample != 0)
//       payload_rows_kernel     one CTA: exclusive scan of the flags -> compact
//                               row per channel, the (tx, rx) pair list, count
//       payload_convert_kernel  fp64 -> fp32 rows with a zero tail to ld
//
// (2) PGM rendering of energy maps (reference io.py:122-137 over
//     EnergyMap.dense, beamform.py:116-128), batched over S maps:
//
//       render_range_kernel     one CTA per map: min / max over the valid
//                               cells (fp64, exact for fp32 inputs)
//       render_pgm_kernel       one thread per output byte, raster order
//                               row r = iy, column c = ix: the cell's own value,
//                               else (stride D > 1) the value of the lattice
//                               cell (ix - ix % D, iy - iy % D) held over its
//                               D x D block, else "no value" -> 0; then
//                               rint(255 * clip((v - vmin) / (vmax - vmin), 0, 1))
//                               with IEEE fp64 _rn operations, so the bytes equal
//                               numpy's; a constant map renders as zeros.

constexpr int IO_THREADS = 256;

__global__ void __launch_bounds__(IO_THREADS) payload_flag_kernel(const double* __restrict__ payload, int n,
                                                                  int* __restrict__ flag) {
  const int ch = blockIdx.x;
  const double* row = payload + (size_t)ch * n;
  int any = 0;
  for (int k = threadIdx.x; k < n && !any; k += IO_THREADS) any = row[k] != 0.0;
  any = __syncthreads_or(any);
  if (threadIdx.x == 0) flag[ch] = any;
}

__global__ void __launch_bounds__(IO_THREADS) payload_rows_kernel(int* __restrict__ flag_row, int m,
                                                                  int32_t* __restrict__ pairs,
                                                                  int32_t* __restrict__ count) {
  __shared__ int warp_sum[IO_THREADS / 32];
  __shared__ int carry;
  const int n_ch = m * m, tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  if (tid == 0) carry = 0;
  __syncthreads();
  for (int base = 0; base < n_ch; base += IO_THREADS) {
    const int ch = base + tid;
    const int f = ch < n_ch ? (flag_row[ch] != 0) : 0;
    int incl = f;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += v;
    }
    if (lane == 31) warp_sum[wid] = incl;
    __syncthreads();
    int before = carry;
    for (int w = 0; w < wid; ++w) before += warp_sum[w];
    const int row = before + incl - f;
    if (ch < n_ch) {
      flag_row[ch] = f ? row : -1;
      if (f) {
        pairs[2 * row] = ch / m;
        pairs[2 * row + 1] = ch % m;
      }
    }
    __syncthreads();
    if (tid == IO_THREADS - 1) carry = before + incl;
    __syncthreads();
  }
  if (tid == 0) {
    int c = carry;
    if (c == 0) {  // an all-zero record keeps channel (0, 0) so every buffer is non-empty
      flag_row[0] = 0;
      pairs[0] = 0;
      pairs[1] = 0;
      c = 1;
    }
    *count = c;
  }
}

__global__ void __launch_bounds__(IO_THREADS) payload_convert_kernel(const double* __restrict__ payload, int n,
                                                                     int ld, const int* __restrict__ row_of,
                                                                     float* __restrict__ out) {
  const int ch = blockIdx.y;
  const int row = row_of[ch];
  if (row < 0) return;
  const double* src = payload + (size_t)ch * n;
  float* dst = out + (size_t)row * ld;
  for (int k = blockIdx.x * IO_THREADS + threadIdx.x; k < ld; k += gridDim.x * IO_THREADS)
    dst[k] = k < n ? __double2float_rn(src[k]) : 0.f;
}

template <typename T>
__global__ void __launch_bounds__(IO_THREADS) render_range_kernel(const T* __restrict__ values,
                                                                  const uint8_t* __restrict__ valid, long long cells,
                                                                  long long map_stride, double* __restrict__ vrange) {
  __shared__ double smin[IO_THREADS / 32], smax[IO_THREADS / 32];
  const int s = blockIdx.x;
  const T* v = values + (size_t)s * map_stride;
  const uint8_t* ok = valid + (size_t)s * map_stride;
  double lo = INFINITY, hi = -INFINITY;
  for (long long i = threadIdx.x; i < cells; i += IO_THREADS) {
    if (ok[i]) {
      const double x = (double)v[i];
      lo = fmin(lo, x);
      hi = fmax(hi, x);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    lo = fmin(lo, __shfl_xor_sync(0xffffffffu, lo, o));
    hi = fmax(hi, __shfl_xor_sync(0xffffffffu, hi, o));
  }
  if ((threadIdx.x & 31) == 0) {
    smin[threadIdx.x >> 5] = lo;
    smax[threadIdx.x >> 5] = hi;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < IO_THREADS / 32; ++w) {
      lo = fmin(lo, smin[w]);
      hi = fmax(hi, smax[w]);
    }
    lo = fmin(lo, smin[0]);
    hi = fmax(hi, smax[0]);
    vrange[2 * s] = lo;
    vrange[2 * s + 1] = hi;
  }
}

template <typename T>
__global__ void __launch_bounds__(IO_THREADS) render_pgm_kernel(const T* __restrict__ values,
                                                                const uint8_t* __restrict__ valid, int nx, int ny,
                                                                long long map_stride, int stride,
                                                                const double* __restrict__ vrange,
                                                                uint8_t* __restrict__ raster) {
  const int s = blockIdx.y;
  const long long cells = (long long)nx * ny;
  const T* v = values + (size_t)s * map_stride;
  const uint8_t* ok = valid + (size_t)s * map_stride;
  uint8_t* out = raster + (size_t)s * cells;
  const double vmin = vrange[2 * s], vmax = vrange[2 * s + 1];
  const bool flat = !(vmax > vmin);
  const double span = __dsub_rn(vmax, vmin);
  for (long long o = (long long)blockIdx.x * IO_THREADS + threadIdx.x; o < cells;
       o += (long long)gridDim.x * IO_THREADS) {
    const int iy = (int)(o / nx), ix = (int)(o - (long long)iy * nx);  // raster row r = iy
    long long c = (long long)ix * ny + iy;                               // map cell (ix, iy), ix-major
    bool have = ok[c];
    if (!have && stride > 1) {
      c = (long long)(ix - ix % stride) * ny + (iy - iy % stride);
      have = ok[c];
    }
    uint8_t byte = 0;
    if (have && !flat) {
      const double norm = __ddiv_rn(__dsub_rn((double)v[c], vmin), span);
      const double pix = fmin(fmax(norm, 0.0), 1.0);
      byte = (uint8_t)rint(__dmul_rn(255.0, pix));
    }
    out[o] = byte;
  }
}

// (3) Compact readback of a framework composite (coarse2fine.py:326-328): the
//     coarse lattice's values (fixed slots per plan) followed by the ROI
//     box's values in (ix, iy, iz) order, so a call reads back n_coarse +
//     |box| floats instead of the whole dense map and its mask (2-D: nz = 1).
__global__ void __launch_bounds__(IO_THREADS) gather_composite_kernel(const float* __restrict__ dense, int ny,
                                                                      int nz, const int* __restrict__ coarse_slots,
                                                                      int n_coarse, const int* __restrict__ region,
                                                                      float* __restrict__ out, long long cap) {
  const long long x0 = region[0], y0 = region[1], z0 = region[2];
  const long long h = region[4] - y0 + 1, dz = region[5] - z0 + 1, plane = h * dz;
  const long long total = n_coarse + (region[3] - x0 + 1) * plane;
  for (long long i = (long long)blockIdx.x * IO_THREADS + threadIdx.x; i < total && i < cap;
       i += (long long)gridDim.x * IO_THREADS) {
    long long slot;
    if (i < n_coarse) {
      slot = coarse_slots[i];
    } else {
      const long long r = i - n_coarse, ax = r / plane, rem = r - ax * plane, ay = rem / dz;
      slot = ((x0 + ax) * ny + y0 + ay) * nz + z0 + (rem - ay * dz);
    }
    out[i] = dense[slot];
  }
}
