// mwb_simulate.cuh — K5 device scan synthesis (simulate.py:111-162 and the BASELINE signal model)
// (included by mwb_kernels.cu inside its anonymous namespace; one translation unit)
#pragma once

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
