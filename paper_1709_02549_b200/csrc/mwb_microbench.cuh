// mwb_microbench.cuh — LDS / FFMA / FFMA2 roofline microbenchmarks (bench.py peaks)
// (included by mwb_kernels.cu inside its anonymous namespace; one translation unit)
#pragma once

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

// shared-memory load-width / broadcast pattern probe: WORDS = 1, 2, 4 (LDS.32/64/128);
// lane address (in units of WORDS words): 0 consecutive, 1 all-same, 2 lane/2,
// 3 lane/4, 4 lane/8, 5 (lane*3)/8 (a delay-like monotone spread)
template <int WORDS>
__global__ void __launch_bounds__(1024) mb_lds_pattern_kernel(float* sink, int pattern) {
  __shared__ __align__(16) float buf[8192];
  for (int i = threadIdx.x; i < 8192; i += blockDim.x) buf[i] = (float)(i & 1023);
  __syncthreads();
  const int lane = threadIdx.x & 31;
  int a;
  switch (pattern) {
    case 0: a = lane; break;
    case 1: a = 0; break;
    case 2: a = lane >> 1; break;
    case 3: a = lane >> 2; break;
    case 4: a = lane >> 3; break;
    default: a = (lane * 3) >> 3; break;
  }
  float acc[4] = {0.f, 0.f, 0.f, 0.f};
  for (int it = 0; it < MB_ITERS / 4; ++it) {
    const int base = ((it * 37) & 63) * 32;  // stays 16-byte aligned per WORDS
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      const float* b = buf + (base + (a + k * 8) * WORDS) % 8192;
      if (WORDS == 1) {
        acc[k & 3] += b[0];
      } else if (WORDS == 2) {
        const float2 v = *reinterpret_cast<const float2*>(b);
        acc[k & 3] += v.x + v.y;
      } else {
        const float4 v = *reinterpret_cast<const float4*>(b);
        acc[k & 3] += (v.x + v.y) + (v.z + v.w);
      }
    }
  }
  const float r = acc[0] + acc[1] + acc[2] + acc[3];
  if (r == 1234.5f) sink[threadIdx.x] = r;
}
