// Probe (development aid, not part of libmwb.so): can tcgen05.mma read the
// Hankel operand B[n = 8k + s, m] = Y[b + m + k][s] straight from a time-major,
// 8-scan-interleaved fp16 plane Y[t][8] with an MN-major no-swizzle smem
// descriptor (core matrix = 8 scans x 8 consecutive time rows of 16 B; MN
// stride SBO = 16 B, i.e. overlapping core matrices; K stride LBO = 128 B)?
// Variant 2 takes the two 8-tap K halves from two different planes (LBO = the
// address difference).  Also times back-to-back MMAs with this operand.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -o tc_hankel_probe tc_hankel_probe.cu
#include <cuda_fp16.h>
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cmath>
#include <vector>

constexpr int M = 128, K = 16, N = 256, L = 64;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__host__ __device__ inline uint32_t kmajor_off(int r, int k) {
  return (r >> 3) * 256 + (k >> 3) * 128 + (r & 7) * 16 + (k & 7) * 2;
}
__device__ __forceinline__ uint64_t smem_desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  return d;
}
__host__ __device__ constexpr uint32_t idesc(int m, int n, int b_mn) {
  return (1u << 4) | ((uint32_t)b_mn << 16) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(m >> 4) << 24);
}
__device__ __forceinline__ void mma(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n"
               ::"r"(d), "l"(a), "l"(b), "r"(id), "r"(acc));
}
__device__ __forceinline__ void wait_bar(uint64_t* bar, uint32_t par) {
  asm volatile("{\n.reg .pred p;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W;\n}\n" ::"r"(
                   smem_u32(bar)), "r"(par) : "memory");
}

// mode 0: B from plane y1 at b1 (both K halves); mode 1: K half 0 from y1 at
// b1, K half 1 from y2 at b2
__global__ void probe(const __half* a, const __half* y1, const __half* y2, int b1, int b2, int mode, float* d) {
  __shared__ __align__(1024) unsigned char sa[M * K * 2];
  __shared__ __align__(1024) __half sy[2][L * 8];
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < M * K; i += blockDim.x) *reinterpret_cast<__half*>(sa + kmajor_off(i / K, i % K)) = a[i];
  for (int i = tid; i < L * 8; i += blockDim.x) {
    sy[0][i] = y1[i];
    sy[1][i] = y2[i];
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tbase)), "r"(256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tbase;
  if (tid == 0) {
    const uint32_t s1 = smem_u32(&sy[0][b1 * 8]), s2 = smem_u32(&sy[1][b2 * 8]);
    const uint32_t lbo = mode == 0 ? 128u : s2 - s1;
    mma(tmem, smem_desc(smem_u32(sa), 128, 256), smem_desc(s1, lbo, 16), idesc(M, N, 1), 0);
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
  }
  wait_bar(&bar, 0);
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const int row = warp * 32 + (tid & 31);
  for (int c = 0; c < N; c += 8) {
    uint32_t v[8];
    const uint32_t addr = tmem + ((uint32_t)(warp * 32) << 16) + c;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                 : "r"(addr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    for (int j = 0; j < 8; ++j) d[row * N + c + j] = __uint_as_float(v[j]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(256));
}

// 6 MMAs per iteration (2 accumulators x 3), B MN-major from planes (mn = 1)
// or K-major (mn = 0); one commit per iteration
__global__ void rate(int iters, int mn, long long* cycles) {
  __shared__ __align__(1024) unsigned char sa[2 * M * K * 2];
  __shared__ __align__(1024) unsigned char sb[2 * N * K * 2];
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < (int)sizeof(sa) / 2; i += blockDim.x) reinterpret_cast<__half*>(sa)[i] = __float2half(0.001f);
  for (int i = tid; i < (int)sizeof(sb) / 2; i += blockDim.x) reinterpret_cast<__half*>(sb)[i] = __float2half(0.001f);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tbase)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tbase;
  if (tid == 0) {
    const uint32_t id = idesc(M, N, mn);
    const uint64_t a0 = smem_desc(smem_u32(sa), 128, 256), a1 = smem_desc(smem_u32(sa) + M * K * 2, 128, 256);
    uint64_t b0, b1;
    if (mn) {
      b0 = smem_desc(smem_u32(sb) + 48, 128, 16);
      b1 = smem_desc(smem_u32(sb) + 4096 + 80, 128, 16);
    } else {
      b0 = smem_desc(smem_u32(sb), 128, 256);
      b1 = smem_desc(smem_u32(sb) + N * K * 2, 128, 256);
    }
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      for (int mb = 0; mb < 2; ++mb) {
        const uint32_t d = tmem + mb * N;
        mma(d, mb ? a1 : a0, b0, id, 1);
        mma(d, mb ? a1 : a0, b1, id, 1);
        mma(d, mb ? a0 : a1, b0, id, 1);
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
    }
    wait_bar(&bar, (uint32_t)((iters - 1) & 1));
    *cycles = clock64() - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}


// Same 6-MMA step as the energy kernels, but with fresh operands every step:
// A from NSLOT rotating 16 KB slots (hi | lo, two M-blocks), B from rotating
// plane addresses (mn = 1) or K-major slots (mn = 0) -- no operand reuse
// across steps, as in the real pipeline.
template <int NSLOT>
__global__ void rate_rot(int iters, int mn, long long* cycles) {
  extern __shared__ __align__(1024) unsigned char dyn[];
  unsigned char* sa = dyn;                       // NSLOT x 16 KB
  unsigned char* sb = dyn + NSLOT * 16384;       // 16 x 8 KB planes / slots
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < (NSLOT * 16384 + 16 * 8192) / 2; i += blockDim.x)
    reinterpret_cast<__half*>(dyn)[i] = __float2half(0.001f);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tbase)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tbase;
  if (tid == 0) {
    const uint32_t id = idesc(M, N, mn);
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      const uint32_t a = smem_u32(sa) + (it % NSLOT) * 16384;
      const uint32_t bp = smem_u32(sb) + (it % 16) * 8192;
      uint64_t bh, bl;
      if (mn) {
        bh = smem_desc(bp + 48, 128, 16);
        bl = smem_desc(bp + 48 + 896, 128, 16);
      } else {
        bh = smem_desc(bp, 128, 256);
        bl = smem_desc(bp + (it % 2) * 0, 128, 256) + 0;
        bl = smem_desc(smem_u32(sb) + ((it + 7) % 16) * 8192, 128, 256);
      }
      for (int mb = 0; mb < 2; ++mb) {
        const uint32_t d = tmem + mb * N;
        const uint64_t ah = smem_desc(a + mb * 4096, 128, 256), al = smem_desc(a + 8192 + mb * 4096, 128, 256);
        mma(d, ah, bh, id, 1);
        mma(d, ah, bl, id, 1);
        mma(d, al, bh, id, 1);
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
    }
    wait_bar(&bar, (uint32_t)((iters - 1) & 1));
    *cycles = clock64() - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

int main() {
  std::vector<__half> ha(M * K), hy1(L * 8), hy2(L * 8);
  std::vector<float> fa(M * K), fy1(L * 8), fy2(L * 8);
  srand(3);
  for (int i = 0; i < M * K; ++i) { fa[i] = (float)((rand() % 17) - 8) / 4.0f; ha[i] = __float2half(fa[i]); }
  for (int i = 0; i < L * 8; ++i) {
    fy1[i] = (float)((rand() % 13) - 6) / 8.0f; hy1[i] = __float2half(fy1[i]);
    fy2[i] = (float)((rand() % 11) - 5) / 8.0f; hy2[i] = __float2half(fy2[i]);
  }
  __half *da, *dy1, *dy2; float* dd;
  cudaMalloc(&da, M * K * 2); cudaMalloc(&dy1, L * 16); cudaMalloc(&dy2, L * 16); cudaMalloc(&dd, M * N * 4);
  cudaMemcpy(da, ha.data(), M * K * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dy1, hy1.data(), L * 16, cudaMemcpyHostToDevice);
  cudaMemcpy(dy2, hy2.data(), L * 16, cudaMemcpyHostToDevice);
  int fails = 0;
  for (int mode = 0; mode < 2; ++mode) {
    for (int b1 : {0, 3, 7}) {
      const int b2 = 5;
      cudaMemset(dd, 0xFF, M * N * 4);
      probe<<<1, 128>>>(da, dy1, dy2, b1, b2, mode, dd);
      cudaError_t e = cudaDeviceSynchronize();
      std::vector<float> hd(M * N);
      cudaMemcpy(hd.data(), dd, M * N * 4, cudaMemcpyDeviceToHost);
      double maxerr = 0; int bad = 0;
      for (int i = 0; i < M; ++i)
        for (int n = 0; n < N; ++n) {
          const int k = n / 8, s = n % 8;
          double acc = 0;
          for (int m = 0; m < K; ++m) {
            const float y = (mode == 0 || m < 8) ? fy1[(b1 + m + k) * 8 + s] : fy2[(b2 + (m - 8) + k) * 8 + s];
            acc += (double)fa[i * K + m] * y;
          }
          const double err = fabs(acc - hd[i * N + n]);
          if (!(err <= maxerr)) maxerr = err;
          if (!(err <= 1e-3) && bad++ < 3) printf("  bad (%d,%d): got %f want %f\n", i, n, hd[i * N + n], acc);
        }
      printf("mode %d b1 %d: %s, max abs err %g, bad %d of %d\n", mode, b1, cudaGetErrorString(e), maxerr, bad, M * N);
      fails += bad != 0;
    }
  }
  long long* dc; cudaMalloc(&dc, 8);
  for (int mn = 0; mn < 2; ++mn)
    for (int iters : {1000, 4000}) {
      rate<<<1, 128>>>(iters, mn, dc);
      cudaDeviceSynchronize();
      long long cyc; cudaMemcpy(&cyc, dc, 8, cudaMemcpyDeviceToHost);
      printf("rate %s iters=%d: %.1f clk per MMA\n", mn ? "MN-major Hankel B" : "K-major B", iters,
             (double)cyc / (iters * 6.0));
    }
  {
    const int smem = 6 * 16384 + 16 * 8192;
    cudaFuncSetAttribute(rate_rot<6>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    for (int mn = 0; mn < 2; ++mn) {
      rate_rot<6><<<1, 128, smem>>>(4000, mn, dc);
      cudaError_t e = cudaDeviceSynchronize();
      long long cyc; cudaMemcpy(&cyc, dc, 8, cudaMemcpyDeviceToHost);
      printf("rotating operands %s: %s %.1f clk per MMA\n", mn ? "MN-major Hankel B" : "K-major B",
             cudaGetErrorString(e), (double)cyc / (4000 * 6.0));
    }
  }
  return fails;
}
