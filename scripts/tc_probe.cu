// Standalone probe of the tcgen05 mechanics the tensor-core energy path uses
// (development aid, not part of libmwb.so): one CTA computes
// D[128 x N] = A[128 x 16] * B[N x 16]^T with fp16 operands in the no-swizzle
// K-major core-matrix layout, fp32 accumulation in TMEM, and checks it on the
// host.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -o tc_probe tc_probe.cu
#include <cuda_fp16.h>
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cmath>
#include <vector>

constexpr int M = 128, K = 16;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// byte offset of element (r, k) of a rows x 16 fp16 K-major operand:
// core matrices of 8 rows x 16 B; LBO = 128 B (k-half), SBO = 256 B (8-row group)
__host__ __device__ inline uint32_t kmajor_off(int r, int k) {
  return (r >> 3) * 256 + (k >> 3) * 128 + (r & 7) * 16 + (k & 7) * 2;
}

__device__ __forceinline__ uint64_t smem_desc(const void* p, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((smem_u32(p) >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // version 1 (sm_100)
  return d;                // base offset 0, lbo mode 0, layout SWIZZLE_NONE (0)
}

__host__ __device__ constexpr uint32_t idesc_f16(int m, int n) {
  return (1u << 4)                      // D format f32
         | (0u << 7) | (0u << 10)       // A, B f16
         | (0u << 15) | (0u << 16)      // K-major both
         | ((uint32_t)(n >> 3) << 17)   // N >> 3
         | ((uint32_t)(m >> 4) << 24);  // M >> 4
}

template <int N>
__global__ void probe(const __half* a, const __half* b, float* d, int* err) {
  __shared__ __align__(1024) unsigned char sa[M * K * 2];
  __shared__ __align__(1024) unsigned char sb[N * K * 2];
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < M * K; i += blockDim.x)
    *reinterpret_cast<__half*>(sa + kmajor_off(i / K, i % K)) = a[i];
  for (int i = tid; i < N * K; i += blockDim.x)
    *reinterpret_cast<__half*>(sb + kmajor_off(i / K, i % K)) = b[i];
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tbase)),
                 "r"(256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tbase;
  if (tid == 0) {
    const uint64_t da = smem_desc(sa, 128, 256), db = smem_desc(sb, 128, 256);
    const uint32_t id = idesc_f16(M, N);
    asm volatile(
        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
        "l"(da), "l"(db), "r"(id), "r"(0));
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
        smem_u32(&bar)));
  }
  // wait for the MMA (phase 0)
  asm volatile(
      "{\n.reg .pred p;\nWAIT:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra WAIT;\n}\n" ::"r"(
          smem_u32(&bar)),
      "r"(0)
      : "memory");
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (warp < 4) {
    const int row = warp * 32 + (tid & 31);
    for (int c = 0; c < N; c += 8) {
      uint32_t v[8];
      const uint32_t addr = tmem + ((uint32_t)(warp * 32) << 16) + c;
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                   : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
                     "=r"(v[7])
                   : "r"(addr));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      for (int j = 0; j < 8; ++j) d[row * N + c + j] = __uint_as_float(v[j]);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(256));
  if (tid == 0) *err = 0;
}

// Same product with A taken from TMEM: thread r writes row r (16 fp16 = 8
// packed 32-bit columns) with tcgen05.st, the MMA reads [a_tmem].
template <int N>
__global__ void probe_tmem_a(const __half* a, const __half* b, float* d) {
  __shared__ __align__(1024) unsigned char sb[N * K * 2];
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < N * K; i += blockDim.x)
    *reinterpret_cast<__half*>(sb + kmajor_off(i / K, i % K)) = b[i];
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tbase)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tbase;
  const uint32_t a_col = 256;  // A operand at columns [256, 264)
  {
    const int row = tid;  // 128 threads: warp w writes lanes 32w..32w+31
    uint32_t r[8];
    for (int j = 0; j < 8; ++j) {
      const __half2 h = __halves2half2(a[row * K + 2 * j], a[row * K + 2 * j + 1]);
      r[j] = *reinterpret_cast<const uint32_t*>(&h);
    }
    const uint32_t addr = tmem + ((uint32_t)(warp * 32) << 16) + a_col;
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(addr), "r"(r[0]),
                 "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]));
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (tid == 0) {
    const uint64_t db = smem_desc(sb, 128, 256);
    const uint32_t id = idesc_f16(M, N);
    asm volatile(
        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(tmem),
        "r"(tmem + a_col), "l"(db), "r"(id), "r"(0));
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
        smem_u32(&bar)));
  }
  asm volatile(
      "{\n.reg .pred p;\nWAIT2:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra WAIT2;\n}\n" ::"r"(
          smem_u32(&bar)),
      "r"(0)
      : "memory");
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  {
    const int row = warp * 32 + (tid & 31);
    for (int c = 0; c < N; c += 8) {
      uint32_t v[8];
      const uint32_t addr = tmem + ((uint32_t)(warp * 32) << 16) + c;
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                   : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
                     "=r"(v[7])
                   : "r"(addr));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      for (int j = 0; j < 8; ++j) d[row * N + c + j] = __uint_as_float(v[j]);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

// Throughput of back-to-back M128 x N x K16 SS MMAs (no-swizzle operands),
// 6 per iteration with a commit per iteration, as the energy kernel issues them.
template <int N>
__global__ void mma_rate(int iters, long long* cycles) {
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
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tbase)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tbase;
  if (tid == 0) {
    const uint32_t id = idesc_f16(M, N);
    const uint64_t a0 = smem_desc(sa, 128, 256), a1 = smem_desc(sa + M * K * 2, 128, 256);
    const uint64_t b0 = smem_desc(sb, 128, 256), b1 = smem_desc(sb + N * K * 2, 128, 256);
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      for (int mb = 0; mb < 2; ++mb) {
        const uint32_t d = tmem + mb * N;
        asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n"
                     ::"r"(d), "l"(mb ? a1 : a0), "l"(b0), "r"(id), "r"(1));
        asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n"
                     ::"r"(d), "l"(mb ? a1 : a0), "l"(b1), "r"(id), "r"(1));
        asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n"
                     ::"r"(d), "l"(mb ? a0 : a1), "l"(b0), "r"(id), "r"(1));
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
    }
    // wait for the last commit's phase
    const uint32_t parity = (uint32_t)((iters - 1) & 1);
    asm volatile(
        "{\n.reg .pred p;\nWAIT3:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra WAIT3;\n}\n" ::"r"(
            smem_u32(&bar)), "r"(parity) : "memory");
    *cycles = clock64() - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

// 2-CTA (cta_group::2) product D[256 x N] = A[256 x 16] * B[N x 16]^T: CTA r
// holds A rows 128 r .. 128 r + 127 and B rows (N / 2) r .. (N / 2)(r + 1) - 1
// at the same shared-memory offsets; the leader issues the MMA; each CTA's
// TMEM receives its 128 rows of D.
template <int N>
__global__ void __cluster_dims__(2, 1, 1) probe_2sm(const __half* a, const __half* b, float* d) {
  __shared__ __align__(1024) unsigned char sa[128 * K * 2];
  __shared__ __align__(1024) unsigned char sb[(N / 2) * K * 2];
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tbase;
  uint32_t rank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < 128 * K; i += blockDim.x)
    *reinterpret_cast<__half*>(sa + kmajor_off(i / K, i % K)) = a[(rank * 128 + i / K) * K + i % K];
  for (int i = tid; i < (N / 2) * K; i += blockDim.x)
    *reinterpret_cast<__half*>(sb + kmajor_off(i / K, i % K)) = b[(rank * (N / 2) + i / K) * K + i % K];
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tbase)),
                 "r"(256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tbase;
  if (rank == 0 && tid == 0) {
    const uint64_t da = smem_desc(sa, 128, 256), db = smem_desc(sb, 128, 256);
    const uint32_t id = idesc_f16(256, N);
    asm volatile(
        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
        "l"(da), "l"(db), "r"(id), "r"(0));
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
            smem_u32(&bar)), "h"((unsigned short)3));
  }
  asm volatile(
      "{\n.reg .pred p;\nWAIT4:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra WAIT4;\n}\n" ::"r"(
          smem_u32(&bar)), "r"(0) : "memory");
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  {
    const int row = warp * 32 + (tid & 31);
    for (int c = 0; c < N; c += 8) {
      uint32_t v[8];
      const uint32_t addr = tmem + ((uint32_t)(warp * 32) << 16) + c;
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                   : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
                     "=r"(v[7])
                   : "r"(addr));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      for (int j = 0; j < 8; ++j) d[(rank * 128 + row) * N + c + j] = __uint_as_float(v[j]);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(256));
}

int main() {
  constexpr int N = 256;
  std::vector<__half> ha(M * K), hb(N * K);
  std::vector<float> fa(M * K), fb(N * K);
  srand(1);
  for (int i = 0; i < M * K; ++i) { fa[i] = (float)((rand() % 17) - 8) / 4.0f; ha[i] = __float2half(fa[i]); }
  for (int i = 0; i < N * K; ++i) { fb[i] = (float)((rand() % 13) - 6) / 8.0f; hb[i] = __float2half(fb[i]); }
  __half *da, *db; float* dd; int* derr;
  cudaMalloc(&da, M * K * 2); cudaMalloc(&db, N * K * 2); cudaMalloc(&dd, M * N * 4); cudaMalloc(&derr, 4);
  cudaMemcpy(da, ha.data(), M * K * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(db, hb.data(), N * K * 2, cudaMemcpyHostToDevice);
  cudaMemset(dd, 0xFF, M * N * 4);
  probe<N><<<1, 128>>>(da, db, dd, derr);
  cudaError_t e = cudaDeviceSynchronize();
  printf("launch: %s\n", cudaGetErrorString(e));
  std::vector<float> hd(M * N);
  cudaMemcpy(hd.data(), dd, M * N * 4, cudaMemcpyDeviceToHost);
  double maxerr = 0; int bad = 0;
  for (int i = 0; i < M; ++i)
    for (int j = 0; j < N; ++j) {
      double s = 0;
      for (int k = 0; k < K; ++k) s += (double)fa[i * K + k] * fb[j * K + k];
      double err = fabs(s - hd[i * N + j]);
      if (err > maxerr) maxerr = err;
      if (err > 1e-3 && bad++ < 5) printf("bad (%d,%d): got %f want %f\n", i, j, hd[i * N + j], s);
    }
  printf("max abs err %g, bad %d of %d\n", maxerr, bad, M * N);
  // A from TMEM
  constexpr int N2 = 192;
  cudaMemset(dd, 0xFF, M * N * 4);
  probe_tmem_a<N2><<<1, 128>>>(da, db, dd);
  e = cudaDeviceSynchronize();
  printf("tmem-A launch: %s\n", cudaGetErrorString(e));
  cudaMemcpy(hd.data(), dd, M * N2 * 4, cudaMemcpyDeviceToHost);
  double maxerr2 = 0; int bad2 = 0;
  for (int i = 0; i < M; ++i)
    for (int j = 0; j < N2; ++j) {
      double s = 0;
      for (int k = 0; k < K; ++k) s += (double)fa[i * K + k] * fb[j * K + k];
      double err = fabs(s - hd[i * N2 + j]);
      if (err > maxerr2) maxerr2 = err;
      if (err > 1e-3 && bad2++ < 5) printf("bad2 (%d,%d): got %f want %f\n", i, j, hd[i * N2 + j], s);
    }
  printf("tmem-A: max abs err %g, bad %d of %d\n", maxerr2, bad2, M * N2);
  {  // 2-CTA pair
    constexpr int N3 = 256;
    std::vector<__half> ha3(256 * K); std::vector<float> fa3(256 * K);
    for (int i = 0; i < 256 * K; ++i) { fa3[i] = (float)((rand() % 15) - 7) / 4.0f; ha3[i] = __float2half(fa3[i]); }
    __half* da3; float* dd3; cudaMalloc(&da3, 256 * K * 2); cudaMalloc(&dd3, 256 * N3 * 4);
    cudaMemcpy(da3, ha3.data(), 256 * K * 2, cudaMemcpyHostToDevice);
    cudaMemset(dd3, 0xFF, 256 * N3 * 4);
    probe_2sm<N3><<<2, 128>>>(da3, db, dd3);
    e = cudaDeviceSynchronize();
    printf("2sm launch: %s\n", cudaGetErrorString(e));
    std::vector<float> hd3(256 * N3);
    cudaMemcpy(hd3.data(), dd3, 256 * N3 * 4, cudaMemcpyDeviceToHost);
    double me = 0; int b3 = 0;
    for (int i = 0; i < 256; ++i)
      for (int j = 0; j < N3; ++j) {
        double sacc = 0;
        for (int k = 0; k < K; ++k) sacc += (double)fa3[i * K + k] * fb[j * K + k];
        const double err = fabs(sacc - hd3[i * N3 + j]);
        if (err > me) me = err;
        if (err > 1e-3 && b3++ < 5) printf("bad3 (%d,%d): got %f want %f\n", i, j, hd3[i * N3 + j], sacc);
      }
    printf("2sm: max abs err %g, bad %d of %d\n", me, b3, 256 * N3);
  }
  long long* dcyc; cudaMalloc(&dcyc, 8);
  for (int iters : {1000, 4000}) {
    mma_rate<256><<<1, 128>>>(iters, dcyc);
    cudaDeviceSynchronize();
    long long cyc; cudaMemcpy(&cyc, dcyc, 8, cudaMemcpyDeviceToHost);
    const double macs = (double)iters * 6 * 128.0 * 256 * 16;
    printf("mma_rate N=256 iters=%d: %lld cycles, %.0f MAC/clk (%.1f clk per MMA)\n", iters, cyc, macs / cyc,
           (double)cyc / (iters * 6.0));
  }
  return (bad != 0) || (bad2 != 0);
}
