// mma_probe.cu -- tcgen05 throughput microbenchmark (B200, sm_100a).
//
// Measures cycles per tcgen05.mma.kind::f16 (bf16, fp32 accumulate, both
// operands K-major SW128 in smem) for the tile shapes the K3-TC kernel can
// use, optionally with 8 warps concurrently streaming the other TMEM buffer
// through tcgen05.ld + relu-sum (the K3 epilogue), and for cta_group::2.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mma_probe mma_probe.cu
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#define CK(x)                                                            \
  do {                                                                   \
    cudaError_t e = (x);                                                 \
    if (e != cudaSuccess) {                                              \
      printf("CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
      return 1;                                                          \
    }                                                                    \
  } while (0)

__constant__ int g_cp = 4;
__constant__ int g_rot = 1;
__constant__ int g_data = 0;  // 0 small positive pattern, 1 Gaussian-like, 2 zeros
__device__ __forceinline__ uint32_t fill_word(uint32_t i) {
  uint32_t h = i * 2654435761u;
  h ^= h >> 13;
  h *= 0x5bd1e995u;
  h ^= h >> 15;
  if (g_data == 0) return 0x3c003c00u ^ (i * 2654435761u & 0x00ff00ffu);
  if (g_data == 2) return 0u;
  // two bf16: random sign, exponent 2^-3..2^0 (like N(0,1) data), random mantissa
  auto one = [](uint32_t x) -> uint32_t {
    return ((x & 1u) << 15) | ((0x7Cu + ((x >> 1) & 3u)) << 7) | ((x >> 3) & 0x7Fu);
  };
  return one(h & 0xFFFFu) | (one(h >> 16) << 16);
}
__device__ __forceinline__ uint32_t su32(const void *p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ uint64_t desc(uint32_t a) {
  return (uint64_t)((a >> 4) & 0x3FFF) | (1ull << 16) | (64ull << 32) |
         (1ull << 46) | (2ull << 61);
}
__device__ __forceinline__ void mbar_wait(uint64_t *b, uint32_t ph) {
  uint32_t ok = 0;
  do {
    asm volatile(
        "{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;"
        " selp.u32 %0,1,0,p;}"
        : "=r"(ok)
        : "r"(su32(b)), "r"(ph)
        : "memory");
  } while (!ok);
}

template <int M, int N, int CG, bool kLdtm, bool kCommit = false, bool kTma = false>
__global__ void __launch_bounds__(320, 1)
    probe(int tiles, int ksteps, unsigned long long *cyc, float *sink,
          const unsigned char *gsrc) {
  extern __shared__ __align__(1024) unsigned char sm_raw[];
  unsigned char *sm =
      (unsigned char *)(((uintptr_t)sm_raw + 1023) & ~(uintptr_t)1023);
  // A: 2 chunks of 128 rows x 128 B; B: 2 chunks of (N/CG) rows x 128 B
  unsigned char *sa = sm;
  unsigned char *sb = sm + 2 * 128 * 128;
  __shared__ uint64_t bar, dummy, tbar[3];
  __shared__ uint32_t slot;
  unsigned char *ring = sm + 2 * 128 * 128 + 2 * (N / CG) * 128;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  for (int i = threadIdx.x; i < (2 * 128 * 128 + 2 * (N / CG) * 128) / 4;
       i += blockDim.x)
    ((uint32_t *)sm)[i] = fill_word(i);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&dummy)));
    for (int i = 0; i < 3; ++i)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&tbar[i])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  uint32_t rank = 0;
  if (CG == 2) asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  if (warp == 1) {
    if (CG == 1) {
      asm volatile(
          "tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::
              "r"(su32(&slot)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    } else {
      asm volatile(
          "tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::
              "r"(su32(&slot)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (CG == 2) {
    asm volatile("barrier.cluster.arrive.release.aligned;");
    asm volatile("barrier.cluster.wait.acquire.aligned;");
  }
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = slot;
  const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) |
                         ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
  volatile __shared__ int stop;
  if (threadIdx.x == 0) stop = 0;
  __syncthreads();
  if (warp == 1 && rank == 0) {
    unsigned long long t0 = clock64();
    for (int t = 0; t < tiles; ++t) {
      const uint32_t d = tmem + (uint32_t)((t & 1) * N);
      if (lane == 0) {
        for (int ks = 0; ks < ksteps; ++ks) {
          const int kc = ks / 4, ko = (ks % 4) * 32;
          uint64_t ad = desc(su32(sa + kc * 128 * 128) + ko);
          uint64_t bd = desc(su32(sb + kc * (N / CG) * 128) + ko);
          uint32_t acc = ks > 0;
          if (CG == 1)
            asm volatile(
                "{.reg .pred p; setp.ne.b32 p, %4, 0;"
                " tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;}" ::
                    "r"(d), "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
          else
            asm volatile(
                "{.reg .pred p; setp.ne.b32 p, %4, 0;"
                " tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;}" ::
                    "r"(d), "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
          if (kCommit && ((t * ksteps + ks + 1) % g_cp == 0)) {
            if (CG == 1)
              asm volatile(
                  "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster."
                  "b64 [%0];" ::"r"(su32(&dummy)));
            else
              asm volatile(
                  "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster."
                  "multicast::cluster.b64 [%0], %1;" ::"r"(su32(&dummy)),
                  "h"((uint16_t)3));
          }
        }
      }
      __syncwarp();
    }
    if (lane == 0) {
      if (CG == 1)
        asm volatile(
            "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster."
            "b64 [%0];" ::"r"(su32(&bar)));
      else
        asm volatile(
            "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster."
            "multicast::cluster.b64 [%0], %1;" ::"r"(su32(&bar)),
            "h"((uint16_t)3));
    }
    __syncwarp();
    mbar_wait(&bar, 0);
    unsigned long long t1 = clock64();
    if (lane == 0) cyc[blockIdx.x] = t1 - t0;
    stop = 1;
  } else if (warp == 1 && CG == 2) {
    mbar_wait(&bar, 0);
    stop = 1;
  } else if (warp == 0 && kTma && lane == 0) {
    // stream 32 KB bulk copies from an L2-resident buffer into a 3-slot ring
    uint32_t ph[3] = {0, 0, 0};
    int it = 0;
    for (int s = 0; s < 3; ++s) {
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&tbar[s])), "r"(32768));
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   ::"r"(su32(ring + s * 32768)), "l"(gsrc + ((it++ * 32768) & ((4 << 20) - 1))), "r"(32768), "r"(su32(&tbar[s])) : "memory");
    }
    while (!stop) {
      for (int s = 0; s < 3 && !stop; ++s) {
        mbar_wait(&tbar[s], ph[s]);
        ph[s] ^= 1;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&tbar[s])), "r"(32768));
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     ::"r"(su32(ring + s * 32768)), "l"(gsrc + ((it++ * 32768) & ((4 << 20) - 1))), "r"(32768), "r"(su32(&tbar[s])) : "memory");
      }
    }
    for (int s = 0; s < 3; ++s) { mbar_wait(&tbar[s], ph[s]); }
    cyc[148 + blockIdx.x] = (unsigned long long)it;
  } else if (warp >= 2 && kLdtm) {
    const int q = warp & 3, half = (warp - 2) >> 2;
    float s = 0.f;
    int it = 0;
    while (!stop) {
      const uint32_t buf = (uint32_t)((it & 1) * N);
      const uint32_t ta = tmem + ((uint32_t)(q * 32) << 16) + buf +
                          (uint32_t)(half * (N / 2));
#pragma unroll 1
      for (int c = 0; c < N / 2; c += 32) {
        uint32_t r[32];
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
            "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,"
            "%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
            : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]),
              "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]), "=r"(r[9]),
              "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
              "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
              "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
              "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]),
              "=r"(r[30]), "=r"(r[31])
            : "r"(ta + c));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
        for (int j = 0; j < 32; ++j) s += fmaxf(__uint_as_float(r[j]), 0.f);
      }
      ++it;
    }
    sink[blockIdx.x * 320 + threadIdx.x] = s;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (CG == 2) {
    asm volatile("barrier.cluster.arrive.release.aligned;");
    asm volatile("barrier.cluster.wait.acquire.aligned;");
  }
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (CG == 1)
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
    else
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

template <int M, int N, int CG, bool kLdtm, bool kCommit = false, bool kTma = false>
int run(const char *name, int tiles, int ksteps, int cp = 4) {
  cudaMemcpyToSymbol(g_cp, &cp, sizeof(int));
  unsigned long long *cyc;
  float *sink;
  CK(cudaMalloc(&cyc, 2 * 148 * 8));
  CK(cudaMemset(cyc, 0, 2 * 148 * 8));
  unsigned char *gsrc;
  CK(cudaMalloc(&gsrc, 4 << 20));
  CK(cudaMemset(gsrc, 1, 4 << 20));
  CK(cudaMalloc(&sink, 148 * 320 * 4));
  size_t smem = 2 * 128 * 128 + 2 * (N / CG) * 128 + 2048 + (kTma ? 3 * 32768 : 0);
  CK(cudaFuncSetAttribute(probe<M, N, CG, kLdtm, kCommit, kTma>,
                          cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(148);
  cfg.blockDim = dim3(320);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CG;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(e0);
    CK(cudaLaunchKernelEx(&cfg, probe<M, N, CG, kLdtm, kCommit, kTma>, tiles, ksteps, cyc, sink, (const unsigned char *)gsrc));
    cudaEventRecord(e1);
    CK(cudaDeviceSynchronize());
  }
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  unsigned long long h[296];
  CK(cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost));
  double tma_bytes = 0;
  for (int i = 0; i < 148; ++i) tma_bytes += (double)h[148 + i] * 32768.0;
  double avg = 0;
  int cnt = 0;
  for (int i = 0; i < 148; ++i)
    if (h[i]) avg += (double)h[i], ++cnt;
  avg /= cnt;
  const double mmas = (double)tiles * ksteps;
  const double macs_per_sm_per_mma = (double)(M / CG) * N * 16;
  const double flops = 2.0 * macs_per_sm_per_mma * mmas * 148;
  printf("%-34s cyc/mma %7.1f  MAC/clk/SM %7.1f  %7.1f TFLOP/s (event %.3f ms) tma %.0f B/clk/SM\n",
         name, avg / mmas, macs_per_sm_per_mma * mmas / avg, flops / ms / 1e9,
         ms, tma_bytes / 148 / avg);
  cudaFree(cyc);
  cudaFree(sink);
  cudaFree(gsrc);
  return 0;
}

// Tight single-thread issuer: the whole MMA role runs on one thread, the
// K-steps of a tile are unrolled with precomputed descriptors, and the two
// per-tile commits (smem slot release + accumulator ready) sit at compile-time
// positions.  Each tile waits on a (pre-satisfied) mbarrier like the kernel.
template <int KS, bool kWait, bool kEpi = false>
__global__ void __launch_bounds__(320, 1)
    probe_tight(int tiles, unsigned long long *cyc) {
  volatile __shared__ int stop_t;
  extern __shared__ __align__(1024) unsigned char sm_raw[];
  unsigned char *sm =
      (unsigned char *)(((uintptr_t)sm_raw + 1023) & ~(uintptr_t)1023);
  unsigned char *sa = sm, *sb = sm + 2 * 128 * 128;
  __shared__ uint64_t bar, b1, b2, ready;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  for (int i = threadIdx.x; i < (2 * 128 * 128 + 2 * 256 * 128) / 4; i += blockDim.x)
    ((uint32_t *)sm)[i] = fill_word(i);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&b1)));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&b2)));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&ready)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (threadIdx.x == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&ready)));
  if (threadIdx.x == 0) stop_t = 0;
  __syncthreads();
  const uint32_t tmem = slot;
  const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(256 >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
  if (warp == 1 && lane == 0) {
    const uint64_t a0 = desc(su32(sa)), b0 = desc(su32(sb));
    unsigned long long t0 = clock64();
    for (int t = 0; t < tiles; ++t) {
      if (kWait) mbar_wait(&ready, 0);
      asm volatile("tcgen05.fence::after_thread_sync;");
      const uint32_t d = tmem + (uint32_t)((t & 1) * 256);
#pragma unroll
      for (int ks = 0; ks < KS; ++ks) {
        if (g_cp == 99 && ks > 0 && ks % 4 == 0) {  // per-chunk wait variant
          mbar_wait(&ready, 0);
          asm volatile("tcgen05.fence::after_thread_sync;");
        }
        const uint64_t ad = a0 + (uint64_t)((ks / 4) * (128 * 128 / 16) + (ks % 4) * 2);
        const uint64_t bd = b0 + (uint64_t)((ks / 4) * (256 * 128 / 16) + (ks % 4) * 2);
        asm volatile(
            "{.reg .pred p; setp.ne.b32 p, %4, 0;"
            " tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;}" ::
                "r"(d), "l"(ad), "l"(bd), "r"(idesc), "r"((uint32_t)(ks > 0)));
        if (ks % 4 == 3 || ks == KS - 1)
          asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&b1)));
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&b2)));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)));
    mbar_wait(&bar, 0);
    cyc[blockIdx.x] = clock64() - t0;
    stop_t = 1;
  } else if (kEpi && warp >= 2) {
    const int q = warp & 3, half = (warp - 2) >> 2;
    float s = 0.f;
    int it = 0;
    while (!stop_t) {
      const uint32_t ta = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)((it & 1) * 256 + half * 128);
#pragma unroll 1
      for (int c = 0; c < 128; c += 32) {
        uint32_t r[32];
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
            "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,"
            "%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
            : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]),
              "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]), "=r"(r[9]),
              "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
              "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
              "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
              "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]),
              "=r"(r[30]), "=r"(r[31])
            : "r"(ta + c));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
        for (int j = 0; j < 32; ++j) s += fmaxf(__uint_as_float(r[j]), 0.f);
      }
      ++it;
    }
    if (s == 12345.f) cyc[148 + threadIdx.x] = 1;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

template <int KS, bool kWait, bool kEpi = false>
int run_tight(const char *name, int tiles) {
  unsigned long long *cyc;
  CK(cudaMalloc(&cyc, 1024 * 8));
  size_t smem = 2 * 128 * 128 + 2 * 256 * 128 + 2048;
  CK(cudaFuncSetAttribute(probe_tight<KS, kWait, kEpi>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float ms = 0;
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(e0);
    probe_tight<KS, kWait, kEpi><<<148, 320, smem>>>(tiles, cyc);
    cudaEventRecord(e1);
    CK(cudaDeviceSynchronize());
    cudaEventElapsedTime(&ms, e0, e1);
  }
  unsigned long long h[148];
  CK(cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost));
  double avg = 0;
  for (int i = 0; i < 148; ++i) avg += (double)h[i];
  avg /= 148;
  printf("%-34s cyc/mma %7.1f  %.1f ms  clk %.0f MHz  %.0f TFLOP/s\n", name,
         avg / ((double)tiles * KS), ms, avg / (ms * 1e3),
         2.0 * 128 * 256 * 16 * (double)tiles * KS * 148 / (ms * 1e9));
  cudaFree(cyc);
  return 0;
}

// Ping-pong probe: the tight MMA issuer and 8 epilogue warps synchronised
// exactly like K3-TC (tfull/tempty mbarriers per TMEM buffer), no TMA.
// NB accumulator buffers of N columns each (NB*N <= 512).
template <int N, int NB, int KS>
__global__ void __launch_bounds__(320, 1)
    probe_pp(int tiles, unsigned long long *cyc, float *sink) {
  extern __shared__ __align__(1024) unsigned char sm_raw[];
  unsigned char *sm =
      (unsigned char *)(((uintptr_t)sm_raw + 1023) & ~(uintptr_t)1023);
  unsigned char *sa = sm, *sb = sm + 2 * 128 * 128;
  __shared__ uint64_t bar, tfull[NB], tempty[NB];
  __shared__ uint32_t slot;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  for (int i = threadIdx.x; i < (2 * 128 * 128 + 2 * N * 128) / 4; i += blockDim.x)
    ((uint32_t *)sm)[i] = fill_word(i);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    for (int b = 0; b < NB; ++b) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&tfull[b])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 8;" ::"r"(su32(&tempty[b])));
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = slot;
  const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
  if (warp == 1 && lane == 0) {
    const uint64_t a0 = desc(su32(sa)), b0 = desc(su32(sb));
    unsigned long long t0 = clock64();
    uint32_t tph = 0;
    for (int t = 0; t < tiles; ++t) {
      const int b = t % NB;
      mbar_wait(&tempty[b], ((tph >> b) & 1u) ^ 1u);
      tph ^= 1u << b;
      asm volatile("tcgen05.fence::after_thread_sync;");
      const uint32_t d = tmem + (uint32_t)(b * N);
#pragma unroll
      for (int ks = 0; ks < KS; ++ks) {
        const uint64_t ad = a0 + (uint64_t)((ks / 4) * (128 * 128 / 16) + (ks % 4) * 2);
        const uint64_t bd = b0 + (uint64_t)((t % g_rot) * (2 * N * 128 / 16)) + (uint64_t)((ks / 4) * (N * 128 / 16) + (ks % 4) * 2);
        asm volatile(
            "{.reg .pred p; setp.ne.b32 p, %4, 0;"
            " tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;}" ::
                "r"(d), "l"(ad), "l"(bd), "r"(idesc), "r"((uint32_t)(ks > 0)));
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&tfull[b])));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)));
    mbar_wait(&bar, 0);
    cyc[blockIdx.x] = clock64() - t0;
  } else if (warp >= 2) {
    const int q = warp & 3, half = (warp - 2) >> 2;
    float s = 0.f;
    uint32_t tph = 0;
    for (int t = 0; t < tiles; ++t) {
      const int b = t % NB;
      mbar_wait(&tfull[b], (tph >> b) & 1u);
      tph ^= 1u << b;
      asm volatile("tcgen05.fence::after_thread_sync;");
      const uint32_t ta = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(b * N + half * (N / 2));
      uint32_t r[N / 2];
#pragma unroll
      for (int c = 0; c < N / 2; c += 32)
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
            "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,"
            "%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
            : "=r"(r[c + 0]), "=r"(r[c + 1]), "=r"(r[c + 2]), "=r"(r[c + 3]), "=r"(r[c + 4]),
              "=r"(r[c + 5]), "=r"(r[c + 6]), "=r"(r[c + 7]), "=r"(r[c + 8]), "=r"(r[c + 9]),
              "=r"(r[c + 10]), "=r"(r[c + 11]), "=r"(r[c + 12]), "=r"(r[c + 13]), "=r"(r[c + 14]),
              "=r"(r[c + 15]), "=r"(r[c + 16]), "=r"(r[c + 17]), "=r"(r[c + 18]), "=r"(r[c + 19]),
              "=r"(r[c + 20]), "=r"(r[c + 21]), "=r"(r[c + 22]), "=r"(r[c + 23]), "=r"(r[c + 24]),
              "=r"(r[c + 25]), "=r"(r[c + 26]), "=r"(r[c + 27]), "=r"(r[c + 28]), "=r"(r[c + 29]),
              "=r"(r[c + 30]), "=r"(r[c + 31])
            : "r"(ta + c));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      asm volatile("tcgen05.fence::before_thread_sync;");
      __syncwarp();
      if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&tempty[b])) : "memory");
#pragma unroll
      for (int j = 0; j < N / 2; ++j) s += fmaxf(__uint_as_float(r[j]), 0.f);
    }
    sink[blockIdx.x * 320 + threadIdx.x] = s;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

template <int N, int NB, int KS>
int run_pp(const char *name, int tiles) {
  unsigned long long *cyc;
  float *sink;
  CK(cudaMalloc(&cyc, 148 * 8));
  CK(cudaMalloc(&sink, 148 * 320 * 4));
  int rot = 1;
  if (const char *r = getenv("PROBE_ROT")) rot = atoi(r);
  cudaMemcpyToSymbol(g_rot, &rot, sizeof(int));
  size_t smem = 2 * 128 * 128 + (size_t)rot * 2 * N * 128 + 2048;
  if (getenv("PROBE_BIG_SMEM")) smem = 224 * 1024;
  CK(cudaFuncSetAttribute(probe_pp<N, NB, KS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  for (int rep = 0; rep < 2; ++rep) {
    probe_pp<N, NB, KS><<<148, 320, smem>>>(tiles, cyc, sink);
    CK(cudaDeviceSynchronize());
  }
  unsigned long long h[148];
  CK(cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost));
  double avg = 0;
  for (int i = 0; i < 148; ++i) avg += (double)h[i];
  avg /= 148;
  const double ideal = (double)N / 2 * KS;  // cycles per tile at 4096 MAC/clk
  printf("%-34s cyc/tile %7.1f  (ideal %5.0f)  eff %.2f\n", name, avg / tiles, ideal, ideal * tiles / avg);
  cudaFree(cyc);
  cudaFree(sink);
  return 0;
}

int main(int argc, char **argv) {
  const int T = 4000, K = 7;
  if (argc > 1 && argv[1][0] == 'c' && argv[1][1] == 'm') {  // commit cost
    int dm = 1;
    cudaMemcpyToSymbol(g_data, &dm, sizeof(int));
    run<128, 256, 1, false>("cg1 N256 no commits", T, K);
    run<128, 256, 1, false, true>("cg1 N256 commit/1", T, K, 1);
    run<128, 256, 1, false, true>("cg1 N256 commit/2", T, K, 2);
    run<128, 256, 1, false, true>("cg1 N256 commit/4", T, K, 4);
    run<128, 256, 1, false, true>("cg1 N256 commit/7", T, K, 7);
    run<128, 256, 1, false, true>("cg1 N256 commit/28", T, K, 28);
    return 0;
  }
  if (argc > 1) {  // cta_group::2 shapes only
    int dm = 1;
    cudaMemcpyToSymbol(g_data, &dm, sizeof(int));
    run<128, 256, 1, false>("cg1 M128 N256", T, K);
    run<256, 256, 2, false>("cg2 M256 N256", T, K);
    run<256, 128, 2, false>("cg2 M256 N128", 2 * T, K);
    run<256, 256, 2, true>("cg2 M256 N256 +ldtm", T, K);
    return 0;
  }
  for (int dm = 0; dm < 3; ++dm) {
    cudaMemcpyToSymbol(g_data, &dm, sizeof(int));
    printf("--- operand data mode %d (0 small-positive, 1 gaussian-like, 2 zeros)\n", dm);
    run_tight<7, true>("tight K7 +wait/tile", T);
    run_tight<7, true, true>("tight K7 +epi LONG", 300000);
    run_pp<256, 2, 7>("pingpong N256 x2 K7", T);
  }
  {
    int dm = 1;
    cudaMemcpyToSymbol(g_data, &dm, sizeof(int));
  }
  run_pp<256, 2, 7>("pingpong N256 x2 K7", T);
  run_pp<128, 4, 7>("pingpong N128 x4 K7", 2 * T);
  run_pp<128, 2, 7>("pingpong N128 x2 K7", 2 * T);
  run_pp<256, 2, 14>("pingpong N256 x2 K14", T);
  run_tight<7, false>("tight K7 2 commits/tile", T);
  run_tight<7, true, true>("tight K7 +epi", T);
  run_tight<7, true, true>("tight K7 +epi LONG", 1500000);
  run_tight<7, true, false>("tight K7 LONG (no epi)", 1500000);
  run_tight<7, true>("tight K7 +wait/tile", T);
  run_tight<2, true>("tight K2 +wait/tile", T);
  run_tight<4, true>("tight K4 +wait/tile", T);
  run_tight<8, true>("tight K8 +wait/tile", T);
  {
    int cp = 99;
    cudaMemcpyToSymbol(g_cp, &cp, sizeof(int));
    run_tight<7, true>("tight K7 +wait/chunk(4)", T);
    run_tight<16, true>("tight K16 +wait/chunk(4)", T);
    cp = 4;
    cudaMemcpyToSymbol(g_cp, &cp, sizeof(int));
  }
  run<128, 256, 1, false>("cg1 M128 N256", T, K);
  run<128, 256, 1, false, true>("cg1 N256 commit/4", T, K, 4);
  run<128, 256, 1, false, true>("cg1 N256 commit/7", T, K, 7);
  run<128, 256, 1, false, true>("cg1 N256 commit/14", T, K, 14);
  run<128, 256, 1, false, true>("cg1 N256 commit/28", T, K, 28);
  run<128, 256, 1, false, true>("cg1 N256 commit/56", T, K, 56);
  run<128, 256, 1, true, true>("cg1 N256 +ldtm commit/7", T, K, 7);
  run<256, 256, 2, false, true>("cg2 N256 commit/7", T, K, 7);
  run<128, 256, 1, false, false, true>("cg1 M128 N256 +tma", T, K);
  run<128, 256, 1, true, true, true>("cg1 M128 N256 +ldtm+commit+tma", T, K);
  run<128, 256, 1, true>("cg1 M128 N256 +ldtm epilogue", T, K);
  run<128, 128, 1, false>("cg1 M128 N128", T, K);
  run<128, 128, 1, true>("cg1 M128 N128 +ldtm", T, K);
  run<128, 64, 1, false>("cg1 M128 N64", T, K);
  run<256, 256, 2, false>("cg2 M256 N256", T, K);
  run<256, 256, 2, true>("cg2 M256 N256 +ldtm", T, K);
  run<256, 128, 2, false>("cg2 M256 N128", T, K);
  return 0;
}
