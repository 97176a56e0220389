// epi_probe.cu -- instruction-mix throughput of the K3-TC relu-sum epilogue.
//
// Per (candidate, point) value x the epilogue must add max(0, x) to a
// running fp32 sum.  Two exact forms:
//   A  t = FMNMX(x, 0)       (ALU pipe)  ; acc += t   (FMA pipe)
//   B  t = FADD(x, |x|) = 2 max(0, x), exact (x + |x| is 0 or 2x)
//                            (FMA pipe)  ; acc2 += t  (FMA pipe)
// and the sign screen S: 32 values AND-ed with LOP3 (ALU).  This measures
// G values/s for A only, B only and mixes of A and B per 12 values, all with
// 12 independent accumulators per thread, 148 SMs x 4 CTAs x 256 threads.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o epi_probe epi_probe.cu
#include <cuda_runtime.h>
#include <stdio.h>

template <int NB>  // NB of every 12 values use form B, the rest form A
__global__ void __launch_bounds__(256) mix_loop(float *out, int iters) {
  float acc[12];
#pragma unroll
  for (int j = 0; j < 12; ++j) acc[j] = (float)(threadIdx.x + j) - 128.f;
#pragma unroll 1
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
#pragma unroll
      for (int j = 0; j < 12; ++j) {
        // x = another chain's accumulator: loop-varying, so nothing is
        // hoisted; 12 independent chains of 2 dependent ops per thread
        const float x = acc[(j + 1) % 12];
        float t;
        if (j < NB) {
          asm volatile("{.reg .f32 a; abs.f32 a, %1; add.f32 %0, %1, a;}"
                       : "=f"(t) : "f"(x));
        } else {
          asm volatile("max.f32 %0, %1, 0f00000000;" : "=f"(t) : "f"(x));
        }
        asm volatile("add.f32 %0, %0, %1;" : "+f"(acc[j]) : "f"(t));
      }
    }
  }
  float s = 0.f;
#pragma unroll
  for (int j = 0; j < 12; ++j) s += acc[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void __launch_bounds__(256) screen_loop(unsigned *out, int iters) {
  unsigned r[32], c[4];
#pragma unroll
  for (int j = 0; j < 32; ++j) r[j] = threadIdx.x * 2654435761u + j;
#pragma unroll
  for (int j = 0; j < 4; ++j) c[j] = threadIdx.x + j;
#pragma unroll 1
  for (int i = 0; i < iters; ++i) {
    // four independent AND chains over 8 values each (32 values per pass)
#pragma unroll
    for (int j = 0; j < 8; j += 2)
#pragma unroll
      for (int q = 0; q < 4; ++q)
        asm volatile("lop3.b32 %0, %0, %1, %2, 0x80;" : "+r"(c[q])
                     : "r"(r[q * 8 + j]), "r"(r[q * 8 + j + 1]));
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = c[0] ^ c[1] ^ c[2] ^ c[3];
}

template <typename K>
static float best_ms(K kern, int blocks, int iters) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  kern(blocks, iters / 10);
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < 10; ++r) {
    cudaEventRecord(e0);
    kern(blocks, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  return best;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk_khz = 0;
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  const int blocks = sms * 4, iters = 20000;
  float *out;
  cudaMalloc(&out, sizeof(float) * blocks * 256);
  const double vals = (double)blocks * 256 * iters * 8 * 12;
  printf("{\"sm_count\": %d, \"max_clock_ghz\": %.3f", sms, clk_khz / 1e6);
#define MIX(NB)                                                              \
  {                                                                          \
    const float ms = best_ms(                                                \
        [&](int b, int it) { mix_loop<NB><<<b, 256>>>(out, it); }, blocks,   \
        iters);                                                              \
    const double g = vals / (ms * 1e-3) / 1e9;                               \
    printf(", \"mix_B%02d_of_12_gvals\": %.1f, \"mix_B%02d_per_clk_sm\": %.1f", \
           NB, g, NB, g * 1e9 / sms / (clk_khz * 1e3));                      \
  }
  MIX(0) MIX(3) MIX(4) MIX(6) MIX(8) MIX(9) MIX(12)
  {
    const float ms = best_ms(
        [&](int b, int it) { screen_loop<<<b, 256>>>((unsigned *)out, it); },
        blocks, iters * 8);
    const double g = (double)blocks * 256 * iters * 8 * 32 / (ms * 1e-3) / 1e9;
    printf(", \"screen_gvals\": %.1f, \"screen_per_clk_sm\": %.1f", g,
           g * 1e9 / sms / (clk_khz * 1e3));
  }
  printf(", \"note\": \"values/clk/SM at the max clock (an upper clock): "
         "A = FMNMX + FADD, B = FADD(x,|x|) + FADD\"}\n");
  return 0;
}
