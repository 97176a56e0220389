// simt_peak.cu -- FP32 FFMA / FP64 DFMA throughput microbenchmark (B200).
//
// The roofline denominators for the SIMT kernels (K3-SIMT, K4 at f32/f64)
// are not in MEASURED_PEAKS.json (which holds HBM copy and cuBLAS bf16), so
// this measures them: every thread runs 8 independent FMA chains for a fixed
// trip count, grid = SMs x 4 CTAs x 256 threads, CUDA events around the
// launch, best of 10.  Also reports cycles via clock64 on CTA 0 so the rate
// can be normalised per SM clock.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o simt_peak simt_peak.cu
//   ./simt_peak   -> one JSON line
#include <cuda_runtime.h>
#include <stdio.h>

template <typename T>
__global__ void __launch_bounds__(256) fma_loop(T *out, int iters, T a, T b,
                                                long long *cyc) {
  T x0 = (T)threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4,
    x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  const long long c0 = clock64();
#pragma unroll 1
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b);
      x3 = fma(x3, a, b); x4 = fma(x4, a, b); x5 = fma(x5, a, b);
      x6 = fma(x6, a, b); x7 = fma(x7, a, b);
    }
  }
  const long long c1 = clock64();
  if (blockIdx.x == 0 && threadIdx.x == 0) *cyc = c1 - c0;
  out[blockIdx.x * blockDim.x + threadIdx.x] =
      x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}

// The relu-sum epilogue of K3 per (candidate, point) pair: one FMNMX (ALU
// pipe) + one FADD (FMA pipe).  Volatile asm keeps both instructions in the
// loop (nothing is hoisted); 8 independent accumulators per thread.
__global__ void __launch_bounds__(256) relu_sum_loop(float *out, int iters,
                                                     long long *cyc) {
  float x[8], acc[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    x[j] = (float)(threadIdx.x + j) - 128.f;
    acc[j] = 0.f;
  }
  const float z = -0.5f;
  const long long c0 = clock64();
#pragma unroll 1
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        float t;  // loop-carried through acc so nothing is hoisted
        asm volatile("max.f32 %0, %1, %2;" : "=f"(t) : "f"(acc[j]), "f"(x[j]));
        asm volatile("add.f32 %0, %1, %2;" : "=f"(acc[j]) : "f"(t), "f"(z));
      }
    }
  }
  const long long c1 = clock64();
  if (blockIdx.x == 0 && threadIdx.x == 0) *cyc = c1 - c0;
  float s = 0.f;
#pragma unroll
  for (int j = 0; j < 8; ++j) s += acc[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// Register outer-product FFMA (the SIMT kernels' inner loop): per thread
// 8 x 8 accumulators fed by 8 + 8 per-thread register operands, no uniform
// or immediate operands (FFMA with three general registers).
__global__ void __launch_bounds__(256) outer_loop(float *out, const float *in,
                                                  int iters) {
  float a[8], b[8], acc[8][8];
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    a[j] = in[(threadIdx.x + j) & 255];
    b[j] = in[(threadIdx.x + 8 + j) & 255];
  }
#pragma unroll
  for (int r = 0; r < 8; ++r)
#pragma unroll
    for (int c = 0; c < 8; ++c) acc[r][c] = 0.f;
#pragma unroll 1
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int r = 0; r < 8; ++r)
#pragma unroll
      for (int c = 0; c < 8; ++c) acc[r][c] = fmaf(a[r], b[c], acc[r][c]);
  }
  float s = 0.f;
#pragma unroll
  for (int r = 0; r < 8; ++r)
#pragma unroll
    for (int c = 0; c < 8; ++c) s += acc[r][c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

static double run_outer(int sms, int iters) {
  const int blocks = sms * 2, threads = 256;
  float *out, *in;
  cudaMalloc(&out, sizeof(float) * blocks * threads);
  cudaMalloc(&in, sizeof(float) * 256);
  cudaMemset(in, 0, sizeof(float) * 256);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  outer_loop<<<blocks, threads>>>(out, in, iters / 10);
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < 10; ++r) {
    cudaEventRecord(e0);
    outer_loop<<<blocks, threads>>>(out, in, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  cudaFree(out);
  cudaFree(in);
  return 2.0 * blocks * threads * (double)iters * 64 / (best * 1e-3) / 1e12;
}

// The relu-sum as the K3-TC epilogue now computes it: per value pair one
// FADD2 forming (x + |x|) = 2 max(0, x) for both values and one FADD2 adding
// them to a pair of running sums (1 instruction per value).  x is another
// chain's sum, so nothing is hoisted; 8 independent pairs per thread.
__global__ void __launch_bounds__(256) relu_fadd2_loop(float *out, int iters) {
  float2 acc[8];
#pragma unroll
  for (int j = 0; j < 8; ++j)
    acc[j] = make_float2((float)(threadIdx.x + j) - 128.f, (float)j - 3.f);
#pragma unroll 1
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const float2 x = acc[(j + 1) & 7];
        const float2 ax = make_float2(fabsf(x.x), fabsf(x.y));
        acc[j] = __fadd2_rn(acc[j], __fadd2_rn(x, ax));
      }
    }
  }
  float s = 0.f;
#pragma unroll
  for (int j = 0; j < 8; ++j) s += acc[j].x + acc[j].y;
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

static double run_relu2(int sms, int iters) {
  const int blocks = sms * 4, threads = 256;
  float *out;
  cudaMalloc(&out, sizeof(float) * blocks * threads);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  relu_fadd2_loop<<<blocks, threads>>>(out, iters / 10);
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < 10; ++r) {
    cudaEventRecord(e0);
    relu_fadd2_loop<<<blocks, threads>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  cudaFree(out);
  const double vals = (double)blocks * threads * iters * 16 * 8 * 2;
  return vals / (best * 1e-3) / 1e9;  // G values/s
}

static double run_relu(int sms, int iters, double *ghz) {
  const int blocks = sms * 4, threads = 256;
  float *out;
  long long *cyc;
  cudaMalloc(&out, sizeof(float) * blocks * threads);
  cudaMalloc(&cyc, sizeof(long long));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  relu_sum_loop<<<blocks, threads>>>(out, iters / 10, cyc);
  cudaDeviceSynchronize();
  float best = 1e30f;
  long long cbest = 0;
  for (int r = 0; r < 10; ++r) {
    cudaEventRecord(e0);
    relu_sum_loop<<<blocks, threads>>>(out, iters, cyc);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) {
      best = ms;
      cudaMemcpy(&cbest, cyc, sizeof(cbest), cudaMemcpyDeviceToHost);
    }
  }
  const double pairs = (double)blocks * threads * iters * 16 * 8;
  *ghz = (double)cbest / (best * 1e-3) / 1e9;
  cudaFree(out);
  cudaFree(cyc);
  return pairs / (best * 1e-3) / 1e9;  // G pairs/s
}

template <typename T>
static double run(int sms, int iters, double *ghz) {
  const int blocks = sms * 4, threads = 256;
  T *out;
  long long *cyc;
  cudaMalloc(&out, sizeof(T) * blocks * threads);
  cudaMalloc(&cyc, sizeof(long long));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  fma_loop<T><<<blocks, threads>>>(out, iters / 10, (T)0.999, (T)0.001, cyc);
  cudaDeviceSynchronize();
  float best = 1e30f;
  long long cbest = 0;
  for (int r = 0; r < 10; ++r) {
    cudaEventRecord(e0);
    fma_loop<T><<<blocks, threads>>>(out, iters, (T)0.999, (T)0.001, cyc);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) {
      best = ms;
      cudaMemcpy(&cbest, cyc, sizeof(cbest), cudaMemcpyDeviceToHost);
    }
  }
  const double fmas = (double)blocks * threads * iters * 16 * 8;
  *ghz = (double)cbest / (best * 1e-3) / 1e9;  // CTA-0 cycles / wall time
  cudaFree(out);
  cudaFree(cyc);
  return 2.0 * fmas / (best * 1e-3) / 1e12;  // TFLOP/s
}

int main() {
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  double g32, g64, gr;
  const double f32 = run<float>(sms, 20000, &g32);
  const double f64 = run<double>(sms, 4000, &g64);
  const double relu = run_relu(sms, 20000, &gr);
  const double outer = run_outer(sms, 20000);
  const double relu2 = run_relu2(sms, 20000);
  (void)g64;
  printf("{\"sm_count\": %d, \"fp32_ffma_tflops\": %.2f,"
         " \"fp32_ffma_reg_outer_tflops\": %.2f,"
         " \"fp64_dfma_tflops\": %.2f, \"relu_sum_gpairs\": %.1f,"
         " \"relu_sum_fadd2_gpairs\": %.1f,"
         " \"clock_ghz_ffma\": %.3f, \"clock_ghz_relu\": %.3f,"
         " \"how\": \"8 independent FMA chains/thread, %d SMs x 4 CTAs x 256 thr,"
         " best of 10, CUDA events; relu_sum = FMNMX + FADD per pair\"}\n",
         sms, f32, outer, f64, relu, relu2, g32, gr, sms);
  return 0;
}
