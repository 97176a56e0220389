// exem_simt_tma.cu -- K3-SIMT (binary32 / binary64 Greedy gains on the CUDA
// cores) with TMA-fed operand tiles, sm_100a.
//
// Same arithmetic as gains_simt_kernel (exem_simt.cu): for a 128-candidate x
// 128-point tile every thread keeps an 8 x 8 register block of dot products
// initialised with -(h_i + b_c) and runs the same sequential fma chain over
// the dimensions, then the relu-sum epilogue
//   partial[split][c] = sum_i max(0, c.v_i - h_i - b_c),  (x2 in K6)
// for the reference's Greedy step (pkg/src/exembatch/optimize.py:61-71) in
// its optimizer-aware form.  Results are bit-identical
// to gains_simt_kernel.
//
// What changes is how operands arrive: the round-1 kernel copies every
// chunk with per-thread cp.async (address arithmetic and a CTA barrier per
// chunk: 85 % issue utilisation with only 87 % of issued instructions FFMA,
// profiles/r01d_simt_ncu.md).  Here one elected thread issues two TMA boxes
// per chunk ([BK dims][128 candidates] of cvt, [BK][128 points] of vt, both
// column-major like the reference's V, src/core.py:286) into an S-stage
// ring with mbarrier completion, and the stage is refilled by the last warp
// that finishes it (no producer role, no CTA barrier per chunk).
#include <cstdlib>

#include "exem_tc_common.cuh"

namespace exem {

namespace {

constexpr int kTM = 128, kTN = 128, kThr = 256, kWarps = kThr / 32;
// ring depth: 4 stages of 16-dimension chunks or 8 of 8 (d_pad % 16 != 0)
template <int BK> constexpr int stages_of() { return BK == 16 ? 4 : 8; }

__device__ __forceinline__ int toff(int t4, int r) {
  return r < 4 ? t4 * 4 + r : 64 + t4 * 4 + (r - 4);
}

template <typename T, int BK>
__global__ void __launch_bounds__(kThr, sizeof(T) == 4 ? 2 : 1)
    gains_simt_tma_kernel(const __grid_constant__ CUtensorMap map_c,
                          const __grid_constant__ CUtensorMap map_v,
                          const double *__restrict__ cnorms, int64_t l,
                          const double *__restrict__ norms,
                          const T *__restrict__ m, int64_t n, int d_pad,
                          int64_t split_pts, double *__restrict__ partial) {
  constexpr int STAGE = 2 * BK * kTM;  // A then B, values
  constexpr int kStages = stages_of<BK>();
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  T *ring = reinterpret_cast<T *>(smem_raw);  // [S][2][BK][128]
  __shared__ __align__(8) uint64_t full[8];
  __shared__ uint32_t rel[8];
  __shared__ T s_b[kTM];
  __shared__ T s_h[kTN];
  const int tid = threadIdx.x, lane = tid & 31;
  const int tx = tid % 16, ty = tid / 16;
  const int64_t c0 = (int64_t)blockIdx.x * kTM;
  const int64_t split = blockIdx.y;
  const int64_t p_begin = split * split_pts;
  const int64_t p_end = n < p_begin + split_pts ? n : p_begin + split_pts;
  const int nk = d_pad / BK;
  const uint32_t ntiles = (uint32_t)((p_end - p_begin + kTN - 1) / kTN);
  const uint32_t total = ntiles * (uint32_t)nk;

  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) {
      tc::mbar_init(&full[s], 1);
      rel[s] = 0;
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (tid < kTM) s_b[tid] = (c0 + tid < l) ? (T)(0.5 * cnorms[c0 + tid]) : T(0);
  __syncthreads();

  auto issue = [&](uint32_t ev) {
    const int s = ev % kStages;
    const int64_t p0 = p_begin + (int64_t)(ev / nk) * kTN;
    const int c = (int)(ev % nk);
    T *dst = ring + s * STAGE;
    tc::mbar_expect_tx(&full[s], (uint32_t)(STAGE * sizeof(T)));
    tc::tma_load_2d(dst, &map_c, &full[s], (int)c0, c * BK);
    tc::tma_load_2d(dst + BK * kTM, &map_v, &full[s], (int)p0, c * BK);
  };
  if (tid == 0)
    for (uint32_t ev = 0; ev < total && ev < (uint32_t)kStages; ++ev) issue(ev);

  double g[8];
#pragma unroll
  for (int r = 0; r < 8; ++r) g[r] = 0.0;
  uint32_t ev = 0;
  for (uint32_t t = 0; t < ntiles; ++t) {
    const int64_t p0 = p_begin + (int64_t)t * kTN;
    __syncthreads();  // previous tile's s_h reads are done
    if (tid < kTN) {
      const int64_t pi = p0 + tid;
      s_h[tid] = pi < p_end ? (T)(0.5 * (norms[pi] - (double)m[pi])) : tinf<T>();
    }
    __syncthreads();
    T acc[8][8];
#pragma unroll
    for (int r = 0; r < 8; ++r)
#pragma unroll
      for (int c = 0; c < 8; ++c)
        acc[r][c] = -(s_h[toff(tx, c)] + s_b[toff(ty, r)]);
    for (int c = 0; c < nk; ++c, ++ev) {
      const int s = ev % kStages;
      tc::mbar_wait_hint(&full[s], (ev / kStages) & 1);
      const T *sa = ring + s * STAGE;
      const T *sb = sa + BK * kTM;
#pragma unroll
      for (int kk = 0; kk < BK; ++kk) {
        T a[8], b[8];
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          a[r] = sa[kk * kTM + ty * 4 + r];
          a[4 + r] = sa[kk * kTM + 64 + ty * 4 + r];
          b[r] = sb[kk * kTN + tx * 4 + r];
          b[4 + r] = sb[kk * kTN + 64 + tx * 4 + r];
        }
#pragma unroll
        for (int r = 0; r < 8; ++r)
#pragma unroll
          for (int q = 0; q < 8; ++q) acc[r][q] = fma(a[r], b[q], acc[r][q]);
      }
      __syncwarp();  // every lane's reads of the stage are consumed
      if (lane == 0) {
        __threadfence_block();
        if (atomicAdd(&rel[s], 1u) == (uint32_t)kWarps - 1) {
          rel[s] = 0;  // nobody touches it before the refill lands
          const uint32_t nev = ev + (uint32_t)kStages;
          if (nev < total) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            issue(nev);
          }
        }
      }
    }
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      T s = T(0);
#pragma unroll
      for (int q = 0; q < 8; ++q) s += tmax(acc[r][q], T(0));
      g[r] += (double)s;
    }
  }
#pragma unroll
  for (int r = 0; r < 8; ++r) {
    double v = g[r];
#pragma unroll
    for (int o = 8; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    const int64_t ci = c0 + toff(ty, r);
    if (tx == 0 && ci < l) partial[split * l + ci] = v;
  }
}

int make_map_simt(CUtensorMap *map, const void *base, bool f64, int64_t ld,
                  int64_t rows, int bk) {
  auto enc = tc::get_encode();
  if (!enc) return 1;
  const int vb = f64 ? 8 : 4;
  cuuint64_t gdim[2] = {(cuuint64_t)ld, (cuuint64_t)rows};
  cuuint64_t gstride[1] = {(cuuint64_t)(ld * vb)};
  cuuint32_t box[2] = {(cuuint32_t)kTM, (cuuint32_t)bk};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(map,
                   f64 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64
                       : CU_TENSOR_MAP_DATA_TYPE_FLOAT32,
                   2, const_cast<void *>(base), gdim, gstride, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? 0 : 1;
}

template <typename T, int BK>
cudaError_t launch_simt_tma(const CUtensorMap &mc, const CUtensorMap &mv,
                            dim3 grid, cudaStream_t st, const double *cnorms,
                            int64_t l, const double *norms, const void *m,
                            int64_t n, int d_pad, int64_t split_pts,
                            double *partial) {
  const size_t smem = (size_t)stages_of<BK>() * 2 * BK * kTM * sizeof(T);
  cudaError_t e = cudaFuncSetAttribute(
      gains_simt_tma_kernel<T, BK>,
      cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  gains_simt_tma_kernel<T, BK><<<grid, kThr, smem, st>>>(
      mc, mv, cnorms, l, norms, (const T *)m, n, d_pad, split_pts, partial);
  return cudaGetLastError();
}

}  // namespace

// K3-SIMT with TMA operands: 0 launched, 1 not applicable (caller uses the
// cp.async kernel), < 0 a CUDA error.  Same grid and partial layout as
// gains_simt_kernel: (candidate tiles of 128, splits).
int gains_simt_tma(int dtype, const void *cvt, int64_t ldc,
                   const double *cnorms, int64_t l, const void *vt, int64_t ld,
                   const double *norms, const void *m, int64_t n, int d_pad,
                   int64_t split_pts, int64_t splits, double *partial,
                   cudaStream_t st) {
  // binary64 only: same-box A/B against the cp.async kernel (tools/simt_ab.py,
  // n = 100k, ms per Greedy step): f64 d = 100 87.1 vs 92.7 (this kernel
  // wins); f32 d = 16 / 100 / 1024 7.81 / 43.9 / 382 vs 7.60 / 39.5 / 374
  // (the cp.async kernel wins: at 4-byte values its one CTA barrier per
  // chunk is cheaper than the per-warp mbarrier round trips).
  // EXEM_SIMT_TMA=1 / EXEM_SIMT_CPASYNC=1 force either (experiments only).
  if (dtype != EXEM_F32 && dtype != EXEM_F64) return 1;
  if (getenv("EXEM_SIMT_CPASYNC")) return 1;
  if (dtype == EXEM_F32 && !getenv("EXEM_SIMT_TMA")) return 1;
  const bool f64 = dtype == EXEM_F64;
  const int bk = d_pad % 16 == 0 ? 16 : 8;
  if (d_pad % bk != 0 || ldc % kTM || ld % kTN) return 1;
  CUtensorMap mc, mv;
  if (make_map_simt(&mc, cvt, f64, ldc, d_pad, bk)) return 1;
  if (make_map_simt(&mv, vt, f64, ld, d_pad, bk)) return 1;
  dim3 grid((unsigned)ceil_div(l, kTM), (unsigned)splits);
  cudaError_t e;
#define EXEM_SIMT_TMA(T, B)                                                   \
  e = launch_simt_tma<T, B>(mc, mv, grid, st, cnorms, l, norms, m, n, d_pad, \
                            split_pts, partial)
  if (f64) {
    if (bk == 16) EXEM_SIMT_TMA(double, 16); else EXEM_SIMT_TMA(double, 8);
  } else {
    if (bk == 16) EXEM_SIMT_TMA(float, 16); else EXEM_SIMT_TMA(float, 8);
  }
#undef EXEM_SIMT_TMA
  return e == cudaSuccess ? 0 : -(int)e;
}

}  // namespace exem
