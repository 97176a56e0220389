// exem_simt.cu -- CUDA-core (FFMA/DFMA) kernels for sm_100a and their
// C-ABI entry points.
//
//   K1 ground_prepare   core.py:286-309        (HBM-bound)
//   K2 set_min / greedy_update / greedy_init  objective.py:113-141,
//                       evaluate.py:105-112, optimize.py:74-76 (HBM-bound)
//   K3 greedy_gains_simt  optimize.py:61-71    (FFMA/DFMA-bound)
//   K4 batch_eval       evaluate.py:142-149,197-270 over pack_batch layout
//                       core.py:331-346        (FFMA/DFMA-bound)
//   K5 argmax_select    optimize.py:73-76      (latency)
//   K6 reduce_partials  evaluate.py:111        (HBM/latency)
//
// All sums are accumulated in fp64 with a fixed reduction order, so every
// output is bit-reproducible for a given (n, split_pts) -- the analogue of the
// reference's fixed COL_BLOCK sweep (core.py:27-30).
#include <cfloat>

#include <cstring>

#include <cstdlib>

#include "exem_common.cuh"

namespace exem {

static thread_local char g_err[1024] = "";
static unsigned long long g_launches = 0;

void set_error(const char *fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}
int fail(int code, const char *fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return code;
}
void count_launch() { __atomic_add_fetch(&g_launches, 1ull, __ATOMIC_RELAXED); }

constexpr int kRedThreads = 256;

// Final fixed-order reduction of block partials (one block).
__global__ void __launch_bounds__(1024)
    reduce_fixed_kernel(const double *__restrict__ in, int64_t count,
                        double *__restrict__ out, int64_t out_index) {
  __shared__ double sh[32];
  double s = 0.0;
  for (int64_t i = threadIdx.x; i < count; i += blockDim.x) s += in[i];
  double r = block_sum<1024>(s, sh);
  if (threadIdx.x == 0) out[out_index] = r;
}

static int reduce_fixed(const double *partials, int64_t count, double *out,
                        int64_t out_index, cudaStream_t st) {
  reduce_fixed_kernel<<<1, 1024, 0, st>>>(partials, count, out, out_index);
  EXEM_LAUNCH_CHECK("reduce_fixed_kernel");
  return EXEM_OK;
}

// ============================================================ K1 prepare
// Non-finite stored values, detected on the device: for f32/f16/bf16 storage
// ||v_i||^2 (accumulated in fp64, which cannot overflow for these widths) is
// finite iff every coordinate is, so a non-finite norm turns the point's aux
// term into NaN and the fixed-order aux sum is NaN iff some stored value is
// inf/NaN (aux terms of finite points are never NaN).  The host raises
// InvalidDataError on it instead of scanning V itself (core.py).  Binary64
// storage keeps the host check (a finite 1e200 would overflow the norm).
template <int DT>
__device__ __forceinline__ double nonfinite_mark(bool mark, double nrm,
                                                 double term) {
  if (DT != EXEM_F64 && mark && !isfinite(nrm))
    return __longlong_as_double(0x7ff8000000000000LL);
  return term;
}

template <int DT, bool VS>
__global__ void __launch_bounds__(kRedThreads)
    ground_prepare_kernel(const typename Traits<DT>::S *__restrict__ src,
                          int64_t n, int d, int d_pad,
                          const typename Traits<DT>::S *__restrict__ e0,
                          typename VtOf<DT, VS>::T *__restrict__ vt, int64_t ld,
                          double *__restrict__ norms,
                          typename Traits<DT>::C *__restrict__ aux,
                          double *__restrict__ partials, bool mark) {
  using S = typename Traits<DT>::S;
  using C = typename Traits<DT>::C;
  using V = typename VtOf<DT, VS>::T;
  __shared__ double sh[32];
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  double nrm = 0.0, dst = 0.0;
  if (i < ld) {
    // HBM-bound: kLoadAheadK1 independent coalesced loads in flight per
    // thread, then the stores and the (same-order) fp64 accumulations
    // (16 for 2-byte sources: the same bytes in flight)
    constexpr int kLoadAheadK1 = sizeof(S) == 2 ? 16 : 8;
    const bool live = i < n;
    int k = 0;
    for (; k + kLoadAheadK1 <= d; k += kLoadAheadK1) {
      C xs[kLoadAheadK1];
#pragma unroll
      for (int u = 0; u < kLoadAheadK1; ++u)
        xs[u] = live ? to_c(src[(int64_t)(k + u) * n + i]) : C(0);
#pragma unroll
      for (int u = 0; u < kLoadAheadK1; ++u) {
        vt[(int64_t)(k + u) * ld + i] = to_vt<V>(xs[u]);
        if (live) {
          double xd = (double)xs[u];
          nrm += xd * xd;
          double df = xd - (double)to_c(e0[k + u]);
          dst += df * df;
        }
      }
    }
    for (; k < d_pad; ++k) {
      C x = C(0);
      if (k < d && live) x = to_c(src[(int64_t)k * n + i]);
      vt[(int64_t)k * ld + i] = to_vt<V>(x);
      if (k < d && live) {
        double xd = (double)x;
        nrm += xd * xd;
        double df = xd - (double)to_c(e0[k]);
        dst += df * df;
      }
    }
    // aux_distances are stored at the storage dtype (core.py:303-305);
    // bfloat16 (not a reference precision) keeps them at binary32.
    C a = C(0);
    if (i < n) a = (DT == EXEM_BF16) ? (C)dst : to_c(from_d<S>(dst));
    if (i < n) {
      norms[i] = nrm;
      aux[i] = a;
    } else {
      norms[i] = 0.0;
      aux[i] = C(0);
    }
    dst = (i < n) ? nonfinite_mark<DT>(mark, nrm, (double)a) : 0.0;
  }
  double r = block_sum<kRedThreads>(dst, sh);
  if (threadIdx.x == 0) partials[blockIdx.x] = r;
}

// K1 for 2-byte storage written as 2-byte vt (EXEM_VT_STORAGE, even n):
// 128 threads per 256 points, two adjacent points per thread, so every V
// access is a 4-byte pair (a warp moves 128 contiguous bytes per dimension)
// and the stored bits are copied untouched.  Per point the same sequential
// fp64 norm / aux accumulation as ground_prepare_kernel, and the block
// partial is block_sum<256>'s tree (pair_block_sum): bit-identical results.
template <int DT>
__global__ void __launch_bounds__(128)
    ground_prepare_pair_kernel(const typename Traits<DT>::S *__restrict__ src,
                               int64_t n, int d, int d_pad,
                               const typename Traits<DT>::S *__restrict__ e0,
                               typename Traits<DT>::S *__restrict__ vt,
                               int64_t ld, double *__restrict__ norms,
                               typename Traits<DT>::C *__restrict__ aux,
                               double *__restrict__ partials, bool mark) {
  using S = typename Traits<DT>::S;
  using C = typename Traits<DT>::C;
  __shared__ double sh[8];
  const int64_t i = (int64_t)blockIdx.x * 256 + 2 * threadIdx.x;
  const bool live = i < n;  // n even: both points of the pair or neither
  double nrm[2] = {0.0, 0.0}, dst[2] = {0.0, 0.0};
  auto accum = [&](uint32_t raw, int k) {
    const S *h = reinterpret_cast<const S *>(&raw);
    const double ek = (double)to_c(e0[k]);
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const double xd = (double)to_c(h[q]);
      nrm[q] += xd * xd;
      const double df = xd - ek;
      dst[q] += df * df;
    }
  };
  constexpr int LA = 8;
  int k = 0;
  for (; k + LA <= d; k += LA) {
    uint32_t xs[LA];
#pragma unroll
    for (int u = 0; u < LA; ++u)
      xs[u] = live ? *reinterpret_cast<const uint32_t *>(src + (int64_t)(k + u) * n + i)
                   : 0u;
#pragma unroll
    for (int u = 0; u < LA; ++u) {
      *reinterpret_cast<uint32_t *>(vt + (int64_t)(k + u) * ld + i) = xs[u];
      if (live) accum(xs[u], k + u);
    }
  }
  for (; k < d_pad; ++k) {
    uint32_t x = 0u;
    if (k < d && live)
      x = *reinterpret_cast<const uint32_t *>(src + (int64_t)k * n + i);
    *reinterpret_cast<uint32_t *>(vt + (int64_t)k * ld + i) = x;
    if (k < d && live) accum(x, k);
  }
  double part[2] = {0.0, 0.0};
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    C a = C(0);
    if (live) a = (DT == EXEM_BF16) ? (C)dst[q] : to_c(from_d<S>(dst[q]));
    norms[i + q] = live ? nrm[q] : 0.0;
    aux[i + q] = a;
    part[q] = live ? nonfinite_mark<DT>(mark, nrm[q], (double)a) : 0.0;
  }
  double r = pair_block_sum(part[0], part[1], sh);
  if (threadIdx.x == 0) partials[blockIdx.x] = r;
}

// K1 for a row-major source (src[i][k], the C-order numpy matrix uploaded
// as is): the block's 256 points are staged through shared memory 32
// dimensions at a time (coalesced reads of the rows, conflict-free column
// reads with a 33-element row pitch), then exactly the per-point arithmetic
// and block partials of ground_prepare_kernel -- results are bit-identical
// to the column-major path.
template <int DT, bool VS>
__global__ void __launch_bounds__(kRedThreads)
    ground_prepare_rows_kernel(const typename Traits<DT>::S *__restrict__ src,
                               int64_t n, int d, int d_pad,
                               const typename Traits<DT>::S *__restrict__ e0,
                               typename VtOf<DT, VS>::T *__restrict__ vt,
                               int64_t ld, double *__restrict__ norms,
                               typename Traits<DT>::C *__restrict__ aux,
                               double *__restrict__ partials, bool mark) {
  using S = typename Traits<DT>::S;
  using C = typename Traits<DT>::C;
  using V = typename VtOf<DT, VS>::T;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  C(*tile)[33] = reinterpret_cast<C(*)[33]>(smem_raw);  // [256][33]
  __shared__ double sh[32];
  const int64_t i0 = (int64_t)blockIdx.x * blockDim.x;
  const int64_t i = i0 + threadIdx.x;
  double nrm = 0.0, dst = 0.0;
  for (int k0 = 0; k0 < d_pad; k0 += 32) {
    __syncthreads();
    // 32 loads per thread, all issued before any shared-memory store
    // (memory-level parallelism; each warp reads one row segment per load)
    C xs[32];
#pragma unroll
    for (int u = 0; u < 32; ++u) {
      const int idx = threadIdx.x + u * kRedThreads;
      const int pp = idx >> 5, kk = idx & 31;
      const int64_t ip = i0 + pp;
      const int k = k0 + kk;
      xs[u] = (k < d && ip < n) ? to_c(src[ip * d + k]) : C(0);
    }
#pragma unroll
    for (int u = 0; u < 32; ++u) {
      const int idx = threadIdx.x + u * kRedThreads;
      tile[idx >> 5][idx & 31] = xs[u];
    }
    __syncthreads();
    if (i < ld) {
      for (int kk = 0; kk < 32 && k0 + kk < d_pad; ++kk) {
        const int k = k0 + kk;
        const C x = tile[threadIdx.x][kk];
        vt[(int64_t)k * ld + i] = to_vt<V>(x);
        if (k < d && i < n) {
          double xd = (double)x;
          nrm += xd * xd;
          double df = xd - (double)to_c(e0[k]);
          dst += df * df;
        }
      }
    }
  }
  if (i < ld) {
    C a = C(0);
    if (i < n) a = (DT == EXEM_BF16) ? (C)dst : to_c(from_d<S>(dst));
    if (i < n) {
      norms[i] = nrm;
      aux[i] = a;
    } else {
      norms[i] = 0.0;
      aux[i] = C(0);
    }
    dst = (i < n) ? nonfinite_mark<DT>(mark, nrm, (double)a) : 0.0;
  } else {
    dst = 0.0;
  }
  double r = block_sum<kRedThreads>(dst, sh);
  if (threadIdx.x == 0) partials[blockIdx.x] = r;
}

// TMA-fed K3-SIMT (exem_simt_tma.cu): 0 launched, 1 not applicable, < 0 a
// CUDA error
int gains_simt_tma(int dtype, const void *cvt, int64_t ldc,
                   const double *cnorms, int64_t l, const void *vt, int64_t ld,
                   const double *norms, const void *m, int64_t n, int d_pad,
                   int64_t split_pts, int64_t splits, double *partial,
                   cudaStream_t st);

// TMA-fed persistent K2 (exem_setmin.cu): 0 launched, 1 shape not covered,
// < 0 a CUDA error
int set_min_tma(int dtype, const void *vt, int64_t ld, int64_t n, int d_pad,
                const double *norms, const void *aux, const void *elems,
                const double *enorms, int k, int include_aux, void *t_out,
                int64_t *label_out, double *partials, void *dist_out,
                int64_t ldd, cudaStream_t st);
int set_min_storage_ok(int dtype, int64_t d, int64_t k, int has_t_out);

// ============================================================ K2 set_min
// min_distances / _set_value / assign_clusters over ONE explicit set
// (objective.py:113-141, evaluate.py:105-112, optimize.py:115-136).
//
// One pass over V for up to KG set elements (64 at f32, 32 at f64; larger
// sets take ceil(k / KG) passes): a CTA owns 256 points; V streams through a
// 4-stage cp.async ring in 8-dimension chunks ([8][256] values, 16-byte
// copies) together with the matching [8][KG] slice of the elements
// (transposed on the fly by 4/8-byte copies, zero-filled past k), and every
// thread keeps a 4-point x KG/4-element block of dot products in registers
// (register-blocked outer product: one 16-byte shared load of 4 points and
// KG/16 vector loads of elements per 4*KG/4 FMAs).  Per point the distances
// use the reference's per-precision form, the minimum keeps the lowest
// element index on ties (strict <, then the lowest index across the four
// element lanes), and the per-256-point block partial of sum_i t_i is the
// same fixed-order block_sum as every other K1/K2 kernel.  Each distance is
// the same sequential fma chain over the dimensions as before tiling.
//
// Algorithmic bytes: n * d * 4 (f32 vt) read once + the elements from L2.
constexpr int kLoadAhead = 8;  // independent V loads in flight (K2 update)
constexpr int kSmP = 256;      // points per CTA
constexpr int kSmBK = 8;       // dimensions per ring stage (= kDimPad)
constexpr int kSmStages = 4;

template <typename C> struct SmVec;
template <> struct SmVec<float> { using V = float4; };
template <> struct SmVec<double> { using V = double2; };

__device__ __forceinline__ void cp_async_small(void *smem, const void *gmem,
                                               int bytes, bool valid) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  const int src = valid ? bytes : 0;  // 0: zero fill
  if (bytes == 4)
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(s),
                 "l"(gmem), "r"(src));
  else
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s),
                 "l"(gmem), "r"(src));
}

template <int DT, int KG>
__global__ void __launch_bounds__(kRedThreads, DT == EXEM_F64 ? 1 : 2)
    set_min_kernel(const typename Traits<DT>::C *__restrict__ vt, int64_t ld,
                   int64_t n, int d_pad, const double *__restrict__ norms,
                   const typename Traits<DT>::C *__restrict__ aux,
                   const typename Traits<DT>::C *__restrict__ elems,
                   const double *__restrict__ enorms, int k, int include_aux,
                   typename Traits<DT>::C *__restrict__ t_out,
                   int64_t *__restrict__ label_out,
                   double *__restrict__ partials,
                   typename Traits<DT>::C *__restrict__ dist_out, int64_t ldd) {
  using C = typename Traits<DT>::C;
  using V4 = typename SmVec<C>::V;
  constexpr int EPT = KG / 4;                   // elements per thread
  constexpr int VPER = 16 / sizeof(C);          // values per 16-byte vector
  extern __shared__ __align__(16) unsigned char smem_raw[];
  C *sv = reinterpret_cast<C *>(smem_raw);                  // [ST][BK][P]
  C *se = sv + kSmStages * kSmBK * kSmP;                    // [ST][BK][KG]
  __shared__ double sh[32];
  __shared__ C st_t[kSmP];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int te = lane & 3;                      // element lane
  const int tp = warp * 8 + (lane >> 2);        // point quad 0..63
  const int64_t i0 = (int64_t)blockIdx.x * kSmP;
  const int nc = d_pad / kSmBK;
  C best[4];
  int64_t lab[4];
#pragma unroll
  for (int p = 0; p < 4; ++p) {
    best[p] = tinf<C>();
    lab[p] = 0;
  }
  for (int g0 = 0; g0 < k; g0 += KG) {
    auto load = [&](int stage, int chunk) {
      C *dv = sv + stage * kSmBK * kSmP;
      C *de = se + stage * kSmBK * KG;
      constexpr int VG = kSmBK * kSmP / VPER;  // 16-byte granules of V
      for (int x = threadIdx.x; x < VG; x += kRedThreads) {
        const int r = x / (kSmP / VPER), c = (x % (kSmP / VPER)) * VPER;
        cp_async16(dv + r * kSmP + c,
                   vt + (int64_t)(chunk * kSmBK + r) * ld + i0 + c);
      }
      for (int x = threadIdx.x; x < kSmBK * KG; x += kRedThreads) {
        const int r = x / KG, e = x % KG;
        const bool ok = g0 + e < k;
        cp_async_small(de + r * KG + e,
                       elems + (int64_t)(ok ? g0 + e : 0) * d_pad +
                           chunk * kSmBK + r,
                       (int)sizeof(C), ok);
      }
    };
    C acc[4][EPT];
#pragma unroll
    for (int p = 0; p < 4; ++p)
#pragma unroll
      for (int j = 0; j < EPT; ++j) acc[p][j] = C(0);
    __syncthreads();  // the previous group's ring is fully consumed
#pragma unroll
    for (int s = 0; s < kSmStages - 1; ++s) {
      if (s < nc) load(s, s);
      cp_async_commit();
    }
    for (int c = 0; c < nc; ++c) {
      cp_async_wait<kSmStages - 2>();
      __syncthreads();
      const int cn = c + kSmStages - 1;
      if (cn < nc) load(cn % kSmStages, cn);
      cp_async_commit();
      const C *cv = sv + (c % kSmStages) * kSmBK * kSmP + tp * 4;
      const C *ce = se + (c % kSmStages) * kSmBK * KG + te * EPT;
#pragma unroll
      for (int kk = 0; kk < kSmBK; ++kk) {
        C pv[4], ev[EPT];
        if constexpr (sizeof(C) == 4) {
          const float4 q = *reinterpret_cast<const float4 *>(cv + kk * kSmP);
          pv[0] = q.x; pv[1] = q.y; pv[2] = q.z; pv[3] = q.w;
        } else {
          const V4 q0 = *reinterpret_cast<const V4 *>(cv + kk * kSmP);
          const V4 q1 = *reinterpret_cast<const V4 *>(cv + kk * kSmP + 2);
          pv[0] = q0.x; pv[1] = q0.y; pv[2] = q1.x; pv[3] = q1.y;
        }
        if constexpr (EPT * sizeof(C) % 16 == 0) {
#pragma unroll
          for (int j = 0; j < EPT; j += VPER) {
            const V4 q = *reinterpret_cast<const V4 *>(ce + kk * KG + j);
            const C *qc = reinterpret_cast<const C *>(&q);
#pragma unroll
            for (int u = 0; u < VPER; ++u) ev[j + u] = qc[u];
          }
        } else {
#pragma unroll
          for (int j = 0; j < EPT; ++j) ev[j] = ce[kk * KG + j];
        }
#pragma unroll
        for (int p = 0; p < 4; ++p)
#pragma unroll
          for (int j = 0; j < EPT; ++j) {
            if (Traits<DT>::kDirect) {
              const C df = pv[p] - ev[j];
              acc[p][j] = fma(df, df, acc[p][j]);
            } else {
              acc[p][j] = fma(pv[p], ev[j], acc[p][j]);
            }
          }
      }
    }
    cp_async_wait<0>();
    // epilogue of the group: distances, running first minimum per point
#pragma unroll
    for (int p = 0; p < 4; ++p) {
      const int64_t i = i0 + tp * 4 + p;
      const C ai = i < n ? (C)norms[i] : C(0);
#pragma unroll
      for (int j = 0; j < EPT; ++j) {
        const int e = g0 + te * EPT + j;
        if (e < k && i < n) {
          const C dist = Traits<DT>::kDirect
                             ? acc[p][j]
                             : gemm_form<C>(acc[p][j], ai, (C)enorms[e]);
          if (dist_out) dist_out[(int64_t)e * ldd + i] = dist;
          if (dist < best[p]) {  // strict: lowest element index wins ties
            best[p] = dist;
            lab[p] = e;
          }
        }
      }
    }
  }
  // first minimum across the four element lanes (lower index on ties)
#pragma unroll
  for (int p = 0; p < 4; ++p) {
#pragma unroll
    for (int o = 1; o < 4; o <<= 1) {
      const C ob = __shfl_xor_sync(0xffffffffu, best[p], o);
      const long long ol = __shfl_xor_sync(0xffffffffu, (long long)lab[p], o);
      if (ob < best[p] || (ob == best[p] && ol < lab[p])) {
        best[p] = ob;
        lab[p] = ol;
      }
    }
    const int64_t i = i0 + tp * 4 + p;
    C t = best[p];
    if (include_aux && i < n) t = tmin(t, aux[i]);
    if (te == 0) {
      st_t[tp * 4 + p] = t;
      if (i < n) {
        if (t_out) t_out[i] = t;
        if (label_out) label_out[i] = lab[p];
      }
    }
  }
  __syncthreads();
  const int64_t i = i0 + threadIdx.x;
  double r = block_sum<kRedThreads>(i < n ? (double)st_t[threadIdx.x] : 0.0,
                                    sh);
  if (threadIdx.x == 0) partials[blockIdx.x] = r;
}

template <int DT, int KG>
static cudaError_t launch_set_min_kg(
    int64_t blocks, cudaStream_t st, const typename Traits<DT>::C *vt,
    int64_t ld, int64_t n, int d_pad, const double *norms,
    const typename Traits<DT>::C *aux, const typename Traits<DT>::C *elems,
    const double *enorms, int k, int include_aux,
    typename Traits<DT>::C *t_out, int64_t *label_out, double *partials,
    typename Traits<DT>::C *dist_out, int64_t ldd) {
  using C = typename Traits<DT>::C;
  const size_t smem = (size_t)kSmStages * kSmBK * (kSmP + KG) * sizeof(C);
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(
        set_min_kernel<DT, KG>, cudaFuncAttributeMaxDynamicSharedMemorySize,
        (int)smem);
    if (e != cudaSuccess) return e;
  }
  set_min_kernel<DT, KG><<<(unsigned)blocks, kRedThreads, smem, st>>>(
      vt, ld, n, d_pad, norms, aux, elems, enorms, k, include_aux, t_out,
      label_out, partials, dist_out, ldd);
  return cudaGetLastError();
}

// Element group KG = the smallest of 8, 16, 32, 64 (32 at f64) covering k:
// small sets compute few dead dot products; the per-element arithmetic is
// the same for every KG, so the distances are identical.
template <int DT>
static cudaError_t launch_set_min(
    int64_t blocks, cudaStream_t st, const typename Traits<DT>::C *vt,
    int64_t ld, int64_t n, int d, const double *norms,
    const typename Traits<DT>::C *aux, const typename Traits<DT>::C *elems,
    int d_pad, const double *enorms, int k, int include_aux,
    typename Traits<DT>::C *t_out, int64_t *label_out, double *partials,
    typename Traits<DT>::C *dist_out = nullptr, int64_t ldd = 0) {
  (void)d;
  if (ld % kSmP != 0 || d_pad % kSmBK != 0) return cudaErrorInvalidValue;
  // the TMA-fed persistent K2 (exem_setmin.cu) whenever the element group is
  // resident in shared memory; this cp.async kernel otherwise
  const int tma = set_min_tma(DT, vt, ld, n, d_pad, norms, aux, elems, enorms,
                              k, include_aux, t_out, label_out, partials,
                              dist_out, ldd, st);
  if (tma == 0) return cudaSuccess;
  if (tma < 0) return (cudaError_t)(-tma);
#define EXEM_SM(KGN)                                                        \
  return launch_set_min_kg<DT, KGN>(blocks, st, vt, ld, n, d_pad, norms,    \
                                    aux, elems, enorms, k, include_aux,     \
                                    t_out, label_out, partials, dist_out,   \
                                    ldd)
  if constexpr (DT != EXEM_F64) {
    if (k > 32) EXEM_SM(64);
  }
  if (k > 16) EXEM_SM(32);
  if (k > 8) EXEM_SM(16);
  EXEM_SM(8);
#undef EXEM_SM
}

// ============================================================ greedy m init
template <typename C>
__global__ void __launch_bounds__(kRedThreads)
    greedy_init_kernel(const C *__restrict__ aux, int64_t n, C *__restrict__ m,
                       double *__restrict__ partials) {
  __shared__ double sh[32];
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  double v = 0.0;
  if (i < n) {
    m[i] = aux[i];
    v = (double)aux[i];
  }
  double r = block_sum<kRedThreads>(v, sh);
  if (threadIdx.x == 0) partials[blockIdx.x] = r;
}

// ============================================================ sieve kernels
// Streaming (Sieve) optimizers keep one m-vector per sieve: M[s][i] =
// min(aux_i, min_{e in S_s} d(v_i, e)).  For an arriving element with
// distances dist[i] = d(v_i, e):
//   sieve_gains:  partial[s][b] = sum_{i in block b} max(0, M[s][i] - dist[i])
//   sieve_update: M[s][i] <- min(M[s][i], dist[i]); partial[b] = block sum
// (fixed-order block partials, reduced by exem_reduce_partials /
// exem_sum_fixed -> deterministic).
template <typename C>
__global__ void __launch_bounds__(kRedThreads)
    sieve_gains_kernel(const C *__restrict__ M, int64_t ldm,
                       const C *__restrict__ dist, int64_t n,
                       double *__restrict__ partial, int64_t nblocks) {
  __shared__ double sh[32];
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t s = blockIdx.y;
  double v = 0.0;
  if (i < n) v = (double)tmax(M[s * ldm + i] - dist[i], C(0));
  const double r = block_sum<kRedThreads>(v, sh);
  if (threadIdx.x == 0) partial[blockIdx.x * gridDim.y + s] = r;
}

template <typename C>
__global__ void __launch_bounds__(kRedThreads)
    sieve_update_kernel(C *__restrict__ m, const C *__restrict__ dist,
                        int64_t n, double *__restrict__ partials) {
  __shared__ double sh[32];
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  double v = 0.0;
  if (i < n) {
    const C mi = tmin(m[i], dist[i]);
    m[i] = mi;
    v = (double)mi;
  }
  const double r = block_sum<kRedThreads>(v, sh);
  if (threadIdx.x == 0) partials[blockIdx.x] = r;
}

// ============================================================ K2 greedy update
// m_i <- min(m_i, d(v_i, c*)), c* read from sel_idx[step] on device.
// Optionally refreshes the TC point operand's folded -h columns.
template <int DT, bool VS>
__global__ void __launch_bounds__(kRedThreads)
    greedy_update_kernel(const typename VtOf<DT, VS>::T *__restrict__ vt,
                         int64_t ld, int64_t n, int d,
                         const double *__restrict__ norms,
                         const typename VtOf<DT, VS>::T *__restrict__ cvt,
                         int64_t ldc, const double *__restrict__ cnorms,
                         const int64_t *__restrict__ sel_idx, int64_t step,
                         typename Traits<DT>::C *__restrict__ m,
                         typename Traits<DT>::S *__restrict__ xp, int64_t kp,
                         double *__restrict__ partials) {
  using C = typename Traits<DT>::C;
  using S = typename Traits<DT>::S;
  __shared__ double sh[32];
  const int64_t c = sel_idx[step];
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  double v = 0.0;
  if (i < n && c < 0) {  // K5 found no valid candidate: S unchanged
    v = (double)m[i];
  } else if (i < n) {
    C acc = C(0);
    int kk = 0;
    // loads ahead (MLP; 16 of 2-byte storage: the same bytes in flight)
    constexpr int LA = VS ? 2 * kLoadAhead : kLoadAhead;
    for (; kk + LA <= d; kk += LA) {
      C xs[LA];
#pragma unroll
      for (int u = 0; u < LA; ++u)
        xs[u] = to_c(vt[(int64_t)(kk + u) * ld + i]);
#pragma unroll
      for (int u = 0; u < LA; ++u) {
        const C y = to_c(cvt[(int64_t)(kk + u) * ldc + c]);
        if (Traits<DT>::kDirect) {
          const C df = xs[u] - y;
          acc = fma(df, df, acc);
        } else {
          acc = fma(xs[u], y, acc);
        }
      }
    }
    for (; kk < d; ++kk) {
      const C x = to_c(vt[(int64_t)kk * ld + i]);
      const C y = to_c(cvt[(int64_t)kk * ldc + c]);
      if (Traits<DT>::kDirect) {
        const C df = x - y;
        acc = fma(df, df, acc);
      } else {
        acc = fma(x, y, acc);
      }
    }
    C dist = Traits<DT>::kDirect
                 ? acc
                 : gemm_form<C>(acc, (C)norms[i], (C)cnorms[c]);
    C mi = tmin(m[i], dist);
    m[i] = mi;
    v = (double)mi;
    if (xp != nullptr) {
      // h_i = (||v_i||^2 - m_i)/2 split into three half pieces (~24 bits).
      double h[3];
      fold_pieces<S>(0.5 * (norms[i] - (double)mi), h);
      S *row = xp + i * kp + d;
      row[0] = from_d<S>(-h[0]);
      row[1] = from_d<S>(-h[1]);
      row[2] = from_d<S>(-h[2]);
    }
  }
  double r = block_sum<kRedThreads>(v, sh);
  if (threadIdx.x == 0) partials[blockIdx.x] = r;
}

// K1 for a row-major source whose 256-row slab fits in shared memory
// (2- and 4-byte storage): the block's rows are one contiguous run of
// 256*d values, copied with 16-byte loads (full 128-byte lines, every byte
// read once) into rows of odd word pitch (conflict-free column reads), then
// the per-point arithmetic and block partials of ground_prepare_kernel --
// bit-identical.  (The 32-dimension tiles of ground_prepare_rows_kernel read
// each row in 64/128-byte pieces that straddle sectors: 0.21-0.48 of HBM.)
constexpr int kSlabMaxBytes = 112 * 1024;  // two CTAs per SM
template <typename S> __host__ __device__ constexpr int slab_pitch(int d) {
  // elements per smem row: an odd number of 4-byte words
  return sizeof(S) == 4 ? (d | 1) : ((((d + 1) / 2) | 1) * 2);
}

template <int DT, bool VS>
__global__ void __launch_bounds__(kRedThreads)
    ground_prepare_slab_kernel(const typename Traits<DT>::S *__restrict__ src,
                               int64_t n, int d, int d_pad,
                               const typename Traits<DT>::S *__restrict__ e0,
                               typename VtOf<DT, VS>::T *__restrict__ vt,
                               int64_t ld, double *__restrict__ norms,
                               typename Traits<DT>::C *__restrict__ aux,
                               double *__restrict__ partials, bool mark) {
  using S = typename Traits<DT>::S;
  using C = typename Traits<DT>::C;
  using V = typename VtOf<DT, VS>::T;
  constexpr int per = 16 / (int)sizeof(S);  // values per 16-byte load
  extern __shared__ __align__(16) unsigned char smem_raw[];
  S *slab = reinterpret_cast<S *>(smem_raw);  // [256][P]
  __shared__ double sh[32];
  const int P = slab_pitch<S>(d);
  const int64_t i0 = (int64_t)blockIdx.x * kRedThreads;
  const int rows = (int)min((int64_t)kRedThreads, n - i0);  // >= 1 (ld < n + 256)
  const int64_t total = (int64_t)rows * d;  // values of the slab
  const S *g = src + i0 * d;                // 16-byte aligned (256*d*sizeof(S))
  const int64_t nv = total / per;
  // running (row, col) of value idx*per, advanced by 256*per per iteration
  const int step = kRedThreads * per;
  int r = (int)(((int64_t)threadIdx.x * per) / d);
  int c = (int)(((int64_t)threadIdx.x * per) - (int64_t)r * d);
  const int dq = step / d, dr = step - dq * d;
  // kU independent 16-byte loads in flight per thread, then their scatter
  constexpr int kU = 8;
  auto scatter = [&](const uint4 &q) {
    const S *qs = reinterpret_cast<const S *>(&q);
    int rr = r, cc = c;
#pragma unroll
    for (int j = 0; j < per; ++j) {
      slab[rr * P + cc] = qs[j];
      if (++cc == d) {
        cc = 0;
        ++rr;
      }
    }
    r += dq;
    c += dr;
    if (c >= d) {
      c -= d;
      ++r;
    }
  };
  int64_t idx = threadIdx.x;
  for (; idx + (kU - 1) * kRedThreads < nv; idx += kU * kRedThreads) {
    uint4 q[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u)
      q[u] = __ldg(reinterpret_cast<const uint4 *>(g) + idx + u * kRedThreads);
#pragma unroll
    for (int u = 0; u < kU; ++u) scatter(q[u]);
  }
  for (; idx < nv; idx += kRedThreads)
    scatter(__ldg(reinterpret_cast<const uint4 *>(g) + idx));
  for (int64_t e = nv * per + threadIdx.x; e < total; e += kRedThreads) {
    const int rr = (int)(e / d);
    slab[rr * P + (int)(e - (int64_t)rr * d)] = g[e];
  }
  __syncthreads();
  const int64_t i = i0 + threadIdx.x;
  const bool live = threadIdx.x < rows;
  double nrm = 0.0, dst = 0.0;
  const S *row = slab + threadIdx.x * P;
  for (int k = 0; k < d_pad; ++k) {
    C x = C(0);
    if (k < d && live) x = to_c(row[k]);
    vt[(int64_t)k * ld + i] = to_vt<V>(x);
    if (k < d && live) {
      const double xd = (double)x;
      nrm += xd * xd;
      const double df = xd - (double)to_c(e0[k]);
      dst += df * df;
    }
  }
  C a = C(0);
  if (live) a = (DT == EXEM_BF16) ? (C)dst : to_c(from_d<S>(dst));
  norms[i] = live ? nrm : 0.0;
  aux[i] = a;
  dst = live ? nonfinite_mark<DT>(mark, nrm, (double)a) : 0.0;
  double rs = block_sum<kRedThreads>(dst, sh);
  if (threadIdx.x == 0) partials[blockIdx.x] = rs;
}

// 0 launched, 1 not applicable (8-byte values, or the slab does not fit),
// < 0 a CUDA error
template <int DT, bool VS>
static int launch_prepare_slab(int64_t blocks, cudaStream_t st,
                               const void *src, int64_t n, int d, int d_pad,
                               const void *e0, void *vt, int64_t ld,
                               double *norms, void *aux, double *scratch,
                               bool mark) {
  using S = typename Traits<DT>::S;
  if constexpr (sizeof(S) <= 4) {
    using C = typename Traits<DT>::C;
    using V = typename VtOf<DT, VS>::T;
    const size_t slab = (size_t)kRedThreads * slab_pitch<S>(d) * sizeof(S);
    if (slab > (size_t)kSlabMaxBytes || !aligned(src, 16) ||
        getenv("EXEM_K1_TILES"))
      return 1;
    cudaError_t e = cudaFuncSetAttribute(
        ground_prepare_slab_kernel<DT, VS>,
        cudaFuncAttributeMaxDynamicSharedMemorySize, (int)slab);
    if (e != cudaSuccess) return -(int)e;
    ground_prepare_slab_kernel<DT, VS><<<(unsigned)blocks, kRedThreads, slab,
                                         st>>>(
        (const S *)src, n, d, d_pad, (const S *)e0, (V *)vt, ld, norms,
        (C *)aux, scratch, mark);
    return 0;
  }
  return 1;
}

// The m-update on 2-byte storage vt (EXEM_VT_STORAGE): two adjacent points
// per thread (4-byte pair loads, 128 threads per 256 points), the same
// per-point direct-form fma chain and xp refresh as greedy_update_kernel,
// block partials by pair_block_sum (bit-identical).
template <int DT>
__global__ void __launch_bounds__(128)
    greedy_update_pair_kernel(const typename Traits<DT>::S *__restrict__ vt,
                              int64_t ld, int64_t n, int d,
                              const double *__restrict__ norms,
                              const typename Traits<DT>::S *__restrict__ cvt,
                              int64_t ldc, const int64_t *__restrict__ sel_idx,
                              int64_t step, float *__restrict__ m,
                              typename Traits<DT>::S *__restrict__ xp,
                              int64_t kp, double *__restrict__ partials) {
  using S = typename Traits<DT>::S;
  __shared__ double sh[8];
  const int64_t c = sel_idx[step];
  const int64_t i = (int64_t)blockIdx.x * 256 + 2 * threadIdx.x;
  double v[2] = {0.0, 0.0};
  if (i < n) {
    const float2 m2 = *reinterpret_cast<const float2 *>(m + i);
    float mi[2] = {m2.x, m2.y};
    if (c >= 0) {  // c < 0: K5 found no valid candidate, S unchanged
      float acc[2] = {0.f, 0.f};
      auto step_k = [&](uint32_t raw, int k) {
        const S *h = reinterpret_cast<const S *>(&raw);
        const float y = to_c(cvt[(int64_t)k * ldc + c]);
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          const float df = to_c(h[q]) - y;
          acc[q] = fmaf(df, df, acc[q]);
        }
      };
      constexpr int LA = 16;
      int kk = 0;
      for (; kk + LA <= d; kk += LA) {
        uint32_t xs[LA];
#pragma unroll
        for (int u = 0; u < LA; ++u)
          xs[u] = *reinterpret_cast<const uint32_t *>(vt + (int64_t)(kk + u) * ld + i);
#pragma unroll
        for (int u = 0; u < LA; ++u) step_k(xs[u], kk + u);
      }
      for (; kk < d; ++kk)
        step_k(*reinterpret_cast<const uint32_t *>(vt + (int64_t)kk * ld + i), kk);
#pragma unroll
      for (int q = 0; q < 2; ++q) mi[q] = tmin(mi[q], acc[q]);
      const bool two = i + 1 < n;
      if (two) {
        *reinterpret_cast<float2 *>(m + i) = make_float2(mi[0], mi[1]);
      } else {
        m[i] = mi[0];
      }
      if (xp != nullptr) {
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          if (q == 1 && !two) break;
          double h[3];
          fold_pieces<S>(0.5 * (norms[i + q] - (double)mi[q]), h);
          S *row = xp + (i + q) * kp + d;
          row[0] = from_d<S>(-h[0]);
          row[1] = from_d<S>(-h[1]);
          row[2] = from_d<S>(-h[2]);
        }
      }
    }
    v[0] = (double)mi[0];
    v[1] = i + 1 < n ? (double)mi[1] : 0.0;
  }
  double r = pair_block_sum(v[0], v[1], sh);
  if (threadIdx.x == 0) partials[blockIdx.x] = r;
}

// launchers of the pair kernels (half tags only; false for f32/f64)
template <int DT>
static bool launch_prepare_pair(int64_t blocks, cudaStream_t st,
                                const void *src, int64_t n, int d, int d_pad,
                                const void *e0, void *vt, int64_t ld,
                                double *norms, void *aux, double *scratch,
                                bool mark) {
  if constexpr (DT == EXEM_F16 || DT == EXEM_BF16) {
    using S = typename Traits<DT>::S;
    using C = typename Traits<DT>::C;
    ground_prepare_pair_kernel<DT><<<(unsigned)blocks, 128, 0, st>>>(
        (const S *)src, n, d, d_pad, (const S *)e0, (S *)vt, ld, norms,
        (C *)aux, scratch, mark);
    return true;
  }
  return false;
}

template <int DT>
static bool launch_update_pair(int64_t blocks, cudaStream_t st, const void *vt,
                               int64_t ld, int64_t n, int d,
                               const double *norms, const void *cvt,
                               int64_t ldc, const int64_t *sel_idx,
                               int64_t step, void *m, void *xp, int64_t kp,
                               double *scratch) {
  if constexpr (DT == EXEM_F16 || DT == EXEM_BF16) {
    using S = typename Traits<DT>::S;
    greedy_update_pair_kernel<DT><<<(unsigned)blocks, 128, 0, st>>>(
        (const S *)vt, ld, n, d, norms, (const S *)cvt, ldc, sel_idx, step,
        (float *)m, (S *)xp, kp, scratch);
    return true;
  }
  return false;
}

// ============================================================ K3 / K4 SIMT
// Register-blocked outer product: CTA tile 128 rows (candidates / sets) x
// 128 points, 256 threads, 8x8 per thread, k-chunks of 8 double-buffered
// with cp.async.  Row r of the thread tile maps to tile row
// (r<4 ? ty*4+r : 64+ty*4+r-4); same for columns with tx.
constexpr int kBM = 128, kBN = 128, kBK = 8, kThreads = 256;

constexpr int kSimtStages = 3;  // cp.async ring: one barrier per k-chunk

template <typename T, int BK = kBK>
struct SimtSmem {
  T a[kSimtStages][BK][kBM];
  T b[kSimtStages][BK][kBN];
};

template <typename T, int BK = kBK>
__device__ __forceinline__ void load_chunk(T (*dst)[kBM], const T *src,
                                           int64_t ldsrc, int64_t col0,
                                           int k0) {
  constexpr int kVec = 16 / sizeof(T);            // elements per 16B
  constexpr int kPerRow = kBM / kVec;             // 16B packets per row
  constexpr int kTotal = BK * kPerRow;            // packets per chunk
#pragma unroll
  for (int p = threadIdx.x; p < kTotal; p += kThreads) {
    const int row = p / kPerRow, col = (p % kPerRow) * kVec;
    cp_async16(&dst[row][col], src + (int64_t)(k0 + row) * ldsrc + col0 + col);
  }
}

// kFull = false: only the first kn dimensions of the chunk are live (the
// last chunk when d is not a multiple of BK: its zero padding dimensions
// would only add exact zeros, so skipping them changes no result)
template <typename T, bool kDirect, int BK = kBK, bool kFull = true>
__device__ __forceinline__ void mma_chunk(const SimtSmem<T, BK> &sm, int buf,
                                          int tx, int ty, T (&acc)[8][8],
                                          int kn = BK) {
#pragma unroll
  for (int kk = 0; kk < BK; ++kk) {
    if constexpr (!kFull) {
      if (kk >= kn) break;
    }
    T a[8], b[8];
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      a[r] = sm.a[buf][kk][ty * 4 + r];
      a[4 + r] = sm.a[buf][kk][64 + ty * 4 + r];
      b[r] = sm.b[buf][kk][tx * 4 + r];
      b[4 + r] = sm.b[buf][kk][64 + tx * 4 + r];
    }
#ifndef EXEM_SIMT_NO_FFMA2
    // binary32: paired FFMA2 (/ FADD2) with a[r] as the broadcast operand --
    // per lane the same IEEE fma (sub) as the scalar loop, so results are
    // bit-identical, at half the issue slots (C2 39.5 -> 35.7 ms per step,
    // profiles/r02_ffma2_ab.log)
    constexpr bool kPaired = sizeof(T) == 4;
#else
    constexpr bool kPaired = false;
#endif
    if constexpr (kPaired) {
#pragma unroll
      for (int r = 0; r < 8; ++r) {
        const float2 ar = make_float2(a[r], a[r]);
#pragma unroll
        for (int c = 0; c < 8; c += 2) {
          float2 t = make_float2(acc[r][c], acc[r][c + 1]);
          if constexpr (kDirect) {
            const float2 df = __fadd2_rn(ar, make_float2(-b[c], -b[c + 1]));
            t = __ffma2_rn(df, df, t);
          } else {
            t = __ffma2_rn(ar, make_float2(b[c], b[c + 1]), t);
          }
          acc[r][c] = t.x;
          acc[r][c + 1] = t.y;
        }
      }
    } else {
#pragma unroll
      for (int r = 0; r < 8; ++r)
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          if (kDirect) {
            const T df = a[r] - b[c];
            acc[r][c] = fma(df, df, acc[r][c]);
          } else {
            acc[r][c] = fma(a[r], b[c], acc[r][c]);
          }
        }
    }
  }
}

// Full-k mainloop for one (row tile, point tile) pair.  kTail: d is not a
// multiple of BK and the last chunk runs only its live dimensions (a
// separate instantiation, so the d % BK == 0 kernels keep the plain loop).
template <typename T, bool kDirect, int BK = kBK, bool kTail = false>
__device__ __forceinline__ void simt_mainloop(SimtSmem<T, BK> &sm, const T *arow,
                                              int64_t lda, int64_t a0,
                                              const T *bpts, int64_t ldb,
                                              int64_t b0, int d_pad, int d,
                                              int tx, int ty,
                                              T (&acc)[8][8]) {
  // Three-buffer cp.async ring: chunk c lives in buffer c % 3 and cp.async
  // group c.  Each iteration waits for its chunk, then ONE barrier both
  // publishes it and proves every thread has finished chunk c-1, whose
  // buffer the load of chunk c+2 then overwrites.
  const int nk = d_pad / BK;
  const int tail = d - (nk - 1) * BK;  // live dimensions of the last chunk
  __syncthreads();  // previous consumers of the ring are done
  load_chunk<T, BK>(sm.a[0], arow, lda, a0, 0);
  load_chunk<T, BK>(sm.b[0], bpts, ldb, b0, 0);
  cp_async_commit();
  if (nk > 1) {
    load_chunk<T, BK>(sm.a[1], arow, lda, a0, BK);
    load_chunk<T, BK>(sm.b[1], bpts, ldb, b0, BK);
  }
  cp_async_commit();
  int buf = 0;
  // kTail: the last chunk is peeled and runs only its live dimensions (the
  // steady-state loop body stays the plain full-chunk code): d = 2
  // 4.40 -> 3.16 ms, d = 100 35.7 -> 35.3 ms per C3 step
  const int nfull = (kTail && tail < BK) ? nk - 1 : nk;
  for (int c = 0; c < nfull; ++c) {
    cp_async_wait<1>();
    __syncthreads();
    if (c + 2 < nk) {
      const int nb = buf == 0 ? 2 : buf - 1;  // (c + 2) % 3
      load_chunk<T, BK>(sm.a[nb], arow, lda, a0, (c + 2) * BK);
      load_chunk<T, BK>(sm.b[nb], bpts, ldb, b0, (c + 2) * BK);
    }
    cp_async_commit();  // (possibly empty: keeps group c+2 = chunk c+2)
    mma_chunk<T, kDirect, BK>(sm, buf, tx, ty, acc);
    buf = buf == 2 ? 0 : buf + 1;
  }
  if constexpr (kTail) {
    if (nfull < nk) {
      cp_async_wait<1>();
      __syncthreads();
      cp_async_commit();
      mma_chunk<T, kDirect, BK, false>(sm, buf, tx, ty, acc, tail);
    }
  }
}

__device__ __forceinline__ int tile_off(int t4, int r) {
  return r < 4 ? t4 * 4 + r : 64 + t4 * 4 + (r - 4);
}

// K3: partial[s][c] = sum_{i in split s} max(0, c.v_i - h_i - b'_c),
//     h_i = (a_i - m_i)/2, b'_c = ||c||^2/2  => 2*that = sum max(0, m_i - d).
// The per-tile constants live in shared memory to keep the 8x8 register
// tile spill-free at 2 CTAs/SM.
template <typename T, int kMinBlocks, int BK = kBK, bool kTail = false>
__global__ void __launch_bounds__(kThreads, kMinBlocks)
    gains_simt_kernel(const T *__restrict__ cvt, int64_t ldc,
                      const double *__restrict__ cnorms, int64_t l,
                      const T *__restrict__ vt, int64_t ld,
                      const double *__restrict__ norms,
                      const T *__restrict__ m, int64_t n, int d_pad, int d,
                      int64_t split_pts, double *__restrict__ partial) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  SimtSmem<T, BK> &sm = *reinterpret_cast<SimtSmem<T, BK> *>(smem_raw);
  __shared__ T s_b[kBM];
  __shared__ T s_h[kBN];
  const int tid = threadIdx.x;
  const int tx = tid % 16, ty = tid / 16;
  const int64_t c0 = (int64_t)blockIdx.x * kBM;
  const int64_t split = blockIdx.y;
  const int64_t p_begin = split * split_pts;
  const int64_t p_end = min(n, p_begin + split_pts);

  if (tid < kBM) s_b[tid] = (c0 + tid < l) ? (T)(0.5 * cnorms[c0 + tid]) : T(0);
  double g[8];
#pragma unroll
  for (int r = 0; r < 8; ++r) g[r] = 0.0;

  for (int64_t p0 = p_begin; p0 < p_end; p0 += kBN) {
    __syncthreads();
    if (tid < kBN) {
      const int64_t pi = p0 + tid;
      s_h[tid] = pi < p_end ? (T)(0.5 * (norms[pi] - (double)m[pi])) : tinf<T>();
    }
    __syncthreads();
    T acc[8][8];
#pragma unroll
    for (int r = 0; r < 8; ++r)
#pragma unroll
      for (int c = 0; c < 8; ++c)
        acc[r][c] = -(s_h[tile_off(tx, c)] + s_b[tile_off(ty, r)]);
    simt_mainloop<T, false, BK, kTail>(sm, cvt, ldc, c0, vt, ld, p0, d_pad, d,
                                       tx, ty, acc);
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      T s = T(0);
#pragma unroll
      for (int c = 0; c < 8; ++c) s += tmax(acc[r][c], T(0));
      g[r] += (double)s;
    }
  }
#pragma unroll
  for (int r = 0; r < 8; ++r) {
    double v = g[r];
#pragma unroll
    for (int o = 8; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    const int64_t ci = c0 + tile_off(ty, r);
    if (tx == 0 && ci < l) partial[split * l + ci] = v;
  }
}

// K4: partial[s][j] = sum_{i in split s} min(aux_i, min_{e<card_j} d(v_i, S_j[e]))
// The running per-(set, point) minima live in shared memory (64 per thread,
// thread-interleaved so the accesses are conflict-free); the GEMM-form
// distances of element e come from the same register-blocked mainloop as K3.
template <typename T>
struct BatchSmem {
  SimtSmem<T> mm;
  T best[64][kThreads];
  T pa[kBN];   // point norms of the tile (compute type)
  T px[kBN];   // point aux distances of the tile
};

template <int DT, bool kTail = false>
__global__ void __launch_bounds__(kThreads, (DT == EXEM_F64 ? 1 : 2))
    batch_eval_kernel(const typename Traits<DT>::C *__restrict__ vt,
                      int64_t ld, int64_t n, int d_pad, int d,
                      const double *__restrict__ norms,
                      const typename Traits<DT>::C *__restrict__ aux,
                      const typename Traits<DT>::C *__restrict__ packed,
                      const double *__restrict__ pnorms,
                      const int32_t *__restrict__ card, int64_t l,
                      int64_t l_pad, int k_max, int64_t split_pts,
                      double *__restrict__ partial) {
  using T = typename Traits<DT>::C;
  constexpr bool kDirect = Traits<DT>::kDirect;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  BatchSmem<T> &sm = *reinterpret_cast<BatchSmem<T> *>(smem_raw);
  __shared__ int s_kmax;
  __shared__ int s_card[kBM];
  const int tid = threadIdx.x;
  const int tx = tid % 16, ty = tid / 16;
  const int64_t j0 = (int64_t)blockIdx.x * kBM;
  const int64_t split = blockIdx.y;
  const int64_t p_begin = split * split_pts;
  const int64_t p_end = min(n, p_begin + split_pts);
  const int64_t ldp = (int64_t)k_max * l_pad;  // stride between dimensions

  if (tid == 0) s_kmax = 0;
  __syncthreads();
  if (tid < kBM) {
    const int cj = (j0 + tid < l) ? card[j0 + tid] : 0;
    s_card[tid] = cj;
    atomicMax(&s_kmax, cj);
  }
  __syncthreads();
  const int kt = s_kmax;  // largest cardinality in this set tile

  double g[8];
#pragma unroll
  for (int r = 0; r < 8; ++r) g[r] = 0.0;

  for (int64_t p0 = p_begin; p0 < p_end; p0 += kBN) {
    __syncthreads();
    if (tid < kBN) {
      const int64_t pi = p0 + tid;
      sm.pa[tid] = pi < p_end ? (T)norms[pi] : T(0);
      sm.px[tid] = pi < p_end ? aux[pi] : T(0);
    }
#pragma unroll
    for (int q = 0; q < 64; ++q) sm.best[q][tid] = tinf<T>();
    for (int e = 0; e < kt; ++e) {
      T acc[8][8];
#pragma unroll
      for (int r = 0; r < 8; ++r)
#pragma unroll
        for (int c = 0; c < 8; ++c) acc[r][c] = T(0);
      // element e of sets j0..j0+127 at dim k: packed[k*ldp + e*l_pad + j]
      simt_mainloop<T, kDirect, kBK, kTail>(sm.mm,
                                            packed + (int64_t)e * l_pad, ldp,
                                            j0, vt, ld, p0, d_pad, d, tx, ty,
                                            acc);
#pragma unroll
      for (int r = 0; r < 8; ++r) {
        const int jr = tile_off(ty, r);
        if (e < s_card[jr]) {  // blank slots (e >= card) never contribute
          T be = T(0);
          if (!kDirect) be = (T)pnorms[(int64_t)e * l_pad + j0 + jr];
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            T dist = kDirect ? acc[r][c]
                             : gemm_form<T>(acc[r][c], sm.pa[tile_off(tx, c)], be);
            sm.best[r * 8 + c][tid] = tmin(sm.best[r * 8 + c][tid], dist);
          }
        }
      }
    }
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      T s = T(0);
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        const int pc = tile_off(tx, c);
        if (p0 + pc < p_end) s += tmin(sm.best[r * 8 + c][tid], sm.px[pc]);
      }
      g[r] += (double)s;
    }
  }
#pragma unroll
  for (int r = 0; r < 8; ++r) {
    double v = g[r];
#pragma unroll
    for (int o = 8; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    const int64_t j = j0 + tile_off(ty, r);
    if (tx == 0 && j < l) partial[split * l + j] = v;
  }
}

// ============================================================ K6 reduce
__global__ void reduce_partials_kernel(const double *__restrict__ partial,
                                       int64_t splits, int64_t l,
                                       double scale, double *__restrict__ out) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= l) return;
  double s = 0.0;
  for (int64_t q = 0; q < splits; ++q) s += partial[q * l + j];
  out[j] = scale * s;
}

// ============================================================ K5 argmax
struct Best {
  double v;
  int64_t i;
};
__device__ __forceinline__ Best better(Best a, Best b) {
  // larger value wins; equal values -> lower index (np.argmax, optimize.py:73)
  if (b.v > a.v || (b.v == a.v && b.i < a.i)) return b;
  return a;
}
__device__ __forceinline__ Best warp_best(Best x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    Best y;
    y.v = __shfl_xor_sync(0xffffffffu, x.v, o);
    y.i = __shfl_xor_sync(0xffffffffu, x.i, o);
    x = better(x, y);
  }
  return x;
}
constexpr int kArgThreads = 1024;
__device__ __forceinline__ Best block_best(Best x) {
  __shared__ double sv[32];
  __shared__ long long si[32];
  x = warp_best(x);
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) {
    sv[w] = x.v;
    si[w] = x.i;
  }
  __syncthreads();
  Best r{-tinf<double>(), INT64_MAX};
  if (w == 0) {
    if (lane < (int)(blockDim.x >> 5)) r = Best{sv[lane], (int64_t)si[lane]};
    r = warp_best(r);
  }
  return r;
}

__global__ void __launch_bounds__(kArgThreads)
    argmax_partial_kernel(const double *__restrict__ g, int64_t l,
                          const uint8_t *__restrict__ selected,
                          double *__restrict__ scratch) {
  Best x{-tinf<double>(), INT64_MAX};
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < l;
       j += (int64_t)gridDim.x * blockDim.x) {
    double v = g[j];
    if (!selected[j] && !(v != v)) x = better(x, Best{v, j});
  }
  x = block_best(x);
  if (threadIdx.x == 0) {
    scratch[2 * blockIdx.x] = x.v;
    scratch[2 * blockIdx.x + 1] = __longlong_as_double((long long)x.i);
  }
}

__global__ void __launch_bounds__(kArgThreads)
    argmax_final_kernel(const double *__restrict__ scratch, int nblocks,
                        uint8_t *__restrict__ selected,
                        const int64_t *__restrict__ index_map, int64_t step,
                        int64_t *__restrict__ sel_idx,
                        double *__restrict__ sel_gain) {
  Best x{-tinf<double>(), INT64_MAX};
  for (int b = threadIdx.x; b < nblocks; b += blockDim.x)
    x = better(x, Best{scratch[2 * b],
                       (int64_t)__double_as_longlong(scratch[2 * b + 1])});
  x = block_best(x);
  if (threadIdx.x == 0) {
    const int64_t j = x.i;
    if (j == INT64_MAX) {
      // no valid candidate (every gain NaN or already selected): sentinel
      // -1, which K2 treats as "S unchanged" and the host turns into an
      // error (never a silent duplicate exemplar)
      sel_idx[step] = -1;
      sel_gain[step] = x.v;
    } else {
      selected[j] = 1;
      sel_idx[step] = index_map ? index_map[j] : j;
      sel_gain[step] = x.v;
    }
  }
}

// ============================================================ peer reduce
// Multi-GPU K5 without NCCL: every rank's local gains vector lives in an
// IPC-shared buffer; after its K3 + K6 a rank publishes a step counter
// (release, system scope).  The consumer kernel on every rank waits for all
// peers' counters (acquire), sums the W local vectors in fixed rank order
// straight out of peer memory over NVLink and runs the argmax partial in the
// same pass -- the collective fused into its consumer, and the summation
// order (hence the picks) independent of the rank's position and of any
// NCCL algorithm choice.
__global__ void peer_publish_kernel(unsigned long long *flag,
                                    unsigned long long value) {
  __threadfence_system();
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(flag), "l"(value)
               : "memory");
}

__device__ __forceinline__ unsigned long long ld_acquire_sys(
    const unsigned long long *p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p)
               : "memory");
  return v;
}

__global__ void __launch_bounds__(kArgThreads)
    peer_argmax_partial_kernel(const double *const *__restrict__ peers,
                               const unsigned long long *const *__restrict__ flags,
                               int world, unsigned long long expect,
                               int64_t l, double scale,
                               double *__restrict__ gains_out,
                               const uint8_t *__restrict__ selected,
                               double *__restrict__ scratch) {
  if (threadIdx.x < world) {
    const unsigned long long *f = flags[threadIdx.x];
    while (ld_acquire_sys(f) < expect) __nanosleep(100);
  }
  __syncthreads();
  Best x{-tinf<double>(), INT64_MAX};
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < l;
       j += (int64_t)gridDim.x * blockDim.x) {
    double v = 0.0;
    for (int r = 0; r < world; ++r) v += peers[r][j];  // fixed rank order
    v *= scale;
    gains_out[j] = v;
    if (!selected[j] && !(v != v)) x = better(x, Best{v, j});
  }
  x = block_best(x);
  if (threadIdx.x == 0) {
    scratch[2 * blockIdx.x] = x.v;
    scratch[2 * blockIdx.x + 1] = __longlong_as_double((long long)x.i);
  }
}

// ============================================================ distances
// out[i][j] = d(a_i, b_j), the reference's per-precision form
// (objective.py:75-90).  64 x 64 output tile per CTA, 256 threads with 4 x 4
// outputs each; k-chunks of 16 staged through shared memory so every a / b
// element is read from global memory once per tile (not once per output);
// per output the k-sum runs sequentially with fma, as before tiling.
constexpr int kDistTile = 64, kDistK = 16;
template <int DT>
__global__ void __launch_bounds__(256)
    distance_matrix_kernel(const typename Traits<DT>::C *__restrict__ a,
                           const double *__restrict__ an, int64_t m,
                           const typename Traits<DT>::C *__restrict__ b,
                           const double *__restrict__ bn, int64_t q, int d,
                           int64_t d_pad, typename Traits<DT>::C *out) {
  using C = typename Traits<DT>::C;
  __shared__ C sa[kDistK][kDistTile + 1];
  __shared__ C sb[kDistK][kDistTile + 1];
  const int64_t i0 = (int64_t)blockIdx.y * kDistTile;
  const int64_t j0 = (int64_t)blockIdx.x * kDistTile;
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  C acc[4][4];
#pragma unroll
  for (int u = 0; u < 4; ++u)
#pragma unroll
    for (int v = 0; v < 4; ++v) acc[u][v] = C(0);
  for (int k0 = 0; k0 < d; k0 += kDistK) {
    // consecutive threads read consecutive k of one row (rows are d_pad
    // long, zero padded): 16-element runs
    for (int e = threadIdx.x; e < kDistTile * kDistK; e += 256) {
      const int r = e / kDistK, kk = e % kDistK, k = k0 + kk;
      const int64_t gi = i0 + r, gj = j0 + r;
      sa[kk][r] = (gi < m && k < d_pad) ? a[gi * d_pad + k] : C(0);
      sb[kk][r] = (gj < q && k < d_pad) ? b[gj * d_pad + k] : C(0);
    }
    __syncthreads();
    const int kn = min(kDistK, d - k0);
    for (int kk = 0; kk < kn; ++kk) {
      C av[4], bv[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) av[u] = sa[kk][ty + 16 * u];
#pragma unroll
      for (int v = 0; v < 4; ++v) bv[v] = sb[kk][tx + 16 * v];
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          if (Traits<DT>::kDirect) {
            const C df = av[u] - bv[v];
            acc[u][v] = fma(df, df, acc[u][v]);
          } else {
            acc[u][v] = fma(av[u], bv[v], acc[u][v]);
          }
        }
    }
    __syncthreads();
  }
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int64_t i = i0 + ty + 16 * u;
    if (i >= m) continue;
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      const int64_t j = j0 + tx + 16 * v;
      if (j >= q) continue;
      out[i * q + j] = Traits<DT>::kDirect
                           ? acc[u][v]
                           : gemm_form<C>(acc[u][v], (C)an[i], (C)bn[j]);
    }
  }
}

template <typename C>
__global__ void row_norms_kernel(const C *x, int64_t rows, int d,
                                 int64_t d_pad, double *out) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= rows) return;
  double s = 0.0;
  for (int k = 0; k < d; ++k) {
    double v = (double)x[r * d_pad + k];
    s += v * v;
  }
  out[r] = s;
}

// pnorms[e][j] = ||S_j[e]||^2 from the packed dim-major layout
// (coalesced over j).
template <typename C>
__global__ void packed_norms_kernel(const C *__restrict__ packed, int d,
                                    int64_t k_max, int64_t l_pad,
                                    double *__restrict__ out) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t total = k_max * l_pad;
  if (idx >= total) return;
  double s = 0.0;
  for (int k = 0; k < d; ++k) {
    const double v = (double)packed[(int64_t)k * total + idx];
    s += v * v;
  }
  out[idx] = s;
}

// Packed round-robin batch from element rows: packed[k][e][j] = the k-th
// coordinate of element e of set j (packed_address order, core.py:320-328),
// compute type, zero for blank slots (e >= card_j), padding dims and padding
// sets.  rows[offsets[j] + e][d] holds set j's elements (storage dtype), so
// the host only concatenates the sets -- no strided host transpose.
template <int DT>
__global__ void pack_elements_kernel(
    const typename Traits<DT>::S *__restrict__ rows,
    const int64_t *__restrict__ offsets, const int32_t *__restrict__ card,
    int64_t l, int64_t l_pad, int k_max, int d, int d_pad,
    typename Traits<DT>::C *__restrict__ packed) {
  using C = typename Traits<DT>::C;
  const int64_t j = (int64_t)blockIdx.x * 32 + threadIdx.x;
  const int e = blockIdx.y;
  if (j >= l_pad) return;
  const bool live = j < l && e < card[j];
  const int64_t base = live ? (offsets[j] + e) * (int64_t)d : 0;
  const int64_t stride_k = (int64_t)k_max * l_pad;
  for (int k = threadIdx.y; k < d_pad; k += blockDim.y) {
    const C v = (live && k < d) ? to_c(rows[base + k]) : C(0);
    packed[(int64_t)k * stride_k + (int64_t)e * l_pad + j] = v;
  }
}

// A packed round-robin batch as the host holds it -- storage dtype,
// [d][k_max][l] (PackedBatch.values, core.py:331-346) -- widened to the
// compute type and zero padded to [d_pad][k_max][l_pad] on the device, so the
// host uploads the raw packed bytes instead of converting them.
template <int DT>
__global__ void widen_packed_kernel(const typename Traits<DT>::S *__restrict__ src,
                                    int64_t l, int64_t l_pad, int k_max, int d,
                                    int d_pad,
                                    typename Traits<DT>::C *__restrict__ dst) {
  using C = typename Traits<DT>::C;
  const int64_t j = (int64_t)blockIdx.x * 128 + threadIdx.x;
  const int e = blockIdx.y;
  if (j >= l_pad) return;
  for (int k = blockIdx.z; k < d_pad; k += gridDim.z) {
    const C v = (k < d && j < l)
                    ? to_c(src[((int64_t)k * k_max + e) * l + j])
                    : C(0);
    dst[((int64_t)k * k_max + e) * l_pad + j] = v;
  }
}

// SieveStreaming over a block of arriving elements: for every sieve row s
// (rows of M, row 0 = aux) and block element b,
//   partial[cta][s][b] = sum_{i in the CTA's points} max(0, M[s][i] - D[b][i])
// 256 threads as 16 x 16, each a 4 (rows) x 4 (elements) register tile of
// fp64 sums; M and D are staged 32 points at a time (coalesced).  A 64 x 64
// (rows x elements) tile per grid.y / grid.z index.
constexpr int kSbTile = 64, kSbPts = 32;

template <typename C>
__global__ void __launch_bounds__(256)
    sieve_block_gains_kernel(const C *__restrict__ M, int64_t ldm, int rows,
                             const C *__restrict__ D, int64_t ldd, int nb,
                             int64_t n, int64_t pts_per_cta,
                             double *__restrict__ partial) {
  __shared__ C Ms[kSbTile][kSbPts + 1];
  __shared__ C Ds[kSbTile][kSbPts + 1];
  const int ts = threadIdx.x >> 4, tb = threadIdx.x & 15;
  const int r0 = blockIdx.y * kSbTile, b0 = blockIdx.z * kSbTile;
  const int64_t p0 = (int64_t)blockIdx.x * pts_per_cta;
  const int64_t p1 = min(n, p0 + pts_per_cta);
  double acc[4][4];
#pragma unroll
  for (int u = 0; u < 4; ++u)
#pragma unroll
    for (int v = 0; v < 4; ++v) acc[u][v] = 0.0;
  for (int64_t q = p0; q < p1; q += kSbPts) {
    __syncthreads();
    for (int idx = threadIdx.x; idx < kSbTile * kSbPts; idx += 256) {
      const int r = idx / kSbPts, c = idx % kSbPts;
      const int64_t i = q + c;
      // padding points contribute max(0, 0 - 0) = 0
      Ms[r][c] = (r0 + r < rows && i < p1) ? M[(int64_t)(r0 + r) * ldm + i] : C(0);
      Ds[r][c] = (b0 + r < nb && i < p1) ? D[(int64_t)(b0 + r) * ldd + i] : C(0);
    }
    __syncthreads();
#pragma unroll 4
    for (int c = 0; c < kSbPts; ++c) {
      C m[4], dd[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) m[u] = Ms[ts * 4 + u][c];
#pragma unroll
      for (int v = 0; v < 4; ++v) dd[v] = Ds[tb * 4 + v][c];
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v)
          acc[u][v] += (double)tmax(m[u] - dd[v], C(0));
    }
  }
  // partial[cta][r][b] over the full (rows x nb) output
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int r = r0 + ts * 4 + u;
    if (r >= rows) continue;
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      const int b = b0 + tb * 4 + v;
      if (b < nb)
        partial[((int64_t)blockIdx.x * rows + r) * nb + b] = acc[u][v];
    }
  }
}

}  // namespace exem

using namespace exem;

// ============================================================ C-ABI
extern "C" {

const char *exem_last_error(void) { return g_err; }
int exem_abi_version(void) { return 4; }
int64_t exem_launch_count(void) {
  return (int64_t)__atomic_load_n(&g_launches, __ATOMIC_RELAXED);
}

int exem_device_info(int device, int *sm_count, int *cc_major, int *cc_minor,
                     int64_t *smem_optin) {
  cudaDeviceProp p;
  cudaError_t e = cudaGetDeviceProperties(&p, device);
  if (e != cudaSuccess)
    return fail(EXEM_ERR_UNSUPPORTED, "cudaGetDeviceProperties: %s",
                cudaGetErrorString(e));
  if (sm_count) *sm_count = p.multiProcessorCount;
  if (cc_major) *cc_major = p.major;
  if (cc_minor) *cc_minor = p.minor;
  if (smem_optin) *smem_optin = (int64_t)p.sharedMemPerBlockOptin;
  return EXEM_OK;
}

int64_t exem_pad_points(int64_t n) {
  return round_up(n < 1 ? 1 : n, kPointPad);
}
int64_t exem_pad_dims(int64_t d) { return round_up(d < 1 ? 1 : d, kDimPad); }
int64_t exem_split_points(int64_t n) {
  // A function of n only, so per-set sums never depend on l, chunking or the
  // number of ranks (cf. fixed COL_BLOCK, core.py:27-30).  Multiple of 256.
  int64_t target = n / 16;
  int64_t p = 1024;
  while (p * 2 <= target && p < 32768) p *= 2;
  return p;
}
int64_t exem_num_splits(int64_t n) {
  return ceil_div(n < 1 ? 1 : n, exem_split_points(n));
}
int64_t exem_tc_kp(int64_t d) { return round_up(d + kTcConst, kTcKChunk); }
int64_t exem_tc_rows(int64_t n) { return round_up(n < 1 ? 1 : n, kPointPad); }
int64_t exem_reduce_scratch(int64_t count) {
  int64_t b = ceil_div(count < 1 ? 1 : count, kRedThreads);
  return b < 2 * 1024 ? 2 * 1024 : b;  // also covers argmax's 2*blocks
}

int exem_ground_prepare(int dtype, const void *src, int64_t n, int64_t d,
                        const void *e0, void *vt, int64_t ld, double *norms,
                        void *aux, double *aux_sum, double *scratch,
                        int check_finite, void *stream) {
  if (n < 1 || d < 1 || ld < n || ld % kPointPad)
    return fail(EXEM_ERR_ARG, "ground_prepare: bad shape n=%lld d=%lld ld=%lld",
                (long long)n, (long long)d, (long long)ld);
  cudaStream_t st = (cudaStream_t)stream;
  const int d_pad = (int)exem_pad_dims(d);
  const int64_t blocks = ceil_div(ld, kRedThreads);
  EXEM_DISPATCH_VT(dtype, DT, VS, {
    using S = typename Traits<DT>::S;
    using C = typename Traits<DT>::C;
    using V = typename VtOf<DT, VS>::T;
    // pair kernel for 2-byte vt: 4-byte aligned source rows need even n
    // (and 4-byte aligned buffers)
    if (VS && n % 2 == 0 && aligned(src, 4) && aligned(vt, 4) &&
        launch_prepare_pair<DT>(blocks, st, src, n, (int)d, d_pad, e0, vt, ld,
                                norms, aux, scratch, check_finite != 0)) {
      EXEM_LAUNCH_CHECK("ground_prepare_pair_kernel");
      break;
    }
    ground_prepare_kernel<DT, VS><<<(unsigned)blocks, kRedThreads, 0, st>>>(
        (const S *)src, n, (int)d, d_pad, (const S *)e0, (V *)vt, ld, norms,
        (C *)aux, scratch, check_finite != 0);
    EXEM_LAUNCH_CHECK("ground_prepare_kernel");
  });
  // aux_sum == NULL: leave the per-256-point block partials in scratch (a
  // streamed slice writes them at its global block offset; exem_sum_fixed
  // then reduces all of them in the same order as a resident build).
  if (!aux_sum) return EXEM_OK;
  return reduce_fixed(scratch, blocks, aux_sum, 0, st);
}

int exem_sum_fixed(const double *in, int64_t count, double *out,
                   int64_t out_index, void *stream) {
  if (count < 1) return fail(EXEM_ERR_ARG, "sum_fixed: count must be >= 1");
  return reduce_fixed(in, count, out, out_index, (cudaStream_t)stream);
}

int exem_host_register(void *host, int64_t bytes) {
  cudaError_t e = cudaHostRegister(host, (size_t)bytes, cudaHostRegisterDefault);
  if (e != cudaSuccess && e != cudaErrorHostMemoryAlreadyRegistered) {
    // a read-only mapping (e.g. a memory-mapped .exem payload) can only be
    // locked read-only
    cudaGetLastError();
    e = cudaHostRegister(host, (size_t)bytes, cudaHostRegisterReadOnly);
  }
  cudaGetLastError();  // never leave a sticky error for the next launch check
  if (e == cudaErrorHostMemoryAlreadyRegistered) return EXEM_OK;
  if (e != cudaSuccess)
    return fail(EXEM_ERR_CUDA, "cudaHostRegister: %s", cudaGetErrorString(e));
  return EXEM_OK;
}

int exem_host_unregister(void *host) {
  cudaError_t e = cudaHostUnregister(host);
  if (e != cudaSuccess && e != cudaErrorHostMemoryNotRegistered)
    return fail(EXEM_ERR_CUDA, "cudaHostUnregister: %s", cudaGetErrorString(e));
  cudaGetLastError();
  return EXEM_OK;
}

int exem_h2d_rows(void *dst, const void *host, int64_t ld_host, int64_t row0,
                  int64_t rows, int64_t d, int64_t elem_bytes, void *stream) {
  if (rows < 1 || d < 1 || row0 < 0 || row0 + rows > ld_host)
    return fail(EXEM_ERR_ARG, "h2d_rows: bad slice [%lld, %lld) of %lld",
                (long long)row0, (long long)(row0 + rows), (long long)ld_host);
  const char *src = (const char *)host + row0 * elem_bytes;
  cudaError_t e = cudaMemcpy2DAsync(dst, (size_t)(rows * elem_bytes), src,
                                    (size_t)(ld_host * elem_bytes),
                                    (size_t)(rows * elem_bytes), (size_t)d,
                                    cudaMemcpyHostToDevice,
                                    (cudaStream_t)stream);
  if (e != cudaSuccess)
    return fail(EXEM_ERR_CUDA, "h2d_rows: %s", cudaGetErrorString(e));
  return EXEM_OK;
}

int exem_set_min_storage_ok(int dtype, int64_t d, int64_t k, int has_t_out) {
  return set_min_storage_ok(dtype, d, k, has_t_out);
}

int exem_set_min(int dtype, const void *vt, int64_t ld, int64_t n, int64_t d,
                 const double *norms, const void *aux, const void *elems,
                 const double *enorms, int64_t k, int include_aux, void *t_out,
                 int64_t *label_out, double *sum_out, double *scratch,
                 void *stream) {
  if (n < 1 || d < 1 || k < 0)
    return fail(EXEM_ERR_ARG, "set_min: bad shape");
  cudaStream_t st = (cudaStream_t)stream;
  const int d_pad = (int)exem_pad_dims(d);
  const int64_t blocks = ceil_div(n, kRedThreads);
  if (dtype & EXEM_VT_STORAGE) {
    // 2-byte storage-typed vt: the TMA-fed K2 only (it widens in registers)
    if (!set_min_storage_ok(dtype, d, k, t_out != nullptr) || ld % kSmP)
      return fail(EXEM_ERR_ARG,
                  "set_min: storage-typed vt is not covered for d=%lld k=%lld "
                  "(exem_set_min_storage_ok)", (long long)d, (long long)k);
    const int tma = set_min_tma(dtype, vt, ld, n, d_pad, norms, aux, elems,
                                enorms, (int)k, include_aux, t_out, label_out,
                                scratch, nullptr, 0, st);
    if (tma != 0)
      return fail(tma > 0 ? EXEM_ERR_ARG : EXEM_ERR_CUDA, "set_min (TMA): %s",
                  tma > 0 ? "shape not covered"
                          : cudaGetErrorString((cudaError_t)(-tma)));
    count_launch();
    if (sum_out) return reduce_fixed(scratch, blocks, sum_out, 0, st);
    return EXEM_OK;
  }
  EXEM_DISPATCH(dtype, DT, {
    using C = typename Traits<DT>::C;
    cudaError_t e = launch_set_min<DT>(
        blocks, st, (const C *)vt, ld, n, (int)d, norms, (const C *)aux,
        (const C *)elems, d_pad, enorms, (int)k, include_aux, (C *)t_out,
        label_out, scratch);
    if (e != cudaSuccess)
      return fail(EXEM_ERR_CUDA, "set_min_kernel: %s", cudaGetErrorString(e));
    count_launch();
  });
  if (sum_out) return reduce_fixed(scratch, blocks, sum_out, 0, st);
  return EXEM_OK;
}

int exem_greedy_init(int dtype, const void *aux, int64_t n, void *m,
                     double *msum_out, double *scratch, void *stream) {
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t blocks = ceil_div(n, kRedThreads);
  if (dtype == EXEM_F64) {
    greedy_init_kernel<double><<<(unsigned)blocks, kRedThreads, 0, st>>>(
        (const double *)aux, n, (double *)m, scratch);
  } else {
    greedy_init_kernel<float><<<(unsigned)blocks, kRedThreads, 0, st>>>(
        (const float *)aux, n, (float *)m, scratch);
  }
  EXEM_LAUNCH_CHECK("greedy_init_kernel");
  return reduce_fixed(scratch, blocks, msum_out, 0, st);
}

int exem_greedy_update(int dtype, const void *vt, int64_t ld, int64_t n,
                       int64_t d, const double *norms, const void *cvt,
                       int64_t ldc, const double *cnorms,
                       const int64_t *sel_idx, int64_t step, void *m,
                       void *xp, int64_t kp, double *msum, double *scratch,
                       void *stream) {
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t blocks = ceil_div(n, kRedThreads);
  EXEM_DISPATCH_VT(dtype, DT, VS, {
    using S = typename Traits<DT>::S;
    using C = typename Traits<DT>::C;
    using V = typename VtOf<DT, VS>::T;
    if (VS && aligned(vt, 4) && aligned(cvt, 2) && aligned(m, 8) &&
        launch_update_pair<DT>(blocks, st, vt, ld, n, (int)d, norms,
                                     cvt, ldc, sel_idx, step, m, xp, kp,
                                     scratch)) {
      EXEM_LAUNCH_CHECK("greedy_update_pair_kernel");
      break;
    }
    greedy_update_kernel<DT, VS><<<(unsigned)blocks, kRedThreads, 0, st>>>(
        (const V *)vt, ld, n, (int)d, norms, (const V *)cvt, ldc, cnorms,
        sel_idx, step, (C *)m, (S *)xp, kp, scratch);
    EXEM_LAUNCH_CHECK("greedy_update_kernel");
  });
  // msum == NULL: leave the per-256-point block partials of sum_i m_i in
  // scratch (a streamed slice writes them at its global block offset)
  if (!msum) return EXEM_OK;
  return reduce_fixed(scratch, blocks, msum, step, st);
}

static int simt_grid_ok(int64_t rows, int64_t n, int64_t split_pts,
                        int64_t splits) {
  if (split_pts < kBN || split_pts % kBN)
    return fail(EXEM_ERR_ARG, "split_pts must be a positive multiple of %d",
                kBN);
  if (splits != ceil_div(n, split_pts))
    return fail(EXEM_ERR_ARG, "splits=%lld != ceil(n/split_pts)=%lld",
                (long long)splits, (long long)ceil_div(n, split_pts));
  if (ceil_div(rows, kBM) > 0x7fffffffll || splits > 65535)
    return fail(EXEM_ERR_ARG, "grid too large");
  return EXEM_OK;
}

int exem_greedy_gains_simt(int dtype, const void *cvt, int64_t ldc,
                           const double *cnorms, int64_t l, const void *vt,
                           int64_t ld, const double *norms, const void *m,
                           int64_t n, int64_t d, int64_t split_pts,
                           double *partial, int64_t splits, void *stream) {
  if (int rc = simt_grid_ok(l, n, split_pts, splits)) return rc;
  if (ldc % kBM || ld % kBN || ldc < round_up(l, kBM))
    return fail(EXEM_ERR_ARG, "greedy_gains_simt: leading dims not padded");
  cudaStream_t st = (cudaStream_t)stream;
  const int d_pad = (int)exem_pad_dims(d);
  // the TMA-fed kernel (exem_simt_tma.cu) when its tensor maps apply
  {
    const int r = gains_simt_tma(dtype, cvt, ldc, cnorms, l, vt, ld, norms, m,
                                 n, d_pad, split_pts, splits, partial, st);
    if (r == 0) {
      count_launch();
      return EXEM_OK;
    }
    if (r < 0)
      return fail(EXEM_ERR_CUDA, "gains_simt_tma_kernel: %s",
                  cudaGetErrorString((cudaError_t)(-r)));
  }
  dim3 grid((unsigned)ceil_div(l, kBM), (unsigned)splits);
  // fp64: k-chunks of 16 (half the ring barriers per DFMA) when d_pad allows
  // it without extra padding -- d = 512 / 1024: 436 -> 413 / 866 -> 822 ms.
  // fp32 with the paired FFMA2 loop: 16 from d_pad = 128 up (d = 512 / 1024:
  // 169.5 -> 167.2 / 337.5 -> 333.1 ms); small d keeps 8 (d = 16: 6.82 vs
  // 6.93 ms) (profiles/r02_simt_bk.log).
  // EXEM_SIMT_BK = 8 | 16 overrides (timing experiments).
  static const int bk_env = getenv("EXEM_SIMT_BK") ? atoi(getenv("EXEM_SIMT_BK")) : 0;
  const bool bk16 = d_pad % 16 == 0 &&
                    (bk_env == 16 ||
                     (bk_env == 0 && (dtype == EXEM_F64 || d_pad >= 128)));
  if (dtype == EXEM_F32 && bk16) {
    size_t smem = sizeof(SimtSmem<float, 16>);
    cudaError_t e = cudaFuncSetAttribute(
        gains_simt_kernel<float, 2, 16>,
        cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess)
      return fail(EXEM_ERR_CUDA, "gains_simt smem: %s", cudaGetErrorString(e));
    gains_simt_kernel<float, 2, 16><<<grid, kThreads, smem, st>>>(
        (const float *)cvt, ldc, cnorms, l, (const float *)vt, ld, norms,
        (const float *)m, n, d_pad, (int)d, split_pts, partial);
    EXEM_LAUNCH_CHECK("gains_simt_kernel<f32,16>");
  } else if (dtype == EXEM_F64 && bk16) {
    size_t smem = sizeof(SimtSmem<double, 16>);
    cudaError_t e = cudaFuncSetAttribute(
        gains_simt_kernel<double, 1, 16>,
        cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess)
      return fail(EXEM_ERR_CUDA, "gains_simt smem: %s", cudaGetErrorString(e));
    gains_simt_kernel<double, 1, 16><<<grid, kThreads, smem, st>>>(
        (const double *)cvt, ldc, cnorms, l, (const double *)vt, ld, norms,
        (const double *)m, n, d_pad, (int)d, split_pts, partial);
    EXEM_LAUNCH_CHECK("gains_simt_kernel<f64,16>");
  } else if (dtype == EXEM_F32) {
    size_t smem = sizeof(SimtSmem<float>);
    if (d % kBK) {  // partial last chunk: its own instantiation
      gains_simt_kernel<float, 2, kBK, true><<<grid, kThreads, smem, st>>>(
          (const float *)cvt, ldc, cnorms, l, (const float *)vt, ld, norms,
          (const float *)m, n, d_pad, (int)d, split_pts, partial);
    } else {
      gains_simt_kernel<float, 2><<<grid, kThreads, smem, st>>>(
          (const float *)cvt, ldc, cnorms, l, (const float *)vt, ld, norms,
          (const float *)m, n, d_pad, (int)d, split_pts, partial);
    }
    EXEM_LAUNCH_CHECK("gains_simt_kernel<f32>");
  } else if (dtype == EXEM_F64) {
    size_t smem = sizeof(SimtSmem<double>);  // 48 KB: needs the opt-in
    cudaError_t e = cudaFuncSetAttribute(
        gains_simt_kernel<double, 1>,
        cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess)
      return fail(EXEM_ERR_CUDA, "gains_simt smem: %s", cudaGetErrorString(e));
    gains_simt_kernel<double, 1><<<grid, kThreads, smem, st>>>(
        (const double *)cvt, ldc, cnorms, l, (const double *)vt, ld, norms,
        (const double *)m, n, d_pad, (int)d, split_pts, partial);
    EXEM_LAUNCH_CHECK("gains_simt_kernel<f64>");
  } else {
    return fail(EXEM_ERR_ARG,
                "greedy_gains_simt handles f32/f64; half precisions use the "
                "tcgen05 path (exem_greedy_gains_tc)");
  }
  return EXEM_OK;
}

int exem_batch_eval(int dtype, const void *vt, int64_t ld, int64_t n,
                    int64_t d, const double *norms, const void *aux,
                    const void *packed, const double *pnorms,
                    const int32_t *card, int64_t l, int64_t l_pad,
                    int64_t k_max, int64_t split_pts, double *partial,
                    int64_t splits, void *stream) {
  if (int rc = simt_grid_ok(l, n, split_pts, splits)) return rc;
  if (l_pad % kBM || l_pad < l || ld % kBN || k_max < 1)
    return fail(EXEM_ERR_ARG, "batch_eval: bad padding l_pad=%lld",
                (long long)l_pad);
  cudaStream_t st = (cudaStream_t)stream;
  const int d_pad = (int)exem_pad_dims(d);
  dim3 grid((unsigned)ceil_div(l, kBM), (unsigned)splits);
  EXEM_DISPATCH(dtype, DT, {
    using C = typename Traits<DT>::C;
    size_t smem = sizeof(BatchSmem<C>);
    // partial last chunk (d % 8 != 0): the instantiation that skips its
    // zero padding dimensions (exact zeros; see simt_mainloop)
    const bool tail = d % kBK != 0;
    cudaError_t e = cudaFuncSetAttribute(
        tail ? (const void *)batch_eval_kernel<DT, true>
             : (const void *)batch_eval_kernel<DT, false>,
        cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess)
      return fail(EXEM_ERR_CUDA, "batch_eval smem: %s", cudaGetErrorString(e));
    if (tail)
      batch_eval_kernel<DT, true><<<grid, kThreads, smem, st>>>(
          (const C *)vt, ld, n, d_pad, (int)d, norms, (const C *)aux,
          (const C *)packed, pnorms, card, l, l_pad, (int)k_max, split_pts,
          partial);
    else
      batch_eval_kernel<DT, false><<<grid, kThreads, smem, st>>>(
          (const C *)vt, ld, n, d_pad, (int)d, norms, (const C *)aux,
          (const C *)packed, pnorms, card, l, l_pad, (int)k_max, split_pts,
          partial);
    EXEM_LAUNCH_CHECK("batch_eval_kernel");
  });
  return EXEM_OK;
}

int exem_reduce_partials(const double *partial, int64_t splits, int64_t l,
                         double scale, double *out, void *stream) {
  cudaStream_t st = (cudaStream_t)stream;
  reduce_partials_kernel<<<(unsigned)ceil_div(l, 256), 256, 0, st>>>(
      partial, splits, l, scale, out);
  EXEM_LAUNCH_CHECK("reduce_partials_kernel");
  return EXEM_OK;
}

int exem_argmax_select(const double *gains, int64_t l, uint8_t *selected,
                       const int64_t *index_map, int64_t step,
                       int64_t *sel_idx, double *sel_gain, double *scratch,
                       void *stream) {
  if (l < 1) return fail(EXEM_ERR_ARG, "argmax over an empty candidate set");
  cudaStream_t st = (cudaStream_t)stream;
  int nb = (int)ceil_div(l, kArgThreads);
  if (nb > 296) nb = 296;  // 2 waves of 148 SMs; grid-stride inside
  argmax_partial_kernel<<<nb, kArgThreads, 0, st>>>(gains, l, selected,
                                                    scratch);
  EXEM_LAUNCH_CHECK("argmax_partial_kernel");
  argmax_final_kernel<<<1, kArgThreads, 0, st>>>(scratch, nb, selected,
                                                 index_map, step, sel_idx,
                                                 sel_gain);
  EXEM_LAUNCH_CHECK("argmax_final_kernel");
  return EXEM_OK;
}

int exem_distance_matrix(int dtype, const void *a, const double *anorms,
                         int64_t m, const void *b, const double *bnorms,
                         int64_t q, int64_t d, int64_t d_pad, void *out,
                         void *stream) {
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t total = m * q;
  if (total == 0) return EXEM_OK;
  EXEM_DISPATCH(dtype, DT, {
    using C = typename Traits<DT>::C;
    const int64_t rows_per = (int64_t)65535 * kDistTile;  // grid.y limit
    for (int64_t r0 = 0; r0 < m; r0 += rows_per) {
      const int64_t mr = m - r0 < rows_per ? m - r0 : rows_per;
      const dim3 grid((unsigned)ceil_div(q, kDistTile),
                      (unsigned)ceil_div(mr, kDistTile));
      distance_matrix_kernel<DT><<<grid, 256, 0, st>>>(
          (const C *)a + r0 * d_pad, anorms + r0, mr, (const C *)b, bnorms, q,
          (int)d, d_pad, (C *)out + r0 * q);
      EXEM_LAUNCH_CHECK("distance_matrix_kernel");
    }
  });
  return EXEM_OK;
}

int exem_row_norms(int dtype, const void *x, int64_t rows, int64_t d,
                   int64_t d_pad, double *out, void *stream) {
  cudaStream_t st = (cudaStream_t)stream;
  if (rows == 0) return EXEM_OK;
  if (dtype == EXEM_F64)
    row_norms_kernel<double><<<(unsigned)ceil_div(rows, 256), 256, 0, st>>>(
        (const double *)x, rows, (int)d, d_pad, out);
  else
    row_norms_kernel<float><<<(unsigned)ceil_div(rows, 256), 256, 0, st>>>(
        (const float *)x, rows, (int)d, d_pad, out);
  EXEM_LAUNCH_CHECK("row_norms_kernel");
  return EXEM_OK;
}

int exem_packed_norms(int dtype, const void *packed, int64_t d, int64_t k_max,
                      int64_t l_pad, double *out, void *stream) {
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t total = k_max * l_pad;
  if (total == 0) return EXEM_OK;
  const unsigned grid = (unsigned)ceil_div(total, 256);
  if (dtype == EXEM_F64)
    packed_norms_kernel<double><<<grid, 256, 0, st>>>((const double *)packed,
                                                      (int)d, k_max, l_pad, out);
  else
    packed_norms_kernel<float><<<grid, 256, 0, st>>>((const float *)packed,
                                                     (int)d, k_max, l_pad, out);
  EXEM_LAUNCH_CHECK("packed_norms_kernel");
  return EXEM_OK;
}

int exem_pack_elements(int dtype, const void *rows, const int64_t *offsets,
                       const int32_t *card, int64_t l, int64_t l_pad,
                       int64_t k_max, int64_t d, void *packed, void *stream) {
  if (l < 1 || k_max < 1 || d < 1 || l_pad < l || k_max > 65535)
    return fail(EXEM_ERR_ARG, "pack_elements: bad shape");
  const int d_pad = (int)exem_pad_dims(d);
  dim3 block(32, 8);
  dim3 grid((unsigned)ceil_div(l_pad, 32), (unsigned)k_max);
  cudaStream_t st = (cudaStream_t)stream;
  EXEM_DISPATCH(dtype, DT, {
    using S = typename Traits<DT>::S;
    using C = typename Traits<DT>::C;
    pack_elements_kernel<DT><<<grid, block, 0, st>>>(
        (const S *)rows, offsets, card, l, l_pad, (int)k_max, (int)d, d_pad,
        (C *)packed);
    EXEM_LAUNCH_CHECK("pack_elements_kernel");
  });
  return EXEM_OK;
}

int exem_widen_packed(int dtype, const void *src, int64_t l, int64_t l_pad,
                      int64_t k_max, int64_t d, void *packed, void *stream) {
  if (l < 1 || k_max < 1 || d < 1 || l_pad < l || k_max > 65535)
    return fail(EXEM_ERR_ARG, "widen_packed: bad shape");
  const int d_pad = (int)exem_pad_dims(d);
  const int zs = d_pad < 64 ? d_pad : 64;
  dim3 grid((unsigned)ceil_div(l_pad, 128), (unsigned)k_max, (unsigned)zs);
  cudaStream_t st = (cudaStream_t)stream;
  EXEM_DISPATCH(dtype, DT, {
    using S = typename Traits<DT>::S;
    using C = typename Traits<DT>::C;
    widen_packed_kernel<DT><<<grid, 128, 0, st>>>(
        (const S *)src, l, l_pad, (int)k_max, (int)d, d_pad, (C *)packed);
    EXEM_LAUNCH_CHECK("widen_packed_kernel");
  });
  return EXEM_OK;
}

int exem_sieve_block_dist(int dtype, const void *vt, int64_t ld, int64_t n,
                          int64_t d, const double *norms, const void *elems,
                          const double *enorms, int64_t nb, void *dist,
                          int64_t ldd, double *scratch, void *stream) {
  if (n < 1 || d < 1 || nb < 1 || ldd < n)
    return fail(EXEM_ERR_ARG, "sieve_block_dist: bad shape");
  cudaStream_t st = (cudaStream_t)stream;
  const int d_pad = (int)exem_pad_dims(d);
  const int64_t blocks = ceil_div(n, kRedThreads);
  EXEM_DISPATCH(dtype, DT, {
    using C = typename Traits<DT>::C;
    // K2's distance arithmetic (identical to exem_set_min with k = 1),
    // every element's distance row written out
    cudaError_t e = launch_set_min<DT>(
        blocks, st, (const C *)vt, ld, n, (int)d, norms, nullptr,
        (const C *)elems, d_pad, enorms, (int)nb, 0, nullptr, nullptr, scratch,
        (C *)dist, ldd);
    if (e != cudaSuccess)
      return fail(EXEM_ERR_CUDA, "set_min_kernel(dist): %s",
                  cudaGetErrorString(e));
    count_launch();
  });
  return EXEM_OK;
}

int64_t exem_sieve_block_scratch(int64_t n, int64_t rows, int64_t nb) {
  const int64_t ctas = n < 32 * 296 ? ceil_div(n, 32) : 296;
  return ctas * rows * nb;
}

int exem_sieve_block_gains(int dtype, const void *M, int64_t ldm, int64_t rows,
                           const void *D, int64_t ldd, int64_t nb, int64_t n,
                           double *gains, double *scratch, void *stream) {
  if (n < 1 || rows < 1 || nb < 1 || ldm < n || ldd < n)
    return fail(EXEM_ERR_ARG, "sieve_block_gains: bad shape");
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t ctas = n < 32 * 296 ? ceil_div(n, 32) : 296;
  const int64_t per = round_up(ceil_div(n, ctas), kSbPts);
  const int64_t used = ceil_div(n, per);
  dim3 grid((unsigned)used, (unsigned)ceil_div(rows, kSbTile),
            (unsigned)ceil_div(nb, kSbTile));
  if (dtype == EXEM_F64)
    sieve_block_gains_kernel<double><<<grid, 256, 0, st>>>(
        (const double *)M, ldm, (int)rows, (const double *)D, ldd, (int)nb, n,
        per, scratch);
  else
    sieve_block_gains_kernel<float><<<grid, 256, 0, st>>>(
        (const float *)M, ldm, (int)rows, (const float *)D, ldd, (int)nb, n,
        per, scratch);
  EXEM_LAUNCH_CHECK("sieve_block_gains_kernel");
  // fixed-order sum over the CTAs' point chunks
  return exem_reduce_partials(scratch, used, rows * nb, 1.0, gains, stream);
}

int exem_sieve_gains(int dtype, const void *M, int64_t ldm, int64_t sieves,
                     const void *dist, int64_t n, double *gains,
                     double *scratch, void *stream) {
  if (n < 1 || sieves < 1 || ldm < n)
    return fail(EXEM_ERR_ARG, "sieve_gains: bad shape");
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t blocks = ceil_div(n, kRedThreads);
  dim3 grid((unsigned)blocks, (unsigned)sieves);
  if (dtype == EXEM_F64)
    sieve_gains_kernel<double><<<grid, kRedThreads, 0, st>>>(
        (const double *)M, ldm, (const double *)dist, n, scratch, blocks);
  else
    sieve_gains_kernel<float><<<grid, kRedThreads, 0, st>>>(
        (const float *)M, ldm, (const float *)dist, n, scratch, blocks);
  EXEM_LAUNCH_CHECK("sieve_gains_kernel");
  // scratch is [blocks][sieves]: the fixed-order column sums are the gains
  return exem_reduce_partials(scratch, blocks, sieves, 1.0, gains, stream);
}

int exem_sieve_update(int dtype, void *m, const void *dist, int64_t n,
                      double *msum, double *scratch, void *stream) {
  if (n < 1) return fail(EXEM_ERR_ARG, "sieve_update: bad shape");
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t blocks = ceil_div(n, kRedThreads);
  if (dtype == EXEM_F64)
    sieve_update_kernel<double><<<(unsigned)blocks, kRedThreads, 0, st>>>(
        (double *)m, (const double *)dist, n, scratch);
  else
    sieve_update_kernel<float><<<(unsigned)blocks, kRedThreads, 0, st>>>(
        (float *)m, (const float *)dist, n, scratch);
  EXEM_LAUNCH_CHECK("sieve_update_kernel");
  return reduce_fixed(scratch, blocks, msum, 0, st);
}

int exem_ipc_alloc(int64_t bytes, void **ptr) {
  if (bytes < 1) return fail(EXEM_ERR_ARG, "ipc_alloc: bytes must be >= 1");
  cudaError_t e = cudaMalloc(ptr, (size_t)bytes);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return fail(EXEM_ERR_OOM, "ipc_alloc: %s", cudaGetErrorString(e));
  }
  return EXEM_OK;
}

int exem_ipc_free(void *ptr) {
  cudaError_t e = cudaFree(ptr);
  if (e != cudaSuccess)
    return fail(EXEM_ERR_CUDA, "ipc_free: %s", cudaGetErrorString(e));
  return EXEM_OK;
}

int exem_ipc_handle(void *ptr, void *handle) {
  cudaIpcMemHandle_t h;
  cudaError_t e = cudaIpcGetMemHandle(&h, ptr);
  if (e != cudaSuccess)
    return fail(EXEM_ERR_CUDA, "cudaIpcGetMemHandle: %s", cudaGetErrorString(e));
  memcpy(handle, &h, sizeof(h));
  return EXEM_OK;
}

int exem_ipc_open(const void *handle, void **ptr) {
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof(h));
  cudaError_t e = cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess);
  if (e != cudaSuccess)
    return fail(EXEM_ERR_CUDA, "cudaIpcOpenMemHandle: %s", cudaGetErrorString(e));
  return EXEM_OK;
}

int exem_ipc_close(void *ptr) {
  cudaError_t e = cudaIpcCloseMemHandle(ptr);
  if (e != cudaSuccess)
    return fail(EXEM_ERR_CUDA, "cudaIpcCloseMemHandle: %s", cudaGetErrorString(e));
  return EXEM_OK;
}

int exem_peer_publish(unsigned long long *flag, unsigned long long value,
                      void *stream) {
  peer_publish_kernel<<<1, 1, 0, (cudaStream_t)stream>>>(flag, value);
  EXEM_LAUNCH_CHECK("peer_publish_kernel");
  return EXEM_OK;
}

int exem_peer_argmax_select(const double *const *peers,
                            const unsigned long long *const *flags, int world,
                            unsigned long long expect, int64_t l, double scale,
                            double *gains_out, uint8_t *selected,
                            int64_t step, int64_t *sel_idx, double *sel_gain,
                            double *scratch, void *stream) {
  if (l < 1 || world < 1 || world > kArgThreads)
    return fail(EXEM_ERR_ARG, "peer_argmax_select: bad shape");
  cudaStream_t st = (cudaStream_t)stream;
  int nb = (int)ceil_div(l, kArgThreads);
  if (nb > 296) nb = 296;
  peer_argmax_partial_kernel<<<nb, kArgThreads, 0, st>>>(
      peers, flags, world, expect, l, scale, gains_out, selected, scratch);
  EXEM_LAUNCH_CHECK("peer_argmax_partial_kernel");
  argmax_final_kernel<<<1, kArgThreads, 0, st>>>(scratch, nb, selected,
                                                 nullptr, step, sel_idx,
                                                 sel_gain);
  EXEM_LAUNCH_CHECK("argmax_final_kernel");
  return EXEM_OK;
}

int exem_ground_prepare_rows(int dtype, const void *src, int64_t n, int64_t d,
                             const void *e0, void *vt, int64_t ld,
                             double *norms, void *aux, double *aux_sum,
                             double *scratch, int check_finite, void *stream) {
  if (n < 1 || d < 1 || ld < n || ld % kPointPad)
    return fail(EXEM_ERR_ARG, "ground_prepare_rows: bad shape");
  cudaStream_t st = (cudaStream_t)stream;
  const int d_pad = (int)exem_pad_dims(d);
  const int64_t blocks = ceil_div(ld, kRedThreads);
  EXEM_DISPATCH_VT(dtype, DT, VS, {
    using S = typename Traits<DT>::S;
    using C = typename Traits<DT>::C;
    using V = typename VtOf<DT, VS>::T;
    {
      const int rc = launch_prepare_slab<DT, VS>(blocks, st, src, n, (int)d,
                                                 d_pad, e0, vt, ld, norms,
                                                 aux, scratch,
                                                 check_finite != 0);
      if (rc < 0)
        return fail(EXEM_ERR_CUDA, "prepare_rows smem: %s",
                    cudaGetErrorString((cudaError_t)(-rc)));
      if (rc == 0) {
        EXEM_LAUNCH_CHECK("ground_prepare_slab_kernel");
        break;
      }
    }
    const size_t smem = (size_t)kRedThreads * 33 * sizeof(C);
    if (smem > 48 * 1024) {
      cudaError_t e = cudaFuncSetAttribute(
          ground_prepare_rows_kernel<DT, VS>,
          cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e != cudaSuccess)
        return fail(EXEM_ERR_CUDA, "prepare_rows smem: %s",
                    cudaGetErrorString(e));
    }
    ground_prepare_rows_kernel<DT, VS><<<(unsigned)blocks, kRedThreads, smem, st>>>(
        (const S *)src, n, (int)d, d_pad, (const S *)e0, (V *)vt, ld, norms,
        (C *)aux, scratch, check_finite != 0);
    EXEM_LAUNCH_CHECK("ground_prepare_rows_kernel");
  });
  if (!aux_sum) return EXEM_OK;
  return reduce_fixed(scratch, blocks, aux_sum, 0, st);
}

int exem_h2d_bytes(void *dst, const void *host, int64_t bytes, void *stream) {
  if (bytes < 1) return EXEM_OK;
  cudaError_t e = cudaMemcpyAsync(dst, host, (size_t)bytes,
                                  cudaMemcpyHostToDevice, (cudaStream_t)stream);
  if (e != cudaSuccess)
    return fail(EXEM_ERR_CUDA, "h2d_bytes: %s", cudaGetErrorString(e));
  return EXEM_OK;
}

}  // extern "C"
