// exem_setmin.cu -- K2 set_min, TMA-fed persistent variant (sm_100a).
//
// min_distances / _set_value / assign_clusters over ONE explicit set
// (reference objective.py:113-141, evaluate.py:105-112, optimize.py:115-136):
//   t_i = min(aux_i, min_e d(v_i, e)),  partial[b] = sum of t_i over the
//   256-point block b (fixed order), labels = first argmin.
//
// Design (K2):
//  * The whole element group (KG <= 64 elements x all d_pad dimensions,
//    transposed to [dim][element], zero padded) is loaded into shared memory
//    ONCE per CTA; CTAs are persistent (2 per SM) and walk 256-point tiles.
//  * V ([d_pad][ld] column-major "vt" layout) streams through an S-stage ring
//    of [BK dims][256 points] boxes loaded by TMA (cp.async.bulk.tensor, one
//    instruction per stage, completion on an mbarrier with expect_tx), so the
//    CTA keeps S x 32 KB in flight with no per-thread copy instructions.  A
//    stage is released by one arrive per warp; thread 0 re-arms it.
//  * Every thread owns PT = KG/8 points x 8 elements of dot products in
//    registers (register-blocked outer product over the dimensions).  Lanes
//    are laid out so each shared-memory vector load of a warp touches one
//    contiguous 128-byte line: per dimension a warp issues PT/4 (points) +
//    2 (elements) conflict-free LDS per 8*PT FMAs.
//  * Distances use the reference's per-precision form and the same
//    sequential fma chain over the dimensions as the other SIMT kernels;
//    the minimum keeps the lowest element index on ties; the per-256-point
//    block partial is the same fixed-order block_sum as K1/K2/streaming, so
//    results are bit-identical to the previous K2.
//
// Algorithmic bytes per launch: n*d*4 (V, read once per
// element group) + 8n (norms) + 4n (aux) + the elements; FFMA work 2*n*k*d.
#include <cstdlib>

#include "exem_tc_common.cuh"

namespace exem {

namespace {

constexpr int kP = 256;        // points per tile (= 256 threads)
constexpr int kThreads = 256;
#ifndef EXEM_K2_UNROLL_WIDE  // experiment: kk unroll of the wide (EG >= 4) shapes
#define EXEM_K2_UNROLL_WIDE 8
#endif
constexpr int kUnrollWide = EXEM_K2_UNROLL_WIDE;
constexpr int kMaxStages = 16; // ring depth: as many 8 KB stages as fit
                               // beside the elements at 2 CTAs per SM
constexpr int kStageBytes = 8 * 1024;
constexpr int kElemSmemMax = 128 * 1024;  // resident element budget
constexpr int kSmemPerSm = 227 * 1024;

// dimensions per ring stage (8 KB of V): exactly d_pad = round_up(d, 8)
// dimensions are streamed (no dead FMAs on padding chunks).  2-byte
// storage-typed V (EXEM_VT_STORAGE): the HBM-bound layouts (EG <= 2) carry
// 16 dimensions per 8 KB stage -- when d_pad is an odd multiple of 8 the
// last box reads 8 rows past d_pad (TMA zero fill, still a full box of
// transaction bytes) that the kernel skips; 4 KB stages of 8 dimensions ran
// at the f32 kernel's stage rate (k = 1: 0.090 ms for half the bytes).  The
// FMA-bound layouts (EG >= 4) keep 8 dimensions in 4 KB stages (16 measured
// 12-19 % slower at k = 50 / 64).
template <typename V, int EG> constexpr int bk_of() {
  return (sizeof(V) == 2 && EG >= 4) ? 8
                                     : kStageBytes / (kP * (int)sizeof(V));
}
template <typename V, int EG> constexpr int stage_bytes() {
  return bk_of<V, EG>() * kP * (int)sizeof(V);
}

// PT consecutive storage-typed points of one dimension, widened (one
// 4/8/16-byte shared load per 2/4/8 points)
template <typename V, int PT, typename C>
__device__ __forceinline__ void load_pts(const V *p, C (&pv)[PT]) {
  constexpr int bytes = PT * (int)sizeof(V);
  if constexpr (bytes == 2) {
    pv[0] = to_c(p[0]);
  } else if constexpr (bytes == 4) {
    const uint32_t raw = *reinterpret_cast<const uint32_t *>(p);
    const V *q = reinterpret_cast<const V *>(&raw);
#pragma unroll
    for (int w = 0; w < PT; ++w) pv[w] = to_c(q[w]);
  } else if constexpr (bytes == 8) {
    const uint2 raw = *reinterpret_cast<const uint2 *>(p);
    const V *q = reinterpret_cast<const V *>(&raw);
#pragma unroll
    for (int w = 0; w < PT; ++w) pv[w] = to_c(q[w]);
  } else {
    constexpr int per = 16 / (int)sizeof(V);
#pragma unroll
    for (int u = 0; u < PT; u += per) {
      const uint4 raw = *reinterpret_cast<const uint4 *>(p + u);
      const V *q = reinterpret_cast<const V *>(&raw);
#pragma unroll
      for (int w = 0; w < per; ++w) pv[u + w] = to_c(q[w]);
    }
  }
}

template <typename C> struct Vec4;
template <> struct Vec4<float> {
  using T = float4;
};
template <> struct Vec4<double> {
  using T = double2;  // two values per 16-byte load
};

constexpr int kWarps = kThreads / 32;

// (C) x, computed no earlier than `dep` is available: keeps the compiler
// from converting a prefetched norm right after its load (which would stall
// the warp on the load at the top of the tile instead of in the epilogue)
template <typename C> __device__ __forceinline__ C late_cast(double x, C dep);
template <> __device__ __forceinline__ float late_cast(double x, float dep) {
  float r;
  asm volatile("{\n\t.reg .f32 t;\n\tmov.f32 t, %2;\n\tcvt.rn.f32.f64 %0, %1;\n\t}"
               : "=f"(r) : "d"(x), "f"(dep));
  return r;
}
template <> __device__ __forceinline__ double late_cast(double x, double) {
  return x;
}

// partials[tile] = xor tree over the kWarps warp sums of tile iteration tt
// (block_sum<256>'s second stage, bit for bit); run by one whole warp
__device__ __forceinline__ void combine_tile(double (&wsum)[2][kWarps],
                                             uint64_t (&wfull)[2],
                                             uint64_t (&wempty)[2],
                                             int64_t tt, int64_t tile,
                                             double *partials, int lane) {
  const int slot = (int)(tt & 1);
  const uint32_t use = (uint32_t)(tt >> 1);
  if (lane == 0) tc::mbar_wait(&wfull[slot], use & 1);
  __syncwarp();
  double r = lane < kWarps ? wsum[slot][lane] : 0.0;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) r += __shfl_xor_sync(0xffffffffu, r, o);
  __syncwarp();
  if (lane == 0) {
    partials[tile] = r;
    tc::mbar_arrive(&wempty[slot]);
  }
}

// Thread layout: EG lanes share a point group of PT = EG points; each lane
// owns ET <= 8 consecutive elements (e = g0 + eg*ET + j), so a group covers
// KG = EG*ET elements with no dead element columns for any k (k = 10:
// EG = 2, ET = 5).  Elements live in smem as [dim][EG][8] (8-wide rows).
// CTAs per SM: each CTA's ring is one serial refill chain, so the
// HBM-bound shapes (few elements per lane) want more of them (k = 1 at 2
// CTAs/SM: 0.107 ms, at 4: 0.084 ms); the register budget follows.
template <int EG>
constexpr int min_ctas() { return EG == 1 ? 4 : (EG == 2 ? 3 : 2); }

template <int DT, int EG, int ET, bool VS>
__global__ void __launch_bounds__(kThreads, min_ctas<EG>())
    set_min_tma_kernel(const __grid_constant__ CUtensorMap vmap,
                       int64_t n, int d_pad, int nstages,
                       const double *__restrict__ norms,
                       const typename Traits<DT>::C *__restrict__ aux,
                       const typename Traits<DT>::C *__restrict__ elems,
                       const double *__restrict__ enorms, int k,
                       int include_aux,
                       typename Traits<DT>::C *__restrict__ t_out,
                       int64_t *__restrict__ label_out,
                       double *__restrict__ partials,
                       typename Traits<DT>::C *__restrict__ dist_out,
                       int64_t ldd) {
  using C = typename Traits<DT>::C;
  using VT = typename VtOf<DT, VS>::T;  // element type of the V stages
  constexpr int BK = bk_of<VT, EG>();
  constexpr int PT = EG;              // points per thread
  constexpr int KG = EG * ET;         // elements per group
  constexpr int ROW = EG * 8;         // smem values per dimension
  constexpr int STAGE = BK * kP;      // values per V stage
  constexpr int kUnrollKK = EG >= 4 ? kUnrollWide : BK;
  // HBM-bound shapes: fetch norms / aux of the tile before its chunk loop
  constexpr bool kPrefetch = PT <= 4;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  VT *sv = reinterpret_cast<VT *>(smem_raw);        // [S][BK][kP]
  C *se = reinterpret_cast<C *>(sv + nstages * STAGE);  // [d_pad][EG][8]
  __shared__ __align__(8) uint64_t full[kMaxStages];
  __shared__ uint32_t rel[kMaxStages];  // warps done with a stage's use
  __shared__ __align__(8) uint64_t wfull[2], wempty[2];
  __shared__ double wsum[2][kWarps];
  __shared__ double s_en[KG];

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int eg = lane & (EG - 1);
  const int pg = warp * (32 / EG) + lane / EG;
  const int64_t tiles = (n + kP - 1) / kP;
  const int64_t my_tiles =
      blockIdx.x < tiles ? (tiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const int nchunks = (d_pad + BK - 1) / BK;

  if (threadIdx.x == 0) {
    for (int s = 0; s < nstages; ++s) {
      tc::mbar_init(&full[s], 1);
      rel[s] = 0;
    }
    for (int s = 0; s < 2; ++s) {
      tc::mbar_init(&wfull[s], kWarps);
      tc::mbar_init(&wempty[s], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  uint32_t ev_use = 0;  // events: (group, tile, chunk)
  const int64_t groups = (k + KG - 1) / KG;
  const uint32_t total = (uint32_t)(groups * my_tiles * nchunks);
  // Self-refilling ring: event ev's box goes to stage ev % S.  There is no
  // producer role: the LAST warp to finish with a stage (a shared-memory
  // counter) issues that stage's next event, so a refill is never late
  // behind a busy producing warp.
  auto issue = [&](uint32_t ev) {
    const int s = ev % nstages;
    const uint32_t within = ev % (uint32_t)(my_tiles * nchunks);
    const int64_t tile = blockIdx.x + (int64_t)(within / nchunks) * gridDim.x;
    const int c = (int)(within % nchunks);
    tc::mbar_expect_tx(&full[s], (uint32_t)(STAGE * sizeof(VT)));
    tc::tma_load_2d(sv + s * STAGE, &vmap, &full[s], (int)(tile * kP), c * BK);
  };
  if (threadIdx.x == 0)
    for (uint32_t ev = 0; ev < total && ev < (uint32_t)nstages; ++ev)
      issue(ev);

  for (int64_t g = 0; g < groups; ++g) {
    const int g0 = (int)(g * KG);
    const bool last = g + 1 == groups;
    // resident element group (zero past k and in the ET..7 pad columns)
    __syncthreads();  // previous group's elements are no longer read
    for (int x = threadIdx.x; x < d_pad * ROW; x += kThreads) {
      const int dim = x / ROW, r = x % ROW, e = (r >> 3) * ET + (r & 7);
      se[x] = ((r & 7) < ET && g0 + e < k)
                  ? elems[(int64_t)(g0 + e) * d_pad + dim] : C(0);
    }
    for (int e = threadIdx.x; e < KG; e += kThreads)
      s_en[e] = g0 + e < k ? enorms[g0 + e] : 0.0;
    __syncthreads();

    for (int64_t tt = 0; tt < my_tiles; ++tt) {
      const int64_t tile = blockIdx.x + tt * gridDim.x;
      const int64_t i0 = tile * kP + pg * PT;
      double nrm[PT];
      C ax[PT];
      if constexpr (kPrefetch) {
#pragma unroll
        for (int p = 0; p < PT; ++p) {
          const bool ok = i0 + p < n;
          nrm[p] = ok ? norms[i0 + p] : 0.0;
          ax[p] = (ok && include_aux) ? aux[i0 + p] : C(0);
        }
      }
      C acc[PT][ET];
#pragma unroll
      for (int p = 0; p < PT; ++p)
#pragma unroll
        for (int j = 0; j < ET; ++j) acc[p][j] = C(0);
      for (int c = 0; c < nchunks; ++c, ++ev_use) {
        const int s = ev_use % nstages;
        // suspend in hardware until the box lands (a spin loop's
        // SYNCS/BRA/ISETP/YIELD were ~15 % of the issued instructions)
        tc::mbar_wait_hint(&full[s], (ev_use / nstages) & 1);
        const VT *cv = sv + s * STAGE + pg * PT;
        const C *ce = se + (c * BK) * ROW + eg * 8;
        auto dim_step = [&](int kk) {
          C pv[PT], ev[8];
          using V4 = typename Vec4<C>::T;
          constexpr int per = 16 / sizeof(C);
          if constexpr (VS) {
            load_pts<VT, PT, C>(cv + kk * kP, pv);
          } else if constexpr (PT == 1) {
            pv[0] = cv[kk * kP];
          } else if constexpr (PT * sizeof(C) == 8) {
            const float2 q = *reinterpret_cast<const float2 *>(cv + kk * kP);
            pv[0] = q.x; pv[1] = q.y;
          } else {
#pragma unroll
            for (int u = 0; u < PT; u += per) {
              const V4 q = *reinterpret_cast<const V4 *>(cv + kk * kP + u);
              const C *qc = reinterpret_cast<const C *>(&q);
#pragma unroll
              for (int w = 0; w < per; ++w) pv[u + w] = qc[w];
            }
          }
#pragma unroll
          for (int u = 0; u < ET; u += per) {
            const V4 q = *reinterpret_cast<const V4 *>(ce + kk * ROW + u);
            const C *qc = reinterpret_cast<const C *>(&q);
#pragma unroll
            for (int w = 0; w < per; ++w) ev[u + w] = qc[w];
          }
#pragma unroll
          for (int p = 0; p < PT; ++p) {
#ifndef EXEM_K2_NO_FFMA2
            // binary32 compute: element pairs through FFMA2 (/ FADD2) with
            // the point as the broadcast operand -- per lane the same IEEE
            // fma / sub as the scalar form (bit-identical), half the issues
            constexpr int JP = sizeof(C) == 4 ? (ET & ~1) : 0;
            if constexpr (JP > 0) {
              const float2 pp = make_float2(pv[p], pv[p]);
#pragma unroll
              for (int j = 0; j < JP; j += 2) {
                float2 t = make_float2(acc[p][j], acc[p][j + 1]);
                if constexpr (Traits<DT>::kDirect) {
                  const float2 df =
                      __fadd2_rn(pp, make_float2(-ev[j], -ev[j + 1]));
                  t = __ffma2_rn(df, df, t);
                } else {
                  t = __ffma2_rn(pp, make_float2(ev[j], ev[j + 1]), t);
                }
                acc[p][j] = t.x;
                acc[p][j + 1] = t.y;
              }
            }
#else
            constexpr int JP = 0;
#endif
#pragma unroll
            for (int j = JP; j < ET; ++j) {
              if constexpr (Traits<DT>::kDirect) {
                const C df = pv[p] - ev[j];
                acc[p][j] = fma(df, df, acc[p][j]);
              } else {
                acc[p][j] = fma(pv[p], ev[j], acc[p][j]);
              }
            }
          }
        };
        if constexpr (BK == 16) {  // 2-byte V: 8 dims, then 8 more unless tail
#pragma unroll
          for (int kk = 0; kk < 8; ++kk) dim_step(kk);
          if (c * BK + 8 < d_pad) {
#pragma unroll
            for (int kk = 8; kk < 16; ++kk) dim_step(kk);
          }
        } else {
#pragma unroll(kUnrollKK)
          for (int kk = 0; kk < BK; ++kk) dim_step(kk);
        }
        __syncwarp();  // every lane's reads of the stage are consumed
        if (lane == 0) {
#ifndef EXEM_K2_NOFENCE
          __threadfence_block();
#endif
          if (atomicAdd(&rel[s], 1u) == (uint32_t)kWarps - 1) {
            rel[s] = 0;  // no other warp touches it before the refill lands
            const uint32_t nev = ev_use + (uint32_t)nstages;
            if (nev < total) {
              asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
              issue(nev);
            }
          }
        }
      }
      // epilogue: distances, first minimum per point within the thread
      // (ascending element index), then across the EG lanes of the point
      // group (lower index on ties); every lane of the group ends with it
      C t[PT];
      int64_t lab[PT];
#pragma unroll
      for (int p = 0; p < PT; ++p) {
        const int64_t i = i0 + p;
        if constexpr (!kPrefetch) {
          nrm[p] = i < n ? norms[i] : 0.0;
          ax[p] = (i < n && include_aux) ? aux[i] : C(0);
        }
        const C ai = late_cast<C>(nrm[p], acc[p][0]);
        C best = tinf<C>();
        int lb = 0;
#pragma unroll
        for (int j = 0; j < ET; ++j) {
          const int el = eg * ET + j;
          const int e = g0 + el;
          if (e < k && i < n) {
            const C dist = Traits<DT>::kDirect
                               ? acc[p][j]
                               : gemm_form<C>(acc[p][j], ai, (C)s_en[el]);
            if (dist_out) dist_out[(int64_t)e * ldd + i] = dist;
            if (dist < best) {
              best = dist;
              lb = e;
            }
          }
        }
#pragma unroll
        for (int o = 1; o < EG; o <<= 1) {
          const C ob = __shfl_xor_sync(0xffffffffu, best, o);
          const int ol = __shfl_xor_sync(0xffffffffu, lb, o);
          if (ob < best || (ob == best && ol < lb)) {
            best = ob;
            lb = ol;
          }
        }
        t[p] = best;
        lab[p] = lb;
        // running minimum across element groups (k > KG) is carried in
        // t_out / label_out (the same lanes own the point in every group)
        if (i < n && g > 0) {
          const C prev = t_out[i];
          if (!(t[p] < prev)) {  // earlier group wins ties (lower index)
            t[p] = prev;
            lab[p] = label_out ? label_out[i] : 0;
          }
        }
        if (last && include_aux && i < n) t[p] = tmin(t[p], ax[p]);
        if (eg == 0 && i < n && (!last || t_out)) t_out[i] = t[p];
        if (eg == 0 && i < n && label_out) label_out[i] = lab[p];
      }
      if (last) {
        // The canonical per-256-point block partial (block_sum<256> of the
        // other K1/K2 kernels: lane c of warp w holds point 32w + c, xor
        // tree in the warp, then an xor tree over the 8 warp sums) without
        // a CTA-wide barrier per tile: the warps deposit their sums in a
        // two-slot ring and the last warp combines tile tt-1 one tile later.
        C mine = C(0);
#pragma unroll
        for (int p = 0; p < PT; ++p) {
          const C v = __shfl_sync(0xffffffffu, t[p], (lane / PT) * EG);
          if (lane % PT == p) mine = v;
        }
        const int64_t ic = tile * kP + warp * 32 + lane;
        double v = ic < n ? (double)mine : 0.0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        const int slot = (int)(tt & 1);
        const uint32_t use = (uint32_t)(tt >> 1);
        if (lane == 0) {
          if (use > 0) tc::mbar_wait(&wempty[slot], (use - 1) & 1);
          wsum[slot][warp] = v;
          tc::mbar_arrive(&wfull[slot]);
        }
        if (warp == kWarps - 1) {
          if (tt > 0) combine_tile(wsum, wfull, wempty, tt - 1, tile - gridDim.x,
                                   partials, lane);
          if (tt + 1 == my_tiles) combine_tile(wsum, wfull, wempty, tt, tile,
                                               partials, lane);
        }
      }
    }
  }
}

template <int DT, int EG, int ET, bool VS>
cudaError_t launch_t(const CUtensorMap &map, int64_t tiles, int sms,
                     cudaStream_t st, int64_t n, int d_pad,
                     const double *norms, const void *aux, const void *elems,
                     const double *enorms, int k, int include_aux,
                     void *t_out, int64_t *label_out, double *partials,
                     void *dist_out, int64_t ldd) {
  using C = typename Traits<DT>::C;
  using VT = typename VtOf<DT, VS>::T;
  constexpr size_t sb = (size_t)stage_bytes<VT, EG>();
  const size_t elem_bytes = (size_t)d_pad * EG * 8 * sizeof(C);
  // 8 KB stages: 5 / 6 / 8 per CTA at 4 / 3 / 2 CTAs per SM (about
  // 130-170 KB in flight per SM); deeper rings with fewer CTAs measured
  // slower (13 stages at 2 CTAs: 0.150 vs 0.084 ms at k = 1).  4 KB stages
  // (2-byte V, EG >= 4) keep the bytes in flight with twice the count.
  int nst = EG == 1 ? 5 : (EG == 2 ? 6 : 8);
  if (sb < (size_t)kStageBytes) nst = nst * 2 > kMaxStages ? kMaxStages : nst * 2;
  size_t smem = (size_t)nst * sb + elem_bytes;
  while (smem + 4096 > (size_t)kSmemPerSm && nst > 2) {
    --nst;
    smem -= sb;
  }
  if (const char *ev = getenv("EXEM_K2_STAGES")) {  // timing experiments only
    const int want = atoi(ev);
    if (want >= 2 && want <= kMaxStages &&
        (size_t)want * sb + elem_bytes + 4096 <= (size_t)kSmemPerSm) {
      nst = want;
      smem = (size_t)nst * sb + elem_bytes;
    }
  }
  cudaError_t e = cudaFuncSetAttribute(
      set_min_tma_kernel<DT, EG, ET, VS>,
      cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int per_sm = 1;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(
          &per_sm, set_min_tma_kernel<DT, EG, ET, VS>, kThreads, smem) !=
          cudaSuccess || per_sm < 1)
    per_sm = 1;
  if (const char *ev = getenv("EXEM_K2_MAXCTA"))  // timing experiments only
    if (atoi(ev) >= 1 && atoi(ev) < per_sm) per_sm = atoi(ev);
  const int grid = (int)(tiles < (int64_t)per_sm * sms ? tiles
                                                       : (int64_t)per_sm * sms);
  set_min_tma_kernel<DT, EG, ET, VS><<<grid, kThreads, smem, st>>>(
      map, n, d_pad, nst, norms, (const C *)aux, (const C *)elems, enorms, k,
      include_aux, (C *)t_out, label_out, partials, (C *)dist_out, ldd);
  return cudaGetLastError();
}

int sm_count() {
  static int sms[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) return 148;
  if (!sms[dev]) cudaDeviceGetAttribute(&sms[dev], cudaDevAttrMultiProcessorCount, dev);
  return sms[dev] ? sms[dev] : 148;
}

// (EG, ET) for k elements: the fewest lanes per point whose 8-element rows
// cover k (EG <= 8, <= 4 at f64), then ET = ceil(k / EG).
void choose(int dtype, int k, int &eg, int &et, bool vs) {
  const int egmax = dtype == EXEM_F64 ? 4 : 8;
  eg = 1;
  while (eg < egmax && eg * 8 < k) eg *= 2;
  et = (k + eg - 1) / eg;
  if (et > 8) et = 8;  // several element groups
  // widened half storage (the streamed slots): 8-wide rows only; 2-byte
  // storage has the binary32 thread layouts (no dead element columns)
  if ((dtype == EXEM_F16 || dtype == EXEM_BF16) && !vs) et = 8;
  if (eg > 1 && et < 5) et = 5;  // instantiated ET range for EG > 1
}

// the TMA kernel runs this shape: the element group fits the resident
// budget and a multi-group set has its t_out carry
bool set_min_tma_covers(int dtype, int d_pad, int k, bool has_t_out, bool vs) {
  if (k < 1 || d_pad % 8 != 0) return false;
  const int eb = dtype == EXEM_F64 ? 8 : 4;  // resident elements: compute type
  int eg, et;
  choose(dtype, k, eg, et, vs);
  if (k > eg * et && !has_t_out) return false;
  return (size_t)d_pad * eg * 8 * eb <= (size_t)kElemSmemMax;
}

}  // namespace

int set_min_storage_ok(int dtype, int64_t d, int64_t k, int has_t_out) {
  const int tag = dtype & ~EXEM_VT_STORAGE;
  if (tag != EXEM_F16 && tag != EXEM_BF16) return 0;
  if (k < 1 || k > (1 << 30) || d < 1) return 0;
  if (!tc::get_encode()) return 0;
  return set_min_tma_covers(tag, (int)round_up(d, kDimPad), (int)k,
                            has_t_out != 0, true) ? 1 : 0;
}

// Returns 1 if the shape is not covered (caller uses the cp.async K2),
// 0 on launch, or a negative CUDA error.  k > EG*ET runs several element
// groups (the running minimum goes through t_out, which must be non-null).
int set_min_tma(int dtype, const void *vt, int64_t ld, int64_t n, int d_pad,
                const double *norms, const void *aux, const void *elems,
                const double *enorms, int k, int include_aux, void *t_out,
                int64_t *label_out, double *partials, void *dist_out,
                int64_t ldd, cudaStream_t st) {
  const bool vs = (dtype & EXEM_VT_STORAGE) != 0;
  dtype &= ~EXEM_VT_STORAGE;
  if (vs && dtype != EXEM_F16 && dtype != EXEM_BF16) return 1;
  if (k < 1 || n < 1 || ld % kP != 0) return 1;
  if (!set_min_tma_covers(dtype, d_pad, k, t_out != nullptr, vs)) return 1;
  const bool f64 = dtype == EXEM_F64;
  const int vb = f64 ? 8 : (vs ? 2 : 4);  // bytes per V value
  int eg, et;
  choose(dtype, k, eg, et, vs);
  const int bk = f64 ? bk_of<double, 1>()
                     : (!vs ? bk_of<float, 1>()
                            : (eg >= 4 ? bk_of<__half, 4>() : bk_of<__half, 1>()));
  CUtensorMap map;
  auto enc = tc::get_encode();
  if (!enc) return 1;
  cuuint64_t gdim[2] = {(cuuint64_t)ld, (cuuint64_t)d_pad};
  cuuint64_t gstride[1] = {(cuuint64_t)(ld * vb)};
  cuuint32_t box[2] = {(cuuint32_t)kP, (cuuint32_t)bk};
  cuuint32_t estr[2] = {1, 1};
  const CUtensorMapDataType tdt =
      f64 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64
          : (!vs ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32
                 : (dtype == EXEM_BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16
                                       : CU_TENSOR_MAP_DATA_TYPE_FLOAT16));
  CUresult r = enc(&map, tdt,
                   2, const_cast<void *>(vt), gdim, gstride, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                   getenv("EXEM_K2_L2P0") ? CU_TENSOR_MAP_L2_PROMOTION_NONE
                                          : CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return 1;
  const int64_t tiles = ceil_div(n, kP);
  const int sms = sm_count();
  cudaError_t e = cudaErrorInvalidValue;
#define EXEM_SMTV(DTV, EGV, ETV, VSV)                                        \
  if (eg == EGV && et == ETV && vs == VSV)                                   \
  e = launch_t<DTV, EGV, ETV, VSV>(map, tiles, sms, st, n, d_pad, norms,    \
                                   aux, elems, enorms, k, include_aux,      \
                                   t_out, label_out, partials, dist_out,    \
                                   ldd)
#define EXEM_SMT(DTV, EGV, ETV) EXEM_SMTV(DTV, EGV, ETV, false)
#define EXEM_SMT_HALF(DTV, EGV) EXEM_SMTV(DTV, EGV, 8, false)
#define EXEM_SMTS_WIDE(DTV, EGV)                                             \
  EXEM_SMTV(DTV, EGV, 5, true); EXEM_SMTV(DTV, EGV, 6, true);               \
  EXEM_SMTV(DTV, EGV, 7, true); EXEM_SMTV(DTV, EGV, 8, true)
#define EXEM_SMTS_ONE(DTV)                                                   \
  EXEM_SMTV(DTV, 1, 1, true); EXEM_SMTV(DTV, 1, 2, true);                   \
  EXEM_SMTV(DTV, 1, 3, true); EXEM_SMTV(DTV, 1, 4, true);                   \
  EXEM_SMTV(DTV, 1, 5, true); EXEM_SMTV(DTV, 1, 6, true);                   \
  EXEM_SMTV(DTV, 1, 7, true); EXEM_SMTV(DTV, 1, 8, true)
#define EXEM_SMT_WIDE(DTV, EGV)                                              \
  EXEM_SMT(DTV, EGV, 5); EXEM_SMT(DTV, EGV, 6); EXEM_SMT(DTV, EGV, 7);      \
  EXEM_SMT(DTV, EGV, 8)
#define EXEM_SMT_ONE(DTV)                                                    \
  EXEM_SMT(DTV, 1, 1); EXEM_SMT(DTV, 1, 2); EXEM_SMT(DTV, 1, 3);            \
  EXEM_SMT(DTV, 1, 4); EXEM_SMT(DTV, 1, 5); EXEM_SMT(DTV, 1, 6);            \
  EXEM_SMT(DTV, 1, 7); EXEM_SMT(DTV, 1, 8)
  switch (dtype) {
    case EXEM_F64:
      EXEM_SMT_ONE(EXEM_F64);
      EXEM_SMT_WIDE(EXEM_F64, 2);
      EXEM_SMT_WIDE(EXEM_F64, 4);
      break;
    case EXEM_F32:
      EXEM_SMT_ONE(EXEM_F32);
      EXEM_SMT_WIDE(EXEM_F32, 2);
      EXEM_SMT_WIDE(EXEM_F32, 4);
      EXEM_SMT_WIDE(EXEM_F32, 8);
      break;
    case EXEM_F16:
      EXEM_SMT_HALF(EXEM_F16, 1); EXEM_SMT_HALF(EXEM_F16, 2);
      EXEM_SMT_HALF(EXEM_F16, 4); EXEM_SMT_HALF(EXEM_F16, 8);
      EXEM_SMTS_ONE(EXEM_F16);
      EXEM_SMTS_WIDE(EXEM_F16, 2); EXEM_SMTS_WIDE(EXEM_F16, 4);
      EXEM_SMTS_WIDE(EXEM_F16, 8);
      break;
    case EXEM_BF16:
      EXEM_SMT_HALF(EXEM_BF16, 1); EXEM_SMT_HALF(EXEM_BF16, 2);
      EXEM_SMT_HALF(EXEM_BF16, 4); EXEM_SMT_HALF(EXEM_BF16, 8);
      EXEM_SMTS_ONE(EXEM_BF16);
      EXEM_SMTS_WIDE(EXEM_BF16, 2); EXEM_SMTS_WIDE(EXEM_BF16, 4);
      EXEM_SMTS_WIDE(EXEM_BF16, 8);
      break;
    default:
      return 1;
  }
#undef EXEM_SMT_HALF
#undef EXEM_SMTS_WIDE
#undef EXEM_SMTS_ONE
#undef EXEM_SMTV
#undef EXEM_SMT_ONE
#undef EXEM_SMT_WIDE
#undef EXEM_SMT
  return e == cudaSuccess ? 0 : -(int)e;
}

}  // namespace exem
