// exem_tc_batch.cu -- K4-TC: tcgen05 evaluation of a batch of EXPLICIT sets
// (the paper's S_multi) at bf16/f16, sm_100a only.
//
// Replaces evaluate_batch / _reference_eval / tiled_evaluate over the packed
// round-robin batch, pkg/src/exembatch/evaluate.py:142-149,197-270 and
// core.py:331-346, for binary16/bfloat16 storage:
//
//   partial[split][j] = sum_{i in split} min(aux_i, min_{e<card_j} d(v_i, S_j[e]))
//
// One MMA row-dot gives D[i][e] = v_i.e - a_i/2 - b_e/2 = -d(v_i, e)/2 with
//   point rows    y_i = [v_i, -h_hi,-h_mid,-h_lo, 1,1,1, 0..]   h = ||v_i||^2/2
//   element rows  x_e = [e,   1,1,1, -b_hi,-b_mid,-b_lo, 0..]  b = ||e||^2/2
// (the K3 operand formats with m = 0; constants split into three half
// pieces, ~24-bit fidelity).  So min_e d = -2 max_e D: the epilogue is a
// per-set max over that set's TMEM columns, then min with aux, then a sum.
//
// Operand roles: points on M (TMEM lanes, streamed by TMA per K chunk),
// set elements on N (the "set tile", stationary in smem for a work item).
// A set tile holds `spt` whole sets, each padded to `w` = round_up(k_max, 8)
// columns; blank slots (e >= card_j) and padding columns are copies of the
// set's element 0, so they never change a minimum and need no masking
// (cf. the blank-slot rule, core.py:227-230).
//
// Roles (320 threads, 1 CTA/SM, persistent over (split, set tile) items):
//   warp 0      TMA producer (set tile once per item; point K-chunks
//               through a `stages`-deep ring)
//   warp 1      TMEM allocator + single-thread MMA issuer (M=128 x
//               N=ncols x K=16), handshakes software-pipelined one chunk
//               ahead so the tensor pipe's ~2-deep queue never drains
//   warps 2-9   epilogue: lane quarter q = warp%4 (TMEM lane access rule),
//               set parity h = (warp-2)/4; per-thread fp64 running sums per
//               set across the item's point tiles, fixed-order xor-shuffle +
//               cross-quarter reduction at item end (deterministic).
#include <cstdlib>

#include "exem_tc_common.cuh"

namespace exem {
namespace tcb {

using namespace exem::tc;

constexpr int BM = 128;                 // points per tile (TMEM lanes)
constexpr int A_CHUNK = BM * 128;       // bytes of one point K-chunk
constexpr int kThreads = 320;
constexpr int kEpiWarps = 8;
constexpr int kMaxSpt = 16;             // sets per set tile (register budget of the epilogue)
constexpr int kSmemBudget = 227 * 1024;
constexpr int kBarBytes = 3072;  // barriers, reductions, plain b
constexpr int kTrace = 256;  // tiles traced on CTA 0
// CTA-0 timeline for timing experiments (tools/tcb_trace.py): compiled in
// only with -DEXEM_TCB_TRACE_BUILD (EXEM_NVCC_FLAGS at build time) -- the
// extra live registers would otherwise spill in the epilogue.
#ifdef EXEM_TCB_TRACE_BUILD
#define TRB(slot, t)                                                       \
  do {                                                                     \
    if (p.trace != nullptr && blockIdx.x == 0 && (t) < kTrace)             \
      p.trace[(slot) * kTrace + (t)] = clock64();                          \
  } while (0)
#else
#define TRB(slot, t) \
  do {               \
  } while (0)
#endif

struct BParams {
  int64_t n;           // points of this slice
  int64_t l;           // sets
  int64_t split_pts;   // points per split (multiple of BM)
  int64_t splits;
  int64_t set_tiles;
  int spt;             // sets per set tile
  int w;               // TMEM columns per set (multiple of 8)
  int ncols;           // MMA N (multiple of 16, >= spt * w)
  int ksteps;          // K=16 MMA steps
  int kchunks;         // 64-wide K chunks per operand row
  int stages;          // point-chunk ring depth
  int bstream;         // 1: set chunks streamed with the point chunks
  int tstage;          // 1: a ring stage holds a whole point tile (all K)
  int gch;             // otherwise: 64-wide K chunks per ring stage (1, 2)
  int dbg;             // timing experiments only (EXEM_TCB_DEBUG), 0 in use
  uint32_t idesc;
  long long *trace;    // timing experiments only (EXEM_TCB_TRACE): CTA-0 timeline
  const float *aux;    // [n] aux distances (compute type)
  int plain;           // 1: unfolded operands, constants added in the epilogue
  const double *norms; // plain: [n] ||v_i||^2
  const float *bs;     // plain: [set rows] ||e||^2 / 2 per set-tile row
  double *partial;     // [splits][l]
};

__device__ __forceinline__ float max8(const uint32_t (&r)[8], float m) {
#pragma unroll
  for (int j = 0; j < 8; ++j) m = fmaxf(m, __uint_as_float(r[j]));
  return m;
}

// Release an accumulator buffer once every lane's tcgen05.ld is complete:
// on this CTA's tempty (CG = 1) or on the pair leader's (CG = 2).
template <int CG>
struct TmemRelease {
  uint64_t *bar;
  int lane;
  __device__ __forceinline__ void operator()() const {
    fence_before();
    __syncwarp();
    if (lane == 0) {
      if constexpr (CG == 2)
        mbar_arrive_cluster(mapa(bar, 0));
      else
        mbar_arrive(bar);
    }
  }
};

// Epilogue of one accumulator tile for one warp, set width W8*8 columns known
// at compile time.  The warp owns sets s = h + 2u (u < nsets); their columns
// are drained with tcgen05.ld x8 into registers in batches of sets
// (EpiShape) and ONE tcgen05.wait::ld per batch -- the TMEM load
// latency is paid once per tile, not once per 32 columns -- and the buffer is
// released right after the last batch's wait, before its arithmetic.
//   t = min(aux_i, max(0, -2 max_e D)),  acc[u] += t   (fp64, per thread)
template <int W8>
struct EpiShape {
  static constexpr int SPT = 32 / W8 < kMaxSpt ? 32 / W8 : kMaxSpt;
  static constexpr int MAXS = (SPT + 1) / 2;  // sets per warp (max)
  // sets per load batch: registers of one batch (8 per group) plus the fp64
  // accumulators within a 116-register budget (ptxas caps this kernel at
  // 168 registers per thread)
  static constexpr int sb() {
    int best = 1;
    for (int s = 1; s <= MAXS; ++s)
      if (s * W8 * 8 + 2 * MAXS <= 116) best = s;
    return best;
  }
  static constexpr int SB = sb();
  static constexpr int NB = (MAXS + SB - 1) / SB;
};

// max over 8 columns of D - b[col] (plain operands: b = ||e||^2/2 of the
// column's element, from shared memory)
__device__ __forceinline__ float max8b(const uint32_t (&r)[8], const float *b,
                                       float m) {
#pragma unroll
  for (int j = 0; j < 8; ++j) m = fmaxf(m, __uint_as_float(r[j]) - b[j]);
  return m;
}

template <int W8, bool kPlain, typename Release>
__device__ __forceinline__ void epi_tile(
    uint32_t taddr, int h, int spt, int w, float ax, float ha, bool valid,
    const float *bsm, double (&acc)[EpiShape<W8>::MAXS],
    const Release &release) {
  const float ninf = -__int_as_float(0x7f800000);
  const int nsets = (spt - h + 1) >> 1;
  if (nsets <= 0) {
    release();
    return;
  }
  if constexpr (W8 * 8 + 2 * EpiShape<W8>::MAXS <= 116) {
    constexpr int SB = EpiShape<W8>::SB;
    constexpr int NB = EpiShape<W8>::NB;
    const int nbat = (nsets + SB - 1) / SB;
#pragma unroll
    for (int b = 0; b < NB; ++b) {
      if (b < nbat) {
        uint32_t r[SB * W8][8];
#pragma unroll
        for (int j = 0; j < SB; ++j) {
          if (b * SB + j < nsets) {
            const uint32_t c0 = taddr + (uint32_t)((h + 2 * (b * SB + j)) * w);
#pragma unroll
            for (int g = 0; g < W8; ++g) TMEM_LD8(c0 + 8 * g, r[j * W8 + g]);
          }
        }
        tmem_wait_ld();
        if (b == nbat - 1) release();
#pragma unroll
        for (int j = 0; j < SB; ++j) {
          if (b * SB + j < nsets) {
            float mx = ninf;
            const int cb = (h + 2 * (b * SB + j)) * w;  // set's first column
#pragma unroll
            for (int g = 0; g < W8; ++g)
              mx = kPlain ? max8b(r[j * W8 + g], bsm + cb + 8 * g, mx)
                          : max8(r[j * W8 + g], mx);
            // folded: min_e d = -2 max D;  plain: min_e d = a - 2 max (D - b)
            const float dm = kPlain ? fmaf(-2.f, mx, ha) : -2.f * mx;
            const float t = fminf(ax, fmaxf(0.f, dm));
            if (valid) acc[b * SB + j] += (double)t;
          }
        }
      }
    }
  } else {
    // w >= 120: at most one set per warp (set h); drain it in sub-batches of
    // 12 groups (96 registers) with a running max
    static_assert(EpiShape<W8>::MAXS == 1, "wide sets: one set per warp");
    constexpr int G = 12;
    constexpr int NS = (W8 + G - 1) / G;
    const uint32_t c0 = taddr + (uint32_t)(h * w);
    float mx = ninf;
#pragma unroll
    for (int sb = 0; sb < NS; ++sb) {
      uint32_t r[G][8];
#pragma unroll
      for (int g = 0; g < G; ++g)
        if (sb * G + g < W8) TMEM_LD8(c0 + 8 * (sb * G + g), r[g]);
      tmem_wait_ld();
      if (sb == NS - 1) release();
#pragma unroll
      for (int g = 0; g < G; ++g)
        if (sb * G + g < W8)
          mx = kPlain ? max8b(r[g], bsm + h * w + 8 * (sb * G + g), mx)
                      : max8(r[g], mx);
    }
    const float dm = kPlain ? fmaf(-2.f, mx, ha) : -2.f * mx;
    const float t = fminf(ax, fmaxf(0.f, dm));
    if (valid) acc[0] += (double)t;
  }
}

// The epilogue warps' whole loop for one set width (W8 = w/8 at compile
// time, so the per-set column runs and the accumulator array are static).
// CG = 2: this CTA holds rows [128*rank, 128*rank+128) of each 256-point
// pair tile; buffers are released on the leader's tempty, and at item end
// the peer's per-set sums travel to the leader through DSMEM (xbuf) so the
// leader writes one fixed-order partial per (split, set).
template <int CG, int W8, bool kPlain>
__device__ __forceinline__ void epilogue_role(const BParams &p, uint32_t tmem,
                                              uint64_t *tfull,
                                              uint64_t *tempty, double *red,
                                              double *xbuf, float *bsm,
                                              uint64_t *xfull,
                                              uint64_t *xempty, int warp,
                                              int lane, int64_t items,
                                              uint32_t rank, int64_t pair,
                                              int64_t npairs) {
  constexpr int MAXS = EpiShape<W8>::MAXS;
  const int ew = warp - 2;       // 0..7
  const int q = warp & 3;        // TMEM lane quarter (lane access rule)
  const int h = ew >> 2;         // set parity handled by this warp
  const int row = q * 32 + lane; // point row within this CTA's tile half
  uint32_t buf = 0, tph = 0, xph = 0;
#ifdef EXEM_TCB_TRACE_BUILD
  int etile = 0;
  const bool tr = warp == 2 && lane == 0;
#endif
  for (int64_t it = pair; it < items; it += npairs) {
    const int64_t st = it % p.set_tiles, sp = it / p.set_tiles;
    const int64_t p0 = sp * p.split_pts;
    const int64_t p1 = min(p.n, p0 + p.split_pts);
    double acc[MAXS];
#pragma unroll
    for (int u = 0; u < MAXS; ++u) acc[u] = 0.0;
    if constexpr (kPlain) {  // the set tile's column constants, once per item
      for (int c = ew * 32 + lane; c < p.ncols; c += kEpiWarps * 32)
        bsm[c] = p.bs[st * p.ncols + c];
      asm volatile("bar.sync 1, %0;" ::"n"(kEpiWarps * 32) : "memory");
    }
    for (int64_t pt = p0; pt < p1; pt += BM * CG) {
      const int64_t pi = pt + BM * rank + row;
      const bool valid = pi < p1;
      const float ax = (valid && !(p.dbg & 8)) ? p.aux[pi] : 0.f;
      const float ha = (kPlain && valid) ? (float)p.norms[pi] : 0.f;
      if (lane == 0) {
        mbar_wait_sleep(&tfull[buf], (tph >> buf) & 1u);
      }
      __syncwarp();
#ifdef EXEM_TCB_TRACE_BUILD
      if (tr) TRB(3, etile);
#endif
      tph ^= 1u << buf;
      fence_after();
      const uint32_t taddr =
          tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(buf * 256);
      TmemRelease<CG> rel{&tempty[buf], lane};
      if (p.dbg & 1)  // timing experiment: no TMEM drain / math
        rel();
      else
        epi_tile<W8, kPlain>(taddr, h, p.spt, p.w, ax, ha, valid, bsm, acc,
                             rel);
#ifdef EXEM_TCB_TRACE_BUILD
      if (tr) TRB(4, etile);
      ++etile;
#endif
      buf ^= 1u;
    }
    // item end: per set, fixed xor tree over the 32 lanes, then the four
    // lane quarters in order (then the pair's two CTAs in order)
#pragma unroll
    for (int u = 0; u < MAXS; ++u) {
      const int s = h + 2 * u;
      if (s < p.spt) {
        double v = acc[u];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (lane == 0) red[q * kMaxSpt + s] = v;
      }
    }
    asm volatile("bar.sync 1, %0;" ::"n"(kEpiWarps * 32) : "memory");
    if (ew == 0) {
      const bool mine = lane < p.spt;
      const double tot =
          mine ? ((red[lane] + red[kMaxSpt + lane]) + red[2 * kMaxSpt + lane]) +
                     red[3 * kMaxSpt + lane]
               : 0.0;
      const int64_t j = st * p.spt + lane;
      if constexpr (CG == 1) {
        if (mine && j < p.l) p.partial[sp * p.l + j] = tot;
      } else if (rank == 1) {
        if (lane == 0) mbar_wait_cluster(xempty, xph ^ 1u);
        __syncwarp();
        if (mine) {
          asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(
                           mapa(&xbuf[lane], 0)),
                       "d"(tot)
                       : "memory");
          asm volatile("fence.acq_rel.cluster;" ::: "memory");
        }
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(mapa(xfull, 0));
      } else {
        if (lane == 0) mbar_wait_cluster(xfull, xph);
        __syncwarp();
        if (mine && j < p.l) p.partial[sp * p.l + j] = tot + xbuf[lane];
        asm volatile("fence.acq_rel.cluster;" ::: "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(mapa(xempty, 1));
      }
      xph ^= 1u;
    }
    asm volatile("bar.sync 1, %0;" ::"n"(kEpiWarps * 32) : "memory");
  }
}

// Issuer loop of one work item with whole-tile point stages (one barrier
// handshake per tile, K3's scheme -- the per-chunk handshake costs ~200+
// cycles of mbarrier latency each, profiles/r01_k4_probe.log): KS K-steps
// unrolled at compile time, the next tile's point stage (full) acquired
// before MMA KS-2 and its accumulator buffer (tempty) before MMA KS-1.
template <int KS>
__device__ __forceinline__ void k4_item_tstage(
    const BParams &p, int ntiles, int &stage, uint32_t &ph, uint32_t &tph,
    uint32_t &buf, int &itile, uint64_t a_base, uint32_t a_step,
    uint64_t b_base, uint32_t b_step, uint32_t tmem, uint64_t *full,
    uint64_t *empty, uint64_t *tfull, uint64_t *tempty) {
  constexpr int WF = KS > 2 ? KS - 2 : 0;
  constexpr int WT = KS > 1 ? KS - 1 : 0;
  mbar_wait(&tempty[buf], ((tph >> buf) & 1u) ^ 1u);
  tph ^= 1u << buf;
  mbar_wait(&full[stage], ph);
  fence_after();
  for (int t = 0; t < ntiles; ++t) {
    const uint32_t d = tmem + buf * 256u;
    const uint64_t ad = a_base + (uint64_t)(stage * a_step);
    const uint32_t nbuf = buf ^ 1u;
    int nstage = stage + 1;
    uint32_t nph = ph;
    if (nstage == p.stages) {
      nstage = 0;
      nph ^= 1u;
    }
    const bool more = t + 1 < ntiles;
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) {
      if (ks == WF && more) {
        mbar_wait(&full[nstage], nph);
        fence_after();
      }
      if (ks == WT && more) {
        mbar_wait(&tempty[nbuf], ((tph >> nbuf) & 1u) ^ 1u);
        tph ^= 1u << nbuf;
        fence_after();
      }
      if (!(p.dbg & 2))
        umma_f16(d, ad + (uint64_t)((ks >> 2) * (A_CHUNK >> 4) + (ks & 3) * 2),
                 b_base + (uint64_t)((ks >> 2) * b_step + (ks & 3) * 2),
                 p.idesc, ks > 0 ? 1u : 0u);
    }
    umma_commit(&empty[stage]);
    umma_commit(&tfull[buf]);
    TRB(2, itile);
    ++itile;
    buf = nbuf;
    stage = nstage;
    ph = nph;
  }
}

// MMA j of an event whose stage holds consecutive 64-wide K chunks: chunk
// j>>2 of the event, K=16 step j&3 inside the 128-B swizzle row.
template <int CG>
__device__ __forceinline__ void issue_mma(const BParams &p, uint32_t d,
                                          uint64_t ad, uint64_t bd,
                                          uint32_t b_step, int kc, int j) {
  if (p.dbg & 2) return;  // timing experiment: no MMA
  const uint64_t a = ad + (uint64_t)((j >> 2) * (A_CHUNK >> 4) + (j & 3) * 2);
  const uint64_t b = bd + (uint64_t)((j >> 2) * b_step + (j & 3) * 2);
  if constexpr (CG == 2)
    umma_f16_pair(d, a, b, p.idesc, (kc | j) ? 1u : 0u);
  else
    umma_f16(d, a, b, p.idesc, (kc | j) ? 1u : 0u);
}

template <int CG>
__global__ void __launch_bounds__(kThreads, 1)
    batch_tc_kernel(const __grid_constant__ CUtensorMap map_p,
                    const __grid_constant__ CUtensorMap map_s,
                    const BParams p) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char *smem = (unsigned char *)(((uintptr_t)smem_raw + 1023) &
                                          ~(uintptr_t)1023);
  const int bh = p.ncols / CG;        // set-tile rows held by this CTA
  const int b_chunk = bh * 128;       // bytes of one set-tile K-chunk half
  const int sb_bytes = p.bstream ? 0 : p.kchunks * b_chunk;
  const int stage_bytes = p.tstage ? p.kchunks * A_CHUNK
                                   : p.gch * A_CHUNK + (p.bstream ? b_chunk : 0);
  unsigned char *sb = smem;                        // stationary set tile
  unsigned char *sa = smem + sb_bytes;             // point-chunk ring
  uint64_t *bars = (uint64_t *)(sa + p.stages * stage_bytes);
  uint64_t *full = bars;                           // [stages]
  uint64_t *empty = bars + p.stages;               // [stages]
  uint64_t *tfull = bars + 2 * p.stages;           // [2]
  uint64_t *tempty = tfull + 2;                    // [2]
  uint64_t *bfull = tempty + 2;                    // [1]
  uint64_t *bempty = bfull + 1;                    // [1]
  uint64_t *xfull = bempty + 1;                    // [1] pair exchange (CTA 0)
  uint64_t *xempty = xfull + 1;                    // [1] pair exchange (CTA 1)
  uint32_t *tmem_slot = (uint32_t *)(xempty + 1);
  double *red = (double *)(tmem_slot + 4);         // [4][kMaxSpt]
  double *xbuf = red + 4 * kMaxSpt;                // [kMaxSpt]
  float *bsm = (float *)(xbuf + kMaxSpt);          // [256] plain: set b

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = CG == 2 ? cluster_rank() : 0u;
  const int64_t pair = blockIdx.x / CG, npairs = gridDim.x / CG;
  if (warp == 0 && lane == 0) {
    for (int s = 0; s < p.stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], kEpiWarps * CG);
    }
    mbar_init(bfull, 1);
    mbar_init(bempty, 1);
    mbar_init(xfull, 1);
    mbar_init(xempty, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&map_p));
    asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&map_s));
  }
  if (warp == 1) {
    if constexpr (CG == 2) {
      asm volatile(
          "tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::
              "r"(su32(tmem_slot)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    } else {
      asm volatile(
          "tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::
              "r"(su32(tmem_slot)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
  }
  fence_before();
  __syncthreads();
  if constexpr (CG == 2) cluster_sync();
  fence_after();
  const uint32_t tmem = *tmem_slot;
  const int64_t items = p.set_tiles * p.splits;

  if (warp == 0) {
    // -------------------------------------------------------------- producer
    // Each CTA loads its own point rows and its half of the set tile; the
    // completions are counted on the leader's barriers (CG = 2).
    if (lane == 0) {
      int stage = 0, ptile = 0;
      uint32_t ph = 0, bph = 0;
      const uint32_t bfull_c = CG == 2 ? mapa(bfull, 0) : 0u;
      for (int64_t it = pair; it < items; it += npairs) {
        const int64_t st = it % p.set_tiles, sp = it / p.set_tiles;
        const int srow = (int)(st * p.ncols) + (int)rank * bh;
        if (!p.bstream) {
          mbar_wait_sleep(bempty, bph ^ 1);
          bph ^= 1;
          if (rank == 0) mbar_expect_tx(bfull, (uint32_t)(CG * sb_bytes));
          for (int kc = 0; kc < p.kchunks; ++kc) {
            if constexpr (CG == 2)
              tma_load_2d_pair(sb + kc * b_chunk, &map_s, bfull_c, kc * KCH, srow);
            else
              tma_load_2d(sb + kc * b_chunk, &map_s, bfull, kc * KCH, srow);
          }
        }
        const int64_t p0 = sp * p.split_pts;
        const int64_t p1 = min(p.n, p0 + p.split_pts);
        for (int64_t pt = p0; pt < p1 && p.tstage; pt += BM, ++ptile) {
          mbar_wait(&empty[stage], ph ^ 1);
          TRB(5, ptile);
          unsigned char *dst = sa + stage * stage_bytes;
          if (p.dbg & 4) {
            mbar_arrive(&full[stage]);
          } else {
            mbar_expect_tx(&full[stage], (uint32_t)stage_bytes);
            for (int kc = 0; kc < p.kchunks; ++kc)
              tma_load_2d(dst + kc * A_CHUNK, &map_p, &full[stage], kc * KCH,
                          (int)pt);
          }
          TRB(6, ptile);
          if (++stage == p.stages) {
            stage = 0;
            ph ^= 1;
          }
        }
        for (int64_t pt = p0; pt < p1 && !p.tstage; pt += BM * CG, ++ptile) {
          const int prow = (int)(pt + BM * rank);
          for (int kc = 0; kc < p.kchunks; kc += p.gch) {
            const int gn = p.kchunks - kc < p.gch ? p.kchunks - kc : p.gch;
            mbar_wait_sleep(&empty[stage], ph ^ 1);
            if (kc == 0) TRB(5, ptile);
            unsigned char *dst = sa + stage * stage_bytes;
            if (p.dbg & 4) {  // timing experiment: no point-operand traffic
              if (rank == 0) mbar_arrive(&full[stage]);
            } else {
              const uint32_t bytes =
                  (uint32_t)(gn * A_CHUNK + (p.bstream ? b_chunk : 0));
              if (rank == 0) mbar_expect_tx(&full[stage], (uint32_t)CG * bytes);
              if constexpr (CG == 2) {
                const uint32_t fc = mapa(&full[stage], 0);
                for (int j = 0; j < gn; ++j)
                  tma_load_2d_pair(dst + j * A_CHUNK, &map_p, fc,
                                   (kc + j) * KCH, prow);
                if (p.bstream)
                  tma_load_2d_pair(dst + A_CHUNK, &map_s, fc, kc * KCH, srow);
              } else {
                for (int j = 0; j < gn; ++j)
                  tma_load_2d(dst + j * A_CHUNK, &map_p, &full[stage],
                              (kc + j) * KCH, prow);
                if (p.bstream)
                  tma_load_2d(dst + A_CHUNK, &map_s, &full[stage], kc * KCH,
                              srow);
              }
            }
            if (kc + gn >= p.kchunks) TRB(6, ptile);
            if (++stage == p.stages) {
              stage = 0;
              ph ^= 1;
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    // (the leader CTA's single thread issues for the pair)
    if (lane == 0 && rank == 0) {
      const uint64_t a_base = sw128_desc(su32(sa));
      const uint64_t b_base = sw128_desc(su32(sb));
      const uint32_t a_step = (uint32_t)(stage_bytes >> 4);
      const uint32_t b_step = (uint32_t)(b_chunk >> 4);
      int stage = 0, itile = 0;
      uint32_t ph = 0, bph = 0, tph = 0, buf = 0;
      for (int64_t it = pair; it < items; it += npairs) {
        const int64_t sp = it / p.set_tiles;
        const int64_t p0 = sp * p.split_pts;
        const int64_t p1 = min(p.n, p0 + p.split_pts);
        const int ntiles = (int)((p1 - p0 + BM * CG - 1) / (BM * CG));
        const int kev = (p.kchunks + p.gch - 1) / p.gch;  // events per tile
        const int nev = ntiles * kev;
        if (!p.bstream) {
          mbar_wait(bfull, bph);
          bph ^= 1;
        }
        if constexpr (CG == 1) {
          if (p.tstage) {
            switch (p.ksteps) {
#define EXEM_K4_ITEM(K)                                                       \
  case K:                                                                     \
    k4_item_tstage<K>(p, ntiles, stage, ph, tph, buf, itile, a_base, a_step, \
                      b_base, b_step, tmem, full, empty, tfull, tempty);      \
    break;
              EXEM_K4_ITEM(1) EXEM_K4_ITEM(2) EXEM_K4_ITEM(3) EXEM_K4_ITEM(4)
              EXEM_K4_ITEM(5) EXEM_K4_ITEM(6) EXEM_K4_ITEM(7)
              default: EXEM_K4_ITEM(8)
#undef EXEM_K4_ITEM
            }
            umma_commit(bempty);
            continue;
          }
        }
        // acquire event 0 (accumulator buffer free + point chunk landed)
        mbar_wait(&tempty[buf], ((tph >> buf) & 1u) ^ 1u);
        TRB(0, itile);
        tph ^= 1u << buf;
        mbar_wait(&full[stage], ph);
        TRB(1, itile);
        fence_after();
        int kc = 0;
        for (int e = 0; e < nev; ++e) {
          const uint32_t d = tmem + buf * 256u;
          const uint64_t ad = a_base + (uint64_t)(stage * a_step);
          const uint64_t bd = p.bstream ? ad + (uint64_t)(A_CHUNK >> 4)
                                        : b_base + (uint64_t)(kc * b_step);
          const int rem = p.ksteps - kc * 4;
          const int nk = rem < 4 * p.gch ? rem : 4 * p.gch;
          // acquisitions for event e+1 (accumulator buffer when e+1 starts a
          // tile, then its point chunk) hide behind this chunk's last two
          // queued MMAs.  (Splitting them -- B stage before MMA nk-2, buffer
          // before nk-1, the better placement for K3 -- measured 1.5x
          // slower here: profiles/r01_k4_probe.log.)
          const int head = nk > 2 ? nk - 2 : 0;
          const bool last = (kc + p.gch >= p.kchunks);
          int nstage = stage + 1;
          uint32_t nph = ph;
          if (nstage == p.stages) {
            nstage = 0;
            nph ^= 1u;
          }
          const bool trc = kc == 1 || (p.kchunks == 1);
          if (trc) TRB(7, itile);
#pragma unroll 1
          for (int j = 0; j < head; ++j)
            issue_mma<CG>(p, d, ad, bd, b_step, kc, j);
          if (trc) TRB(8, itile);
          if (e + 1 < nev) {
            if (last) {
              const uint32_t nb = buf ^ 1u;
              mbar_wait(&tempty[nb], ((tph >> nb) & 1u) ^ 1u);
              TRB(0, itile + 1);
              tph ^= 1u << nb;
            }
            mbar_wait(&full[nstage], nph);
            if (last) TRB(1, itile + 1);
            // the tcgen05 fence orders the next MMAs' TMEM writes after the
            // epilogue's reads (tempty); smem data landed by TMA needs none
            if (last) fence_after();
          }
          if (trc) TRB(9, itile);
#pragma unroll 1
          for (int j = head; j < nk; ++j)
            issue_mma<CG>(p, d, ad, bd, b_step, kc, j);
          if (trc) TRB(10, itile);
          if constexpr (CG == 2) umma_commit_pair(&empty[stage]);
          else umma_commit(&empty[stage]);
          if (trc) TRB(11, itile);
          if (last) {
            if constexpr (CG == 2) umma_commit_pair(&tfull[buf]);
            else umma_commit(&tfull[buf]);
            TRB(2, itile);
            ++itile;
            buf ^= 1u;
            kc = 0;
          } else {
            kc += p.gch;
          }
          stage = nstage;
          ph = nph;
        }
        if (!p.bstream) {
          if constexpr (CG == 2) umma_commit_pair(bempty);
          else umma_commit(bempty);
        }
      }
    }
    __syncwarp();
  } else {
    // -------------------------------------------------------------- epilogue
    switch (p.w >> 3) {
#define EXEM_EPI_CASE(W)                                                     \
  case W:                                                                    \
    if (p.plain)                                                             \
      epilogue_role<CG, W, true>(p, tmem, tfull, tempty, red, xbuf, bsm,     \
                                 xfull, xempty, warp, lane, items, rank,     \
                                 pair, npairs);                              \
    else                                                                     \
      epilogue_role<CG, W, false>(p, tmem, tfull, tempty, red, xbuf, bsm,    \
                                  xfull, xempty, warp, lane, items, rank,    \
                                  pair, npairs);                             \
    break;
      EXEM_EPI_CASE(1) EXEM_EPI_CASE(2) EXEM_EPI_CASE(3) EXEM_EPI_CASE(4)
      EXEM_EPI_CASE(5) EXEM_EPI_CASE(6) EXEM_EPI_CASE(7) EXEM_EPI_CASE(8)
      EXEM_EPI_CASE(9) EXEM_EPI_CASE(10) EXEM_EPI_CASE(11) EXEM_EPI_CASE(12)
      EXEM_EPI_CASE(13) EXEM_EPI_CASE(14) EXEM_EPI_CASE(15) EXEM_EPI_CASE(16)
      EXEM_EPI_CASE(17) EXEM_EPI_CASE(18) EXEM_EPI_CASE(19) EXEM_EPI_CASE(20)
      EXEM_EPI_CASE(21) EXEM_EPI_CASE(22) EXEM_EPI_CASE(23) EXEM_EPI_CASE(24)
      EXEM_EPI_CASE(25) EXEM_EPI_CASE(26) EXEM_EPI_CASE(27) EXEM_EPI_CASE(28)
      EXEM_EPI_CASE(29) EXEM_EPI_CASE(30) EXEM_EPI_CASE(31) EXEM_EPI_CASE(32)
#undef EXEM_EPI_CASE
      default: break;
    }
  }

  fence_before();
  __syncthreads();
  if constexpr (CG == 2) cluster_sync();
  if (warp == 1) {
    fence_after();
    if constexpr (CG == 2)
      asm volatile(
          "tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem));
    else
      asm volatile(
          "tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

// ---------------------------------------------------------------- packing
// Set-tile operand rows from the packed round-robin batch
// packed[d_pad][k_max][l_pad] (compute type, packed_address order,
// core.py:320-328).  Row r = tile*ncols + s*w + e holds element
// (e < card_j ? e : 0) of set j = tile*spt + s, then the folded constants;
// rows of sets j >= l and padding columns past spt*w are zero.
template <int DT>
__global__ void pack_sets_kernel(const float *__restrict__ packed,
                                 const double *__restrict__ pnorms,
                                 const int32_t *__restrict__ card, int64_t l,
                                 int64_t l_pad, int k_max, int d, int spt,
                                 int w, int ncols, int64_t rows,
                                 typename Traits<DT>::S *__restrict__ x,
                                 int64_t kp, float *__restrict__ bs) {
  using S = typename Traits<DT>::S;
  const int64_t r = (int64_t)blockIdx.x * blockDim.y + threadIdx.y;
  if (r >= rows) return;
  const int64_t tile = r / ncols;
  const int c = (int)(r % ncols);
  const int s = c / w, e = c % w;
  const int64_t j = tile * spt + s;
  const bool real = s < spt && j < l;
  const int src = real ? (e < card[j] ? e : 0) : 0;
  const int64_t ldp = (int64_t)k_max * l_pad;
  if (bs != nullptr && threadIdx.x == 0)  // plain: the column's b = ||e||^2/2
    bs[r] = real ? (float)(0.5 * pnorms[(int64_t)src * l_pad + j]) : 0.f;
  for (int k = threadIdx.x; k < kp; k += blockDim.x) {
    double v = 0.0;
    if (real && (bs == nullptr || k < d)) {
      if (k < d) {
        v = (double)packed[(int64_t)k * ldp + (int64_t)src * l_pad + j];
      } else if (k < d + 3) {
        v = 1.0;
      } else if (k < d + kTcConst) {
        const double t = 0.5 * pnorms[(int64_t)src * l_pad + j];
        const double t0 = (double)to_c(from_d<S>(t));
        const double t1 = (double)to_c(from_d<S>(t - t0));
        const double t2 = (double)to_c(from_d<S>(t - t0 - t1));
        const int piece = k - d - 3;
        v = -(piece == 0 ? t0 : (piece == 1 ? t1 : t2));
      }
    }
    x[r * kp + k] = from_d<S>(v);
  }
}

// Plain point rows [v, 0..] (kp = round_up(d, 64)) for unfolded K4-TC.
template <int DT>
__global__ void pack_plain_kernel(const float *__restrict__ vt, int64_t ld,
                                  int64_t n, int d,
                                  typename Traits<DT>::S *__restrict__ x,
                                  int64_t kp, int64_t rows) {
  using S = typename Traits<DT>::S;
  __shared__ float tile[32][33];
  const int64_t r0 = (int64_t)blockIdx.x * 32;
  const int k0 = blockIdx.y * 32;
  for (int ty = threadIdx.y; ty < 32; ty += blockDim.y) {
    const int k = k0 + ty;
    const int64_t r = r0 + threadIdx.x;
    tile[ty][threadIdx.x] = (k < d && r < n) ? vt[(int64_t)k * ld + r] : 0.f;
  }
  __syncthreads();
  for (int ty = threadIdx.y; ty < 32; ty += blockDim.y) {
    const int64_t r = r0 + ty;
    const int k = k0 + threadIdx.x;
    if (r < rows && k < kp) x[r * kp + k] = from_d<S>((double)tile[threadIdx.x][ty]);
  }
}

}  // namespace tcb
}  // namespace exem

using namespace exem;

extern "C" {

int exem_tc_set_geometry(int64_t k_max, int32_t *spt, int32_t *w,
                         int32_t *ncols) {
  if (k_max < 1) return fail(EXEM_ERR_ARG, "k_max must be >= 1");
  const int64_t ww = round_up(k_max, 8);
  if (ww > 256)
    return fail(EXEM_ERR_UNSUPPORTED,
                "tcgen05 batch path holds a set in <= 256 TMEM columns "
                "(k_max=%lld)", (long long)k_max);
  int64_t s = 256 / ww;
  if (s > tcb::kMaxSpt) s = tcb::kMaxSpt;
  if (const char *e = getenv("EXEM_TCB_SPT")) {  // timing experiments only
    const int64_t f = atoll(e);
    if (f >= 1 && f < s) s = f;
  }
  *spt = (int32_t)s;
  *w = (int32_t)ww;
  *ncols = (int32_t)round_up(s * ww, 16);
  return EXEM_OK;
}

int64_t exem_tc_set_rows(int64_t l, int64_t k_max) {
  int32_t spt, w, nc;
  if (exem_tc_set_geometry(k_max, &spt, &w, &nc) != EXEM_OK) return -1;
  return ceil_div(l < 1 ? 1 : l, spt) * nc;
}

int64_t exem_tc_batch_plain(int64_t d) {
  // unfolded operands when folding the six constant columns would cost a
  // whole extra 64-wide K chunk (d = 59..64 mod 64, e.g. d = 256)
  return round_up(d, kTcKChunk) < exem_tc_kp(d) ? 1 : 0;
}

int64_t exem_tc_batch_kp(int64_t d) {
  return exem_tc_batch_plain(d) ? round_up(d, kTcKChunk) : exem_tc_kp(d);
}

int exem_tc_pack_points_plain(int dtype, const void *vt, int64_t ld,
                              int64_t n, int64_t d, void *xp, void *stream) {
  if (dtype != EXEM_BF16 && dtype != EXEM_F16)
    return fail(EXEM_ERR_ARG, "TC operands are bf16/f16 only");
  const int64_t kp = round_up(d, kTcKChunk), rows = exem_tc_rows(n);
  dim3 grid((unsigned)ceil_div(rows, 32), (unsigned)ceil_div(kp, 32));
  dim3 block(32, 8);
  cudaStream_t st = (cudaStream_t)stream;
  if (dtype == EXEM_BF16)
    tcb::pack_plain_kernel<EXEM_BF16><<<grid, block, 0, st>>>(
        (const float *)vt, ld, n, (int)d, (__nv_bfloat16 *)xp, kp, rows);
  else
    tcb::pack_plain_kernel<EXEM_F16><<<grid, block, 0, st>>>(
        (const float *)vt, ld, n, (int)d, (__half *)xp, kp, rows);
  EXEM_LAUNCH_CHECK("tc_pack_points_plain");
  return EXEM_OK;
}

int exem_tc_pack_sets(int dtype, const void *packed, const double *pnorms,
                      const int32_t *card, int64_t l, int64_t l_pad,
                      int64_t k_max, int64_t d, void *xs, float *bs,
                      void *stream) {
  if (dtype != EXEM_BF16 && dtype != EXEM_F16)
    return fail(EXEM_ERR_ARG, "TC operands are bf16/f16 only");
  int32_t spt, w, nc;
  if (int rc = exem_tc_set_geometry(k_max, &spt, &w, &nc)) return rc;
  const int64_t rows = exem_tc_set_rows(l, k_max);
  const int64_t kp = bs ? round_up(d, kTcKChunk) : exem_tc_kp(d);
  dim3 block(64, 4);
  dim3 grid((unsigned)ceil_div(rows, 4));
  cudaStream_t st = (cudaStream_t)stream;
  if (dtype == EXEM_BF16)
    tcb::pack_sets_kernel<EXEM_BF16><<<grid, block, 0, st>>>(
        (const float *)packed, pnorms, card, l, l_pad, (int)k_max, (int)d, spt,
        w, nc, rows, (__nv_bfloat16 *)xs, kp, bs);
  else
    tcb::pack_sets_kernel<EXEM_F16><<<grid, block, 0, st>>>(
        (const float *)packed, pnorms, card, l, l_pad, (int)k_max, (int)d, spt,
        w, nc, rows, (__half *)xs, kp, bs);
  EXEM_LAUNCH_CHECK("tc_pack_sets");
  return EXEM_OK;
}

int exem_batch_eval_tc(int dtype, const void *xp, int64_t n, const void *aux,
                       const double *norms, const void *xs, const float *bs,
                       int64_t l, int64_t k_max, int64_t d, int64_t split_pts,
                       double *partial, int64_t splits, void *stream) {
  using namespace exem::tcb;
  if (dtype != EXEM_BF16 && dtype != EXEM_F16)
    return fail(EXEM_ERR_ARG, "batch_eval_tc is bf16/f16 only");
  if (n < 1 || l < 1) return fail(EXEM_ERR_ARG, "empty batch or ground set");
  if (split_pts < BM || split_pts % BM)
    return fail(EXEM_ERR_ARG, "split_pts must be a multiple of %d", BM);
  if (splits != ceil_div(n, split_pts))
    return fail(EXEM_ERR_ARG, "splits mismatch");
  int dev = 0, sms = 0, major = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
  if (major != 10)
    return fail(EXEM_ERR_UNSUPPORTED,
                "tcgen05 path needs an sm_100 (B200) device, found sm_%d",
                major * 10);
  BParams prm;
  int32_t spt, w, nc;
  if (int rc = exem_tc_set_geometry(k_max, &spt, &w, &nc)) return rc;
  const bool plain = bs != nullptr;
  if (plain && norms == nullptr)
    return fail(EXEM_ERR_ARG, "batch_eval_tc: plain operands need norms");
  const int64_t kp = plain ? round_up(d, kTcKChunk) : exem_tc_kp(d);
  prm.plain = plain ? 1 : 0;
  prm.norms = norms;
  prm.bs = bs;
  prm.n = n;
  prm.l = l;
  prm.split_pts = split_pts;
  prm.splits = splits;
  prm.set_tiles = ceil_div(l, spt);
  prm.spt = spt;
  prm.w = w;
  prm.ncols = nc;
  prm.ksteps = (int)ceil_div(d + (plain ? 0 : kTcConst), 16);
  prm.kchunks = (int)(kp / KCH);
  // Single-CTA tiles by default.  EXEM_TCB_CG=2 selects CTA pairs
  // (cta_group::2, M = 256, each CTA holding half of the set tile, 9 instead
  // of 5 point-chunk stages at d = 256): correct (tests) but measured no
  // faster at d = 256 and 1.4x slower at d = 100 (tools/k4_cg_compare.sh,
  // profiles/r01_k4_probe.log) -- the per-chunk cross-SM handshake costs
  // more than the deeper ring saves.
  int cg = 1;
  if (const char *e = getenv("EXEM_TCB_CG")) cg = atoi(e) == 2 ? 2 : 1;
  prm.idesc = make_idesc(dtype == EXEM_BF16, BM * cg, nc);
  prm.aux = (const float *)aux;
  {
    const char *dbg = getenv("EXEM_TCB_DEBUG");
    prm.dbg = dbg ? atoi(dbg) : 0;
  }
  prm.partial = partial;
  prm.trace = nullptr;
  const char *trace_path = getenv("EXEM_TCB_TRACE");
  if (trace_path) {
    cudaMalloc(&prm.trace, 12 * kTrace * sizeof(long long));
    cudaMemset(prm.trace, 0, 12 * kTrace * sizeof(long long));
  }
  const int b_chunk = (nc / cg) * 128;
  const int avail = kSmemBudget - kBarBytes - 1024;
  // set tile stationary when it leaves room for >= 3 point-chunk stages
  const bool bstream = (avail - prm.kchunks * b_chunk) / A_CHUNK < 3;
  const int sb_bytes = bstream ? 0 : prm.kchunks * b_chunk;
  // whole-tile point stages (one handshake per tile) when >= 3 fit and the
  // K loop unrolls (K <= 128); EXEM_TCB_DEBUG 128 disables (timing only)
  const bool tstage = cg == 1 && !bstream && prm.ksteps <= 8 &&
                      (avail - sb_bytes) / (prm.kchunks * A_CHUNK) >= 3 &&
                      !(prm.dbg & 128);
  prm.tstage = tstage ? 1 : 0;
  // otherwise two K chunks per stage when >= 2 such stages fit: half the
  // per-stage handshakes (d = 256: 149 -> 134 ms with only 2 stages,
  // profiles/r01_k4_probe.log); EXEM_TCB_G forces 1 or 2 (experiments)
  int gch = (!tstage && !bstream && prm.kchunks >= 2 &&
             (avail - sb_bytes) / (2 * A_CHUNK) >= 2) ? 2 : 1;
  if (const char *e = getenv("EXEM_TCB_G"))
    if (!tstage && !bstream) gch = atoi(e) == 2 && prm.kchunks >= 2 ? 2 : 1;
  prm.gch = gch;
  const int stage_bytes = tstage ? prm.kchunks * A_CHUNK
                                 : gch * A_CHUNK + (bstream ? b_chunk : 0);
  int stages = (avail - sb_bytes) / stage_bytes;
  if (stages > 16) stages = 16;
  if (stages < 2) return fail(EXEM_ERR_UNSUPPORTED, "set tile too large for smem");
  prm.stages = stages;
  prm.bstream = bstream ? 1 : 0;
  const size_t smem = (size_t)sb_bytes + (size_t)stages * stage_bytes +
                      kBarBytes + 1024;
  CUtensorMap mp, ms;
  if (int rc = make_map(&mp, xp, dtype, exem_tc_rows(n), kp, BM)) return rc;
  if (int rc = make_map(&ms, xs, dtype, exem_tc_set_rows(l, k_max), kp,
                        nc / cg))
    return rc;
  const int64_t items = prm.set_tiles * splits;
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute at[1];
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = (cudaStream_t)stream;
  cudaError_t e;
  if (cg == 2) {
    e = cudaFuncSetAttribute(batch_tc_kernel<2>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem);
    if (e != cudaSuccess)
      return fail(EXEM_ERR_CUDA, "smem attr: %s", cudaGetErrorString(e));
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int clusters = 0;
    cfg.gridDim = dim3((unsigned)(sms & ~1));
    e = cudaOccupancyMaxActiveClusters(&clusters, batch_tc_kernel<2>, &cfg);
    if (e != cudaSuccess || clusters < 1)
      return fail(EXEM_ERR_CUDA, "no co-resident CTA pairs: %s",
                  cudaGetErrorString(e));
    const int64_t pairs = items < clusters ? items : clusters;
    cfg.gridDim = dim3((unsigned)(2 * pairs));
    if (getenv("EXEM_TCB_VERBOSE"))
      fprintf(stderr, "batch_tc<2>: clusters=%d grid=%u stages=%d smem=%zu "
              "bstream=%d\n", clusters, cfg.gridDim.x, stages, smem,
              (int)bstream);
    e = cudaLaunchKernelEx(&cfg, batch_tc_kernel<2>, mp, ms, prm);
  } else {
    e = cudaFuncSetAttribute(batch_tc_kernel<1>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem);
    if (e != cudaSuccess)
      return fail(EXEM_ERR_CUDA, "smem attr: %s", cudaGetErrorString(e));
    cfg.gridDim = dim3((unsigned)(items < sms ? items : sms));
    e = cudaLaunchKernelEx(&cfg, batch_tc_kernel<1>, mp, ms, prm);
  }
  if (e != cudaSuccess)
    return fail(EXEM_ERR_CUDA, "batch_tc_kernel launch: %s",
                cudaGetErrorString(e));
  if (prm.trace) {  // timing experiment: dump the CTA-0 timeline
    static long long host[12 * kTrace];
    cudaStreamSynchronize((cudaStream_t)stream);
    cudaMemcpy(host, prm.trace, sizeof(host), cudaMemcpyDeviceToHost);
    cudaFree(prm.trace);
    if (FILE *f = fopen(trace_path, "w")) {
      for (int t = 0; t < kTrace; ++t)
        for (int s2 = 0; s2 < 12; ++s2)
          fprintf(f, "%lld%c", host[s2 * kTrace + t], s2 == 11 ? '\n' : ' ');
      fclose(f);
    }
  }
  EXEM_LAUNCH_CHECK("batch_tc_kernel");
  return EXEM_OK;
}

}  // extern "C"
