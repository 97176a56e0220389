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
// A set tile holds `spt` = min(16, 256 / k_max) sets, column-interleaved:
// column c is slot c / spt of set c % spt (the packed batch's own round-robin
// order, core.py:331-346), so N = round_up(spt * k_max, 16) with no per-set
// padding (k_max = 50: 5 sets in N = 256, not 4 in 224).  Blank slots
// (e >= card_j) and padding columns are copies of the set's element 0, so
// they never change a minimum and need no masking (cf. the blank-slot rule,
// core.py:227-230).
//
// Roles (320 threads, 1 CTA/SM, persistent over (split, set tile) items):
//   warp 0      TMA producer (set tile once per item; point K-chunks
//               through a `stages`-deep ring)
//   warp 1      TMEM allocator + single-thread MMA issuer (M=128 x
//               N=ncols x K=16), handshakes software-pipelined one chunk
//               ahead so the tensor pipe's ~2-deep queue never drains
//   warps 2-9   epilogue: lane quarter q = warp%4 (TMEM lane access rule),
//               column-group / set parity h = (warp-2)/4 (maxima swapped
//               through smem); per-thread fp64 running sums per set across the item's point tiles, fixed-order xor-shuffle +
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
// Sets per set tile: up to 16 in the main kernel; small sets (k_max <= 10)
// use a separate instantiation with up to 32 (N = 16 k_max < 256 left the
// MMAs short of the sync skeleton; a run-time switch inside one kernel
// slowed the C5 shape by 17 %, so the wide variant is its own kernel)
constexpr int kMaxSpt = 16;
constexpr int kMaxSptWide = 32;
constexpr int kSmemBudget = 227 * 1024;
// barriers, reductions, plain b, and the [2][MAXS][BM] maxima exchange
__host__ __device__ constexpr int bar_bytes(int maxs) {
  return 3072 + 2 * maxs * BM * 4;
}
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

// Timing-probe masks (EXEM_TCB_DEBUG: 1 no epilogue, 2 no MMA, 4 no point
// TMA, 8 no aux load) exist only in a probe build (-DEXEM_TCB_PROBE_BUILD via
// EXEM_NVCC_FLAGS): K3 showed such branches alone can cost ~20 % of a step.
#ifdef EXEM_TCB_PROBE_BUILD
#define TCB_PROBE(p, bit) (((p).dbg & (bit)) != 0)
#else
#define TCB_PROBE(p, bit) false
#endif

struct BParams {
  int64_t n;           // points of this slice
  int64_t l;           // sets
  int64_t split_pts;   // points per split (multiple of BM)
  int64_t splits;
  int64_t set_tiles;
  int spt;             // sets per set tile
  int w;               // slots per set (= k_max; columns interleaved)
  int ncols;           // MMA N (multiple of 16, >= spt * w)
  int ksteps;          // K=16 MMA steps
  int kchunks;         // 64-wide K chunks per operand row
  int stages;          // point-chunk ring depth
  int bstream;         // 1: set chunks streamed with the point chunks
  int tstage;          // 1: a ring stage holds a whole point tile (all K)
  int gch;             // otherwise: 64-wide K chunks per ring stage (1, 2)
  int dbg;             // timing experiments only (EXEM_TCB_DEBUG), 0 in use
  int late;            // 1: next accumulator buffer acquired after the commit
  uint32_t idesc;
  long long *trace;    // timing experiments only (EXEM_TCB_TRACE): CTA-0 timeline
  const float *aux;    // [n] aux distances (compute type)
  int plain;           // 1: unfolded operands, constants added in the epilogue
  const double *norms; // plain: [n] ||v_i||^2
  const float *bs;     // plain: [set rows] ||e||^2 / 2 per set-tile row
  double *partial;     // [splits][l]
};

// Work items (split sp, set tile st) of one CTA.  A cluster of MC CTAs takes
// units (split, group of MC adjacent set tiles): CTA rank r scores set tile
// MC*g + r against the SAME point tiles, which are multicast to all MC CTAs
// (each CTA loads 1/MC of every point chunk: 1/MC of the L2 -> SM traffic).
// A spare tile (st >= set_tiles, odd set_tiles) reads TMA's zero fill and
// writes nothing.
struct WorkSplit {
  int64_t first, step, units, groups;  // groups = ceil(set_tiles / MC)
  int mc;
  uint32_t rank;
  __device__ __forceinline__ void item(int64_t u, int64_t &st,
                                       int64_t &sp) const {
    sp = u / groups;
    st = (int64_t)mc * (u % groups) + rank;
  }
};

// Release an accumulator buffer once every lane's tcgen05.ld is complete.
struct TmemRelease {
  uint64_t *bar;
  int lane;
  __device__ __forceinline__ void operator()() const {
    fence_before();
    __syncwarp();
    if (lane == 0) mbar_arrive(bar);
  }
};

// Epilogue of one accumulator tile for one warp.  Set tiles are column-
// interleaved: column c holds slot c / SPT of set c % SPT (exem_tc_pack_sets),
// so with SPT known at compile time every column's set is static.  The two
// warps of a TMEM lane quarter split the tile's 8-column groups (g = 2i + HH,
// an even split for any N), each folds its columns into per-set maxima pm[],
// and they swap the maxima of the sets the other one owns (set parity) through
// shared memory -- one 64-thread named barrier per tile.  Columns are drained
// with tcgen05.ld x8 in batches of 8 groups and one tcgen05.wait::ld per
// batch; the buffer is released right after the last batch's wait.
//   t = min(aux_i, max(0, -2 max_e D)),  acc[u] += t   (fp64, per thread)
template <int SPT>
struct EpiShape {
  static constexpr int OWN = (SPT + 1) / 2;  // sets finalised per warp (max)
  static constexpr int GB = 8;               // 8-column groups per ld batch
};

// xch: this buffer's [MAXS][BM] exchange slots (set-major, row-minor:
// conflict-free).
template <int SPT, int HH, bool kPlain, typename Release>
__device__ __forceinline__ void epi_tile(
    uint32_t taddr, int ngroups, int q, int row, float ax, float ha,
    bool valid, const float *bsm, float *xch,
    double (&acc)[EpiShape<SPT>::OWN], const Release &release) {
  constexpr int GB = EpiShape<SPT>::GB;
  const float ninf = -__int_as_float(0x7f800000);
  float pm[SPT];
#pragma unroll
  for (int s = 0; s < SPT; ++s) pm[s] = ninf;
  const int mine = (ngroups - HH + 1) >> 1;  // this warp's groups (>= 1)
#pragma unroll
  for (int b = 0; b < 16 / GB; ++b) {
    if (b * GB < mine) {
      uint32_t r[GB][8];
#pragma unroll
      for (int i = 0; i < GB; ++i)
        if (b * GB + i < mine)
          TMEM_LD8(taddr + (uint32_t)(8 * (2 * (b * GB + i) + HH)), r[i]);
      tmem_wait_ld();
      if ((b + 1) * GB >= mine) release();
#pragma unroll
      for (int i = 0; i < GB; ++i) {
        if (b * GB + i < mine) {
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            const int c = 8 * (2 * (b * GB + i) + HH) + k;  // static
            float v = __uint_as_float(r[i][k]);
            if constexpr (kPlain) v -= bsm[c];
            pm[c % SPT] = fmaxf(pm[c % SPT], v);
          }
        }
      }
    }
  }
  if (mine <= 0) release();
  // swap maxima: this warp finalises sets s = HH (mod 2)
#pragma unroll
  for (int s = 1 - HH; s < SPT; s += 2) xch[s * BM + row] = pm[s];
  asm volatile("bar.sync %0, 64;" ::"r"(2 + q) : "memory");
#pragma unroll
  for (int u = 0; u < EpiShape<SPT>::OWN; ++u) {
    const int s = HH + 2 * u;
    if (s < SPT) {
      const float mx = fmaxf(pm[s], xch[s * BM + row]);
      // folded: min_e d = -2 max D;  plain: min_e d = a - 2 max (D - b)
      const float dm = kPlain ? fmaf(-2.f, mx, ha) : -2.f * mx;
      const float t = fminf(ax, fmaxf(0.f, dm));
      if (valid) acc[u] += (double)t;
    }
  }
}

// The epilogue warps' whole loop for one sets-per-tile count (SPT at compile
// time, so every column's set and the accumulator array are static) and one
// group parity HH.  Work items follow the producer's order (item_of).
template <int SPT, int HH, bool kPlain, int MAXS>
__device__ __forceinline__ void epilogue_role(const BParams &p, uint32_t tmem,
                                              uint64_t *tfull,
                                              uint64_t *tempty, double *red,
                                              float *bsm, float *xch, int warp,
                                              int lane, const WorkSplit &ws) {
  constexpr int OWN = EpiShape<SPT>::OWN;
  const int ew = warp - 2;       // 0..7
  const int q = warp & 3;        // TMEM lane quarter (lane access rule)
  const int row = q * 32 + lane; // point row within the tile
  const int ngroups = p.ncols >> 3;
  uint32_t buf = 0, tph = 0;
#ifdef EXEM_TCB_TRACE_BUILD
  int etile = 0;
  const bool tr = warp == 2 && lane == 0;
#endif
  for (int64_t u = ws.first; u < ws.units; u += ws.step) {
    int64_t st, sp;
    ws.item(u, st, sp);
    const int64_t p0 = sp * p.split_pts;
    const int64_t p1 = min(p.n, p0 + p.split_pts);
    double acc[OWN];
#pragma unroll
    for (int k = 0; k < OWN; ++k) acc[k] = 0.0;
    if constexpr (kPlain) {  // the set tile's column constants, once per item
      for (int c = ew * 32 + lane; c < p.ncols; c += kEpiWarps * 32)
        bsm[c] = st < p.set_tiles ? p.bs[st * p.ncols + c] : 0.f;
      asm volatile("bar.sync 1, %0;" ::"n"(kEpiWarps * 32) : "memory");
    }
    for (int64_t pt = p0; pt < p1; pt += BM) {
      const int64_t pi = pt + row;
      const bool valid = pi < p1;
      const float ax = (valid && !TCB_PROBE(p, 8)) ? p.aux[pi] : 0.f;
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
#ifdef EXEM_TCB_TRACE_BUILD
      if (tr) TRB(12, etile);
#endif
      const uint32_t taddr =
          tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(buf * 256);
      TmemRelease rel{&tempty[buf], lane};
      if (TCB_PROBE(p, 1)) {  // timing experiment: no TMEM drain / math
        rel();
      } else {
#ifdef EXEM_TCB_TRACE_BUILD
        struct Traced {  // release + timestamp (slot 13)
          TmemRelease r;
          const BParams &p;
          bool tr;
          int etile;
          __device__ void operator()() const {
            r();
            if (tr) TRB(13, etile);
          }
        } trel{rel, p, tr, etile};
        epi_tile<SPT, HH, kPlain>(taddr, ngroups, q, row, ax, ha, valid, bsm,
                                  xch + buf * (MAXS * BM), acc, trel);
#else
        epi_tile<SPT, HH, kPlain>(taddr, ngroups, q, row, ax, ha, valid, bsm,
                                  xch + buf * (MAXS * BM), acc, rel);
#endif
      }
#ifdef EXEM_TCB_TRACE_BUILD
      if (tr) TRB(4, etile);
      ++etile;
#endif
      buf ^= 1u;
    }
    // item end: per set, fixed xor tree over the 32 lanes, then the four
    // lane quarters in order
#pragma unroll
    for (int k = 0; k < OWN; ++k) {
      const int s = HH + 2 * k;
      if (s < SPT) {
        double v = acc[k];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (lane == 0) red[q * MAXS + s] = v;
      }
    }
    asm volatile("bar.sync 1, %0;" ::"n"(kEpiWarps * 32) : "memory");
    if (ew == 0) {
      const int64_t j = st * SPT + lane;  // >= l for a cluster's spare tile
      if (lane < SPT && j < p.l)
        p.partial[sp * p.l + j] =
            ((red[lane] + red[MAXS + lane]) + red[2 * MAXS + lane]) +
            red[3 * MAXS + lane];
    }
    asm volatile("bar.sync 1, %0;" ::"n"(kEpiWarps * 32) : "memory");
  }
}

// Issuer loop of one work item with whole-tile point stages (one barrier
// handshake per tile, K3's scheme -- the per-chunk handshake costs ~200+
// cycles of mbarrier latency each, profiles/r01_k4_probe.log): KS K-steps
// unrolled at compile time, the next tile's point stage (full) acquired
// before MMA KS-2 and its accumulator buffer (tempty) before MMA KS-1.
template <int MC>
__device__ __forceinline__ void release_stage(uint64_t *bar);

template <int KS, int MC, bool kLate>
__device__ __forceinline__ void k4_item_tstage(
    const BParams &p, int ntiles, int &stage, uint32_t &ph, uint32_t &tph,
    uint32_t &buf, int &itile, uint64_t a_base, uint32_t a_step,
    uint64_t b_base, uint32_t b_step, uint32_t tmem, uint64_t *full,
    uint64_t *empty, uint64_t *tfull, uint64_t *tempty) {
  constexpr int WF = KS > 2 ? KS - 2 : 0;
  constexpr int WT = KS > 1 ? KS - 1 : 0;
  mbar_wait(&tempty[buf], ((tph >> buf) & 1u) ^ 1u);
  TRB(0, itile);
  tph ^= 1u << buf;
  mbar_wait(&full[stage], ph);
  TRB(1, itile);
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
        TRB(1, itile + 1);
        fence_after();
      }
      if (!kLate && ks == WT && more) {
        mbar_wait(&tempty[nbuf], ((tph >> nbuf) & 1u) ^ 1u);
        TRB(0, itile + 1);
        tph ^= 1u << nbuf;
        fence_after();
      }
      if (!TCB_PROBE(p, 2))
        umma_f16(d, ad + (uint64_t)((ks >> 2) * (A_CHUNK >> 4) + (ks & 3) * 2),
                 b_base + (uint64_t)((ks >> 2) * b_step + (ks & 3) * 2),
                 p.idesc, ks > 0 ? 1u : 0u);
    }
    release_stage<MC>(&empty[stage]);
    umma_commit(&tfull[buf]);
    TRB(2, itile);
    if (kLate && more) {
      // the next buffer is acquired only after this tile's commit, so the
      // commit (and the epilogue of this tile) never waits for the release
      // of the previous tile -- the epilogue-bound shapes' critical chain
      mbar_wait(&tempty[nbuf], ((tph >> nbuf) & 1u) ^ 1u);
      TRB(0, itile + 1);
      tph ^= 1u << nbuf;
      fence_after();
    }
    ++itile;
    buf = nbuf;
    stage = nstage;
    ph = nph;
  }
}

// MMA j of an event whose stage holds consecutive 64-wide K chunks: chunk
// j>>2 of the event, K=16 step j&3 inside the 128-B swizzle row.
__device__ __forceinline__ void issue_mma(const BParams &p, uint32_t d,
                                          uint64_t ad, uint64_t bd,
                                          uint32_t b_step, int kc, int j) {
  if (TCB_PROBE(p, 2)) return;  // timing experiment: no MMA
  const uint64_t a = ad + (uint64_t)((j >> 2) * (A_CHUNK >> 4) + (j & 3) * 2);
  const uint64_t b = bd + (uint64_t)((j >> 2) * b_step + (j & 3) * 2);
  umma_f16(d, a, b, p.idesc, (kc | j) ? 1u : 0u);
}

// Release a point stage: on this CTA's empty barrier, or (MC > 1) on every
// cluster CTA's -- their producers multicast into this CTA's copy.
template <int MC>
__device__ __forceinline__ void release_stage(uint64_t *bar) {
  if constexpr (MC > 1)
    umma_commit_mc(bar, (uint16_t)((1u << MC) - 1));
  else
    umma_commit(bar);
}

// MC: CTAs per cluster sharing every point tile by TMA multicast (1 = none).
// map_p: the point operand with BM/MC-row boxes.
template <int MC, int MAXS>
__global__ void __launch_bounds__(kThreads, 1)
    batch_tc_kernel(const __grid_constant__ CUtensorMap map_p,
                    const __grid_constant__ CUtensorMap map_s,
                    const BParams p) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char *smem = (unsigned char *)(((uintptr_t)smem_raw + 1023) &
                                          ~(uintptr_t)1023);
  const int b_chunk = p.ncols * 128;  // bytes of one set-tile K-chunk
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
  uint32_t *tmem_slot = (uint32_t *)(bempty + 1);
  double *red = (double *)(tmem_slot + 4);         // [4][MAXS]
  float *bsm = (float *)(red + 4 * MAXS);          // [256] plain: set b
  float *xch = bsm + 256;                          // [2][MAXS][BM]

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  WorkSplit ws;
  ws.mc = MC;
  ws.rank = MC > 1 ? cluster_rank() : 0u;
  ws.groups = (p.set_tiles + MC - 1) / MC;
  ws.units = ws.groups * p.splits;
  ws.first = blockIdx.x / MC;
  ws.step = gridDim.x / MC;
  if (warp == 0 && lane == 0) {
    for (int s = 0; s < p.stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], MC);  // one commit per cluster CTA
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], kEpiWarps);
    }
    mbar_init(bfull, 1);
    mbar_init(bempty, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&map_p));
    asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&map_s));
  }
  if (warp == 1) {
    asm volatile(
        "tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::
            "r"(su32(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  fence_before();
  __syncthreads();
  if constexpr (MC > 1) cluster_sync();  // peers' barriers initialised
  fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // -------------------------------------------------------------- producer
    if (lane == 0) {
      int stage = 0, ptile = 0;
      uint32_t ph = 0, bph = 0;
      const uint16_t mask = (uint16_t)((1u << MC) - 1);
      const int prow_off = (int)ws.rank * (BM / MC);   // this CTA's rows
      const int pdst_off = (int)ws.rank * (A_CHUNK / MC);
      for (int64_t u = ws.first; u < ws.units; u += ws.step) {
        int64_t st, sp;
        ws.item(u, st, sp);
        // a cluster's spare tile (st >= set_tiles) re-reads tile 0: valid
        // memory, results never written
        const int srow = st < p.set_tiles ? (int)(st * p.ncols) : 0;
        if (!p.bstream) {
          mbar_wait_sleep(bempty, bph ^ 1);
          bph ^= 1;
          mbar_expect_tx(bfull, (uint32_t)sb_bytes);
          for (int kc = 0; kc < p.kchunks; ++kc)
            tma_load_2d(sb + kc * b_chunk, &map_s, bfull, kc * KCH, srow);
        }
        const int64_t p0 = sp * p.split_pts;
        const int64_t p1 = min(p.n, p0 + p.split_pts);
        for (int64_t pt = p0; pt < p1; pt += BM, ++ptile) {
          const int ng = p.tstage ? p.kchunks : p.gch;  // chunks per stage
          for (int kc = 0; kc < p.kchunks; kc += ng) {
            const int gn = p.kchunks - kc < ng ? p.kchunks - kc : ng;
            mbar_wait(&empty[stage], ph ^ 1);
            if (kc == 0) TRB(5, ptile);
            unsigned char *dst = sa + stage * stage_bytes;
            if (TCB_PROBE(p, 4)) {  // timing experiment: no point-operand traffic
              mbar_arrive(&full[stage]);
            } else {
              mbar_expect_tx(&full[stage],
                             (uint32_t)(gn * A_CHUNK + (p.bstream ? b_chunk : 0)));
              for (int j = 0; j < gn; ++j) {
                if constexpr (MC > 1)
                  tma_load_2d_mc(dst + j * A_CHUNK + pdst_off, &map_p,
                                 &full[stage], (kc + j) * KCH,
                                 (int)pt + prow_off, mask);
                else
                  tma_load_2d(dst + j * A_CHUNK, &map_p, &full[stage],
                              (kc + j) * KCH, (int)pt);
              }
              if (p.bstream)
                tma_load_2d(dst + A_CHUNK, &map_s, &full[stage], kc * KCH,
                            srow);
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
    if (lane == 0) {
      const uint64_t a_base = sw128_desc(su32(sa));
      const uint64_t b_base = sw128_desc(su32(sb));
      const uint32_t a_step = (uint32_t)(stage_bytes >> 4);
      const uint32_t b_step = (uint32_t)(b_chunk >> 4);
      int stage = 0, itile = 0;
      uint32_t ph = 0, bph = 0, tph = 0, buf = 0;
      for (int64_t u = ws.first; u < ws.units; u += ws.step) {
        int64_t st, sp;
        ws.item(u, st, sp);
        const int64_t p0 = sp * p.split_pts;
        const int64_t p1 = min(p.n, p0 + p.split_pts);
        const int ntiles = (int)((p1 - p0 + BM - 1) / BM);
        const int kev = (p.kchunks + p.gch - 1) / p.gch;  // events per tile
        const int nev = ntiles * kev;
        if (!p.bstream) {
          mbar_wait(bfull, bph);
          bph ^= 1;
        }
        if (p.tstage) {
          switch (p.ksteps) {
#define EXEM_K4_ITEM(K)                                                       \
  case K:                                                                     \
    if (p.late)                                                               \
      k4_item_tstage<K, MC, true>(p, ntiles, stage, ph, tph, buf, itile,      \
                                  a_base, a_step, b_base, b_step, tmem, full, \
                                  empty, tfull, tempty);                      \
    else                                                                      \
      k4_item_tstage<K, MC, false>(p, ntiles, stage, ph, tph, buf, itile,     \
                                   a_base, a_step, b_base, b_step, tmem,      \
                                   full, empty, tfull, tempty);               \
    break;
            EXEM_K4_ITEM(1) EXEM_K4_ITEM(2) EXEM_K4_ITEM(3) EXEM_K4_ITEM(4)
            EXEM_K4_ITEM(5) EXEM_K4_ITEM(6) EXEM_K4_ITEM(7)
            default: EXEM_K4_ITEM(8)
#undef EXEM_K4_ITEM
          }
          umma_commit(bempty);
          continue;
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
          // full events (one or two whole 64-wide chunks) issue from
          // compile-time unrolled code: the issuing thread is the critical
          // path (K3's experience), the runtime loop only covers ragged tails
          if (nk == 8) {
#pragma unroll
            for (int j = 0; j < 6; ++j) issue_mma(p, d, ad, bd, b_step, kc, j);
          } else if (nk == 4) {
#pragma unroll
            for (int j = 0; j < 2; ++j) issue_mma(p, d, ad, bd, b_step, kc, j);
          } else {
#pragma unroll 1
            for (int j = 0; j < head; ++j) issue_mma(p, d, ad, bd, b_step, kc, j);
          }
          if (trc) TRB(8, itile);
          if (e + 1 < nev) {
            if (last && !p.late) {
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
          if (nk == 8) {
#pragma unroll
            for (int j = 6; j < 8; ++j) issue_mma(p, d, ad, bd, b_step, kc, j);
          } else if (nk == 4) {
#pragma unroll
            for (int j = 2; j < 4; ++j) issue_mma(p, d, ad, bd, b_step, kc, j);
          } else {
#pragma unroll 1
            for (int j = head; j < nk; ++j) issue_mma(p, d, ad, bd, b_step, kc, j);
          }
          if (trc) TRB(10, itile);
          release_stage<MC>(&empty[stage]);
          if (trc) TRB(11, itile);
          if (last) {
            umma_commit(&tfull[buf]);
            TRB(2, itile);
            if (p.late && e + 1 < nev) {  // see k4_item_tstage<.., kLate>
              const uint32_t nb = buf ^ 1u;
              mbar_wait(&tempty[nb], ((tph >> nb) & 1u) ^ 1u);
              TRB(0, itile + 1);
              tph ^= 1u << nb;
              fence_after();
            }
            ++itile;
            buf ^= 1u;
            kc = 0;
          } else {
            kc += p.gch;
          }
          stage = nstage;
          ph = nph;
        }
        if (!p.bstream) umma_commit(bempty);
      }
    }
    __syncwarp();
  } else {
    // -------------------------------------------------------------- epilogue
    const bool hh = (warp - 2) >= 4;  // 8-column group parity of this warp
#define EXEM_EPI_ROLE(S, H, PL)                                              \
  epilogue_role<S, H, PL, MAXS>(p, tmem, tfull, tempty, red, bsm, xch, warp, \
                                lane, ws)
#define EXEM_EPI_CASE(S)                                                     \
  case S:                                                                    \
    if (p.plain) {                                                           \
      if (hh) EXEM_EPI_ROLE(S, 1, true); else EXEM_EPI_ROLE(S, 0, true);     \
    } else {                                                                 \
      if (hh) EXEM_EPI_ROLE(S, 1, false); else EXEM_EPI_ROLE(S, 0, false);   \
    }                                                                        \
    break;
    // each instantiation compiles only its own set-count class
    if constexpr (MAXS == kMaxSpt) {
      switch (p.spt) {
        EXEM_EPI_CASE(1) EXEM_EPI_CASE(2) EXEM_EPI_CASE(3) EXEM_EPI_CASE(4)
        EXEM_EPI_CASE(5) EXEM_EPI_CASE(6) EXEM_EPI_CASE(7) EXEM_EPI_CASE(8)
        EXEM_EPI_CASE(9) EXEM_EPI_CASE(10) EXEM_EPI_CASE(11) EXEM_EPI_CASE(12)
        EXEM_EPI_CASE(13) EXEM_EPI_CASE(14) EXEM_EPI_CASE(15) EXEM_EPI_CASE(16)
        default: break;
      }
    } else {
      switch (p.spt) {
        EXEM_EPI_CASE(17) EXEM_EPI_CASE(18) EXEM_EPI_CASE(19) EXEM_EPI_CASE(20)
        EXEM_EPI_CASE(21) EXEM_EPI_CASE(22) EXEM_EPI_CASE(23) EXEM_EPI_CASE(24)
        EXEM_EPI_CASE(25) EXEM_EPI_CASE(26) EXEM_EPI_CASE(27) EXEM_EPI_CASE(28)
        EXEM_EPI_CASE(29) EXEM_EPI_CASE(30) EXEM_EPI_CASE(31) EXEM_EPI_CASE(32)
        default: break;
      }
    }
#undef EXEM_EPI_CASE
#undef EXEM_EPI_ROLE
  }

  fence_before();
  __syncthreads();
  if constexpr (MC > 1) cluster_sync();  // no multicast / commit in flight
  if (warp == 1) {
    fence_after();
    asm volatile(
        "tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

// ---------------------------------------------------------------- packing
// Set-tile operand rows from the packed round-robin batch
// packed[d_pad][k_max][l_pad] (compute type, packed_address order,
// core.py:320-328).  Column-interleaved like the packed batch itself: row
// r = tile*ncols + c holds slot e = c / spt of set j = tile*spt + c % spt --
// element (e < card_j ? e : 0), then the folded constants -- so blank slots
// and the padding columns past spt*k_max repeat the set's element 0 (never
// change a minimum, need no mask).  Rows of sets j >= l are zero.
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
  const int s = c % spt, e = c / spt;
  const int64_t j = tile * spt + s;
  const bool real = j < l;
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
        v = fold_one<S>(k - d);
      } else if (k < d + kTcConst) {
        double p[3];
        fold_pieces<S>(0.5 * pnorms[(int64_t)src * l_pad + j], p);
        v = -p[k - d - 3];
      }
    }
    x[r * kp + k] = from_d<S>(v);
  }
}

// Plain point rows [v, 0..] (kp = round_up(d, 64)) for unfolded K4-TC.
template <int DT, bool VS>
__global__ void pack_plain_kernel(const typename VtOf<DT, VS>::T *__restrict__ vt,
                                  int64_t ld,
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
    tile[ty][threadIdx.x] = (k < d && r < n) ? to_c(vt[(int64_t)k * ld + r]) : 0.f;
  }
  __syncthreads();
  for (int ty = threadIdx.y; ty < 32; ty += blockDim.y) {
    const int64_t r = r0 + ty;
    const int k = k0 + threadIdx.x;
    if (r < rows && k < kp) x[r * kp + k] = from_d<S>((double)tile[threadIdx.x][ty]);
  }
}

// Launch one persistent CTA per SM (clusters of MC), at most one per unit.
template <int MC, int MAXS>
cudaError_t launch_batch(const BParams &prm, const CUtensorMap &mp,
                         const CUtensorMap &ms, size_t smem, int sms,
                         int64_t splits, void *stream) {
  cudaError_t e = cudaFuncSetAttribute(
      batch_tc_kernel<MC, MAXS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
      (int)smem);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute at[1];
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = (cudaStream_t)stream;
  const int64_t units = (prm.set_tiles + MC - 1) / MC * splits;
  int64_t clusters = sms / MC;
  if (MC > 1) {
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = MC;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cfg.gridDim = dim3((unsigned)(clusters * MC));
    int active = 0;
    e = cudaOccupancyMaxActiveClusters(&active, batch_tc_kernel<MC, MAXS>,
                                       &cfg);
    if (e != cudaSuccess) return e;
    if (active < 1) return cudaErrorLaunchOutOfResources;
    if (active < clusters) clusters = active;
  }
  if (units < clusters) clusters = units;
  cfg.gridDim = dim3((unsigned)(clusters * MC));
  if (getenv("EXEM_TCB_VERBOSE"))
    fprintf(stderr, "batch_tc<%d,%d>: grid=%u stages=%d smem=%zu bstream=%d "
            "tstage=%d gch=%d\n", MC, MAXS, cfg.gridDim.x, prm.stages, smem,
            prm.bstream, prm.tstage, prm.gch);
  return cudaLaunchKernelEx(&cfg, batch_tc_kernel<MC, MAXS>, mp, ms, prm);
}

}  // namespace tcb
}  // namespace exem

using namespace exem;

extern "C" {

int exem_tc_set_geometry(int64_t k_max, int32_t *spt, int32_t *w,
                         int32_t *ncols) {
  if (k_max < 1) return fail(EXEM_ERR_ARG, "k_max must be >= 1");
  const int64_t ww = k_max;  // slots per set (interleaved, no padding)
  if (ww > 256)
    return fail(EXEM_ERR_UNSUPPORTED,
                "tcgen05 batch path holds a set in <= 256 TMEM columns "
                "(k_max=%lld)", (long long)k_max);
  int64_t s = 256 / ww;
  // more than 16 sets per tile (the small-set kernel) only where it wins:
  // k_max <= 10 (d = 100 / 256: k = 5 +14 % / +65 %, k = 8 +9 % / +40 %,
  // k = 10 +3 % / +12 %; k = 12..15 0 to -14 %, profiles/r02_k4_small_sets.log)
  if (s > tcb::kMaxSpt && ww > 10) s = tcb::kMaxSpt;
  if (s > tcb::kMaxSptWide) s = tcb::kMaxSptWide;
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
  const int tag = dtype & ~EXEM_VT_STORAGE;
  if (tag != EXEM_BF16 && tag != EXEM_F16)
    return fail(EXEM_ERR_ARG, "TC operands are bf16/f16 only");
  const int64_t kp = round_up(d, kTcKChunk), rows = exem_tc_rows(n);
  dim3 grid((unsigned)ceil_div(rows, 32), (unsigned)ceil_div(kp, 32));
  dim3 block(32, 8);
  cudaStream_t st = (cudaStream_t)stream;
  const bool vs = (dtype & EXEM_VT_STORAGE) != 0;
#define EXEM_PACK(DT, VS)                                                    \
  tcb::pack_plain_kernel<DT, VS><<<grid, block, 0, st>>>(                    \
      (const typename VtOf<DT, VS>::T *)vt, ld, n, (int)d,                   \
      (typename Traits<DT>::S *)xp, kp, rows)
  if (tag == EXEM_BF16) {
    if (vs) EXEM_PACK(EXEM_BF16, true); else EXEM_PACK(EXEM_BF16, false);
  } else {
    if (vs) EXEM_PACK(EXEM_F16, true); else EXEM_PACK(EXEM_F16, false);
  }
#undef EXEM_PACK
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
  prm.idesc = make_idesc(dtype == EXEM_BF16, BM, nc);
  // Acquire the next accumulator buffer after a tile's commit (instead of
  // before its last MMA) when few, wide sets make the epilogue the longer
  // leg: d = 100, 1M x 4096 sets, |S| = 50 / 64 / 100: 42.0 -> 39.3,
  // 53.0 -> 48.7, 96.3 -> 88.1 ms; |S| <= 32 (spt >= 8) is slower that way
  // and the chunked-stage layouts (d > 122) do not care
  // (tools/k4_late.sh, profiles/r01_k4_probe.log).  EXEM_TCB_LATE overrides.
  prm.late = spt <= 5 ? 1 : 0;
  if (const char *e = getenv("EXEM_TCB_LATE")) prm.late = atoi(e) ? 1 : 0;
  prm.aux = (const float *)aux;
  {
    const char *dbg = getenv("EXEM_TCB_DEBUG");
    prm.dbg = dbg ? atoi(dbg) : 0;
  }
  prm.partial = partial;
  prm.trace = nullptr;
  const char *trace_path = getenv("EXEM_TCB_TRACE");
  if (trace_path) {
    cudaMalloc(&prm.trace, 16 * kTrace * sizeof(long long));
    cudaMemset(prm.trace, 0, 16 * kTrace * sizeof(long long));
  }
  const int b_chunk = nc * 128;
  const int maxs = spt > kMaxSpt ? kMaxSptWide : kMaxSpt;
  const int kBarBytes = bar_bytes(maxs);
  const int avail = kSmemBudget - kBarBytes - 1024;
  // set tile stationary when it leaves room for >= 3 point-chunk stages
  const bool bstream = (avail - prm.kchunks * b_chunk) / A_CHUNK < 3;
  const int sb_bytes = bstream ? 0 : prm.kchunks * b_chunk;
  // whole-tile point stages (one handshake per tile) when >= 3 fit and the
  // K loop unrolls (K <= 128); EXEM_TCB_DEBUG 128 disables (timing only)
  const bool tstage = !bstream && prm.ksteps <= 8 &&
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
  // Point tiles shared by TMA multicast across clusters of MC CTAs scoring
  // adjacent set tiles (default 2; EXEM_TCB_MC = 1, 2 or 4 for experiments).
  // The streamed-set-tile layout keeps MC = 1.
  int mc = 2;
  if (const char *e = getenv("EXEM_TCB_MC")) {
    const int f = atoi(e);
    mc = (f == 1 || f == 4) ? f : 2;
  }
  if (bstream) mc = 1;
  CUtensorMap mp, ms;
  if (int rc = make_map(&mp, xp, dtype, exem_tc_rows(n), kp, BM / mc)) return rc;
  if (int rc = make_map(&ms, xs, dtype, exem_tc_set_rows(l, k_max), kp, nc))
    return rc;
  cudaError_t e;
  if (maxs == kMaxSptWide) {  // small sets: the 32-set-tile kernel
    e = mc == 1 ? launch_batch<1, kMaxSptWide>(prm, mp, ms, smem, sms, splits,
                                               stream)
                : launch_batch<2, kMaxSptWide>(prm, mp, ms, smem, sms, splits,
                                               stream);
  } else {
    switch (mc) {
      case 1: e = launch_batch<1, kMaxSpt>(prm, mp, ms, smem, sms, splits, stream); break;
      case 4: e = launch_batch<4, kMaxSpt>(prm, mp, ms, smem, sms, splits, stream); break;
      default: e = launch_batch<2, kMaxSpt>(prm, mp, ms, smem, sms, splits, stream); break;
    }
  }
  if (e != cudaSuccess)
    return fail(EXEM_ERR_CUDA, "batch_tc_kernel launch: %s",
                cudaGetErrorString(e));
  if (prm.trace) {  // timing experiment: dump the CTA-0 timeline
    static long long host[16 * kTrace];
    cudaStreamSynchronize((cudaStream_t)stream);
    cudaMemcpy(host, prm.trace, sizeof(host), cudaMemcpyDeviceToHost);
    cudaFree(prm.trace);
    if (FILE *f = fopen(trace_path, "w")) {
      for (int t = 0; t < kTrace; ++t)
        for (int s2 = 0; s2 < 16; ++s2)
          fprintf(f, "%lld%c", host[s2 * kTrace + t], s2 == 15 ? '\n' : ' ');
      fclose(f);
    }
  }
  EXEM_LAUNCH_CHECK("batch_tc_kernel");
  return EXEM_OK;
}

}  // extern "C"
