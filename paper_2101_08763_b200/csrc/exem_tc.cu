// exem_tc.cu -- tcgen05 / TMEM / TMA kernel for the optimizer-aware batched
// Greedy gains (K3-TC), sm_100a only.
//
// Replaces the per-step batch of explicit sets S u {c} that greedy_maximize
// builds and evaluates, pkg/src/exembatch/optimize.py:61-71 (through
// evaluate.py:142-149 / objective.py:75-90), by one persistent launch that
// evaluates every candidate of the step:
//
//   D[c][i] = x_c . y_i  with  x_c = [c, 1,1,1, -b_hi,-b_mid,-b_lo, 0..]
//                              y_i = [v_i, -h_hi,-h_mid,-h_lo, 1,1,1, 0..]
//   b = ||c||^2/2, h_i = (||v_i||^2 - m_i)/2   =>   D = (m_i - d(v_i,c))/2
//   partial[split][c] = sum_{i in split} max(0, D[c][i])   (x2 in K6)
//
// Roles (64 + 128*Q threads, 1 CTA/SM, persistent over (split, candidate
// tile)):
//   warps 0..4Q-1  epilogue: tcgen05.ld 32x32b -> relu-sum per
//               candidate row in registers (fp32 per tile, fp64 across
//               tiles), fixed-order merge of the column groups, one store
//               per candidate.  Warp w drains TMEM lane quarter w % 4.
//   warp kProdWarp  TMA producer: candidate tile (A, stationary per item)
//               and point tiles (B, streamed per 64-wide K chunk) into
//               128B-swizzled smem, mbarrier complete_tx.
//   warp kMmaWarp   TMEM allocator + single-thread tcgen05.mma issuer,
//               M=128 candidates x N=256 points x K=16, fp32 accum in TMEM,
//               two accumulator buffers (2 x 256 columns) so the epilogue
//               of tile t overlaps the MMAs of tile t+1.
#include <cstdlib>

#include "exem_tc_common.cuh"

namespace exem {
namespace tc {

constexpr int BM = 128;            // candidates per tile (TMEM lanes)
constexpr int BN = 256;            // points per tile (TMEM columns)
constexpr int A_CHUNK = BM * 128;  // bytes of one A K-chunk
constexpr int B_CHUNK = BN * 128;  // bytes of one B K-chunk
// Epilogue column groups Q: each TMEM lane quarter (32 candidates) is
// drained by Q warps, each taking BN / Q columns of a tile (a template
// parameter of the kernel; the host picks it per launch).  Q = 4 (16
// epilogue warps, 4 per SMSP) halves each warp's drain + relu-sum chain per
// tile: on data with many positive gains (a 16-blob mixture) that chain sets
// the tile period and Q = 4 is 16 % faster; on data where the sign screen
// skips almost everything (centred Gaussian) Q = 2 is 2 % faster
// (tools/k3_ab.py).
template <int Q, int BNv = BN> struct Epi {
  static constexpr int kCols = BNv / Q;       // accumulator columns per warp
  static constexpr int kWarps = 4 * Q;        // epilogue warps
  static constexpr int kThreads = 64 + 32 * kWarps;
  // Role warps.  The SMSP arbiter favours the highest warp id, so the
  // single MMA-issuing thread (whose every instruction is on the tensor
  // pipe's critical path) and the TMA producer take the two highest warp
  // ids; the epilogue warps 0..kWarps-1 keep warp % 4 = their TMEM lane
  // quarter.
  static constexpr int kProdWarp = kWarps;
  static constexpr int kMmaWarp = kWarps + 1;
};
constexpr int kSmemBudget = 227 * 1024;
constexpr int kBarBytes = 2048;  // barriers (<= 4 TMEM buffers), slot, red
constexpr int kTrace = 256;  // tiles traced on CTA 0 (EXEM_TC_TRACE)
// CTA-0 timeline (EXEM_TC_TRACE, tools/tc_trace.py): probe builds only
// (-DEXEM_TC_PROBE_BUILD), like the EXEM_TC_DEBUG masks.
#ifdef EXEM_TC_PROBE_BUILD
#define TR(slot, t)                                                        \
  do {                                                                     \
    if (p.trace != nullptr && blockIdx.x == 0 && (t) < kTrace)             \
      p.trace[(slot) * kTrace + (t)] = clock64();                          \
  } while (0)
#else
#define TR(slot, t) \
  do {              \
  } while (0)
#endif

// NK back-to-back MMAs over one 64-wide K chunk in a single asm block: the
// descriptors advance by 32 B (2 in the >>4 address field) per K=16 step.
// kFirst: the first MMA overwrites the accumulator (start of a tile).
#define EXEM_MMA1(P)                                                         \
  "tcgen05.mma.cta_group::1.kind::f16 [%0], a, b, %3, " P ";\n\t"
#define EXEM_STEP "add.s64 a, a, 2;\n\tadd.s64 b, b, 2;\n\t"
template <int NK, bool kFirst>
__device__ __forceinline__ void umma_chunk(uint32_t d, uint64_t ad,
                                           uint64_t bd, uint32_t idesc) {
  static_assert(NK >= 1 && NK <= 4, "1..4 MMAs per 64-wide chunk");
  if constexpr (NK == 1)
    asm volatile("{\n\t.reg .b64 a, b;\n\t.reg .pred pf, pt;\n\t"
                 "setp.ne.b32 pf, %4, 0;\n\tsetp.eq.b32 pt, 0, 0;\n\t"
                 "mov.b64 a, %1;\n\tmov.b64 b, %2;\n\t" EXEM_MMA1("pf") "}" ::
                     "r"(d), "l"(ad), "l"(bd), "r"(idesc), "r"(kFirst ? 0 : 1)
                 : "memory");
  if constexpr (NK == 2)
    asm volatile("{\n\t.reg .b64 a, b;\n\t.reg .pred pf, pt;\n\t"
                 "setp.ne.b32 pf, %4, 0;\n\tsetp.eq.b32 pt, 0, 0;\n\t"
                 "mov.b64 a, %1;\n\tmov.b64 b, %2;\n\t" EXEM_MMA1("pf")
                     EXEM_STEP EXEM_MMA1("pt") "}" ::"r"(d),
                 "l"(ad), "l"(bd), "r"(idesc), "r"(kFirst ? 0 : 1)
                 : "memory");
  if constexpr (NK == 3)
    asm volatile("{\n\t.reg .b64 a, b;\n\t.reg .pred pf, pt;\n\t"
                 "setp.ne.b32 pf, %4, 0;\n\tsetp.eq.b32 pt, 0, 0;\n\t"
                 "mov.b64 a, %1;\n\tmov.b64 b, %2;\n\t" EXEM_MMA1("pf")
                     EXEM_STEP EXEM_MMA1("pt") EXEM_STEP EXEM_MMA1("pt") "}" ::
                         "r"(d),
                 "l"(ad), "l"(bd), "r"(idesc), "r"(kFirst ? 0 : 1)
                 : "memory");
  if constexpr (NK == 4)
    asm volatile("{\n\t.reg .b64 a, b;\n\t.reg .pred pf, pt;\n\t"
                 "setp.ne.b32 pf, %4, 0;\n\tsetp.eq.b32 pt, 0, 0;\n\t"
                 "mov.b64 a, %1;\n\tmov.b64 b, %2;\n\t" EXEM_MMA1("pf")
                     EXEM_STEP EXEM_MMA1("pt") EXEM_STEP EXEM_MMA1("pt")
                         EXEM_STEP EXEM_MMA1("pt") "}" ::"r"(d),
                 "l"(ad), "l"(bd), "r"(idesc), "r"(kFirst ? 0 : 1)
                 : "memory");
}
template <bool kFirst>
__device__ __forceinline__ void umma_chunk_n(int nk, uint32_t d, uint64_t ad,
                                             uint64_t bd, uint32_t idesc) {
  switch (nk) {
    case 1: umma_chunk<1, kFirst>(d, ad, bd, idesc); break;
    case 2: umma_chunk<2, kFirst>(d, ad, bd, idesc); break;
    case 3: umma_chunk<3, kFirst>(d, ad, bd, idesc); break;
    default: umma_chunk<4, kFirst>(d, ad, bd, idesc); break;
  }
}

// All K steps of one whole-tile stage, fully unrolled (compile-time
// descriptor offsets): A chunks are A_CHUNK apart, B chunks B_CHUNK apart,
// K=16 steps 32 B apart inside a 128-B swizzle row.
template <int KS, int BNv = BN>
__device__ __forceinline__ void issue_tile(uint32_t d, uint64_t a0,
                                           uint64_t b0, uint32_t idesc) {
#pragma unroll
  for (int ks = 0; ks < KS; ++ks) {
    constexpr uint32_t kA = 128 * 128 >> 4, kB = BNv * 128 >> 4;
    umma_f16(d, a0 + (uint64_t)((ks >> 2) * kA + (ks & 3) * 2),
             b0 + (uint64_t)((ks >> 2) * kB + (ks & 3) * 2), idesc,
             ks > 0 ? 1u : 0u);
  }
}

// MMAs [LO, HI) of one whole-tile stage.
template <int LO, int HI, int BNv = BN>
__device__ __forceinline__ void issue_range(uint32_t d, uint64_t a0,
                                            uint64_t b0, uint32_t idesc) {
#pragma unroll
  for (int ks = LO; ks < HI; ++ks) {
    constexpr uint32_t kA = 128 * 128 >> 4, kB = BNv * 128 >> 4;
    umma_f16(d, a0 + (uint64_t)((ks >> 2) * kA + (ks & 3) * 2),
             b0 + (uint64_t)((ks >> 2) * kB + (ks & 3) * 2), idesc,
             ks > 0 ? 1u : 0u);
  }
}

// MMA issuer state carried across work items.
struct MmaState {
  int stage;
  uint32_t ph, tph, buf;
  int tile_no;
};


// One work item (a split's point tiles against the stationary candidate
// tile) with a software-pipelined handshake: the two acquisitions for tile
// t+1 -- B stage landed (full) and accumulator buffer free (tempty) -- are
// placed before MMA index WF / WT of tile t, so their latency hides behind
// queued tensor work instead of opening a bubble in the ~2-deep MMA queue.
// Index KS = after the whole tile (and its commits).  Measured at C4
// (tools/k3_waits.sh, profiles/r01_k3_waits.log): WF = KS-2, WT = KS-1 is
// 6 % faster than both before KS-2 (185.4 -> 173.5 ms); waiting for tempty
// after the tile costs 25 %.
template <int KS, int WF, int WT, int CS, int BNv, typename P>
__device__ __forceinline__ void mma_item_waits(
    const P &p, int ntiles, MmaState &s, uint64_t a_desc0, uint64_t b_desc0,
    uint32_t stage_step, uint32_t tmem, uint64_t *full, uint64_t *empty,
    uint64_t *tfull, uint64_t *tempty) {
  mbar_wait(&tempty[s.buf], ((s.tph >> s.buf) & 1u) ^ 1u);
  s.tph ^= 1u << s.buf;
  mbar_wait(&full[s.stage], s.ph);
  fence_after();
  for (int t = 0; t < ntiles; ++t) {
    constexpr uint32_t kNB = 512 / BNv;  // TMEM accumulator buffers
    const uint32_t d = tmem + s.buf * (uint32_t)BNv;
    const uint64_t b0 = b_desc0 + (uint64_t)(s.stage * stage_step);
    const uint32_t nbuf = s.buf + 1u == kNB ? 0u : s.buf + 1u;
    int nstage = s.stage + 1;
    uint32_t nph = s.ph;
    if (nstage == p.stages) {
      nstage = 0;
      nph ^= 1u;
    }
    const bool more = t + 1 < ntiles;
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) {
      if (ks == WT && more) {
        TR(0, s.tile_no + 1);
        mbar_wait(&tempty[nbuf], ((s.tph >> nbuf) & 1u) ^ 1u);
        TR(1, s.tile_no + 1);
        s.tph ^= 1u << nbuf;
        fence_after();
      }
      if (ks == WF && more) {
        mbar_wait(&full[nstage], nph);
        TR(2, s.tile_no + 1);
        fence_after();
      }
      constexpr uint32_t kA = 128 * 128 >> 4, kB = BNv * 128 >> 4;
      umma_f16(d, a_desc0 + (uint64_t)((ks >> 2) * kA + (ks & 3) * 2),
               b0 + (uint64_t)((ks >> 2) * kB + (ks & 3) * 2), p.idesc,
               ks > 0 ? 1u : 0u);
    }
    if constexpr (CS > 1)  // every cluster CTA's B stage (multicast)
      umma_commit_mc(&empty[s.stage], (uint16_t)((1u << CS) - 1));
    else
      umma_commit(&empty[s.stage]);
    umma_commit(&tfull[s.buf]);
    TR(3, s.tile_no);
    if (WT == KS && more) {
      TR(0, s.tile_no + 1);
      mbar_wait(&tempty[nbuf], ((s.tph >> nbuf) & 1u) ^ 1u);
      TR(1, s.tile_no + 1);
      s.tph ^= 1u << nbuf;
      fence_after();
    }
    if (WF == KS && more) {
      mbar_wait(&full[nstage], nph);
      TR(2, s.tile_no + 1);
      fence_after();
    }
    ++s.tile_no;
    s.buf = nbuf;
    s.stage = nstage;
    s.ph = nph;
  }
}



// AND of 32 words as a balanced tree (depth 5 instead of a 31-deep chain;
// the compiler fuses pairs of levels into 3-input LOP3s)
__device__ __forceinline__ uint32_t and32(const uint32_t (&r)[32]) {
  uint32_t a[16];
#pragma unroll
  for (int j = 0; j < 16; ++j) a[j] = r[j] & r[j + 16];
#pragma unroll
  for (int w = 8; w > 0; w >>= 1)
#pragma unroll
    for (int j = 0; j < w; ++j) a[j] &= a[j + w];
  return a[0];
}
#ifdef EXEM_TC_RELU_FMNMX
__device__ __forceinline__ void relu_acc_fmnmx(const uint32_t (&r)[32],
                                               float &se, float &so) {
#pragma unroll
  for (int j = 0; j < 32; j += 2) {
    se += fmaxf(__uint_as_float(r[j]), 0.f);
    so += fmaxf(__uint_as_float(r[j + 1]), 0.f);
  }
}
#endif
// acc.x += 2 max(0, r[2j]), acc.y += 2 max(0, r[2j+1]) in ascending j.
// x + |x| is exactly 2 max(0, x) (0 or 2x), and one FADD2 with the |.|
// operand modifier forms it for a register pair; a second FADD2 adds the
// pair to the two running sums.  FADD2 issues at half the FADD rate, so this
// runs at the FMNMX + FADD speed (tools/simt_peak.cu: 18.6 vs 18.3 T
// values/s) while keeping the ALU pipe free for the sign screens.  The
// doubled sums are halved once (exact), so they equal the FMNMX + FADD sums
// bit for bit unless a partial sum is subnormal.
// Four independent FADD2 chains per 32 values (pairs j = 4q + c go to chain
// c), combined in a fixed tree: the chain's latency, not the FADD2 issue
// rate, bounded a warp's relu-sum when most chunks fire (16 dependent FADD2
// per chunk behind each taken sign-screen branch).
__device__ __forceinline__ void relu_acc(const uint32_t (&r)[32],
                                         float2 &acc) {
#ifdef EXEM_TC_RELU_CHAIN1  // A/B experiment: one chain per 32 values
#pragma unroll
  for (int j = 0; j < 32; j += 2) {
    const float2 x = make_float2(__uint_as_float(r[j]),
                                 __uint_as_float(r[j + 1]));
    const float2 ax = make_float2(fabsf(x.x), fabsf(x.y));
    acc = __fadd2_rn(acc, __fadd2_rn(x, ax));
  }
#else
  float2 c[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const float2 x = make_float2(__uint_as_float(r[2 * q]),
                                 __uint_as_float(r[2 * q + 1]));
    c[q] = __fadd2_rn(x, make_float2(fabsf(x.x), fabsf(x.y)));
  }
#pragma unroll
  for (int j = 8; j < 32; j += 2) {
    const float2 x = make_float2(__uint_as_float(r[j]),
                                 __uint_as_float(r[j + 1]));
    const float2 ax = make_float2(fabsf(x.x), fabsf(x.y));
    c[(j >> 1) & 3] = __fadd2_rn(c[(j >> 1) & 3], __fadd2_rn(x, ax));
  }
  acc = __fadd2_rn(acc, __fadd2_rn(__fadd2_rn(c[0], c[1]),
                                   __fadd2_rn(c[2], c[3])));
#endif
}


// Timing-probe switches (EXEM_TC_DEBUG masks, EXEM_TC_WAITS) exist only in
// a probe build (-DEXEM_TC_PROBE_BUILD via EXEM_NVCC_FLAGS): even untaken,
// such branches in the issuer / epilogue loops can cost a large share of a
// step (K3 power wall).
#ifdef EXEM_TC_PROBE_BUILD
#define TC_PROBE(p, bit) (((p).dbg & (bit)) != 0)
#define TC_PROBE_ANY(p, mask) (((p).dbg & (mask)) != 0)
#define TC_WAIT_SPIN(p) (((p).wait_mode & 8) != 0)
#else
#define TC_PROBE(p, bit) false
#define TC_PROBE_ANY(p, mask) false
#define TC_WAIT_SPIN(p) false
#endif

struct Params {
  int64_t l;            // candidates
  int64_t n;            // points of this shard
  int64_t split_pts;    // points per split (multiple of BN)
  int64_t splits;
  int64_t cand_tiles;
  int ksteps;           // K=16 MMA steps  (ceil((d+6)/16))
  int kchunks;          // 64-wide K chunks loaded per operand tile
  int stages;           // B pipeline depth (in K chunks)
  int dbg;              // timing experiments only (EXEM_TC_DEBUG), 0 in use
  int wait_mode;        // timing experiments: 8 = epilogue spins on tfull (EXEM_TC_WAITS)
  int tile_stage;       // 1: a pipeline stage holds a whole B tile
  uint32_t idesc;
  double *partial;
  long long *trace;     // timing experiments only (EXEM_TC_TRACE)
  // optional: += number of (candidate row, 32-point chunk) screens that
  // found a value >= +0 (the relu-sum work actually done; the host uses it
  // to pick the epilogue width Q for the following steps)
  unsigned long long *hits;
};

// kCS > 1: kCS-CTA cluster; the CTAs score adjacent candidate tiles against
// the same point tiles, each loading 1/kCS of every B tile and multicasting
// it to all (1/kCS of the L2 -> SM traffic for B, less power, a higher
// clock under the cap); a B stage is refilled only when every CTA's MMAs
// released it (empty barriers count kCS, commits multicast).  map_ph: the
// point operand with 256/kCS-row boxes.
// kBN: points per tile = TMEM columns per accumulator buffer; 512 / kBN
// buffers.  256 (two buffers) in use; 128 (four buffers) is a timing
// experiment (EXEM_TC_BN=128), measured slower at small d.
template <bool kAStream, int kCS, int kQ, int kBN>
__global__ void __launch_bounds__(Epi<kQ, kBN>::kThreads, 1)
    gains_tc_kernel(const __grid_constant__ CUtensorMap map_c,
                    const __grid_constant__ CUtensorMap map_p,
                    const __grid_constant__ CUtensorMap map_ph,
                    const Params p) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  // 1024-align the dynamic smem base (swizzle atoms).
  unsigned char *smem = (unsigned char *)(((uintptr_t)smem_raw + 1023) &
                                          ~(uintptr_t)1023);
  constexpr int kBChunk = kBN * 128;   // bytes of one B K-chunk
  constexpr int kNB = 512 / kBN;       // TMEM accumulator buffers
  const int a_bytes = kAStream ? 0 : p.kchunks * A_CHUNK;
  const int stage_bytes =
      p.tile_stage ? p.kchunks * kBChunk : kBChunk + (kAStream ? A_CHUNK : 0);
  unsigned char *sa = smem;                      // stationary A chunks
  unsigned char *sb = smem + a_bytes;            // stages
  uint64_t *bars = (uint64_t *)(sb + p.stages * stage_bytes);
  uint64_t *full = bars;                         // [stages]
  uint64_t *empty = bars + p.stages;             // [stages]
  uint64_t *tfull = bars + 2 * p.stages;         // [kNB]
  uint64_t *tempty = tfull + kNB;                // [kNB]
  uint64_t *afull = tempty + kNB;                // [1]
  uint64_t *aempty = afull + 1;                  // [1]
  uint32_t *tmem_slot = (uint32_t *)(aempty + 1);
  double *red = (double *)(tmem_slot + 4);       // [BM] half-merge buffer

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int kEpiCols = Epi<kQ, kBN>::kCols;
  constexpr int kEpiWarps = Epi<kQ, kBN>::kWarps;
  constexpr int kProdWarp = Epi<kQ, kBN>::kProdWarp;
  constexpr int kMmaWarp = Epi<kQ, kBN>::kMmaWarp;

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < p.stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kCS);
    }
    for (int b = 0; b < kNB; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], kEpiWarps);
    }
    mbar_init(afull, 1);
    mbar_init(aempty, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&map_c));
    asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&map_p));
  }
  if (warp == kMmaWarp) {
    asm volatile(
        "tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::
            "r"(su32(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  fence_before();
  __syncthreads();
  if constexpr (kCS > 1) cluster_sync();  // peers' barriers initialised
  fence_after();
  const uint32_t tmem = *tmem_slot;

  // work item = (split, candidate unit); a unit is one candidate tile, or
  // with clusters kCS adjacent tiles (CTA rank r of the cluster takes
  // kCS*u + r)
  const uint32_t crank = kCS > 1 ? cluster_rank() : 0u;
  const int64_t cunits = (p.cand_tiles + kCS - 1) / kCS;
  const int64_t wid = blockIdx.x / kCS;
  const int64_t nwork = gridDim.x / kCS;
  const int64_t items = cunits * p.splits;

  if (warp == kProdWarp) {
    // ------------------------------------------------------------ producer
    if (lane == 0) {
      int stage = 0;
      uint32_t ph = 0, aph = 0;
      for (int64_t it = wid; it < items; it += nwork) {
        const int64_t ct = kCS * (it % cunits) + crank;
        const int64_t sp = it / cunits;
        const int crow = (int)(ct * BM);
        if (!kAStream) {
          mbar_wait(aempty, aph ^ 1);
          aph ^= 1;
          mbar_expect_tx(afull, (uint32_t)(p.kchunks * A_CHUNK));
          for (int kc = 0; kc < p.kchunks; ++kc)
            tma_load_2d(sa + kc * A_CHUNK, &map_c, afull, kc * KCH, crow);
        }
        const int64_t p0 = sp * p.split_pts;
        const int64_t p1 = min(p.n, p0 + p.split_pts);
        for (int64_t pt = p0; pt < p1; pt += kBN) {
          // whole-tile stages: one stage = every K chunk of the B tile
          const int per_stage = p.tile_stage ? p.kchunks : 1;
          for (int kc0 = 0; kc0 < p.kchunks; kc0 += per_stage) {
            if (!TC_PROBE(p, 16)) mbar_wait_sleep(&empty[stage], ph ^ 1);
            unsigned char *dst = sb + stage * stage_bytes;
            if (TC_PROBE(p, 4)) {  // timing experiment: no operand traffic
              mbar_arrive(&full[stage]);
            } else if (kCS > 1) {
              // this CTA's 1/kCS of the B tile, to every CTA of the cluster
              mbar_expect_tx(&full[stage], (uint32_t)stage_bytes);
              for (int j = 0; j < per_stage; ++j)
                tma_load_2d_mc(dst + j * kBChunk + crank * (kBChunk / kCS),
                               &map_ph, &full[stage], (kc0 + j) * KCH,
                               (int)(pt + crank * (kBN / kCS)),
                               (uint16_t)((1u << kCS) - 1));
            } else {
              mbar_expect_tx(&full[stage], (uint32_t)stage_bytes);
              for (int j = 0; j < per_stage; ++j)
                tma_load_2d(dst + j * kBChunk, &map_p, &full[stage],
                            (kc0 + j) * KCH, (int)pt);
              if (kAStream)
                tma_load_2d(dst + kBChunk, &map_c, &full[stage], kc0 * KCH,
                            crow);
            }
            if (++stage == p.stages) {
              stage = 0;
              ph ^= 1;
            }
          }
        }
      }
    }
  } else if (warp == kMmaWarp) {
    // ------------------------------------------------------------ MMA issuer
    // One thread runs the whole role.  With whole-tile stages the K-steps of
    // a tile are issued back to back after a single barrier wait; the
    // timeline tool (EXEM_TC_TRACE, tools/tc_trace.py) showed per-chunk
    // synchronisation inside a tile costing ~2x in tensor-pipe time.
    if (lane == 0) {
      const uint64_t a_desc0 = sw128_desc(su32(sa));
      const uint64_t b_desc0 = sw128_desc(su32(sb));
      const uint32_t stage_step = (uint32_t)(stage_bytes >> 4);
      int stage = 0;
      uint32_t ph = 0, aph = 0, tph = 0;  // tph: bit b = phase of buffer b
      uint32_t buf = 0;
      int tile_no = 0;
      for (int64_t it = wid; it < items; it += nwork) {
        const int64_t sp = it / cunits;
        if (!kAStream) {
          mbar_wait(afull, aph);
          aph ^= 1;
        }
        const int64_t p0 = sp * p.split_pts;
        const int64_t p1 = min(p.n, p0 + p.split_pts);
        if (p.tile_stage && p.ksteps <= 8 && !TC_PROBE_ANY(p, ~5)) {
          // software-pipelined handshake (see mma_item_waits)
          const int ntiles = (int)((p1 - p0 + kBN - 1) / kBN);
          MmaState ms{stage, ph, tph, buf, tile_no};
          const uint32_t st_step = stage_step;
          switch (p.ksteps) {
#define EXEM_K3_ITEM(K)                                                       \
  case K:                                                                     \
    mma_item_waits<K, (K > 2 ? K - 2 : 0), (K > 1 ? K - 1 : 0), kCS, kBN>(   \
        p, ntiles, ms, a_desc0, b_desc0, st_step, tmem, full, empty, tfull,   \
        tempty);                                                              \
    break;
            EXEM_K3_ITEM(1) EXEM_K3_ITEM(2) EXEM_K3_ITEM(3) EXEM_K3_ITEM(4)
            EXEM_K3_ITEM(5) EXEM_K3_ITEM(6) EXEM_K3_ITEM(7)
            default: EXEM_K3_ITEM(8)
#undef EXEM_K3_ITEM
          }
          stage = ms.stage;
          ph = ms.ph;
          tph = ms.tph;
          buf = ms.buf;
          tile_no = ms.tile_no;
        }
        for (int64_t pt = p0;
             pt < p1 && !(p.tile_stage && p.ksteps <= 8 && !TC_PROBE_ANY(p, ~5));
             pt += kBN) {
          TR(0, tile_no);
          mbar_wait(&tempty[buf], ((tph >> buf) & 1u) ^ 1u);
          TR(1, tile_no);
          tph ^= 1u << buf;
          fence_after();  // TMEM WAR vs the epilogue's tcgen05.ld
          const uint32_t dcol = tmem + buf * (uint32_t)kBN;
          if (p.tile_stage) {
            if (!TC_PROBE(p, 8)) mbar_wait(&full[stage], ph);
            TR(2, tile_no);
            const uint64_t bd0 = b_desc0 + (uint64_t)((TC_PROBE(p, 128) ? 0 : stage) * stage_step);
            if (!TC_PROBE(p, 2)) {
              switch (p.ksteps) {  // compile-time K for d <= 122
                case 1: issue_tile<1, kBN>(dcol, a_desc0, bd0, p.idesc); break;
                case 2: issue_tile<2, kBN>(dcol, a_desc0, bd0, p.idesc); break;
                case 3: issue_tile<3, kBN>(dcol, a_desc0, bd0, p.idesc); break;
                case 4: issue_tile<4, kBN>(dcol, a_desc0, bd0, p.idesc); break;
                case 5: issue_tile<5, kBN>(dcol, a_desc0, bd0, p.idesc); break;
                case 6: issue_tile<6, kBN>(dcol, a_desc0, bd0, p.idesc); break;
                case 7: issue_tile<7, kBN>(dcol, a_desc0, bd0, p.idesc); break;
                case 8: issue_tile<8, kBN>(dcol, a_desc0, bd0, p.idesc); break;
                default:
#pragma unroll 1
                  for (int ks = 0; ks < p.ksteps; ++ks) {
                    const uint32_t off_a = (uint32_t)((ks >> 2) * (A_CHUNK >> 4) + (ks & 3) * 2);
                    const uint32_t off_b = (uint32_t)((ks >> 2) * (kBChunk >> 4) + (ks & 3) * 2);
                    umma_f16(dcol, a_desc0 + off_a, bd0 + off_b, p.idesc,
                             ks > 0 ? 1u : 0u);
                  }
              }
            }
            if (!TC_PROBE(p, 16)) {
              if constexpr (kCS > 1)
                umma_commit_mc(&empty[stage], (uint16_t)((1u << kCS) - 1));
              else umma_commit(&empty[stage]);
            }
            if (++stage == p.stages) {
              stage = 0;
              ph ^= 1;
            }
          } else {
            int ks_left = p.ksteps;
            for (int kc = 0; kc < p.kchunks; ++kc) {
              mbar_wait(&full[stage], ph);
              if (kc == 0) TR(2, tile_no);
              const uint64_t bd = b_desc0 + (uint64_t)(stage * stage_step);
              const uint64_t ad =
                  kAStream ? bd + (uint64_t)(kBChunk >> 4)
                           : a_desc0 + (uint64_t)(kc * (A_CHUNK >> 4));
              const int nk = ks_left < KCH / 16 ? ks_left : KCH / 16;
              if (!TC_PROBE(p, 2)) {
                // whole chunks from compile-time unrolled code (the single
                // issuing thread is the critical path; K4-TC measured 1.06-
                // 1.31x from this), the runtime loop only for a ragged tail
                if (nk == KCH / 16) {
#pragma unroll
                  for (int j = 0; j < KCH / 16; ++j)
                    umma_f16(dcol, ad + (uint64_t)(2 * j),
                             bd + (uint64_t)(2 * j), p.idesc,
                             (kc | j) ? 1u : 0u);
                } else {
#pragma unroll 1
                  for (int j = 0; j < nk; ++j)
                    umma_f16(dcol, ad + (uint64_t)(2 * j),
                             bd + (uint64_t)(2 * j), p.idesc,
                             (kc | j) ? 1u : 0u);
                }
              }
              ks_left -= KCH / 16;
              if constexpr (kCS > 1)
                umma_commit_mc(&empty[stage], (uint16_t)((1u << kCS) - 1));
              else umma_commit(&empty[stage]);
              if (++stage == p.stages) {
                stage = 0;
                ph ^= 1;
              }
            }
          }
          umma_commit(&tfull[buf]);
          TR(3, tile_no);
          ++tile_no;
          buf = buf + 1u == (uint32_t)kNB ? 0u : buf + 1u;
        }
        if (!kAStream) umma_commit(aempty);
      }
    }
    __syncwarp();
  } else {
    // ------------------------------------------------------------ epilogue
    const int ew = warp;                // 0..kEpiWarps-1
    const int q = warp & 3;             // TMEM lane quarter of this warp
    const int grp = ew >> 2;            // column group of the 256-wide tile
    const int row = q * 32 + lane;      // candidate row within the tile
    uint32_t buf = 0, tph = 0;  // tph: bit b = phase of buffer b
    int tile_no = 0;
    uint32_t nhit = 0;
    const bool tr = (warp == 0 && lane == 0);
    for (int64_t it = wid; it < items; it += nwork) {
      const int64_t ct = kCS * (it % cunits) + crank;
      const int64_t sp = it / cunits;
      const int64_t p0 = sp * p.split_pts;
      const int64_t p1 = min(p.n, p0 + p.split_pts);
      double g = 0.0;
      for (int64_t pt = p0; pt < p1; pt += kBN) {
        if (tr) TR(4, tile_no);
        // one lane polls the barrier; the warp sync orders the others
        if (lane == 0) {
          if (TC_WAIT_SPIN(p))
            mbar_wait(&tfull[buf], (tph >> buf) & 1u);
          else
#ifdef EXEM_TC_EPI_SLEEP  // A/B experiment: nanosleep back-off (round 1)
            mbar_wait_sleep(&tfull[buf], (tph >> buf) & 1u);
#else
            mbar_wait_hint(&tfull[buf], (tph >> buf) & 1u);
#endif
        }
        __syncwarp();
        if (tr) TR(5, tile_no);
        tph ^= 1u << buf;
        fence_after();
        const uint32_t taddr = tmem + ((uint32_t)(q * 32) << 16) +
                               (uint32_t)(buf * kBN + grp * kEpiCols);
        // Drain this warp's 32 x kEpiCols slice of the accumulator into
        // registers first and release the TMEM buffer immediately, so the
        // MMA of tile t+kNB never waits on this tile's arithmetic.
        uint32_t r[kEpiCols / 32][32];
#pragma unroll
        for (int c = 0; c < kEpiCols / 32; ++c) TMEM_LD32(taddr + 32 * c, r[c]);
        tmem_wait_ld();
        fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[buf]);
        if (tr) TR(6, tile_no);
        if (TC_PROBE(p, 1)) {  // timing experiment: no epilogue arithmetic
          g += (double)__uint_as_float(r[0][0] ^ r[kEpiCols / 32 - 1][31]);
          buf = buf + 1u == (uint32_t)kNB ? 0u : buf + 1u;
          ++tile_no;
          continue;
        }
        // relu-sum with a sign-bit screen: max(0, D) contributes only where
        // D >= +0, and almost every (candidate, point) pair has D < 0 (a
        // candidate helps only points closer to it than their current
        // exemplar).  AND-ing the raw bits of 32 values (LOP3, 3 inputs per
        // op) leaves the sign bit set iff all 32 are negative, so the relu
        // work runs only for chunks that can contribute.  Skipped chunks
        // would only have added +0, so the sums are bit-identical.
#ifdef EXEM_TC_RELU_FMNMX  // A/B experiment: FMNMX + FADD per value
        float s[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int c = 0; c < kEpiCols / 32; ++c)
          if ((int)and32(r[c]) >= 0)
            relu_acc_fmnmx(r[c], s[2 * (c & 1)], s[2 * (c & 1) + 1]);
        g += (double)((s[0] + s[1]) + (s[2] + s[3]));
#else
        // one pair of running sums per 32-column chunk (independent FADD2
        // chains), combined in a fixed tree
        constexpr int NC = kEpiCols / 32;
        float2 a[NC];
#pragma unroll
        for (int c = 0; c < NC; ++c) {
          a[c] = make_float2(0.f, 0.f);
          if ((int)and32(r[c]) >= 0) {
            relu_acc(r[c], a[c]);
            ++nhit;
          }
        }
        float sc[NC];
#pragma unroll
        for (int c = 0; c < NC; ++c) sc[c] = a[c].x + a[c].y;
#pragma unroll
        for (int w = NC / 2; w > 0; w >>= 1)
#pragma unroll
          for (int c = 0; c < w; ++c) sc[c] = sc[c] + sc[c + w];
        g += (double)(sc[0] * 0.5f);
#endif
        if (tr) TR(7, tile_no);
        ++tile_no;
        buf = buf + 1u == (uint32_t)kNB ? 0u : buf + 1u;
      }
      // fixed-order merge of the column groups: ((g0 + g1) + g2) + g3
      // through one [BM] buffer
#pragma unroll 1
      for (int gq = 1; gq < kQ; ++gq) {
        if (grp == gq) red[row] = g;
        asm volatile("bar.sync 1, %0;" ::"n"(kEpiWarps * 32) : "memory");
        if (grp == 0) g += red[row];
        asm volatile("bar.sync 1, %0;" ::"n"(kEpiWarps * 32) : "memory");
      }
      if (grp == 0) {
        const int64_t c = ct * BM + row;
        if (c < p.l) p.partial[sp * p.l + c] = g;
      }
    }
    if (p.hits) {
      const uint32_t w = __reduce_add_sync(0xffffffffu, nhit);
      if (lane == 0 && w) atomicAdd(p.hits, (unsigned long long)w);
    }
  }

  fence_before();
  __syncthreads();
  if constexpr (kCS > 1) cluster_sync();  // no multicast / commit in flight
  if (warp == kMmaWarp) {
    fence_after();
    asm volatile(
        "tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

// ---------------------------------------------------------------- packing
// Transposes the SIMT layout vt[d_pad][ld] into point-major half rows and
// appends the folded constant columns (see header comment).
template <int DT, bool kCand, bool VS>
__global__ void pack_kernel(const typename VtOf<DT, VS>::T *__restrict__ vt,
                            int64_t ld,
                            int64_t n, int d, const double *__restrict__ norms,
                            const float *__restrict__ m,
                            typename Traits<DT>::S *__restrict__ x, int64_t kp,
                            int64_t rows) {
  using S = typename Traits<DT>::S;
  __shared__ float tile[32][33];
  const int64_t r0 = (int64_t)blockIdx.x * 32;
  const int k0 = blockIdx.y * 32;
  // load vt[k0+ty][r0+tx] (coalesced along points)
  for (int ty = threadIdx.y; ty < 32; ty += blockDim.y) {
    const int k = k0 + ty;
    const int64_t r = r0 + threadIdx.x;
    tile[ty][threadIdx.x] = (k < d && r < n) ? to_c(vt[(int64_t)k * ld + r]) : 0.f;
  }
  __syncthreads();
  for (int ty = threadIdx.y; ty < 32; ty += blockDim.y) {
    const int64_t r = r0 + ty;
    const int k = k0 + threadIdx.x;
    if (r >= rows || k >= kp) continue;
    double v = 0.0;
    if (r < n) {
      if (k < d) {
        v = (double)tile[threadIdx.x][ty];
      } else if (k < d + kTcConst) {
        const int c = k - d;
        const bool ones = kCand ? (c < 3) : (c >= 3);
        if (ones) {
          v = fold_one<S>(kCand ? c : c - 3);
        } else {
          const double t = kCand ? 0.5 * norms[r]
                                 : 0.5 * (norms[r] - (m ? (double)m[r] : 0.0));
          double p[3];
          fold_pieces<S>(t, p);
          v = -p[kCand ? c - 3 : c];
        }
      }
    }
    x[r * kp + k] = from_d<S>(v);
  }
}


// ------------------------------------------- split-bf16 binary32 operands
// An fp32 value x is split into three bf16 pieces x0 + x1 + x2 (x0 = bf16(x),
// x1 = bf16(x - x0), x2 = bf16(x - x0 - x1): 24 significant bits, exact for
// binary32).  Laying the pieces out along K as
//   candidate row  [c0, c0, c1, c0, c1, c2, 1,1,1, -b0,-b1,-b2, 0..]
//   point row      [v0, v1, v0, v2, v1, v0, -h0,-h1,-h2, 1,1,1, 0..]
// makes one bf16 row-dot over K' = 6d+6 equal to
//   c.v (all piece products with i+j <= 2; each is exact in fp32, the dropped
//   ones are < 2^-24 relative) - h - b,
// i.e. the K3 quantity D at binary32 accuracy on the tensor cores: the
// unchanged gains_tc_kernel runs on these rows with "d" = 6d.
__device__ __forceinline__ void split3(float x, __nv_bfloat16 (&o)[3]) {
  o[0] = __float2bfloat16_rn(x);
  const float r1 = x - __bfloat162float(o[0]);
  o[1] = __float2bfloat16_rn(r1);
  o[2] = __float2bfloat16_rn(r1 - __bfloat162float(o[1]));
}

template <bool kCand>
__global__ void pack_split3_kernel(const float *__restrict__ vt, int64_t ld,
                                   int64_t n, int d,
                                   const double *__restrict__ norms,
                                   const float *__restrict__ m,
                                   __nv_bfloat16 *__restrict__ x, int64_t kp,
                                   int64_t rows) {
  // piece order of the six d-wide segments (see above)
  constexpr int kCandPiece[6] = {0, 0, 1, 0, 1, 2};
  constexpr int kPointPiece[6] = {0, 1, 0, 2, 1, 0};
  const int64_t r = (int64_t)blockIdx.x * blockDim.y + threadIdx.y;
  if (r >= rows) return;
  __nv_bfloat16 *row = x + r * kp;
  const __nv_bfloat16 zero = __float2bfloat16_rn(0.f);
  for (int64_t k = threadIdx.x; k < kp; k += blockDim.x) {
    __nv_bfloat16 v = zero;
    if (r < n) {
      if (k < 6 * (int64_t)d) {
        const int seg = (int)(k / d), dim = (int)(k % d);
        __nv_bfloat16 pc[3];
        split3(vt[(int64_t)dim * ld + r], pc);
        v = pc[kCand ? kCandPiece[seg] : kPointPiece[seg]];
      } else if (k < 6 * (int64_t)d + kTcConst) {
        const int c = (int)(k - 6 * (int64_t)d);
        const bool ones = kCand ? (c < 3) : (c >= 3);
        if (ones) {
          v = __float2bfloat16_rn(1.f);
        } else {
          const double t = kCand ? 0.5 * norms[r]
                                 : 0.5 * (norms[r] - (m ? (double)m[r] : 0.0));
          const double t0 = (double)__bfloat162float(__double2bfloat16(t));
          const double t1 = (double)__bfloat162float(__double2bfloat16(t - t0));
          const double t2 =
              (double)__bfloat162float(__double2bfloat16(t - t0 - t1));
          const int piece = kCand ? c - 3 : c;
          v = __double2bfloat16(-(piece == 0 ? t0 : (piece == 1 ? t1 : t2)));
        }
      }
    }
    row[k] = v;
  }
}

// Rewrite only the three -h columns (at column hcol) of point rows after an
// m-update: h_i = (||v_i||^2 - m_i)/2 in three bf16 pieces.
__global__ void refresh_h_kernel(const double *__restrict__ norms,
                                 const float *__restrict__ m, int64_t n,
                                 __nv_bfloat16 *__restrict__ x, int64_t kp,
                                 int64_t hcol) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double h = 0.5 * (norms[i] - (double)m[i]);
  const double t0 = (double)__bfloat162float(__double2bfloat16(h));
  const double t1 = (double)__bfloat162float(__double2bfloat16(h - t0));
  const double t2 = (double)__bfloat162float(__double2bfloat16(h - t0 - t1));
  __nv_bfloat16 *row = x + i * kp + hcol;
  row[0] = __double2bfloat16(-t0);
  row[1] = __double2bfloat16(-t1);
  row[2] = __double2bfloat16(-t2);
}

}  // namespace tc
}  // namespace exem

using namespace exem;

extern "C" {

int exem_tc_pack_candidates(int dtype, const void *vt, int64_t ld, int64_t n,
                            int64_t d, const double *norms, void *xc,
                            void *stream) {
  const int tag = dtype & ~EXEM_VT_STORAGE;
  if (tag != EXEM_BF16 && tag != EXEM_F16)
    return fail(EXEM_ERR_ARG, "TC operands are bf16/f16 only");
  const int64_t kp = exem_tc_kp(d), rows = exem_tc_rows(n);
  dim3 grid((unsigned)ceil_div(rows, 32), (unsigned)ceil_div(kp, 32));
  dim3 block(32, 8);
  cudaStream_t st = (cudaStream_t)stream;
  const bool vs = (dtype & EXEM_VT_STORAGE) != 0;
#define EXEM_PACK(DT, VS)                                                    \
  tc::pack_kernel<DT, true, VS><<<grid, block, 0, st>>>(                     \
      (const typename VtOf<DT, VS>::T *)vt, ld, n, (int)d, norms, nullptr,   \
      (typename Traits<DT>::S *)xc, kp, rows)
  if (tag == EXEM_BF16) {
    if (vs) EXEM_PACK(EXEM_BF16, true); else EXEM_PACK(EXEM_BF16, false);
  } else {
    if (vs) EXEM_PACK(EXEM_F16, true); else EXEM_PACK(EXEM_F16, false);
  }
#undef EXEM_PACK
  EXEM_LAUNCH_CHECK("tc_pack_candidates");
  return EXEM_OK;
}

int exem_tc_pack_points(int dtype, const void *vt, int64_t ld, int64_t n,
                        int64_t d, const double *norms, const void *m,
                        void *xp, void *stream) {
  const int tag = dtype & ~EXEM_VT_STORAGE;
  if (tag != EXEM_BF16 && tag != EXEM_F16)
    return fail(EXEM_ERR_ARG, "TC operands are bf16/f16 only");
  const int64_t kp = exem_tc_kp(d), rows = exem_tc_rows(n);
  dim3 grid((unsigned)ceil_div(rows, 32), (unsigned)ceil_div(kp, 32));
  dim3 block(32, 8);
  cudaStream_t st = (cudaStream_t)stream;
  const bool vs = (dtype & EXEM_VT_STORAGE) != 0;
#define EXEM_PACK(DT, VS)                                                    \
  tc::pack_kernel<DT, false, VS><<<grid, block, 0, st>>>(                    \
      (const typename VtOf<DT, VS>::T *)vt, ld, n, (int)d, norms,            \
      (const float *)m, (typename Traits<DT>::S *)xp, kp, rows)
  if (tag == EXEM_BF16) {
    if (vs) EXEM_PACK(EXEM_BF16, true); else EXEM_PACK(EXEM_BF16, false);
  } else {
    if (vs) EXEM_PACK(EXEM_F16, true); else EXEM_PACK(EXEM_F16, false);
  }
#undef EXEM_PACK
  EXEM_LAUNCH_CHECK("tc_pack_points");
  return EXEM_OK;
}

int exem_greedy_gains_tc(int dtype, const void *xc, int64_t l, const void *xp,
                         int64_t n, int64_t d, int64_t split_pts,
                         double *partial, int64_t splits, void *stream) {
  return exem_greedy_gains_tc_ex(dtype, xc, l, xp, n, d, split_pts, partial,
                                 splits, 0, nullptr, stream);
}

int exem_greedy_gains_tc_ex(int dtype, const void *xc, int64_t l,
                            const void *xp, int64_t n, int64_t d,
                            int64_t split_pts, double *partial, int64_t splits,
                            int epi_groups, unsigned long long *screen_hits,
                            void *stream) {
  using namespace exem::tc;
  if (epi_groups != 0 && epi_groups != 2 && epi_groups != 4)
    return fail(EXEM_ERR_ARG, "epi_groups must be 0 (default), 2 or 4");
  const int q = epi_groups == 4 ? 4 : 2;
  if (dtype != EXEM_BF16 && dtype != EXEM_F16)
    return fail(EXEM_ERR_ARG, "greedy_gains_tc is bf16/f16 only");
  if (split_pts < BN || split_pts % BN)
    return fail(EXEM_ERR_ARG, "split_pts must be a multiple of %d", BN);
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
  const int64_t kp = exem_tc_kp(d);
  const int kchunks = (int)(kp / KCH);
  const int ksteps = (int)ceil_div(d + kTcConst, 16);
  Params prm;
  prm.l = l;
  prm.n = n;
  prm.split_pts = split_pts;
  prm.splits = splits;
  prm.cand_tiles = ceil_div(l, BM);
  prm.ksteps = ksteps;
  prm.kchunks = kchunks;
  prm.partial = partial;
  prm.hits = screen_hits;
  {
    const char *dbg = getenv("EXEM_TC_DEBUG");
    prm.dbg = dbg ? atoi(dbg) : 0;
    const char *wm = getenv("EXEM_TC_WAITS");
    prm.wait_mode = wm ? atoi(wm) : 0;
  }
  prm.trace = nullptr;
  const char *trace_path = getenv("EXEM_TC_TRACE");
  if (trace_path) {
    cudaMalloc(&prm.trace, 16 * kTrace * sizeof(long long));
    cudaMemset(prm.trace, 0, 16 * kTrace * sizeof(long long));
  }
  // A stationary when it leaves room for >= 3 B chunk stages.
  const int avail = kSmemBudget - kBarBytes - 1024;
  const bool astream = (avail - kchunks * A_CHUNK) / B_CHUNK < 3;
  // Whole-tile stages (one barrier handshake per B tile) when >= 3 fit.
  const bool tile_stage =
      !astream && (avail - kchunks * A_CHUNK) / (kchunks * B_CHUNK) >= 3;
  // 256-point tiles in two TMEM buffers.  EXEM_TC_BN = 128 (timing
  // experiments, whole-tile stages only) runs 128-point tiles in four
  // buffers: measured slower even at d = 2 / 16 / 20 (1.92 / 2.02 / 2.02 vs
  // 1.51 / 1.53 / 1.53 ms per C3 step) -- the per-tile epilogue cost, not
  // the two-buffer release chain, bounds the small-d tiles.
  int bn = BN;
  if (const char *eb = getenv("EXEM_TC_BN"))
    if (tile_stage && !astream && atoi(eb) == 128) bn = 128;
  prm.idesc = make_idesc(dtype == EXEM_BF16, BM, bn);
  const int b_chunk = bn * 128;
  const int stage_bytes = tile_stage ? kchunks * b_chunk
                                     : b_chunk + (astream ? A_CHUNK : 0);
  int stages = (avail - (astream ? 0 : kchunks * A_CHUNK)) / stage_bytes;
  if (stages > 8) stages = 8;
  if (const char *ms = getenv("EXEM_TC_STAGES")) stages = atoi(ms);  // timing only
  prm.stages = stages;
  prm.tile_stage = tile_stage ? 1 : 0;
  const size_t smem = (size_t)(astream ? 0 : kchunks * A_CHUNK) +
                      (size_t)stages * stage_bytes + kBarBytes + 1024;
  CUtensorMap mc, mp;
  if (int rc = make_map(&mc, xc, dtype, exem_tc_rows(l), kp, BM)) return rc;
  if (int rc = make_map(&mp, xp, dtype, exem_tc_rows(n), kp, bn)) return rc;
  // clusters sharing B tiles by TMA multicast (whole-tile stages, the
  // pipelined issuer): cluster size 2 by default, EXEM_TC_MC = 0 | 1 | 2 | 4
  // (0/1: none) for timing experiments
  int cs = (tile_stage && !astream && ksteps <= 8 && prm.dbg == 0) ? 2 : 1;
  if (const char *e = getenv("EXEM_TC_MC"))
    if (cs > 1) cs = atoi(e) >= 4 ? 4 : (atoi(e) >= 2 ? 2 : 1);
  if (bn != BN && cs > 2) cs = 2;  // the narrow tiles have pairs only
  const bool mcast = cs > 1;
  CUtensorMap mph;  // bn/cs-row boxes: one CTA's share of a B tile
  if (int rc = make_map(&mph, xp, dtype, exem_tc_rows(n), kp, bn / cs))
    return rc;
  cudaStream_t st = (cudaStream_t)stream;
  cudaError_t e;
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute at[1];
  cfg.blockDim = dim3(q == 4 ? Epi<4>::kThreads : Epi<2>::kThreads);  // any BN
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  // one kernel instantiation per (A streamed, cluster size, Q, tile width)
  auto pick = [&](bool as, int c) {
#define EXEM_K3_PICK(AS, CS, B)                                               \
  (q == 4 ? gains_tc_kernel<AS, CS, 4, B> : gains_tc_kernel<AS, CS, 2, B>)
    if (bn == 128)
      return c == 2 ? EXEM_K3_PICK(false, 2, 128) : EXEM_K3_PICK(false, 1, 128);
    return as ? EXEM_K3_PICK(true, 1, BN)
              : (c == 4 ? EXEM_K3_PICK(false, 4, BN)
                        : (c == 2 ? EXEM_K3_PICK(false, 2, BN)
                                  : EXEM_K3_PICK(false, 1, BN)));
#undef EXEM_K3_PICK
  };
  auto kern = pick(astream, cs);
  e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)smem);
  if (e != cudaSuccess)
    return fail(EXEM_ERR_CUDA, "smem attr: %s", cudaGetErrorString(e));
  if (mcast) {
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cs;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cfg.gridDim = dim3((unsigned)(sms / cs * cs));
    int clusters = 0;
    e = cudaOccupancyMaxActiveClusters(&clusters, kern, &cfg);
    if (e != cudaSuccess || clusters < 1)
      return fail(EXEM_ERR_CUDA, "no co-resident CTA clusters: %s",
                  cudaGetErrorString(e));
    const int64_t units = (prm.cand_tiles + cs - 1) / cs * splits;
    cfg.gridDim = dim3((unsigned)(cs * (units < clusters ? units : clusters)));
    e = cudaLaunchKernelEx(&cfg, kern, mc, mp, mph, prm);
  } else {
    const int64_t items = prm.cand_tiles * splits;
    cfg.gridDim = dim3((unsigned)(items < sms ? items : sms));
    e = cudaLaunchKernelEx(&cfg, kern, mc, mp, mph, prm);
  }
  if (e != cudaSuccess)
    return fail(EXEM_ERR_CUDA, "gains_tc_kernel launch: %s",
                cudaGetErrorString(e));
  EXEM_LAUNCH_CHECK("gains_tc_kernel");
  if (prm.trace) {  // timing experiment: dump the CTA-0 timeline
    static long long host[16 * kTrace];
    cudaStreamSynchronize(st);
    cudaMemcpy(host, prm.trace, sizeof(host), cudaMemcpyDeviceToHost);
    cudaFree(prm.trace);
    if (FILE *f = fopen(trace_path, "w")) {
      for (int t = 0; t < kTrace; ++t) {
        for (int s = 0; s < 10; ++s)
          fprintf(f, "%lld%c", host[s * kTrace + t], s == 9 ? '\n' : ' ');
      }
      fclose(f);
    }
  }
  return EXEM_OK;
}

int64_t exem_tc_split_dim(int64_t d) { return 6 * d; }

int exem_tc_pack_split(int role, const void *vt, int64_t ld, int64_t n,
                       int64_t d, const double *norms, const void *m,
                       void *x, void *stream) {
  if (n < 1 || d < 1) return fail(EXEM_ERR_ARG, "tc_pack_split: bad shape");
  const int64_t kp = exem_tc_kp(6 * d), rows = exem_tc_rows(n);
  dim3 block(64, 4);
  dim3 grid((unsigned)ceil_div(rows, 4));
  cudaStream_t st = (cudaStream_t)stream;
  if (role == 0)
    tc::pack_split3_kernel<true><<<grid, block, 0, st>>>(
        (const float *)vt, ld, n, (int)d, norms, nullptr, (__nv_bfloat16 *)x,
        kp, rows);
  else
    tc::pack_split3_kernel<false><<<grid, block, 0, st>>>(
        (const float *)vt, ld, n, (int)d, norms, (const float *)m,
        (__nv_bfloat16 *)x, kp, rows);
  EXEM_LAUNCH_CHECK("tc_pack_split");
  return EXEM_OK;
}

int exem_tc_refresh_h(const double *norms, const void *m, int64_t n, void *x,
                      int64_t kp, int64_t hcol, void *stream) {
  if (n < 1) return EXEM_OK;
  tc::refresh_h_kernel<<<(unsigned)ceil_div(n, 256), 256, 0,
                         (cudaStream_t)stream>>>(
      norms, (const float *)m, n, (__nv_bfloat16 *)x, kp, hcol);
  EXEM_LAUNCH_CHECK("tc_refresh_h");
  return EXEM_OK;
}

}  // extern "C"
