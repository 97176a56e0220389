/*
 * exem_b200.h -- C-ABI of the B200-native exemplar-clustering evaluator.
 *
 * Drop-in boundary for the evaluation path of the reference package
 * `exembatch` (arXiv 2101.08763 re-implementation).  The reference binds no
 * native code: its plugin point is the backend string dispatch in
 * pkg/src/exembatch/evaluate.py:42,59-65,282-293 plus the batch dissimilarity
 * pkg/src/exembatch/objective.py:24-61,75-90.  Every function below replaces
 * one numeric step of that Python path (file:line cited per entry point);
 * the Python package `paper_2101_08763_b200` binds them with ctypes exactly
 * as INTEGRATION.md shows.
 *
 * Conventions
 *  - Plain pointers + sizes only.  Every pointer argument is DEVICE memory
 *    owned by the caller unless stated otherwise; nothing is retained across
 *    calls and the library allocates no persistent device memory.
 *  - `stream` is a cudaStream_t passed as void* (NULL = legacy default).
 *    All calls are asynchronous and stream-ordered; none synchronises.
 *  - Return value is an EXEM_* status; exem_last_error() gives a
 *    thread-local message for the last non-zero status.
 *  - Device layouts:
 *      SIMT layout  vt[d_pad][ld]  column-major points (the reference's
 *                   F-order, pkg/src/exembatch/core.py:286), compute type
 *                   float (f16/bf16/f32 storage) or double (f64), zero padded.
 *      TC layout    x[rows][kp]    point-major, K-contiguous half operand
 *                   (bf16/f16) with d data columns followed by 6 folded
 *                   constant columns; TMA 128B-swizzle friendly.
 */
#ifndef EXEM_B200_H
#define EXEM_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- dtype tags (Precision, pkg/src/exembatch/core.py:33-94; +bf16) ---- */
#define EXEM_F16 0
#define EXEM_BF16 1
#define EXEM_F32 2
#define EXEM_F64 3

/* OR'd into the dtype tag of the entry points that take the column-major
 * V buffer `vt` (exem_ground_prepare[_rows] as output; exem_set_min,
 * exem_greedy_update (vt and cvt), exem_tc_pack_candidates/_points/
 * _points_plain as input): for bf16/f16 ground sets `vt` holds the 2-byte
 * STORAGE values instead of their binary32 widening -- half the HBM bytes
 * of K1/K2/the m-update and one fewer 4-byte copy of V.  Arithmetic is
 * unchanged (values are widened in registers), so results are bit-identical
 * to the widened layout.  Rejected (EXEM_ERR_ARG) with f32/f64 tags and by
 * entry points that do not list it. */
#define EXEM_VT_STORAGE 0x100

/* ---- status codes -> pkg/src/exembatch/errors.py:4-41 ---- */
#define EXEM_OK 0
#define EXEM_ERR_ARG 1         /* ValueError / DimensionMismatchError        */
#define EXEM_ERR_OOM 2         /* OutOfMemoryError (errors.py:28)            */
#define EXEM_ERR_CUDA 3        /* ExemError (CUDA launch / runtime failure)  */
#define EXEM_ERR_DATA 4        /* InvalidDataError (errors.py:20)            */
#define EXEM_ERR_UNSUPPORTED 5 /* ExemError: no sm_100a device / bad dtype   */

const char *exem_last_error(void);
int exem_abi_version(void); /* 4: EXEM_VT_STORAGE (2-byte vt); 3: exem_greedy_gains_tc_ex (2: check_finite in K1, interleaved K4-TC set tiles) */

/* Device query: SM count, compute capability, opt-in shared memory. */
int exem_device_info(int device, int *sm_count, int *cc_major, int *cc_minor,
                     int64_t *smem_optin);

/* ---- layout helpers (pure host arithmetic, no device work) ---- */
int64_t exem_pad_points(int64_t n);          /* ld of the SIMT layout        */
int64_t exem_pad_dims(int64_t d);            /* d_pad of the SIMT layout     */
int64_t exem_split_points(int64_t n);        /* points per partial-sum split */
int64_t exem_num_splits(int64_t n);          /* ceil(n / split_points)       */
int64_t exem_tc_kp(int64_t d);               /* K stride of the TC operand   */
int64_t exem_tc_rows(int64_t n);             /* row count of the TC operand  */
int64_t exem_reduce_scratch(int64_t count);  /* doubles of scratch needed by
                                                the fixed-order reductions  */

/*
 * K1  ground_prepare
 * Replaces build_ground_set's numeric part, pkg/src/exembatch/core.py:286-309
 * (storage cast, aux_distances = d(v_i, e0), aux sum).
 *   src      [d][n] column-major storage-dtype values (the F-order buffer,
 *            GroundSet.data core.py:152-155), device.
 *   e0       [d] storage-dtype auxiliary vector, device.
 *   vt       out [d_pad][ld] compute-type SIMT layout (zero padded).
 *   norms    out [ld] double, ||v_i||^2 of the stored values (0 on padding).
 *   aux      out [ld] compute type, d(v_i, e0) rounded through the storage
 *            dtype (the reference stores aux_distances at dt, core.py:304).
 *   aux_sum  out [1] double, sum_i aux_i in fixed order.
 *   scratch  exem_reduce_scratch(n) doubles.
 *   check_finite  != 0 (f32/f16/bf16 storage): a point with a non-finite
 *            stored value contributes NaN to the aux sum, so aux_sum is NaN
 *            iff V holds inf/NaN -- the device-side replacement of the
 *            reference's host scan (core.py:282-283).
 */
int exem_ground_prepare(int dtype, const void *src, int64_t n, int64_t d,
                        const void *e0, void *vt, int64_t ld, double *norms,
                        void *aux, double *aux_sum, double *scratch,
                        int check_finite, void *stream);

/*
 * Low-memory regime (north-star item c): V stays in (pinned) host memory and
 * streams through the device in split-aligned row slices.
 *   exem_host_register / _unregister  page-lock an existing host buffer
 *            (the F-order GroundSet.data, core.py:152-155) for async DMA.
 *   exem_h2d_rows  rows [row0, row0+rows) of a column-major [d][ld_host]
 *            host matrix -> a dense [d][rows] device buffer (one 2-D DMA).
 *   exem_sum_fixed out[out_index] = fixed-order sum of `count` block
 *            partials (the final step of K1/K2 sums; with per-slice block
 *            partials at their global offsets the result is bit-identical
 *            to the resident computation).
 * K1 with aux_sum == NULL, K2 (set_min) with sum_out == NULL and
 * greedy_update with msum == NULL leave their per-256-point block partials
 * in `scratch` instead of reducing them.
 */
int exem_host_register(void *host, int64_t bytes);
int exem_host_unregister(void *host);
int exem_h2d_rows(void *dst, const void *host, int64_t ld_host, int64_t row0,
                  int64_t rows, int64_t d, int64_t elem_bytes, void *stream);
int exem_sum_fixed(const double *in, int64_t count, double *out,
                   int64_t out_index, void *stream);

/* K1 for a ROW-major source src[n][d] (a C-order numpy matrix uploaded as
 * is, no host transpose); outputs and aux block partials bit-identical to
 * exem_ground_prepare. */
int exem_ground_prepare_rows(int dtype, const void *src, int64_t n, int64_t d,
                             const void *e0, void *vt, int64_t ld,
                             double *norms, void *aux, double *aux_sum,
                             double *scratch, int check_finite, void *stream);
/* Plain async host -> device copy (a contiguous row slice of a row-major
 * host matrix in the low-memory regime). */
int exem_h2d_bytes(void *dst, const void *host, int64_t bytes, void *stream);

/*
 * K2  set_min -- per-point minimum over one explicit element set
 * Replaces min_distances, pkg/src/exembatch/objective.py:113-141, and the
 * sum inside _set_value, pkg/src/exembatch/evaluate.py:105-112.
 *   elems    [k][d_pad] compute-type element rows (device).
 *   enorms   [k] double ||e||^2.
 *   include_aux  1: t_i = min(aux_i, min_e d) (objective.py:138-139).
 *   t_out    optional [n] compute type (NULL to skip).
 *   label_out optional [n] int64 argmin element, lowest index on ties
 *            (assign_clusters, pkg/src/exembatch/optimize.py:115-136).
 *   sum_out  optional [1] double fixed-order sum_i t_i.
 */
/* 1 when exem_set_min runs (dtype | EXEM_VT_STORAGE) for this shape (the
 * TMA-fed K2; the cp.async K2 reads widened vt only); has_t_out: a t_out
 * buffer will be passed (needed when k exceeds one element group). */
int exem_set_min_storage_ok(int dtype, int64_t d, int64_t k, int has_t_out);
int exem_set_min(int dtype, const void *vt, int64_t ld, int64_t n, int64_t d,
                 const double *norms, const void *aux, const void *elems,
                 const double *enorms, int64_t k, int include_aux, void *t_out,
                 int64_t *label_out, double *sum_out, double *scratch,
                 void *stream);

/*
 * K4  batch_eval -- explicit packed sets (the paper's S_multi)
 * Replaces evaluate_batch / _reference_eval / tiled_evaluate,
 * pkg/src/exembatch/evaluate.py:142-149,197-270,273-293, over the packed
 * round-robin layout of pack_batch, pkg/src/exembatch/core.py:331-346:
 *   packed   [d_pad][k_max][l_pad] compute type; value (j,e,dim) at
 *            dim*(k_max*l_pad) + e*l_pad + j  (packed_address, core.py:320).
 *   pnorms   [k_max][l_pad] double ||S_j[e]||^2.
 *   card     [l] int32 cardinalities; slots e >= card[j] are never used.
 *   partial  out [splits][l] double, sum over the split's points of
 *            t_i(S_j) = min(aux_i, min_e d(v_i, S_j[e])).
 *   split_pts  points per partial-sum split (exem_split_points of the
 *            GLOBAL n); a row shard / streamed slice of V must start on a
 *            split boundary, so per-set sums never depend on sharding.
 *   splits   ceil(n / split_pts) for the n points passed here.
 */
int exem_batch_eval(int dtype, const void *vt, int64_t ld, int64_t n,
                    int64_t d, const double *norms, const void *aux,
                    const void *packed, const double *pnorms,
                    const int32_t *card, int64_t l, int64_t l_pad,
                    int64_t k_max, int64_t split_pts, double *partial,
                    int64_t splits, void *stream);

/*
 * K3  greedy_gains -- optimizer-aware batched evaluation of every
 * S u {c} of one Greedy step in one launch
 * Replaces the batch built and evaluated in greedy_maximize,
 * pkg/src/exembatch/optimize.py:61-71 (via evaluate.py:142-149).
 * Computes G_c = sum_i max(0, m_i - d(v_i, c)) for every candidate row c,
 * with m_i = min(aux_i, min_{s in S} d(v_i, s)) held on device.
 * SIMT form (f32/f64):
 *   cvt      [d_pad][ldc] candidate SIMT layout (== vt for Greedy).
 *   cnorms   [ldc] double ||c||^2.
 *   vt/norms/m  point shard (SIMT layout), m in compute type.
 *   partial  out [splits][l] double.
 */
int exem_greedy_gains_simt(int dtype, const void *cvt, int64_t ldc,
                           const double *cnorms, int64_t l, const void *vt,
                           int64_t ld, const double *norms, const void *m,
                           int64_t n, int64_t d, int64_t split_pts,
                           double *partial, int64_t splits, void *stream);

/*
 * K3-TC  tcgen05 form (bf16/f16 operands, fp32 TMEM accumulators):
 *   xc   [tc_rows(l)][kp] candidate operand rows  [c, 1,1,1, -b_hi,-b_mid,-b_lo]
 *   xp   [tc_rows(n)][kp] point operand rows      [v, -h_hi,-h_mid,-h_lo, 1,1,1]
 *   with b = ||c||^2/2 and h_i = (||v_i||^2 - m_i)/2, so one MMA row-dot is
 *   D = (m_i - d(v_i,c))/2; partial receives sum_i max(0, D) * 2.
 */
int exem_greedy_gains_tc(int dtype, const void *xc, int64_t l, const void *xp,
                         int64_t n, int64_t d, int64_t split_pts,
                         double *partial, int64_t splits, void *stream);
/*
 * Same as exem_greedy_gains_tc with the epilogue width chosen by the caller:
 *   epi_groups   0 (default = 2), 2 or 4 warps per TMEM lane quarter (4:
 *                faster when many (candidate, point) gains are positive,
 *                e.g. clustered data; 2: when the sign screen skips most)
 *   screen_hits  NULL, or a device counter that receives += the number of
 *                (candidate row, 32-point chunk) screens that found a value
 *                >= 0 (the relu-sum work done; lets the caller choose
 *                epi_groups for the next steps).  Results do not depend on
 *                epi_groups beyond fp32 summation order inside a tile.
 */
int exem_greedy_gains_tc_ex(int dtype, const void *xc, int64_t l,
                            const void *xp, int64_t n, int64_t d,
                            int64_t split_pts, double *partial, int64_t splits,
                            int epi_groups, unsigned long long *screen_hits,
                            void *stream);

/*
 * K4-TC  batch_eval_tc -- explicit packed sets on tensor cores (bf16/f16).
 * Replaces evaluate_batch / tiled_evaluate, pkg/src/exembatch/evaluate.py:
 * 142-149,197-270, for half storage (same partial[splits][l] contract as
 * exem_batch_eval).  Points on M (TMEM lanes), set elements on N:
 *   xp   [tc_rows(n)][kp] point operand built by exem_tc_pack_points with
 *        m = NULL (h_i = ||v_i||^2 / 2).
 *   aux  [n] float aux distances (compute type).
 *   xs   [tc_set_rows(l, k_max)][kp] set-tile operand (exem_tc_pack_sets).
 * exem_tc_set_geometry: a set tile holds `spt` = min(16, 256 / k_max) sets
 * of `w` = k_max slots, column-interleaved (column c = slot c / spt of set
 * c % spt), MMA N = ncols = round_up(spt * w, 16); EXEM_ERR_UNSUPPORTED when
 * k_max > 256 (the caller then uses exem_batch_eval).
 */
int exem_tc_set_geometry(int64_t k_max, int32_t *spt, int32_t *w,
                         int32_t *ncols);
int64_t exem_tc_set_rows(int64_t l, int64_t k_max);
int exem_tc_pack_sets(int dtype, const void *packed, const double *pnorms,
                      const int32_t *card, int64_t l, int64_t l_pad,
                      int64_t k_max, int64_t d, void *xs, float *bs,
                      void *stream);
int exem_batch_eval_tc(int dtype, const void *xp, int64_t n, const void *aux,
                       const double *norms, const void *xs, const float *bs,
                       int64_t l, int64_t k_max, int64_t d, int64_t split_pts,
                       double *partial, int64_t splits, void *stream);
/* Plain (unfolded) K4-TC operands, used when folding the six constant
 * columns would add a whole 64-wide K chunk (exem_tc_batch_plain(d) = 1,
 * e.g. d = 256): point rows [v, 0..] and set rows [e, 0..] with stride
 * exem_tc_batch_kp(d) = round_up(d, 64); exem_tc_pack_sets with bs != NULL
 * writes plain set rows and bs[row] = ||e||^2/2, and exem_batch_eval_tc with
 * bs != NULL adds the constants in the epilogue from bs and norms
 * (min_e d = ||v||^2 - 2 max_e (v.e - ||e||^2/2)). */
int64_t exem_tc_batch_plain(int64_t d);
int64_t exem_tc_batch_kp(int64_t d);
int exem_tc_pack_points_plain(int dtype, const void *vt, int64_t ld,
                              int64_t n, int64_t d, void *xp, void *stream);

/*
 * Binary32 on tensor cores (split-bf16): each fp32 coordinate is split into
 * three bf16 pieces and the pieces are laid out along K (6d columns, then
 * the folded constants) so that exem_greedy_gains_tc with d' =
 * exem_tc_split_dim(d) computes the K3 gains at binary32 accuracy
 * (all piece products with i+j <= 2, each exact in fp32).
 *   role 0: candidate rows from vt/norms; role 1: point rows from vt/norms/m.
 *   exem_tc_refresh_h rewrites the three -h columns (at hcol = 6d) of point
 *   rows from norms and an updated m (after exem_greedy_update).
 */
int64_t exem_tc_split_dim(int64_t d);
int exem_tc_pack_split(int role, const void *vt, int64_t ld, int64_t n,
                       int64_t d, const double *norms, const void *m,
                       void *x, void *stream);
int exem_tc_refresh_h(const double *norms, const void *m, int64_t n, void *x,
                      int64_t kp, int64_t hcol, void *stream);

/* Build the TC candidate operand from the SIMT layout (+ norms). */
int exem_tc_pack_candidates(int dtype, const void *vt, int64_t ld, int64_t n,
                            int64_t d, const double *norms, void *xc,
                            void *stream);
/* Build / refresh the TC point operand from the SIMT layout, norms and m
 * (m = NULL: h_i = ||v_i||^2/2, the K4-TC point operand). */
int exem_tc_pack_points(int dtype, const void *vt, int64_t ld, int64_t n,
                        int64_t d, const double *norms, const void *m,
                        void *xp, void *stream);

/*
 * K6  reduce_partials: G[j] = scale * sum_{s} partial[s][j], fixed order.
 * Replaces np.sum(t, dtype=acc) per set, pkg/src/exembatch/evaluate.py:111.
 */
int exem_reduce_partials(const double *partial, int64_t splits, int64_t l,
                         double scale, double *out, void *stream);

/*
 * K5  argmax_select: masked argmax over G (first maximum = lowest index,
 * pkg/src/exembatch/optimize.py:73), marks it selected, appends it to the
 * device-resident trajectory: sel_idx[step], sel_gain[step].
 *   selected  [l] uint8 mask (1 = already in S, excluded).
 *   index_map optional [l] int64 candidate row -> ground index (NULL: identity)
 */
int exem_argmax_select(const double *gains, int64_t l, uint8_t *selected,
                       const int64_t *index_map, int64_t step,
                       int64_t *sel_idx, double *sel_gain, double *scratch,
                       void *stream);

/*
 * K2  greedy_update: m_i <- min(m_i, d(v_i, c*)) for c* = sel_idx[step]
 * (the exemplar just chosen, read on device -- no host round trip), and
 * msum[step] = sum_i m_i (fixed order) -- pkg/src/exembatch/optimize.py:74-76.
 *   cvt/ldc   candidate SIMT layout the index refers to.
 *   xp/kp     optional TC point operand (NULL for f32/f64): its folded -h
 *             columns are rewritten from the new m_i.
 */
int exem_greedy_update(int dtype, const void *vt, int64_t ld, int64_t n,
                       int64_t d, const double *norms, const void *cvt,
                       int64_t ldc, const double *cnorms,
                       const int64_t *sel_idx, int64_t step, void *m,
                       void *xp, int64_t kp, double *msum, double *scratch,
                       void *stream);

/* m_i <- aux_i (start of a Greedy run); msum_out = sum aux (fixed order). */
int exem_greedy_init(int dtype, const void *aux, int64_t n, void *m,
                     double *msum_out, double *scratch, void *stream);

/*
 * Distance matrix for Dissimilarity.distances / _squared_euclidean_batch,
 * pkg/src/exembatch/objective.py:42-61,75-90:  out[i][j] = d(a_i, b_j).
 *   a [m][d_pad], b [q][d_pad] compute type row-major; out [m][q] compute.
 */
int exem_distance_matrix(int dtype, const void *a, const double *anorms,
                         int64_t m, const void *b, const double *bnorms,
                         int64_t q, int64_t d, int64_t d_pad, void *out,
                         void *stream);

/* Packed round-robin batch [d_pad][k_max][l_pad] (compute type) from the
 * concatenated element rows of the l sets: rows[offsets[j] + e][d] (storage
 * dtype, row-major), card[j] = |S_j|; blank slots / padding are zero.  The
 * device-side form of pack_batch, pkg/src/exembatch/core.py:331-346. */
int exem_pack_elements(int dtype, const void *rows, const int64_t *offsets,
                       const int32_t *card, int64_t l, int64_t l_pad,
                       int64_t k_max, int64_t d, void *packed, void *stream);

/* The packed batch as PackedBatch.values holds it (storage dtype,
 * [d][k_max][l], pkg/src/exembatch/core.py:331-346) widened to the compute
 * type and zero padded to [d_pad][k_max][l_pad] on the device. */
int exem_widen_packed(int dtype, const void *src, int64_t l, int64_t l_pad,
                      int64_t k_max, int64_t d, void *packed, void *stream);

/* pnorms[e][j] = ||S_j[e]||^2 of a packed [d_pad][k_max][l_pad] batch
 * (the element norms e2 of objective.py:84, computed once per batch). */
int exem_packed_norms(int dtype, const void *packed, int64_t d, int64_t k_max,
                      int64_t l_pad, double *out, void *stream);

/* Row norms ||x_r||^2 (double) of a [rows][d_pad] compute-type matrix. */
int exem_row_norms(int dtype, const void *x, int64_t rows, int64_t d,
                   int64_t d_pad, double *out, void *stream);

/* SieveStreaming over a BLOCK of nb arriving elements (sieve.py):
 * exem_sieve_block_dist writes dist[b][i] = d(v_i, elems[b]) with K2's
 * arithmetic (identical to exem_set_min, k = 1); exem_sieve_block_gains then
 * computes gains[s][b] = sum_i max(0, M[s][i] - dist[b][i]) for every sieve
 * row s < rows (fp64, fixed order), scratch = exem_sieve_block_scratch. */
int exem_sieve_block_dist(int dtype, const void *vt, int64_t ld, int64_t n,
                          int64_t d, const double *norms, const void *elems,
                          const double *enorms, int64_t nb, void *dist,
                          int64_t ldd, double *scratch, void *stream);
int64_t exem_sieve_block_scratch(int64_t n, int64_t rows, int64_t nb);
int exem_sieve_block_gains(int dtype, const void *M, int64_t ldm, int64_t rows,
                           const void *D, int64_t ldd, int64_t nb, int64_t n,
                           double *gains, double *scratch, void *stream);

/*
 * Sieve streaming (north star: "the Greedy and streaming optimizers"; the
 * reference ships none, SPEC.md:9,402 -- see sieve.py).  Each sieve s keeps
 * an m-vector M[s][0..n) (row stride ldm) = per-point minimum over its set
 * and aux.  For one arriving element with dist[i] = d(v_i, e) (exem_set_min
 * with k = 1, include_aux = 0):
 *   exem_sieve_gains   gains[s] = sum_i max(0, M[s][i] - dist[i]) (fixed
 *                      order; scratch >= ceil(n/256) * sieves doubles)
 *   exem_sieve_update  m <- min(m, dist) for one sieve row; msum[0] = sum m
 */
int exem_sieve_gains(int dtype, const void *M, int64_t ldm, int64_t sieves,
                     const void *dist, int64_t n, double *gains,
                     double *scratch, void *stream);
int exem_sieve_update(int dtype, void *m, const void *dist, int64_t n,
                      double *msum, double *scratch, void *stream);

/*
 * Multi-GPU K5 over peer memory (no NCCL on the per-step path; distributed.py
 * PeerGains).  Shared buffers are allocated here (their base pointers are
 * what CUDA IPC exports) and owned by the caller:
 *   exem_ipc_alloc / exem_ipc_free      cudaMalloc / cudaFree
 *   exem_ipc_handle / exem_ipc_open / exem_ipc_close  64-byte CUDA IPC handle
 *   exem_peer_publish   after this rank's K3 + K6: flag = value (release,
 *                       system scope; stream-ordered after the gains)
 *   exem_peer_argmax_select  waits until every peer's flag >= expect, sums
 *       the W peers' local gains in fixed rank order (x scale) into
 *       gains_out and takes the masked argmax (as exem_argmax_select).
 *   peers / flags: device arrays of W device pointers (peer-mapped).
 */
int exem_ipc_alloc(int64_t bytes, void **ptr);
int exem_ipc_free(void *ptr);
int exem_ipc_handle(void *ptr, void *handle);
int exem_ipc_open(const void *handle, void **ptr);
int exem_ipc_close(void *ptr);
int exem_peer_publish(unsigned long long *flag, unsigned long long value,
                      void *stream);
int exem_peer_argmax_select(const double *const *peers,
                            const unsigned long long *const *flags, int world,
                            unsigned long long expect, int64_t l, double scale,
                            double *gains_out, uint8_t *selected,
                            int64_t step, int64_t *sel_idx, double *sel_gain,
                            double *scratch, void *stream);

/* Number of kernels this library launched since load (evidence counter). */
int64_t exem_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif /* EXEM_B200_H */
