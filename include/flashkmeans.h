/*
 * flashkmeans.h -- C ABI of the B200-native flash-kmeans hot path.
 *
 * The reference (flashmeans 0.1.0, /root/reference/pkg/src/flashmeans) has no
 * foreign-function boundary of its own: its "native seam" is a set of Numba
 * @njit kernels that fill caller-allocated NumPy buffers (_kernels.py:18-171)
 * behind three Python operators.  Each entry point below replaces one of
 * those operators at the same granularity, with the same ownership rule
 * (caller allocates every output, the library only writes views):
 *
 *   fk_assign     <- flash_assign          flash_assign.py:135-222
 *                    (dist_block + rowmin_merge, _kernels.py:32-82;
 *                     assign_tile_fast, _kernels.py:85-104)
 *   fk_update     <- sort_inverse_update   sort_inverse.py:106-149
 *                    (counting_sort + segment_stats + merge_segments,
 *                     _kernels.py:118-171)
 *   fk_normalize  <- normalize             baseline.py:127-150
 *   fk_row_norms  <- row_norms             core.py:307-318 (_kernels.py:21-29)
 *   fk_objective  <- _objective_row        pipeline.py:65-68
 *   fk_scatter    <- scatter_update        baseline.py:108-124 (foil only)
 *
 * Conventions
 *   - extern "C", plain pointers and sizes; no torch / CUDA types.  `stream`
 *     is a cudaStream_t passed as void* (NULL = legacy default stream).
 *   - Every call is stream-ordered, never synchronizes the host and never
 *     allocates device memory: scratch comes from a caller-owned workspace
 *     sized by the matching *_workspace query.
 *   - Inside one call, consecutive kernels may use programmatic dependent
 *     launch (each waits for its predecessor's completion before touching
 *     memory), so stream order toward the caller's later work is unchanged.
 *   - All data pointers are DEVICE pointers.  Layouts are batch-major,
 *     row-major: X (B,N,d), C (B,K,d), ids (B,N) int32, sums (B,K,d) f64,
 *     counts (B,K) int64 -- the reference's shapes and dtypes
 *     (core.py:109-233).
 *   - Errors are status codes, validated before any launch (the reference
 *     raises ValueError before any kernel call, flash_assign.py:152-157);
 *     FK_EINVAL maps to ValueError in the Python layer.
 *   - The library is reentrant; its only global state is a lazily built,
 *     thread-safe per-device table of kernel attributes (AOT sm_100a SASS,
 *     no JIT).
 */
#ifndef FLASHKMEANS_H_
#define FLASHKMEANS_H_

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define FK_API __attribute__((visibility("default")))
#else
#define FK_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  FK_OK = 0,
  FK_EINVAL = 1,        /* bad shape / dtype / pointer / id                    */
  FK_EUNSUPPORTED = 2,  /* shape outside the precompiled buckets or no sm_100 */
  FK_ECUDA = 3,         /* a CUDA runtime error; see fk_last_cuda_error()     */
  FK_EWORKSPACE = 4     /* workspace smaller than the *_workspace query        */
} fk_status;

typedef enum {
  FK_F32 = 0,   /* "single" (core.py:22)                                       */
  FK_BF16 = 1,  /* bf16 data: tcgen05 path, fp32 accumulation                  */
  FK_F16 = 2,   /* fp16 data: tcgen05 path, fp32 accumulation                  */
  FK_F64 = 3    /* "double" (core.py:22)                                       */
} fk_dtype;

typedef enum {
  FK_ASSIGN_EXACT = 0,  /* dot_mode="exact": Appendix-A arithmetic, bitwise for f32/f64 */
  FK_ASSIGN_FAST = 1    /* dot_mode="fast":  tensor cores (bf16/f16), fp32 accumulate   */
} fk_assign_mode;

FK_API const char* fk_version(void);
FK_API const char* fk_status_string(fk_status s);
/* Last CUDA error string seen by this thread (valid until the next call). */
FK_API const char* fk_last_cuda_error(void);
/* 1 if `device` is an sm_100 part this library has SASS for, else 0. */
FK_API int fk_device_supported(int device);
/* Load every kernel of the library on the current device now instead of at
 * its first launch (lazy module loading), so a first call on a new shape
 * pays no loading time (time-to-first-run, reference PAPER.md:392-395 and
 * the `ttfr` bench, cli.py:261-336).  Idempotent per device.  The Python
 * package calls it when it binds a device. */
FK_API fk_status fk_preload(void);

/* ---------------------------------------------------------------- assign
 * Nearest-centroid assignment without materializing the N x K distances.
 *   X, C      : (B,N,d), (B,K,d) in dtype `dt`
 *   idx_out   : (B,N) int32, lowest centroid id among equal minima
 *   mind_out  : (B,N) squared distance to the chosen centroid; element type
 *               is the data type for FK_F32/FK_F64 and float32 for
 *               FK_BF16/FK_F16
 *   idx_prev  : optional (B,N) int32; when given, *changed_flag (int32, device)
 *               is OR-ed with 1 if any id differs from idx_prev
 *               (the lloyd_run repeat test, pipeline.py:137)
 * FK_F32/FK_F64 are bitwise equal to the reference's dot_mode="exact": for
 * d <= 128 and problems above ~6.7e7 multiply-adds through the certified
 * tensor-core path (fk_assign_split below, X's split operand built in the
 * workspace), otherwise through the exact CUDA-core mirror.  FK_BF16/FK_F16
 * run the tcgen05 kernel for d <= 256 (rows of 16-byte multiples) and a
 * CUDA-core kernel otherwise.
 * bias      : optional (FK_BF16/FK_F16 only) the tensor-core bias operand of C,
 *             (B, fk_assign_bias_rows(K), 16) bf16 = [hi, mid, lo, 0...] split of
 *             ||c||^2/2, as written by fk_normalize(bias_out) or fk_assign_bias;
 *             NULL computes it inside the call (one extra pass over C).          */
FK_API size_t fk_assign_workspace(fk_dtype dt, int64_t B, int64_t N, int64_t K, int64_t d);
FK_API int64_t fk_assign_bias_rows(int64_t K);
FK_API fk_status fk_assign_bias(fk_dtype dt, const void* C, int64_t B, int64_t K, int64_t d,
                                void* bias_out, void* stream);
FK_API fk_status fk_assign(fk_dtype dt, const void* X, const void* C, const void* bias, int64_t B,
                           int64_t N, int64_t K, int64_t d, int32_t* idx_out, void* mind_out,
                           const int32_t* idx_prev, int32_t* changed_flag, void* workspace,
                           size_t workspace_bytes, void* stream);

/* ------------------------------------------------- assign, f32 / f64 data
 * The certified tensor-core path for the reference's own precisions
 * (flash_assign dot_mode "exact" / "fast", flash_assign.py:203-208;
 * dist_block and assign_tile_fast, _kernels.py:32-45, 85-104), d <= 128:
 *   xsplit : fk_assign_xsplit_bytes of device memory: the (B, N, 32*ceil(d/16))
 *            bf16 rows [hi | lo] of X, v = hi + lo + O(2^-16 v), then the
 *            reference's exact ||x||^2 (row_norms, core.py:307-318); written
 *            once by fk_assign_xsplit, reusable while X is unchanged (a Lloyd
 *            run builds it once).
 *   dot_mode FK_DOT_EXACT: tcgen05 estimate of every distance (3 bf16 MMAs
 *            per K=16 step, fp32 accumulation) + per-row certificate that the
 *            estimated argmin is the reference's; uncertified rows (near and
 *            exact ties, non-finite data) rerun the exact CUDA-core mirror.
 *            Output bitwise equal to the reference's exact mode.
 *   FK_DOT_FAST: the reference's relaxed mode (held to rtol 1e-6,
 *            test_flash_assign.py:172-178) is served by the same certified
 *            path, i.e. exactly: an uncertified tensor-core argmin can differ
 *            from exact when two centroids are closer than the estimate's
 *            error (~2^-16 |x||c|), which f64 reassociation never causes.
 *   FK_DOT_MIRROR: the exact CUDA-core mirror for every row (xsplit unused).
 * Workspace: fk_assign_split_workspace (does not include xsplit).           */
enum { FK_DOT_EXACT = 0, FK_DOT_FAST = 1, FK_DOT_MIRROR = 2 };
/* Diagnostic: how many rows of each batch element the last fk_assign_split
 * call on `workspace` sent to the exact fallback (B int32 to host memory;
 * synchronizes `stream`).  For fk_assign's own f32/f64 calls pass its
 * workspace offset by fk_assign_xsplit_bytes.                              */
FK_API fk_status fk_assign_split_fallback_rows(fk_dtype dt, int64_t B, int64_t N, int64_t K,
                                               int64_t d, const void* workspace,
                                               int32_t* counts_host, void* stream);
FK_API size_t fk_assign_xsplit_bytes(fk_dtype dt, int64_t B, int64_t N, int64_t d);
FK_API fk_status fk_assign_xsplit(fk_dtype dt, const void* X, int64_t B, int64_t N, int64_t d,
                                  void* xsplit_out, void* stream);
FK_API size_t fk_assign_split_workspace(fk_dtype dt, int64_t B, int64_t N, int64_t K, int64_t d);
FK_API fk_status fk_assign_split(fk_dtype dt, const void* X, const void* xsplit, const void* C,
                                 int64_t B, int64_t N, int64_t K, int64_t d, int32_t dot_mode,
                                 int32_t* idx_out, void* mind_out, const int32_t* idx_prev,
                                 int32_t* changed_flag, void* workspace, size_t workspace_bytes,
                                 void* stream);

/* ---------------------------------------------------------------- update
 * Per-cluster sums (f64) and counts (int64) from (X, ids) by a device stable
 * counting sort of ids followed by warp-level segmented reductions over the
 * sorted order (X is never permuted).  Deterministic: every addition order is
 * fixed by (ids, shape, SM count), so repeated calls return the same bits; ids
 * outside [0, K) are skipped (the Python layer rejects them beforehand, as
 * the reference does).  `accumulate`=0 overwrites sums/counts,
 * 1 adds into them (chunked streaming, PartialStats.combine pipeline.py:250).
 * `update_chunk` is the reference's chunk (TilingConfig.update_chunk); it
 * only defines *merges_out (device int64, incremented by the segment count the
 * reference would record, sort_inverse.py:165).  merges_out may be NULL.    */
FK_API size_t fk_update_workspace(fk_dtype dt, int64_t B, int64_t N, int64_t K, int64_t d);
FK_API fk_status fk_update(fk_dtype dt, const void* X, const int32_t* ids, int64_t B, int64_t N,
                    int64_t K, int64_t d, int64_t update_chunk, int32_t accumulate, double* sums,
                    int64_t* counts, int64_t* merges_out, void* workspace, size_t workspace_bytes,
                    void* stream);

/* The update's first pass folded into the assign (a Lloyd iteration's
 * assign -> update pair on bf16/fp16 data; the counting step of
 * counting_sort, _kernels.py:118-132, sort_inverse.py:67-78):
 *   fk_update_hist_slots: where the block histogram table of an update
 *     workspace lives -- hist_table (B * hist_bpb rows of K int32), hist_inval
 *     (B * hist_bpb int32), the blocks per batch element and points per block,
 *     and clear_words: the int32 words from hist_table on that must be zero
 *     before the first fk_assign_hist (FK_EUNSUPPORTED for f32/f64 data or
 *     K > 16384: use fk_update);
 *   fk_assign_hist: fk_assign (bf16/fp16, tensor-core path) whose epilogue
 *     also adds each row's id into that table (ids outside [0, K) into
 *     hist_inval); the table must be zero on entry;
 *   fk_update_prehist: fk_update without its histogram pass, reading the
 *     table the assign built; it leaves the table zeroed again for the next
 *     fk_assign_hist.  Results are bitwise those of fk_assign + fk_update.  */
FK_API fk_status fk_update_hist_slots(fk_dtype dt, int64_t B, int64_t N, int64_t K, int64_t d,
                                      void* workspace, int32_t** hist_table, int32_t** hist_inval,
                                      int64_t* hist_bpb, int64_t* hist_per, int64_t* clear_words);
FK_API fk_status fk_assign_hist(fk_dtype dt, const void* X, const void* C, const void* bias, int64_t B,
                                int64_t N, int64_t K, int64_t d, int32_t* idx_out, void* mind_out,
                                const int32_t* idx_prev, int32_t* changed_flag, void* workspace,
                                size_t workspace_bytes, int32_t* hist_table, int32_t* hist_inval,
                                int64_t hist_bpb, int64_t hist_per, const float* xnorm, void* stream);
/* xnorm (optional, fk_assign_hist): (B, N) fp32 ||x||^2 of X written once per
 * data set by fk_assign_row_norms (same K), which sums every row exactly as
 * the tensor-core epilogue would from its shared-memory tile -- min_dists are
 * bitwise unchanged and the epilogue skips that sum on every call.          */
FK_API fk_status fk_assign_row_norms(fk_dtype dt, const void* X, int64_t B, int64_t N, int64_t K,
                                     int64_t d, float* xnorm_out, void* stream);
FK_API fk_status fk_update_prehist(fk_dtype dt, const void* X, const int32_t* ids, int64_t B,
                                   int64_t N, int64_t K, int64_t d, int64_t update_chunk,
                                   int32_t accumulate, double* sums, int64_t* counts, int64_t* merges_out,
                                   void* workspace, size_t workspace_bytes, void* stream);

/* Stable argsort of the ids alone (argsort_assignments / counting_sort,
 * sort_inverse.py:67-78, _kernels.py:118-132): the order the update's segmented
 * reductions walk.  order_out (B*N int32): flat point indices b*N + i, grouped
 * by key b*K + id, ascending point index inside a key (np.argsort
 * kind="stable"); ids outside [0, K) are left out, so only the first
 * offsets_out[B*K] entries are written.  offsets_out (B*K+1 int64): start of
 * each key's run.  Workspace: fk_update_workspace(dt, B, N, K, 1).            */
FK_API fk_status fk_argsort(const int32_t* ids, int64_t B, int64_t N, int64_t K, int32_t* order_out,
                            int64_t* offsets_out, void* workspace, size_t workspace_bytes,
                            void* stream);

/* ------------------------------------------------------------- normalize
 * c = fl_T(sums / counts) per cluster; clusters with count 0 keep `prev`
 * bitwise and get empty_mask=1.  prev/out are (B,K,d) in `master_dt`
 * (FK_F32 or FK_F64); `operand_out` (optional, (B,K,d) in `operand_dt`)
 * receives the rounded copy used as the next MMA operand.  `max_shift2`
 * (optional, device f64 scalar, must be pre-zeroed) receives
 * max_k sum_j (out-prev)^2 (pipeline._max_shift before the sqrt).  out may
 * alias prev.                                                                */
FK_API fk_status fk_normalize(fk_dtype master_dt, const double* sums, const int64_t* counts,
                       const void* prev, void* out, fk_dtype operand_dt, void* operand_out,
                       uint8_t* empty_mask, double* max_shift2, int64_t B, int64_t K, int64_t d,
                       void* bias_out, void* stream);
/* bias_out (optional, with a bf16/fp16 operand_out): also write the next
 * assign's bias operand of operand_out (see fk_assign), bitwise what
 * fk_assign_bias would compute.                                              */

/* Exact row norms in the data precision (f32/f64), core.row_norms semantics. */
FK_API fk_status fk_row_norms(fk_dtype dt, const void* M, int64_t rows, int64_t d, void* out,
                       void* stream);

/* objective[b] = sum_i mind[b,i] in f64 (pipeline._objective_row); mind is
 * f32 (FK_F32/FK_BF16/FK_F16 data) or f64.  Deterministic fixed-order
 * reduction; for f32 min_dists every f64 partial is exact in practice, so it
 * equals numpy's np.sum(m, dtype=float64) bit for bit.                      */
FK_API size_t fk_objective_workspace(int64_t B, int64_t N);
/* The two halves of fk_objective for the device-resident loop:
 * fk_objective_partials writes B * ceil(N / 8192) partials (numpy's buffer order);
 * fk_loop_tail (one launch at the end of an iteration) reduces them into
 * objective[b] (bitwise fk_objective's result) and, when history is given,
 * into history[*history_row * B + b] (then ++*history_row: the row index
 * lives on the device so a replayed CUDA graph fills successive rows); it
 * copies [*changed, *max_shift2, *merges] into flags_out[3] (f64) and clears
 * the three for the next iteration.                                          */
FK_API fk_status fk_objective_partials(fk_dtype mind_dt, const void* mind, int64_t B, int64_t N,
                                       double* partials, void* stream);
FK_API fk_status fk_loop_tail(const double* partials, int64_t B, int64_t N, double* objective,
                              double* history, int64_t* history_row, int32_t* changed,
                              double* max_shift2, int64_t* merges, double* flags_out, void* stream);
/* fk_normalize + fk_objective_partials + fk_loop_tail in ONE launch (the end
 * of a single-device iteration): the normalize blocks also compute the
 * objective partials of `mind` (same blocks and trees, so the same doubles)
 * and the last block to finish runs fk_loop_tail's work.  `counter` is a
 * device uint32 that is 0 before the call and left at 0.                   */
FK_API fk_status fk_normalize_loop_tail(fk_dtype master_dt, const double* sums, const int64_t* counts,
                                        const void* prev, void* out, fk_dtype operand_dt,
                                        void* operand_out, uint8_t* empty_mask, double* max_shift2,
                                        int64_t B, int64_t K, int64_t d, void* bias_out,
                                        fk_dtype mind_dt, const void* mind, int64_t N, double* partials,
                                        double* objective, double* history, int64_t* history_row,
                                        int32_t* changed_flag, int64_t* merges, double* flags_out,
                                        uint32_t* counter, void* stream);
FK_API fk_status fk_objective(fk_dtype mind_dt, const void* mind, int64_t B, int64_t N, double* out,
                       void* workspace, size_t workspace_bytes, void* stream);

/* Baseline scatter (one f64 atomic merge per point element): the contended
 * foil of baseline.scatter_update, kept for ncu comparison only.            */
FK_API fk_status fk_scatter(fk_dtype dt, const void* X, const int32_t* ids, int64_t B, int64_t N,
                     int64_t K, int64_t d, double* sums, int64_t* counts, void* stream);

/* ------------------------------------------------------ multi-GPU exchange
 * Packs (unpack = 0) counts (B*K int64), objective (B f64) and the changed
 * flag (int32) behind the sums in the single f64 all-reduce buffer
 * red = [sums (B*K*d) | counts | objective | changed] -- `red` points at the
 * counts part -- or unpacks the reduced values (changed = sum > 0).  One launch
 * each way around the per-iteration NCCL all-reduce of the point-sharded path. */
FK_API fk_status fk_stats_pack(int32_t unpack, int64_t* counts, double* objective, int32_t* changed,
                               double* red, int64_t BK, int64_t B, void* stream);
/* The reference's synchronized_merges for one update over GLOBAL counts
 * (B,K) int64 -- sort_inverse.py:159-165 evaluated on the all-reduced counts,
 * so a point-sharded run reports the single-process count: each non-empty
 * key's run [s, e) of its batch element meets floor((e-1)/chunk) -
 * floor(s/chunk) + 1 update chunks.  *merges = result (accumulate = 0) or
 * += result.                                                                 */
FK_API fk_status fk_merges_from_counts(const int64_t* counts, int64_t B, int64_t K,
                                       int64_t update_chunk, int64_t* merges, int32_t accumulate,
                                       void* stream);

/* ---------------------------------------------------------- reseed_farthest
 * The E points farthest from their assigned centroids, in the reference's
 * order: distance descending, ties to the lowest point index
 * (_farthest_order / _FarthestTracker, pipeline.py:76-89, 283-309).
 *   mind   : (B,N) f32 or f64 assigned distances (fk_assign's min_dists)
 *   idx_out: (B,E) int64 point indices
 * A radix select over the unique 96-bit keys (f64 distance bits, inverted
 * index) finds the E-th largest key on the device, then the E winners are
 * sorted in shared memory -- no sort of all N, no host round trip.
 * E <= 8192 (FK_EUNSUPPORTED beyond), N < 2^32.                             */
FK_API size_t fk_farthest_workspace(int64_t B, int64_t E);
FK_API fk_status fk_farthest(fk_dtype mind_dt, const void* mind, int64_t B, int64_t N, int64_t E,
                             int64_t* idx_out, void* workspace, size_t workspace_bytes, void* stream);

/* ------------------------------------------------------------- k-means++
 * D^2 seeding of init_centroids(method="kmeanspp") on the device:
 *   fk_kmeanspp        <- _kmeanspp_indices      core.py:342-357
 *   fk_kmeanspp_sweep  <- the per-chunk sweep of _streaming_kmeanspp
 *                         (pipeline.py:435-443)
 *   fk_kmeanspp_select <- total = min_d2.sum(); rng.choice(n, p=min_d2/total)
 *                         (core.py:350-353, pipeline.py:446-450)
 * The chosen indices equal the reference's for the same data and draws, bit for
 * bit: distances and `total` follow numpy's pairwise summation order in f64,
 * and choice() -- cumsum / normalise / searchsorted(side="right") -- is
 * resolved from an exact prefix with a certified error window, falling back
 * to numpy's literal serial cumsum when the draw lands inside it.
 * The random stream stays with the caller (numpy PCG64 substream (seed, b)):
 *   idx    : (B,K) int64; in: idx[b,0] = rng.integers(N); out: idx[b,1..K-1]
 *   u      : (B,K-1) f64, u[b,j-1] = the rng.random() double of draw j
 *   halted : (B) int32 out: K, or the first draw j whose total was 0.  The
 *            reference then draws rng.integers(N) for j..K-1 (the table stays
 *            all-zero), which the caller replays on its generator; idx[b, j..]
 *            is left untouched.
 *   min_d2 : (B,N) f64 scratch (the reference's resident weight table).
 * Distances are computed from the exact f64 upcast of the data (f32, f64,
 * bf16, f16).  Rows need d*8 <= 200 KiB.  The in-core sweep skips rows whose
 * minimum provably cannot change (triangle inequality against the nearest
 * chosen center, with rounding margins), so later draws read only the rows
 * near the new center; the results are unchanged bit for bit.                */
/* K and d size the in-core pruning state of fk_kmeanspp; the streaming pieces
 * (init / select) need only fk_kmeanspp_workspace(B, N, 0, 0).               */
FK_API size_t fk_kmeanspp_workspace(int64_t B, int64_t N, int64_t K, int64_t d);
FK_API fk_status fk_kmeanspp(fk_dtype dt, const void* X, int64_t B, int64_t N, int64_t d,
                             int64_t K, const double* u, int64_t* idx, int32_t* halted,
                             double* min_d2, void* workspace, size_t workspace_bytes, void* stream);
/* Streaming pieces.  fk_kmeanspp_init sets halted[b] = K.  A sweep covers rows
 * [0, rows) of X (B, rows, d) with batch stride x_batch_stride elements
 * against centers (B, d) (batch stride c_batch_stride elements), writing
 * min_d2 rows [0, rows) (batch stride m_batch_stride): first != 0 stores the
 * distance, else the running minimum.  Sweeps for draw j skip batch elements
 * with halted[b] < j.  fk_kmeanspp_select then picks idx[b, j] from the full
 * (B, N) table.                                                               */
FK_API fk_status fk_kmeanspp_init(int32_t* halted, int64_t B, int64_t N, int64_t K,
                                  void* workspace, size_t workspace_bytes, void* stream);
FK_API fk_status fk_kmeanspp_sweep(fk_dtype dt, const void* X, int64_t B, int64_t rows, int64_t d,
                                   int64_t x_batch_stride, const void* centers,
                                   int64_t c_batch_stride, double* min_d2, int64_t m_batch_stride,
                                   int32_t first, const int32_t* halted, int64_t j, void* stream);
FK_API fk_status fk_kmeanspp_select(const double* min_d2, int64_t B, int64_t N, const double* u,
                                    int64_t K, int64_t j, int64_t* idx, int32_t* halted,
                                    void* workspace, size_t workspace_bytes, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* FLASHKMEANS_H_ */
