/* dfa2c.h — C-ABI drop-in boundary for DiTFastAttnV2's fused head-wise
 * attention path on B200 (sm_100a).
 *
 * The reference (/root/reference/proj) exposes this path as the namespace
 * `dfa2` C++ free-function API (include/dfa2/ *.hpp headers, linked statically as
 * dfa2_core). This header is the thin C layer the host C++ (include/dfa2/)
 * and any FFI (ctypes, cgo, JNI) call. Plain pointers,
 * sizes and integer status codes; no C++ or torch types cross it.
 *
 * Conventions
 *  - Device tensors are bf16, contiguous row-major [batch, H, N, d] (the
 *    reference's [H, N, d] per sample, inc/tensor.hpp:86-93, with a leading
 *    batch axis; the reference runs one sample).
 *  - Plans are host arrays: kinds[H] (DFA2C_FULL|ARROW|CACHED) and
 *    windows[H] (Arrow window radius in blocks), mirroring HeadStrategy /
 *    LayerPlan (inc/dispatch.hpp:12-37).
 *  - Block masks are host uint8 [nb*nb], row-major, nb = ceil(N/B)
 *    (BlockMask, inc/arrow.hpp:12-34).
 *  - Every function returns a dfa2c_status; dfa2c_last_error() holds the
 *    message of the last failure on the calling thread. Status codes mirror
 *    the reference exception taxonomy (inc/errors.hpp:8-45). Validation is
 *    complete before any device work or cache mutation, as in
 *    src/dispatch.cpp:34-54.
 *  - Calls that take a cudaStream_t (passed as void*) are asynchronous on
 *    that stream unless stated otherwise; NULL means the legacy stream.
 */
#ifndef DFA2C_H
#define DFA2C_H

#include <stdint.h>

#if defined(__GNUC__)
#pragma GCC visibility push(default)
#endif
#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    DFA2C_OK = 0,
    DFA2C_SHAPE = 1,        /* dfa2::ShapeError */
    DFA2C_NONFINITE = 2,    /* dfa2::NonFiniteError */
    DFA2C_FULLY_MASKED = 3, /* dfa2::FullyMaskedRowError */
    DFA2C_CACHE_MISS = 4,   /* dfa2::CacheMissError */
    DFA2C_DEGENERATE = 5,   /* dfa2::DegenerateReferenceError */
    DFA2C_PLAN = 6,         /* dfa2::PlanValidationError */
    DFA2C_IO = 7,           /* dfa2::IoError */
    DFA2C_ORACLE = 8,       /* dfa2::OracleError */
    DFA2C_CUDA = 9,         /* CUDA runtime / driver failure */
    DFA2C_UNSUPPORTED = 10  /* shape outside what the sm_100a kernels support */
} dfa2c_status;

enum { DFA2C_FULL = 0, DFA2C_ARROW = 1, DFA2C_CACHED = 2 }; /* StrategyKind */
/* Flag OR-ed into kinds[h] of dfa2c_mha_forward(_host): head h belongs to
 * the layer plan (it counts for scheduling decisions) but this call neither
 * computes, copies nor commits it, and leaves its output rows untouched.
 * Lets several calls (e.g. one per GPU) split one layer by heads while every
 * head's result stays bitwise what the single call produces. */
enum { DFA2C_SKIP = 0x100 };
enum { DFA2C_VISUAL_FIRST = 0, DFA2C_TEXT_FIRST = 1 };     /* TokenOrder */
enum { DFA2C_BF16 = 0, DFA2C_F32 = 1, DFA2C_F64 = 2 };    /* element type */
enum { DFA2C_RSE_STANDARD = 0, DFA2C_RSE_LITERAL = 1 };     /* RseMode */

/* AttentionDims (inc/tensor.hpp:56-72). */
typedef struct {
    int64_t n_heads;
    int64_t head_dim;
    int64_t n_visual;
    int64_t n_text;
    int32_t order; /* DFA2C_VISUAL_FIRST | DFA2C_TEXT_FIRST */
} dfa2c_dims;

const char* dfa2c_last_error(void);
const char* dfa2c_version(void);

/* ---- host-only plan arithmetic (no GPU needed; bit-exact) -------------- */

/* build_arrow_mask (inc/arrow.hpp:45; src/arrow.cpp:113-153). active may be
 * NULL to query nb only; otherwise it receives nb*nb bytes. */
int dfa2c_arrow_mask(const dfa2c_dims* dims, int64_t block, int64_t window,
                     uint8_t* active, int64_t* nb);
/* BlockMask::active_positions, flops_count, sparsity_ratio
 * (inc/arrow.hpp:31-53; src/arrow.cpp:95-104, 155-169). Any output may be NULL. */
int dfa2c_mask_stats(const uint8_t* active, int64_t seq_len, int64_t block,
                     int64_t head_dim, int64_t* active_positions, int64_t* flops,
                     double* sparsity);
/* dense_flops (inc/arrow.hpp:50; src/arrow.cpp:161-163). */
int64_t dfa2c_dense_flops(int64_t seq_len, int64_t head_dim);
/* plan_flops (inc/dispatch.hpp:51-52; src/dispatch.cpp:93-120). */
int dfa2c_plan_flops(const dfa2c_dims* dims, int64_t block, const int32_t* kinds,
                     const int64_t* windows, int64_t* flops);
/* CompressionPlan::validate + flops_total/flops_dense_total/aggregate_sparsity
 * (inc/plan.hpp:30-42; src/plan.cpp:33-73) over a timestep-major [T*L*H]
 * plan (layers[t*L + l], src/plan.cpp:25-31). Outputs may be NULL. */
int dfa2c_plan_aggregate(const dfa2c_dims* dims, int64_t n_timesteps, int64_t n_layers,
                         int64_t block, const int32_t* kinds, const int64_t* windows,
                         int64_t* flops_total, int64_t* flops_dense, double* sparsity);
/* The per-head tile scheduler's tile set for one head strategy: for every
 * 128-row query tile i, the KV tiles (dfa2c_kv_tile_keys() keys each) the
 * kernel will compute, in ascending order. row_ptr[n_qtiles+1] (CSR),
 * cols[] (kv tile | 1<<31 when the tile needs element masking: a mask block
 * boundary inside the tile or a ragged tail). Pass cols == NULL to query
 * the count in *n_tiles. kind FULL or ARROW. */
int64_t dfa2c_kv_tile_keys(void);
int dfa2c_tile_set(const dfa2c_dims* dims, int64_t block, int32_t kind, int64_t window,
                   int64_t* row_ptr, uint32_t* cols, int64_t* n_tiles);

/* ---- HeadCache (inc/cache.hpp:15-32; src/cache.cpp) --------------------
 * Device-resident: one bf16 slot [batch, N, d] per (layer, head), laid out
 * per layer as [batch, H, N, d] so cached heads copy back with the same
 * offsets as the output. produced_at bookkeeping is host-side. n_layers is
 * a capacity hint: any layer index >= 0 is accepted (storage grows), as in
 * the reference's map-backed cache. */
typedef struct dfa2c_cache dfa2c_cache;
int dfa2c_cache_create(int64_t n_layers, int64_t n_heads, int64_t batch,
                       int64_t seq_len, int64_t head_dim, dfa2c_cache** cache);
int dfa2c_cache_destroy(dfa2c_cache* cache);
int dfa2c_cache_has(const dfa2c_cache* cache, int64_t layer, int64_t head, int32_t* has);
int dfa2c_cache_produced_at(const dfa2c_cache* cache, int64_t layer, int64_t head,
                            int64_t* t); /* DFA2C_CACHE_MISS when empty */
int dfa2c_cache_staleness(const dfa2c_cache* cache, int64_t layer, int64_t head,
                          int64_t t, int64_t* staleness);
/* store: copies a device bf16 [batch, N, d] tensor into the slot (deep copy,
 * HeadCache::store). fetch: slot -> device [batch, N, d]. */
int dfa2c_cache_store(dfa2c_cache* cache, int64_t layer, int64_t head, const void* src,
                      int64_t t, void* stream);
int dfa2c_cache_fetch(const dfa2c_cache* cache, int64_t layer, int64_t head, void* dst,
                      void* stream);
int dfa2c_cache_clear(dfa2c_cache* cache);
int dfa2c_cache_size(const dfa2c_cache* cache, int64_t* n_entries);
int dfa2c_cache_bytes(const dfa2c_cache* cache, int64_t* bytes);

/* ---- the fused joint-attention call ------------------------------------
 * multi_strategy_attention (inc/dispatch.hpp:44-47; src/dispatch.cpp:30-91):
 * ONE kernel launch computes every Full and Arrow head with the sm_100a
 * tcgen05/TMA flash kernel over only the tiles the head's mask keeps, copies
 * every Cached head's stored slot into `out`, and commits computed heads to
 * the cache (dual store) — cached heads read the pre-call slot state and
 * keep their produced_at. `cache` may be NULL only if no head is Cached (then
 * nothing is committed). q/k/v/out: device bf16 [batch, H, N, d]. */
int dfa2c_mha_forward(const void* q, const void* k, const void* v, int64_t batch,
                      const dfa2c_dims* dims, int64_t block, const int32_t* kinds,
                      const int64_t* windows, dfa2c_cache* cache, int64_t layer,
                      int64_t t, void* out, void* stream);

/* Same call with HOST buffers (the reference's host-tensor calling
 * convention, inc/dispatch.hpp:44-47): q/k/v/out are host bf16
 * [batch, H, N, d] (pinned for full overlap; pageable works, slower). Only
 * the computed heads' q/k/v are uploaded, in head groups on a copy stream;
 * each group's fused launch starts as soon as its inputs land and its
 * outputs download while later groups upload and compute. Cached heads'
 * outputs go straight from the cache slot to `out`. The call is
 * asynchronous on `stream`: `out` is final once the stream reaches it.
 * Host inputs are read from the moment of the call (uploads may start
 * before earlier work on `stream` completes, overlapping the previous
 * call's download), so they must be ready when the call is made — as with
 * the reference's synchronous call.
 * Same validation, cache semantics and results as dfa2c_mha_forward. */
int dfa2c_mha_forward_host(const void* q, const void* k, const void* v, int64_t batch,
                           const dfa2c_dims* dims, int64_t block, const int32_t* kinds,
                           const int64_t* windows, dfa2c_cache* cache, int64_t layer,
                           int64_t t, void* out, void* stream);

/* ---- one layer on W GPUs (src/dispatch.cpp:62-83) --------
 * Every (sample, head, query block) is independent, so the layer shards with
 * no exchange inside it. dfa2c_mha_forward_sharded is the multi-GPU
 * multi_strategy_attention, called by every rank with the SAME replicated
 * q/k/v and plan:
 *  - the layer's (sample, head, query-tile pair) sequence is cut into
 *    `world` contiguous ranges of near-equal cost (cost = the pair's kept KV
 *    tiles; a Cached head's pair = its copy), so rank r owns one contiguous
 *    span [row_bounds[r], row_bounds[r+1]) of the flattened [batch*H*N]
 *    output rows and its ONE fused launch computes / copies / commits only
 *    those rows over all 148 SMs;
 *  - pairs longer than 1/(8*148) of the layer run as key chunks (split-KV
 *    against a fixed 8-GPU reference), so the bits of every head are the same
 *    for every `world` (1, 2, 4, 8 ... give identical outputs);
 *  - with nccl_comm (an ncclComm_t of `world` ranks, this rank = `rank`; the
 *    library binds libnccl.so.2 at run time) the ranges are all-gathered in
 *    place into `out` (one NCCL group of W broadcasts over NVLink/NVSwitch),
 *    and the other ranks' computed rows are committed into this rank's cache
 *    so every rank's cache is complete (a Cached head can then be served by
 *    whichever rank owns its rows at the next timestep). Without a comm the
 *    caller gathers `out` itself and then calls dfa2c_shard_commit.
 * row_bounds (optional, [world + 1]) receives the row ranges. Cached heads
 * need their slots on every rank (true when every layer runs through this
 * call). Asynchronous on `stream`. */
int dfa2c_mha_forward_sharded(const void* q, const void* k, const void* v, int64_t batch,
                              const dfa2c_dims* dims, int64_t block, const int32_t* kinds,
                              const int64_t* windows, dfa2c_cache* cache, int64_t layer, int64_t t,
                              void* out, int32_t rank, int32_t world, void* nccl_comm,
                              int64_t* row_bounds, void* stream);
/* The same sharded layer assembled over PEER MEMORY instead of a collective:
 * outs[world] holds every rank's output buffer as mapped in this process
 * (outs[rank] is this rank's own; the others opened with dfa2c_ipc_open).
 * This rank's ONE fused launch stores each output box of its row range to
 * its own out AND to every peer's, from the kernel epilogue over NVLink, so
 * the transfer overlaps the computation tile by tile and no all-gather runs.
 * Once every rank's launch has completed (the caller's cross-rank sync), all
 * outs hold the whole layer, bitwise the single-GPU sharded result; call
 * dfa2c_shard_commit to complete this rank's cache with the other rows.
 * world <= 8. Asynchronous on `stream`. */
int dfa2c_mha_forward_sharded_p2p(const void* q, const void* k, const void* v, int64_t batch,
                                  const dfa2c_dims* dims, int64_t block, const int32_t* kinds,
                                  const int64_t* windows, dfa2c_cache* cache, int64_t layer, int64_t t,
                                  void* const* outs, int32_t rank, int32_t world, int64_t* row_bounds,
                                  void* stream);
/* CUDA IPC for the peer buffers: a 64-byte handle + byte offset of a device
 * pointer (any pointer inside an allocation), its mapping in another process
 * (peer access enabled lazily), and the unmapping (same offset). */
int dfa2c_ipc_handle(const void* ptr, char* handle /* 64 bytes */, int64_t* offset);
int dfa2c_ipc_open(const char* handle, int64_t offset, void** ptr);
int dfa2c_ipc_close(void* ptr, int64_t offset);
/* The row ranges dfa2c_mha_forward_sharded gives each of `world` ranks for
 * this layer (host only, no GPU): row_bounds[world + 1] over the flattened
 * [batch*H*N] rows; bitwise the bounds the sharded call reports. */
int dfa2c_shard_rows(int64_t batch, const dfa2c_dims* dims, int64_t block, const int32_t* kinds,
                     const int64_t* windows, int32_t world, int64_t* row_bounds);
/* After a caller-side gather of a sharded call's `out`: commit the computed
 * heads' rows outside this rank's range into `cache`. */
int dfa2c_shard_commit(int64_t batch, const dfa2c_dims* dims, const int32_t* kinds, dfa2c_cache* cache,
                       int64_t layer, const int64_t* row_bounds, int32_t rank, int32_t world,
                       const void* out, void* stream);
/* NCCL plumbing for C / C++ callers without their own communicator.
 * dfa2c_nccl_unique_id fills 128 bytes on one rank (share them out of band);
 * every rank then calls dfa2c_nccl_comm_init with its rank (collective). */
int dfa2c_nccl_available(void);
int dfa2c_nccl_unique_id(char* id /* 128 bytes */);
int dfa2c_nccl_comm_init(const char* id, int32_t world, int32_t rank, void** comm);
int dfa2c_nccl_comm_destroy(void* comm);
/* In-place all-gather of unequal row ranges [row_bounds[r], row_bounds[r+1])
 * (rows of row_bytes bytes) of buf: one NCCL group of `world` broadcasts. */
int dfa2c_allgather_rows(void* comm, void* buf, const int64_t* row_bounds, int32_t world,
                         int64_t row_bytes, void* stream);

/* Split-KV scheduling for latency-bound layers (process-wide; default from
 * the environment, DFA2_SPLIT_KV=1). When on, a query-tile pair whose key
 * tiles cost more than the layer's average load per SM (reference 148 SMs)
 * runs as key chunks combined in a fixed order by the CTA finishing last:
 * e.g. a late-timestep layer with most heads Cached drops from being bound
 * by one arrow head's text rows. Results stay deterministic (independent
 * of batch, launch split and device) but each head then also depends on the
 * other heads' strategies, so the default is off (bitwise head isolation). */
int dfa2c_set_split_kv(int32_t on);

/* sparse_attention_forward (inc/arrow.hpp:59-63; src/arrow.cpp:171-208) for
 * `n_heads` independent [N, d] heads sharing one arbitrary block mask
 * (host bytes, nb*nb). Empty mask rows -> DFA2C_FULLY_MASKED. */
int dfa2c_sparse_attention_forward(const void* q, const void* k, const void* v,
                                   void* out, int64_t n_heads, int64_t seq_len,
                                   int64_t head_dim, const uint8_t* active,
                                   int64_t block, void* stream);
/* dense_tiled_attention (inc/arrow.hpp:67-69; src/arrow.cpp:210-228). */
int dfa2c_dense_attention_forward(const void* q, const void* k, const void* v, void* out,
                                  int64_t n_heads, int64_t seq_len, int64_t head_dim,
                                  void* stream);

/* attention_reference (inc/tensor.hpp:86-93; src/tensor.cpp:73-114, 268-295):
 * the reference's ground-truth masked attention at the CALLER's precision —
 * dtype DFA2C_F32 or DFA2C_F64, q/k/v/out device [n_heads, N, d] of that
 * type, computed in that type by a SIMT kernel (no bf16, no tensor cores):
 * scores, row max, exp, row sum, out = sum_j (w_j / sum) v_j. An independent
 * checker for the bf16 path (run_bench's oracle gate, cmd_verify); results
 * agree with the reference's sequential loops to rounding (~1e-6 relative in
 * f32). active (host nb*nb bytes, nb = ceil(N/block)) may be NULL (no mask);
 * an empty mask row -> DFA2C_FULLY_MASKED before any compute. head_dim <= 512.
 * Asynchronous on `stream` (synchronises when a mask is given). */
int dfa2c_attention_reference(const void* q, const void* k, const void* v, void* out, int32_t dtype,
                              int64_t n_heads, int64_t seq_len, int64_t head_dim, const uint8_t* active,
                              int64_t block, void* stream);

/* ---- calibration RSE query ---------------------------------------------
 * rse (inc/calibrate.hpp:18-20; src/calibrate.cpp:18-87) for `n_heads`
 * contiguous heads of `numel` elements each (y_m, y_o device, dtype
 * DFA2C_BF16, DFA2C_F32 or DFA2C_F64): fp64 accumulation, deterministic fixed-order
 * reduction. Writes out[n_heads] (HOST doubles) and synchronizes the
 * stream; DFA2C_DEGENERATE if any head's reference has zero variance. */
int dfa2c_rse(const void* y_m, const void* y_o, int32_t dtype, int64_t n_heads,
              int64_t numel, int32_t mode, double* out, void* stream);
/* Asynchronous variant: out_dev is a DEVICE double[n_heads]; degenerate
 * heads yield NaN instead of an error. */
int dfa2c_rse_async(const void* y_m, const void* y_o, int32_t dtype, int64_t n_heads,
                    int64_t numel, int32_t mode, double* out_dev, void* stream);

/* Element-type conversion of n device elements (DFA2C_BF16 / F32 / F64;
 * to bf16: round to nearest even). The C++ drop-in converts the reference's
 * f32 host tensors on the device with it. Asynchronous on `stream`. */
int dfa2c_convert(const void* src, int32_t src_dtype, void* dst, int32_t dst_dtype, int64_t n,
                  void* stream);

/* influence_for_layer (inc/calibrate.hpp:80-86; src/calibrate.cpp:193-253)
 * for one sample (batch 1): 1 original (all Full) + |M| candidate
 * evaluations, M = n_windows Arrow(w) candidates then Cached when
 * include_cached != 0 (make_candidates, src/calibrate.cpp:89-103).
 * influence[H*M] host (h*M + m), +inf where ineligible (Cached at t == 0 or
 * empty slot). original / method_outputs are optional device outputs
 * ([H,N,d] and [M,H,N,d] bf16); evals (optional) += 1 + M (the
 * reference's count of layer-level evaluations, whatever the launch count).
 * Synchronous.
 * When block == 128, the head dim is read in place (64, or 72..128 step 8)
 * and 1 <= n_windows <= 15, the original and every Arrow candidate come from
 * ONE fused launch: arrow masks are nested in w, so each
 * query tile folds its key tiles band by band and a snapshot of O / l after
 * band i is candidate i's output. Those outputs equal the per-candidate
 * passes' up to the key-tile fold order (bf16 rounding). */
int dfa2c_influence_for_layer(const void* q, const void* k, const void* v,
                              const dfa2c_dims* dims, int64_t block,
                              const int64_t* windows, int64_t n_windows,
                              int32_t include_cached, const dfa2c_cache* cache,
                              int64_t layer, int64_t t, int32_t mode, double* influence,
                              void* original, void* method_outputs, int64_t* evals,
                              void* stream);

/* Asynchronous influence_for_layer: the same launches, nothing synchronised.
 * rse_host (HOST double[M*H], pinned for true asynchrony) receives the raw
 * per-(m, h) RSE at index m*H + h when the stream reaches it; eligible (HOST
 * uint8[M*H], written before return) marks the measured entries.
 * dfa2c_influence_finalize turns both into influence[h*M + m] (+inf where
 * ineligible; DFA2C_DEGENERATE on a zero-variance reference). Lets a
 * calibration driver solve layer l while the GPU measures layer l+1. */
int dfa2c_influence_for_layer_async(const void* q, const void* k, const void* v,
                                    const dfa2c_dims* dims, int64_t block,
                                    const int64_t* windows, int64_t n_windows,
                                    int32_t include_cached, const dfa2c_cache* cache,
                                    int64_t layer, int64_t t, int32_t mode, double* rse_host,
                                    uint8_t* eligible, void* original, void* method_outputs,
                                    int64_t* evals, void* stream);
int dfa2c_influence_finalize(const double* rse_host, const uint8_t* eligible, int64_t n_heads,
                             int64_t n_methods, double* influence);

/* Drops every cached work list (plans are rebuilt on their next use) and
 * returns the library pool's unused device memory to the driver on the
 * current device (head-cache layers and in-flight scratch stay). The pool
 * otherwise keeps its memory for fast stream-ordered reuse. Synchronises
 * the device. */
int dfa2c_release_cached_memory(void);

/* Fused calibration pass switch (process-wide; default on, environment
 * DFA2_INFLUENCE_FUSED=0 turns it off): 0 = one launch per candidate, whose
 * outputs are bitwise dfa2c_mha_forward's for the same strategy. */
int dfa2c_set_influence_fused(int32_t on);
int32_t dfa2c_influence_fused_enabled(void);

/* ---- per-layer plan selection (calibration driver) ----------------------
 * The selection problem of calibrate_model (inc/plansolver.hpp:19-75;
 * src/calibrate.cpp:314-320): per head pick Full (full_cost, influence 0)
 * or one method m with finite influence[h*M + m] <= selection_cap, keeping
 * the summed influence <= delta, minimising the summed cost. Ties: lower
 * summed influence, then the lexicographically smaller choice vector
 * (method index, Full after every method). delta == 0 -> all Full.
 * choice[H] receives -1 (Full) or a method index. exhaustive != 0
 * enumerates every assignment (test oracle; (M+1)^H <= 1e7). Invalid
 * problems -> DFA2C_SHAPE (std::invalid_argument in the reference). */
double dfa2c_selection_cap(double coeff, int64_t n_heads, double delta);
int dfa2c_plan_solve(int64_t n_heads, int64_t n_methods, const double* influence,
                     double full_cost, const double* method_cost, double delta, double coeff,
                     int32_t exhaustive, int64_t* choice, double* objective,
                     double* total_influence, int64_t* nodes);
/* LP relaxation optimum (fractional multiple-choice knapsack) of the same problem. */
int dfa2c_plan_lp_bound(int64_t n_heads, int64_t n_methods, const double* influence,
                        double full_cost, const double* method_cost, double delta, double coeff,
                        double* bound);
/* analytic_costs: full_cost = 1, Arrow(w) = active fraction of its mask,
 * Cached = 0 (kinds/windows[n_methods] describe the candidates). */
int dfa2c_analytic_costs(const dfa2c_dims* dims, int64_t block, const int32_t* kinds,
                         const int64_t* windows, int64_t n_methods, double* full_cost,
                         double* method_cost);

/* ---- plan files (JSON version 1) ---------------------------------------
 * The reference's plan file format (inc/plan.hpp:44-52; src/plan.cpp:109-228):
 * {version, dims:{T,L,H,d,n_visual,n_text,block}, delta, coeff, window_set,
 *  plan:[{t, layer, heads:[{kind, window_blocks?}]}], influence_digest},
 * written with the same text layout as the reference (sorted keys, 2-space
 * indent, trailing newline). Plans are flat timestep-major arrays
 * kinds/windows[(t*L + l)*H + h] (CompressionPlan::at, src/plan.cpp:25-31). */
typedef struct {
    int64_t n_timesteps, n_layers, n_heads, head_dim, n_visual, n_text, block_size;
    double delta, coeff;
    int64_t n_window_set; /* entries of window_set */
    int64_t digest_len;   /* influence_digest bytes (excl. NUL); set by from_json */
} dfa2c_plan_header;
/* plan_to_json: buf may be NULL to query *len (bytes, excl. NUL); otherwise
 * cap must be >= *len + 1. No validation (as in the reference). */
int dfa2c_plan_to_json(const dfa2c_plan_header* hdr, const int32_t* kinds, const int64_t* windows,
                       const int64_t* window_set, const char* influence_digest, char* buf,
                       int64_t cap, int64_t* len);
/* plan_from_json: parses and validates (CompressionPlan::validate);
 * malformed text and schema violations -> DFA2C_PLAN. text_len < 0 means
 * NUL-terminated. Call with kinds == NULL to learn the header (sizes), then
 * with kinds/windows [T*L*H], window_set [n_window_set] and digest
 * [digest_len + 1]. */
int dfa2c_plan_from_json(const char* text, int64_t text_len, dfa2c_plan_header* hdr,
                         int32_t* kinds, int64_t* windows, int64_t* window_set, char* digest,
                         int64_t digest_cap);
/* fnv1a_hex (inc/plan.hpp:57-58): FNV-1a 64 of n bytes as 16 hex chars + NUL. */
int dfa2c_fnv1a_hex(const void* bytes, int64_t n, char* out);

/* ---- device workload generator ------------------------
 * The reference's synthetic MMDiT stream (generate(), src/workload.cpp:
 * 120-228: default locality/drift profiles, positional features from its
 * own seeded mt19937_64 draws, a per-timestep random walk) produced on the
 * GPU: per-element gaussians come from a counter-based Philox stream keyed
 * by the reference's derive_seed(seed, layer, head, t, tag), so any slot is
 * a pure function of (seed, t, layer) — same distribution as the reference,
 * not the same bits (dfa2::generate on the host stays bit-identical for
 * small streams). Each layer's walk state stays in HBM (fp32 [3, H, N, d],
 * allocated on first use); dfa2c_workload_slot writes slot (t, layer) as
 * bf16 q/k/v [H, N, d] on `stream`, stepping the layer's walk forward (or
 * restarting it for an earlier t). head_dim % 4 == 0. Not thread-safe. */
typedef struct dfa2c_workload dfa2c_workload;
int dfa2c_workload_create(const dfa2c_dims* dims, int64_t n_layers, int64_t block, uint64_t seed,
                          dfa2c_workload** w);
int dfa2c_workload_destroy(dfa2c_workload* w);
int dfa2c_workload_profile(const dfa2c_workload* w, int64_t layer, int64_t head, double* locality,
                           double* drift);
int dfa2c_workload_slot(dfa2c_workload* w, int64_t t, int64_t layer, void* q, void* k, void* v,
                        void* stream);

/* Kernel launches issued by this library since load (evidence counter). */
int64_t dfa2c_launch_count(void);
/* Debug: device buffer (int64 [2][4096][8]) receiving per-tile clock64 stamps
 * of CTA 0 from kernels built with -DDFA2_TRACE=1 (NULL disables). */
void dfa2c_debug_set_trace(void* dev_buffer);
/* Debug / test hook (no device work): the work-list scheduler's CTA
 * assignment for items of the given costs over n_ctas CTAs — LPT, then with
 * refine != 0 the move / swap improvement of the costliest CTA. cta_of[i]
 * receives item i's CTA, *max_load the costliest CTA's load. */
int dfa2c_debug_schedule(const double* costs, int64_t n, int32_t n_ctas, int32_t refine, int32_t* cta_of,
                         double* max_load);

#ifdef __cplusplus
}
#endif
#if defined(__GNUC__)
#pragma GCC visibility pop
#endif
#endif /* DFA2C_H */
