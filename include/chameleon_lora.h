/*
 * chameleon_lora.h — C ABI of the B200-native batched heterogeneous-rank LoRA apply.
 *
 * This is the drop-in boundary for the one data-parallel hot path of Chameleon
 * (arXiv 2411.17741).  In the reference (`/root/reference/pkg/src/adaptersim`) the path
 * has no FFI at all: LoRA compute exists only as the modelled cost term of
 * `CostModel.step_duration` (engine.py:59-78, term at 67-77), adapter residency is the
 * pure-Python `AdapterCache` (adapter_cache.py:65-328) and host->GPU adapter loads are a
 * simulated FIFO link (`LinkState.enqueue`, engine.py:100-121).  Every entry point below
 * replaces one of those seams with real device work; the Python package
 * `paper_2411_17741_b200` binds them with ctypes.
 *
 * Conventions
 *  - All functions return 0 on success or a negative `cham_status` code.  No exception
 *    crosses the ABI.  `cham_last_error()` returns a thread-local message for the last
 *    failure.
 *  - Streams are passed as `void*` (a `cudaStream_t`); NULL means the legacy default stream.
 *  - Device pointers are plain `void*` / `int*`; sizes are in elements unless named `bytes`.
 *  - int32 tables (perm, seg_off, seg_slot, seg_rank, n_seg) live in device memory.
 *  - dtype: CHAM_F32 (fp32 storage, fp32 math) or CHAM_BF16 (bf16 storage, fp32 accumulate).
 */
#ifndef CHAMELEON_LORA_H
#define CHAMELEON_LORA_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define CHAM_API __attribute__((visibility("default")))
#else
#define CHAM_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  CHAM_OK = 0,
  CHAM_ERR_INVALID = -1,   /* bad argument (shape, alignment, range) */
  CHAM_ERR_CUDA = -2,      /* a CUDA runtime call failed */
  CHAM_ERR_OOM = -3,       /* device / pinned allocation failed */
  CHAM_ERR_LIMIT = -4,     /* a compiled-in limit was exceeded (segments, tokens, rank) */
  CHAM_ERR_UNSUPPORTED = -5
} cham_status;

enum { CHAM_F32 = 0, CHAM_BF16 = 1 };

/* Compiled-in limits (queried so the host side can validate before launching). */
typedef struct {
  int max_rank;           /* largest adapter rank a slot can hold (rows; multiple of 8 padding) */
  int max_segments;       /* largest segment count one lora_apply accepts */
  int max_jobs;           /* projections sharing one segment table in one launch */
  int max_requests;       /* largest batch the device segment builder accepts */
  int rows_per_page;      /* rank rows per pool page (8) */
  int tokens_per_tile;    /* decode kernel token tile */
  int prefill_min_tokens; /* segments at least this long are routed to the tcgen05 kernel */
} cham_limits;

typedef struct cham_pool cham_pool;

CHAM_API const char* cham_last_error(void);
CHAM_API int cham_get_limits(cham_limits* out);
CHAM_API int cham_device_sm_count(int device, int* out);

/* ---------------------------------------------------------------------------------------
 * Paged adapter pool (replaces AdapterCache residency bookkeeping's *storage* side:
 * `begin_load` (adapter_cache.py:144-151) reserves pages, `finish_load` (153-159) is the
 * completion of `cham_pool_fill_async`; `_evict` (220-226) returns pages to the host-side
 * allocator.  Decisions stay in the host cache, bit-exact with the reference).
 *
 * Layout: a page holds 8 rank rows of one adapter for every (layer, projection).  Inside
 * a page, (layer, proj) blocks are stored in order; each block is A^T [8, h_in] followed by
 * B [8, h_out], both tiled in 1 KiB atoms of 8 rows x 128 bytes with the 128-byte XOR
 * swizzle (16-byte chunk c of row j stored at chunk c ^ j).  page_bytes =
 * sum_{l,p} 8 * (h_in[p] + h_out[p]) * elem_bytes (16 MiB for Llama-2-7B bf16 q/k/v/o).
 * ------------------------------------------------------------------------------------- */
CHAM_API int cham_pool_create(cham_pool** out, int device, int n_pages, int n_layers, int n_proj,
                     const int* h_in, const int* h_out, int dtype, int n_slots,
                     int max_tokens);
CHAM_API int cham_pool_destroy(cham_pool* pool);
CHAM_API int cham_pool_page_bytes(const cham_pool* pool, size_t* out);
CHAM_API int cham_pool_block_offsets(const cham_pool* pool, int layer, int proj, size_t* a_off,
                            size_t* b_off);
/* Device base of page 0 (pages are contiguous: page p at base + p * page_bytes). */
CHAM_API int cham_pool_base(const cham_pool* pool, void** out);
/* Bind `slot` to `rank` rows stored in `pages[0 .. ceil(rank/8))`; rank 0 unbinds. The
 * device slot table is updated on `stream` (stream-ordered with later applies). */
CHAM_API int cham_pool_set_slot(cham_pool* pool, int slot, int rank, const int* pages, int n_pages,
                       void* stream);
/* Copy a packed adapter (ceil(rank/8) pages back to back, host memory — pinned for true
 * async) into the slot's pages on `stream`, then record `done` (cudaEvent_t, may be NULL).
 * Replaces LinkState.enqueue (engine.py:115-121). */
CHAM_API int cham_pool_fill_async(cham_pool* pool, int slot, const void* host_src, size_t bytes,
                         void* stream, void* done);
/* Same, but from a device buffer (used by the bench to populate the pool quickly). */
CHAM_API int cham_pool_fill_from_device(cham_pool* pool, int slot, const void* dev_src, size_t bytes,
                               void* stream);

/* Copy `bytes` of pool storage starting at byte `offset` from page 0's base into `dst`
 * (host or device memory; synchronous on `stream`).  Introspection / tests. */
CHAM_API int cham_pool_copy_out(const cham_pool* pool, size_t offset, size_t bytes, void* dst, void* stream);

/* Routing of prefill-sized segments to the tcgen05 kernels (K3, bf16 pools whose h_in and
 * h_out are multiples of 128).  A segment with >= min_tokens tokens and rank <= 128 runs on
 * the tensor cores; every other segment runs on the decode GEMV kernel.  min_tokens <= 0
 * disables the tcgen05 path.  min/max_segment_tokens are optional host hints about the
 * segments of the steps that follow (0 / -1 = unknown): with max < min_tokens the tcgen05
 * kernels are not launched, with min >= min_tokens the decode kernel is not launched.  Set
 * the route before cham_build_plan and keep it for the step (the plan and the launches must
 * agree).  Default: min_tokens = 64 (prefill_min_tokens of cham_limits), no hints. */
CHAM_API int cham_pool_set_prefill_route(cham_pool* pool, int min_tokens, int min_segment_tokens,
                                         int max_segment_tokens);

/* Cross-apply weight prefetch (no reference counterpart: the reference simulates the step,
 * engine.py:67-77).  cham_pool_set_next_apply names the (layer, projections) that the caller
 * launches right after the NEXT apply on this pool, with the same segment table and plan;
 * it is consumed (cleared) by that apply.  Its CTAs, once they run out of units, pull the
 * first `bytes` (cham_pool_set_l2_prefetch, default 0 = off) of the hinted apply's A blocks,
 * in the hinted apply's unit order, into L2 — HBM work that does not depend on the current
 * apply, done while its tail and the launch boundary leave bandwidth idle.  Results never
 * depend on the hint (a wrong hint only wastes bandwidth).  n_projs <= 0 clears it. */
CHAM_API int cham_pool_set_next_apply(cham_pool* pool, int layer, int n_projs, const int* projs);
CHAM_API int cham_pool_set_l2_prefetch(cham_pool* pool, long long bytes);

/* Device-side error word of the pool's kernels (0 = none).  Kernels that meet a
 * compiled-in limit only known on the device (segment count read from n_seg_dev, more than
 * kPrefillMaxTiles prefill tiles, plan totals above max_tokens) leave y untouched and set
 * it to CHAM_ERR_LIMIT.  Synchronises `stream`; clear != 0 resets the word.
 * Pools are limited to 65535 pages and 65535 max_tokens (cham_pool_create). */
CHAM_API int cham_pool_device_error(cham_pool* pool, int* device_error, int clear, void* stream);

/* Debug: record a per-item timeline of the decode kernel into `dev_buf`
 * (2 x [sm_count][items_per_cta][8] u64 — shrink kernel then expand kernel: producer issue
 * ns, kind<<32|bytes, consumer start ns, consumer end ns).  NULL disables.  Not for production use (adds global stores). */
CHAM_API int cham_debug_set_trace(cham_pool* pool, void* dev_buf, int items_per_cta);

/* Pack one adapter into page format on the host.  a: [n_layers][n_proj][h_in[p]][rank]
 * (column layout of `x @ A`), b: [n_layers][n_proj][rank][h_out[p]], both row-major in the
 * pool dtype; out: ceil(rank/8) * page_bytes bytes (pad rows are zero).  For projection
 * p the A/B pointers are at the running offsets of the previous (l,p) blocks. */
CHAM_API int cham_pack_adapter_host(const cham_pool* pool, int rank, const void* a, const void* b,
                           void* out);
/* Same packing from an explicit geometry (no pool, no GPU needed). */
CHAM_API int cham_pack_adapter_host_geom(int n_layers, int n_proj, const int* h_in, const int* h_out,
                                         int dtype, int rank, const void* a, const void* b, void* out);
/* Device variant of the same packing (a, b, out in device memory). */
CHAM_API int cham_pack_adapter_device(const cham_pool* pool, int rank, const void* a, const void* b,
                             void* out, void* stream);

/* ---------------------------------------------------------------------------------------
 * Segment-table builder (K4) — replaces the per-request Python loop of
 * CostModel.step_duration (engine.py:64-76).  Requests are in batch order (prefills then
 * decoders, engine.py:443-451); request i owns tokens [sum_{j<i} ntok_j, ... + ntok_i).
 * Output: a stable group-by-slot of the requests (ties keep batch order), segments in
 * ascending slot order; perm[k] = original token index at grouped position k;
 * seg_off[S+1]; seg_slot[S]; seg_rank[S]; n_seg[0] = S.  Requests with slot < 0 carry no
 * adapter and are left out of perm.  n_req <= max_requests.
 * ------------------------------------------------------------------------------------- */
CHAM_API int cham_build_segments(const int* req_slot, const int* req_rank, const int* req_ntok,
                        int n_req, int* perm, int* seg_off, int* seg_slot, int* seg_rank,
                        int* n_seg, void* stream);

/* ---------------------------------------------------------------------------------------
 * Batched heterogeneous-rank LoRA apply: y[t] += (x[t] . A_slot) . B_slot for every token
 * t of every segment, A/B read from the pool pages of the segment's slot for (layer, proj).
 * The reference operator is lora_apply(x, y, slot_ids, segment offsets, ranks); it replaces
 * the modelled term adapter_compute_per_rank_token_us * adapter_units (engine.py:67-77).
 *   x: [T, h_in[proj]] and y: [T, h_out[proj]], row-major, pool dtype; y is updated in place.
 *   n_tokens: rows of x / y (T); every perm entry and seg_off[S] must be <= T <= the
 *   pool's max_tokens.
 *   perm: grouped position -> token row (NULL = identity).
 *   n_seg >= 0: host segment count; n_seg < 0: read the count from n_seg_dev (device).
 *   plan: optional launch plan from cham_build_plan for this segment table (NULL = the
 *   kernels derive it themselves, at a few microseconds per launch).
 * Decode-sized segments run the fused shrink->expand GEMV kernel; segments of at least
 * prefill_min_tokens tokens in bf16 run the tcgen05 kernel.
 * ------------------------------------------------------------------------------------- */
CHAM_API int cham_lora_apply(cham_pool* pool, int layer, int proj, const void* x, void* y,
                    int n_tokens, const int* perm, const int* seg_off, const int* seg_slot,
                    const int* seg_rank, int n_seg, const int* n_seg_dev, const void* plan, void* stream);

/* Launch plan for one segment table against the pool's current slot table, built on the
 * device by one CTA: segment prefix sums, largest-rank-first order, page ids, perm, and a
 * 32-byte work descriptor per shrink unit / expand tile.  Valid while the slots of the batch
 * stay bound (their adapters are pinned for the step), so one plan serves every
 * (layer, projection) apply of a step.  `plan` is device memory of cham_plan_bytes(pool)
 * bytes, 16-byte aligned. */
CHAM_API size_t cham_plan_bytes(const cham_pool* pool);
CHAM_API int cham_build_plan(cham_pool* pool, const int* perm, const int* seg_off, const int* seg_slot,
                             const int* seg_rank, int n_seg, const int* n_seg_dev, void* plan,
                             void* stream);

/* Several projections of one layer that share the token batch (e.g. q/k/v over the same
 * normed hidden state) in ONE launch.  All projections must have equal h_in and h_out. */
CHAM_API int cham_lora_apply_multi(cham_pool* pool, int layer, int n_jobs, const int* projs,
                          const void* const* xs, void* const* ys, int n_tokens,
                          const int* perm,
                          const int* seg_off, const int* seg_slot, const int* seg_rank,
                          int n_seg, const int* n_seg_dev, const void* plan, void* stream);

/* Tensor-parallel halves (config C5).  shrink: v[k, 0:r] = x[perm[k]] . A_slot (fp32, rows
 * laid out [grouped position][v_stride]); expand: y[perm[k]] += v[k] . B_slot.  With A
 * sharded on h_in across ranks the caller all-reduces v between the two calls. */
CHAM_API int cham_lora_shrink(cham_pool* pool, int layer, int proj, const void* x, float* v,
                     int v_stride, int n_tokens, const int* perm, const int* seg_off, const int* seg_slot,
                     const int* seg_rank, int n_seg, const int* n_seg_dev, const void* plan, void* stream);
CHAM_API int cham_lora_expand(cham_pool* pool, int layer, int proj, const float* v, int v_stride,
                     void* y, int n_tokens, const int* perm, const int* seg_off, const int* seg_slot,
                     const int* seg_rank, int n_seg, const int* n_seg_dev, const void* plan, void* stream);

/* Tensor-parallel halves over several projections of one layer in ONE launch each: job j
 * (projection projs[j]) owns v columns [j * v_cols, (j + 1) * v_cols) of every v row, so the
 * q/k/v shrink outputs land side by side in the single buffer that is all-reduced.  shrink:
 * the projections must share h_in; expand: they must share h_out.  n_jobs <= 4,
 * n_jobs * v_cols <= v_stride, v_cols a multiple of 4; ranks beyond v_cols are dropped. */
CHAM_API int cham_lora_shrink_multi(cham_pool* pool, int layer, int n_jobs, const int* projs,
                     const void* const* xs, float* v, int v_stride, int v_cols, int n_tokens,
                     const int* perm, const int* seg_off, const int* seg_slot, const int* seg_rank,
                     int n_seg, const int* n_seg_dev, const void* plan, void* stream);
CHAM_API int cham_lora_expand_multi(cham_pool* pool, int layer, int n_jobs, const int* projs,
                     const float* v, int v_stride, int v_cols, void* const* ys, int n_tokens,
                     const int* perm, const int* seg_off, const int* seg_slot, const int* seg_rank,
                     int n_seg, const int* n_seg_dev, const void* plan, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* CHAMELEON_LORA_H */
