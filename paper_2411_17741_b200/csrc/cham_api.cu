// cham_api.cu — extern "C" LoRA-apply entry points (see include/chameleon_lora.h).
#include "cham_pool.h"

namespace cham {
int decode_entry(cham_pool* pool, int layer, int n_jobs, const int* projs, const void* const* xs,
                 void* const* ys, int n_tokens, const int* perm, const int* seg_off, const int* seg_slot,
                 const int* seg_rank, int n_seg, const int* n_seg_dev, const void* plan, void* stream, int mode,
                 float* v_out, const float* v_in, int v_stride, int v_cols);
size_t plan_bytes(const cham_pool* pool);
int build_plan_entry(cham_pool* pool, const int* perm, const int* seg_off, const int* seg_slot,
                     const int* seg_rank, int n_seg, const int* n_seg_dev, void* plan, void* stream);
}

using namespace cham;

extern "C" {

int cham_lora_apply(cham_pool* pool, int layer, int proj, const void* x, void* y, int n_tokens,
                    const int* perm, const int* seg_off, const int* seg_slot, const int* seg_rank,
                    int n_seg, const int* n_seg_dev, const void* plan, void* stream) {
  const void* xs[1] = {x};
  void* ys[1] = {y};
  return decode_entry(pool, layer, 1, &proj, xs, ys, n_tokens, perm, seg_off, seg_slot, seg_rank, n_seg,
                      n_seg_dev, plan, stream, /*MODE_FUSED*/ 0, nullptr, nullptr, 0, 0);
}

int cham_lora_apply_multi(cham_pool* pool, int layer, int n_jobs, const int* projs, const void* const* xs,
                          void* const* ys, int n_tokens, const int* perm, const int* seg_off,
                          const int* seg_slot, const int* seg_rank, int n_seg, const int* n_seg_dev,
                          const void* plan, void* stream) {
  if (!projs || !xs || !ys) return fail(CHAM_ERR_INVALID, "cham_lora_apply_multi: null argument");
  return decode_entry(pool, layer, n_jobs, projs, xs, ys, n_tokens, perm, seg_off, seg_slot, seg_rank, n_seg,
                      n_seg_dev, plan, stream, 0, nullptr, nullptr, 0, 0);
}

int cham_lora_shrink(cham_pool* pool, int layer, int proj, const void* x, float* v, int v_stride,
                     int n_tokens, const int* perm, const int* seg_off, const int* seg_slot,
                     const int* seg_rank, int n_seg, const int* n_seg_dev, const void* plan, void* stream) {
  if (!v || v_stride <= 0) return fail(CHAM_ERR_INVALID, "cham_lora_shrink: v / v_stride");
  const void* xs[1] = {x};
  void* ys[1] = {nullptr};
  return decode_entry(pool, layer, 1, &proj, xs, ys, n_tokens, perm, seg_off, seg_slot, seg_rank, n_seg,
                      n_seg_dev, plan, stream, /*MODE_SHRINK*/ 1, v, nullptr, v_stride, v_stride);
}

int cham_lora_expand(cham_pool* pool, int layer, int proj, const float* v, int v_stride, void* y,
                     int n_tokens, const int* perm, const int* seg_off, const int* seg_slot,
                     const int* seg_rank, int n_seg, const int* n_seg_dev, const void* plan, void* stream) {
  if (!v || v_stride <= 0) return fail(CHAM_ERR_INVALID, "cham_lora_expand: v / v_stride");
  const void* xs[1] = {nullptr};
  void* ys[1] = {y};
  return decode_entry(pool, layer, 1, &proj, xs, ys, n_tokens, perm, seg_off, seg_slot, seg_rank, n_seg,
                      n_seg_dev, plan, stream, /*MODE_EXPAND*/ 2, nullptr, v, v_stride, v_stride);
}

int cham_lora_shrink_multi(cham_pool* pool, int layer, int n_jobs, const int* projs, const void* const* xs, float* v,
                           int v_stride, int v_cols, int n_tokens, const int* perm, const int* seg_off,
                           const int* seg_slot, const int* seg_rank, int n_seg, const int* n_seg_dev, const void* plan,
                           void* stream) {
  if (!projs || !xs || !v || v_stride <= 0) return fail(CHAM_ERR_INVALID, "cham_lora_shrink_multi: null argument");
  void* ys[kMaxJobs] = {};
  return decode_entry(pool, layer, n_jobs, projs, xs, ys, n_tokens, perm, seg_off, seg_slot, seg_rank, n_seg,
                      n_seg_dev, plan, stream, /*MODE_SHRINK*/ 1, v, nullptr, v_stride, v_cols);
}

int cham_lora_expand_multi(cham_pool* pool, int layer, int n_jobs, const int* projs, const float* v, int v_stride,
                           int v_cols, void* const* ys, int n_tokens, const int* perm, const int* seg_off,
                           const int* seg_slot, const int* seg_rank, int n_seg, const int* n_seg_dev, const void* plan,
                           void* stream) {
  if (!projs || !ys || !v || v_stride <= 0) return fail(CHAM_ERR_INVALID, "cham_lora_expand_multi: null argument");
  const void* xs[kMaxJobs] = {};
  return decode_entry(pool, layer, n_jobs, projs, xs, ys, n_tokens, perm, seg_off, seg_slot, seg_rank, n_seg,
                      n_seg_dev, plan, stream, /*MODE_EXPAND*/ 2, nullptr, v, v_stride, v_cols);
}

size_t cham_plan_bytes(const cham_pool* pool) { return pool ? plan_bytes(pool) : 0; }

int cham_build_plan(cham_pool* pool, const int* perm, const int* seg_off, const int* seg_slot,
                    const int* seg_rank, int n_seg, const int* n_seg_dev, void* plan, void* stream) {
  return build_plan_entry(pool, perm, seg_off, seg_slot, seg_rank, n_seg, n_seg_dev, plan, stream);
}

size_t cham_plan_bytes_internal(const cham_pool* pool) { return plan_bytes(pool); }

}  // extern "C"
