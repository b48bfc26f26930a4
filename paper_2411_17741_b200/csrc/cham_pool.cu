// cham_pool.cu — paged adapter pool in HBM, slot table, pinned miss fills, page packing.
//
// Reference seams replaced:
//   AdapterCache.begin_load / finish_load (adapter_cache.py:144-159): page reservation +
//     cham_pool_fill_async completion event;
//   LinkState.enqueue (engine.py:115-121): a real pinned cudaMemcpyAsync on a side stream;
//   DEFAULT_BYTES_PER_RANK_UNIT (model.py:23-26): page_bytes / 8 equals the reference's
//     2 MiB-per-rank byte model for Llama-2-7B q/k/v/o in bf16.
#include <algorithm>
#include <cstring>
#include <string>

#include <vector>

#include "cham_pool.h"

namespace cham {

static thread_local std::string g_last_error;

void set_error(const std::string& msg) { g_last_error = msg; }

int fail(int code, const std::string& msg) {
  set_error(msg);
  return code;
}

int cuda_fail(cudaError_t e, const char* what) {
  set_error(std::string(what) + ": " + cudaGetErrorString(e));
  return e == cudaErrorMemoryAllocation ? CHAM_ERR_OOM : CHAM_ERR_CUDA;
}

struct SlotRow {
  int pages[kMaxPagesPerSlot];
};

__global__ void set_slot_kernel(int* slot_pages, int* slot_rank, int slot, int rank,
                                SlotRow row) {
  int i = threadIdx.x;
  if (i < kMaxPagesPerSlot) slot_pages[slot * kMaxPagesPerSlot + i] = row.pages[i];
  if (i == 0) slot_rank[slot] = rank;
}

// One thread per 16-byte output chunk of one page.  a: [L][P][h_in][rank], b: [L][P][rank][h_out]
template <int ES>
__global__ void pack_kernel(const char* __restrict__ a, const char* __restrict__ b,
                            char* __restrict__ out, int rank, int n_lp, const int* __restrict__ hin_lp,
                            const int* __restrict__ hout_lp, const long long* __restrict__ aoff_lp,
                            const long long* __restrict__ boff_lp,
                            const long long* __restrict__ asrc_lp,
                            const long long* __restrict__ bsrc_lp, long long page_bytes) {
  const int page = blockIdx.y;
  const long long chunk = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const long long n_chunks = page_bytes / 16;
  if (chunk >= n_chunks) return;
  const long long byte = chunk * 16;
  // locate the (l,p) block and A/B part by scanning (n_lp is small: <= a few hundred)
  int lp = 0;
  while (lp + 1 < n_lp && aoff_lp[lp + 1] <= byte) ++lp;
  const bool is_b = byte >= boff_lp[lp];
  const long long blk = byte - (is_b ? boff_lp[lp] : aoff_lp[lp]);
  const int atom = static_cast<int>(blk / kAtomBytes);
  const int in_atom = static_cast<int>(blk % kAtomBytes);
  const int j = in_atom / kRowBytes;
  const int stored_chunk = (in_atom % kRowBytes) / 16;
  const int logical_chunk = stored_chunk ^ j;
  constexpr int EPV = 16 / ES;
  constexpr int ATOM_E = kRowBytes / ES;
  const int r = page * kRowsPerPage + j;
  alignas(16) char buf[16];
  for (int e = 0; e < EPV; ++e) {
    const int col = atom * ATOM_E + logical_chunk * EPV + e;  // k (A) or n (B)
    const char* src = nullptr;
    if (r < rank) {
      if (!is_b) {
        src = a + asrc_lp[lp] + ((long long)col * rank + r) * ES;
      } else {
        src = b + bsrc_lp[lp] + ((long long)r * hout_lp[lp] + col) * ES;
      }
    }
    for (int q = 0; q < ES; ++q) buf[e * ES + q] = src ? src[q] : 0;
  }
  *reinterpret_cast<uint4*>(out + page * page_bytes + byte) = *reinterpret_cast<uint4*>(buf);
}

}  // namespace cham

using namespace cham;

extern "C" {

const char* cham_last_error(void) { return cham::g_last_error.c_str(); }

int cham_get_limits(cham_limits* out) {
  if (!out) return fail(CHAM_ERR_INVALID, "cham_get_limits: null");
  out->max_rank = kMaxRank;
  out->max_segments = kMaxSegments;
  out->max_jobs = kMaxJobs;
  out->max_requests = kMaxRequests;
  out->rows_per_page = kRowsPerPage;
  out->tokens_per_tile = 4;
  out->prefill_min_tokens = kPrefillMinTokens;  // default of bf16 pools (cham_pool_set_prefill_route)
  return CHAM_OK;
}

int cham_device_sm_count(int device, int* out) {
  if (!out) return fail(CHAM_ERR_INVALID, "null");
  CHAM_CUDA(cudaDeviceGetAttribute(out, cudaDevAttrMultiProcessorCount, device));
  return CHAM_OK;
}

int cham_pool_create(cham_pool** out, int device, int n_pages, int n_layers, int n_proj,
                     const int* h_in, const int* h_out, int dtype, int n_slots, int max_tokens) {
  if (!out || !h_in || !h_out) return fail(CHAM_ERR_INVALID, "cham_pool_create: null argument");
  *out = nullptr;
  if (n_pages < 0 || n_layers <= 0 || n_proj <= 0 || n_slots <= 0 || max_tokens <= 0)
    return fail(CHAM_ERR_INVALID, "cham_pool_create: non-positive geometry");
  if (dtype != CHAM_F32 && dtype != CHAM_BF16)
    return fail(CHAM_ERR_INVALID, "cham_pool_create: dtype must be CHAM_F32 or CHAM_BF16");
  // the step plan stores page ids and token rows as 16-bit values
  if (n_pages > kMaxPoolPages)
    return fail(CHAM_ERR_LIMIT, "cham_pool_create: n_pages exceeds " + std::to_string(kMaxPoolPages));
  if (max_tokens > kMaxPoolTokens)
    return fail(CHAM_ERR_LIMIT, "cham_pool_create: max_tokens exceeds " + std::to_string(kMaxPoolTokens));
  const int es = dtype == CHAM_F32 ? 4 : 2;
  const int atom_e = kRowBytes / es;
  int hin_max = 0;
  for (int p = 0; p < n_proj; ++p) {
    if (h_in[p] <= 0 || h_out[p] <= 0 || h_in[p] % atom_e || h_out[p] % atom_e)
      return fail(CHAM_ERR_INVALID, "cham_pool_create: h_in/h_out must be positive multiples of " +
                                        std::to_string(atom_e));
    if ((long long)h_in[p] * es > (long long)kMaxKChunks * kActRowBytes)
      return fail(CHAM_ERR_LIMIT, "cham_pool_create: h_in too large");
    hin_max = std::max(hin_max, h_in[p]);
  }
  cham_pool* pool = new cham_pool();
  pool->device = device;
  pool->n_pages = n_pages;
  pool->n_layers = n_layers;
  pool->n_proj = n_proj;
  pool->dtype = dtype;
  pool->es = es;
  pool->n_slots = n_slots;
  pool->max_tokens = max_tokens;
  pool->h_in.assign(h_in, h_in + n_proj);
  pool->h_out.assign(h_out, h_out + n_proj);
  size_t off = 0;
  for (int l = 0; l < n_layers; ++l)
    for (int p = 0; p < n_proj; ++p) {
      pool->a_off.push_back(off);
      off += (size_t)kRowsPerPage * h_in[p] * es;
      pool->b_off.push_back(off);
      off += (size_t)kRowsPerPage * h_out[p] * es;
    }
  pool->page_bytes = off;
  pool->prefill_ok = dtype == CHAM_BF16;
  for (int p = 0; p < n_proj; ++p)
    if (h_in[p] % 128 || h_out[p] % 128) pool->prefill_ok = false;
  pool->prefill_min_tokens = pool->prefill_ok ? kPrefillMinTokens : 0;
  pool->vws_kc = (int)((hin_max * es + kActRowBytes - 1) / kActRowBytes);
  pool->slot_rank.assign(n_slots, 0);
  pool->slot_pages.assign((size_t)n_slots * kMaxPagesPerSlot, -1);

  int prev = 0;
  cudaGetDevice(&prev);
  auto cleanup = [&](int code, const std::string& msg) {
    cudaFree(pool->base);
    cudaFree(pool->d_slot_pages);
    cudaFree(pool->d_slot_rank);
    cudaFree(pool->d_ctr);
    cudaFree(pool->d_vws);
    cudaFree(pool->d_plan);
    cudaFree(pool->d_pvimg);
    cudaFree(pool->d_ppart);
    cudaFree(pool->d_pctr);
    cudaFree(pool->d_iota);
    cudaFree(pool->d_split);
    cudaFree(pool->d_split_ctr);
    delete pool;
    cudaSetDevice(prev);
    return fail(code, msg);
  };
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) return cleanup(CHAM_ERR_CUDA, std::string("cudaSetDevice: ") + cudaGetErrorString(e));
  cudaDeviceGetAttribute(&pool->sm_count, cudaDevAttrMultiProcessorCount, device);
  if (n_pages > 0) {
    e = cudaMalloc(&pool->base, (size_t)n_pages * pool->page_bytes);
    if (e != cudaSuccess)
      return cleanup(CHAM_ERR_OOM, "cham_pool_create: cannot allocate " +
                                       std::to_string((size_t)n_pages * pool->page_bytes) +
                                       " bytes of pages");
  }
  e = cudaMalloc(&pool->d_slot_pages, sizeof(int) * (size_t)n_slots * kMaxPagesPerSlot);
  if (e == cudaSuccess) e = cudaMalloc(&pool->d_slot_rank, sizeof(int) * (size_t)n_slots);
  const size_t n_ctr = cham::ctr_ints(max_tokens);
  if (e == cudaSuccess) e = cudaMalloc(&pool->d_ctr, sizeof(int) * n_ctr);
  if (e == cudaSuccess)
    e = cudaMalloc(&pool->d_vws, 2 * sizeof(float) * (size_t)kMaxJobs * max_tokens * kMaxRank);
  if (e == cudaSuccess) {
    extern size_t cham_plan_bytes_internal(const cham_pool*);
    e = cudaMalloc(&pool->d_plan, cham_plan_bytes_internal(pool));
  }
  {
    int hout_max = 0;
    for (int p = 0; p < n_proj; ++p) hout_max = hout_max > h_out[p] ? hout_max : h_out[p];
    pool->split_ncc = (int)(((size_t)hout_max * es + kSplitNcb - 1) / kSplitNcb);
  }
  const size_t n_split = (size_t)kMaxJobs * kSplitCap * pool->split_ncc;
  if (e == cudaSuccess)  // fp32 partial: kSplitTG tokens x (kSplitNcb / es) columns per slot
    e = cudaMalloc(&pool->d_split, n_split * kSplitTG * (kSplitNcb / es) * sizeof(float));
  if (e == cudaSuccess) e = cudaMalloc(&pool->d_split_ctr, 2 * n_split * sizeof(int));
  if (e == cudaSuccess) e = cudaMemset(pool->d_split_ctr, 0, 2 * n_split * sizeof(int));
  if (e == cudaSuccess && pool->prefill_ok)
    e = cudaMalloc(&pool->d_pvimg, (size_t)kMaxJobs * kPrefillMaxTiles * kPrefillVImg);
  if (e == cudaSuccess && pool->prefill_ok)
    e = cudaMalloc(&pool->d_ppart, (size_t)kMaxJobs * kPrefillMaxTiles * kPrefillPart);
  if (e == cudaSuccess && pool->prefill_ok) e = cudaMalloc(&pool->d_pctr, sizeof(int) * prefill_ctr_ints());
  if (e == cudaSuccess && pool->prefill_ok) e = cudaMemset(pool->d_pctr, 0, sizeof(int) * prefill_ctr_ints());
  if (e == cudaSuccess && pool->prefill_ok) e = cudaMalloc(&pool->d_iota, sizeof(int) * (size_t)max_tokens);
  if (e == cudaSuccess && pool->prefill_ok) {
    std::vector<int> iota(max_tokens);
    for (int i = 0; i < max_tokens; ++i) iota[i] = i;
    e = cudaMemcpy(pool->d_iota, iota.data(), sizeof(int) * (size_t)max_tokens, cudaMemcpyHostToDevice);
  }
  if (e != cudaSuccess) return cleanup(CHAM_ERR_OOM, "cham_pool_create: workspace allocation failed");
  cudaMemset(pool->d_slot_pages, 0xff, sizeof(int) * (size_t)n_slots * kMaxPagesPerSlot);
  cudaMemset(pool->d_slot_rank, 0, sizeof(int) * (size_t)n_slots);
  cudaMemset(pool->d_ctr, 0, sizeof(int) * n_ctr);
  e = cudaDeviceSynchronize();
  if (e != cudaSuccess) return cleanup(CHAM_ERR_CUDA, std::string("cham_pool_create: ") + cudaGetErrorString(e));
  cudaSetDevice(prev);
  *out = pool;
  return CHAM_OK;
}

int cham_pool_destroy(cham_pool* pool) {
  if (!pool) return CHAM_OK;
  cudaDeviceSynchronize();
  cudaFree(pool->base);
  cudaFree(pool->d_slot_pages);
  cudaFree(pool->d_slot_rank);
  cudaFree(pool->d_ctr);
  cudaFree(pool->d_vws);
  cudaFree(pool->d_plan);
  cudaFree(pool->d_pvimg);
  cudaFree(pool->d_ppart);
  cudaFree(pool->d_pctr);
  cudaFree(pool->d_iota);
  cudaFree(pool->d_split);
  cudaFree(pool->d_split_ctr);
  delete pool;
  return CHAM_OK;
}

int cham_pool_set_prefill_route(cham_pool* pool, int min_tokens, int min_segment_tokens,
                                int max_segment_tokens) {
  if (!pool) return fail(CHAM_ERR_INVALID, "cham_pool_set_prefill_route: null pool");
  if (min_tokens > 0 && !pool->prefill_ok)
    return fail(CHAM_ERR_UNSUPPORTED,
                "cham_pool_set_prefill_route: the tcgen05 path needs a bf16 pool with h_in, h_out multiples of 128");
  pool->prefill_min_tokens = min_tokens > 0 ? min_tokens : 0;
  pool->route_min_seg = min_segment_tokens > 0 ? min_segment_tokens : 0;
  pool->route_max_seg = max_segment_tokens >= 0 ? max_segment_tokens : (1 << 30);
  return CHAM_OK;
}

int cham_pool_set_next_apply(cham_pool* pool, int layer, int n_projs, const int* projs) {
  if (!pool) return fail(CHAM_ERR_INVALID, "cham_pool_set_next_apply: null pool");
  if (n_projs <= 0) {
    pool->next_n = 0;
    return CHAM_OK;
  }
  if (n_projs > cham::kMaxJobs || !projs) return fail(CHAM_ERR_INVALID, "cham_pool_set_next_apply: 1..max_jobs projections");
  if (layer < 0 || layer >= pool->n_layers) return fail(CHAM_ERR_INVALID, "cham_pool_set_next_apply: layer out of range");
  for (int j = 0; j < n_projs; ++j) {
    if (projs[j] < 0 || projs[j] >= pool->n_proj) return fail(CHAM_ERR_INVALID, "cham_pool_set_next_apply: proj out of range");
    if (pool->h_in[projs[j]] != pool->h_in[projs[0]])
      return fail(CHAM_ERR_INVALID, "cham_pool_set_next_apply: projections must share h_in");
    pool->next_a_off[j] = pool->a_off[(size_t)layer * pool->n_proj + projs[j]];
  }
  pool->next_a_bytes = kRowsPerPage * pool->h_in[projs[0]] * pool->es;
  pool->next_n = n_projs;
  return CHAM_OK;
}

int cham_pool_set_l2_prefetch(cham_pool* pool, long long bytes) {
  if (!pool || bytes < 0) return fail(CHAM_ERR_INVALID, "cham_pool_set_l2_prefetch: null pool or negative budget");
  pool->l2_prefetch_bytes = bytes;
  return CHAM_OK;
}

int cham_pool_page_bytes(const cham_pool* pool, size_t* out) {
  if (!pool || !out) return fail(CHAM_ERR_INVALID, "null");
  *out = pool->page_bytes;
  return CHAM_OK;
}

int cham_pool_block_offsets(const cham_pool* pool, int layer, int proj, size_t* a_off, size_t* b_off) {
  if (!pool || layer < 0 || layer >= pool->n_layers || proj < 0 || proj >= pool->n_proj)
    return fail(CHAM_ERR_INVALID, "cham_pool_block_offsets: bad layer/proj");
  const int lp = layer * pool->n_proj + proj;
  if (a_off) *a_off = pool->a_off[lp];
  if (b_off) *b_off = pool->b_off[lp];
  return CHAM_OK;
}

int cham_pool_base(const cham_pool* pool, void** out) {
  if (!pool || !out) return fail(CHAM_ERR_INVALID, "null");
  *out = pool->base;
  return CHAM_OK;
}

int cham_pool_set_slot(cham_pool* pool, int slot, int rank, const int* pages, int n_pages,
                       void* stream) {
  if (!pool) return fail(CHAM_ERR_INVALID, "cham_pool_set_slot: null pool");
  if (slot < 0 || slot >= pool->n_slots) return fail(CHAM_ERR_INVALID, "cham_pool_set_slot: slot out of range");
  if (rank < 0 || rank > kMaxRank) return fail(CHAM_ERR_LIMIT, "cham_pool_set_slot: rank exceeds max_rank");
  const int need = (rank + kRowsPerPage - 1) / kRowsPerPage;
  if (n_pages != need) return fail(CHAM_ERR_INVALID, "cham_pool_set_slot: n_pages != ceil(rank/8)");
  SlotRow row;
  for (int i = 0; i < kMaxPagesPerSlot; ++i) row.pages[i] = -1;
  for (int i = 0; i < n_pages; ++i) {
    if (!pages || pages[i] < 0 || pages[i] >= pool->n_pages)
      return fail(CHAM_ERR_INVALID, "cham_pool_set_slot: page id out of range");
    row.pages[i] = pages[i];
  }
  for (int i = 0; i < kMaxPagesPerSlot; ++i)
    pool->slot_pages[(size_t)slot * kMaxPagesPerSlot + i] = row.pages[i];
  pool->slot_rank[slot] = rank;
  set_slot_kernel<<<1, 32, 0, (cudaStream_t)stream>>>(pool->d_slot_pages, pool->d_slot_rank, slot,
                                                      rank, row);
  CHAM_CUDA(cudaGetLastError());
  return CHAM_OK;
}

static int fill_common(cham_pool* pool, int slot, const void* src, size_t bytes, void* stream,
                       cudaMemcpyKind kind) {
  if (!pool || !src) return fail(CHAM_ERR_INVALID, "cham_pool_fill: null argument");
  if (slot < 0 || slot >= pool->n_slots) return fail(CHAM_ERR_INVALID, "cham_pool_fill: slot out of range");
  const int rank = pool->slot_rank[slot];
  const int np = (rank + kRowsPerPage - 1) / kRowsPerPage;
  if (np == 0) return fail(CHAM_ERR_INVALID, "cham_pool_fill: slot is not bound (set_slot first)");
  if (bytes != (size_t)np * pool->page_bytes)
    return fail(CHAM_ERR_INVALID, "cham_pool_fill: bytes != ceil(rank/8) * page_bytes");
  const char* s = static_cast<const char*>(src);
  for (int i = 0; i < np; ++i) {
    const int page = pool->slot_pages[(size_t)slot * kMaxPagesPerSlot + i];
    CHAM_CUDA(cudaMemcpyAsync(pool->base + (size_t)page * pool->page_bytes, s + (size_t)i * pool->page_bytes,
                              pool->page_bytes, kind, (cudaStream_t)stream));
  }
  return CHAM_OK;
}

int cham_pool_fill_async(cham_pool* pool, int slot, const void* host_src, size_t bytes, void* stream,
                         void* done) {
  int rc = fill_common(pool, slot, host_src, bytes, stream, cudaMemcpyHostToDevice);
  if (rc) return rc;
  if (done) CHAM_CUDA(cudaEventRecord((cudaEvent_t)done, (cudaStream_t)stream));
  return CHAM_OK;
}

int cham_pool_fill_from_device(cham_pool* pool, int slot, const void* dev_src, size_t bytes, void* stream) {
  return fill_common(pool, slot, dev_src, bytes, stream, cudaMemcpyDeviceToDevice);
}

int cham_pool_device_error(cham_pool* pool, int* device_error, int clear, void* stream) {
  if (!pool || !device_error) return fail(CHAM_ERR_INVALID, "cham_pool_device_error: null argument");
  int v = 0;
  CHAM_CUDA(cudaMemcpyAsync(&v, pool->d_ctr + 2, sizeof(int), cudaMemcpyDeviceToHost, (cudaStream_t)stream));
  CHAM_CUDA(cudaStreamSynchronize((cudaStream_t)stream));
  if (clear && v) {
    CHAM_CUDA(cudaMemsetAsync(pool->d_ctr + 2, 0, sizeof(int), (cudaStream_t)stream));
    CHAM_CUDA(cudaStreamSynchronize((cudaStream_t)stream));
  }
  *device_error = v;
  return CHAM_OK;
}

int cham_debug_set_trace(cham_pool* pool, void* dev_buf, int items_per_cta) {
  if (!pool || (dev_buf && items_per_cta <= 0)) return fail(CHAM_ERR_INVALID, "cham_debug_set_trace: bad argument");
  pool->d_trace = static_cast<unsigned long long*>(dev_buf);
  pool->trace_cap = dev_buf ? items_per_cta : 0;
  return CHAM_OK;
}

int cham_pool_copy_out(const cham_pool* pool, size_t offset, size_t bytes, void* dst, void* stream) {
  if (!pool || !dst) return fail(CHAM_ERR_INVALID, "cham_pool_copy_out: null argument");
  if (offset + bytes > (size_t)pool->n_pages * pool->page_bytes)
    return fail(CHAM_ERR_INVALID, "cham_pool_copy_out: range outside the pool");
  CHAM_CUDA(cudaMemcpyAsync(dst, pool->base + offset, bytes, cudaMemcpyDefault, (cudaStream_t)stream));
  CHAM_CUDA(cudaStreamSynchronize((cudaStream_t)stream));
  return CHAM_OK;
}

int cham_pack_adapter_host_geom(int n_layers, int n_proj, const int* h_in, const int* h_out, int dtype, int rank,
                                const void* a, const void* b, void* out) {
  if (!h_in || !h_out || !a || !b || !out || n_layers <= 0 || n_proj <= 0)
    return fail(CHAM_ERR_INVALID, "cham_pack_adapter_host_geom: bad argument");
  if (dtype != CHAM_F32 && dtype != CHAM_BF16) return fail(CHAM_ERR_INVALID, "cham_pack_adapter_host_geom: dtype");
  if (rank <= 0 || rank > kMaxRank) return fail(CHAM_ERR_LIMIT, "cham_pack_adapter_host_geom: bad rank");
  const int es = dtype == CHAM_F32 ? 4 : 2;
  const int atom_e = kRowBytes / es;
  size_t page_bytes = 0;
  for (int p = 0; p < n_proj; ++p) {
    if (h_in[p] <= 0 || h_out[p] <= 0 || h_in[p] % atom_e || h_out[p] % atom_e)
      return fail(CHAM_ERR_INVALID, "cham_pack_adapter_host_geom: h_in/h_out must be multiples of the atom width");
    page_bytes += (size_t)kRowsPerPage * (h_in[p] + h_out[p]) * es;
  }
  page_bytes *= n_layers;
  const int np = (rank + kRowsPerPage - 1) / kRowsPerPage;
  const char* ca = static_cast<const char*>(a);
  const char* cb = static_cast<const char*>(b);
  char* co = static_cast<char*>(out);
  std::memset(co, 0, (size_t)np * page_bytes);
  size_t off = 0, asrc = 0, bsrc = 0;
  for (int l = 0; l < n_layers; ++l)
    for (int p = 0; p < n_proj; ++p) {
      const int hin = h_in[p], hout = h_out[p];
      const size_t aoff = off, boff = off + (size_t)kRowsPerPage * hin * es;
      off = boff + (size_t)kRowsPerPage * hout * es;
      for (int r = 0; r < rank; ++r) {
        const int page = r / kRowsPerPage, j = r % kRowsPerPage;
        char* pg = co + (size_t)page * page_bytes;
        for (int k = 0; k < hin; ++k)
          std::memcpy(pg + aoff + (size_t)(k / atom_e) * kAtomBytes + atom_offset(j, k % atom_e, es),
                      ca + asrc + ((size_t)k * rank + r) * es, es);
        for (int n = 0; n < hout; ++n)
          std::memcpy(pg + boff + (size_t)(n / atom_e) * kAtomBytes + atom_offset(j, n % atom_e, es),
                      cb + bsrc + ((size_t)r * hout + n) * es, es);
      }
      asrc += (size_t)hin * rank * es;
      bsrc += (size_t)rank * hout * es;
    }
  return CHAM_OK;
}

int cham_pack_adapter_host(const cham_pool* pool, int rank, const void* a, const void* b, void* out) {
  if (!pool) return fail(CHAM_ERR_INVALID, "cham_pack_adapter_host: null pool");
  return cham_pack_adapter_host_geom(pool->n_layers, pool->n_proj, pool->h_in.data(), pool->h_out.data(),
                                     pool->dtype, rank, a, b, out);
}

int cham_pack_adapter_device(const cham_pool* pool, int rank, const void* a, const void* b, void* out,
                             void* stream) {
  if (!pool || !a || !b || !out) return fail(CHAM_ERR_INVALID, "cham_pack_adapter_device: null argument");
  if (rank <= 0 || rank > kMaxRank) return fail(CHAM_ERR_LIMIT, "cham_pack_adapter_device: bad rank");
  const int n_lp = pool->n_layers * pool->n_proj;
  std::vector<int> hin(n_lp), hout(n_lp);
  std::vector<long long> aoff(n_lp), boff(n_lp), asrc(n_lp), bsrc(n_lp);
  long long as = 0, bs = 0;
  for (int l = 0; l < pool->n_layers; ++l)
    for (int p = 0; p < pool->n_proj; ++p) {
      const int lp = l * pool->n_proj + p;
      hin[lp] = pool->h_in[p];
      hout[lp] = pool->h_out[p];
      aoff[lp] = (long long)pool->a_off[lp];
      boff[lp] = (long long)pool->b_off[lp];
      asrc[lp] = as;
      bsrc[lp] = bs;
      as += (long long)hin[lp] * rank * pool->es;
      bs += (long long)rank * hout[lp] * pool->es;
    }
  // small metadata block in device memory (freed after the stream completes the kernel)
  const size_t meta_bytes = n_lp * (2 * sizeof(int) + 4 * sizeof(long long));
  char* meta = nullptr;
  CHAM_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&meta), meta_bytes, (cudaStream_t)stream));
  std::vector<char> h(meta_bytes);
  size_t o = 0;
  auto put = [&](const void* src, size_t n) { std::memcpy(h.data() + o, src, n); o += n; };
  put(aoff.data(), n_lp * 8); put(boff.data(), n_lp * 8); put(asrc.data(), n_lp * 8);
  put(bsrc.data(), n_lp * 8); put(hin.data(), n_lp * 4); put(hout.data(), n_lp * 4);
  CHAM_CUDA(cudaMemcpyAsync(meta, h.data(), meta_bytes, cudaMemcpyHostToDevice, (cudaStream_t)stream));
  const long long* d_aoff = reinterpret_cast<const long long*>(meta);
  const long long* d_boff = d_aoff + n_lp;
  const long long* d_asrc = d_boff + n_lp;
  const long long* d_bsrc = d_asrc + n_lp;
  const int* d_hin = reinterpret_cast<const int*>(d_bsrc + n_lp);
  const int* d_hout = d_hin + n_lp;
  const int np = (rank + kRowsPerPage - 1) / kRowsPerPage;
  const long long n_chunks = (long long)pool->page_bytes / 16;
  dim3 grid((unsigned)((n_chunks + 255) / 256), np);
  if (pool->es == 4)
    pack_kernel<4><<<grid, 256, 0, (cudaStream_t)stream>>>(
        (const char*)a, (const char*)b, (char*)out, rank, n_lp, d_hin, d_hout, d_aoff, d_boff, d_asrc,
        d_bsrc, (long long)pool->page_bytes);
  else
    pack_kernel<2><<<grid, 256, 0, (cudaStream_t)stream>>>(
        (const char*)a, (const char*)b, (char*)out, rank, n_lp, d_hin, d_hout, d_aoff, d_boff, d_asrc,
        d_bsrc, (long long)pool->page_bytes);
  CHAM_CUDA(cudaGetLastError());
  CHAM_CUDA(cudaFreeAsync(meta, (cudaStream_t)stream));
  return CHAM_OK;
}

}  // extern "C"
