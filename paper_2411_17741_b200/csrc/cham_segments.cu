// cham_segments.cu — K4: device-side segment-table builder.
//
// Replaces the per-request Python loop of CostModel.step_duration (engine.py:64-76), which
// walks the step's batch (prefills with input_tokens each, decoders with one token each,
// engine.py:443-451) one request at a time.  Here one CTA of 1024 threads builds the
// stable group-by-slot of up to 4096 requests with a block radix sort (CUB, stable) over
// only the bits the batch's largest slot needs (7 bits = 2 digit passes for 100 adapters,
// instead of 8 passes over slot << 12 | request), block scans for token offsets and segment
// ids, and writes perm / seg_off / seg_slot / seg_rank.  Slots must be < 2^20.  Canonical form (bit-exact with oracle/segments_ref.py): segments in ascending slot order,
// requests inside a segment in batch order, tokens of a request contiguous.
#include <cub/block/block_radix_sort.cuh>
#include <cub/block/block_scan.cuh>

#include "cham_pool.h"

namespace cham {
namespace seg {

constexpr int kThreads = 1024;
constexpr int kItems = kMaxRequests / kThreads;  // 4
static_assert(kItems * kThreads == kMaxRequests, "request capacity");

__global__ void __launch_bounds__(kThreads, 1)
build_segments_kernel(const int* __restrict__ req_slot, const int* __restrict__ req_rank,
                      const int* __restrict__ req_ntok, int n_req, int* __restrict__ perm,
                      int* __restrict__ seg_off, int* __restrict__ seg_slot,
                      int* __restrict__ seg_rank, int* __restrict__ n_seg) {
  using Sort = cub::BlockRadixSort<unsigned, kThreads, kItems, int>;
  using Scan = cub::BlockScan<int, kThreads>;
  __shared__ union {
    typename Sort::TempStorage sort;
    typename Scan::TempStorage scan;
  } tmp;
  __shared__ unsigned last_key[kThreads];
  __shared__ int total_tokens, total_segs;
  __shared__ unsigned s_max_slot;

  const int tid = threadIdx.x;
  // 1) token offsets in batch order (blocked arrangement: thread t owns requests 4t..4t+3)
  int ntok[kItems];
#pragma unroll
  for (int i = 0; i < kItems; ++i) {
    const int r = tid * kItems + i;
    ntok[i] = r < n_req ? max(req_ntok[r], 0) : 0;
  }
  int off[kItems];
  if (tid == 0) s_max_slot = 0;
  Scan(tmp.scan).ExclusiveSum(ntok, off);
  int slot_in[kItems];
  unsigned my_max = 0;
#pragma unroll
  for (int i = 0; i < kItems; ++i) {
    const int r = tid * kItems + i;
    const int s = r < n_req ? req_slot[r] : -1;
    slot_in[i] = (s >= 0 && s < (1 << 20)) ? s : -1;
    if (slot_in[i] >= 0) my_max = max(my_max, static_cast<unsigned>(slot_in[i]) + 1);
  }
  __syncthreads();
  if (my_max) atomicMax(&s_max_slot, my_max);
  __syncthreads();

  // 2) stable sort of key = slot (batch order kept inside a slot: CUB's radix sort is
  //    stable and the input is in batch order); the value is the request index.  No adapter
  //    -> key = largest slot + 1, sorts last.  Only the bits of that sentinel are sorted.
  //    The value packs the request's first token (< 2^20: a step holds at most 65535 tokens,
  //    kMaxPoolTokens) above its 12-bit index.
  const unsigned sentinel = s_max_slot;  // largest valid slot + 1
  const int end_bit = max(1, 32 - __clz(sentinel));
  unsigned key[kItems];
  int val[kItems];
#pragma unroll
  for (int i = 0; i < kItems; ++i) {
    key[i] = slot_in[i] >= 0 ? static_cast<unsigned>(slot_in[i]) : sentinel;
    val[i] = (off[i] << 12) | (tid * kItems + i);
  }
  Sort(tmp.sort).Sort(key, val, 0, end_bit);
  __syncthreads();

  // 3) token positions in grouped order and segment ids
  int gtok[kItems], flag[kItems];
  last_key[tid] = key[kItems - 1];
  __syncthreads();
  unsigned prev = tid > 0 ? last_key[tid - 1] : 0xfffffffeu;
#pragma unroll
  for (int i = 0; i < kItems; ++i) {
    const bool valid = key[i] != sentinel;
    gtok[i] = valid ? max(req_ntok[val[i] & 4095], 0) : 0;
    flag[i] = valid && key[i] != prev ? 1 : 0;
    prev = key[i];
  }
  int gpos[kItems], segid[kItems];
  int tot_tok, tot_seg;
  Scan(tmp.scan).ExclusiveSum(gtok, gpos, tot_tok);
  __syncthreads();
  Scan(tmp.scan).ExclusiveSum(flag, segid, tot_seg);
  if (tid == 0) {
    total_tokens = tot_tok;
    total_segs = tot_seg;
  }
#pragma unroll
  for (int i = 0; i < kItems; ++i) {
    if (key[i] == sentinel) continue;
    const int r = val[i] & 4095;
    if (flag[i]) {
      seg_off[segid[i]] = gpos[i];
      seg_slot[segid[i]] = static_cast<int>(key[i]);
      seg_rank[segid[i]] = req_rank[r];
    }
    const int base = static_cast<unsigned>(val[i]) >> 12;
    for (int k = 0; k < gtok[i]; ++k) perm[gpos[i] + k] = base + k;
  }
  __syncthreads();
  if (tid == 0) {
    seg_off[total_segs] = total_tokens;
    *n_seg = total_segs;
  }
}

}  // namespace seg
}  // namespace cham

using namespace cham;

extern "C" int cham_build_segments(const int* req_slot, const int* req_rank, const int* req_ntok,
                                   int n_req, int* perm, int* seg_off, int* seg_slot, int* seg_rank,
                                   int* n_seg, void* stream) {
  if (n_req < 0 || n_req > kMaxRequests)
    return fail(CHAM_ERR_LIMIT, "cham_build_segments: n_req must be in [0, max_requests]");
  if ((n_req > 0 && (!req_slot || !req_rank || !req_ntok)) || !seg_off || !seg_slot || !seg_rank ||
      !n_seg || !perm)
    return fail(CHAM_ERR_INVALID, "cham_build_segments: null argument");
  seg::build_segments_kernel<<<1, seg::kThreads, 0, (cudaStream_t)stream>>>(
      req_slot, req_rank, req_ntok, n_req, perm, seg_off, seg_slot, seg_rank, n_seg);
  CHAM_CUDA(cudaGetLastError());
  return CHAM_OK;
}
