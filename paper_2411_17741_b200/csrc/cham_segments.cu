// cham_segments.cu — K4: device-side segment-table builder.
//
// Replaces the per-request Python loop of CostModel.step_duration (engine.py:64-76), which
// walks the step's batch (prefills with input_tokens each, decoders with one token each,
// engine.py:443-451) one request at a time.  Here one CTA of 1024 threads builds the
// stable group-by-slot of up to 4096 requests with a block radix sort (CUB, stable), block
// scans for token offsets and segment ids, and writes perm / seg_off / seg_slot / seg_rank.
// Slots must be < 2^20 - 1.  Canonical form (bit-exact with oracle/segments_ref.py): segments in ascending slot order,
// requests inside a segment in batch order, tokens of a request contiguous.
#include <cub/block/block_radix_sort.cuh>
#include <cub/block/block_reduce.cuh>
#include <cub/block/block_scan.cuh>

#include "cham_pool.h"

namespace cham {
namespace seg {

constexpr int kItems = 4;  // requests per thread
// Two block sizes: 256 threads cover batches of <= 1024 requests (every decode step of the
// benchmarks), 1024 threads the full kMaxRequests.  The sort only runs over the key bits in
// use: 12 request-index bits plus the width of the largest slot of the batch.
template <int kThreads>
__global__ void __launch_bounds__(kThreads, 1)
build_segments_kernel(const int* __restrict__ req_slot, const int* __restrict__ req_rank,
                      const int* __restrict__ req_ntok, int n_req, int* __restrict__ perm,
                      int* __restrict__ seg_off, int* __restrict__ seg_slot,
                      int* __restrict__ seg_rank, int* __restrict__ n_seg) {
  using Sort = cub::BlockRadixSort<unsigned, kThreads, kItems, int>;
  using Scan = cub::BlockScan<int, kThreads>;
  using Reduce = cub::BlockReduce<int, kThreads>;
  __shared__ union {
    typename Sort::TempStorage sort;
    typename Scan::TempStorage scan;
    typename Reduce::TempStorage reduce;
  } tmp;
  __shared__ unsigned last_key[kThreads];
  __shared__ int total_tokens, total_segs, slot_max_all;

  const int tid = threadIdx.x;
  // 1) token offsets in batch order (blocked arrangement: thread t owns requests 4t..4t+3)
  int ntok[kItems];
#pragma unroll
  for (int i = 0; i < kItems; ++i) {
    const int r = tid * kItems + i;
    ntok[i] = r < n_req ? max(req_ntok[r], 0) : 0;
  }
  int off[kItems];
  Scan(tmp.scan).ExclusiveSum(ntok, off);
  __syncthreads();

  // 2) sort of key = slot << 12 | request index (unique keys, so batch order is kept inside
  //    a slot); the value carries the request's first token.  No adapter -> slot max + 1, so
  //    it sorts last inside the sorted bits (marked 0xffffffff afterwards).
  int smax = -1;
#pragma unroll
  for (int i = 0; i < kItems; ++i) {
    const int r = tid * kItems + i;
    const int s = r < n_req ? req_slot[r] : -1;
    if (s >= 0 && s < (1 << 20) - 1) smax = max(smax, s);
  }
  smax = Reduce(tmp.reduce).Reduce(smax, cub::Max());  // valid in thread 0
  if (tid == 0) slot_max_all = smax;
  __syncthreads();
  const unsigned none = static_cast<unsigned>(slot_max_all + 1);
  const int key_bits = 12 + (32 - __clz(static_cast<int>(none)));
  unsigned key[kItems];
  int val[kItems];
#pragma unroll
  for (int i = 0; i < kItems; ++i) {
    const int r = tid * kItems + i;
    const int s = r < n_req ? req_slot[r] : -1;
    key[i] = (((s >= 0 && s < (1 << 20) - 1) ? static_cast<unsigned>(s) : none) << 12) | static_cast<unsigned>(r);
    val[i] = off[i];
  }
  Sort(tmp.sort).Sort(key, val, 0, key_bits);
  __syncthreads();
#pragma unroll
  for (int i = 0; i < kItems; ++i)
    if ((key[i] >> 12) == none) key[i] = 0xffffffffu;

  // 3) token positions in grouped order and segment ids
  int gtok[kItems], flag[kItems];
  last_key[tid] = key[kItems - 1];
  __syncthreads();
  unsigned prev = tid > 0 ? (last_key[tid - 1] >> 12) : 0xfffffffeu;
#pragma unroll
  for (int i = 0; i < kItems; ++i) {
    const bool valid = key[i] != 0xffffffffu;
    gtok[i] = valid ? max(req_ntok[key[i] & 4095], 0) : 0;
    flag[i] = valid && (key[i] >> 12) != prev ? 1 : 0;
    prev = key[i] >> 12;
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
    if (key[i] == 0xffffffffu) continue;
    const int r = key[i] & 4095;
    if (flag[i]) {
      seg_off[segid[i]] = gpos[i];
      seg_slot[segid[i]] = static_cast<int>(key[i] >> 12);
      seg_rank[segid[i]] = req_rank[r];
    }
    const int base = val[i];
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
  if (n_req <= 256 * seg::kItems)
    seg::build_segments_kernel<256><<<1, 256, 0, (cudaStream_t)stream>>>(req_slot, req_rank, req_ntok, n_req, perm,
                                                                         seg_off, seg_slot, seg_rank, n_seg);
  else
    seg::build_segments_kernel<1024><<<1, 1024, 0, (cudaStream_t)stream>>>(req_slot, req_rank, req_ntok, n_req, perm,
                                                                           seg_off, seg_slot, seg_rank, n_seg);
  CHAM_CUDA(cudaGetLastError());
  return CHAM_OK;
}
