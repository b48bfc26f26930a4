// cham_pool.h — internal definition of the paged adapter pool (not part of the C ABI).
#pragma once

#include <vector>

#include "cham_common.cuh"

struct cham_pool {
  int device = 0;
  int n_pages = 0;
  int n_layers = 0;
  int n_proj = 0;
  int dtype = CHAM_BF16;
  int es = 2;  // element bytes
  int n_slots = 0;
  int max_tokens = 0;
  int sm_count = 148;
  std::vector<int> h_in, h_out;
  std::vector<size_t> a_off, b_off;  // byte offset of (l*n_proj+p) A / B block inside a page
  size_t page_bytes = 0;
  char* base = nullptr;                // n_pages * page_bytes, device
  int* d_slot_pages = nullptr;         // [n_slots][kMaxPagesPerSlot]
  int* d_slot_rank = nullptr;          // [n_slots]
  std::vector<int> slot_rank;          // host mirror
  std::vector<int> slot_pages;         // host mirror [n_slots][kMaxPagesPerSlot]
  // decode / shrink / expand workspace (one launch at a time per pool)
  int* d_ctr = nullptr;                // [2] error; [16..31] / [32..47]: per-parity launch counters;
                                       // [64..): 2 x [kMaxJobs][max_tokens] per-tile v-ready counters
  float* d_vws = nullptr;              // 2 x [kMaxJobs][max_tokens][vws_kc][kMaxRank] (ping-pong)
  int vws_kc = 1;
  unsigned long long apply_count = 0;  // selects the v / counter ping-pong sets
  void* d_plan = nullptr;              // scratch plan for calls without a step-level plan
  unsigned long long* d_trace = nullptr;  // debug timeline buffer (caller-owned)
  int trace_cap = 0;
  // tcgen05 prefill routing (cham_prefill.cu): segments with >= prefill_min_tokens tokens and
  // rank <= kPrefillMaxRank run the tensor-core kernels; the decode plan skips them.
  bool prefill_ok = false;             // bf16 pool, every h_in / h_out a multiple of 128
  int prefill_min_tokens = 0;          // 0 = tcgen05 path disabled
  int route_min_seg = 0;               // host hints about the next steps' segment lengths
  int route_max_seg = 1 << 30;
  char* d_pvimg = nullptr;             // prefill V images [kMaxJobs][kPrefillMaxTiles][32 KiB] (bf16, one per tile)
  float* d_ppart = nullptr;            // prefill split-K fp32 partials [kMaxJobs][kPrefillMaxTiles][64 KiB]
  int* d_iota = nullptr;               // identity token rows [max_tokens] (prefill calls without perm)
  int* d_pctr = nullptr;               // prefill counters: 2 parity sets + tile V flags
  int prefill_epoch = 0;               // prefill launches so far (tile flags, counter parity)
  float* d_split = nullptr;            // decode page-half partials [kMaxJobs][kSplitCap][split_ncc][4][2048 B cols]
  int* d_split_ctr = nullptr;          // 2 parity x [kMaxJobs][kSplitCap][split_ncc]
  int split_ncc = 1;                   // 2048-byte column chunks of the widest h_out
  // Next-apply hint (cham_pool_set_next_apply): the (layer, projections) the caller launches
  // right after the next apply on the same plan.  That apply's CTAs, once out of units, pull
  // the first l2_prefetch_bytes of the hinted apply's A blocks into L2 (one-shot).
  int next_n = 0;
  size_t next_a_off[cham::kMaxJobs] = {};
  int next_a_bytes = 0;                // bytes of one page's A block of the hinted projections
  long long l2_prefetch_bytes = 0;     // budget per hinted apply (0 = off)
};

namespace cham {
constexpr int kPrefillMinTokens = 64;  // default routing threshold (segment tokens)
constexpr int kPrefillMaxRank = 128;   // largest rank on the tcgen05 path (TMEM / smem budget)
constexpr int kPrefillMaxSplit = 8;    // shrink split-K factor bound (workspace sizing)
constexpr int kPrefillMaxTiles = 256;  // 128-row prefill tiles per apply (workspace sizing)
constexpr int kPrefillCtrSet = 4 + kPrefillMaxTiles + kPrefillMaxTiles * cham::kMaxJobs;  // one parity set:
// dispatch, done, spare x2, tile V counters [tiles], split-K arrival counters [tiles][groups]
constexpr size_t kPrefillPart = 131072;                // fp32 split-K partial bytes per (job, tile): 2 K ranges at 128 rows x rank 128
constexpr size_t kPrefillVImg = 32768;                // V image bytes per (job, tile)
inline size_t prefill_ctr_ints() { return 2 * kPrefillCtrSet + kPrefillMaxTiles; }

constexpr int kMaxPoolPages = 65535;   // plan page ids are uint16 (cham_decode.cu Plan::pages)
constexpr int kMaxPoolTokens = 65535;  // plan token rows are uint16 (Plan::perm)

constexpr int kSplitCap = 128;         // decode expand tiles split into page halves per apply
constexpr int kSplitTG = 4;            // tokens per decode tile (decode::TG)
constexpr int kSplitNcb = 2048;        // bytes of one B row per decode expand unit

// d_ctr layout: launch counters, then the per-parity tile-ready counters of the decode kernel
constexpr int kTileCtrBase = 64;
inline size_t ctr_ints(int max_tokens) { return kTileCtrBase + 2 * (size_t)kMaxJobs * max_tokens; }

// Threshold the plan and the launches use for this pool: segments with at least this many
// tokens (and rank <= kPrefillMaxRank) go to the tcgen05 kernels.  INT_MAX = none.
inline int prefill_route_thr(const cham_pool* pool) {
  if (!pool->prefill_ok || pool->prefill_min_tokens <= 0) return 1 << 30;
  if (pool->route_max_seg < pool->prefill_min_tokens) return 1 << 30;
  return pool->prefill_min_tokens;
}
__host__ __device__ inline bool is_prefill_segment(int n_tok, int rank, int thr) {
  return n_tok >= thr && rank > 0 && rank <= kPrefillMaxRank;
}

// Byte offset of element (row j, element e) inside a 1 KiB swizzled atom.
__host__ __device__ inline uint32_t atom_offset(int j, int e, int es) {
  const int byte = e * es;
  const int chunk = byte >> 4;
  return static_cast<uint32_t>(j * kRowBytes + (((chunk ^ j) & 7) << 4) + (byte & 15));
}
}  // namespace cham
