// cham_decode.cu — segmented shrink (h_in -> r) and expand (r -> h_out, accumulated into y)
// for decode-sized segments: ONE persistent, warp-specialised kernel per lora_apply; an
// expand stage waits only for the shrink units of its own pages (no grid barrier);
// consecutive applies overlap through programmatic dependent launch (PDL).
//
// Reference seam: CostModel.step_duration's LoRA term (engine.py:67-77) models
//   adapter_units = sum_decoders rank + sum_prefills rank * input_tokens
// as 0.155 us per rank*token (model.py:172); these kernels perform that work for real:
// for every token t of segment s, y[t] += (x[t] . A_slot(s)) . B_slot(s).
//
// Design:
//  * A tile is <= 4 tokens of one segment.  Work is dispatched in *units* that loop over
//    several pipeline stages (a K-loop), so every TMA bulk copy is large:
//      K1 unit = (job, tile, page):  nkc stages, each = 32 KiB of A (8 rank rows x 2048
//               bf16 of h_in) + the tile's x rows for that k-chunk; the 8 x T partial sums
//               stay in registers across the stages, so v is written once, final.
//      K2 unit = (job, tile, 1024-column chunk): ceil(np/2) stages, each = two pages x
//               16 KiB of B with those pages' v slices; the y rows ride on the last stage
//               (tiles of <= 4 pages: 2048-column units, one page per stage).
//  * Units come from ONE global counter, all shrink units then all expand units, each in
//    LPT order (adapters of larger page count first); two units are fetched ahead of the
//    one being issued and one more claim is in flight.
//  * Two producer warps (producer 0 claims and forwards the unit ids, producer 1 issues
//    every other stage; plan in shared memory), 8 consumer warps (packed FFMA2, fp32
//    accumulate), one publisher warp: a finished shrink unit's v rows are released with one
//    `red.release.gpu.or` of its page bit into the tile's mask; an expand stage acquires the
//    bits of its pages before its v copy.  Weights are issued before griddepcontrol.wait,
//    activations after it.
//  * Counters and the fp32 v workspace ping-pong by apply parity.  Producer 0 of every CTA
//    re-arms the previous apply's counter slice right after griddepcontrol.wait and only then
//    signals launch_dependents, so apply n+1 starts with zeroed counters and no CTA ends with
//    a last-CTA reset; every CTA executes griddepcontrol.wait, so apply n completes after
//    apply n-1 and the v buffer of apply n-2 is free when apply n writes it.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>

#include "cham_pool.h"

namespace cham {
int encode_f32_map(CUtensorMap* m, const void* base, int rows, int cols, int pitch, int box_cols, int box_rows);
int prefill_launch(cham_pool* pool, int layer, int n_jobs, const int* projs, const void* const* xs,
                   void* const* ys, int n_tokens, const int* perm, const int* seg_off, const int* seg_slot,
                   const int* seg_rank, int n_seg, const int* n_seg_dev, void* stream, int mode, float* v_out,
                   const float* v_in, int v_stride);
namespace decode {

#ifndef CHAM_EXP_NOCOMPUTE
#define CHAM_EXP_NOCOMPUTE 0  // experiment builds only: consumers skip the math (data-movement ceiling)
#endif
constexpr bool kNoCompute = CHAM_EXP_NOCOMPUTE != 0;
#ifndef CHAM_MMA_SHRINK
#define CHAM_MMA_SHRINK 0  // 1: bf16 shrink on mma.sync (A/B on C2: 99.4k vs 114.9k tok/s FFMA2)
#endif
constexpr bool kMmaShrink = CHAM_MMA_SHRINK != 0;
#ifndef CHAM_MMA_EXPAND
#define CHAM_MMA_EXPAND 0  // 1: bf16 expand on mma.sync (A/B on C2: 104.0k vs 114.9k tok/s FFMA2)
#endif
constexpr bool kMmaExpand = CHAM_MMA_EXPAND != 0;

constexpr int TG = 4;                        // tokens per tile
#ifndef CHAM_NSTAGE
#define CHAM_NSTAGE 4
#endif
#ifndef CHAM_ACHUNK
#define CHAM_ACHUNK 32768
#endif
#ifndef CHAM_EXPG
#define CHAM_EXPG 2
#endif
constexpr int NSTAGE = CHAM_NSTAGE;          // ring depth
constexpr int A_CHUNK = CHAM_ACHUNK;         // K1: adapter bytes per stage (8 rows x A_CHUNK/8)
constexpr int X_ROW = A_CHUNK / kRowsPerPage;  // K1: x bytes per token per stage (k-chunk)
constexpr int EX_PAGES = CHAM_EXPG;          // K2: adapter pages per stage (1 or 2)
static_assert(X_ROW <= kActRowBytes && (EX_PAGES == 1 || EX_PAGES == 2), "stage geometry");
constexpr int X_PITCH = X_ROW + 16;         // staged x rows: +16 B so ldmatrix rows hit distinct banks
constexpr int K1_STAGE = A_CHUNK + TG * X_PITCH;
// K2 geometry tiers, chosen by the adapter's page count np so that every expand unit is at
// most two 32 KiB stages (uniform units keep the dynamic dispatch balanced to the end —
// with unit sizes from 16 to 256 KiB, large units claimed late by the look-ahead dispatch
// made an ~8 us tail):
//   tier 0 (np <= 4):  units of 2048 B per B row, 2 pages per stage (16 KiB page copies)
//   tier 1 (np <= 8):  1024 B per B row, 4 pages per stage (8 KiB copies)
//   tier 2 (np <= 16): 512 B per B row, 8 pages per stage (4 KiB copies)
constexpr int NTIER = 3;
constexpr int NCB_SMALL = 2048;              // bytes of one B row per unit, tier 0
__host__ __device__ constexpr int tier_ncb(int t) { return NCB_SMALL >> t; }
__host__ __device__ constexpr int tier_pitch(int t) {  // page pitch in a stage (+ bank skew)
  return (NCB_SMALL >> t) * kRowsPerPage + (64 >> t);
}
#ifndef CHAM_TIERS
#define CHAM_TIERS 0  // 1: page-count tiers (A/B on C2: 98.1k vs 110.3k tok/s without)
#endif
__host__ __device__ constexpr int tier_of_np(int np) {  // CHAM_TIERS: highest tier used
  return CHAM_TIERS == 0 ? 0 : np <= 4 ? 0 : (np <= 8 || CHAM_TIERS == 1) ? 1 : 2;
}
#ifndef CHAM_EX_DEPTH
#define CHAM_EX_DEPTH 1  // expand dispatch look-ahead (A/B on C2: 1 -> 114.2k, 2 -> 110.2k tok/s)
#endif
#ifndef CHAM_SH_DEPTH
#define CHAM_SH_DEPTH 1  // shrink dispatch look-ahead (A/B on C2: 1 -> 118.5k, 2 -> 117.2k, 3 -> 114.0k)
#endif
constexpr int K2_B = (CHAM_TIERS ? 2 : EX_PAGES) * tier_pitch(0);
static_assert(CHAM_TIERS == 0 || (4 * tier_pitch(1) <= K2_B && 8 * tier_pitch(2) <= K2_B), "stage layout");
constexpr int K2_Y = K2_B;
constexpr int K2_V = K2_Y + TG * NCB_SMALL;
constexpr int K2_STAGE = K2_V + 8 * TG * kRowsPerPage * 4;  // v slice [page][token][8 rows]
// Wide expand geometry for small-rank tiles (np <= CHAM_WIDE_NP pages): units of 2048 B per
// B row (2048 bf16 columns), ONE page per stage, one consumer thread per 16-byte column chunk
// holding all 8 rank rows — no sibling combine, no divergent y update, and twice the bytes
// per unit of the tier-0 geometry, whose 1-page stages were consumer- and issue-bound
// (0.9 us per 25 KB stage on C2).  Stage layout: B [8 rows][4096 B] | y [TG][4096 B] | v [TG][8].
#ifndef CHAM_WIDE_NP
#define CHAM_WIDE_NP 4  // A/B (tok/s, page-ready tiles, release publication): C2 4 -> 131.2k, 8 -> 132.0k, 16 -> 115.3k; C5 4 -> 24.25k, 8 -> 23.5k
#endif
constexpr int kWideNp = CHAM_WIDE_NP;
constexpr int TIER_W = 3;
constexpr int NCB_WIDE = 4096;
constexpr int K2W_Y = kRowsPerPage * NCB_WIDE;
constexpr int K2W_V = K2W_Y + TG * NCB_WIDE;
constexpr int PQ = 16;             // publisher ring depth (tile counters to release)
constexpr int GROUP_WARPS = 8;
constexpr int GROUP_THREADS = GROUP_WARPS * 32;
constexpr int NTHREADS = 32 + GROUP_THREADS;      // plan kernel; apply kernel adds the publisher warp
// Producer warps of the apply kernel.  With 2, producer pid issues the ring stages with
// seq % 2 == pid (both walk the same unit stream: producer 0 claims the units and hands the
// ids to producer 1 through a shared-memory queue), so two stages' issue latencies overlap.
#ifndef CHAM_NPROD
#define CHAM_NPROD 2
#endif
constexpr int NPROD = CHAM_NPROD;
static_assert(NPROD == 1 || NPROD == 2, "one or two producer warps");
constexpr int APPLY_THREADS = NTHREADS + 32 * NPROD;  // consumers, producer 0, publisher, producer 1
constexpr int UQN = 8;  // unit-id queue depth, producer 0 -> producer 1
static_assert(GROUP_THREADS == 2 * (tier_ncb(0) / 16) && GROUP_THREADS == 4 * (tier_ncb(1) / 16) &&
                  GROUP_THREADS == 8 * (tier_ncb(2) / 16),
              "K2 maps 2 << tier threads per 16-byte column chunk");
constexpr int PLAN_SEGS = 512;
constexpr int PLAN_PAGES = 2048;
constexpr int PLAN_TOKENS = 2048;
static_assert(PLAN_SEGS == kMaxSegments, "limits");

enum Mode { MODE_FUSED = 0, MODE_SHRINK = 1, MODE_EXPAND = 2 };
enum Kind { KIND_END = 0, KIND_SHRINK = 1, KIND_EXPAND = 2, KIND_PHASE = 3 };

struct Job {
  const char* x;
  char* y;
  long long a_off;
  long long b_off;
};

struct Params {
  CUtensorMap vmap;   // MODE_EXPAND: v_in as [positions][v_stride] fp32, boxes of 8 ranks x TG tokens
  const char* base;
  long long page_bytes;
  const int* slot_pages;
  int h_in, h_out;
  int n_jobs;
  Job jobs[kMaxJobs];
  const int* perm;
  const int* seg_off;
  const int* seg_slot;
  const int* seg_rank;
  int n_seg;
  const int* n_seg_dev;
  int* ctr;        // [0] next shrink unit, [1] finished CTAs, [4] next expand unit
  // CHAM_ZERO_NEXT: the other parity's counter set (the previous apply's), re-armed by this
  // apply's producers right after griddepcontrol.wait, before launch_dependents
  int* zero_ctr;
  int* zero_tile;
  long long zero_tile_n;
  int* zero_split;
  long long zero_split_n;
  int* tile_ctr;   // MODE_FUSED: [job][expand tile] shrink units finished (v rows published)
  float* split_buf;   // page-half partials [job][split tile][col chunk][TG][cols of a chunk]
  int* split_ctr;     // [job][split tile][col chunk]: half 0 published its partial
  int split_ncc;      // column chunks per split tile (scratch geometry)
  int* err;
  float* vws;      // this apply's compact v buffer: [job][sum_s T_s * rpad_s]
  long long vws_job_stride;
  int max_tokens;
  float* v_out;       // MODE_SHRINK: v [positions][v_stride]
  const float* v_in;  // MODE_EXPAND: v [positions][v_stride]
  int v_stride;
  int v_cols;         // columns of one job's v slice: job j's v starts at column j * v_cols
  unsigned long long* trace;  // debug: [cta][seq][8] globaltimer stamps (null = off)
  int trace_cap;
  const void* plan;           // Plan header + unit descriptors (cham_build_plan)
  long long desc_cap;
  int prefill_thr;            // segments routed to the tcgen05 kernels (cham_prefill.cu) are skipped
  // next-apply L2 prefetch (cham_pool_set_next_apply): A blocks of the hinted apply's first
  // nx_items shrink units (its unit order: job-major, descriptor order), claimed through ctr[5]
  int nx_jobs;
  int nx_items;
  int nx_a_bytes;
  long long nx_a_off[kMaxJobs];
};

// Per-stage record written by the producer, read by the consumers after the full barrier.
struct Meta {
  int kind;
  int nst;    // stages in this unit (set on every stage)
  int job, seg, pos0, T, np;
  int g;      // K1: page index of the unit
  int kc;     // K1: k-chunk of this stage
  int pg0;    // K2: first page of this stage
  int npg;    // K2: pages in this stage (1 or 2)
  int col0, ncols;
  int vrow;   // K2: floats per staged v row
  int lpg;    // K2: log2(pages per stage) = log2(threads per column chunk)
  int ncb;    // K2: bytes of one B row in this unit
  int pitch;  // K2: page pitch in the stage
  int nq;     // K2: 16-byte column chunks in this unit
  int xm;     // K2: 0 plain, 1 page half 0 (write partial), 2 page half 1 (combine stage last)
  int sidx;   // K2: split scratch / flag slot
  int rows[TG];
};

struct alignas(16) Plan {
  int seg_off[PLAN_SEGS + 1];
  int seg_sr[PLAN_SEGS];      // (slot << 9) | rank
  int seg_pg[PLAN_SEGS + 1];  // prefix of pages -> pages[]
  int v_start[PLAN_SEGS + 1]; // prefix of nt_s * TG * rpad_s -> v, per tile [page][TG][8]
  int sh_start[PLAN_SEGS + 1];  // K1 units prefix (LPT order, indexed by segment)
  int ex_start[PLAN_SEGS + 1];  // K2 tiles prefix (LPT order); units = tiles x column chunks
  int order[PLAN_SEGS];         // K2 segment order: decreasing page count
  int bucket[kMaxPagesPerSlot + 2];
  uint16_t pages[PLAN_PAGES];
  uint16_t perm[PLAN_TOKENS];
  int scan[NTHREADS / 32][4];
  int totals[6];  // K1 units/job, K2 tiles/job, tokens, pages, v floats/job, segments with work
  int n_seg;
  int sh_lpt[PLAN_SEGS + 1];  // K1 unit prefix by LPT position
  int cls_pos[kMaxPagesPerSlot + 2];  // LPT positions where the page-count classes start
  int n_cls;
  int n_split;  // leading LPT expand tiles split into page halves (np > kSplitNp)
  int order_pos[PLAN_SEGS];  // segment -> position in the LPT order
  long long desc_cap;        // descriptor capacity (entries) after the header
};
static_assert(sizeof(Plan) % 16 == 0, "the plan is moved with one bulk copy");

// 32-byte work descriptors written by the plan kernel right after the Plan header:
// first one per shrink unit (job-independent, segment order), then one per expand tile
// (LPT order).  The producer fetches the descriptor of unit k+1 while it streams unit k.
struct alignas(16) UnitDesc {
  int seg;
  int pos0;
  int meta;     // tcount | np << 8 | g << 16   (g: shrink page index)
  int aux;      // shrink: pool page id of page g; expand: offset of the tile's v rows
  int rows[TG]; // token rows of the tile (perm)
};
static_assert(sizeof(UnitDesc) == 32, "descriptor layout");
__host__ __device__ inline long long plan_desc_capacity(int max_tokens) {
  // shrink units <= T * kMaxPagesPerSlot, expand tiles <= T
  return (long long)max_tokens * (kMaxPagesPerSlot + 1);
}

constexpr int MAX_BLOCKS = 2 * (kMaxPagesPerSlot + 1);
// Expand units of tiles whose adapter has more than kSplitNp pages are split into two page
// halves: half 0 leaves its fp32 partial sums in a scratch slot, half 1 adds them (plus its
// own and y) in a final combine stage.  Long units (8 stages at rank 128) otherwise leave the
// CTAs that took them running long after the rest finished.
#ifndef CHAM_SPLIT_NP
#define CHAM_SPLIT_NP 0  // 0 = off (A/B on C2: 8 -> 99.6k, off -> 113.3k tok/s on the same box)
#endif
constexpr int kSplitNp = CHAM_SPLIT_NP;
// Alternative for the large-rank tiles (np > 8): the tier-2 expand geometry (8 pages x 256
// columns per stage, 2-stage units, 16 column chunks per tile) instead of the page halves.
// 2: on (A/B on C2: 101.1k vs 114.6k tok/s off), 0: off.
#ifndef CHAM_BIG_TIER
#define CHAM_BIG_TIER 0
#endif
constexpr int kBigTier = CHAM_BIG_TIER;
static_assert(TG == kSplitTG && NCB_SMALL == kSplitNcb, "split scratch geometry (cham_pool.h)");
#ifndef CHAM_STAGGER
#define CHAM_STAGGER 0  // 1: S(0) S(1) E(0) S(2) E(1) ... (A/B on C2: 103.5k vs 118.5k tok/s for S... E...)
#endif
constexpr bool kStagger = CHAM_STAGGER != 0;
#ifndef CHAM_ASPLIT
#define CHAM_ASPLIT 1  // bulk copies per shrink stage's A chunk
#endif
#ifndef CHAM_STAGGER_1JOB
#define CHAM_STAGGER_1JOB 0  // stagger gap for single-projection launches only
#endif
struct Schedule {
  int n;
  int wide[MAX_BLOCKS];       // expand block in the wide geometry
  int start[MAX_BLOCKS + 1];  // unit prefix
  int kind[MAX_BLOCKS];       // KIND_SHRINK / KIND_EXPAND
  int a[MAX_BLOCKS], e[MAX_BLOCKS];  // LPT positions [a, e) of the class
};

// rounded to 128 B: every stage base must satisfy the TMA tensor-copy alignment (TP v boxes)
constexpr int STAGE_BYTES = ((K1_STAGE > K2_STAGE ? K1_STAGE : K2_STAGE) + 127) / 128 * 128;
static_assert(kWideNp == 0 || K2W_V + TG * kRowsPerPage * 4 <= STAGE_BYTES, "wide expand stage layout");
static_assert(GROUP_THREADS == NCB_WIDE / 16, "wide expand: one consumer thread per 16-byte column chunk");
constexpr int SCRATCH_BYTES = TG * kMaxRank * 4;  // K2 v rows; K1 uses the first 1 KiB
struct Shared {
  alignas(128) unsigned char stage[NSTAGE][STAGE_BYTES];
  alignas(16) unsigned char scratch[SCRATCH_BYTES];
  uint64_t full[NSTAGE];
  uint64_t empty[NSTAGE];
  Meta meta[NSTAGE];
  uint64_t plan_bar;
  int last_cta;  // this CTA re-arms the counters at exit
  int* pub_slot[PQ];
  unsigned pub_bits[PQ];
  uint64_t pub_full[PQ], pub_empty[PQ];
  int unit_mailbox;
  int uq_id[UQN];  // unit ids, producer 0 -> producer 1
  uint64_t uq_full[UQN], uq_empty[UQN];
  Schedule sched;
  Plan plan;
};
static_assert(sizeof(Shared) <= 227 * 1024, "decode kernel shared memory exceeds the 227 KiB per-CTA limit");
using K1Shared = Shared;
using K2Shared = Shared;

__host__ __device__ inline int ceil_div(int a, int b) { return (a + b - 1) / b; }
__host__ __device__ constexpr int cpow2(int v) { return v <= 1 ? 1 : 2 * cpow2((v + 1) / 2); }
__host__ __device__ constexpr int clog2(int v) { return v <= 1 ? 0 : 1 + clog2(v / 2); }

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch_dependents() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// Counter re-arming (CHAM_ZERO_NEXT).  Apply n counts in parity set n % 2.  Once its
// griddepcontrol.wait returned, apply n-1 (the other set's user) is complete, so producer 0 of
// every CTA zeroes its slice of the other set and only then signals launch_dependents: apply
// n+1 cannot start before every slice is zero, and no CTA of apply n needs a last-CTA reset
// (an L2 atomic and a fence on every CTA's exit path) any more.
#ifndef CHAM_ZERO_NEXT
#define CHAM_ZERO_NEXT 1
#endif
constexpr bool kZeroNext = CHAM_ZERO_NEXT != 0;
__device__ __forceinline__ void after_wait(const Params& p, int pid) {
  if (!kZeroNext) {
    pdl_launch_dependents();
    return;
  }
  if (pid != 0) return;  // producer 0 signals, after the re-arm
  const int lane = threadIdx.x & 31;
  const long long step = (long long)gridDim.x * 32;
  for (long long i = (long long)blockIdx.x * 32 + lane; i < p.zero_tile_n; i += step) p.zero_tile[i] = 0;
  for (long long i = (long long)blockIdx.x * 32 + lane; i < p.zero_split_n; i += step) p.zero_split[i] = 0;
  if (blockIdx.x == 0 && lane < 16) p.zero_ctr[lane] = 0;
  __threadfence();
  __syncwarp();
  pdl_launch_dependents();
}

// Reduce-scatter of NV (power of two <= 32) per-lane partial sums across a warp: returns
// the warp-wide sum of value index (lane >> (5 - log2 NV)).
template <int NV>
__device__ __forceinline__ float warp_reduce_scatter(float (&v)[NV], int lane) {
  int n = NV;
#pragma unroll
  for (int w = 16; w >= 1; w >>= 1) {
    if (n > 1) {
      const bool upper = (lane & w) != 0;
#pragma unroll
      for (int i = 0; i < NV / 2; ++i) {
        if (i < n / 2) {
          const float send = upper ? v[i] : v[i + n / 2];
          const float keep = upper ? v[i + n / 2] : v[i];
          v[i] = keep + __shfl_xor_sync(0xffffffffu, send, w);
        }
      }
      n >>= 1;
    } else {
      v[0] += __shfl_xor_sync(0xffffffffu, v[0], w);
    }
  }
  return v[0];
}

// index of the last entry s in [0, S) with start[s] <= v (start non-decreasing)
__device__ __forceinline__ int seg_search(const int* start, int S, int v) {
  int lo = 0, hi = S;
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (start[mid] <= v) lo = mid; else hi = mid;
  }
  return lo;
}

template <typename T>
__device__ __forceinline__ int n_kchunks(const Params& p) {
  return ceil_div(p.h_in * Elem<T>::kBytes, X_ROW);
}
template <typename T>
__device__ __forceinline__ int n_colchunks(const Params& p, int tier) {
  return ceil_div(p.h_out * Elem<T>::kBytes, tier == TIER_W ? NCB_WIDE : tier_ncb(tier));
}

// Builds the launch plan in shared memory (all NTHREADS threads).  It depends only on the
// segment table and the slot table, so one plan serves every (layer, projection) of a step.
__device__ bool build_plan(const Params& p, Plan& pl, int S, UnitDesc* desc = nullptr) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid < kMaxPagesPerSlot + 2) pl.bucket[tid] = 0;
  const int per = ceil_div(S, NTHREADS);
  const int s0 = min(S, tid * per), s1 = min(S, s0 + per);
  int lsh = 0, lpg = 0, lv = 0;
  for (int s = s0; s < s1; ++s) {
    const int o0 = p.seg_off[s], o1 = p.seg_off[s + 1];
    const int slot = p.seg_slot[s];
    const int rank = slot >= 0 ? min(p.seg_rank[s], kMaxRank) : 0;
    pl.seg_off[s] = o0;
    // segments of the tcgen05 prefill path carry no decode work (rank 0 here)
    const bool pre = is_prefill_segment(o1 - o0, rank, p.prefill_thr);
    pl.seg_sr[s] = (slot >= 0 && !pre) ? ((slot << 9) | rank) : 0;
    // same page count as the second pass (0 for prefill-routed segments): the unit, page and
    // v prefixes must not leave holes
    const int np = (slot >= 0 && !pre) ? ceil_div(rank, kRowsPerPage) : 0;
    const int nt = ceil_div(o1 - o0, TG);
    lsh += nt * np;
    lpg += np;
    lv += nt * TG * np * kRowsPerPage;
  }
  int ish = lsh, ipg = lpg, iv = lv;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int a = __shfl_up_sync(0xffffffffu, ish, o);
    const int c = __shfl_up_sync(0xffffffffu, ipg, o);
    const int d = __shfl_up_sync(0xffffffffu, iv, o);
    if (lane >= o) { ish += a; ipg += c; iv += d; }
  }
  if (lane == 31) { pl.scan[warp][0] = ish; pl.scan[warp][1] = ipg; pl.scan[warp][2] = iv; }
  __syncthreads();
  int bsh = 0, bpg = 0, bv = 0;
  for (int w = 0; w < warp; ++w) { bsh += pl.scan[w][0]; bpg += pl.scan[w][1]; bv += pl.scan[w][2]; }
  bsh += ish - lsh;
  bpg += ipg - lpg;
  bv += iv - lv;
  for (int s = s0; s < s1; ++s) {
    const int np = ceil_div(pl.seg_sr[s] & 511, kRowsPerPage);
    const int T_s = p.seg_off[s + 1] - pl.seg_off[s];
    pl.sh_start[s] = bsh;
    pl.seg_pg[s] = bpg;
    pl.v_start[s] = bv;
    bsh += ceil_div(T_s, TG) * np;
    bpg += np;
    bv += ceil_div(T_s, TG) * TG * np * kRowsPerPage;
    if (np > 0 && T_s > 0) atomicAdd(&pl.bucket[np], 1);
  }
  if (tid == NTHREADS - 1) {
    pl.sh_start[S] = bsh;
    pl.seg_pg[S] = bpg;
    pl.v_start[S] = bv;
    const int ntok = S > 0 ? p.seg_off[S] : 0;
    pl.seg_off[S] = ntok;
    pl.totals[0] = bsh;
    pl.totals[2] = ntok;
    pl.totals[3] = bpg;
    pl.totals[4] = bv;
    pl.n_seg = S;
  }
  __syncthreads();
  if (pl.totals[2] > p.max_tokens) return false;
  // LPT order for K2: bucket offsets by decreasing page count, then scatter segments
  if (tid == 0) {
    int acc = 0, ncls = 0;
    for (int np = kMaxPagesPerSlot; np >= 1; --np) {
      const int c = pl.bucket[np];
      if (c > 0) pl.cls_pos[ncls++] = acc;  // one class per page count present
      pl.bucket[np] = acc;
      acc += c;
    }
    pl.cls_pos[ncls] = acc;
    pl.n_cls = ncls;
    pl.totals[5] = acc;  // segments with work
  }
  __syncthreads();
  for (int s = s0; s < s1; ++s) {
    const int np = ceil_div(pl.seg_sr[s] & 511, kRowsPerPage);
    const int T_s = pl.seg_off[s + 1] - pl.seg_off[s];
    if (np > 0 && T_s > 0) {
      const int oi = atomicAdd(&pl.bucket[np], 1);
      pl.order[oi] = s;
      pl.order_pos[s] = oi;
    }
  }
  if (pl.totals[3] <= PLAN_PAGES) {
    for (int s = s0; s < s1; ++s) {
      const int slot = pl.seg_sr[s] >> 9;
      const int np = ceil_div(pl.seg_sr[s] & 511, kRowsPerPage);
      for (int g = 0; g < np; ++g)
        pl.pages[pl.seg_pg[s] + g] = (uint16_t)__ldg(p.slot_pages + slot * kMaxPagesPerSlot + g);
    }
  }
  if (pl.totals[2] <= PLAN_TOKENS) {
    for (int i = tid; i < pl.totals[2]; i += NTHREADS)
      pl.perm[i] = (uint16_t)(p.perm ? __ldg(p.perm + i) : i);
  }
  __syncthreads();
  // K2 tile prefix and K1 unit prefix over the LPT order (one warp scans; <= 512 entries).
  // Both phases walk the segments largest-rank first: when the first expand units are
  // dispatched, the shrink units still in flight belong to the small tiles at the end of the
  // order, so the per-tile v-ready waits of the expand producer almost never block.
  const int nw = pl.totals[5];
  if (warp == 0) {
    int carry = 0, carry_sh = 0;
    for (int base = 0; base < nw; base += 32) {
      const int i = base + lane;
      int u = 0, ush = 0, s = 0;
      if (i < nw) {
        s = pl.order[i];
        u = ceil_div(pl.seg_off[s + 1] - pl.seg_off[s], TG);
        ush = u * ceil_div(pl.seg_sr[s] & 511, kRowsPerPage);
      }
      int inc = u, inc_sh = ush;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int a = __shfl_up_sync(0xffffffffu, inc, o);
        const int b = __shfl_up_sync(0xffffffffu, inc_sh, o);
        if (lane >= o) { inc += a; inc_sh += b; }
      }
      if (i < nw) {
        pl.ex_start[i] = carry + inc - u;
        pl.sh_lpt[i] = carry_sh + inc_sh - ush;
        pl.sh_start[s] = carry_sh + inc_sh - ush;
      }
      carry += __shfl_sync(0xffffffffu, inc, 31);
      carry_sh += __shfl_sync(0xffffffffu, inc_sh, 31);
    }
    if (lane == 0) {
      pl.ex_start[nw] = carry;
      pl.sh_lpt[nw] = carry_sh;
      pl.totals[1] = carry;
      // split tiles: the LPT prefix whose adapters have more than kSplitNp pages
      int nsplit = 0;
      if ((kSplitNp > 0 || kBigTier > 0) && !kStagger) {
        nsplit = carry;
        for (int c = 0; c < pl.n_cls; ++c) {
          const int np_c = ceil_div(pl.seg_sr[pl.order[pl.cls_pos[c]]] & 511, kRowsPerPage);
          if (np_c <= (kSplitNp > 0 ? kSplitNp : 8)) {
            nsplit = pl.ex_start[pl.cls_pos[c]];
            break;
          }
        }
        nsplit = min(nsplit, kSplitCap);
      }
      pl.n_split = nsplit;
    }
  }
  __syncthreads();
  if (desc) {
    // descriptors: shrink units [0, totals[0]) then expand tiles [totals[0], + totals[1])
    if ((long long)pl.totals[0] + pl.totals[1] > p.desc_cap) return false;
    UnitDesc* dex = desc + pl.totals[0];
    for (int s = s0; s < s1; ++s) {
      const int o0 = pl.seg_off[s], T_s = pl.seg_off[s + 1] - o0;
      const int slot = pl.seg_sr[s] >> 9;
      const int np = ceil_div(pl.seg_sr[s] & 511, kRowsPerPage);
      if (np == 0 || T_s == 0) continue;
      const int nt = ceil_div(T_s, TG);
      for (int t = 0; t < nt; ++t) {
        UnitDesc d;
        d.seg = s;
        d.pos0 = o0 + t * TG;
        const int tc = min(TG, T_s - t * TG);
        for (int i = 0; i < TG; ++i) {
          const int pos = d.pos0 + min(i, tc - 1);
          d.rows[i] = p.perm ? __ldg(p.perm + pos) : pos;
        }
        for (int g = 0; g < np; ++g) {
          d.meta = tc | (np << 8) | (g << 16);
          d.aux = __ldg(p.slot_pages + slot * kMaxPagesPerSlot + g);
          desc[pl.sh_start[s] + t * np + g] = d;
        }
        d.meta = tc | (np << 8);
        d.aux = pl.v_start[s] + t * TG * np * kRowsPerPage;  // [page][TG][8] block of the tile
        dex[pl.ex_start[pl.order_pos[s]] + t] = d;
      }
    }
  }
  return true;
}

__device__ __forceinline__ int page_of(const Params& p, const Plan& pl, bool pages_smem, int s, int slot, int g) {
  return pages_smem ? (int)pl.pages[pl.seg_pg[s] + g] : __ldg(p.slot_pages + slot * kMaxPagesPerSlot + g);
}
__device__ __forceinline__ int row_of(const Params& p, const Plan& pl, bool perm_smem, int pos) {
  return perm_smem ? (int)pl.perm[pos] : (p.perm ? __ldg(p.perm + pos) : pos);
}



// Barriers + plan header (one bulk copy; the plan was written by an earlier kernel of the
// step, so it may be read before the PDL wait).
__device__ __forceinline__ bool prologue(const Params& p, Shared& sm) {
  if (threadIdx.x == 0) {
    for (int i = 0; i < NSTAGE; ++i) {
      mbar_init(&sm.full[i], 1);
      mbar_init(&sm.empty[i], GROUP_THREADS);
    }
    mbar_init(&sm.plan_bar, 1);
    for (int i = 0; i < UQN; ++i) {
      mbar_init(&sm.uq_full[i], 1);
      mbar_init(&sm.uq_empty[i], 1);
    }
    for (int i = 0; i < PQ; ++i) {
      mbar_init(&sm.pub_full[i], 1);
      mbar_init(&sm.pub_empty[i], 1);
    }
    fence_mbar_init();
    mbar_arrive_expect_tx(&sm.plan_bar, sizeof(Plan));
    bulk_g2s(&sm.plan, p.plan, sizeof(Plan), &sm.plan_bar, policy_evict_last());
  }
  __syncthreads();
  mbar_wait(&sm.plan_bar, 0);
  return sm.plan.totals[2] <= p.max_tokens;
}

__device__ __forceinline__ void abort_launch(const Params& p) {
  pdl_wait();
  if (threadIdx.x < 32) after_wait(p, 0);  // the next apply's counters are still re-armed
  if (threadIdx.x == 0 && blockIdx.x == 0) *p.err = CHAM_ERR_LIMIT;
}

__device__ __forceinline__ void trace_producer(const Params& p, int seq, unsigned long long t_it,
                                               unsigned long long t_ready, int kind, uint32_t bytes) {
  if (p.trace && seq < p.trace_cap - 1) {
    unsigned long long* tr = p.trace + ((long long)blockIdx.x * p.trace_cap + seq) * 8;
    tr[0] = gtimer();
    tr[1] = ((unsigned long long)kind << 32) | bytes;
    tr[4] = t_it;
    tr[5] = t_ready;
  }
}
// per-CTA life stamps in the last trace slot: 0 entry, 1 plan ready, 2 producer 0 past the
// PDL wait, 3 consumers done, 4 exit
__device__ __forceinline__ void trace_cta(const Params& p, int field) {
  if (p.trace) p.trace[((long long)blockIdx.x * p.trace_cap + p.trace_cap - 1) * 8 + field] = gtimer();
}
__device__ __forceinline__ void trace_consumer(const Params& p, int seq, int field) {
  if (p.trace && seq < p.trace_cap - 1) p.trace[((long long)blockIdx.x * p.trace_cap + seq) * 8 + field] = gtimer();
}

// =========================================================================== K1: shrink
// One unit: nst stages (k-chunks) of one page of one tile; the consumers keep the 8 x NT
// dot products in registers across the stages and write the final v rows at the end.
// The v rows of a finished shrink unit are released to the expand producers (tile counter
// += 1) by a dedicated publisher warp: its gpu-scope fence waits for the stores to be
// acknowledged, which would otherwise stall a consumer warp (and with it the stage release)
// for a full store round trip on every unit.
__device__ __forceinline__ void post_publish(Shared& sm, int& npub, int* ctr, unsigned bits = 0u) {
  const int k = npub++;
  const int slot = k % PQ;
  if (k >= PQ) mbar_wait(&sm.pub_empty[slot], ((k / PQ) - 1) & 1);
  sm.pub_slot[slot] = ctr;
  sm.pub_bits[slot] = bits;
  mbar_arrive(&sm.pub_full[slot]);
}

// ---------------------------------------------------------------- K1 on the tensor cores (bf16)
// The shrink of a 4-token tile against one page is a [T x K] . [K x 8] product: each consumer
// warp runs mma.sync m16n8k16 (bf16 in, fp32 accumulate) over its 1/8 of the stage's K range,
// x rows as the A operand (tokens padded to 16: rows >= T repeat row 0 and are discarded) and
// the page's A^T rows (already K-major and 128 B-swizzled) as the B operand via ldmatrix; the
// eight warp partials are summed through shared memory at the end of the unit.
__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t (&r)[4]) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(addr));
}
__device__ __forceinline__ void ldsm_x2(uint32_t addr, uint32_t (&r)[2]) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x2.shared.b16 {%0,%1}, [%2];" : "=r"(r[0]), "=r"(r[1]) : "r"(addr));
}
__device__ __forceinline__ void mma_16816(float (&d)[4], const uint32_t (&a)[4], const uint32_t (&b)[2]) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
}

template <int NT>
__device__ __forceinline__ void shrink_unit_mma(const Params& p, const Plan& pl, K1Shared& sm, int& seq,
                                                const Meta& m0, float* red, int ct, int lane, int gw, int& npub) {
  constexpr int ES = 2;
  constexpr int NACC = 4;  // independent accumulators: consecutive k-steps do not wait on each other
  float dd[NACC][4];
#pragma unroll
  for (int i = 0; i < NACC; ++i) dd[i][0] = dd[i][1] = dd[i][2] = dd[i][3] = 0.f;
  // ldmatrix row addresses: x (A operand) row rr = lane % 8 + 8 * ((lane / 8) & 1), k half lane / 16;
  // A^T (B operand) rank row j = lane % 8, k half (lane / 8) & 1
  const int rr = (lane & 7) + 8 * ((lane >> 3) & 1);
  const int xrow = rr < NT ? rr : 0;
  const int xko = (lane >> 4) * 8;
  const int bj = lane & 7, bko = ((lane >> 3) & 1) * 8;
  for (int k = 0; k < m0.nst; ++k, ++seq) {
    const int stage = seq % NSTAGE;
    if (k > 0) mbar_wait(&sm.full[stage], (seq / NSTAGE) & 1);
    if (ct == 0) trace_consumer(p, seq, 2);
    const Meta& m = sm.meta[stage];
    const unsigned char* st = sm.stage[stage];
    const int kel = min(X_ROW, p.h_in * ES - m.kc * X_ROW) / ES;  // K elements in this stage
    const int per_warp = kel / GROUP_WARPS;                        // multiple of 16 (h_in % 128 == 0)
    const uint32_t xbase = smem_u32(st + A_CHUNK + xrow * X_PITCH) + xko * ES;
    const uint32_t abase = smem_u32(st);
    if (!kNoCompute) {
      for (int k0 = gw * per_warp; k0 < (gw + 1) * per_warp; k0 += 16 * NACC) {
#pragma unroll
        for (int i = 0; i < NACC; ++i) {
          const int kk = k0 + i * 16;
          if (kk < (gw + 1) * per_warp) {
            uint32_t a[4], b[2];
            ldsm_x4(xbase + kk * ES, a);
            const int kb = kk + bko;  // this lane's 8-element K chunk of the B rows
            ldsm_x2(abase + (kb >> 6) * kAtomBytes + bj * kRowBytes + ((((kb >> 3) & 7) ^ bj) << 4), b);
            mma_16816(dd[i], a, b);
          }
        }
      }
    }
    if (ct == 0) trace_consumer(p, seq, 3);
    mbar_arrive(&sm.empty[stage]);  // this stage has been read: hand it back
  }
  // C fragment: d[0], d[1] = (token row lane / 4, rank rows 2 (lane % 4), +1); rows >= NT are padding
  float d[2] = {0.f, 0.f};
#pragma unroll
  for (int i = 0; i < NACC; ++i) {
    d[0] += dd[i][0];
    d[1] += dd[i][1];
  }
  named_bar_sync(1, GROUP_THREADS);  // the previous unit's readers of `red` are done
  const int g = lane >> 2, c2 = (lane & 3) * 2;
  if (g < NT) {
    red[(gw * TG + g) * kRowsPerPage + c2] = d[0];
    red[(gw * TG + g) * kRowsPerPage + c2 + 1] = d[1];
  }
  named_bar_sync(1, GROUP_THREADS);
  if (ct < NT * kRowsPerPage) {
    const int t = ct / kRowsPerPage, j = ct % kRowsPerPage;
    float sum = 0.f;
#pragma unroll
    for (int w2 = 0; w2 < GROUP_WARPS; ++w2) sum += red[(w2 * TG + t) * kRowsPerPage + j];
    const int row = m0.g * kRowsPerPage + j;
    if (p.v_out) {
      if (row < p.v_cols) p.v_out[(long long)(m0.pos0 + t) * p.v_stride + m0.job * p.v_cols + row] = sum;  // TP
    } else {
      const int tile = (m0.pos0 - pl.seg_off[m0.seg]) / TG;
      const long long vb = pl.v_start[m0.seg] + (long long)tile * TG * m0.np * kRowsPerPage;
      p.vws[m0.job * p.vws_job_stride + vb + (m0.g * TG + t) * kRowsPerPage + j] = sum;
      asm volatile("fence.proxy.async.global;" ::: "memory");  // read later by TMA (async proxy)
    }
  }
  if (p.tile_ctr && gw == 0) {
    // this page's v rows of the tile are final: hand the tile counter to the publisher warp
    __syncwarp();
    if (lane == 0) {
      const int tile = pl.ex_start[pl.order_pos[m0.seg]] + (m0.pos0 - pl.seg_off[m0.seg]) / TG;
      post_publish(sm, npub, p.tile_ctr + m0.job * pl.totals[1] + tile, 1u << m0.g);
    }
  }
}

template <typename T, int NT>
__device__ __forceinline__ void shrink_unit(const Params& p, const Plan& pl, K1Shared& sm, int& seq, const Meta& m0,
                                            float* red, int ct, int lane, int gw, int& npub) {
  constexpr int ES = Elem<T>::kBytes;
  constexpr int EPV = Elem<T>::kEPV;
  constexpr int NP2 = EPV / 2;
  constexpr int NTR = cpow2(NT);
  constexpr int NV = kRowsPerPage * NTR;
  float2 acc2[kRowsPerPage][NT];
#pragma unroll
  for (int j = 0; j < kRowsPerPage; ++j)
#pragma unroll
    for (int t = 0; t < NT; ++t) acc2[j][t] = make_float2(0.f, 0.f);
  for (int k = 0; k < m0.nst; ++k, ++seq) {
    const int stage = seq % NSTAGE;
    if (k > 0) mbar_wait(&sm.full[stage], (seq / NSTAGE) & 1);
    if (ct == 0) trace_consumer(p, seq, 2);
    const Meta& m = sm.meta[stage];
    const unsigned char* st = sm.stage[stage];
    const int kbytes = min(X_ROW, p.h_in * ES - m.kc * X_ROW);
    const unsigned char* X = st + A_CHUNK;
    for (int q = ct; q < (kNoCompute ? 0 : kbytes >> 4); q += GROUP_THREADS) {
      const int a = q >> 3, c = q & 7;
      float2 xf[NT][NP2];
#pragma unroll
      for (int t = 0; t < NT; ++t) Elem<T>::unpack2(lds128(X + t * X_PITCH + q * 16), xf[t]);
#pragma unroll
      for (int j = 0; j < kRowsPerPage; ++j) {
        float2 af[NP2];
        Elem<T>::unpack2(lds128(st + a * kAtomBytes + j * kRowBytes + (((c ^ j) & 7) << 4)), af);
#pragma unroll
        for (int e = 0; e < NP2; ++e)
#pragma unroll
          for (int t = 0; t < NT; ++t) acc2[j][t] = __ffma2_rn(af[e], xf[t][e], acc2[j][t]);
      }
    }
    if (ct == 0) trace_consumer(p, seq, 3);
    mbar_arrive(&sm.empty[stage]);  // this stage has been read: hand it back
  }
  float v[NV];
#pragma unroll
  for (int j = 0; j < kRowsPerPage; ++j)
#pragma unroll
    for (int t = 0; t < NTR; ++t) v[j * NTR + t] = t < NT ? acc2[j][t].x + acc2[j][t].y : 0.f;
  const float mine = warp_reduce_scatter<NV>(v, lane);
  constexpr int SHIFT = 5 - clog2(NV);
  named_bar_sync(1, GROUP_THREADS);  // the previous unit's readers of `red` are done
  if ((lane & ((1 << SHIFT) - 1)) == 0) red[gw * 32 + (lane >> SHIFT)] = mine;
  named_bar_sync(1, GROUP_THREADS);
  if (ct < NV) {
    float sum = 0.f;
#pragma unroll
    for (int w2 = 0; w2 < GROUP_WARPS; ++w2) sum += red[w2 * 32 + ct];
    const int j = ct / NTR, t = ct % NTR;
    if (t < NT) {
      const int row = m0.g * kRowsPerPage + j;
      if (p.v_out) {
        if (row < p.v_cols) p.v_out[(long long)(m0.pos0 + t) * p.v_stride + m0.job * p.v_cols + row] = sum;  // TP
      } else {
        // tile-major layout [page][TG][8 rows]: each expand stage copies its pages' slice
        const int tile = (m0.pos0 - pl.seg_off[m0.seg]) / TG;
        const long long vb = pl.v_start[m0.seg] + (long long)tile * TG * m0.np * kRowsPerPage;
        p.vws[m0.job * p.vws_job_stride + vb + (m0.g * TG + t) * kRowsPerPage + j] = sum;
        asm volatile("fence.proxy.async.global;" ::: "memory");  // read later by TMA (async proxy)
      }
    }
  }
  if (p.tile_ctr && gw == 0) {
    // this page's v rows of the tile are final: hand the tile counter to the publisher warp
    __syncwarp();
    if (lane == 0) {
      const int tile = pl.ex_start[pl.order_pos[m0.seg]] + (m0.pos0 - pl.seg_off[m0.seg]) / TG;
      post_publish(sm, npub, p.tile_ctr + m0.job * pl.totals[1] + tile, 1u << m0.g);
    }
  }
}

// ---------------------------------------------------------------- K2 on the tensor cores (bf16)
// Y[T x 1024] += V[T x 16] . B[16 x 1024] per stage of two pages: each consumer warp owns 128
// columns = 16 mma.sync m16n8k16 tiles; V (fp32 in the stage) is rounded to bf16 into the A
// fragment (tokens padded to 16 rows, a lone page's missing 8 K rows zeroed), B comes straight
// from the page layout (8 rank rows x 64 columns per swizzled atom) with ldmatrix.trans.
__device__ __forceinline__ void ldsm_x2_trans(uint32_t addr, uint32_t (&r)[2]) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x2.trans.shared.b16 {%0,%1}, [%2];" : "=r"(r[0]), "=r"(r[1]) : "r"(addr));
}

template <int NT>
__device__ __forceinline__ void expand_unit_mma(const Params& p, Shared& sm, int& seq, const Meta& m0, int ct,
                                                int lane, int gw) {
  constexpr int NTILE = (NCB_SMALL / 2) / 8 / GROUP_WARPS;  // 16 n-tiles of 8 columns per warp
  float d[NTILE][4];
#pragma unroll
  for (int i = 0; i < NTILE; ++i) d[i][0] = d[i][1] = d[i][2] = d[i][3] = 0.f;
  const int g = lane >> 2, c2 = (lane & 3) * 2;
  const int bj = lane & 7, bpg = (lane >> 3) & 1;  // ldmatrix row: rank row j of page bpg
  const int wcol = gw * NTILE * 8;                  // this warp's first column in the unit
  for (int k = 0; k < m0.nst; ++k, ++seq) {
    const int stage = seq % NSTAGE;
    if (k > 0) mbar_wait(&sm.full[stage], (seq / NSTAGE) & 1);
    if (ct == 0) trace_consumer(p, seq, 2);
    const Meta& m = sm.meta[stage];
    const unsigned char* st = sm.stage[stage];
    if (!kNoCompute) {
      const float* Vst = reinterpret_cast<const float*>(st + K2_V);  // [page in stage][TG][8]
      uint32_t a[4] = {0u, 0u, 0u, 0u};
      if (g < NT) {
        a[0] = pack_bf16x2(Vst[(0 * TG + g) * kRowsPerPage + c2], Vst[(0 * TG + g) * kRowsPerPage + c2 + 1]);
        if (m.npg == 2)
          a[2] = pack_bf16x2(Vst[(1 * TG + g) * kRowsPerPage + c2], Vst[(1 * TG + g) * kRowsPerPage + c2 + 1]);
      }
      // a lone page: its B rows stand in for the missing page (finite; multiplied by zero)
      const uint32_t bbase = smem_u32(st + (m.npg == 2 ? bpg : 0) * m0.pitch) + bj * kRowBytes;
#pragma unroll
      for (int i = 0; i < NTILE; ++i) {
        const int n0 = wcol + i * 8;
        if (n0 * 2 < m0.ncols * 2) {
          uint32_t b[2];
          const int at = n0 >> 6, c = (n0 >> 3) & 7;
          ldsm_x2_trans(bbase + at * kAtomBytes + (((c ^ bj) & 7) << 4), b);
          mma_16816(d[i], a, b);
        }
      }
    }
    if (k == m0.nst - 1 && g < NT) {
      // epilogue: y rows (staged bf16 in this stage) += D, stored straight to global
      const unsigned char* yst = st + K2_Y + g * m0.ncb;
      char* ydst = p.jobs[m0.job].y + ((long long)m0.rows[g] * p.h_out + m0.col0) * 2;
#pragma unroll
      for (int i = 0; i < NTILE; ++i) {
        const int col = wcol + i * 8 + c2;
        if (col < m0.ncols) {
          const uint32_t yv = *reinterpret_cast<const uint32_t*>(yst + col * 2);
          *reinterpret_cast<uint32_t*>(ydst + col * 2) = pack_bf16x2(bf_lo(yv) + d[i][0], bf_hi(yv) + d[i][1]);
        }
      }
    }
    if (ct == 0) trace_consumer(p, seq, 3);
    mbar_arrive(&sm.empty[stage]);
  }
}

// =========================================================================== K2: expand
// One unit: output tile [NT tokens x ncols]; stages walk the adapter's pages PG at a time.
// Thread (q, h) owns 16-byte column chunk q = ct >> lpg and page pg0 + h of each stage
// (h = ct & (PG-1)); a lone page in a PG = 2 stage is split in row halves instead.
template <typename T, int NT>
__device__ __forceinline__ void expand_unit(const Params& p, Shared& sm, int& seq, const Meta& m0, int ct, int& npub) {
  constexpr int ES = Elem<T>::kBytes;
  constexpr int EPV = Elem<T>::kEPV;
  constexpr int NP2 = EPV / 2;
  const int lpg = m0.lpg;
  const int npgmax = 1 << lpg;
  const int h = ct & (npgmax - 1), q = ct >> lpg;
  const int a = q >> 3, c = q & 7;
  const bool active = q < m0.nq && q * EPV < m0.ncols;
  float2 acc[NT][NP2];
#pragma unroll
  for (int t = 0; t < NT; ++t)
#pragma unroll
    for (int e = 0; e < NP2; ++e) acc[t][e] = make_float2(0.f, 0.f);
  for (int k = 0; k < m0.nst; ++k, ++seq) {
    const int stage = seq % NSTAGE;
    if (k > 0) mbar_wait(&sm.full[stage], (seq / NSTAGE) & 1);
    if (ct == 0) trace_consumer(p, seq, 2);
    const Meta& m = sm.meta[stage];
    const unsigned char* st = sm.stage[stage];
    const float* Vst = reinterpret_cast<const float*>(st + (lpg == 0 ? K2W_V : K2_V));  // [page in stage][TG][8]
    if (active && !kNoCompute && m.npg > 0) {
      if (lpg != 1 || m.npg == 2) {
        // own page pg0 + h: all 8 rows, fully unrolled
        if (h < m.npg) {
          const unsigned char* Bg = st + h * m0.pitch;
          float vv[NT][kRowsPerPage];
#pragma unroll
          for (int t = 0; t < NT; ++t) {
            const float4 lo = *reinterpret_cast<const float4*>(Vst + (h * TG + t) * kRowsPerPage);
            const float4 hi = *reinterpret_cast<const float4*>(Vst + (h * TG + t) * kRowsPerPage + 4);
            vv[t][0] = lo.x; vv[t][1] = lo.y; vv[t][2] = lo.z; vv[t][3] = lo.w;
            vv[t][4] = hi.x; vv[t][5] = hi.y; vv[t][6] = hi.z; vv[t][7] = hi.w;
          }
          float2 bf[kRowsPerPage][NP2];
#pragma unroll
          for (int j = 0; j < kRowsPerPage; ++j)
            Elem<T>::unpack2(lds128(Bg + a * kAtomBytes + j * kRowBytes + (((c ^ j) & 7) << 4)), bf[j]);
#pragma unroll
          for (int j = 0; j < kRowsPerPage; ++j)
#pragma unroll
            for (int t = 0; t < NT; ++t) {
              const float2 v2 = make_float2(vv[t][j], vv[t][j]);
#pragma unroll
              for (int e = 0; e < NP2; ++e) acc[t][e] = __ffma2_rn(v2, bf[j][e], acc[t][e]);
            }
        }
      } else {
        // PG = 2 stage with a single page: rows 4h .. 4h+3
        float vv[NT][4];
#pragma unroll
        for (int t = 0; t < NT; ++t) {
          const float4 v4 = *reinterpret_cast<const float4*>(Vst + t * kRowsPerPage + h * 4);
          vv[t][0] = v4.x; vv[t][1] = v4.y; vv[t][2] = v4.z; vv[t][3] = v4.w;
        }
        float2 bf[4][NP2];
#pragma unroll
        for (int jj = 0; jj < 4; ++jj) {
          const int j = h * 4 + jj;
          Elem<T>::unpack2(lds128(st + a * kAtomBytes + j * kRowBytes + (((c ^ j) & 7) << 4)), bf[jj]);
        }
#pragma unroll
        for (int jj = 0; jj < 4; ++jj)
#pragma unroll
          for (int t = 0; t < NT; ++t) {
            const float2 v2 = make_float2(vv[t][jj], vv[t][jj]);
#pragma unroll
            for (int e = 0; e < NP2; ++e) acc[t][e] = __ffma2_rn(v2, bf[jj][e], acc[t][e]);
          }
      }
    }
    if (k == m0.nst - 1) {
      // epilogue on the last stage (it carries the y rows): combine the partial sums of the
      // sibling lanes (adjacent), add into y, store
      for (int o = 1; o < npgmax; o <<= 1) {
#pragma unroll
        for (int t = 0; t < NT; ++t)
#pragma unroll
          for (int e = 0; e < NP2; ++e) {
            acc[t][e].x += __shfl_xor_sync(0xffffffffu, acc[t][e].x, o);
            acc[t][e].y += __shfl_xor_sync(0xffffffffu, acc[t][e].y, o);
          }
      }
      const int ncol_unit = m0.ncb / ES;
      if (active) {
#pragma unroll
        for (int t = 0; t < NT; ++t) {
          if ((t & (npgmax - 1)) == h) {  // sibling h stores tokens t == h (mod PG)
            if (m0.xm == 1) {
              // page half 0: leave the fp32 partial for half 1 (read by its producer's TMA)
              float4* dst = reinterpret_cast<float4*>(p.split_buf + ((long long)m0.sidx * TG + t) * ncol_unit + q * EPV);
#pragma unroll
              for (int e = 0; e < NP2; e += 2)
                dst[e / 2] = make_float4(acc[t][e].x, acc[t][e].y, acc[t][e + 1].x, acc[t][e + 1].y);
              asm volatile("fence.proxy.async.global;" ::: "memory");
              continue;
            }
            float yv[EPV];
            Elem<T>::unpack(lds128(st + (lpg == 0 ? K2W_Y : K2_Y) + t * m0.ncb + q * 16), yv);
            if (m0.xm == 2) {  // combine stage: add half 0's partial
              const float4* pv = reinterpret_cast<const float4*>(st + (t * ncol_unit + q * EPV) * 4);
#pragma unroll
              for (int e = 0; e < NP2; e += 2) {
                const float4 f = pv[e / 2];
                acc[t][e].x += f.x; acc[t][e].y += f.y; acc[t][e + 1].x += f.z; acc[t][e + 1].y += f.w;
              }
            }
#pragma unroll
            for (int e = 0; e < NP2; ++e) {
              yv[2 * e] += acc[t][e].x;
              yv[2 * e + 1] += acc[t][e].y;
            }
            char* dst = p.jobs[m0.job].y + ((long long)m0.rows[t] * p.h_out + m0.col0) * ES + q * 16;
            *reinterpret_cast<uint4*>(dst) = Elem<T>::pack(yv);
          }
        }
      }
      if (m0.xm == 1) {
        // every partial of the slot is written: hand its flag to the publisher warp
        named_bar_sync(1, GROUP_THREADS);
        if (ct == 0) post_publish(sm, npub, p.split_ctr + m0.sidx);
      }
    }
    if (ct == 0) trace_consumer(p, seq, 3);
    mbar_arrive(&sm.empty[stage]);
  }
}

// =========================================================================== fused kernel
// Dynamic unit dispatch for the producer warp: lanes [0, depth) each hold one outstanding
// counter value (an atomicAdd issued depth-1 units earlier).  The raw atomic result is kept
// untouched until the slot is consumed, so the warp never waits on the counter's L2 round
// trip.  The first unit of every CTA is static.  Unit index = slot value + gridDim.x.
// Plain (non-aggregated) fetch-and-increment (atom.inc cannot be warp-aggregated; the
// aggregated atomicAdd reads its result with a shuffle at once = an L2 round-trip stall).
__device__ __forceinline__ int atom_add_lazy(int* p) {
  int old;
  asm volatile("atom.global.inc.u32 %0, [%1], 2147483647;" : "=r"(old) : "l"(p) : "memory");
  return old;
}

struct UnitQueue {
  int q;  // this lane's raw slot value (lanes < depth)
  int head;
  int depth;
  int* ctr;
  int total;
  volatile int* xfer;  // shared-memory mailbox: only the head lane reads its own slot
  __device__ __forceinline__ void init(int* c, int tot, int d, int lane, int* mailbox) {
    ctr = c;
    total = tot;
    depth = d;
    xfer = mailbox;
    head = 0;
    q = 1 << 29;
    if (lane == 0) q = (int)blockIdx.x - (int)gridDim.x;
    else if (lane < depth) q = atom_add_lazy(ctr);
  }
  // next unit index for this CTA, or -1 when the unit space is exhausted
  __device__ __forceinline__ int next(int lane) {
    for (;;) {
      // a shuffle would read q in every lane and wait on every outstanding atomic
      if (lane == head) *xfer = q;
      __syncwarp();
      const int u = *xfer + (int)gridDim.x;
      __syncwarp();
      const int h = head;
      head = head + 1 == depth ? 0 : head + 1;
      if (u < total) {
        if (lane == h) q = atom_add_lazy(ctr);  // refill; the result is read depth-1 units later
        return u;
      }
      if (!__any_sync(0xffffffffu, lane < depth && q + (int)gridDim.x < total)) return -1;
    }
  }
};

__device__ __forceinline__ void ldg_desc(const UnitDesc* d, int4& a, int4& b) {
  const int4* q = reinterpret_cast<const int4*>(d);
  a = __ldg(q);
  b = __ldg(q + 1);
}

// The producer's unit stream.  Segments are grouped into classes of equal page count np,
// largest first (the LPT order of the plan).  Every class c contributes a block of shrink
// units S(c) (job, 4-token tile, page) and a block of expand units E(c) (tile, job,
// 1024-column chunk), dispatched from ONE counter in the order
//     S(0) S(1) E(0) S(2) E(1) ... S(C-1) E(C-2) E(C-1)
// so the long expand units of the large-rank tiles start while shrink work is still in
// flight (instead of after all of it), and each E(c) follows its S(c) by one class: by the
// time an expand unit is claimed its tile's v rows are (nearly always) published.
// MODE_SHRINK streams the S blocks only, MODE_EXPAND the E blocks only.
template <typename T>
__device__ void build_schedule(const Params& p, const Plan& pl, int mode, Schedule& sc) {
  const int J = p.n_jobs;
  const int ncc = n_colchunks<T>(p, 0);
  int n = 0, acc = 0;
  auto add = [&](int kind, int a, int e, bool wide = false) {
    const int t0 = pl.ex_start[a], t1 = pl.ex_start[e];
    if (wide) {
      const int units = J * n_colchunks<T>(p, TIER_W) * (t1 - t0);
      if (units <= 0) return;
      sc.kind[n] = kind;
      sc.wide[n] = 1;
      sc.a[n] = a;
      sc.e[n] = e;
      sc.start[n] = acc;
      acc += units;
      ++n;
      return;
    }
    const int nsp = max(0, min(pl.n_split, t1) - t0);  // split tiles inside the block
    const bool big_tier = kBigTier == 2;
    const int ncc2 = n_colchunks<T>(p, 2);
    const int units = kind == KIND_SHRINK ? J * (pl.sh_lpt[e] - pl.sh_lpt[a])
                      : big_tier          ? J * (ncc * (t1 - t0 - nsp) + ncc2 * nsp)
                      : kSplitNp > 0      ? J * ncc * (t1 - t0 + nsp)
                                          : J * ncc * (t1 - t0);
    if (units <= 0) return;
    sc.kind[n] = kind;
    sc.wide[n] = 0;
    sc.a[n] = a;
    sc.e[n] = e;
    sc.start[n] = acc;
    acc += units;
    ++n;
  };
  const int C = pl.n_cls;
  const int gap = kStagger ? CHAM_STAGGER : (J == 1 ? CHAM_STAGGER_1JOB : 0);
  if (gap > 0) {
    // E(c) follows S(c + gap): the classes between give S(c) time to complete
    for (int c = 0; c < C; ++c) {
      if (mode != MODE_EXPAND) add(KIND_SHRINK, pl.cls_pos[c], pl.cls_pos[c + 1]);
      if (mode != MODE_SHRINK && c >= gap) add(KIND_EXPAND, pl.cls_pos[c - gap], pl.cls_pos[c - gap + 1]);
    }
    if (mode != MODE_SHRINK)
      for (int c = max(0, C - gap); c < C; ++c) add(KIND_EXPAND, pl.cls_pos[c], pl.cls_pos[c + 1]);
  } else {
    if (mode != MODE_EXPAND) add(KIND_SHRINK, pl.cls_pos[0], pl.cls_pos[C]);
    if (mode != MODE_SHRINK) {
      // classes are in decreasing page count: the small-rank tail takes the wide geometry
      int cw = C;
      if (kWideNp > 0 && kSplitNp == 0 && kBigTier == 0) {
        cw = 0;
        while (cw < C && ceil_div(pl.seg_sr[pl.order[pl.cls_pos[cw]]] & 511, kRowsPerPage) > kWideNp) ++cw;
      }
      add(KIND_EXPAND, pl.cls_pos[0], pl.cls_pos[cw]);
      if (cw < C) add(KIND_EXPAND, pl.cls_pos[cw], pl.cls_pos[C], true);
    }
  }
  sc.start[n] = acc;
  sc.n = n;
}

// unit -> (block, job, descriptor index, column chunk)
struct UnitPos {
  int kind, job, di, cc, half, tier;
};
template <typename T>
__device__ __forceinline__ UnitPos locate(const Params& p, const Plan& pl, const Schedule& sc, int u) {
  int b = 0;
  while (b + 1 < sc.n && sc.start[b + 1] <= u) ++b;
  const int rel = u - sc.start[b];
  UnitPos r;
  r.kind = sc.kind[b];
  if (r.kind == KIND_SHRINK) {
    const int span = pl.sh_lpt[sc.e[b]] - pl.sh_lpt[sc.a[b]];
    r.job = rel / span;
    r.di = pl.sh_lpt[sc.a[b]] + (rel - r.job * span);
    r.cc = 0;
    r.half = -1;
    r.tier = 0;
  } else if (sc.wide[b]) {
    const int nccw = n_colchunks<T>(p, TIER_W);
    const int per_tile = p.n_jobs * nccw;
    r.tier = TIER_W;
    r.half = -1;
    r.di = pl.ex_start[sc.a[b]] + rel / per_tile;
    const int jc = rel - (rel / per_tile) * per_tile;
    r.job = jc / nccw;
    r.cc = jc - r.job * nccw;
  } else {
    const int ncc = n_colchunks<T>(p, 0);
    const int per_tile = p.n_jobs * ncc;
    const int t0 = pl.ex_start[sc.a[b]];
    const int nsp = max(0, min(pl.n_split, pl.ex_start[sc.e[b]]) - t0);
    const bool big_tier = kBigTier == 2;
    int jc;
    r.tier = 0;
    if (big_tier && rel < nsp * p.n_jobs * n_colchunks<T>(p, 2)) {  // large-rank tiles, tier-2 geometry
      const int ncc2 = n_colchunks<T>(p, 2), per2 = p.n_jobs * ncc2;
      r.half = -1;
      r.tier = 2;
      r.di = t0 + rel / per2;
      jc = rel % per2;
      r.job = jc / ncc2;
      r.cc = jc - r.job * ncc2;
      return r;
    } else if (big_tier) {
      const int r2 = rel - nsp * p.n_jobs * n_colchunks<T>(p, 2);
      r.half = -1;
      r.di = t0 + nsp + r2 / per_tile;
      jc = r2 % per_tile;
    } else if (kSplitNp > 0 && rel < 2 * nsp * per_tile) {  // split tiles: (tile, job, chunk) x 2 page halves
      r.half = rel & 1;
      r.di = t0 + (rel >> 1) / per_tile;
      jc = (rel >> 1) % per_tile;
    } else {
      const int r2 = rel - 2 * nsp * per_tile;
      r.half = -1;
      r.di = t0 + nsp + r2 / per_tile;  // expand tile
      jc = r2 % per_tile;
    }
    r.job = jc / ncc;
    r.cc = jc - r.job * ncc;
  }
  return r;
}

#ifndef CHAM_PUB_FENCE
#define CHAM_PUB_FENCE 0  // publisher: fence + relaxed atomic (1) or one release reduction / release OR (0); A/B on C2 with page-ready tiles: 131.5k vs 132.8k (wide 8)
#endif
constexpr bool kPubFence = CHAM_PUB_FENCE != 0;
#ifndef CHAM_PAGE_READY
#define CHAM_PAGE_READY 1  // 1: tile counters as page bitmasks, an expand stage waits for its own pages only (round 1: C2 117.0k vs 117.3k; round 2: 131.0k vs 130.3k)
#endif
constexpr bool kPageReady = CHAM_PAGE_READY != 0;
// pages [pg0, pg0 + n) of a tile as a mask (np <= 32 pages per adapter)
__device__ __forceinline__ unsigned page_bits(int pg0, int n) {
  return (n >= 32 ? 0xffffffffu : ((1u << n) - 1u)) << pg0;
}
// all np shrink units of the tile published (counter or page mask)
__device__ __forceinline__ bool tile_ready(int v, int np) {
  return kPageReady ? ((unsigned)v & page_bits(0, np)) == page_bits(0, np) : v >= np;
}
#ifndef CHAM_EARLY_A
#define CHAM_EARLY_A 0  // 1: A chunks of the whole first ring pass before griddepcontrol.wait (C2 114.0k vs 115.2k off)
#endif
// x copies of the first ring pass held back until the previous kernel has completed, so the
// adapter (A) parts of up to NSTAGE stages stream while that kernel drains.  Per lane: its x
// row's source; the stage, barrier and size are uniform.
struct PendingX {
  const char* src[NSTAGE];
  uint32_t dst[NSTAGE];
  uint32_t bar[NSTAGE];
  uint32_t bytes[NSTAGE];
  bool on[NSTAGE];
  int n;
};
__device__ __forceinline__ void pend_add(PendingX& q, const char* src, void* dst, uint64_t* bar, uint32_t bytes, bool on) {
#pragma unroll
  for (int i = 0; i < NSTAGE; ++i)
    if (i == q.n) {
      q.src[i] = src;
      q.dst[i] = smem_u32(dst);
      q.bar[i] = smem_u32(bar);
      q.bytes[i] = bytes;
      q.on[i] = on;
    }
  ++q.n;
}
// wait for the previous kernel (x, y and the workspaces may be its outputs), then issue the
// held-back x copies
__device__ __forceinline__ void pend_flush(const Params& p, int pid, PendingX& q, bool& waited, uint64_t pol_x) {
  if (waited) return;
  pdl_wait();
  after_wait(p, pid);
  waited = true;
#pragma unroll
  for (int i = 0; i < NSTAGE; ++i)
    if (i < q.n && q.on[i])
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
          "[%0], [%1], %2, [%3], %4;" ::"r"(q.dst[i]),
          "l"(q.src[i]), "r"(q.bytes[i]), "r"(q.bar[i]), "l"(pol_x)
          : "memory");
  q.n = 0;
}

template <typename T>
__device__ __forceinline__ int issue_shrink(const Params& p, Shared& sm, int seq, bool& waited, PendingX& pend, int job,
                                            int4 da, int4 db, int pid) {
  constexpr int ES = Elem<T>::kBytes;
  const int lane = threadIdx.x & 31;
  const int nkc = n_kchunks<T>(p);
  const int natoms = p.h_in * ES / kRowBytes;
  const uint64_t pol_w = policy_evict_first();  // weights: streamed once per step
  const uint64_t pol_x = policy_evict_last();   // x rows: re-read by every page of the tile
  const int s = da.x, pos0 = da.y;
  const int tcount = da.z & 0xff, np = (da.z >> 8) & 0xff, g = da.z >> 16;
  const int row = lane == 0 ? db.x : lane == 1 ? db.y : lane == 2 ? db.z : db.w;
  const Job& jb = p.jobs[job];
  const char* a_src = p.base + (long long)da.w * p.page_bytes + jb.a_off;
  for (int kc = 0; kc < nkc; ++kc, ++seq) {
    if (NPROD > 1 && (seq & 1) != pid) continue;  // the other producer's stage
    const unsigned long long t_it = p.trace ? gtimer() : 0;
    const int stage = seq % NSTAGE;
    const int a0 = kc * (A_CHUNK / kAtomBytes);
    const uint32_t a_bytes = min(A_CHUNK / kAtomBytes, natoms - a0) * kAtomBytes;
    const uint32_t x_bytes = a_bytes / kRowsPerPage;
    unsigned char* st = sm.stage[stage];
    // a stage's second use waits for consumers that need their x rows: release them first
    if (seq >= NSTAGE) pend_flush(p, pid, pend, waited, pol_x);
    if (lane == 0) mbar_wait(&sm.empty[stage], ((seq / NSTAGE) & 1) ^ 1);
    const unsigned long long t_ready = p.trace ? gtimer() : 0;
    __syncwarp();
    Meta& m = sm.meta[stage];
    if (lane < tcount) m.rows[lane] = row;
    __syncwarp();  // every Meta store precedes lane 0's release-arrive below
    if (lane == 0) {
      m.kind = KIND_SHRINK; m.nst = nkc; m.job = job; m.seg = s; m.pos0 = pos0; m.T = tcount; m.np = np;
      m.g = g; m.kc = kc;
      mbar_arrive_expect_tx(&sm.full[stage], a_bytes + x_bytes * tcount);
    }
    __syncwarp();
    {
      // the A chunk as CHAM_ASPLIT copies issued by different lanes
      const uint32_t part = a_bytes / CHAM_ASPLIT;
      if (lane < CHAM_ASPLIT) {
        const uint32_t nb = lane == CHAM_ASPLIT - 1 ? a_bytes - part * (CHAM_ASPLIT - 1) : part;
        bulk_g2s(st + lane * part, a_src + (long long)a0 * kAtomBytes + lane * part, nb, &sm.full[stage], pol_w);
      }
    }
    const char* x_src = jb.x + ((long long)row * p.h_in) * ES + (long long)kc * X_ROW;
    if (!waited && CHAM_EARLY_A) {  // x may be produced by the previous kernel: hold it back
      pend_add(pend, x_src, st + A_CHUNK + lane * X_PITCH, &sm.full[stage], x_bytes, lane < tcount);
    } else {
      pend_flush(p, pid, pend, waited, pol_x);
      if (lane < tcount) bulk_g2s(st + A_CHUNK + lane * X_PITCH, x_src, x_bytes, &sm.full[stage], pol_x);
    }
    if (lane == 0) trace_producer(p, seq, t_it, t_ready, 1, a_bytes + x_bytes * tcount);
    __syncwarp();
  }
  return seq;
}

template <typename T>
__device__ __forceinline__ int issue_expand(const Params& p, Shared& sm, int seq, bool& waited, PendingX& pend,
                                            bool fused, int job, int cc, int tile, int half, int tier, int4 da,
                                            int4 db, int rdy, int unit, int pid) {
  constexpr int ES = Elem<T>::kBytes;
  pend_flush(p, pid, pend, waited, policy_evict_last());
  const Plan& pl = sm.plan;
  const int lane = threadIdx.x & 31;
  const int NTL = pl.totals[1];
  const bool pages_smem = pl.totals[3] <= PLAN_PAGES;
  const uint64_t pol_w = policy_evict_first();
  const int s = da.x, pos0 = da.y;
  const int tcount = da.z & 0xff, np = (da.z >> 8) & 0xff;
  const int vbase = da.w;
  const int row = lane == 0 ? db.x : lane == 1 ? db.y : lane == 2 ? db.z : db.w;
  const int slot = pl.seg_sr[s] >> 9;
  // tier 0: two consumer threads per 16-byte column chunk (EX_PAGES pages per stage; one page
  // is split in row halves); tier 2: eight threads, one page each, 8 pages per stage
  const bool wide = tier == TIER_W;
  const int lpg = wide ? 0 : tier == 2 ? 3 : 1;
  const int pgs = wide ? 1 : tier == 2 ? 8 : EX_PAGES;
  const int ncb = wide ? NCB_WIDE : tier_ncb(tier);
  const int pitch = wide ? K2W_Y : tier_pitch(tier);
  const int yoff = wide ? K2W_Y : K2_Y;
  const int voff = wide ? K2W_V : K2_V;
  const int ncol_unit = ncb / ES;
  const int col0 = cc * ncol_unit;
  const int ncols = min(ncol_unit, p.h_out - col0);
  const uint32_t b_bytes = ncols * ES * kRowsPerPage;  // per page
  const uint32_t y_bytes = ncols * ES;                  // per token
  const int rpad = np * kRowsPerPage;
  const int vrow = p.v_in ? min(rpad, p.v_cols) : rpad;
  // page range of this unit: all pages, or one half of them (the second half adds a combine stage)
  const int pb = half == 1 ? np / 2 : 0, pe = half == 0 ? np / 2 : np;
  const int nst_pg = ceil_div(pe - pb, pgs);
  const int nst = nst_pg + (half == 1 ? 1 : 0);
  const int xm = half + 1;
  const int sidx = half >= 0 ? (job * kSplitCap + tile) * p.split_ncc + cc : 0;
  const Job& jb = p.jobs[job];
  bool v_checked = false;  // this producer has seen the tile's v rows published
  for (int k = 0; k < nst; ++k, ++seq) {
    if (NPROD > 1 && (seq & 1) != pid) continue;  // the other producer's stage
    const unsigned long long t_it = p.trace ? gtimer() : 0;
    const int stage = seq % NSTAGE;
    unsigned char* st = sm.stage[stage];
    if (k == nst_pg) {
      // half 1's combine stage: y rows + half 0's fp32 partial (published through split_ctr)
      const uint32_t part_bytes = ncol_unit * 4;  // per token
      if (lane == 0) {
        mbar_wait(&sm.empty[stage], ((seq / NSTAGE) & 1) ^ 1);
        while (ld_acquire_gpu(p.split_ctr + sidx) < 1) __nanosleep(32);
        asm volatile("fence.proxy.async.global;" ::: "memory");
      }
      __syncwarp();
      Meta& m = sm.meta[stage];
      if (lane < tcount) m.rows[lane] = row;
      __syncwarp();
      if (lane == 0) {
        m.kind = KIND_EXPAND; m.nst = nst; m.job = job; m.seg = s; m.pos0 = pos0; m.T = tcount; m.np = np;
        m.pg0 = pe; m.npg = 0; m.col0 = col0; m.ncols = ncols; m.vrow = vrow;
        m.lpg = lpg; m.ncb = ncb; m.pitch = pitch; m.nq = ncb / 16; m.xm = xm; m.sidx = sidx;
        mbar_arrive_expect_tx(&sm.full[stage], (y_bytes + part_bytes) * tcount);
        bulk_g2s(st, p.split_buf + (long long)sidx * TG * ncol_unit, part_bytes * tcount, &sm.full[stage], pol_w);
      }
      if (lane < tcount) {
        bulk_g2s(st + yoff + lane * ncb, jb.y + ((long long)row * p.h_out + col0) * ES, y_bytes, &sm.full[stage], pol_w);
      }
      __syncwarp();
      continue;
    }
    const int pg0 = pb + k * pgs;
    const int npg = min(pgs, pe - pg0);
    const bool y_here = half < 0 && k == nst - 1;  // plain units: the last stage carries the y rows
    // every stage carries its pages' v slice; the last one also the y rows.  With a
    // caller-provided v (TP) only pages inside v_stride are copied, the rest are zeroed.
    const int npg_in = p.v_in ? max(0, min(npg, vrow / kRowsPerPage - pg0)) : npg;
    const uint32_t v_bytes = p.v_in ? npg_in * TG * kRowsPerPage * 4 : npg * TG * kRowsPerPage * 4;
    uint32_t bytes = b_bytes * npg + v_bytes;
    if (y_here) bytes += y_bytes * tcount;
    int pgid = 0;
    if (lane < npg) pgid = page_of(p, pl, pages_smem, s, slot, pg0 + lane);
    if (lane == 0) mbar_wait(&sm.empty[stage], ((seq / NSTAGE) & 1) ^ 1);
    const unsigned long long t_ready = p.trace ? gtimer() : 0;
    __syncwarp();
    if (p.v_in && npg_in < npg) {
      for (int c2 = lane; c2 < (npg - npg_in) * tcount; c2 += 32) {
        const int hh = npg_in + c2 / tcount, t = c2 % tcount;
        float4* z = reinterpret_cast<float4*>(st + voff + (hh * TG + t) * kRowsPerPage * 4);
        z[0] = make_float4(0.f, 0.f, 0.f, 0.f);
        z[1] = make_float4(0.f, 0.f, 0.f, 0.f);
      }
      fence_proxy_async_shared();  // generic zero stores before later TMA writes to the stage
      __syncwarp();
    }
    Meta& m = sm.meta[stage];
    if (lane < tcount) m.rows[lane] = row;
    __syncwarp();  // every Meta store precedes lane 0's release-arrive below
    if (lane == 0) {
      m.kind = KIND_EXPAND; m.nst = nst; m.job = job; m.seg = s; m.pos0 = pos0; m.T = tcount; m.np = np;
      m.pg0 = pg0; m.npg = npg; m.col0 = col0; m.ncols = ncols; m.vrow = vrow;
      m.lpg = lpg; m.ncb = ncb; m.pitch = pitch; m.nq = ncb / 16; m.xm = xm; m.sidx = sidx;
      mbar_arrive_expect_tx(&sm.full[stage], bytes);
    }
    // B pages of this stage (weights: independent of phase 1 and of the previous kernel)
    if (lane < npg) {
      const char* src = p.base + (long long)pgid * p.page_bytes + jb.b_off + (long long)col0 * ES * kRowsPerPage;
      bulk_g2s(st + lane * pitch, src, b_bytes, &sm.full[stage], pol_w);
    }
    if (!waited) {  // y may be produced by the previous kernel
      pdl_wait();
      after_wait(p, pid);
      waited = true;
    }
    if (y_here && lane < tcount)
      bulk_g2s(st + yoff + lane * ncb, jb.y + ((long long)row * p.h_out + col0) * ES, y_bytes, &sm.full[stage], pol_w);
    if (fused && kPageReady) {
      // this stage's v rows are final once the shrink units of ITS pages published (writers:
      // v stores, proxy fence; publisher warp: gpu fence, page bit).  The mask was peeked when
      // the unit was claimed and is refreshed only while a needed page is still in flight.
      const unsigned need = page_bits(pg0, npg);
      if (lane == 0) {
        if (((unsigned)rdy & need) != need) {
          const int* c = p.tile_ctr + job * NTL + tile;
          while ((((unsigned)(rdy = ld_acquire_gpu(c))) & need) != need) __nanosleep(20);
        } else {
          fence_acquire_gpu();  // acquire pattern for the relaxed peek
        }
        fence_proxy_async_global();
      }
      __syncwarp();
    } else if (fused && !v_checked) {
      // (first stage of the unit THIS producer issues: with two producers the other one
      // issues every other stage and checks the counter itself)
      // the tile's v rows are complete once all np shrink units of (job, tile) published
      // (writers: v stores, proxy fence; publisher warp: gpu fence, counter).  The counter
      // was peeked when the unit was claimed; only a tile still in flight then is polled.
      if (lane == 0) {
        if (rdy < np) {
          const int* c = p.tile_ctr + job * NTL + tile;
          while (ld_acquire_gpu(c) < np) __nanosleep(20);
        } else {
          // the counter was peeked relaxed: this fence turns that read into an acquire
          // (happens-after the publishers' releases) before the v rows are read
          fence_acquire_gpu();
        }
        fence_proxy_async_global();  // generic-proxy v stores -> the bulk copy below
      }
      __syncwarp();
      v_checked = true;
    }
    if (p.v_in) {
      // TP: v [position][v_stride] -> stage [page][token][8]: one 2-D box (8 ranks x TG
      // positions; rows past the tile are read and ignored, past the buffer zero-filled) per page
      if (lane < npg_in)
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint "
            "[%0], [%1, {%2, %3}], [%4], %5;" ::"r"(smem_u32(st + voff + lane * TG * kRowsPerPage * 4)),
            "l"(reinterpret_cast<uint64_t>(&p.vmap)), "r"(job * p.v_cols + (pg0 + lane) * kRowsPerPage), "r"(pos0),
            "r"(smem_u32(&sm.full[stage])), "l"(pol_w)
            : "memory");
    } else if (lane == 0) {
      bulk_g2s(st + voff, p.vws + job * p.vws_job_stride + vbase + pg0 * TG * kRowsPerPage, v_bytes, &sm.full[stage],
               pol_w);
    }
    if (lane == 0) {
      trace_producer(p, seq, t_it, t_ready, 2, bytes);
      if (p.trace && seq < p.trace_cap - 1) {
        p.trace[((long long)blockIdx.x * p.trace_cap + seq) * 8 + 6] = unit;
        p.trace[((long long)blockIdx.x * p.trace_cap + seq) * 8 + 7] = (np << 8) | tcount;
      }
    }
    __syncwarp();
  }
  return seq;
}

template <typename T>
__device__ __forceinline__ int produce_all(const Params& p, Shared& sm, int seq, bool& waited, int mode, int pid) {
  PendingX pend;
  pend.n = 0;
  const Plan& pl = sm.plan;
  const int lane = threadIdx.x & 31;
  const bool fused = mode == MODE_FUSED;
  Schedule& sc = sm.sched;
  // producer 0 builds the schedule; producer 1 reads it only after receiving a unit id
  // (the queue's mbarrier orders the schedule stores before)
  if (pid == 0 && lane == 0) build_schedule<T>(p, pl, mode, sc);
  __syncwarp();
  const int total = pid == 0 ? sc.start[sc.n] : 0;
  const int NTL = pl.totals[1];
  const UnitDesc* desc = reinterpret_cast<const UnitDesc*>(static_cast<const char*>(p.plan) + sizeof(Plan));
  UnitQueue uq;
  if (pid == 0) uq.init(p.ctr, total, CHAM_SH_DEPTH, lane, &sm.unit_mailbox);
  // the CTA's unit stream: producer 0 claims and forwards, producer 1 receives
  int nq = 0;
  auto next_unit = [&]() {
    int u = -1;
    if (NPROD == 1) return uq.next(lane);
    const int q = nq % UQN;
    if (pid == 0) {
      u = uq.next(lane);
      if (lane == 0) {
        if (nq >= UQN) mbar_wait(&sm.uq_empty[q], ((nq / UQN) - 1) & 1);
        sm.uq_id[q] = u;
        mbar_arrive(&sm.uq_full[q]);
      }
    } else {
      if (lane == 0) {
        mbar_wait(&sm.uq_full[q], (nq / UQN) & 1);
        u = sm.uq_id[q];
        mbar_arrive(&sm.uq_empty[q]);
      }
      u = __shfl_sync(0xffffffffu, u, 0);
    }
    ++nq;
    return u;
  };
  // descriptor and (expand) tile-ready counter of a unit, fetched one unit ahead (relaxed)
  auto fetch = [&](int u, UnitPos& up, int4& a, int4& b, int& rdy) {
    up = locate<T>(p, pl, sc, u);
    ldg_desc(desc + (up.kind == KIND_SHRINK ? up.di : pl.totals[0] + up.di), a, b);
    rdy = 0;
    if (up.kind == KIND_EXPAND && fused && lane == 0) {
      const int* c = p.tile_ctr + up.job * NTL + up.di;
      asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(rdy) : "l"(c) : "memory");
    }
  };
  // Units are fetched (descriptor loads from L2, tile-counter peek) two units ahead of the
  // one being issued, so a stream of one-stage units does not wait on the L2 round trip.
  struct Fetched {
    int unit, rdy;
    UnitPos up;
    int4 a, b;
  };
  auto take = [&](Fetched& f) {
    f.unit = next_unit();
    f.rdy = 0;
    if (f.unit >= 0) fetch(f.unit, f.up, f.a, f.b, f.rdy);
  };
  Fetched f0, f1;
  take(f0);
  f1.unit = -1;
  if (f0.unit >= 0) take(f1);
  while (f0.unit >= 0) {
    Fetched f2;
    f2.unit = -1;
    if (f1.unit >= 0) take(f2);
    if (f0.up.kind == KIND_SHRINK)
      seq = issue_shrink<T>(p, sm, seq, waited, pend, f0.up.job, f0.a, f0.b, pid);
    else
      seq = issue_expand<T>(p, sm, seq, waited, pend, fused, f0.up.job, f0.up.cc, f0.up.di, f0.up.half, f0.up.tier, f0.a,
                            f0.b, f0.rdy, f0.unit, pid);
    f0 = f1;
    f1 = f2;
  }
  pend_flush(p, pid, pend, waited, policy_evict_last());
  return seq;
}

// Out of units: pull the hinted next apply's first A blocks into L2 (evict_last, so they
// survive until that apply's evict_first reads).  Items are the next apply's shrink units in
// its own claim order (job-major, descriptor order over the SAME plan), spread statically
// over the CTAs (item u -> CTA u % grid): one SM's TMA engine moves ~50 GB/s, so a CTA that
// took many items would hold its SM's copy queue for tens of microseconds.
__device__ __noinline__ void prefetch_next_apply(const Params& p, const Plan& pl, int lane) {
  const int per_job = pl.totals[0];
  const int total = min(p.nx_items, per_job * p.nx_jobs);
  const int G = gridDim.x;
  const UnitDesc* desc = reinterpret_cast<const UnitDesc*>(static_cast<const char*>(p.plan) + sizeof(Plan));
  const uint64_t pol = policy_evict_last();
  for (int u = blockIdx.x + lane * G; u < total; u += 32 * G) {
    const int job = u / per_job, di = u - job * per_job;
    const int page = __ldg(&desc[di].aux);
    asm volatile("cp.async.bulk.prefetch.L2.global.L2::cache_hint [%0], %1, %2;" ::"l"(
                     p.base + (long long)page * p.page_bytes + p.nx_a_off[job]),
                 "r"(p.nx_a_bytes), "l"(pol)
                 : "memory");
  }
}

// Marker stage (end of the unit stream).
__device__ __forceinline__ void post_marker(Shared& sm, int seq, int kind) {
  const int st = seq % NSTAGE;
  mbar_wait(&sm.empty[st], ((seq / NSTAGE) & 1) ^ 1);
  sm.meta[st].kind = kind;
  mbar_arrive(&sm.full[st]);
}

// One launch per lora_apply: phase 1 (shrink units) then phase 2 (expand units) from one
// CTA-local stream; an expand unit waits only for its own tile's shrink units (per-tile
// counters), not for the whole grid.  MODE_SHRINK runs phase 1 only (v to v_out),
// MODE_EXPAND phase 2 only (v_in).
template <typename T>
__global__ void __launch_bounds__(APPLY_THREADS, 1) lora_apply_kernel(const __grid_constant__ Params p, int mode) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  Shared& sm = *reinterpret_cast<Shared*>(smem_raw);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) trace_cta(p, 0);
  if (!prologue(p, sm)) {
    abort_launch(p);
    return;
  }
  if (tid == 0) trace_cta(p, 1);
  const bool fused = mode == MODE_FUSED;
  // The producer is the highest-numbered warp: the SM's warp schedulers favour higher warp
  // ids, so the producer is never starved by the FMA-heavy consumer warps on its SMSP.
  if (warp == GROUP_WARPS + 1) {
    // publisher: releases finished shrink units' v rows (tile counter += 1) in post order
    if (lane == 0) {
      for (int k = 0;; ++k) {
        const int slot = k % PQ;
        mbar_wait(&sm.pub_full[slot], (k / PQ) & 1);
        int* c = sm.pub_slot[slot];
        const unsigned bits = sm.pub_bits[slot];
        mbar_arrive(&sm.pub_empty[slot]);
        if (!c) break;
        if (kPubFence) __threadfence();  // explicit fence before the release (A/B switch)
        if (kPageReady && bits) {  // page g of the tile is final
          if (kPubFence)
            atomicOr(reinterpret_cast<unsigned*>(c), bits);
          else
            red_release_gpu_or(reinterpret_cast<unsigned*>(c), bits);  // release, cumulative as below
        } else if (kPubFence)
          atomicAdd(c, 1);  // tile counters without page masks; split-unit partials
        else
          red_release_gpu_add(c, 1);  // release is cumulative over the consumers' v stores
                                      // (acquired through pub_full)
      }
    }
  } else if (warp == GROUP_WARPS || warp == GROUP_WARPS + 2) {
    const int pid = warp == GROUP_WARPS ? 0 : 1;
    bool waited = false;
    int seq = 0;
    seq = produce_all<T>(p, sm, seq, waited, mode, pid);
    if (!waited) {
      pdl_wait();
      after_wait(p, pid);  // a CTA without units still re-arms its slice
    }
    if (lane == 0 && (NPROD == 1 || (seq & 1) == pid)) post_marker(sm, seq, KIND_END);
    if (pid == 0 && p.nx_items > 0) prefetch_next_apply(p, sm.plan, lane);
  } else {
    const int ct = tid;  // consumer warps 0 .. GROUP_WARPS-1
    const int gw = ct >> 5;
    float* red = reinterpret_cast<float*>(sm.scratch);
    int npub = 0;  // consumer thread 0: tile counters posted to the publisher
    int seq = 0;
    for (;;) {
      const int stage = seq % NSTAGE;
      mbar_wait(&sm.full[stage], (seq / NSTAGE) & 1);
      const Meta m0 = sm.meta[stage];
      if (m0.kind == KIND_END) {
        if (ct == 0) post_publish(sm, npub, nullptr);  // the publisher exits
        break;
      }
      if (m0.kind == KIND_SHRINK) {
        switch (m0.T) {
          case 1:
            if (kMmaShrink && Elem<T>::kDtype == CHAM_BF16 && p.h_in % 128 == 0) shrink_unit_mma<1>(p, sm.plan, sm, seq, m0, red, ct, lane, gw, npub);
            else shrink_unit<T, 1>(p, sm.plan, sm, seq, m0, red, ct, lane, gw, npub);
            break;
          case 2:
            if (kMmaShrink && Elem<T>::kDtype == CHAM_BF16 && p.h_in % 128 == 0) shrink_unit_mma<2>(p, sm.plan, sm, seq, m0, red, ct, lane, gw, npub);
            else shrink_unit<T, 2>(p, sm.plan, sm, seq, m0, red, ct, lane, gw, npub);
            break;
          case 3:
            if (kMmaShrink && Elem<T>::kDtype == CHAM_BF16 && p.h_in % 128 == 0) shrink_unit_mma<3>(p, sm.plan, sm, seq, m0, red, ct, lane, gw, npub);
            else shrink_unit<T, 3>(p, sm.plan, sm, seq, m0, red, ct, lane, gw, npub);
            break;
          default:
            if (kMmaShrink && Elem<T>::kDtype == CHAM_BF16 && p.h_in % 128 == 0) shrink_unit_mma<4>(p, sm.plan, sm, seq, m0, red, ct, lane, gw, npub);
            else shrink_unit<T, 4>(p, sm.plan, sm, seq, m0, red, ct, lane, gw, npub);
            break;
        }
      } else {
        switch (m0.T) {
          case 1:
            if (kMmaExpand && Elem<T>::kDtype == CHAM_BF16 && m0.xm == 0 && m0.lpg == 1) expand_unit_mma<1>(p, sm, seq, m0, ct, lane, gw);
            else expand_unit<T, 1>(p, sm, seq, m0, ct, npub);
            break;
          case 2:
            if (kMmaExpand && Elem<T>::kDtype == CHAM_BF16 && m0.xm == 0 && m0.lpg == 1) expand_unit_mma<2>(p, sm, seq, m0, ct, lane, gw);
            else expand_unit<T, 2>(p, sm, seq, m0, ct, npub);
            break;
          case 3:
            if (kMmaExpand && Elem<T>::kDtype == CHAM_BF16 && m0.xm == 0 && m0.lpg == 1) expand_unit_mma<3>(p, sm, seq, m0, ct, lane, gw);
            else expand_unit<T, 3>(p, sm, seq, m0, ct, npub);
            break;
          default:
            if (kMmaExpand && Elem<T>::kDtype == CHAM_BF16 && m0.xm == 0 && m0.lpg == 1) expand_unit_mma<4>(p, sm, seq, m0, ct, lane, gw);
            else expand_unit<T, 4>(p, sm, seq, m0, ct, npub);
            break;
        }
      }
    }
  }
  // the last CTA re-arms the unit counters and the tile counters for the next launch
  if (tid == 0) trace_cta(p, 3);
  if (kZeroNext) {  // the next apply re-arms this parity's counters (after_wait)
    if (tid == 0) trace_cta(p, 4);
    return;
  }
  __syncthreads();
  if (tid == 0) {
    __threadfence();
    sm.last_cta = atomicAdd(p.ctr + 1, 1) == (int)gridDim.x - 1;
  }
  __syncthreads();
  if (sm.last_cta) {
    if (p.tile_ctr) {
      const int n = p.n_jobs * sm.plan.totals[1];
      for (int i = tid; i < n; i += APPLY_THREADS) p.tile_ctr[i] = 0;
    }
    {
      const int per = sm.plan.n_split * p.split_ncc;  // used slots of each job
      for (int i = tid; i < p.n_jobs * per; i += APPLY_THREADS)
        p.split_ctr[(i / per) * kSplitCap * p.split_ncc + i % per] = 0;
    }
    if (tid == 0) {
      p.ctr[0] = 0;
      p.ctr[4] = 0;
      p.ctr[1] = 0;
    }
    __threadfence();
  }
  if (tid == 0) trace_cta(p, 4);
}

// One CTA builds the step's plan and writes it to global memory (consumed by every
// lora_apply of the step through Params::plan).
__global__ void __launch_bounds__(NTHREADS, 1) build_plan_kernel(const __grid_constant__ Params p, Plan* out) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  Plan& pl = *reinterpret_cast<Plan*>(smem_raw);
  const int S = p.n_seg >= 0 ? p.n_seg : *p.n_seg_dev;
  bool ok = S >= 0 && S <= PLAN_SEGS;
  if (ok) ok = build_plan(p, pl, S, reinterpret_cast<UnitDesc*>(out + 1));
  if (threadIdx.x == 0) pl.desc_cap = p.desc_cap;
  __syncthreads();
  if (!ok) {
    if (threadIdx.x == 0) {
      *p.err = CHAM_ERR_LIMIT;
      out->totals[2] = 1 << 30;  // consumers of this plan will refuse it
    }
    return;
  }
  const int4* src = reinterpret_cast<const int4*>(&pl);
  int4* dst = reinterpret_cast<int4*>(out);
  for (int i = threadIdx.x; i < (int)(sizeof(Plan) / 16); i += NTHREADS) dst[i] = src[i];
}

template <typename T>
int launch(cham_pool* pool, Params& prm, int mode, cudaStream_t stream) {
  static bool attr_set[2] = {false, false};
  auto kern = lora_apply_kernel<T>;
  const int smem = sizeof(Shared);
  if (!attr_set[Elem<T>::kDtype]) {
    CHAM_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    attr_set[Elem<T>::kDtype] = true;
  }
  // ping-pong v workspace: apply n uses buffer n % 2 (see the ordering argument above)
  prm.vws_job_stride = (long long)pool->max_tokens * kMaxRank;
  prm.vws = pool->d_vws + (pool->apply_count & 1) * (size_t)kMaxJobs * prm.vws_job_stride;
  // counters ping-pong like the v buffer: apply n+1 may start (PDL) while apply n's last
  // CTA is still re-arming its own counter set
  prm.ctr = pool->d_ctr + 16 + (pool->apply_count & 1) * 16;
  prm.tile_ctr = mode == MODE_FUSED ? pool->d_ctr + kTileCtrBase + (pool->apply_count & 1) * (size_t)kMaxJobs *
                                                                      pool->max_tokens
                                    : nullptr;
  prm.split_buf = pool->d_split;
  prm.split_ncc = pool->split_ncc;
  prm.split_ctr = pool->d_split_ctr + (pool->apply_count & 1) * (size_t)kMaxJobs * kSplitCap * pool->split_ncc;
  prm.err = pool->d_ctr + 2;
  {
    const int o = (pool->apply_count + 1) & 1;  // the other parity: the previous apply's set
    prm.zero_ctr = pool->d_ctr + 16 + o * 16;
    prm.zero_tile = pool->d_ctr + kTileCtrBase + o * (size_t)kMaxJobs * pool->max_tokens;
    prm.zero_tile_n = (long long)kMaxJobs * pool->max_tokens;
    prm.zero_split = pool->d_split_ctr + o * (size_t)kMaxJobs * kSplitCap * pool->split_ncc;
    prm.zero_split_n = (long long)kMaxJobs * kSplitCap * pool->split_ncc;
  }
  ++pool->apply_count;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(pool->sm_count);
  cfg.blockDim = dim3(APPLY_THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  CHAM_CUDA(cudaLaunchKernelEx(&cfg, kern, prm, mode));
  return CHAM_OK;
}

}  // namespace decode

size_t plan_bytes(const cham_pool* pool) {
  return sizeof(decode::Plan) + sizeof(decode::UnitDesc) * (size_t)decode::plan_desc_capacity(pool->max_tokens);
}

int build_plan_entry(cham_pool* pool, const int* perm, const int* seg_off, const int* seg_slot,
                     const int* seg_rank, int n_seg, const int* n_seg_dev, void* plan, void* stream) {
  using namespace decode;
  if (!pool || !plan || !seg_off || !seg_slot || !seg_rank) return fail(CHAM_ERR_INVALID, "cham_build_plan: null argument");
  if (n_seg < 0 && !n_seg_dev) return fail(CHAM_ERR_INVALID, "cham_build_plan: n_seg < 0 needs n_seg_dev");
  if (n_seg > PLAN_SEGS) return fail(CHAM_ERR_LIMIT, "cham_build_plan: too many segments");
  if (reinterpret_cast<uintptr_t>(plan) & 15) return fail(CHAM_ERR_INVALID, "cham_build_plan: plan must be 16-byte aligned");
  Params prm{};
  prm.slot_pages = pool->d_slot_pages;
  prm.perm = perm;
  prm.seg_off = seg_off;
  prm.seg_slot = seg_slot;
  prm.seg_rank = seg_rank;
  prm.n_seg = n_seg;
  prm.n_seg_dev = n_seg_dev;
  prm.max_tokens = pool->max_tokens;
  prm.err = pool->d_ctr + 2;
  prm.desc_cap = plan_desc_capacity(pool->max_tokens);
  prm.prefill_thr = prefill_route_thr(pool);
  build_plan_kernel<<<1, NTHREADS, sizeof(Plan), (cudaStream_t)stream>>>(prm, static_cast<Plan*>(plan));
  CHAM_CUDA(cudaGetLastError());
  return CHAM_OK;
}

// Shared validation + parameter setup for the four entry points.
int decode_entry(cham_pool* pool, int layer, int n_jobs, const int* projs, const void* const* xs,
                 void* const* ys, int n_tokens, const int* perm, const int* seg_off, const int* seg_slot,
                 const int* seg_rank, int n_seg, const int* n_seg_dev, const void* plan, void* stream, int mode,
                 float* v_out, const float* v_in, int v_stride, int v_cols) {
  using namespace decode;
  if (!pool) return fail(CHAM_ERR_INVALID, "lora_apply: null pool");
  if (layer < 0 || layer >= pool->n_layers) return fail(CHAM_ERR_INVALID, "lora_apply: layer out of range");
  if (n_jobs <= 0 || n_jobs > kMaxJobs) return fail(CHAM_ERR_LIMIT, "lora_apply: 1..max_jobs projections per launch");
  if (n_seg == 0 || n_tokens == 0) return CHAM_OK;  // nothing to do (also for empty tensors)
  if (!seg_off || !seg_slot || !seg_rank) return fail(CHAM_ERR_INVALID, "lora_apply: null segment table");
  if (n_seg < 0 && !n_seg_dev) return fail(CHAM_ERR_INVALID, "lora_apply: n_seg < 0 needs n_seg_dev");
  if (n_seg > PLAN_SEGS) return fail(CHAM_ERR_LIMIT, "lora_apply: too many segments");
  if (n_tokens < 0 || n_tokens > pool->max_tokens)
    return fail(CHAM_ERR_LIMIT, "lora_apply: n_tokens exceeds the pool's max_tokens");
  if ((v_in || v_out) && (v_stride <= 0 || v_stride % 4))
    return fail(CHAM_ERR_INVALID, "lora_shrink/expand: v_stride must be a positive multiple of 4");
  if (v_cols <= 0) v_cols = v_stride;
  if ((v_in || v_out) && (v_cols % 4 || (long long)n_jobs * v_cols > v_stride))
    return fail(CHAM_ERR_INVALID, "lora_shrink/expand: v_cols must be a multiple of 4 with n_jobs * v_cols <= v_stride");
  Params prm{};
  prm.base = pool->base;
  prm.page_bytes = (long long)pool->page_bytes;
  prm.slot_pages = pool->d_slot_pages;
  const int p0 = projs[0];
  if (p0 < 0 || p0 >= pool->n_proj) return fail(CHAM_ERR_INVALID, "lora_apply: proj out of range");
  prm.h_in = pool->h_in[p0];
  prm.h_out = pool->h_out[p0];
  prm.n_jobs = n_jobs;
  for (int j = 0; j < n_jobs; ++j) {
    const int pj = projs[j];
    if (pj < 0 || pj >= pool->n_proj) return fail(CHAM_ERR_INVALID, "lora_apply: proj out of range");
    // shrink reads only h_in, expand only h_out; the fused apply needs both equal
    if ((mode != MODE_EXPAND && pool->h_in[pj] != prm.h_in) || (mode != MODE_SHRINK && pool->h_out[pj] != prm.h_out))
      return fail(CHAM_ERR_INVALID, "lora_apply_multi: projections must share h_in (shrink) / h_out (expand)");
    const int lp = layer * pool->n_proj + pj;
    if (mode != MODE_EXPAND && !xs[j]) return fail(CHAM_ERR_INVALID, "lora_apply: null x");
    if (mode != MODE_SHRINK && !ys[j]) return fail(CHAM_ERR_INVALID, "lora_apply: null y");
    if ((reinterpret_cast<uintptr_t>(xs[j]) | reinterpret_cast<uintptr_t>(ys[j])) & 15)
      return fail(CHAM_ERR_INVALID, "lora_apply: x and y must be 16-byte aligned");
    prm.jobs[j].x = static_cast<const char*>(xs[j]);
    prm.jobs[j].y = static_cast<char*>(ys[j]);
    prm.jobs[j].a_off = (long long)pool->a_off[lp];
    prm.jobs[j].b_off = (long long)pool->b_off[lp];
  }
  prm.perm = perm;
  prm.seg_off = seg_off;
  prm.seg_slot = seg_slot;
  prm.seg_rank = seg_rank;
  prm.n_seg = n_seg;
  prm.n_seg_dev = n_seg_dev;
  prm.max_tokens = pool->max_tokens;
  prm.v_out = mode == MODE_SHRINK ? v_out : nullptr;
  prm.v_in = mode == MODE_EXPAND ? v_in : nullptr;
  prm.v_stride = v_stride;
  prm.v_cols = v_cols;
  if (prm.v_in) {
    const int rc = encode_f32_map(&prm.vmap, v_in, n_tokens, v_stride, v_stride, kRowsPerPage, TG);
    if (rc) return rc;
  }
  prm.trace = pool->d_trace;
  prm.trace_cap = pool->trace_cap;
  prm.desc_cap = plan_desc_capacity(pool->max_tokens);
  if (!plan) {
    // no step-level plan: build one for this call into the pool's scratch plan
    int rc = build_plan_entry(pool, perm, seg_off, seg_slot, seg_rank, n_seg, n_seg_dev, pool->d_plan, stream);
    if (rc) return rc;
    plan = pool->d_plan;
  }
  prm.plan = plan;
  prm.prefill_thr = prefill_route_thr(pool);
  if (pool->next_n > 0 && pool->l2_prefetch_bytes > 0 && mode == MODE_FUSED) {
    prm.nx_jobs = pool->next_n;
    prm.nx_a_bytes = pool->next_a_bytes;
    prm.nx_items = (int)std::min<long long>(pool->l2_prefetch_bytes / pool->next_a_bytes, 1 << 30);
    for (int j = 0; j < pool->next_n; ++j) prm.nx_a_off[j] = (long long)pool->next_a_off[j];
  }
  pool->next_n = 0;  // one-shot
  const bool pre = prm.prefill_thr < (1 << 30) && n_tokens >= prm.prefill_thr;
  if (pre && mode != MODE_FUSED && n_jobs > 1) {
    // the prefill kernel's TP halves take one projection: one call per job on its v columns
    for (int j = 0; j < n_jobs; ++j) {
      const int rc = decode_entry(pool, layer, 1, projs + j, xs + j, ys + j, n_tokens, perm, seg_off, seg_slot,
                                  seg_rank, n_seg, n_seg_dev, plan, stream, mode, v_out ? v_out + j * v_cols : nullptr,
                                  v_in ? v_in + j * v_cols : nullptr, v_stride, v_cols);
      if (rc) return rc;
    }
    return CHAM_OK;
  }
  // with a host guarantee that every segment is prefill-sized, the decode kernel has no work
  const bool dec = !pre || pool->route_min_seg < prm.prefill_thr;
  int rc = CHAM_OK;
  if (dec) {
    rc = pool->dtype == CHAM_BF16 ? launch<__nv_bfloat16>(pool, prm, mode, (cudaStream_t)stream)
                                  : launch<float>(pool, prm, mode, (cudaStream_t)stream);
    if (rc) return rc;
  }
  if (pre)
    rc = prefill_launch(pool, layer, n_jobs, projs, xs, ys, n_tokens, perm, seg_off, seg_slot, seg_rank, n_seg,
                        n_seg_dev, stream, mode, v_out, v_in, v_stride);
  return rc;
}

}  // namespace cham
