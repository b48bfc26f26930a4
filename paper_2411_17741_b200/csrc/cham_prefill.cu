// cham_prefill.cu — K3: the tensor-core (tcgen05) path for prefill-sized segments.
//
// Reference seam: the prefill half of CostModel.step_duration's LoRA term (engine.py:67-77):
// a prefill contributes rank * input_tokens adapter units (engine.py:70, 75-76); this kernel
// performs that work for real, y[t] += (x[t] . A_slot) . B_slot, for every segment with at
// least `prefill_min_tokens` tokens (rank <= 128, bf16).
//
// ONE persistent, warp-specialised kernel per lora_apply (K3), one CTA per SM, 12
// warps: 0-7 epilogue (two sets of four, each set covering the 128 TMEM lanes), 8 publisher
// (probes both sets' queues; warp 9 is the second loader with CHAM_PF_LD2, else idle), 10 MMA
// issuer, 11 loader (TMA + dispatch; the highest warp id, so the schedulers favour it).  A tile
// is up to 128 token rows of one segment (UMMA M = 128).  The ring has two 48 KiB stages.
// Units come from one dynamic counter, phase-1 units first (shrink units in LPT order: tiles
// by rank, descending; K split <= 2):
//   shrink unit (tile, K range kq of ks, job group): D[128 x rp] (TMEM, fp32) = X . A^T over the
//        range, for every job of the group from ONE x stage (q/k/v share x, so x crosses
//        HBM->SM once per K range).  Stages carry kpc 64-column k-chunks: x by TMA tensor loads
//        of exactly the tile's rows (64-row boxes, or 1-row boxes when the rows are not
//        consecutive tokens), A^T page atoms by bulk copies straight from the pool layout
//        (K-major SWIZZLE_128B already).  With ks > 1 the epilogue writes the range's fp32
//        partial; the last of the ks arrivals (per tile and job group) sums the partials in K
//        order — deterministic, one bf16 rounding — into the tile's V image (bf16, K-major
//        SWIZZLE_128B: exactly the UMMA A-operand layout); with ks = 1 the image is written
//        directly.  The publisher releases the image (tile counter += 1).
//   expand unit (tile, job, CW = 256 columns): the loader waits for the tile's images, copies
//        the V image (one bulk copy, double-buffered), then streams the B page slices of the
//        unit's 64-column groups (MN-major SWIZZLE_128B — the pool layout again).  D2[128 x 64]
//        = V . B per group into one of two TMEM accumulators; the epilogue thread of token
//        row r loads its 128-byte y piece of the group into registers one group ahead, adds
//        D2 and stores it back — no separate elementwise kernel, no y in shared memory.
// Expand units wait only for their own tile, so the phases overlap across tiles.  Counters
// ping-pong by launch parity; each launch re-arms the previous launch's set after its
// griddepcontrol.wait (no last-CTA reset).  The path is
// HBM-bound (AI ~15 flop/B at C3): tensor cores are used because the CUDA-core FMA ceiling
// (~51-74 TFLOP/s) is below what the HBM roofline demands.
#include <cuda.h>
#include <cudaTypedefs.h>

#include "cham_pool.h"

namespace cham {
namespace prefill {

constexpr int BM = 128;                 // tokens per tile (UMMA M)
constexpr int MAXR = kPrefillMaxRank;   // rank rows per adapter on this path
#ifndef CHAM_PF_NS
#define CHAM_PF_NS 2  // ring stages x bytes: A/B on C3 (tok/s): 4 x 32K 630k, 3 x 32K 651k, 2 x 64K 656k, 2 x 48K 677k
#endif
#ifndef CHAM_PF_VBUF
#define CHAM_PF_VBUF (2 * 128 * 128)
#endif
constexpr int NS = CHAM_PF_NS;          // ring stages
#ifndef CHAM_PF_LD2
#define CHAM_PF_LD2 0  // 1: two loader warps in the expand phase (alternate unit positions; the second publisher warp loads); A/B on C3: 709k vs 763k — the epilogue (y RMW, ~1.7 us per group per set) then limits, and the 64 KiB stages it needs cost 3%
#endif
constexpr bool kLd2 = CHAM_PF_LD2 != 0;
#ifndef CHAM_PF_PUB1
#define CHAM_PF_PUB1 1  // one publisher warp probes both epilogue sets' queues (test_wait); 0: one warp per set
#endif
constexpr bool kPub1 = CHAM_PF_PUB1 != 0;
#ifndef CHAM_PF_STAGE
// two big stages: shrink stages carry 2-3 K-chunks (A copies of 2-3 KiB, not 1 KiB); with two
// loaders every expand unit must fit one stage (4 groups x 16 KiB of B at rank 128)
#define CHAM_PF_STAGE (CHAM_PF_LD2 ? 65536 : 49152)
#endif
constexpr int STAGE = CHAM_PF_STAGE;    // bytes per ring stage
constexpr int VPAD = BM * 128 - 4096;   // worst over-read past a V buffer: 16 KiB - the smallest x block
constexpr int VBUF = CHAM_PF_VBUF;      // V images of one (job, tile): ks partials x K-blocks x mp rows x 128 B
#ifndef CHAM_PF_PDL
#define CHAM_PF_PDL 1  // programmatic dependent launch for the prefill kernel
#endif
#ifndef CHAM_PF_YREG
#define CHAM_PF_YREG 1  // expand y path: 1 = epilogue registers (ld/st.global, ring stages carry B only), 0 = y rows staged in the ring
#endif
constexpr bool kYReg = CHAM_PF_YREG != 0;
#ifndef CHAM_PF_YPF
#define CHAM_PF_YPF 1  // register y path: L2 prefetch of the set's later groups at unit start
#endif
constexpr bool kYPrefetch = CHAM_PF_YPF != 0;
#ifndef CHAM_PF_CW
#define CHAM_PF_CW 256  // expand unit width; A/B on C3: 256 -> 642k, 512 -> 625k, 1024 -> 553k tok/s
#endif
constexpr int CW = CHAM_PF_CW;          // expand unit columns
constexpr int NGRP = CW / 64;           // 64-column MMA groups per expand unit
#ifndef CHAM_PF_UQ
#define CHAM_PF_UQ 8
#endif
constexpr int UQ = CHAM_PF_UQ;          // unit-id ring depth
#ifndef CHAM_PF_ZATOM
#define CHAM_PF_ZATOM 1  // odd page counts read their K padding from one zero atom (the last K step's stride points at it); 0: the loader zero-fills a pad atom per stage (A/B on C3: 775.9k vs 774.0k tok/s)
#endif
constexpr bool kZeroAtom = CHAM_PF_ZATOM != 0;
#ifndef CHAM_PF_ZERO_NEXT
#define CHAM_PF_ZERO_NEXT 1  // counters re-armed by the next launch after its griddepcontrol.wait
#endif
constexpr bool kPfZeroNext = CHAM_PF_ZERO_NEXT != 0;
#ifndef CHAM_PF_KS_MAX
#define CHAM_PF_KS_MAX 2  // largest shrink K-split; A/B on C3 with 2 x 48K stages: 8 677k, 2 744k, 1 663k tok/s
#endif
#ifndef CHAM_PF_KS_WAVES
#define CHAM_PF_KS_WAVES 2  // shrink K-split: grow until the phase-1 units fill this many waves
#endif
#ifndef CHAM_PF_CD
#define CHAM_PF_CD 1  // outstanding unit claims per loader (A/B on C3: 1 -> 590k, 4 -> 347k tok/s: early claims of expand units block on unready tiles)
#endif
constexpr int CD = CHAM_PF_CD;
#ifndef CHAM_PF_EXSTATIC
#define CHAM_PF_EXSTATIC 0  // 1: expand units assigned statically, round-robin (A/B on C3: 539k vs 634k tok/s dynamic)
#endif
constexpr bool kExStatic = CHAM_PF_EXSTATIC != 0;
constexpr int MAX_TILES = kPrefillMaxTiles;
constexpr int NTHREADS = 384;           // warps 0-7 epilogue (two sets of 4), 8-9 publishers, 10 MMA, 11 loader
// The loader is the highest-numbered warp (the warp schedulers favour higher warp ids, so the
// serial dispatch + copy-issue chain is not starved by the ALU-heavy epilogue warps).
#ifndef CHAM_PF_LOADER_HI
#define CHAM_PF_LOADER_HI 1  // 0: the round-1 numbering (loader 8, MMA 9, publishers 10-11)
#endif
constexpr int W_LOAD = CHAM_PF_LOADER_HI ? 11 : 8, W_MMA = CHAM_PF_LOADER_HI ? 10 : 9,
              W_PUB = CHAM_PF_LOADER_HI ? 8 : 10;
constexpr int W_LOAD2 = W_PUB + 1;  // kLd2: the second loader (one publisher serves both sets)
constexpr int kUnitLoaderDone = -2;  // kLd2: a loader ran out of units (its later positions are skipped)
constexpr int PQN = 8;                  // publish ring depth per epilogue set
constexpr int TMEM_COLS = 512;
// TMEM: two shrink accumulators of TM_SH columns, then NACC expand accumulators of 64 columns
// (2 x 128 + 2 x 64: one expand group per epilogue set in flight between the MMA warp and
// the epilogue; four measured 0.6% slower)
#ifndef CHAM_PF_NACC
#define CHAM_PF_NACC 2  // expand accumulators; A/B on C3 (register y path): 2 -> 762k, 4 -> 757k, 6 (TM_SH 64) -> 743k
#endif
#ifndef CHAM_PF_TMSH
#define CHAM_PF_TMSH (CHAM_PF_YREG ? 128 : 192)
#endif
constexpr int NACC = CHAM_PF_NACC;
constexpr int TM_SH = CHAM_PF_TMSH;
constexpr int TM_EX = 2 * TM_SH;
static_assert(TM_EX + NACC * 64 <= TMEM_COLS, "TMEM budget");
constexpr int BAR_EPI = 1;              // named barriers 1, 2: the 128 threads of epilogue set 0, 1

enum Mode { MODE_FUSED = 0, MODE_SHRINK = 1, MODE_EXPAND = 2 };

struct Job {
  const char* x;
  char* y;
  long long a_off;
  long long b_off;
};

// Activation tensor maps of one job: a 64-column x 64-row box for contiguous rows and a
// 64-column x 1-row box for gathered ones, both SWIZZLE_128B (x for shrink, y for expand).
struct alignas(64) Maps {
  CUtensorMap x64, x1, y64, y1, y32;  // y32: 32-row boxes of the standalone expand kernel
};

struct alignas(64) Params {
  Maps maps[kMaxJobs];
  Job jobs[kMaxJobs];
  const char* base;
  long long page_bytes;
  const int* slot_pages;
  int h_in, h_out;
  int n_jobs;
  int mode;
  int no_expand;           // MODE_FUSED without expand units: V images only (expand_kernel follows)
  int x_shared;            // every job reads the same x (q/k/v): one x stage serves the group
  const int* perm;
  const int* seg_off;
  const int* seg_slot;
  const int* seg_rank;
  int n_seg;
  const int* n_seg_dev;
  int thr;                 // routing threshold (segment tokens)
  int epoch;               // launch id (tile V flags), parity selects the counter set
  int* ctr;                // this parity's counters: [0] dispatch, [1] finished CTAs, [2] error
  int* tile_cnt;           // this parity's tile counters [MAX_TILES]: reduced V images published
  int* arrive;             // this parity's split-K arrival counters [MAX_TILES][kMaxJobs] (tile, job group)
  float* ppart;            // fp32 split-K partials [job][tile][kPrefillPart / 4]
  int* err;
  int* zero_set;           // CHAM_PF_ZERO_NEXT: the other parity's counter set (the previous launch's)
  int zero_n;
  char* vimg;              // V images [job][tile][VBUF]
  float* v_out;            // MODE_SHRINK: v [position][v_stride]
  const float* v_in;       // MODE_EXPAND: v [position][v_stride]
  int v_stride;
  int n_pages, n_tokens;   // pool pages, activation rows (bounds checks of CHAM_PF_CHECK builds)
  unsigned long long* trace;  // debug timeline [cta][unit k][8] (null = off)
  int trace_cap;
};

// ------------------------------------------------------------------ PTX wrappers (tcgen05)
__device__ __forceinline__ uint32_t idesc_bf16(int M, int N, bool b_mn_major) {
  // kind::f16 instruction descriptor: D fp32, A/B bf16, A K-major, B K- or MN-major
  return (1u << 4) | (1u << 7) | (1u << 10) | ((b_mn_major ? 1u : 0u) << 16) |
         ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
// SWIZZLE_128B shared-memory matrix descriptor (sm_100 version 1)
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr & 0x3FFFFu) >> 4) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46) | (2ull << 61);
}
__device__ __forceinline__ void mma_bf16(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tmem_alloc(uint32_t* dst) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst)),
               "n"(TMEM_COLS));
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "n"(TMEM_COLS));
}
// 32 lanes x 32 consecutive fp32 columns: thread `lane` of the warp gets row (lane base + lane)
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float (&v)[32]) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}
// two 32-column loads, one wait
__device__ __forceinline__ void tmem_ld32x2(uint32_t taddr, float (&v0)[32], float (&v1)[32]) {
  uint32_t r[64];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[32]), "=r"(r[33]), "=r"(r[34]), "=r"(r[35]), "=r"(r[36]), "=r"(r[37]), "=r"(r[38]), "=r"(r[39]),
        "=r"(r[40]), "=r"(r[41]), "=r"(r[42]), "=r"(r[43]), "=r"(r[44]), "=r"(r[45]), "=r"(r[46]), "=r"(r[47]),
        "=r"(r[48]), "=r"(r[49]), "=r"(r[50]), "=r"(r[51]), "=r"(r[52]), "=r"(r[53]), "=r"(r[54]), "=r"(r[55]),
        "=r"(r[56]), "=r"(r[57]), "=r"(r[58]), "=r"(r[59]), "=r"(r[60]), "=r"(r[61]), "=r"(r[62]), "=r"(r[63])
      : "r"(taddr + 32));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) {
    v0[i] = __uint_as_float(r[i]);
    v1[i] = __uint_as_float(r[32 + i]);
  }
}
// 2-D TMA tensor load (box defined by the map) completing on an mbarrier
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar,
                                            uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint "
      "[%0], [%1, {%2, %3}], [%4], %5;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}
// the same without an L2 cache hint
__device__ __forceinline__ void tma_load_2d_nohint(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes "
      "[%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}
// 2-D TMA tensor store smem -> global (bulk async-group of the issuing thread)
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, int c0, int c1, const void* src) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(c0), "r"(c1), "r"(smem_u32(src))
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void prefetch_map(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}
__device__ __forceinline__ uint32_t swz(int row, int chunk) {  // 16-byte chunk of a 128-byte row
  return (uint32_t)(row * 128 + (((chunk ^ row) & 7) << 4));
}
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
// debug timeline: field 0 loader claim, 1 loader issued, 2 MMA first stage ready, 3 MMA
// issued, 4 epilogue accumulators ready, 5 epilogue end, 6 unit id | kind << 32, 7 loader
// got the unit's first ring slot
__device__ __forceinline__ void trace_put(const Params& p, int k, int field, unsigned long long v) {
  if (p.trace && k < p.trace_cap) p.trace[((long long)blockIdx.x * p.trace_cap + k) * 8 + field] = v;
}
// loader detail timeline (debug): the first half of the debug buffer (the decode kernel's,
// unused while a prefill-only chain runs): 0 unit ring slot free, 1 next unit id known, 2 V
// buffer free, 3 tile ready, 4 V copy issued, 5 first ring stage free
__device__ __forceinline__ void trace_ld(const Params& p, int k, int field) {
  if (p.trace && k < p.trace_cap)
    p.trace[(((long long)blockIdx.x - (long long)gridDim.x) * p.trace_cap + k) * 8 + field] = gtimer();
}
// debug breadcrumbs of the CTA's own progress (trace builds only): slot trace_cap - 1,
// written by thread 0 and pushed to memory at system scope (the trace may be host-mapped)
__device__ __forceinline__ void crumb(const Params& p, int field, unsigned long long v) {
  if (p.trace && threadIdx.x == 0) {
    p.trace[((long long)blockIdx.x * p.trace_cap + p.trace_cap - 1) * 8 + field] = v;
    __threadfence_system();
  }
}
#ifndef CHAM_PF_MMA_SYNC
#define CHAM_PF_MMA_SYNC 0  // 1: the MMA warp waits for each shrink stage's MMAs (fault-hunt experiment)
#endif
#ifndef CHAM_PF_LATE_ALLOC
#define CHAM_PF_LATE_ALLOC 0  // 1: tcgen05.alloc after griddepcontrol.wait (fault-hunt experiment)
#endif
#ifndef CHAM_PF_XPOL_NORMAL
#define CHAM_PF_XPOL_NORMAL 1  // x load L2 policy: 0 evict_last, 1 evict_normal (default), 2 evict_first, 3 no hint.
// evict_last faulted the context ("unspecified launch failure") in nearly every run when
// another kernel had just rewritten x (dirty L2 lines) and the launches were PDL-chained;
// 0 faults in 30 runs with any of 1-3 (scripts/fault_repro.py kb/e2e)
#endif
#ifndef CHAM_PF_NOPFMAP
#define CHAM_PF_NOPFMAP 0  // fault-hunt experiment: 1 skips prefetch.tensormap
#endif
#ifndef CHAM_PF_PROXYFENCE
#define CHAM_PF_PROXYFENCE 0  // fault-hunt experiment: 1 adds fence.proxy.async.global after griddepcontrol.wait
#endif
#ifndef CHAM_PF_NOACQ
#define CHAM_PF_NOACQ 0  // fault-hunt experiment: 1 drops the acquire fence after a satisfied peek
#endif
#ifndef CHAM_PF_DRAIN
#define CHAM_PF_DRAIN 1  // drain the MMA warp's commit arrivals before the CTA exits
#endif
constexpr bool kDrain = CHAM_PF_DRAIN != 0;
// debug breadcrumb of the MMA warp's progress inside a shrink unit (trace builds with
// CHAM_PF_WATCHDOG): slot trace_cap - 15 = {unit k, stage, seq, state, time}
__device__ __forceinline__ void mma_mark(const Params& p, int k, int s, int seq, int state);
#ifndef CHAM_PF_WATCHDOG
#define CHAM_PF_WATCHDOG 0  // debug builds: report mbarrier waits longer than 30 us into the trace
#endif
// Debug builds (CHAM_PF_WATCHDOG, trace on): a wait that is not satisfied after 30 us writes,
// once per warp, the barrier's raw state and the waiter into trace slot cap-2-warp, then keeps
// waiting.  Otherwise a plain mbarrier wait.
__device__ __forceinline__ void pf_wait(const Params& p, uint64_t* bar, uint32_t parity, int tag, int a, int b) {
  // CHAM_PF_WATCHDOG 2: watch only the stage-full waits (tags 9, 11, 15), the others plain
  if (!CHAM_PF_WATCHDOG || !p.trace || (CHAM_PF_WATCHDOG == 2 && tag != 9 && tag != 11 && tag != 15)) {
    mbar_wait(bar, parity);
    return;
  }
  const unsigned long long t0 = gtimer();
  bool rep = false;
  while (!mbar_try_wait(bar, parity)) {
    if (!rep && (threadIdx.x & 31) == 0 && gtimer() - t0 > 30000ull) {
      rep = true;
      unsigned long long raw;
      asm volatile("ld.shared.b64 %0, [%1];" : "=l"(raw) : "r"(smem_u32(bar)) : "memory");
      unsigned long long* d =
          p.trace + ((long long)blockIdx.x * p.trace_cap + p.trace_cap - 2 - (threadIdx.x >> 5)) * 8;
      d[1] = raw;
      d[2] = parity;
      d[3] = (unsigned long long)(smem_u32(bar));
      d[4] = (unsigned long long)(unsigned)a;
      d[5] = (unsigned long long)(unsigned)b;
      d[6] = gtimer();
      d[7] = (unsigned long long)p.epoch;
      d[0] = (unsigned long long)(tag + 1);
      __threadfence_system();
    }
  }
}
__device__ __forceinline__ void mma_mark(const Params& p, int k, int s, int seq, int state) {
  if (CHAM_PF_WATCHDOG && p.trace && (threadIdx.x & 31) == 0) {
    unsigned long long* d = p.trace + ((long long)blockIdx.x * p.trace_cap + p.trace_cap - 15) * 8;
    d[0] = k;
    d[1] = s;
    d[2] = seq;
    d[3] = state;
    d[4] = gtimer();
    d[5] = p.epoch;
    __threadfence_system();
  }
}
__device__ __forceinline__ void mbar_arrive_cnt(uint64_t* bar, uint32_t n) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(n) : "memory");
}
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

__device__ __forceinline__ void x_load(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar, uint64_t pol) {
  if (CHAM_PF_XPOL_NORMAL == 3) tma_load_2d_nohint(dst, map, c0, c1, bar);
  else tma_load_2d(dst, map, c0, c1, bar, pol);
}

// ------------------------------------------------------------------ tiles and units
struct Tile {
  int pos0;  // first position (perm order) of the tile's rows
  int m;     // rows (<= 128)
  int slot;
  int rank;
  int ks;    // shrink K-split of this tile (its ks partial V images must fit one V buffer)
};
struct TileList {
  int n_tiles;
  int ks;           // shrink K-split factor
  int u1;           // phase-1 units
  int u_total;
  int ncc, ept;     // expand: column chunks per (tile, job); units per tile (n_jobs x ncc)
  float inv_ncc, inv_ept;  // their reciprocals (fast division on the loader's path)
  int sh_start[MAX_TILES + 1];  // phase-1 unit prefix over the LPT order
  int ord[MAX_TILES];            // LPT order of the phase-1 units: position -> tile (rank descending)
  Tile t[MAX_TILES];
};

__host__ __device__ __forceinline__ int rpad(int rank) { return (rank + 15) & ~15; }
__host__ __device__ __forceinline__ int mpad(int m) { return (m + 63) & ~63; }  // 64-row TMA boxes
// jobs sharing one shrink stage: all of them when their A^T atoms fit a 16 KiB region
__device__ __forceinline__ int jobs_per_group(const Params& p, int rank) {
  return (p.mode == MODE_FUSED && p.x_shared && p.n_jobs * (rpad(rank) / 8) <= 16 && p.n_jobs * rpad(rank) <= TM_SH)
             ? p.n_jobs : 1;
}
// job groups of a tile (jobs_per_group is n_jobs or 1): no integer division on the loader's path
__device__ __forceinline__ int n_groups(const Params& p, int rank) { return jobs_per_group(p, rank) == 1 ? p.n_jobs : 1; }

// Warp 0 of every CTA builds the same tile list (deterministic): prefill segments in table
// order, each cut into 128-row tiles; phase-1 unit prefix per tile.  Returns false on overflow.
__device__ bool build_tiles(const Params& p, TileList& tl, int grid) {
  const int lane = threadIdx.x & 31;
  int S = p.n_seg >= 0 ? p.n_seg : *p.n_seg_dev;
  S = max(0, min(S, kMaxSegments));
  int tiles = 0;
  bool ok = true;
  for (int base = 0; base < S; base += 32) {
    const int s = base + lane;
    int o0 = 0, T = 0, slot = -1, rank = 0;
    if (s < S) {
      o0 = __ldg(p.seg_off + s);
      T = __ldg(p.seg_off + s + 1) - o0;
      slot = __ldg(p.seg_slot + s);
      rank = __ldg(p.seg_rank + s);
    }
    const bool f = s < S && slot >= 0 && is_prefill_segment(T, rank, p.thr);
    const int nt = f ? (T + BM - 1) / BM : 0;
    int inc = nt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int a = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += a;
    }
    const int first = tiles + inc - nt;
    if (first + nt > MAX_TILES) ok = false;
    else
      for (int i = 0; i < nt; ++i) {
        Tile t;
        t.pos0 = o0 + i * BM;
        t.m = min(BM, T - i * BM);
        t.slot = slot;
        t.rank = rank;
        tl.t[first + i] = t;
      }
    tiles += __shfl_sync(0xffffffffu, inc, 31);
  }
  ok = __all_sync(0xffffffffu, ok);
  if (!ok) return false;
  // K-split: about two phase-1 units per CTA, K loops of >= 8 chunks
  const int nkc = p.h_in / 64;
  int groups = 0;
  for (int t = lane; t < tiles; t += 32) groups += n_groups(p, tl.t[t].rank);
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) groups += __shfl_xor_sync(0xffffffffu, groups, o);
  int ks = 1;
  if (p.mode == MODE_FUSED)
    while (ks < CHAM_PF_KS_MAX && groups * ks < CHAM_PF_KS_WAVES * grid && nkc % (2 * ks) == 0 && nkc / (2 * ks) >= 8)
      ks *= 2;
  // LPT order of the phase-1 units: tiles by padded rank, descending (stable) — the long
  // K loops of the large-rank tiles start first instead of forming the launch's tail
  {
    int pos = 0;
    for (int b = MAXR / 16; b >= 1; --b)
      for (int base = 0; base < tiles; base += 32) {
        const int t = base + lane;
        const bool f = t < tiles && rpad(tl.t[t].rank) / 16 == b;
        const unsigned m = __ballot_sync(0xffffffffu, f);
        if (f) tl.ord[pos + __popc(m & ((1u << lane) - 1))] = t;
        pos += __popc(m);
      }
    __syncwarp();
  }
  // phase-1 unit prefix over the LPT order (vbuild units in MODE_EXPAND: one per tile)
  int carry = 0;
  for (int base = 0; base < tiles; base += 32) {
    const int k = base + lane;
    int u = 0;
    if (k < tiles) {
      const int t = tl.ord[k];
      int kt = ks;
      const int part = mpad(tl.t[t].m) * rpad(tl.t[t].rank) * 4;  // one K range's fp32 partial
      while (kt > 1 && kt * part > (int)kPrefillPart) kt >>= 1;
      tl.t[t].ks = kt;
      u = p.mode == MODE_EXPAND ? 1 : kt * n_groups(p, tl.t[t].rank);
    }
    int inc = u;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int a = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += a;
    }
    if (k < tiles) tl.sh_start[k] = carry + inc - u;
    carry += __shfl_sync(0xffffffffu, inc, 31);
  }
  if (lane == 0) {
    tl.n_tiles = tiles;
    tl.ks = ks;
    tl.sh_start[tiles] = carry;
    tl.u1 = carry;
    const int ncc = (p.h_out + CW - 1) / CW;
    tl.u_total = carry + ((p.mode == MODE_SHRINK || p.no_expand) ? 0 : tiles * p.n_jobs * ncc);
    tl.ncc = ncc;
    tl.ept = p.n_jobs * ncc;
    tl.inv_ncc = 1.0f / (float)ncc;
    tl.inv_ept = 1.0f / (float)tl.ept;
  }
  return true;
}

// n / d for 0 <= n < 2^22 by the reciprocal (one correction step: the float quotient is off
// by at most one there); replaces the ~30-instruction integer division on the loader's
// per-unit path.  Unit counts stay far below 2^22; the tile peek of an exhausted claim
// (n ~ 2^29) gets a quotient within a few units of the true one, which the caller clamps.
__device__ __forceinline__ int fdiv(int n, int d, float inv) {
  int q = __float2int_rz(__int2float_rn(n) * inv);
  const int r = n - q * d;
  q += r >= d ? 1 : r < 0 ? -1 : 0;
  return q;
}

__device__ __forceinline__ int tile_of_unit(const TileList& tl, int u) {
  int lo = 0, hi = tl.n_tiles;
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (tl.sh_start[mid] <= u) lo = mid; else hi = mid;
  }
  return lo;
}

// Everything every role derives from a unit id.
struct Unit {
  int kind;    // 1 shrink, 2 expand, 3 vbuild (MODE_EXPAND phase 1)
  int tile, pos0, m, mp, slot, rank, rp, np;
  int kq, job0, jps;  // shrink: K range, first job, jobs in the group
  int job, col0;      // expand
  int ngrp;           // expand: 64-column groups in the unit
  int kpc, nst;       // chunks (shrink) / groups (expand) per stage, stages
  int nchunks;        // shrink: k-chunks in the unit
  int ks;             // the tile's shrink K-split (fp32 partials reduced into ONE V image)
  int vstride;        // bytes of the tile's V image (K-blocks x mp rows x 128 B)
  int xb;             // bytes of one activation chunk/group in smem (mp rows x 128 B)
  int bstride;        // expand: bytes of one group's B slices (np rounded up to even, x 1 KiB)
};

__device__ __forceinline__ Unit make_unit(const Params& p, const TileList& tl, int u) {
  Unit x;
  int k = 0;  // LPT position of a phase-1 unit's tile
  if (u < tl.u1) {
    k = tile_of_unit(tl, u);
    x.tile = tl.ord[k];
    x.kind = p.mode == MODE_EXPAND ? 3 : 1;
  } else {
    const int ncc = tl.ncc;
    const int r = u - tl.u1;
    x.tile = fdiv(r, tl.ept, tl.inv_ept);
    const int jc = r - x.tile * tl.ept;
    x.job = fdiv(jc, ncc, tl.inv_ncc);
    x.col0 = (jc - x.job * ncc) * CW;
    x.kind = 2;
  }
  const Tile& t = tl.t[x.tile];
  x.pos0 = t.pos0;
  x.m = t.m;
  x.mp = mpad(t.m);
  x.slot = t.slot;
  x.rank = t.rank;
  x.rp = rpad(t.rank);
  x.np = (t.rank + 7) / 8;
  x.xb = x.mp * 128;
  x.bstride = (x.rp / 8) * kAtomBytes;
  x.ks = t.ks;
  x.vstride = ((x.rp + 63) / 64) * x.xb;
  if (x.kind == 1) {
    const int rem = u - tl.sh_start[k];
    const int lks = __ffs(t.ks) - 1;  // ks is a power of two
    x.kq = rem & (t.ks - 1);
    x.jps = jobs_per_group(p, t.rank);
    x.job0 = (rem >> lks) * x.jps;
    x.nchunks = (p.h_in / 64) >> lks;
    const int chunk_bytes = x.xb + x.jps * (x.rp / 8) * kAtomBytes;
    x.kpc = max(1, min(4, min(STAGE / chunk_bytes, x.nchunks)));
    x.nst = (x.nchunks + x.kpc - 1) / x.kpc;
  } else if (x.kind == 2) {
    x.ngrp = min(NGRP, (p.h_out - x.col0) / 64);
    x.kpc = kYReg ? max(1, min(NGRP, STAGE / x.bstride)) : max(1, min(4, STAGE / (x.bstride + x.xb)));
    x.nst = (x.ngrp + x.kpc - 1) / x.kpc;
  } else {
    x.kpc = 0;
    x.nst = 0;
  }
  return x;
}

// Token rows of one 32-row block of a tile as seen by a loader lane: the block is contiguous
// when its rows are consecutive tokens (one TMA box), else each lane loads its own row.
// Per-unit global reads of the loader (token rows of the tile, adapter page ids), issued one
// unit ahead so their L2 round trip overlaps the current unit's copies.
struct Prefetch {
  int rows[4];  // lane l: row of tile position 32 b + l (clamped to the last row)
  int page;     // lane l < np: pool page l of the adapter
};
__device__ __forceinline__ Prefetch prefetch_unit(const Params& p, const TileList& tl, int u_id, int lane) {
  // Every load is unconditional (clamped to a valid unit): the values are consumed one unit
  // later, and a predicated load merged with a default would make the loader wait for it now.
  Prefetch f;
  if (tl.u_total == 0) {  // no prefill work in this apply
    f.page = 0;
#pragma unroll
    for (int b = 0; b < 4; ++b) f.rows[b] = 0;
    return f;
  }
  const bool ok = u_id >= 0 && u_id < tl.u_total;
  const int uu = ok ? u_id : 0;
  const int ti = uu < tl.u1 ? tl.ord[tile_of_unit(tl, uu)] : fdiv(uu - tl.u1, tl.ept, tl.inv_ept);
  const Tile& t = tl.t[ti];
  f.page = __ldg(p.slot_pages + t.slot * kMaxPagesPerSlot + min(lane, kMaxPagesPerSlot - 1));
#pragma unroll
  for (int b = 0; b < 4; ++b) {
    const int pos = t.pos0 + min(b * 32 + lane, t.m - 1);
    f.rows[b] = __ldg(p.perm + pos);  // perm is never null (identity rows from the pool)
  }
  return f;
}
#ifndef CHAM_WARM_L2
#define CHAM_WARM_L2 0  // A/B on C3: 461.7k (on) vs 520.8k tok/s (off)
#endif
constexpr bool kWarmL2 = CHAM_WARM_L2 != 0;
#ifndef CHAM_PF_WARM_Y
#define CHAM_PF_WARM_Y 0  // 1: (A/B on C3: 592k vs 635k tok/s off) the loader pulls an expand unit's y rows into L2 when it claims the unit
#endif
constexpr bool kWarmY = CHAM_PF_WARM_Y != 0 && CHAM_PF_YREG != 0;
#ifndef CHAM_EXP_NOEPI
#define CHAM_EXP_NOEPI 0  // experiment builds only: 1 the expand epilogue skips the y update (stores), 2 also
                          // the y loads, 3 also the accumulator reads (released unread)
#endif
constexpr bool kNoEpi = CHAM_EXP_NOEPI != 0;
#ifndef CHAM_PF_CHECK
#define CHAM_PF_CHECK 0  // debug builds: bounds-check every copy the loader issues, trap with a report
#endif
#define PF_CHECK(cond, code, a, b)                                                                          \
  do {                                                                                                    \
    if (CHAM_PF_CHECK && !(cond)) {                                                                       \
      printf("PF_CHECK %d failed: cta %d warp %d lane %d a=%lld b=%lld\n", (code), (int)blockIdx.x,     \
             (int)(threadIdx.x >> 5), (int)(threadIdx.x & 31), (long long)(a), (long long)(b));           \
      __trap();                                                                                           \
    }                                                                                                     \
  } while (0)
// Warm L2 with a unit's operands as long contiguous runs (one x/y row range per token, one
// run of atoms per adapter page): the TMA box loads then move 128-byte row pieces out of L2
// instead of scattering 128-byte requests over DRAM pages.
__device__ __forceinline__ void warm_l2(const Params& p, const Unit& u, const Prefetch& f, int lane) {
  if (u.kind == 1) {
    const int kc0 = u.kq * u.nchunks;
#pragma unroll
    for (int b = 0; b < 4; ++b)
      if (b * 32 + lane < u.m)
        bulk_prefetch_l2(p.jobs[u.job0].x + ((long long)f.rows[b] * p.h_in + kc0 * 64) * 2, u.nchunks * 128);
    if (lane < u.np)
      for (int j = 0; j < u.jps; ++j)
        bulk_prefetch_l2(p.base + (long long)f.page * p.page_bytes + p.jobs[u.job0 + j].a_off + (long long)kc0 * kAtomBytes,
                         u.nchunks * kAtomBytes);
  } else if (u.kind == 2) {
#pragma unroll
    for (int b = 0; b < 4; ++b)
      if (b * 32 + lane < u.m)
        bulk_prefetch_l2(p.jobs[u.job].y + ((long long)f.rows[b] * p.h_out + u.col0) * 2, u.ngrp * 128);
    if (lane < u.np)
      bulk_prefetch_l2(p.base + (long long)f.page * p.page_bytes + p.jobs[u.job].b_off + (long long)(u.col0 / 64) * kAtomBytes,
                       u.ngrp * kAtomBytes);
  }
}

// 64-row block h of the tile: one TMA box when its (up to) 64 valid rows are consecutive tokens
__device__ __forceinline__ bool block64(const bool (&contig)[4], const int (&rows)[4], int nblk, int h) {
  bool ok = contig[2 * h];
  if (2 * h + 1 < nblk)
    ok = ok && contig[2 * h + 1] &&
         __shfl_sync(0xffffffffu, rows[2 * h + 1], 0) == __shfl_sync(0xffffffffu, rows[2 * h], 0) + 32;
  return ok;
}

// Token row of block `blk` for this lane; `contig` = the block's rows are consecutive tokens
// (one TMA box), else each lane moves its own row.
__device__ __forceinline__ int block_row(const Prefetch& f, const Unit& u, int blk, int lane, bool& contig) {
  const int r = blk * 32 + lane;
  const int row = f.rows[blk];
  const int first = __shfl_sync(0xffffffffu, row, 0);
  contig = __all_sync(0xffffffffu, r >= u.m || row == first + lane);
  return row;
}

// ------------------------------------------------------------------ shared memory
struct Shared {
  alignas(1024) unsigned char ring[NS][STAGE];
  // The UMMA A operand always spans 128 rows: the rows past a partial image's mp rows are
  // read (and ignored) from whatever follows it.  Each V buffer has its own pad so that read
  // never overlaps the other buffer, which the loader may be filling (TMA) at the same time.
  alignas(1024) unsigned char vbuf[2][VBUF + VPAD];
  alignas(1024) unsigned char zero_atom[kZeroAtom ? kAtomBytes : 16];  // above every ring stage
  uint64_t full[NS], empty[NS];
  uint64_t tfull_sh[2], tempty_sh[2], tfull_ex[NACC], tempty_ex[NACC];
  uint64_t vfull[2], vempty[2];
  uint64_t drain;  // the MMA warp's last commit: every earlier commit arrival has landed
  uint64_t ho_bar;  // kLd2: loader 0 hands the odd expand positions to loader 1
  int ho_k0, ho_seq0, ho_nex0, ho_ok;
  uint64_t ufull[UQ], uempty[UQ];
  int uslot[UQ];
  uint32_t tmem_base;
  int last[2];
  int flag;
  int last_arr[2];  // epilogue set es: its shrink unit was the tile group's last split-K arrival
  // epilogue set es -> publisher warp W_PUB + es: finished shrink units / V images
  int pq_tile[2][PQN];
  int pq_kind[2][PQN];  // 0 end, 1 split-K partials written (count, last one reduces), 2 V written
  uint64_t pq_full[2][PQN], pq_empty[2][PQN];
  TileList tl;
};

static_assert(sizeof(Shared) <= 227 * 1024, "prefill kernel shared memory exceeds the 227 KiB per-CTA limit");

// V image of (job, tile): K-block b (64 ranks) of row r, 16-byte chunk c at
// b * mp*128 + r*128 + ((c ^ r) & 7) * 16 — the K-major SWIZZLE_128B A-operand layout.
__device__ __forceinline__ char* vimg_of(const Params& p, int job, int tile) {
  return p.vimg + ((long long)job * MAX_TILES + tile) * VBUF;
}
// fp32 split-K partials of (job, tile): [kq][mp rows][rp ranks]
__device__ __forceinline__ float* part_of(const Params& p, int job, int tile) {
  return p.ppart + ((size_t)job * MAX_TILES + tile) * (kPrefillPart / sizeof(float));
}
// ranks [c0, c0 + 32) of row r (v[i] = rank c0 + i; ranks >= nvals are written as zero),
// clipped to the rp columns of the image
__device__ __forceinline__ void write_v_chunk(char* img, const Unit& u, int r, int c0, const float (&v)[32],
                                              int nvals) {
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int c8 = (c0 >> 3) + q;
    if (c8 * 8 < u.rp) {
      float f[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) f[i] = c0 + q * 8 + i < nvals ? v[q * 8 + i] : 0.f;
      const uint4 w = make_uint4(pack_bf16x2(f[0], f[1]), pack_bf16x2(f[2], f[3]), pack_bf16x2(f[4], f[5]),
                                 pack_bf16x2(f[6], f[7]));
      *reinterpret_cast<uint4*>(img + (c8 >> 3) * u.xb + swz(r, c8 & 7)) = w;
    }
  }
}

__device__ __forceinline__ bool s_first_group_ok(int g0, int ngrp) { return g0 < ngrp; }

// Epilogue set -> its publisher warp.  The set's partial / V stores precede the post through
// the set's named barrier (CTA-scope ordering) and the release of pq_full; the publisher's
// gpu-scope fences are cumulative, so the epilogue warps never wait on a store round trip.
__device__ __forceinline__ void post_event(const Params& p, Shared& sm, int es, int& npost, int tile, int kind, int et) {
  asm volatile("fence.proxy.async.global;" ::: "memory");  // this thread's V stores -> TMA reads
  named_bar_sync(BAR_EPI + es, 128);
  if (et == 0) {
    const int k = npost;
    const int q = k % PQN;
    if (k >= PQN) pf_wait(p, &sm.pq_empty[es][q], ((k / PQN) - 1) & 1, 1, k, 0);
    sm.pq_tile[es][q] = tile;
    sm.pq_kind[es][q] = kind;
    mbar_arrive(&sm.pq_full[es][q]);
  }
  ++npost;
}

// Publisher warp: one finished phase-1 unit (its partial V image written) -> tile counter
// += 1 (release).  Expand units of the tile wait for all of the tile's units.
__device__ void publisher(const Params& p, Shared& sm, int es) {
  const int lane = threadIdx.x & 31;
  for (int k = 0;; ++k) {
    const int q = k % PQN;
    pf_wait(p, &sm.pq_full[es][q], (k / PQN) & 1, 2, k, 0);
    const int tile = sm.pq_tile[es][q], kind = sm.pq_kind[es][q];
    __syncwarp();
    if (lane == 0) mbar_arrive(&sm.pq_empty[es][q]);
    if (kind == 0) break;
    if (lane == 0) {
      __threadfence();  // cumulative over the epilogue set's image stores
      red_release_gpu_add(p.tile_cnt + tile, 1);
    }
  }
}

// One publisher warp for both epilogue sets (CHAM_PF_LD2: the other warp loads): the two
// queues are probed without blocking, each in its own order.
__device__ void publisher_both(const Params& p, Shared& sm) {
  const int lane = threadIdx.x & 31;
  int k[2] = {0, 0};
  bool done[2] = {false, false};
  while (!done[0] || !done[1]) {
    bool any = false;
#pragma unroll
    for (int es = 0; es < 2; ++es) {
      if (done[es]) continue;
      const int q = k[es] % PQN;
      if (!mbar_test_wait(&sm.pq_full[es][q], (k[es] / PQN) & 1)) continue;
      any = true;
      const int tile = sm.pq_tile[es][q], kind = sm.pq_kind[es][q];
      __syncwarp();
      if (lane == 0) mbar_arrive(&sm.pq_empty[es][q]);
      ++k[es];
      if (kind == 0) {
        done[es] = true;
        continue;
      }
      if (lane == 0) {
        __threadfence();  // cumulative over the epilogue set's image stores
        red_release_gpu_add(p.tile_cnt + tile, 1);
      }
    }
    if (!any) __nanosleep(32);
  }
}

// =========================================================================== the kernel
__global__ void __launch_bounds__(NTHREADS, 1) fused_kernel(const __grid_constant__ Params p) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  Shared& sm = *reinterpret_cast<Shared*>(smem_raw);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  crumb(p, 6, (unsigned long long)p.epoch);
  crumb(p, 0, gtimer());
  if (tid == 0) {
    for (int i = 0; i < NS; ++i) {
      mbar_init(&sm.full[i], 1);
      mbar_init(&sm.empty[i], 1 + 8);  // MMA commit + one arrival per epilogue warp
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&sm.tfull_sh[i], 1);
      mbar_init(&sm.tempty_sh[i], 4);

      mbar_init(&sm.vfull[i], 1);
      mbar_init(&sm.vempty[i], 1);
    }
    for (int i = 0; i < NACC; ++i) {
      mbar_init(&sm.tfull_ex[i], 1);
      mbar_init(&sm.tempty_ex[i], 4);
    }
    mbar_init(&sm.drain, 1);
    mbar_init(&sm.ho_bar, 1);
    for (int i = 0; i < UQ; ++i) {
      mbar_init(&sm.ufull[i], 1);
      mbar_init(&sm.uempty[i], 1 + 8);
    }
    for (int e = 0; e < 2; ++e)
      for (int i = 0; i < PQN; ++i) {
        mbar_init(&sm.pq_full[e][i], 1);
        mbar_init(&sm.pq_empty[e][i], 1);
      }
    fence_mbar_init();
  }
  if (kZeroAtom && warp == W_MMA) {  // zeros for the MMA's async-proxy reads (before the CTA barrier below)
    for (int i = lane; i < kAtomBytes / 16; i += 32) reinterpret_cast<uint4*>(sm.zero_atom)[i] = make_uint4(0, 0, 0, 0);
    fence_proxy_async_shared();
  }
  if (!CHAM_PF_NOPFMAP && warp == W_LOAD && lane < p.n_jobs) {
    prefetch_map(&p.maps[lane].x64);
    prefetch_map(&p.maps[lane].x1);
    prefetch_map(&p.maps[lane].y64);
    prefetch_map(&p.maps[lane].y1);
  }
  if (warp == W_MMA) {
    // CHAM_PF_LATE_ALLOC: take the tensor memory only once the previous kernel has completed
    if (CHAM_PF_LATE_ALLOC) pdl_wait();
    tmem_alloc(&sm.tmem_base);
    tc_fence_before();
  }
  if (warp == 0) sm.flag = build_tiles(p, sm.tl, gridDim.x) ? 1 : 0;
  __syncthreads();
  tc_fence_after();
  const TileList& tl = sm.tl;
  const uint32_t tmem = sm.tmem_base;
  crumb(p, 1, gtimer());
  pdl_wait();  // x, y, v and the workspaces may belong to the previous kernel
  if (CHAM_PF_PROXYFENCE) fence_proxy_async_global();
  crumb(p, 2, gtimer());
  if (kPfZeroNext) {
    // the previous launch (the other parity's user) is complete: re-arm its counter set, a
    // slice per CTA, before this launch lets the next one start (no last-CTA reset at exit)
    for (int i = blockIdx.x * NTHREADS + tid; i < p.zero_n; i += gridDim.x * NTHREADS) p.zero_set[i] = 0;
    __threadfence();
    __syncthreads();
  }
  pdl_launch_dependents();
  if (!sm.flag) {
    if (tid == 0 && blockIdx.x == 0) *p.err = CHAM_ERR_LIMIT;
  } else if (warp == W_LOAD || (kLd2 && warp == W_LOAD2)) {
    // ---------------------------------------------------------------- loader + dispatch
    // kLd2: loader 0 runs the shrink phase alone; at its first expand unit (position k0) it
    // hands positions k0 + 1, k0 + 3, ... to loader 1 and keeps k0, k0 + 2, ...  Every expand
    // unit is one ring stage and one V buffer, so position parity owns one stage and one V
    // buffer: each loader's waits stay in its own order.  A loader out of units posts
    // kUnitLoaderDone; the consumers then skip its positions.
    const int ld = (kLd2 && warp == W_LOAD2) ? 1 : 0;
    const uint64_t pol_w = policy_evict_first();  // adapter pages: streamed
    const uint64_t pol_x = CHAM_PF_XPOL_NORMAL == 1 ? policy_evict_normal() : CHAM_PF_XPOL_NORMAL == 2 ? policy_evict_first() : policy_evict_last();  // x: re-read by the other job groups / K ranges
    const uint64_t pol_y = policy_evict_first();
    // first unit static, the rest from the counter: lanes 0 .. CD-1 each hold one outstanding
    // claim (consumed round-robin and refilled at once), so a unit's id never waits for the
    // atomic's round trip
    //   (CHAM_PF_EXSTATIC=1 assigns the expand units statically, CTA c taking u1 + c, u1 + c + G,
    //   ...: no atomic on the loader's path, but it lost the A/B — tiles become ready unevenly.)
    int next = blockIdx.x;
    int claim = 1 << 29, chead = 0;
    bool dyn = true;
    int ex_j = 0;
    bool two = false;                // two-loader positions (k0 + ld + 2i)
    int h_k0 = 0, h_seq0 = 0, h_nex0 = 0;
    bool idle = false;               // loader 1 without a handoff
    if (ld == 1) {
      mbar_wait(&sm.ho_bar, 0);
      idle = !sm.ho_ok;
      h_k0 = sm.ho_k0;
      h_seq0 = sm.ho_seq0;
      h_nex0 = sm.ho_nex0;
      two = true;
      int c0 = 1 << 29;
      if (!idle && lane == 0) c0 = atomicAdd(p.ctr, 1);
      next = __shfl_sync(0xffffffffu, c0, 0) + gridDim.x;
    } else if (kExStatic && next >= tl.u1) {
      dyn = false;
      next = tl.u1 + blockIdx.x;
      ex_j = 1;
    }
    if (dyn && lane < CD && next < tl.u_total) claim = atomicAdd(p.ctr, 1);
    // published phase-1 units of an expand unit's tile, read without blocking one unit ahead
    auto peek_flag = [&](int u) {  // unconditional (clamped) load: the value is used one unit later
      int v;
      const int* f = p.tile_cnt + min(fdiv(max(u - tl.u1, 0), tl.ept, tl.inv_ept), MAX_TILES - 1);
      asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(f) : "memory");
      return v;
    };
    int flag = peek_flag(next);
    Prefetch pf = prefetch_unit(p, tl, next, lane);
    if (kWarmL2 && next < tl.u_total) warm_l2(p, make_unit(p, tl, next), pf, lane);
    int seq = 0, nex = 0;
    for (int k = ld == 0 ? 0 : h_k0 + 1; !idle; k += two ? 2 : 1) {
      if (k > 0 && lane == 0 && p.trace) trace_put(p, k - 1, 1, gtimer());
      const int u_id = __shfl_sync(0xffffffffu, next < tl.u_total ? next : -1, 0);
      if (kLd2 && ld == 0 && !two && p.mode == MODE_FUSED && u_id >= tl.u1) {
        // the first expand unit: from here on one stage and one V buffer per unit
        h_k0 = k;
        h_seq0 = seq;
        h_nex0 = nex;
        if (lane == 0) {
          sm.ho_k0 = k;
          sm.ho_seq0 = seq;
          sm.ho_nex0 = nex;
          sm.ho_ok = 1;
          mbar_arrive(&sm.ho_bar);  // release: the handoff values above
        }
        two = true;
      }
      if (two) {  // this loader's stage and V buffer sequence at position k
        seq = h_seq0 + (k - h_k0);
        nex = h_nex0 + (k - h_k0);
      }
      // publish the unit id to the MMA and epilogue warps
      const int q = k % UQ;
      if (lane == 0) {
        if (k >= UQ) pf_wait(p, &sm.uempty[q], ((k / UQ) - 1) & 1, 3, k, 0);
        sm.uslot[q] = (u_id < 0 && two) ? kUnitLoaderDone : u_id;
        mbar_arrive(&sm.ufull[q]);
        trace_ld(p, k, 0);
      }
      if (u_id < 0) break;
      // The next unit's claim and its lookahead loads (tile counter peek, page ids, token
      // rows); their values are consumed one unit later.  (Issuing them after the expand
      // unit's acquire fence instead: A/B on C3 588k vs 600k tok/s.)
      const int cur_flag = flag;
      const Prefetch cf = pf;
      auto advance = [&]() {
        // the lanes' claims were issued together, so their order is not the counter's; an
        // exhausted claim (>= the unit count) is skipped until every lane's is
        if (kExStatic && !dyn) {
          next = tl.u1 + blockIdx.x + ex_j * gridDim.x;
          ++ex_j;
        } else for (;;) {
          const int h = chead;
          chead = chead + 1 == CD ? 0 : chead + 1;
          next = __shfl_sync(0xffffffffu, claim, h) + gridDim.x;
          if (kExStatic && next >= tl.u1) {  // phase-1 units exhausted: the static expand list
            dyn = false;
            next = tl.u1 + blockIdx.x;
            ex_j = 1;
            break;
          }
          if (next < tl.u_total) {
            if (lane == h) claim = atomicAdd(p.ctr, 1);
            break;
          }
          if (lane == h) claim = 1 << 29;
          if (!__any_sync(0xffffffffu, lane < CD && claim + (int)gridDim.x < tl.u_total)) break;
        }
        if (lane == 0) trace_ld(p, k, 1);
        flag = peek_flag(next);
        if (lane == 0) trace_ld(p, k, 6);
        pf = prefetch_unit(p, tl, next, lane);
      };
      advance();
      if (lane == 0) trace_ld(p, k, 7);
      const Unit u = make_unit(p, tl, u_id);
      if (lane == 0 && p.trace) {
        trace_put(p, k, 0, gtimer());
        trace_put(p, k, 6, (unsigned long long)u_id | ((unsigned long long)u.kind << 32));
      }
      if (u.kind == 3) continue;
      const int my_page = cf.page;
      if (u.kind == 1) {
        // ---- shrink: x chunks of the tile + A^T atoms of every job of the group
        const int nblk = (u.m + 31) / 32;
        bool contig[4];
        int rows[4];
#pragma unroll
        for (int b = 0; b < 4; ++b) rows[b] = b < nblk ? block_row(cf, u, b, lane, contig[b]) : 0;
        const bool c64[2] = {block64(contig, rows, nblk, 0), nblk > 2 && block64(contig, rows, nblk, 1)};
        const int kc0 = u.kq * u.nchunks;
        const int np_pad = u.rp / 8;
        for (int s = 0; s < u.nst; ++s, ++seq) {
          const int st = seq % NS;
          const int c_first = s * u.kpc;
          const int nch = min(u.kpc, u.nchunks - c_first);
          if (seq >= NS) pf_wait(p, &sm.empty[st], ((seq / NS) - 1) & 1, 4, seq, u_id);
          if (s == 0 && lane == 0 && p.trace) trace_put(p, k, 7, gtimer());
          uint32_t bytes = nch * u.jps * u.np * kAtomBytes;
#pragma unroll
          for (int h = 0; h < 2; ++h)
            if (h * 64 < u.m) bytes += nch * (c64[h] ? 64 * 128 : min(64, u.m - h * 64) * 128);
          PF_CHECK(bytes <= STAGE && u.kpc * u.xb + u.jps * np_pad * u.kpc * kAtomBytes <= STAGE, 1, bytes, u.kpc);
          PF_CHECK(kc0 + c_first + nch <= p.h_in / 64 && nch > 0, 2, kc0 + c_first + nch, nch);
          PF_CHECK(lane >= u.np || (my_page >= 0 && my_page < p.n_pages), 3, my_page, u.slot);
          PF_CHECK(u.job0 + u.jps <= p.n_jobs && u.tile < tl.n_tiles, 4, u.job0, u.tile);
#pragma unroll
          for (int b = 0; b < 4; ++b) PF_CHECK(b * 32 >= u.m || (rows[b] >= 0 && rows[b] < p.n_tokens), 5, rows[b], b);
          if (lane == 0) mbar_arrive_expect_tx(&sm.full[st], bytes);
          __syncwarp();
          unsigned char* stg = sm.ring[st];
          for (int i = 0; i < nch; ++i) {
            const int kc = kc0 + c_first + i;
            unsigned char* xdst = stg + i * u.xb;
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              if (h * 64 >= u.m) continue;
              if (c64[h]) {
                if (lane == 0)
                  x_load(xdst + h * 64 * 128, &p.maps[u.job0].x64, kc * 64, rows[2 * h], &sm.full[st], pol_x);
              } else {
#pragma unroll
                for (int b = 2 * h; b < 2 * h + 2; ++b)
                  if (b * 32 + lane < u.m)
                    x_load(xdst + (b * 32 + lane) * 128, &p.maps[u.job0].x1, kc * 64, rows[b], &sm.full[st], pol_x);
              }
            }
          }
          // A^T atoms [job][page][chunk]: one copy of the stage's nch chunks per (job, page)
          unsigned char* adst = stg + u.kpc * u.xb;
          for (int j = 0; j < u.jps; ++j) {
            if (lane < u.np) {
              const char* src = p.base + (long long)my_page * p.page_bytes + p.jobs[u.job0 + j].a_off +
                                (long long)(kc0 + c_first) * kAtomBytes;
              bulk_g2s(adst + (j * np_pad + lane) * u.kpc * kAtomBytes, src, nch * kAtomBytes, &sm.full[st], pol_w);
            }
          }
        }
      } else {
        // ---- expand: V image of (job, tile), then B slices + y rows per 64-column group
        const int vb = nex & 1;
        if (lane == 0) {
          if (nex >= 2) pf_wait(p, &sm.vempty[vb], ((nex >> 1) - 1) & 1, 5, nex, u_id);
          trace_ld(p, k, 2);
          // every phase-1 unit of the tile has published its partial V image
          const int need = p.mode == MODE_EXPAND ? 1 : n_groups(p, u.rank);  // reduced images of the tile
          if (cur_flag < need) {
            while (ld_acquire_gpu(p.tile_cnt + u.tile) < need) __nanosleep(32);
          } else if (!CHAM_PF_NOACQ) {
            fence_acquire_gpu();  // the relaxed peek saw the count: acquire pattern before the V read
          }
          fence_proxy_async_global();
          trace_ld(p, k, 3);
          const uint32_t vbytes = u.vstride;
          PF_CHECK(vbytes <= VBUF && vbytes > 0 && u.tile < tl.n_tiles && u.job < p.n_jobs, 6, vbytes, u.tile);
          mbar_arrive_expect_tx(&sm.vfull[vb], vbytes);
          bulk_g2s(sm.vbuf[vb], vimg_of(p, u.job, u.tile), vbytes, &sm.vfull[vb], pol_w);
          trace_ld(p, k, 4);
        }
        __syncwarp();
        ++nex;
        const int nblk = (u.m + 31) / 32;
        bool contig[4] = {false, false, false, false};
        int rows[4] = {0, 0, 0, 0};
        bool c64[2] = {false, false};
        if (!kYReg) {  // the staged-y path's TMA boxes (the register path loads y in the epilogue)
#pragma unroll
          for (int b = 0; b < 4; ++b) rows[b] = b < nblk ? block_row(cf, u, b, lane, contig[b]) : 0;
          c64[0] = block64(contig, rows, nblk, 0);
          c64[1] = nblk > 2 && block64(contig, rows, nblk, 1);
        }
        const bool pad = !kZeroAtom && (u.rp / 8) > u.np;
        for (int s = 0; s < u.nst; ++s, ++seq) {
          const int st = seq % NS;
          const int g_first = s * u.kpc;
          const int ng = min(u.kpc, u.ngrp - g_first);
          if (seq >= NS) pf_wait(p, &sm.empty[st], ((seq / NS) - 1) & 1, 6, seq, u_id);
          if (s == 0 && lane == 0 && p.trace) trace_put(p, k, 7, gtimer());
          if (s == 0 && lane == 0) trace_ld(p, k, 5);
          unsigned char* stg = sm.ring[st];
          if (pad) {
            // odd page count: the K rows rank..rp of every group are a zero atom (page np)
            for (int c = lane; c < ng * 64; c += 32)
              reinterpret_cast<uint4*>(stg + u.np * u.kpc * kAtomBytes)[c] = make_uint4(0, 0, 0, 0);
            fence_proxy_async_shared();
          }
          __syncwarp();
          uint32_t bytes = ng * u.np * kAtomBytes;
          if (!kYReg) {
#pragma unroll
            for (int h = 0; h < 2; ++h)
              if (h * 64 < u.m) bytes += ng * (c64[h] ? 64 * 128 : min(64, u.m - h * 64) * 128);
          }
          PF_CHECK(bytes <= STAGE && u.kpc * u.bstride + (kYReg ? 0 : ng * u.xb) <= STAGE && ng > 0, 7, bytes, ng);
          PF_CHECK(u.col0 / 64 + g_first + ng <= p.h_out / 64, 8, u.col0, g_first);
          PF_CHECK(lane >= u.np || (my_page >= 0 && my_page < p.n_pages), 9, my_page, u.slot);
#pragma unroll
          for (int b = 0; b < 4; ++b) PF_CHECK(b * 32 >= u.m || (rows[b] >= 0 && rows[b] < p.n_tokens), 10, rows[b], b);
          if (lane == 0) mbar_arrive_expect_tx(&sm.full[st], bytes);
          __syncwarp();
          // B atoms [page][group]: one copy of the stage's ng groups per page
          if (lane < u.np) {
            const char* src = p.base + (long long)my_page * p.page_bytes + p.jobs[u.job].b_off +
                              (long long)(u.col0 / 64 + g_first) * kAtomBytes;
            bulk_g2s(stg + lane * u.kpc * kAtomBytes, src, ng * kAtomBytes, &sm.full[st], pol_w);
          }
          for (int g = 0; g < (kYReg ? 0 : ng); ++g) {
            const int col = u.col0 + (g_first + g) * 64;
            unsigned char* ydst = stg + u.kpc * u.bstride + g * u.xb;
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              if (h * 64 >= u.m) continue;
              if (c64[h]) {
                if (lane == 0) tma_load_2d(ydst + h * 64 * 128, &p.maps[u.job].y64, col, rows[2 * h], &sm.full[st], pol_y);
              } else {
#pragma unroll
                for (int b = 2 * h; b < 2 * h + 2; ++b)
                  if (b * 32 + lane < u.m)
                    tma_load_2d(ydst + (b * 32 + lane) * 128, &p.maps[u.job].y1, col, rows[b], &sm.full[st], pol_y);
              }
            }
          }
        }
      }
      if (kWarmL2 && next < tl.u_total) warm_l2(p, make_unit(p, tl, next), pf, lane);
    }
    if (kLd2 && ld == 0 && !two && lane == 0) {  // no expand units here: loader 1 has nothing to do
      sm.ho_ok = 0;
      mbar_arrive(&sm.ho_bar);
    }
  } else if ((kLd2 || kPub1) && warp == W_PUB) {
    publisher_both(p, sm);
  } else if (!kPub1 && (warp == W_PUB || warp == W_PUB + 1)) {
    publisher(p, sm, warp - W_PUB);
  } else if (warp == W_PUB + 1) {
    // kPub1 without kLd2: the second publisher warp has no role
  } else if (warp == W_MMA) {
    // ---------------------------------------------------------------- MMA issuer
    int seq = 0, nsh = 0, nex = 0, ngrp = 0, ndrain = 0;
    int skip_par = -1;  // CHAM_PF_LD2: position parity of the loader that finished first
    const uint32_t idesc_ex = idesc_bf16(BM, 64, true);
    for (int k = 0;; ++k) {
      if (k > 0 && lane == 0 && p.trace) trace_put(p, k - 1, 3, gtimer());
      if (skip_par >= 0 && (k & 1) == skip_par) {  // the finished loader's position: its stage
        ++seq;                                      // and V buffer advance, nothing else
        ++nex;
        continue;
      }
      const int q = k % UQ;
      pf_wait(p, &sm.ufull[q], (k / UQ) & 1, 7, k, 0);
      const int u_id = sm.uslot[q];
      __syncwarp();
      if (lane == 0) mbar_arrive(&sm.uempty[q]);
      if (u_id == kUnitLoaderDone && skip_par < 0) {
        ++seq;
        ++nex;
        skip_par = k & 1;
        continue;
      }
      if (u_id < 0) {
        if (lane == 0) sm.last[1] = ndrain;  // drain phases used (CHAM_PF_MMA_SYNC)
        __syncwarp();
        break;
      }
      const Unit u = make_unit(p, tl, u_id);
      if (u.kind == 3) continue;
      if (u.kind == 1) {
        const int ab = nsh & 1;
        if (nsh >= 2) pf_wait(p, &sm.tempty_sh[ab], ((nsh >> 1) - 1) & 1, 8, nsh, u_id);
        tc_fence_after();
        // (one MMA of N = jps * rp for the whole group would read x once per K step, but it
        // faulted intermittently in long PDL chains: one MMA per job)
        const uint32_t idesc = idesc_bf16(BM, u.rp, false);
        for (int s = 0; s < u.nst; ++s, ++seq) {
          const int st = seq % NS;
          const int nch = min(u.kpc, u.nchunks - s * u.kpc);
          mma_mark(p, k, s, seq, 1);  // waiting for the stage
          if (lane == 0 && p.trace) trace_put(p, k, 3, (1ull << 62) | ((unsigned long long)s << 8) | 1);
          pf_wait(p, &sm.full[st], (seq / NS) & 1, 9, seq, u_id);
          if (lane == 0 && p.trace) trace_put(p, k, 3, (1ull << 62) | ((unsigned long long)s << 8) | 2);
          mma_mark(p, k, s, seq, 2);  // issuing
          if (s == 0 && lane == 0 && p.trace) trace_put(p, k, 2, gtimer());
          tc_fence_after();
          if (lane == 0) {
            const uint32_t base = smem_u32(sm.ring[st]);
            for (int i = 0; i < nch; ++i) {
              const uint32_t xa = base + i * u.xb;
              for (int j = 0; j < u.jps; ++j) {
                // A^T atoms [job][page][chunk]: the pages of chunk i are kpc atoms apart
                const uint32_t aa = base + u.kpc * u.xb + (j * (u.rp / 8) * u.kpc + i) * kAtomBytes;
                const uint32_t d = tmem + ab * TM_SH + j * u.rp;
#pragma unroll
                for (int kk = 0; kk < 4; ++kk)
                  mma_bf16(d, sdesc(xa + kk * 32, 16, 1024), sdesc(aa + kk * 32, 16, u.kpc * kAtomBytes), idesc,
                           (s | i | kk) ? 1u : 0u);
              }
            }
            mma_commit(&sm.empty[st]);
            mbar_arrive_cnt(&sm.empty[st], 8);  // the epilogue warps never read shrink stages
            if (s == u.nst - 1) mma_commit(&sm.tfull_sh[ab]);
            mma_mark(p, k, s, seq, 3);  // issued + committed
            if (p.trace) trace_put(p, k, 3, (1ull << 62) | ((unsigned long long)s << 8) | 3);
            if (CHAM_PF_MMA_SYNC) {  // fault-hunt experiment: one stage of MMAs in flight at a time
              mma_commit(&sm.drain);
              mbar_wait(&sm.drain, ndrain & 1);
            }
          }
          ++ndrain;
          __syncwarp();
        }
        ++nsh;
      } else {
        const int vb = nex & 1;
        pf_wait(p, &sm.vfull[vb], (nex >> 1) & 1, 10, nex, u_id);
        tc_fence_after();
        const uint32_t va = smem_u32(sm.vbuf[vb]);
        for (int s = 0; s < u.nst; ++s, ++seq) {
          const int st = seq % NS;
          const int ng = min(u.kpc, u.ngrp - s * u.kpc);
          pf_wait(p, &sm.full[st], (seq / NS) & 1, 11, seq, u_id);
          if (s == 0 && lane == 0 && p.trace) trace_put(p, k, 2, gtimer());
          tc_fence_after();
          const uint32_t base = smem_u32(sm.ring[st]);
          for (int g = 0; g < ng; ++g, ++ngrp) {
            const int acc = ngrp % NACC;
            if (ngrp >= NACC) pf_wait(p, &sm.tempty_ex[acc], ((ngrp / NACC) - 1) & 1, 12, ngrp, u_id);
            tc_fence_after();
            if (lane == 0) {
              const uint32_t ba = base + g * kAtomBytes;  // B atoms [page][group]
              // D2 = V . B over the tile's (reduced) V image
              const int nk = u.rp / 16;
              const bool zpad = kZeroAtom && 2 * nk > u.np;  // odd page count: K rows rank..rp
              for (int kk = 0; kk < nk; ++kk) {
                const uint64_t ad = sdesc(va + (kk >> 2) * u.xb + (kk & 3) * 32, 16, 1024);
                const uint32_t b0 = ba + kk * 2 * u.kpc * kAtomBytes;
                // the second 8-row K group of the last step comes from the zero atom
                const uint32_t ks = (zpad && kk == nk - 1) ? smem_u32(sm.zero_atom) - b0 : u.kpc * kAtomBytes;
                const uint64_t bd = sdesc(b0, kAtomBytes, ks);
                mma_bf16(tmem + TM_EX + acc * 64, ad, bd, idesc_ex, kk ? 1u : 0u);
              }
              mma_commit(&sm.tfull_ex[acc]);
            }
            __syncwarp();
          }
          if (lane == 0) {
            mma_commit(&sm.empty[st]);
            if (kYReg) mbar_arrive_cnt(&sm.empty[st], 8);  // the epilogue never reads B-only stages
            if (s == u.nst - 1) mma_commit(&sm.vempty[vb]);
          }
          __syncwarp();
        }
        ++nex;
      }
    }
  } else {
    // ---------------------------------------------------------------- epilogue warps 0-7
    // Two sets of four warps (es = warp / 4), each covering all 128 rows (TMEM lane quarter
    // = warp % 4): set es drains the shrink units with nsh % 2 == es and the expand groups
    // with ngrp % 2 == es, i.e. exactly the TMEM accumulator buffer es.
    const int es = warp >> 2, wq = warp & 3;
    const int r = wq * 32 + lane;  // tile row == TMEM lane
    const uint32_t lane_off = (uint32_t)(wq * 32) << 16;
    int seq = 0, nsh = 0, ngrp = 0, nvb = 0, npost = 0;
    int skip_par = -1;  // CHAM_PF_LD2: position parity of the loader that finished first
    for (int k = 0;; ++k) {
      if (k > 0 && tid == 0 && p.trace) trace_put(p, k - 1, 5, gtimer());
      if (skip_par >= 0 && (k & 1) == skip_par) {
        ++seq;
        continue;
      }
      const int q = k % UQ;
      pf_wait(p, &sm.ufull[q], (k / UQ) & 1, 13, k, 0);
      const int u_id = sm.uslot[q];
      __syncwarp();
      if (lane == 0) mbar_arrive(&sm.uempty[q]);
      if (u_id == kUnitLoaderDone && skip_par < 0) {
        ++seq;
        skip_par = k & 1;
        continue;
      }
      if (u_id < 0) {
        post_event(p, sm, es, npost, 0, 0, r);  // the publisher exits
        break;
      }
      const Unit u = make_unit(p, tl, u_id);
      const int pos = u.pos0 + min(r, u.m - 1);
      if (u.kind == 3) {
        // ---- MODE_EXPAND phase 1: caller's v rows -> V image
        if ((nvb++ & 1) != es) continue;
        if (r < u.mp) {
          const int nv = r < u.m ? min(u.rank, p.v_stride) : 0;
          const float* src = p.v_in + (long long)pos * p.v_stride;
          for (int c0 = 0; c0 < u.rp; c0 += 32) {
            float v[32];
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] = c0 + i < nv ? src[c0 + i] : 0.f;
            write_v_chunk(vimg_of(p, 0, u.tile), u, r, c0, v, nv);
          }
        }
        post_event(p, sm, es, npost, u.tile, 2, r);
        continue;
      }
      if (u.kind == 1) {
        // ---- shrink: drain the accumulators (the MMA warp releases the stages)
        seq += u.nst;
        const int ab = nsh & 1;
        if (ab != es) {
          ++nsh;
          continue;
        }
        pf_wait(p, &sm.tfull_sh[ab], (nsh >> 1) & 1, 14, nsh, u_id);
        if (r == 0 && p.trace) trace_put(p, k, 4, gtimer());
        tc_fence_after();
        ++nsh;
        const bool split = p.mode == MODE_FUSED && u.ks > 1;
        for (int j = 0; j < u.jps; ++j) {
          const int job = u.job0 + j;
          for (int c0 = 0; c0 < u.rank; c0 += 32) {
            float v[32];
            tmem_ld32(tmem + ab * TM_SH + j * u.rp + c0 + lane_off, v);
            if (p.mode == MODE_SHRINK) {
              if (r < u.m) {
                const int nv = min(u.rank, p.v_stride);
                float* dst = p.v_out + (long long)pos * p.v_stride;
#pragma unroll
                for (int i = 0; i < 32; ++i)
                  if (c0 + i < nv) dst[c0 + i] = v[i];
              }
            } else if (split) {
              // this K range's fp32 partial row (rows >= m are never read back)
              if (r < u.m) {
                float4* dst = reinterpret_cast<float4*>(part_of(p, job, u.tile) + ((size_t)u.kq * u.mp + r) * u.rp + c0);
#pragma unroll
                for (int i = 0; i < 8; ++i)
                  if (c0 + i * 4 < u.rp) dst[i] = make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
              }
            } else if (r < u.mp) {
              write_v_chunk(vimg_of(p, job, u.tile), u, r, c0, v, r < u.m ? u.rank : 0);  // the tile's V image
            }
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&sm.tempty_sh[ab]);
        if (p.mode == MODE_SHRINK) continue;
        if (split) {
          // split-K arrival: the last of the tile's ks units of this job group sums the ks fp32
          // partials in K order (deterministic) and writes the ONE bf16 V image
          named_bar_sync(BAR_EPI + es, 128);
          if (r == 0) {
            __threadfence();  // release: this set's partial stores before the arrival
            const int old = atomicAdd(p.arrive + u.tile * kMaxJobs + u.job0 / u.jps, 1);
            __threadfence();  // acquire: the other units' partials after the arrival
            sm.last_arr[es] = old == u.ks - 1;
          }
          named_bar_sync(BAR_EPI + es, 128);
          if (!sm.last_arr[es]) continue;
          for (int j = 0; j < u.jps; ++j) {
            const int job = u.job0 + j;
            const float* base = part_of(p, job, u.tile);
            if (r < u.mp)
              for (int c0 = 0; c0 < u.rank; c0 += 32) {
                float v[32];
#pragma unroll
                for (int i = 0; i < 32; ++i) v[i] = 0.f;
                if (r < u.m)
                  for (int kq = 0; kq < u.ks; ++kq) {
                    const float4* src = reinterpret_cast<const float4*>(base + ((size_t)kq * u.mp + r) * u.rp + c0);
#pragma unroll
                    for (int i = 0; i < 8; ++i)
                      if (c0 + i * 4 < u.rp) {
                        const float4 q = __ldcg(src + i);
                        v[4 * i] += q.x; v[4 * i + 1] += q.y; v[4 * i + 2] += q.z; v[4 * i + 3] += q.w;
                      }
                  }
                write_v_chunk(vimg_of(p, job, u.tile), u, r, c0, v, r < u.m ? u.rank : 0);
              }
          }
        }
        post_event(p, sm, es, npost, u.tile, 2, r);
        continue;
      }
      // ---- expand: y rows += D2 per 64-column group.  Each thread adds its row in place in
      // the staged y tile; then the warp stores its 32 rows coalesced (8 lanes per 128-byte
      // row, 4 rows per instruction) instead of 32 rows x 16 B per instruction.
      const int yrow_idx = __ldg(p.perm + pos);
      const bool valid = r < u.m;
      char* const ybase_g = p.jobs[u.job].y;
      if (kYReg) {
        // Each thread owns tile row r (TMEM lane r): its 128-byte y piece of a 64-column group
        // is loaded into registers one of its groups ahead (the loads overlap the B copies and
        // the MMAs), D2 is added, and the row piece is stored back.  The ring carries B only.
        seq += u.nst;
        char* const yrow = ybase_g + (long long)yrow_idx * p.h_out * 2 + (long long)u.col0 * 2;
        const int g0 = (es - (ngrp & 1)) & 1;  // this set's first group of the unit
        uint4 ya[8], yb[8];
        auto yload = [&](int g, uint4 (&buf)[8]) {
          if (CHAM_EXP_NOEPI < 2 && valid && g < u.ngrp) {
#pragma unroll
            for (int i = 0; i < 8; ++i) buf[i] = __ldcs(reinterpret_cast<const uint4*>(yrow + g * 128) + i);
          }
        };
        auto yupdate = [&](int g, uint4 (&buf)[8]) {
          const int gi = ngrp + g;
          const int acc = gi % NACC;
          if (CHAM_EXP_NOEPI == 3) {  // experiment: the epilogue releases the accumulator unread
            if (lane == 0) mbar_arrive(&sm.tempty_ex[acc]);
            return;
          }
          pf_wait(p, &sm.tfull_ex[acc], (gi / NACC) & 1, 16, gi, u_id);
          tc_fence_after();
          float d0[32], d1[32];
          tmem_ld32x2(tmem + TM_EX + acc * 64 + lane_off, d0, d1);
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&sm.tempty_ex[acc]);
          if (valid && !kNoEpi) {
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              const float* d = i < 4 ? d0 + i * 8 : d1 + (i - 4) * 8;
              float f[8];
              Elem<__nv_bfloat16>::unpack(buf[i], f);
#pragma unroll
              for (int e = 0; e < 8; ++e) f[e] += d[e];
              __stcs(reinterpret_cast<uint4*>(yrow + g * 128) + i, Elem<__nv_bfloat16>::pack(f));
            }
          }
        };
        if (kYPrefetch && valid)  // this set's later groups of the unit: DRAM -> L2 now, registers later
          for (int g = g0 + 2; g < u.ngrp; g += 2)
            asm volatile("prefetch.global.L2 [%0];" ::"l"(yrow + g * 128) : "memory");
        if (s_first_group_ok(g0, u.ngrp)) yload(g0, ya);
        for (int g = g0; g < u.ngrp; g += 4) {
          yload(g + 2, yb);
          yupdate(g, ya);
          if (g + 2 >= u.ngrp) break;
          yload(g + 4, ya);
          yupdate(g + 2, yb);
        }
        if (r == 0 && p.trace) trace_put(p, k, 4, gtimer());
        ngrp += u.ngrp;
        continue;
      }
      for (int s = 0; s < u.nst; ++s, ++seq) {
        const int st = seq % NS;
        const int ng = min(u.kpc, u.ngrp - s * u.kpc);
        pf_wait(p, &sm.full[st], (seq / NS) & 1, 15, seq, u_id);  // the y rows of this stage have landed
        if (s == 0 && tid == 0 && p.trace) trace_put(p, k, 4, gtimer());
        const unsigned char* ybase = sm.ring[st] + u.kpc * u.bstride;
        for (int g = 0; g < ng; ++g, ++ngrp) {
          const int acc = ngrp & 1;
          if (acc != es) continue;  // the other set's group
          pf_wait(p, &sm.tfull_ex[acc], (ngrp >> 1) & 1, 16, ngrp, u_id);
          tc_fence_after();
          float d0[32], d1[32];
          const uint32_t ta = tmem + TM_EX + acc * 64 + lane_off;
          tmem_ld32x2(ta, d0, d1);
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&sm.tempty_ex[acc]);
          const int col0 = u.col0 + (s * u.kpc + g) * 64;
          unsigned char* yg = const_cast<unsigned char*>(ybase) + g * u.xb;
          if (kNoEpi) continue;  // experiment builds: data-movement ceiling without the y update
          if (valid) {
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              const float* d = i < 4 ? d0 + i * 8 : d1 + (i - 4) * 8;
              float f[8];
              Elem<__nv_bfloat16>::unpack(lds128(yg + swz(r, i)), f);
#pragma unroll
              for (int e = 0; e < 8; ++e) f[e] += d[e];
              const uint4 w = Elem<__nv_bfloat16>::pack(f);
              asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};" ::"r"(smem_u32(yg + swz(r, i))), "r"(w.x), "r"(w.y),
                           "r"(w.z), "r"(w.w)
                           : "memory");
            }
          }
          __syncwarp();
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const int rr = i * 4 + (lane >> 3);  // row of this warp's block
            const int c = lane & 7;              // 16-byte chunk of the row
            const int grow = __shfl_sync(0xffffffffu, yrow_idx, rr);
            if (wq * 32 + rr < u.m) {
              const uint4 w = lds128(yg + swz(wq * 32 + rr, c));
              *reinterpret_cast<uint4*>(ybase_g + ((long long)grow * p.h_out + col0 + c * 8) * 2) = w;
            }
          }
        }
        // the in-place y updates above are generic-proxy writes into a stage the loader will
        // refill with TMA (async proxy): order them before the release
        fence_proxy_async_shared();
        __syncwarp();
        if (lane == 0) mbar_arrive(&sm.empty[st]);
      }
    }
  }
  // the last CTA re-arms this parity's counters
  crumb(p, 3, gtimer());
  if (kDrain && warp == W_MMA) {
    // tcgen05.commit arrivals are asynchronous: a CTA that exits with one in flight lets it
    // land in the shared memory of the next CTA on this SM (PDL starts it right away), on
    // that CTA's freshly initialised barriers.  One more commit, waited for, drains them.
    if (lane == 0) mma_commit(&sm.drain);
    __syncwarp();
    mbar_wait(&sm.drain, CHAM_PF_MMA_SYNC ? (sm.last[1] & 1) : 0);
  }
  __syncthreads();
  crumb(p, 4, gtimer());
  if (warp == W_MMA) {
    tc_fence_after();
    tmem_dealloc(tmem);
  }
  if (kPfZeroNext) {  // the next launch re-arms this parity's counters
    crumb(p, 5, gtimer());
    return;
  }
  if (tid == 0) {
    __threadfence();
    sm.last[0] = atomicAdd(p.ctr + 1, 1) == (int)gridDim.x - 1;
  }
  __syncthreads();
  if (sm.last[0]) {
    for (int i = tid; i < MAX_TILES; i += NTHREADS) p.tile_cnt[i] = 0;
    for (int i = tid; i < MAX_TILES * kMaxJobs; i += NTHREADS) p.arrive[i] = 0;
    if (tid == 0) {
      p.ctr[0] = 0;
      p.ctr[1] = 0;
    }
    __threadfence();
  }
  crumb(p, 5, gtimer());
}


// =========================================================================== expand kernel
// The standalone expand phase of a prefill apply (CHAM_PF_SPLITX): the fused kernel runs in
// shrink-only mode (no_expand: it publishes the tiles' V images and stops), then this kernel
// streams y += V . B with no dependency left inside the launch — every V image is final once
// griddepcontrol.wait returns — so the work is split statically: each CTA owns one contiguous
// range of items (tile, job, column block), balanced by bytes, and runs it as a plain pipeline
// without claims, readiness polls or per-unit global round trips on the loader's path.
//   warp 0 loader: per item one ring stage = the y rows of the item's G 64-column groups
//          (TMA, 32-row SWIZZLE_128B boxes, 1-row boxes for non-consecutive rows) + the B page
//          slices of those groups (bulk copies straight from the page layout, [page][group]
//          atoms: the MN-major SWIZZLE_128B B operand); per run of items of one (tile, job)
//          the V image (double-buffered).
//   warp 1 MMA: D[128 x 64] = V . B per group into one of eight TMEM accumulators.
//   warps 2-5 epilogue: thread = tile row = TMEM lane; adds D to its y row piece IN the stage
//          (swizzled 16-byte chunks: conflict-free), then the warp TMA-stores its 32 rows back
//          (one box when they are 32 consecutive valid tokens, else one row box per row).
// Arithmetic is the fused kernel's: the same V image, the same UMMA sequence, y + D rounded
// once to bf16 — the two paths give bit-identical y.
#ifndef CHAM_PF_SPLITX
#define CHAM_PF_SPLITX 0  // 1: fused-mode applies run as shrink-only fused kernel + expand_kernel (A/B on C3: 540k vs 630k tok/s fused)
#endif
#ifndef CHAM_PFX_NS
#define CHAM_PFX_NS 6
#endif
constexpr int XNS = CHAM_PFX_NS;     // ring stages
constexpr int XSTAGE = 24576;        // bytes per stage (y of G groups of <= 64 rows + their B slices)
constexpr int XACC = 8;              // TMEM accumulators of 64 fp32 columns (all 512 columns)
#ifndef CHAM_PFX_SETS
#define CHAM_PFX_SETS 2              // epilogue sets (4 warps each) working on alternate items
#endif
constexpr int XSETS = CHAM_PFX_SETS;
constexpr int X_THREADS = 64 + 128 * XSETS;  // warp 0 loader, 1 MMA, then the epilogue sets
constexpr int XROWS = 64;            // rows of an expand item (a half of a 128-row tile)
constexpr int XYB = XROWS * 128;     // y bytes of one 64-column group of an item
constexpr int XVB = 2 * XYB;         // V buffer: the item rows of <= 2 K-blocks (rank <= 128)
#ifndef CHAM_PFX_IDY
#define CHAM_PFX_IDY 1  // y added on the tensor cores: D = I . Y + V . B (epilogue: convert + store only)
#endif
constexpr bool kIdY = CHAM_PFX_IDY != 0;
#ifndef CHAM_PFX_EXP
#define CHAM_PFX_EXP 0  // experiment builds: 1 the epilogue skips the y add, 2 waits for each item's stores
#endif
#ifndef CHAM_PFX_LAG
#define CHAM_PFX_LAG 1               // items (of one set) whose y stores may still read their stage
#endif
constexpr int XLAG = CHAM_PFX_LAG;
static_assert(XACC * 64 <= TMEM_COLS, "TMEM budget");
static_assert(XNS > XSETS * (XLAG + 1), "ring depth");

struct XShared {
  alignas(1024) unsigned char stage[XNS][XSTAGE];
  // two V buffers + one pad: the UMMA A operand spans 128 rows, the image has 64 per K-block
  alignas(1024) unsigned char vbuf[2 * XVB + XYB];
  // kIdY: A operand [128 rows x 64 K] = the identity on rows < 64 (K-major SWIZZLE_128B)
  alignas(1024) unsigned char ident[kIdY ? BM * 128 : 16];
  uint64_t full[XNS], empty[XNS];
  uint64_t tfull[XACC], tempty[XACC];
  uint64_t vfull[2], vempty[2];
  uint64_t drain;
  uint32_t tmem_base;
  int ok;
  int lo, hi;            // this CTA's items [lo, hi)
  int t0, h0, j0, cb0;   // (tile, half, job, column block) of item lo
  TileList tl;
};
static_assert(sizeof(XShared) <= 227 * 1024, "expand kernel shared memory exceeds 227 KiB");

// Per-tile item geometry: G 64-column groups per item, as many as one stage holds.
struct XGeom {
  int rp, np, npad;  // ranks (16-padded), pages, pages incl. the zero pad
  int nh;            // 64-row halves of the tile
  int G, ncb;        // groups per item, items per (tile, half, job)
  int xb;            // K-block stride of the tile's V image (mp rows x 128 B)
};
__device__ __forceinline__ XGeom xgeom(const Params& p, const Tile& t) {
  XGeom g;
  g.rp = rpad(t.rank);
  g.np = (t.rank + 7) / 8;
  g.npad = g.rp / 8;
  g.nh = (t.m + XROWS - 1) / XROWS;
  g.xb = mpad(t.m) * 128;
  g.G = max(1, min(8, XSTAGE / (XYB + g.npad * kAtomBytes)));
  const int ngr = p.h_out / 64;
  g.ncb = (ngr + g.G - 1) / g.G;
  return g;
}
// Byte weight of one item of tile t (y read + written, B read): the balance unit.
__device__ __forceinline__ long long xweight(const Tile& t, const XGeom& g) {
  return (long long)g.G * (2LL * min(t.m, XROWS) * 128 + (long long)g.np * kAtomBytes);
}

// Warp 0: this CTA's item range, by byte weight (items in (tile, half, job, block) order).
__device__ void x_range(const Params& p, XShared& sm) {
  const int lane = threadIdx.x & 31;
  const TileList& tl = sm.tl;
  const int n = tl.n_tiles;
  const int K = (n + 31) / 32;  // tiles per lane, contiguous
  const int ta = min(n, lane * K), tb = min(n, ta + K);
  long long w = 0;
  int items = 0;
  for (int t = ta; t < tb; ++t) {
    const XGeom g = xgeom(p, tl.t[t]);
    const int it = g.nh * p.n_jobs * g.ncb;
    items += it;
    w += it * xweight(tl.t[t], g);
  }
  long long wpre = w;
  int ipre = items;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const long long a = __shfl_up_sync(0xffffffffu, wpre, o);
    const int b = __shfl_up_sync(0xffffffffu, ipre, o);
    if (lane >= o) {
      wpre += a;
      ipre += b;
    }
  }
  const long long W = __shfl_sync(0xffffffffu, wpre, 31);
  const int NI = __shfl_sync(0xffffffffu, ipre, 31);
  wpre -= w;  // exclusive
  ipre -= items;
  // the first item whose start weight is >= S, and its (tile, half, job, block)
  auto locate = [&](long long S, int (&res)[5]) {
    const bool mine = S >= wpre && S < wpre + w;
    const unsigned bal = __ballot_sync(0xffffffffu, mine);
    int r[5] = {NI, n, 0, 0, 0};
    if (mine && lane == __ffs(bal) - 1) {
      long long acc = wpre;
      int ib = ipre;
      for (int t = ta; t < tb; ++t) {
        const XGeom g = xgeom(p, tl.t[t]);
        const long long wi = xweight(tl.t[t], g);
        const int it = g.nh * p.n_jobs * g.ncb;
        if (S < acc + it * wi) {
          const int k = (int)((S - acc + wi - 1) / wi);
          if (k >= it) {
            r[0] = ib + it;
            r[1] = t + 1;
          } else {
            r[0] = ib + k;
            r[1] = t;
            r[2] = k / (p.n_jobs * g.ncb);
            r[3] = (k / g.ncb) % p.n_jobs;
            r[4] = k % g.ncb;
          }
          break;
        }
        acc += it * wi;
        ib += it;
      }
    }
    const int src = bal ? __ffs(bal) - 1 : 0;
#pragma unroll
    for (int i = 0; i < 5; ++i) {
      const int v = __shfl_sync(0xffffffffu, r[i], src);
      res[i] = bal ? v : (i == 0 ? NI : i == 1 ? n : 0);
    }
  };
  const long long S0 = W * (long long)blockIdx.x / gridDim.x;
  const long long S1 = W * (long long)(blockIdx.x + 1) / gridDim.x;
  int r0[5], r1[5];
  locate(S0, r0);
  int hi = NI;
  if (blockIdx.x + 1 != gridDim.x) {
    locate(S1, r1);
    hi = r1[0];
  }
  if (lane == 0) {
    sm.lo = r0[0];
    sm.hi = max(r0[0], hi);
    sm.t0 = r0[1];
    sm.h0 = r0[2];
    sm.j0 = r0[3];
    sm.cb0 = r0[4];
  }
}

// Item cursor: (tile, half, job, column block) in item order.
struct XCursor {
  int t, h, j, cb;
  __device__ __forceinline__ void next(int n_jobs, const XGeom& g) {
    if (++cb == g.ncb) {
      cb = 0;
      if (++j == n_jobs) {
        j = 0;
        if (++h == g.nh) {
          h = 0;
          ++t;
        }
      }
    }
  }
};

// debug timeline (trace builds): the first half of the debug buffer, units 64 + i: item i of
// the CTA's range: 0 loader issued, 1 MMA got the stage, 2 epilogue got it, 3 epilogue done;
// unit 63: lo, hi, start time
__device__ __forceinline__ void xtrace(const Params& p, int i, int field, unsigned long long v) {
  const int k = 64 + i;
  if (p.trace && k < p.trace_cap)
    p.trace[(((long long)blockIdx.x - (long long)gridDim.x) * p.trace_cap + k) * 8 + field] = v;
}

__global__ void __launch_bounds__(X_THREADS, 1) expand_kernel(const __grid_constant__ Params p) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  XShared& sm = *reinterpret_cast<XShared*>(smem_raw);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int i = 0; i < XNS; ++i) {
      mbar_init(&sm.full[i], 1);
      mbar_init(&sm.empty[i], 1 + 128);  // MMA commit + every epilogue thread (its stores read)
    }
    for (int i = 0; i < XACC; ++i) {
      mbar_init(&sm.tfull[i], 1);
      mbar_init(&sm.tempty[i], 4);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&sm.vfull[i], 1);
      mbar_init(&sm.vempty[i], 1);
    }
    mbar_init(&sm.drain, 1);
    fence_mbar_init();
  }
  if (warp == 0 && lane < p.n_jobs) {
    prefetch_map(&p.maps[lane].y32);
    prefetch_map(&p.maps[lane].y1);
  }
  if (kIdY) {
    for (int i = tid; i < BM * 8; i += X_THREADS) {  // row i / 8, 16-byte chunk i % 8 (K cols 8c..8c+7)
      const int rr = i >> 3, ch = i & 7;
      uint32_t w[4] = {0, 0, 0, 0};
      if (rr < XROWS && (rr >> 3) == ch) w[(rr & 7) >> 1] = (rr & 1) ? 0x3F800000u : 0x00003F80u;
      *reinterpret_cast<uint4*>(sm.ident + swz(rr, ch)) = make_uint4(w[0], w[1], w[2], w[3]);
    }
    fence_proxy_async_shared();  // generic stores -> the UMMA's async-proxy reads
  }
  if (warp == 1) {
    tmem_alloc(&sm.tmem_base);
    tc_fence_before();
  }
  if (warp == 0) {
    const bool ok = build_tiles(p, sm.tl, gridDim.x);
    if (lane == 0) sm.ok = ok ? 1 : 0;
    if (ok) x_range(p, sm);
  }
  __syncthreads();
  tc_fence_after();
  const TileList& tl = sm.tl;
  const uint32_t tmem = sm.tmem_base;
  const int lo = sm.ok ? sm.lo : 0, hi = sm.ok ? sm.hi : 0;
  if (!sm.ok && tid == 0 && blockIdx.x == 0) *p.err = CHAM_ERR_LIMIT;
  if (tid == 0) {
    xtrace(p, -1, 0, lo);
    xtrace(p, -1, 1, hi);
    xtrace(p, -1, 2, gtimer());
  }
  const int ngr = p.h_out / 64;
  if (warp == 0) {
    // ---------------------------------------------------------------- loader
    const uint64_t pol_w = policy_evict_first();
    const uint64_t pol_y = policy_evict_first();
    XCursor c{sm.t0, sm.h0, sm.j0, sm.cb0};
    int cur_t = -1, cur_h = -1, cur_j = -1, nrun = -1, seq = 0, mh = 0;
    int rows[2] = {0, 0}, rf[2] = {0, 0};  // this lane's row / the 32-row block's first row
    bool c32[2] = {false, false};
    int page = 0;
    XGeom g{};
    bool waited = false;
    for (int it = lo; it < hi; ++it, c.next(p.n_jobs, g)) {
      const Tile& T = tl.t[c.t];
      if (c.t != cur_t) {
        g = xgeom(p, T);
        page = __ldg(p.slot_pages + T.slot * kMaxPagesPerSlot + min(lane, kMaxPagesPerSlot - 1));
      }
      if (c.t != cur_t || c.h != cur_h) {
        mh = min(XROWS, T.m - c.h * XROWS);
#pragma unroll
        for (int b = 0; b < 2; ++b) {
          rows[b] = __ldg(p.perm + T.pos0 + c.h * XROWS + min(b * 32 + lane, mh - 1));
          rf[b] = __shfl_sync(0xffffffffu, rows[b], 0);
          c32[b] = __all_sync(0xffffffffu, b * 32 + lane >= mh || rows[b] == rf[b] + lane);
        }
      }
      if (!waited) {  // V images (the shrink kernel) and y (earlier applies) come from earlier grids
        pdl_wait();
        pdl_launch_dependents();
        waited = true;
      }
      if (c.t != cur_t || c.h != cur_h || c.j != cur_j) {
        ++nrun;
        const int vb = nrun & 1;
        const int nkb = (g.rp + 63) / 64;
        if (lane == 0) {
          if (nrun >= 2) mbar_wait(&sm.vempty[vb], ((nrun >> 1) - 1) & 1);
          mbar_arrive_expect_tx(&sm.vfull[vb], nkb * XYB);
        }
        __syncwarp();
        // the half's 64 rows of each K-block of the tile's V image
        if (lane < nkb)
          bulk_g2s(sm.vbuf + vb * XVB + lane * XYB, vimg_of(p, c.j, c.t) + lane * g.xb + c.h * XYB, XYB,
                   &sm.vfull[vb], pol_w);
        cur_t = c.t;
        cur_h = c.h;
        cur_j = c.j;
      }
      const int s = seq % XNS;
      if (lane == 0 && seq >= XNS) mbar_wait(&sm.empty[s], ((seq / XNS) - 1) & 1);
      __syncwarp();
      unsigned char* st = sm.stage[s];
      unsigned char* bst = st + g.G * XYB;  // B atoms [page][group], page stride G KiB
      const int col0 = c.cb * g.G * 64;
      const int ng = min(g.G, ngr - c.cb * g.G);
      if (g.npad > g.np) {
        // zero atoms for the K rows rank..rp (V is zero there; 0 x stale NaN would not be)
        uint4* z = reinterpret_cast<uint4*>(bst + g.np * g.G * kAtomBytes);
        for (int i = lane; i < (g.npad - g.np) * g.G * (kAtomBytes / 16); i += 32) z[i] = make_uint4(0, 0, 0, 0);
        fence_proxy_async_shared();
      }
      __syncwarp();
      // both 32-row blocks consecutive: one 64-row box per group
      const bool c64 = mh > 32 && c32[0] && c32[1] && rf[1] == rf[0] + 32;
      uint32_t ybytes = 0;
#pragma unroll
      for (int b = 0; b < 2; ++b)
        if (b * 32 < mh) ybytes += c32[b] ? 32 * 128 : min(32, mh - b * 32) * 128;
      if (CHAM_PFX_EXP == 4) ybytes = 0;
      if (kIdY && (mh < XROWS || !c32[0] || !c32[1])) {
        // the identity MMA reads all 64 y rows of a group: rows no box covers must be finite
        for (int gi = 0; gi < ng; ++gi)
#pragma unroll
          for (int b = 0; b < 2; ++b) {
            if (c32[b] && b * 32 < mh) continue;  // the box fills all 32 rows
            for (int i = lane; i < 32 * 8; i += 32) {
              const int rr = b * 32 + (i >> 3);
              if (rr >= mh) *reinterpret_cast<uint4*>(st + gi * XYB + rr * 128 + (i & 7) * 16) = make_uint4(0, 0, 0, 0);
            }
          }
        fence_proxy_async_shared();
        __syncwarp();
      }
      if (lane == 0) mbar_arrive_expect_tx(&sm.full[s], ng * (g.np * kAtomBytes + ybytes));
      __syncwarp();
      if (lane < g.np)
        bulk_g2s(bst + lane * g.G * kAtomBytes,
                 p.base + (long long)page * p.page_bytes + p.jobs[c.j].b_off + (long long)(col0 / 64) * kAtomBytes,
                 ng * kAtomBytes, &sm.full[s], pol_w);
      for (int gi = 0; gi < (CHAM_PFX_EXP == 4 ? 0 : ng); ++gi) {
        unsigned char* yd = st + gi * XYB;
        if (c64 && CHAM_PFX_EXP == 3) {
          if (lane == 0) tma_load_2d(yd, &p.maps[c.j].y64, col0 + gi * 64, rf[0], &sm.full[s], pol_y);
          continue;
        }
#pragma unroll
        for (int b = 0; b < 2; ++b) {
          if (b * 32 >= mh) continue;
          if (c32[b]) {
            if (lane == 0) tma_load_2d(yd + b * 32 * 128, &p.maps[c.j].y32, col0 + gi * 64, rf[b], &sm.full[s], pol_y);
          } else if (b * 32 + lane < mh) {
            tma_load_2d(yd + (b * 32 + lane) * 128, &p.maps[c.j].y1, col0 + gi * 64, rows[b], &sm.full[s], pol_y);
          }
        }
      }
      if (lane == 0) xtrace(p, it - lo, 0, gtimer());
      ++seq;
    }
    if (!waited) {
      pdl_wait();
      pdl_launch_dependents();
    }
  } else if (warp == 1) {
    // ---------------------------------------------------------------- MMA issuer
    const uint32_t idesc = idesc_bf16(BM, 64, true);
    XCursor c{sm.t0, sm.h0, sm.j0, sm.cb0};
    int cur_t = -1, cur_h = -1, cur_j = -1, nrun = -1, seq = 0, nacc = 0;
    XGeom g{};
    for (int it = lo; it < hi; ++it) {
      if (c.t != cur_t) g = xgeom(p, tl.t[c.t]);
      if (c.t != cur_t || c.h != cur_h || c.j != cur_j) {
        ++nrun;
        mbar_wait(&sm.vfull[nrun & 1], (nrun >> 1) & 1);
        cur_t = c.t;
        cur_h = c.h;
        cur_j = c.j;
      }
      const int s = seq % XNS;
      mbar_wait(&sm.full[s], (seq / XNS) & 1);
      if (lane == 0) xtrace(p, it - lo, 1, gtimer());
      tc_fence_after();
      const uint32_t va = smem_u32(sm.vbuf + (nrun & 1) * XVB);
      const uint32_t bb = smem_u32(sm.stage[s] + g.G * XYB);
      const int ng = min(g.G, ngr - c.cb * g.G);
      for (int gi = 0; gi < ng; ++gi, ++nacc) {
        const int a = nacc % XACC;
        if (nacc >= XACC) mbar_wait(&sm.tempty[a], ((nacc / XACC) - 1) & 1);
        tc_fence_after();
        if (lane == 0) {
          if (kIdY) {  // D = I . Y: the group's y rows (MN-major SWIZZLE_128B B operand, K = rows)
            const uint32_t ia = smem_u32(sm.ident), yb = smem_u32(sm.stage[s] + gi * XYB);
            for (int kk = 0; kk < XROWS / 16; ++kk)
              mma_bf16(tmem + a * 64, sdesc(ia + kk * 32, 16, 1024), sdesc(yb + kk * 2 * kAtomBytes, kAtomBytes, kAtomBytes),
                       idesc, kk ? 1u : 0u);
          }
          for (int kk = 0; kk < g.rp / 16; ++kk) {
            const uint64_t ad = sdesc(va + (kk >> 2) * XYB + (kk & 3) * 32, 16, 1024);
            const uint64_t bd = sdesc(bb + gi * kAtomBytes + kk * 2 * g.G * kAtomBytes, kAtomBytes, g.G * kAtomBytes);
            mma_bf16(tmem + a * 64, ad, bd, idesc, (kIdY || kk) ? 1u : 0u);
          }
          mma_commit(&sm.tfull[a]);
        }
        __syncwarp();
      }
      const int vb = nrun & 1;
      XCursor nx = c;
      nx.next(p.n_jobs, g);
      const bool run_end = it + 1 == hi || nx.t != c.t || nx.h != c.h || nx.j != c.j;
      if (lane == 0) {
        mma_commit(&sm.empty[s]);
        if (run_end) mma_commit(&sm.vempty[vb]);
      }
      __syncwarp();
      c = nx;
      ++seq;
    }
    // drain: the commit arrivals above are asynchronous and must land before the CTA exits
    if (lane == 0) mma_commit(&sm.drain);
    __syncwarp();
    mbar_wait(&sm.drain, 0);
  } else {
    // ---------------------------------------------------------------- epilogue sets
    // set es (warps 2 + 4 es .. 5 + 4 es, one per TMEM lane quarter) takes the items with
    // (item - lo) % XSETS == es; every set walks the whole item stream for the cursors
    const int es = (warp - 2) >> 2;
    const int eq = warp & 3;                 // TMEM lane quarter of this warp
    const int r = eq * 32 + lane;            // item row (rows >= 64 are the UMMA's padding)
    const uint32_t lane_off = (uint32_t)(eq * 32) << 16;
    XCursor c{sm.t0, sm.h0, sm.j0, sm.cb0};
    int cur_t = -1, cur_h = -1, seq = 0, nacc = 0;
    int pend[XLAG + 1];                      // stages whose stores may still read them
#pragma unroll
    for (int i = 0; i <= XLAG; ++i) pend[i] = -1;
    int row = 0, row0 = 0, mh_cur = 0;
    bool box = false, valid = false;
    XGeom g{};
    for (int it = lo; it < hi; ++it) {
      const Tile& T = tl.t[c.t];
      if (c.t != cur_t) g = xgeom(p, T);
      if ((it - lo) % XSETS != es) {  // another set's item
        nacc += min(g.G, ngr - c.cb * g.G);
        c.next(p.n_jobs, g);
        ++seq;
        continue;
      }
      if (c.t != cur_t || c.h != cur_h) {
        const int mh = min(XROWS, T.m - c.h * XROWS);
        mh_cur = mh;
        valid = r < mh;
        row = __ldg(p.perm + T.pos0 + c.h * XROWS + min(r, mh - 1));
        row0 = __shfl_sync(0xffffffffu, row, 0);
        // one 32-row box store when the warp's rows are 32 consecutive valid tokens
        box = __all_sync(0xffffffffu, valid && row == row0 + lane);
        cur_t = c.t;
        cur_h = c.h;
      }
      const int s = seq % XNS;
      mbar_wait(&sm.full[s], (seq / XNS) & 1);
      if (eq == 0 && lane == 0) xtrace(p, it - lo, 2, gtimer());
      unsigned char* st = sm.stage[s];
      const int col0 = c.cb * g.G * 64;
      const int ng = min(g.G, ngr - c.cb * g.G);
      for (int gi = 0; gi < ng; ++gi, ++nacc) {
        const int a = nacc % XACC;
        mbar_wait(&sm.tfull[a], (nacc / XACC) & 1);
        tc_fence_after();
        float d0[32], d1[32];
        const bool wvalid = eq * 32 < mh_cur;  // warp-uniform: this quarter holds item rows
        if (!kIdY || wvalid) tmem_ld32x2(tmem + a * 64 + lane_off, d0, d1);
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&sm.tempty[a]);
        if (kIdY) {
          if (valid) {  // D = y + V . B in fp32: round once, back into the stage for the TMA store
            unsigned char* yr = st + gi * XYB;
#pragma unroll
            for (int ch = 0; ch < 8; ++ch) {
              const float* d = ch < 4 ? d0 + ch * 8 : d1 + (ch - 4) * 8;
              float f[8];
#pragma unroll
              for (int e = 0; e < 8; ++e) f[e] = d[e];
              *reinterpret_cast<uint4*>(yr + swz(r, ch)) = Elem<__nv_bfloat16>::pack(f);
            }
          }
          continue;
        }
        if (eq == 0 && lane == 0 && gi == 0) xtrace(p, it - lo, 7, gtimer());  // group 0's accumulator in registers
        if (valid && CHAM_PFX_EXP != 1) {
          unsigned char* yr = st + gi * XYB;
          uint4 yv[8];  // all eight 16-byte chunks of the row piece in flight at once
#pragma unroll
          for (int ch = 0; ch < 8; ++ch) yv[ch] = *reinterpret_cast<const uint4*>(yr + swz(r, ch));
#pragma unroll
          for (int ch = 0; ch < 8; ++ch) {
            float f[8];
            Elem<__nv_bfloat16>::unpack(yv[ch], f);
            const float* d = ch < 4 ? d0 + ch * 8 : d1 + (ch - 4) * 8;
#pragma unroll
            for (int e = 0; e < 8; ++e) f[e] += d[e];
            *reinterpret_cast<uint4*>(yr + swz(r, ch)) = Elem<__nv_bfloat16>::pack(f);
          }
        }
      }
      if (eq == 0 && lane == 0) xtrace(p, it - lo, 4, gtimer());
      // the generic-proxy y writes -> the TMA stores (async proxy) of this warp's rows
      fence_proxy_async_shared();
      __syncwarp();
      if (eq == 0 && lane == 0) xtrace(p, it - lo, 5, gtimer());
      if (box) {
        if (lane == 0)
          for (int gi = 0; gi < ng; ++gi)
            tma_store_2d(&p.maps[c.j].y32, col0 + gi * 64, row0, st + gi * XYB + eq * 32 * 128);
      } else if (valid) {
        for (int gi = 0; gi < ng; ++gi)
          tma_store_2d(&p.maps[c.j].y1, col0 + gi * 64, row, st + gi * XYB + r * 128);
      }
      bulk_commit();
      if (eq == 0 && lane == 0) xtrace(p, it - lo, 6, gtimer());
      if (CHAM_PFX_EXP == 2) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      // the stores of the item XLAG back have read their stage: release it
      asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(XLAG) : "memory");
#pragma unroll
      for (int i = XLAG; i > 0; --i) pend[i] = pend[i - 1];
      pend[0] = s;
      if (pend[XLAG] >= 0) mbar_arrive(&sm.empty[pend[XLAG]]);
      if (eq == 0 && lane == 0) xtrace(p, it - lo, 3, gtimer());
      c.next(p.n_jobs, g);
      ++seq;
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");  // every y store performed
  }
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem);
  }
}

}  // namespace prefill

namespace {
PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  }
  return fn;
}

// [rows x cols] bf16 row-major activation: boxes of 64 columns x box_rows rows, 128-byte swizzle
int encode_act_map(CUtensorMap* m, const void* base, int rows, int cols, int box_rows) {
  auto fn = encode_fn();
  if (!fn) return fail(CHAM_ERR_CUDA, "cuTensorMapEncodeTiled is unavailable");
  const cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  const cuuint64_t strides[1] = {(cuuint64_t)cols * 2};
  const cuuint32_t box[2] = {64, (cuuint32_t)box_rows};
  const cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(CHAM_ERR_CUDA, "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
  return CHAM_OK;
}
}  // namespace

// [rows x cols] fp32 row-major (row pitch `pitch` floats), unswizzled boxes of box_cols x
// box_rows: the decode kernel's TP v operand (one box = one page's 8 ranks of a token tile).
int encode_f32_map(CUtensorMap* m, const void* base, int rows, int cols, int pitch, int box_cols, int box_rows) {
  auto fn = encode_fn();
  if (!fn) return fail(CHAM_ERR_CUDA, "cuTensorMapEncodeTiled is unavailable");
  const cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  const cuuint64_t strides[1] = {(cuuint64_t)pitch * 4};
  const cuuint32_t box[2] = {(cuuint32_t)box_cols, (cuuint32_t)box_rows};
  const cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(base), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(CHAM_ERR_CUDA, "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
  return CHAM_OK;
}

// Launch the fused tcgen05 kernel for the prefill segments of this apply.
// mode: 0 fused, 1 shrink only (v_out, TP), 2 expand only (v_in, TP).
int prefill_launch(cham_pool* pool, int layer, int n_jobs, const int* projs, const void* const* xs,
                   void* const* ys, int n_tokens, const int* perm, const int* seg_off, const int* seg_slot,
                   const int* seg_rank, int n_seg, const int* n_seg_dev, void* stream, int mode, float* v_out,
                   const float* v_in, int v_stride) {
  using namespace prefill;
  static bool attr_set = false;
  if (!attr_set) {
    CHAM_CUDA(cudaFuncSetAttribute(fused_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(Shared)));
    CHAM_CUDA(cudaFuncSetAttribute(expand_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(XShared)));
    attr_set = true;
  }
  // fused mode as two launches: shrink-only fused kernel (V images), then expand_kernel
  const bool splitx = mode == MODE_FUSED && CHAM_PF_SPLITX;
  if (mode != MODE_FUSED && n_jobs != 1) return fail(CHAM_ERR_INVALID, "prefill shrink/expand take one projection");
  Params prm{};
  prm.base = pool->base;
  prm.page_bytes = (long long)pool->page_bytes;
  prm.n_pages = pool->n_pages;
  prm.n_tokens = n_tokens;
  prm.slot_pages = pool->d_slot_pages;
  prm.h_in = pool->h_in[projs[0]];
  prm.h_out = pool->h_out[projs[0]];
  prm.n_jobs = n_jobs;
  prm.mode = mode;
  prm.x_shared = 1;
  for (int j = 1; j < n_jobs; ++j)
    if (xs[j] != xs[0]) prm.x_shared = 0;
  for (int j = 0; j < n_jobs; ++j) {
    const int lp = layer * pool->n_proj + projs[j];
    prm.jobs[j].x = static_cast<const char*>(xs[j]);
    prm.jobs[j].y = static_cast<char*>(ys[j]);
    prm.jobs[j].a_off = (long long)pool->a_off[lp];
    prm.jobs[j].b_off = (long long)pool->b_off[lp];
  }
  // an unconditional row load: `perm ? perm[pos] : pos` would compile to a load merged with a
  // select that waits for the load where it is issued (one L2 round trip per loader unit)
  prm.perm = perm ? perm : pool->d_iota;
  prm.seg_off = seg_off;
  prm.seg_slot = seg_slot;
  prm.seg_rank = seg_rank;
  prm.n_seg = n_seg;
  prm.n_seg_dev = n_seg_dev;
  prm.thr = prefill_route_thr(pool);
  prm.epoch = ++pool->prefill_epoch;
  int* pc = pool->d_pctr + (prm.epoch & 1) * (kPrefillCtrSet);
  prm.zero_set = pool->d_pctr + ((prm.epoch + 1) & 1) * (kPrefillCtrSet);
  prm.zero_n = kPrefillCtrSet;
  prm.ctr = pc;
  prm.tile_cnt = pc + 4;
  prm.arrive = pc + 4 + kPrefillMaxTiles;
  prm.ppart = pool->d_ppart;
  prm.err = pool->d_ctr + 2;
  prm.vimg = pool->d_pvimg;
  prm.v_out = v_out;
  prm.v_in = v_in;
  prm.v_stride = v_stride;
  if (pool->d_trace) {  // second half of the debug buffer (the first is the decode kernel's)
    prm.trace = pool->d_trace + (size_t)pool->sm_count * pool->trace_cap * 8;
    prm.trace_cap = pool->trace_cap;
  }
  for (int j = 0; j < n_jobs; ++j) {
    int rc = CHAM_OK;
    if (mode != MODE_EXPAND) {
      rc = encode_act_map(&prm.maps[j].x64, xs[j], n_tokens, prm.h_in, 64);
      if (!rc) rc = encode_act_map(&prm.maps[j].x1, xs[j], n_tokens, prm.h_in, 1);
    }
    if (!rc && mode != MODE_SHRINK) {
      rc = encode_act_map(&prm.maps[j].y64, ys[j], n_tokens, prm.h_out, 64);
      if (!rc) rc = encode_act_map(&prm.maps[j].y1, ys[j], n_tokens, prm.h_out, 1);
      if (!rc && splitx) rc = encode_act_map(&prm.maps[j].y32, ys[j], n_tokens, prm.h_out, 32);
    }
    if (rc) return rc;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(pool->sm_count);
  cfg.blockDim = dim3(NTHREADS);
  cfg.dynamicSmemBytes = sizeof(Shared);
  cfg.stream = (cudaStream_t)stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = CHAM_PF_PDL ? 1 : 0;
  prm.no_expand = splitx ? 1 : 0;
  CHAM_CUDA(cudaLaunchKernelEx(&cfg, fused_kernel, prm));
  if (splitx) {
    cfg.blockDim = dim3(X_THREADS);
    cfg.dynamicSmemBytes = sizeof(XShared);
    CHAM_CUDA(cudaLaunchKernelEx(&cfg, expand_kernel, prm));
  }
  return CHAM_OK;
}

}  // namespace cham
