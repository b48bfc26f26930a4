// cham_prefill.cu — K3: the tensor-core (tcgen05) path for prefill-sized segments.
//
// Reference seam: the prefill half of CostModel.step_duration's LoRA term (engine.py:67-77):
// a prefill contributes rank * input_tokens adapter units (engine.py:70, 75-76); these
// kernels perform that work for real, y[t] += (x[t] . A_slot) . B_slot, for every segment
// with at least `prefill_min_tokens` tokens (rank <= 128, bf16).
//
// Two launches per lora_apply (K3):
//  P1 shrink  unit = (job, 128-token tile, K-split):  D1[128 x rp] (TMEM, fp32) =
//             X_tile[128 x K/ks] . A^T[rp x K/ks]^T.  X arrives by TMA tensor loads (one
//             128-row box per 64-column stage when the tile's token rows are contiguous — the
//             rows of a prefill request are — else one 1-row box per token: a TMA gather),
//             A^T pages by 1 KiB bulk copies straight from the page layout, which already is
//             the K-major SWIZZLE_128B canonical layout.  The epilogue writes fp32 partial
//             v rows to a workspace (or, for the TP half, the final v to v_out).
//  P2 expand  unit = (job, tile, 512 output columns):  V = sum of the K-split partials,
//             rounded to bf16 into a K-major SWIZZLE_128B smem tile (zero beyond the rank);
//             per 64-column group D2[128 x 64] (TMEM) = V . B with the B page slices used as
//             MN-major SWIZZLE_128B operands (again the page layout itself); the y tile of the
//             group is TMA-loaded into the same stage, and the epilogue adds D2 and stores the
//             rows back — no separate elementwise kernel.
// Both kernels are persistent (one CTA per SM) and warp-specialised: warps 0-3 epilogue
// (TMEM lanes 0-127, one token row per thread), warp 4 loads (TMA), warp 5 issues the MMAs.
// Stage rings are mbarrier pipelines; TMEM accumulators are double-buffered so the epilogue
// of one unit overlaps the MMAs of the next.  The path is HBM-bound (AI ~15 flop/B at C3);
// tensor cores are used because the CUDA-core FMA ceiling (~51-74 TFLOP/s) is below what the
// HBM roofline demands.
#include <cuda.h>
#include <cudaTypedefs.h>

#include "cham_pool.h"

namespace cham {
namespace prefill {

constexpr int BM = 128;                 // tokens per tile (UMMA M)
constexpr int BK = 64;                  // shrink K elements per stage (one 128-byte swizzle atom)
constexpr int MAXR = kPrefillMaxRank;   // rank rows per adapter on this path
constexpr int S1 = 6;                   // shrink ring stages
constexpr int X_STAGE = BM * 128;       // 16 KiB
constexpr int A_STAGE = MAXR * 128;     // 16 KiB (one 1 KiB atom per page)
constexpr int BN = 64;                  // expand N per MMA group (one atom)
constexpr int NSUB = 8;                 // expand groups per unit (512 columns)
constexpr int S2 = 4;                   // expand ring stages
constexpr int B_STAGE = MAXR * 128;     // 16 KiB
constexpr int Y_STAGE = BM * 128;       // 16 KiB
constexpr int V_TILE = BM * MAXR * 2;   // 32 KiB
constexpr int NSEG = kMaxSegments;
constexpr int NTHREADS = 192;           // warps 0-3 epilogue, 4 loader, 5 MMA
constexpr int P1_TMEM = 256;            // two 128-column fp32 accumulators
constexpr int P2_TMEM = 128;            // two 64-column fp32 accumulators

struct Job {
  const char* x;
  char* y;
  long long a_off;
  long long b_off;
};

// Activation tensor maps of one job (x for P1, y for P2): a 64-column x 128-row box for
// contiguous tiles and a 64-column x 1-row box for gathered ones, both SWIZZLE_128B.
struct alignas(64) Maps {
  CUtensorMap tile;
  CUtensorMap row;
};

struct alignas(64) Params {
  Maps maps[kMaxJobs];
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
  int thr;             // routing threshold (segment tokens)
  int grid1;           // P1 grid size (the K-split factor is derived from it)
  int split_ok;        // 0: no K-split (TP shrink writes final v)
  float* vout;         // P1 output: [job][ks][pos][ld]
  const float* vin;    // P2 input
  long long v_job_stride, v_ks_stride;
  int ld;              // floats per v row
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
template <int COLS>
__device__ __forceinline__ void tmem_alloc(uint32_t* dst) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst)), "n"(COLS));
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
}
template <int COLS>
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "n"(COLS));
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
// 2-D TMA tensor load (box defined by the map) completing on an mbarrier
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar,
                                            uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint "
      "[%0], [%1, {%2, %3}], [%4], %5;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}
__device__ __forceinline__ void prefetch_map(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}
__device__ __forceinline__ void sts128(uint32_t addr, uint4 v) {
  asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};" ::"r"(addr), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
               : "memory");
}
__device__ __forceinline__ uint32_t swz(int row, int chunk) {  // 16-byte chunk of a 128-byte row
  return (uint32_t)(row * 128 + (((chunk ^ row) & 7) << 4));
}

// ------------------------------------------------------------------ tile list (per CTA)
struct TileList {
  int n_tiles;
  int n_pseg;
  int pseg[NSEG];          // prefill segment -> segment index
  int tstart[NSEG + 1];    // tile prefix over prefill segments
  int s_off[NSEG];
  int s_T[NSEG];
  int s_slot[NSEG];
  int s_rank[NSEG];
};

// All threads: read the segment table into smem, compact the prefill segments (stable),
// prefix their 128-token tile counts.  Deterministic: P1 and P2 derive the same list.
__device__ void build_tiles(const Params& p, TileList& tl) {
  const int tid = threadIdx.x, lane = tid & 31;
  int S = p.n_seg >= 0 ? p.n_seg : *p.n_seg_dev;
  S = max(0, min(S, NSEG));
  for (int s = tid; s < S; s += blockDim.x) {
    const int o0 = __ldg(p.seg_off + s), o1 = __ldg(p.seg_off + s + 1);
    tl.s_off[s] = o0;
    tl.s_T[s] = o1 - o0;
    tl.s_slot[s] = __ldg(p.seg_slot + s);
    tl.s_rank[s] = __ldg(p.seg_rank + s);
  }
  __syncthreads();
  if (tid < 32) {
    int cnt = 0, tiles = 0;
    for (int base = 0; base < S; base += 32) {
      const int s = base + lane;
      const bool f = s < S && tl.s_slot[s] >= 0 && is_prefill_segment(tl.s_T[s], tl.s_rank[s], p.thr);
      const unsigned m = __ballot_sync(0xffffffffu, f);
      const int nt = f ? (tl.s_T[s] + BM - 1) / BM : 0;
      int inc = nt;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int a = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += a;
      }
      if (f) {
        const int i = cnt + __popc(m & ((1u << lane) - 1));
        tl.pseg[i] = s;
        tl.tstart[i] = tiles + inc - nt;
      }
      cnt += __popc(m);
      tiles += __shfl_sync(0xffffffffu, inc, 31);
    }
    if (lane == 0) {
      tl.n_pseg = cnt;
      tl.n_tiles = tiles;
      tl.tstart[cnt] = tiles;
    }
  }
  __syncthreads();
}

// prefill-segment index owning tile t
__device__ __forceinline__ int tile_pseg(const TileList& tl, int t) {
  int lo = 0, hi = tl.n_pseg;
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (tl.tstart[mid] <= t) lo = mid; else hi = mid;
  }
  return lo;
}

__device__ __forceinline__ int choose_ks(const Params& p, int n_tiles) {
  const int nkc = p.h_in / BK;
  if (!p.split_ok) return 1;
  int ks = 1;
  // about four units per CTA: balances the tail without shrinking the K loops below 8 stages
  while (ks < kPrefillMaxSplit && n_tiles * p.n_jobs * ks < 4 * p.grid1 && nkc % (2 * ks) == 0 && nkc / (2 * ks) >= 8)
    ks *= 2;
  return ks;
}

struct Unit {
  int job, seg, row0, m, rank, rp, np, slot;
};
__device__ __forceinline__ Unit make_unit(const Params& p, const TileList& tl, int job, int t) {
  Unit u;
  const int i = tile_pseg(tl, t);
  u.job = job;
  u.seg = tl.pseg[i];
  const int tile_in_seg = t - tl.tstart[i];
  u.row0 = tl.s_off[u.seg] + tile_in_seg * BM;
  u.m = min(BM, tl.s_T[u.seg] - tile_in_seg * BM);
  u.rank = tl.s_rank[u.seg];
  u.rp = (u.rank + 15) & ~15;
  u.np = (u.rank + kRowsPerPage - 1) / kRowsPerPage;
  u.slot = tl.s_slot[u.seg];
  return u;
}

// Token rows of a unit's tile as seen by the loader warp: lane l holds rows l, l+32, l+64,
// l+96 (perm applied); `contig` = the m rows are consecutive (one TMA box per stage).
struct TileRows {
  int row[4];
  int first;
  bool contig;
};
__device__ __forceinline__ TileRows tile_rows(const Params& p, int row0, int m, int lane) {
  TileRows t;
  bool ok = true;
  t.first = p.perm ? __ldg(p.perm + row0) : row0;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int r = lane + 32 * i;
    const int pos = row0 + min(r, m - 1);
    t.row[i] = p.perm ? __ldg(p.perm + pos) : pos;
    if (r < m) ok &= t.row[i] == t.first + r;
  }
  t.contig = __all_sync(0xffffffffu, ok);
  return t;
}

// Loader-warp helper: one activation stage (64 columns at c0) of the tile into smem.
__device__ __forceinline__ void load_act(const Maps& mp, const TileRows& tr, int m, int c0, unsigned char* dst,
                                         uint64_t* bar, uint64_t pol, int lane) {
  if (tr.contig) {
    if (lane == 0) tma_load_2d(dst, &mp.tile, c0, tr.first, bar, pol);
  } else {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int r = lane + 32 * i;
      if (r < m) tma_load_2d(dst + r * 128, &mp.row, c0, tr.row[i], bar, pol);
    }
  }
}
__device__ __forceinline__ uint32_t act_bytes(const TileRows& tr, int m) { return tr.contig ? BM * 128 : m * 128; }

// =========================================================================== P1: shrink
struct P1Shared {
  alignas(1024) unsigned char x[S1][X_STAGE];
  alignas(1024) unsigned char a[S1][A_STAGE];
  uint64_t full[S1], empty[S1], tfull[2], tempty[2];
  uint32_t tmem_base;
  TileList tl;
};

__global__ void __launch_bounds__(NTHREADS, 1) shrink_kernel(const __grid_constant__ Params p) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  P1Shared& sm = *reinterpret_cast<P1Shared*>(smem_raw);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int i = 0; i < S1; ++i) {
      mbar_init(&sm.full[i], 1);
      mbar_init(&sm.empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&sm.tfull[i], 1);
      mbar_init(&sm.tempty[i], 128);
    }
    fence_mbar_init();
  }
  if (warp == 4 && lane < p.n_jobs) {
    prefetch_map(&p.maps[lane].tile);
    prefetch_map(&p.maps[lane].row);
  }
  if (warp == 5) {
    tmem_alloc<P1_TMEM>(&sm.tmem_base);
    tc_fence_before();
  }
  build_tiles(p, sm.tl);  // contains __syncthreads
  tc_fence_after();
  const uint32_t tmem = sm.tmem_base;
  const int n_tiles = sm.tl.n_tiles;
  const int ks = choose_ks(p, n_tiles);
  const int nkc = p.h_in / BK / ks;  // stages per unit
  const int n_units = n_tiles * ks * p.n_jobs;

  if (warp == 4) {
    // ---------------- loader: X by TMA tensor loads, A^T by 1 KiB page bulk copies
    const uint64_t pol_w = policy_evict_first();
    const uint64_t pol_x = policy_evict_last();  // the other jobs of the tile re-read x from L2
    int seq = 0;
    for (int uu = blockIdx.x; uu < n_units; uu += gridDim.x) {
      const int job = uu % p.n_jobs, rem = uu / p.n_jobs;
      const Unit u = make_unit(p, sm.tl, job, rem / ks);
      const int kq = rem % ks;
      const TileRows tr = tile_rows(p, u.row0, u.m, lane);
      const char* blk0 = p.base + p.jobs[job].a_off;
      const long long pg = lane < u.np ? (long long)__ldg(p.slot_pages + u.slot * kMaxPagesPerSlot + lane) : 0;
      const uint32_t bytes = act_bytes(tr, u.m) + u.np * kAtomBytes;
      for (int k = 0; k < nkc; ++k, ++seq) {
        const int st = seq % S1;
        if (seq >= S1) mbar_wait(&sm.empty[st], ((seq / S1) - 1) & 1);
        if (lane == 0) mbar_arrive_expect_tx(&sm.full[st], bytes);
        __syncwarp();
        const int kc = kq * nkc + k;
        load_act(p.maps[job], tr, u.m, kc * BK, sm.x[st], &sm.full[st], pol_x, lane);
        if (lane < u.np)
          bulk_g2s(sm.a[st] + lane * kAtomBytes, blk0 + pg * p.page_bytes + (long long)kc * kAtomBytes, kAtomBytes,
                   &sm.full[st], pol_w);
      }
    }
  } else if (warp == 5) {
    // ---------------- MMA issuer
    int seq = 0, ui = 0;
    for (int uu = blockIdx.x; uu < n_units; uu += gridDim.x, ++ui) {
      const int job = uu % p.n_jobs, rem = uu / p.n_jobs;
      const Unit u = make_unit(p, sm.tl, job, rem / ks);
      const int acc = ui & 1;
      if (ui >= 2) mbar_wait(&sm.tempty[acc], ((ui >> 1) - 1) & 1);
      tc_fence_after();
      const uint32_t idesc = idesc_bf16(BM, u.rp, false);
      const uint32_t d = tmem + acc * 128;
      for (int k = 0; k < nkc; ++k, ++seq) {
        const int st = seq % S1;
        mbar_wait(&sm.full[st], (seq / S1) & 1);
        tc_fence_after();
        if (lane == 0) {
          const uint32_t xa = smem_u32(sm.x[st]), aa = smem_u32(sm.a[st]);
#pragma unroll
          for (int j = 0; j < BK / 16; ++j) {
            const uint64_t ad = sdesc(xa + j * 32, 16, 1024);
            const uint64_t bd = sdesc(aa + j * 32, 16, kAtomBytes);
            mma_bf16(d, ad, bd, idesc, (k | j) ? 1u : 0u);
          }
          mma_commit(&sm.empty[st]);
          if (k == nkc - 1) mma_commit(&sm.tfull[acc]);
        }
        __syncwarp();
      }
    }
  } else {
    // ---------------- epilogue warps 0-3: TMEM -> fp32 partial v rows
    int ui = 0;
    for (int uu = blockIdx.x; uu < n_units; uu += gridDim.x, ++ui) {
      const int job = uu % p.n_jobs, rem = uu / p.n_jobs;
      const Unit u = make_unit(p, sm.tl, job, rem / ks);
      const int kq = rem % ks;
      const int acc = ui & 1;
      mbar_wait(&sm.tfull[acc], (ui >> 1) & 1);
      tc_fence_after();
      const int r = warp * 32 + lane;
      float* dst = p.vout + job * p.v_job_stride + kq * p.v_ks_stride + (long long)(u.row0 + r) * p.ld;
      for (int c0 = 0; c0 < u.rank; c0 += 32) {
        float v[32];
        tmem_ld32(tmem + acc * 128 + c0 + ((uint32_t)(warp * 32) << 16), v);
        if (r < u.m) {
#pragma unroll
          for (int i = 0; i < 32; i += 4)
            if (c0 + i < u.rank) *reinterpret_cast<float4*>(dst + c0 + i) = make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]);
        }
      }
      tc_fence_before();
      mbar_arrive(&sm.tempty[acc]);
    }
  }
  __syncthreads();
  if (warp == 5) {
    tc_fence_after();
    tmem_dealloc<P1_TMEM>(tmem);
  }
}

// =========================================================================== P2: expand
struct P2Shared {
  alignas(1024) unsigned char v[2][V_TILE];
  alignas(1024) unsigned char b[S2][B_STAGE];
  alignas(1024) unsigned char y[S2][Y_STAGE];
  uint64_t full[S2], empty[S2], vfull[2], vempty[2], tfull[2], tempty[2];
  uint32_t tmem_base;
  TileList tl;
};

__global__ void __launch_bounds__(NTHREADS, 1) expand_kernel(const __grid_constant__ Params p) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  P2Shared& sm = *reinterpret_cast<P2Shared*>(smem_raw);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int i = 0; i < S2; ++i) {
      mbar_init(&sm.full[i], 1);
      mbar_init(&sm.empty[i], 1 + 128);  // MMA commit (B read) + 128 epilogue threads (y read)
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&sm.vfull[i], 128);
      mbar_init(&sm.vempty[i], 1);
      mbar_init(&sm.tfull[i], 1);
      mbar_init(&sm.tempty[i], 128);
    }
    fence_mbar_init();
  }
  if (warp == 4 && lane < p.n_jobs) {
    prefetch_map(&p.maps[lane].tile);
    prefetch_map(&p.maps[lane].row);
  }
  if (warp == 5) {
    tmem_alloc<P2_TMEM>(&sm.tmem_base);
    tc_fence_before();
  }
  build_tiles(p, sm.tl);
  tc_fence_after();
  const uint32_t tmem = sm.tmem_base;
  const int n_tiles = sm.tl.n_tiles;
  const int ks = choose_ks(p, n_tiles);
  const int ncols_unit = NSUB * BN;
  const int nq = (p.h_out + ncols_unit - 1) / ncols_unit;
  const int n_units = n_tiles * nq * p.n_jobs;

  if (warp == 4) {
    // ---------------- loader: per 64-column group, one 1 KiB B slice per page + the y tile
    const uint64_t pol_w = policy_evict_first();
    const uint64_t pol_y = policy_evict_last();  // written back right after
    int seq = 0;
    for (int uu = blockIdx.x; uu < n_units; uu += gridDim.x) {
      const int job = uu / (n_tiles * nq), rem = uu % (n_tiles * nq);
      const Unit u = make_unit(p, sm.tl, job, rem / nq);
      const int n0 = (rem % nq) * ncols_unit;
      const int nsub = min(NSUB, (p.h_out - n0) / BN);
      const TileRows tr = tile_rows(p, u.row0, u.m, lane);
      const char* blk0 = p.base + p.jobs[job].b_off;
      const long long pg = lane < u.np ? (long long)__ldg(p.slot_pages + u.slot * kMaxPagesPerSlot + lane) : 0;
      const bool pad = u.rp / kRowsPerPage > u.np;  // odd page count: zero pad page (K rows rank..rp)
      const uint32_t bytes = act_bytes(tr, u.m) + u.np * kAtomBytes;
      for (int c = 0; c < nsub; ++c, ++seq) {
        const int st = seq % S2;
        if (seq >= S2) mbar_wait(&sm.empty[st], ((seq / S2) - 1) & 1);
        if (pad) {
          uint4* z = reinterpret_cast<uint4*>(sm.b[st] + u.np * kAtomBytes);
          z[lane] = make_uint4(0, 0, 0, 0);
          z[lane + 32] = make_uint4(0, 0, 0, 0);
          fence_proxy_async_shared();
        }
        __syncwarp();
        if (lane == 0) mbar_arrive_expect_tx(&sm.full[st], bytes);
        __syncwarp();
        const int col = n0 + c * BN;
        if (lane < u.np)
          bulk_g2s(sm.b[st] + lane * kAtomBytes, blk0 + pg * p.page_bytes + (long long)(col / 64) * kAtomBytes,
                   kAtomBytes, &sm.full[st], pol_w);
        load_act(p.maps[job], tr, u.m, col, sm.y[st], &sm.full[st], pol_y, lane);
      }
    }
  } else if (warp == 5) {
    // ---------------- MMA issuer
    int seq = 0, gi = 0, ui = 0;
    const uint32_t idesc = idesc_bf16(BM, BN, true);
    for (int uu = blockIdx.x; uu < n_units; uu += gridDim.x, ++ui) {
      const int job = uu / (n_tiles * nq), rem = uu % (n_tiles * nq);
      const Unit u = make_unit(p, sm.tl, job, rem / nq);
      const int n0 = (rem % nq) * ncols_unit;
      const int nsub = min(NSUB, (p.h_out - n0) / BN);
      const int vb = ui & 1;
      mbar_wait(&sm.vfull[vb], (ui >> 1) & 1);
      tc_fence_after();
      for (int c = 0; c < nsub; ++c, ++seq, ++gi) {
        const int st = seq % S2, acc = gi & 1;
        if (gi >= 2) mbar_wait(&sm.tempty[acc], ((gi >> 1) - 1) & 1);
        mbar_wait(&sm.full[st], (seq / S2) & 1);
        tc_fence_after();
        if (lane == 0) {
          const uint32_t va = smem_u32(sm.v[vb]), ba = smem_u32(sm.b[st]);
          for (int j = 0; j < u.rp / 16; ++j) {
            const uint64_t ad = sdesc(va + (j >> 2) * (BM * 128) + (j & 3) * 32, 16, 1024);
            const uint64_t bd = sdesc(ba + j * 2 * kAtomBytes, kAtomBytes, kAtomBytes);
            mma_bf16(tmem + acc * BN, ad, bd, idesc, j ? 1u : 0u);
          }
          mma_commit(&sm.empty[st]);
          mma_commit(&sm.tfull[acc]);
          if (c == nsub - 1) mma_commit(&sm.vempty[vb]);
        }
        __syncwarp();
      }
    }
  } else {
    // ---------------- warps 0-3: build V (bf16, swizzled), then y += D2 per group
    const int r = warp * 32 + lane;  // tile row == TMEM lane
    int seq = 0, gi = 0, ui = 0;
    for (int uu = blockIdx.x; uu < n_units; uu += gridDim.x, ++ui) {
      const int job = uu / (n_tiles * nq), rem = uu % (n_tiles * nq);
      const Unit u = make_unit(p, sm.tl, job, rem / nq);
      const int n0 = (rem % nq) * ncols_unit;
      const int nsub = min(NSUB, (p.h_out - n0) / BN);
      const int vb = ui & 1;
      const bool valid = r < u.m;
      const int pos = u.row0 + min(r, u.m - 1);
      const int row = p.perm ? __ldg(p.perm + pos) : pos;
      if (ui >= 2) mbar_wait(&sm.vempty[vb], ((ui >> 1) - 1) & 1);
      {
        const float* vsrc = p.vin + job * p.v_job_stride + (long long)pos * p.ld;
        const uint32_t vbase = smem_u32(sm.v[vb]);
        for (int cj = 0; cj < u.rp / 8; ++cj) {
          float f[8];
#pragma unroll
          for (int i = 0; i < 8; ++i) f[i] = 0.f;
          if (valid && cj * 8 < u.rank) {
            for (int kq = 0; kq < ks; ++kq) {
              const float4 lo = *reinterpret_cast<const float4*>(vsrc + kq * p.v_ks_stride + cj * 8);
              const float4 hi = *reinterpret_cast<const float4*>(vsrc + kq * p.v_ks_stride + cj * 8 + 4);
              f[0] += lo.x; f[1] += lo.y; f[2] += lo.z; f[3] += lo.w;
              f[4] += hi.x; f[5] += hi.y; f[6] += hi.z; f[7] += hi.w;
            }
#pragma unroll
            for (int i = 0; i < 8; ++i)
              if (cj * 8 + i >= u.rank) f[i] = 0.f;
          }
          const uint4 w = make_uint4(pack_bf16x2(f[0], f[1]), pack_bf16x2(f[2], f[3]), pack_bf16x2(f[4], f[5]),
                                     pack_bf16x2(f[6], f[7]));
          sts128(vbase + (cj >> 3) * (BM * 128) + swz(r, cj & 7), w);
        }
      }
      fence_proxy_async_shared();
      mbar_arrive(&sm.vfull[vb]);
      char* yrow = p.jobs[job].y + (long long)row * p.h_out * 2;
      for (int c = 0; c < nsub; ++c, ++seq, ++gi) {
        const int st = seq % S2, acc = gi & 1;
        const int col0 = n0 + c * BN;
        mbar_wait(&sm.tfull[acc], (gi >> 1) & 1);
        tc_fence_after();
        float d0[32], d1[32];
        const uint32_t ta = tmem + acc * BN + ((uint32_t)(warp * 32) << 16);
        tmem_ld32(ta, d0);
        tmem_ld32(ta + 32, d1);
        tc_fence_before();
        mbar_arrive(&sm.tempty[acc]);
        mbar_wait(&sm.full[st], (seq / S2) & 1);  // the y tile of this group has landed
        uint4 yv[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) yv[i] = lds128(sm.y[st] + swz(r, i));
        mbar_arrive(&sm.empty[st]);
        if (valid) {
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const float* d = i < 4 ? d0 + i * 8 : d1 + (i - 4) * 8;
            float f[8];
            Elem<__nv_bfloat16>::unpack(yv[i], f);
#pragma unroll
            for (int e = 0; e < 8; ++e) f[e] += d[e];
            *reinterpret_cast<uint4*>(yrow + (col0 + i * 8) * 2) = Elem<__nv_bfloat16>::pack(f);
          }
        }
      }
    }
  }
  __syncthreads();
  if (warp == 5) {
    tc_fence_after();
    tmem_dealloc<P2_TMEM>(tmem);
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

// Launch P1 (unless mode == expand-only) and P2 (unless mode == shrink-only) for the
// prefill segments of this apply.  mode: 0 fused, 1 shrink (v_out), 2 expand (v_in).
int prefill_launch(cham_pool* pool, int layer, int n_jobs, const int* projs, const void* const* xs,
                   void* const* ys, int n_tokens, const int* perm, const int* seg_off, const int* seg_slot,
                   const int* seg_rank, int n_seg, const int* n_seg_dev, void* stream, int mode, float* v_out,
                   const float* v_in, int v_stride) {
  using namespace prefill;
  static bool attr_set = false;
  if (!attr_set) {
    CHAM_CUDA(cudaFuncSetAttribute(shrink_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(P1Shared)));
    CHAM_CUDA(cudaFuncSetAttribute(expand_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(P2Shared)));
    attr_set = true;
  }
  Params prm{};
  prm.base = pool->base;
  prm.page_bytes = (long long)pool->page_bytes;
  prm.slot_pages = pool->d_slot_pages;
  prm.h_in = pool->h_in[projs[0]];
  prm.h_out = pool->h_out[projs[0]];
  prm.n_jobs = n_jobs;
  for (int j = 0; j < n_jobs; ++j) {
    const int lp = layer * pool->n_proj + projs[j];
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
  prm.thr = prefill_route_thr(pool);
  prm.grid1 = pool->sm_count;
  cudaStream_t s = (cudaStream_t)stream;
  if (mode == 0) {
    prm.split_ok = 1;
    prm.ld = MAXR;
    prm.v_ks_stride = (long long)pool->max_tokens * MAXR;
    prm.v_job_stride = prm.v_ks_stride * kPrefillMaxSplit;
    prm.vout = pool->d_pws;
    prm.vin = pool->d_pws;
  } else {
    prm.split_ok = 0;
    prm.ld = v_stride;
    prm.v_ks_stride = 0;
    prm.v_job_stride = 0;
    prm.vout = v_out;
    prm.vin = v_in;
  }
  if (mode != 2) {
    for (int j = 0; j < n_jobs; ++j) {
      int rc = encode_act_map(&prm.maps[j].tile, xs[j], n_tokens, prm.h_in, BM);
      if (!rc) rc = encode_act_map(&prm.maps[j].row, xs[j], n_tokens, prm.h_in, 1);
      if (rc) return rc;
    }
    shrink_kernel<<<pool->sm_count, NTHREADS, sizeof(P1Shared), s>>>(prm);
    CHAM_CUDA(cudaGetLastError());
  }
  if (mode != 1) {
    for (int j = 0; j < n_jobs; ++j) {
      int rc = encode_act_map(&prm.maps[j].tile, ys[j], n_tokens, prm.h_out, BM);
      if (!rc) rc = encode_act_map(&prm.maps[j].row, ys[j], n_tokens, prm.h_out, 1);
      if (rc) return rc;
    }
    expand_kernel<<<pool->sm_count, NTHREADS, sizeof(P2Shared), s>>>(prm);
    CHAM_CUDA(cudaGetLastError());
  }
  return CHAM_OK;
}

}  // namespace cham
