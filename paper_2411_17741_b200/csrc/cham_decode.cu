// cham_decode.cu — K1 (segmented shrink, h_in -> r) and K2 (segmented expand, r -> h_out,
// accumulated into y) for decode-sized segments: two persistent, warp-specialised kernels
// chained with programmatic dependent launch (PDL).
//
// Reference seam: CostModel.step_duration's LoRA term (engine.py:67-77) models
//   adapter_units = sum_decoders rank + sum_prefills rank * input_tokens
// as 0.155 us per rank*token (model.py:172); these kernels perform that work for real:
// for every token t of segment s, y[t] += (x[t] . A_slot(s)) . B_slot(s).
//
// Design:
//  * Work is cut into ~32 KiB items of adapter bytes.  K1 items = (job, tile, page,
//    k-chunk); K2 items = (job, tile, column chunk); a tile is <= 4 tokens of one segment.
//    CTA b owns the contiguous item range [b*N/G, (b+1)*N/G) and walks it with an
//    incremental decoder (no per-item search, division or atomic).
//  * Warp 0 is the producer: it decodes an item from a shared-memory plan (segments, page
//    ids and perm are cached in smem, so the loop never waits on L2) and issues 1-D bulk
//    async copies (TMA engine) into a 4-stage ring completing on mbarriers.  Weight tiles
//    (A or B pages) do not depend on the previous kernel and are issued before
//    griddepcontrol.wait; activations / v are issued after it.
//  * Two consumer groups of 4 warps take alternate stages.  K1: every thread owns 16-byte
//    k-columns of all 8 rank rows; fp32 FMAs; butterfly reduce-scatter across the warp;
//    cross-warp sum -> v partial (fp32) in a ping-pong workspace.  K2: the stage holds the
//    B atoms, the y rows and the tile's v partials; the group sums the k-chunk partials,
//    FMAs against B, reduces across the sibling lanes holding other pages, adds into the
//    staged y rows and stores y.  No separate elementwise kernel touches y.
//  * K1 -> K2 ordering is the kernel boundary (griddepcontrol.wait in K2 before it copies
//    v); no fences, flags or spin-waits inside either kernel.  Every CTA executes
//    griddepcontrol.wait before exiting, so grid n completes after grid n-1 and the
//    ping-pong v buffer of apply n-2 is free when apply n writes it.
#include "cham_pool.h"

namespace cham {
namespace decode {

constexpr int TG = 4;                       // tokens per tile
constexpr int NSTAGE = 4;
constexpr int ADAPTER_BYTES = 32768;        // adapter bytes per item
constexpr int PAGE_PAD = 16;                // K2: per-page skew to spread smem banks
constexpr int ACT_ROW_BYTES = ADAPTER_BYTES / kRowsPerPage;  // 4 KiB activations per token (K1)
static_assert(ACT_ROW_BYTES == kActRowBytes, "pool workspace geometry");
constexpr int Y_ROW_BYTES = 2048;           // K2: y bytes per token per item (<= 128 chunks)
constexpr int V_BYTES = 8192;               // K2: staged v partials per item
constexpr int K1_STAGE = ADAPTER_BYTES + TG * ACT_ROW_BYTES;
constexpr int K2_B_REGION = ADAPTER_BYTES + kMaxPagesPerSlot * PAGE_PAD;
constexpr int K2_STAGE = K2_B_REGION + TG * Y_ROW_BYTES + V_BYTES;
constexpr int NGROUP = 1;                   // one consumer group: 3 stages in flight ahead of it
constexpr int GROUP_WARPS = 8;
constexpr int MAX_NQ = Y_ROW_BYTES / 16;    // K2: 16-byte column chunks per item
constexpr int GROUP_THREADS = GROUP_WARPS * 32;
constexpr int NTHREADS = 32 + NGROUP * GROUP_THREADS;
constexpr int PLAN_SEGS = 512;              // segments per launch (plan lives in shared memory)
constexpr int PLAN_PAGES = 2048;            // page ids cached in shared memory (else from L2)
constexpr int PLAN_TOKENS = 2048;           // perm entries cached in shared memory (else from L2)
static_assert(PLAN_SEGS == kMaxSegments, "limits");

enum Mode { MODE_FUSED = 0, MODE_SHRINK = 1, MODE_EXPAND = 2 };
enum Kind { KIND_END = 0, KIND_SHRINK = 1, KIND_EXPAND = 2 };

struct Job {
  const char* x;
  char* y;
  long long a_off;
  long long b_off;
};

struct Params {
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
  int* ctr;        // [0] next item, [1] finished CTAs (per kernel); ctr[2] of the pool = error
  int* err;
  float* vws;      // this apply's buffer: [job][max_tokens][vws_kc][kMaxRank]
  int vws_kc;
  int max_tokens;
  const float* v_in;  // MODE_EXPAND: v [positions][v_stride] (kc = 1)
  int v_stride;
  unsigned long long* trace;  // debug: [cta][seq][4] globaltimer stamps (null = off)
  int trace_cap;
};

struct Meta {
  int kind, job, pos0, T, g, kc, np, col0, ncols, nq, p2, vrow;
  int rows[TG];
};

struct Plan {
  int sh_start[PLAN_SEGS + 1];
  int ex_start[PLAN_SEGS + 1];
  int seg_off[PLAN_SEGS + 1];
  int seg_pg[PLAN_SEGS + 1];  // prefix of pages per segment into `pages`
  int seg_sr[PLAN_SEGS];      // (slot << 9) | rank
  int ex_cost_start[PLAN_SEGS + 1];  // prefix of expand cost (B bytes / 128) per job
  uint16_t pages[PLAN_PAGES];
  uint16_t perm[PLAN_TOKENS];
  int scan[NTHREADS / 32][4];
  int totals[5];  // shrink items/job, expand items/job, tokens, pages, expand cost/job
};

template <int STAGE_BYTES, int SCRATCH_BYTES>
struct Shared {
  alignas(128) unsigned char stage[NSTAGE][STAGE_BYTES];
  alignas(16) unsigned char scratch[NGROUP][SCRATCH_BYTES];
  uint64_t full[NSTAGE];
  uint64_t empty[NSTAGE];
  Meta meta[NSTAGE];
  Plan plan;
  int last_cta;
};
using K1Shared = Shared<K1_STAGE, GROUP_WARPS * 32 * 4>;
using K2Shared = Shared<K2_STAGE, TG * kMaxRank * 4>;

__host__ __device__ inline int ceil_div(int a, int b) { return (a + b - 1) / b; }
__host__ __device__ inline int pow2ceil(int v) {
  int p = 1;
  while (p < v) p <<= 1;
  return p;
}
// K2 geometry for a segment with np pages: p2 = pow2ceil(np) sibling lanes share one
// 16-byte column chunk (one page each); nq column chunks per item.
__host__ __device__ inline int expand_p2(int np) { return pow2ceil(np); }
__host__ __device__ inline int expand_nq(int p2) { return min(MAX_NQ, 256 / p2); }

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch_dependents() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// Items per segment for K1 / K2, and the per-item K2 cost (B bytes / 128) used to
// balance the expand work across CTAs.
template <typename T>
__device__ __forceinline__ void plan_counts(const Params& p, int T_s, int rank, int& n_sh, int& n_ex,
                                            int& ex_cost) {
  constexpr int ES = Elem<T>::kBytes;
  constexpr int EPV = Elem<T>::kEPV;
  const int np = ceil_div(rank, kRowsPerPage);
  const int nt = ceil_div(T_s, TG);
  if (np == 0 || nt == 0) {
    n_sh = n_ex = ex_cost = 0;
    return;
  }
  const int nkc = ceil_div(p.h_in * ES, ACT_ROW_BYTES);
  const int nq = expand_nq(expand_p2(np));
  n_sh = nt * np * nkc;
  n_ex = nt * ceil_div(p.h_out, nq * EPV);
  ex_cost = np * nq;
}

// index of the last segment s with start[s] <= v (start non-decreasing, start[0] = 0)
__device__ __forceinline__ int seg_search(const int* start, int S, int v) {
  int lo = 0, hi = S;
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (start[mid] <= v) lo = mid; else hi = mid;
  }
  return lo;
}


// Reduce-scatter of NV (power of two <= 32) per-lane partial sums across a warp: returns
// the warp-wide sum of value index (lane >> (5 - log2 NV)).  Halving rounds first, then
// plain xor rounds once every lane holds a single value.
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

__host__ __device__ constexpr int cpow2(int v) { return v <= 1 ? 1 : 2 * cpow2((v + 1) / 2); }
__host__ __device__ constexpr int clog2(int v) { return v <= 1 ? 0 : 1 + clog2(v / 2); }

// Builds the launch plan in shared memory (all threads).  Returns false on overflow.
template <typename T>
__device__ bool build_plan(const Params& p, Plan& pl, int S) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int per = ceil_div(S, NTHREADS);
  const int s0 = min(S, tid * per), s1 = min(S, s0 + per);
  int lsh = 0, lex = 0, lpg = 0, lco = 0;
  for (int s = s0; s < s1; ++s) {
    const int o0 = p.seg_off[s], o1 = p.seg_off[s + 1];
    const int slot = p.seg_slot[s];
    const int rank = slot >= 0 ? min(p.seg_rank[s], kMaxRank) : 0;
    pl.seg_off[s] = o0;
    pl.seg_sr[s] = slot >= 0 ? ((slot << 9) | rank) : 0;
    int a, b, c;
    plan_counts<T>(p, o1 - o0, rank, a, b, c);
    lsh += a;
    lex += b;
    lpg += ceil_div(rank, kRowsPerPage);
    lco += b * c;
  }
  int ish = lsh, iex = lex, ipg = lpg, ico = lco;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int a = __shfl_up_sync(0xffffffffu, ish, o);
    const int b = __shfl_up_sync(0xffffffffu, iex, o);
    const int c = __shfl_up_sync(0xffffffffu, ipg, o);
    const int d = __shfl_up_sync(0xffffffffu, ico, o);
    if (lane >= o) { ish += a; iex += b; ipg += c; ico += d; }
  }
  if (lane == 31) { pl.scan[warp][0] = ish; pl.scan[warp][1] = iex; pl.scan[warp][2] = ipg; pl.scan[warp][3] = ico; }
  __syncthreads();
  int bsh = 0, bex = 0, bpg = 0, bco = 0;
  for (int w = 0; w < warp; ++w) {
    bsh += pl.scan[w][0]; bex += pl.scan[w][1]; bpg += pl.scan[w][2]; bco += pl.scan[w][3];
  }
  bsh += ish - lsh;
  bex += iex - lex;
  bpg += ipg - lpg;
  bco += ico - lco;
  for (int s = s0; s < s1; ++s) {
    const int rank = pl.seg_sr[s] & 511;
    int a, b, c;
    plan_counts<T>(p, p.seg_off[s + 1] - pl.seg_off[s], rank, a, b, c);
    pl.sh_start[s] = bsh;
    pl.ex_start[s] = bex;
    pl.seg_pg[s] = bpg;
    pl.ex_cost_start[s] = bco;
    bsh += a;
    bex += b;
    bpg += ceil_div(rank, kRowsPerPage);
    bco += b * c;
  }
  if (tid == NTHREADS - 1) {
    pl.sh_start[S] = bsh;
    pl.ex_start[S] = bex;
    pl.seg_pg[S] = bpg;
    pl.ex_cost_start[S] = bco;
    pl.totals[4] = bco;
    const int ntok = S > 0 ? p.seg_off[S] : 0;
    pl.seg_off[S] = ntok;
    pl.totals[0] = bsh;
    pl.totals[1] = bex;
    pl.totals[2] = ntok;
    pl.totals[3] = bpg;
  }
  __syncthreads();
  if (pl.totals[2] > p.max_tokens) return false;
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
  return true;
}

struct ItemPos {
  int job, s, local;
};
__device__ __forceinline__ ItemPos locate(const int* start, int per_job, int S, int item) {
  ItemPos ip;
  ip.job = item / per_job;
  const int rem = item - ip.job * per_job;
  ip.s = seg_search(start, S, rem);
  ip.local = rem - start[ip.s];
  return ip;
}

__device__ __forceinline__ int page_of(const Params& p, const Plan& pl, bool pages_smem, int s, int slot, int g) {
  return pages_smem ? (int)pl.pages[pl.seg_pg[s] + g] : __ldg(p.slot_pages + slot * kMaxPagesPerSlot + g);
}
__device__ __forceinline__ int row_of(const Params& p, const Plan& pl, bool perm_smem, int pos) {
  return perm_smem ? (int)pl.perm[pos] : (p.perm ? __ldg(p.perm + pos) : pos);
}

// Two END markers (one per consumer group) at sequence numbers seq and seq + 1.
template <class SH>
__device__ __forceinline__ void post_end(SH& sm, int seq) {
  for (int k = 0; k < NGROUP; ++k) {
    const int sq = seq + k, st = sq % NSTAGE;
    mbar_wait(&sm.empty[st], ((sq / NSTAGE) & 1) ^ 1);
    sm.meta[st].kind = KIND_END;
    mbar_arrive(&sm.full[st]);
  }
}

template <class SH>
__device__ __forceinline__ bool prologue(const Params& p, SH& sm, int& S_out) {
  const int tid = threadIdx.x;
  const int S = p.n_seg >= 0 ? p.n_seg : *p.n_seg_dev;
  S_out = S;
  if (S > PLAN_SEGS || S < 0) return false;
  if (tid == 0) {
    for (int i = 0; i < NSTAGE; ++i) {
      mbar_init(&sm.full[i], 1);
      mbar_init(&sm.empty[i], GROUP_THREADS);
    }
    fence_mbar_init();
  }
  return true;
}

__device__ __forceinline__ void abort_launch(const Params& p) {
  pdl_wait();
  if (threadIdx.x == 0 && blockIdx.x == 0) *p.err = CHAM_ERR_LIMIT;
}


// K1 consumer work for one item with NT (1..4) tokens: partial v rows [g*8, g*8+8) for
// k-chunk kc.  Releases the stage as soon as its shared memory has been read.
template <typename T, int NT>
__device__ __forceinline__ void shrink_item(const Params& p, const Meta& m, const unsigned char* st,
                                            uint64_t* empty_bar, float* red, int ct, int lane, int gw,
                                            int bar_id) {
  constexpr int ES = Elem<T>::kBytes;
  constexpr int EPV = Elem<T>::kEPV;
  constexpr int NP2 = EPV / 2;
  constexpr int NTR = cpow2(NT);                  // tokens padded to a power of two
  constexpr int NV = kRowsPerPage * NTR;          // values reduced per item
  float2 acc2[kRowsPerPage][NT];
#pragma unroll
  for (int j = 0; j < kRowsPerPage; ++j)
#pragma unroll
    for (int t = 0; t < NT; ++t) acc2[j][t] = make_float2(0.f, 0.f);
  const int kbytes = min(ACT_ROW_BYTES, p.h_in * ES - m.kc * ACT_ROW_BYTES);
  const int nqk = kbytes >> 4;
  const unsigned char* X = st + ADAPTER_BYTES;
  for (int q = ct; q < nqk; q += GROUP_THREADS) {
    const int a = q >> 3, c = q & 7;
    float2 xf[NT][NP2];
#pragma unroll
    for (int t = 0; t < NT; ++t) Elem<T>::unpack2(lds128(X + t * ACT_ROW_BYTES + q * 16), xf[t]);
#pragma unroll
    for (int j = 0; j < kRowsPerPage; ++j) {
      float2 af[NP2];
      Elem<T>::unpack2(lds128(st + a * kAtomBytes + j * kRowBytes + (((c ^ j) & 7) << 4)), af);
#pragma unroll
      for (int k = 0; k < NP2; ++k)
#pragma unroll
        for (int t = 0; t < NT; ++t) acc2[j][t] = __ffma2_rn(af[k], xf[t][k], acc2[j][t]);
    }
  }
  mbar_arrive(empty_bar);  // the stage has been read: hand it back to the producer
  float v[NV];
#pragma unroll
  for (int j = 0; j < kRowsPerPage; ++j)
#pragma unroll
    for (int t = 0; t < NTR; ++t) v[j * NTR + t] = t < NT ? acc2[j][t].x + acc2[j][t].y : 0.f;
  const float mine = warp_reduce_scatter<NV>(v, lane);
  constexpr int SHIFT = 5 - clog2(NV);
  named_bar_sync(bar_id, GROUP_THREADS);  // previous item's readers of `red` are done
  if ((lane & ((1 << SHIFT) - 1)) == 0) red[gw * 32 + (lane >> SHIFT)] = mine;
  named_bar_sync(bar_id, GROUP_THREADS);
  if (ct < NV) {
    float sum = 0.f;
#pragma unroll
    for (int w2 = 0; w2 < GROUP_WARPS; ++w2) sum += red[w2 * 32 + ct];
    const int j = ct / NTR, t = ct % NTR;
    if (t < NT)
      p.vws[(((long long)m.job * p.max_tokens + m.pos0 + t) * p.vws_kc + m.kc) * kMaxRank + m.g * kRowsPerPage + j] =
          sum;
  }
}

// K2 consumer work for one item with NT (1..4) tokens.
template <typename T, int NT>
__device__ __forceinline__ void expand_item(const Params& p, const Meta& m, const unsigned char* st, float* vs,
                                            int nkc, int ct, int bar_id) {
  constexpr int ES = Elem<T>::kBytes;
  constexpr int EPV = Elem<T>::kEPV;
  constexpr int NP2 = EPV / 2;
  const int rows = m.np * kRowsPerPage;
  const bool v_staged = m.vrow > 0;
  const int vrow = v_staged ? m.vrow : -m.vrow;
  named_bar_sync(bar_id, GROUP_THREADS);  // previous item's readers of vs are done
  const float* Vs = reinterpret_cast<const float*>(st + K2_B_REGION + TG * Y_ROW_BYTES);
  for (int idx = ct; idx < NT * rows; idx += GROUP_THREADS) {
    const int t = idx / rows, r = idx - t * rows;
    float sum = 0.f;
    if (r < vrow) {
      for (int k2 = 0; k2 < nkc; ++k2) {
        if (v_staged) {
          sum += Vs[(t * nkc + k2) * vrow + r];
        } else if (p.v_in) {
          sum += __ldg(p.v_in + (long long)(m.pos0 + t) * p.v_stride + r);
        } else {
          sum += __ldg(p.vws + (((long long)m.job * p.max_tokens + m.pos0 + t) * p.vws_kc + k2) * kMaxRank + r);
        }
      }
    }
    vs[t * kMaxRank + r] = sum;
  }
  named_bar_sync(bar_id, GROUP_THREADS);
  const int p2 = m.p2;
  const int gi = ct & (p2 - 1);
  const int q = ct / p2;  // threads with q >= nq idle in the FMA phase (rank-8 items)
  float2 acc[NT][NP2];
#pragma unroll
  for (int t = 0; t < NT; ++t)
#pragma unroll
    for (int k = 0; k < NP2; ++k) acc[t][k] = make_float2(0.f, 0.f);
  const bool active = q < m.nq && q * EPV < m.ncols;
  if (active) {
    const int a = q >> 3, c = q & 7;
    for (int g = gi; g < m.np; g += p2) {
      const unsigned char* Bg = st + g * (m.nq * kRowBytes + PAGE_PAD);
      float vv[NT][kRowsPerPage];  // v[t][g*8 .. g*8+7]: two 16-byte loads per token
#pragma unroll
      for (int t = 0; t < NT; ++t) {
        const float4 lo = *reinterpret_cast<const float4*>(vs + t * kMaxRank + g * kRowsPerPage);
        const float4 hi = *reinterpret_cast<const float4*>(vs + t * kMaxRank + g * kRowsPerPage + 4);
        vv[t][0] = lo.x; vv[t][1] = lo.y; vv[t][2] = lo.z; vv[t][3] = lo.w;
        vv[t][4] = hi.x; vv[t][5] = hi.y; vv[t][6] = hi.z; vv[t][7] = hi.w;
      }
#pragma unroll
      for (int j = 0; j < kRowsPerPage; ++j) {
        float2 bf[NP2];
        Elem<T>::unpack2(lds128(Bg + a * kAtomBytes + j * kRowBytes + (((c ^ j) & 7) << 4)), bf);
#pragma unroll
        for (int t = 0; t < NT; ++t) {
          const float2 v2 = make_float2(vv[t][j], vv[t][j]);
#pragma unroll
          for (int k = 0; k < NP2; ++k) acc[t][k] = __ffma2_rn(v2, bf[k], acc[t][k]);
        }
      }
    }
  }
  for (int o = 1; o < p2; o <<= 1) {
#pragma unroll
    for (int t = 0; t < NT; ++t)
#pragma unroll
      for (int k = 0; k < NP2; ++k) {
        acc[t][k].x += __shfl_xor_sync(0xffffffffu, acc[t][k].x, o);
        acc[t][k].y += __shfl_xor_sync(0xffffffffu, acc[t][k].y, o);
      }
  }
  if (active) {
    const unsigned char* Y = st + K2_B_REGION;
#pragma unroll
    for (int t = 0; t < NT; ++t) {
      // the p2 sibling lanes hold identical sums; lane gi stores tokens t == gi (mod p2)
      if ((t & (p2 - 1)) == gi) {
        float yf[EPV];
        Elem<T>::unpack(lds128(Y + t * Y_ROW_BYTES + q * 16), yf);
#pragma unroll
        for (int k = 0; k < NP2; ++k) {
          yf[2 * k] += acc[t][k].x;
          yf[2 * k + 1] += acc[t][k].y;
        }
        char* dst = p.jobs[m.job].y + ((long long)m.rows[t] * p.h_out + m.col0) * ES + q * 16;
        *reinterpret_cast<uint4*>(dst) = Elem<T>::pack(yf);
      }
    }
  }
}

// =========================================================================== K1: shrink
template <typename T>
__global__ void __launch_bounds__(NTHREADS, 1) lora_shrink_kernel(const __grid_constant__ Params p) {
  constexpr int ES = Elem<T>::kBytes;
  constexpr int EPV = Elem<T>::kEPV;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  K1Shared& sm = *reinterpret_cast<K1Shared*>(smem_raw);
  Plan& pl = sm.plan;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  int S;
  if (!prologue(p, sm, S) || !build_plan<T>(p, pl, S)) {
    abort_launch(p);
    return;
  }
  const int SH = pl.totals[0];
  const bool pages_smem = pl.totals[3] <= PLAN_PAGES;
  const bool perm_smem = pl.totals[2] <= PLAN_TOKENS;
  const int total = p.n_jobs * SH;
  const int nkc = ceil_div(p.h_in * ES, ACT_ROW_BYTES);
  const int natoms = p.h_in * ES / kRowBytes;

  if (warp == 0) {
    // ------------------------------------------------------------------ producer
    const uint64_t pol_w = policy_evict_first();  // weights: streamed once per step
    const uint64_t pol_x = policy_evict_last();   // x rows: re-read by every page item
    // this CTA's contiguous share of the item space, walked with an incremental decoder
    const int i0 = (int)((long long)total * blockIdx.x / gridDim.x);
    const int i1 = (int)((long long)total * (blockIdx.x + 1) / gridDim.x);
    int job = 0, s = 0, tile = 0, g = 0, kc = 0;
    int o0 = 0, Ts = 0, slot = 0, np = 0, nt = 0;
    auto load_seg = [&]() {
      o0 = pl.seg_off[s];
      Ts = pl.seg_off[s + 1] - o0;
      slot = pl.seg_sr[s] >> 9;
      np = ceil_div(pl.seg_sr[s] & 511, kRowsPerPage);
      nt = ceil_div(Ts, TG);
    };
    if (i0 < i1) {
      const ItemPos ip = locate(pl.sh_start, SH, S, i0);
      job = ip.job;
      s = ip.s;
      load_seg();
      const int per_tile = np * nkc;
      tile = ip.local / per_tile;
      const int r2 = ip.local - tile * per_tile;
      g = r2 / nkc;
      kc = r2 - g * nkc;
    }
    bool waited = false;
    int seq = 0;
    for (int item = i0; item < i1; ++item, ++seq) {
      const unsigned long long t_it = p.trace ? gtimer() : 0;
      const int stage = seq % NSTAGE;
      const int pos0 = o0 + tile * TG;
      const int tcount = min(TG, Ts - tile * TG);
      const int a0 = kc * (ADAPTER_BYTES / kAtomBytes);
      const uint32_t a_bytes = min(ADAPTER_BYTES / kAtomBytes, natoms - a0) * kAtomBytes;
      const uint32_t x_bytes = a_bytes / kRowsPerPage;
      const Job& jb = p.jobs[job];
      unsigned char* st = sm.stage[stage];
      int row = 0, pg = 0;
      if (lane < tcount) row = row_of(p, pl, perm_smem, pos0 + lane);
      if (lane == 0) pg = page_of(p, pl, pages_smem, s, slot, g);
      if (lane == 0) mbar_wait(&sm.empty[stage], ((seq / NSTAGE) & 1) ^ 1);
      const unsigned long long t_ready = p.trace ? gtimer() : 0;
      __syncwarp();
      Meta& m = sm.meta[stage];
      if (lane == 0) {
        m.kind = KIND_SHRINK; m.job = job; m.pos0 = pos0; m.T = tcount; m.g = g; m.kc = kc; m.np = np;
        mbar_arrive_expect_tx(&sm.full[stage], a_bytes + x_bytes * tcount);
        bulk_g2s(st, p.base + (long long)pg * p.page_bytes + jb.a_off + (long long)a0 * kAtomBytes, a_bytes,
                 &sm.full[stage], pol_w);
      }
      if (!waited) {  // x may be produced by the previous kernel
        pdl_wait();
        pdl_launch_dependents();
        waited = true;
      }
      if (lane < tcount) {
        const char* src = jb.x + ((long long)row * p.h_in + (long long)kc * (ACT_ROW_BYTES / ES)) * ES;
        bulk_g2s(st + ADAPTER_BYTES + lane * ACT_ROW_BYTES, src, x_bytes, &sm.full[stage], pol_x);
      }
      if (p.trace && lane == 0 && seq < p.trace_cap) {
        unsigned long long* tr = p.trace + ((long long)blockIdx.x * p.trace_cap + seq) * 8;
        tr[0] = gtimer();
        tr[1] = (1ull << 32) | (a_bytes + x_bytes * tcount);
        tr[4] = t_it;
        tr[5] = t_ready;
      }
      // advance (kc fastest, then page, tile, segment, job)
      if (++kc == nkc) {
        kc = 0;
        if (++g == np) {
          g = 0;
          if (++tile == nt) {
            tile = 0;
            do {
              if (++s == S) { s = 0; ++job; }
            } while (job < p.n_jobs && pl.sh_start[s + 1] == pl.sh_start[s]);
            if (job < p.n_jobs) load_seg();
          }
        }
      }
      __syncwarp();
    }
    if (!waited) pdl_wait();
    if (lane == 0) post_end(sm, seq);
  } else {
    // ------------------------------------------------------------------ consumers
    const int grp = (warp - 1) / GROUP_WARPS;
    const int ct = tid - 32 - grp * GROUP_THREADS;
    const int gw = ct >> 5;
    const int bar_id = 1 + grp;
    float* red = reinterpret_cast<float*>(sm.scratch[grp]);
    for (int seq = grp;; seq += NGROUP) {
      const int stage = seq % NSTAGE;
      mbar_wait(&sm.full[stage], (seq / NSTAGE) & 1);
      const Meta m = sm.meta[stage];
      if (m.kind == KIND_END) break;
      if (p.trace && ct == 0 && seq < p.trace_cap)
        p.trace[((long long)blockIdx.x * p.trace_cap + seq) * 8 + 2] = gtimer();
      const unsigned char* st = sm.stage[stage];
      switch (m.T) {
        case 1: shrink_item<T, 1>(p, m, st, &sm.empty[stage], red, ct, lane, gw, bar_id); break;
        case 2: shrink_item<T, 2>(p, m, st, &sm.empty[stage], red, ct, lane, gw, bar_id); break;
        case 3: shrink_item<T, 3>(p, m, st, &sm.empty[stage], red, ct, lane, gw, bar_id); break;
        default: shrink_item<T, 4>(p, m, st, &sm.empty[stage], red, ct, lane, gw, bar_id); break;
      }
      if (p.trace && ct == 0 && seq < p.trace_cap)
        p.trace[((long long)blockIdx.x * p.trace_cap + seq) * 8 + 3] = gtimer();
    }
  }
}

// =========================================================================== K2: expand
template <typename T>
__global__ void __launch_bounds__(NTHREADS, 1) lora_expand_kernel(const __grid_constant__ Params p) {
  constexpr int ES = Elem<T>::kBytes;
  constexpr int EPV = Elem<T>::kEPV;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  K2Shared& sm = *reinterpret_cast<K2Shared*>(smem_raw);
  Plan& pl = sm.plan;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  int S;
  if (!prologue(p, sm, S) || !build_plan<T>(p, pl, S)) {
    abort_launch(p);
    return;
  }
  const int EX = pl.totals[1];
  const bool pages_smem = pl.totals[3] <= PLAN_PAGES;
  const bool perm_smem = pl.totals[2] <= PLAN_TOKENS;
  const int total = p.n_jobs * EX;
  const int nkc = p.v_in ? 1 : ceil_div(p.h_in * ES, ACT_ROW_BYTES);

  if (warp == 0) {
    // ------------------------------------------------------------------ producer
    const uint64_t pol_stream = policy_evict_first();
    // this CTA's share of the expand work, balanced by bytes (rank-8 items carry half)
    const long long cost_job = pl.totals[4];
    auto item_at_cost = [&](long long c) -> int {
      if (cost_job == 0) return 0;
      const int jb = (int)(c / cost_job);
      if (jb >= p.n_jobs) return total;
      const int rem = (int)(c - jb * cost_job);
      const int sg = seg_search(pl.ex_cost_start, S, rem);
      int np_s, dummy1, dummy2, unit;
      plan_counts<T>(p, pl.seg_off[sg + 1] - pl.seg_off[sg], pl.seg_sr[sg] & 511, dummy1, np_s, unit);
      (void)dummy2;
      const int local = unit > 0 ? ceil_div(rem - pl.ex_cost_start[sg], unit) : 0;
      return jb * EX + pl.ex_start[sg] + min(local, np_s);
    };
    const long long cost_all = cost_job * p.n_jobs;
    const int i0 = item_at_cost(cost_all * blockIdx.x / gridDim.x);
    const int i1 = blockIdx.x + 1 == gridDim.x ? total : item_at_cost(cost_all * (blockIdx.x + 1) / gridDim.x);
    int job = 0, s = 0, tile = 0, cc = 0;
    int o0 = 0, Ts = 0, slot = 0, np = 0, nt = 0, p2 = 1, nq = 0, nc = 0, nexp = 0;
    auto load_seg = [&]() {
      o0 = pl.seg_off[s];
      Ts = pl.seg_off[s + 1] - o0;
      slot = pl.seg_sr[s] >> 9;
      np = ceil_div(pl.seg_sr[s] & 511, kRowsPerPage);
      nt = ceil_div(Ts, TG);
      p2 = expand_p2(np);
      nq = expand_nq(p2);
      nc = nq * EPV;
      nexp = ceil_div(p.h_out, nc);
    };
    if (i0 < i1) {
      const ItemPos ip = locate(pl.ex_start, EX, S, i0);
      job = ip.job;
      s = ip.s;
      load_seg();
      tile = ip.local / nexp;
      cc = ip.local - tile * nexp;
    }
    bool waited = false;
    int seq = 0;
    for (int item = i0; item < i1; ++item, ++seq) {
      const unsigned long long t_it = p.trace ? gtimer() : 0;
      const int stage = seq % NSTAGE;
      const int col0 = cc * nc;
      const int ncols = min(nc, p.h_out - col0);
      const int pos0 = o0 + tile * TG;
      const int tcount = min(TG, Ts - tile * TG);
      const uint32_t b_bytes = ncols * ES * kRowsPerPage;  // per page
      const uint32_t y_bytes = ncols * ES;                  // per token
      const int vrow = p.v_in ? min(np * kRowsPerPage, p.v_stride) : np * kRowsPerPage;  // floats per v row
      const uint32_t v_row_bytes = vrow * 4;
      const int nv = tcount * nkc;  // v rows staged
      const bool v_staged = nv * (int)v_row_bytes <= V_BYTES;
      const Job& jb = p.jobs[job];
      unsigned char* st = sm.stage[stage];
      int row = 0;
      if (lane < tcount) row = row_of(p, pl, perm_smem, pos0 + lane);
      if (lane == 0) mbar_wait(&sm.empty[stage], ((seq / NSTAGE) & 1) ^ 1);
      const unsigned long long t_ready = p.trace ? gtimer() : 0;
      __syncwarp();
      Meta& m = sm.meta[stage];
      if (lane == 0) {
        m.kind = KIND_EXPAND; m.job = job; m.pos0 = pos0; m.T = tcount; m.np = np; m.col0 = col0;
        m.ncols = ncols; m.nq = nq; m.p2 = p2; m.vrow = v_staged ? vrow : -vrow;
        mbar_arrive_expect_tx(&sm.full[stage], b_bytes * np + y_bytes * tcount + (v_staged ? nv * v_row_bytes : 0));
      }
      if (lane < tcount) m.rows[lane] = row;
      // weights and y rows do not depend on the shrink kernel: issue them first
      for (int c = lane; c < np; c += 32) {
        const int pgc = page_of(p, pl, pages_smem, s, slot, c);
        const char* src = p.base + (long long)pgc * p.page_bytes + jb.b_off +
                          (long long)(col0 * ES / kRowBytes) * kAtomBytes;
        bulk_g2s(st + c * (nq * kRowBytes + PAGE_PAD), src, b_bytes, &sm.full[stage], pol_stream);
      }
      if (lane < tcount)
        bulk_g2s(st + K2_B_REGION + lane * Y_ROW_BYTES, jb.y + ((long long)row * p.h_out + col0) * ES, y_bytes,
                 &sm.full[stage], pol_stream);
      if (!waited) {  // v is produced by the shrink kernel
        pdl_wait();
        pdl_launch_dependents();
        waited = true;
      }
      if (v_staged) {
        for (int c = lane; c < nv; c += 32) {
          const int t = c / nkc, k2 = c - t * nkc;
          const float* src = p.v_in ? p.v_in + (long long)(pos0 + t) * p.v_stride
                                    : p.vws + (((long long)job * p.max_tokens + pos0 + t) * p.vws_kc + k2) * kMaxRank;
          bulk_g2s(st + K2_B_REGION + TG * Y_ROW_BYTES + c * v_row_bytes, src, v_row_bytes, &sm.full[stage],
                   pol_stream);
        }
      }
      if (p.trace && lane == 0 && seq < p.trace_cap) {
        unsigned long long* tr = p.trace + ((long long)blockIdx.x * p.trace_cap + seq) * 8;
        tr[0] = gtimer();
        tr[1] = (2ull << 32) | (b_bytes * np + y_bytes * tcount + (v_staged ? nv * v_row_bytes : 0));
        tr[4] = t_it;
        tr[5] = t_ready;
      }
      // advance (column chunk fastest, then tile, segment, job)
      if (++cc == nexp) {
        cc = 0;
        if (++tile == nt) {
          tile = 0;
          do {
            if (++s == S) { s = 0; ++job; }
          } while (job < p.n_jobs && pl.ex_start[s + 1] == pl.ex_start[s]);
          if (job < p.n_jobs) load_seg();
        }
      }
      __syncwarp();
    }
    if (!waited) pdl_wait();
    if (lane == 0) post_end(sm, seq);
  } else {
    // ------------------------------------------------------------------ consumers
    const int grp = (warp - 1) / GROUP_WARPS;
    const int ct = tid - 32 - grp * GROUP_THREADS;
    const int bar_id = 1 + grp;
    float* vs = reinterpret_cast<float*>(sm.scratch[grp]);  // [TG][kMaxRank]
    for (int seq = grp;; seq += NGROUP) {
      const int stage = seq % NSTAGE;
      mbar_wait(&sm.full[stage], (seq / NSTAGE) & 1);
      const Meta m = sm.meta[stage];
      if (m.kind == KIND_END) break;
      if (p.trace && ct == 0 && seq < p.trace_cap)
        p.trace[((long long)blockIdx.x * p.trace_cap + seq) * 8 + 2] = gtimer();
      const unsigned char* st = sm.stage[stage];
      switch (m.T) {
        case 1: expand_item<T, 1>(p, m, st, vs, nkc, ct, bar_id); break;
        case 2: expand_item<T, 2>(p, m, st, vs, nkc, ct, bar_id); break;
        case 3: expand_item<T, 3>(p, m, st, vs, nkc, ct, bar_id); break;
        default: expand_item<T, 4>(p, m, st, vs, nkc, ct, bar_id); break;
      }
      if (p.trace && ct == 0 && seq < p.trace_cap)
        p.trace[((long long)blockIdx.x * p.trace_cap + seq) * 8 + 3] = gtimer();
      mbar_arrive(&sm.empty[stage]);
    }
  }
}

// TP shrink: fold the k-chunk partials of every grouped position into v_out [pos][v_stride].
__global__ void fold_partials_kernel(const float* __restrict__ vws, int vws_kc, int nkc,
                                     const int* __restrict__ seg_off, const int* __restrict__ seg_slot,
                                     const int* __restrict__ seg_rank, int n_seg, const int* __restrict__ n_seg_dev,
                                     float* __restrict__ v_out, int v_stride) {
  const int S = n_seg >= 0 ? n_seg : *n_seg_dev;
  for (int s = blockIdx.x; s < S; s += gridDim.x) {
    const int slot = seg_slot[s];
    const int rows = slot >= 0 ? min(ceil_div(min(seg_rank[s], kMaxRank), kRowsPerPage) * kRowsPerPage, v_stride) : 0;
    const int o0 = seg_off[s], o1 = seg_off[s + 1];
    for (int idx = threadIdx.x; idx < (o1 - o0) * rows; idx += blockDim.x) {
      const int t = idx / rows, r = idx - t * rows;
      const float* src = vws + ((long long)(o0 + t) * vws_kc) * kMaxRank + r;
      float sum = 0.f;
      for (int k = 0; k < nkc; ++k) sum += src[k * kMaxRank];
      v_out[(long long)(o0 + t) * v_stride + r] = sum;
    }
  }
}

template <typename KernelT>
int launch_pdl(KernelT kern, int smem, const cham_pool* pool, const Params& prm, cudaStream_t stream) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(pool->sm_count);
  cfg.blockDim = dim3(NTHREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  CHAM_CUDA(cudaLaunchKernelEx(&cfg, kern, prm));
  return CHAM_OK;
}

template <typename T>
int launch(cham_pool* pool, Params& prm, int mode, float* v_out, int v_stride, cudaStream_t stream) {
  static bool attr_set[2] = {false, false};
  auto k1 = lora_shrink_kernel<T>;
  auto k2 = lora_expand_kernel<T>;
  const int s1 = sizeof(K1Shared), s2 = sizeof(K2Shared);
  if (!attr_set[Elem<T>::kDtype]) {
    CHAM_CUDA(cudaFuncSetAttribute(k1, cudaFuncAttributeMaxDynamicSharedMemorySize, s1));
    CHAM_CUDA(cudaFuncSetAttribute(k2, cudaFuncAttributeMaxDynamicSharedMemorySize, s2));
    attr_set[Elem<T>::kDtype] = true;
  }
  // ping-pong v workspace: apply n uses buffer n % 2 (see the ordering argument above)
  const size_t buf_floats = (size_t)kMaxJobs * pool->max_tokens * pool->vws_kc * kMaxRank;
  Params p1 = prm;
  p1.vws = pool->d_vws + (pool->apply_count & 1) * buf_floats;
  p1.ctr = pool->d_ctr;
  p1.err = pool->d_ctr + 2;
  Params p2 = p1;
  p2.ctr = pool->d_ctr + 4;
  if (p2.trace) p2.trace += (size_t)pool->sm_count * p2.trace_cap * 8;  // K2 timeline in the second half
  ++pool->apply_count;
  if (mode != MODE_EXPAND) {
    int rc = launch_pdl(k1, s1, pool, p1, stream);
    if (rc) return rc;
  }
  if (mode == MODE_SHRINK) {
    fold_partials_kernel<<<pool->sm_count, 256, 0, stream>>>(
        p1.vws, p1.vws_kc, ceil_div(prm.h_in * (int)sizeof(T), ACT_ROW_BYTES), prm.seg_off, prm.seg_slot,
        prm.seg_rank, prm.n_seg, prm.n_seg_dev, v_out, v_stride);
    CHAM_CUDA(cudaGetLastError());
    return CHAM_OK;
  }
  return launch_pdl(k2, s2, pool, p2, stream);
}

}  // namespace decode

// Shared validation + parameter setup for the four entry points.
int decode_entry(cham_pool* pool, int layer, int n_jobs, const int* projs, const void* const* xs,
                 void* const* ys, int n_tokens, const int* perm, const int* seg_off, const int* seg_slot,
                 const int* seg_rank, int n_seg, const int* n_seg_dev, void* stream, int mode,
                 float* v_out, const float* v_in, int v_stride) {
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
  if (mode != MODE_FUSED && n_jobs != 1) return fail(CHAM_ERR_INVALID, "shrink/expand take one projection");
  if (v_in && (v_stride % 4)) return fail(CHAM_ERR_INVALID, "lora_expand: v_stride must be a multiple of 4");
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
    if (pool->h_in[pj] != prm.h_in || pool->h_out[pj] != prm.h_out)
      return fail(CHAM_ERR_INVALID, "lora_apply_multi: projections must share h_in and h_out");
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
  prm.vws_kc = pool->vws_kc;
  prm.max_tokens = pool->max_tokens;
  prm.v_in = v_in;
  prm.v_stride = v_stride;
  prm.trace = pool->d_trace;
  prm.trace_cap = pool->trace_cap;
  if (pool->dtype == CHAM_BF16)
    return launch<__nv_bfloat16>(pool, prm, mode, v_out, v_stride, (cudaStream_t)stream);
  return launch<float>(pool, prm, mode, v_out, v_stride, (cudaStream_t)stream);
}

}  // namespace cham
