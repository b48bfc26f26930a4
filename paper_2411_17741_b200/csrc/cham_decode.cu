// cham_decode.cu — K1+K2: fused segmented shrink (h_in -> r) and expand (r -> h_out, +=
// into y) for decode-sized segments, as ONE persistent warp-specialised kernel.
//
// Reference seam: CostModel.step_duration's LoRA term (engine.py:67-77) models
//   adapter_units = sum_decoders rank + sum_prefills rank * input_tokens
// as 0.155 us per rank*token (model.py:172); this kernel performs that work for real:
// for every token t of segment s, y[t] += (x[t] . A_slot(s)) . B_slot(s).
//
// Design:
//  * Work is cut into ~32 KiB "items" of adapter bytes: shrink items (tile, page, k-chunk)
//    and expand items (tile, column chunk); a tile is <= 4 tokens of one segment.  All
//    shrink items precede all expand items; CTA b runs items b, b+G, b+2G, ... in order.
//  * Warp 0 is the producer: it decodes an item from a shared-memory plan and issues 1-D
//    bulk async copies (TMA engine) of the adapter atoms and the tile's activation rows
//    into a 4-stage ring, completing on mbarriers.
//  * Two consumer groups of 4 warps take alternate stages.  Shrink: every thread owns
//    16-byte k-columns of all 8 rank rows, fp32 FMAs, butterfly reduce-scatter across the
//    warp, cross-warp sum -> v partial in a global workspace, then a release-increment of
//    the tile's counter.  Expand: wait (acquire) until the tile's shrink items are done,
//    sum the k-chunk partials into shared memory, FMA against the B atoms, reduce across
//    the pages held by sibling lanes, add into the y rows staged by the producer and store.
//    No separate elementwise kernel touches y.
//  * Deadlock freedom: a CTA processes its items in increasing order and every expand item
//    is numbered after every shrink item, so the shrink items an expand waits for are
//    already in flight in their own CTA and never wait on anything.
#include "cham_pool.h"

namespace cham {
namespace decode {

constexpr int TG = 4;                       // tokens per tile
constexpr int NSTAGE = 4;
constexpr int ADAPTER_BYTES = 32768;        // adapter bytes per item
constexpr int PAGE_PAD = 16;                // expand: per-page skew to spread smem banks
constexpr int ADAPTER_REGION = ADAPTER_BYTES + kMaxPagesPerSlot * PAGE_PAD;
constexpr int ACT_ROW_BYTES = ADAPTER_BYTES / kRowsPerPage;  // 4 KiB activations per token
static_assert(ACT_ROW_BYTES == kActRowBytes, "pool workspace geometry");
constexpr int STAGE_BYTES = ADAPTER_REGION + TG * ACT_ROW_BYTES;
constexpr int NGROUP = 2;
constexpr int GROUP_WARPS = 4;
constexpr int GROUP_THREADS = GROUP_WARPS * 32;
constexpr int NTHREADS = 32 + NGROUP * GROUP_THREADS;
constexpr int PLAN_SEGS = 512;              // segments per launch (plan lives in shared memory)
constexpr int PLAN_PAGES = 2048;            // page ids cached in shared memory (else read from L2)
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
  int* ctr;        // [1] finished CTAs, [2] error flag
  int* tile_done;  // [job][max_tokens]
  float* vws;      // [job][max_tokens][vws_kc][kMaxRank]
  int vws_kc;
  int max_tokens;
  int mode;
  float* v_out;       // MODE_SHRINK
  const float* v_in;  // MODE_EXPAND
  int v_stride;
  unsigned long long* trace;  // debug: [cta][seq][4] globaltimer stamps (null = off)
  int trace_cap;
};

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

struct Meta {
  int kind, job, pos0, T, g, kc, np, col0, ncols, nq, p2, need;
  int rows[TG];
};

struct Shared {
  alignas(16) unsigned char stage[NSTAGE][STAGE_BYTES];
  uint64_t full[NSTAGE];
  uint64_t empty[NSTAGE];
  Meta meta[NSTAGE];
  int sh_start[PLAN_SEGS + 1];
  int ex_start[PLAN_SEGS + 1];
  int seg_off[PLAN_SEGS + 1];
  int seg_pg[PLAN_SEGS + 1];  // prefix of pages per segment into `pages`
  int seg_sr[PLAN_SEGS];      // (slot << 9) | rank, slot -1 -> 0 rank
  uint16_t pages[PLAN_PAGES];
  uint16_t perm[PLAN_TOKENS];
  float red[NGROUP][GROUP_WARPS][32];
  float vs[NGROUP][TG][kMaxRank];
  int scan[NTHREADS / 32][3];
  int flag[NGROUP];
  int totals[4];  // shrink items/job, expand items/job, tokens, pages
};

__host__ __device__ inline int ceil_div(int a, int b) { return (a + b - 1) / b; }
__host__ __device__ inline int pow2ceil(int v) {
  int p = 1;
  while (p < v) p <<= 1;
  return p;
}
// Expand geometry for a segment with np pages: P2 lanes share one 16-byte column chunk.
__host__ __device__ inline int expand_p2(int np) { return pow2ceil(ceil_div(np, 2)); }

template <typename T>
__device__ __forceinline__ void plan_counts(const Params& p, int T_s, int rank, int& n_sh,
                                            int& n_ex) {
  constexpr int ES = Elem<T>::kBytes;
  constexpr int EPV = Elem<T>::kEPV;
  const int np = ceil_div(rank, kRowsPerPage);
  const int nt = ceil_div(T_s, TG);
  if (np == 0 || nt == 0) {
    n_sh = n_ex = 0;
    return;
  }
  const int nkc = ceil_div(p.h_in * ES, ACT_ROW_BYTES);
  const int nq = GROUP_THREADS / expand_p2(np);
  const int nexp = ceil_div(p.h_out, nq * EPV);
  n_sh = p.mode == MODE_EXPAND ? 0 : nt * np * nkc;
  n_ex = p.mode == MODE_SHRINK ? 0 : nt * nexp;
}

// index of the last segment s with start[s] <= v (start is non-decreasing, start[0] = 0)
__device__ __forceinline__ int seg_search(const int* start, int S, int v) {
  int lo = 0, hi = S;  // answer in [0, S)
  while (hi - lo > 1) {
    int mid = (lo + hi) >> 1;
    if (start[mid] <= v) lo = mid; else hi = mid;
  }
  return lo;
}

template <typename T>
__global__ void __launch_bounds__(NTHREADS, 1) lora_decode_kernel(const __grid_constant__ Params p) {
  constexpr int ES = Elem<T>::kBytes;
  constexpr int EPV = Elem<T>::kEPV;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  Shared& sm = *reinterpret_cast<Shared*>(smem_raw);
  const int tid = threadIdx.x;
  const int warp = tid >> 5;
  const int lane = tid & 31;

  // ------------------------------------------------------------------ plan (all threads)
  const int S = p.n_seg >= 0 ? p.n_seg : *p.n_seg_dev;
  if (S > PLAN_SEGS || S < 0) {
    if (tid == 0 && blockIdx.x == 0) p.ctr[2] = CHAM_ERR_LIMIT;
    return;
  }
  if (tid == 0) {
    for (int i = 0; i < NSTAGE; ++i) {
      mbar_init(&sm.full[i], 1);
      mbar_init(&sm.empty[i], GROUP_THREADS);
    }
    fence_mbar_init();
  }
  {
    const int per = ceil_div(S, NTHREADS);
    const int s0 = min(S, tid * per), s1 = min(S, s0 + per);
    int lsh = 0, lex = 0, lpg = 0;
    for (int s = s0; s < s1; ++s) {
      const int o0 = p.seg_off[s], o1 = p.seg_off[s + 1];
      const int slot = p.seg_slot[s];
      const int rank = slot >= 0 ? min(p.seg_rank[s], kMaxRank) : 0;
      sm.seg_off[s] = o0;
      sm.seg_sr[s] = slot >= 0 ? ((slot << 9) | rank) : 0;
      int a, b;
      plan_counts<T>(p, o1 - o0, rank, a, b);
      lsh += a;
      lex += b;
      lpg += ceil_div(rank, kRowsPerPage);
    }
    // block exclusive scan of (lsh, lex, lpg)
    int ish = lsh, iex = lex, ipg = lpg;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int a = __shfl_up_sync(0xffffffffu, ish, o);
      const int b = __shfl_up_sync(0xffffffffu, iex, o);
      const int c = __shfl_up_sync(0xffffffffu, ipg, o);
      if (lane >= o) { ish += a; iex += b; ipg += c; }
    }
    if (lane == 31) { sm.scan[warp][0] = ish; sm.scan[warp][1] = iex; sm.scan[warp][2] = ipg; }
    __syncthreads();
    int bsh = 0, bex = 0, bpg = 0;
    for (int w = 0; w < warp; ++w) { bsh += sm.scan[w][0]; bex += sm.scan[w][1]; bpg += sm.scan[w][2]; }
    bsh += ish - lsh;
    bex += iex - lex;
    bpg += ipg - lpg;
    for (int s = s0; s < s1; ++s) {
      const int rank = sm.seg_sr[s] & 511;
      int a, b;
      plan_counts<T>(p, p.seg_off[s + 1] - sm.seg_off[s], rank, a, b);
      sm.sh_start[s] = bsh;
      sm.ex_start[s] = bex;
      sm.seg_pg[s] = bpg;
      bsh += a;
      bex += b;
      bpg += ceil_div(rank, kRowsPerPage);
    }
    if (tid == NTHREADS - 1) {
      sm.sh_start[S] = bsh;
      sm.ex_start[S] = bex;
      sm.seg_pg[S] = bpg;
      sm.seg_off[S] = S > 0 ? p.seg_off[S] : 0;
      sm.totals[0] = bsh;
      sm.totals[1] = bex;
      sm.totals[2] = S > 0 ? p.seg_off[S] : 0;
      sm.totals[3] = bpg;
    }
    __syncthreads();
    // page ids and perm into shared memory when they fit (the producer then never waits on L2)
    if (sm.totals[3] <= PLAN_PAGES) {
      for (int s = s0; s < s1; ++s) {
        const int slot = sm.seg_sr[s] >> 9;
        const int np = ceil_div(sm.seg_sr[s] & 511, kRowsPerPage);
        for (int g = 0; g < np; ++g)
          sm.pages[sm.seg_pg[s] + g] = (uint16_t)__ldg(p.slot_pages + slot * kMaxPagesPerSlot + g);
      }
    }
    if (sm.totals[2] <= PLAN_TOKENS) {
      for (int i = tid; i < sm.totals[2]; i += NTHREADS)
        sm.perm[i] = (uint16_t)(p.perm ? __ldg(p.perm + i) : i);
    }
    __syncthreads();
  }
  const int SH = sm.totals[0], EX = sm.totals[1], NTOK = sm.totals[2];
  const bool pages_smem = sm.totals[3] <= PLAN_PAGES;
  const bool perm_smem = NTOK <= PLAN_TOKENS;
  if (NTOK > p.max_tokens) {
    if (tid == 0 && blockIdx.x == 0) p.ctr[2] = CHAM_ERR_LIMIT;
    return;
  }
  const int total = p.n_jobs * (SH + EX);
  const int nkc = ceil_div(p.h_in * ES, ACT_ROW_BYTES);

  if (warp == 0) {
    // ================================================================ producer warp
    const uint64_t pol_stream = policy_evict_first();  // adapter bytes: read once per step
    const uint64_t pol_act = policy_evict_last();      // x rows: re-read by every page item
    int seq = 0;
    for (int item = blockIdx.x;; item += gridDim.x, ++seq) {
      const int stage = seq % NSTAGE;
      const uint32_t parity = ((seq / NSTAGE) & 1) ^ 1;
      if (lane == 0) mbar_wait(&sm.empty[stage], parity);
      __syncwarp();
      Meta& m = sm.meta[stage];
      if (item >= total) {
        // two END markers so that both consumer groups terminate
        if (lane == 0) {
          m.kind = KIND_END;
          mbar_arrive(&sm.full[stage]);
          const int seq2 = seq + 1, st2 = seq2 % NSTAGE;
          mbar_wait(&sm.empty[st2], ((seq2 / NSTAGE) & 1) ^ 1);
          sm.meta[st2].kind = KIND_END;
          mbar_arrive(&sm.full[st2]);
        }
        break;
      }
      int kind, job, rem;
      if (item < p.n_jobs * SH) {
        kind = KIND_SHRINK; job = item / SH; rem = item - job * SH;
      } else {
        const int e = item - p.n_jobs * SH;
        kind = KIND_EXPAND; job = e / EX; rem = e - job * EX;
      }
      const int* start = kind == KIND_SHRINK ? sm.sh_start : sm.ex_start;
      const int s = seg_search(start, S, rem);
      const int local = rem - start[s];
      const int o0 = sm.seg_off[s];
      const int Ts = sm.seg_off[s + 1] - o0;
      const int sr = sm.seg_sr[s];
      const int slot = sr >> 9, rank = sr & 511;
      const int np = ceil_div(rank, kRowsPerPage);
      const Job& jb = p.jobs[job];
      unsigned char* st = sm.stage[stage];
      int tile, g = 0, kc = 0, col0 = 0, ncols = 0, nq = 0, p2 = 1;
      if (kind == KIND_SHRINK) {
        const int per_tile = np * nkc;
        tile = local / per_tile;
        const int r2 = local - tile * per_tile;
        g = r2 / nkc;
        kc = r2 - g * nkc;
      } else {
        p2 = expand_p2(np);
        nq = GROUP_THREADS / p2;
        const int nc = nq * EPV;
        const int nexp = ceil_div(p.h_out, nc);
        tile = local / nexp;
        const int cc = local - tile * nexp;
        col0 = cc * nc;
        ncols = min(nc, p.h_out - col0);
      }
      const int pos0 = o0 + tile * TG;
      const int tcount = min(TG, Ts - tile * TG);
      // bytes this stage will receive
      uint32_t a_bytes, act_bytes, n_adapter_copies;
      if (kind == KIND_SHRINK) {
        const int natoms = p.h_in * ES / kRowBytes;
        const int a0 = kc * (ADAPTER_BYTES / kAtomBytes);
        const int na = min(ADAPTER_BYTES / kAtomBytes, natoms - a0);
        a_bytes = na * kAtomBytes;
        act_bytes = a_bytes / kRowsPerPage;  // x row chunk
        n_adapter_copies = 1;
      } else {
        a_bytes = ncols * ES * kRowsPerPage;  // per page
        act_bytes = ncols * ES;               // y row chunk
        n_adapter_copies = np;
      }
      if (lane == 0) {
        m.kind = kind; m.job = job; m.pos0 = pos0; m.T = tcount; m.g = g; m.kc = kc; m.np = np;
        m.col0 = col0; m.ncols = ncols; m.nq = nq; m.p2 = p2; m.need = np * nkc;
      }
      // lane c issues copy c: adapter atoms first, then one activation row per token
      const int ncopy = n_adapter_copies + tcount;
      int row = 0, pg = 0;
      const bool is_row = lane >= (int)n_adapter_copies && lane < ncopy;
      if (is_row) {
        const int pos = pos0 + lane - n_adapter_copies;
        row = perm_smem ? (int)sm.perm[pos] : (p.perm ? __ldg(p.perm + pos) : pos);
        m.rows[lane - n_adapter_copies] = row;
      } else if (lane < (int)n_adapter_copies) {
        const int gg = kind == KIND_SHRINK ? g : lane;
        pg = pages_smem ? (int)sm.pages[sm.seg_pg[s] + gg] : __ldg(p.slot_pages + slot * kMaxPagesPerSlot + gg);
      }
      __syncwarp();
      if (lane == 0)
        mbar_arrive_expect_tx(&sm.full[stage], a_bytes * n_adapter_copies + act_bytes * tcount);
      __syncwarp();
      if (lane < (int)n_adapter_copies) {
        if (kind == KIND_SHRINK) {
          const char* src = p.base + (long long)pg * p.page_bytes + jb.a_off + (long long)kc * ADAPTER_BYTES;
          bulk_g2s(st, src, a_bytes, &sm.full[stage], pol_stream);
        } else {
          const char* src = p.base + (long long)pg * p.page_bytes + jb.b_off +
                            (long long)(col0 * ES / kRowBytes) * kAtomBytes;
          bulk_g2s(st + lane * (nq * kRowBytes + PAGE_PAD), src, a_bytes, &sm.full[stage], pol_stream);
        }
      } else if (is_row) {
        const int t = lane - n_adapter_copies;
        if (kind == KIND_SHRINK) {
          const char* src = jb.x + ((long long)row * p.h_in + (long long)kc * (ACT_ROW_BYTES / ES)) * ES;
          bulk_g2s(st + ADAPTER_REGION + t * ACT_ROW_BYTES, src, act_bytes, &sm.full[stage], pol_act);
        } else {
          const char* src = jb.y + ((long long)row * p.h_out + col0) * ES;
          bulk_g2s(st + ADAPTER_REGION + t * ACT_ROW_BYTES, src, act_bytes, &sm.full[stage], pol_stream);
        }
      }
      if (p.trace && lane == 0 && seq < p.trace_cap) {
        unsigned long long* tr = p.trace + ((long long)blockIdx.x * p.trace_cap + seq) * 4;
        tr[0] = gtimer();
        tr[1] = ((unsigned long long)kind << 32) | (unsigned)(a_bytes * n_adapter_copies + act_bytes * tcount);
      }
      __syncwarp();
    }
  } else {
    // ================================================================ consumer groups
    const int grp = (warp - 1) / GROUP_WARPS;
    const int ct = tid - 32 - grp * GROUP_THREADS;  // thread index in group
    const int gw = ct >> 5;                         // warp index in group
    const int bar_id = 1 + grp;
    for (int seq = grp;; seq += NGROUP) {
      const int stage = seq % NSTAGE;
      mbar_wait(&sm.full[stage], (seq / NSTAGE) & 1);
      const Meta m = sm.meta[stage];
      if (m.kind == KIND_END) break;
      if (p.trace && ct == 0 && seq < p.trace_cap)
        p.trace[((long long)blockIdx.x * p.trace_cap + seq) * 4 + 2] = gtimer();
      const unsigned char* st = sm.stage[stage];
      const Job& jb = p.jobs[m.job];
      if (m.kind == KIND_SHRINK) {
        // ---------------------------------------------------------------- shrink
        float acc[kRowsPerPage][TG];
#pragma unroll
        for (int j = 0; j < kRowsPerPage; ++j)
#pragma unroll
          for (int t = 0; t < TG; ++t) acc[j][t] = 0.f;
        const int kbytes = min(ACT_ROW_BYTES, p.h_in * ES - m.kc * ACT_ROW_BYTES);
        const int nqk = kbytes >> 4;
        const unsigned char* X = st + ADAPTER_REGION;
        for (int q = ct; q < nqk; q += GROUP_THREADS) {
          const int a = q >> 3, c = q & 7;
          float xf[TG][EPV];
#pragma unroll
          for (int t = 0; t < TG; ++t) {
            if (t < m.T) {
              Elem<T>::unpack(lds128(X + t * ACT_ROW_BYTES + q * 16), xf[t]);
            } else {
#pragma unroll
              for (int e = 0; e < EPV; ++e) xf[t][e] = 0.f;
            }
          }
#pragma unroll
          for (int j = 0; j < kRowsPerPage; ++j) {
            float af[EPV];
            Elem<T>::unpack(lds128(st + a * kAtomBytes + j * kRowBytes + (((c ^ j) & 7) << 4)), af);
#pragma unroll
            for (int t = 0; t < TG; ++t)
#pragma unroll
              for (int e = 0; e < EPV; ++e) acc[j][t] = fmaf(af[e], xf[t][e], acc[j][t]);
          }
        }
        // butterfly reduce-scatter: 32 values (j*TG + t) over 32 lanes -> lane holds idx=lane
        float v[32];
#pragma unroll
        for (int j = 0; j < kRowsPerPage; ++j)
#pragma unroll
          for (int t = 0; t < TG; ++t) v[j * TG + t] = acc[j][t];
#pragma unroll
        for (int w = 16; w >= 1; w >>= 1) {
          const bool upper = (lane & w) != 0;
#pragma unroll
          for (int i = 0; i < w; ++i) {
            const float send = upper ? v[i] : v[i + w];
            const float keep = upper ? v[i + w] : v[i];
            v[i] = keep + __shfl_xor_sync(0xffffffffu, send, w);
          }
        }
        sm.red[grp][gw][lane] = v[0];
        named_bar_sync(bar_id, GROUP_THREADS);
        if (ct < 32) {
          float s = 0.f;
#pragma unroll
          for (int w2 = 0; w2 < GROUP_WARPS; ++w2) s += sm.red[grp][w2][ct];
          const int j = ct / TG, t = ct % TG;
          if (t < m.T) {
            float* dst = p.vws + (((long long)m.job * p.max_tokens + m.pos0 + t) * p.vws_kc + m.kc) * kMaxRank +
                         m.g * kRowsPerPage + j;
            *dst = s;
          }
        }
        named_bar_sync(bar_id, GROUP_THREADS);
        int* done = p.tile_done + (long long)m.job * p.max_tokens + m.pos0;
        if (p.mode == MODE_FUSED) {
          // one thread publishes: the barrier orders the group's partial-sum stores before
          // its cumulative release (gpu scope) of the tile counter
          if (ct == 0) {
            __threadfence();
            red_release_gpu_add(done, 1);
          }
        } else {
          // MODE_SHRINK: the last item of the tile folds the k-chunk partials into v_out
          if (ct == 0) {
            __threadfence();
            sm.flag[grp] = atom_acq_rel_gpu_add(done, 1) == m.need - 1;
          }
          named_bar_sync(bar_id, GROUP_THREADS);
          if (sm.flag[grp]) {
            const int rows = min(m.np * kRowsPerPage, p.v_stride);
            for (int idx = ct; idx < m.T * rows; idx += GROUP_THREADS) {
              const int t = idx / rows, r = idx - t * rows;
              const float* src = p.vws + (((long long)m.job * p.max_tokens + m.pos0 + t) * p.vws_kc) * kMaxRank + r;
              float s = 0.f;
              for (int k2 = 0; k2 < nkc; ++k2) s += __ldcg(src + k2 * kMaxRank);
              p.v_out[(long long)(m.pos0 + t) * p.v_stride + r] = s;
            }
          }
        }
      } else {
        // ---------------------------------------------------------------- expand
        if (p.mode == MODE_FUSED) {
          if (ct == 0) {
            const int* done = p.tile_done + (long long)m.job * p.max_tokens + m.pos0;
            while (ld_acquire_gpu(done) < m.need) __nanosleep(64);
          }
          named_bar_sync(bar_id, GROUP_THREADS);
        }
        const int rows = m.np * kRowsPerPage;
        for (int idx = ct; idx < m.T * rows; idx += GROUP_THREADS) {
          const int t = idx / rows, r = idx - t * rows;
          float s = 0.f;
          if (p.mode == MODE_FUSED) {
            const float* src = p.vws + (((long long)m.job * p.max_tokens + m.pos0 + t) * p.vws_kc) * kMaxRank + r;
            for (int k2 = 0; k2 < nkc; ++k2) s += __ldcg(src + k2 * kMaxRank);
          } else {
            s = r < p.v_stride ? __ldg(p.v_in + (long long)(m.pos0 + t) * p.v_stride + r) : 0.f;
          }
          sm.vs[grp][t][r] = s;
        }
        named_bar_sync(bar_id, GROUP_THREADS);
        const int p2 = m.p2;
        const int gi = ct & (p2 - 1);
        const int q = ct / p2;
        float acc[TG][EPV];
#pragma unroll
        for (int t = 0; t < TG; ++t)
#pragma unroll
          for (int e = 0; e < EPV; ++e) acc[t][e] = 0.f;
        const bool active = q * EPV < m.ncols;
        if (active) {
          const int a = q >> 3, c = q & 7;
          for (int g = gi; g < m.np; g += p2) {
            const unsigned char* Bg = st + g * (m.nq * kRowBytes + PAGE_PAD);
#pragma unroll
            for (int j = 0; j < kRowsPerPage; ++j) {
              float bf[EPV];
              Elem<T>::unpack(lds128(Bg + a * kAtomBytes + j * kRowBytes + (((c ^ j) & 7) << 4)), bf);
#pragma unroll
              for (int t = 0; t < TG; ++t) {
                const float vv = t < m.T ? sm.vs[grp][t][g * kRowsPerPage + j] : 0.f;
#pragma unroll
                for (int e = 0; e < EPV; ++e) acc[t][e] = fmaf(vv, bf[e], acc[t][e]);
              }
            }
          }
        }
        for (int o = 1; o < p2; o <<= 1) {
#pragma unroll
          for (int t = 0; t < TG; ++t)
#pragma unroll
            for (int e = 0; e < EPV; ++e) acc[t][e] += __shfl_xor_sync(0xffffffffu, acc[t][e], o);
        }
        if (active) {
          const unsigned char* Y = st + ADAPTER_REGION;
#pragma unroll
          for (int t = 0; t < TG; ++t) {
            // the p2 sibling lanes hold identical sums; lane gi stores tokens t == gi (mod p2)
            if (t < m.T && (t & (p2 - 1)) == gi) {
              float yf[EPV];
              Elem<T>::unpack(lds128(Y + t * ACT_ROW_BYTES + q * 16), yf);
#pragma unroll
              for (int e = 0; e < EPV; ++e) yf[e] += acc[t][e];
              char* dst = jb.y + ((long long)m.rows[t] * p.h_out + m.col0) * ES + q * 16;
              *reinterpret_cast<uint4*>(dst) = Elem<T>::pack(yf);
            }
          }
        }
      }
      if (p.trace && ct == 0 && seq < p.trace_cap)
        p.trace[((long long)blockIdx.x * p.trace_cap + seq) * 4 + 3] = gtimer();
      // release the stage (every consumer thread of the group arrives)
      mbar_arrive(&sm.empty[stage]);
    }
  }

  // ---------------------------------------------------------------- teardown / reset
  __syncthreads();
  if (p.mode != MODE_EXPAND) {
    if (tid == 0) {
      __threadfence();
      sm.flag[0] = atomicAdd(p.ctr + 1, 1) == (int)gridDim.x - 1;
    }
    __syncthreads();
    if (sm.flag[0]) {
      __threadfence();
      for (int j = 0; j < p.n_jobs; ++j)
        for (int i = tid; i < NTOK; i += NTHREADS) p.tile_done[(long long)j * p.max_tokens + i] = 0;
      if (tid == 0) p.ctr[1] = 0;
    }
  }
}

template <typename T>
int launch(const cham_pool* pool, Params& prm, cudaStream_t stream) {
  static bool attr_set[2] = {false, false};
  auto kern = lora_decode_kernel<T>;
  const int smem = sizeof(Shared);
  if (!attr_set[Elem<T>::kDtype]) {
    CHAM_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    attr_set[Elem<T>::kDtype] = true;
  }
  kern<<<pool->sm_count, NTHREADS, smem, stream>>>(prm);
  CHAM_CUDA(cudaGetLastError());
  return CHAM_OK;
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
  prm.ctr = pool->d_ctr;
  prm.tile_done = pool->d_tile_done;
  prm.vws = pool->d_vws;
  prm.vws_kc = pool->vws_kc;
  prm.max_tokens = pool->max_tokens;
  prm.mode = mode;
  prm.v_out = v_out;
  prm.v_in = v_in;
  prm.v_stride = v_stride;
  prm.trace = pool->d_trace;
  prm.trace_cap = pool->trace_cap;
  if (pool->dtype == CHAM_BF16) return launch<__nv_bfloat16>(pool, prm, (cudaStream_t)stream);
  return launch<float>(pool, prm, (cudaStream_t)stream);
}

}  // namespace cham
