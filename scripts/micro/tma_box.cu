// Microbenchmark: HBM read throughput of 2-D TMA box loads (64 bf16 columns x 32 rows,
// SWIZZLE_128B — the prefill kernel's activation tiles) over a [rows x 4096] bf16 matrix,
// for two traversal orders: row-block-major (consecutive boxes of a CTA share rows) and
// column-chunk-major (consecutive boxes are 32 rows further down the same 128-byte column
// strip).  Compared with 1-D bulk copies of whole contiguous rows.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mb_init(uint64_t* b, int c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(b)), "r"(c)); }
__device__ __forceinline__ void mb_expect(uint64_t* b, uint32_t n) { asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(sa(b)), "r"(n) : "memory"); }
__device__ __forceinline__ void mb_arrive(uint64_t* b) { asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(sa(b)) : "memory"); }
__device__ __forceinline__ void mb_wait(uint64_t* b, uint32_t ph) {
  uint32_t ok = 0;
  while (!ok) asm volatile("{.reg .pred p; mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}" : "=r"(ok) : "r"(sa(b)), "r"(ph) : "memory");
}
__device__ __forceinline__ void tma2d(void* dst, const CUtensorMap* m, int c0, int c1, uint64_t* bar) {
  asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
               ::"r"(sa(dst)), "l"(reinterpret_cast<uint64_t>(m)), "r"(c0), "r"(c1), "r"(sa(bar)) : "memory");
}
__device__ __forceinline__ void bulk(void* d, const void* s, uint32_t n, uint64_t* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(sa(d)), "l"(s), "r"(n), "r"(sa(b)) : "memory");
}

constexpr int NST = 8, BOXES = 4, BOX = 64 * 32 * 2;  // 8 stages x 16 KiB
// mode 0: row-block-major boxes, 1: column-chunk-major boxes, 2: 1-D bulk rows (4 x 4 KiB per stage)
__global__ void run(const __grid_constant__ CUtensorMap map, const char* base, int rows, int cols, int mode,
                    unsigned long long* sink) {
  extern __shared__ __align__(1024) unsigned char sm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(sm);
  uint64_t* empty = full + NST;
  unsigned char* buf = sm + 1024;
  if (threadIdx.x == 0) {
    for (int i = 0; i < NST; ++i) { mb_init(&full[i], 1); mb_init(&empty[i], 32); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nrb = rows / 32, ncc = cols / 64;
  const long long nbox = (long long)nrb * ncc;
  const long long nst_total = nbox / BOXES;
  if (warp == 0) {
    int seq = 0;
    for (long long s = blockIdx.x; s < nst_total; s += gridDim.x, ++seq) {
      const int st = seq % NST;
      if (seq >= NST) mb_wait(&empty[st], ((seq / NST) - 1) & 1);
      if (lane == 0) mb_expect(&full[st], BOXES * BOX);
      __syncwarp();
      if (lane < BOXES) {
        const long long b = s * BOXES + lane;
        unsigned char* dst = buf + (size_t)st * BOXES * BOX + lane * BOX;
        if (mode == 0) tma2d(dst, &map, (int)(b % ncc) * 64, (int)(b / ncc) * 32, &full[st]);
        else if (mode == 1) tma2d(dst, &map, (int)(b / nrb) * 64, (int)(b % nrb) * 32, &full[st]);
        else if (mode == 2) bulk(dst, base + b * BOX, BOX, &full[st]);
      }
      if (mode >= 3) {  // the same 16 KiB per stage as (mode - 2) x 1 KiB ... copies
        const int per = mode == 3 ? 1024 : 2048;
        const int nc = BOXES * BOX / per;
        for (int c = lane; c < nc; c += 32)
          bulk(buf + (size_t)st * BOXES * BOX + c * per, base + s * BOXES * BOX + (long long)c * per, per, &full[st]);
      }
    }
  } else if (warp == 1) {
    int seq = 0;
    unsigned long long acc = 0;
    for (long long s = blockIdx.x; s < nst_total; s += gridDim.x, ++seq) {
      const int st = seq % NST;
      mb_wait(&full[st], (seq / NST) & 1);
      acc += buf[(size_t)st * BOXES * BOX + lane * 64];
      mb_arrive(&empty[st]);
    }
    if (acc == 0xdeadbeef) *sink = acc;
  }
}

int main() {
  const int rows = 131072, cols = 4096;  // 1 GiB bf16
  char* src;
  cudaMalloc(&src, (size_t)rows * cols * 2);
  cudaMemset(src, 1, (size_t)rows * cols * 2);
  unsigned long long* sink;
  cudaMalloc(&sink, 8);
  void* f = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q);
  auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  CUtensorMap map;
  const cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  const cuuint64_t strides[1] = {(cuuint64_t)cols * 2};
  const cuuint32_t box[2] = {64, 32};
  const cuuint32_t estr[2] = {1, 1};
  enc(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, src, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int smem = 1024 + NST * BOXES * BOX;
  cudaFuncSetAttribute(run, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const char* names[5] = {"2-D boxes, row-block-major", "2-D boxes, column-chunk-major", "1-D bulk copies 4 KiB",
                          "1-D bulk copies 1 KiB", "1-D bulk copies 2 KiB"};
  for (int mode = 0; mode < 5; ++mode) {
    float best = 1e9;
    for (int it = 0; it < 3; ++it) {
      cudaEventRecord(e0);
      run<<<sms, 64, smem>>>(map, src, rows, cols, mode, sink);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (ms < best) best = ms;
    }
    printf("%-32s %7.0f GB/s\n", names[mode], (double)rows * cols * 2 / (best * 1e-3) / 1e9);
  }
  printf("status %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
