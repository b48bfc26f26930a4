// Microbenchmark: HBM read throughput of a persistent TMA bulk-copy ring (1-D cp.async.bulk),
// as a function of copy size, ring depth, CTAs per SM and copies per stage.  Consumers only
// wait for the data and release the stage (no math).  Used to size the decode/prefill rings.
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mb_init(uint64_t* b, int c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(b)), "r"(c)); }
__device__ __forceinline__ void mb_expect(uint64_t* b, uint32_t n) { asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(sa(b)), "r"(n) : "memory"); }
__device__ __forceinline__ void mb_arrive(uint64_t* b) { asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(sa(b)) : "memory"); }
__device__ __forceinline__ void mb_wait(uint64_t* b, uint32_t ph) {
  uint32_t ok = 0;
  while (!ok) asm volatile("{.reg .pred p; mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}" : "=r"(ok) : "r"(sa(b)), "r"(ph) : "memory");
}
__device__ __forceinline__ void bulk(void* d, const void* s, uint32_t n, uint64_t* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(sa(d)), "l"(s), "r"(n), "r"(sa(b)) : "memory");
}

__global__ void stream(const char* src, size_t total, int copy_bytes, int nstage, int per_stage, unsigned long long* sink) {
  extern __shared__ __align__(1024) unsigned char sm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(sm);
  uint64_t* empty = full + 16;
  unsigned char* buf = sm + 1024;
  const int stage_bytes = copy_bytes * per_stage;
  if (threadIdx.x == 0) {
    for (int i = 0; i < nstage; ++i) { mb_init(&full[i], 1); mb_init(&empty[i], 32); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const size_t chunk = (size_t)stage_bytes;
  const size_t nchunks = total / chunk;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) {
    int seq = 0;
    for (size_t c = blockIdx.x; c < nchunks; c += gridDim.x, ++seq) {
      const int st = seq % nstage;
      if (seq >= nstage) mb_wait(&empty[st], ((seq / nstage) - 1) & 1);
      if (lane == 0) mb_expect(&full[st], stage_bytes);
      __syncwarp();
      if (lane < per_stage) bulk(buf + (size_t)st * stage_bytes + lane * copy_bytes, src + c * chunk + (size_t)lane * copy_bytes, copy_bytes, &full[st]);
    }
  } else if (warp == 1) {
    int seq = 0;
    unsigned long long acc = 0;
    for (size_t c = blockIdx.x; c < nchunks; c += gridDim.x, ++seq) {
      const int st = seq % nstage;
      mb_wait(&full[st], (seq / nstage) & 1);
      acc += buf[(size_t)st * stage_bytes + lane * 64];
      mb_arrive(&empty[st]);
    }
    if (acc == 0xdeadbeef) *sink = acc;
  }
}

int main() {
  const size_t total = (size_t)4 << 30;  // 4 GiB >> L2
  char* src;
  cudaMalloc(&src, total);
  cudaMemset(src, 1, total);
  unsigned long long* sink;
  cudaMalloc(&sink, 8);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaFuncSetAttribute(stream, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  struct Cfg { int copy, nst, per, ctas; };
  std::vector<Cfg> cfgs;
  for (int copy : {4096, 8192, 16384, 32768})
    for (int per : {1, 2, 4})
      for (int nst : {2, 4, 6, 8})
        for (int ctas : {1, 2}) {
          const size_t smem = 1024 + (size_t)copy * per * nst;
          if (smem * ctas > 220 * 1024) continue;
          cfgs.push_back({copy, nst, per, ctas});
        }
  printf("copy_KB per_stage stages ctas_per_sm inflight_KB_per_sm GB/s\n");
  for (auto c : cfgs) {
    const size_t smem = 1024 + (size_t)c.copy * c.per * c.nst;
    float best = 1e9;
    for (int it = 0; it < 3; ++it) {
      cudaEventRecord(e0);
      stream<<<sms * c.ctas, 64, smem>>>(src, total, c.copy, c.nst, c.per, sink);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (ms < best) best = ms;
    }
    const size_t moved = (total / ((size_t)c.copy * c.per)) * c.copy * c.per;
    printf("%3d %d %d %d %5zu %7.0f\n", c.copy / 1024, c.per, c.nst, c.ctas, (size_t)c.copy * c.per * c.nst * c.ctas / 1024,
           moved / (best * 1e-3) / 1e9);
  }
  cudaError_t e = cudaDeviceSynchronize();
  printf("status %s\n", cudaGetErrorString(e));
  return 0;
}
