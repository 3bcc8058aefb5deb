// Probe: G warps (one per "layer"), each issuing 6-MMA batches (M=128, N=96,
// K=16, SS) into its own TMEM region, committing to its own mbarrier and
// waiting for it before the next batch -- no epilogue.  Reports per-warp
// issue cycles (6 MMAs + commit) and batch round-trip cycles.
//   nvcc -gencode arch=compute_100a,code=sm_100a -shared -Xcompiler -fPIC -o debug/libissueprobe.so debug/issue_probe.cu
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46);
}

__global__ void probe(long long *out, int iters) {
  extern __shared__ __align__(1024) uint8_t sm[];   // A: 2 planes x 2 KB, B: 6 tiles x 5 KB
  __shared__ uint64_t bars[8];
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < (4096 + 30720) / 4; i += blockDim.x) reinterpret_cast<uint32_t *>(sm)[i] = 0x3c003c00u;
  if (threadIdx.x < 8) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bars[threadIdx.x])));
  asm volatile("fence.mbarrier_init.release.cluster;");
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tslot + warp * 96;
  const uint32_t idesc = (1u << 4) | ((uint32_t)(96 >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
  const uint64_t a = desc(smem_u32(sm), 2048, 128), b = desc(smem_u32(sm + 4096), 2560, 128);
  const uint32_t bar = smem_u32(&bars[warp]);
  long long issue = 0, t_start = clock64();
  uint32_t ph = 0;
  for (int it = 0; it < iters; ++it) {
    long long t0 = clock64();
    asm volatile(
        "{\n\t.reg .pred e, p;\n\t.reg .b64 ta, tb;\n\t"
        "setp.ne.b32 p, 1, 0;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t"
        "add.s64 ta, %1, 256;\n\tadd.s64 tb, %2, 320;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], ta, tb, %3, p;\n\t"
        "add.s64 ta, %1, 1;\n\tadd.s64 tb, %2, 640;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], ta, tb, %3, p;\n\t"
        "add.s64 ta, %1, 257;\n\tadd.s64 tb, %2, 960;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], ta, tb, %3, p;\n\t"
        "add.s64 ta, %1, 2;\n\tadd.s64 tb, %2, 1280;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], ta, tb, %3, p;\n\t"
        "add.s64 ta, %1, 258;\n\tadd.s64 tb, %2, 1600;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], ta, tb, %3, p;\n\t"
        "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%4];\n\t}"
        ::"r"(tmem), "l"(a), "l"(b), "r"(idesc), "r"(bar) : "memory");
    issue += clock64() - t0;
    asm volatile("{\n\t.reg .pred P1;\nW:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t@!P1 bra W;\n\t}"
                 ::"r"(bar), "r"(ph) : "memory");
    ph ^= 1;
  }
  long long total = clock64() - t_start;
  if (lane == 0) { out[2 * warp] = issue; out[2 * warp + 1] = total; }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tslot));
}

extern "C" int run(long long *out, int warps, int iters) {
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 4096 + 30720);
  probe<<<1, 32 * warps, 4096 + 30720>>>(out, iters);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
  return 0;
}
