// Latency microbenchmark of the synchronisation / TMEM primitives the fused
// kernel's epilogue uses, with the tensor core idle or busy (warp 1 issuing
// N=96 MMAs back to back).
#include <cuda_runtime.h>
#include <stdint.h>

__device__ __forceinline__ uint64_t desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46);
}

__global__ void prim_kernel(int iters, int busy, long long *out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar, bar2;
  __shared__ uint32_t tslot;
  __shared__ volatile int stop;
  const int tid = threadIdx.x, warp = tid / 32, lane = tid & 31;
  for (int i = tid; i < 64 * 1024 / 4; i += blockDim.x) ((uint32_t *)smem)[i] = 0;
  if (tid == 0) stop = 0;
  asm volatile("fence.proxy.async.shared::cta;");
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
        (uint32_t)__cvta_generic_to_shared(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(&bar)));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(&bar2)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tslot;
  const uint32_t sb = (uint32_t)__cvta_generic_to_shared(smem);
  const uint32_t b1 = (uint32_t)__cvta_generic_to_shared(&bar);
  if (warp == 1) {
    if (busy) {
      const uint32_t idesc = (1u << 4) | ((uint32_t)(96 >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
      const uint64_t ad = desc(sb, 2080, 128), bd = desc(sb + 20000, 2560, 128);
      while (!stop) {
        for (int k = 0; k < 16; ++k)
          asm volatile("{\n\t.reg .pred p, e;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                       "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem + 256),
                       "l"(ad), "l"(bd), "r"(idesc), "r"(1));
        __syncwarp();
      }
    }
  } else if (warp == 0) {
    const uint32_t tl = tmem;  // lanes 0-31
    long long acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    uint32_t v[16];
    for (int it = 0; it < iters; ++it) {
      long long c0 = clock64();
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
          : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
            "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
          : "r"(tl));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      long long c1 = clock64();
      asm volatile(
          "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(tl + 32),
          "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]),
          "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
          : "memory");
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      long long c2 = clock64();
      asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};" ::"r"(sb + 40000 + lane * 16), "r"(v[0]), "r"(v[1]),
                   "r"(v[2]), "r"(v[3]) : "memory");
      asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};" ::"r"(sb + 42080 + lane * 16), "r"(v[4]), "r"(v[5]),
                   "r"(v[6]), "r"(v[7]) : "memory");
      long long c3 = clock64();
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      long long c4 = clock64();
      __syncwarp();
      if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(b1) : "memory");
      long long c5 = clock64();
      // wait for the phase we just completed (already complete)
      if (lane == 0)
        asm volatile("{\n\t.reg .pred P1;\nW:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t@P1 bra D;\n\tbra W;\nD:\n\t}" ::"r"(b1),
                     "r"((uint32_t)(it & 1)));
      __syncwarp();
      long long c6 = clock64();
      acc[0] += c1 - c0; acc[1] += c2 - c1; acc[2] += c3 - c2; acc[3] += c4 - c3;
      acc[4] += c5 - c4; acc[5] += c6 - c5;
    }
    if (lane == 0) for (int k = 0; k < 6; ++k) out[k] = acc[k] / iters;
    stop = 1;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

extern "C" int run_prim(int iters, int busy, long long *host) {
  long long *d;
  cudaMalloc(&d, 64);
  cudaFuncSetAttribute(prim_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  prim_kernel<<<1, 64, 64 * 1024>>>(iters, busy, d);
  cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(host, d, 48, cudaMemcpyDeviceToHost);
  cudaFree(d);
  return (int)e;
}
