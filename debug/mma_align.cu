// Microbenchmark: tcgen05.mma kind::f16 M=128 N=96 K=16 throughput in the
// training conv's operand layout (K-major, no swizzle; A rows 16 B apart, B
// the doubled-ky tile), by A start alignment: SHIFT 0 = every MMA's A start
// 128-B aligned, 1 = the conv's kx = 0,1,2 starts (-16 B, 0, +16 B), 2 = all
// +16 B.  One CTA per SM, back-to-back batches of 18 MMAs, one commit each.
//   nvcc -gencode arch=compute_100a,code=sm_100a -shared -Xcompiler -fPIC -o debug/libmmaalign.so debug/mma_align.cu
#include <cuda_runtime.h>
#include <stdint.h>

__device__ __forceinline__ uint64_t desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46);
}
__device__ __forceinline__ void mma(uint32_t d, uint64_t a, uint64_t b, uint32_t acc) {
  constexpr uint32_t IDESC = (1u << 4) | ((uint32_t)(96 >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
               "l"(a), "l"(b), "r"(IDESC), "r"(acc) : "memory");
}

template <int SHIFT>
__global__ void bench(int batches, long long *out, int mode) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint64_t cb[4];
  __shared__ uint32_t tslot;
  const int tid = threadIdx.x;
  for (int i = tid; i < 160 * 1024 / 4; i += blockDim.x) {
    uint32_t x = (uint32_t)i * 2654435761u;
    x ^= x >> 13;
    const uint32_t h0 = 0x3800u | (x & 0x3FFu) | ((x >> 10) & 1u) << 15;
    const uint32_t h1 = 0x3800u | ((x >> 11) & 0x3FFu) | ((x >> 21) & 1u) << 15;
    ((uint32_t *)smem)[i] = h0 | (h1 << 16);
  }
  asm volatile("fence.proxy.async.shared::cta;");
  if (tid < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
        (uint32_t)__cvta_generic_to_shared(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(&bar)));
    for (int k = 0; k < 4; ++k) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(&cb[k])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tslot;
  if (tid == 0) {
    const uint32_t sb = (uint32_t)__cvta_generic_to_shared(smem);
    // B: 2 parts x 6 tiles of 5120 B at 0; A: 2 parts x 8 KB at 64 KB (+16 B guard)
    const uint64_t b0 = desc(sb, 2560, 128), a0 = desc(sb + 65536 + 1024, 2048, 128);
    constexpr uint64_t AP = 8192 >> 4, BP = 30720 >> 4, TB = 5120 >> 4, KH = 4096 >> 4;
    long long t0 = clock64();
    for (int r = 0; r < batches; ++r) {
      // mode 2: at most two batches in flight; mode 3: one
      const int lag = mode == 2 ? 2 : 1;
      if (mode >= 2 && r >= lag) {
        const uint32_t wb = (uint32_t)__cvta_generic_to_shared(&cb[(r - lag) & 3]);
        const uint32_t par = ((r - lag) >> 2) & 1;
        asm volatile("{\n\t.reg .pred P1;\nW:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t@!P1 bra W;\n\t}"
                     ::"r"(wb), "r"(par) : "memory");
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      }
      const uint32_t d = tmem + (uint32_t)((r & 3) * 96);
      const uint64_t b = b0 + ((r % 3) * 512 >> 4);
      uint32_t acc = 0;
#pragma unroll
      for (int kx = 0; kx < 3; ++kx)
#pragma unroll
        for (int kh = 0; kh < 2; ++kh) {
          const int sh = SHIFT == 0 ? 0 : (SHIFT == 1 ? kx - 1 : 1);
          const uint64_t a = a0 + kh * KH + sh, bb = b + (kx * 2 + kh) * TB;
          mma(d, a + AP, bb, acc);
          acc = 1;
          mma(d, a, bb + BP, 1);
        }
#pragma unroll
      for (int kx = 0; kx < 3; ++kx)
#pragma unroll
        for (int kh = 0; kh < 2; ++kh) {
          const int sh = SHIFT == 0 ? 0 : (SHIFT == 1 ? kx - 1 : 1);
          mma(d, a0 + kh * KH + sh, b + (kx * 2 + kh) * TB, 1);
        }
      if (mode >= 1)
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
            (uint32_t)__cvta_generic_to_shared(&cb[r & 3])) : "memory");
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
        (uint32_t)__cvta_generic_to_shared(&bar)) : "memory");
    asm volatile("{\n\t.reg .pred P1;\nW:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t@!P1 bra W;\n\t}"
                 ::"r"((uint32_t)__cvta_generic_to_shared(&bar)) : "memory");
    const long long t1 = clock64();
    if (blockIdx.x == 0) { out[0] = t1 - t0; }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (tid < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

extern "C" int run(int shift, int batches, int nblk, long long *out_host, int mode) {
  long long *d;
  cudaMalloc(&d, 16);
  const int smem = 160 * 1024;
  if (shift == 0) { cudaFuncSetAttribute(bench<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem); bench<0><<<nblk, 128, smem>>>(batches, d, mode); }
  if (shift == 1) { cudaFuncSetAttribute(bench<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem); bench<1><<<nblk, 128, smem>>>(batches, d, mode); }
  if (shift == 2) { cudaFuncSetAttribute(bench<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem); bench<2><<<nblk, 128, smem>>>(batches, d, mode); }
  cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(out_host, d, 8, cudaMemcpyDeviceToHost);
  cudaFree(d);
  return e == cudaSuccess ? 0 : 1;
}
