// Microbenchmark: tcgen05.mma kind::f16 M=128 issue/throughput in the shape
// the fused conv kernel uses: per "row", 6 MMAs (3 kx shifts x 2 K halves)
// whose descriptors are runtime base + compile-time offsets.
#include <cuda_runtime.h>
#include <stdint.h>

__device__ __forceinline__ uint64_t desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46);
}
__device__ __forceinline__ void mma_plain(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
               "l"(a), "l"(b), "r"(idesc), "r"(1));
}
__device__ __forceinline__ void mma_elect(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc) {
  asm volatile("{\n\t.reg .pred p, e;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
               "l"(a), "l"(b), "r"(idesc), "r"(1));
}

template <int N, int MODE>
__global__ void mma_kernel(int rows, long long *out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint64_t cbar[2];
  __shared__ uint32_t tslot;
  const int tid = threadIdx.x;
  for (int i = tid; i < 200 * 1024 / 4; i += blockDim.x) {
    uint32_t x = (uint32_t)i * 2654435761u;
    x ^= x >> 13;
    // random fp16 pairs in [-1, 1) (MODE 9/10) or zeros
    const uint32_t h0 = 0x3800u | (x & 0x3FFu) | ((x >> 10) & 1u) << 15;
    const uint32_t h1 = 0x3800u | ((x >> 11) & 0x3FFu) | ((x >> 21) & 1u) << 15;
    ((uint32_t *)smem)[i] = (MODE >= 9) ? (h0 | (h1 << 16)) : 0u;
  }
  asm volatile("fence.proxy.async.shared::cta;");
  if (tid < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
        (uint32_t)__cvta_generic_to_shared(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(&bar)));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(&cbar[0])));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(&cbar[1])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const int warp_u = __shfl_sync(0xffffffffu, tid / 32, 0);
  const uint32_t tmem = __shfl_sync(0xffffffffu, tslot, 0);
  const bool issuer = (MODE == 0) ? (tid == 0) : (warp_u == 0);
  __shared__ volatile int stop_flag;
  if (tid == 0) stop_flag = 0;
  __syncthreads();
  if (MODE >= 6 && warp_u >= 1) {
    const uint32_t sb = (uint32_t)__cvta_generic_to_shared(smem);
    const int lane = tid & 31, w = warp_u;
    uint32_t v[16];
    for (int i = 0; i < 16; ++i) v[i] = i;
    while (!stop_flag) {
      if (MODE == 6 || MODE == 8) {
        for (int k = 0; k < 8; ++k) {
          const uint32_t a = sb + 40000 + ((w * 8 + k) % 16) * 512 + lane * 16;
          asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};" ::"r"(a), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]) : "memory");
          asm volatile("ld.shared.v4.b32 {%0,%1,%2,%3}, [%4];" : "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]) : "r"(a + 16) : "memory");
        }
      }
      if (MODE == 7 || MODE == 8) {
        const uint32_t tl = tmem + ((uint32_t)((w & 3) * 32) << 16) + 384;
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
              "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
            : "r"(tl));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        asm volatile(
            "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(tl + 16),
            "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]),
            "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]) : "memory");
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      }
    }
  }
  if (issuer) {
    const uint32_t sb = (uint32_t)__cvta_generic_to_shared(smem);
    constexpr uint32_t idesc = (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    long long t0 = clock64();
    for (int r = 0; r < rows; ++r) {
      const int q = r & 1;
      const int rot = r % 3;
      const int o = rot == 0 ? 1 : (rot == 1 ? 0 : 2);
      // MODE 10: spread over 4 "layers" (distinct A buffers and weight tiles)
      const int layer = (MODE == 10) ? (r & 3) : 0;
      const uint32_t a_base = sb + 130000 + layer * 16640 + q * 8320;
      const uint32_t w_base = sb + layer * 30720 + o * 512;
      const uint32_t d = tmem + (MODE == 3 ? (r & 3) * N : 0);
#pragma unroll
      for (int kx = 0; kx < 3; ++kx) {
#pragma unroll
        for (int kh = 0; kh < 2; ++kh) {
          const uint64_t ad = desc(a_base + kh * 4160 + kx * 16, 2080, 128);
          const uint64_t bd = desc(w_base + (kx * 2 + kh) * 5120, 2560, 128);
          if (MODE == 0) mma_plain(d, ad, bd, idesc);
          else mma_elect(d, ad, bd, idesc);
        }
      }
      if (MODE == 11) {
        if ((tid & 31) == 0)
          asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
              (uint32_t)__cvta_generic_to_shared(&cbar[0])));
        if ((tid & 31) == 0)
          asm volatile("{\n\t.reg .pred P1;\nW:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t@P1 bra D;\n\tbra W;\nD:\n\t}" ::"r"(
              (uint32_t)__cvta_generic_to_shared(&cbar[0])), "r"((uint32_t)(r & 1)));
        __syncwarp();
      }
      if (MODE >= 4 && MODE <= 10 && (tid & 31) == 0) {
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
            (uint32_t)__cvta_generic_to_shared(&cbar[0])));
        if (MODE == 5)
          asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
              (uint32_t)__cvta_generic_to_shared(&cbar[1])));
      }
      __syncwarp();
    }
    long long t1 = clock64();
    if (MODE == 0 || (tid & 31) == 0)
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
          (uint32_t)__cvta_generic_to_shared(&bar)));
    asm volatile("{\n\t.reg .pred P1;\nW:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t@P1 bra D;\n\tbra W;\nD:\n\t}" ::"r"(
        (uint32_t)__cvta_generic_to_shared(&bar)));
    long long t2 = clock64();
    if ((tid & 31) == 0) { out[0] = t1 - t0; out[1] = t2 - t0; }
    stop_flag = 1;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (tid < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

extern "C" int run_mma_bench(int N, int mode, int rows, int nblocks, long long *host) {
  long long *d;
  cudaMalloc(&d, 16);
  const int smem = 200 * 1024;
#define L(NN, MM)                                                                                \
  if (N == NN && mode == MM) {                                                                   \
    cudaFuncSetAttribute(mma_kernel<NN, MM>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem); \
    mma_kernel<NN, MM><<<nblocks, (MM >= 6 ? 544 : 128), smem>>>(rows, d);                                         \
  }
  L(32, 0) L(32, 1) L(32, 3) L(96, 0) L(96, 1) L(96, 3) L(128, 0) L(128, 1) L(128, 3)
  L(256, 0) L(256, 1) L(96, 4) L(96, 5) L(128, 5) L(96, 6) L(96, 7) L(96, 8) L(96, 9) L(96, 10) L(96, 11) L(32, 11) L(256, 11)
  cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(host, d, 16, cudaMemcpyDeviceToHost);
  cudaFree(d);
  return (int)e;
}
