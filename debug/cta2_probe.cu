// Probe: tcgen05.mma.cta_group::2 (M=256 across a CTA pair, N=96, K=16,
// f16 -> f32) with A = 128x16 per CTA and B = 48x16 per CTA (each CTA holds
// half of N), K-major no-swizzle descriptors; commit multicast to both CTAs.
//   nvcc -gencode arch=compute_100a,code=sm_100a -shared -Xcompiler -fPIC -o debug/libcta2probe.so debug/cta2_probe.cu
#include <cooperative_groups.h>
#include <cstdint>
#include <cstdio>
#include <cuda_fp16.h>

namespace cg = cooperative_groups;

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46);
}

// A: [128 rows][16 k] fp16 -> smem core-matrix layout: row m at (m/8)*128 + (m%8)*16 within a
// K-chunk plane (8 k per 16 B); plane kc at kc * PA.  B same with 48 rows, plane stride PB.
constexpr int PA = 128 * 16, PB = 48 * 16;

__global__ void __cluster_dims__(2, 1, 1) probe(const __half *A, const __half *B, float *D) {
  __shared__ __align__(1024) uint8_t sa[2 * PA];
  __shared__ __align__(1024) uint8_t sb[2 * PB];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  cg::cluster_group cluster = cg::this_cluster();
  const unsigned rank = cluster.block_rank();
  const int tid = threadIdx.x;
  // fill A (this CTA's 128 rows) and B (this CTA's 48 rows of N)
  for (int i = tid; i < 128 * 16; i += blockDim.x) {
    const int m = i / 16, k = i % 16;
    *reinterpret_cast<__half *>(sa + (k / 8) * PA + m * 16 + (k % 8) * 2) = A[(rank * 128 + m) * 16 + k];
  }
  for (int i = tid; i < 48 * 16; i += blockDim.x) {
    const int n = i / 16, k = i % 16;
    *reinterpret_cast<__half *>(sb + (k / 8) * PB + n * 16 + (k % 8) * 2) = B[(rank * 48 + n) * 16 + k];
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (tid < 32) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(smem_u32(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  cluster.sync();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tslot;
  if (rank == 0 && tid < 32) {
    const uint32_t idesc = (1u << 4) | ((uint32_t)(96 >> 3) << 17) | ((uint32_t)(256 >> 4) << 24);
    const uint64_t ad = desc(smem_u32(sa), PA, 128), bd = desc(smem_u32(sb), PB, 128);
    asm volatile(
        "{\n\t.reg .pred e, p;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "setp.ne.b32 p, 0, 0;\n\t"
        "@e tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t"
        "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%4], %5;\n\t}"
        ::"r"(tmem), "l"(ad), "l"(bd), "r"(idesc), "r"(smem_u32(&bar)), "h"((uint16_t)3)
        : "memory");
  }
  asm volatile(
      "{\n\t.reg .pred P1;\nW:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t@!P1 bra W;\n\t}" ::"r"(
          smem_u32(&bar))
      : "memory");
  asm volatile("tcgen05.fence::after_thread_sync;");
  const int w = tid >> 5;
  for (int c0 = 0; c0 < 96; c0 += 32) {
    uint32_t r[32];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
          "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
          "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(tmem + ((uint32_t)(w * 32) << 16) + c0));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    for (int i = 0; i < 32; ++i) D[(rank * 128 + tid) * 96 + c0 + i] = __uint_as_float(r[i]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  cluster.sync();
  if (tid < 32) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 128;" ::"r"(tmem));
}

extern "C" int run_probe(const void *A, const void *B, float *D) {
  probe<<<2, 128>>>((const __half *)A, (const __half *)B, D);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
  return 0;
}

template <int CG>
__global__ void __cluster_dims__(2, 1, 1) tput(long long *cycles, int niter) {
  __shared__ __align__(1024) uint8_t sa[2 * PA];
  __shared__ __align__(1024) uint8_t sb[2 * 160 * 16];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  cg::cluster_group cluster = cg::this_cluster();
  const unsigned rank = cluster.block_rank();
  const int tid = threadIdx.x;
  for (int i = tid; i < 2 * PA / 4; i += blockDim.x) reinterpret_cast<uint32_t *>(sa)[i] = 0x3c003c00u;
  for (int i = tid; i < 2 * 160 * 16 / 4; i += blockDim.x) reinterpret_cast<uint32_t *>(sb)[i] = 0x3c003c00u;
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (tid < 32) {
    if (CG == 2) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(smem_u32(&tslot)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(smem_u32(&tslot)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  cluster.sync();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tslot;
  if ((CG == 1 || rank == 0) && tid < 32) {
    const uint32_t idesc = (1u << 4) | ((uint32_t)(96 >> 3) << 17) | ((uint32_t)((CG == 2 ? 256 : 128) >> 4) << 24);
    const uint64_t ad = desc(smem_u32(sa), PA, 128), bd = desc(smem_u32(sb), (CG == 2 ? 48 : 96) * 16, 128);
    long long t0 = clock64();
    for (int it = 0; it < niter; ++it) {
      if (CG == 2)
        asm volatile("{\n\t.reg .pred e, p;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, 1, 0;\n\t"
                     "@e tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}"
                     ::"r"(tmem), "l"(ad + (it & 1)), "l"(bd), "r"(idesc) : "memory");
      else
        asm volatile("{\n\t.reg .pred e, p;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, 1, 0;\n\t"
                     "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}"
                     ::"r"(tmem), "l"(ad + (it & 1)), "l"(bd), "r"(idesc) : "memory");
    }
    if (CG == 2)
      asm volatile("{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
                   "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n\t}"
                   ::"r"(smem_u32(&bar)), "h"((uint16_t)3) : "memory");
    else
      asm volatile("{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
                   "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}"
                   ::"r"(smem_u32(&bar)) : "memory");
    asm volatile("{\n\t.reg .pred P1;\nW:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t@!P1 bra W;\n\t}"
                 ::"r"(smem_u32(&bar)) : "memory");
    if (tid == 0) cycles[blockIdx.x] = clock64() - t0;
  } else if (CG == 2) {
    asm volatile("{\n\t.reg .pred P1;\nW:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t@!P1 bra W;\n\t}"
                 ::"r"(smem_u32(&bar)) : "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  cluster.sync();
  if (tid < 32) {
    if (CG == 2) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 128;" ::"r"(tmem));
    else asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(tmem));
  }
}

extern "C" int run_tput(int cg2, long long *cycles, int niter, int nclusters) {
  if (cg2) tput<2><<<2 * nclusters, 128>>>(cycles, niter);
  else tput<1><<<2 * nclusters, 128>>>(cycles, niter);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
  return 0;
}

// ping-pong latency: CTA r waits on its own barrier, then arrives remotely on
// the peer's barrier (mapa + mbarrier.arrive.release.cluster)
__global__ void __cluster_dims__(2, 1, 1) pingpong(long long *out, int iters) {
  __shared__ uint64_t bar;
  cg::cluster_group cluster = cg::this_cluster();
  const unsigned rank = cluster.block_rank();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  cluster.sync();
  if (threadIdx.x == 0) {
    uint32_t remote;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(smem_u32(&bar)), "r"(rank ^ 1));
    long long t0 = clock64();
    uint32_t ph = 0;
    for (int i = 0; i < iters; ++i) {
      if (rank == 0) asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote) : "memory");
      asm volatile("{\n\t.reg .pred P1;\nW:\n\tmbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P1, [%0], %1;\n\t@!P1 bra W;\n\t}"
                   ::"r"(smem_u32(&bar)), "r"(ph) : "memory");
      ph ^= 1;
      if (rank == 1) asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote) : "memory");
    }
    out[rank] = clock64() - t0;
  }
  cluster.sync();
}
extern "C" int run_pingpong(long long *out, int iters) {
  pingpong<<<2, 32>>>(out, iters);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
  return 0;
}
