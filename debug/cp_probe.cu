// Probe: cp.async.bulk (global -> smem, mbarrier complete_tx) and
// tcgen05.cp.128x256b (smem -> TMEM) with a K-major no-swizzle descriptor
// (8-row core matrices of 16 B, SBO = 128 B between row groups, LBO = plane
// stride between the two 16-B halves of a row).  Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -shared -Xcompiler -fPIC -o debug/libcpprobe.so debug/cp_probe.cu
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void probe(const float *src, float *out, int plane_bytes) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const int tid = threadIdx.x;
  const uint32_t b = smem_u32(&bar);
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (tid < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"(smem_u32(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tslot;
  // 8 planes of 128 lanes x 16 B (4 fp32): plane g holds channels 4g..4g+3
  if (tid == 0) {
    const uint32_t bytes = 8 * 2048;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(bytes) : "memory");
    for (int g = 0; g < 8; ++g)
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
              smem_u32(smem) + g * plane_bytes),
          "l"(src + g * 512), "r"(2048), "r"(b)
          : "memory");
  }
  // wait
  asm volatile(
      "{\n\t.reg .pred P1;\nW:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t@!P1 bra W;\n\t}" ::"r"(b)
      : "memory");
  if (tid == 0) {
    for (int k = 0; k < 4; ++k) {
      const uint32_t sa = smem_u32(smem) + 2 * k * plane_bytes;
      const uint64_t desc = (uint64_t)((sa >> 4) & 0x3FFF) | ((uint64_t)((plane_bytes >> 4) & 0x3FFF) << 16) |
                            ((uint64_t)(128 >> 4) << 32) | (1ull << 46);
      asm volatile("tcgen05.cp.cta_group::1.128x256b [%0], %1;" ::"r"(tmem + 8 * k), "l"(desc) : "memory");
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(b) : "memory");
  }
  asm volatile(
      "{\n\t.reg .pred P1;\nW2:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 1;\n\t@!P1 bra W2;\n\t}" ::"r"(b)
      : "memory");
  asm volatile("tcgen05.fence::after_thread_sync;");
  const int w = tid >> 5;
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(tmem + ((uint32_t)(w * 32) << 16)));
  asm volatile("tcgen05.wait::ld.sync.aligned;");
  for (int i = 0; i < 32; ++i) out[tid * 32 + i] = __uint_as_float(r[i]);
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (tid < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(tmem));
}

extern "C" int run_probe(const float *src, float *out, int plane_bytes) {
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * plane_bytes + 1024);
  probe<<<1, 128, 8 * plane_bytes + 1024>>>(src, out, plane_bytes);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
  return 0;
}
