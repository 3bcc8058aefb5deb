// Training 3x3 convolution 32 -> 32 on tcgen05 with split-bf16 operands.
//
// Replaces conv3x3_fwd_kernel<32,32> of the training path: the residual
// blocks' forward convs (nn.py:46-60, 91-95) and their input gradients, which
// conv_simt.cu runs as forward convs with transposed / flipped weights
// (nn.py:62-77, 97-100).  Same epilogue options: bias, ReLU mask, residual
// add, ReLU.  NCHW fp32 in and out, so the rest of the pipeline is unchanged.
//
// Precision: each fp32 operand is split into three bf16 parts x = x0 + x1 +
// x2 (x0 = bf16(x), x1 = bf16(x - x0), x2 = bf16(x - x0 - x1): 24 mantissa
// bits, the fp32 exponent range); a product keeps the six terms xi*wj with
// i + j <= 2, accumulated in fp32 TMEM (six kind::f16 MMAs, bf16 rate =
// 2x tf32), i.e. fp32-level accuracy -- needed: with 3xTF32 (~2^-21 per
// product) the 32 chained input-gradient convs of the paper architecture
// missed the 1e-4 bar (1.3e-3).
//
// Structure (the fused forward's row streaming, one layer):
// * a strip is 128 pixel lanes of the virtual side-by-side image (the B
//   images laid next to each other with one zero column between), with 126
//   output lanes (halo 1);
// * rows stream top to bottom; MMA(r) for input row r adds into output rows
//   r+1, r, r-1, a 3-slot TMEM ring reached through a window of the doubled
//   ky sequence [2,1,0,2,1] (N = 96), 36 MMAs per row (3 kx x 2 K-halves x
//   6 split products);
// * one CTA per SM: the weights (three bf16 parts, 90 KB) are split into
//   UMMA tiles by every CTA from the OIHW fp32 tensor, two input rows (three
//   parts, 48 KB) are double buffered; 8 warps, thread = (pixel lane,
//   16-channel half).
#include "common.cuh"
#include "tc_ptx.cuh"

#include <cuda_bf16.h>

namespace ht {
namespace tct {

using namespace ::ht::tc;

constexpr int C = 32;
constexpr int M = 128;
constexpr int S = M - 2;              // output lanes per strip
constexpr int NSL = 5;                // doubled ky sequence [2,1,0,2,1]
constexpr int NPART = 3;              // bf16 parts of an fp32 value
constexpr int PLANE = M * 16;         // 8 channels x 128 lanes (bf16)
constexpr int ROW = 4 * PLANE;        // 32 channels of a row, one part
constexpr int TILE = 2 * NSL * C * 16;  // B tile for (kx, 16-channel K-half): 160 rows x 32 B
constexpr int W_BYTES = NPART * 3 * 2 * TILE;
constexpr int A_OFF = W_BYTES;
constexpr int A_BYTES = 2 * NPART * ROW;    // 2 buffers x 3 parts
constexpr int BAR_OFF = A_OFF + A_BYTES;
// barriers acc_full[2], ready[2], stg_full[2], TMEM address
constexpr int STG_OFF = BAR_OFF + 128;
// one TMA box: 132 px x 32 channels fp32 ([ch][px]); a box's first column
// must be a multiple of 4 (16 B), so it starts up to 3 px left of lane 0
constexpr int BOXW = M + 4;
constexpr int BOX = BOXW * C * 4;
constexpr int STG_SLOT = 2 * BOX;     // a strip row spans at most two images (W + 1 >= 128)
constexpr int SMEM_LDG = STG_OFF;
constexpr int SMEM_TMA = STG_OFF + 2 * STG_SLOT;
constexpr int NRING = 4;              // TMEM rings (input row mod 4), 96 columns each
constexpr int NWORK = 256;            // worker threads: 2 channel halves x 4 lane quarters
constexpr int NTHR = NWORK + 32;      // + one MMA-issuer warp
constexpr int HC = C / 2;             // channels per thread
constexpr uint32_t IDESC_BF16 =
    (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(96 >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
__constant__ int c_ky[NSL] = {2, 1, 0, 2, 1};

// x = x0 + x1 + x2 (bf16 parts; the remainders are exact in fp32)
__device__ __forceinline__ void split3(float x, __nv_bfloat16 &p0, __nv_bfloat16 &p1, __nv_bfloat16 &p2) {
  p0 = __float2bfloat16_rn(x);
  const float r1 = x - __bfloat162float(p0);
  p1 = __float2bfloat16_rn(r1);
  p2 = __float2bfloat16_rn(r1 - __bfloat162float(p1));
}
// split3 of a pair with packed conversions (one cvt.rn.bf16x2 per part: half
// the conversion-pipe instructions); p_i = {part i of x (low), of y (high)}
__device__ __forceinline__ void split3x2(float x, float y, uint32_t &p0, uint32_t &p1, uint32_t &p2) {
  auto cvt2 = [](float lo, float hi) {
    const __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
    return *reinterpret_cast<const uint32_t *>(&v);
  };
  p0 = cvt2(x, y);
  const float rx = x - __uint_as_float(p0 << 16), ry = y - __uint_as_float(p0 & 0xFFFF0000u);
  p1 = cvt2(rx, ry);
  const float sx = rx - __uint_as_float(p1 << 16), sy = ry - __uint_as_float(p1 & 0xFFFF0000u);
  p2 = cvt2(sx, sy);
}
__device__ __forceinline__ uint32_t pack_bf2(__nv_bfloat16 a, __nv_bfloat16 b) {
  return (uint32_t)__bfloat16_as_ushort(a) | ((uint32_t)__bfloat16_as_ushort(b) << 16);
}

// One input row into its own TMEM ring: for kx in 0..2, K-half kh in 0..1 (16
// channels) and the six split products (i, j) with i + j <= 2:
// D[128 x 96] += A_i[128 x 16] * B_j[96 x 16]^T.  The thirty small correction
// products go first (the first overwrites the ring: no re-init), the six
// main products (0, 0) last, so the large partial sums see only six fp32
// accumulation steps -- the tensor core's accumulation error stays at the
// SIMT level.  Descriptors are the six bases plus immediate offsets (16-B units).
__device__ __forceinline__ void mma36_row(uint32_t d, uint64_t a0, uint64_t a1, uint64_t a2, uint64_t b0,
                                          uint64_t b1, uint64_t b2, uint32_t bar_acc) {
  asm volatile(
      "{\n\t.reg .pred e, p, z;\n\t.reg .b64 ta, tb;\n\t"
      "setp.ne.b32 p, 1, 0;\n\t"
      "setp.ne.b32 z, 0, 0;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "add.s64 ta, %1, -1;\n\tadd.s64 tb, %5, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], ta, tb, %7, z;\n\t"
      "add.s64 ta, %2, -1;\n\tadd.s64 tb, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], ta, tb, %7, p;\n\t"
      "add.s64 ta, %1, -1;\n\tadd.s64 tb, %6, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], ta, tb, %7, p;\n\t"
      "add.s64 ta, %2, -1;\n\tadd.s64 tb, %5, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], ta, tb, %7, p;\n\t"
      "add.s64 ta, %3, -1;\n\tadd.s64 tb, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], ta, tb, %7, p;\n\t"
      "add.s64 ta, %1, 255;\n\tadd.s64 tb, %5, 320;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], ta, tb, %7, p;\n\t"
      "add.s64 ta, %2, 255;\n\tadd.s64 tb, %4, 320;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], ta, tb, %7, p;\n\t"
      "add.s64 ta, %1, 255;\n\tadd.s64 tb, %6, 320;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], ta, tb, %7, p;\n\t"
      "add.s64 ta, %2, 255;\n\tadd.s64 tb, %5, 320;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], ta, tb, %7, p;\n\t"
      "add.s64 ta, %3, 255;\n\tadd.s64 tb, %4, 320;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], ta, tb, %7, p;\n\t"
      "add.s64 ta, %1, 0;\n\tadd.s64 tb, %5, 640;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], ta, tb, %7, p;\n\t"
      "add.s64 ta, %2, 0;\n\tadd.s64 tb, %4, 640;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], ta, tb, %7, p;\n\t"
      "add.s64 ta, %1, 0;\n\tadd.s64 tb, %6, 640;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], ta, tb, %7, p;\n\t"
      "add.s64 ta, %2, 0;\n\tadd.s64 tb, %5, 640;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], ta, tb, %7, p;\n\t"
      "add.s64 ta, %3, 0;\n\tadd.s64 tb, %4, 640;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], ta, tb, %7, p;\n\t"
      "add.s64 ta, %1, 256;\n\tadd.s64 tb, %5, 960;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], ta, tb, %7, p;\n\t"
      "add.s64 ta, %2, 256;\n\tadd.s64 tb, %4, 960;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], ta, tb, %7, p;\n\t"
      "add.s64 ta, %1, 256;\n\tadd.s64 tb, %6, 960;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], ta, tb, %7, p;\n\t"
      "add.s64 ta, %2, 256;\n\tadd.s64 tb, %5, 960;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], ta, tb, %7, p;\n\t"
      "add.s64 ta, %3, 256;\n\tadd.s64 tb, %4, 960;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], ta, tb, %7, p;\n\t"
      "add.s64 ta, %1, 1;\n\tadd.s64 tb, %5, 1280;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], ta, tb, %7, p;\n\t"
      "add.s64 ta, %2, 1;\n\tadd.s64 tb, %4, 1280;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], ta, tb, %7, p;\n\t"
      "add.s64 ta, %1, 1;\n\tadd.s64 tb, %6, 1280;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], ta, tb, %7, p;\n\t"
      "add.s64 ta, %2, 1;\n\tadd.s64 tb, %5, 1280;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], ta, tb, %7, p;\n\t"
      "add.s64 ta, %3, 1;\n\tadd.s64 tb, %4, 1280;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], ta, tb, %7, p;\n\t"
      "add.s64 ta, %1, 257;\n\tadd.s64 tb, %5, 1600;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], ta, tb, %7, p;\n\t"
      "add.s64 ta, %2, 257;\n\tadd.s64 tb, %4, 1600;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], ta, tb, %7, p;\n\t"
      "add.s64 ta, %1, 257;\n\tadd.s64 tb, %6, 1600;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], ta, tb, %7, p;\n\t"
      "add.s64 ta, %2, 257;\n\tadd.s64 tb, %5, 1600;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], ta, tb, %7, p;\n\t"
      "add.s64 ta, %3, 257;\n\tadd.s64 tb, %4, 1600;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], ta, tb, %7, p;\n\t"
      "add.s64 ta, %1, -1;\n\tadd.s64 tb, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], ta, tb, %7, p;\n\t"
      "add.s64 ta, %1, 255;\n\tadd.s64 tb, %4, 320;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], ta, tb, %7, p;\n\t"
      "add.s64 ta, %1, 0;\n\tadd.s64 tb, %4, 640;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], ta, tb, %7, p;\n\t"
      "add.s64 ta, %1, 256;\n\tadd.s64 tb, %4, 960;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], ta, tb, %7, p;\n\t"
      "add.s64 ta, %1, 1;\n\tadd.s64 tb, %4, 1280;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], ta, tb, %7, p;\n\t"
      "add.s64 ta, %1, 257;\n\tadd.s64 tb, %4, 1600;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], ta, tb, %7, p;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%8];\n\t}"
      ::"r"(d), "l"(a0), "l"(a1), "l"(a2), "l"(b0), "l"(b1), "l"(b2), "r"(IDESC_BF16), "r"(bar_acc)
      : "memory");
}

#ifdef CT_TL
// debug timeline of CTA 0, warp 0 lane 0: per step (r, after barrier+issue,
// MMA(r) seen, drained, split, stored+loaded)
__device__ long long g_ctl[4096][6];
#define CTL(k) do { if (blockIdx.x == 0 && threadIdx.x == 0 && ctl_n < 4096) g_ctl[ctl_n][k] = clock64(); } while (0)
#else
#define CTL(k) do {} while (0)
#endif

struct ConvParams {
  CUtensorMap tm_x;  // TX: x as (W, C, H, B) fp32, box 128 x 32 x 1 x 1
  const float *x, *w, *bias, *mask, *resid;
  float *out;
  int B, H, W, VW, relu;
  int n_strips;
  long long chunk;   // strip-rows per CTA (strip-major)
};

__device__ __forceinline__ void tma_load_4d(uint32_t dst, const CUtensorMap *map, int c0, int c1, int c2, int c3,
                                            uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, "
      "%5}], [%6];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(bar)
      : "memory");
}

// TX: input rows arrive by TMA (issued two rows ahead by the issuer warp) into
// a two-slot staging ring instead of per-thread loads -- an LDG still in
// flight at a split's proxy fence (a CTA memory barrier) would stall it.
template <bool TX>
__global__ void __launch_bounds__(NTHR, 1) conv_tc_kernel(const __grid_constant__ ConvParams P) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const int tid = threadIdx.x, lane = tid & 31;
  const int warp = __shfl_sync(0xffffffffu, tid >> 5, 0);
  const uint32_t sbase = smem_u32(smem);
  // MMA(x) commits to acc_full[x & 1]: two batches can be in flight
  auto acc_full = [&](int x) { return sbase + BAR_OFF + 8u * (uint32_t)(x & 1); };
  // ready[x & 1]: the 8 worker warps split input row x (and drained the row
  // whose ring MMA(x) reuses) -- the issuer warp may issue MMA(x)
  auto ready = [&](int x) { return sbase + BAR_OFF + 16 + 8u * (uint32_t)(x & 1); };
  auto stg_full = [&](int x) { return sbase + BAR_OFF + 32 + 8u * (uint32_t)(x & 1); };
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(smem + BAR_OFF + 48);
  if (tid == 0) {
    mbar_init(acc_full(0), 1);
    mbar_init(acc_full(1), 1);
    mbar_init(ready(0), NWORK / 32);
    mbar_init(ready(1), NWORK / 32);
    mbar_init(stg_full(0), 1);
    mbar_init(stg_full(1), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  // weights: OIHW fp32 -> three bf16 parts, UMMA tiles [part][kx][kh] of 160
  // rows (slice s, co) x 2 K-chunks (8 channels, 16 B), K-major core matrices
  for (int i = tid; i < 3 * 2 * 2 * NSL * C * 8; i += NTHR) {
    const int e = i & 7, co = (i >> 3) % C, s = (i >> 3) / C % NSL;
    const int kc = (i >> 3) / C / NSL % 2, kh = (i >> 3) / C / NSL / 2 % 2, kx = (i >> 3) / C / NSL / 4;
    const int ci = kh * 16 + kc * 8 + e, ky = c_ky[s];
    __nv_bfloat16 w0, w1, w2;
    split3(P.w[((co * C + ci) * 3 + ky) * 3 + kx], w0, w1, w2);
    const int off = (kx * 2 + kh) * TILE + kc * (NSL * C * 16) + (s * C + co) * 16 + e * 2;
    *reinterpret_cast<__nv_bfloat16 *>(smem + off) = w0;
    *reinterpret_cast<__nv_bfloat16 *>(smem + 6 * TILE + off) = w1;
    *reinterpret_cast<__nv_bfloat16 *>(smem + 12 * TILE + off) = w2;
  }
  for (int i = tid; i < A_BYTES / 16; i += NTHR)
    reinterpret_cast<uint4 *>(smem + A_OFF)[i] = make_uint4(0, 0, 0, 0);
  fence_proxy_async();
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = __shfl_sync(0xffffffffu, *tmem_slot, 0);
  // two warpgroups: warp w serves TMEM lane quarter w & 3 (pixel lanes) and
  // channel half w >> 2 (16 channels) -- twice the warps of one pixel per
  // thread, for the epilogue's and loader's memory latency
  const int wq = warp & 3, half = warp >> 2;
  const uint32_t tlane = tmem + ((uint32_t)(wq * 32) << 16);
  const int l = wq * 32 + lane;
  const int c0 = half * HC;
  const uint64_t adesc0 = umma_desc(sbase, PLANE, 128);
  const uint64_t bdesc0 = (adesc0 & ~(0x3FFFull << 16)) | ((uint64_t)((NSL * C * 16) >> 4) << 16);
  const size_t plane = (size_t)P.H * P.W;
  const long long range = P.H;
  const long long q0 = (long long)blockIdx.x * P.chunk;
  const long long q1 = min(q0 + P.chunk, (long long)P.n_strips * range);
  if (warp == NWORK / 32) {
    // ---- MMA issuer: MMA(x) for every input row x of every segment, as soon
    //      as the workers have split row x and drained the row whose ring it
    //      overwrites.  Blocking on a full tensor-pipe queue here costs the
    //      workers nothing (they never issue).
    uint32_t ph_rdy = 0;
    for (long long qq = q0; qq < q1;) {
      const int s = (int)(qq / range);
      const long long end = min(q1, (long long)(s + 1) * range);
      const int R0 = (int)(qq - (long long)s * range), R1 = (int)(end - (long long)s * range);
      qq = end;
      const int A = max(R0 - 1, 0), Bn = min(R1 + 1, P.H);
      // TX: input row x of this strip -> staging slot x & 1 (one box per image
      // the strip touches; out-of-image pixels arrive as zeros)
      const int v0 = s * S - 1, b0 = max(v0, 0) / (P.W + 1);
      auto tma_row = [&](int x) {
        if (lane == 0) {
          const int nbox = b0 + 1 < P.B ? 2 : 1;
          mbar_expect_tx(stg_full(x), nbox * BOX);
          for (int k = 0; k < nbox; ++k)
            tma_load_4d(sbase + STG_OFF + (x & 1) * STG_SLOT + k * BOX, &P.tm_x, (v0 - (b0 + k) * (P.W + 1)) & ~3, 0, x,
                        b0 + k, stg_full(x));
        }
      };
      if constexpr (TX) {
        tma_row(A);
        if (A + 1 < Bn) tma_row(A + 1);
      }
      for (int x = A; x < Bn; ++x) {
        if (lane == 0) mbar_wait(ready(x), (ph_rdy >> (x & 1)) & 1);
        ph_rdy ^= 1u << (x & 1);
        __syncwarp();
        // row x was split: its staging slot takes row x+2 (before the MMAs,
        // whose issue can block on a full tensor-pipe queue)
        if constexpr (TX) {
          if (x + 2 < Bn) tma_row(x + 2);
        }
        __syncwarp();
        tc_fence_after();
        const int xm3 = x % 3;
        const int o = xm3 == 0 ? 1 : (xm3 == 1 ? 0 : 2);         // B window for rows (x+1, x, x-1)
        const uint64_t a = adesc0 + ((A_OFF + (x & 1) * NPART * ROW) >> 4);
        const uint64_t bw = bdesc0 + ((o * C * 16) >> 4);
        mma36_row(tmem + (uint32_t)((x % NRING) * 3 * C), a, a + (ROW >> 4), a + ((2 * ROW) >> 4), bw,
                  bw + ((6 * TILE) >> 4), bw + ((12 * TILE) >> 4), acc_full(x));
        __syncwarp();
      }
    }
  } else {
  uint32_t ph_acc = 0, ph_stg = 0;
#ifdef CT_TL
  int ctl_n = 0;
#endif
  float xin[HC], vals[HC];
  float bv[HC], mv[HC], rv[HC];   // bias of this thread's channels; next row's mask / residual
  constexpr size_t NO_ROW = ~(size_t)0;
  float pend[HC];                 // output row awaiting its stores
  size_t pend_o0 = NO_ROW;
#pragma unroll
  for (int i = 0; i < HC; ++i) bv[i] = P.bias ? __ldg(P.bias + c0 + i) : 0.f;
  for (long long qq = q0; qq < q1;) {
    const int s = (int)(qq / range);
    const long long end = min(q1, (long long)(s + 1) * range);
    const int R0 = (int)(qq - (long long)s * range), R1 = (int)(end - (long long)s * range);
    qq = end;
    const int A = max(R0 - 1, 0), Bn = min(R1 + 1, P.H);
    const int v = s * S - 1 + l;
    const int b = v >= 0 ? v / (P.W + 1) : 0, col = v >= 0 ? v % (P.W + 1) : 0;
    const bool in_img = v >= 0 && v < P.VW && col < P.W;
    const bool lane_valid = l >= 1 && l < 1 + S && in_img;
    const float *xb = P.x + ((size_t)b * C + c0) * plane + col;
    auto load_row = [&](int row) {
      if constexpr (!TX) {
#pragma unroll
        for (int i = 0; i < HC; ++i) xin[i] = 0.f;
        if (in_img && row < Bn) {
#pragma unroll
          for (int i = 0; i < HC; ++i) xin[i] = __ldg(xb + (size_t)i * plane + (size_t)row * P.W);
        }
      }
    };
    // TX: this thread's 16 channels of staged row `row` (box of its image)
    const int kbox = in_img ? b - max(s * S - 1, 0) / (P.W + 1) : -1;
    // lane l of box k sits at column l + ((c_k) & 3), c_k = the box's lane-0 column
    const int kcol = (s * S - 1) - (max(s * S - 1, 0) / (P.W + 1) + max(kbox, 0)) * (P.W + 1);
    const int koff = l + (kcol & 3);
    auto stage_row = [&](int row) {
      if constexpr (TX) {
        if (lane == 0) mbar_wait(stg_full(row), (ph_stg >> (row & 1)) & 1);
        ph_stg ^= 1u << (row & 1);
        __syncwarp();
        const float *src = reinterpret_cast<const float *>(smem + STG_OFF + (row & 1) * STG_SLOT + max(kbox, 0) * BOX) +
                           c0 * BOXW + koff;
#pragma unroll
        for (int i = 0; i < HC; ++i) xin[i] = kbox >= 0 ? src[i * BOXW] : 0.f;
      }
    };
    // this thread's 16 channels of an input row -> three bf16 parts in the
    // row's A buffer (visible to the MMAs after the next CTA barrier)
    auto split_row = [&](int row) {
      const uint32_t dst = sbase + A_OFF + (row & 1) * NPART * ROW + (2 * half) * PLANE + l * 16;
#pragma unroll
      for (int g = 0; g < 2; ++g) {
        uint32_t w[3][4];
#pragma unroll
        for (int k2 = 0; k2 < 4; ++k2) {
          split3x2(xin[8 * g + 2 * k2], xin[8 * g + 2 * k2 + 1], w[0][k2], w[1][k2], w[2][k2]);
        }
#pragma unroll
        for (int pp = 0; pp < 3; ++pp)
          st_shared_v4(dst + pp * ROW + g * PLANE, w[pp][0], w[pp][1], w[pp][2], w[pp][3]);
      }
      fence_proxy_async();
    };
    // Input row x's products go to TMEM ring x mod 4 (three 32-column slots:
    // output rows mod 3); output row d is the sum of the slots d mod 3 of the
    // rings of input rows d-1, d, d+1.  The issuer warp runs MMA(r+1) as soon
    // as row r+1 is split and row r-2 drained (ring (r+1) mod 4 last held row
    // r-3), so the tensor pipe has the next row queued while the workers wait
    // for MMA(r), drain row r-1, split row r+2 and store row r-1.
    // mask / residual values of output row `row` for the epilogue (one row ahead)
    auto load_epi = [&](int row) {
      if (!(P.mask || P.resid) || !(row >= R0 && row < R1 && lane_valid)) return;
      const size_t o0 = ((size_t)b * C + c0) * plane + (size_t)row * P.W + col;
#pragma unroll
      for (int i = 0; i < HC; ++i) {
        if (P.mask) mv[i] = __ldg(P.mask + o0 + (size_t)i * plane);
        if (P.resid) rv[i] = __ldg(P.resid + o0 + (size_t)i * plane);
      }
    };
    // deferred stores of the previous output row
    auto flush = [&]() {
      if (pend_o0 != NO_ROW) {
#pragma unroll
        for (int i = 0; i < HC; ++i) P.out[pend_o0 + (size_t)i * plane] = pend[i];
        pend_o0 = NO_ROW;
      }
    };
    load_row(A);                       // split in the first iteration (r = A-2)
    load_epi(R0);
    int tm3 = ((A - 3) % 3 + 3) % 3;   // slot of row r-1 at t = A-2
    for (int r = A - 2; r <= Bn; ++r) {
#ifdef CT_TL
      if (blockIdx.x == 0 && threadIdx.x == 0 && ctl_n < 4096) g_ctl[ctl_n][0] = r;
#endif
      CTL(1);
      const int d = r - 1, slot = tm3;
      tm3 = tm3 == 2 ? 0 : tm3 + 1;
      CTL(2);
      // ---- 2. MMA(r) done (and every earlier MMA; MMA(r+1) may still run)
      if (r >= A && r < Bn) {
        if (lane == 0) mbar_wait(acc_full(r), (ph_acc >> (r & 1)) & 1);
        ph_acc ^= 1u << (r & 1);
        __syncwarp();
        tc_fence_after();
      }
      // ---- 3. finished output row d -> registers: slots d mod 3 of the rings
      //         of input rows d-1, d, d+1 (a row outside [A, Bn) is zero
      //         padding: its ring holds an older row)
      CTL(3);
      const bool drain = d >= A && d < Bn;
      if (drain) {
#pragma unroll
        for (int i = 0; i < HC; ++i) vals[i] = 0.f;
#pragma unroll
        for (int k = -1; k <= 1; ++k) {
          const int xr = d + k;
          if (xr < A || xr >= Bn) continue;
          float part[HC];
          tmem_ld16(tlane + (xr % NRING) * 3 * C + slot * C + c0, part);
#pragma unroll
          for (int i = 0; i < HC; ++i) vals[i] += part[i];
        }
      }
      // ---- 4. input row r+2 -> the three bf16 A planes of buffer (r+2)&1
      //         (last read by MMA(r), retired in step 2)
      CTL(4);
      if (r + 2 >= A && r + 2 < Bn) {
        stage_row(r + 2);
#ifdef CT_TL
        if (blockIdx.x == 0 && threadIdx.x == 0 && ctl_n < 4096) g_ctl[ctl_n][0] = clock64();
#endif
        split_row(r + 2);
        // row r+2 split, row r-1 drained (the last reader of ring (r+2) mod 4)
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(ready(r + 2));
      }
      flush();
      CTL(5);
      // ---- 5. prefetch input row r+3 (split next step: a whole step of
      //         latency cover -- every split's proxy fence waits for the
      //         loads outstanding at that point, so they must be a step old)
      if (r + 2 >= A && r + 2 < Bn) load_row(r + 3);
      // ---- 6. epilogue of row d (overlaps MMA(r+1)); its mask / residual
      //         values were loaded a step earlier; then those of row d+1.
      //         Its stores go out after the next step's split, so that
      //         split's proxy fence finds them a step old.
      const bool store_d = drain && d >= R0 && d < R1 && lane_valid;
      if (store_d) {
        pend_o0 = ((size_t)b * C + c0) * plane + (size_t)d * P.W + col;
#pragma unroll
        for (int i = 0; i < HC; ++i) {
          float y = vals[i] + bv[i];
          if (P.mask) y = mv[i] > 0.f ? y : 0.f;
          if (P.resid) y += rv[i];
          if (P.relu) y = fmaxf(y, 0.f);
          pend[i] = y;
        }
      }
      load_epi(d + 1);
#ifdef CT_TL
      ++ctl_n;
#endif
    }
    flush();
  }
  }   // workers
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

}  // namespace tct
#ifdef CT_TL
extern "C" int ht_debug_conv_timeline(long long *host) {
  return (int)cudaMemcpyFromSymbol(host, tct::g_ctl, sizeof(long long) * 4096 * 6);
}
#endif

// x, out, mask, resid: (B, 32, H, W) fp32; w: (32, 32, 3, 3) fp32 OIHW.
int conv_tc32(const float *x, int B, int H, int W, const float *w, const float *bias, const float *mask,
              const float *resid, float *out, int relu, cudaStream_t st) {
  using namespace tct;
  if (int rc = ensure_smem_attr((const void *)conv_tc_kernel<false>, SMEM_LDG)) return rc;
  if (int rc = ensure_smem_attr((const void *)conv_tc_kernel<true>, SMEM_TMA)) return rc;
  int dev = 0, n_sm = 148;
  HT_CUDA(cudaGetDevice(&dev));
  HT_CUDA(cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev));
  ConvParams p{};
  p.x = x; p.w = w; p.bias = bias; p.mask = mask; p.resid = resid; p.out = out;
  p.B = B; p.H = H; p.W = W; p.VW = B * (W + 1); p.relu = relu;
  p.n_strips = (p.VW + S - 1) / S;
  const long long total = (long long)p.n_strips * H;
  long long grid = n_sm;
  if (total < grid * 8) grid = (total + 7) / 8;
  if (grid < 1) grid = 1;
  p.chunk = (total + grid - 1) / grid;
  grid = (total + p.chunk - 1) / p.chunk;
  // TMA-staged rows need 16-B row strides and strips spanning <= 2 images
  if (W % 4 == 0 && W + 1 >= M) {
    auto enc = tensor_map_encoder();
    HT_REQUIRE(enc != nullptr, "cuTensorMapEncodeTiled unavailable");
    const cuuint64_t row = (cuuint64_t)W * 4, planeb = row * H;
    cuuint64_t dims[4] = {(cuuint64_t)W, (cuuint64_t)C, (cuuint64_t)H, (cuuint64_t)B};
    cuuint64_t strides[3] = {planeb, row, planeb * C};
    cuuint32_t box[4] = {(cuuint32_t)BOXW, (cuuint32_t)C, 1, 1};
    cuuint32_t estr[4] = {1, 1, 1, 1};
    const CUresult r = enc(&p.tm_x, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, const_cast<float *>(x), dims, strides, box,
                           estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    HT_REQUIRE(r == CUDA_SUCCESS, "cuTensorMapEncodeTiled failed (%d)", (int)r);
    conv_tc_kernel<true><<<(unsigned)grid, NTHR, SMEM_TMA, st>>>(p);
  } else {
    conv_tc_kernel<false><<<(unsigned)grid, NTHR, SMEM_LDG, st>>>(p);
  }
  count_launch();
  HT_CHECK_LAUNCH();
  return HT_OK;
}

}  // namespace ht
