// K1: fused tensor-core policy forward + sigmoid/threshold epilogue, sm_100a.
//
// Replaces PolicyNetwork.forward (nn.py:138-150) and the threshold of
// rl.infer_halftone (rl.py:306-311).  Design:
//
// * Row streaming.  A CTA owns a 128-pixel-wide strip of the "virtual image"
//   (the B images laid side by side, one zero column between neighbours) and
//   a band of rows.  Each UMMA M-tile is one strip row: 128 pixels = 128 TMEM
//   lanes.  The network runs as passes of <=5 conv layers; inside a pass every
//   layer streams rows top to bottom in a diagonal wavefront (layer j consumes
//   its input row t-2j at step t), so only two input rows per layer live in
//   shared memory and the per-pass halo is G columns/rows (G = layers in pass).
// * Implicit GEMM per input row r of a layer: for each horizontal tap kx and
//   K half kh, one tcgen05.mma (kind::f16, M=128, N=3*32, K=16) with
//     A = the row's fp16 activations shifted by kx pixels (a 16-byte shift of
//         the UMMA start address in a K-major, no-swizzle, row-linear layout),
//     B = the weights of all three vertical taps ky stacked along N,
//     D = three 32-column TMEM accumulators: output rows r+1, r, r-1.
//   The three output rows live in a 3-slot TMEM ring (slot = row mod 3); the
//   B operand is a window into a doubled ky sequence [2,1,0,2,1] so every row
//   maps onto the ring with a single N=96 MMA and no wrap-around.
// * Residual stream in fp32: a conv2 accumulator slot is initialised (via
//   tcgen05.st) with x + bias before its first MMA, so the skip add is free;
//   the fp32 x rows are carried in registers of the epilogue threads or read
//   from the pass input.  conv_in takes (c, z) split into fp16 hi/lo pairs
//   (and hi/lo weights) so its input is represented to ~fp32 accuracy.
// * Per-layer zero padding (nn.py:50): out-of-image pixels are forced to 0 in
//   every epilogue; out-of-image rows issue no MMAs.
// * Roles (544 threads): warp 0 lane 0 issues all MMAs; warps 1-16 are the
//   epilogue in two sets (even / odd layers); set 0 also loads the pass input rows (TMEM -> registers -> bias,
//   ReLU, fp16 -> next layer's shared-memory row / global x / p,h).
//   Producer/consumer hand-offs use mbarriers; tcgen05.commit signals MMA
//   completion.
#include <cuda_fp16.h>

#include <type_traits>

#include "common.cuh"
#include "fwd_tc.cuh"

namespace ht {
namespace tc {

// compile-time reverse loop: f(integral_constant<N-1>), ..., f(integral_constant<0>)
template <int N, typename F>
__device__ __forceinline__ void rev_for(F &&f) {
  if constexpr (N > 0) {
    f(std::integral_constant<int, N - 1>{});
    rev_for<N - 1>(f);
  }
}

enum : int { K_IN = 0, K_C1 = 1, K_C2 = 2, K_OUT = 3 };

template <bool HI, int NBK, bool HO>
struct Plan {
  static constexpr int G = (HI ? 1 : 0) + 2 * NBK + (HO ? 1 : 0);
  static constexpr int kind(int j) {
    return (HI && j == 0) ? K_IN : (HO && j == G - 1) ? K_OUT : (((j - (HI ? 1 : 0)) % 2 == 0) ? K_C1 : K_C2);
  }
  static constexpr int nk(int j) { return kind(j) == K_IN ? 1 : 2; }
  static constexpr int ns(int j) { return kind(j) == K_OUT ? 16 : 32; }
  static constexpr int wbytes(int j) { return 3 * nk(j) * tile_bytes(ns(j)); }
  static constexpr int abytes(int j) { return nk(j) * 2 * PLANE; }
  static constexpr int w_off(int j) { return j == 0 ? 0 : w_off(j - 1) + wbytes(j - 1); }
  static constexpr int W_TOTAL = w_off(G - 1) + wbytes(G - 1);
  static constexpr int a_off(int j) { return j == 0 ? W_TOTAL : a_off(j - 1) + 2 * abytes(j - 1); }
  static constexpr int A_END = a_off(G - 1) + 2 * abytes(G - 1);
  static constexpr int BIAS_OFF = A_END;                       // G*32 fp32
  static constexpr int BAR_OFF = BIAS_OFF + G * 32 * 4;        // barriers (8 B each)
  // barriers: a_full[G][2], a_empty[G][2], acc_full[G], acc_free[G]
  static constexpr int NBAR = 6 * G;
  static constexpr int TMEMP_OFF = BAR_OFF + NBAR * 8;
  static constexpr int SMEM = TMEMP_OFF + 16;
  static constexpr int tcol(int j) { return j == 0 ? 0 : tcol(j - 1) + 3 * ns(j - 1); }
  static constexpr int TCOLS = tcol(G - 1) + 3 * ns(G - 1);
  // layer j writes its output into the next layer's A buffer
  static constexpr bool feeds_next(int j) { return j < G - 1; }
  // layer j's output is the residual of layer j+2 (a conv2)
  static constexpr bool holds(int j) {
    return (kind(j) == K_IN || kind(j) == K_C2) && j + 2 < G && kind(j + 2) == K_C2;
  }
  static constexpr int hold_idx(int j) { return j <= 0 ? 0 : hold_idx(j - 1) + (holds(j - 1) ? 1 : 0); }
};

// ---------------------------------------------------------------------------
// PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}
#ifdef HT_TRACE
#define TRACE(...) do { if (blockIdx.x == 0) printf(__VA_ARGS__); } while (0)
#else
#define TRACE(...) do {} while (0)
#endif
#ifdef HT_WATCHDOG
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  uint32_t ok = 0;
  for (long long it = 0; !ok; ++it) {
    asm volatile(
        "{\n\t.reg .pred P1;\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n\tselp.u32 %0, 1, 0, P1;\n\t}"
        : "=r"(ok) : "r"(bar), "r"(parity) : "memory");
    if (it == (1ll << 22)) {
      uint32_t base;
      asm volatile("mov.u32 %0, %%dynamic_smem_size;" : "=r"(base));
      extern __shared__ __align__(1024) uint8_t smem[];
      printf("WATCHDOG block %d thread %d bar_off %u parity %u (smem %u)\n", blockIdx.x, threadIdx.x,
             bar - (uint32_t)__cvta_generic_to_shared(smem), parity, base);
      asm volatile("trap;");
    }
  }
}
#else
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@P1 bra DONE_%=;\n\t"
      "bra WAIT_%=;\n"
      "DONE_%=:\n\t}" ::"r"(bar),
      "r"(parity)
      : "memory");
}
#endif
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar)
               : "memory");
}
__device__ __forceinline__ void tc_mma(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(1));
}
// UMMA shared-memory descriptor: K-major, no swizzle, version 1 (sm_100)
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46);
}
// instruction descriptor: f16 x f16 -> f32, K-major A/B, M=128, N
__host__ __device__ constexpr uint32_t idesc_f16(int n) {
  return (1u << 4) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[16]) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ float tmem_ld1(uint32_t taddr) {
  uint32_t r;
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(r) : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
  return __uint_as_float(r);
}
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const float (&v)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
          taddr),
      "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])),
      "r"(__float_as_uint(v[3])), "r"(__float_as_uint(v[4])), "r"(__float_as_uint(v[5])),
      "r"(__float_as_uint(v[6])), "r"(__float_as_uint(v[7])), "r"(__float_as_uint(v[8])),
      "r"(__float_as_uint(v[9])), "r"(__float_as_uint(v[10])), "r"(__float_as_uint(v[11])),
      "r"(__float_as_uint(v[12])), "r"(__float_as_uint(v[13])), "r"(__float_as_uint(v[14])),
      "r"(__float_as_uint(v[15]))
      : "memory");
}
__device__ __forceinline__ void tmem_st16_zero(uint32_t taddr) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1};" ::"r"(taddr),
      "r"(0u)
      : "memory");
}
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

__device__ __forceinline__ uint32_t pack_h2(float a, float b) {
  __half2 h = __floats2half2_rn(a, b);
  return *reinterpret_cast<uint32_t *>(&h);
}
__device__ __forceinline__ void st_shared_v4(uint32_t addr, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};" ::"r"(addr), "r"(a), "r"(b), "r"(c), "r"(d)
               : "memory");
}

// ---------------------------------------------------------------------------
struct TcParams {
  const uint8_t *w;     // this pass's weight tiles (same byte image as smem)
  const float *bias;    // G x 32 fp32
  const float *c, *z;   // HI: (B, rows, W) fp32 planes
  const float *x_in;    // !HI: (rows, 8, VW, 4) fp32 (channel-group planar)
  float *x_out;         // !HO: (rows, 8, VW, 4) fp32
  float *p;             // HO: (B, out_rows, W) (nullable)
  uint8_t *h;           // HO: (B, out_rows, W) (nullable)
  int *flag;            // HO: non-finite logit flag
  int B, W, VW, rows;   // rows = window rows held by the pass buffers
  int S, n_strips;      // strip stride (valid lanes) and count
  int r_lo, r_hi;       // output rows [r_lo, r_hi) of this pass (window-relative)
  long long chunk;      // strip-rows per CTA: CTA i owns [i*chunk, (i+1)*chunk) of
                        // the strip-major (strip, row) space, split into segments
  int out_rows;         // HO: rows of p/h (== r_hi - r_lo)
};

constexpr int NTHREADS = 544;  // warp 0: MMA issuer | warps 1-16: epilogue (2 sets of 8)

template <bool HI, int NBK, bool HO>
__global__ void __launch_bounds__(NTHREADS, 1) tc_pass_kernel(const __grid_constant__ TcParams P) {
  using PL = Plan<HI, NBK, HO>;
  constexpr int G = PL::G;
  extern __shared__ __align__(1024) uint8_t smem[];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t sbase = smem_u32(smem);
  const uint32_t bar0 = sbase + PL::BAR_OFF;
  auto a_full = [&](int j, int q) { return bar0 + 8u * (j * 2 + q); };
  auto a_empty = [&](int j, int q) { return bar0 + 8u * (2 * G + j * 2 + q); };
  auto acc_full = [&](int j) { return bar0 + 8u * (4 * G + j); };
  auto acc_free = [&](int j) { return bar0 + 8u * (5 * G + j); };
  float *bias_s = reinterpret_cast<float *>(smem + PL::BIAS_OFF);

  // ---- setup: barriers, zeroed row buffers, weights, biases, TMEM ----------
  if (tid == 0) {
    for (int j = 0; j < G; ++j) {
      const uint32_t prod = 8u;  // one epilogue set (set 0 also loads layer 0's rows)
      mbar_init(a_full(j, 0), prod);
      mbar_init(a_full(j, 1), prod);
      mbar_init(a_empty(j, 0), 1);
      mbar_init(a_empty(j, 1), 1);
      mbar_init(acc_full(j), 1);
      mbar_init(acc_free(j), 8);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  {
    const uint4 zero = make_uint4(0, 0, 0, 0);
    uint4 *ab = reinterpret_cast<uint4 *>(smem + PL::W_TOTAL);
    for (int i = tid; i < (PL::A_END - PL::W_TOTAL) / 16; i += NTHREADS) ab[i] = zero;
    const uint4 *wg = reinterpret_cast<const uint4 *>(P.w);
    uint4 *ws = reinterpret_cast<uint4 *>(smem);
    for (int i = tid; i < PL::W_TOTAL / 16; i += NTHREADS) ws[i] = __ldg(wg + i);
    for (int i = tid; i < G * 32; i += NTHREADS) bias_s[i] = __ldg(P.bias + i);
  }
  fence_proxy_async();
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(smem + PL::TMEMP_OFF);
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  // Balanced work split: this CTA owns strip-rows [q0, q1) of the strip-major
  // (strip, output row) space; it walks them as one segment per strip touched.
  const long long range = P.r_hi - P.r_lo;
  const long long q0 = (long long)blockIdx.x * P.chunk;
  const long long q1 = min(q0 + P.chunk, (long long)P.n_strips * range);
  // segment geometry at position q (identical in every role); returns the
  // position after the segment
  auto seg_geom = [&](long long q, int &v0, int &A, int &Bn, int &R0, int &R1) -> long long {
    const int s = (int)(q / range);
    const long long end = min(q1, (long long)(s + 1) * range);
    v0 = s * P.S - G;
    R0 = P.r_lo + (int)(q - (long long)s * range);
    R1 = P.r_lo + (int)(end - (long long)s * range);
    A = max(R0 - G, 0);
    Bn = min(R1 + G, P.rows);
    return end;
  };

  if (warp == 0) {
    // ===================== MMA issuer (one thread) ============================
    if (lane == 0) {
      uint32_t ph_afull = 0, ph_free = 0;
      for (long long q = q0; q < q1;) {
        int v0, A, Bn, R0, R1;
        q = seg_geom(q, v0, A, Bn, R0, R1);
        for (int t = A; t < Bn + 2 * (G - 1); ++t) {
          rev_for<G>([&](auto JC) {
            constexpr int j = decltype(JC)::value;
            const int r = t - 2 * j;
            if (r >= A && r < Bn) {
              const int q = r & 1;
              mbar_wait(a_full(j, q), (ph_afull >> (2 * j + q)) & 1);
              ph_afull ^= 1u << (2 * j + q);
              mbar_wait(acc_free(j), (ph_free >> j) & 1);
              ph_free ^= 1u << j;
              tc_fence_after();
              const int rot = r % 3;
              const int o = rot == 0 ? 1 : (rot == 1 ? 0 : 2);
              constexpr int ns = PL::ns(j), nk = PL::nk(j);
              constexpr uint32_t idesc = idesc_f16(3 * ns);
              const uint32_t a_base = sbase + PL::a_off(j) + q * PL::abytes(j);
              const uint32_t w_base = sbase + PL::w_off(j) + o * ns * 16;
              const uint32_t d = tmem + PL::tcol(j);
#pragma unroll
              for (int kx = 0; kx < 3; ++kx) {
#pragma unroll
                for (int kh = 0; kh < nk; ++kh) {
                  const uint64_t ad = umma_desc(a_base + kh * 2 * PLANE + kx * 16, PLANE, 128);
                  const uint64_t bd = umma_desc(w_base + (kx * nk + kh) * tile_bytes(ns),
                                                NSLICE * ns * 16, 128);
                  tc_mma(d, ad, bd, idesc);
                }
              }
              tc_commit(a_empty(j, q));
              tc_commit(acc_full(j));
              TRACE("MMA t=%d j=%d r=%d issued\n", t, j, r);
            }
            // no commit on the drain-only step r == Bn: the last row's data is
            // covered by the previous completion, and two back-to-back
            // completions could let a slow waiter miss a parity phase
          });
        }
      }
    }
  } else {
    // ===================== epilogue: two warp sets ============================
    // Set s handles the layers j with j % 2 == s (a conv2 and the layer that
    // holds its residual are two layers apart, so they share a set and the fp32
    // residual rows stay in the same thread's registers).  Within a set the 8
    // warps cover the 4 TMEM lane quarters x 2 channel halves.  Set 0 also
    // streams the pass input rows into layer 0's A buffer, one row ahead, with
    // the global loads prefetched a further row ahead in registers.
    const int ew = (warp - 1) & 7;
    const int quarter = warp & 3, hf = ew >> 2;
    const int l = quarter * 32 + lane;
    const uint32_t tlane = tmem + ((uint32_t)(quarter * 32) << 16);
    // one code path per set: the compiler then only keeps that set's
    // register arrays live (held / pre for conv2 residuals, pf for loads)
    auto epilogue = [&](auto SETC) {
      constexpr int set = decltype(SETC)::value;
      uint32_t ph_full = 0, ph_empty = 0, ph_in = 0;
      float held[2][16];
      float pre[16];
      constexpr int NV = HI ? 2 : 16;
      float pf[NV];
  #pragma unroll
      for (int i = 0; i < 16; ++i) { held[0][i] = held[1][i] = pre[i] = 0.f; }
      for (long long qq = q0; qq < q1;) {
        int v0, A, Bn, R0, R1;
        qq = seg_geom(qq, v0, A, Bn, R0, R1);
        const int v = v0 + l;
        const int b = v >= 0 ? v / (P.W + 1) : -1, col = v >= 0 ? v % (P.W + 1) : -1;
        const bool in_img = v >= 0 && v < P.VW && col < P.W;
        const bool lane_valid = l >= G && l < G + P.S && v >= 0 && v < P.VW;
        // pass buffers are channel-group planar: [row][group of 4 channels][v][4]
        // (float4 index), so a warp's 16-byte accesses are 512 contiguous bytes
        auto xoff = [&](int row, int g) { return ((size_t)row * 8 + g) * P.VW + v; };
        auto load_resid = [&](int e) {
  #pragma unroll
          for (int i = 0; i < 16; ++i) pre[i] = 0.f;
          if constexpr (!HI) {
            if (e < Bn && v >= 0 && v < P.VW) {
  #pragma unroll
              for (int i = 0; i < 4; ++i) {
                const float4 f = __ldg(reinterpret_cast<const float4 *>(P.x_in) + xoff(e, 4 * hf + i));
                pre[4 * i] = f.x; pre[4 * i + 1] = f.y; pre[4 * i + 2] = f.z; pre[4 * i + 3] = f.w;
              }
            }
          }
        };
        if constexpr (!HI) {
          if (set == 1) load_resid(A);   // layer 1 (a conv2) takes its residual from the pass input
        }
        // pass input row t -> registers (set 0): (c, z) or 16 channels of x
        auto load_in = [&](int t) {
  #pragma unroll
          for (int i = 0; i < NV; ++i) pf[i] = 0.f;
          if (!in_img || t >= Bn) return;
          if constexpr (HI) {
            const size_t idx = ((size_t)b * P.rows + t) * P.W + col;
            pf[0] = __ldg(P.c + idx);
            pf[1] = __ldg(P.z + idx);
          } else {
  #pragma unroll
            for (int i = 0; i < 4; ++i) {
              const float4 f = __ldg(reinterpret_cast<const float4 *>(P.x_in) + xoff(t, 4 * hf + i));
              pf[4 * i] = f.x; pf[4 * i + 1] = f.y; pf[4 * i + 2] = f.z; pf[4 * i + 3] = f.w;
            }
          }
        };
        // registers (row t) -> layer 0's A buffer, then prefetch row t+1
        auto store_in = [&](int t) {
          const int q = t & 1;
          if (t - 2 >= A) {
            if (lane == 0) mbar_wait(a_empty(0, q), (ph_in >> q) & 1);
            ph_in ^= 1u << q;
            __syncwarp();
          }
          const uint32_t dst = sbase + PL::a_off(0) + q * PL::abytes(0) + (l + 1) * 16;
          if constexpr (HI) {
            if (hf == 0) {
              // K=16 channel slots: [c_hi, c_lo, c_hi, z_hi, z_lo, z_hi, 0, 0 | 0 x 8]
              const __half ch = __float2half_rn(pf[0]);
              const __half cl = __float2half_rn(pf[0] - __half2float(ch));
              const __half zh = __float2half_rn(pf[1]);
              const __half zl = __float2half_rn(pf[1] - __half2float(zh));
              __half2 p0 = __halves2half2(ch, cl), p1 = __halves2half2(ch, zh), p2 = __halves2half2(zl, zh);
              st_shared_v4(dst, *reinterpret_cast<uint32_t *>(&p0), *reinterpret_cast<uint32_t *>(&p1),
                           *reinterpret_cast<uint32_t *>(&p2), 0u);
            }
          } else {
            const uint32_t d2 = dst + (2 * hf) * PLANE;
            st_shared_v4(d2, pack_h2(pf[0], pf[1]), pack_h2(pf[2], pf[3]), pack_h2(pf[4], pf[5]),
                         pack_h2(pf[6], pf[7]));
            st_shared_v4(d2 + PLANE, pack_h2(pf[8], pf[9]), pack_h2(pf[10], pf[11]), pack_h2(pf[12], pf[13]),
                         pack_h2(pf[14], pf[15]));
          }
          fence_proxy_async();
          __syncwarp();
          if (lane == 0) mbar_arrive(a_full(0, q));
          if (lane == 0) TRACE("LOAD warp %d stored row %d\n", warp, t);
          load_in(t + 1);
        };
        if (set == 0) load_in(A);
        for (int t = A - 2; t <= Bn + 2 * (G - 1); ++t) {
          rev_for<G>([&](auto JC) {
            constexpr int j = decltype(JC)::value;
            if constexpr ((j & 1) != set) return;
            else {
            constexpr int kind = PL::kind(j), ns = PL::ns(j);
            const int r = t - 2 * j;
            if (r >= A && r < Bn) {
              if (lane == 0) mbar_wait(acc_full(j), (ph_full >> j) & 1);
              if (lane == 0) TRACE("EPI warp %d t=%d j=%d acc_full ok\n", warp, t, j);
              ph_full ^= 1u << j;
              __syncwarp();
              tc_fence_after();
            }
            const int d = r - 1, e = r + 2;
            const bool do_drain = d >= A && d < Bn;
            const bool do_init = e >= A && e < Bn;
            // ---- 1. load the finished row d from TMEM ----
            float val[16];
            float logit = 0.f;
            if (do_drain) {
              const uint32_t taddr = tlane + PL::tcol(j) + (d % 3) * ns;
              if constexpr (kind == K_OUT) {
                if (hf == 0) logit = tmem_ld1(taddr);
              } else {
                tmem_ld16(taddr + hf * 16, val);
              }
            }
            // ---- 2. initialise slot of row e (same slot as d: after the load) and
            //         release the MMA for this layer's next row ----
            if (do_init) {
              // in place: the held / prefetched residual row is consumed exactly once
              const uint32_t taddr = tlane + PL::tcol(j) + (e % 3) * ns;
              if constexpr (kind == K_C2) {
                if constexpr (j >= 2 && PL::holds(j >= 2 ? j - 2 : 0)) {
                  constexpr int hi_ = PL::hold_idx(j - 2);
  #pragma unroll
                  for (int i = 0; i < 16; ++i) held[hi_][i] += bias_s[j * 32 + hf * 16 + i];
                  tmem_st16(taddr + hf * 16, held[hi_]);
                } else {
  #pragma unroll
                  for (int i = 0; i < 16; ++i) pre[i] += bias_s[j * 32 + hf * 16 + i];
                  tmem_st16(taddr + hf * 16, pre);
                }
              } else if (kind != K_OUT || hf == 0) {
                tmem_st16_zero(taddr + (kind == K_OUT ? 0 : hf * 16));
              }
            }
            if (r + 1 >= A && r + 1 < Bn) {
              tmem_wait_st();
              tc_fence_before();
              __syncwarp();
              if (lane == 0) mbar_arrive(acc_free(j));
            }
            if constexpr (kind == K_C2 && !(j >= 2 && PL::holds(j >= 2 ? j - 2 : 0))) {
              if (do_init) load_resid(e + 1);
            }
            // ---- 3. epilogue math + hand-off of row d ----
            if (do_drain) {
              if constexpr (kind == K_OUT) {
                if (hf == 0) {
                  logit += bias_s[j * 32];
                  if (lane_valid && in_img && d >= R0 && d < R1) {
                    if (!isfinite(logit)) atomicOr(P.flag, 1);
                    const size_t o = ((size_t)b * P.out_rows + (d - P.r_lo)) * P.W + col;
                    if (P.p) P.p[o] = 1.f / (1.f + __expf(-logit));
                    if (P.h) P.h[o] = logit >= 0.f ? 1 : 0;
                  }
                }
              } else {
  #pragma unroll
                for (int i = 0; i < 16; ++i) {
                  float x = val[i];
                  if constexpr (kind == K_IN) x += bias_s[j * 32 + hf * 16 + i];
                  if constexpr (kind == K_C1) x = fmaxf(x + bias_s[j * 32 + hf * 16 + i], 0.f);
                  val[i] = in_img ? x : 0.f;
                }
                if constexpr (PL::holds(j)) {
  #pragma unroll
                  for (int i = 0; i < 16; ++i) held[PL::hold_idx(j)][i] = val[i];
                }
                if constexpr (PL::feeds_next(j)) {
                  const int q = d & 1;
                  if (d - 2 >= A) {
                    if (lane == 0) mbar_wait(a_empty(j + 1, q), (ph_empty >> (2 * (j + 1) + q)) & 1);
                    ph_empty ^= 1u << (2 * (j + 1) + q);
                    __syncwarp();
                  }
                  const uint32_t dst = sbase + PL::a_off(j + 1) + q * PL::abytes(j + 1) + (l + 1) * 16 +
                                       (2 * hf) * PLANE;
                  st_shared_v4(dst, pack_h2(val[0], val[1]), pack_h2(val[2], val[3]), pack_h2(val[4], val[5]),
                               pack_h2(val[6], val[7]));
                  st_shared_v4(dst + PLANE, pack_h2(val[8], val[9]), pack_h2(val[10], val[11]),
                               pack_h2(val[12], val[13]), pack_h2(val[14], val[15]));
                  fence_proxy_async();
                  __syncwarp();
                  if (lane == 0) mbar_arrive(a_full(j + 1, q));
                } else {
                  // last layer of a non-output pass: fp32 x -> global
                  if (lane_valid && d >= R0 && d < R1) {
                    float4 *dstg = reinterpret_cast<float4 *>(P.x_out);
  #pragma unroll
                    for (int i = 0; i < 4; ++i)
                      dstg[xoff(d, 4 * hf + i)] = make_float4(val[4 * i], val[4 * i + 1], val[4 * i + 2], val[4 * i + 3]);
                  }
                }
              }
            }
            }  // layer of this set
          });
          if (set == 0 && t + 1 >= A && t + 1 < Bn) store_in(t + 1);
        }
        // consume the trailing a_empty completions of the buffers we produce into
  #pragma unroll
        for (int j = 0; j + 1 < G; ++j) {
          if ((j & 1) != set) continue;
          for (int t = max(A, Bn - 2); t < Bn; ++t) {
            const int q = t & 1;
            if (lane == 0) mbar_wait(a_empty(j + 1, q), (ph_empty >> (2 * (j + 1) + q)) & 1);
            ph_empty ^= 1u << (2 * (j + 1) + q);
          }
        }
        if (set == 0) {
          for (int t = max(A, Bn - 2); t < Bn; ++t) {
            const int q = t & 1;
            if (lane == 0) mbar_wait(a_empty(0, q), (ph_in >> q) & 1);
            ph_in ^= 1u << q;
          }
        }
        __syncwarp();
      }
    };
    if (((warp - 1) >> 3) == 0) epilogue(std::integral_constant<int, 0>{});
    else epilogue(std::integral_constant<int, 1>{});
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

// ---------------------------------------------------------------------------
// weight packing: fp64 params -> fp16 UMMA tiles (doubled ky sequence)
__constant__ int c_ky_of_slice[NSLICE] = {2, 1, 0, 2, 1};

__global__ void pack_tc_kernel(const double *__restrict__ prm, int NB, __half *__restrict__ dst,
                               float *__restrict__ bias) {
  const NetGeom g(C, NB);
  const int64_t n_half = weight_bytes(NB) / 2;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n_half;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t byte = i * 2;
    int kind, nk, ns;
    int64_t lstart, woff;
    if (byte < W_IN_BYTES) {
      kind = K_IN; nk = 1; ns = 32; lstart = 0; woff = g.in_w;
    } else if (byte < weight_offset_out(NB)) {
      const int ci = (int)((byte - W_IN_BYTES) / W_MID_BYTES);
      kind = K_C1; nk = 2; ns = 32; lstart = weight_offset_mid(ci);
      woff = (ci % 2 == 0) ? g.w1(ci / 2) : g.w2(ci / 2);
    } else {
      kind = K_OUT; nk = 2; ns = 16; lstart = weight_offset_out(NB); woff = g.out_w;
    }
    const int64_t off = byte - lstart;
    const int tb = tile_bytes(ns);
    const int tile = (int)(off / tb), within = (int)(off % tb);
    const int kx = tile / nk, kh = tile % nk;
    const int chunk = within / (NSLICE * ns * 16);
    const int n = (within / 16) % (NSLICE * ns);
    const int e = (within % 16) / 2;
    const int slice = n / ns, co = n % ns, ky = c_ky_of_slice[slice];
    float val = 0.f;
    if (kind == K_IN) {
      const int k = chunk * 8 + e;
      if (k < 6) {
        const int cin = k < 3 ? 0 : 1;
        const double w = prm[woff + ((int64_t)co * 2 + cin) * 9 + ky * 3 + kx];
        const __half hi = __float2half_rn((float)w);
        const float lo = (float)(w - (double)__half2float(hi));
        const int kk = k % 3;
        val = (kk == 2) ? __half2float(__float2half_rn(lo)) : __half2float(hi);
      }
    } else {
      const int ci = kh * 16 + chunk * 8 + e;
      const int cout = kind == K_OUT ? 1 : C;
      if (co < cout) val = (float)prm[woff + ((int64_t)co * C + ci) * 9 + ky * 3 + kx];
    }
    dst[i] = __float2half_rn(val);
  }
  // biases
  const int nb = (int)bias_floats(NB);
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nb; i += gridDim.x * blockDim.x) {
    const int layer = i / 32, co = i % 32;
    double b = 0.0;
    if (layer == 0) b = prm[g.in_b + co];
    else if (layer <= 2 * NB) {
      const int k = layer - 1;
      b = prm[(k % 2 == 0 ? g.b1(k / 2) : g.b2(k / 2)) + co];
    } else if (co == 0) b = prm[g.out_b];
    bias[i] = (float)b;
  }
}

int pack(const double *params, int NB, void *tc_dst, float *bias_dst, cudaStream_t st) {
  pack_tc_kernel<<<512, 256, 0, st>>>(params, NB, (__half *)tc_dst, bias_dst);
  HT_CHECK_LAUNCH();
  return HT_OK;
}

// ---------------------------------------------------------------------------
// host side: pass plan + launches
int64_t workspace_bytes(int NB, int B, int H, int W, int in_rows) {
  (void)NB; (void)H;
  const int64_t VW = (int64_t)B * (W + 1);
  return 2 * (int64_t)in_rows * VW * 32 * 4 + 256;
}

struct PassDesc {
  bool hi, ho;
  int nbk;
  int layer0;  // index of first layer (0 = conv_in, 1.. = convs, 2NB+1 = conv_out)
};

template <bool HI, int NBK, bool HO>
static int launch_pass(const TcParams &prm, int grid, cudaStream_t st) {
  using PL = Plan<HI, NBK, HO>;
  static_assert(PL::TCOLS <= 512, "TMEM columns exceeded");
  static_assert(PL::SMEM <= 232448, "shared memory exceeded");
  auto kern = tc_pass_kernel<HI, NBK, HO>;
  static bool attr = false;
  if (!attr) {
    HT_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, PL::SMEM));
    attr = true;
  }
  timing_mark_begin(st, (HI ? 100 : 0) + NBK * 10 + (HO ? 1 : 0));
  kern<<<grid, NTHREADS, PL::SMEM, st>>>(prm);
  timing_mark_end(st);
  count_launch();
  HT_CHECK_LAUNCH();
  return HT_OK;
}

int run(const void *tc_w, const float *tc_b, int NB, const float *c, const float *z, int B, int H,
        int W, int in_row0, int in_rows, int out_row0, int out_rows, float *p, uint8_t *h,
        void *ws, int64_t ws_bytes, int *flag_dev, cudaStream_t st) {
  (void)H;
  const int64_t need = workspace_bytes(NB, B, H, W, in_rows);
  HT_REQUIRE(ws_bytes >= need, "workspace too small: %lld < %lld", (long long)ws_bytes, (long long)need);
  int dev = 0, n_sm = 148;
  HT_CUDA(cudaGetDevice(&dev));
  HT_CUDA(cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev));
  const int VW = B * (W + 1);
  HT_REQUIRE((int64_t)in_rows * VW * 32 < (1ll << 31) * 16, "image too large");
  float *xa = (float *)ws;
  float *xb = xa + (size_t)in_rows * VW * 32;
  // pass plan (layers: conv_in, 2*NB convs, conv_out)
  PassDesc passes[64];
  int np = 0;
  {
    const int nb0 = NB < 2 ? NB : 2;
    passes[np++] = {true, false, nb0, 0};
    int done = nb0;
    while (NB - done > 2) { passes[np++] = {false, false, 2, 1 + 2 * done}; done += 2; }
    passes[np++] = {false, true, NB - done, 1 + 2 * done};
  }
  const uint8_t *wbase = (const uint8_t *)tc_w;
  const float *in_x = nullptr;
  float *out_x = xa;
  for (int pi = 0; pi < np; ++pi) {
    const PassDesc &pd = passes[pi];
    const int G = (pd.hi ? 1 : 0) + 2 * pd.nbk + (pd.ho ? 1 : 0);
    TcParams prm{};
    prm.w = wbase + (pd.layer0 == 0 ? 0 : weight_offset_mid(pd.layer0 - 1));
    prm.bias = tc_b + 32 * pd.layer0;
    prm.c = c; prm.z = z;
    prm.x_in = in_x;
    prm.x_out = pd.ho ? nullptr : out_x;
    prm.p = p; prm.h = h; prm.flag = flag_dev;
    prm.B = B; prm.W = W; prm.VW = VW; prm.rows = in_rows;
    prm.S = M - 2 * G;
    prm.n_strips = (VW + prm.S - 1) / prm.S;
    prm.r_lo = pd.ho ? out_row0 - in_row0 : 0;
    prm.r_hi = pd.ho ? out_row0 - in_row0 + out_rows : in_rows;
    prm.out_rows = out_rows;
    // balanced split of the strip-major (strip, row) space over the SMs; each
    // CTA gets >= 8G rows so halo recompute stays small
    const long long total = (long long)prm.n_strips * (prm.r_hi - prm.r_lo);
    long long grid = n_sm;
    if (total < grid * 8 * G) grid = (total + 8 * G - 1) / (8 * G);
    if (grid < 1) grid = 1;
    prm.chunk = (total + grid - 1) / grid;
    grid = (total + prm.chunk - 1) / prm.chunk;
    const int g = (int)grid;
    int rc;
    if (pd.hi && pd.nbk == 2 && !pd.ho) rc = launch_pass<true, 2, false>(prm, g, st);
    else if (pd.hi && pd.nbk == 1 && !pd.ho) rc = launch_pass<true, 1, false>(prm, g, st);
    else if (pd.hi && pd.nbk == 0 && !pd.ho) rc = launch_pass<true, 0, false>(prm, g, st);
    else if (!pd.hi && pd.nbk == 2 && !pd.ho) rc = launch_pass<false, 2, false>(prm, g, st);
    else if (!pd.hi && pd.nbk == 2 && pd.ho) rc = launch_pass<false, 2, true>(prm, g, st);
    else if (!pd.hi && pd.nbk == 1 && pd.ho) rc = launch_pass<false, 1, true>(prm, g, st);
    else if (!pd.hi && pd.nbk == 0 && pd.ho) rc = launch_pass<false, 0, true>(prm, g, st);
    else return fail(HT_E_UNSUPPORTED, "no kernel for pass (hi=%d nbk=%d ho=%d)", pd.hi, pd.nbk, pd.ho);
    if (rc) return rc;
    in_x = out_x;
    out_x = (out_x == xa) ? xb : xa;
  }
  return HT_OK;
}

}  // namespace tc
}  // namespace ht
