// K1: fused tensor-core policy forward + sigmoid/threshold epilogue, sm_100a.
//
// Replaces PolicyNetwork.forward (nn.py:138-150) and the threshold of
// rl.infer_halftone (rl.py:306-311).  Design:
//
// * Row streaming.  A CTA owns a 128-pixel-wide strip of the "virtual image"
//   (the B images laid side by side, one zero column between neighbours) and
//   a band of rows.  Each UMMA M-tile is one strip row: 128 pixels = 128 TMEM
//   lanes.  The network runs as passes of <=4 conv layers; inside a pass every
//   layer streams rows top to bottom in a diagonal wavefront (layer j consumes
//   its input row t-3j at step t), so three input rows per layer live in
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
// * Roles (128*G threads): one 4-warp group per layer drains its TMEM ring,
//   re-initialises slots, issues its own MMAs (elected lane) and hands rows on
//   (TMEM -> registers -> bias, ReLU, fp16 -> next layer's shared-memory row /
//   global x / p,h).  Group 0 also loads the pass input rows.  Hand-offs use
//   mbarriers; tcgen05.commit signals MMA completion.
#include <cuda_fp16.h>

#include <type_traits>

#include "common.cuh"
#include "fwd_tc.cuh"
#include "tc_ptx.cuh"

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
// Wavefront skew: layer j processes input row t - SKEW*j at step t, so a row
// handed over at step t is consumed at step t+1 and a layer never waits on a
// hand-off of the same step.
constexpr int SKEW = 3;
// Input-row buffers per layer (Plan::NAB): three decouple producer and
// consumer fully; two suffice when shared memory is tight (a producer then
// waits, via a_empty, only for the consumer's MMA issued two steps earlier).
// A plan takes three when the layout still fits the 196 KB carveout, so the
// L1 left for the pass-buffer loads stays >= 60 KB.
constexpr int SMEM_L1_FRIENDLY = 196 * 1024 - 1024;
constexpr int NLINK = 4;   // residual rows in flight between a holder and its conv2


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
  // NAB input-row buffers per layer (ring indexed by row)
  static constexpr int a_bytes_total(int nab) {
    int t = 0;
    for (int j = 0; j < G; ++j) t += nab * abytes(j);
    return t;
  }
  static constexpr int NAB =
      W_TOTAL + A_PHASE + a_bytes_total(3) + ((2 * 3 + 1) * G + 2 * NLINK) * 8 + 16 <= SMEM_L1_FRIENDLY ? 3 : 2;
  static constexpr int a_off(int j) { return j == 0 ? W_TOTAL + A_PHASE : a_off(j - 1) + NAB * abytes(j - 1); }
  static constexpr int A_END = a_off(G - 1) + NAB * abytes(G - 1);
  // barriers: a_full[G][3], a_empty[G][3], acc_full[G], link_full[4], link_empty[4]
  static constexpr int BAR_OFF = A_END;
  static constexpr int NBAR = (2 * NAB + 1) * G + 2 * NLINK;
  static constexpr int TMEMP_OFF = BAR_OFF + NBAR * 8;
  static constexpr int SMEM = TMEMP_OFF + 16;
  static constexpr int tcol(int j) { return j == 0 ? 0 : tcol(j - 1) + 3 * ns(j - 1); }
  static constexpr int LINK_COL = tcol(G - 1) + 3 * ns(G - 1);   // residual link: 4 rows x 32 fp32
  static constexpr int TCOLS = LINK_COL + 32 * NLINK;
  static constexpr bool feeds_next(int j) { return j < G - 1; }
  // layer j's output is the residual of layer j+2 (a conv2) -> written to the TMEM link
  static constexpr bool holds(int j) {
    return (kind(j) == K_IN || kind(j) == K_C2) && j + 2 < G && kind(j + 2) == K_C2;
  }
  // a conv2 whose residual comes from the pass input (global) instead of the link
  static constexpr bool global_resid(int j) { return kind(j) == K_C2 && !(j >= 2 && holds(j - 2)); }
};

// ---------------------------------------------------------------------------
// PTX helpers
#ifdef HT_TIMELINE
// debug timeline of CTA 0: per-role private slots (no atomics), (ev, t, j, clock)
__device__ long long g_tl[4][4 * 16384];
#define TL_DECL int tl_n_ = 0;
#define TL(role, ev, t, j) do { if (blockIdx.x == 0 && tl_n_ < 16384) { long long *p_ = &g_tl[role][4 * tl_n_++]; \
  p_[0] = (ev); p_[1] = (t); p_[2] = (j); p_[3] = clock64(); } } while (0)
#else
#define TL_DECL
#define TL(role, ev, t, j) do {} while (0)
#endif
#ifdef HT_PROF
// per (group, warp-in-group 0/1) cycle accumulators of CTA 0, lane 0
__device__ long long g_prof[8][16];
#define PROF_DECL long long pacc_[16] = {0}; long long pt_ = clock64();
#define PROF_MARK(k) do { long long n_ = clock64(); pacc_[k] += n_ - pt_; pt_ = n_; } while (0)
#define PROF_DUMP(slot) do { if (blockIdx.x == 0 && lane == 0 && (slot) < 8) \
  for (int k_ = 0; k_ < 16; ++k_) g_prof[slot][k_] = pacc_[k_]; } while (0)
#else
#define PROF_DECL
#define PROF_MARK(k) do {} while (0)
#define PROF_DUMP(set) do {} while (0)
#endif
#ifdef HT_TRACE
#define TRACE(...) do { if (blockIdx.x == 0) printf(__VA_ARGS__); } while (0)
#else
#define TRACE(...) do {} while (0)
#endif
__device__ __forceinline__ void tc_mma(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(1));
}
// one elected lane of a converged warp issues the MMA (keeps operands uniform)
__device__ __forceinline__ void tc_mma_elect(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(1));
}
// One row's MMA batch: for kx in 0..2, kh in 0..NK-1 one M=128 x N=3*NS x K=16
// UMMA with A = a + kh*AK + kx and B = b + (kx*NK + kh)*TB (descriptor units of
// 16 B), then commit to acc_full (and a_empty when bar_e != 0).  One elect for
// the whole batch and immediate offsets keep the issue to a few instructions.
template <int NK, int NS>
__device__ __forceinline__ void mma_row(uint32_t d, uint64_t a, uint64_t b, uint32_t bar_acc, uint32_t bar_e) {
  constexpr uint32_t idesc = (1u << 4) | ((uint32_t)((3 * NS) >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
  constexpr long long AK = (2 * 2176) >> 4;   // checked against PLANE below
  constexpr long long TB = (2 * 5 * NS * 16) >> 4;
  if constexpr (NK == 2) {
    asm volatile(
        "{\n\t.reg .pred e, p, q;\n\t.reg .b64 a1, a2, a3, a4, a5, b1, b2, b3, b4, b5;\n\t"
        "setp.ne.b32 p, %3, 0;\n\t"
        "setp.ne.b32 q, %5, 0;\n\t"
        "add.s64 a1, %1, %6;\n\tadd.s64 b1, %2, %7;\n\t"
        "add.s64 a2, %1, 1;\n\tadd.s64 b2, %2, %8;\n\t"
        "add.s64 a3, %1, %9;\n\tadd.s64 b3, %2, %10;\n\t"
        "add.s64 a4, %1, 2;\n\tadd.s64 b4, %2, %11;\n\t"
        "add.s64 a5, %1, %12;\n\tadd.s64 b5, %2, %13;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %14, p;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a1, b1, %14, p;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a2, b2, %14, p;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a3, b3, %14, p;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a4, b4, %14, p;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a5, b5, %14, p;\n\t"
        "and.pred q, q, e;\n\t"
        "@q tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%5];\n\t"
        "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%4];\n\t}"
        ::"r"(d), "l"(a), "l"(b), "r"(1), "r"(bar_acc), "r"(bar_e),
        "n"(AK), "n"(TB), "n"(2 * TB), "n"(AK + 1), "n"(3 * TB), "n"(4 * TB), "n"(AK + 2), "n"(5 * TB),
        "r"(idesc)
        : "memory");
  } else {
    asm volatile(
        "{\n\t.reg .pred e, p, q;\n\t.reg .b64 a1, a2, b1, b2;\n\t"
        "setp.ne.b32 p, %3, 0;\n\t"
        "setp.ne.b32 q, %5, 0;\n\t"
        "add.s64 a1, %1, 1;\n\tadd.s64 b1, %2, %6;\n\t"
        "add.s64 a2, %1, 2;\n\tadd.s64 b2, %2, %7;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %8, p;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a1, b1, %8, p;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a2, b2, %8, p;\n\t"
        "and.pred q, q, e;\n\t"
        "@q tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%5];\n\t"
        "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%4];\n\t}"
        ::"r"(d), "l"(a), "l"(b), "r"(1), "r"(bar_acc), "r"(bar_e), "n"(TB), "n"(2 * TB), "r"(idesc)
        : "memory");
  }
}
static_assert(PLANE == 2176, "mma_row's A chunk offset assumes PLANE == 2176");

// ---------------------------------------------------------------------------
struct TcParams {
  const uint8_t *w;     // this pass's weight tiles (same byte image as smem)
  int layer0;           // index of the pass's first layer (0 = conv_in)
  const float *c, *z;   // HI: (B, rows, W) fp32 planes
  const float *x_in;    // !HI: (rows, 8, VW, 4) fp32 (channel-group planar)
  float *x_out;         // !HO: (rows, 8, VW, 4) fp32
  float *p;             // HO: (B, out_rows, W) (nullable)
  uint8_t *h;           // HO: (B, out_rows, W) (nullable)
  uint32_t *pbm;        // HO: PBM P4 payload as words (nullable; zeroed, padded to 4 B)
  int pbm_rb;           // bytes per PBM row, ceil(W / 8)
  int *flag;            // HO: non-finite logit flag
  int B, W, VW, rows;   // rows = window rows held by the pass buffers
  long long pitch;      // pass-buffer pixels per (row, channel group): x_pitch(VW)
  int S, n_strips;      // strip stride (valid lanes) and count
  int r_lo, r_hi;       // output rows [r_lo, r_hi) of this pass (window-relative)
  long long chunk;      // strip-rows per CTA: CTA i owns [i*chunk, (i+1)*chunk) of
                        // the strip-major (strip, row) space, split into segments
  int out_rows;         // HO: rows of p/h (== r_hi - r_lo)
  int steps;            // HO: output lattice i/steps (1 = binary halftone)
  // this pass's biases (<= 4 layers x 32), read from the kernel-parameter
  // constant bank (not SMEM: the tensor core's operand reads saturate
  // shared-memory bandwidth).  Per launch, so concurrent forwards of
  // different networks never share mutable state.
  float bias[4][32];
};

#define PBIAS(j, i) P.bias[(j)][(i)]

// One 4-warp group per layer (128 threads = the 128 pixel lanes of a strip
// row; warp k of a group owns TMEM lane quarter k; each thread owns one pixel
// and all 32 channels).  Per step t a group, for its layer j and input row
// r = t - SKEW*j:
//   1. waits for MMA(r) to complete (acc_full; retires all earlier MMAs too)
//   2. loads the finished output row d = r-1 from its TMEM slot
//   3. row d: bias, ReLU, zero padding, residual-link write, fp16 pack
//   4. re-initialises that slot for row e = r+2 (zero, or residual + bias;
//      the residual comes from the pass input or from the TMEM link)
//   5. (layer 0 only) stores pass-input row r+1 into its A buffer
//   6. group barrier, then one elected thread issues MMA(r+1) (6 UMMAs); the
//      previous layer handed row r+1 over at step t-1 (a_full)
//   7. hands row d on while MMA(r+1) runs: fp16 row into the next layer's A
//      buffer (d mod 3), or fp32 x to global / p,h for the output layer.
// With SKEW = 3 no layer waits on a hand-off of the same step, so every group
// re-issues as soon as its own accumulator is drained and the tensor pipe
// always has queued work from some layer.
template <bool HI, int NBK, bool HO>
__global__ void __launch_bounds__(128 * Plan<HI, NBK, HO>::G, 1) tc_pass_kernel(const __grid_constant__ TcParams P) {
  using PL = Plan<HI, NBK, HO>;
  constexpr int G = PL::G;
  constexpr int NT = 128 * G;
  constexpr int NABUF = PL::NAB;
  extern __shared__ __align__(1024) uint8_t smem[];
  // the next pass may be scheduled now: its CTAs take SMs as ours exit and
  // run their prologue (weights, barriers, TMEM) before waiting for us
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int tid = threadIdx.x, lane = tid & 31;
  const int warp = __shfl_sync(0xffffffffu, tid >> 5, 0);   // warp-uniform
  const uint32_t sbase = smem_u32(smem);
  const uint32_t bar0 = sbase + PL::BAR_OFF;
  auto a_full = [&](int j, int q) { return bar0 + 8u * (j * NABUF + q); };
  auto a_empty = [&](int j, int q) { return bar0 + 8u * (NABUF * G + j * NABUF + q); };
  auto acc_full = [&](int j) { return bar0 + 8u * (2 * NABUF * G + j); };
  auto link_full = [&](int q) { return bar0 + 8u * ((2 * NABUF + 1) * G + q); };
  auto link_empty = [&](int q) { return bar0 + 8u * ((2 * NABUF + 1) * G + NLINK + q); };

  // ---- setup: barriers, zeroed row buffers, weights, TMEM --------------------
  if (tid == 0) {
    for (int j = 0; j < G; ++j) {
      for (int q = 0; q < NABUF; ++q) {
        mbar_init(a_full(j, q), 4);   // the producing group's 4 warps
        mbar_init(a_empty(j, q), 1);  // tcgen05.commit
      }
      mbar_init(acc_full(j), 1);
    }
    for (int q = 0; q < NLINK; ++q) {
      mbar_init(link_full(q), 4);
      mbar_init(link_empty(q), 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  {
    const uint4 zero = make_uint4(0, 0, 0, 0);
    uint4 *ab = reinterpret_cast<uint4 *>(smem + PL::W_TOTAL);
    for (int i = tid; i < (PL::A_END - PL::W_TOTAL) / 16; i += NT) ab[i] = zero;
    const uint4 *wg = reinterpret_cast<const uint4 *>(P.w);
    uint4 *ws = reinterpret_cast<uint4 *>(smem);
    for (int i = tid; i < PL::W_TOTAL / 16; i += NT) ws[i] = __ldg(wg + i);
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
  const uint32_t tmem = __shfl_sync(0xffffffffu, *tmem_slot, 0);
  // programmatic dependent launch: the previous pass (which wrote our input
  // rows and last read the buffer we write) has completed past this point
  asm volatile("griddepcontrol.wait;" ::: "memory");

  // Balanced work split: this CTA owns strip-rows [q0, q1) of the strip-major
  // (strip, output row) space; it walks them as one segment per strip touched.
  const long long range = P.r_hi - P.r_lo;
  const long long q0 = (long long)blockIdx.x * P.chunk;
  const long long q1 = min(q0 + P.chunk, (long long)P.n_strips * range);
  auto seg_geom = [&](long long q, int &v0, int &A, int &Bn, int &R0, int &R1) -> long long {
    const int s = (int)(q / range);
    const long long end = min(q1, (long long)(s + 1) * range);
    v0 = s * P.S - STRIP_L;
    R0 = P.r_lo + (int)(q - (long long)s * range);
    R1 = P.r_lo + (int)(end - (long long)s * range);
    A = max(R0 - G, 0);
    Bn = min(R1 + G, P.rows);
    return end;
  };

  const int wq = warp & 3;                 // lane quarter == warp index within the group
  const int l = wq * 32 + lane;            // strip lane (pixel) of this thread
  const uint32_t tlane = tmem + ((uint32_t)(wq * 32) << 16);

  auto group = [&](auto JC) {
    constexpr int j = decltype(JC)::value;
    constexpr int kind = PL::kind(j), ns = PL::ns(j), nk = PL::nk(j);
    constexpr bool LINK_IN = kind == K_C2 && !PL::global_resid(j);
    constexpr bool GRES = PL::global_resid(j) && !HI;
    uint32_t ph_acc = 0, ph_af = 0, ph_ae = 0, ph_lf = 0, ph_le = 0;
    TL_DECL
    // timeline of the mid pass only (CTA 0, warp 0 of each group, lane 0)
#define TLG(ev) do { if constexpr (!HI && !HO) { if (wq == 0 && lane == 0) TL(j, ev, t, r); } } while (0)
    float vals[32];
    // layer 0: pass-input rows / global-residual conv2: residual rows, prefetched
    // one step ahead (aux = next row to use)
    float aux[32];
    PROF_DECL
    for (long long qq = q0; qq < q1;) {
      int v0, A, Bn, R0, R1;
      qq = seg_geom(qq, v0, A, Bn, R0, R1);
      const int v = v0 + l;
      const int b = v >= 0 ? v / (P.W + 1) : -1, col = v >= 0 ? v % (P.W + 1) : -1;
      const bool in_img = v >= 0 && v < P.VW && col < P.W;
      const bool lane_valid = l >= STRIP_L && l < STRIP_L + P.S && v >= 0 && v < P.VW;
      // pass buffers are channel-group planar: [row][group of 4 channels][v][4]
      auto xoff = [&](int row, int g) { return ((size_t)row * 8 + g) * P.pitch + v + XPAD; };
      auto load_row32 = [&](int row, float (&dst)[32]) {   // fp32 x row (0 outside)
#pragma unroll
        for (int i = 0; i < 32; ++i) dst[i] = 0.f;
        if (row < Bn && v >= 0 && v < P.VW) {
#pragma unroll
          for (int g = 0; g < 8; ++g) {
            const float4 f = ldg_stream(reinterpret_cast<const float4 *>(P.x_in) + xoff(row, g));
            dst[4 * g] = f.x; dst[4 * g + 1] = f.y; dst[4 * g + 2] = f.z; dst[4 * g + 3] = f.w;
          }
        }
      };
      auto load_in = [&](int row, float (&dst)[32]) {      // pass input row
        if constexpr (HI) {
          dst[0] = dst[1] = 0.f;
          if (in_img && row < Bn) {
            const size_t idx = ((size_t)b * P.rows + row) * P.W + col;
            dst[0] = __ldg(P.c + idx);
            dst[1] = __ldg(P.z + idx);
          }
        } else {
          load_row32(row, dst);
        }
      };
      // one-row prefetch: aux holds the next row to use; refill after use
      auto advance = [&](int row) {
        if constexpr (j == 0) load_in(row, aux);
        else load_row32(row, aux);
      };
      if constexpr (j == 0) load_in(A, aux);
      if constexpr (GRES) load_row32(A, aux);
      // a warp whose 32 pixels are all inside the image skips the zero padding
      const bool warp_in = __all_sync(0xffffffffu, in_img);
      const int t_end = Bn + SKEW * (G - 1);
      int tm3 = ((A - 3 - SKEW * j) % 3 + 3) % 3;   // (r - 1) mod 3 at t = A - 2, tracked incrementally
      for (int t = A - 2; t <= t_end; ++t) {
        const int r = t - SKEW * j;
        const int d = r - 1, e = r + 2;
        const int slot = tm3;                      // slot (and A buffer) of rows d and e (e = d + 3)
        tm3 = tm3 == 2 ? 0 : tm3 + 1;
        if (r < A - 2 || r > Bn) continue;         // layer idle at this step
        auto &resbuf = aux;
        auto &inbuf = aux;
        PROF_MARK(0);
        // ---- 1. wait for MMA(r) (it also retires every earlier MMA of this layer)
        if (r >= A && r < Bn) {
          if (lane == 0) mbar_wait(acc_full(j), ph_acc & 1);
          ph_acc ^= 1u;
          __syncwarp();
          tc_fence_after();
        }
        PROF_MARK(1);
        TLG(1);
        const uint32_t taddr = tlane + PL::tcol(j) + slot * ns;
        // ---- 2. finished row d -> registers
        const bool drain = d >= A && d < Bn;
        if (drain) {
          if constexpr (kind == K_OUT) vals[0] = tmem_ld1(taddr);
          else tmem_ld32(taddr, vals);
        }
        PROF_MARK(2);
        TLG(6);
        TLG(7);
        // ---- 3. re-initialise the slot for row e: zero (bias is added at
        //         hand-off) or, for a conv2, residual + bias
        if (e >= A && e < Bn) {
          if constexpr (kind == K_C2) {
            if constexpr (LINK_IN) {
              const int lq = e & (NLINK - 1);
              if (lane == 0) mbar_wait(link_full(lq), (ph_lf >> lq) & 1);
              ph_lf ^= 1u << lq;
              __syncwarp();
              tc_fence_after();
              tmem_ld32(tlane + PL::LINK_COL + lq * 32, resbuf);
              tc_fence_before();
              __syncwarp();
              if (lane == 0) mbar_arrive(link_empty(lq));
#pragma unroll
              for (int i = 0; i < 32; ++i) resbuf[i] += PBIAS(j, i);
              tmem_st32(taddr, resbuf);
            } else {
#pragma unroll
              for (int i = 0; i < 32; ++i) resbuf[i] += PBIAS(j, i);
              tmem_st32(taddr, resbuf);
              if constexpr (GRES) advance(e + 1);
            }
          } else if constexpr (kind == K_OUT) {
            tmem_st16_zero(taddr);
          } else {
            tmem_st32_zero(taddr);
          }
        }
        PROF_MARK(3);
        TLG(8);
        // ---- 4. layer 0: pass-input row r+1 -> its A buffer.  The previous
        //         row there (r+1-NABUF) was read by an MMA retired in step 1.
        const int rn = r + 1;
        const int rot = slot == 0 ? 2 : slot - 1;  // (r+1) mod 3: TMEM ring position of row r+1
        const int qn = NABUF == 3 ? rot : (rn & 1);  // A buffer of row r+1
        const bool issue = rn >= A && rn < Bn;
        if constexpr (j == 0) {
          if (issue) {
            const uint32_t dst = sbase + PL::a_off(0) + qn * PL::abytes(0) + (l + 1) * 16;
            if constexpr (HI) {
              // K=16 channel slots: [c_hi, c_lo, c_hi, z_hi, z_lo, z_hi, 0, 0 | 0 x 8]
              const __half ch = __float2half_rn(inbuf[0]);
              const __half cl = __float2half_rn(inbuf[0] - __half2float(ch));
              const __half zh = __float2half_rn(inbuf[1]);
              const __half zl = __float2half_rn(inbuf[1] - __half2float(zh));
              __half2 p0 = __halves2half2(ch, cl), p1 = __halves2half2(ch, zh), p2 = __halves2half2(zl, zh);
              st_shared_v4(dst, *reinterpret_cast<uint32_t *>(&p0), *reinterpret_cast<uint32_t *>(&p1),
                           *reinterpret_cast<uint32_t *>(&p2), 0u);
            } else {
#pragma unroll
              for (int c4 = 0; c4 < 4; ++c4)
                st_shared_v4(dst + c4 * PLANE, pack_h2(inbuf[8 * c4], inbuf[8 * c4 + 1]),
                             pack_h2(inbuf[8 * c4 + 2], inbuf[8 * c4 + 3]), pack_h2(inbuf[8 * c4 + 4], inbuf[8 * c4 + 5]),
                             pack_h2(inbuf[8 * c4 + 6], inbuf[8 * c4 + 7]));
            }
            fence_proxy_async();
            advance(rn + 1);
          }
        }
        PROF_MARK(4);
        // ---- 5. group barrier, then issue MMA(r+1): its input row was handed
        //         over by layer j-1 at step t-1
        if (issue) {
          tmem_wait_st();
          tc_fence_before();
          named_bar(1 + j, 128);
          PROF_MARK(6);
          TLG(2);
          if (wq == 0) {
            if constexpr (j > 0) {
              if (lane == 0) mbar_wait(a_full(j, qn), (ph_af >> qn) & 1);
              ph_af ^= 1u << qn;
            }
            __syncwarp();
            PROF_MARK(7);
            TLG(3);
            tc_fence_after();
            const int o = rot == 0 ? 1 : (rot == 1 ? 0 : 2);   // B window for output rows (r+2, r+1, r)
            constexpr uint32_t lbo_b = NSLICE * ns * 16;
            const uint64_t adesc0 = umma_desc(sbase, PLANE, 128);
            const uint64_t bdesc0 = (adesc0 & ~(0x3FFFull << 16)) | ((uint64_t)(lbo_b >> 4) << 16);
            const uint32_t a_add = (PL::a_off(j) + qn * PL::abytes(j)) >> 4;
            const uint32_t b_add = (PL::w_off(j) + o * ns * 16) >> 4;
            mma_row<nk, ns>(tmem + PL::tcol(j), adesc0 + a_add, bdesc0 + b_add, acc_full(j),
                            j > 0 ? a_empty(j, qn) : 0u);
            __syncwarp();
            PROF_MARK(8);
            TLG(4);
          }
        }
        // ---- 6. row d: activation, residual link, fp16 pack (after the issue:
        //         off the drain -> issue critical path)
        uint32_t hv[16];
        if constexpr (kind != K_OUT) {
          if (drain) {
#pragma unroll
            for (int i = 0; i < 32; ++i) {
              float x = vals[i];
              if constexpr (kind != K_C2) x += PBIAS(j, i);
              if constexpr (kind == K_C1) x = fmaxf(x, 0.f);
              vals[i] = x;
            }
            if (!warp_in) {
#pragma unroll
              for (int i = 0; i < 32; ++i) vals[i] = in_img ? vals[i] : 0.f;
            }
            if constexpr (PL::feeds_next(j)) {
#pragma unroll
              for (int i = 0; i < 16; ++i) hv[i] = pack_h2(vals[2 * i], vals[2 * i + 1]);
            }
          }
        }
        // ---- 7. hand row d on (overlaps MMA(r+1))
        if (drain) {
          if constexpr (kind == K_OUT) {
            const float logit = vals[0] + PBIAS(j, 0);
            const bool px = lane_valid && in_img && d >= R0 && d < R1;
            if (px) {
              if (!isfinite(logit)) atomicOr(P.flag, 1);
              const size_t o = ((size_t)b * P.out_rows + (d - P.r_lo)) * P.W + col;
              if (P.p) P.p[o] = 1.f / (1.f + __expf(-logit));
              if (P.h) P.h[o] = level_of(logit, P.steps);
            }
            if (P.pbm) {
              // PBM P4 bits straight from the logits (imagecore.py:289-297:
              // bit = 1 - h = black, MSB first, rows padded to bytes): the
              // warp's bits are OR-reduced per 32-bit word of the payload
              // (its 32 columns touch <= 3 words per image row; a strip's
              // edge word is shared with the neighbouring strip's CTA)
              uint32_t widx = 0xffffffffu, val = 0u;
              if (px) {
                const uint32_t byte =
                    (uint32_t)(((size_t)b * P.out_rows + (d - P.r_lo)) * P.pbm_rb + (col >> 3));
                widx = byte >> 2;
                val = (logit >= 0.f ? 0u : 1u) << (7 - (col & 7) + 8 * (byte & 3));
              }
              const unsigned peers = __match_any_sync(0xffffffffu, widx);
              const uint32_t orv = __reduce_or_sync(peers, val);
              if (px && orv && lane == __ffs(peers) - 1) atomicOr(P.pbm + widx, orv);
            }
          } else if constexpr (PL::feeds_next(j)) {
            const int q = NABUF == 3 ? slot : (d & 1);   // A buffer of row d
            PROF_MARK(9);
            if (d - NABUF >= A) {
              if (lane == 0) mbar_wait(a_empty(j + 1, q), (ph_ae >> q) & 1);
              ph_ae ^= 1u << q;
              __syncwarp();
            }
            PROF_MARK(10);
            const uint32_t dst = sbase + PL::a_off(j + 1) + q * PL::abytes(j + 1) + (l + 1) * 16;
#pragma unroll
            for (int c4 = 0; c4 < 4; ++c4)
              st_shared_v4(dst + c4 * PLANE, hv[4 * c4], hv[4 * c4 + 1], hv[4 * c4 + 2], hv[4 * c4 + 3]);
            PROF_MARK(11);
            fence_proxy_async();
            PROF_MARK(12);
            __syncwarp();
            if (lane == 0) mbar_arrive(a_full(j + 1, q));
            PROF_MARK(13);
            // the residual link for layer j+2 after the hand-off to layer
            // j+1 (the link has steps of slack, the hand-off does not:
            // mid pass 1.546 -> 1.520 ms)
            if constexpr (PL::holds(j)) {
              const int lq = d & (NLINK - 1);
              PROF_MARK(14);
              if (d - NLINK >= A) {
                if (lane == 0) mbar_wait(link_empty(lq), (ph_le >> lq) & 1);
                ph_le ^= 1u << lq;
                __syncwarp();
              }
              PROF_MARK(15);
              tc_fence_after();
              tmem_st32(tlane + PL::LINK_COL + lq * 32, vals);
              tmem_wait_st();
              tc_fence_before();
              __syncwarp();
              if (lane == 0) mbar_arrive(link_full(lq));
            }
          } else {
            // last layer of a non-output pass: fp32 x -> global
            if (lane_valid && d >= R0 && d < R1) {
              float4 *dstg = reinterpret_cast<float4 *>(P.x_out);
#pragma unroll
              for (int g = 0; g < 8; ++g)
                dstg[xoff(d, g)] = make_float4(vals[4 * g], vals[4 * g + 1], vals[4 * g + 2], vals[4 * g + 3]);
            }
          }
        }
        PROF_MARK(5);
        TLG(5);
      }
      // consume the trailing completions this group waits on as a producer
      if constexpr (PL::feeds_next(j)) {
        for (int rr = max(A, Bn - NABUF); rr < Bn; ++rr) {
          const int q = rr % NABUF;
          if (lane == 0) mbar_wait(a_empty(j + 1, q), (ph_ae >> q) & 1);
          ph_ae ^= 1u << q;
        }
      }
      if constexpr (PL::holds(j)) {
        for (int rr = max(A, Bn - NLINK); rr < Bn; ++rr) {
          const int lq = rr & (NLINK - 1);
          if (lane == 0) mbar_wait(link_empty(lq), (ph_le >> lq) & 1);
          ph_le ^= 1u << lq;
        }
      }
      __syncwarp();
    }
    if (wq < 2 && !HO && !HI) PROF_DUMP(j * 2 + wq);
  };
  // dispatch: warps [4j, 4j+4) run layer j
  const int grp = warp >> 2;
  if constexpr (G >= 1) { if (grp == 0) group(std::integral_constant<int, 0>{}); }
  if constexpr (G >= 2) { if (grp == 1) group(std::integral_constant<int, 1>{}); }
  if constexpr (G >= 3) { if (grp == 2) group(std::integral_constant<int, 2>{}); }
  if constexpr (G >= 4) { if (grp == 3) group(std::integral_constant<int, 3>{}); }

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
  return 2 * (int64_t)in_rows * x_pitch((int)VW) * 32 * 4 + 256;
}

struct PassDesc {
  bool hi, ho;
  int nbk;
  int layer0;  // index of first layer (0 = conv_in, 1.. = convs, 2NB+1 = conv_out)
};

// pdl: launched as a programmatic dependent of the previous pass (its
// prologue overlaps that pass's tail); not while per-pass timing events are
// recorded between the launches
template <bool HI, int NBK, bool HO>
static int launch_pass(const TcParams &prm, int grid, cudaStream_t st, bool pdl) {
  using PL = Plan<HI, NBK, HO>;
  static_assert(PL::G <= 4 && PL::G <= STRIP_L, "at most 4 layers per pass (halo <= STRIP_L lanes)");
  static_assert(PL::TCOLS <= 512, "TMEM columns exceeded");
  static_assert(PL::SMEM <= 232448, "shared memory exceeded");
  auto kern = tc_pass_kernel<HI, NBK, HO>;
  if (int rc = ensure_smem_attr((const void *)kern, PL::SMEM)) return rc;
  timing_mark_begin(st, (HI ? 100 : 0) + NBK * 10 + (HO ? 1 : 0));
  if (pdl && !timing_enabled()) {
    cudaLaunchConfig_t cfg{};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.gridDim = dim3((unsigned)grid, 1, 1);
    cfg.blockDim = dim3(128 * PL::G, 1, 1);
    cfg.dynamicSmemBytes = PL::SMEM;
    cfg.stream = st;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    HT_CUDA(cudaLaunchKernelEx(&cfg, kern, prm));
  } else {
    kern<<<grid, 128 * PL::G, PL::SMEM, st>>>(prm);
  }
  timing_mark_end(st);
  count_launch();
  HT_CHECK_LAUNCH();
  return HT_OK;
}

int run(const void *tc_w, const float *tc_b, int NB, const float *c, const float *z, int B, int H,
        int W, int in_row0, int in_rows, int out_row0, int out_rows, float *p, uint8_t *h,
        uint32_t *pbm_words, void *ws, int64_t ws_bytes, int *flag_dev, int levels, cudaStream_t st) {
  (void)H;
  const int64_t need = workspace_bytes(NB, B, H, W, in_rows);
  HT_REQUIRE(ws_bytes >= need, "workspace too small: %lld < %lld", (long long)ws_bytes, (long long)need);
  int dev = 0, n_sm = 148;
  HT_CUDA(cudaGetDevice(&dev));
  HT_CUDA(cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev));
  const int VW = B * (W + 1);
  HT_REQUIRE((int64_t)in_rows * VW * 32 < (1ll << 31) * 16, "image too large");
  float *xa = (float *)ws;
  float *xb = xa + (size_t)in_rows * x_pitch(VW) * 32;
  // pass plan (layers: conv_in, 2*NB convs, conv_out)
  constexpr int MAX_PASSES = 64;
  HT_REQUIRE(NB / 2 + 2 <= MAX_PASSES, "too many residual blocks for the fused forward (%d)", NB);
  const float *hb = nullptr;
  if (int rc = host_biases(tc_b, bias_floats(NB), st, &hb)) return rc;
  PassDesc passes[MAX_PASSES];
  int np = 0;
  {
    // <= 4 layers per pass: conv_in + 1 block | 2 blocks ... | <=1 block + conv_out
    const int nb0 = NB < 1 ? NB : 1;
    passes[np++] = {true, false, nb0, 0};
    int done = nb0;
    while (NB - done > 1) { passes[np++] = {false, false, 2, 1 + 2 * done}; done += 2; }
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
    prm.layer0 = pd.layer0;
    for (int j = 0; j < G; ++j)
      for (int i = 0; i < 32; ++i) prm.bias[j][i] = hb[(pd.layer0 + j) * 32 + i];
    prm.c = c; prm.z = z;
    prm.x_in = in_x;
    prm.x_out = pd.ho ? nullptr : out_x;
    prm.p = p; prm.h = h; prm.flag = flag_dev;
    prm.pbm = pd.ho ? pbm_words : nullptr;
    prm.pbm_rb = (W + 7) / 8;
    prm.B = B; prm.W = W; prm.VW = VW; prm.rows = in_rows;
    prm.S = STRIP_S;
    prm.pitch = x_pitch(VW);
    prm.n_strips = (VW + prm.S - 1) / prm.S;
    prm.r_lo = pd.ho ? out_row0 - in_row0 : 0;
    prm.r_hi = pd.ho ? out_row0 - in_row0 + out_rows : in_rows;
    prm.out_rows = out_rows;
    prm.steps = levels - 1;
    // balanced split of the strip-major (strip, row) space over the SMs.  A
    // small image still spreads over every SM (down to G rows per CTA):
    // idle SMs are worth more than the extra halo recompute -- the latency
    // of one 256^2 image drops from 0.86 to 0.59 ms (debug/latency_sweep.py)
    const long long total = (long long)prm.n_strips * (prm.r_hi - prm.r_lo);
    long long grid = n_sm;
    if (total < grid * G) grid = (total + G - 1) / G;
    if (grid < 1) grid = 1;
    prm.chunk = (total + grid - 1) / grid;
    grid = (total + prm.chunk - 1) / prm.chunk;
    const int g = (int)grid;
    int rc;
    if (pd.hi && pd.nbk == 1 && !pd.ho) rc = launch_pass<true, 1, false>(prm, g, st, pi > 0);
    else if (pd.hi && pd.nbk == 0 && !pd.ho) rc = launch_pass<true, 0, false>(prm, g, st, pi > 0);
    else if (!pd.hi && pd.nbk == 2 && !pd.ho) rc = launch_pass<false, 2, false>(prm, g, st, pi > 0);
    else if (!pd.hi && pd.nbk == 1 && pd.ho) rc = launch_pass<false, 1, true>(prm, g, st, pi > 0);
    else if (!pd.hi && pd.nbk == 0 && pd.ho) rc = launch_pass<false, 0, true>(prm, g, st, pi > 0);
    else return fail(HT_E_UNSUPPORTED, "no kernel for pass (hi=%d nbk=%d ho=%d)", pd.hi, pd.nbk, pd.ho);
    if (rc) return rc;
    in_x = out_x;
    out_x = (out_x == xa) ? xb : xa;
  }
  return HT_OK;
}

}  // namespace tc
}  // namespace ht

#ifdef HT_PROF
extern "C" int ht_debug_prof(long long *host) {
  cudaMemcpyFromSymbol(host, ht::tc::g_prof, sizeof(long long) * 128);
  return 0;
}
#endif
#ifdef HT_TIMELINE
extern "C" int ht_debug_timeline(long long *host) {
  cudaMemcpyFromSymbol(host, ht::tc::g_tl, sizeof(long long) * 4 * 4 * 16384);
  cudaMemset(nullptr, 0, 0);
  static long long zeros[4 * 4 * 16384];
  cudaMemcpyToSymbol(ht::tc::g_tl, zeros, sizeof(zeros));
  return 0;
}
#endif
