// Training 3x3 convolution 32 -> 32 on tcgen05, version 2: scaled fp16 pairs
// and role-split warps.  Same contract as conv_tc.cu (the residual blocks'
// forward convs nn.py:46-60, 91-95 and their input gradients nn.py:62-77,
// 97-100, run as forward convs with transposed / flipped weights): NCHW fp32
// in and out, epilogue bias, ReLU mask, residual add, ReLU.
//
// Precision: every input row x is scaled by a power of two 2^sx (row max |x|
// -> [2^13, 2^14)) and split into two fp16 parts x0 + x1 (x1 = the fp16
// rounding of the remainder: 22 significant bits), the weights likewise with
// one per-layer scale 2^sw.  A row's products x0 w0 + x0 w1 + x1 w0 (three
// kind::f16 MMAs per tap and K-half, 18 per row) accumulate in fp32 in the
// row's own TMEM ring, and the drain multiplies each ring by 2^-(sx + sw)
// (exact) before summing the three rings of an output row.  Error ~2^-22
// of the row scale per product -- the SIMT fp32 class; the per-row scale keeps
// the tiny input gradients of the backward pass (1e-9 and below) in fp16's
// normal range.  conv_tc.cu's split bf16 needs six products for the same
// class (bf16 has 8 significant bits).
//
// Structure (one CTA per SM, strips of 128 pixel lanes with 126 output lanes,
// rows streamed top to bottom, MMA(x) for input row x adding into output rows
// x+1, x, x-1 of TMEM ring x mod 4 through the doubled-ky B window):
// * two MMA issuer warps (alternate rows): the 18 MMAs of row x once the
//   splitters have written it and the drainers have freed ring x mod 4 --
//   while one warp's issue blocks on the tensor pipe's shallow queue the
//   other waits for its next row;
// * TMA producer warps: input rows into a staging ring (3 slots; 2 when the
//   launch has a mask / residual input, whose rows a second producer stages
//   in a 2-slot ring of their own, two output rows ahead);
// * 4 splitter warps (thread = pixel lane, 32 channels): staged row -> row
//   max (warp reduce + 4-warp barrier) -> scaled fp16 pair planes in one of
//   the A buffers (3; 2 with an epilogue input).  They touch no global
//   memory, so the proxy fence that publishes the planes to the tensor core
//   waits for nothing else;
// * 8 drainer warps (thread = pixel lane x 16 channels): wait for the MMAs of
//   an output row's three input rows, unscale and sum the rings (one at a
//   time), release the ring, epilogue with the staged mask / residual,
//   coalesced NCHW stores deferred past the next row's loads.
// Splitting, MMAs and draining of different rows overlap: the tensor pipe
// works on MMA(x) while row x+1 is split and row x-2 is drained.  Launched
// as a programmatic dependent of the previous kernel (the prologue -- weight
// split, barriers, TMEM -- overlaps its tail; griddepcontrol.wait before the
// first read of its output).  PAIR (opt-in, ht_set_conv_pair): the same on
// CTA pairs with tcgen05.mma.cta_group::2 (measured slower, kept tested).
#include "common.cuh"
#include "tc_ptx.cuh"

#include <cuda_fp16.h>

namespace ht {
namespace tct2 {

using namespace ::ht::tc;

constexpr int C = 32;
constexpr int M = 128;
constexpr int S = M - 2;                  // output lanes per strip
constexpr int NSL = 5;                    // doubled ky sequence [2,1,0,2,1]
constexpr int NPART = 2;                  // fp16 parts
constexpr int PLANE = M * 16;             // 8 channels x 128 lanes (fp16)
constexpr int ROW = 4 * PLANE;            // 32 channels of a row, one part
// B tile (kx, K-half): WROWS rows x 2 K-chunks x 16 B.  One CTA holds all
// 160 rows of the doubled ky sequence; a CTA pair (cta_group::2, M = 256)
// splits every N = 96 window between its CTAs (rows [0, 48) of the window
// in CTA 0, [48, 96) in CTA 1, at the same address), so each holds 112.
template <bool PAIR>
struct WLay {
  static constexpr int WROWS = PAIR ? 112 : NSL * C;
  static constexpr int TILE = 2 * WROWS * 16;
  static constexpr int KSTRIDE = WROWS * 16;          // B K-chunk stride (LBO)
  static constexpr int W_BYTES = NPART * 6 * TILE;
};
constexpr int BOXW = M + 4;               // box: 132 px x 32 channels fp32, [ch][px]
constexpr int BOX = BOXW * C * 4;
constexpr int STG_SLOT = 2 * BOX;         // a strip row spans at most two images
constexpr int NRING1 = 4;                 // TMEM rings of 96 columns, one CTA per strip (five measured no faster)
constexpr int NRING2 = 5;                 // CTA pairs: one more row of slack for the cross-CTA ring release
// barriers (8 B each): acc_full[8], ready[8], ring_free[NRING], stg_full[<=3],
// stg_empty[<=3], epi_full[2], epi_empty[2].  acc_full / ready are indexed by
// row & 7 so that no waiter is ever two phases behind its barrier: the two
// issuer warps wait on alternate rows' ready barriers, and the splitters can
// run NAB rows past a slow issuer.
constexpr int NSEQ = 8;
constexpr int B_ACC = 0, B_RDY = 8, B_FREE = 16, B_STG = 21, B_STE = 24, B_EF = 27, B_EE = 29, NBARS = 32;
// Shared-memory layout.  Without an epilogue input: three A buffers and
// three staging slots (TMA three rows ahead); with one, its rows take two
// staging slots of their own and the others drop to two each (227 KB).
template <bool EPI, bool PAIR>
struct Lay2 {
  static constexpr int A_OFF = WLay<PAIR>::W_BYTES;
  static constexpr int NAB = EPI ? 2 : 3;     // A buffers
  static constexpr int NSTG = EPI ? 2 : 3;    // input-row staging slots
  static constexpr int NESTG = EPI ? 2 : 0;   // epilogue-input (mask / residual) row slots
  static constexpr int A_BYTES = NAB * NPART * ROW;
  static constexpr int STG_OFF = A_OFF + A_BYTES;   // (W_BYTES is a multiple of 1 KB)
  static constexpr int ESTG_OFF = STG_OFF + NSTG * STG_SLOT;
  static constexpr int BAR_OFF = ESTG_OFF + NESTG * STG_SLOT;
  static constexpr int MISC_OFF = BAR_OFF + NBARS * 8;   // tmem slot, pad, sx[8], red[2][8], wred[24]
  static constexpr int SMEM = MISC_OFF + 384;
  static_assert(STG_OFF % 1024 == 0 && ESTG_OFF % 1024 == 0 && BOX % 128 == 0,
                "TMA destinations must stay 128-B aligned");
  static_assert(SMEM <= 232448, "shared memory exceeded");
};
constexpr int NSPL = 128, NDRN = 256;
constexpr int NISS = 2;                         // MMA issuer warps (even / odd rows)
constexpr int NTHR = NSPL + NDRN + 32 * NISS + 64;   // + issuers + two TMA producer warps
constexpr int HC = C / 2;
constexpr int SCALE_TOP = 14;             // scaled max |x| in [2^(SCALE_TOP-1), 2^SCALE_TOP)
constexpr uint32_t IDESC = (1u << 4) | ((uint32_t)(96 >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
constexpr uint32_t IDESC2 = (1u << 4) | ((uint32_t)(96 >> 3) << 17) | ((uint32_t)((2 * M) >> 4) << 24);
__constant__ int c_ky2[NSL] = {2, 1, 0, 2, 1};

__device__ __forceinline__ float exp2i(int e) { return __int_as_float((127 + e) << 23); }
// scale exponent of a block whose max |x| is m (0 / NaN -> 0), clamped to +-60
__device__ __forceinline__ int scale_exp(float m) {
  if (!(m > 0.f)) return 0;
  const int e = ((__float_as_int(m) >> 23) & 0xff) - 127;
  return max(-60, min(60, SCALE_TOP - 1 - e));
}
// v = x0 + x1 with x0 = fp16(v), x1 = fp16(v - x0); pairs packed as half2
__device__ __forceinline__ void split2h(float a, float b, uint32_t &p0, uint32_t &p1) {
  const __half2 h = __floats2half2_rn(a, b);
  const float2 hf = __half22float2(h);
  const __half2 l = __floats2half2_rn(a - hf.x, b - hf.y);
  p0 = *reinterpret_cast<const uint32_t *>(&h);
  p1 = *reinterpret_cast<const uint32_t *>(&l);
}
// cta_group::2: M = 256 over the CTA pair (issued by CTA 0; A and B halves
// read from the same shared-memory offsets of both CTAs, D in both TMEMs)
__device__ __forceinline__ void mma_f16_pair(uint32_t d, uint64_t a, uint64_t b, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
      "l"(a), "l"(b), "r"(IDESC2), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void commit_pair(uint32_t bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(bar),
      "h"((uint16_t)3)
      : "memory");
}
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
// the same shared-memory offset in CTA `rank` of the cluster
__device__ __forceinline__ uint32_t map_cta(uint32_t addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
__device__ __forceinline__ void mbar_wait_cluster(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n"
      "WAITC_%=:\n\t"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P1, [%0], %1, 0x989680;\n\t"
      "@P1 bra DONEC_%=;\n\t"
      "bra WAITC_%=;\n"
      "DONEC_%=:\n\t}" ::"r"(bar),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void mma_f16(uint32_t d, uint64_t a, uint64_t b, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
      "l"(a), "l"(b), "r"(IDESC), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void tma_load_4d(uint32_t dst, const CUtensorMap *map, int c0, int c1, int c2, int c3,
                                            uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, "
      "%5}], [%6];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(bar)
      : "memory");
}
// three 16-column TMEM loads, one wait
__device__ __forceinline__ void tmem_ld16x3(uint32_t t0, uint32_t t1, uint32_t t2, uint32_t (&r)[3][16]) {
#define HT_LD16(T, R)                                                                                          \
  asm volatile(                                                                                                \
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];" \
      : "=r"(R[0]), "=r"(R[1]), "=r"(R[2]), "=r"(R[3]), "=r"(R[4]), "=r"(R[5]), "=r"(R[6]), "=r"(R[7]),       \
        "=r"(R[8]), "=r"(R[9]), "=r"(R[10]), "=r"(R[11]), "=r"(R[12]), "=r"(R[13]), "=r"(R[14]), "=r"(R[15])  \
      : "r"(T))
  HT_LD16(t0, r[0]);
  HT_LD16(t1, r[1]);
  HT_LD16(t2, r[2]);
#undef HT_LD16
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

#ifdef CT2_TL
// debug timeline of CTA 0 (lane 0 of the issuer, splitter warp 0, drainer
// warp 4): [role][row][event] = clock64
__device__ long long g_ctl2[3][1024][6];
#define TL2(role, n, k) do { if (blockIdx.x == 0 && lane == 0 && (n) < 1024) g_ctl2[role][n][k] = clock64(); } while (0)
#else
#define TL2(role, n, k) do {} while (0)
#endif

struct Conv2Params {
  CUtensorMap tm_x;   // x as (W, C, H, B) fp32, box 132 x 32 x 1 x 1
  CUtensorMap tm_e;   // the mask or residual, same geometry (EPI kernels)
  int is_mask;
  const float *w, *bias, *mask, *resid;
  float *out;
  // training-path extras (conv_tc2_32_ex): ReLU bits written by a forward
  // conv1 / read by the input gradient of conv2 instead of an fp32 mask, one
  // uint16 per (image, channel half, pixel) = bit i: channel half*16+i > 0;
  // accum: out += conv (red.global.add) -- the conv1 input gradient adds onto
  // the skip gradient in place instead of reading it as a residual
  uint16_t *bits_out;
  const uint16_t *bits_in;
  int accum;
  int B, H, W, VW, relu;
  int n_strips;
  long long chunk;    // strip-rows per CTA (strip-major; per CTA pair: strip-pair rows)
};

// the strip-major (strip, row) range [q0, q1) of a CTA, walked as segments
struct Seg {
  int s, R0, R1, A, Bn;
};
__device__ __forceinline__ long long next_seg(long long qq, long long q1, int H, Seg &g) {
  g.s = (int)(qq / H);
  const long long end = min(q1, (long long)(g.s + 1) * H);
  g.R0 = (int)(qq - (long long)g.s * H);
  g.R1 = (int)(end - (long long)g.s * H);
  g.A = max(g.R0 - 1, 0);
  g.Bn = min(g.R1 + 1, H);
  return end;
}

template <bool EPI, bool PAIR>
__global__ void __launch_bounds__(NTHR, 1) conv_tc2_kernel(const __grid_constant__ Conv2Params P) {
  using L = Lay2<EPI, PAIR>;
  using WL = WLay<PAIR>;
  constexpr int NAB = L::NAB, NSTG = L::NSTG, NESTG = EPI ? L::NESTG : 1;
  constexpr int A_BYTES = L::A_BYTES, STG_OFF = L::STG_OFF, ESTG_OFF = L::ESTG_OFF;
  constexpr int BAR_OFF = L::BAR_OFF, MISC_OFF = L::MISC_OFF, A_OFF = L::A_OFF;
  constexpr int TILE = WL::TILE;
  // PAIR: CTA `rank` of the pair owns strip 2 u + rank of strip pair u; CTA 0
  // issues the pair's MMAs, both CTAs' splitters / drainers arrive on CTA 0's
  // ready / ring_free barriers
  const uint32_t rank = PAIR ? cluster_rank() : 0u;
  constexpr int NRING = PAIR ? NRING2 : NRING1;
  extern __shared__ __align__(1024) uint8_t smem[];
  pdl_launch_dependents();
  const int tid = threadIdx.x, lane = tid & 31;
  const int warp = __shfl_sync(0xffffffffu, tid >> 5, 0);
  const uint32_t sbase = smem_u32(smem);
  auto bar = [&](int k) { return sbase + BAR_OFF + 8u * (uint32_t)k; };
  auto acc_full = [&](long long g) { return bar(B_ACC + (int)(g % NSEQ)); };
  auto ready = [&](long long g) { return bar(B_RDY + (int)(g % NSEQ)); };
  // parity of row g's phase on its acc_full / ready barrier
  auto seq_par = [](long long g) { return (uint32_t)(g / NSEQ) & 1u; };
  auto ring_free = [&](long long g) { return bar(B_FREE + (int)(g % NRING)); };
  auto stg_full = [&](long long g) { return bar(B_STG + (int)(g % NSTG)); };
  auto stg_empty = [&](long long g) { return bar(B_STE + (int)(g % NSTG)); };
  auto epi_full = [&](long long g) { return bar(B_EF + (int)(g % NESTG)); };
  auto epi_empty = [&](long long g) { return bar(B_EE + (int)(g % NESTG)); };
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(smem + MISC_OFF);
  int *sx_s = reinterpret_cast<int *>(smem + MISC_OFF + 8);        // [8] row scale by g & 7
  int *red = reinterpret_cast<int *>(smem + MISC_OFF + 48);        // [2][8] row-max partials
  int *wred = reinterpret_cast<int *>(smem + MISC_OFF + 112);      // [24] weight-max partials
  float *bias_s = reinterpret_cast<float *>(smem + MISC_OFF + 208); // [32] bias
  if (tid == 0) {
    for (int k = 0; k < NSEQ; ++k) {
      mbar_init(bar(B_ACC + k), 1);
      // PAIR: CTA 1's splitters / drainers arrive locally and one forwarder
      // warp passes each completed phase on to CTA 0 (a cluster-scope
      // release in every splitter / drainer warp cost ~1,300 cycles each)
      mbar_init(bar(B_RDY + k), NSPL / 32 + (PAIR && rank == 0 ? 1 : 0));
    }
    for (int k = 0; k < NRING; ++k) mbar_init(bar(B_FREE + k), NDRN / 32 + (PAIR && rank == 0 ? 1 : 0));
    for (int k = 0; k < NSTG; ++k) {
      mbar_init(bar(B_STG + k), 1);
      mbar_init(bar(B_STE + k), NSPL / 32);
    }
    for (int k = 0; k < L::NESTG; ++k) {
      mbar_init(bar(B_EF + k), 1);
      mbar_init(bar(B_EE + k), NDRN / 32);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  // ---- weights: per-layer scale, two fp16 parts in UMMA tiles [part][kx][kh]
  {
    float m = 0.f;
    for (int i = tid; i < C * C * 9; i += NTHR) m = fmaxf(m, fabsf(__ldg(P.w + i)));
    m = __int_as_float(__reduce_max_sync(0xffffffffu, __float_as_int(m)));
    if (lane == 0) wred[warp] = __float_as_int(m);
  }
  __syncthreads();
  int sw;
  {
    float m = 0.f;
    for (int k = 0; k < NTHR / 32; ++k) m = fmaxf(m, __int_as_float(wred[k]));
    sw = scale_exp(m);
  }
  const float wsc = exp2i(sw);
  for (int i = tid; i < 3 * 2 * 2 * NSL * C * 4; i += NTHR) {
    // one (e pair) of a B row: 2 channels -> 4 B per part
    const int ep = i & 3, co = (i >> 2) % C, s = (i >> 2) / C % NSL;
    const int kc = (i >> 2) / C / NSL % 2, kh = (i >> 2) / C / NSL / 2 % 2, kx = (i >> 2) / C / NSL / 4;
    const int ci = kh * 16 + kc * 8 + 2 * ep, ky = c_ky2[s];
    const int wrow = s * C + co - (PAIR ? 48 * (int)rank : 0);   // row of this CTA's tile
    if (wrow < 0 || wrow >= WL::WROWS) continue;
    const float wa = __ldg(P.w + ((co * C + ci) * 3 + ky) * 3 + kx) * wsc;
    const float wb = __ldg(P.w + ((co * C + ci + 1) * 3 + ky) * 3 + kx) * wsc;
    uint32_t p0, p1;
    split2h(wa, wb, p0, p1);
    const int off = (kx * 2 + kh) * TILE + kc * WL::KSTRIDE + wrow * 16 + ep * 4;
    *reinterpret_cast<uint32_t *>(smem + off) = p0;
    *reinterpret_cast<uint32_t *>(smem + 6 * TILE + off) = p1;
  }
  for (int i = tid; i < A_BYTES / 16; i += NTHR)
    reinterpret_cast<uint4 *>(smem + A_OFF)[i] = make_uint4(0, 0, 0, 0);
  if (tid < C) bias_s[tid] = P.bias ? __ldg(P.bias + tid) : 0.f;
  fence_proxy_async();
  if (warp == 0) {
    if constexpr (PAIR) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_slot)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_slot)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
  }
  tc_fence_before();
  if constexpr (PAIR) {
    // both CTAs' barriers initialised and weights written before any remote
    // arrive or pair MMA
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  } else {
    __syncthreads();
  }
  tc_fence_after();
  const uint32_t tmem = __shfl_sync(0xffffffffu, *tmem_slot, 0);
  // launched as a programmatic dependent: the prologue above (weights,
  // barriers, TMEM) overlapped the previous kernel; its outputs (our input,
  // mask / residual) are complete past this point
  pdl_wait();
  const size_t plane = (size_t)P.H * P.W;
  // PAIR: the q space is (strip pair, row), one range per CTA pair
  const long long n_units = PAIR ? (P.n_strips + 1) / 2 : P.n_strips;
  const long long q0 = (long long)(PAIR ? blockIdx.x / 2 : blockIdx.x) * P.chunk;
  const long long q1 = min(q0 + P.chunk, n_units * P.H);
  // this CTA's strip of segment unit u; a pair's second strip past the last
  // one stays in the loops (zero inputs, no stores) with its TMA boxes
  // pointed inside the tensor
  auto strip_of = [&](int u) { return PAIR ? 2 * u + (int)rank : u; };
  auto box_image = [&](int v0) { return min(max(v0, 0) / (P.W + 1), P.B - 1); };
  const int WP = P.W + 1;

  if (warp == (NSPL + NDRN) / 32 + NISS + 1) {
    // ================= producer: epilogue-input rows (mask / residual) ======
    if (lane == 0 && EPI) {
      long long ge = 0;
      for (long long qq = q0; qq < q1;) {
        Seg sg;
        qq = next_seg(qq, q1, P.H, sg);
        sg.s = strip_of(sg.s);
        const bool empty = sg.s >= P.n_strips;   // (PAIR: a pair's missing second strip)
        const int v0 = sg.s * S - 1, b0 = empty ? 0 : box_image(v0);
        const int nbox = (!empty && b0 + 1 < P.B && v0 + M - 1 >= (b0 + 1) * WP) ? 2 : 1;
        const int c0a = empty ? 0 : (v0 - b0 * WP) & ~3, c0b = (v0 - (b0 + 1) * WP) & ~3;
        for (int d = sg.R0; d < sg.R1; ++d, ++ge) {
          if (ge >= NESTG) mbar_wait(epi_empty(ge), (uint32_t)((ge / NESTG) - 1) & 1u);
          const uint32_t fb = epi_full(ge), dst = sbase + ESTG_OFF + (uint32_t)(ge % NESTG) * STG_SLOT;
          mbar_expect_tx(fb, nbox * BOX);
          tma_load_4d(dst, &P.tm_e, c0a, 0, d, b0, fb);
          if (nbox == 2) tma_load_4d(dst + BOX, &P.tm_e, c0b, 0, d, b0 + 1, fb);
        }
      }
    }
  } else if (warp == (NSPL + NDRN) / 32 + NISS) {
    // ================= producer: input rows by TMA, NSTG rows ahead ========
    if (lane == 0) {
      long long tg = 0;
      for (long long qq = q0; qq < q1;) {
        Seg sg;
        qq = next_seg(qq, q1, P.H, sg);
        sg.s = strip_of(sg.s);
        const bool empty = sg.s >= P.n_strips;   // (PAIR: a pair's missing second strip)
        const int v0 = sg.s * S - 1, b0 = empty ? 0 : box_image(v0);
        const int nbox = (!empty && b0 + 1 < P.B && v0 + M - 1 >= (b0 + 1) * WP) ? 2 : 1;
        const int c0a = empty ? 0 : (v0 - b0 * WP) & ~3, c0b = (v0 - (b0 + 1) * WP) & ~3;
        for (int x = sg.A; x < sg.Bn; ++x, ++tg) {
          // slot tg % NSTG was read by the splitters of row tg - NSTG
          if (tg >= NSTG) mbar_wait(stg_empty(tg), (uint32_t)((tg / NSTG) - 1) & 1u);
          const uint32_t fb = stg_full(tg), dst = sbase + STG_OFF + (uint32_t)(tg % NSTG) * STG_SLOT;
          mbar_expect_tx(fb, nbox * BOX);
          tma_load_4d(dst, &P.tm_x, c0a, 0, x, b0, fb);
          if (nbox == 2) tma_load_4d(dst + BOX, &P.tm_x, c0b, 0, x, b0 + 1, fb);
        }
      }
    }
  } else if (warp >= (NSPL + NDRN) / 32) {
    if (PAIR && rank != 0) {
      // CTA 1: the pair's MMAs are issued by CTA 0; warp iss forwards this
      // CTA's ready (iss 0) / ring_free (iss 1) phases to CTA 0, row by row
      const int iss = warp - (NSPL + NDRN) / 32;
      long long n_rows = 0;
      for (long long qq = q0; qq < q1;) {
        Seg sg;
        qq = next_seg(qq, q1, P.H, sg);
        n_rows += sg.Bn - sg.A;
      }
      if (lane == 0) {
        for (long long g = 0; g < n_rows; ++g) {
          if (iss == 0) {
            mbar_wait(ready(g), seq_par(g));
            mbar_arrive_cluster(map_cta(ready(g), 0));
          } else {
            mbar_wait(ring_free(g), (uint32_t)(g / NRING) & 1u);
            tc_fence_after();
            tc_fence_before();
            mbar_arrive_cluster(map_cta(ring_free(g), 0));
          }
        }
      }
      __syncwarp();
    } else {
    // ================= issuers: 18 MMAs per row, rows alternating between two
    // warps: while one warp's issue blocks on the tensor pipe's queue, the
    // other waits for its next row's inputs and ring, so the pipe is fed with
    // no gap between batches
    const int iss = warp - (NSPL + NDRN) / 32;
    const uint64_t adesc0 = umma_desc(sbase, PLANE, 128);
    const uint64_t bdesc0 = (adesc0 & ~(0x3FFFull << 16)) | ((uint64_t)(WL::KSTRIDE >> 4) << 16);
    long long g = 0;
    for (long long qq = q0; qq < q1;) {
      Seg sg;
      qq = next_seg(qq, q1, P.H, sg);
        sg.s = strip_of(sg.s);
      int xm3 = sg.A % 3;
      for (int x = sg.A; x < sg.Bn; ++x, ++g, xm3 = xm3 == 2 ? 0 : xm3 + 1) {
        if ((int)(g % NISS) != iss) continue;
        TL2(0, g, 0);
        if (lane == 0) {
          if constexpr (PAIR) mbar_wait_cluster(ready(g), seq_par(g));
          else mbar_wait(ready(g), seq_par(g));
        }
        __syncwarp();
        TL2(0, g, 1);
        TL2(0, g, 2);
        if (g >= NRING) {
          if (lane == 0) {
            if constexpr (PAIR) mbar_wait_cluster(ring_free(g), (uint32_t)((g / NRING) - 1) & 1u);
            else mbar_wait(ring_free(g), (uint32_t)((g / NRING) - 1) & 1u);
          }
          __syncwarp();
        }
        TL2(0, g, 3);
        tc_fence_after();
        if (lane == 0) {
          const int o = xm3 == 0 ? 1 : (xm3 == 1 ? 0 : 2);   // B window for rows (x+1, x, x-1)
          const uint32_t d = tmem + (uint32_t)((g % NRING) * 3 * C);
          const uint64_t a0 = adesc0 + ((A_OFF + (uint32_t)(g % NAB) * NPART * ROW) >> 4);
          const uint64_t b0 = bdesc0 + ((o * C * 16) >> 4);
          constexpr uint64_t AP = ROW >> 4, BP = (6 * TILE) >> 4, TB = TILE >> 4, KH = (2 * PLANE) >> 4;
          // corrections x1 w0 and x0 w1 first (the first one overwrites the
          // ring), the main products x0 w0 last
          uint32_t acc = 0;
#pragma unroll
          for (int kx = 0; kx < 3; ++kx)
#pragma unroll
            for (int kh = 0; kh < 2; ++kh) {
              const uint64_t a = a0 + kh * KH + kx - 1, b = b0 + (kx * 2 + kh) * TB;
              if constexpr (PAIR) {
                mma_f16_pair(d, a + AP, b, acc);
                mma_f16_pair(d, a, b + BP, 1);
              } else {
                mma_f16(d, a + AP, b, acc);
                mma_f16(d, a, b + BP, 1);
              }
              acc = 1;
            }
#pragma unroll
          for (int kx = 0; kx < 3; ++kx)
#pragma unroll
            for (int kh = 0; kh < 2; ++kh) {
              if constexpr (PAIR) mma_f16_pair(d, a0 + kh * KH + kx - 1, b0 + (kx * 2 + kh) * TB, 1);
              else mma_f16(d, a0 + kh * KH + kx - 1, b0 + (kx * 2 + kh) * TB, 1);
            }
          if constexpr (PAIR) commit_pair(acc_full(g));
          else tc_commit(acc_full(g));
        }
        __syncwarp();
        TL2(0, g, 4);
      }
    }
    }
  } else if (warp < NSPL / 32) {
    // ================= splitters: staged row -> scaled fp16 pair planes =====
    const int l = tid;   // pixel lane, all 32 channels
    long long g = 0;
    for (long long qq = q0; qq < q1;) {
      Seg sg;
      qq = next_seg(qq, q1, P.H, sg);
        sg.s = strip_of(sg.s);
      const int v0 = sg.s * S - 1, v = v0 + l;
      const int b = v >= 0 ? v / WP : 0, col = v >= 0 ? v % WP : 0;
      const bool in_img = v >= 0 && v < P.VW && col < P.W;
      const int b0 = max(v0, 0) / WP;
      const int kbox = in_img ? b - b0 : -1;
      const int kcol = v0 - (b0 + max(kbox, 0)) * WP;
      const int koff = l + (kcol & 3);
      for (int x = sg.A; x < sg.Bn; ++x, ++g) {
        if (warp == 0) TL2(1, g, 0);
        if (lane == 0) mbar_wait(stg_full(g), (uint32_t)(g / NSTG) & 1u);
        __syncwarp();
        if (warp == 0) TL2(1, g, 1);
        float xin[C];
        const float *src = reinterpret_cast<const float *>(smem + STG_OFF + (uint32_t)(g % NSTG) * STG_SLOT +
                                                           max(kbox, 0) * BOX) + koff;
        float m = 0.f;
#pragma unroll
        for (int i = 0; i < C; ++i) {
          xin[i] = kbox >= 0 ? src[i * BOXW] : 0.f;
          m = fmaxf(m, fabsf(xin[i]));
        }
        m = __int_as_float(__reduce_max_sync(0xffffffffu, __float_as_int(m)));
        // this warp's reads of the staging slot are done
        if (lane == 0) {
          mbar_arrive(stg_empty(g));
          red[(g & 1) * 4 + warp] = __float_as_int(m);
        }
        named_bar(1, NSPL);
        {
          const int4 ra = *reinterpret_cast<const int4 *>(red + (g & 1) * 4);
          m = __int_as_float(max(max(ra.x, ra.y), max(ra.z, ra.w)));
        }
        const int sx = scale_exp(m);
        const float sc = exp2i(sx);
        if (warp == 0) TL2(1, g, 2);
        // A buffer g % NAB was last read by MMA(g - NAB)
        if (g >= NAB) {
          if (lane == 0) mbar_wait(acc_full(g - NAB), seq_par(g - NAB));
          __syncwarp();
        }
        if (warp == 0) TL2(1, g, 3);
        const uint32_t dst = sbase + A_OFF + (uint32_t)(g % NAB) * NPART * ROW + l * 16;
#pragma unroll
        for (int kc = 0; kc < 4; ++kc) {
          uint32_t h[4], lo[4];
#pragma unroll
          for (int k2 = 0; k2 < 4; ++k2)
            split2h(xin[8 * kc + 2 * k2] * sc, xin[8 * kc + 2 * k2 + 1] * sc, h[k2], lo[k2]);
          st_shared_v4(dst + kc * PLANE, h[0], h[1], h[2], h[3]);
          st_shared_v4(dst + ROW + kc * PLANE, lo[0], lo[1], lo[2], lo[3]);
        }
        if (tid == 0) sx_s[g & 7] = sx;
        fence_proxy_async();
        __syncwarp();
        if (lane == 0) mbar_arrive(ready(g));
        if (warp == 0) TL2(1, g, 4);
      }
    }
  } else {
    // ================= drainers: rings -> output rows =======================
    const int wd = warp - NSPL / 32;
    const int wq = warp & 3, half = wd >> 2;
    const uint32_t tlane = tmem + ((uint32_t)(wq * 32) << 16);
    const int l = wq * 32 + lane, c0 = half * HC;
    // the one epilogue input of a launch (the training path passes a ReLU
    // mask or a residual, never both: conv_tc2_32 requires that) arrives by
    // TMA, two output rows ahead, in the epilogue staging ring
    float bv[HC];
#pragma unroll
    for (int i = 0; i < HC; ++i) bv[i] = P.bias ? __ldg(P.bias + c0 + i) : 0.f;
    constexpr bool has_epi = EPI;
    const bool is_mask = P.is_mask != 0;
    long long gbase = 0, ge = 0;
    for (long long qq = q0; qq < q1;) {
      Seg sg;
      qq = next_seg(qq, q1, P.H, sg);
        sg.s = strip_of(sg.s);
      const int v = sg.s * S - 1 + l;
      const int b = v >= 0 ? v / WP : 0, col = v >= 0 ? v % WP : 0;
      const bool in_img = v >= 0 && v < P.VW && col < P.W;
      const bool lane_valid = l >= 1 && l < 1 + S && in_img;
      const size_t obase = ((size_t)b * C + c0) * plane + col;
      // this lane's column in the staged epilogue boxes (as the splitters')
      const int eb0 = max(sg.s * S - 1, 0) / WP;
      const int ekbox = in_img ? b - eb0 : -1;
      const int ekcol = (sg.s * S - 1) - (eb0 + max(ekbox, 0)) * WP;
      const int ekoff = max(ekbox, 0) * (BOX / 4) + l + (ekcol & 3) + c0 * BOXW;
      auto gx = [&](int x) { return gbase + (x - sg.A); };
      auto release = [&](int x) {   // ring of input row x: every output row it feeds is drained
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(ring_free(gx(x)));
      };
      // output row awaiting its stores: issued after the next row's epilogue
      // loads, so those never queue behind them
      float y[HC];
      size_t pend = ~(size_t)0;
      auto flush = [&]() {
        if (pend != ~(size_t)0) {
          float *dst = P.out + pend;
          if (!EPI && P.accum) {
#pragma unroll
            for (int i = 0; i < HC; ++i) red_add_f32(dst + (size_t)i * plane, y[i]);
          } else {
#pragma unroll
            for (int i = 0; i < HC; ++i) dst[(size_t)i * plane] = y[i];
          }
          pend = ~(size_t)0;
        }
      };
      // ReLU bits of (image b, this channel half): one uint16 per pixel
      const size_t bbase = ((size_t)b * 2 + half) * plane + col;
      auto drain_row = [&](int d) {
        float e[HC];
        uint32_t mb = 0xffffu;
        // (issued before the completion wait: its latency hides behind it)
        if (!EPI && P.bits_in && lane_valid) mb = __ldg(P.bits_in + bbase + (size_t)d * P.W);
        if (has_epi) {
          // this row's mask / residual from its staging slot; the slot is
          // released at once (the arrive orders the reads before it)
          if (lane == 0) mbar_wait(epi_full(ge), (uint32_t)(ge / NESTG) & 1u);
          __syncwarp();
          const float *src = reinterpret_cast<const float *>(smem + ESTG_OFF + (uint32_t)(ge % NESTG) * STG_SLOT) + ekoff;
#pragma unroll
          for (int i = 0; i < HC; ++i) e[i] = src[i * BOXW];
          __syncwarp();
          if (lane == 0) mbar_arrive(epi_empty(ge));
        }
        ++ge;
        flush();
        // MMAs of input rows d-1, d, d+1 done (two issuer warps: no order
        // between their commits, so each is waited for)
        if (warp == 4) TL2(2, gx(d), 0);
        if (lane == 0) {
          for (int xr = max(d - 1, sg.A); xr <= min(d + 1, sg.Bn - 1); ++xr) {
            const long long gt = gx(xr);
            mbar_wait(acc_full(gt), seq_par(gt));
          }
        }
        __syncwarp();
        if (warp == 4) TL2(2, gx(d), 1);
        tc_fence_after();
        const int slot = d % 3;
        int sxr[3];
#pragma unroll
        for (int k = 0; k < 3; ++k) {
          const int xr = min(max(d - 1 + k, sg.A), sg.Bn - 1);
          sxr[k] = sx_s[gx(xr) & 7];
        }
#pragma unroll
        for (int i = 0; i < HC; ++i) y[i] = bv[i];
        // the three rings one at a time (16 registers), each unscaled exactly;
        // a ring of a row outside the segment holds stale values: skipped
#pragma unroll
        for (int k = 0; k < 3; ++k) {
          const int xr = d - 1 + k;
          if (xr < sg.A || xr >= sg.Bn) continue;
          float r[HC];
          tmem_ld16(tlane + (uint32_t)((gx(xr) % NRING) * 3 * C + slot * C + c0), r);
          const float f = exp2i(-(sxr[k] + sw));
#pragma unroll
          for (int i = 0; i < HC; ++i) y[i] = fmaf(r[i], f, y[i]);
        }
        if (warp == 4) TL2(2, gx(d), 5);
        // the ring of input row d-1 fed rows d-2, d-1, d: free now
        if (d - 1 >= sg.A) release(d - 1);
        if (warp == 4) TL2(2, gx(d), 2);
#pragma unroll
        for (int i = 0; i < HC; ++i) {
          if (has_epi) {
            if (is_mask) y[i] = e[i] > 0.f ? y[i] : 0.f;
            else y[i] += e[i];
          }
          if (!EPI) y[i] = (mb >> i) & 1u ? y[i] : 0.f;
          if (P.relu) y[i] = fmaxf(y[i], 0.f);
        }
        if (!EPI && P.bits_out && lane_valid) {
          uint32_t bits = 0;
#pragma unroll
          for (int i = 0; i < HC; ++i) bits |= (y[i] > 0.f ? 1u : 0u) << i;
          P.bits_out[bbase + (size_t)d * P.W] = (uint16_t)bits;
        }
        if (lane_valid) pend = obase + (size_t)d * P.W;
        if (warp == 4) TL2(2, gx(d), 3);
        if (warp == 4) TL2(2, gx(d), 4);
      };
      for (int d = sg.R0; d < sg.R1; ++d) drain_row(d);
      flush();
      // rings of the rows below the last output row
      for (int x = max(sg.A, sg.R1 - 1); x < sg.Bn; ++x) release(x);
      gbase += sg.Bn - sg.A;
    }
  }
  tc_fence_before();
  if constexpr (PAIR) {
    // the pair's last MMAs wrote both TMEMs: no CTA frees its TMEM (or exits,
    // releasing shared memory the peer's MMAs read) before both are done
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  } else {
    __syncthreads();
  }
  if (warp == 0) {
    tc_fence_after();
    if constexpr (PAIR) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem));
    else asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

}  // namespace tct2
#ifdef CT2_TL
extern "C" int ht_debug_conv2_timeline(long long *host) {
  return (int)cudaMemcpyFromSymbol(host, tct2::g_ctl2, sizeof(long long) * 3 * 1024 * 6);
}
#endif

// true when the shape suits the TMA-staged kernel (16-B row strides, a strip
// row spans at most two images)
bool conv_tc2_eligible(int W) { return W % 4 == 0 && W + 1 >= tct2::M; }

// 0: one CTA per strip (cta_group::1), 1: CTA pairs (cta_group::2, M = 256)
int g_conv_tc2_pair = 0;

int conv_tc2_32_ex(const float *x, int B, int H, int W, const float *w, const float *bias, const float *mask,
                   const float *resid, float *out, int relu, uint16_t *bits_out, const uint16_t *bits_in,
                   int accum, cudaStream_t st);
int conv_tc2_32(const float *x, int B, int H, int W, const float *w, const float *bias, const float *mask,
                const float *resid, float *out, int relu, cudaStream_t st) {
  return conv_tc2_32_ex(x, B, H, W, w, bias, mask, resid, out, relu, nullptr, nullptr, 0, st);
}

int conv_tc2_32_ex(const float *x, int B, int H, int W, const float *w, const float *bias, const float *mask,
                   const float *resid, float *out, int relu, uint16_t *bits_out, const uint16_t *bits_in,
                   int accum, cudaStream_t st) {
  using namespace tct2;
  HT_REQUIRE(conv_tc2_eligible(W), "conv_tc2: unsupported width %d", W);
  HT_REQUIRE(!(mask && resid), "conv_tc2: a ReLU mask and a residual in one launch");
  HT_REQUIRE(!((mask || resid) && (bits_in || bits_out || accum)),
             "conv_tc2: ReLU bits / accumulation only without an fp32 epilogue input");
  const bool pair = g_conv_tc2_pair != 0;
  if (int rc = ensure_smem_attr((const void *)conv_tc2_kernel<false, false>, Lay2<false, false>::SMEM)) return rc;
  if (int rc = ensure_smem_attr((const void *)conv_tc2_kernel<true, false>, Lay2<true, false>::SMEM)) return rc;
  if (int rc = ensure_smem_attr((const void *)conv_tc2_kernel<false, true>, Lay2<false, true>::SMEM)) return rc;
  if (int rc = ensure_smem_attr((const void *)conv_tc2_kernel<true, true>, Lay2<true, true>::SMEM)) return rc;
  int dev = 0, n_sm = 148;
  HT_CUDA(cudaGetDevice(&dev));
  HT_CUDA(cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev));
  Conv2Params p{};
  p.w = w; p.bias = bias; p.mask = mask; p.resid = resid; p.out = out;
  p.bits_out = bits_out; p.bits_in = bits_in; p.accum = accum;
  p.B = B; p.H = H; p.W = W; p.VW = B * (W + 1); p.relu = relu;
  p.n_strips = (p.VW + S - 1) / S;
  // work units: (strip, row), or (strip pair, row) for CTA pairs
  const long long units = pair ? (p.n_strips + 1) / 2 : p.n_strips;
  const long long total = units * H;
  long long grid = pair ? n_sm / 2 : n_sm;
  if (total < grid * 8) grid = (total + 7) / 8;
  if (grid < 1) grid = 1;
  p.chunk = (total + grid - 1) / grid;
  grid = (total + p.chunk - 1) / p.chunk;
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
  const float *epi = mask ? mask : resid;
  p.is_mask = mask != nullptr;
  if (epi) {
    const CUresult re = enc(&p.tm_e, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, const_cast<float *>(epi), dims, strides, box,
                            estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    HT_REQUIRE(re == CUDA_SUCCESS, "cuTensorMapEncodeTiled failed (%d)", (int)re);
  }
  if (!pair) {
    if (epi) HT_CUDA(launch_pdl(conv_tc2_kernel<true, false>, (unsigned)grid, NTHR, Lay2<true, false>::SMEM, st, p));
    else HT_CUDA(launch_pdl(conv_tc2_kernel<false, false>, (unsigned)grid, NTHR, Lay2<false, false>::SMEM, st, p));
  } else {
    cudaLaunchConfig_t cfg{};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.gridDim = dim3((unsigned)(2 * grid), 1, 1);
    cfg.blockDim = dim3(NTHR, 1, 1);
    cfg.dynamicSmemBytes = epi ? Lay2<true, true>::SMEM : Lay2<false, true>::SMEM;
    cfg.stream = st;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (epi) HT_CUDA(cudaLaunchKernelEx(&cfg, conv_tc2_kernel<true, true>, p));
    else HT_CUDA(cudaLaunchKernelEx(&cfg, conv_tc2_kernel<false, true>, p));
  }
  count_launch();
  HT_CHECK_LAUNCH();
  return HT_OK;
}

}  // namespace ht
