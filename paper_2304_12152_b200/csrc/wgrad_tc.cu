// Weight (and bias) gradient of the 32 -> 32 training convs on tcgen05.
//
// Replaces conv3x3_wgrad32_kernel (conv_simt.cu) on the training path: the
// residual blocks' dW = sum over pixels of dout (x) im2col(x) (nn.py:62-77,
// 97-100 of the reference compute it with numpy einsums in float64).
//
// As a GEMM with the pixels as the reduction (K) dimension:
//   D[(ky', ci)][(s, kx, co)] += x[ci][y - 1 + ky'][p] * dout[co][y + s][p - kx + 1]
// for a pair of dout rows y, y+1 (s = 0, 1) and the four x rows y-1 .. y+2
// (ky' = 0..3): M = 4 x 32 = 128, N = 2 x 3 x 32 = 192, K = 16 pixels per MMA.
// Block (ky', s) holds tap ky = ky' - s; the two blocks with ky' - s outside
// 0..2 are wasted (6 of 8 useful), the price of a full 128-row MMA.  The kx
// shift cannot be a descriptor offset (2 B along K), so the dout rows are
// written three times, shifted.  The sums stay in TMEM for all of a CTA's
// tiles and are added into the fp64 dW once at the end.
//
// Precision: split bf16 operands (x = x0 + x1 [+ x2]); NP = 2 keeps the
// three products with i + j <= 1 (~2^-16 per product), NP = 3 the six with
// i + j <= 2 (fp32 level).  dW feeds Adam directly (no chain of layers for
// errors to grow along); the tests hold both against fp64.
//
// Tiles: one dout row pair x WT = 32 pixels of one image, interleaved over
// the CTAs (all SMs sweep the same image rows together: whole DRAM pages,
// halo rows from L2).  Warp roles:
// * a producer warp streams each tile's raw fp32 boxes with TMA (x: 4 rows x
//   32 channels x 32 px, 128-B swizzled; dout: 2 rows x 32 channels x 44 px,
//   176-B rows) into an NR-slot ring -- out-of-image pixels arrive
//   as zeros, no load instructions or bounds checks in the converters;
// * 16 converter warps split a raw slot into bf16 parts: 8 warps write the
//   x rows straight into the MMA's A operand in TMEM (TMEM lane quarter = x
//   row, lane = channel, bf16 pairs of 16 pixels per warp), 8 warps the
//   shifted dout copies as UMMA core matrices in shared memory (two
//   buffers); keeping A out of shared memory cuts the operand traffic of a
//   pipe the converters and the MMAs share;
// * one warp issues the MMAs in tile order;
// * the tensor core adds into its fp32 accumulator with an error that grows
//   with the chain length (1.2e-5 with one chain per CTA over 8 x 256^2), so
//   D is restarted every F tiles and four flusher warps add it into a second
//   TMEM accumulator with fp32 (RN) adds: the error no longer grows with the
//   batch.
#include "common.cuh"
#include "tc_ptx.cuh"

#include <cuda.h>
#include <cuda_bf16.h>
#include <cudaTypedefs.h>

namespace ht {
namespace wgt {

using namespace ::ht::tc;

constexpr int C = 32;
#ifndef WG_F2
#define WG_F2 32   // tiles per two-part chain: 16 -> 32 measured 136.4 -> 131.7 us per launch, tests unchanged
#endif
constexpr int TY = 2;                 // dout rows per tile (one row pair)
constexpr int WT = 32;                // pixels per tile row (WT / 16 K-steps)
constexpr int XR = TY + 2;            // x rows per tile
constexpr int CGB = (WT / 8) * 128;   // one 8-channel group of a row: WT/8 core matrices (8 ch x 8 px)
constexpr int ROWB = 4 * CGB;         // 32 channels of a row, one part
constexpr int NCOL = 2 * 3 * C;       // 192 accumulator columns (s, kx, co)
constexpr int NCONV = 512;            // converter threads
constexpr int D_UNITS = TY * C * (WT / 8);   // (dout row, channel, 8-pixel chunk)
static_assert(XR * C == 128 && D_UNITS == NCONV - 256, "x rows on warps 0-3 / 12-15, dout units on 4-11");
// dout box: pixels x0-4 .. x0+39 (the innermost box start must be 16-B
// aligned; 176-B rows keep 8 consecutive channels on distinct bank groups)
constexpr int DBOX = 44;
constexpr int RAW_X = XR * C * WT * 4;          // 16 KB, 128-B swizzled rows (y, c)
constexpr int RAW_D = TY * C * DBOX * 4;        // 11 KB
constexpr int RAW_SLOT = (RAW_X + RAW_D + 1023) / 1024 * 1024;
constexpr uint32_t IDESC =
    (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(NCOL >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
// TMEM: chain accumulator D (192 columns), the x operand A (NB buffers x NP
// parts x 16 columns: 32 pixels of bf16 pairs per lane), running sum D2
constexpr int D_COL = 0, A_COL = 192, D2_COL = 288;

template <int NP>
struct Lay {
  static constexpr int NPROD = NP == 2 ? 3 : 6;
  static constexpr int F = NP == 2 ? WG_F2 : 8;      // tiles per accumulation chain (192 MMAs with two parts, 96 with three)
  static constexpr int NR = 4;                       // raw ring slots
  // operand buffers: converters fill tile t+NB-1 while the MMAs of tile t run
  // (three for two parts: the converters then never wait on the MMAs' commit
  // round trip; the x operands of NB buffers x NP parts fit TMEM columns
  // 192..287 either way)
  static constexpr int NB = NP == 2 ? 3 : 2;
  static_assert(A_COL + NB * NP * 16 <= D2_COL, "TMEM operand buffers overlap D2");
  static constexpr int D_ROW = 3 * ROWB;   // three kx-shifted copies of a dout row
  static constexpr int D_PART = TY * D_ROW;
  static constexpr int BUF = (NP * D_PART + 1023) / 1024 * 1024;   // dout operand (B) only
  static constexpr int A_BUF_COLS = NP * 16;
  static constexpr int RAW_OFF = NB * BUF;
  // raw_full[NR], raw_empty[NR], op_full[NB], op_free[NB], d_full, d_empty
  static constexpr int BAR_OFF = RAW_OFF + NR * RAW_SLOT;
  static constexpr int NBARS = 2 * NR + 2 * NB + 2;
  static constexpr int DB_OFF = BAR_OFF + NBARS * 8;
  static constexpr int TMEMP_OFF = DB_OFF + C * 4;
  static constexpr int SMEM = TMEMP_OFF + 16 + 1024;   // + alignment slack
  static constexpr int MMA_WARP = NCONV / 32, TMA_WARP = MMA_WARP + 1, FLUSH_WARP0 = MMA_WARP + 2;
  static constexpr int NTHR = NCONV + 64 + 128;
};

// (a, b) -> NP packed bf16x2 words, a in the low half: part p of both values
// (x = x0 + x1 [+ x2], the remainders exact in fp32); packed conversions
// (one F2FP per pair and part) keep the converters off the conversion pipe
template <int NP>
__device__ __forceinline__ void split_pair(float a, float b, uint32_t (&w)[NP]) {
  float ra = a, rb = b;
#pragma unroll
  for (int p = 0; p < NP; ++p) {
    const __nv_bfloat162 h = __floats2bfloat162_rn(ra, rb);
    w[p] = *reinterpret_cast<const uint32_t *>(&h);
    if (p + 1 < NP) {
      ra -= __uint_as_float(w[p] << 16);
      rb -= __uint_as_float(w[p] & 0xffff0000u);
    }
  }
}
// bf16 pair (hi half of lo_word, lo half of hi_word): the odd-aligned pair
__device__ __forceinline__ uint32_t mid_pair(uint32_t lo_word, uint32_t hi_word) {
  return __byte_perm(lo_word, hi_word, 0x5432);
}
// 8 consecutive values -> one 16-B core-matrix row per part
template <int NP>
__device__ __forceinline__ void store8(uint32_t dst, uint32_t part_stride, const float (&v)[8]) {
  uint32_t w[4][NP];
#pragma unroll
  for (int k = 0; k < 4; ++k) split_pair<NP>(v[2 * k], v[2 * k + 1], w[k]);
#pragma unroll
  for (int p = 0; p < NP; ++p) st_shared_v4(dst + p * part_stride, w[0][p], w[1][p], w[2][p], w[3][p]);
}

// D (TMEM) += A (TMEM, 128 lanes x 16 bf16) * B (shared-memory descriptor)^T
__device__ __forceinline__ void mma_bf16_ta(uint32_t d, uint32_t a_tmem, uint64_t b, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
      "r"(a_tmem), "l"(b), "r"(IDESC), "r"(acc)
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

#ifdef WG_TL
// debug timeline of CTA 0: role 0 converters (warp 0), 8 MMA, 9 flushers
__device__ long long g_wtl[10][1024][4];
#define WTL(role, i, a, b, c) do { if (blockIdx.x == 0 && lane == 0 && (i) < 1024) { \
  g_wtl[role][i][0] = (a); g_wtl[role][i][1] = (b); g_wtl[role][i][2] = (c); g_wtl[role][i][3] = clock64(); } } while (0)
#else
#define WTL(role, i, a, b, c) do {} while (0)
#endif

struct WgParams {
  // (W, C, H, B) fp32 views of x and dout: x box 32 x 32 x 4 (128-B swizzle),
  // dout box 44 x 32 x 2
  CUtensorMap tm_x, tm_d;
  int B, H, W, tiles_y, tiles_x;
  long long n_tiles;
  double *dw, *db;
};

template <int NP>
__global__ void __launch_bounds__(Lay<NP>::NTHR, 1) wgrad_tc_kernel(const __grid_constant__ WgParams P) {
  using L = Lay<NP>;
  extern __shared__ uint8_t smem_raw[];
  pdl_launch_dependents();
  const int tid = threadIdx.x, lane = tid & 31;
  const int warp = __shfl_sync(0xffffffffu, tid >> 5, 0);
  // 1024-B alignment for the swizzled TMA boxes
  const uint32_t sraw = smem_u32(smem_raw);
  const uint32_t sbase = (sraw + 1023u) & ~1023u;
  uint8_t *smem = smem_raw + (sbase - sraw);
  const uint32_t raw_full0 = sbase + L::BAR_OFF, raw_empty0 = raw_full0 + 8 * L::NR;
  const uint32_t op_full0 = raw_empty0 + 8 * L::NR, op_free0 = op_full0 + 8 * L::NB;
  const uint32_t d_full = op_free0 + 8 * L::NB, d_empty = d_full + 8;
  float *db_s = reinterpret_cast<float *>(smem + L::DB_OFF);
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(smem + L::TMEMP_OFF);
  if (tid == 0) {
    for (int i = 0; i < L::NR; ++i) {
      mbar_init(raw_full0 + 8 * i, 1);
      mbar_init(raw_empty0 + 8 * i, NCONV / 32);
    }
    for (int i = 0; i < L::NB; ++i) {
      mbar_init(op_full0 + 8 * i, NCONV / 32);
      mbar_init(op_free0 + 8 * i, 1);
    }
    mbar_init(d_full, 1);
    mbar_init(d_empty, 4);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (tid < C) db_s[tid] = 0.f;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = __shfl_sync(0xffffffffu, *tmem_slot, 0);
  pdl_wait();   // (programmatic dependent launch: x and dout are complete from here)

  // tiles interleaved over the CTAs (tile blockIdx.x + i * gridDim.x), x fastest
  const long long stride = gridDim.x;
  const int n_tiles = (int)max(0ll, (P.n_tiles - blockIdx.x + stride - 1) / stride);
  if (warp < L::MMA_WARP) {
    // ---- converters: raw slot -> split-bf16 operands.  Warps 0-3 and 12-15:
    //      x row r = warp & 3 (TMEM lane quarter = ky'), lane = channel,
    //      pixels 0-15 / 16-31 into the A operand in TMEM.  Warps 4-11: the
    //      256 dout units into the B core matrices in shared memory.
    const bool xw = warp < 4 || warp >= 12;
    const int xh = warp >= 12 ? 1 : 0;         // pixel half of the x row
    const int u = tid - 128;
    const int c8 = u & 7, kc = (u >> 3) & 3, cg = (u >> 5) & 3, yy = u >> 7;   // dout unit (u < D_UNITS)
    const int c = xw ? lane : cg * 8 + c8;
    const uint32_t a_lane = tmem + ((uint32_t)((warp & 3) * 32) << 16) + A_COL + xh * 8;
    float dbacc = 0.f;
    for (int i_t = 0; i_t < n_tiles; ++i_t) {
      const int slot = i_t % L::NR, q = i_t % L::NB;
      const long long tl0 = clock64();
      long long tlr = 0;
      if (lane == 0) {
        mbar_wait(raw_full0 + 8 * slot, (i_t / L::NR) & 1);
        tlr = clock64();
        if (i_t >= L::NB) mbar_wait(op_free0 + 8 * q, ((i_t / L::NB) - 1) & 1);
      }
      (void)tlr;
      __syncwarp();
      tc_fence_after();
      const long long tl1 = clock64();
      const uint32_t raw = sbase + L::RAW_OFF + slot * RAW_SLOT;
      const uint32_t buf = sbase + q * L::BUF;
      if (xw) {
        // swizzled raw row R = r * 32 + c: logical 16-B chunk j at j ^ (c & 7)
        const uint32_t row = raw + (uint32_t)((warp & 3) * C + c) * 128;
        uint32_t w[NP][8];
#pragma unroll
        for (int jj = 0; jj < 4; ++jj) {
          const int j = xh * 4 + jj;
          const float4 f = ld_shared_f4(row + ((j ^ (c & 7)) << 4));
          uint32_t p0[NP], p1[NP];
          split_pair<NP>(f.x, f.y, p0);
          split_pair<NP>(f.z, f.w, p1);
#pragma unroll
          for (int p = 0; p < NP; ++p) {
            w[p][2 * jj] = p0[p];
            w[p][2 * jj + 1] = p1[p];
          }
        }
#pragma unroll
        for (int p = 0; p < NP; ++p) tmem_st8u(a_lane + q * L::A_BUF_COLS + p * 16, w[p]);
        tmem_wait_st();
      } else if (u < D_UNITS) {
        // dout row yy: box pixel e = p - (x0 - 4); values p = x0 + 8 kc - 1 .. + 8 are e = 8 kc + 3 .. 8 kc + 12
        const uint32_t row = raw + RAW_X + (uint32_t)(yy * C + c) * (DBOX * 4) + kc * 32;
        const float4 a = ld_shared_f4(row), b = ld_shared_f4(row + 16), e = ld_shared_f4(row + 32),
                     f = ld_shared_f4(row + 48);
        const float dv[10] = {a.w, b.x, b.y, b.z, b.w, e.x, e.y, e.z, e.w, f.x};
#pragma unroll
        for (int i = 1; i <= 8; ++i) dbacc += dv[i];
        // pairs (0,1) .. (8,9) split once; B_kx[p] = dout[p - kx + 1]: kx = 0
        // the pairs from (2,3), kx = 2 from (0,1), kx = 1 the odd-aligned pairs
        uint32_t ev[5][NP];
#pragma unroll
        for (int i = 0; i < 5; ++i) split_pair<NP>(dv[2 * i], dv[2 * i + 1], ev[i]);
        const uint32_t dst = buf + yy * L::D_ROW + cg * CGB + kc * 128 + c8 * 16;
#pragma unroll
        for (int p = 0; p < NP; ++p) {
          st_shared_v4(dst + p * L::D_PART, ev[1][p], ev[2][p], ev[3][p], ev[4][p]);
          st_shared_v4(dst + ROWB + p * L::D_PART, mid_pair(ev[0][p], ev[1][p]), mid_pair(ev[1][p], ev[2][p]),
                       mid_pair(ev[2][p], ev[3][p]), mid_pair(ev[3][p], ev[4][p]));
          st_shared_v4(dst + 2 * ROWB + p * L::D_PART, ev[0][p], ev[1][p], ev[2][p], ev[3][p]);
        }
      }
      fence_proxy_async();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(raw_empty0 + 8 * slot);
        mbar_arrive(op_full0 + 8 * q);
      }
      if (warp == 0) WTL(0, i_t, tl0, tl1, tlr);
    }
    if (!xw && u < D_UNITS) atomicAdd(&db_s[c], dbacc);
  } else if (warp == L::TMA_WARP) {
    // ---- producer: raw boxes of tile i into slot i % NR
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&P.tm_x)) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&P.tm_d)) : "memory");
      for (int i_t = 0; i_t < n_tiles; ++i_t) {
        const int slot = i_t % L::NR;
        if (i_t >= L::NR) mbar_wait(raw_empty0 + 8 * slot, ((i_t / L::NR) - 1) & 1);
        const long long t = blockIdx.x + (long long)i_t * stride;
        const long long img = t / ((long long)P.tiles_y * P.tiles_x);
        const int rem = (int)(t - img * P.tiles_y * P.tiles_x);
        const int b = (int)img, ty = rem / P.tiles_x, tx = rem % P.tiles_x;
        const int y0 = ty * TY, x0 = tx * WT;
        const uint32_t raw = sbase + L::RAW_OFF + slot * RAW_SLOT;
        mbar_expect_tx(raw_full0 + 8 * slot, RAW_X + RAW_D);
        tma_load_4d(raw, &P.tm_x, x0, 0, y0 - 1, b, raw_full0 + 8 * slot);
        tma_load_4d(raw + RAW_X, &P.tm_d, x0 - 4, 0, y0, b, raw_full0 + 8 * slot);
      }
    }
    __syncwarp();
  } else if (warp == L::MMA_WARP) {
    // ---- MMA warp: tiles in order; chains of F tiles into D (the first MMA
    //      of a chain overwrites it), each handed to the flushers
    for (int i_t = 0; i_t < n_tiles; ++i_t) {
      const int q = i_t % L::NB;
      const int f = i_t / L::F;
      const bool chain_start = i_t % L::F == 0;
      const bool chain_end = i_t % L::F == L::F - 1 || i_t == n_tiles - 1;
      const long long tm0 = clock64();
      long long tm1 = 0;
      if (lane == 0) {
        if (chain_start && f >= 1) mbar_wait(d_empty, (f - 1) & 1);
        tm1 = clock64();
        mbar_wait(op_full0 + 8 * q, (i_t / L::NB) & 1);
      }
      __syncwarp();
      tc_fence_after();
      if (lane == 0) {
        const uint32_t buf = sbase + q * L::BUF;
        // B: K-major, no swizzle: K core matrices 128 B apart, 8-row groups
        // CGB apart; A: part pa, K-step ks at TMEM column +pa*16 + ks*8
        const uint64_t d0 = umma_desc(buf, 128, CGB);
        const uint32_t a0 = tmem + A_COL + q * L::A_BUF_COLS;
#pragma unroll
        for (int ks = 0; ks < WT / 16; ++ks)
#pragma unroll
          for (int pr = 0; pr < L::NPROD; ++pr) {
            constexpr int pa_tab[6] = {0, 0, 1, 0, 1, 2}, pb_tab[6] = {0, 1, 0, 2, 1, 0};
            const uint32_t bo = (pb_tab[pr] * L::D_PART + ks * 256) >> 4;
            const bool first = chain_start && ks == 0 && pr == 0;
            mma_bf16_ta(tmem + D_COL, a0 + pa_tab[pr] * 16 + ks * 8, d0 + bo, first ? 0u : 1u);
          }
        tc_commit(op_free0 + 8 * q);
        if (chain_end) tc_commit(d_full);
      }
      WTL(8, i_t, tm0, tm1, 0);
      __syncwarp();
    }
  } else {
    // ---- flushers (one per TMEM lane quarter): D2 += D in fp32, so the
    //      tensor core's accumulation chains stay F tiles long
    const uint32_t lrow = (uint32_t)((warp & 3) * 32) << 16;
    const int n_chains = (n_tiles + L::F - 1) / L::F;
    for (int f = 0; f < n_chains; ++f) {
      const long long tf0 = clock64();
      if (lane == 0) mbar_wait(d_full, f & 1);
      __syncwarp();
      const long long tf1 = clock64();
      tc_fence_after();
#pragma unroll 1
      for (int cc = 0; cc < NCOL; cc += 32) {
        float v[32];
        tmem_ld32(tmem + lrow + D_COL + cc, v);
        if (f > 0) {
          float a[32];
          tmem_ld32(tmem + lrow + D2_COL + cc, a);
#pragma unroll
          for (int i = 0; i < 32; ++i) v[i] += a[i];
        }
        tmem_st32(tmem + lrow + D2_COL + cc, v);
      }
      tmem_wait_st();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(d_empty);
      if (warp == L::FLUSH_WARP0) WTL(9, f, tf0, tf1, 0);
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  // ---- D2 -> dW (fp64) by the converter warps: TMEM lane = ky' * 32 + ci,
  //      column = (s, kx, co).  Every dW element has two entries (s = 0, 1;
  //      ky' = ky + s): D2 goes through shared memory (the operand and raw
  //      buffers are free now) and each element is added with one fp64
  //      atomic instead of two (the 148 CTAs' atomics on the same 9216
  //      addresses are the kernel's tail: ~20 us per launch with two)
  if (n_tiles > 0 && warp < L::MMA_WARP) {
    constexpr int CPW = NCOL / (NCONV / 128);   // columns per warp
    constexpr int DP2 = NCOL + 1;               // padded row: conflict-free column-wise stores
    static_assert(128 * DP2 * 4 <= L::BAR_OFF, "D2 staging exceeds the free buffers");
    float *d2s = reinterpret_cast<float *>(smem);
    const int quarter = warp & 3;
    const int c_lo = (warp >> 2) * CPW;
#pragma unroll
    for (int cc = 0; cc < CPW; cc += 16) {
      float v[16];
      tmem_ld16(tmem + ((uint32_t)(quarter * 32) << 16) + D2_COL + c_lo + cc, v);
#pragma unroll
      for (int i = 0; i < 16; ++i) d2s[(quarter * 32 + lane) * DP2 + c_lo + cc + i] = v[i];
    }
    named_bar(1, NCONV);
    for (int t = tid; t < C * C * 9; t += NCONV) {
      const int co = t % C, kx = (t / C) % 3, ky = (t / (3 * C)) % 3, ci = t / (9 * C);
      double sum = 0.0;
#pragma unroll
      for (int sp = 0; sp < TY; ++sp) sum += (double)d2s[((ky + sp) * C + ci) * DP2 + (sp * 3 + kx) * C + co];
      atomicAdd(P.dw + ((size_t)(co * C + ci) * 3 + ky) * 3 + kx, sum);
    }
  }
  if (tid < C && P.db) atomicAdd(P.db + tid, (double)db_s[tid]);
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

// (W, C, H, B) view of an NCHW fp32 tensor; box (bw, 32, bh, 1)
static int make_map(CUtensorMap *map, const float *base, int B, int H, int W, int bw, int bh, bool swz) {
  auto enc = tensor_map_encoder();
  HT_REQUIRE(enc != nullptr, "cuTensorMapEncodeTiled unavailable");
  const cuuint64_t row = (cuuint64_t)W * 4, planeb = row * H;
  cuuint64_t dims[4] = {(cuuint64_t)W, (cuuint64_t)C, (cuuint64_t)H, (cuuint64_t)B};
  cuuint64_t strides[3] = {planeb, row, planeb * C};
  cuuint32_t box[4] = {(cuuint32_t)bw, (cuuint32_t)C, (cuuint32_t)bh, 1};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  const CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, const_cast<float *>(base), dims, strides, box,
                         estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                         swz ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                         CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  HT_REQUIRE(r == CUDA_SUCCESS, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return HT_OK;
}

template <int NP>
static int launch(const float *x, const float *dout, int B, int H, int W, double *dw, double *db, cudaStream_t st) {
  using L = Lay<NP>;
  static_assert(L::SMEM <= 232448, "shared memory exceeded");
  if (int rc = ensure_smem_attr((const void *)wgrad_tc_kernel<NP>, L::SMEM)) return rc;
  if (B <= 0 || H <= 0 || W <= 0) return HT_OK;
  int dev = 0, n_sm = 148;
  HT_CUDA(cudaGetDevice(&dev));
  HT_CUDA(cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev));
  WgParams p{};
  int rc = make_map(&p.tm_x, x, B, H, W, WT, XR, true);
  if (rc) return rc;
  rc = make_map(&p.tm_d, dout, B, H, W, DBOX, TY, false);
  if (rc) return rc;
  p.B = B; p.H = H; p.W = W; p.dw = dw; p.db = db;
  p.tiles_y = (H + TY - 1) / TY;
  p.tiles_x = (W + WT - 1) / WT;
  p.n_tiles = (long long)B * p.tiles_y * p.tiles_x;
  const long long grid = p.n_tiles < n_sm ? p.n_tiles : n_sm;
  HT_CUDA(launch_pdl(wgrad_tc_kernel<NP>, (unsigned)grid, L::NTHR, L::SMEM, st, p));
  count_launch();
  HT_CHECK_LAUNCH();
  return HT_OK;
}

}  // namespace wgt

#ifdef WG_TL
extern "C" void *ht_debug_wtl_ptr() {
  void *p = nullptr;
  cudaGetSymbolAddress(&p, wgt::g_wtl);
  return p;
}
#endif

// dw (32, 32, 3, 3) and db (32) fp64 accumulate (+=) the gradient of a 3x3
// pad-1 conv with x, dout (B, 32, H, W) fp32 (W % 4 == 0: TMA row strides).
// parts: 2 or 3 bf16 parts.
int wgrad_tc32(const float *x, const float *dout, int B, int H, int W, double *dw, double *db, int parts,
               cudaStream_t st) {
  return parts == 3 ? wgt::launch<3>(x, dout, B, H, W, dw, db, st) : wgt::launch<2>(x, dout, B, H, W, dw, db, st);
}

}  // namespace ht
