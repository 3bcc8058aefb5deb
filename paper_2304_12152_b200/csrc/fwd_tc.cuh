// Fused tensor-core policy forward (K1) -- interface shared with pack.cu and
// the C-ABI.  Design notes live in fwd_tc.cu and DESIGN.md.
#pragma once
#include <stdint.h>

#include <cuda_runtime.h>

namespace ht {
namespace tc {

constexpr int C = 32;          // channels the fused kernel is built for (PRESET_PAPER)
constexpr int M = 128;         // pixels per UMMA M-tile (one strip row)
constexpr int NPIX = M + 2;    // A row buffer pixels: one zero pixel each side
// bytes per 8-channel K-chunk plane of a row: NPIX pixels rounded up to whole
// 128-B lines so every plane of a row starts at the same bank phase
constexpr int PLANE = (NPIX * 16 + 127) / 128 * 128;
// A-row buffers start 16 B before a 128-B boundary, so pixel 0 of a strip row
// (buffer pixel 1) is line aligned and a warp's 512-B store is 4 wavefronts
constexpr int A_PHASE = 112;
// strip geometry, identical for every pass: a strip row holds lanes
// [STRIP_L, STRIP_L + STRIP_S) of output plus >= G halo lanes each side.
// Pass buffers store column v at v + XPAD with a pitch that is a multiple of 8
// pixels, so lane 0 of every strip row (v = s*STRIP_S - STRIP_L) is 128-B
// aligned in the fp32 channel-group-planar layout.
constexpr int STRIP_L = 4;
constexpr int STRIP_S = M - 2 * STRIP_L;
constexpr int XPAD = STRIP_L;
static_assert(STRIP_S % 8 == 0, "strip stride must keep 128-B alignment");
__host__ __device__ inline int64_t x_pitch(int VW) { return ((int64_t)VW + XPAD + 7) / 8 * 8; }
constexpr int NSLICE = 5;      // doubled ky sequence [2,1,0,2,1] (rotation windows)

// weight tile bytes for one (kx, kh) UMMA K-step: 2 K-chunks x 5*ns rows x 16 B
constexpr int tile_bytes(int ns) { return 2 * NSLICE * ns * 16; }
constexpr int W_IN_BYTES = 3 * 1 * tile_bytes(32);   // conv_in: K=16 (split c/z)
constexpr int W_MID_BYTES = 3 * 2 * tile_bytes(32);  // 32->32 conv: K=32
constexpr int W_OUT_BYTES = 3 * 2 * tile_bytes(16);  // conv_out: K=32, N padded 1->16

__host__ __device__ inline int64_t weight_bytes(int NB) {
  return (int64_t)W_IN_BYTES + (int64_t)2 * NB * W_MID_BYTES + W_OUT_BYTES;
}
__host__ __device__ inline int64_t weight_offset_mid(int conv_idx /*0-based over the 2*NB convs*/) {
  return (int64_t)W_IN_BYTES + (int64_t)conv_idx * W_MID_BYTES;
}
__host__ __device__ inline int64_t weight_offset_out(int NB) { return (int64_t)W_IN_BYTES + (int64_t)2 * NB * W_MID_BYTES; }
// fp32 biases: conv_in (32) | 2*NB convs (32 each) | conv_out (padded 32)
__host__ __device__ inline int64_t bias_floats(int NB) { return (int64_t)32 * (2 * NB + 2); }

int pack(const double *params, int NB, void *tc_dst, float *bias_dst, cudaStream_t st);

// workspace bytes for run(): two fp32 NHWC pass buffers of the virtual
// side-by-side image + flag
int64_t workspace_bytes(int NB, int B, int H, int W, int in_rows);

int run(const void *tc_w, const float *tc_b, int NB, const float *c, const float *z, int B,
        int H, int W, int in_row0, int in_rows, int out_row0, int out_rows, float *p,
        uint8_t *h, uint32_t *pbm_words, void *ws, int64_t ws_bytes, int *flag_dev, int levels,
        cudaStream_t st);

}  // namespace tc
}  // namespace ht
