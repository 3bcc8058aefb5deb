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
constexpr int PLANE = NPIX * 16;  // bytes per 8-channel K-chunk plane of a row
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
        uint8_t *h, void *ws, int64_t ws_bytes, int *flag_dev, cudaStream_t st);

}  // namespace tc
}  // namespace ht
