// ht_halftone: the inference entry point (K1 + PBM epilogue) and its
// workspace sizing.  Replaces rl.infer_halftone's forward + threshold
// (rl.py:306-311) and feeds imagecore.save_pbm's payload (imagecore.py:289-297).
#include "common.cuh"
#include "fwd_tc.cuh"

namespace ht {
int simt_halftone(const void *packed, int C, int NB, const float *c, const float *z, int B,
                  int H, int W, int in_row0, int in_rows, int out_row0, int out_rows, float *p,
                  uint8_t *h, void *ws, int64_t ws_bytes, int *nonfinite_dev, int levels,
                  cudaStream_t st);
int64_t simt_halftone_ws(int C, int B, int W, int in_rows);

// PBM P4 payload from a uint8 halftone (1 = white): bit = 1 - h, MSB first,
// rows padded to whole bytes with 0 bits (np.packbits, imagecore.py:293-294).
__global__ void pbm_pack_kernel(const uint8_t *__restrict__ h, int64_t rows, int W,
                                uint8_t *__restrict__ out) {
  const int rb = (W + 7) / 8;
  const int64_t n = rows * rb;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = i / rb;
    const int byte = (int)(i % rb);
    const uint8_t *hr = h + row * W;
    uint8_t v = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int x = byte * 8 + k;
      const uint8_t bit = (x < W) ? (uint8_t)(1 - hr[x]) : 0;
      v |= bit << (7 - k);
    }
    out[i] = v;
  }
}
}  // namespace ht

extern "C" {

int ht_halftone_workspace_bytes(int C, int NB, int B, int H, int W, int in_rows, int out_rows,
                                int impl, int64_t *bytes) {
  if (B < 1 || H < 1 || W < 1 || in_rows < 1) return ht::fail(HT_E_INVALID, "empty image");
  int64_t base = 256;  // flag
  if (impl == 0 && C == ht::tc::C)   // PBM words (K1 writes the payload bits itself)
    *bytes = base + ht::align256(((int64_t)B * out_rows * ((W + 7) / 8) + 3) / 4 * 4) +
             ht::tc::workspace_bytes(NB, B, H, W, in_rows);
  else                               // uint8 h scratch for the PBM pack kernel
    *bytes = base + ht::align256((int64_t)B * out_rows * W) + ht::simt_halftone_ws(C, B, W, in_rows);
  return HT_OK;
}

}  // extern "C"

static int halftone_impl(const void *packed, int C, int NB, const float *c, const float *z, int B, int H,
                int W, int in_row0, int in_rows, int out_row0, int out_rows, float *p,
                uint8_t *h, uint8_t *pbm, void *ws, int64_t ws_bytes, int impl, int levels,
                void *stream) {
  ht::reset_launches();
  HT_REQUIRE(B >= 1 && H >= 1 && W >= 1, "input must be non-empty (B=%d H=%d W=%d)", B, H, W);
  HT_REQUIRE(in_row0 >= 0 && in_rows >= 1 && in_row0 + in_rows <= H, "bad input row window");
  HT_REQUIRE(out_row0 >= in_row0 && out_rows >= 1 && out_row0 + out_rows <= in_row0 + in_rows,
             "output rows must lie inside the input rows");
  HT_REQUIRE(impl == 0 || impl == 1, "impl must be 0 (tensor core) or 1 (simt)");
  HT_REQUIRE(levels >= 2 && levels <= 256, "levels must be in [2, 256]");
  HT_REQUIRE(levels == 2 || pbm == nullptr, "the PBM payload is binary (levels = 2)");
  if (impl == 0 && C != ht::tc::C)
    return ht::fail(HT_E_UNSUPPORTED, "fused tensor-core forward is built for channels=%d (got %d)",
                    ht::tc::C, C);
  int64_t need = 0;
  int rc = ht_halftone_workspace_bytes(C, NB, B, H, W, in_rows, out_rows, impl, &need);
  if (rc) return rc;
  HT_REQUIRE(ws_bytes >= need, "workspace too small: %lld < %lld", (long long)ws_bytes,
             (long long)need);
  cudaStream_t st = (cudaStream_t)stream;
  char *wsb = (char *)ws;
  int *flag = (int *)wsb;
  HT_CUDA(cudaMemsetAsync(flag, 0, sizeof(int), st));
  const int64_t pbm_bytes = (int64_t)B * out_rows * ((W + 7) / 8);
  if (impl == 0) {
    // K1 ORs the PBM bits into 32-bit words: straight into the caller's
    // buffer when it is word-aligned and whole words long, else into a padded
    // workspace copy (then one device copy of the exact payload)
    HT_REQUIRE(pbm_bytes < (1ll << 34), "PBM payload too large");
    uint32_t *words = (uint32_t *)(wsb + 256);
    const bool direct = pbm && ((uintptr_t)pbm % 4 == 0) && pbm_bytes % 4 == 0;
    if (direct) words = (uint32_t *)pbm;
    const int64_t wbytes = (pbm_bytes + 3) / 4 * 4;
    char *rest = wsb + 256 + ht::align256(wbytes);
    const int64_t rest_bytes = ws_bytes - (rest - wsb);
    if (pbm) HT_CUDA(cudaMemsetAsync(words, 0, wbytes, st));
    ht::PackLayout L = ht::pack_layout(C, NB);
    rc = ht::tc::run((const char *)packed + L.tc_off, (const float *)((const char *)packed + L.tcb_off),
                     NB, c, z, B, H, W, in_row0, in_rows, out_row0, out_rows, p, h, pbm ? words : nullptr,
                     rest, rest_bytes, flag, levels, st);
    if (rc) return rc;
    if (pbm && !direct) HT_CUDA(cudaMemcpyAsync(pbm, words, pbm_bytes, cudaMemcpyDeviceToDevice, st));
    return HT_OK;
  }
  uint8_t *hscratch = (uint8_t *)(wsb + 256);
  char *rest = wsb + 256 + ht::align256((int64_t)B * out_rows * W);
  const int64_t rest_bytes = ws_bytes - (rest - wsb);
  uint8_t *hout = h ? h : (pbm ? hscratch : nullptr);
  rc = ht::simt_halftone(packed, C, NB, c, z, B, H, W, in_row0, in_rows, out_row0, out_rows, p,
                         hout, rest, rest_bytes, flag, levels, st);
  if (rc) return rc;
  if (pbm) {
    const int64_t n = (int64_t)B * out_rows * ((W + 7) / 8);
    const int grid = (int)((n + 255) / 256 < 4096 ? (n + 255) / 256 : 4096);
    ht::pbm_pack_kernel<<<grid, 256, 0, st>>>(hout, (int64_t)B * out_rows, W, pbm);
    ht::count_launch();
    HT_CHECK_LAUNCH();
  }
  return HT_OK;
}

extern "C" {

int ht_halftone(const void *packed, int C, int NB, const float *c, const float *z, int B, int H,
                int W, int in_row0, int in_rows, int out_row0, int out_rows, float *p,
                uint8_t *h, uint8_t *pbm, void *ws, int64_t ws_bytes, int impl, void *stream) {
  return halftone_impl(packed, C, NB, c, z, B, H, W, in_row0, in_rows, out_row0, out_rows, p, h,
                       pbm, ws, ws_bytes, impl, 2, stream);
}

// Multitone inference (multitone.infer_multitone, multitone.py:70-76): q =
// index of the nearest level i/(levels-1) (half-steps round up), uint8.
int ht_multitone(const void *packed, int C, int NB, const float *c, const float *z, int B, int H,
                 int W, int in_row0, int in_rows, int out_row0, int out_rows, int levels, float *p,
                 uint8_t *q, void *ws, int64_t ws_bytes, int impl, void *stream) {
  return halftone_impl(packed, C, NB, c, z, B, H, W, in_row0, in_rows, out_row0, out_rows, p, q,
                       nullptr, ws, ws_bytes, impl, levels, stream);
}

// Non-finite flag of the last ht_halftone that used `ws` (reads 4 bytes;
// synchronises the stream).  Returns HT_E_NONFINITE when set (nn.py:147-148).
int ht_halftone_check(const void *ws, void *stream) {
  int f = 0;
  cudaStream_t st = (cudaStream_t)stream;
  HT_CUDA(cudaMemcpyAsync(&f, ws, sizeof(int), cudaMemcpyDeviceToHost, st));
  HT_CUDA(cudaStreamSynchronize(st));
  if (f) return ht::fail(HT_E_NONFINITE, "non-finite logits");
  return HT_OK;
}

}  // extern "C"
