// ht_pack_params: repack the flat float64 parameter vector (params() order,
// nn.py:118-122) into every layout the kernels consume.
#include <cuda_fp16.h>

#include "common.cuh"
#include "fwd_tc.cuh"

namespace ht {

PackLayout pack_layout(int C, int NB) {
  NetGeom g(C, NB);
  PackLayout L;
  L.f32_off = 0;
  L.f32t_off = align256(L.f32_off + g.total * 4);
  L.tc_off = align256(L.f32t_off + g.total * 4);
  L.tcb_off = align256(L.tc_off + tc::weight_bytes(NB));
  L.total = align256(L.tcb_off + tc::bias_floats(NB) * 4);
  return L;
}

__global__ void pack_f32_kernel(const double *__restrict__ p, float *__restrict__ f32,
                                int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    f32[i] = (float)p[i];
}

// transposed + spatially flipped copies: for a conv with weight w[co][ci][3][3]
// at offset `off`, wt[ci][co][a][b] = w[co][ci][2-a][2-b] at the same offset.
// Biases are copied unchanged (unused).
__global__ void pack_f32t_kernel(const double *__restrict__ p, float *__restrict__ wt, int C,
                                 int NB) {
  NetGeom g(C, NB);
  const int nconv = 2 * NB + 2;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < g.total;
       i += (int64_t)gridDim.x * blockDim.x) {
    // locate conv containing i
    int64_t off = 0;
    int cout = C, cin = 2;
    bool is_w = false;
    int64_t base = 0;
    for (int k = 0; k < nconv; ++k) {
      if (k == 0) { off = g.in_w; cout = C; cin = 2; }
      else if (k == nconv - 1) { off = g.out_w; cout = 1; cin = C; }
      else { const int b = (k - 1) / 2; off = ((k - 1) % 2 == 0) ? g.w1(b) : g.w2(b); cout = C; cin = C; }
      const int64_t wsz = (int64_t)cout * cin * 9;
      if (i >= off && i < off + wsz) { is_w = true; base = off; break; }
    }
    if (!is_w) { wt[i] = (float)p[i]; continue; }
    const int64_t r = i - base;  // index in the transposed tensor [cin][cout][a][b]
    const int bb = (int)(r % 3), a = (int)((r / 3) % 3);
    const int co = (int)((r / 9) % cout), ci = (int)(r / (9 * cout));
    wt[i] = (float)p[base + (((int64_t)co * cin + ci) * 3 + (2 - a)) * 3 + (2 - bb)];
  }
}

}  // namespace ht

extern "C" {

int ht_packed_bytes(int channels, int blocks, int64_t *bytes) {
  if (channels < 1 || blocks < 0) return ht::fail(HT_E_INVALID, "bad architecture");
  *bytes = ht::pack_layout(channels, blocks).total;
  return HT_OK;
}

int ht_pack_params(const double *params, int C, int NB, void *packed, void *stream) {
  if (C < 1 || NB < 0) return ht::fail(HT_E_INVALID, "bad architecture");
  cudaStream_t st = (cudaStream_t)stream;
  ht::NetGeom g(C, NB);
  ht::PackLayout L = ht::pack_layout(C, NB);
  char *base = (char *)packed;
  ht::pack_f32_kernel<<<256, 256, 0, st>>>(params, (float *)(base + L.f32_off), g.total);
  HT_CHECK_LAUNCH();
  ht::pack_f32t_kernel<<<256, 256, 0, st>>>(params, (float *)(base + L.f32t_off), C, NB);
  HT_CHECK_LAUNCH();
  if (C == ht::tc::C) {
    int rc = ht::tc::pack(params, NB, base + L.tc_off, (float *)(base + L.tcb_off), st);
    if (rc) return rc;
    rc = ht::note_bias_pack(base + L.tcb_off, st);
    if (rc) return rc;
  }
  return HT_OK;
}

}  // extern "C"
