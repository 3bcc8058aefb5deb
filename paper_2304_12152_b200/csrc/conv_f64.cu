// Drop-in Conv2d forward / backward in float64 (nn.py:36-80), any channel
// counts: the reference's layer-level API (Conv2d.forward / .backward,
// ResidualBlock, and PolicyNetwork with in_channels != 2), computed on the
// device in the reference's float64.  The network-level hot paths use the
// fused / tensor-core kernels instead (fwd_tc.cu, conv_tc.cu).
//
// Convention (nn.py:46-60, pinned by test_nn.py:33-41): cross-correlation
// with zero padding 1, out[b,o,y,x] = bias[o] + sum_{i,ky,kx}
// x[b,i,y+ky-1,x+kx-1] w[o,i,ky,kx].
#include "common.cuh"

namespace ht {

__global__ void conv_f64_fwd_kernel(const double *__restrict__ x, int B, int Ci, int Co, int H, int W,
                                    const double *__restrict__ w, const double *__restrict__ bias,
                                    double *__restrict__ out) {
  const int64_t n = (int64_t)B * Co * H * W;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int xx = (int)(i % W), yy = (int)((i / W) % H);
    const int o = (int)((i / ((int64_t)H * W)) % Co);
    const int64_t b = i / ((int64_t)Co * H * W);
    double acc = bias ? bias[o] : 0.0;
    for (int ci = 0; ci < Ci; ++ci) {
      const double *xp = x + ((b * Ci + ci) * H) * (int64_t)W;
      const double *wp = w + ((int64_t)o * Ci + ci) * 9;
      for (int ky = 0; ky < 3; ++ky) {
        const int sy = yy + ky - 1;
        if (sy < 0 || sy >= H) continue;
        for (int kx = 0; kx < 3; ++kx) {
          const int sx = xx + kx - 1;
          if (sx < 0 || sx >= W) continue;
          acc += xp[(int64_t)sy * W + sx] * wp[ky * 3 + kx];
        }
      }
    }
    out[i] = acc;
  }
}

// dx[b,i,y,x] = sum_{o,ky,kx} dout[b,o,y-ky+1,x-kx+1] w[o,i,ky,kx]
__global__ void conv_f64_dgrad_kernel(const double *__restrict__ dout, int B, int Ci, int Co, int H, int W,
                                      const double *__restrict__ w, double *__restrict__ dx) {
  const int64_t n = (int64_t)B * Ci * H * W;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int xx = (int)(i % W), yy = (int)((i / W) % H);
    const int ci = (int)((i / ((int64_t)H * W)) % Ci);
    const int64_t b = i / ((int64_t)Ci * H * W);
    double acc = 0.0;
    for (int o = 0; o < Co; ++o) {
      const double *dp = dout + ((b * Co + o) * H) * (int64_t)W;
      const double *wp = w + ((int64_t)o * Ci + ci) * 9;
      for (int ky = 0; ky < 3; ++ky) {
        const int sy = yy - ky + 1;
        if (sy < 0 || sy >= H) continue;
        for (int kx = 0; kx < 3; ++kx) {
          const int sx = xx - kx + 1;
          if (sx < 0 || sx >= W) continue;
          acc += dp[(int64_t)sy * W + sx] * wp[ky * 3 + kx];
        }
      }
    }
    dx[i] = acc;
  }
}

// dw[o,i,ky,kx] += sum_{b,y,x} dout[b,o,y,x] x[b,i,y+ky-1,x+kx-1]   (one
// block per weight element; fixed-order block reduction), db[o] += sum dout
__global__ void conv_f64_wgrad_kernel(const double *__restrict__ x, const double *__restrict__ dout, int B, int Ci,
                                      int Co, int H, int W, double *__restrict__ dw, double *__restrict__ db) {
  const int e = blockIdx.x;                       // weight element, or Co*Ci*9 + o for the bias
  const bool is_bias = e >= Co * Ci * 9;
  const int o = is_bias ? e - Co * Ci * 9 : e / (Ci * 9);
  const int ci = is_bias ? 0 : (e / 9) % Ci;
  const int ky = is_bias ? 1 : (e % 9) / 3, kx = is_bias ? 1 : e % 3;
  const int64_t HW = (int64_t)H * W, n = (int64_t)B * HW;
  double acc = 0.0;
  for (int64_t j = threadIdx.x; j < n; j += blockDim.x) {
    const int64_t b = j / HW;
    const int yy = (int)((j % HW) / W), xx = (int)(j % W);
    const double g = dout[(b * Co + o) * HW + (int64_t)yy * W + xx];
    if (is_bias) {
      acc += g;
    } else {
      const int sy = yy + ky - 1, sx = xx + kx - 1;
      if (sy >= 0 && sy < H && sx >= 0 && sx < W) acc += g * x[(b * Ci + ci) * HW + (int64_t)sy * W + sx];
    }
  }
  __shared__ double red[32];
  for (int s = 16; s > 0; s >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, s);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int k = 0; k < (int)(blockDim.x >> 5); ++k) t += red[k];
    if (is_bias) db[o] += t;
    else dw[e] += t;
  }
}

static int grid_for(int64_t n) { return (int)((n + 255) / 256 < 16384 ? (n + 255) / 256 : 16384); }

}  // namespace ht

extern "C" {

int ht_conv3x3_f64(const double *x, int B, int Ci, int Co, int H, int W, const double *w, const double *bias,
                   double *out, void *stream) {
  HT_REQUIRE(B >= 1 && Ci >= 1 && Co >= 1 && H >= 1 && W >= 1, "empty conv");
  const int64_t n = (int64_t)B * Co * H * W;
  ht::conv_f64_fwd_kernel<<<ht::grid_for(n), 256, 0, (cudaStream_t)stream>>>(x, B, Ci, Co, H, W, w, bias, out);
  ht::count_launch();
  HT_CHECK_LAUNCH();
  return HT_OK;
}

int ht_conv3x3_f64_backward(const double *x, const double *dout, int B, int Ci, int Co, int H, int W,
                            const double *w, double *dw, double *db, double *dx, void *stream) {
  HT_REQUIRE(B >= 1 && Ci >= 1 && Co >= 1 && H >= 1 && W >= 1, "empty conv");
  cudaStream_t st = (cudaStream_t)stream;
  if (dw && db) {
    ht::conv_f64_wgrad_kernel<<<Co * Ci * 9 + Co, 256, 0, st>>>(x, dout, B, Ci, Co, H, W, dw, db);
    ht::count_launch();
    HT_CHECK_LAUNCH();
  }
  if (dx) {
    const int64_t n = (int64_t)B * Ci * H * W;
    ht::conv_f64_dgrad_kernel<<<ht::grid_for(n), 256, 0, st>>>(dout, B, Ci, Co, H, W, w, dx);
    ht::count_launch();
    HT_CHECK_LAUNCH();
  }
  return HT_OK;
}

}  // extern "C"
