// K5 / K7: periodogram, ring statistics, anisotropy loss and its gradient,
// fp64 (complex128 like numpy.fft).
//
// Reference: periodogram (spectral.py:17-24), ring partition (39-55),
// _ring_sums / rapsd (67-88), _loss_pieces / anisotropy_loss /
// anisotropy_loss_backward (100-133).  The 2-D DFT is evaluated as two
// separable 1-D DFT passes with an exact twiddle table (angle index reduced
// mod N before sin/cos), so any image size is supported.
#include <math.h>

#include "common.cuh"

namespace ht {

// twiddle table tw[k] = exp(-2 pi i k / N), k in [0, N)
__global__ void twiddle_kernel(double2 *__restrict__ tw, int N) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= N) return;
  double s, c;
  sincospi(-2.0 * (double)k / (double)N, &s, &c);
  tw[k] = make_double2(c, s);
}

// forward row DFT of real input: Y[b][y][kx] = sum_x x[b][y][x] tw_W[(kx*x) mod W]
__global__ void dft_rows_real_kernel(const float *__restrict__ x, int B, int H, int W,
                                     const double2 *__restrict__ tw, double2 *__restrict__ Y) {
  const int64_t n = (int64_t)B * H * W;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int kx = (int)(i % W);
    const int64_t row = i / W;
    const float *xr = x + row * W;
    double re = 0.0, im = 0.0;
    int idx = 0;
    for (int xx = 0; xx < W; ++xx) {
      const double v = (double)xr[xx];
      const double2 t = tw[idx];
      re += v * t.x;
      im += v * t.y;
      idx += kx;
      if (idx >= W) idx -= W;
    }
    Y[i] = make_double2(re, im);
  }
}

// column DFT (complex): Z[b][ky][kx] = sum_y Y[b][y][kx] tw_H[(sgn*ky*y) mod H]
// conj = 1 uses the conjugate twiddles (inverse transform, unnormalised).
__global__ void dft_cols_kernel(const double2 *__restrict__ Y, int B, int H, int W,
                                const double2 *__restrict__ tw, int conj,
                                double2 *__restrict__ Z) {
  const int64_t n = (int64_t)B * H * W;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int kx = (int)(i % W);
    const int ky = (int)((i / W) % H);
    const int64_t b = i / ((int64_t)H * W);
    const double2 *col = Y + b * H * W + kx;
    double re = 0.0, im = 0.0;
    int idx = 0;
    for (int y = 0; y < H; ++y) {
      const double2 v = col[(int64_t)y * W];
      double2 t = tw[idx];
      if (conj) t.y = -t.y;
      re += v.x * t.x - v.y * t.y;
      im += v.x * t.y + v.y * t.x;
      idx += ky;
      if (idx >= H) idx -= H;
    }
    Z[i] = make_double2(re, im);
  }
}

// inverse row DFT keeping the real part: out[b][y][x] = scale/N * Re sum_kx
//   G[b][y][kx] conj(tw_W)[(kx*x) mod W]
__global__ void idft_rows_real_kernel(const double2 *__restrict__ G, int B, int H, int W,
                                      const double2 *__restrict__ tw, double scale,
                                      float *__restrict__ out) {
  const int64_t n = (int64_t)B * H * W;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int xx = (int)(i % W);
    const int64_t row = i / W;
    const double2 *gr = G + row * W;
    double re = 0.0;
    int idx = 0;
    for (int kx = 0; kx < W; ++kx) {
      const double2 v = gr[kx];
      const double2 t = tw[idx];  // conj: (t.x, -t.y)
      re += v.x * t.x + v.y * t.y;
      idx += xx;
      if (idx >= W) idx -= W;
    }
    out[i] = (float)(re * scale);
  }
}

// ring sums of P = |X|^2 / N per image: sums[b][ring] (spectral.py:67-71)
__global__ void ring_power_kernel(const double2 *__restrict__ X, int B, int HW,
                                  const int32_t *__restrict__ ring, int n_rings,
                                  double *__restrict__ sums) {
  extern __shared__ double hist[];
  const int b = blockIdx.y;
  for (int r = threadIdx.x; r < n_rings; r += blockDim.x) hist[r] = 0.0;
  __syncthreads();
  const double inv = 1.0 / (double)HW;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < HW; i += gridDim.x * blockDim.x) {
    const int r = ring[i];
    if (r < 0) continue;
    const double2 v = X[(int64_t)b * HW + i];
    atomicAdd(&hist[r], (v.x * v.x + v.y * v.y) * inv);
  }
  __syncthreads();
  for (int r = threadIdx.x; r < n_rings; r += blockDim.x)
    if (hist[r] != 0.0) atomicAdd(&sums[(int64_t)b * n_rings + r], hist[r]);
}

// dev = P - ring mean on rings with count > 1 (DC and singletons -> 0);
// loss[b] += sum dev^2; G = dev * X (for the gradient)   spectral.py:100-133
// mode 1 (rapsd): ssq[b][ring] += dev^2 over all rings (spectral.py:80-83)
__global__ void ring_dev_kernel(const double2 *__restrict__ X, int B, int HW,
                                const int32_t *__restrict__ ring,
                                const int32_t *__restrict__ counts, int n_rings,
                                const double *__restrict__ sums, int mode,
                                double *__restrict__ loss, double2 *__restrict__ G,
                                double *__restrict__ ssq) {
  const int b = blockIdx.y;
  const double inv = 1.0 / (double)HW;
  double acc = 0.0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < HW; i += gridDim.x * blockDim.x) {
    const int r = ring[i];
    const double2 v = X[(int64_t)b * HW + i];
    const double P = (v.x * v.x + v.y * v.y) * inv;
    double dev = 0.0;
    if (r >= 0) {
      const int cnt = counts[r];
      const double mean = sums[(int64_t)b * n_rings + r] / (double)cnt;
      if (mode == 0) {
        if (cnt > 1) dev = P - mean;
      } else {
        dev = P - mean;
        atomicAdd(&ssq[(int64_t)b * n_rings + r], dev * dev);
      }
    }
    if (mode == 0) {
      acc += dev * dev;
      if (G) G[(int64_t)b * HW + i] = make_double2(dev * v.x, dev * v.y);
    }
  }
  if (mode == 0) {
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0) atomicAdd(&loss[b], acc);
  }
}

// rapsd finalisation (spectral.py:80-88): power = sums/counts,
// anis = ssq / (power^2 (count-1)) where count > 1 and power > 0, else NaN
__global__ void rapsd_final_kernel(const double *__restrict__ sums, const double *__restrict__ ssq,
                                   const int32_t *__restrict__ counts, int B, int n_rings,
                                   const double2 *__restrict__ X, int HW,
                                   double *__restrict__ power, double *__restrict__ anis,
                                   double *__restrict__ dc) {
  const int64_t n = (int64_t)B * n_rings;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int r = (int)(i % n_rings);
    const int cnt = counts[r];
    const double pw = sums[i] / (double)cnt;
    power[i] = pw;
    anis[i] = (cnt > 1 && pw > 0.0) ? ssq[i] / (pw * pw * (double)(cnt - 1)) : nan("");
    if (r == 0) {
      const int64_t b = i / n_rings;
      const double2 v = X[b * HW];
      dc[b] = (v.x * v.x + v.y * v.y) / (double)HW;
    }
  }
}

struct SpecWs {
  double2 *twW, *twH, *Y, *X, *G;
  double *sums, *ssq;
};
static int64_t spec_ws_bytes(int B, int H, int W, int n_rings) {
  const int64_t n = (int64_t)B * H * W;
  return align256(16 * (int64_t)W) + align256(16 * (int64_t)H) + 3 * align256(16 * n) +
         2 * align256(8 * (int64_t)B * n_rings);
}
static SpecWs spec_ws(void *ws, int B, int H, int W, int n_rings) {
  char *p = (char *)ws;
  const int64_t n = (int64_t)B * H * W;
  SpecWs s;
  s.twW = (double2 *)p; p += align256(16 * (int64_t)W);
  s.twH = (double2 *)p; p += align256(16 * (int64_t)H);
  s.Y = (double2 *)p; p += align256(16 * n);
  s.X = (double2 *)p; p += align256(16 * n);
  s.G = (double2 *)p; p += align256(16 * n);
  s.sums = (double *)p; p += align256(8 * (int64_t)B * n_rings);
  s.ssq = (double *)p;
  return s;
}

static int forward_dft(const float *x, int B, int H, int W, const SpecWs &s, cudaStream_t st) {
  twiddle_kernel<<<(W + 255) / 256, 256, 0, st>>>(s.twW, W);
  twiddle_kernel<<<(H + 255) / 256, 256, 0, st>>>(s.twH, H);
  const int64_t n = (int64_t)B * H * W;
  const int grid = (int)((n + 255) / 256 < 8192 ? (n + 255) / 256 : 8192);
  dft_rows_real_kernel<<<grid, 256, 0, st>>>(x, B, H, W, s.twW, s.Y);
  dft_cols_kernel<<<grid, 256, 0, st>>>(s.Y, B, H, W, s.twH, 0, s.X);
  count_launch(4);
  HT_CHECK_LAUNCH();
  return HT_OK;
}

}  // namespace ht

extern "C" {

int ht_spectral_workspace_bytes(int B, int H, int W, int n_rings, int64_t *bytes) {
  *bytes = ht::spec_ws_bytes(B, H, W, n_rings);
  return HT_OK;
}

int ht_anisotropy(const float *x, int B, int H, int W, const int32_t *ring, const int32_t *counts,
                  int n_rings, double scale, double *loss, float *grad, void *ws, int64_t ws_bytes,
                  void *stream) {
  HT_REQUIRE(B >= 1 && H >= 1 && W >= 1 && n_rings >= 1, "empty input");
  HT_REQUIRE(ws_bytes >= ht::spec_ws_bytes(B, H, W, n_rings), "workspace too small");
  cudaStream_t st = (cudaStream_t)stream;
  ht::SpecWs s = ht::spec_ws(ws, B, H, W, n_rings);
  HT_CUDA(cudaMemsetAsync(s.sums, 0, sizeof(double) * B * n_rings, st));
  HT_CUDA(cudaMemsetAsync(loss, 0, sizeof(double) * B, st));
  int rc = ht::forward_dft(x, B, H, W, s, st);
  if (rc) return rc;
  const int HW = H * W;
  dim3 rg((HW + 255) / 256 < 64 ? (HW + 255) / 256 : 64, B);
  ht::ring_power_kernel<<<rg, 256, n_rings * sizeof(double), st>>>(s.X, B, HW, ring, n_rings,
                                                                      s.sums);
  ht::ring_dev_kernel<<<rg, 256, 0, st>>>(s.X, B, HW, ring, counts, n_rings, s.sums, 0, loss,
                                          grad ? s.G : nullptr, nullptr);
  ht::count_launch(2);
  HT_CHECK_LAUNCH();
  if (grad) {
    // grad = 4 Re(IFFT2(dev * X)) * scale; ifft2 carries 1/N (numpy)
    const int64_t n = (int64_t)B * H * W;
    const int grid = (int)((n + 255) / 256 < 8192 ? (n + 255) / 256 : 8192);
    ht::dft_cols_kernel<<<grid, 256, 0, st>>>(s.G, B, H, W, s.twH, 1, s.Y);
    ht::idft_rows_real_kernel<<<grid, 256, 0, st>>>(s.Y, B, H, W, s.twW, 4.0 * scale / (double)HW,
                                                    grad);
    ht::count_launch(2);
    HT_CHECK_LAUNCH();
  }
  return HT_OK;
}

int ht_rapsd(const float *x, int B, int H, int W, const int32_t *ring, const int32_t *counts,
             int n_rings, double *power, double *anis, double *dc, void *ws, int64_t ws_bytes,
             void *stream) {
  HT_REQUIRE(B >= 1 && H >= 1 && W >= 1 && n_rings >= 1, "empty input");
  HT_REQUIRE(ws_bytes >= ht::spec_ws_bytes(B, H, W, n_rings), "workspace too small");
  cudaStream_t st = (cudaStream_t)stream;
  ht::SpecWs s = ht::spec_ws(ws, B, H, W, n_rings);
  HT_CUDA(cudaMemsetAsync(s.sums, 0, sizeof(double) * B * n_rings, st));
  HT_CUDA(cudaMemsetAsync(s.ssq, 0, sizeof(double) * B * n_rings, st));
  int rc = ht::forward_dft(x, B, H, W, s, st);
  if (rc) return rc;
  const int HW = H * W;
  dim3 rg((HW + 255) / 256 < 64 ? (HW + 255) / 256 : 64, B);
  ht::ring_power_kernel<<<rg, 256, n_rings * sizeof(double), st>>>(s.X, B, HW, ring, n_rings,
                                                                      s.sums);
  ht::ring_dev_kernel<<<rg, 256, 0, st>>>(s.X, B, HW, ring, counts, n_rings, s.sums, 1, nullptr,
                                          nullptr, s.ssq);
  const int64_t nr = (int64_t)B * n_rings;
  ht::rapsd_final_kernel<<<(unsigned)((nr + 255) / 256), 256, 0, st>>>(
      s.sums, s.ssq, counts, B, n_rings, s.X, HW, power, anis, dc);
  ht::count_launch(3);
  HT_CHECK_LAUNCH();
  return HT_OK;
}

}  // extern "C"
