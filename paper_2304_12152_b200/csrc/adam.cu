// K6: Adam.step (nn.py:175-186) over the flat float64 parameter vector, and
// the bin_gap reduction of rl.train_step (rl.py:255).
#include "common.cuh"

namespace ht {

__global__ void adam_kernel(double *__restrict__ p, const double *__restrict__ g,
                            double *__restrict__ m, double *__restrict__ v, int64_t n, double lr,
                            double b1, double b2, double eps, double c1, double c2) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double gi = g[i];
    const double mi = b1 * m[i] + (1.0 - b1) * gi;
    const double vi = b2 * v[i] + (1.0 - b2) * (gi * gi);
    m[i] = mi;
    v[i] = vi;
    p[i] -= lr * (mi / c1) / (sqrt(vi / c2) + eps);
  }
}

__global__ void bin_gap_kernel(const float *__restrict__ p, int64_t n, double *__restrict__ out) {
  double s = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double q = p[i];
    s += fabs(q - rint(q));
  }
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  __shared__ double red[32];
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x < 32) {
    s = threadIdx.x < blockDim.x / 32 ? red[threadIdx.x] : 0.0;
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (threadIdx.x == 0) atomicAdd(out, s);
  }
}

}  // namespace ht

extern "C" {

int ht_adam_step(double *params, const double *grad, double *m, double *v, int64_t n, int t,
                 double lr, double b1, double b2, double eps, void *stream) {
  HT_REQUIRE(n >= 0 && t >= 1, "bad Adam arguments (n=%lld, t=%d)", (long long)n, t);
  const double c1 = 1.0 - pow(b1, (double)t);
  const double c2 = 1.0 - pow(b2, (double)t);
  const int grid = (int)((n + 255) / 256 < 1184 ? (n + 255) / 256 : 1184);
  if (n == 0) return HT_OK;
  ht::adam_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(params, grad, m, v, n, lr, b1, b2, eps, c1,
                                                          c2);
  ht::count_launch();
  HT_CHECK_LAUNCH();
  return HT_OK;
}

int ht_bin_gap_sum(const float *p, int64_t n, double *out, void *stream) {
  if (n <= 0) return HT_OK;
  const int grid = (int)((n + 255) / 256 < 592 ? (n + 255) / 256 : 592);
  ht::bin_gap_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(p, n, out);
  ht::count_launch();
  HT_CHECK_LAUNCH();
  return HT_OK;
}

}  // extern "C"
