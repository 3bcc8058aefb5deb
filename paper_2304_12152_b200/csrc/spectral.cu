// K5 / K7: periodogram, ring statistics, anisotropy loss and its gradient,
// fp64 (complex128 like numpy.fft).
//
// Reference: periodogram (spectral.py:17-24), ring partition (39-55),
// _ring_sums / rapsd (67-88), _loss_pieces / anisotropy_loss /
// anisotropy_loss_backward (100-133).  The 2-D DFTs are batched cuFFT Z2Z
// transforms (library FFT, as numpy uses pocketfft; plans cached per
// (device, B, H, W)); the ring reductions, deviations and the gradient's
// real-part epilogue are the kernels below.  Inputs may be float32 (the
// training path's probability maps) or float64 (the drop-in API keeps the
// reference's float64 arrays float64).
#include <cufft.h>
#include <math.h>

#include <mutex>
#include <tuple>
#include <map>

#include "common.cuh"

namespace ht {

// real input -> complex128 (the FFT operand)
template <typename T>
__global__ void to_complex_kernel(const T *__restrict__ x, int64_t n, double2 *__restrict__ X) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    X[i] = make_double2((double)x[i], 0.0);
}

// out = scale * Re(Y) (inverse transform epilogue; cuFFT is unnormalised)
template <typename T>
__global__ void real_part_kernel(const double2 *__restrict__ Y, int64_t n, double scale, T *__restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = (T)(scale * Y[i].x);
}

// P = |X|^2 / N (periodogram, spectral.py:23-24)
__global__ void power_kernel(const double2 *__restrict__ X, int64_t n, double inv, double *__restrict__ P) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double2 v = X[i];
    P[i] = (v.x * v.x + v.y * v.y) * inv;
  }
}

// The spectrum is given either as X (complex, P = |X|^2/N) or as P itself.
struct Spec {
  const double2 *X;
  const double *P;
  double inv;
  __device__ __forceinline__ double power(int64_t i) const {
    if (P) return P[i];
    const double2 v = X[i];
    return (v.x * v.x + v.y * v.y) * inv;
  }
};

// ring sums of P per image: sums[b][ring] (spectral.py:67-71)
__global__ void ring_power_kernel(Spec S, int B, int HW, const int32_t *__restrict__ ring, int n_rings,
                                  double *__restrict__ sums) {
  extern __shared__ double hist[];
  const int b = blockIdx.y;
  for (int r = threadIdx.x; r < n_rings; r += blockDim.x) hist[r] = 0.0;
  __syncthreads();
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < HW; i += gridDim.x * blockDim.x) {
    const int r = ring[i];
    if (r < 0) continue;
    atomicAdd(&hist[r], S.power((int64_t)b * HW + i));
  }
  __syncthreads();
  for (int r = threadIdx.x; r < n_rings; r += blockDim.x)
    if (hist[r] != 0.0) atomicAdd(&sums[(int64_t)b * n_rings + r], hist[r]);
}

// dev = P - ring mean on rings with count > 1 (DC and singletons -> 0);
// loss[b] += sum dev^2; G = dev * X (for the gradient)   spectral.py:100-133
// mode 1 (rapsd): ssq[b][ring] += dev^2 over all rings (spectral.py:80-83)
__global__ void ring_dev_kernel(Spec S, int B, int HW, const int32_t *__restrict__ ring,
                                const int32_t *__restrict__ counts, int n_rings,
                                const double *__restrict__ sums, int mode, double *__restrict__ loss,
                                double2 *__restrict__ G, double *__restrict__ ssq) {
  const int b = blockIdx.y;
  double acc = 0.0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < HW; i += gridDim.x * blockDim.x) {
    const int r = ring[i];
    const int64_t gi = (int64_t)b * HW + i;
    const double P = S.power(gi);
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
      if (G) {
        const double2 v = S.X[gi];
        G[gi] = make_double2(dev * v.x, dev * v.y);
      }
    }
  }
  if (mode == 0) {
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0) atomicAdd(&loss[b], acc);
  }
}

// rapsd finalisation (spectral.py:80-88): power = sums/counts,
// anis = ssq / (power^2 (count-1)) where count > 1 and power > 0, else NaN,
// dc = P[0, 0]
__global__ void rapsd_final_kernel(const double *__restrict__ sums, const double *__restrict__ ssq,
                                   const int32_t *__restrict__ counts, int B, int n_rings, Spec S, int HW,
                                   double *__restrict__ power, double *__restrict__ anis,
                                   double *__restrict__ dc) {
  const int64_t n = (int64_t)B * n_rings;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int r = (int)(i % n_rings);
    const int cnt = counts[r];
    const double pw = sums[i] / (double)cnt;
    power[i] = pw;
    anis[i] = (cnt > 1 && pw > 0.0) ? ssq[i] / (pw * pw * (double)(cnt - 1)) : nan("");
    if (r == 0) {
      const int64_t b = i / n_rings;
      dc[b] = S.power(b * HW);
    }
  }
}

struct SpecWs {
  double2 *X, *G;
  double *sums, *ssq;
};
static int64_t spec_ws_bytes(int B, int H, int W, int n_rings) {
  const int64_t n = (int64_t)B * H * W;
  return 2 * align256(16 * n) + 2 * align256(8 * (int64_t)B * (n_rings > 0 ? n_rings : 1));
}
static SpecWs spec_ws(void *ws, int B, int H, int W, int n_rings) {
  char *p = (char *)ws;
  const int64_t n = (int64_t)B * H * W;
  SpecWs s;
  s.X = (double2 *)p; p += align256(16 * n);
  s.G = (double2 *)p; p += align256(16 * n);
  s.sums = (double *)p; p += align256(8 * (int64_t)B * (n_rings > 0 ? n_rings : 1));
  s.ssq = (double *)p;
  return s;
}

static int grid_of(int64_t n) { return (int)((n + 255) / 256 < 8192 ? (n + 255) / 256 : 8192); }

// batched 2-D Z2Z plan for (B, H, W) on the current device (cached)
static int fft_plan(int B, int H, int W, cudaStream_t st, cufftHandle *out) {
  static std::mutex mu;
  static std::map<std::tuple<int, int, int, int>, cufftHandle> plans;
  int dev = 0;
  HT_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(mu);
  auto key = std::make_tuple(dev, B, H, W);
  auto it = plans.find(key);
  cufftHandle h;
  if (it == plans.end()) {
    int dims[2] = {H, W};
    if (cufftPlanMany(&h, 2, dims, nullptr, 1, H * W, nullptr, 1, H * W, CUFFT_Z2Z, B) != CUFFT_SUCCESS)
      return fail(HT_E_CUDA, "cufftPlanMany(%d x %d, batch %d) failed", H, W, B);
    plans[key] = h;
  } else {
    h = it->second;
  }
  if (cufftSetStream(h, st) != CUFFT_SUCCESS) return fail(HT_E_CUDA, "cufftSetStream failed");
  *out = h;
  return HT_OK;
}

// X = FFT2(x) for B real images
template <typename T>
static int forward_fft(const T *x, int B, int H, int W, double2 *X, cudaStream_t st) {
  const int64_t n = (int64_t)B * H * W;
  to_complex_kernel<T><<<grid_of(n), 256, 0, st>>>(x, n, X);
  count_launch();
  HT_CHECK_LAUNCH();
  cufftHandle h;
  if (int rc = fft_plan(B, H, W, st, &h)) return rc;
  if (cufftExecZ2Z(h, (cufftDoubleComplex *)X, (cufftDoubleComplex *)X, CUFFT_FORWARD) != CUFFT_SUCCESS)
    return fail(HT_E_CUDA, "cufftExecZ2Z (forward) failed");
  return HT_OK;
}

template <typename T>
static int anisotropy(const T *x, int B, int H, int W, const int32_t *ring, const int32_t *counts, int n_rings,
                      double scale, double *loss, T *grad, void *ws, int64_t ws_bytes, cudaStream_t st) {
  HT_REQUIRE(B >= 1 && H >= 1 && W >= 1 && n_rings >= 1, "empty input");
  HT_REQUIRE(ws_bytes >= spec_ws_bytes(B, H, W, n_rings), "workspace too small");
  SpecWs s = spec_ws(ws, B, H, W, n_rings);
  HT_CUDA(cudaMemsetAsync(s.sums, 0, sizeof(double) * B * n_rings, st));
  HT_CUDA(cudaMemsetAsync(loss, 0, sizeof(double) * B, st));
  if (int rc = forward_fft(x, B, H, W, s.X, st)) return rc;
  const int HW = H * W;
  const Spec S{s.X, nullptr, 1.0 / (double)HW};
  dim3 rg((HW + 255) / 256 < 64 ? (HW + 255) / 256 : 64, B);
  ring_power_kernel<<<rg, 256, n_rings * sizeof(double), st>>>(S, B, HW, ring, n_rings, s.sums);
  ring_dev_kernel<<<rg, 256, 0, st>>>(S, B, HW, ring, counts, n_rings, s.sums, 0, loss, grad ? s.G : nullptr,
                                      nullptr);
  count_launch(2);
  HT_CHECK_LAUNCH();
  if (grad) {
    // grad = 4 Re(IFFT2(dev * X)) * scale; numpy's ifft2 carries the 1/N
    cufftHandle h;
    if (int rc = fft_plan(B, H, W, st, &h)) return rc;
    if (cufftExecZ2Z(h, (cufftDoubleComplex *)s.G, (cufftDoubleComplex *)s.G, CUFFT_INVERSE) != CUFFT_SUCCESS)
      return fail(HT_E_CUDA, "cufftExecZ2Z (inverse) failed");
    const int64_t n = (int64_t)B * HW;
    real_part_kernel<T><<<grid_of(n), 256, 0, st>>>(s.G, n, 4.0 * scale / (double)HW, grad);
    count_launch();
    HT_CHECK_LAUNCH();
  }
  return HT_OK;
}

// rapsd of the spectrum S (spectral.py:74-88)
static int rapsd_of(const Spec &S, int B, int HW, const int32_t *ring, const int32_t *counts, int n_rings,
                    double *power, double *anis, double *dc, const SpecWs &s, cudaStream_t st) {
  HT_CUDA(cudaMemsetAsync(s.sums, 0, sizeof(double) * B * n_rings, st));
  HT_CUDA(cudaMemsetAsync(s.ssq, 0, sizeof(double) * B * n_rings, st));
  dim3 rg((HW + 255) / 256 < 64 ? (HW + 255) / 256 : 64, B);
  ring_power_kernel<<<rg, 256, n_rings * sizeof(double), st>>>(S, B, HW, ring, n_rings, s.sums);
  ring_dev_kernel<<<rg, 256, 0, st>>>(S, B, HW, ring, counts, n_rings, s.sums, 1, nullptr, nullptr, s.ssq);
  const int64_t nr = (int64_t)B * n_rings;
  rapsd_final_kernel<<<(unsigned)((nr + 255) / 256), 256, 0, st>>>(s.sums, s.ssq, counts, B, n_rings, S, HW,
                                                                    power, anis, dc);
  count_launch(3);
  HT_CHECK_LAUNCH();
  return HT_OK;
}

template <typename T>
static int rapsd(const T *x, int B, int H, int W, const int32_t *ring, const int32_t *counts, int n_rings,
                 double *power, double *anis, double *dc, void *ws, int64_t ws_bytes, cudaStream_t st) {
  HT_REQUIRE(B >= 1 && H >= 1 && W >= 1 && n_rings >= 1, "empty input");
  HT_REQUIRE(ws_bytes >= spec_ws_bytes(B, H, W, n_rings), "workspace too small");
  SpecWs s = spec_ws(ws, B, H, W, n_rings);
  if (int rc = forward_fft(x, B, H, W, s.X, st)) return rc;
  const Spec S{s.X, nullptr, 1.0 / (double)(H * W)};
  return rapsd_of(S, B, H * W, ring, counts, n_rings, power, anis, dc, s, st);
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
  return ht::anisotropy<float>(x, B, H, W, ring, counts, n_rings, scale, loss, grad, ws, ws_bytes,
                               (cudaStream_t)stream);
}

int ht_anisotropy_f64(const double *x, int B, int H, int W, const int32_t *ring, const int32_t *counts,
                      int n_rings, double scale, double *loss, double *grad, void *ws, int64_t ws_bytes,
                      void *stream) {
  return ht::anisotropy<double>(x, B, H, W, ring, counts, n_rings, scale, loss, grad, ws, ws_bytes,
                                (cudaStream_t)stream);
}

int ht_rapsd(const float *x, int B, int H, int W, const int32_t *ring, const int32_t *counts,
             int n_rings, double *power, double *anis, double *dc, void *ws, int64_t ws_bytes,
             void *stream) {
  return ht::rapsd<float>(x, B, H, W, ring, counts, n_rings, power, anis, dc, ws, ws_bytes,
                          (cudaStream_t)stream);
}

int ht_rapsd_f64(const double *x, int B, int H, int W, const int32_t *ring, const int32_t *counts,
                 int n_rings, double *power, double *anis, double *dc, void *ws, int64_t ws_bytes,
                 void *stream) {
  return ht::rapsd<double>(x, B, H, W, ring, counts, n_rings, power, anis, dc, ws, ws_bytes,
                           (cudaStream_t)stream);
}

int ht_periodogram_f64(const double *x, int B, int H, int W, double *P, void *ws, int64_t ws_bytes,
                       void *stream) {
  HT_REQUIRE(B >= 1 && H >= 1 && W >= 1, "empty input");
  HT_REQUIRE(ws_bytes >= ht::spec_ws_bytes(B, H, W, 1), "workspace too small");
  cudaStream_t st = (cudaStream_t)stream;
  ht::SpecWs s = ht::spec_ws(ws, B, H, W, 1);
  if (int rc = ht::forward_fft(x, B, H, W, s.X, st)) return rc;
  const int64_t n = (int64_t)B * H * W;
  ht::power_kernel<<<ht::grid_of(n), 256, 0, st>>>(s.X, n, 1.0 / (double)(H * W), P);
  ht::count_launch();
  HT_CHECK_LAUNCH();
  return HT_OK;
}

int ht_rapsd_power_f64(const double *P, int B, int H, int W, const int32_t *ring, const int32_t *counts,
                       int n_rings, double *power, double *anis, double *dc, void *ws, int64_t ws_bytes,
                       void *stream) {
  HT_REQUIRE(B >= 1 && H >= 1 && W >= 1 && n_rings >= 1, "empty input");
  HT_REQUIRE(ws_bytes >= ht::spec_ws_bytes(B, H, W, n_rings), "workspace too small");
  ht::SpecWs s = ht::spec_ws(ws, B, H, W, n_rings);
  const ht::Spec S{nullptr, P, 0.0};
  return ht::rapsd_of(S, B, H * W, ring, counts, n_rings, power, anis, dc, s, (cudaStream_t)stream);
}

}  // extern "C"
