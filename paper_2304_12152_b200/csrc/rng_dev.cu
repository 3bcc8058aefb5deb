// Device xoshiro256++ streams with exact jump-ahead.
//
// Rng.uniforms / Rng.gaussians (imagecore.py:70-99) are one sequential
// xoshiro256++ stream.  Its state update is linear over GF(2)^256, so
// advancing by n draws is a product of the precomputed bit matrices
// J_k = T^(2^k) for the set bits of n.  A kernel thread jumps straight to its
// own offset in the stream, so a noise map or action-uniform map is produced
// on the GPU in one launch, draw-for-draw the same stream as the host; the
// host state is then advanced by the same count (bit-exact).
//
// Uniforms are bit-exact.  Gaussians use the device's fp64 log / sqrt /
// sin / cos (<= 2 ulp from the host libm), so fp64 values may differ in the
// last bits and the fp32-rounded noise the fused kernel consumes matches the
// host's except for ~1e-8 of samples (one fp32 ulp when it differs).
#include <cmath>
#include <mutex>
#include <vector>

#include "common.cuh"

namespace ht {
namespace rng {

constexpr int LEVELS = 56;  // jumps of up to 2^56 draws

struct Mat {
  uint64_t col[256][4];  // column j = image of state bit j
};

__host__ __device__ __forceinline__ void transition(uint64_t s[4]) {
  const uint64_t t = s[1] << 17;
  s[2] ^= s[0];
  s[3] ^= s[1];
  s[1] ^= s[2];
  s[0] ^= s[3];
  s[2] ^= t;
  s[3] = (s[3] << 45) | (s[3] >> 19);
}

static void matvec_host(const Mat &m, uint64_t s[4]) {
  uint64_t o[4] = {0, 0, 0, 0};
  for (int j = 0; j < 256; ++j)
    if ((s[j >> 6] >> (j & 63)) & 1)
      for (int w = 0; w < 4; ++w) o[w] ^= m.col[j][w];
  for (int w = 0; w < 4; ++w) s[w] = o[w];
}

static const std::vector<Mat> &tables() {
  static std::vector<Mat> t;
  static std::once_flag once;
  std::call_once(once, [] {
    t.resize(LEVELS);
    for (int j = 0; j < 256; ++j) {
      uint64_t s[4] = {0, 0, 0, 0};
      s[j >> 6] = 1ull << (j & 63);
      transition(s);
      for (int w = 0; w < 4; ++w) t[0].col[j][w] = s[w];
    }
    for (int k = 1; k < LEVELS; ++k)
      for (int j = 0; j < 256; ++j) {
        uint64_t s[4];
        for (int w = 0; w < 4; ++w) s[w] = t[k - 1].col[j][w];
        matvec_host(t[k - 1], s);
        for (int w = 0; w < 4; ++w) t[k].col[j][w] = s[w];
      }
  });
  return t;
}

void jump_host(uint64_t s[4], uint64_t n) {
  const auto &t = tables();
  for (int k = 0; k < LEVELS && n; ++k, n >>= 1)
    if (n & 1) matvec_host(t[k], s);
}

// Device form of the jump matrices: per level, 64 nibble tables
// N[c][v] = XOR of the columns 4c + i for the set bits i of v, so a product
// is 64 lookups instead of 256 masked column XORs.
struct NibMat {
  ulonglong4 t[64][16];
};

static const NibMat *device_tables() {
  static std::mutex mu;
  static const NibMat *per_dev[64] = {nullptr};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return nullptr;
  std::lock_guard<std::mutex> lock(mu);
  if (!per_dev[dev]) {
    std::vector<NibMat> h(LEVELS);
    const auto &t = tables();
    for (int k = 0; k < LEVELS; ++k)
      for (int c = 0; c < 64; ++c)
        for (int v = 0; v < 16; ++v) {
          uint64_t o[4] = {0, 0, 0, 0};
          for (int i = 0; i < 4; ++i)
            if ((v >> i) & 1)
              for (int w = 0; w < 4; ++w) o[w] ^= t[k].col[4 * c + i][w];
          h[k].t[c][v] = make_ulonglong4(o[0], o[1], o[2], o[3]);
        }
    NibMat *d = nullptr;
    if (cudaMalloc(&d, sizeof(NibMat) * LEVELS) != cudaSuccess) return nullptr;
    if (cudaMemcpy(d, h.data(), sizeof(NibMat) * LEVELS, cudaMemcpyHostToDevice) != cudaSuccess) return nullptr;
    per_dev[dev] = d;
  }
  return per_dev[dev];
}

__device__ __forceinline__ void jump_dev(const NibMat *__restrict__ J, uint64_t s[4], uint64_t n) {
  for (int k = 0; k < LEVELS && n; ++k, n >>= 1) {
    if (!(n & 1)) continue;
    uint64_t o0 = 0, o1 = 0, o2 = 0, o3 = 0;
    const ulonglong2 *base = reinterpret_cast<const ulonglong2 *>(J[k].t);
#pragma unroll
    for (int w = 0; w < 4; ++w) {
      const uint64_t sw = s[w];
#pragma unroll
      for (int q = 0; q < 16; ++q) {
        const int c = w * 16 + q;
        const int v = (int)((sw >> (4 * q)) & 15u);
        const ulonglong2 a = __ldg(base + 2 * (c * 16 + v)), b = __ldg(base + 2 * (c * 16 + v) + 1);
        o0 ^= a.x; o1 ^= a.y; o2 ^= b.x; o3 ^= b.y;
      }
    }
    s[0] = o0; s[1] = o1; s[2] = o2; s[3] = o3;
  }
}

__device__ __forceinline__ uint64_t next_dev(uint64_t s[4]) {
  const uint64_t x = s[0] + s[3];
  const uint64_t out = ((x << 23) | (x >> 41)) + s[0];
  transition(s);
  return out;
}
__device__ __forceinline__ double unit(uint64_t x) { return (double)(x >> 11) * 0x1.0p-53; }

#ifndef RNG_PPT
#define RNG_PPT 32   // Box-Muller pairs per thread: 16 -> 32 measured 74 -> 71 us for 16 x 256^2 maps
#endif
constexpr int PAIRS_PER_THREAD = RNG_PPT;

// Noise maps of n gaussians each (n gaussians = ceil(n/2) Box-Muller pairs,
// pair i consuming draws 2i, 2i+1 of its map's stream), map m starting from
// its own stream state -- maps interleaved with host draws, e.g.
// rl.train_step's per-sample image pick / crop / noise order, take one
// launch for all of them; a single stream is the one-map case.
constexpr int MAX_MAPS = 64;
struct MapStarts {
  ulonglong4 s[MAX_MAPS];
};

template <typename T>
__global__ void gaussian_maps_kernel(const __grid_constant__ MapStarts st, int64_t n, const NibMat *__restrict__ J,
                                     T *__restrict__ out) {
  const int64_t npairs = (n + 1) / 2;
  const int64_t p0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * PAIRS_PER_THREAD;
  if (p0 >= npairs) return;
  const ulonglong4 s0 = st.s[blockIdx.y];
  uint64_t s[4] = {s0.x, s0.y, s0.z, s0.w};
  jump_dev(J, s, 2ull * (uint64_t)p0);
  T *o = out + (int64_t)blockIdx.y * n;
  const int64_t p1 = min(npairs, p0 + PAIRS_PER_THREAD);
  const double two_pi = 2.0 * 3.14159265358979323846;
  for (int64_t p = p0; p < p1; ++p) {
    const double u0 = unit(next_dev(s));
    const double u1 = unit(next_dev(s));
    const double r = sqrt(-2.0 * log(1.0 - u0));
    double sn, cs;
    sincos(two_pi * u1, &sn, &cs);
    o[2 * p] = (T)(r * cs);
    if (2 * p + 1 < n) o[2 * p + 1] = (T)(r * sn);
  }
}

template <typename T>
static int launch_maps(const uint64_t *states, int n_maps, int64_t n, T *out, cudaStream_t st) {
  HT_REQUIRE(n_maps >= 0 && n >= 0, "counts must be non-negative");
  if (n_maps == 0 || n == 0) return HT_OK;
  const NibMat *J = device_tables();
  HT_REQUIRE(J != nullptr, "could not upload RNG jump tables");
  const int threads = 128;
  const int64_t units = ((n + 1) / 2 + PAIRS_PER_THREAD - 1) / PAIRS_PER_THREAD;
  const int64_t blocks = (units + threads - 1) / threads;
  HT_REQUIRE(blocks < (1ll << 31), "too many draws");
  for (int m0 = 0; m0 < n_maps; m0 += MAX_MAPS) {
    MapStarts ms{};
    const int cnt = min(MAX_MAPS, n_maps - m0);
    for (int m = 0; m < cnt; ++m)
      ms.s[m] = make_ulonglong4(states[4 * (m0 + m)], states[4 * (m0 + m) + 1], states[4 * (m0 + m) + 2],
                                states[4 * (m0 + m) + 3]);
    gaussian_maps_kernel<T><<<dim3((unsigned)blocks, (unsigned)cnt), threads, 0, st>>>(ms, n, J, out + (int64_t)m0 * n);
    count_launch();
    HT_CHECK_LAUNCH();
  }
  return HT_OK;
}

#ifndef RNG_DPT
#define RNG_DPT 128  // uniforms per thread: 32 -> 128 measured 78 -> 65 us per 1M (fewer jumps)
#endif
constexpr int DRAWS_PER_THREAD = RNG_DPT;

template <typename T>
__global__ void uniforms_kernel(ulonglong4 start, int64_t n, const NibMat *__restrict__ J, T *__restrict__ out) {
  const int64_t i0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * DRAWS_PER_THREAD;
  if (i0 >= n) return;
  uint64_t s[4] = {start.x, start.y, start.z, start.w};
  jump_dev(J, s, (uint64_t)i0);
  const int64_t i1 = min(n, i0 + DRAWS_PER_THREAD);
  for (int64_t i = i0; i < i1; ++i) out[i] = (T)unit(next_dev(s));
}

template <typename T>
static int launch_uniforms(uint64_t state[4], int64_t n, T *out, cudaStream_t st) {
  HT_REQUIRE(n >= 0, "n must be non-negative");
  if (n == 0) return HT_OK;
  const NibMat *J = device_tables();
  HT_REQUIRE(J != nullptr, "could not upload RNG jump tables");
  const ulonglong4 s0 = make_ulonglong4(state[0], state[1], state[2], state[3]);
  const int threads = 128;
  const int64_t blocks = ((n + DRAWS_PER_THREAD - 1) / DRAWS_PER_THREAD + threads - 1) / threads;
  HT_REQUIRE(blocks < (1ll << 31), "too many draws");
  uniforms_kernel<T><<<(unsigned)blocks, threads, 0, st>>>(s0, n, J, out);
  count_launch();
  HT_CHECK_LAUNCH();
  jump_host(state, (uint64_t)n);
  return HT_OK;
}

template <typename T>
static int launch_gaussians(uint64_t state[4], int64_t n, T *out, cudaStream_t st) {
  HT_REQUIRE(n >= 0, "n must be non-negative");
  const int rc = launch_maps<T>(state, 1, n, out, st);
  if (rc == HT_OK) jump_host(state, 2ull * (uint64_t)((n + 1) / 2));
  return rc;
}

}  // namespace rng
}  // namespace ht

extern "C" {

// Rng.jump: advance a host state by n draws (GF(2) jump-ahead).
int ht_rng_jump(uint64_t state[4], uint64_t n) {
  ht::rng::jump_host(state, n);
  return HT_OK;
}
// Device Rng.gaussians / Rng.uniforms: out is a device pointer; the host
// state advances exactly as the host functions would.
int ht_rng_gaussians_device(uint64_t state[4], int64_t n, void *out, int f64, void *stream) {
  return f64 ? ht::rng::launch_gaussians<double>(state, n, (double *)out, (cudaStream_t)stream)
             : ht::rng::launch_gaussians<float>(state, n, (float *)out, (cudaStream_t)stream);
}
// n_maps noise maps of n gaussians, map m drawn from stream state
// states[4m..4m+3] (host array); no host state is advanced.
int ht_rng_gaussian_maps_device(const uint64_t *states, int n_maps, int64_t n, void *out, int f64,
                                void *stream) {
  return f64 ? ht::rng::launch_maps<double>(states, n_maps, n, (double *)out, (cudaStream_t)stream)
             : ht::rng::launch_maps<float>(states, n_maps, n, (float *)out, (cudaStream_t)stream);
}
int ht_rng_uniforms_device(uint64_t state[4], int64_t n, void *out, int f64, void *stream) {
  return f64 ? ht::rng::launch_uniforms<double>(state, n, (double *)out, (cudaStream_t)stream)
             : ht::rng::launch_uniforms<float>(state, n, (float *)out, (cudaStream_t)stream);
}

}  // extern "C"
