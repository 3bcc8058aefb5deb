// C-ABI plumbing: error strings, launch counting, device check and the
// bit-exact host RNG (imagecore.py:14-120) used for input preparation.
#include <math.h>
#include <stdarg.h>
#include <string.h>

#include <mutex>
#include <unordered_map>
#include <utility>
#include <vector>

#include "common.cuh"

namespace ht {

int ensure_smem_attr(const void *kernel, int bytes) {
  static std::mutex mu;
  static std::unordered_map<const void *, uint64_t> done;   // kernel -> device bit mask
  int dev = 0;
  HT_CUDA(cudaGetDevice(&dev));
  const uint64_t bit = 1ull << (dev & 63);
  std::lock_guard<std::mutex> lk(mu);
  uint64_t &mask = done[kernel];
  if (!(mask & bit)) {
    HT_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
    mask |= bit;
  }
  return HT_OK;
}

namespace {
struct BiasEntry {
  uint64_t gen = 0, seen = ~0ull;
  cudaEvent_t packed = nullptr;     // recorded on the packing stream
  std::vector<float> host;
};
std::mutex g_bias_mu;
std::unordered_map<const void *, BiasEntry> g_bias;
}  // namespace

int note_bias_pack(const void *tcb_dev, cudaStream_t st) {
  std::lock_guard<std::mutex> lk(g_bias_mu);
  BiasEntry &e = g_bias[tcb_dev];
  e.gen++;
  if (!e.packed) HT_CUDA(cudaEventCreateWithFlags(&e.packed, cudaEventDisableTiming));
  HT_CUDA(cudaEventRecord(e.packed, st));
  return HT_OK;
}

int host_biases(const float *tcb_dev, int64_t n, cudaStream_t st, const float **out) {
  (void)st;
  std::lock_guard<std::mutex> lk(g_bias_mu);
  BiasEntry &e = g_bias[tcb_dev];
  if (e.seen != e.gen || (int64_t)e.host.size() != n) {
    // after the pack that wrote them, whatever stream it ran on
    e.host.resize(n);
    if (e.packed) HT_CUDA(cudaEventSynchronize(e.packed));
    HT_CUDA(cudaMemcpy(e.host.data(), tcb_dev, sizeof(float) * n, cudaMemcpyDeviceToHost));
    e.seen = e.gen;
  }
  *out = e.host.data();
  return HT_OK;
}

static thread_local char g_err[1024] = "";
static thread_local int g_launches = 0;

void set_error(const char *fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

int fail(int code, const char *fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return code;
}

void count_launch(int n) { g_launches += n; }
void reset_launches() { g_launches = 0; }

struct TimedLaunch {
  cudaEvent_t a, b;
  int tag;
};
static thread_local bool g_timing = false;
static thread_local std::vector<TimedLaunch> g_timed;
static thread_local std::vector<cudaEvent_t> g_event_pool;

static cudaEvent_t pool_event() {
  if (!g_event_pool.empty()) {
    cudaEvent_t e = g_event_pool.back();
    g_event_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  cudaEventCreate(&e);
  return e;
}
bool timing_enabled() { return g_timing; }
void timing_mark_begin(cudaStream_t st, int tag) {
  if (!g_timing) return;
  TimedLaunch t{pool_event(), pool_event(), tag};
  cudaEventRecord(t.a, st);
  g_timed.push_back(t);
}
void timing_mark_end(cudaStream_t st) {
  if (!g_timing || g_timed.empty()) return;
  cudaEventRecord(g_timed.back().b, st);
}

int g_train_conv_impl = 0;
int g_wgrad_parts = 2;
extern int g_edge_conv_impl;
extern int g_train_bits;
extern int g_conv_tc2_pair;

// ---- xoshiro256++ / splitmix64 (imagecore.py:14-21, 52-64) -------------
static inline uint64_t splitmix64(uint64_t &s) {
  s += 0x9E3779B97F4A7C15ull;
  uint64_t z = s;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
static inline uint64_t rotl(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }
static inline uint64_t xoshiro_next(uint64_t *s) {
  const uint64_t out = rotl(s[0] + s[3], 23) + s[0];
  const uint64_t t = s[1] << 17;
  s[2] ^= s[0];
  s[3] ^= s[1];
  s[1] ^= s[2];
  s[0] ^= s[3];
  s[2] ^= t;
  s[3] = rotl(s[3], 45);
  return out;
}
static inline double to_unit(uint64_t x) { return (double)(x >> 11) * 0x1.0p-53; }

}  // namespace ht

extern "C" {

const char *ht_last_error(void) { return ht::g_err; }
int ht_version(void) { return 100; }

int ht_last_launch_count(int *count) {
  if (count) *count = ht::g_launches;
  return HT_OK;
}

// Per-launch event timing of the fused forward's pass kernels.
int ht_timing_enable(int on) {
  ht::g_timing = on != 0;
  return HT_OK;
}
// Pre-creates n event pairs for the timing hooks, so a timed region does not
// pay for event creation (the first timed step would otherwise).
int ht_timing_reserve(int n) {
  while ((int)ht::g_event_pool.size() < 2 * n) {
    cudaEvent_t e;
    HT_CUDA(cudaEventCreate(&e));
    ht::g_event_pool.push_back(e);
  }
  return HT_OK;
}
// Copies up to `max` (tag, milliseconds) pairs recorded since the last read
// (synchronises on the recorded events), then clears the record.
int ht_timing_read(int *tags, float *ms, int max, int *count) {
  int n = 0;
  for (auto &t : ht::g_timed) {
    if (n < max) {
      HT_CUDA(cudaEventSynchronize(t.b));
      float v = 0.f;
      HT_CUDA(cudaEventElapsedTime(&v, t.a, t.b));
      tags[n] = t.tag;
      ms[n] = v;
      ++n;
    }
    ht::g_event_pool.push_back(t.a);
    ht::g_event_pool.push_back(t.b);
  }
  ht::g_timed.clear();
  *count = n;
  return HT_OK;
}

// Training convolutions: 0 = tcgen05 kernels for the 32 -> 32 convs
// (default; scaled fp16 pairs where the shape allows TMA staging, split bf16
// otherwise), 1 = fp32 SIMT kernels only (cross-check), 2 = tcgen05 with the
// split-bf16 conv everywhere, 3 = same as 0.
int ht_set_train_conv_impl(int impl) {
  if (impl < 0 || impl > 3) return ht::fail(HT_E_INVALID, "impl must be 0 (tensor core), 1 (simt), 2 (split bf16) or 3 (fp16 pairs)");
  ht::g_train_conv_impl = impl;
  return HT_OK;
}

// Training conv v2 on CTA pairs (cta_group::2): 0 = off (default), 1 = on.
int ht_set_conv_pair(int on) {
  if (on != 0 && on != 1) return ht::fail(HT_E_INVALID, "on must be 0 or 1");
  ht::g_conv_tc2_pair = on;
  return HT_OK;
}

// Edge (conv_in / conv_out) weight gradients: 0 = warp-row kernel
// (default), 1 = the generic SIMT tile kernel (cross-check).
int ht_set_edge_conv_impl(int impl) {
  if (impl != 0 && impl != 1) return ht::fail(HT_E_INVALID, "impl must be 0 or 1");
  ht::g_edge_conv_impl = impl;
  return HT_OK;
}

int ht_set_train_bits(int on) {
  if (on != 0 && on != 1) return ht::fail(HT_E_INVALID, "on must be 0 or 1");
  ht::g_train_bits = on;
  return HT_OK;
}

int ht_set_wgrad_parts(int parts) {
  if (parts != 2 && parts != 3) return ht::fail(HT_E_INVALID, "parts must be 2 or 3");
  ht::g_wgrad_parts = parts;
  return HT_OK;
}

int ht_device_supported(int device, int *supported) {
  cudaDeviceProp prop;
  HT_CUDA(cudaGetDeviceProperties(&prop, device));
  *supported = (prop.major == 10 && prop.minor == 0) ? 1 : 0;
  return HT_OK;
}

// Rng.__init__ (imagecore.py:43-50): four splitmix64 outputs.
int ht_rng_seed(uint64_t seed, uint64_t state[4]) {
  uint64_t s = seed;
  for (int i = 0; i < 4; ++i) state[i] = ht::splitmix64(s);
  return HT_OK;
}

// Rng.uniforms (imagecore.py:70-86): (x >> 11) * 2^-53, row-major.
int ht_rng_uniforms(uint64_t state[4], int64_t n, double *out) {
  if (n < 0) return ht::fail(HT_E_INVALID, "n must be non-negative");
  for (int64_t i = 0; i < n; ++i) out[i] = ht::to_unit(ht::xoshiro_next(state));
  return HT_OK;
}

}  // extern "C"

// Rng.gaussians (imagecore.py:88-99): Box-Muller on consumed pairs
// (u1 = 1 - u_even, u2 = u_odd), r cos / r sin interleaved; odd n burns
// the last sine.
template <typename T>
static int gaussians_impl(uint64_t state[4], int64_t n, T *out) {
  if (n < 0) return ht::fail(HT_E_INVALID, "n must be non-negative");
  const double two_pi = 2.0 * M_PI;
  for (int64_t i = 0; i < n; i += 2) {
    const double u0 = ht::to_unit(ht::xoshiro_next(state));
    const double u1 = ht::to_unit(ht::xoshiro_next(state));
    const double r = sqrt(-2.0 * log(1.0 - u0));
    const double th = two_pi * u1;
    out[i] = (T)(r * cos(th));
    if (i + 1 < n) out[i + 1] = (T)(r * sin(th));
  }
  return HT_OK;
}

extern "C" {
int ht_rng_gaussians(uint64_t state[4], int64_t n, double *out) {
  return gaussians_impl<double>(state, n, out);
}
int ht_rng_gaussians_f32(uint64_t state[4], int64_t n, float *out) {
  return gaussians_impl<float>(state, n, out);
}

int ht_num_params(int channels, int blocks, int64_t *n) {
  if (channels < 1 || blocks < 0)
    return ht::fail(HT_E_INVALID, "channels must be positive and blocks non-negative");
  *n = ht::NetGeom(channels, blocks).total;
  return HT_OK;
}

}  // extern "C"
