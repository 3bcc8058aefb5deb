// Shared helpers for the htb200 CUDA library: status/error plumbing and the
// parameter-vector geometry of PolicyNetwork (nn.py:106-122).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include <string>

#include "../../include/htb200.h"

namespace ht {

// thread-local last error message (ht_last_error)
void set_error(const char *fmt, ...);
int fail(int code, const char *fmt, ...);

#define HT_CUDA(call)                                                        \
  do {                                                                       \
    cudaError_t e_ = (call);                                                 \
    if (e_ != cudaSuccess)                                                   \
      return ::ht::fail(HT_E_CUDA, "%s failed: %s (%s:%d)", #call,           \
                        cudaGetErrorString(e_), __FILE__, __LINE__);         \
  } while (0)

#define HT_CHECK_LAUNCH()                                                    \
  do {                                                                       \
    cudaError_t e_ = cudaGetLastError();                                     \
    if (e_ != cudaSuccess)                                                   \
      return ::ht::fail(HT_E_CUDA, "kernel launch failed: %s (%s:%d)",       \
                        cudaGetErrorString(e_), __FILE__, __LINE__);         \
  } while (0)

#define HT_REQUIRE(cond, ...)                                                \
  do {                                                                       \
    if (!(cond)) return ::ht::fail(HT_E_INVALID, __VA_ARGS__);               \
  } while (0)

// per-thread launch counter (ht_last_launch_count)
void count_launch(int n = 1);
void reset_launches();

// optional per-launch CUDA-event timing (ht_timing_*): when enabled, the
// fused forward brackets every pass launch with events on its stream.
bool timing_enabled();
void timing_mark_begin(cudaStream_t st, int tag);
void timing_mark_end(cudaStream_t st);

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per (kernel, device):
// the attribute belongs to the device context, so a process driving several
// GPUs must set it on each of them.
int ensure_smem_attr(const void *kernel, int bytes);

// Host copy of a packed network's fp32 bias section (ht_pack_params writes it
// on the device).  The fused forward passes each pass's biases as kernel
// parameters, so concurrent forwards of different networks on different
// streams never share a mutable constant bank.  The copy is refreshed (wait
// for the event ht_pack_params recorded after its pack, then a 4 KB D2H) only
// after ht_pack_params rewrote the section.
int note_bias_pack(const void *tcb_dev, cudaStream_t st);
int host_biases(const float *tcb_dev, int64_t n, cudaStream_t st, const float **out);

// Offsets of the parameter tensors in the flat params() vector
// (nn.py:118-122): conv_in, then per block conv1 / conv2, then conv_out.
struct NetGeom {
  int C, NB;
  int64_t in_w, in_b;           // conv_in weight (C,2,3,3), bias (C)
  int64_t blk0;                 // start of block 0
  int64_t blk_stride;           // 2*(C*C*9 + C)
  int64_t out_w, out_b;         // conv_out weight (1,C,3,3), bias (1)
  int64_t total;
  __host__ __device__ NetGeom(int C_, int NB_) : C(C_), NB(NB_) {
    in_w = 0;
    in_b = (int64_t)C * 2 * 9;
    blk0 = in_b + C;
    blk_stride = 2 * ((int64_t)C * C * 9 + C);
    out_w = blk0 + blk_stride * NB;
    out_b = out_w + (int64_t)C * 9;
    total = out_b + 1;
  }
  __host__ __device__ int64_t w1(int b) const { return blk0 + blk_stride * b; }
  __host__ __device__ int64_t b1(int b) const { return w1(b) + (int64_t)C * C * 9; }
  __host__ __device__ int64_t w2(int b) const { return b1(b) + C; }
  __host__ __device__ int64_t b2(int b) const { return w2(b) + (int64_t)C * C * 9; }
};

// Packed device weight image (ht_pack_params).  All sections 256-B aligned.
//   f32     : fp32 copy of the flat params (SIMT forward, OIHW)
//   f32t    : per conv, transposed + spatially flipped fp32 weights
//             wt[ci][co][a][b] = w[co][ci][2-a][2-b] (dgrad as a forward conv)
//   tc      : fp16 UMMA operand tiles for the fused forward (fwd_tc.cu)
//   tcb     : fp32 biases for the fused forward
struct PackLayout {
  int64_t f32_off, f32t_off, tc_off, tcb_off, total;
};
PackLayout pack_layout(int C, int NB);

inline int64_t align256(int64_t x) { return (x + 255) & ~(int64_t)255; }

// Output level of a logit on the lattice i/steps (multitone.quantize_multitone,
// multitone.py:61-67: nearest level, half-steps round up).  steps = 1 is the
// binary rule h = (p >= 0.5) = (logit >= 0) of rl.infer_halftone (rl.py:311).
__device__ __forceinline__ uint8_t level_of(float logit, int steps) {
  if (steps == 1) return logit >= 0.f ? 1 : 0;
  const float v = 1.f / (1.f + expf(-logit));
  const float q = floorf(v * (float)steps + 0.5f);
  return (uint8_t)fminf(fmaxf(q, 0.f), (float)steps);
}

}  // namespace ht
