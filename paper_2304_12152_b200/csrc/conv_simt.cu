// FP32 SIMT convolution kernels: the training forward (activations kept for
// backward), the backward (dgrad + wgrad), and the reference-precision
// inference cross-check path (ht_halftone impl=1).
//
// Reference semantics: Conv2d.forward/backward (nn.py:46-77) -- 3x3
// cross-correlation, stride 1, zero padding 1 applied to EVERY layer's input;
// ResidualBlock (nn.py:91-100); PolicyNetwork (nn.py:138-160).  Tensors are
// NCHW float32; gradients accumulate into a flat float64 vector in
// params() order.
#include <mutex>
#include <set>
#include <math.h>

#include <vector>

#include "common.cuh"

namespace ht {

// ---------------------------------------------------------------------------
// forward conv: out[b,co,y,x] = epi( bias[co] + sum_{ci,ky,kx}
//                 x[b,ci,y+ky-1,x+kx-1] * w[co,ci,ky,kx] )
// epi: mask-multiply (mask>0), residual add, relu -- in that order.  With
// w = transposed+flipped weights and no bias this is the dgrad.
constexpr int FT_X = 32, FT_Y = 8, F_CHUNK = 8;

template <int CIN, int COUT>
__global__ void __launch_bounds__(128)
conv3x3_fwd_kernel(const float *__restrict__ x, int H, int W,
                   const float *__restrict__ w, const float *__restrict__ bias,
                   const float *__restrict__ mask, const float *__restrict__ resid,
                   float *__restrict__ out, int relu) {
  constexpr int CC = CIN < F_CHUNK ? CIN : F_CHUNK;
  constexpr int TXP = FT_X + 2, TYP = FT_Y + 2;
  __shared__ float ws[CIN * 9 * COUT];       // [ci][ky][kx][co]
  __shared__ float xs[CC][TYP][TXP + 1];
  const int b = blockIdx.z;
  const int x0 = blockIdx.x * FT_X, y0 = blockIdx.y * FT_Y;
  const int tid = threadIdx.x;
  const int tx = (tid % 16) * 2, ty = tid / 16;  // 2 pixels per thread
  for (int i = tid; i < CIN * 9 * COUT; i += 128) {
    const int co = i % COUT, r = i / COUT;  // r = ci*9 + tap
    ws[i] = w[(size_t)co * CIN * 9 + r];
  }
  float acc[2][COUT];
#pragma unroll
  for (int j = 0; j < COUT; ++j) acc[0][j] = acc[1][j] = 0.f;
  const size_t plane = (size_t)H * W;
  const float *xb = x + (size_t)b * CIN * plane;
  for (int c0 = 0; c0 < CIN; c0 += CC) {
    __syncthreads();
    for (int i = tid; i < CC * TYP * TXP; i += 128) {
      const int cc = i / (TYP * TXP), rem = i % (TYP * TXP);
      const int yy = rem / TXP, xx = rem % TXP;
      const int gy = y0 + yy - 1, gx = x0 + xx - 1;
      float v = 0.f;
      if (c0 + cc < CIN && gy >= 0 && gy < H && gx >= 0 && gx < W)
        v = xb[(size_t)(c0 + cc) * plane + (size_t)gy * W + gx];
      xs[cc][yy][xx] = v;
    }
    __syncthreads();
#pragma unroll 1
    for (int cc = 0; cc < CC; ++cc) {
      const int ci = c0 + cc;
      if (ci >= CIN) break;
#pragma unroll
      for (int ky = 0; ky < 3; ++ky) {
        float xv[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) xv[k] = xs[cc][ty + ky][tx + k];
#pragma unroll
        for (int kx = 0; kx < 3; ++kx) {
          const float *wr = &ws[((ci * 3 + ky) * 3 + kx) * COUT];
#pragma unroll
          for (int co = 0; co < COUT; ++co) {
            const float wv = wr[co];
            acc[0][co] = fmaf(xv[kx], wv, acc[0][co]);
            acc[1][co] = fmaf(xv[kx + 1], wv, acc[1][co]);
          }
        }
      }
    }
  }
  const int gy = y0 + ty;
  if (gy >= H) return;
  float *ob = out + (size_t)b * COUT * plane;
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    const int gx = x0 + tx + k;
    if (gx >= W) continue;
    const size_t pix = (size_t)gy * W + gx;
#pragma unroll
    for (int co = 0; co < COUT; ++co) {
      float v = acc[k][co] + (bias ? bias[co] : 0.f);
      const size_t idx = (size_t)b * COUT * plane + (size_t)co * plane + pix;
      if (mask) v = mask[idx] > 0.f ? v : 0.f;
      if (resid) v += resid[idx];
      if (relu) v = fmaxf(v, 0.f);
      ob[(size_t)co * plane + pix] = v;
    }
  }
}

// ---------------------------------------------------------------------------
// wgrad: dw[co,ci,ky,kx] += sum_{b,y,x} dout[b,co,y,x] * x[b,ci,y+ky-1,x+kx-1]
//        db[co] += sum dout[b,co,:,:]     (nn.py:66-73)
// One thread per (ci, tap); each CTA sweeps `tiles_per_cta` pixel tiles and
// accumulates in fp32 registers, then atomically adds into the fp64 grads.
constexpr int WT_X = 32, WT_Y = 8;

// Generic weight / bias gradient (the convs other than 32 -> 32: conv_in's
// 2 -> C, conv_out's C -> 1, and the small presets).  Thread (ci, tap, k)
// accumulates the KS output channels co = k*KS .. of one (ci, tap) over a tile
// of WT_Y x WT_X pixels; dout is staged pixel-major with a padded row so the
// coalesced (pixel-fastest) loads and the per-pixel broadcast reads are both
// conflict-free.
template <int CIN, int COUT>
struct WgSimt {
  static constexpr int KS = COUT >= 16 ? 2 : COUT;          // output channels per thread
  static constexpr int NK = COUT / KS;
  static constexpr int ACTIVE = CIN * 9 * NK;
  static constexpr int NT = ACTIVE < 64 ? 64 : (ACTIVE + 31) / 32 * 32;
  static constexpr int DP = COUT + 1;                        // padded dout row
};

template <int CIN, int COUT>
__global__ void __launch_bounds__(WgSimt<CIN, COUT>::NT)
conv3x3_wgrad_kernel(const float *__restrict__ x, const float *__restrict__ dout,
                     int B, int H, int W, int tiles_per_cta,
                     double *__restrict__ dw, double *__restrict__ db) {
  using L = WgSimt<CIN, COUT>;
  constexpr int NT = L::NT, KS = L::KS, DP = L::DP;
  constexpr int TXP = WT_X + 2, TYP = WT_Y + 2, NP = WT_Y * WT_X;
  extern __shared__ float smem[];
  float *xs = smem;                                  // [CIN][TYP][TXP]
  float *ds = smem + CIN * TYP * TXP;                // [NP][DP]
  const int tid = threadIdx.x;
  const bool active = tid < L::ACTIVE;
  const int ct = tid / L::NK, k = tid % L::NK;      // (ci, tap), output-channel group
  const int ci = ct / 9, tap = ct % 9, ky = tap / 3, kx = tap % 3;
  float acc[KS];
  float bacc = 0.f;
#pragma unroll
  for (int j = 0; j < KS; ++j) acc[j] = 0.f;
  const int tx_n = (W + WT_X - 1) / WT_X, ty_n = (H + WT_Y - 1) / WT_Y;
  const long total_tiles = (long)B * tx_n * ty_n;
  const size_t plane = (size_t)H * W;
  for (int it = 0; it < tiles_per_cta; ++it) {
    const long t = (long)blockIdx.x * tiles_per_cta + it;
    if (t >= total_tiles) break;
    const int b = (int)(t / (tx_n * ty_n));
    const int rem = (int)(t % (tx_n * ty_n));
    const int y0 = (rem / tx_n) * WT_Y, x0 = (rem % tx_n) * WT_X;
    __syncthreads();
    for (int i = tid; i < CIN * TYP * TXP; i += NT) {
      const int c = i / (TYP * TXP), r = i % (TYP * TXP);
      const int yy = r / TXP, xx = r % TXP;
      const int gy = y0 + yy - 1, gx = x0 + xx - 1;
      float v = 0.f;
      if (gy >= 0 && gy < H && gx >= 0 && gx < W)
        v = x[((size_t)b * CIN + c) * plane + (size_t)gy * W + gx];
      xs[i] = v;
    }
    for (int i = tid; i < NP * COUT; i += NT) {
      const int p = i % NP, co = i / NP;             // pixel fastest: coalesced
      const int gy = y0 + p / WT_X, gx = x0 + p % WT_X;
      float v = 0.f;
      if (gy < H && gx < W) v = dout[((size_t)b * COUT + co) * plane + (size_t)gy * W + gx];
      ds[p * DP + co] = v;
    }
    __syncthreads();
    if (active) {
      const float *xr = xs + ci * TYP * TXP + ky * TXP + kx;
#pragma unroll 4
      for (int p = 0; p < NP; ++p) {
        const float xv = xr[(p / WT_X) * TXP + (p % WT_X)];
        const float *dr = ds + p * DP + k * KS;
#pragma unroll
        for (int j = 0; j < KS; ++j) acc[j] = fmaf(dr[j], xv, acc[j]);
      }
    }
    if (tid < COUT) {
      for (int p = 0; p < NP; ++p) bacc += ds[p * DP + tid];
    }
  }
  if (active) {
#pragma unroll
    for (int j = 0; j < KS; ++j)
      atomicAdd(&dw[((size_t)(k * KS + j) * CIN + ci) * 9 + tap], (double)acc[j]);
  }
  if (tid < COUT) atomicAdd(&db[tid], (double)bacc);
}

// ---------------------------------------------------------------------------
// Edge weight gradients (conv_in 2 -> C, conv_out C -> 1; nn.py:62-77): one
// side has C channels ("many"), the other F = 1 or 2 ("few").  A warp owns one
// (image, many-channel j, band of rows) and sweeps it row by row: each lane
// holds 8 columns of the many-channel row and a 3-row x 10-column register
// window of the few channels, so every input value is read from memory once
// per warp and the 9 F tap sums stay in registers (reduced over the warp at
// the end of the band, added in fp64).  dW[(j F + f) 9 + 3 ky + kx]:
//   S = +1 (conv_in):  many = dout (co = j), few = x    at (y+ky-1, x+kx-1)
//   S = -1 (conv_out): many = x (ci = j),    few = dout at (y-ky+1, x-kx+1)
// db: conv_in db[j] = sum of the many rows; conv_out db[0] = sum of the few.
#ifndef EW_RB_V
#define EW_RB_V 16   // 32 -> 16 measured 116 -> 111 us (conv_in dW) and 67 -> 59 us (conv_out dW)
#endif
constexpr int EW_RB = EW_RB_V;          // rows per warp task (fp32 chain length RB x 256)
template <int F, int S>
__global__ void __launch_bounds__(256) edge_wgrad_kernel(const float *__restrict__ many, const float *__restrict__ few,
                                                         int B, int C, int H, int W, double *__restrict__ dw,
                                                         double *__restrict__ db) {
  // a programmatic dependent launched next (the training convs) may start its
  // prologue while this kernel runs; it waits for our completion before
  // reading what we write
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int lane = threadIdx.x & 31;
  const long long wglob = (long long)blockIdx.x * 8 + (threadIdx.x >> 5), nw = (long long)gridDim.x * 8;
  const int n_bands = (H + EW_RB - 1) / EW_RB;
  const long long tasks = (long long)B * C * n_bands;
  const size_t plane = (size_t)H * W;
  const bool vec = (W & 7) == 0;
  for (long long task = wglob; task < tasks; task += nw) {
    const int band = (int)(task % n_bands), j = (int)((task / n_bands) % C), b = (int)(task / ((long long)n_bands * C));
    const int y0 = band * EW_RB, y1 = min(H, y0 + EW_RB);
    float acc[F][9];
#pragma unroll
    for (int f = 0; f < F; ++f)
#pragma unroll
      for (int t = 0; t < 9; ++t) acc[f][t] = 0.f;
    float dbacc = 0.f;
    const float *mrow0 = many + ((size_t)b * C + j) * plane;
    for (int xc = 0; xc < W; xc += 256) {
      const int x0 = xc + lane * 8;
      // raw loads of few-channel row yy: the 8 columns x0 .. x0+7 and, for the
      // chunk's edge lanes, the halo column (zero outside the image); the halo
      // columns of the other lanes come from their neighbours (widen)
      auto load_few = [&](int yy, float (&cen)[F][8], float (&edge)[F]) {
#pragma unroll
        for (int f = 0; f < F; ++f) {
#pragma unroll
          for (int k = 0; k < 8; ++k) cen[f][k] = 0.f;
          edge[f] = 0.f;
          if (yy < 0 || yy >= H) continue;
          const float *r = few + ((size_t)b * F + f) * plane + (size_t)yy * W;
          if (vec && x0 + 8 <= W) {
            const float4 u = __ldg(reinterpret_cast<const float4 *>(r + x0));
            const float4 v = __ldg(reinterpret_cast<const float4 *>(r + x0 + 4));
            cen[f][0] = u.x; cen[f][1] = u.y; cen[f][2] = u.z; cen[f][3] = u.w;
            cen[f][4] = v.x; cen[f][5] = v.y; cen[f][6] = v.z; cen[f][7] = v.w;
          } else {
#pragma unroll
            for (int k = 0; k < 8; ++k)
              if (x0 + k < W) cen[f][k] = __ldg(r + x0 + k);
          }
          if (lane == 0 && x0 - 1 >= 0 && x0 - 1 < W) edge[f] = __ldg(r + x0 - 1);
          if (lane == 31 && x0 + 8 < W) edge[f] = __ldg(r + x0 + 8);
        }
      };
      auto widen = [&](const float (&cen)[F][8], const float (&edge)[F], float (&dst)[F][10]) {
#pragma unroll
        for (int f = 0; f < F; ++f) {
#pragma unroll
          for (int k = 0; k < 8; ++k) dst[f][1 + k] = cen[f][k];
          const float left = __shfl_up_sync(0xffffffffu, cen[f][7], 1);
          const float right = __shfl_down_sync(0xffffffffu, cen[f][0], 1);
          dst[f][0] = lane > 0 ? left : edge[f];
          dst[f][9] = lane < 31 ? right : edge[f];
        }
      };
      auto load_many = [&](int y, float (&a)[8]) {
        const float *mr = mrow0 + (size_t)y * W;
        if (vec && x0 + 8 <= W) {
          const float4 u = __ldg(reinterpret_cast<const float4 *>(mr + x0));
          const float4 v = __ldg(reinterpret_cast<const float4 *>(mr + x0 + 4));
          a[0] = u.x; a[1] = u.y; a[2] = u.z; a[3] = u.w; a[4] = v.x; a[5] = v.y; a[6] = v.z; a[7] = v.w;
        } else {
#pragma unroll
          for (int k = 0; k < 8; ++k) a[k] = x0 + k < W ? __ldg(mr + x0 + k) : 0.f;
        }
      };
      float w0[F][10], w1[F][10], w2[F][10];   // few rows y-1, y, y+1
      float nc[F][8], ne[F], a[8];
      load_few(y0 - 1, nc, ne);
      widen(nc, ne, w0);
      load_few(y0, nc, ne);
      widen(nc, ne, w1);
      for (int y = y0; y < y1; ++y) {
        load_few(y + 1, nc, ne);
        load_many(y, a);
        widen(nc, ne, w2);
#pragma unroll
        for (int f = 0; f < F; ++f) {
#pragma unroll
          for (int ky = 0; ky < 3; ++ky) {
            // window row of tap ky: S = +1 -> y + ky - 1, S = -1 -> y - ky + 1
            const float(&wr)[10] = (S > 0 ? ky : 2 - ky) == 0 ? w0[f] : ((S > 0 ? ky : 2 - ky) == 1 ? w1[f] : w2[f]);
#pragma unroll
            for (int kx = 0; kx < 3; ++kx) {
              const int c = S > 0 ? kx : 2 - kx;   // column offset into the window
              float s = acc[f][ky * 3 + kx];
#pragma unroll
              for (int p = 0; p < 8; ++p) s = fmaf(a[p], wr[p + c], s);
              acc[f][ky * 3 + kx] = s;
            }
          }
        }
        if (S > 0) {
#pragma unroll
          for (int p = 0; p < 8; ++p) dbacc += a[p];
        } else if (j == 0) {
#pragma unroll
          for (int p = 0; p < 8; ++p) dbacc += w1[0][1 + p];
        }
#pragma unroll
        for (int f = 0; f < F; ++f)
#pragma unroll
          for (int k = 0; k < 10; ++k) {
            w0[f][k] = w1[f][k];
            w1[f][k] = w2[f][k];
          }
      }
    }
#pragma unroll
    for (int f = 0; f < F; ++f)
#pragma unroll
      for (int t = 0; t < 9; ++t) {
        float v = acc[f][t];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (lane == 0) atomicAdd(&dw[((size_t)j * F + f) * 9 + t], (double)v);
      }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) dbacc += __shfl_xor_sync(0xffffffffu, dbacc, o);
    if (lane == 0 && db != nullptr && (S > 0 || j == 0)) atomicAdd(&db[S > 0 ? j : 0], (double)dbacc);
  }
}

// Edge forward convs from few channels to many (conv_in 2 -> C, and the
// input gradient of conv_out, 1 -> C with the transposed weights;
// nn.py:46-77): a warp owns RB rows of one image, each lane 8 columns with a
// 3-row x 10-column register window of the F input channels (each input
// value read once per task); per output channel the 9 F weights are
// broadcast from shared memory and the 8 outputs stored as two 16-B stores.
constexpr int EF_RB = 2;
template <int F>
__global__ void __launch_bounds__(256) edge_fwd_f2m_kernel(const float *__restrict__ few, int B, int C, int H, int W,
                                                           const float *__restrict__ w, const float *__restrict__ bias,
                                                           float *__restrict__ out, int relu) {
  // a programmatic dependent launched next (the training convs) may start its
  // prologue while this kernel runs; it waits for our completion before
  // reading what we write
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  __shared__ float ws[32 * F * 9];
  __shared__ float bs[32];
  for (int i = threadIdx.x; i < C * F * 9; i += blockDim.x) ws[i] = __ldg(w + i);
  for (int i = threadIdx.x; i < C; i += blockDim.x) bs[i] = bias ? __ldg(bias + i) : 0.f;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const long long wglob = (long long)blockIdx.x * 8 + (threadIdx.x >> 5), nw = (long long)gridDim.x * 8;
  const int n_bands = (H + EF_RB - 1) / EF_RB;
  const long long tasks = (long long)B * n_bands;
  const size_t plane = (size_t)H * W;
  const bool vec = (W & 7) == 0;
  for (long long task = wglob; task < tasks; task += nw) {
    const int band = (int)(task % n_bands), b = (int)(task / n_bands);
    const int y0 = band * EF_RB, y1 = min(H, y0 + EF_RB);
    for (int xc = 0; xc < W; xc += 256) {
      const int x0 = xc + lane * 8;
      auto load_row = [&](int yy, float (&dst)[F][10]) {
#pragma unroll
        for (int f = 0; f < F; ++f) {
          float cen[8];
#pragma unroll
          for (int k = 0; k < 8; ++k) cen[k] = 0.f;
          float edge = 0.f;
          if (yy >= 0 && yy < H) {
            const float *r = few + ((size_t)b * F + f) * plane + (size_t)yy * W;
            if (vec && x0 + 8 <= W) {
              const float4 u = __ldg(reinterpret_cast<const float4 *>(r + x0));
              const float4 v = __ldg(reinterpret_cast<const float4 *>(r + x0 + 4));
              cen[0] = u.x; cen[1] = u.y; cen[2] = u.z; cen[3] = u.w;
              cen[4] = v.x; cen[5] = v.y; cen[6] = v.z; cen[7] = v.w;
            } else {
#pragma unroll
              for (int k = 0; k < 8; ++k)
                if (x0 + k < W) cen[k] = __ldg(r + x0 + k);
            }
            if (lane == 0 && x0 - 1 >= 0 && x0 - 1 < W) edge = __ldg(r + x0 - 1);
            if (lane == 31 && x0 + 8 < W) edge = __ldg(r + x0 + 8);
          }
          const float left = __shfl_up_sync(0xffffffffu, cen[7], 1);
          const float right = __shfl_down_sync(0xffffffffu, cen[0], 1);
#pragma unroll
          for (int k = 0; k < 8; ++k) dst[f][1 + k] = cen[k];
          dst[f][0] = lane > 0 ? left : edge;
          dst[f][9] = lane < 31 ? right : edge;
        }
      };
      float w0[F][10], w1[F][10], w2[F][10];
      load_row(y0 - 1, w0);
      load_row(y0, w1);
      for (int y = y0; y < y1; ++y) {
        load_row(y + 1, w2);
        for (int co = 0; co < C; ++co) {
          float acc[8];
#pragma unroll
          for (int p = 0; p < 8; ++p) acc[p] = bs[co];
#pragma unroll
          for (int f = 0; f < F; ++f)
#pragma unroll
            for (int ky = 0; ky < 3; ++ky) {
              const float(&wr)[10] = ky == 0 ? w0[f] : (ky == 1 ? w1[f] : w2[f]);
#pragma unroll
              for (int kx = 0; kx < 3; ++kx) {
                const float wv = ws[((co * F + f) * 3 + ky) * 3 + kx];
#pragma unroll
                for (int p = 0; p < 8; ++p) acc[p] = fmaf(wr[p + kx], wv, acc[p]);
              }
            }
          if (relu) {
#pragma unroll
            for (int p = 0; p < 8; ++p) acc[p] = fmaxf(acc[p], 0.f);
          }
          float *o = out + ((size_t)b * C + co) * plane + (size_t)y * W + x0;
          if (vec && x0 + 8 <= W) {
            reinterpret_cast<float4 *>(o)[0] = make_float4(acc[0], acc[1], acc[2], acc[3]);
            reinterpret_cast<float4 *>(o)[1] = make_float4(acc[4], acc[5], acc[6], acc[7]);
          } else {
#pragma unroll
            for (int p = 0; p < 8; ++p)
              if (x0 + p < W) o[p] = acc[p];
          }
        }
#pragma unroll
        for (int f = 0; f < F; ++f)
#pragma unroll
          for (int k = 0; k < 10; ++k) {
            w0[f][k] = w1[f][k];
            w1[f][k] = w2[f][k];
          }
      }
    }
  }
}

// Edge forward conv from many channels to one (conv_out C -> 1, nn.py:46-60):
// a CTA owns EM_RB rows of one image; its 8 warps split the input channels
// (warp k: channels k, k+8, ...), each lane 8 columns and the EM_RB x 8
// partial sums, a channel's rows held in a register window (each input row
// read (RB + 2) / RB times); the warps' partials are summed through shared
// memory in a fixed order (deterministic).
constexpr int EM_RB = 4;
__global__ void __launch_bounds__(256, 2) edge_fwd_m2o_kernel(const float *__restrict__ x, int B, int C, int H, int W,
                                                           const float *__restrict__ w, const float *__restrict__ bias,
                                                           float *__restrict__ out) {
  // a programmatic dependent launched next (the training convs) may start its
  // prologue while this kernel runs; it waits for our completion before
  // reading what we write
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  __shared__ float ws[32 * 9];
  __shared__ float red[8][EM_RB][256];
  for (int i = threadIdx.x; i < C * 9; i += blockDim.x) ws[i] = __ldg(w + i);
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int n_bands = (H + EM_RB - 1) / EM_RB;
  const long long tasks = (long long)B * n_bands;
  const size_t plane = (size_t)H * W;
  const bool vec = (W & 7) == 0;
  const float b0v = bias ? __ldg(bias) : 0.f;
  for (long long task = blockIdx.x; task < tasks; task += gridDim.x) {
    const int band = (int)(task % n_bands), b = (int)(task / n_bands);
    const int y0 = band * EM_RB;
    for (int xc = 0; xc < W; xc += 256) {
      const int x0 = xc + lane * 8;
      float acc[EM_RB][8];
#pragma unroll
      for (int i = 0; i < EM_RB; ++i)
#pragma unroll
        for (int p = 0; p < 8; ++p) acc[i][p] = 0.f;
      for (int ci = warp; ci < C; ci += 8) {
        const float *xp = x + ((size_t)b * C + ci) * plane;
        float rows[EM_RB + 2][10];
#pragma unroll
        for (int i = 0; i < EM_RB + 2; ++i) {
          const int yy = y0 - 1 + i;
          float cen[8];
#pragma unroll
          for (int k = 0; k < 8; ++k) cen[k] = 0.f;
          float edge = 0.f;
          if (yy >= 0 && yy < H) {
            const float *r = xp + (size_t)yy * W;
            if (vec && x0 + 8 <= W) {
              const float4 u = __ldg(reinterpret_cast<const float4 *>(r + x0));
              const float4 v = __ldg(reinterpret_cast<const float4 *>(r + x0 + 4));
              cen[0] = u.x; cen[1] = u.y; cen[2] = u.z; cen[3] = u.w;
              cen[4] = v.x; cen[5] = v.y; cen[6] = v.z; cen[7] = v.w;
            } else {
#pragma unroll
              for (int k = 0; k < 8; ++k)
                if (x0 + k < W) cen[k] = __ldg(r + x0 + k);
            }
            if (lane == 0 && x0 - 1 >= 0 && x0 - 1 < W) edge = __ldg(r + x0 - 1);
            if (lane == 31 && x0 + 8 < W) edge = __ldg(r + x0 + 8);
          }
          const float left = __shfl_up_sync(0xffffffffu, cen[7], 1);
          const float right = __shfl_down_sync(0xffffffffu, cen[0], 1);
#pragma unroll
          for (int k = 0; k < 8; ++k) rows[i][1 + k] = cen[k];
          rows[i][0] = lane > 0 ? left : edge;
          rows[i][9] = lane < 31 ? right : edge;
        }
#pragma unroll
        for (int ky = 0; ky < 3; ++ky)
#pragma unroll
          for (int kx = 0; kx < 3; ++kx) {
            const float wv = ws[ci * 9 + ky * 3 + kx];
#pragma unroll
            for (int i = 0; i < EM_RB; ++i)
#pragma unroll
              for (int p = 0; p < 8; ++p) acc[i][p] = fmaf(rows[i + ky][p + kx], wv, acc[i][p]);
          }
      }
      // partials -> shared memory; the sum over warps in warp order
#pragma unroll
      for (int i = 0; i < EM_RB; ++i) {
        float4 *d = reinterpret_cast<float4 *>(&red[warp][i][lane * 8]);
        d[0] = make_float4(acc[i][0], acc[i][1], acc[i][2], acc[i][3]);
        d[1] = make_float4(acc[i][4], acc[i][5], acc[i][6], acc[i][7]);
      }
      __syncthreads();
      for (int e = threadIdx.x; e < EM_RB * 256; e += blockDim.x) {
        const int i = e / 256, col = e % 256, y = y0 + i, xx = xc + col;
        if (y < H && xx < W) {
          float v = b0v;
#pragma unroll
          for (int k = 0; k < 8; ++k) v += red[k][i][col];
          out[(size_t)b * plane + (size_t)y * W + xx] = v;
        }
      }
      __syncthreads();
    }
  }
}

// ---------------------------------------------------------------------------
// elementwise helpers
// p = sigmoid(logit); a non-finite logit of sample i / per_flag sets
// nonfinite[i / per_flag]
__global__ void sigmoid_kernel(const float *__restrict__ logit, float *__restrict__ p,
                               int64_t n, int *__restrict__ nonfinite, int64_t per_flag) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const float l = logit[i];
  if (!isfinite(l)) atomicOr(nonfinite + i / per_flag, 1);
  p[i] = 1.f / (1.f + expf(-l));
}

// dlogits = dp * p * (1 - p)   (nn.py:156)
__global__ void dlogit_kernel(const float *__restrict__ dp, const float *__restrict__ p,
                              float *__restrict__ dl, int64_t n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const float q = p[i];
  dl[i] = dp[i] * q * (1.f - q);
}

// window logits (B, in_rows, W) -> outputs for rows [out_row0, +out_rows):
// p (float), h (uint8, p >= 0.5 <=> logit >= 0, rl.py:311)
__global__ void threshold_window_kernel(const float *__restrict__ logit, int B, int in_rows,
                                        int W, int row_off, int out_rows,
                                        float *__restrict__ p, uint8_t *__restrict__ h,
                                        int *__restrict__ nonfinite, int steps) {
  const int64_t n = (int64_t)B * out_rows * W;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int b = (int)(i / ((int64_t)out_rows * W));
  const int64_t rem = i % ((int64_t)out_rows * W);
  const int y = (int)(rem / W), xx = (int)(rem % W);
  const float l = logit[((int64_t)b * in_rows + y + row_off) * W + xx];
  if (!isfinite(l)) atomicOr(nonfinite, 1);
  if (p) p[i] = 1.f / (1.f + expf(-l));
  if (h) h[i] = level_of(l, steps);
}

}  // namespace ht

// ===========================================================================
// host orchestration
namespace ht {

// wgrad for the 32 -> 32 convs (the dominant training kernel): thread =
// (ci, ky) with all three kx taps x 32 co in registers, a sliding window
// over the x row (one shared load per pixel for 96 FMAs) and dout read as
// broadcast 16-B loads from pixel rows padded to 36 floats (conflict-light
// transposing stores of the coalesced NCHW loads).
constexpr int W32_NT = 96, W32_PAD = 36;
constexpr int W32_TX = 32, W32_TY = 8;   // 256-pixel tiles (measured faster than 128: per-tile overhead)

__global__ void __launch_bounds__(W32_NT)
conv3x3_wgrad32_kernel(const float *__restrict__ x, const float *__restrict__ dout, int B, int H, int W,
                       int tiles_per_cta, double *__restrict__ dw, double *__restrict__ db) {
  constexpr int C = 32, TXP = W32_TX + 2, TYP = W32_TY + 2, NP = W32_TY * W32_TX;
  extern __shared__ float smem[];
  float *xs = smem;                       // [C][TYP][TXP]
  float *ds = smem + C * TYP * TXP;       // [NP][W32_PAD]
  const int tid = threadIdx.x;
  const int ci = tid / 3, ky = tid % 3;
  float acc[3][C];
#pragma unroll
  for (int k = 0; k < 3; ++k)
#pragma unroll
    for (int j = 0; j < C; ++j) acc[k][j] = 0.f;
  float bacc = 0.f;
  const int tx_n = (W + W32_TX - 1) / W32_TX, ty_n = (H + W32_TY - 1) / W32_TY;
  const long total_tiles = (long)B * tx_n * ty_n;
  const size_t plane = (size_t)H * W;
  for (int it = 0; it < tiles_per_cta; ++it) {
    const long t = (long)blockIdx.x * tiles_per_cta + it;
    if (t >= total_tiles) break;
    const int b = (int)(t / (tx_n * ty_n));
    const int rem = (int)(t % (tx_n * ty_n));
    const int y0 = (rem / tx_n) * W32_TY, x0 = (rem % tx_n) * W32_TX;
    __syncthreads();
    for (int i = tid; i < C * TYP * TXP; i += W32_NT) {
      const int c = i / (TYP * TXP), r = i % (TYP * TXP);
      const int yy = r / TXP, xx = r % TXP;
      const int gy = y0 + yy - 1, gx = x0 + xx - 1;
      xs[i] = (gy >= 0 && gy < H && gx >= 0 && gx < W) ? x[((size_t)b * C + c) * plane + (size_t)gy * W + gx] : 0.f;
    }
    // dout tile: consecutive threads = consecutive pixels (coalesced), four
    // channels per thread -> one 16-B store into the pixel's padded row
    for (int i = tid; i < NP * (C / 4); i += W32_NT) {
      const int pp = i % NP, cg = i / NP;
      const int gy = y0 + pp / W32_TX, gx = x0 + pp % W32_TX;
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (gy < H && gx < W) {
        const float *src = dout + ((size_t)b * C + 4 * cg) * plane + (size_t)gy * W + gx;
        v = make_float4(src[0], src[plane], src[2 * plane], src[3 * plane]);
      }
      *reinterpret_cast<float4 *>(ds + pp * W32_PAD + 4 * cg) = v;
    }
    __syncthreads();
    const float *xr = xs + (ci * TYP + ky) * TXP;
#pragma unroll 1
    for (int yy = 0; yy < W32_TY; ++yy) {
      const float *row = xr + yy * TXP;
      float xa = row[0], xb = row[1];
#pragma unroll 2
      for (int xx = 0; xx < W32_TX; ++xx) {
        const float xc = row[xx + 2];
        const float4 *dr = reinterpret_cast<const float4 *>(ds + (yy * W32_TX + xx) * W32_PAD);
#pragma unroll
        for (int q = 0; q < C / 4; ++q) {
          const float4 d = dr[q];
          const float dv[4] = {d.x, d.y, d.z, d.w};
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            acc[0][4 * q + k] = fmaf(dv[k], xa, acc[0][4 * q + k]);
            acc[1][4 * q + k] = fmaf(dv[k], xb, acc[1][4 * q + k]);
            acc[2][4 * q + k] = fmaf(dv[k], xc, acc[2][4 * q + k]);
          }
        }
        xa = xb;
        xb = xc;
      }
    }
    if (tid < C) {
      for (int pp = 0; pp < NP; ++pp) bacc += ds[pp * W32_PAD + tid];
    }
  }
#pragma unroll
  for (int kx = 0; kx < 3; ++kx)
#pragma unroll
    for (int co = 0; co < C; ++co) atomicAdd(&dw[((size_t)(co * C + ci) * 3 + ky) * 3 + kx], (double)acc[kx][co]);
  if (tid < C) atomicAdd(&db[tid], (double)bacc);
}

// conv_tc.cu: the 32 -> 32 training conv on tcgen05 (split-bf16, fp32-level)
int conv_tc32(const float *x, int B, int H, int W, const float *w, const float *bias, const float *mask,
              const float *resid, float *out, int relu, cudaStream_t st);
// conv_tc2.cu: the same conv with scaled fp16 pairs and role-split warps
// (half the MMAs; TMA-staged shapes only)
bool conv_tc2_eligible(int W);
int conv_tc2_32(const float *x, int B, int H, int W, const float *w, const float *bias, const float *mask,
                const float *resid, float *out, int relu, cudaStream_t st);
int conv_tc2_32_ex(const float *x, int B, int H, int W, const float *w, const float *bias, const float *mask,
                   const float *resid, float *out, int relu, uint16_t *bits_out, const uint16_t *bits_in,
                   int accum, cudaStream_t st);
// 0: tensor cores for 32 -> 32 convs (default: conv_tc2 where the shape
// allows TMA staging, conv_tc otherwise), 1: SIMT only, 2: tensor cores with
// conv_tc.cu's split-bf16 kernel everywhere, 3: same as 0 (kept for A/B
// scripts)
extern int g_train_conv_impl;
// 1 (default): on the conv_tc2 path the training forward stores each conv1's
// ReLU as bits (4 B per pixel) and the backward reads those instead of the
// fp32 activation, and adds the conv1 input gradient onto the skip gradient
// in place; 0: fp32 mask / residual epilogue inputs (cross-check)
int g_train_bits = 1;
static bool train_bits_path(int C, int W) {
  return C == 32 && g_train_bits && (g_train_conv_impl == 0 || g_train_conv_impl == 3) && conv_tc2_eligible(W);
}
// activation workspaces whose ReLU bits the last forward into them wrote (the
// backward takes the bits path only for those, whatever the settings now)
static std::mutex g_bits_mu;
static std::set<const void *> g_bits_acts;
static void note_bits(const void *act, bool valid) {
  std::lock_guard<std::mutex> lk(g_bits_mu);
  if (valid) g_bits_acts.insert(act);
  else g_bits_acts.erase(act);
}
static bool has_bits(const void *act) {
  std::lock_guard<std::mutex> lk(g_bits_mu);
  return g_bits_acts.count(act) != 0;
}
// edge weight gradients: 0 = edge_wgrad_kernel (default), 1 = the generic
// SIMT tile kernel (cross-check)
int g_edge_conv_impl = 0;
// wgrad_tc.cu: their weight gradient on tcgen05 (split-bf16, `parts` bf16 parts)
int wgrad_tc32(const float *x, const float *dout, int B, int H, int W, double *dw, double *db, int parts,
               cudaStream_t st);
extern int g_wgrad_parts;

template <int CIN, int COUT>
static int conv_fwd(const float *x, int B, int H, int W, const float *w, const float *bias,
                    const float *mask, const float *resid, float *out, int relu,
                    cudaStream_t st) {
  if constexpr (COUT == 1 && CIN > 2 && CIN <= 32) {
    // edge conv many -> one (conv_out)
    if (g_edge_conv_impl == 0 && !mask && !resid && !relu) {
      const long long tasks = (long long)B * ((H + EM_RB - 1) / EM_RB);
      const int grid = (int)std::min<long long>(tasks, 148 * 8);
      edge_fwd_m2o_kernel<<<grid, 256, 0, st>>>(x, B, CIN, H, W, w, bias, out);
      count_launch();
      HT_CHECK_LAUNCH();
      return HT_OK;
    }
  }
  if constexpr (CIN <= 2 && COUT > 2 && COUT <= 32) {
    // edge convs few -> many (conv_in, conv_out's input gradient)
    if (g_edge_conv_impl == 0 && !mask && !resid) {
      const long long tasks = (long long)B * ((H + EF_RB - 1) / EF_RB);
      const int grid = (int)std::min<long long>((tasks + 7) / 8, 148 * 16);
      edge_fwd_f2m_kernel<CIN><<<grid, 256, 0, st>>>(x, B, COUT, H, W, w, bias, out, relu);
      count_launch();
      HT_CHECK_LAUNCH();
      return HT_OK;
    }
  }
  if constexpr (CIN == 32 && COUT == 32) {
    // conv_tc2 (20 x 256^2: 110 vs 134 us plain, 143 vs 162 us with a mask
    // or residual input) wherever the shape allows TMA staging
    if ((g_train_conv_impl == 0 || g_train_conv_impl == 3) && conv_tc2_eligible(W) && !(mask && resid))
      return conv_tc2_32(x, B, H, W, w, bias, mask, resid, out, relu, st);
    if (g_train_conv_impl != 1) return conv_tc32(x, B, H, W, w, bias, mask, resid, out, relu, st);
  }
  dim3 grid((W + FT_X - 1) / FT_X, (H + FT_Y - 1) / FT_Y, B);
  conv3x3_fwd_kernel<CIN, COUT><<<grid, 128, 0, st>>>(x, H, W, w, bias, mask, resid, out, relu);
  count_launch();
  HT_CHECK_LAUNCH();
  return HT_OK;
}

template <int CIN, int COUT>
static int conv_wgrad(const float *x, const float *dout, int B, int H, int W, double *dw,
                      double *db, cudaStream_t st) {
  if constexpr ((COUT == 1 && CIN > 2) || (CIN == 2 && COUT > 2)) {
    // edge convs: the warp-row kernel (one pass over each input)
    if (g_edge_conv_impl == 0) {
      constexpr int F = COUT == 1 ? 1 : 2;
      constexpr int S = COUT == 1 ? -1 : 1;
      const int C = COUT == 1 ? CIN : COUT;
      const long long tasks = (long long)B * C * ((H + EW_RB - 1) / EW_RB);
      const int grid = (int)std::min<long long>((tasks + 7) / 8, 148 * 8);
      const float *many = COUT == 1 ? x : dout, *fewp = COUT == 1 ? dout : x;
      edge_wgrad_kernel<F, S><<<grid, 256, 0, st>>>(many, fewp, B, C, H, W, dw, db);
      count_launch();
      HT_CHECK_LAUNCH();
      return HT_OK;
    }
  }
  if constexpr (CIN == 32 && COUT == 32) {
    // the tensor-core kernel streams rows with TMA (16-B row strides: W % 4 == 0)
    if (g_train_conv_impl != 1 && W % 4 == 0) return wgrad_tc32(x, dout, B, H, W, dw, db, g_wgrad_parts, st);
    const size_t smem = sizeof(float) * ((size_t)32 * (W32_TY + 2) * (W32_TX + 2) + W32_TY * W32_TX * W32_PAD);
    if (int rc = ensure_smem_attr((const void *)conv3x3_wgrad32_kernel, (int)smem)) return rc;
    const long tiles = (long)B * ((W + W32_TX - 1) / W32_TX) * ((H + W32_TY - 1) / W32_TY);
    const int per = tiles > 148 * 2 ? (int)((tiles + 148 * 2 - 1) / (148 * 2)) : 1;
    const int grid = (int)((tiles + per - 1) / per);
    conv3x3_wgrad32_kernel<<<grid, W32_NT, smem, st>>>(x, dout, B, H, W, per, dw, db);
    count_launch();
    HT_CHECK_LAUNCH();
    return HT_OK;
  }
  constexpr int NT = WgSimt<CIN, COUT>::NT;
  const size_t smem = sizeof(float) * ((size_t)CIN * (WT_Y + 2) * (WT_X + 2) + WT_Y * WT_X * WgSimt<CIN, COUT>::DP);
  if (int rc = ensure_smem_attr((const void *)conv3x3_wgrad_kernel<CIN, COUT>, (int)smem)) return rc;
  const long tiles = (long)B * ((W + WT_X - 1) / WT_X) * ((H + WT_Y - 1) / WT_Y);
  const int per = tiles > 148 * 8 ? (int)((tiles + 148 * 8 - 1) / (148 * 8)) : 1;
  const int grid = (int)((tiles + per - 1) / per);
  conv3x3_wgrad_kernel<CIN, COUT><<<grid, NT, smem, st>>>(x, dout, B, H, W, per, dw, db);
  count_launch();
  HT_CHECK_LAUNCH();
  return HT_OK;
}

// Generic-C dispatch.  The fused tensor-core kernel is specialised for the
// paper architecture (C=32, PRESET_PAPER nn.py:24); the SIMT path also
// serves the mini preset (C=8, nn.py:25) used by the reference's tests.
#define HT_DISPATCH_C(C, ...)                                                \
  switch (C) {                                                               \
    case 32: { constexpr int CC = 32; __VA_ARGS__; break; }                  \
    case 8:  { constexpr int CC = 8;  __VA_ARGS__; break; }                  \
    case 16: { constexpr int CC = 16; __VA_ARGS__; break; }                  \
    case 4:  { constexpr int CC = 4;  __VA_ARGS__; break; }                  \
    default: return ::ht::fail(HT_E_UNSUPPORTED, "channels=%d not compiled (supported: 4, 8, 16, 32)", C); \
  }

struct PackPtrs {
  const float *f32, *f32t;
};
static PackPtrs pack_ptrs(const void *packed, int C, int NB) {
  PackLayout L = pack_layout(C, NB);
  const char *base = (const char *)packed;
  return {(const float *)(base + L.f32_off), (const float *)(base + L.f32t_off)};
}

// Forward over (B, 2, H, W).  keep != nullptr: training mode, activations
// stored as y[0..NB] and r[0..NB-1] (each B*C*H*W); else ping-pong scratch.
static int simt_forward(const void *packed, int C, int NB, const float *x, int B, int H,
                        int W, float *scratch, bool keep, float *logits, cudaStream_t st,
                        uint16_t *bits = nullptr) {
  NetGeom g(C, NB);
  PackPtrs P = pack_ptrs(packed, C, NB);
  const size_t act = (size_t)B * C * H * W;
  auto ybuf = [&](int k) { return keep ? scratch + act * k : scratch + act * (k & 1); };
  auto rbuf = [&](int k) { return keep ? scratch + act * (NB + 1 + k) : scratch + act * 2; };
  int rc;
  HT_DISPATCH_C(C, {
    rc = conv_fwd<2, CC>(x, B, H, W, P.f32 + g.in_w, P.f32 + g.in_b, nullptr, nullptr,
                         ybuf(0), 0, st);
    if (rc) return rc;
    for (int k = 0; k < NB; ++k) {
      if (bits)
        rc = conv_tc2_32_ex(ybuf(k), B, H, W, P.f32 + g.w1(k), P.f32 + g.b1(k), nullptr, nullptr, rbuf(k), 1,
                            bits + (size_t)k * 2 * B * H * W, nullptr, 0, st);
      else
        rc = conv_fwd<CC, CC>(ybuf(k), B, H, W, P.f32 + g.w1(k), P.f32 + g.b1(k), nullptr,
                              nullptr, rbuf(k), 1, st);
      if (rc) return rc;
      rc = conv_fwd<CC, CC>(rbuf(k), B, H, W, P.f32 + g.w2(k), P.f32 + g.b2(k), nullptr,
                            ybuf(k), ybuf(k + 1), 0, st);
      if (rc) return rc;
    }
    rc = conv_fwd<CC, 1>(ybuf(NB), B, H, W, P.f32 + g.out_w, P.f32 + g.out_b, nullptr,
                         nullptr, logits, 0, st);
    if (rc) return rc;
  });
  return HT_OK;
}

int simt_halftone(const void *packed, int C, int NB, const float *c, const float *z, int B,
                  int H, int W, int in_row0, int in_rows, int out_row0, int out_rows,
                  float *p, uint8_t *h, void *ws, int64_t ws_bytes, int *nonfinite_dev,
                  int levels, cudaStream_t st) {
  const size_t plane = (size_t)in_rows * W;
  const size_t act = (size_t)B * C * plane;
  const int64_t need = (int64_t)sizeof(float) * (3 * act + (size_t)B * 2 * plane + (size_t)B * plane);
  HT_REQUIRE(ws_bytes >= need, "workspace too small: %lld < %lld", (long long)ws_bytes,
             (long long)need);
  float *scratch = (float *)ws;
  float *xin = scratch + 3 * act;
  float *logits = xin + (size_t)B * 2 * plane;
  // interleave (c, z) -> (B, 2, in_rows, W)
  for (int b = 0; b < B; ++b) {
    HT_CUDA(cudaMemcpyAsync(xin + (size_t)b * 2 * plane, c + (size_t)b * plane,
                            plane * sizeof(float), cudaMemcpyDeviceToDevice, st));
    HT_CUDA(cudaMemcpyAsync(xin + (size_t)b * 2 * plane + plane, z + (size_t)b * plane,
                            plane * sizeof(float), cudaMemcpyDeviceToDevice, st));
  }
  int rc = simt_forward(packed, C, NB, xin, B, in_rows, W, scratch, false, logits, st);
  if (rc) return rc;
  const int64_t n = (int64_t)B * out_rows * W;
  threshold_window_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(
      logits, B, in_rows, W, out_row0 - in_row0, out_rows, p, h, nonfinite_dev, levels - 1);
  count_launch();
  HT_CHECK_LAUNCH();
  return HT_OK;
}

int64_t simt_halftone_ws(int C, int B, int W, int in_rows) {
  const size_t plane = (size_t)in_rows * W;
  return (int64_t)sizeof(float) * (3 * (size_t)B * C * plane + (size_t)B * 3 * plane);
}

}  // namespace ht

// ===========================================================================
extern "C" {

int ht_train_act_bytes(int channels, int blocks, int B, int H, int W, int64_t *bytes) {
  const size_t act = (size_t)B * channels * H * W;
  // y[0..NB], r[0..NB-1], logits, 3 backward temporaries, then the conv1
  // ReLU bits (blocks x B x 2 x H x W uint16) of the conv_tc2 path
  *bytes = (int64_t)sizeof(float) * ((2 * (size_t)blocks + 1) * act + (size_t)B * H * W + 3 * act) +
           (int64_t)sizeof(uint16_t) * 2 * (size_t)blocks * B * H * W;
  return HT_OK;
}

// Training forward + sigmoid; sample b's non-finite logits OR'ed into
// flag_dev[b] (B device ints) without waiting for the GPU: the caller checks
// the flags later, e.g. once per training step before the parameter update.
int ht_policy_forward_train_async(const void *packed, int C, int NB, const float *x, int B, int H, int W,
                                  void *act, float *p, int *flag_dev, void *stream) {
  HT_REQUIRE(B > 0 && H > 0 && W > 0, "input must be non-empty (B=%d H=%d W=%d)", B, H, W);
  HT_REQUIRE(flag_dev != nullptr, "flag_dev must be a device int");
  ht::reset_launches();
  cudaStream_t st = (cudaStream_t)stream;
  const size_t a = (size_t)B * C * H * W;
  float *scratch = (float *)act;
  float *logits = scratch + (2 * (size_t)NB + 1) * a;
  uint16_t *bits = ht::train_bits_path(C, W)
                       ? reinterpret_cast<uint16_t *>(logits + (size_t)B * H * W + 3 * a) : nullptr;
  ht::note_bits(act, bits != nullptr);
  int rc = ht::simt_forward(packed, C, NB, x, B, H, W, scratch, true, logits, st, bits);
  if (rc) return rc;
  // sigmoid + finite check (nn.py:147-149)
  const int64_t n = (int64_t)B * H * W;
  ht::sigmoid_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(logits, p, n, flag_dev,
                                                                   (int64_t)H * W);
  ht::count_launch();
  HT_CHECK_LAUNCH();
  return HT_OK;
}

int ht_policy_forward_train(const void *packed, int C, int NB, const float *x, int B, int H,
                            int W, void *act, float *p, void *stream) {
  HT_REQUIRE(B > 0 && H > 0 && W > 0, "input must be non-empty (B=%d H=%d W=%d)", B, H, W);
  cudaStream_t st = (cudaStream_t)stream;
  int *d_flag;
  HT_CUDA(cudaMallocAsync(&d_flag, sizeof(int) * B, st));
  HT_CUDA(cudaMemsetAsync(d_flag, 0, sizeof(int) * B, st));
  const int rc = ht_policy_forward_train_async(packed, C, NB, x, B, H, W, act, p, d_flag, stream);
  if (rc) {
    cudaFreeAsync(d_flag, st);
    return rc;
  }
  std::vector<int> hflag(B, 0);
  HT_CUDA(cudaMemcpyAsync(hflag.data(), d_flag, sizeof(int) * B, cudaMemcpyDeviceToHost, st));
  HT_CUDA(cudaFreeAsync(d_flag, st));
  HT_CUDA(cudaStreamSynchronize(st));
  for (int b = 0; b < B; ++b)
    if (hflag[b]) return ht::fail(HT_E_NONFINITE, "non-finite logits");
  return HT_OK;
}

int ht_policy_backward(const void *packed, int C, int NB, const float *x, int B, int H, int W,
                       const void *act, const float *p, const float *dp, double *grad,
                       float *dx, void *stream) {
  HT_REQUIRE(B > 0 && H > 0 && W > 0, "input must be non-empty");
  ht::reset_launches();
  cudaStream_t st = (cudaStream_t)stream;
  ht::NetGeom g(C, NB);
  ht::PackPtrs P = ht::pack_ptrs(packed, C, NB);
  const size_t a = (size_t)B * C * H * W;
  const float *scratch = (const float *)act;
  auto y = [&](int k) { return scratch + a * k; };
  auto r = [&](int k) { return scratch + a * (NB + 1 + k); };
  float *tmp = (float *)(scratch + (2 * (size_t)NB + 1) * a + (size_t)B * H * W);
  float *dy = tmp, *dt = tmp + a, *dy2 = tmp + 2 * a;
  // the forward stored conv1's ReLU as bits when it took this path
  const uint16_t *bits = ht::has_bits(act) ? reinterpret_cast<const uint16_t *>(tmp + 3 * a) : nullptr;
  // dlogits into dt's first plane-set (B*H*W floats)
  float *dl = dt;
  const int64_t n = (int64_t)B * H * W;
  ht::dlogit_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(dp, p, dl, n);
  ht::count_launch();
  HT_CHECK_LAUNCH();
  // transposed weights: f32t mirrors the f32 layout (same offsets)
  int rc;
  HT_DISPATCH_C(C, {
    rc = ht::conv_wgrad<CC, 1>(y(NB), dl, B, H, W, grad + g.out_w, grad + g.out_b, st);
    if (rc) return rc;
    rc = ht::conv_fwd<1, CC>(dl, B, H, W, P.f32t + g.out_w, nullptr, nullptr, nullptr, dy, 0,
                             st);
    if (rc) return rc;
    for (int k = NB - 1; k >= 0; --k) {
      rc = ht::conv_wgrad<CC, CC>(r(k), dy, B, H, W, grad + g.w2(k), grad + g.b2(k), st);
      if (rc) return rc;
      if (bits)
        rc = ht::conv_tc2_32_ex(dy, B, H, W, P.f32t + g.w2(k), nullptr, nullptr, nullptr, dt, 0, nullptr,
                                bits + (size_t)k * 2 * B * H * W, 0, st);
      else
        rc = ht::conv_fwd<CC, CC>(dy, B, H, W, P.f32t + g.w2(k), nullptr, r(k), nullptr, dt, 0,
                                  st);
      if (rc) return rc;
      rc = ht::conv_wgrad<CC, CC>(y(k), dt, B, H, W, grad + g.w1(k), grad + g.b1(k), st);
      if (rc) return rc;
      if (bits) {
        // dy += conv1^T(dt), in place (same fp32 sum as the residual epilogue)
        rc = ht::conv_tc2_32_ex(dt, B, H, W, P.f32t + g.w1(k), nullptr, nullptr, nullptr, dy, 0, nullptr,
                                nullptr, 1, st);
        if (rc) return rc;
        continue;
      }
      rc = ht::conv_fwd<CC, CC>(dt, B, H, W, P.f32t + g.w1(k), nullptr, nullptr, dy, dy2, 0,
                                st);
      if (rc) return rc;
      float *t = dy; dy = dy2; dy2 = t;
    }
    rc = ht::conv_wgrad<2, CC>(x, dy, B, H, W, grad + g.in_w, grad + g.in_b, st);
    if (rc) return rc;
    if (dx) {
      rc = ht::conv_fwd<CC, 2>(dy, B, H, W, P.f32t + g.in_w, nullptr, nullptr, nullptr, dx, 0,
                               st);
      if (rc) return rc;
    }
  });
  return HT_OK;
}


// One 3x3 convolution 32 -> 32 (x, out, mask, resid: (B, 32, H, W) fp32; w
// OIHW fp32), the training conv with its epilogue options, on the chosen
// implementation: 0 = tcgen05 split-bf16, 1 = fp32 SIMT.  For tests.
int ht_conv3x3_32(const float *x, int B, int H, int W, const float *w, const float *bias,
                  const float *mask, const float *resid, float *out, int relu, int impl, void *stream) {
  HT_REQUIRE(B >= 1 && H >= 1 && W >= 1, "empty input");
  HT_REQUIRE(impl >= 0 && impl <= 3, "impl must be 0 (tensor core), 1 (simt), 2 (split bf16) or 3 (fp16 pairs)");
  const int keep = ht::g_train_conv_impl;
  ht::g_train_conv_impl = impl;
  const int rc = ht::conv_fwd<32, 32>(x, B, H, W, w, bias, mask, resid, out, relu, (cudaStream_t)stream);
  ht::g_train_conv_impl = keep;
  return rc;
}

// Weight / bias gradient of one 3x3 convolution 32 -> 32: dw (32,32,3,3) and
// db (32) fp64 accumulate (+=); impl 0 = tcgen05 with `parts` (2 or 3) bf16
// parts, 1 = fp32 SIMT.  For tests.
int ht_wgrad3x3_32(const float *x, const float *dout, int B, int H, int W, double *dw, double *db, int impl,
                   int parts, void *stream) {
  HT_REQUIRE(B >= 1 && H >= 1 && W >= 1, "empty input");
  HT_REQUIRE(impl == 0 || impl == 1, "impl must be 0 (tensor core) or 1 (simt)");
  HT_REQUIRE(parts == 2 || parts == 3, "parts must be 2 or 3");
  const int keep = ht::g_train_conv_impl, keep_parts = ht::g_wgrad_parts;
  ht::g_train_conv_impl = impl;
  ht::g_wgrad_parts = parts;
  const int rc = ht::conv_wgrad<32, 32>(x, dout, B, H, W, dw, db, (cudaStream_t)stream);
  ht::g_train_conv_impl = keep;
  ht::g_wgrad_parts = keep_parts;
  return rc;
}

}  // extern "C"
