// K3 + K4: action sampling, reward maps and the local-expectation (LE)
// flip-reward signal, fp64 math (the training signal is ~1e-5 and must stay
// within 1e-4 relative of the reference).
//
// Reference (region="full"; L output levels i/(L-1), L=2 the binary policy):
//   sampling      two-point cast of p onto the lattice (floor, ceil, p_ceil =
//                 frac) and m = u < p_ceil ? ceil : floor   rl.py:40-69
//                 (L=2: m = (u < p) bit for bit)
//   RewardContext f = conv(., k) (true convolution), window sums mu/E[..]
//                 by correlation with the SSIM window w; sigma_c, SSIM,
//                 CSSIM, reward map, scalar R         metrics.py:165-204, 95-107
//   delta_map     dSSE = 2 d corr(e,k) + d^2 corr(1,k^2); dCS summed over the
//                 window positions b covering a        metrics.py:333-392
//   estimators    per pixel from the flip delta D (moving pixel a to the other
//                 support point):
//                 local expectation  (m == ceil ? D : -D) * (L-1)    rl.py:96-109
//                 COMA (L=2)         h=1: (1-q) D / q, h=0: -q D / (1-q),
//                                    q = clip(p, 1e-7, 1-1e-7)      rl.py:117-129
//                 REINFORCE variants use the per-image reward only
//                 (ht_reinforce_signal)                             rl.py:132-136
#include "common.cuh"

namespace ht {

constexpr int RT = 16;            // output tile edge
constexpr int RMAXK = 11;         // max stencil size supported (odd; the reference default is 11)
constexpr int RH = RMAXK / 2;     // max halo

__device__ __forceinline__ double ssim3(double mx, double my, double sxx, double syy, double sxy,
                                        double c1, double c2, double *parts = nullptr) {
  // metrics.py:95-107
  const double vx = fmax(sxx - mx * mx, 0.0);
  const double vy = fmax(syy - my * my, 0.0);
  const double cov = sxy - mx * my;
  const double sx = sqrt(vx), sy = sqrt(vy);
  const double c3 = c2 / 2.0;
  const double lum = (2.0 * mx * my + c1) / (mx * mx + my * my + c1);
  const double con = (2.0 * sx * sy + c2) / (vx + vy + c2);
  const double str = (cov + c3) / (sx * sy + c3);
  if (parts) {
    parts[0] = lum;
    parts[1] = con;
    parts[2] = str;
  }
  return lum * con * str;
}

constexpr int NMAPS = 8;
constexpr int LE_NQ = 9;    // staged window-centre quantities of the delta kernel
constexpr int LE_SMEM = (LE_NQ * (RT + 2 * RH) * (RT + 2 * RH) + 2 * RMAXK * RMAXK) * 8;
// RewardContext's remaining maps (metrics.py:188-204), written on request:
//   [0] f_h  [1] f_c  [2] luminance  [3] contrast  [4] structure
//   [5] cssim_map  [6] reward_map
constexpr int NEXTRA = 7;

// two-point cast (rl.py:40-57): floor / ceil lattice values and upper mass
__device__ __forceinline__ void cast_two_point(double v, int steps, double &fl, double &ce, double &frac) {
  const double scaled = v * steps;
  const double idx = floor(scaled);
  frac = scaled - idx;
  fl = idx / steps;
  ce = frac == 0.0 ? fl : fmin(idx + 1.0, (double)steps) / steps;
}

// Stage 1: per pixel maps.  Workspace layout per image (doubles, n = H*W):
//   [0] e  [1] mu_h  [2] shc  [3] mu_c  [4] scc  [5] sigma_c  [6] ssim  [7] shh
// plus per-image sums[2] = {sum e^2, sum cssim}.  Also writes m, and the
// NEXTRA maps of the drop-in RewardContext when `extra` is given.  T is the
// input type: float32 on the training path, float64 for the drop-in API.
template <typename T>
__global__ void __launch_bounds__(256)
reward_maps_kernel(const T *__restrict__ p, const double *__restrict__ u,
                   const T *__restrict__ c, int H, int W, const double *__restrict__ k,
                   int ks, const double *__restrict__ w, int wsz, double c1, double c2,
                   double gain, double w_s, int steps, T *__restrict__ m_out,
                   double *__restrict__ maps, double *__restrict__ sums, double *__restrict__ extra) {
  const int b = blockIdx.z;
  const int x0 = blockIdx.x * RT, y0 = blockIdx.y * RT;
  const int hk = ks / 2, hw = wsz / 2, hh = hk > hw ? hk : hw;
  const int TP = RT + 2 * RH;
  __shared__ double sm[RT + 2 * RH][RT + 2 * RH + 1];
  __shared__ double sc[RT + 2 * RH][RT + 2 * RH + 1];
  __shared__ double sk[RMAXK * RMAXK], sw[RMAXK * RMAXK];
  __shared__ double red[2][8];
  // separable window (the reference's SSIM window is the normalised outer
  // product of a sampled 1-D Gaussian, hvs.py:54-64): w_ij = a_i a_j with
  // a_i = sum_j w_ij; the five window sums then take 2 x wsz products each
  // instead of wsz^2 (horizontal pass into hs, vertical pass per pixel)
  __shared__ double sa[RMAXK], sb1[RMAXK];
  __shared__ double hs[5][RT + 2 * RH][RT];
  __shared__ double hf[2][RT + 2 * RH][RT];
  __shared__ int sep, sepk;
  const size_t n = (size_t)H * W;
  const T *pb = p + b * n;
  const double *ub = u + b * n;
  const T *cb = c + b * n;
  for (int i = threadIdx.x; i < ks * ks; i += 256) sk[i] = k[i];
  for (int i = threadIdx.x; i < wsz * wsz; i += 256) sw[i] = w[i];
  __syncthreads();
  // (the same for the HVS kernel k when it is a Gaussian, hvs.py:54-64; the
  // Nasanen kernel is not separable and keeps the 2-D loop)
  if (threadIdx.x < wsz) {
    double r = 0.0;
    for (int j = 0; j < wsz; ++j) r += sw[threadIdx.x * wsz + j];
    sa[threadIdx.x] = r;
  } else if (threadIdx.x >= 32 && threadIdx.x < 32 + ks) {
    const int i = threadIdx.x - 32;
    double r = 0.0;
    for (int j = 0; j < ks; ++j) r += sk[i * ks + j];
    sb1[i] = r;
  }
  __syncthreads();
  if (threadIdx.x < 64) {
    // warp 0 checks w, warp 1 checks k: max |w_ij - a_i a_j| against max |w|
    const bool isw = threadIdx.x < 32;
    const int sz = isw ? wsz : ks;
    const double *m2 = isw ? sw : sk;
    const double *f1 = isw ? sa : sb1;
    double mx = 0.0, err = 0.0;
    for (int t = threadIdx.x & 31; t < sz * sz; t += 32) {
      const double v = m2[t];
      mx = fmax(mx, fabs(v));
      err = fmax(err, fabs(v - f1[t / sz] * f1[t % sz]));
    }
    for (int o = 16; o > 0; o >>= 1) {
      mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
      err = fmax(err, __shfl_xor_sync(0xffffffffu, err, o));
    }
    // a few ulps for the reference's Gaussians; far above for other kernels
    if ((threadIdx.x & 31) == 0) {
      if (isw) sep = err <= 1e-14 * mx;
      else sepk = err <= 1e-14 * mx;
    }
  }
  for (int i = threadIdx.x; i < TP * TP; i += 256) {
    const int yy = i / TP, xx = i % TP;
    const int gy = y0 + yy - RH, gx = x0 + xx - RH;
    double mv = 0.0, cv = 0.0;
    if (gy >= 0 && gy < H && gx >= 0 && gx < W) {
      const size_t idx = (size_t)gy * W + gx;
      if (ub) {
        double fl, ce, frac;
        cast_two_point((double)pb[idx], steps, fl, ce, frac);
        mv = ub[idx] < frac ? ce : fl;
      } else {
        mv = (double)pb[idx];                 // action map given (RewardContext)
      }
      cv = (double)cb[idx];
    }
    sm[yy][xx] = mv;
    sc[yy][xx] = cv;
  }
  __syncthreads();
  if (sep) {
    for (int i = threadIdx.x; i < TP * RT; i += 256) {
      const int yy = i / RT, xx = i % RT;
      double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0, a4 = 0.0;
      for (int j = 0; j < wsz; ++j) {
        const double wv = sa[j];
        const double mv = sm[yy][xx + RH + j - hw], cv = sc[yy][xx + RH + j - hw];
        a0 += wv * mv;
        a1 += wv * (mv * mv);
        a2 += wv * (mv * cv);
        a3 += wv * cv;
        a4 += wv * (cv * cv);
      }
      hs[0][yy][xx] = a0; hs[1][yy][xx] = a1; hs[2][yy][xx] = a2; hs[3][yy][xx] = a3; hs[4][yy][xx] = a4;
    }
  }
  if (sepk) {
    // convolution rows: h[yy][x] = sum_j b_j img[yy][x - (j - hk)]
    for (int i = threadIdx.x; i < TP * RT; i += 256) {
      const int yy = i / RT, xx = i % RT;
      double a0 = 0.0, a1 = 0.0;
      for (int j = 0; j < ks; ++j) {
        const double kv = sb1[j];
        a0 += kv * sm[yy][xx + RH - (j - hk)];
        a1 += kv * sc[yy][xx + RH - (j - hk)];
      }
      hf[0][yy][xx] = a0;
      hf[1][yy][xx] = a1;
    }
  }
  if (sep || sepk) __syncthreads();
  const int tx = threadIdx.x % RT, ty = threadIdx.x / RT;
  const int gy = y0 + ty, gx = x0 + tx;
  double e2 = 0.0, cs = 0.0;
  if (gy < H && gx < W) {
    // f = conv(img, k): f[y,x] = sum_ij k[i,j] img[y-(i-hk), x-(j-hk)]
    double fh = 0.0, fc = 0.0;
    if (sepk) {
      for (int i = 0; i < ks; ++i) {
        const double kv = sb1[i];
        fh += kv * hf[0][ty + RH - (i - hk)][tx];
        fc += kv * hf[1][ty + RH - (i - hk)][tx];
      }
    } else {
      for (int i = 0; i < ks; ++i)
        for (int j = 0; j < ks; ++j) {
          const double kv = sk[i * ks + j];
          const int yy = ty + RH - (i - hk), xx = tx + RH - (j - hk);
          fh += kv * sm[yy][xx];
          fc += kv * sc[yy][xx];
        }
    }
    // window sums by correlation with w
    double muh = 0.0, shc = 0.0, muc = 0.0, scc = 0.0, shh = 0.0;
    if (sep) {
      for (int i = 0; i < wsz; ++i) {
        const double wv = sa[i];
        const int yy = ty + RH + i - hw;
        muh += wv * hs[0][yy][tx];
        shh += wv * hs[1][yy][tx];
        shc += wv * hs[2][yy][tx];
        muc += wv * hs[3][yy][tx];
        scc += wv * hs[4][yy][tx];
      }
    } else {
      for (int i = 0; i < wsz; ++i)
        for (int j = 0; j < wsz; ++j) {
          const double wv = sw[i * wsz + j];
          const int yy = ty + RH + i - hw, xx = tx + RH + j - hw;
          const double mv = sm[yy][xx], cv = sc[yy][xx];
          muh += wv * mv;
          shh += wv * (mv * mv);
          shc += wv * (mv * cv);
          muc += wv * cv;
          scc += wv * (cv * cv);
        }
    }
    const double sig = fmin(gain * sqrt(fmax(scc - muc * muc, 0.0)), 1.0);
    double parts[3];
    const double s = ssim3(muh, muc, shh, scc, shc, c1, c2, parts);
    const double e = fh - fc;
    const size_t idx = (size_t)gy * W + gx;
    double *mb = maps + (size_t)b * NMAPS * n;
    mb[0 * n + idx] = e;
    mb[1 * n + idx] = muh;
    mb[2 * n + idx] = shc;
    mb[3 * n + idx] = muc;
    mb[4 * n + idx] = scc;
    mb[5 * n + idx] = sig;
    mb[6 * n + idx] = s;
    mb[7 * n + idx] = shh;
    m_out[b * n + idx] = (T)sm[ty + RH][tx + RH];
    e2 = e * e;
    cs = sig * s + (1.0 - sig);
    if (extra) {
      double *xb = extra + (size_t)b * NEXTRA * n;
      xb[0 * n + idx] = fh;
      xb[1 * n + idx] = fc;
      xb[2 * n + idx] = parts[0];
      xb[3 * n + idx] = parts[1];
      xb[4 * n + idx] = parts[2];
      xb[5 * n + idx] = cs;
      xb[6 * n + idx] = -e2 + w_s * cs;
    }
  }
  (void)hh;
  for (int o = 16; o > 0; o >>= 1) {
    e2 += __shfl_xor_sync(0xffffffffu, e2, o);
    cs += __shfl_xor_sync(0xffffffffu, cs, o);
  }
  if ((threadIdx.x & 31) == 0) {
    red[0][threadIdx.x >> 5] = e2;
    red[1][threadIdx.x >> 5] = cs;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0.0, bsum = 0.0;
    for (int i = 0; i < 8; ++i) { a += red[0][i]; bsum += red[1][i]; }
    atomicAdd(&sums[2 * b], a);
    atomicAdd(&sums[2 * b + 1], bsum);
  }
}

// Stage 2: delta for moving every pixel to its other support point, then
// the estimator's signal (scaled), per pixel a.  estimator: 0 = local
// expectation, 1 = COMA (binary only).
template <typename T, typename TO>
__global__ void __launch_bounds__(256)
reward_le_kernel(const T *__restrict__ m_in, const T *__restrict__ p, const T *__restrict__ other,
                 const T *__restrict__ c, int H, int W, const double *__restrict__ k, int ks, const double *__restrict__ w, int wsz,
                 double c1, double c2, double w_s, double scale, int steps, int estimator,
                 const double *__restrict__ maps, TO *__restrict__ signal) {
  const int b = blockIdx.z;
  const int x0 = blockIdx.x * RT, y0 = blockIdx.y * RT;
  const int hk = ks / 2, hw = wsz / 2;
  constexpr int TP = RT + 2 * RH;
  // window-centre quantities around the tile, staged once per centre (each
  // centre serves up to 121 pixels): e, mu_h, shc, shh, mu_c,
  // mu_c^2 + C1, v_c + C2, sigma_c, SSIM (v_c = max(E[c^2] - mu_c^2, 0))
  extern __shared__ double smem_le[];
  double (*sb)[TP][TP] = reinterpret_cast<double (*)[TP][TP]>(smem_le);
  double *sk = smem_le + LE_NQ * TP * TP, *sw = sk + RMAXK * RMAXK;
  const size_t n = (size_t)H * W;
  const double *mb = maps + (size_t)b * NMAPS * n;
  for (int i = threadIdx.x; i < ks * ks; i += 256) sk[i] = k[i];
  for (int i = threadIdx.x; i < wsz * wsz; i += 256) sw[i] = w[i];
  for (int i = threadIdx.x; i < TP * TP; i += 256) {
    const int yy = i / TP, xx = i % TP;
    const int gy = y0 + yy - RH, gx = x0 + xx - RH;
    const bool in = gy >= 0 && gy < H && gx >= 0 && gx < W;
    const size_t idx = in ? (size_t)gy * W + gx : 0;
    const double muc = in ? mb[3 * n + idx] : 0.0, scc = in ? mb[4 * n + idx] : 0.0;
    const double vc = fmax(scc - muc * muc, 0.0);
    sb[0][yy][xx] = in ? mb[0 * n + idx] : 0.0;   // e
    sb[1][yy][xx] = in ? mb[1 * n + idx] : 0.0;   // mu_h
    sb[2][yy][xx] = in ? mb[2 * n + idx] : 0.0;   // shc
    sb[3][yy][xx] = in ? mb[7 * n + idx] : 0.0;   // shh
    sb[4][yy][xx] = muc;
    sb[5][yy][xx] = muc * muc + c1;
    sb[6][yy][xx] = vc + c2;
    sb[7][yy][xx] = in ? mb[5 * n + idx] : 0.0;   // sigma_c
    sb[8][yy][xx] = in ? mb[6 * n + idx] : 0.0;   // SSIM before
  }
  __syncthreads();
  const int tx = threadIdx.x % RT, ty = threadIdx.x / RT;
  const int gy = y0 + ty, gx = x0 + tx;
  if (gy >= H || gx >= W) return;
  const size_t ia = (size_t)gy * W + gx;
  const T mf = m_in[b * n + ia];
  double ma = (double)mf;
  const double ca = (double)c[b * n + ia];
  // other support point (rl.py:98-99): m == ceil ? floor : ceil
  const double pa = (double)p[b * n + ia];
  double lv, hv, frac;
  cast_two_point(pa, steps, lv, hv, frac);
  // m_out may be float32: recover the exact lattice value of a sampled action
  const bool at_ceil = mf == (T)hv;
  if (!other) ma = at_ceil ? hv : lv;
  // other - h: the given substitution, or the other support point (+-1 for
  // L=2; 0 where the support collapsed)
  const double d = other ? (double)other[b * n + ia] - ma : (at_ceil ? lv : hv) - ma;
  // dSSE = 2 d corr(e, k)[a] + d^2 sum_{y in image} k[y - a + hk]^2
  double ce = 0.0, k2 = 0.0;
  for (int i = 0; i < ks; ++i) {
    const int yy = gy + i - hk;
    if (yy < 0 || yy >= H) continue;
    for (int j = 0; j < ks; ++j) {
      const int xx = gx + j - hk;
      if (xx < 0 || xx >= W) continue;
      const double kv = sk[i * ks + j];
      ce += kv * sb[0][ty + RH + i - hk][tx + RH + j - hk];
      k2 += kv * kv;
    }
  }
  const double dsse = 2.0 * d * ce + d * d * k2;
  // dCS[a] = sum over window centres b = a - (dy,dx), in image, of
  //          sigma_c[b] (SSIM_b(after) - SSIM_b(before)),  wd = w[hw+dy, hw+dx]
  double dcs = 0.0;
  // d == 0: the window statistics do not move, so every SSIM term cancels
  // exactly (as in the reference's numpy evaluation; recomputing s1 here
  // could differ from the stored s0 in the last bit)
  if (w_s != 0.0 && d != 0.0) {
    const double dh = 2.0 * ma * d + d * d, dc = d * ca, c3 = c2 / 2.0;
    for (int dy = -hw; dy <= hw; ++dy) {
      const int by = gy - dy;
      if (by < 0 || by >= H) continue;
      for (int dx = -hw; dx <= hw; ++dx) {
        const int bx = gx - dx;
        if (bx < 0 || bx >= W) continue;
        const double wd = sw[(hw + dy) * wsz + (hw + dx)];
        const int sy = ty + RH - dy, sx = tx + RH - dx;
        // SSIM_b after the edit (metrics.py:95-107 with the window sums moved
        // by wd * (d, 2 h d + d^2, d c)).  With C3 = C2 / 2 the contrast
        // factor's numerator is exactly twice the structure factor's
        // denominator (2 s_h s_c + C2 = 2 (s_h s_c + C3), exact in binary
        // floating point), so contrast x structure = 2 (cov + C3) /
        // (v_h + v_c + C2): no square root, one division
        const double mh = sb[1][sy][sx] + wd * d;
        const double muc = sb[4][sy][sx];
        const double vx = fmax(sb[3][sy][sx] + wd * dh - mh * mh, 0.0);
        const double cov = sb[2][sy][sx] + wd * dc - mh * muc;
        const double num = (2.0 * mh * muc + c1) * (2.0 * (cov + c3));
        const double den = (mh * mh + sb[5][sy][sx]) * (vx + sb[6][sy][sx]);
        dcs += sb[7][sy][sx] * (num / den - sb[8][sy][sx]);
      }
    }
  }
  const double delta = (-dsse + w_s * dcs) / (double)n;
  double sigv;
  if (estimator == 2) {
    sigv = delta;                              // raw delta map (metrics.delta_map)
  } else if (estimator == 1) {
    // COMA: -dlogpi(p, h) (R - baseline), baseline = q R_up + (1-q) R_down
    const double q = fmin(fmax(pa, 1e-7), 1.0 - 1e-7);
    sigv = ma == 1.0 ? (1.0 - q) * delta / q : -q * delta / (1.0 - q);
  } else {
    // local expectation: -(sign * delta) / (1/(L-1)), sign = -1 where m == ceil
    sigv = (at_ceil ? delta : -delta) * (double)steps;
  }
  signal[b * n + ia] = (TO)(sigv * scale);
}

__global__ void reinforce_kernel(const float *__restrict__ p, const float *__restrict__ m, int64_t total,
                                 int64_t n, const double *__restrict__ reward, double baseline, double scale,
                                 float *__restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const double q = fmin(fmax((double)p[i], 1e-7), 1.0 - 1e-7);
    const double dl = m[i] == 1.0f ? 1.0 / q : -1.0 / (1.0 - q);
    out[i] = (float)(-dl * (reward[i / n] - baseline) * scale);
  }
}

__global__ void reward_finalize_kernel(const double *__restrict__ sums, int B, double n,
                                       double w_s, double *__restrict__ reward) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  const double mse = sums[2 * b] / n;
  const double css = sums[2 * b + 1] / n;
  reward[b] = -mse + w_s * css;
}

}  // namespace ht

extern "C" {

int ht_reward_workspace_bytes(int B, int H, int W, int64_t *bytes) {
  *bytes = (int64_t)sizeof(double) * ((int64_t)B * ht::NMAPS * H * W + 2 * (int64_t)B) + 256;
  return HT_OK;
}

int ht_reward_signal(const float *p, const double *u, const float *other, const float *c, int B, int H, int W,
                     const double *k, int ks, const double *w, int wsz, double w_s, double c1,
                     double c2, double gain, int levels, int estimator, double scale, float *m_out,
                     float *signal_out, double *reward_out, void *ws, int64_t ws_bytes, void *stream) {
  HT_REQUIRE(B >= 1 && H >= 1 && W >= 1, "empty batch");
  HT_REQUIRE(ks % 2 == 1 && ks <= ht::RMAXK && wsz % 2 == 1 && wsz <= ht::RMAXK,
             "stencils must be odd and at most %d wide", ht::RMAXK);
  HT_REQUIRE(levels >= 2 && levels <= 256, "levels must be in [2, 256]");
  HT_REQUIRE(estimator == 0 || (estimator == 1 && levels == 2) || (estimator == 2 && other != nullptr),
             "estimator must be 0 (local expectation), 1 (COMA, binary policies only) or 2 "
             "(delta map, needs `other`)");
  HT_REQUIRE(u != nullptr || estimator == 2 || signal_out == nullptr,
             "estimator signals need sampled actions (u)");
  HT_REQUIRE(m_out != nullptr, "m_out is required");
  int64_t need = 0;
  ht_reward_workspace_bytes(B, H, W, &need);
  HT_REQUIRE(ws_bytes >= need, "workspace too small");
  cudaStream_t st = (cudaStream_t)stream;
  double *maps = (double *)ws;
  double *sums = maps + (size_t)B * ht::NMAPS * H * W;
  HT_CUDA(cudaMemsetAsync(sums, 0, sizeof(double) * 2 * B, st));
  dim3 grid((W + ht::RT - 1) / ht::RT, (H + ht::RT - 1) / ht::RT, B);
  ht::reward_maps_kernel<float><<<grid, 256, 0, st>>>(p, u, c, H, W, k, ks, w, wsz, c1, c2, gain, w_s,
                                                      levels - 1, m_out, maps, sums, nullptr);
  ht::count_launch();
  HT_CHECK_LAUNCH();
  if (signal_out) {
    if (int rc = ht::ensure_smem_attr((const void *)ht::reward_le_kernel<float, float>, ht::LE_SMEM)) return rc;
    ht::reward_le_kernel<float, float><<<grid, 256, ht::LE_SMEM, st>>>(m_out, p, other, c, H, W, k, ks, w, wsz, c1, c2,
                                                             w_s, scale, levels - 1, estimator, maps, signal_out);
    ht::count_launch();
    HT_CHECK_LAUNCH();
  }
  if (reward_out) {
    ht::reward_finalize_kernel<<<(B + 127) / 128, 128, 0, st>>>(sums, B, (double)H * W, w_s,
                                                                 reward_out);
    ht::count_launch();
    HT_CHECK_LAUNCH();
  }
  return HT_OK;
}

int ht_reward_le(const float *p, const double *u, const float *c, int B, int H, int W,
                 const double *k, int ks, const double *w, int wsz, double w_s, double c1,
                 double c2, double gain, double scale, float *m_out, float *signal_out,
                 double *reward_out, void *ws, int64_t ws_bytes, void *stream) {
  return ht_reward_signal(p, u, nullptr, c, B, H, W, k, ks, w, wsz, w_s, c1, c2, gain, 2, 0, scale, m_out,
                          signal_out, reward_out, ws, ws_bytes, stream);
}

// Drop-in RewardContext (metrics.py:165-204) on float64 action maps h and
// contones c (region "full"): maps_out (B, 8, H, W) = e, mu_h, shc, mu_c,
// scc, sigma_c, ssim, shh; extra_out (B, 7, H, W) = f_h, f_c, luminance,
// contrast, structure, cssim_map, reward_map; sums_out (B, 2) = sum e^2,
// sum cssim; h_out (B, H, W) a copy of the action maps (scratch).
int ht_reward_context_f64(const double *h, const double *c, int B, int H, int W, const double *k, int ks,
                          const double *w, int wsz, double w_s, double c1, double c2, double gain,
                          double *maps_out, double *extra_out, double *sums_out, double *h_out,
                          void *stream) {
  HT_REQUIRE(B >= 1 && H >= 1 && W >= 1, "empty batch");
  HT_REQUIRE(ks % 2 == 1 && ks <= ht::RMAXK && wsz % 2 == 1 && wsz <= ht::RMAXK,
             "stencils must be odd and at most %d wide", ht::RMAXK);
  HT_REQUIRE(maps_out && sums_out && h_out, "maps_out, sums_out and h_out are required");
  cudaStream_t st = (cudaStream_t)stream;
  HT_CUDA(cudaMemsetAsync(sums_out, 0, sizeof(double) * 2 * B, st));
  dim3 grid((W + ht::RT - 1) / ht::RT, (H + ht::RT - 1) / ht::RT, B);
  ht::reward_maps_kernel<double><<<grid, 256, 0, st>>>(h, nullptr, c, H, W, k, ks, w, wsz, c1, c2, gain, w_s, 1,
                                                       h_out, maps_out, sums_out, extra_out);
  ht::count_launch();
  HT_CHECK_LAUNCH();
  return HT_OK;
}

// Drop-in delta_map (metrics.py:333-392) in float64: delta_out[a] =
// R(h with pixel a -> other[a]) - R(h) for every pixel a.  Workspace:
// ht_reward_workspace_bytes(B, H, W) + 8 * B * H * W bytes.
int ht_reward_delta_f64(const double *h, const double *other, const double *c, int B, int H, int W,
                        const double *k, int ks, const double *w, int wsz, double w_s, double c1, double c2,
                        double gain, double *delta_out, void *ws, int64_t ws_bytes, void *stream) {
  HT_REQUIRE(B >= 1 && H >= 1 && W >= 1, "empty batch");
  HT_REQUIRE(ks % 2 == 1 && ks <= ht::RMAXK && wsz % 2 == 1 && wsz <= ht::RMAXK,
             "stencils must be odd and at most %d wide", ht::RMAXK);
  int64_t need = 0;
  ht_reward_workspace_bytes(B, H, W, &need);
  HT_REQUIRE(ws_bytes >= need + 8 * (int64_t)B * H * W, "workspace too small");
  cudaStream_t st = (cudaStream_t)stream;
  double *maps = (double *)ws;
  double *sums = maps + (size_t)B * ht::NMAPS * H * W;
  double *m = (double *)((char *)ws + need);
  HT_CUDA(cudaMemsetAsync(sums, 0, sizeof(double) * 2 * B, st));
  dim3 grid((W + ht::RT - 1) / ht::RT, (H + ht::RT - 1) / ht::RT, B);
  ht::reward_maps_kernel<double><<<grid, 256, 0, st>>>(h, nullptr, c, H, W, k, ks, w, wsz, c1, c2, gain, w_s, 1,
                                                       m, maps, sums, nullptr);
  if (int rc = ht::ensure_smem_attr((const void *)ht::reward_le_kernel<double, double>, ht::LE_SMEM)) return rc;
  ht::reward_le_kernel<double, double><<<grid, 256, ht::LE_SMEM, st>>>(m, h, other, c, H, W, k, ks, w, wsz, c1, c2, w_s,
                                                             1.0, 1, 2, maps, delta_out);
  ht::count_launch(2);
  HT_CHECK_LAUNCH();
  return HT_OK;
}

// REINFORCE (rl.py:132-136): signal = -dlogpi(p, h) (R_b - baseline) * scale,
// dlogpi = 1/q where h = 1, -1/(1-q) where h = 0, q = clip(p, 1e-7, 1-1e-7).
int ht_reinforce_signal(const float *p, const float *m, int B, int64_t n, const double *reward,
                        double baseline, double scale, float *signal_out, void *stream) {
  HT_REQUIRE(B >= 1 && n >= 1, "empty batch");
  const int64_t total = (int64_t)B * n;
  const int grid = (int)((total + 255) / 256 < 8192 ? (total + 255) / 256 : 8192);
  ht::reinforce_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(p, m, total, n, reward, baseline, scale,
                                                                 signal_out);
  ht::count_launch();
  HT_CHECK_LAUNCH();
  return HT_OK;
}

}  // extern "C"
