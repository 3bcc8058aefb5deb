/*
 * htb200.h -- C-ABI of the B200-native halftoning hot path (arXiv 2304.12152).
 *
 * Drop-in boundary for the reference package `htlab` (pure Python/NumPy,
 * /root/reference/pkg/src/htlab).  Every entry point names the reference
 * interface it replaces (file:line, relative to that directory).  The Python
 * host layer `paper_2304_12152_b200` binds these with ctypes and mirrors the
 * reference's Python API on top.
 *
 * Conventions
 *   - plain pointers and sizes only; no torch types.  Pointers named *_dev
 *     are CUDA device pointers; `stream` is a cudaStream_t (NULL = legacy
 *     default stream).  All kernels are sm_100a.
 *   - every function returns an int status: HT_OK (0) or one of HT_E_*;
 *     ht_last_error() returns the message of the last failure on the calling
 *     thread.  The host layer maps HT_E_INVALID -> ValueError,
 *     HT_E_NONFINITE -> FloatingPointError (nn.py:147-148), others ->
 *     RuntimeError.
 *   - images are row-major float32 (B, H, W) planes; the library never frees
 *     caller memory.
 *   - parameters are one flat float64 buffer in PolicyNetwork.params() order
 *     (nn.py:118-122): conv_in.w (C,2,3,3), conv_in.b (C), then per residual
 *     block conv1.w (C,C,3,3), conv1.b, conv2.w, conv2.b, then conv_out.w
 *     (1,C,3,3), conv_out.b (1).  Weights are OIHW, cross-correlation
 *     convention (nn.py:46-60).
 */
#ifndef HTB200_H
#define HTB200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HT_OK 0
#define HT_E_INVALID 1     /* bad shape / argument  -> ValueError          */
#define HT_E_NONFINITE 2   /* non-finite logits     -> FloatingPointError  */
#define HT_E_CUDA 3        /* CUDA runtime failure  -> RuntimeError        */
#define HT_E_UNSUPPORTED 4 /* arch / config not supported                  */

/* ---- library ---------------------------------------------------------- */
const char *ht_last_error(void);
int ht_version(void);
/* 1 if `device` is an sm_100 part this library's cubins run on. */
int ht_device_supported(int device, int *supported);

/* ---- host RNG: bit-exact xoshiro256++ / splitmix64 / Box-Muller ---------
 * Replaces imagecore.Rng (imagecore.py:35-120) and gaussian_noise_map
 * (imagecore.py:155-159) for host-side input preparation.  state[4] is the
 * xoshiro state (Rng.state_words()). */
int ht_rng_seed(uint64_t seed, uint64_t state[4]);            /* Rng.__init__ imagecore.py:43-50 */
int ht_rng_uniforms(uint64_t state[4], int64_t n, double *out); /* Rng.uniforms imagecore.py:70-86 */
int ht_rng_gaussians(uint64_t state[4], int64_t n, double *out);/* Rng.gaussians imagecore.py:88-99 */
int ht_rng_gaussians_f32(uint64_t state[4], int64_t n, float *out);
/* Advance state by n draws without producing them (GF(2) jump-ahead; the
 * same stream position Rng.uniforms(n) would leave).  Not in the reference:
 * the building block for the device streams below. */
int ht_rng_jump(uint64_t state[4], uint64_t n);
/* Device Rng.gaussians / Rng.uniforms: writes n values to
 * the device buffer `out` (fp64 if f64 != 0, else fp32) on `stream`, each
 * thread jumping to its own offset of the stream; the host state advances
 * exactly as the host call would (uniforms: n draws; gaussians:
 * 2*ceil(n/2)).  Uniforms are bit-exact; gaussians use the device's fp64
 * log/sin/cos (<= 2 ulp from libm: fp32-rounded values match the host
 * stream except for ~1e-8 of samples, by one fp32 ulp).  Replaces the
 * host loops of gaussian_noise_map (imagecore.py:155-159) and the action
 * uniforms of rl.sample_actions (rl.py:67-69). */
int ht_rng_gaussians_device(uint64_t state[4], int64_t n, void *out, int f64, void *stream);
int ht_rng_uniforms_device(uint64_t state[4], int64_t n, void *out, int f64, void *stream);
/* n_maps noise maps of n gaussians in one launch, map m drawn from the stream
 * state states[4m..4m+3] (host array), written at out + m*n; no host state
 * advances (the caller recorded the states and jumped past each map). */
int ht_rng_gaussian_maps_device(const uint64_t *states, int n_maps, int64_t n, void *out, int f64,
                                void *stream);

/* ---- policy network parameters ----------------------------------------- */
/* Number of float64 parameters of PolicyNetwork(channels, blocks, in_ch=2). */
int ht_num_params(int channels, int blocks, int64_t *n);
/* Bytes of the packed device weight image produced by ht_pack_params. */
int ht_packed_bytes(int channels, int blocks, int64_t *bytes);
/* Repack the flat float64 parameters (device) into the kernels' layouts:
 * fp32 OIHW + transposed/flipped copies for the SIMT training kernels and
 * the fp16 UMMA K-major tiles of the fused tensor-core forward.  Must be
 * re-run whenever the parameters change (Adam step, checkpoint load). */
int ht_pack_params(const double *params_dev, int channels, int blocks,
                   void *packed_dev, void *stream);

/* ---- K1: fused inference forward + sigmoid + threshold ------------------
 * Replaces PolicyNetwork.forward (nn.py:138-150) + rl.infer_halftone's
 * threshold `p >= 0.5` (rl.py:306-311; L=2 twin multitone.py:61-67).
 * c_dev/z_dev hold rows [in_row0, in_row0+in_rows) of B images of full
 * height H and width W (image stride in_rows*W).  Produces rows
 * [out_row0, out_row0+out_rows) (must lie inside the input rows, with a
 * 34-row receptive-field halo available unless at a true image edge).
 * Outputs (each optional, NULL to skip), image stride out_rows*W:
 *   p_dev   float32 probabilities
 *   h_dev   uint8 halftone, 1 = white (p >= 0.5)
 *   pbm_dev PBM P4 payload bytes: per row ceil(W/8) bytes, bit 1 = black,
 *           MSB first (imagecore.save_pbm, imagecore.py:289-297)
 * workspace: ht_halftone_workspace_bytes() bytes of device scratch.
 * impl: 0 = fused tcgen05 tensor-core kernel (default), 1 = fp32 SIMT
 * layer-by-layer kernels (reference-precision cross-check).            */
int ht_halftone_workspace_bytes(int channels, int blocks, int B, int H, int W,
                                int in_rows, int out_rows, int impl,
                                int64_t *bytes);
int ht_halftone(const void *packed_dev, int channels, int blocks,
                const float *c_dev, const float *z_dev, int B, int H, int W,
                int in_row0, int in_rows, int out_row0, int out_rows,
                float *p_dev, uint8_t *h_dev, uint8_t *pbm_dev,
                void *workspace_dev, int64_t workspace_bytes, int impl,
                void *stream);
/* Multitone inference (multitone.infer_multitone / quantize_multitone,
 * multitone.py:61-76): same forward as ht_halftone, the
 * epilogue writes q_dev = index of the nearest level i/(levels-1) of p
 * (half-steps round up) as uint8; levels in [2, 256] (2 = ht_halftone's h). */
int ht_multitone(const void *packed_dev, int channels, int blocks,
                 const float *c_dev, const float *z_dev, int B, int H, int W,
                 int in_row0, int in_rows, int out_row0, int out_rows, int levels,
                 float *p_dev, uint8_t *q_dev, void *workspace_dev,
                 int64_t workspace_bytes, int impl, void *stream);
/* Reads the non-finite-logit flag the last ht_halftone left in `workspace_dev`
 * (synchronises `stream`); HT_E_NONFINITE if set (nn.py:147-148). */
int ht_halftone_check(const void *workspace_dev, void *stream);
/* Number of kernel launches the last ht_halftone on this thread issued. */
int ht_last_launch_count(int *count);
/* Measurement hooks (bench.py): when enabled, every fused-forward pass launch
 * on this thread is bracketed by CUDA events on its stream; ht_timing_read
 * returns (tag, ms) per launch since the last read.  tag = 100*has_conv_in +
 * 10*blocks_in_pass + has_conv_out. */
int ht_timing_enable(int on);
/* Pre-creates n (begin, end) event pairs for the hooks (no event creation
 * inside a timed region). */
int ht_timing_reserve(int n);
int ht_timing_read(int *tags, float *ms, int max, int *count);

/* Training convolutions (nn.py:46-77): 0 = the 32 -> 32 convs of the residual
 * blocks (forward, input gradient and weight gradient) on tcgen05 (default:
 * scaled fp16 pairs where the shape allows TMA staging, W % 4 == 0 and
 * W >= 127; split-bf16 operands otherwise), 1 = fp32 SIMT kernels only
 * (cross-check), 2 = tcgen05 with split-bf16 operands everywhere, 3 = same
 * as 0.  Process-wide. */
int ht_set_train_conv_impl(int impl);
/* bf16 parts of the tensor-core weight gradient: 2 (three products,
 * ~2^-16 per product; default -- the config-5 step stays at 1.6e-5 of the
 * reference normwise per tensor, tests/test_gpu_train_cfg5.py) or 3 (six
 * products, fp32 level). */
int ht_set_wgrad_parts(int parts);
/* Training edge convs (conv_in 2 -> C, conv_out C -> 1; forward, weight
 * gradients and conv_out's input gradient, nn.py:46-77): 0 = warp-row
 * kernels reading each input once (default), 1 = the generic SIMT tile
 * kernels (cross-check).  Process-wide. */
int ht_set_edge_conv_impl(int impl);
/* Training ReLU bits (the _relu_mask of ResidualBlock, nn.py:89-100): 1 =
 * on the TMA-staged training-conv path the forward stores each conv1's ReLU
 * as bits (4 B per pixel) that conv2's input gradient reads instead of the
 * fp32 activation, and conv1's input gradient is added onto the skip
 * gradient in place (default); 0 = fp32 mask / residual epilogue inputs
 * (cross-check).  Process-wide; a backward follows what its forward did. */
int ht_set_train_bits(int on);
/* The training conv v2 (conv_tc2.cu) on CTA pairs: tcgen05.mma.cta_group::2
 * (M = 256, each CTA holding half of every weight window) -- 1 = on,
 * 0 = one CTA per strip.  Process-wide. */
int ht_set_conv_pair(int on);
/* One 32 -> 32 training convolution (x, out, mask, resid (B,32,H,W) fp32, w
 * OIHW (32,32,3,3) fp32; bias / mask / resid may be NULL): out = conv(x) +
 * bias, zeroed where mask <= 0, + resid, ReLU if relu -- Conv2d.forward
 * (nn.py:46-60) and the epilogues of the block backward (nn.py:97-100) --
 * on impl 0 (tcgen05) or 1 (fp32 SIMT).  For parity tests. */
int ht_conv3x3_32(const float *x, int B, int H, int W, const float *w, const float *bias,
                  const float *mask, const float *resid, float *out, int relu, int impl,
                  void *stream);
/* Weight / bias gradient of one such convolution (Conv2d.backward's dW, db,
 * nn.py:62-77): dw (32,32,3,3) and db (32) fp64 are accumulated into (+=);
 * impl 0 = tcgen05 with `parts` bf16 parts (2 or 3), 1 = fp32 SIMT. */
int ht_wgrad3x3_32(const float *x, const float *dout, int B, int H, int W, double *dw, double *db,
                   int impl, int parts, void *stream);

/* ---- K1' / K2: training forward (stores activations) and backward -------
 * Replaces PolicyNetwork.forward/backward (nn.py:138-160) incl.
 * ResidualBlock (nn.py:91-100) and Conv2d (nn.py:46-77), fp32 math.
 * x_dev: (B, 2, H, W) float32.  act_dev: ht_train_act_bytes() bytes.
 * p_dev: (B, H, W) float32 output.  Returns HT_E_NONFINITE on non-finite
 * logits (nn.py:147-148).  The 32 -> 32 convs run on tcgen05 (scaled fp16
 * pairs where the shape allows TMA staging, split bf16 otherwise), the edge
 * convs in fp32 SIMT (see ht_set_train_conv_impl).  The workspace holds the
 * activations, three backward temporaries and the conv1 ReLU bits
 * (ht_set_train_bits); ht_policy_backward takes the workspace its forward
 * filled. */
int ht_train_act_bytes(int channels, int blocks, int B, int H, int W,
                       int64_t *bytes);
int ht_policy_forward_train(const void *packed_dev, int channels, int blocks,
                            const float *x_dev, int B, int H, int W,
                            void *act_dev, float *p_dev, void *stream);
/* Same without waiting for the GPU: sample b's non-finite logits are OR'ed
 * into flag_dev[b] (B device ints the caller zeroes and checks later --
 * rl.train_step checks them once per step, before the parameter update, and
 * raises as nn.py:147-148 would). */
int ht_policy_forward_train_async(const void *packed_dev, int channels, int blocks,
                                  const float *x_dev, int B, int H, int W,
                                  void *act_dev, float *p_dev, int *flag_dev, void *stream);
/* dp_dev (B,H,W) float32 = dL/dp injected at the sigmoid output.
 * grad_dev: flat float64 gradient in params() order, ACCUMULATED (+=) like
 * the reference's .grad (nn.py:66-73; caller zeroes, nn.py:134-136).
 * dx_dev (B,2,H,W) float32 or NULL. */
int ht_policy_backward(const void *packed_dev, int channels, int blocks,
                       const float *x_dev, int B, int H, int W,
                       const void *act_dev, const float *p_dev,
                       const float *dp_dev, double *grad_dev, float *dx_dev,
                       void *stream);

/* ---- K3 + K4: sampled actions, reward maps, LE flip-reward signal -------
 * Replaces rl._sample_two_point (rl.py:67-69, L=2), metrics.RewardContext
 * (metrics.py:165-204, region="full"), metrics.delta_map +
 * _delta_cssim_map (metrics.py:333-392) and rl.le_signal (rl.py:96-109).
 * p, c: (B,H,W) float32, u (B,H,W) float64 uniforms; m_out (B,H,W) float32
 * sampled actions (u < p); stencils up to 11x11 (hvs_size default 11);
 * signal_out (B,H,W) float32 = le_signal * scale; reward_out (B) float64
 * scalar R per image.  k_hvs / w_ssim: ksize x ksize / wsize x wsize
 * float64 stencils (host constants, hvs.py:54-103).                     */
int ht_reward_le(const float *p_dev, const double *u_dev, const float *c_dev,
                 int B, int H, int W, const double *k_hvs_dev, int ksize,
                 const double *w_ssim_dev, int wsize, double w_s, double c1,
                 double c2, double gain, double scale, float *m_out_dev,
                 float *signal_out_dev, double *reward_out_dev,
                 void *workspace_dev, int64_t workspace_bytes, void *stream);
int ht_reward_workspace_bytes(int B, int H, int W, int64_t *bytes);
/* General form (L output levels, estimators):
 *   u_dev != NULL: actions sampled by the two-point cast of p onto the
 *     lattice i/(L-1) (rl._cast_two_point / _sample_two_point, rl.py:40-69);
 *   u_dev == NULL: p_dev holds the action map itself (RewardContext).
 *   estimator 0: local expectation, (m == ceil ? D : -D) * (L-1)
 *              (rl.le_signal, rl.py:96-109; multitone_le, multitone.py:56-59)
 *   estimator 1: COMA (rl.coma_signal, rl.py:117-129), L = 2 only
 *   estimator 2: raw delta D(a -> other[a]) (metrics.delta_map, needs
 *              other_dev: (B,H,W) float32 substitute values)
 * where D is the reward change of moving pixel a to the other support point
 * (or to other[a]).  signal_out = signal * scale.  ht_reward_le is this
 * entry with L = 2, estimator 0. */
int ht_reward_signal(const float *p_dev, const double *u_dev, const float *other_dev,
                     const float *c_dev, int B, int H, int W, const double *k_hvs_dev,
                     int ksize, const double *w_ssim_dev, int wsize, double w_s, double c1,
                     double c2, double gain, int levels, int estimator, double scale,
                     float *m_out_dev, float *signal_out_dev, double *reward_out_dev,
                     void *workspace_dev, int64_t workspace_bytes, void *stream);
/* REINFORCE / REINFORCE with mean baseline (rl.reinforce_signal,
 * rl.py:132-136): signal = -dlogpi(p, m) (reward[b] - baseline) * scale,
 * dlogpi = 1/q (m = 1) or -1/(1-q) (m = 0), q = clip(p, 1e-7, 1 - 1e-7);
 * p, m, signal (B, n) float32, reward (B) float64. */
int ht_reinforce_signal(const float *p_dev, const float *m_dev, int B, int64_t n,
                        const double *reward_dev, double baseline, double scale,
                        float *signal_out_dev, void *stream);

/* Drop-in RewardContext (metrics.py:165-204, region "full") on float64
 * action maps h and contones c, computed in float64: maps_out (B,8,H,W) =
 * e, mu_h, shc, mu_c, scc, sigma_c, ssim, shh; extra_out (B,7,H,W) = f_h,
 * f_c, luminance, contrast, structure, cssim_map, reward_map (may be NULL);
 * sums_out (B,2) = sum e^2, sum cssim; h_out (B,H,W) scratch copy of h.  */
int ht_reward_context_f64(const double *h_dev, const double *c_dev, int B,
                          int H, int W, const double *k_hvs_dev, int ks,
                          const double *w_ssim_dev, int wsz, double w_s,
                          double c1, double c2, double gain,
                          double *maps_out_dev, double *extra_out_dev,
                          double *sums_out_dev, double *h_out_dev,
                          void *stream);
/* Drop-in delta_map (metrics.py:333-392) in float64: delta_out (B,H,W) =
 * R(h with pixel a -> other[a]) - R(h).  Workspace:
 * ht_reward_workspace_bytes(B,H,W) + 8*B*H*W bytes.                      */
int ht_reward_delta_f64(const double *h_dev, const double *other_dev,
                        const double *c_dev, int B, int H, int W,
                        const double *k_hvs_dev, int ks,
                        const double *w_ssim_dev, int wsz, double w_s,
                        double c1, double c2, double gain,
                        double *delta_out_dev, void *workspace_dev,
                        int64_t workspace_bytes, void *stream);

/* ---- K5 / K7: spectral ---------------------------------------------------
 * anisotropy_loss / anisotropy_loss_backward (spectral.py:100-133) for B
 * images: loss_out (B) float64, grad_out (B,H,W) float32 = dL/dx * scale.
 * ring_dev (H*W) int32 dense ring index (-1 = DC), counts_dev (n_rings)
 * int32 (spectral.py:39-55).  grad_out may be NULL.                      */
int ht_spectral_workspace_bytes(int B, int H, int W, int n_rings,
                                int64_t *bytes);
int ht_anisotropy(const float *x_dev, int B, int H, int W,
                  const int32_t *ring_dev, const int32_t *counts_dev,
                  int n_rings, double scale, double *loss_out_dev,
                  float *grad_out_dev, void *workspace_dev,
                  int64_t workspace_bytes, void *stream);
/* Same for float64 images (spectral.anisotropy_loss on float64 arrays
 * keeps the reference's precision); grad_out (B,H,W) float64.           */
int ht_anisotropy_f64(const double *x_dev, int B, int H, int W,
                      const int32_t *ring_dev, const int32_t *counts_dev,
                      int n_rings, double scale, double *loss_out_dev,
                      double *grad_out_dev, void *workspace_dev,
                      int64_t workspace_bytes, void *stream);
/* rapsd (spectral.py:74-88) of the periodogram (spectral.py:17-24) of B
 * images: power_out / anis_out (B, n_rings) float64, dc_out (B).        */
int ht_rapsd(const float *x_dev, int B, int H, int W,
             const int32_t *ring_dev, const int32_t *counts_dev, int n_rings,
             double *power_out_dev, double *anis_out_dev, double *dc_out_dev,
             void *workspace_dev, int64_t workspace_bytes, void *stream);
int ht_rapsd_f64(const double *x_dev, int B, int H, int W,
                 const int32_t *ring_dev, const int32_t *counts_dev, int n_rings,
                 double *power_out_dev, double *anis_out_dev, double *dc_out_dev,
                 void *workspace_dev, int64_t workspace_bytes, void *stream);
/* periodogram (spectral.py:17-24): P_out (B,H,W) float64 = |FFT2(x)|^2/N.
 * Workspace: ht_spectral_workspace_bytes(B, H, W, 1).                   */
int ht_periodogram_f64(const double *x_dev, int B, int H, int W,
                       double *P_out_dev, void *workspace_dev,
                       int64_t workspace_bytes, void *stream);
/* rapsd(p_hat, part) (spectral.py:74-88) of given periodograms P (B,H,W). */
int ht_rapsd_power_f64(const double *P_dev, int B, int H, int W,
                       const int32_t *ring_dev, const int32_t *counts_dev,
                       int n_rings, double *power_out_dev,
                       double *anis_out_dev, double *dc_out_dev,
                       void *workspace_dev, int64_t workspace_bytes,
                       void *stream);

/* ---- drop-in layer API in float64 (nn.py:36-103) ------------------------
 * Conv2d.forward: out (B,Co,H,W) = bias + x (B,Ci,H,W) correlated with w
 * (Co,Ci,3,3), zero padding 1 (nn.py:46-60).  bias may be NULL.
 * Conv2d.backward (nn.py:62-77): dw (Co,Ci,3,3) += dL/dw, db (Co) += dL/db
 * (both may be NULL), dx (B,Ci,H,W) = dL/dx (may be NULL).              */
int ht_conv3x3_f64(const double *x_dev, int B, int Ci, int Co, int H, int W,
                   const double *w_dev, const double *bias_dev,
                   double *out_dev, void *stream);
int ht_conv3x3_f64_backward(const double *x_dev, const double *dout_dev,
                            int B, int Ci, int Co, int H, int W,
                            const double *w_dev, double *dw_dev,
                            double *db_dev, double *dx_dev, void *stream);

/* ---- K6: Adam (nn.py:163-186) on the flat float64 parameter vector ----- */
int ht_adam_step(double *params_dev, const double *grad_dev, double *m_dev,
                 double *v_dev, int64_t n, int t, double lr, double beta1,
                 double beta2, double eps, void *stream);

/* ---- small device reductions used by rl.train_step (rl.py:254-255) ----- */
/* out[0] += sum |p - rint(p)| over n elements (bin_gap numerator). */
int ht_bin_gap_sum(const float *p_dev, int64_t n, double *out_dev,
                   void *stream);

#ifdef __cplusplus
}
#endif
#endif /* HTB200_H */
