/*
 * stanza_b200.h -- C ABI of the B200-native Stanza layer-separated step.
 *
 * The reference (stanza-sim 0.1.0, /root/reference/pkg/src/stanza) has no C
 * ABI: its per-layer operator contract is the Python pair
 *     forward(layer, params, x, labels=None) -> (y, cache)
 *     backward(layer, params, cache, gy)    -> (gx, [gW, gb])   (sums)
 * in tensor_core.py:153-301, plus sgd_step (tensor_core.py:366-388).  Each
 * entry point below replaces one layer kind / phase of that contract and is
 * what a reference-side FFI (ctypes) would bind.
 *
 * Conventions
 *   - all tensors are fp32 (labels int32), row-major, device pointers owned
 *     by the caller; layouts are the reference's: activations NCHW, conv W
 *     [O,C,k,k], FC W [in,out] (tensor_core.py:81-88);
 *   - ws / ws_bytes: optional caller workspace for split-K partials (pass
 *     NULL, 0 to disable split-K);
 *   - stream: a cudaStream_t passed as void*;
 *   - returns 0 on success, 1 invalid argument (the reference raises
 *     ShapeMismatch, tensor_core.py:25-26), 2 CUDA launch error,
 *     3 workspace too small; stz_last_error() describes the failure.
 *   - gradients are batch SUMS, as in the reference; the only division by
 *     the global batch is the inv_n argument of stz_sgd_momentum.
 */
#ifndef STANZA_B200_H
#define STANZA_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ABI version (2) and the last error message of the calling thread. */
int stz_abi_version(void);
const char* stz_last_error(void);

/* Number of kernels this library has launched (bench evidence). */
unsigned long long stz_launch_count(void);

/* GEMM producer: 1 (default) = TMA (tiled / im2col tensor maps) where the
 * shapes allow it, with each MN-major tile fetched as one 3D box; 2 = TMA
 * with one 2D box per 32 MN-major rows; 0 = the cp.async gather kernel for
 * every GEMM (the GPU tests run all and compare). */
int stz_set_tma(int on);

/* Thin (64-wide, unpaired) GEMM tiles as two 128-row halves per CTA sharing
 * one B stage and one 256-row A box: 0 (default) when the GEMM has enough row
 * tiles to fill the GPU, 1 never, 2 always (tests). */
int stz_set_mh(int mode);

/* 1 (default): GEMMs with >= 2 row tiles run on CTA pairs (cta_group::2
 * UMMA, 256-row tiles, each CTA stages half of the B tile); 0: one CTA per
 * 128-row tile.  The GPU tests run both. */
int stz_set_cluster(int on);

/* 1 (default): stride-1 unpadded convolutions run on the shifted-window
 * ("band") implicit GEMM, one shared-memory band per channel block serving
 * every tap; 2: padded stride-1 convolutions (and input gradients) too
 * (measured slower, kept for coverage); 0: the im2col TMA GEMM.  The GPU
 * tests run all three. */
int stz_set_band(int on);
/* split-K GEMMs: 1 the last split of each tile reduces in-kernel (when the
 * tiles cover the GPU and splits <= 4), 0 (default) a separate reduce pass;
 * tests compare both */
int stz_set_fixup(int on);

/* Force the TMA GEMM tile (tests / tuning): width bn in {64, 96, 128, 192,
 * 256}, cl = 2 for CTA pairs (required for 256; 64 / 96 run unpaired),
 * splits = K splits (0 = the cost model's count for that tile, never below the
 * per-tile accumulation cap).  bn = 0 restores the cost-model choice.  The
 * setting is process-global host state read at launch, so a caller brackets
 * one call with it (paper_1812_10624_b200/_lib.py: call, autotune_tiles). */
int stz_set_tile(int bn, int cl, int splits);

/* GEMM pipeline diagnostics (results are WRONG while set): 1 skips epilogue
 * stores, 2 skips the MMAs, 4 skips the TMA loads.  0 = normal. */
int stz_set_debug(int flags);

/* Tuning/experiment knob: cap the K extent one CTA accumulates (0 = auto). */
int stz_set_max_k_per_split(int k);

/* Conv2d forward, replaces tensor_core.py:161-181 (+ReLU :213-214 when
 * relu != 0).  x [N,C,H,W], w [O,C,k,k], b [O] -> y [N,O,OH,OW]. */
int stz_conv2d_fwd(const float* x, const float* w, const float* b, float* y, int N, int C, int H,
                   int W, int O, int k, int s, int p, int relu, void* ws, size_t ws_bytes,
                   void* stream);

/* Conv2d input gradient, replaces tensor_core.py:257-258,:260.
 * gy [N,O,OH,OW], w -> gx [N,C,H,W]; mask (nullable) = output of the ReLU
 * feeding this conv: gx is zeroed where mask <= 0 (tensor_core.py:291-293). */
int stz_conv2d_bwd_data(const float* gy, const float* w, float* gx, const float* mask, int N,
                        int C, int H, int W, int O, int k, int s, int p, void* ws,
                        size_t ws_bytes, void* stream);

/* Conv2d weight/bias gradient sums, replaces tensor_core.py:253-259.
 * x [N,C,H,W], gy [N,O,OH,OW] -> gw [O,C,k,k], gb [O] (gb nullable). */
int stz_conv2d_bwd_filter(const float* x, const float* gy, float* gw, float* gb, int N, int C,
                          int H, int W, int O, int k, int s, int p, void* ws, size_t ws_bytes,
                          void* stream);

/* FullyConnected forward y = x @ W + b (+ReLU), replaces tensor_core.py:205-211.
 * x [M,in], W [in,out], b [out] -> y [M,out]. */
int stz_fc_fwd(const float* x, const float* w, const float* b, float* y, int M, int in_dim,
               int out_dim, int relu, void* ws, size_t ws_bytes, void* stream);

/* FC input gradient gx = gy @ W^T, replaces tensor_core.py:286; optional
 * ReLU mask as in stz_conv2d_bwd_data. */
int stz_fc_bwd_data(const float* gy, const float* w, float* gx, const float* mask, int M,
                    int in_dim, int out_dim, void* ws, size_t ws_bytes, void* stream);

/* FC weight/bias gradient sums gW = x^T @ gy, gb = colsum(gy), replaces
 * tensor_core.py:287-288. */
int stz_fc_bwd_weight(const float* x, const float* gy, float* gw, float* gb, int M, int in_dim,
                      int out_dim, void* ws, size_t ws_bytes, void* stream);

/* MaxPool2d forward with first-max argmax (uint8 index kh*k+kw), replaces
 * tensor_core.py:183-198. */
int stz_maxpool2d_fwd(const float* x, float* y, uint8_t* arg, int N, int C, int H, int W, int k,
                      int s, void* stream);

/* MaxPool2d backward (gather form, float64 sums), replaces
 * tensor_core.py:263-276; optional ReLU mask on the pool input. */
int stz_maxpool2d_bwd(const float* gy, const uint8_t* arg, float* gx, const float* mask, int N,
                      int C, int H, int W, int k, int s, void* stream);

/* Standalone ReLU, replaces tensor_core.py:213-214 / :291-293 (src is the
 * ReLU input or output: both are > 0 at the same cells). */
int stz_relu_fwd(const float* x, float* y, size_t n, void* stream);
int stz_relu_bwd(const float* gy, const float* src, float* gx, size_t n, void* stream);

/* SoftmaxCrossEntropy forward+backward in one pass (float64 inside),
 * replaces tensor_core.py:216-228 and :295-299: per-sample losses [M] and
 * the gradient of the loss SUM, p - onehot, [M,C]. */
int stz_softmax_ce(const float* logits, const int* labels, float* losses, float* dlogits, int M,
                   int C, void* stream);

/* Deterministic float64 sum of n floats (the iteration loss sum,
 * stanza_runtime.py:273); accumulate != 0 adds into *out instead of
 * overwriting it (several FC workers' sums into one slot). */
int stz_sum_f32(const float* x, size_t n, double* out, int accumulate, void* stream);

/* Momentum SGD from gradient sums in the reference's exact fp32 op order,
 * replaces tensor_core.py:366-388: v = v*mu + g*inv_n; w = w - lr*v.
 * inv_n = float32(1)/float32(n_conv*K) computed by the caller. */
int stz_sgd_momentum(float* w, float* v, const float* g, size_t n, float lr, float mu,
                     float inv_n, void* stream);

/* dst += src (fp32).  Sums FC-replica gradient vectors when several FC
 * workers share one GPU -- the single-device stand-in for the FC-group
 * allreduce (stanza_runtime.py:320-337); on >1 GPU NCCL does this. */
int stz_vec_add(float* dst, const float* src, size_t n, void* stream);

/* ===========================================================================
 * Hot path on split-plane tensors (engine.BlockEngine).
 *
 * A logical fp32 tensor is three bf16 planes P0,P1,P2 (uint16 storage, plane
 * stride `ps` elements) with T = P0 + P1 + P2 exactly.  Conv activations are
 * NHWC with channels padded to C8 = roundup(C, 8); flat activations and FC
 * weights are row-major [rows][D8].  Conv weights are re-packed after every
 * update as wf[O][kh][kw][C8] (forward) and wd[C][kh][kw][O8] (input
 * gradient); FC W [in][out] as [in][out8] planes.  Every GEMM is the tcgen05
 * BF16x6 kernel; fp32 master parameters stay in the reference layouts.
 * ===========================================================================
 */

/* layout conversion (batch input, FC-block input, weights, debug read-back) */
int stzx_pack_nchw(const float* x, void* xp, size_t ps, int N, int C, int H, int W, int C8,
                   void* stream);
int stzx_unpack_nhwc(const void* xp, size_t ps, float* x, int N, int C, int H, int W, int C8,
                     void* stream);
int stzx_pack_rows(const float* x, void* xp, size_t ps, int M, int D, int D8, void* stream);
int stzx_unpack_rows(const void* xp, size_t ps, float* x, int M, int D, int D8, void* stream);
int stzx_pack_conv_w(const float* w, void* wf, size_t psf, void* wd, size_t psd, int O, int C,
                     int k, int C8, int O8, void* stream);
int stzx_nhwc_to_flat(const void* x, size_t psx, void* y, size_t psy, int N, int C, int H, int W,
                      int C8, int D8, void* stream);
int stzx_flat_to_nhwc(const void* y, size_t psy, void* x, size_t psx, int N, int C, int H, int W,
                      int C8, int D8, void* stream);

/* Conv2d forward (tensor_core.py:161-181 + fused ReLU): y NHWC [N][OH][OW][O8]. */
int stzx_conv_fwd(const void* x, size_t psx, const void* wf, size_t psw, const float* bias,
                  void* y, size_t psy, int N, int C8, int H, int W, int O, int O8, int k, int s,
                  int p, int relu, void* ws, size_t ws_bytes, void* stream);
/* Conv2d input gradient (tensor_core.py:257-260), ReLU mask = plane 0 of the
 * conv input when a ReLU produced it (nullable). */
int stzx_conv_dgrad(const void* g, size_t psg, const void* wd, size_t psw, void* gx, size_t psgx,
                    const void* mask, int N, int C, int C8, int H, int W, int O8, int k, int s,
                    int p, void* ws, size_t ws_bytes, void* stream);
/* Conv2d weight / bias gradient sums into fp32 [O,C,k,k] / [O] (tensor_core.py:253-259). */
int stzx_conv_wgrad(const void* x, size_t psx, const void* g, size_t psg, float* gw, float* gb,
                    int accumulate, int N, int C, int C8, int H, int W, int O, int O8, int k,
                    int s, int p, void* ws, size_t ws_bytes, void* stream);
/* FC forward (tensor_core.py:205-211): split output (y) or fp32 logits (y_f32). */
int stzx_fc_fwd(const void* x, size_t psx, const void* w, size_t psw, const float* bias, void* y,
                size_t psy, float* y_f32, int M, int in_dim, int in8, int out_dim, int out8,
                int relu, void* ws, size_t ws_bytes, void* stream);
/* FC input gradient (tensor_core.py:286) with optional ReLU mask. */
int stzx_fc_dgrad(const void* g, size_t psg, const void* w, size_t psw, void* gx, size_t psgx,
                  const void* mask, int M, int in_dim, int in8, int out8, void* ws,
                  size_t ws_bytes, void* stream);
/* FC weight / bias gradient sums (tensor_core.py:287-288).  The engine-level
 * weight-gradient entries take `accumulate`: 0 writes gw / gb, 1 adds into
 * them (micro-batches of one iteration summing into the same gradient). */
int stzx_fc_wgrad(const void* x, size_t psx, const void* g, size_t psg, float* gw, float* gb,
                  int accumulate, int M, int in_dim, int in8, int out_dim, int out8, void* ws,
                  size_t ws_bytes, void* stream);

/* Bias gradient on its own: out[n] (+)= sum over the R rows of split-plane
 * g [R][ld] of column n < N, float64 sums in a fixed order rounded once
 * (tensor_core.py:259 / :288) -- the colsum the weight-gradient entries run
 * when given gb, issued separately so it can run on another stream. */
int stzx_colsum(const void* g, size_t psg, int R, int N, int ld, float* out, int accumulate,
                void* ws, size_t ws_bytes, void* stream);

/* stzx_fc_wgrad fused with the momentum step when one FC worker owns the
 * layer: the weight gradient of W [in][out] is consumed in the
 * GEMM epilogue -- w / v (fp32 [in][out], 16-byte aligned) get
 * tensor_core.py:366-388's update (v = mu*v + g*inv_n; w -= lr*v) and the
 * split-plane GEMM copy `planes` ([in][out8], psw elements apart) is
 * rewritten; gW is never stored.  accumulate = 1 adds the earlier
 * micro-batches' sum held in gw first.  With wb != NULL the bias gradient
 * (column sums of g, written to gb) updates (wb, vb) the same way.  The
 * flat-block update then skips these ranges (stz_plane_range with
 * planes == NULL and D == 0). */
int stzx_fc_wgrad_sgd(const void* x, size_t psx, const void* g, size_t psg, float* w, float* v,
                      void* planes, size_t psw, float* wb, float* vb, float* gw, float* gb,
                      int accumulate, int M, int in_dim, int in8, int out_dim, int out8, float lr,
                      float mu, float inv_n, void* ws, size_t ws_bytes, void* stream);
/* MaxPool2d (tensor_core.py:183-198 / :263-276); flat_ld > 0 selects the
 * CHW-flat [N][flat_ld] layout for y / gy (the FC-block boundary). */
int stzx_maxpool_fwd(const void* x, size_t psx, void* y, size_t psy, uint8_t* arg, int N, int C,
                     int C8, int H, int W, int k, int s, int flat_ld, void* stream);
int stzx_maxpool_bwd(const void* gy, size_t psg, const uint8_t* arg, void* gx, size_t psx,
                     const void* mask, int N, int C, int C8, int H, int W, int k, int s,
                     int flat_ld, void* stream);
/* standalone ReLU on split planes */
int stzx_relu_fwd(const void* x, size_t psx, void* y, size_t psy, size_t n, void* stream);
int stzx_relu_bwd(const void* gy, size_t psg, const void* src, void* gx, size_t psx, size_t n,
                  void* stream);
/* Forward of a strided conv as its space-to-depth stride-1 form (ks x ks
 * taps over Cs8-channel blocks; channels >= Creal are zero padding, so the
 * shifted-window kernel skips their 16-deep k steps). */
int stzx_conv_fwd_s2d(const void* x, size_t psx, const void* wf, size_t psw, const float* bias,
                      void* y, size_t psy, int N, int Creal, int Cs8, int Hs, int Ws, int O, int O8,
                      int ks, int relu, void* ws, size_t ws_bytes, void* stream);
/* Space-to-depth form of a strided first conv (AlexNet conv1, 11x11/4 on 3
 * channels): the padded input is regrouped into s x s blocks, giving a
 * stride-1 ceil(k/s) x ceil(k/s) conv over C*s*s (padded to Cs8) channels
 * that runs on the TMA kernel; the forward uses stzx_conv_fwd on the packed
 * tensors, the weight gradient maps back to [O,C,k,k]. */
int stzx_pack_s2d(const float* x, void* xp, size_t ps, int N, int C, int H, int W, int s, int p,
                  int Hs, int Ws, int Cs8, void* stream);
int stzx_pack_conv_w_s2d(const float* w, void* wf, size_t ps, int O, int C, int k, int s,
                         int Cs8, void* stream);
int stzx_conv_wgrad_s2d(const void* x, size_t psx, const void* g, size_t psg, float* gw,
                        float* gb, int accumulate, int N, int C, int Cs8, int Hs, int Ws, int O,
                        int O8, int k, int s, void* ws, size_t ws_bytes, void* stream);
/* ResNet-trunk kinds.  The reference has no such layers
 * (tensor_core.py:37-74 stops at SoftmaxCrossEntropy), so there is no
 * reference entry point to replace; semantics are the oracle's
 * (oracle/stanza_oracle.py: bn_forward, bn_backward, gap_forward, gap_backward,
 * residual), parity
 * unpinned.  BatchNorm runs in training mode with float64 statistics per
 * group of `group` samples (one CONV worker's batch); `stats` is caller-owned
 * double [N/group][C8][2] = (mean, rstd), written by the forward and read by
 * the backward.  y = ((x-mean)*rstd)*gamma + beta (+ res, fp32 add) (ReLU). */
int stzx_bn_fwd(const void* x, size_t psx, const float* gamma, const float* beta, const void* res,
                size_t psr, void* y, size_t psy, double* stats, int N, int HW, int C, int C8,
                int group, float eps, int relu, void* ws, size_t ws_bytes, void* stream);
/* dgamma / dbeta batch sums (added with `accumulate`), gx nullable; `mask`
 * (nullable): g is the gradient of a ReLU output, masked where plane 0 of
 * `mask` (that output) is not > 0 (a residual block's final ReLU).
 * `gbias_in` (nullable, needs gx): the batch sum of gx per channel -- the
 * gradient of a bias added to x (the producing conv's) -- from the same pass
 * that writes gx (float64 sums of the fp32 gx values, fixed order). */
int stzx_bn_bwd(const void* g, size_t psg, const void* mask, const void* x, size_t psx,
                const double* stats,
                const float* gamma, float* ggamma, float* gbeta, float* gbias_in, int accumulate,
                void* gx, size_t psgx, int N, int HW, int C, int C8, int group, void* ws,
                size_t ws_bytes, void* stream);
/* global average pool NHWC [N][HW][C8] <-> rows [N][C8] (float64 sums / HW) */
int stzx_gap_fwd(const void* x, size_t psx, void* y, size_t psy, int N, int HW, int C8,
                 void* stream);
int stzx_gap_bwd(const void* gy, size_t psg, void* gx, size_t psx, int N, int HW, int C8,
                 void* stream);
/* Every conv layer's weight repack in one launch (after each update): job
 * i = stzx_pack_conv2_w's arguments (wd may be NULL: no input-gradient copy);
 * at most 160 jobs. */
typedef struct {
  const float* w;
  void* wf;
  void* wd;
  size_t psf, psd;
  int O, C, kh, kw, C8, O8;
} stz_conv_pack;
int stzx_pack_conv_w_multi(const stz_conv_pack* jobs, int n, void* stream);

/* ---- Inception-V3 kinds (not in the reference: semantics
 * restated in oracle/stanza_oracle.py, parity unpinned) ---- */
/* Rectangular conv (kh x kw kernel, padding (ph, pw): 1xn / nx1) on the TMA
 * im2col path (C8 % 32 == 0 for fwd / wgrad, O8 % 32 and stride 1 for
 * dgrad); the square entries above are these with kh = kw, ph = pw. */
int stzx_pack_conv2_w(const float* w, void* wf, size_t psf, void* wd, size_t psd, int O, int C,
                      int kh, int kw, int C8, int O8, void* stream);
int stzx_conv2_fwd(const void* x, size_t psx, const void* wf, size_t psw, const float* bias,
                   void* y, size_t psy, int N, int C8, int H, int W, int O, int O8, int kh, int kw,
                   int s, int ph, int pw, int relu, void* ws, size_t ws_bytes, void* stream);
int stzx_conv2_dgrad(const void* g, size_t psg, const void* wd, size_t psw, void* gx, size_t psgx,
                     const void* mask, int N, int C, int C8, int H, int W, int O8, int kh, int kw,
                     int s, int ph, int pw, void* ws, size_t ws_bytes, void* stream);
int stzx_conv2_wgrad(const void* x, size_t psx, const void* g, size_t psg, float* gw, float* gb,
                     int accumulate, int N, int C, int C8, int H, int W, int O, int O8, int kh,
                     int kw, int s, int ph, int pw, void* ws, size_t ws_bytes, void* stream);
/* AvgPool2d, zero padding p (2p <= k), every window divided by k*k: float64
 * window sums (forward) / float64 sums of g/(k*k) over covering windows
 * (backward, gather form), NHWC split planes [N][H][W][C8]. */
int stzx_avgpool_fwd(const void* x, size_t psx, void* y, size_t psy, int N, int C8, int H,
                     int W, int k, int s, int p, void* stream);
int stzx_avgpool_bwd(const void* gy, size_t psg, void* gx, size_t psx, int N, int C8, int H, int W,
                     int k, int s, int p, void* stream);
/* Channel-slice copy of split-plane rows (the Inception concat and its
 * backward): dst[r][d0 + c] = src[r][s0 + c], c < C; row pitches src8 / dst8;
 * C, s0, d0, pitches multiples of 8.  mask != NULL (pitch mask8, offset m0):
 * zero where the mask (a ReLU output) is not > 0 -- a branch's closing ReLU
 * backward fused into the copy. */
int stzx_copy_channels(const void* src, size_t pss, int src8, int s0, void* dst, size_t psd,
                       int dst8, int d0, size_t rows, int C, const void* mask, int mask8, int m0,
                       void* stream);
/* y = ((x0 + x1) + x2) + x3 (fp32 RN, the first nin of 2..4 inputs, host
 * arrays of pointers / plane strides), n a multiple of 8: the Inception
 * concat's input gradient in branch order. */
int stzx_add_n(const void* const* xs, const size_t* ps, int nin, void* y, size_t psy, size_t n,
               void* stream);

/* y = a + b elementwise (fp32 RN), n a multiple of 8: residual input
 * gradients; b masked by a ReLU output (plane 0 > 0) when mask_b != NULL */
int stzx_add(const void* a, size_t psa, const void* b, size_t psb, const void* mask_b, void* y,
             size_t psy, size_t n, void* stream);
/* SoftmaxCE on fp32 logits -> losses + split dlogits [M][C8]. */
int stzx_softmax_ce(const float* logits, const int* labels, float* losses, void* dz, size_t psd,
                    int M, int C, int C8, void* stream);

/* ===========================================================================
 * Gradient exchange + update over NVLink peer memory (replaces the
 * reference's _exchange_phase, stanza_runtime.py:309-338 -> allreduce_sum,
 * collectives.py:117-157, and _update_phase, stanza_runtime.py:340-350 ->
 * unpack_vector tensor_core.py:510-524 + sgd_step tensor_core.py:366-388).
 *
 * One role group (the CONV workers, or the FC workers when n_fc > 1) of
 * nranks processes, one per GPU.  Each member owns three device buffers that
 * every other member maps through CUDA IPC: its flat gradient vector, a
 * reduced-gradient vector of the same length and a block of
 * STZ_PEER_FLAG_WORDS uint32 flag words (zeroed once).  Pointer arrays are
 * HOST arrays of nranks device pointers indexed by group rank (the local
 * member's own entries are its local pointers).
 * ===========================================================================
 */
#define STZ_IPC_HANDLE_BYTES 64
#define STZ_PEER_FLAG_WORDS 32

/* CUDA IPC: handle (STZ_IPC_HANDLE_BYTES) of the allocation holding dptr and
 * dptr's byte offset in it; open maps a peer's allocation (returns its base),
 * close unmaps it. */
int stz_ipc_handle(const void* dptr, void* handle, size_t* offset);
int stz_ipc_open(const void* handle, void** base);
int stz_ipc_close(void* base);

/* Timeout after which a peer wait (exchange barrier, link get) gives up: it
 * writes a status word (flags[17] of the exchange block, word
 * STZ_LINK_STATUS of the link block), later kernels of that member skip
 * their work, and the host raises MissingSource (the reference's
 * stanza_runtime.py:37-38, :77-82, :295-299); 0 restores the default 60 s. */
int stz_set_peer_timeout_ms(unsigned long long ms);

/* Stream-ordered barrier of the group: returns (on the stream) once every
 * member's stream reached its matching barrier call. */
int stz_peer_barrier(unsigned* const* flags, int nranks, int me, void* stream);

/* Member `me` sums chunk `me` (256-byte aligned, ceil(n/nranks) rounded up)
 * of every member's gradient in group-rank order and stores the sum into the
 * same chunk of every member's reduced buffer. */
int stz_peer_reduce_push(const float* const* grads, float* const* red, int nranks, int me,
                         size_t n, void* stream);

/* A slice [off, off+len) of the flat parameter vector whose split-plane GEMM
 * copy is a row-major [len/D][D8] matrix (FC W [in][out8], planes ps
 * elements apart); off % 4 == 0.  planes == NULL with D == 0 marks a slice
 * that the update skips (already updated by stzx_fc_wgrad_sgd). */
typedef struct {
  size_t off, len;
  void* planes;
  size_t ps;
  int D, D8;
} stz_plane_range;

/* stz_sgd_momentum fused with the split-plane weight repack of the given
 * ranges (sorted, disjoint, <= 16 including the gaps between them). */
int stz_sgd_momentum_pack(float* w, float* v, const float* g, size_t n, float lr, float mu,
                          float inv_n, const stz_plane_range* ranges, int nranges, void* stream);

/* The whole exchange + update of one member: barrier, reduce-push, barrier,
 * then SGD + repack of its replica from its reduced buffer (nranks == 1: SGD
 * + repack from grads[0]).  Every member ends with bit-identical w, v. */
int stz_allreduce_sgd(const float* const* grads, float* const* red, unsigned* const* flags,
                      int nranks, int me, float* w, float* v, size_t n, float lr, float mu,
                      float inv_n, const stz_plane_range* ranges, int nranges, void* stream);

/* ===========================================================================
 * CONV <-> FC link over peer memory: the many-to-one activation gather
 * (_activations_phase + collect_group_activations, stanza_runtime.py:64-85,
 * :228-253) and the one-to-many boundary-gradient scatter (_boundary_phase,
 * :278-307) of the layer-separated step, one message per (CONV worker,
 * micro-batch), 4 bytes per element on the link.
 *
 * Every rank owns a link flag block of STZ_LINK_FLAG_WORDS uint32 (zeroed
 * once; IPC-mapped by its link peers) and an fp32 staging buffer for what it
 * receives.  Per step: stz_link_begin on every rank; the sender's
 * stz_link_put stores its split-plane rows as fp32 into the receiver's
 * staging rows (and labels into the receiver's label rows) and then publishes
 * its epoch in the receiver's message slot; the receiver's stz_link_get waits
 * for the slots of one micro-batch and splits the staged rows into its local
 * split-plane buffer.  All stream-ordered device work (no host sync).
 * ===========================================================================
 */
#define STZ_LINK_FLAG_WORDS 256
#define STZ_LINK_SLOTS 192
#define STZ_LINK_EPOCH 240
#define STZ_LINK_STATUS 241

/* epoch += 1 on the rank's link block (once per step, before its puts/gets) */
int stz_link_begin(unsigned* flags, void* stream);

/* src: split planes [rows][D8] (plane stride ps, 16-byte aligned); dst: the
 * receiver's fp32 staging rows [rows][D] (peer pointer); labels (optional):
 * rows int32 copied to labels_dst (peer pointer); then
 * *remote_slot = this rank's epoch (release, system scope). */
int stz_link_put(const void* src, size_t ps, int rows, int D, int D8, float* dst,
                 const int* labels, int* labels_dst, unsigned* my_flags, unsigned* remote_slot,
                 void* stream);

/* Wait until my_flags[slot0 + i*slot_stride] >= this rank's epoch for every
 * i < nslots (timeout: status word, see stz_set_peer_timeout_ms), then
 * src fp32 [rows][D] -> split planes dst [rows][D8] (plane stride ps). */
int stz_link_get(const float* src, int rows, int D, void* dst, size_t ps, int D8,
                 unsigned* my_flags, int slot0, int nslots, int slot_stride, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* STANZA_B200_H */
