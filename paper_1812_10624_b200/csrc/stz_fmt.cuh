// Split-plane format kernels: packing / unpacking, weight layouts, max-pool,
// ReLU, softmax-CE and column sums on the hot-path formats (stz_split.cuh).
//
// Reference semantics restated (file:line under /root/reference/pkg/src/stanza):
//   maxpool fwd/bwd  tensor_core.py:183-198 / :263-276 (first max, fp64 sums)
//   relu fwd/bwd     tensor_core.py:213-214 / :291-293
//   softmax-CE       tensor_core.py:216-228 / :295-299 (fp64 inside)
//   bias sums        tensor_core.py:259, :288 (fp64)
//   flatten          tensor_core.py:200-203 (CHW order)
#pragma once

#include "stz_split.cuh"

namespace stz {

#define STZ_GRID_LOOP(i, total)                                                     \
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < (total); \
       i += (size_t)gridDim.x * blockDim.x)

// fp32 NCHW -> NHWC split planes (channels padded to C8 with zeros)
__global__ void pack_nchw_kernel(const float* __restrict__ x, bf16_t* __restrict__ xp, size_t ps,
                                 int N, int C, int H, int W, int C8) {
  const int chunks = C8 / 8;
  const size_t total = (size_t)N * H * W * chunks;
  STZ_GRID_LOOP(i, total) {
    const int cc = (int)(i % chunks);
    const size_t pix = i / chunks;  // (n, h, w)
    const int hw = (int)(pix % ((size_t)H * W));
    const size_t n = pix / ((size_t)H * W);
    float v[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int c = cc * 8 + j;
      v[j] = c < C ? x[(n * C + c) * H * W + hw] : 0.f;
    }
    store_split8(xp + pix * C8 + cc * 8, ps, v);
  }
}

// NHWC split planes -> fp32 NCHW
__global__ void unpack_nhwc_kernel(const bf16_t* __restrict__ xp, size_t ps, float* __restrict__ x,
                                   int N, int C, int H, int W, int C8) {
  const size_t total = (size_t)N * C * H * W;
  STZ_GRID_LOOP(i, total) {
    const int hw = (int)(i % ((size_t)H * W));
    const int c = (int)((i / ((size_t)H * W)) % C);
    const size_t n = i / ((size_t)C * H * W);
    x[i] = load_split(xp, ps, (n * H * W + hw) * C8 + c);
  }
}

// fp32 rows [M][D] -> split planes [M][D8]
__global__ void pack_rows_kernel(const float* __restrict__ x, bf16_t* __restrict__ xp, size_t ps,
                                 int M, int D, int D8) {
  const int chunks = D8 / 8;
  const size_t total = (size_t)M * chunks;
  STZ_GRID_LOOP(i, total) {
    const int cc = (int)(i % chunks);
    const size_t m = i / chunks;
    float v[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int d = cc * 8 + j;
      v[j] = d < D ? x[m * D + d] : 0.f;
    }
    store_split8(xp + m * D8 + cc * 8, ps, v);
  }
}

__global__ void unpack_rows_kernel(const bf16_t* __restrict__ xp, size_t ps, float* __restrict__ x,
                                   int M, int D, int D8) {
  const size_t total = (size_t)M * D;
  STZ_GRID_LOOP(i, total) {
    x[i] = load_split(xp, ps, (i / D) * D8 + i % D);
  }
}

// conv W [O, C, k, k] -> forward B planes wf[O][tap][C8] and input-gradient
// B planes wd[C][tap][O8]  (tap = kh*k + kw; zeros in the channel padding)
__global__ void pack_conv_w_kernel(const float* __restrict__ w, bf16_t* __restrict__ wf,
                                   size_t psf, bf16_t* __restrict__ wd, size_t psd, int O, int C,
                                   int kk, int C8, int O8) {
  const size_t nf = (size_t)O * kk * C8, nd = (size_t)C * kk * O8;
  STZ_GRID_LOOP(i, nf + nd) {
    if (i < nf) {
      const int c = (int)(i % C8);
      const int tap = (int)((i / C8) % kk);
      const int o = (int)(i / ((size_t)C8 * kk));
      store_split(wf, psf, i, c < C ? w[((size_t)o * C + c) * kk + tap] : 0.f);
    } else {
      const size_t j = i - nf;
      const int o = (int)(j % O8);
      const int tap = (int)((j / O8) % kk);
      const int c = (int)(j / ((size_t)O8 * kk));
      store_split(wd, psd, j, o < O ? w[((size_t)o * C + c) * kk + tap] : 0.f);
    }
  }
}

// NHWC split planes [N][H][W][C8] <-> CHW-flat split planes [N][D8]
// (flatten in the reference's CHW order when no max-pool precedes it)
__global__ void nhwc_to_flat_kernel(const bf16_t* __restrict__ x, size_t psx, bf16_t* __restrict__ y,
                                    size_t psy, int N, int C, int H, int W, int C8, int D8) {
  const size_t D = (size_t)C * H * W;
  STZ_GRID_LOOP(i, (size_t)N * D8) {
    const size_t n = i / D8, d = i % D8;
    if (d >= D) {
      store_split(y, psy, i, 0.f);
      continue;
    }
    const int c = (int)(d / ((size_t)H * W)), hw = (int)(d % ((size_t)H * W));
    const size_t src = (n * H * W + hw) * C8 + c;
    y[i] = x[src];
    y[i + psy] = x[src + psx];
    y[i + 2 * psy] = x[src + 2 * psx];
  }
}

__global__ void flat_to_nhwc_kernel(const bf16_t* __restrict__ y, size_t psy, bf16_t* __restrict__ x,
                                    size_t psx, int N, int C, int H, int W, int C8, int D8) {
  STZ_GRID_LOOP(i, (size_t)N * H * W * C8) {
    const int c = (int)(i % C8);
    const size_t pix = i / C8;
    const int hw = (int)(pix % ((size_t)H * W));
    const size_t n = pix / ((size_t)H * W);
    if (c >= C) {
      store_split(x, psx, i, 0.f);
      continue;
    }
    const size_t src = n * D8 + (size_t)c * H * W + hw;
    x[i] = y[src];
    x[i + psx] = y[src + psy];
    x[i + 2 * psx] = y[src + 2 * psy];
  }
}

// max-pool forward on NHWC split planes.  Output NHWC [N][OH][OW][C8]
// (flat_ld == 0) or CHW-flat [N][flat_ld] (the FC-block input, reference
// flatten order).  arg (uint8, kh*k+kw of the first maximum) is indexed
// NHWC [N][OH][OW][C8] in both modes.
__global__ void maxpool_fwd_split_kernel(const bf16_t* __restrict__ x, size_t psx,
                                         bf16_t* __restrict__ y, size_t psy,
                                         uint8_t* __restrict__ arg, int N, int C, int C8, int H,
                                         int W, int k, int s, int OH, int OW, int flat_ld) {
  STZ_GRID_LOOP(i, (size_t)N * OH * OW * C8) {
    const int c = (int)(i % C8);
    const size_t opix = i / C8;
    const int ow = (int)(opix % OW), oh = (int)((opix / OW) % OH);
    const size_t n = opix / ((size_t)OH * OW);
    float best = 0.f;
    int bi = 0;
    if (c < C) {
      const size_t base = ((n * H + (size_t)oh * s) * W + (size_t)ow * s) * C8 + c;
      best = load_split(x, psx, base);
      for (int kh = 0; kh < k; ++kh)
        for (int kw = 0; kw < k; ++kw) {
          const float v = load_split(x, psx, base + ((size_t)kh * W + kw) * C8);
          if (v > best) {
            best = v;
            bi = kh * k + kw;
          }
        }
    }
    arg[i] = (uint8_t)bi;
    if (flat_ld == 0) {
      store_split(y, psy, i, best);
    } else if (c < C) {
      store_split(y, psy, n * flat_ld + ((size_t)c * OH + oh) * OW + ow, best);
    }
  }
}

// zero the CHW-flat tail columns [C*OH*OW, flat_ld) once per buffer
__global__ void zero_flat_tail_kernel(bf16_t* __restrict__ y, size_t psy, int N, int D, int ld) {
  const int tail = ld - D;
  STZ_GRID_LOOP(i, (size_t)N * tail) {
    store_split(y, psy, (i / tail) * ld + D + i % tail, 0.f);
  }
}

// max-pool backward, gather form: every input cell (NHWC) sums in float64,
// in the reference's (kh, kw) order, the output gradients whose argmax it
// was; gy is NHWC (flat_ld == 0) or CHW-flat.  mask = plane 0 of the pool
// input when a ReLU fed the pool (its backward fused here).
__global__ void maxpool_bwd_split_kernel(const bf16_t* __restrict__ gy, size_t psg,
                                         const uint8_t* __restrict__ arg,
                                         bf16_t* __restrict__ gx, size_t psx,
                                         const bf16_t* __restrict__ mask, int N, int C, int C8,
                                         int H, int W, int k, int s, int OH, int OW,
                                         int flat_ld) {
  STZ_GRID_LOOP(i, (size_t)N * H * W * C8) {
    const int c = (int)(i % C8);
    const size_t pix = i / C8;
    const int w = (int)(pix % W), h = (int)((pix / W) % H);
    const size_t n = pix / ((size_t)H * W);
    double acc = 0.0;
    if (c < C) {
      const int th = h - k + 1, tw = w - k + 1;
      const int oh_lo = th <= 0 ? 0 : (th + s - 1) / s, ow_lo = tw <= 0 ? 0 : (tw + s - 1) / s;
      const int oh_hi = min(OH - 1, h / s), ow_hi = min(OW - 1, w / s);
      for (int oh = oh_hi; oh >= oh_lo; --oh)
        for (int ow = ow_hi; ow >= ow_lo; --ow) {
          const size_t o = ((n * OH + oh) * OW + ow) * C8 + c;
          if (arg[o] == (uint8_t)((h - oh * s) * k + (w - ow * s))) {
            const size_t gi = flat_ld == 0 ? o : n * flat_ld + ((size_t)c * OH + oh) * OW + ow;
            acc += (double)load_split(gy, psg, gi);
          }
        }
    }
    float v = (float)acc;
    if (mask && !(bf2f(mask[i]) > 0.f)) v = 0.f;
    store_split(gx, psx, i, v);
  }
}

// standalone ReLU on split planes (sign and zero-ness live in plane 0)
__global__ void relu_fwd_split_kernel(const bf16_t* __restrict__ x, size_t psx,
                                      bf16_t* __restrict__ y, size_t psy, size_t n) {
  STZ_GRID_LOOP(i, n) {
    const bool neg = bf2f(x[i]) < 0.f;
    y[i] = neg ? 0 : x[i];
    y[i + psy] = neg ? 0 : x[i + psx];
    y[i + 2 * psy] = neg ? 0 : x[i + 2 * psx];
  }
}

__global__ void relu_bwd_split_kernel(const bf16_t* __restrict__ gy, size_t psg,
                                      const bf16_t* __restrict__ src, bf16_t* __restrict__ gx,
                                      size_t psx, size_t n) {
  STZ_GRID_LOOP(i, n) {
    const bool keep = bf2f(src[i]) > 0.f;
    gx[i] = keep ? gy[i] : 0;
    gx[i + psx] = keep ? gy[i + psg] : 0;
    gx[i + 2 * psx] = keep ? gy[i + 2 * psg] : 0;
  }
}

template <int T>
__device__ double blk_sum(double v, double* red) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  if (w == 0) {
    v = l < T / 32 ? red[l] : 0.0;
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (l == 0) red[0] = v;
  }
  __syncthreads();
  return red[0];
}

template <int T>
__device__ double blk_max(double v, double* red) {
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  if (w == 0) {
    v = l < T / 32 ? red[l] : -INFINITY;
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    if (l == 0) red[0] = v;
  }
  __syncthreads();
  return red[0];
}

// softmax-CE on fp32 logits [M][C]: per-sample loss (fp32) and the gradient
// of the loss SUM, p - onehot, written as split planes [M][C8]
__global__ void __launch_bounds__(256) softmax_ce_split_kernel(
    const float* __restrict__ z, const int* __restrict__ labels, float* __restrict__ loss,
    bf16_t* __restrict__ dz, size_t psd, int C, int C8) {
  __shared__ double red[32];
  const int row = blockIdx.x;
  const float* zr = z + (size_t)row * C;
  double mx = -INFINITY;
  for (int j = threadIdx.x; j < C; j += 256) mx = fmax(mx, (double)zr[j]);
  mx = blk_max<256>(mx, red);
  double se = 0.0;
  for (int j = threadIdx.x; j < C; j += 256) se += exp((double)zr[j] - mx);
  se = blk_sum<256>(se, red);
  const int lab = labels[row];
  for (int j = threadIdx.x; j < C8; j += 256) {
    float g = 0.f;
    if (j < C) {
      double p = exp((double)zr[j] - mx) / se;
      if (j == lab) p -= 1.0;
      g = (float)p;
    }
    store_split(dz, psd, (size_t)row * C8 + j, g);
  }
  if (threadIdx.x == 0) loss[row] = (float)(-log(exp((double)zr[lab] - mx) / se));
}

// column sums of split planes [R][ld] (first N columns) in float64, two
// deterministic passes: per-block partials, then a fixed-order final sum.
constexpr int CS_ROWS = 256;  // rows per partial block

__global__ void __launch_bounds__(256) colsum_partial_kernel(const bf16_t* __restrict__ g,
                                                             size_t ps, int R, int N, int ld,
                                                             double* __restrict__ part) {
  const int r0 = blockIdx.x * CS_ROWS;
  const int r1 = min(R, r0 + CS_ROWS);
  for (int c0 = blockIdx.y * 256; c0 < N; c0 += 256 * gridDim.y) {
    const int c = c0 + threadIdx.x;
    double s = 0.0;
    if (c < N)
      for (int r = r0; r < r1; ++r) s += (double)load_split(g, ps, (size_t)r * ld + c);
    if (c < N) part[(size_t)blockIdx.x * N + c] = s;
  }
}

__global__ void colsum_final_kernel(const double* __restrict__ part, int blocks, int N,
                                    float* __restrict__ out) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= N) return;
  double s = 0.0;
  for (int b = 0; b < blocks; ++b) s += part[(size_t)b * N + c];
  out[c] = (float)s;
}

}  // namespace stz
