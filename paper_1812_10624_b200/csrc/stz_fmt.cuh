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
                                 int N, int C, int H, int W, int C8, FastDiv d_chunks,
                                 FastDiv d_hw) {
  const uint32_t total = (uint32_t)N * H * W * (C8 / 8);
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    uint32_t pix, cc, n, hw;
    d_chunks.divmod(i, pix, cc);  // pix = (n, h, w)
    d_hw.divmod(pix, n, hw);
    float v[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int c = (int)cc * 8 + j;
      v[j] = c < C ? __ldg(x + ((size_t)n * C + c) * H * W + hw) : 0.f;
    }
    store_split8(xp + (size_t)pix * C8 + cc * 8, ps, v);
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

// Space-to-depth for a strided first conv (AlexNet conv1: 11x11 stride 4 on
// 3 channels).  With the input zero-padded by p, window row ih' = oh*s + kh;
// s2d pixel (i, j) holds channels c' = (dy*s + dx)*C + c of padded input
// (i*s + dy, j*s + dx).  The conv becomes a stride-1, unpadded k' x k'
// (k' = ceil(k/s)) conv over C*s*s channels: tap (kh', kw'), channel c'
// carries original tap (kh'*s + dy, kw'*s + dx) -- zero where that exceeds k.
// fp32 NCHW -> s2d NHWC split planes [N][Hs][Ws][Cs8]
__global__ void pack_s2d_kernel(const float* __restrict__ x, bf16_t* __restrict__ xp, size_t ps,
                                int N, int C, int H, int W, int s, int pad, int Hs, int Ws,
                                int Cs8, FastDiv d_chunks, FastDiv d_ws, FastDiv d_hs) {
  const uint32_t total = (uint32_t)N * Hs * Ws * (Cs8 / 8);
  const int Cs = C * s * s;
  for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < total; t += gridDim.x * blockDim.x) {
    uint32_t pix, cc, r, j, n, i;
    d_chunks.divmod(t, pix, cc);
    d_ws.divmod(pix, r, j);
    d_hs.divmod(r, n, i);
    float v[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int cp = (int)cc * 8 + q;
      float val = 0.f;
      if (cp < Cs) {
        const int c = cp % C, d = cp / C, dy = d / s, dx = d % s;
        const int ih = (int)i * s + dy - pad, iw = (int)j * s + dx - pad;
        if ((unsigned)ih < (unsigned)H && (unsigned)iw < (unsigned)W)
          val = __ldg(x + (((size_t)n * C + c) * H + ih) * W + iw);
      }
      v[q] = val;
    }
    store_split8(xp + (size_t)pix * Cs8 + cc * 8, ps, v);
  }
}

// conv W [O, C, k, k] -> s2d forward B planes wf[O][kh'*ks + kw'][Cs8]
__global__ void pack_s2d_w_kernel(const float* __restrict__ w, bf16_t* __restrict__ wf,
                                  size_t ps, int O, int C, int k, int s, int ks, int Cs8) {
  const size_t total = (size_t)O * ks * ks * Cs8;
  const int Cs = C * s * s;
  STZ_GRID_LOOP(i, total) {
    const int cp = (int)(i % Cs8);
    const int tap = (int)((i / Cs8) % (ks * ks));
    const int o = (int)(i / ((size_t)Cs8 * ks * ks));
    float val = 0.f;
    if (cp < Cs) {
      const int c = cp % C, d = cp / C, dy = d / s, dx = d % s;
      const int kh = (tap / ks) * s + dy, kw = (tap % ks) * s + dx;
      if (kh < k && kw < k) val = w[(((size_t)o * C + c) * k + kh) * k + kw];
    }
    store_split(wf, ps, i, val);
  }
}

// conv W [O, C, k, k] -> forward B planes wf[O][tap][C8] (tap = kh*k + kw)
// and input-gradient B planes wd[C][t][O8] with FLIPPED taps
// t = (k-1-kh)*k + (k-1-kw), the order in which the input gradient walks
// the output-gradient window (zeros in the channel padding)
__global__ void pack_conv_w_kernel(const float* __restrict__ w, bf16_t* __restrict__ wf,
                                   size_t psf, bf16_t* __restrict__ wd, size_t psd, int O, int C,
                                   int kk, int C8, int O8, int ksz) {
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
      const int t = (int)((j / O8) % kk);
      const int c = (int)(j / ((size_t)O8 * kk));
      const int tap = kk - 1 - t;  // (k-1-th)*k + (k-1-tw)
      store_split(wd, psd, j, o < O ? w[((size_t)o * C + c) * kk + tap] : 0.f);
    }
  }
}

// Every conv layer of a block in one launch (the refresh after each update):
// job j covers elements [start[j], start[j+1]) of the concatenated
// [forward copy | input-gradient copy] ranges, laid out as pack_conv_w_kernel's
struct ConvPackJob {
  const float* w;
  bf16_t* wf;
  bf16_t* wd;
  size_t psf, psd;
  int O, C, kk, C8, O8;
  int cb;          // input channels per tile (even; 32 o x cb c x kk taps staged in shared memory)
  int tile0;       // first tile of this job
  int vec;         // cb % 8 == 0 and 16-byte aligned planes: 8-element stores
};
constexpr int kMaxConvPack = 160;
constexpr int kPackSpan = 288;   // cb * kk words per output channel in a tile
struct ConvPackTable {
  int n, tiles;
  ConvPackJob j[kMaxConvPack];
};

// One tile = 32 output channels x cb input channels x all kk taps of one
// job: read w[o][c0 .. c0+cb)[*] as contiguous runs (coalesced), stage it in
// shared memory, then write the forward operand wf [O][kk][C8] (c-runs) and
// the flipped input-gradient operand wd [C][kk][O8] (o-runs) from it, two
// elements per 4-byte store.  Padded channels are zeros.
__global__ void __launch_bounds__(256) pack_conv_w_multi_kernel(const __grid_constant__ ConvPackTable t) {
  __shared__ float tile[32 * (kPackSpan + 1)];
  int lo = 0, hi = t.n - 1;           // last job with tile0 <= blockIdx.x
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (t.j[mid].tile0 <= (int)blockIdx.x) lo = mid; else hi = mid - 1;
  }
  const ConvPackJob& J = t.j[lo];
  const int kk = J.kk, cb = J.cb, span = cb * kk, ld = span + 1;
  const int ncb = (J.C8 + cb - 1) / cb;
  const int tl = (int)blockIdx.x - J.tile0;
  const int o0 = (tl / ncb) * 32, c0 = (tl % ncb) * cb;
  for (int idx = threadIdx.x; idx < 32 * span; idx += blockDim.x) {
    const int ol = idx / span, rem = idx - ol * span;
    const int o = o0 + ol, c = c0 + rem / kk;
    tile[ol * ld + rem] = (o < J.O && c < J.C) ? __ldg(J.w + ((size_t)o * J.C + c0) * kk + rem) : 0.f;
  }
  __syncthreads();
  if (J.vec) {
    // wf[o][tap][c], c fastest: 8 channels per thread, one 16-byte store per plane
    const int cg8 = cb >> 3;
    for (int idx = threadIdx.x; idx < 32 * kk * cg8; idx += blockDim.x) {
      const int ol = idx / (kk * cg8), rem = idx - ol * kk * cg8;
      const int tap = rem / cg8, cl = 8 * (rem - tap * cg8);
      const int o = o0 + ol, c = c0 + cl;
      if (o >= J.O || c >= J.C8) continue;
      float v[8];
#pragma unroll
      for (int t = 0; t < 8; ++t) v[t] = tile[ol * ld + (cl + t) * kk + tap];
      store_split8(J.wf + ((size_t)o * kk + tap) * J.C8 + c, J.psf, v);
    }
    if (!J.wd) return;
    // wd[c][tt][o], o fastest, tap = kk - 1 - tt: 8 output channels per thread
    for (int idx = threadIdx.x; idx < 4 * span; idx += blockDim.x) {
      const int cl = idx / (4 * kk), rem = idx - cl * 4 * kk;
      const int tt = rem >> 2, ol = 8 * (rem & 3);
      const int o = o0 + ol, c = c0 + cl;
      if (c >= J.C || o >= J.O8) continue;
      const int src = cl * kk + (kk - 1 - tt);
      float v[8];
#pragma unroll
      for (int t = 0; t < 8; ++t) v[t] = tile[(ol + t) * ld + src];
      store_split8(J.wd + ((size_t)c * kk + tt) * J.O8 + o, J.psd, v);
    }
    return;
  }
  // wf[o][tap][c], c fastest, pairs (c, c+1): C8, c0 and cb are even
  const int hb = cb >> 1;
  for (int idx = threadIdx.x; idx < 32 * kk * hb; idx += blockDim.x) {
    const int ol = idx / (kk * hb), rem = idx - ol * kk * hb;
    const int tap = rem / hb, cl = 2 * (rem - tap * hb);
    const int o = o0 + ol, c = c0 + cl;
    if (o < J.O && c < J.C8)
      store_split2(J.wf, J.psf, ((size_t)o * kk + tap) * J.C8 + c, tile[ol * ld + cl * kk + tap],
                   tile[ol * ld + (cl + 1) * kk + tap]);
  }
  if (!J.wd) return;
  // wd[c][tt][o], o fastest, pairs (o, o+1), tap = kk - 1 - tt (both tap axes flipped)
  for (int idx = threadIdx.x; idx < 16 * span; idx += blockDim.x) {
    const int cl = idx / (16 * kk), rem = idx - cl * 16 * kk;
    const int tt = rem >> 4, ol = 2 * (rem & 15);
    const int o = o0 + ol, c = c0 + cl;
    const int src = cl * kk + (kk - 1 - tt);
    if (c < J.C && o < J.O8)
      store_split2(J.wd, J.psd, ((size_t)c * kk + tt) * J.O8 + o, tile[ol * ld + src],
                   tile[(ol + 1) * ld + src]);
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

// 8-channel vector helpers on split planes (16-byte aligned chunks)
__device__ __forceinline__ void load_split8(const bf16_t* p, size_t ps, float (&v)[8]) {
  const uint4 a = *reinterpret_cast<const uint4*>(p);
  const uint4 b = *reinterpret_cast<const uint4*>(p + ps);
  const uint4 c = *reinterpret_cast<const uint4*>(p + 2 * ps);
  const uint32_t aw[4] = {a.x, a.y, a.z, a.w}, bw[4] = {b.x, b.y, b.z, b.w},
                 cw[4] = {c.x, c.y, c.z, c.w};
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    v[2 * j] = join3((bf16_t)(aw[j] & 0xFFFF), (bf16_t)(bw[j] & 0xFFFF), (bf16_t)(cw[j] & 0xFFFF));
    v[2 * j + 1] = join3((bf16_t)(aw[j] >> 16), (bf16_t)(bw[j] >> 16), (bf16_t)(cw[j] >> 16));
  }
}

// max-pool forward on NHWC split planes, one thread per (output pixel, 8
// channels).  Output NHWC [N][OH][OW][C8] (flat_ld == 0) or CHW-flat
// [N][flat_ld] (the FC-block input, reference flatten order).  arg (uint8,
// kh*k+kw of the FIRST maximum, scanning kh-major / kw-minor) is indexed NHWC
// [N][OH][OW][C8] in both modes.
__global__ void maxpool_fwd_split_kernel(const bf16_t* __restrict__ x, size_t psx,
                                         bf16_t* __restrict__ y, size_t psy,
                                         uint8_t* __restrict__ arg, int N, int C, int C8, int H,
                                         int W, int k, int s, int OH, int OW, int flat_ld,
                                         FastDiv d_ch, FastDiv d_ow, FastDiv d_oh) {
  const uint32_t total = (uint32_t)N * OH * OW * (C8 / 8);
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    uint32_t opix, cc, t, ow, n, oh;
    d_ch.divmod(i, opix, cc);
    d_ow.divmod(opix, t, ow);
    d_oh.divmod(t, n, oh);
    const size_t base = (((size_t)n * H + (size_t)oh * s) * W + (size_t)ow * s) * C8 + cc * 8;
    float best[8];
    int bi[8];
    load_split8(x + base, psx, best);
#pragma unroll
    for (int j = 0; j < 8; ++j) bi[j] = 0;
    for (int kh = 0; kh < k; ++kh)
      for (int kw = 0; kw < k; ++kw) {
        if ((kh | kw) == 0) continue;
        float v[8];
        load_split8(x + base + ((size_t)kh * W + kw) * C8, psx, v);
#pragma unroll
        for (int j = 0; j < 8; ++j)
          if (v[j] > best[j]) {
            best[j] = v[j];
            bi[j] = kh * k + kw;
          }
      }
    const size_t o = (size_t)opix * C8 + cc * 8;
    uint2 packed;
    packed.x = (uint32_t)bi[0] | ((uint32_t)bi[1] << 8) | ((uint32_t)bi[2] << 16) |
               ((uint32_t)bi[3] << 24);
    packed.y = (uint32_t)bi[4] | ((uint32_t)bi[5] << 8) | ((uint32_t)bi[6] << 16) |
               ((uint32_t)bi[7] << 24);
    *reinterpret_cast<uint2*>(arg + o) = packed;
#pragma unroll
    for (int j = 0; j < 8; ++j)
      if ((int)(cc * 8 + j) >= C) best[j] = 0.f;
    if (flat_ld == 0) {
      store_split8(y + o, psy, best);
    } else {
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int c = (int)cc * 8 + j;
        if (c < C) store_split(y, psy, (size_t)n * flat_ld + ((size_t)c * OH + oh) * OW + ow, best[j]);
      }
    }
  }
}

// Row-tiled form of maxpool_fwd_split_kernel for NHWC outputs (same
// comparisons in the same order, so bit-identical): one block per (image,
// TOH output rows).  The input rows the tile's windows read are joined from
// their three bf16 planes into fp32 shared memory once -- the untiled kernel
// joined each input pixel once per window reading it (9 joins per output at
// 3x3/2 against (2 TOH + 1) W / (TOH OW) here).
__global__ void __launch_bounds__(256) maxpool_fwd_tiled_kernel(
    const bf16_t* __restrict__ x, size_t psx, bf16_t* __restrict__ y, size_t psy,
    uint8_t* __restrict__ arg, int C, int C8, int H, int W, int k, int s, int OH, int OW,
    int TOH, FastDiv d_ch, FastDiv d_w, FastDiv d_ow) {
  extern __shared__ float4 poolf_smem4[];
  float* xs = reinterpret_cast<float*>(poolf_smem4);
  const int tiles = (OH + TOH - 1) / TOH;
  const int n = blockIdx.x / tiles, tt = blockIdx.x - n * tiles;
  const int oh0 = tt * TOH, oh1 = min(OH, oh0 + TOH);
  const int h0 = oh0 * s, h1 = min(H, (oh1 - 1) * s + k);
  const int groups = (h1 - h0) * W * (C8 / 8);
  for (int i = threadIdx.x; i < groups; i += blockDim.x) {
    uint32_t pr, cc, r, w;
    d_ch.divmod((uint32_t)i, pr, cc);
    d_w.divmod(pr, r, w);
    float v[8];
    load_split8(x + (((size_t)n * H + h0 + r) * W + w) * C8 + cc * 8, psx, v);
    float4* d = reinterpret_cast<float4*>(xs + (size_t)i * 8);
    d[0] = make_float4(v[0], v[1], v[2], v[3]);
    d[1] = make_float4(v[4], v[5], v[6], v[7]);
  }
  __syncthreads();
  const int outs = (oh1 - oh0) * OW * (C8 / 8);
  for (int i = threadIdx.x; i < outs; i += blockDim.x) {
    uint32_t pr, cc, r, ow;
    d_ch.divmod((uint32_t)i, pr, cc);
    d_ow.divmod(pr, r, ow);
    const int oh = oh0 + (int)r;
    const float* b0 = xs + (((size_t)(oh * s - h0) * W + ow * s) * C8 + cc * 8);
    float best[8];
    int bi[8];
    {
      const float4 p0 = *reinterpret_cast<const float4*>(b0);
      const float4 p1 = *reinterpret_cast<const float4*>(b0 + 4);
      best[0] = p0.x; best[1] = p0.y; best[2] = p0.z; best[3] = p0.w;
      best[4] = p1.x; best[5] = p1.y; best[6] = p1.z; best[7] = p1.w;
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) bi[j] = 0;
    for (int kh = 0; kh < k; ++kh)
      for (int kw = 0; kw < k; ++kw) {
        if ((kh | kw) == 0) continue;
        const float* q = b0 + ((size_t)kh * W + kw) * C8;
        const float4 p0 = *reinterpret_cast<const float4*>(q);
        const float4 p1 = *reinterpret_cast<const float4*>(q + 4);
        const float v[8] = {p0.x, p0.y, p0.z, p0.w, p1.x, p1.y, p1.z, p1.w};
#pragma unroll
        for (int j = 0; j < 8; ++j)
          if (v[j] > best[j]) {
            best[j] = v[j];
            bi[j] = kh * k + kw;
          }
      }
    const size_t o = (((size_t)n * OH + oh) * OW + ow) * C8 + cc * 8;
    uint2 packed;
    packed.x = (uint32_t)bi[0] | ((uint32_t)bi[1] << 8) | ((uint32_t)bi[2] << 16) |
               ((uint32_t)bi[3] << 24);
    packed.y = (uint32_t)bi[4] | ((uint32_t)bi[5] << 8) | ((uint32_t)bi[6] << 16) |
               ((uint32_t)bi[7] << 24);
    *reinterpret_cast<uint2*>(arg + o) = packed;
#pragma unroll
    for (int j = 0; j < 8; ++j)
      if ((int)(cc * 8 + j) >= C) best[j] = 0.f;
    store_split8(y + o, psy, best);
  }
}

// zero the CHW-flat tail columns [C*OH*OW, flat_ld) once per buffer
__global__ void zero_flat_tail_kernel(bf16_t* __restrict__ y, size_t psy, int N, int D, int ld) {
  const int tail = ld - D;
  STZ_GRID_LOOP(i, (size_t)N * tail) {
    store_split(y, psy, (i / tail) * ld + D + i % tail, 0.f);
  }
}

// max-pool backward, gather form, one thread per (input pixel, 8 channels):
// every input cell sums in float64, in the reference's (kh, kw) order, the
// output gradients whose argmax it was; gy is NHWC (flat_ld == 0) or
// CHW-flat.  mask = plane 0 of the pool input when a ReLU fed the pool (its
// backward fused here).
__global__ void maxpool_bwd_split_kernel(const bf16_t* __restrict__ gy, size_t psg,
                                         const uint8_t* __restrict__ arg,
                                         bf16_t* __restrict__ gx, size_t psx,
                                         const bf16_t* __restrict__ mask, int N, int C, int C8,
                                         int H, int W, int k, int s, int OH, int OW,
                                         int flat_ld, FastDiv d_ch, FastDiv d_w, FastDiv d_h) {
  const uint32_t total = (uint32_t)N * H * W * (C8 / 8);
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    uint32_t pix, cc, t, w, n, h;
    d_ch.divmod(i, pix, cc);
    d_w.divmod(pix, t, w);
    d_h.divmod(t, n, h);
    double acc[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[j] = 0.0;
    const int th = (int)h - k + 1, tw = (int)w - k + 1;
    const int oh_lo = th <= 0 ? 0 : (th + s - 1) / s, ow_lo = tw <= 0 ? 0 : (tw + s - 1) / s;
    const int oh_hi = min(OH - 1, (int)h / s), ow_hi = min(OW - 1, (int)w / s);
    for (int oh = oh_hi; oh >= oh_lo; --oh)
      for (int ow = ow_hi; ow >= ow_lo; --ow) {
        const size_t o = (((size_t)n * OH + oh) * OW + ow) * C8 + cc * 8;
        const uint2 a2 = *reinterpret_cast<const uint2*>(arg + o);
        const uint32_t want = (uint32_t)(((int)h - oh * s) * k + ((int)w - ow * s));
        float g[8];
        if (flat_ld == 0) {
          load_split8(gy + o, psg, g);
        } else {
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const int c = (int)cc * 8 + j;
            g[j] = c < C ? load_split(gy, psg,
                                      (size_t)n * flat_ld + ((size_t)c * OH + oh) * OW + ow)
                         : 0.f;
          }
        }
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const uint32_t aj = ((j < 4 ? a2.x : a2.y) >> (8 * (j & 3))) & 0xFFu;
          if (aj == want) acc[j] += (double)g[j];
        }
      }
    const size_t xi = (size_t)pix * C8 + cc * 8;
    float v[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] = (int)(cc * 8 + j) < C ? (float)acc[j] : 0.f;
    if (mask) {
      const uint4 mk = *reinterpret_cast<const uint4*>(mask + xi);
      const uint32_t mw[4] = {mk.x, mk.y, mk.z, mk.w};
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const bf16_t mb = (bf16_t)((mw[j >> 1] >> (16 * (j & 1))) & 0xFFFF);
        if (!(bf2f(mb) > 0.f)) v[j] = 0.f;
      }
    }
    store_split8(gx + xi, psx, v);
  }
}

// ---- max-pool, faster forms -------------------------------------------------

// backward, NHWC gy, compile-time window (K, S): the <= ceil(K/S)^2 windows
// covering a cell are known up front, so every load (argmax bytes, gradient
// planes, ReLU mask) is issued before the float64 accumulation, which keeps
// the reference's (kh, kw) order (oh, ow descending).
template <int K, int S>
__global__ void maxpool_bwd_nhwc_kernel(const bf16_t* __restrict__ gy, size_t psg,
                                        const uint8_t* __restrict__ arg,
                                        bf16_t* __restrict__ gx, size_t psx,
                                        const bf16_t* __restrict__ mask, int N, int C, int C8,
                                        int H, int W, int OH, int OW, FastDiv d_ch, FastDiv d_w,
                                        FastDiv d_h) {
  constexpr int R = (K + S - 1) / S;
  const uint32_t total = (uint32_t)N * H * W * (C8 / 8);
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    uint32_t pix, cc, t, w, n, h;
    d_ch.divmod(i, pix, cc);
    d_w.divmod(pix, t, w);
    d_h.divmod(t, n, h);
    const size_t xi = (size_t)pix * C8 + cc * 8;
    uint4 mk = make_uint4(0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu);
    if (mask) mk = __ldg(reinterpret_cast<const uint4*>(mask + xi));
    const int oh_hi = min(OH - 1, (int)h / S), ow_hi = min(OW - 1, (int)w / S);
    bool ok[R][R];
    uint2 ar[R][R];
    float g[R][R][8];
#pragma unroll
    for (int a = 0; a < R; ++a)
#pragma unroll
      for (int b = 0; b < R; ++b) {
        const int oh = oh_hi - a, ow = ow_hi - b;
        ok[a][b] = oh >= 0 && ow >= 0 && (int)h - oh * S < K && (int)w - ow * S < K;
        if (ok[a][b]) {
          const size_t o = (((size_t)n * OH + oh) * OW + ow) * C8 + cc * 8;
          ar[a][b] = __ldg(reinterpret_cast<const uint2*>(arg + o));
          load_split8(gy + o, psg, g[a][b]);
        }
      }
    double acc[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[j] = 0.0;
#pragma unroll
    for (int a = 0; a < R; ++a)
#pragma unroll
      for (int b = 0; b < R; ++b) {
        if (!ok[a][b]) continue;
        const uint32_t want =
            (uint32_t)(((int)h - (oh_hi - a) * S) * K + ((int)w - (ow_hi - b) * S));
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const uint32_t aj = ((j < 4 ? ar[a][b].x : ar[a][b].y) >> (8 * (j & 3))) & 0xFFu;
          if (aj == want) acc[j] += (double)g[a][b][j];
        }
      }
    const uint32_t mw[4] = {mk.x, mk.y, mk.z, mk.w};
    float v[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const uint32_t hb = (mw[j >> 1] >> (16 * (j & 1))) & 0xFFFFu;   // bf16 > 0
      const bool keep = !mask || (hb != 0u && hb < 0x8000u);
      v[j] = ((int)(cc * 8 + j) < C && keep) ? (float)acc[j] : 0.f;
    }
    store_split8(gx + xi, psx, v);
  }
}

// Row-tiled form of maxpool_bwd_nhwc_kernel (same values, same summation
// order, so bit-identical): one block per (image, TOH output rows).  The
// gradient windows the tile's input rows read -- output rows [oh_lo, oh_hi]
// -- are joined from their three bf16 planes into fp32 ONCE, into shared
// memory with their argmax bytes; the per-input-pixel gather then reads
// shared memory.  The untiled kernel re-joined every window for each of the
// up to R*R input pixels that read it (K = 3, S = 2: 4 candidate windows per
// pixel), which made it instruction-bound (profiles/r02/op/pool2_bwd_*:
// 68% issue slots busy at 0.25 of HBM).  Input rows [S*oh0, S*(oh0+TOH)) of
// the tile, the last tile through H (rows past every window get zero).
template <int K, int S>
__global__ void __launch_bounds__(512) maxpool_bwd_tiled_kernel(
    const bf16_t* __restrict__ gy, size_t psg, const uint8_t* __restrict__ arg,
    bf16_t* __restrict__ gx, size_t psx, const bf16_t* __restrict__ mask, int C, int C8, int H,
    int W, int OH, int OW, int TOH, FastDiv d_ch, FastDiv d_ow, FastDiv d_w) {
  constexpr int R = (K + S - 1) / S;
  extern __shared__ float4 pool_smem4[];
  const int tiles = (OH + TOH - 1) / TOH;
  const int n = blockIdx.x / tiles, tt = blockIdx.x - n * tiles;
  const int oh0 = tt * TOH;
  const int h_lo = S * oh0, h_hi = tt == tiles - 1 ? H : min(H, S * (oh0 + TOH));
  // windows covering rows [h_lo, h_hi): oh*S <= h <= oh*S + K - 1
  const int w_lo = max(0, (h_lo - K + S) / S), w_hi = min(OH - 1, (h_hi - 1) / S);
  const int nrows = w_hi - w_lo + 1;
  const int rowc = OW * C8;                       // values per window row
  float* gs = reinterpret_cast<float*>(pool_smem4);
  uint8_t* as = reinterpret_cast<uint8_t*>(gs + (size_t)nrows * rowc);
  const int groups = nrows * OW * (C8 / 8);
  for (int i = threadIdx.x; i < groups; i += blockDim.x) {
    uint32_t rw, cc, r, ow;
    d_ch.divmod((uint32_t)i, rw, cc);
    d_ow.divmod(rw, r, ow);
    const size_t o = (((size_t)n * OH + w_lo + r) * OW + ow) * C8 + cc * 8;
    float g[8];
    load_split8(gy + o, psg, g);
    const uint2 a = __ldg(reinterpret_cast<const uint2*>(arg + o));
    float4* d = reinterpret_cast<float4*>(gs + (size_t)i * 8);
    d[0] = make_float4(g[0], g[1], g[2], g[3]);
    d[1] = make_float4(g[4], g[5], g[6], g[7]);
    *reinterpret_cast<uint2*>(as + (size_t)i * 8) = a;
  }
  __syncthreads();
  const int pix_groups = (h_hi - h_lo) * W * (C8 / 8);
  for (int i = threadIdx.x; i < pix_groups; i += blockDim.x) {
    uint32_t pr, cc, hr, w;
    d_ch.divmod((uint32_t)i, pr, cc);
    d_w.divmod(pr, hr, w);
    const int h = h_lo + (int)hr;
    const size_t xi = (((size_t)n * H + h) * W + w) * C8 + cc * 8;
    uint4 mk = make_uint4(0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu);
    if (mask) mk = __ldg(reinterpret_cast<const uint4*>(mask + xi));
    const int oh_hi = min(OH - 1, h / S), ow_hi = min(OW - 1, (int)w / S);
    double acc[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[j] = 0.0;
#pragma unroll
    for (int a = 0; a < R; ++a)
#pragma unroll
      for (int b = 0; b < R; ++b) {
        const int oh = oh_hi - a, ow = ow_hi - b;
        if (oh < 0 || ow < 0 || h - oh * S >= K || (int)w - ow * S >= K) continue;
        const size_t si = ((size_t)(oh - w_lo) * OW + ow) * C8 + cc * 8;
        const uint2 ar = *reinterpret_cast<const uint2*>(as + si);
        const uint32_t want = (uint32_t)((h - oh * S) * K + ((int)w - ow * S));
        const uint32_t rep = want * 0x01010101u;
        const uint32_t m0 = __vcmpeq4(ar.x, rep), m1 = __vcmpeq4(ar.y, rep);
        if ((m0 | m1) == 0u) continue;
        const float4 g0 = *reinterpret_cast<const float4*>(gs + si);
        const float4 g1 = *reinterpret_cast<const float4*>(gs + si + 4);
        const float gv[8] = {g0.x, g0.y, g0.z, g0.w, g1.x, g1.y, g1.z, g1.w};
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const uint32_t mj = ((j < 4 ? m0 : m1) >> (8 * (j & 3))) & 1u;
          if (mj) acc[j] += (double)gv[j];
        }
      }
    const uint32_t mw[4] = {mk.x, mk.y, mk.z, mk.w};
    float v[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const uint32_t hb = (mw[j >> 1] >> (16 * (j & 1))) & 0xFFFFu;   // bf16 > 0
      const bool keep = !mask || (hb != 0u && hb < 0x8000u);
      v[j] = ((int)(cc * 8 + j) < C && keep) ? (float)acc[j] : 0.f;
    }
    store_split8(gx + xi, psx, v);
  }
}

// forward into the CHW-flat FC boundary, one block per image: windows are
// scanned NHWC (coalesced, 8 channels per thread), the maxima land in shared
// memory in flat (c, oh, ow) order and leave as coalesced 8-element rows; the
// row's padding columns [C*OH*OW, flat_ld) are zeroed here too.
__global__ void maxpool_fwd_flat_kernel(const bf16_t* __restrict__ x, size_t psx,
                                        bf16_t* __restrict__ y, size_t psy,
                                        uint8_t* __restrict__ arg, int C, int C8, int H, int W,
                                        int k, int s, int OH, int OW, int flat_ld) {
  extern __shared__ float sflat[];   // [C * OH * OW]
  const int n = blockIdx.x;
  const int chunks = C8 / 8, items = OH * OW * chunks, D = C * OH * OW;
  for (int it = threadIdx.x; it < items; it += blockDim.x) {
    const int cc = it % chunks, opix = it / chunks, oh = opix / OW, ow = opix % OW;
    const size_t base = (((size_t)n * H + (size_t)oh * s) * W + (size_t)ow * s) * C8 + cc * 8;
    float best[8];
    int bi[8];
    load_split8(x + base, psx, best);
#pragma unroll
    for (int j = 0; j < 8; ++j) bi[j] = 0;
    for (int kh = 0; kh < k; ++kh)
      for (int kw = 0; kw < k; ++kw) {
        if ((kh | kw) == 0) continue;
        float v[8];
        load_split8(x + base + ((size_t)kh * W + kw) * C8, psx, v);
#pragma unroll
        for (int j = 0; j < 8; ++j)
          if (v[j] > best[j]) {
            best[j] = v[j];
            bi[j] = kh * k + kw;
          }
      }
    uint2 packed;
    packed.x = (uint32_t)bi[0] | ((uint32_t)bi[1] << 8) | ((uint32_t)bi[2] << 16) |
               ((uint32_t)bi[3] << 24);
    packed.y = (uint32_t)bi[4] | ((uint32_t)bi[5] << 8) | ((uint32_t)bi[6] << 16) |
               ((uint32_t)bi[7] << 24);
    *reinterpret_cast<uint2*>(arg + ((size_t)n * OH * OW + opix) * C8 + cc * 8) = packed;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int c = cc * 8 + j;
      if (c < C) sflat[(c * OH + oh) * OW + ow] = best[j];
    }
  }
  __syncthreads();
  bf16_t* row = y + (size_t)n * flat_ld;
  for (int q = threadIdx.x; q < flat_ld / 8; q += blockDim.x) {
    float v[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] = q * 8 + j < D ? sflat[q * 8 + j] : 0.f;
    store_split8(row + q * 8, psy, v);
  }
}

// backward from the CHW-flat FC boundary, one block per image: the image's
// gradient row is staged in shared memory (coalesced), then every input cell
// gathers in float64, (kh, kw) order, as maxpool_bwd_split_kernel does.
__global__ void maxpool_bwd_flat_kernel(const bf16_t* __restrict__ gy, size_t psg,
                                        const uint8_t* __restrict__ arg,
                                        bf16_t* __restrict__ gx, size_t psx,
                                        const bf16_t* __restrict__ mask, int C, int C8, int H,
                                        int W, int k, int s, int OH, int OW, int flat_ld) {
  extern __shared__ float sflat[];   // [C * OH * OW]
  const int n = blockIdx.x;
  const int D = C * OH * OW;
  const bf16_t* row = gy + (size_t)n * flat_ld;
  for (int q = threadIdx.x; q < (D + 7) / 8; q += blockDim.x) {
    float v[8];
    load_split8(row + q * 8, psg, v);   // flat_ld % 8 == 0: the padded tail is readable
#pragma unroll
    for (int j = 0; j < 8; ++j)
      if (q * 8 + j < D) sflat[q * 8 + j] = v[j];
  }
  __syncthreads();
  const int chunks = C8 / 8, items = H * W * chunks;
  for (int it = threadIdx.x; it < items; it += blockDim.x) {
    const int cc = it % chunks, pix = it / chunks, h = pix / W, w = pix % W;
    const size_t xi = ((size_t)n * H * W + pix) * C8 + cc * 8;
    double acc[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[j] = 0.0;
    const int th = h - k + 1, tw = w - k + 1;
    const int oh_lo = th <= 0 ? 0 : (th + s - 1) / s, ow_lo = tw <= 0 ? 0 : (tw + s - 1) / s;
    const int oh_hi = min(OH - 1, h / s), ow_hi = min(OW - 1, w / s);
    for (int oh = oh_hi; oh >= oh_lo; --oh)
      for (int ow = ow_hi; ow >= ow_lo; --ow) {
        const uint2 a2 = __ldg(reinterpret_cast<const uint2*>(
            arg + (((size_t)n * OH + oh) * OW + ow) * C8 + cc * 8));
        const uint32_t want = (uint32_t)((h - oh * s) * k + (w - ow * s));
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const int c = cc * 8 + j;
          const uint32_t aj = ((j < 4 ? a2.x : a2.y) >> (8 * (j & 3))) & 0xFFu;
          if (aj == want && c < C) acc[j] += (double)sflat[(c * OH + oh) * OW + ow];
        }
      }
    uint4 mk = make_uint4(0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu);
    if (mask) mk = __ldg(reinterpret_cast<const uint4*>(mask + xi));
    const uint32_t mw[4] = {mk.x, mk.y, mk.z, mk.w};
    float v[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const uint32_t hb = (mw[j >> 1] >> (16 * (j & 1))) & 0xFFFFu;
      const bool keep = !mask || (hb != 0u && hb < 0x8000u);
      v[j] = (cc * 8 + j < C && keep) ? (float)acc[j] : 0.f;
    }
    store_split8(gx + xi, psx, v);
  }
}

// space-to-depth input pack, one block per (image, s2d row i): the C x S
// input rows i*S - pad .. i*S - pad + S - 1 are read coalesced and staged in
// shared memory as [c][dy][dx][j] (the s2d column j fastest, so the gather
// below is conflict-free), then every s2d pixel of the row leaves as 16-byte
// 8-channel chunks per plane.  C and S are compile-time (AlexNet conv1: 3, 4),
// which turns every index division into a multiply / shift -- the generic
// form of this kernel was bound by integer division.
template <int C, int S>
__global__ void pack_s2d_rows_kernel(const float* __restrict__ x, bf16_t* __restrict__ xp,
                                     size_t ps, int H, int W, int pad, int Hs, int Ws, int Cs8) {
  extern __shared__ float srows[];   // [C][S][S][Ws]
  const int n = blockIdx.x / Hs, i = blockIdx.x % Hs;
  const int WS = Ws * S;   // padded-input columns the row covers
  // stage: row r = c*S + dy, columns col in [0, WS); one column per thread,
  // all C*S rows' loads in flight before the shared stores
  for (int col = threadIdx.x; col < WS; col += blockDim.x) {
    const int iw = col - pad;
    const bool col_ok = iw >= 0 && iw < W;
    float v[C * S];
#pragma unroll
    for (int r = 0; r < C * S; ++r) {
      const int c = r / S, dy = r % S;
      const int ih = i * S + dy - pad;
      v[r] = (col_ok && ih >= 0 && ih < H) ? __ldg(x + (((size_t)n * C + c) * H + ih) * W + iw)
                                           : 0.f;
    }
#pragma unroll
    for (int r = 0; r < C * S; ++r) srows[(r * S + col % S) * Ws + col / S] = v[r];
  }
  __syncthreads();
  constexpr int CS = C * S * S;
  const int chunks = Cs8 / 8;
  bf16_t* out = xp + ((size_t)n * Hs + i) * Ws * Cs8;
  for (int q = threadIdx.x; q < Ws * chunks; q += blockDim.x) {
    const int cc = q % chunks, j = q / chunks;
    float v[8];
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      const int cp = cc * 8 + t;
      // channel cp = (dy*S + dx)*C + c  ->  srows[c][dy][dx][j]
      v[t] = cp < CS ? srows[((cp % C) * S * S + cp / C) * Ws + j] : 0.f;
    }
    store_split8(out + (size_t)j * Cs8 + cc * 8, ps, v);
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
  // a label outside [0, C) (the reference raises IndexError on it) never
  // indexes memory: the loss is NaN, which the harness reports as NonFinite
  if (threadIdx.x == 0)
    loss[row] = (lab >= 0 && lab < C) ? (float)(-log(exp((double)zr[lab] - mx) / se)) : __int_as_float(0x7fc00000);
}

// column sums of split planes [R][ld] (first N columns) in float64, two
// deterministic passes.  Pass 1: block b covers rows [b*rpb, (b+1)*rpb); a
// thread owns one 8-column chunk (16-byte loads per plane) and a row lane;
// lanes are reduced through shared memory in fixed order -> part[b][N8].
// Pass 2: fixed-order sum over blocks.
__global__ void __launch_bounds__(256) colsum_partial_kernel(const bf16_t* __restrict__ g,
                                                             size_t ps, int R, int N8, int ld,
                                                             int rows_per_block,
                                                             double* __restrict__ part) {
  __shared__ double red[256 * 8];
  const int chunks = N8 / 8;
  const int per_pass = chunks < 256 ? chunks : 256;
  const int lanes = 256 / per_pass;
  const int tc = threadIdx.x % per_pass, tl = threadIdx.x / per_pass;
  const int r0 = blockIdx.x * rows_per_block;
  const int r1 = min(R, r0 + rows_per_block);
  for (int c0 = 0; c0 < chunks; c0 += per_pass) {
    const int cc = c0 + tc;
    double acc[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[j] = 0.0;
    if (tl < lanes && cc < chunks) {
      // four rows' loads in flight per step; each thread's adds stay in row order
      int r = r0 + tl;
      for (; r + 3 * lanes < r1; r += 4 * lanes) {
        float v[4][8];
#pragma unroll
        for (int u = 0; u < 4; ++u) load_split8(g + (size_t)(r + u * lanes) * ld + cc * 8, ps, v[u]);
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
          for (int j = 0; j < 8; ++j) acc[j] += (double)v[u][j];
      }
      for (; r < r1; r += lanes) {
        float v[8];
        load_split8(g + (size_t)r * ld + cc * 8, ps, v);
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[j] += (double)v[j];
      }
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) red[threadIdx.x * 8 + j] = acc[j];
    __syncthreads();
    for (int e = threadIdx.x; e < per_pass * 8; e += 256) {
      const int c = e / 8, j = e % 8;
      if (c0 + c < chunks) {
        double t = 0.0;
        for (int l = 0; l < lanes; ++l) t += red[(l * per_pass + c) * 8 + j];
        part[(size_t)blockIdx.x * N8 + (c0 + c) * 8 + j] = t;
      }
    }
    __syncthreads();
  }
}

// one warp per column: lane-strided partial sums + a fixed shuffle tree
__global__ void __launch_bounds__(256) colsum_final_kernel(const double* __restrict__ part,
                                                           int blocks, int N, int N8,
                                                           float* __restrict__ out,
                                                           int accumulate) {
  const int c = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (c >= N) return;
  double s = 0.0;
  int b = lane;
  for (; b + 224 < blocks; b += 256) {   // eight blocks' loads in flight per step
    double v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = part[(size_t)(b + 32 * u) * N8 + c];
#pragma unroll
    for (int u = 0; u < 8; ++u) s += v[u];
  }
  for (; b < blocks; b += 32) s += part[(size_t)b * N8 + c];
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) out[c] = accumulate ? __fadd_rn(out[c], (float)s) : (float)s;
}

}  // namespace stz
