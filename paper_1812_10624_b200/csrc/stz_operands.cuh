// Operand "gather" views and the GEMM epilogue.
//
// Every contraction on the hot path is C[M,N] = sum_k A(m,k) * B(k,n) where
// A and B are read straight out of the reference layouts (NCHW activations,
// conv W [O,C,k,k], FC W [in,out]) -- implicit GEMM, no im2col buffers.
// A view exposes
//     Row row(int r)                 per-row context, built once per tile
//     float4 load(const Row&, int k0) elements k0..k0+3 of that row (0 past
//                                    the edge, in padding, or off-stride)
// so the producer warps of both GEMM cores can stage 4-wide K chunks.
//
// Reference semantics each view restates (file:line under
// /root/reference/pkg/src/stanza):
//   Im2col     conv forward taps           tensor_core.py:176-179
//   DgradG/W   conv input gradient         tensor_core.py:257-258, :260
//   WgradX/G   conv weight gradient        tensor_core.py:256
//   RowK/ColK  FC x@W, g@W^T, x^T@g        tensor_core.py:210, :286-287
#pragma once

#include "stz_common.cuh"

namespace stz {

// elem(r, k) = p[r*ld + k]          (K contiguous)
struct ViewRowK {
  const float* p;
  int rows, K, ld;
  int vec;  // ld % 4 == 0 and p 16-byte aligned
  struct Row {
    const float* ptr;
  };
  __device__ __forceinline__ Row row(int r) const {
    return Row{r < rows ? p + (size_t)r * ld : nullptr};
  }
  __device__ __forceinline__ float4 load(const Row& rw, int k0) const {
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    if (rw.ptr == nullptr || k0 >= K) return v;
    if (vec && k0 + 3 < K) return __ldg(reinterpret_cast<const float4*>(rw.ptr + k0));
    v.x = __ldg(rw.ptr + k0);
    if (k0 + 1 < K) v.y = __ldg(rw.ptr + k0 + 1);
    if (k0 + 2 < K) v.z = __ldg(rw.ptr + k0 + 2);
    if (k0 + 3 < K) v.w = __ldg(rw.ptr + k0 + 3);
    return v;
  }
};

// elem(r, k) = p[k*ld + r]          (rows contiguous)
struct ViewColK {
  const float* p;
  int rows, K, ld;
  struct Row {
    const float* ptr;
  };
  __device__ __forceinline__ Row row(int r) const {
    return Row{r < rows ? p + r : nullptr};
  }
  __device__ __forceinline__ float4 load(const Row& rw, int k0) const {
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    if (rw.ptr == nullptr || k0 >= K) return v;
    const float* q = rw.ptr + (size_t)k0 * ld;
    v.x = __ldg(q);
    if (k0 + 1 < K) v.y = __ldg(q + ld);
    if (k0 + 2 < K) v.z = __ldg(q + 2 * (size_t)ld);
    if (k0 + 3 < K) v.w = __ldg(q + 3 * (size_t)ld);
    return v;
  }
};

// Conv forward A: row m = (n, oh, ow), k = (c, kh, kw):
// x[n, c, oh*s - p + kh, ow*s - p + kw], zero in the padding.
struct ViewIm2col {
  const float* x;
  int M, K, C, H, W, OW, s, pad, ksz;
  FastDiv d_ohw, d_ow, d_kk, d_k;
  struct Row {
    long long base;  // offset of x[n, 0, ih0, iw0] (may be negative)
    int ih0, iw0;
    bool ok;
  };
  __device__ __forceinline__ Row row(int m) const {
    Row r;
    r.ok = m < M;
    uint32_t n, j, oh, ow;
    d_ohw.divmod(r.ok ? m : 0, n, j);
    d_ow.divmod(j, oh, ow);
    r.ih0 = (int)oh * s - pad;
    r.iw0 = (int)ow * s - pad;
    r.base = (long long)n * C * H * W + (long long)r.ih0 * W + r.iw0;
    return r;
  }
  __device__ __forceinline__ float elem(const Row& r, int k) const {
    if (!r.ok || k >= K) return 0.f;
    uint32_t c, t, kh, kw;
    d_kk.divmod(k, c, t);
    d_k.divmod(t, kh, kw);
    const int ih = r.ih0 + (int)kh, iw = r.iw0 + (int)kw;
    if ((unsigned)ih >= (unsigned)H || (unsigned)iw >= (unsigned)W) return 0.f;
    return __ldg(x + r.base + (long long)c * H * W + (long long)kh * W + kw);
  }
  __device__ __forceinline__ float4 load(const Row& r, int k0) const {
    return make_float4(elem(r, k0), elem(r, k0 + 1), elem(r, k0 + 2), elem(r, k0 + 3));
  }
};

// Conv input-gradient A: row m = (n, h, w), k = (o, kh, kw):
// gy[n, o, (h + p - kh)/s, (w + p - kw)/s] when the division is exact and
// lands inside the output; zero otherwise.
struct ViewDgradG {
  const float* g;
  int M, K, O, OH, OW, s, pad, ksz;
  FastDiv d_hw, d_w, d_kk, d_k;
  struct Row {
    long long base;  // n * O * OH * OW
    int y0, x0;      // h + p, w + p
    bool ok;
  };
  __device__ __forceinline__ Row row(int m) const {
    Row r;
    r.ok = m < M;
    uint32_t n, j, h, w;
    d_hw.divmod(r.ok ? m : 0, n, j);
    d_w.divmod(j, h, w);
    r.base = (long long)n * O * OH * OW;
    r.y0 = (int)h + pad;
    r.x0 = (int)w + pad;
    return r;
  }
  __device__ __forceinline__ float elem(const Row& r, int k) const {
    if (!r.ok || k >= K) return 0.f;
    uint32_t o, t, kh, kw;
    d_kk.divmod(k, o, t);
    d_k.divmod(t, kh, kw);
    int ty = r.y0 - (int)kh, tx = r.x0 - (int)kw;
    if (ty < 0 || tx < 0) return 0.f;
    if (s != 1) {
      if ((ty % s) != 0 || (tx % s) != 0) return 0.f;
      ty /= s;
      tx /= s;
    }
    if (ty >= OH || tx >= OW) return 0.f;
    return __ldg(g + r.base + (long long)o * OH * OW + (long long)ty * OW + tx);
  }
  __device__ __forceinline__ float4 load(const Row& r, int k0) const {
    return make_float4(elem(r, k0), elem(r, k0 + 1), elem(r, k0 + 2), elem(r, k0 + 3));
  }
};

// Conv input-gradient B: row = input channel c, k = (o, kh, kw): w[o, c, kh, kw].
struct ViewDgradW {
  const float* w;
  int C, K, kk;
  FastDiv d_kk;
  struct Row {
    int c;
    bool ok;
  };
  __device__ __forceinline__ Row row(int c) const { return Row{c, c < C}; }
  __device__ __forceinline__ float elem(const Row& r, int k) const {
    if (!r.ok || k >= K) return 0.f;
    uint32_t o, t;
    d_kk.divmod(k, o, t);
    return __ldg(w + ((size_t)o * C + r.c) * kk + t);
  }
  __device__ __forceinline__ float4 load(const Row& r, int k0) const {
    return make_float4(elem(r, k0), elem(r, k0 + 1), elem(r, k0 + 2), elem(r, k0 + 3));
  }
};

// Conv weight-gradient A (M side): row = (c, kh, kw), k = (n, oh, ow):
// x[n, c, oh*s - p + kh, ow*s - p + kw].
struct ViewWgradX {
  const float* x;
  int rows, K, C, H, W, OW, s, pad, ksz;
  FastDiv d_kk, d_k, d_ohw, d_ow;
  struct Row {
    long long off;  // c*H*W + kh*W + kw
    int kh, kw;
    bool ok;
  };
  __device__ __forceinline__ Row row(int r) const {
    Row o;
    o.ok = r < rows;
    uint32_t c, t, kh, kw;
    d_kk.divmod(o.ok ? r : 0, c, t);
    d_k.divmod(t, kh, kw);
    o.kh = (int)kh;
    o.kw = (int)kw;
    o.off = (long long)c * H * W + (long long)kh * W + kw;
    return o;
  }
  __device__ __forceinline__ float elem(const Row& r, int k) const {
    if (!r.ok || k >= K) return 0.f;
    uint32_t n, j, oh, ow;
    d_ohw.divmod(k, n, j);
    d_ow.divmod(j, oh, ow);
    const int ih0 = (int)oh * s - pad, iw0 = (int)ow * s - pad;
    const int ih = ih0 + r.kh, iw = iw0 + r.kw;
    if ((unsigned)ih >= (unsigned)H || (unsigned)iw >= (unsigned)W) return 0.f;
    return __ldg(x + (long long)n * C * H * W + (long long)ih0 * W + iw0 + r.off);
  }
  __device__ __forceinline__ float4 load(const Row& r, int k0) const {
    return make_float4(elem(r, k0), elem(r, k0 + 1), elem(r, k0 + 2), elem(r, k0 + 3));
  }
};

// Conv weight-gradient B (N side): row = output channel o, k = (n, oh, ow):
// gy[n, o, oh, ow].
struct ViewWgradG {
  const float* g;
  int O, K, OHW;
  FastDiv d_ohw;
  struct Row {
    long long off;
    bool ok;
  };
  __device__ __forceinline__ Row row(int o) const {
    return Row{(long long)o * OHW, o < O};
  }
  __device__ __forceinline__ float elem(const Row& r, int k) const {
    if (!r.ok || k >= K) return 0.f;
    uint32_t n, j;
    d_ohw.divmod(k, n, j);
    return __ldg(g + (long long)n * O * OHW + r.off + j);
  }
  __device__ __forceinline__ float4 load(const Row& r, int k0) const {
    return make_float4(elem(r, k0), elem(r, k0 + 1), elem(r, k0 + 2), elem(r, k0 + 3));
  }
};

// Epilogue: out[idx(m, n)] = mask(relu(acc + bias[n])), with
// idx(m, n) = (m / mdiv) * ld_hi + (m % mdiv) * ld_lo + n * ld_n
// (covers row-major FC outputs, NCHW conv outputs and the transposed
// weight-gradient store).  `mask` fuses the backward of a preceding ReLU:
// keep the value only where mask[idx] > 0 (tensor_core.py:291-293 with the
// ReLU output standing in for its input; both are > 0 at the same cells).
struct Epilogue {
  float* out;
  int M, N;
  FastDiv d_m;
  long long ld_hi, ld_lo, ld_n;
  const float* bias;
  const float* mask;
  int relu;
  __device__ __forceinline__ long long index(int m, int n) const {
    uint32_t q, r;
    d_m.divmod((uint32_t)m, q, r);
    return (long long)q * ld_hi + (long long)r * ld_lo + (long long)n * ld_n;
  }
  __device__ __forceinline__ void store(int m, int n, float acc) const {
    if (m >= M || n >= N) return;
    const long long idx = index(m, n);
    float v = acc;
    if (bias) v = __fadd_rn(v, __ldg(bias + n));
    if (relu && v < 0.f) v = 0.f;  // NaN propagates like np.maximum
    if (mask && !(__ldg(mask + idx) > 0.f)) v = 0.f;
    out[idx] = v;
  }
};

}  // namespace stz
