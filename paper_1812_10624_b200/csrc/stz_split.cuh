// Split-plane tensor format and the cp.async tcgen05 GEMM (the hot path).
//
// Format.  A logical fp32 tensor T is stored as three bf16 planes
// P0, P1, P2 (same shape, `ps` elements apart) with T = P0 + P1 + P2
// EXACTLY: P0 = rn_bf16(T), P1 = rn_bf16(T - P0), P2 = T - P0 - P1 (the
// residuals of an fp32 value have <= 16 and <= 8 significant bits).  Conv
// activations are NHWC with channels padded to C8 = roundup(C, 8); flat
// activations / FC weights are row-major with rows padded to a multiple of
// 8.  Every 16-byte "piece" (8 consecutive elements along the contiguous
// dimension) is therefore one aligned cp.async.
//
// GEMM.  C[M,N] = sum_k A(m,k) B(k,n) with A, B given as split-plane views.
// The BF16x6 product b0*b0 | b0*b1 + b1*b0 + b1*b1 + b0*b2 + b2*b0 runs on
// tcgen05 (kind::f16, fp32 accumulate) into two TMEM accumulators, summed in
// fp32 RN by the epilogue.  Why two: measured on B200 (round 1 precision
// probes), the tensor core sums same-exponent products exactly
// but truncates bits shifted out during alignment, so every MMA into an
// accumulator D costs a bias of up to ~1 ulp(D) toward zero; the cross terms
// land in a separate "small" accumulator whose ulp is ~2^-8 of the big one.
// (TF32x3 was measured too: tf32 product sums are ~20-bit accurate; dropped.)  Producers (8 warps, two groups alternating
// k-blocks) only compute piece addresses and issue cp.async (zero-fill for
// padding / out-of-range); completion is signalled to the MMA thread through
// the stage's mbarrier after cp.async.wait_group + fence.proxy.async.
#pragma once

#include "stz_common.cuh"

namespace stz {

using bf16_t = uint16_t;

__device__ __forceinline__ float bf2f(bf16_t b) { return __uint_as_float((uint32_t)b << 16); }

__device__ __forceinline__ float join3(bf16_t a, bf16_t b, bf16_t c) {
  return __fadd_rn(__fadd_rn(bf2f(a), bf2f(b)), bf2f(c));
}

__device__ __forceinline__ float load_split(const bf16_t* p, size_t ps, size_t i) {
  return join3(p[i], p[i + ps], p[i + 2 * ps]);
}

__device__ __forceinline__ void store_split(bf16_t* p, size_t ps, size_t i, float x) {
  bf16_t a, b, c;
  split_bf16x3(x, a, b, c);
  p[i] = a;
  p[i + ps] = b;
  p[i + 2 * ps] = c;
}

// 2 consecutive values -> one 4-byte store per plane (p + i 4-byte aligned, ps even)
__device__ __forceinline__ void store_split2(bf16_t* p, size_t ps, size_t i, float x, float y) {
  bf16_t a0, a1, a2, b0, b1, b2;
  split_bf16x3(x, a0, a1, a2);
  split_bf16x3(y, b0, b1, b2);
  *reinterpret_cast<uint32_t*>(p + i) = (uint32_t)a0 | ((uint32_t)b0 << 16);
  *reinterpret_cast<uint32_t*>(p + i + ps) = (uint32_t)a1 | ((uint32_t)b1 << 16);
  *reinterpret_cast<uint32_t*>(p + i + 2 * ps) = (uint32_t)a2 | ((uint32_t)b2 << 16);
}

// 8 consecutive values -> one 16-byte store per plane (dst 16-byte aligned)
__device__ __forceinline__ void store_split8(bf16_t* p, size_t ps, const float (&v)[8]) {
  uint32_t w0[4], w1[4], w2[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    bf16_t a0, a1, a2, c0, c1, c2;
    split_bf16x3(v[2 * j], a0, a1, a2);
    split_bf16x3(v[2 * j + 1], c0, c1, c2);
    w0[j] = (uint32_t)a0 | ((uint32_t)c0 << 16);
    w1[j] = (uint32_t)a1 | ((uint32_t)c1 << 16);
    w2[j] = (uint32_t)a2 | ((uint32_t)c2 << 16);
  }
  *reinterpret_cast<uint4*>(p) = make_uint4(w0[0], w0[1], w0[2], w0[3]);
  *reinterpret_cast<uint4*>(p + ps) = make_uint4(w1[0], w1[1], w1[2], w1[3]);
  *reinterpret_cast<uint4*>(p + 2 * ps) = make_uint4(w2[0], w2[1], w2[2], w2[3]);
}

// ---------------------------------------------------------------------------
// cp.async
// ---------------------------------------------------------------------------

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, bool valid) {
  // src-size 0 -> 16 zero bytes; src must still be a mapped address
  asm volatile("cp.async.ca.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src),
               "r"(valid ? 16 : 0)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() {
  asm volatile("cp.async.commit_group;" ::: "memory");
}
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// ---------------------------------------------------------------------------
// operand views: piece(r, k) -> plane-0 pointer of 8 contiguous bf16, or null
//   K-major : r = row, k = first of 8 consecutive K indices
//   MN-major: r = first of 8 consecutive rows, k = one K index
// ---------------------------------------------------------------------------

// dense row-major planes, K contiguous: elem(r, k) = p[r*ld + k]
struct SvRowsK {
  static constexpr bool MN = false;
  const bf16_t* p;
  size_t ps;
  int rows, K, ld;
  __device__ __forceinline__ const bf16_t* p_any() const { return p; }
  __device__ __forceinline__ const bf16_t* piece(int r, int k) const {
    return (r < rows && k < K) ? p + (size_t)r * ld + k : nullptr;
  }
};

// dense planes with the ROW dimension contiguous: elem(r, k) = p[k*ld + r]
struct SvRowsMN {
  static constexpr bool MN = true;
  const bf16_t* p;
  size_t ps;
  int rows, K, ld;
  __device__ __forceinline__ const bf16_t* p_any() const { return p; }
  __device__ __forceinline__ const bf16_t* piece(int r0, int k) const {
    return (r0 < rows && k < K) ? p + (size_t)k * ld + r0 : nullptr;
  }
};

// conv forward A (implicit im2col over NHWC planes), K-major:
// row m = (n, oh, ow), k = (kh, kw, c):  X[n, oh*s-p+kh, ow*s-p+kw, c]
struct SvConvFwdA {
  static constexpr bool MN = false;
  const bf16_t* x;
  size_t ps;
  int M, K, H, W, C8, OW, s, pad;
  FastDiv d_ohw, d_ow, d_c8, d_k;
  __device__ __forceinline__ const bf16_t* p_any() const { return x; }
  __device__ __forceinline__ const bf16_t* piece(int m, int k) const {
    if (m >= M || k >= K) return nullptr;
    uint32_t n, j, oh, ow, tap, c0, kh, kw;
    d_ohw.divmod(m, n, j);
    d_ow.divmod(j, oh, ow);
    d_c8.divmod(k, tap, c0);
    d_k.divmod(tap, kh, kw);
    const int ih = (int)(oh * s + kh) - pad, iw = (int)(ow * s + kw) - pad;
    if ((unsigned)ih >= (unsigned)H || (unsigned)iw >= (unsigned)W) return nullptr;
    return x + (((size_t)n * H + ih) * W + iw) * C8 + c0;
  }
};

// conv input-gradient A over NHWC gradient planes G[N, OH, OW, O8], K-major:
// row m = (n, h, w), k = (th, tw, o) with flipped taps kh = k-1-th,
// kw = k-1-tw (matches the wd packing): G[n, (h+p-kh)/s, (w+p-kw)/s, o]
struct SvConvDgradA {
  static constexpr bool MN = false;
  const bf16_t* g;
  size_t ps;
  int M, K, OH, OW, O8, s, pad;
  FastDiv d_hw, d_w, d_o8, d_k;
  __device__ __forceinline__ const bf16_t* p_any() const { return g; }
  __device__ __forceinline__ const bf16_t* piece(int m, int k) const {
    if (m >= M || k >= K) return nullptr;
    uint32_t n, j, h, w, tap, o0, kh, kw;
    d_hw.divmod(m, n, j);
    d_w.divmod(j, h, w);
    d_o8.divmod(k, tap, o0);
    d_k.divmod(tap, kh, kw);
    kh = d_k.d - 1 - kh;  // flipped tap order
    kw = d_k.d - 1 - kw;
    int ty = (int)(h + pad) - (int)kh, tx = (int)(w + pad) - (int)kw;
    if (ty < 0 || tx < 0) return nullptr;
    if (s != 1) {
      if (ty % s || tx % s) return nullptr;
      ty /= s;
      tx /= s;
    }
    if (ty >= OH || tx >= OW) return nullptr;
    return g + (((size_t)n * OH + ty) * OW + tx) * O8 + o0;
  }
};

// conv weight-gradient A over NHWC input planes, MN-major:
// row r = (kh, kw, c) (c fastest, 8 at a time), k = output pixel (n, oh, ow)
struct SvConvWgradA {
  static constexpr bool MN = true;
  const bf16_t* x;
  size_t ps;
  int rows, K, H, W, C8, OW, s, pad;
  FastDiv d_c8, d_k, d_ohw, d_ow;
  __device__ __forceinline__ const bf16_t* p_any() const { return x; }
  __device__ __forceinline__ const bf16_t* piece(int r0, int k) const {
    if (r0 >= rows || k >= K) return nullptr;
    uint32_t tap, c0, kh, kw, n, j, oh, ow;
    d_c8.divmod(r0, tap, c0);
    d_k.divmod(tap, kh, kw);
    d_ohw.divmod(k, n, j);
    d_ow.divmod(j, oh, ow);
    const int ih = (int)(oh * s + kh) - pad, iw = (int)(ow * s + kw) - pad;
    if ((unsigned)ih >= (unsigned)H || (unsigned)iw >= (unsigned)W) return nullptr;
    return x + (((size_t)n * H + ih) * W + iw) * C8 + c0;
  }
};

// ---------------------------------------------------------------------------
// epilogues: store8(m, n0, v) for 8 consecutive columns n0..n0+7 of row m.
// HAS_BIAS epilogues split it as bias8(n0, b) (column bias, 0 past N) +
// store8_nb(m, n0, v + b), so the TMA kernel can issue the bias loads before
// its TMEM loads and keep them off the critical path.
// ---------------------------------------------------------------------------

// 8 consecutive fp32 values at p (n0 .. n0+7, zeros at n >= N)
__device__ __forceinline__ void ldg8_f32(const float* p, int n0, int N, float (&b)[8]) {
  if (n0 + 8 <= N && (reinterpret_cast<uintptr_t>(p + n0) & 15) == 0) {
    const float4 x = __ldg(reinterpret_cast<const float4*>(p + n0));
    const float4 y = __ldg(reinterpret_cast<const float4*>(p + n0) + 1);
    b[0] = x.x; b[1] = x.y; b[2] = x.z; b[3] = x.w;
    b[4] = y.x; b[5] = y.y; b[6] = y.z; b[7] = y.w;
  } else {
#pragma unroll
    for (int j = 0; j < 8; ++j) b[j] = n0 + j < N ? __ldg(p + n0 + j) : 0.f;
  }
}

// split planes, row-major [M][ld] (NHWC pixels or flat rows); columns in
// [N, ld) are written as zeros (channel padding).  bias / ReLU / ReLU-mask
// (mask = plane 0 of the ReLU output in the same layout: > 0 keeps).
struct EpSplit {
  bf16_t* out;
  size_t ps;
  int M, N, ld;
  const float* bias;
  const bf16_t* mask;
  int relu;
  // strided row scatter (a 1x1 stride-rs conv's input gradient): GEMM row
  // m = (n, oh, ow) of the output grid lands on input pixel (n, rs*oh, rs*ow)
  // of the rH x rW input; rs = 0 keeps rows in place
  // (+ offsets ro_h, ro_w: one phase of a strided conv's input gradient)
  int rs = 0, rH = 0, rW = 0, ro_h = 0, ro_w = 0;
  FastDiv rd_ow, rd_oh;
  static constexpr bool HAS_BIAS = true;
  static constexpr bool STAGED = true;
  __device__ __forceinline__ void bias8(int n0, float (&b)[8]) const {
    if (bias) {
      ldg8_f32(bias, n0, N, b);
    } else {
#pragma unroll
      for (int j = 0; j < 8; ++j) b[j] = 0.f;
    }
  }
  __device__ __forceinline__ size_t row_of(int m) const {
    if (!rs) return (size_t)m;
    uint32_t q, ow, n, oh;
    rd_ow.divmod((uint32_t)m, q, ow);
    rd_oh.divmod(q, n, oh);
    return ((size_t)n * rH + (size_t)rs * oh + ro_h) * rW + (size_t)rs * ow + ro_w;
  }
  // staged path, before the split: ReLU, zeros at n >= N (the ReLU mask is
  // applied to the planes by store_planes)
  __device__ __forceinline__ void prep8(int n0, float (&v)[8]) const {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      float x = v[j];
      if (relu && x < 0.f) x = 0.f;
      v[j] = n0 + j < N ? x : 0.f;
    }
  }
  // staged path: the three planes' 16 bytes of row m, columns n0..n0+7
  __device__ __forceinline__ void store_planes(int m, int n0, uint4 (&pl)[3]) const {
    if (n0 >= ld) return;
    const size_t base = row_of(m) * ld + n0;
    if (mask) {
      // a masked element is 0 in every plane (split of +0)
      const uint4 mk = __ldg(reinterpret_cast<const uint4*>(mask + base));
      const uint32_t mw[4] = {mk.x, mk.y, mk.z, mk.w};
      uint32_t keep[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const uint32_t lo = mw[j] & 0xFFFFu, hi = mw[j] >> 16;
        keep[j] = ((lo != 0u && lo < 0x8000u) ? 0x0000FFFFu : 0u) |
                  ((hi != 0u && hi < 0x8000u) ? 0xFFFF0000u : 0u);
      }
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        pl[k].x &= keep[0];
        pl[k].y &= keep[1];
        pl[k].z &= keep[2];
        pl[k].w &= keep[3];
      }
    }
    *reinterpret_cast<uint4*>(out + base) = pl[0];
    *reinterpret_cast<uint4*>(out + base + ps) = pl[1];
    *reinterpret_cast<uint4*>(out + base + 2 * ps) = pl[2];
  }
  // v already includes the bias
  __device__ __forceinline__ void store8_nb(int m, int n0, float (&v)[8]) const {
    if (m >= M || n0 >= ld) return;
    size_t row = (size_t)m;
    if (rs) {
      uint32_t q, ow, n, oh;
      rd_ow.divmod((uint32_t)m, q, ow);
      rd_oh.divmod(q, n, oh);
      row = ((size_t)n * rH + (size_t)rs * oh + ro_h) * rW + (size_t)rs * ow + ro_w;
    }
    const size_t base = row * ld + n0;
    uint4 mk = make_uint4(0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu);
    if (mask) mk = __ldg(reinterpret_cast<const uint4*>(mask + base));   // 8 bf16, 16-B aligned
    const uint32_t mw[4] = {mk.x, mk.y, mk.z, mk.w};
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      float x = v[j];
      if (n0 + j < N) {
        if (relu && x < 0.f) x = 0.f;
        // bf16 > 0: sign bit clear and not +0 (mask = plane 0 of a ReLU output)
        const uint32_t h = (mw[j >> 1] >> (16 * (j & 1))) & 0xFFFFu;
        if (mask && !(h != 0u && h < 0x8000u)) x = 0.f;
      } else {
        x = 0.f;
      }
      v[j] = x;
    }
    store_split8(out + base, ps, v);
  }
  __device__ __forceinline__ void store8(int m, int n0, float (&v)[8]) const {
    if (bias && n0 < N) {
      float b[8];
      bias8(n0, b);
#pragma unroll
      for (int j = 0; j < 8; ++j) v[j] = __fadd_rn(v[j], b[j]);
    }
    store8_nb(m, n0, v);
  }
  // 16 columns of row m (v includes the bias): one 256-bit store per plane,
  // i.e. whole 32-byte sectors, where the row segment is 32-byte aligned and
  // in range; else two store8_nb
  __device__ __forceinline__ void store16_nb(int m, int n0, float (&v)[16]) const {
    if (m >= M || n0 >= ld) return;
    const size_t base = (size_t)m * ld + n0;
    if (rs || n0 + 16 > ld || ((reinterpret_cast<uintptr_t>(out + base) |
                                 reinterpret_cast<uintptr_t>(out + base + ps)) & 31)) {
      float a[8], b[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        a[j] = v[j];
        b[j] = v[8 + j];
      }
      store8_nb(m, n0, a);
      store8_nb(m, n0 + 8, b);
      return;
    }
    uint32_t mw[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) mw[j] = 0xFFFFFFFFu;
    if (mask) {
      const uint4 m0 = __ldg(reinterpret_cast<const uint4*>(mask + base));
      const uint4 m1 = __ldg(reinterpret_cast<const uint4*>(mask + base + 8));
      mw[0] = m0.x; mw[1] = m0.y; mw[2] = m0.z; mw[3] = m0.w;
      mw[4] = m1.x; mw[5] = m1.y; mw[6] = m1.z; mw[7] = m1.w;
    }
    uint32_t w[3][8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      float x2[2];
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int jj = 2 * j + e;
        float x = v[jj];
        if (n0 + jj < N) {
          if (relu && x < 0.f) x = 0.f;
          const uint32_t h = (mw[j] >> (16 * e)) & 0xFFFFu;
          if (mask && !(h != 0u && h < 0x8000u)) x = 0.f;
        } else {
          x = 0.f;
        }
        x2[e] = x;
      }
      bf16_t a0, a1, a2, c0, c1, c2;
      split_bf16x3(x2[0], a0, a1, a2);
      split_bf16x3(x2[1], c0, c1, c2);
      w[0][j] = (uint32_t)a0 | ((uint32_t)c0 << 16);
      w[1][j] = (uint32_t)a1 | ((uint32_t)c1 << 16);
      w[2][j] = (uint32_t)a2 | ((uint32_t)c2 << 16);
    }
#pragma unroll
    for (int k = 0; k < 3; ++k)
      asm volatile("st.global.v8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(out + base + k * ps),
                   "r"(w[k][0]), "r"(w[k][1]), "r"(w[k][2]), "r"(w[k][3]), "r"(w[k][4]),
                   "r"(w[k][5]), "r"(w[k][6]), "r"(w[k][7])
                   : "memory");
  }
};

// fp32 output with the general index (m/mdiv)*ld_hi + (m%mdiv)*ld_lo + n*ld_n
// (row-major logits, NCHW reference layout, transposed weight gradients)
struct EpF32 {
  float* out;
  int M, N;
  FastDiv d_m;
  long long ld_hi, ld_lo, ld_n;
  const float* bias;
  const float* mask;  // fp32, same indexing as out
  int relu;
  int accumulate;     // 1: out += value (micro-batch gradient sums)
  static constexpr bool HAS_BIAS = true;
  static constexpr bool STAGED = false;
  __device__ __forceinline__ void bias8(int n0, float (&b)[8]) const {
    if (bias) {
      ldg8_f32(bias, n0, N, b);
    } else {
#pragma unroll
      for (int j = 0; j < 8; ++j) b[j] = 0.f;
    }
  }
  __device__ __forceinline__ void store8_nb(int m, int n0, float (&v)[8]) const {
    if (m >= M) return;
    uint32_t q, r;
    d_m.divmod((uint32_t)m, q, r);
    const long long row = (long long)q * ld_hi + (long long)r * ld_lo;
    if (ld_n == 1 && n0 + 8 <= N && !mask &&
        (reinterpret_cast<uintptr_t>(out + row + n0) & 15) == 0) {   // views may be offset
      float w[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        float x = v[j];
        if (relu && x < 0.f) x = 0.f;
        w[j] = x;
      }
      float4* dst = reinterpret_cast<float4*>(out + row + n0);
      if (accumulate) {
        const float4 a = dst[0], b = dst[1];
        w[0] = __fadd_rn(a.x, w[0]); w[1] = __fadd_rn(a.y, w[1]);
        w[2] = __fadd_rn(a.z, w[2]); w[3] = __fadd_rn(a.w, w[3]);
        w[4] = __fadd_rn(b.x, w[4]); w[5] = __fadd_rn(b.y, w[5]);
        w[6] = __fadd_rn(b.z, w[6]); w[7] = __fadd_rn(b.w, w[7]);
      }
      if ((reinterpret_cast<uintptr_t>(dst) & 31) == 0) {
        stg256(out + row + n0, w);
      } else {
        dst[0] = make_float4(w[0], w[1], w[2], w[3]);
        dst[1] = make_float4(w[4], w[5], w[6], w[7]);
      }
      return;
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int n = n0 + j;
      if (n >= N) break;
      const long long idx = row + (long long)n * ld_n;
      float x = v[j];
      if (relu && x < 0.f) x = 0.f;
      if (mask && !(__ldg(mask + idx) > 0.f)) x = 0.f;
      out[idx] = accumulate ? __fadd_rn(out[idx], x) : x;
    }
  }
  __device__ __forceinline__ void store8(int m, int n0, float (&v)[8]) const {
    if (bias && n0 < N) {
      float b[8];
      bias8(n0, b);
#pragma unroll
      for (int j = 0; j < 8; ++j) v[j] = __fadd_rn(v[j], b[j]);
    }
    store8_nb(m, n0, v);
  }
};

// conv weight gradient: row m = (tap, c) with c in [0, C8), column n = o ->
// gw[o, c, kh, kw] (reference layout); padded channels c >= C are dropped
struct EpConvWgrad {
  float* gw;
  int M, N, C, kk;
  FastDiv d_c8;
  int accumulate;   // 1: gw += value (micro-batch gradient sums)
  static constexpr bool HAS_BIAS = false;
  static constexpr bool STAGED = false;
  __device__ __forceinline__ void bias8(int, float (&)[8]) const {}
  __device__ __forceinline__ void store8_nb(int m, int n0, float (&v)[8]) const { store8(m, n0, v); }
  __device__ __forceinline__ void store8(int m, int n0, float (&v)[8]) const {
    if (m >= M) return;
    uint32_t tap, c;
    d_c8.divmod((uint32_t)m, tap, c);
    if ((int)c >= C) return;
    const size_t base = (size_t)c * kk + tap;
#pragma unroll
    for (int j = 0; j < 8; ++j)
      if (n0 + j < N) {
        float* d = gw + (size_t)(n0 + j) * C * kk + base;
        *d = accumulate ? __fadd_rn(*d, v[j]) : v[j];
      }
  }
};

// weight gradient of a space-to-depth conv (stz_fmt.cuh pack_s2d_kernel):
// row m = (tap', c') over Cs8 channels -> gw[o, c, kh'*s+dy, kw'*s+dx],
// dropping padded channels and taps beyond k
struct EpConvWgradS2D {
  float* gw;
  int M, N, C, k, s, ks, Cs;
  FastDiv d_cs8;
  int accumulate;   // 1: gw += value
  static constexpr bool HAS_BIAS = false;
  static constexpr bool STAGED = false;
  __device__ __forceinline__ void bias8(int, float (&)[8]) const {}
  __device__ __forceinline__ void store8_nb(int m, int n0, float (&v)[8]) const { store8(m, n0, v); }
  __device__ __forceinline__ void store8(int m, int n0, float (&v)[8]) const {
    if (m >= M) return;
    uint32_t tap, cp;
    d_cs8.divmod((uint32_t)m, tap, cp);
    if ((int)cp >= Cs) return;
    const int c = (int)cp % C, d = (int)cp / C, dy = d / s, dx = d % s;
    const int kh = (int)(tap / ks) * s + dy, kw = (int)(tap % ks) * s + dx;
    if (kh >= k || kw >= k) return;
    const size_t base = ((size_t)c * k + kh) * k + kw;
#pragma unroll
    for (int j = 0; j < 8; ++j)
      if (n0 + j < N) {
        float* d = gw + (size_t)(n0 + j) * C * k * k + base;
        *d = accumulate ? __fadd_rn(*d, v[j]) : v[j];
      }
  }
};

// ---------------------------------------------------------------------------
// the tcgen05 split-plane GEMM
// ---------------------------------------------------------------------------

constexpr int SG_BM = 128;
constexpr int SG_THREADS = 288;  // 8 producer warps (2 groups) + 1 MMA warp
constexpr int SG_DEPTH = 1;      // cp.async groups a producer keeps in flight

template <int BN, int BK>
struct SgCfg {
  static constexpr int CH = BK / 8;                    // 16-byte K pieces per row
  static constexpr int A_BYTES = SG_BM * BK * 2;       // one plane of the A tile
  static constexpr int B_BYTES = BN * BK * 2;
  static constexpr int STAGE_BYTES = 3 * (A_BYTES + B_BYTES);
  static constexpr int STAGES = (200 * 1024) / STAGE_BYTES > 8 ? 8 : (200 * 1024) / STAGE_BYTES;
  static constexpr int SMEM = STAGES * STAGE_BYTES + 256;
  static constexpr int A_PIECES = SG_BM * BK / 8 / 128; // per producer thread per stage
  static constexpr int B_PIECES = BN * BK / 8 / 128;
  static constexpr int KSTEPS = BK / 16;
  static constexpr int TMEM_COLS = BN <= 16 ? 32 : BN <= 32 ? 64 : BN <= 64 ? 128 : BN <= 128 ? 256 : 512;
  static constexpr uint32_t SBO = CH * 128;
  static constexpr uint32_t LBO = 128;
  static_assert(STAGES >= 2 * (SG_DEPTH + 1), "producer pipeline needs more stages");
  static_assert(A_PIECES >= 1 && B_PIECES >= 1, "tile too small for 128 producers");
};

__host__ __device__ constexpr uint32_t sg_idesc(int m, int n, bool a_mn, bool b_mn) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((a_mn ? 1u : 0u) << 15) |
         ((b_mn ? 1u : 0u) << 16) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(m >> 4) << 24);
}

// producer piece q (0 <= q < R*BK/8) of an R-row operand tile:
// returns (row or row-group start, k offset in tile, smem byte offset)
template <bool MN, int R, int BK>
__device__ __forceinline__ void sg_piece(int q, int& r, int& kt, uint32_t& soff) {
  constexpr int CH = BK / 8;
  if (!MN) {
    const int mi = q & 7, kc = (q >> 3) % CH, mg = q / (8 * CH);
    r = mg * 8 + mi;
    kt = kc * 8;
    soff = (uint32_t)((mg * CH + kc) * 128 + mi * 16);
  } else {
    const int kin = q & 7, mg = (q >> 3) % (R / 8), kg = q / R;
    r = mg * 8;
    kt = kg * 8 + kin;
    soff = (uint32_t)((mg * CH + kg) * 128 + kin * 16);
  }
}

template <int BN, int BK, class VA, class VB, class EP>
__global__ void __launch_bounds__(SG_THREADS, 1)
    sgemm_kernel(VA va, VB vb, EP ep, float* __restrict__ partial, int M, int N, int K,
                 int k_per_split) {
  using Cfg = SgCfg<BN, BK>;
  constexpr int STAGES = Cfg::STAGES;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + STAGES * Cfg::STAGE_BYTES);
  uint64_t* empty_bar = full_bar + STAGES;
  uint64_t* done_bar = empty_bar + STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done_bar + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m0 = blockIdx.x * SG_BM, n0 = blockIdx.y * BN;
  const int kbeg = blockIdx.z * k_per_split;
  const int kend = min(K, kbeg + k_per_split);
  const int nkb = cdiv(kend - kbeg, BK);

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full_bar[s], 128);
      mbar_init(&empty_bar[s], 1);
    }
    mbar_init(done_bar, 1);
    mbar_fence_init();
  }
  if (warp == 8) tmem_alloc(tmem_slot, Cfg::TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const uint32_t smem_base = smem_u32(smem);

  if (warp < 8) {
    // ---------------- producers: cp.async pieces --------------------------
    const int grp = warp >> 2;
    const int t = threadIdx.x & 127;
    int issued = 0, arrived = 0;
    for (int kb = grp; kb < nkb; kb += 2) {
      const int stage = kb % STAGES;
      mbar_wait(&empty_bar[stage], ((kb / STAGES) & 1) ^ 1);
      const int kt0 = kbeg + kb * BK;
      const uint32_t st = smem_base + stage * Cfg::STAGE_BYTES;
#pragma unroll
      for (int i = 0; i < Cfg::A_PIECES; ++i) {
        int r, kt;
        uint32_t so;
        sg_piece<VA::MN, SG_BM, BK>(t + 128 * i, r, kt, so);
        const bf16_t* src = va.piece(m0 + r, kt0 + kt);
        const bool ok = src != nullptr && (kt0 + kt) < kend;
        const bf16_t* s0 = ok ? src : va.p_any();
#pragma unroll
        for (int p = 0; p < 3; ++p)
          cp_async16(st + p * Cfg::A_BYTES + so, s0 + (ok ? p * va.ps : 0), ok);
      }
#pragma unroll
      for (int i = 0; i < Cfg::B_PIECES; ++i) {
        int r, kt;
        uint32_t so;
        sg_piece<VB::MN, BN, BK>(t + 128 * i, r, kt, so);
        const bf16_t* src = vb.piece(n0 + r, kt0 + kt);
        const bool ok = src != nullptr && (kt0 + kt) < kend;
        const bf16_t* s0 = ok ? src : vb.p_any();
#pragma unroll
        for (int p = 0; p < 3; ++p)
          cp_async16(st + 3 * Cfg::A_BYTES + p * Cfg::B_BYTES + so, s0 + (ok ? p * vb.ps : 0),
                     ok);
      }
      cp_async_commit();
      ++issued;
      if (issued > SG_DEPTH) {
        cp_async_wait<SG_DEPTH>();
        fence_proxy_async_smem();
        mbar_arrive(&full_bar[(grp + 2 * arrived) % STAGES]);
        ++arrived;
      }
    }
    cp_async_wait<0>();
    fence_proxy_async_smem();
    while (arrived < issued) {
      mbar_arrive(&full_bar[(grp + 2 * arrived) % STAGES]);
      ++arrived;
    }

    if (grp == 0) {
      // ---------------- epilogue: TMEM (big + small) -> registers -> ep ----
      mbar_wait(done_bar, 0);
      tc_fence_after();
      const int q = warp & 3;
      const int m = m0 + q * 32 + lane;
      const int npad = cdiv(N, 8) * 8;
#pragma unroll 1
      for (int c = 0; c < BN; c += 16) {
        if (n0 + c >= npad) break;
        uint32_t r[16], rs[16];
        const uint32_t taddr = tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)c;
        tmem_ld16(taddr, r);
        tmem_ld16(taddr + BN, rs);
        tmem_ld_wait();
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int nb = n0 + c + 8 * h;
          if (nb >= npad) break;
          float v[8];
#pragma unroll
          for (int j = 0; j < 8; ++j)
            v[j] = __fadd_rn(__uint_as_float(r[8 * h + j]), __uint_as_float(rs[8 * h + j]));
          if (partial) {
            if (m < M) {
              float4* dst = reinterpret_cast<float4*>(
                  partial + ((size_t)blockIdx.z * M + m) * npad + nb);
              dst[0] = make_float4(v[0], v[1], v[2], v[3]);
              dst[1] = make_float4(v[4], v[5], v[6], v[7]);
            }
          } else {
            ep.store8(m, nb, v);
          }
        }
      }
    }
  } else if (lane == 0) {
    // ---------------- MMA issuer --------------------------------------------
    constexpr uint32_t idesc = sg_idesc(SG_BM, BN, VA::MN, VB::MN);
    // (a plane, b plane) per MMA; the last is the big b0*b0 term
    constexpr int AP[6] = {0, 2, 1, 0, 1, 0};
    constexpr int BP[6] = {2, 0, 1, 1, 0, 0};
    for (int kb = 0; kb < nkb; ++kb) {
      const int stage = kb % STAGES;
      mbar_wait(&full_bar[stage], (kb / STAGES) & 1);
      tc_fence_after();
      const uint32_t a0 = smem_base + stage * Cfg::STAGE_BYTES;
      const uint32_t b0 = a0 + 3 * Cfg::A_BYTES;
#pragma unroll
      for (int j = 0; j < Cfg::KSTEPS; ++j) {
        const uint32_t off = j * 2 * Cfg::LBO;
#pragma unroll
        for (int i = 0; i < 6; ++i) {
          const uint64_t da = umma_desc_kmajor(a0 + AP[i] * Cfg::A_BYTES + off, Cfg::LBO, Cfg::SBO);
          const uint64_t db = umma_desc_kmajor(b0 + BP[i] * Cfg::B_BYTES + off, Cfg::LBO, Cfg::SBO);
          const bool big = i == 5;
          const bool first = (kb | j) == 0 && (big || i == 0);
          umma_f16(tmem_base + (big ? 0u : (uint32_t)BN), da, db, idesc, first ? 0u : 1u);
        }
      }
      umma_commit(&empty_bar[stage]);
    }
    umma_commit(done_bar);
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 8) {
    tc_fence_after();
    tmem_dealloc(tmem_base, Cfg::TMEM_COLS);
  }
}

// deterministic split-K reduction (fixed split order) + epilogue, 8 columns
// per thread
template <class EP>
__global__ void sgemm_reduce_kernel(const float* __restrict__ partial, int splits, int M, int N,
                                    EP ep) {
  const int npad = cdiv(N, 8) * 8;
  const int chunks = npad / 8;
  const size_t total = (size_t)M * chunks;
  const size_t zs = (size_t)M * npad;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total;
       i += (size_t)gridDim.x * blockDim.x) {
    const int m = (int)(i / chunks), nb = (int)(i % chunks) * 8;
    const float* src = partial + (size_t)m * npad + nb;
    float v[8];
    float4 a = reinterpret_cast<const float4*>(src)[0], b = reinterpret_cast<const float4*>(src)[1];
    v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
    // four splits' loads in flight at a time; the adds keep the fixed split order
    for (int z0 = 1; z0 < splits; z0 += 4) {
      float4 pa[4], pb[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        if (z0 + u < splits) {
          pa[u] = __ldg(reinterpret_cast<const float4*>(src + (z0 + u) * zs));
          pb[u] = __ldg(reinterpret_cast<const float4*>(src + (z0 + u) * zs) + 1);
        }
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        if (z0 + u < splits) {
          v[0] = __fadd_rn(v[0], pa[u].x); v[1] = __fadd_rn(v[1], pa[u].y);
          v[2] = __fadd_rn(v[2], pa[u].z); v[3] = __fadd_rn(v[3], pa[u].w);
          v[4] = __fadd_rn(v[4], pb[u].x); v[5] = __fadd_rn(v[5], pb[u].y);
          v[6] = __fadd_rn(v[6], pb[u].z); v[7] = __fadd_rn(v[7], pb[u].w);
        }
      }
    }
    ep.store8(m, nb, v);
  }
}

// Split-K reduction for many splits (S >= 16): the plain kernel above gives
// one thread per 8-column chunk a serial walk over all S partials, which is
// latency-bound when M*N is small (conv1's weight gradient: 4,608 threads x
// 118 splits).  Here a block of 256 threads covers 32 chunks x 8 z-lanes;
// lane l sums splits l, l+8, l+16, ... in order, and the 8 lane sums are then
// added in lane order through shared memory -- a fixed order, so the result
// is deterministic (it differs from the serial order only by fp32 rounding).
template <class EP>
__global__ void __launch_bounds__(256) sgemm_reduce_wide_kernel(const float* __restrict__ partial,
                                                                 int splits, int M, int N, EP ep) {
  __shared__ float red[8][32][9];
  const int npad = cdiv(N, 8) * 8;
  const int chunks = npad / 8;
  const size_t total = (size_t)M * chunks;
  const size_t zs = (size_t)M * npad;
  const int cl = threadIdx.x & 31, zl = threadIdx.x >> 5;
  for (size_t base = (size_t)blockIdx.x * 32; base < total; base += (size_t)gridDim.x * 32) {
    const size_t i = base + cl;
    float v[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] = 0.f;
    if (i < total) {
      const int m = (int)(i / chunks), nb = (int)(i % chunks) * 8;
      const float* src = partial + (size_t)m * npad + nb;
      for (int z = zl; z < splits; z += 16) {
        const bool two = z + 8 < splits;
        const float4 a = __ldg(reinterpret_cast<const float4*>(src + z * zs));
        const float4 b = __ldg(reinterpret_cast<const float4*>(src + z * zs) + 1);
        float4 c = make_float4(0.f, 0.f, 0.f, 0.f), d = c;
        if (two) {
          c = __ldg(reinterpret_cast<const float4*>(src + (z + 8) * zs));
          d = __ldg(reinterpret_cast<const float4*>(src + (z + 8) * zs) + 1);
        }
        v[0] = __fadd_rn(v[0], a.x); v[1] = __fadd_rn(v[1], a.y);
        v[2] = __fadd_rn(v[2], a.z); v[3] = __fadd_rn(v[3], a.w);
        v[4] = __fadd_rn(v[4], b.x); v[5] = __fadd_rn(v[5], b.y);
        v[6] = __fadd_rn(v[6], b.z); v[7] = __fadd_rn(v[7], b.w);
        if (two) {
          v[0] = __fadd_rn(v[0], c.x); v[1] = __fadd_rn(v[1], c.y);
          v[2] = __fadd_rn(v[2], c.z); v[3] = __fadd_rn(v[3], c.w);
          v[4] = __fadd_rn(v[4], d.x); v[5] = __fadd_rn(v[5], d.y);
          v[6] = __fadd_rn(v[6], d.z); v[7] = __fadd_rn(v[7], d.w);
        }
      }
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) red[zl][cl][j] = v[j];
    __syncthreads();
    if (zl == 0 && i < total) {
#pragma unroll
      for (int l = 1; l < 8; ++l)
#pragma unroll
        for (int j = 0; j < 8; ++j) v[j] = __fadd_rn(v[j], red[l][cl][j]);
      const int m = (int)(i / chunks), nb = (int)(i % chunks) * 8;
      ep.store8(m, nb, v);
    }
    __syncthreads();
  }
}

}  // namespace stz
