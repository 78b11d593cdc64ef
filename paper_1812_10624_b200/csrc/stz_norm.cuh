// ResNet-trunk kernels on the split-plane formats:
// training-mode BatchNorm, global average pooling and the residual add.
//
// The reference has none of these layer kinds (tensor_core.py:37-74); their
// semantics are the oracle's (oracle/stanza_oracle.py bn_forward /
// bn_backward / gap_forward / gap_backward / "residual"), all statistics and
// per-element arithmetic in float64 with one fp32 rounding, reductions in a
// fixed order (deterministic).  Every kernel is HBM-bound: 8 channels per
// thread as 16-byte loads of each plane.
//
// BatchNorm statistics are per GROUP of `group` samples (one CONV worker's
// batch) so that the co-located single-GPU trunk, which runs n_c workers'
// batches as one N = n_c*K pass, normalises exactly as each worker would.
#pragma once

#include <cooperative_groups.h>

#include "stz_fmt.cuh"

namespace stz {

// gradient of a ReLU output -> gradient of its input: zero where the output
// (plane 0, whose sign is the value's) is not > 0
__device__ __forceinline__ void apply_mask8(const bf16_t* m, float (&v)[8]) {
  const uint4 w = *reinterpret_cast<const uint4*>(m);
  const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    if (!(bf2f((bf16_t)(ws[j] & 0xFFFF)) > 0.f)) v[2 * j] = 0.f;
    if (!(bf2f((bf16_t)(ws[j] >> 16)) > 0.f)) v[2 * j + 1] = 0.f;
  }
}

// Per (group, row slice, channel) float64 partial sums.
//   forward : (sum x, sum x^2)
//   backward: (sum g, sum g*x); the finalize forms sum g*xhat =
//             rstd*(sum g*x - mean*sum g) (fp32 products are exact in float64)
// Block = 256 threads as L channel-chunk lanes x R row lanes (L = min(chunks
// left in this 32-chunk tile, 32), R = 256 / L); grid (slices, groups, tiles).
// Several rows' loads are in flight per thread (the loop is latency-bound with
// one); each thread's adds stay in row order.
template <bool BWD>
__global__ void __launch_bounds__(256, 2) bn_reduce_kernel(
    const bf16_t* __restrict__ x, size_t psx, const bf16_t* __restrict__ g, size_t psg,
    const bf16_t* __restrict__ mask, double* __restrict__ partial, int HW, int C8, int group,
    int rows_per_slice) {
  __shared__ double red[256][16];
  const int nch = C8 / 8, ct = blockIdx.z;
  const int L = min(nch - ct * 32, 32), R = 256 / L;
  const int t = threadIdx.x, cl = t % L, rl = t / L;
  const int gi = blockIdx.y, slice = blockIdx.x, nslices = gridDim.x;
  const size_t grows = (size_t)group * HW, grow0 = (size_t)gi * grows;
  const size_t r0 = (size_t)slice * rows_per_slice;
  const size_t r1 = min(grows, r0 + (size_t)rows_per_slice);
  const int cc = ct * 32 + cl;
  double s[8], q[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) s[j] = q[j] = 0.0;
  auto acc_row = [&](const float (&v)[8], const float (&gv)[8]) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const double a = BWD ? (double)gv[j] : (double)v[j];
      s[j] += a;
      q[j] = fma(a, (double)v[j], q[j]);
    }
  };
  auto load_row = [&](size_t r, float (&v)[8], float (&gv)[8]) {
    const size_t off = (grow0 + r) * C8 + (size_t)cc * 8;
    load_split8(x + off, psx, v);
    if (BWD) {
      load_split8(g + off, psg, gv);
      if (mask) apply_mask8(mask + off, gv);
    }
  };
  constexpr int U = BWD ? 2 : 4;   // rows in flight (the backward loads two operands)
  if (rl < R) {
    size_t r = r0 + rl;
    for (; r + (U - 1) * (size_t)R < r1; r += U * (size_t)R) {
      float v[U][8], gv[U][8];
#pragma unroll
      for (int u = 0; u < U; ++u) load_row(r + u * (size_t)R, v[u], gv[u]);
#pragma unroll
      for (int u = 0; u < U; ++u) acc_row(v[u], gv[u]);
    }
    for (; r < r1; r += R) {
      float v[8], gv[8];
      load_row(r, v, gv);
      acc_row(v, gv);
    }
  }
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    red[t][j] = s[j];
    red[t][8 + j] = q[j];
  }
  __syncthreads();
  for (int idx = t; idx < L * 16; idx += 256) {   // (lane, quantity): fixed-order sum over row lanes
    const int lane = idx % L, jj = idx / L;
    double acc = 0.0;
    for (int r = 0; r < R; ++r) acc += red[r * L + lane][jj];
    const int c = (ct * 32 + lane) * 8 + (jj & 7);
    partial[(((size_t)gi * nslices + slice) * C8 + c) * 2 + (jj >> 3)] = acc;
  }
}

// lane's share of a (sum, sum2) pair column: slices lane, lane + 32, ... in
// order, eight slices' loads in flight per step (the finals are latency-bound)
__device__ __forceinline__ void bn_sum_slices(const double* __restrict__ p, size_t stride,
                                              int nslices, int lane, double& s, double& q) {
  int k = lane;
  for (; k + 224 < nslices; k += 256) {
    double2 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = *reinterpret_cast<const double2*>(p + (size_t)(k + 32 * u) * stride);
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      s += v[u].x;
      q += v[u].y;
    }
  }
  for (; k < nslices; k += 32) {
    const double2 v = *reinterpret_cast<const double2*>(p + (size_t)k * stride);
    s += v.x;
    q += v.y;
  }
}

// forward finalize: per (group, channel) mean and rstd = 1/sqrt(var + eps),
// var = E[x^2] - mean^2 (float64; clamped at 0), kept in `stats` for the
// backward; and the apply pass's affine form y = x*A + B, A = rstd*gamma,
// B = beta - mean*A (float64; padded channels A = B = 0)
__global__ void bn_stats_final_kernel(const double* __restrict__ partial, double* __restrict__ stats,
                                      double2* __restrict__ coef, const float* __restrict__ gamma,
                                      const float* __restrict__ beta, int G, int nslices, int C,
                                      int C8, double m, double eps) {
  // one warp per (group, channel): lanes take slices l, l+32, ... and a fixed
  // xor-shuffle tree combines them (deterministic)
  const int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (i >= G * C8) return;
  const int gi = i / C8, c = i % C8;
  double s = 0.0, q = 0.0;
  bn_sum_slices(partial + ((size_t)gi * nslices * C8 + c) * 2, (size_t)C8 * 2, nslices, lane, s, q);
  for (int o = 16; o > 0; o >>= 1) {
    s += __shfl_xor_sync(0xffffffffu, s, o);
    q += __shfl_xor_sync(0xffffffffu, q, o);
  }
  if (lane) return;
  const double mean = s / m;
  const double var = fmax(q / m - mean * mean, 0.0);
  const double rstd = 1.0 / sqrt(var + eps);
  stats[(size_t)i * 2] = mean;
  stats[(size_t)i * 2 + 1] = rstd;
  const double A = c < C ? rstd * (double)gamma[c] : 0.0;
  coef[i] = make_double2(A, c < C ? (double)beta[c] - mean * A : 0.0);
}

// backward finalize: per-group (sum g, sum g*xhat) -> the apply pass's
// affine form gx = P*g + Q*x + R with coef = gamma*rstd/m:
//   P = coef*m, Q = -coef*sgx*rstd, R = coef*(sgx*rstd*mean - sg)
// and the parameter-gradient batch sums dgamma = sum g*xhat, dbeta = sum g
// over all groups (written, or added in fp32 with `accumulate`)
__global__ void bn_bwd_final_kernel(const double* __restrict__ partial,
                                    const double* __restrict__ stats,
                                    const float* __restrict__ gamma, double4* __restrict__ coef,
                                    float* __restrict__ ggamma, float* __restrict__ gbeta, int G,
                                    int nslices, int C, int C8, double m, int accumulate) {
  // one warp per channel (groups in order; slices over the lanes, fixed tree)
  const int c = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (c >= C8) return;
  double tg = 0.0, tgx = 0.0;
  for (int gi = 0; gi < G; ++gi) {
    double s = 0.0, q = 0.0;
    bn_sum_slices(partial + ((size_t)gi * nslices * C8 + c) * 2, (size_t)C8 * 2, nslices, lane, s,
                  q);
    for (int o = 16; o > 0; o >>= 1) {
      s += __shfl_xor_sync(0xffffffffu, s, o);
      q += __shfl_xor_sync(0xffffffffu, q, o);
    }
    const size_t i = (size_t)gi * C8 + c;
    const double mean = stats[i * 2], rstd = stats[i * 2 + 1];
    q = rstd * (q - mean * s);   // sum g*x -> sum g*xhat
    const double cf = c < C ? (double)gamma[c] * rstd / m : 0.0;
    if (lane == 0)
      coef[i] = make_double4(cf * m, -cf * q * rstd, cf * (q * rstd * mean - s), 0.0);
    tg += s;
    tgx += q;
  }
  if (c < C && lane == 0) {
    ggamma[c] = accumulate ? __fadd_rn(ggamma[c], (float)tgx) : (float)tgx;
    gbeta[c] = accumulate ? __fadd_rn(gbeta[c], (float)tg) : (float)tg;
  }
}

// The apply passes use the reduce kernels' block shape: L channel-chunk lanes
// x R row lanes over a slice of rows.  The float64 coefficients of the (at
// most two) sample groups a slice touches are staged in shared memory as
// [group][quantity][j][lane] (consecutive lanes -> consecutive words); the
// host makes slices no longer than a group, so a slice spans at most two.
// Four rows' loads are in flight per thread.
constexpr int BN_APPLY_U = 4;

template <int NQ, typename CT>
__device__ __forceinline__ void bn_stage_coef(double* sc, const CT* __restrict__ coef, int g_lo,
                                              int ng, int C8, int ct, int L) {
  for (int i = threadIdx.x; i < ng * NQ * 8 * L; i += blockDim.x) {
    const int lane = i % L, j = (i / L) % 8, qd = (i / (8 * L)) % NQ, gg = i / (8 * L * NQ);
    const double* src = reinterpret_cast<const double*>(&coef[(size_t)(g_lo + gg) * C8 + (ct * 32 + lane) * 8 + j]);
    sc[((gg * NQ + qd) * 8 + j) * 32 + lane] = src[qd];
  }
}

// y = x*A + B (float64, one rounding), then optionally + residual (fp32
// add) and ReLU.  grid (slices, channel tiles).
__global__ void __launch_bounds__(256, 2) bn_apply_kernel(
    const bf16_t* __restrict__ x, size_t psx, const double2* __restrict__ coef,
    const bf16_t* __restrict__ res, size_t psr, bf16_t* __restrict__ y, size_t psy,
    uint32_t rows, uint32_t rows_per_slice, FastDiv d_grows, int C8, int relu) {
  __shared__ double sc[2 * 2 * 8 * 32];
  const int nch = C8 / 8, ct = blockIdx.y;
  const int L = min(nch - ct * 32, 32), R = 256 / L;
  const int t = threadIdx.x, cl = t % L, rl = t / L;
  const int cc = ct * 32 + cl;
  const uint32_t r0 = blockIdx.x * rows_per_slice, r1 = min(rows, r0 + rows_per_slice);
  if (r0 >= r1) return;
  const uint32_t g_lo = d_grows.div(r0), ng = d_grows.div(r1 - 1) - g_lo + 1;   // <= 2
  bn_stage_coef<2>(sc, coef, (int)g_lo, (int)ng, C8, ct, L);
  __syncthreads();
  if (rl >= R) return;
  auto row = [&](uint32_t r, float (&v)[8], const float (&rr)[8]) {
    const uint32_t gg = d_grows.div(r) - g_lo;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const double A = sc[((gg * 2 + 0) * 8 + j) * 32 + cl];
      const double B = sc[((gg * 2 + 1) * 8 + j) * 32 + cl];
      float o = (float)fma((double)v[j], A, B);
      if (res) o = __fadd_rn(o, rr[j]);
      if (relu) o = o > 0.f ? o : 0.f;
      v[j] = o;
    }
    store_split8(y + (size_t)r * C8 + cc * 8, psy, v);
  };
  uint32_t r = r0 + rl;
  for (; r + (BN_APPLY_U - 1) * (uint32_t)R < r1; r += BN_APPLY_U * (uint32_t)R) {
    float v[BN_APPLY_U][8], rr[BN_APPLY_U][8];
#pragma unroll
    for (int u = 0; u < BN_APPLY_U; ++u) {
      const size_t off = (size_t)(r + u * R) * C8 + cc * 8;
      load_split8(x + off, psx, v[u]);
      if (res) load_split8(res + off, psr, rr[u]);
    }
#pragma unroll
    for (int u = 0; u < BN_APPLY_U; ++u) row(r + u * R, v[u], rr[u]);
  }
  for (; r < r1; r += R) {
    const size_t off = (size_t)r * C8 + cc * 8;
    float v[8], rr[8];
    load_split8(x + off, psx, v);
    if (res) load_split8(res + off, psr, rr);
    row(r, v, rr);
  }
}

// gx = P*g + Q*x + R (float64, one rounding); g masked by a ReLU output
// when `mask` is given
__global__ void __launch_bounds__(256, 2) bn_bwd_apply_kernel(
    const bf16_t* __restrict__ g, size_t psg, const bf16_t* __restrict__ mask,
    const bf16_t* __restrict__ x, size_t psx, const double4* __restrict__ coef,
    bf16_t* __restrict__ gx, size_t psgx, double* __restrict__ bpart, uint32_t rows,
    uint32_t rows_per_slice, FastDiv d_grows, int C8) {
  __shared__ double sc[2 * 3 * 8 * 32];
  __shared__ double red[256 * 8];
  const int nch = C8 / 8, ct = blockIdx.y;
  const int L = min(nch - ct * 32, 32), R = 256 / L;
  const int t = threadIdx.x, cl = t % L, rl = t / L;
  const int cc = ct * 32 + cl;
  const uint32_t r0 = blockIdx.x * rows_per_slice, r1 = min(rows, r0 + rows_per_slice);
  if (r0 >= r1) {   // an empty trailing slice still owns its partials
    if (bpart)
      for (int e = t; e < L * 8; e += 256) bpart[(size_t)blockIdx.x * C8 + ct * 256 + e] = 0.0;
    return;
  }
  const uint32_t g_lo = d_grows.div(r0), ng = d_grows.div(r1 - 1) - g_lo + 1;   // <= 2
  bn_stage_coef<3>(sc, coef, (int)g_lo, (int)ng, C8, ct, L);
  __syncthreads();
  double bs[8];   // batch sums of this thread's gx values (the input bias gradient)
#pragma unroll
  for (int j = 0; j < 8; ++j) bs[j] = 0.0;
  auto row = [&](uint32_t r, float (&v)[8], const float (&gv)[8]) {
    const uint32_t gg = d_grows.div(r) - g_lo;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const double P = sc[((gg * 3 + 0) * 8 + j) * 32 + cl];
      const double Q = sc[((gg * 3 + 1) * 8 + j) * 32 + cl];
      const double Rc = sc[((gg * 3 + 2) * 8 + j) * 32 + cl];
      v[j] = (float)fma(P, (double)gv[j], fma(Q, (double)v[j], Rc));
      bs[j] += (double)v[j];
    }
    store_split8(gx + (size_t)r * C8 + cc * 8, psgx, v);
  };
  uint32_t r = rl < R ? r0 + rl : r1;
  for (; r + (BN_APPLY_U - 1) * (uint32_t)R < r1; r += BN_APPLY_U * (uint32_t)R) {
    float v[BN_APPLY_U][8], gv[BN_APPLY_U][8];
#pragma unroll
    for (int u = 0; u < BN_APPLY_U; ++u) {
      const size_t off = (size_t)(r + u * R) * C8 + cc * 8;
      load_split8(x + off, psx, v[u]);
      load_split8(g + off, psg, gv[u]);
      if (mask) apply_mask8(mask + off, gv[u]);
    }
#pragma unroll
    for (int u = 0; u < BN_APPLY_U; ++u) row(r + u * R, v[u], gv[u]);
  }
  for (; r < r1; r += R) {
    const size_t off = (size_t)r * C8 + cc * 8;
    float v[8], gv[8];
    load_split8(x + off, psx, v);
    load_split8(g + off, psg, gv);
    if (mask) apply_mask8(mask + off, gv);
    row(r, v, gv);
  }
  if (!bpart) return;
  // fixed-order sum over the row lanes -> bpart[slice][c]
#pragma unroll
  for (int j = 0; j < 8; ++j) red[t * 8 + j] = bs[j];
  __syncthreads();
  for (int e = t; e < L * 8; e += 256) {
    const int lane = e >> 3, j = e & 7;
    double acc = 0.0;
    for (int q = 0; q < R; ++q) acc += red[(q * L + lane) * 8 + j];
    bpart[(size_t)blockIdx.x * C8 + (ct * 32 + lane) * 8 + j] = acc;
  }
}

// global average pool: NHWC [N][HW][C8] -> rows [N][C8] (= NHWC [N][1][1][C8])
__global__ void gap_fwd_kernel(const bf16_t* __restrict__ x, size_t psx, bf16_t* __restrict__ y,
                               size_t psy, int N, int HW, int C8) {
  const int nch = C8 / 8;
  STZ_GRID_LOOP(i, (size_t)N * nch) {
    const size_t n = i / nch;
    const int cc = (int)(i % nch);
    double s[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) s[j] = 0.0;
    for (int p = 0; p < HW; ++p) {
      float v[8];
      load_split8(x + (n * HW + p) * C8 + (size_t)cc * 8, psx, v);
#pragma unroll
      for (int j = 0; j < 8; ++j) s[j] += (double)v[j];
    }
    float o[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) o[j] = (float)__ddiv_rn(s[j], (double)HW);
    store_split8(y + n * C8 + (size_t)cc * 8, psy, o);
  }
}

__global__ void gap_bwd_kernel(const bf16_t* __restrict__ gy, size_t psg, bf16_t* __restrict__ gx,
                               size_t psx, int N, int HW, int C8) {
  const int nch = C8 / 8;
  STZ_GRID_LOOP(i, (size_t)N * HW * nch) {
    const size_t pix = i / nch, n = pix / HW;
    const int cc = (int)(i % nch);
    float v[8];
    load_split8(gy + n * C8 + (size_t)cc * 8, psg, v);
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] = (float)__ddiv_rn((double)v[j], (double)HW);
    store_split8(gx + pix * C8 + (size_t)cc * 8, psx, v);
  }
}

// y = a + b (fp32 RN), n elements (multiple of 8); b masked by a ReLU output
// (plane 0 > 0) when `mask_b` is given
__global__ void add_split_kernel(const bf16_t* __restrict__ a, size_t psa,
                                 const bf16_t* __restrict__ b, size_t psb,
                                 const bf16_t* __restrict__ mask_b, bf16_t* __restrict__ y,
                                 size_t psy, size_t n8) {
  STZ_GRID_LOOP(i, n8) {
    float va[8], vb[8];
    load_split8(a + i * 8, psa, va);
    load_split8(b + i * 8, psb, vb);
    if (mask_b) apply_mask8(mask_b + i * 8, vb);
#pragma unroll
    for (int j = 0; j < 8; ++j) va[j] = __fadd_rn(va[j], vb[j]);
    store_split8(y + i * 8, psy, va);
  }
}


// ---------------------------------------------------------------------------
// Inception-V3 kinds (§8f row 4; semantics oracle/stanza_oracle.py
// avgpool_forward / avgpool_backward / "concat")
// ---------------------------------------------------------------------------

// AvgPool2d forward, NHWC split planes, 8 channels per thread: float64 sum of
// the window taps in (kh, kw) order (padding contributes nothing), divided by
// k*k, one fp32 rounding
__global__ void __launch_bounds__(256) avgpool_fwd_kernel(const bf16_t* __restrict__ x, size_t psx,
                                                          bf16_t* __restrict__ y, size_t psy,
                                                          int N, int H, int W, int C8, int OH,
                                                          int OW, int k, int s, int p) {
  const int nch = C8 / 8;
  const double kk = (double)(k * k);
  STZ_GRID_LOOP(i, (size_t)N * OH * OW * nch) {
    const int cc = (int)(i % nch);
    const size_t pix = i / nch;
    const int ow = (int)(pix % OW), oh = (int)((pix / OW) % OH);
    const size_t n = pix / ((size_t)OW * OH);
    double acc[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[j] = 0.0;
    for (int kh = 0; kh < k; ++kh) {
      const int h = oh * s + kh - p;
      if (h < 0 || h >= H) continue;
      for (int kw = 0; kw < k; ++kw) {
        const int w = ow * s + kw - p;
        if (w < 0 || w >= W) continue;
        float v[8];
        load_split8(x + ((n * H + h) * W + w) * C8 + (size_t)cc * 8, psx, v);
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[j] += (double)v[j];
      }
    }
    float o[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) o[j] = (float)__ddiv_rn(acc[j], kk);
    store_split8(y + pix * C8 + (size_t)cc * 8, psy, o);
  }
}

// AvgPool2d backward (gather form): input cell (h, w) sums g[oh, ow] / (k*k)
// (float64 quotient per term) over the windows covering it, in (kh, kw) order
__global__ void __launch_bounds__(256) avgpool_bwd_kernel(const bf16_t* __restrict__ gy, size_t psg,
                                                          bf16_t* __restrict__ gx, size_t psx,
                                                          int N, int H, int W, int C8, int OH,
                                                          int OW, int k, int s, int p) {
  const int nch = C8 / 8;
  const double kk = (double)(k * k);
  const double rk = 1.0 / kk;   // RN(1/kk)
  STZ_GRID_LOOP(i, (size_t)N * H * W * nch) {
    const int cc = (int)(i % nch);
    const size_t pix = i / nch;
    const int w = (int)(pix % W), h = (int)((pix / W) % H);
    const size_t n = pix / ((size_t)W * H);
    double acc[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[j] = 0.0;
    for (int kh = 0; kh < k; ++kh) {
      const int th = h + p - kh;
      if (th < 0 || th % s) continue;
      const int oh = th / s;
      if (oh >= OH) continue;
      for (int kw = 0; kw < k; ++kw) {
        const int tw = w + p - kw;
        if (tw < 0 || tw % s) continue;
        const int ow = tw / s;
        if (ow >= OW) continue;
        float v[8];
        load_split8(gy + ((n * OH + oh) * OW + ow) * C8 + (size_t)cc * 8, psg, v);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          // v / kk correctly rounded without a division: q0 = RN(v * RN(1/kk)) is
          // faithful, the remainder v - q0*kk is exact (fma), and one
          // correction step RN(q0 + r * RN(1/kk)) is the correctly rounded
          // quotient (Markstein) -- the same double as __ddiv_rn
          const double x = (double)v[j], q0 = x * rk, r = fma(-q0, kk, x);
          acc[j] += fma(r, rk, q0);
        }
      }
    }
    float o[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) o[j] = (float)acc[j];
    store_split8(gx + pix * C8 + (size_t)cc * 8, psx, o);
  }
}

// channel-slice copy of split-plane rows: dst[r][d0 + c] = src[r][s0 + c] for
// c < C (C, s0, d0, both row pitches multiples of 8): the Inception concat
// (branch output -> its channel slice) and its backward (slice -> branch).
// With `mask` (row pitch mask8, offset m0): zero where the mask value (a ReLU
// output, plane 0) is not > 0 -- the branch's closing ReLU backward, fused
__global__ void __launch_bounds__(256) copy_channels_kernel(const bf16_t* __restrict__ src,
                                                            size_t pss, int src8, int s0,
                                                            bf16_t* __restrict__ dst, size_t psd,
                                                            int dst8, int d0, size_t R, int C,
                                                            const bf16_t* __restrict__ mask,
                                                            int mask8, int m0) {
  const int nch = C / 8;
  STZ_GRID_LOOP(i, R * nch) {
    const size_t r = i / nch;
    const int cc = (int)(i % nch) * 8;
    const bf16_t* a = src + r * src8 + s0 + cc;
    bf16_t* b = dst + r * dst8 + d0 + cc;
    if (mask) {
      float v[8];
      load_split8(a, pss, v);
      apply_mask8(mask + r * mask8 + m0 + cc, v);
      store_split8(b, psd, v);
      continue;
    }
#pragma unroll
    for (int q = 0; q < 3; ++q)
      *reinterpret_cast<uint4*>(b + q * psd) = __ldg(reinterpret_cast<const uint4*>(a + q * pss));
  }
}

// y = ((x0 + x1) + x2) + x3 (fp32 RN, the first n inputs): the Inception
// concat's input gradient, one pass over every branch's input gradient
__global__ void __launch_bounds__(256) add_n_split_kernel(const bf16_t* __restrict__ x0,
                                                          const bf16_t* __restrict__ x1,
                                                          const bf16_t* __restrict__ x2,
                                                          const bf16_t* __restrict__ x3,
                                                          size_t psx0, size_t psx1, size_t psx2,
                                                          size_t psx3, int n, bf16_t* y,
                                                          size_t psy, size_t n8) {
  STZ_GRID_LOOP(i, n8) {
    float acc[8], v[8];
    load_split8(x0 + i * 8, psx0, acc);
    load_split8(x1 + i * 8, psx1, v);
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[j] = __fadd_rn(acc[j], v[j]);
    if (n > 2) {
      load_split8(x2 + i * 8, psx2, v);
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[j] = __fadd_rn(acc[j], v[j]);
    }
    if (n > 3) {
      load_split8(x3 + i * 8, psx3, v);
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[j] = __fadd_rn(acc[j], v[j]);
    }
    store_split8(y + i * 8, psy, acc);
  }
}


// ---------------------------------------------------------------------------
// One-launch BatchNorm (forward and backward) for the step's graphs
// ---------------------------------------------------------------------------
//
// The three-launch form above (reduce, finalize, apply) costs two kernel
// boundaries per BatchNorm and reads the input twice; at ResNet-50's later
// stages (1568-6272 rows at K = 32) a BatchNorm is a few MB and the launches,
// not the bytes, set its time (profiles/r02: 25-35 us for 2-15 MB).  Here one
// cooperative grid (every CTA resident: cudaLaunchAttributeCooperative) runs
// the phases with grid-wide barriers between them:
//
//   1  each CTA = (group, row slice, 256-channel tile) loads its rows once --
//      x (and g, ReLU-masked) as fp32 kept in shared memory up to `kcap` rows
//      per thread -- and writes its float64 partial sums (as bn_reduce_kernel)
//   2  the grid's warps finalize every (group, channel) -- the same float64
//      formulas as bn_stats_final_kernel / bn_bwd_final_kernel
//   3  each CTA applies the affine form to its rows from shared memory
//      (re-reading only rows beyond the cache) and stores y / gx
//   4  (backward with a producing-conv bias) per-slice sums of gx, then the
//      grid's warps sum them per channel in slice order (colsum_final_kernel)
//
// Every sum runs in a fixed order (deterministic); the float64 arithmetic per
// element is the three-launch path's.
constexpr int BNF_THREADS = 512;
constexpr int BNF_RED_Q = 4;   // quantities per block-reduction round

struct BnFusedParams {
  const bf16_t* x; size_t psx;
  const bf16_t* g; size_t psg;         // backward: output gradient
  const bf16_t* mask;                  // backward: ReLU output masking g (or null)
  const bf16_t* res; size_t psr;       // forward: residual added after the affine (or null)
  bf16_t* y; size_t psy;               // forward: y; backward: gx (null: no input gradient)
  double* partial;                     // [G][spg][C8][2]
  double* stats;                       // [G][C8][2] (mean, rstd): forward writes, backward reads
  const float* gamma; const float* beta;
  float* ggamma; float* gbeta;         // backward: parameter gradients
  float* gbias;                        // backward: the producing conv's bias gradient (or null)
  double* bpart;                       // [G * spg][C8] per-slice gx sums (gbias)
  double m, eps;
  size_t grows;                        // rows per group (group * HW)
  int C, C8, G, spg, tiles, rps, kcap, relu, accumulate;
};

__device__ __forceinline__ void bnf_put(float4* c, const float (&v)[8]) {
  c[0] = make_float4(v[0], v[1], v[2], v[3]);
  c[1] = make_float4(v[4], v[5], v[6], v[7]);
}
__device__ __forceinline__ void bnf_get(const float4* c, float (&v)[8]) {
  const float4 a = c[0], b = c[1];
  v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
  v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
}

// fixed-order sum over the R row lanes of NQ per-thread quantities ->
// out(lane, quantity, value) for lane < L (rounds of BNF_RED_Q quantities)
template <int NQ, class F>
__device__ __forceinline__ void bnf_block_reduce(double* red, const double (&val)[NQ], int L, int R,
                                                 F&& out) {
  const int t = threadIdx.x;
#pragma unroll
  for (int q0 = 0; q0 < NQ; q0 += BNF_RED_Q) {
#pragma unroll
    for (int j = 0; j < BNF_RED_Q; ++j) red[j * BNF_THREADS + t] = val[q0 + j];
    __syncthreads();
    if (t < L * BNF_RED_Q) {
      const int lane = t % L, j = t / L;
      double acc = 0.0;
      for (int r = 0; r < R; ++r) acc += red[j * BNF_THREADS + r * L + lane];
      out(lane, q0 + j, acc);
    }
    __syncthreads();
  }
}

template <bool BWD>
__global__ void __launch_bounds__(BNF_THREADS, 1) bn_fused_kernel(const __grid_constant__ BnFusedParams p) {
  extern __shared__ float4 bnf_cache[];
  __shared__ double red[BNF_RED_Q * BNF_THREADS];
  __shared__ double sc[3 * 8 * 32];
  cooperative_groups::grid_group grid = cooperative_groups::this_grid();
  const int nch = p.C8 / 8;
  const int b = blockIdx.x, ct = b % p.tiles, rest = b / p.tiles;
  const int slice = rest % p.spg, gi = rest / p.spg;
  const int L = min(nch - ct * 32, 32), R = BNF_THREADS / L;
  const int t = threadIdx.x, cl = t % L, rl = t / L;
  const bool act = rl < R;
  const int cc = ct * 32 + cl;
  const size_t grow0 = (size_t)gi * p.grows;
  const size_t r0 = min(p.grows, (size_t)slice * p.rps), r1 = min(p.grows, r0 + (size_t)p.rps);
  const int nslot = R * L, slot = rl * L + cl;
  float4* cx = bnf_cache;                                    // [kcap][nslot][2]
  float4* cgr = bnf_cache + (size_t)p.kcap * nslot * 2;      // backward: g
  const int warp = t >> 5, lane = t & 31;
  const int gw = b * (BNF_THREADS / 32) + warp, nw = gridDim.x * (BNF_THREADS / 32);

  // ---- phase 1: load (cache) + float64 partial sums ------------------------
  {
    double s[8], q[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) s[j] = q[j] = 0.0;
    auto load_row = [&](size_t r, int k, float (&v)[8], float (&gv)[8]) {
      const size_t off = (grow0 + r) * p.C8 + (size_t)cc * 8;
      load_split8(p.x + off, p.psx, v);
      if (BWD) {
        load_split8(p.g + off, p.psg, gv);
        if (p.mask) apply_mask8(p.mask + off, gv);
      }
      if (k < p.kcap) {
        bnf_put(cx + ((size_t)k * nslot + slot) * 2, v);
        if (BWD) bnf_put(cgr + ((size_t)k * nslot + slot) * 2, gv);
      }
    };
    auto acc_row = [&](const float (&v)[8], const float (&gv)[8]) {
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const double a = BWD ? (double)gv[j] : (double)v[j];
        s[j] += a;
        q[j] = fma(a, (double)v[j], q[j]);
      }
    };
    constexpr int U = BWD ? 2 : 4;
    if (act) {
      size_t r = r0 + rl;
      int k = 0;
      for (; r + (U - 1) * (size_t)R < r1; r += U * (size_t)R, k += U) {
        float v[U][8], gv[U][8];
#pragma unroll
        for (int u = 0; u < U; ++u) load_row(r + u * (size_t)R, k + u, v[u], gv[u]);
#pragma unroll
        for (int u = 0; u < U; ++u) acc_row(v[u], gv[u]);
      }
      for (; r < r1; r += R, ++k) {
        float v[8], gv[8];
        load_row(r, k, v, gv);
        acc_row(v, gv);
      }
    }
    double val[16];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      val[j] = act ? s[j] : 0.0;
      val[8 + j] = act ? q[j] : 0.0;
    }
    double* part = p.partial + ((size_t)gi * p.spg + slice) * p.C8 * 2;
    bnf_block_reduce<16>(red, val, L, R, [&](int ln, int jj, double a) {
      part[((size_t)(ct * 32 + ln) * 8 + (jj & 7)) * 2 + (jj >> 3)] = a;
    });
  }
  grid.sync();

  // ---- phase 2: finalize per (group, channel) ------------------------------
  if (!BWD) {
    for (int i = gw; i < p.G * p.C8; i += nw) {
      const int g2 = i / p.C8, c = i % p.C8;
      double s = 0.0, q = 0.0;
      bn_sum_slices(p.partial + ((size_t)g2 * p.spg * p.C8 + c) * 2, (size_t)p.C8 * 2, p.spg,
                    lane, s, q);
      for (int o = 16; o > 0; o >>= 1) {
        s += __shfl_xor_sync(0xffffffffu, s, o);
        q += __shfl_xor_sync(0xffffffffu, q, o);
      }
      if (lane == 0) {
        const double mean = s / p.m;
        const double var = fmax(q / p.m - mean * mean, 0.0);
        const double rstd = 1.0 / sqrt(var + p.eps);
        p.stats[(size_t)i * 2] = mean;
        p.stats[(size_t)i * 2 + 1] = rstd;
      }
    }
  } else {
    for (int c = gw; c < p.C8; c += nw) {
      double tg = 0.0, tgx = 0.0;
      for (int g2 = 0; g2 < p.G; ++g2) {
        double s = 0.0, q = 0.0;
        bn_sum_slices(p.partial + ((size_t)g2 * p.spg * p.C8 + c) * 2, (size_t)p.C8 * 2, p.spg,
                      lane, s, q);
        for (int o = 16; o > 0; o >>= 1) {
          s += __shfl_xor_sync(0xffffffffu, s, o);
          q += __shfl_xor_sync(0xffffffffu, q, o);
        }
        const size_t i = (size_t)g2 * p.C8 + c;
        const double mean = p.stats[i * 2], rstd = p.stats[i * 2 + 1];
        q = rstd * (q - mean * s);   // sum g*x -> sum g*xhat
        // the partials are no longer needed: keep (sum g, sum g*xhat) in slot 0
        if (lane == 0) {
          p.partial[((size_t)g2 * p.spg * p.C8 + c) * 2] = s;
          p.partial[((size_t)g2 * p.spg * p.C8 + c) * 2 + 1] = q;
        }
        tg += s;
        tgx += q;
      }
      if (c < p.C && lane == 0) {
        p.ggamma[c] = p.accumulate ? __fadd_rn(p.ggamma[c], (float)tgx) : (float)tgx;
        p.gbeta[c] = p.accumulate ? __fadd_rn(p.gbeta[c], (float)tg) : (float)tg;
      }
    }
  }
  if (BWD && !p.y) return;   // uniform over the grid: no input gradient
  grid.sync();

  // ---- phase 3: apply --------------------------------------------------------
  // this CTA's coefficients: forward (A, B), backward (P, Q, R) as float64
  constexpr int NQ = BWD ? 3 : 2;
  for (int i = t; i < 8 * L; i += BNF_THREADS) {
    const int ln = i % L, j = i / L, c = (ct * 32 + ln) * 8 + j;
    const size_t gc = (size_t)gi * p.C8 + c;
    const double mean = p.stats[gc * 2], rstd = p.stats[gc * 2 + 1];
    if (!BWD) {
      const double A = c < p.C ? rstd * (double)p.gamma[c] : 0.0;
      sc[(0 * 8 + j) * 32 + ln] = A;
      sc[(1 * 8 + j) * 32 + ln] = c < p.C ? (double)p.beta[c] - mean * A : 0.0;
    } else {
      const double* f = p.partial + ((size_t)gi * p.spg * p.C8 + c) * 2;
      const double s = f[0], q = f[1];
      const double cf = c < p.C ? (double)p.gamma[c] * rstd / p.m : 0.0;
      sc[(0 * 8 + j) * 32 + ln] = cf * p.m;
      sc[(1 * 8 + j) * 32 + ln] = -cf * q * rstd;
      sc[(2 * 8 + j) * 32 + ln] = cf * (q * rstd * mean - s);
    }
  }
  __syncthreads();
  double bs[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) bs[j] = 0.0;
  if (act) {
    // one row per step: the rows beyond the cache are few once the largest
    // tensors take the three-launch path (U rows in flight here measured
    // slower: the cached rows' shared loads serialise behind them)
    size_t r = r0 + rl;
    int k = 0;
    for (; r < r1; r += R, ++k) {
      const size_t off = (grow0 + r) * p.C8 + (size_t)cc * 8;
      float v[8], gv[8], rr[8];
      if (k < p.kcap) {
        bnf_get(cx + ((size_t)k * nslot + slot) * 2, v);
        if (BWD) bnf_get(cgr + ((size_t)k * nslot + slot) * 2, gv);
      } else {
        load_split8(p.x + off, p.psx, v);
        if (BWD) {
          load_split8(p.g + off, p.psg, gv);
          if (p.mask) apply_mask8(p.mask + off, gv);
        }
      }
      if (!BWD && p.res) load_split8(p.res + off, p.psr, rr);
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        if (!BWD) {
          float o = (float)fma((double)v[j], sc[j * 32 + cl], sc[(8 + j) * 32 + cl]);
          if (p.res) o = __fadd_rn(o, rr[j]);
          if (p.relu) o = o > 0.f ? o : 0.f;
          v[j] = o;
        } else {
          v[j] = (float)fma(sc[j * 32 + cl], (double)gv[j],
                            fma(sc[(8 + j) * 32 + cl], (double)v[j], sc[(16 + j) * 32 + cl]));
          bs[j] += (double)v[j];
        }
      }
      store_split8(p.y + off, p.psy, v);
    }
  }
  if (!BWD || !p.gbias) return;   // uniform

  // ---- phase 4: the producing conv's bias gradient = column sums of gx -----
  {
    double val[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) val[j] = act ? bs[j] : 0.0;
    double* bp = p.bpart + ((size_t)gi * p.spg + slice) * p.C8;
    bnf_block_reduce<8>(red, val, L, R, [&](int ln, int jj, double a) {
      bp[(ct * 32 + ln) * 8 + jj] = a;
    });
  }
  grid.sync();
  const int ns = p.G * p.spg;
  for (int c = gw; c < p.C; c += nw) {
    double s = 0.0;
    for (int k = lane; k < ns; k += 32) s += p.bpart[(size_t)k * p.C8 + c];
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) p.gbias[c] = p.accumulate ? __fadd_rn(p.gbias[c], (float)s) : (float)s;
  }
}

}  // namespace stz
