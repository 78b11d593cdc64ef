// C-ABI for the Stanza B200 hot path (declared in include/stanza_b200.h).
//
// Every entry takes device pointers owned by the caller (PyTorch), sizes,
// an optional caller workspace and a cudaStream_t passed as void*.  Nothing
// here allocates device memory.  Return value: 0 = ok, else an STZ_E* code;
// stz_last_error() holds the message.
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>

#include "stz_gemm.cuh"
#include "../../include/stanza_b200.h"

using namespace stz;

namespace {

thread_local std::string g_err;
int g_impl = 0;  // 0 = tcgen05 BF16x6 (product), 1 = SIMT fp32, 2 = tcgen05 TF32x3
int g_num_sms = 0;
int g_max_kps = 0;  // >0: cap the K range one CTA accumulates (experiments/tests)

enum { STZ_OK = 0, STZ_EINVAL = 1, STZ_ECUDA = 2, STZ_EWORKSPACE = 3 };

int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

unsigned long long g_launches = 0;  // kernels launched through this library

int check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(STZ_ECUDA, "%s: %s", what, cudaGetErrorString(e));
  ++g_launches;
  return STZ_OK;
}

int num_sms() {
  if (g_num_sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
    if (g_num_sms <= 0) g_num_sms = 148;
  }
  return g_num_sms;
}

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }
inline bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

template <class S, int BN, int BK, class VA, class VB>
void launch_tc(const VA& va, const VB& vb, const Epilogue& epi, float* partial, int M, int N,
               int K, int kps, int splits, cudaStream_t st) {
  using Cfg = TcCfg<S, BN, BK>;
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(gemm_tc_kernel<S, BN, BK, VA, VB>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM);
    attr_set = true;
  }
  dim3 grid(cdiv(M, TC_BM), cdiv(N, BN), splits);
  gemm_tc_kernel<S, BN, BK, VA, VB><<<grid, TC_THREADS, Cfg::SMEM, st>>>(va, vb, epi, partial, M,
                                                                           N, K, kps);
}

template <class S, class VA, class VB>
void launch_tc_bn(int BN, const VA& va, const VB& vb, const Epilogue& epi, float* partial, int M,
                  int N, int K, int kps, int splits, cudaStream_t st) {
  if (BN == 32) launch_tc<S, 32, 32>(va, vb, epi, partial, M, N, K, kps, splits, st);
  else if (BN == 64) launch_tc<S, 64, 32>(va, vb, epi, partial, M, N, K, kps, splits, st);
  else if (BN == 128) launch_tc<S, 128, 32>(va, vb, epi, partial, M, N, K, kps, splits, st);
  else launch_tc<S, 256, 16>(va, vb, epi, partial, M, N, K, kps, splits, st);
}

// C[M,N] = A(M,K) . B(K,N) through the views, epilogue applied once.
template <class VA, class VB>
int run_gemm(const char* what, const VA& va, const VB& vb, const Epilogue& epi, int M, int N,
             int K, void* ws, size_t ws_bytes, cudaStream_t st) {
  if (M <= 0 || N <= 0) return STZ_OK;
  if (K <= 0) return fail(STZ_EINVAL, "%s: empty contraction (K=%d)", what, K);
  int BN, BK;
  if (g_impl == 1) {
    BN = 64;
    BK = 16;
  } else {
    BN = N <= 32 ? 32 : N <= 64 ? 64 : N <= 128 ? 128 : 256;
    BK = BN == 256 ? 16 : 32;
  }
  const int tiles = cdiv(M, TC_BM) * cdiv(N, BN);
  const int nkb = cdiv(K, BK);
  const int target = 2 * num_sms();
  int splits = 1;
  if (tiles < target && nkb >= 8) {
    splits = cdiv(target, tiles);
    if (splits > nkb / 4) splits = nkb / 4;
    const size_t per = (size_t)M * N * sizeof(float);
    const size_t fit = ws ? ws_bytes / per : 0;
    if ((size_t)splits > fit) splits = (int)fit;
    if (splits < 2) splits = 1;
  }
  if (g_max_kps > 0 && K > g_max_kps) {
    const size_t per = (size_t)M * N * sizeof(float);
    const int want = cdiv(K, g_max_kps);
    const int fit = ws ? (int)(ws_bytes / per) : 1;
    splits = want < fit ? want : fit;
    if (splits < 1) splits = 1;
  }
  const int kps = cdiv(nkb, splits) * BK;
  splits = cdiv(K, kps);
  float* partial = splits > 1 ? static_cast<float*>(ws) : nullptr;

  if (g_impl == 1) {
    dim3 grid(cdiv(M, 128), cdiv(N, 64), splits);
    gemm_simt_kernel<VA, VB><<<grid, 256, 0, st>>>(va, vb, epi, partial, M, N, K, kps);
  } else if (g_impl == 2) {
    launch_tc_bn<SchemeTF32x3>(BN, va, vb, epi, partial, M, N, K, kps, splits, st);
  } else {
    launch_tc_bn<SchemeBF16x6>(BN, va, vb, epi, partial, M, N, K, kps, splits, st);
  }
  int rc = check_launch(what);
  if (rc) return rc;
  if (splits > 1) {
    const size_t total = (size_t)M * N;
    int blocks = (int)((total + 255) / 256);
    if (blocks > 8 * num_sms()) blocks = 8 * num_sms();
    splitk_reduce_kernel<<<blocks, 256, 0, st>>>(partial, splits, M, N, epi);
    rc = check_launch("splitk_reduce");
  }
  return rc;
}

Epilogue make_epi(float* out, int M, int N, uint32_t mdiv, long long ld_hi, long long ld_lo,
                  long long ld_n, const float* bias, const float* mask, int relu) {
  Epilogue e;
  e.out = out;
  e.M = M;
  e.N = N;
  e.d_m = FastDiv(mdiv);
  e.ld_hi = ld_hi;
  e.ld_lo = ld_lo;
  e.ld_n = ld_n;
  e.bias = bias;
  e.mask = mask;
  e.relu = relu;
  return e;
}

constexpr uint32_t kRowMajor = 1u << 30;  // m / kRowMajor == 0 for every row index

// ---------------------------------------------------------------------------
// elementwise / reduction kernels
// ---------------------------------------------------------------------------

// tensor_core.py:183-198 -- first maximum in kh-major, kw-minor order
__global__ void maxpool_fwd_kernel(const float* __restrict__ x, float* __restrict__ y,
                                   uint8_t* __restrict__ arg, int NC, int H, int W, int k, int s,
                                   int OH, int OW) {
  const size_t total = (size_t)NC * OH * OW;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total;
       i += (size_t)gridDim.x * blockDim.x) {
    const int ow = (int)(i % OW);
    const int oh = (int)((i / OW) % OH);
    const size_t nc = i / ((size_t)OH * OW);
    const float* xp = x + nc * H * W + (size_t)oh * s * W + (size_t)ow * s;
    float best = xp[0];
    int bi = 0;
    for (int kh = 0; kh < k; ++kh)
      for (int kw = 0; kw < k; ++kw) {
        const float v = xp[kh * W + kw];
        if (v > best) {
          best = v;
          bi = kh * k + kw;
        }
      }
    y[i] = best;
    arg[i] = (uint8_t)bi;
  }
}

// tensor_core.py:263-276 as a gather: every input cell sums, in float64 and
// in the reference's (kh, kw) order, the output gradients whose argmax it
// was.  Optional mask fuses the backward of a ReLU that fed the pool.
__global__ void maxpool_bwd_kernel(const float* __restrict__ gy, const uint8_t* __restrict__ arg,
                                   float* __restrict__ gx, const float* __restrict__ mask, int NC,
                                   int H, int W, int k, int s, int OH, int OW) {
  const size_t total = (size_t)NC * H * W;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total;
       i += (size_t)gridDim.x * blockDim.x) {
    const int w = (int)(i % W);
    const int h = (int)((i / W) % H);
    const size_t nc = i / ((size_t)H * W);
    const int th = h - k + 1, tw = w - k + 1;
    const int oh_lo = th <= 0 ? 0 : (th + s - 1) / s;
    const int ow_lo = tw <= 0 ? 0 : (tw + s - 1) / s;
    const int oh_hi = min(OH - 1, h / s), ow_hi = min(OW - 1, w / s);
    double acc = 0.0;
    for (int oh = oh_hi; oh >= oh_lo; --oh) {      // kh = h - oh*s ascending
      for (int ow = ow_hi; ow >= ow_lo; --ow) {    // kw = w - ow*s ascending
        const size_t o = (nc * OH + oh) * OW + ow;
        if (arg[o] == (uint8_t)((h - oh * s) * k + (w - ow * s))) acc += (double)gy[o];
      }
    }
    float v = (float)acc;
    if (mask && !(mask[i] > 0.f)) v = 0.f;
    gx[i] = v;
  }
}

__global__ void relu_fwd_kernel(const float* __restrict__ x, float* __restrict__ y, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x) {
    const float v = x[i];
    y[i] = v < 0.f ? 0.f : v;
  }
}

__global__ void relu_bwd_kernel(const float* __restrict__ gy, const float* __restrict__ src,
                                float* __restrict__ gx, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x)
    gx[i] = src[i] > 0.f ? gy[i] : 0.f;
}

template <int T>
__device__ double block_sum(double v, double* red) {
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
__device__ double block_max(double v, double* red) {
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

// tensor_core.py:216-228 and :295-299 in float64: per-sample loss
// -log softmax[label] and the gradient of the loss SUM, p - onehot.
__global__ void __launch_bounds__(256) softmax_ce_kernel(const float* __restrict__ z,
                                                         const int* __restrict__ labels,
                                                         float* __restrict__ loss,
                                                         float* __restrict__ dz, int C) {
  __shared__ double red[32];
  const int row = blockIdx.x;
  const float* zr = z + (size_t)row * C;
  double mx = -INFINITY;
  for (int j = threadIdx.x; j < C; j += 256) mx = fmax(mx, (double)zr[j]);
  mx = block_max<256>(mx, red);
  double se = 0.0;
  for (int j = threadIdx.x; j < C; j += 256) se += exp((double)zr[j] - mx);
  se = block_sum<256>(se, red);
  const int lab = labels[row];
  float* dr = dz + (size_t)row * C;
  for (int j = threadIdx.x; j < C; j += 256) {
    double p = exp((double)zr[j] - mx) / se;
    if (j == lab) p -= 1.0;
    dr[j] = (float)p;
  }
  if (threadIdx.x == 0) loss[row] = (float)(-log(exp((double)zr[lab] - mx) / se));
}

// deterministic float64 sum of an fp32 vector (one block)
__global__ void __launch_bounds__(1024) sum_f32_kernel(const float* __restrict__ x, size_t n,
                                                       double* __restrict__ out, int accumulate) {
  __shared__ double red[32];
  double s = 0.0;
  for (size_t i = threadIdx.x; i < n; i += 1024) s += (double)x[i];
  s = block_sum<1024>(s, red);
  if (threadIdx.x == 0) *out = accumulate ? *out + s : s;
}

// FC bias gradient, tensor_core.py:288: column sums in float64
__global__ void fc_bias_grad_kernel(const float* __restrict__ g, float* __restrict__ gb, int M,
                                    int N) {
  const int n = blockIdx.x * blockDim.x + threadIdx.x;
  if (n >= N) return;
  double s = 0.0;
  for (int m = 0; m < M; ++m) s += (double)g[(size_t)m * N + n];
  gb[n] = (float)s;
}

// conv bias gradient, tensor_core.py:259: sum over (n, h, w) in float64
__global__ void __launch_bounds__(256) conv_bias_grad_kernel(const float* __restrict__ g,
                                                             float* __restrict__ gb, int N, int O,
                                                             int HW) {
  __shared__ double red[32];
  const int o = blockIdx.x;
  double s = 0.0;
  for (int n = 0; n < N; ++n) {
    const float* p = g + ((size_t)n * O + o) * HW;
    for (int j = threadIdx.x; j < HW; j += 256) s += (double)p[j];
  }
  s = block_sum<256>(s, red);
  if (threadIdx.x == 0) gb[o] = (float)s;
}

// tensor_core.py:366-388, exact fp32 op order and no contraction:
// v = v*mu; v = v + g*inv_n; w = w - lr*v
__device__ __forceinline__ void sgd1(float& w, float& v, float g, float lr, float mu, float inv_n) {
  v = __fadd_rn(__fmul_rn(v, mu), __fmul_rn(g, inv_n));
  w = __fsub_rn(w, __fmul_rn(lr, v));
}

__global__ void sgd_kernel(float* __restrict__ w, float* __restrict__ v,
                           const float* __restrict__ g, size_t n, float lr, float mu,
                           float inv_n) {
  const size_t n4 = n / 4;
  float4* w4 = reinterpret_cast<float4*>(w);
  float4* v4 = reinterpret_cast<float4*>(v);
  const float4* g4 = reinterpret_cast<const float4*>(g);
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4;
       i += (size_t)gridDim.x * blockDim.x) {
    float4 a = w4[i], b = v4[i];
    const float4 c = g4[i];
    sgd1(a.x, b.x, c.x, lr, mu, inv_n);
    sgd1(a.y, b.y, c.y, lr, mu, inv_n);
    sgd1(a.z, b.z, c.z, lr, mu, inv_n);
    sgd1(a.w, b.w, c.w, lr, mu, inv_n);
    w4[i] = a;
    v4[i] = b;
  }
  for (size_t i = n4 * 4 + blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x)
    sgd1(w[i], v[i], g[i], lr, mu, inv_n);
}

// dst += src, fp32 (emulated allreduce of replica gradients, fixed order)
__global__ void vec_add_kernel(float* __restrict__ dst, const float* __restrict__ src, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x)
    dst[i] = __fadd_rn(dst[i], src[i]);
}

int grid_for(size_t n, int threads = 256) {
  size_t b = (n + threads - 1) / threads;
  const size_t cap = (size_t)num_sms() * 16;
  if (b > cap) b = cap;
  return b < 1 ? 1 : (int)b;
}

}  // namespace

// ===========================================================================
// exported C ABI
// ===========================================================================
extern "C" {

int stz_abi_version(void) { return 1; }

const char* stz_last_error(void) { return g_err.c_str(); }

int stz_set_gemm_impl(int impl) {
  if (impl < 0 || impl > 2) return fail(STZ_EINVAL, "gemm impl must be 0, 1 or 2, got %d", impl);
  g_impl = impl;
  return STZ_OK;
}

int stz_get_gemm_impl(void) { return g_impl; }

unsigned long long stz_launch_count(void) { return g_launches; }

int stz_set_max_k_per_split(int k) {
  if (k < 0) return fail(STZ_EINVAL, "max_k_per_split must be >= 0");
  g_max_kps = k;
  return STZ_OK;
}

int stz_conv2d_fwd(const float* x, const float* w, const float* b, float* y, int N, int C, int H,
                   int W, int O, int k, int s, int p, int relu, void* ws, size_t ws_bytes,
                   void* stream) {
  const int OH = (H + 2 * p - k) / s + 1, OW = (W + 2 * p - k) / s + 1;
  if (N < 0 || C <= 0 || O <= 0 || k <= 0 || s <= 0 || p < 0 || OH <= 0 || OW <= 0)
    return fail(STZ_EINVAL, "conv2d_fwd: bad shape N=%d C=%d H=%d W=%d O=%d k=%d s=%d p=%d", N, C,
                H, W, O, k, s, p);
  const int M = N * OH * OW, K = C * k * k;
  ViewIm2col va{x, M, K, C, H, W, OW, s, p, k,
                FastDiv(OH * OW), FastDiv(OW), FastDiv(k * k), FastDiv(k)};
  ViewRowK vb{w, O, K, K, (K % 4 == 0 && aligned16(w)) ? 1 : 0};
  Epilogue e = make_epi(y, M, O, OH * OW, (long long)O * OH * OW, 1, OH * OW, b, nullptr, relu);
  return run_gemm("conv2d_fwd", va, vb, e, M, O, K, ws, ws_bytes, as_stream(stream));
}

int stz_conv2d_bwd_data(const float* gy, const float* w, float* gx, const float* mask, int N,
                        int C, int H, int W, int O, int k, int s, int p, void* ws,
                        size_t ws_bytes, void* stream) {
  const int OH = (H + 2 * p - k) / s + 1, OW = (W + 2 * p - k) / s + 1;
  if (N < 0 || C <= 0 || O <= 0 || k <= 0 || s <= 0 || p < 0 || OH <= 0 || OW <= 0)
    return fail(STZ_EINVAL, "conv2d_bwd_data: bad shape");
  const int M = N * H * W, K = O * k * k;
  ViewDgradG va{gy, M, K, O, OH, OW, s, p, k,
                FastDiv(H * W), FastDiv(W), FastDiv(k * k), FastDiv(k)};
  ViewDgradW vb{w, C, K, k * k, FastDiv(k * k)};
  Epilogue e = make_epi(gx, M, C, H * W, (long long)C * H * W, 1, H * W, nullptr, mask, 0);
  return run_gemm("conv2d_bwd_data", va, vb, e, M, C, K, ws, ws_bytes, as_stream(stream));
}

int stz_conv2d_bwd_filter(const float* x, const float* gy, float* gw, float* gb, int N, int C,
                          int H, int W, int O, int k, int s, int p, void* ws, size_t ws_bytes,
                          void* stream) {
  const int OH = (H + 2 * p - k) / s + 1, OW = (W + 2 * p - k) / s + 1;
  if (N <= 0 || C <= 0 || O <= 0 || k <= 0 || s <= 0 || p < 0 || OH <= 0 || OW <= 0)
    return fail(STZ_EINVAL, "conv2d_bwd_filter: bad shape");
  const int CKK = C * k * k, K = N * OH * OW;
  cudaStream_t st = as_stream(stream);
  ViewWgradX va{x, CKK, K, C, H, W, OW, s, p, k,
                FastDiv(k * k), FastDiv(k), FastDiv(OH * OW), FastDiv(OW)};
  ViewWgradG vb{gy, O, K, OH * OW, FastDiv(OH * OW)};
  // C[ckk, o] stored transposed into gw[o, ckk]
  Epilogue e = make_epi(gw, CKK, O, kRowMajor, 0, 1, CKK, nullptr, nullptr, 0);
  int rc = run_gemm("conv2d_bwd_filter", va, vb, e, CKK, O, K, ws, ws_bytes, st);
  if (rc) return rc;
  if (gb) {
    conv_bias_grad_kernel<<<O, 256, 0, st>>>(gy, gb, N, O, OH * OW);
    rc = check_launch("conv_bias_grad");
  }
  return rc;
}

int stz_fc_fwd(const float* x, const float* w, const float* b, float* y, int M, int in_dim,
               int out_dim, int relu, void* ws, size_t ws_bytes, void* stream) {
  if (M < 0 || in_dim <= 0 || out_dim <= 0) return fail(STZ_EINVAL, "fc_fwd: bad shape");
  ViewRowK va{x, M, in_dim, in_dim, (in_dim % 4 == 0 && aligned16(x)) ? 1 : 0};
  ViewColK vb{w, out_dim, in_dim, out_dim};
  Epilogue e = make_epi(y, M, out_dim, kRowMajor, 0, out_dim, 1, b, nullptr, relu);
  return run_gemm("fc_fwd", va, vb, e, M, out_dim, in_dim, ws, ws_bytes, as_stream(stream));
}

int stz_fc_bwd_data(const float* gy, const float* w, float* gx, const float* mask, int M,
                    int in_dim, int out_dim, void* ws, size_t ws_bytes, void* stream) {
  if (M < 0 || in_dim <= 0 || out_dim <= 0) return fail(STZ_EINVAL, "fc_bwd_data: bad shape");
  ViewRowK va{gy, M, out_dim, out_dim, (out_dim % 4 == 0 && aligned16(gy)) ? 1 : 0};
  ViewRowK vb{w, in_dim, out_dim, out_dim, (out_dim % 4 == 0 && aligned16(w)) ? 1 : 0};
  Epilogue e = make_epi(gx, M, in_dim, kRowMajor, 0, in_dim, 1, nullptr, mask, 0);
  return run_gemm("fc_bwd_data", va, vb, e, M, in_dim, out_dim, ws, ws_bytes,
                  as_stream(stream));
}

int stz_fc_bwd_weight(const float* x, const float* gy, float* gw, float* gb, int M, int in_dim,
                      int out_dim, void* ws, size_t ws_bytes, void* stream) {
  if (M <= 0 || in_dim <= 0 || out_dim <= 0) return fail(STZ_EINVAL, "fc_bwd_weight: bad shape");
  cudaStream_t st = as_stream(stream);
  ViewColK va{x, in_dim, M, in_dim};
  ViewColK vb{gy, out_dim, M, out_dim};
  Epilogue e = make_epi(gw, in_dim, out_dim, kRowMajor, 0, out_dim, 1, nullptr, nullptr, 0);
  int rc = run_gemm("fc_bwd_weight", va, vb, e, in_dim, out_dim, M, ws, ws_bytes, st);
  if (rc) return rc;
  if (gb) {
    fc_bias_grad_kernel<<<cdiv(out_dim, 256), 256, 0, st>>>(gy, gb, M, out_dim);
    rc = check_launch("fc_bias_grad");
  }
  return rc;
}

int stz_maxpool2d_fwd(const float* x, float* y, uint8_t* arg, int N, int C, int H, int W, int k,
                      int s, void* stream) {
  const int OH = (H - k) / s + 1, OW = (W - k) / s + 1;
  if (k <= 0 || s <= 0 || OH <= 0 || OW <= 0 || k * k > 256)
    return fail(STZ_EINVAL, "maxpool2d_fwd: bad shape");
  const size_t total = (size_t)N * C * OH * OW;
  if (total == 0) return STZ_OK;
  maxpool_fwd_kernel<<<grid_for(total), 256, 0, as_stream(stream)>>>(x, y, arg, N * C, H, W, k,
                                                                      s, OH, OW);
  return check_launch("maxpool2d_fwd");
}

int stz_maxpool2d_bwd(const float* gy, const uint8_t* arg, float* gx, const float* mask, int N,
                      int C, int H, int W, int k, int s, void* stream) {
  const int OH = (H - k) / s + 1, OW = (W - k) / s + 1;
  if (k <= 0 || s <= 0 || OH <= 0 || OW <= 0) return fail(STZ_EINVAL, "maxpool2d_bwd: bad shape");
  const size_t total = (size_t)N * C * H * W;
  if (total == 0) return STZ_OK;
  maxpool_bwd_kernel<<<grid_for(total), 256, 0, as_stream(stream)>>>(gy, arg, gx, mask, N * C, H,
                                                                      W, k, s, OH, OW);
  return check_launch("maxpool2d_bwd");
}

int stz_relu_fwd(const float* x, float* y, size_t n, void* stream) {
  if (n == 0) return STZ_OK;
  relu_fwd_kernel<<<grid_for(n), 256, 0, as_stream(stream)>>>(x, y, n);
  return check_launch("relu_fwd");
}

int stz_relu_bwd(const float* gy, const float* src, float* gx, size_t n, void* stream) {
  if (n == 0) return STZ_OK;
  relu_bwd_kernel<<<grid_for(n), 256, 0, as_stream(stream)>>>(gy, src, gx, n);
  return check_launch("relu_bwd");
}

int stz_softmax_ce(const float* logits, const int* labels, float* losses, float* dlogits, int M,
                   int C, void* stream) {
  if (M < 0 || C <= 0) return fail(STZ_EINVAL, "softmax_ce: bad shape");
  if (M == 0) return STZ_OK;
  softmax_ce_kernel<<<M, 256, 0, as_stream(stream)>>>(logits, labels, losses, dlogits, C);
  return check_launch("softmax_ce");
}

int stz_sum_f32(const float* x, size_t n, double* out, int accumulate, void* stream) {
  sum_f32_kernel<<<1, 1024, 0, as_stream(stream)>>>(x, n, out, accumulate);
  return check_launch("sum_f32");
}

int stz_sgd_momentum(float* w, float* v, const float* g, size_t n, float lr, float mu,
                     float inv_n, void* stream) {
  if (n == 0) return STZ_OK;
  if (!aligned16(w) || !aligned16(v) || !aligned16(g))
    return fail(STZ_EINVAL, "sgd_momentum: buffers must be 16-byte aligned");
  sgd_kernel<<<grid_for(n / 4 + 1), 256, 0, as_stream(stream)>>>(w, v, g, n, lr, mu, inv_n);
  return check_launch("sgd_momentum");
}

int stz_vec_add(float* dst, const float* src, size_t n, void* stream) {
  if (n == 0) return STZ_OK;
  vec_add_kernel<<<grid_for(n), 256, 0, as_stream(stream)>>>(dst, src, n);
  return check_launch("vec_add");
}

}  // extern "C"
