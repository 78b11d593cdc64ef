// C-ABI for the Stanza B200 hot path (declared in include/stanza_b200.h).
//
// Two levels:
//   stz_*   reference-layout operator contract (fp32 NCHW / row-major, the
//           layouts of /root/reference/pkg/src/stanza/tensor_core.py); each
//           GEMM op packs its inputs into split planes in the caller
//           workspace and runs the same tcgen05 kernel as the hot path.
//   stzx_*  the fused hot path on split-plane tensors (stz_split.cuh),
//           driven by engine.BlockEngine.
// Every entry takes device pointers owned by the caller (PyTorch), sizes, an
// optional caller workspace and a cudaStream_t passed as void*.  Nothing here
// allocates device memory.  0 = ok, else an STZ_E* code; stz_last_error()
// holds the message.
#include <algorithm>
#include <climits>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "stz_fmt.cuh"
#include "stz_norm.cuh"
#include "stz_tma.cuh"
#include "stz_band.cuh"
#include "stz_bandw.cuh"
#include "stz_peer.cuh"

#include <cuda.h>
#include <mutex>
#include <unordered_map>
#include "../../include/stanza_b200.h"

using namespace stz;

namespace {

thread_local std::string g_err;
int g_num_sms = 0;
int g_max_kps = 0;  // >0: cap the K range one CTA accumulates (tuning knob)
// STZ_TRACE=1: print every TMA GEMM's schedule (shape, tile, pairs, split-K, waves) to stderr
const bool g_trace = [] {
  const char* e = getenv("STZ_TRACE");
  return e && *e == '1';
}();
unsigned long long g_launches = 0;

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
inline int rup8(int v) { return (v + 7) / 8 * 8; }
inline const bf16_t* cb(const void* p) { return reinterpret_cast<const bf16_t*>(p); }
inline bf16_t* mb(void* p) { return reinterpret_cast<bf16_t*>(p); }

int grid_for(size_t n, int threads = 256) {
  size_t b = (n + threads - 1) / threads;
  const size_t cap = (size_t)num_sms() * 16;
  if (b > cap) b = cap;
  return b < 1 ? 1 : (int)b;
}

// bump allocator over the caller workspace (256-byte aligned carving)
struct Carve {
  uint8_t* p;
  size_t left;
  Carve(void* ws, size_t bytes) : p(static_cast<uint8_t*>(ws)), left(ws ? bytes : 0) {}
  template <class T>
  T* take(size_t n) {
    size_t bytes = (n * sizeof(T) + 255) / 256 * 256;
    if (bytes > left) return nullptr;
    T* r = reinterpret_cast<T*>(p);
    p += bytes;
    left -= bytes;
    return r;
  }
};

// ---------------------------------------------------------------------------
// fp32 reference-layout elementwise kernels
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
  // a label outside [0, C) (the reference raises IndexError on it) never
  // indexes memory: the loss is NaN, which the harness reports as NonFinite
  if (threadIdx.x == 0)
    loss[row] = (lab >= 0 && lab < C) ? (float)(-log(exp((double)zr[lab] - mx) / se)) : __int_as_float(0x7fc00000);
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



// ---------------------------------------------------------------------------
// split-plane GEMM dispatch
// ---------------------------------------------------------------------------

template <int BN, int BK, class VA, class VB, class EP>
void launch_sg(const VA& va, const VB& vb, const EP& ep, float* partial, int M, int N, int K,
               int kps, int splits, cudaStream_t st) {
  using Cfg = SgCfg<BN, BK>;
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(sgemm_kernel<BN, BK, VA, VB, EP>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM);
    attr_set = true;
  }
  dim3 grid(cdiv(M, SG_BM), cdiv(N, BN), splits);
  sgemm_kernel<BN, BK, VA, VB, EP><<<grid, SG_THREADS, Cfg::SMEM, st>>>(va, vb, ep, partial, M, N,
                                                                          K, kps);
}

// split-K reduction launcher: the lane-parallel kernel when there are many
// splits, else the one-thread-per-chunk serial walk
template <class EP>
void launch_reduce(const float* partial, int splits, int M, int N, const EP& ep, cudaStream_t st) {
  const size_t total = (size_t)M * (rup8(N) / 8);
  if (splits >= 16) {
    const size_t blocks = (total + 31) / 32;
    const size_t cap = (size_t)num_sms() * 8;
    sgemm_reduce_wide_kernel<EP><<<(int)(blocks < cap ? blocks : cap), 256, 0, st>>>(
        partial, splits, M, N, ep);
  } else {
    sgemm_reduce_kernel<EP><<<grid_for(total), 256, 0, st>>>(partial, splits, M, N, ep);
  }
}

// C[M,N] = A(M,K) . B(K,N) over split-plane views; ep applied once.
template <class VA, class VB, class EP>
int run_sgemm(const char* what, const VA& va, const VB& vb, const EP& ep, int M, int N, int K,
              void* ws, size_t ws_bytes, cudaStream_t st) {
  if (M <= 0 || N <= 0) return STZ_OK;
  if (K <= 0) return fail(STZ_EINVAL, "%s: empty contraction (K=%d)", what, K);
  const int BN = N <= 32 ? 32 : N <= 64 ? 64 : N <= 128 ? 128 : 256;
  const int BK = BN == 256 ? 16 : 32;
  const int tiles = cdiv(M, SG_BM) * cdiv(N, BN);
  const int nkb = cdiv(K, BK);
  const int npad = rup8(N);
  const size_t per = (size_t)M * npad * sizeof(float);
  const int fit = ws ? (int)(ws_bytes / per) : 1;
  int splits = 1;
  if (tiles < 2 * num_sms() && nkb >= 8) {
    splits = cdiv(2 * num_sms(), tiles);
    if (splits > nkb / 4) splits = nkb / 4;
  }
  if (g_max_kps > 0 && K > g_max_kps) splits = cdiv(K, g_max_kps);
  if (splits > fit) splits = fit;
  if (splits < 1) splits = 1;
  const int kps = cdiv(nkb, splits) * BK;
  splits = cdiv(K, kps);
  float* partial = splits > 1 ? static_cast<float*>(ws) : nullptr;
  if (BN == 32) launch_sg<32, 32>(va, vb, ep, partial, M, N, K, kps, splits, st);
  else if (BN == 64) launch_sg<64, 32>(va, vb, ep, partial, M, N, K, kps, splits, st);
  else if (BN == 128) launch_sg<128, 32>(va, vb, ep, partial, M, N, K, kps, splits, st);
  else launch_sg<256, 16>(va, vb, ep, partial, M, N, K, kps, splits, st);
  int rc = check_launch(what);
  if (rc) return rc;
  if (splits > 1) {
    launch_reduce(partial, splits, M, N, ep, st);
    rc = check_launch("sgemm_reduce");
  }
  return rc;
}


// ---------------------------------------------------------------------------
// TMA operands (tensor maps via the driver entry points, cached)
// ---------------------------------------------------------------------------

typedef CUresult (*EncTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                               const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                               const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                               CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
typedef CUresult (*EncIm2colFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                const cuuint64_t*, const cuuint64_t*, const int*, const int*,
                                cuuint32_t, cuuint32_t, const cuuint32_t*, CUtensorMapInterleave,
                                CUtensorMapSwizzle, CUtensorMapL2promotion,
                                CUtensorMapFloatOOBfill);
EncTiledFn g_enc_tiled = nullptr;
EncIm2colFn g_enc_im2col = nullptr;
int g_use_tma = 1;
std::unordered_map<std::string, CUtensorMap> g_map_cache;

bool tma_ready() {
  if (g_enc_tiled && g_enc_im2col) return true;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&g_enc_tiled),
                              cudaEnableDefault, &q) != cudaSuccess ||
      q != cudaDriverEntryPointSuccess)
    g_enc_tiled = nullptr;
  if (cudaGetDriverEntryPoint("cuTensorMapEncodeIm2col", reinterpret_cast<void**>(&g_enc_im2col),
                              cudaEnableDefault, &q) != cudaSuccess ||
      q != cudaDriverEntryPointSuccess)
    g_enc_im2col = nullptr;
  return g_enc_tiled && g_enc_im2col;
}

template <class... T>
std::string cache_key(T... v) {
  std::string k;
  const long long vals[] = {static_cast<long long>(v)...};
  k.assign(reinterpret_cast<const char*>(vals), sizeof(vals));
  return k;
}

bool enc_tiled(CUtensorMap* out, const void* base, uint64_t inner, uint64_t outer,
               uint64_t ld_elems, uint32_t box_inner, uint32_t box_outer, bool swizzle = true) {
  const std::string key = cache_key(0, (uintptr_t)base, inner, outer, ld_elems, box_inner,
                                    box_outer, swizzle ? 1 : 0);
  auto it = g_map_cache.find(key);
  if (it != g_map_cache.end()) {
    *out = it->second;
    return true;
  }
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {ld_elems * 2};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t es[2] = {1, 1};
  CUresult r = g_enc_tiled(out, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims,
                           strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                           swizzle ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_NONE,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return false;
  g_map_cache.emplace(key, *out);
  return true;
}

// the three split planes of a [rows][K] operand (plane stride ps elements) as
// one 3D map {K, rows, plane}: a box {32, R, 3} lands the planes R*64 bytes
// apart, exactly the layout of three {32, R} boxes
bool enc_planes3(CUtensorMap* out, const void* base, uint64_t K, uint64_t rows, uint64_t ld,
                 uint64_t ps, uint32_t R) {
  if ((ps * 2) % 16 || (ld * 2) % 16) return false;
  const std::string key = cache_key(5, (uintptr_t)base, K, rows, ld, ps, R);
  auto it = g_map_cache.find(key);
  if (it != g_map_cache.end()) {
    *out = it->second;
    return true;
  }
  cuuint64_t dims[3] = {K, rows, 3};
  cuuint64_t strides[2] = {ld * 2, ps * 2};
  cuuint32_t box[3] = {32, R, 3};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = g_enc_tiled(out, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims,
                           strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                           CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return false;
  g_map_cache.emplace(key, *out);
  return true;
}

bool enc_im2col(CUtensorMap* out, const void* base, int N, int H, int W, int C8, int s, int lo,
                int hi, int pixels, int chans = 32, int lo_h = INT_MIN, int hi_h = INT_MIN) {
  if (lo_h == INT_MIN) lo_h = lo;
  if (hi_h == INT_MIN) hi_h = hi;
  const std::string key = cache_key(1, (uintptr_t)base, N, H, W, C8, s, lo, hi, pixels, chans,
                                    lo_h, hi_h);
  auto it = g_map_cache.find(key);
  if (it != g_map_cache.end()) {
    *out = it->second;
    return true;
  }
  cuuint64_t dims[4] = {(cuuint64_t)C8, (cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)N};
  cuuint64_t strides[3] = {(cuuint64_t)C8 * 2, (cuuint64_t)W * C8 * 2, (cuuint64_t)H * W * C8 * 2};
  int lower[2] = {lo, lo_h}, upper[2] = {hi, hi_h};   // {W, H}
  cuuint32_t es[4] = {1, (cuuint32_t)s, (cuuint32_t)s, 1};
  CUresult r = g_enc_im2col(out, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(base), dims,
                            strides, lower, upper, (cuuint32_t)chans, (cuuint32_t)pixels, es,
                            CU_TENSOR_MAP_INTERLEAVE_NONE,
                            chans == 64 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B,
                            CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return false;
  g_map_cache.emplace(key, *out);
  return true;
}

// NHWC [N][H][W][C8] planes as a 4D tiled map with box {32, bw, bh, 1} and the
// 64-byte swizzle: the shifted-window conv's band (out-of-range boxes zero-fill)
bool enc_band4d(CUtensorMap* out, const void* base, int N, int H, int W, int C8, int bw, int bh) {
  const std::string key = cache_key(3, (uintptr_t)base, N, H, W, C8, bw, bh);
  auto it = g_map_cache.find(key);
  if (it != g_map_cache.end()) {
    *out = it->second;
    return true;
  }
  cuuint64_t dims[4] = {(cuuint64_t)C8, (cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)N};
  cuuint64_t strides[3] = {(cuuint64_t)C8 * 2, (cuuint64_t)W * C8 * 2, (cuuint64_t)H * W * C8 * 2};
  cuuint32_t box[4] = {32, (cuuint32_t)bw, (cuuint32_t)bh, 1};
  cuuint32_t es[4] = {1, 1, 1, 1};
  CUresult r = g_enc_tiled(out, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(base), dims,
                           strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                           CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return false;
  g_map_cache.emplace(key, *out);
  return true;
}

// [rows][K] planes, K contiguous (row stride ld), tile of R rows
bool op_tiled_k(TgOperand& op, const bf16_t* p, size_t ps, int rows, int K, int ld, int R) {
  op = TgOperand{};
  op.mode = TG_TILED_K;
  op.nbox = 1;
  op.box_rows = R;
  op.box_bytes = R * 64;
  for (int pl = 0; pl < 3; ++pl)
    if (!enc_tiled(&op.map[pl], p + pl * ps, (uint64_t)K, (uint64_t)rows, (uint64_t)ld, 32,
                   (uint32_t)R))
      return false;
  return true;
}

// [K][rows] viewed as 3D {rows % 32, K, rows / 32} (strides ld, 32 elements):
// box {32, 32, groups} = an MN-major tile of 32*groups rows, SW64 atoms
bool enc_mn3d(CUtensorMap* out, const void* base, uint64_t rows, uint64_t K, uint64_t ld,
              uint32_t groups) {
  const std::string key = cache_key(3, (uintptr_t)base, rows, K, ld, groups);
  auto it = g_map_cache.find(key);
  if (it != g_map_cache.end()) {
    *out = it->second;
    return true;
  }
  cuuint64_t dims[3] = {32, K, rows / 32};
  cuuint64_t strides[2] = {ld * 2, 64};
  cuuint32_t box[3] = {32, 32, groups};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = g_enc_tiled(out, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims,
                           strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                           CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return false;
  g_map_cache.emplace(key, *out);
  return true;
}

int g_mn3d = 1;   // stz_set_tma(2): no 3D MN-major boxes, no SW128 im2col boxes (tests compare)

// [K][rows] planes, rows contiguous (row stride ld), tile of R rows (R % 32 == 0).
// rows % 32 == 0: one 3D box per plane per k-block; else R/32 2D boxes
bool op_tiled_mn(TgOperand& op, const bf16_t* p, size_t ps, int rows, int K, int ld, int R) {
  op = TgOperand{};
  op.mode = TG_TILED_MN;
  op.mn3d = g_mn3d && rows % 32 == 0 && R % 32 == 0;
  op.nbox = op.mn3d ? 1 : R / 32;
  op.box_bytes = op.mn3d ? R * 64 : 2048;
  for (int pl = 0; pl < 3; ++pl) {
    const bool ok = op.mn3d ? enc_mn3d(&op.map[pl], p + pl * ps, (uint64_t)rows, (uint64_t)K,
                                       (uint64_t)ld, (uint32_t)(R / 32))
                            : enc_tiled(&op.map[pl], p + pl * ps, (uint64_t)rows, (uint64_t)K,
                                        (uint64_t)ld, 32, 32);
    if (!ok) return false;
  }
  return true;
}

// NHWC [N][H][W][C8] planes read as im2col; output grid OHxOW enumerates the
// window starts (oh*s + lo, ow*s + lo); taps (th, tw) are TMA offsets
bool op_im2col(TgOperand& op, bool mn, const bf16_t* p, size_t ps, int N, int H, int W, int C8,
               int ksz, int s, int lo, int hi, int OH, int OW, int R, int lo_h = INT_MIN,
               int hi_h = INT_MIN) {
  if (lo_h == INT_MIN) lo_h = lo;
  if (hi_h == INT_MIN) hi_h = hi;
  op = TgOperand{};
  op.mode = mn ? TG_IM2COL_MN : TG_IM2COL_K;
  // MN-major (weight-gradient A): 64-channel SW128 boxes when the channels allow
  op.sw128 = mn && g_mn3d && C8 % 64 == 0 && R % 64 == 0;
  op.nbox = mn ? R / (op.sw128 ? 64 : 32) : 1;
  op.box_bytes = op.sw128 ? 4096 : 2048;
  op.lo = lo;
  op.lo_h = lo_h;
  op.s = s;
  op.C8 = C8;
  op.ksz = ksz;
  op.d_ohw = FastDiv(OH * OW);
  op.d_ow = FastDiv(OW);
  op.d_c8 = FastDiv(C8);
  op.d_k = FastDiv(ksz);
  for (int pl = 0; pl < 3; ++pl)
    if (!enc_im2col(&op.map[pl], p + pl * ps, N, H, W, C8, s, lo, hi, mn ? 32 : R,
                    op.sw128 ? 64 : 32, lo_h, hi_h))
      return false;
  return true;
}

// Tile shape.  The split-plane GEMMs are bound by the L2 -> SM operand feed
// (measured with stz_set_debug: skipping the MMAs barely shortens them,
// skipping the loads halves them), so the choice minimises operand bytes per
// MMA cycle: CTA pairs (cta_group::2, 256-row tiles, each CTA stages half of
// B) when there are >= 2 row tiles; width 256 / 192 with one TMEM set when N
// allows, else 128 double-buffered, 64 for thin outputs.
int g_use_cluster = 1;   // CTA pairs (stz_set_cluster)
int g_debug = 0;         // GEMM pipeline diagnostics (stz_set_debug)

struct TgShape {
  int BN, CL, splits;
  double cost;
  int MH = 1;   // 2: two 128-row halves per CTA (thin unpaired tiles)
};
int g_mh_mode = 0;   // stz_set_mh: 0 auto, 1 never, 2 whenever the tile is thin

// Predicted seconds for a TMA GEMM with tile (BN, CL) and `sp` K-splits:
//   waves * (k-blocks per item + per-item overhead) * t_kb + partial sums
// t_kb = max(12 MMAs at max(48, BN/2) cycles, the stage's operand bytes at
// ~27 B/cycle/SM of effective L2 -> SM feed), both measured (tools/mma_bench.cu and the
// stz_set_debug runs); one TMEM set (BN >= 192) serialises the epilogue with
// the next item's mainloop; partial sums are mostly L2-resident.
// MH = 2 halves the A boxes per row (one 256-row box) and fetches B once for
// both halves; TMA cost is per box (tools/tma_bench.cu), credited as 0.8x feed.
double tg_cost(int M, int N, int K, int BN, int CL, int sp, int MH = 1) {
  const double clk = 1.9e9;
  const int sms = num_sms() / CL;
  const int tiles = cdiv(M, TG_BM * CL * MH) * cdiv(N, BN);
  const int nkb = cdiv(K, TG_BK);
  const double mma_cyc = 12.0 * MH * (BN / 2 > 48 ? BN / 2 : 48);
  const double stage_bytes = 3.0 * (TG_BM * MH * TG_BK * 2 + (double)(BN / CL) * TG_BK * 2);
  const double feed_cyc = stage_bytes / 27.0 * (MH == 2 ? 0.8 : 1.0);
  const double t_kb = (mma_cyc > feed_cyc ? mma_cyc : feed_cyc) / clk;
  const double t_epi = BN >= 192 ? 1.0 * t_kb : 0.0;
  const double t_item0 = 4.0 * t_kb + t_epi + 2e-6;
  const double waves = (double)cdiv(tiles * sp, sms);
  double cost = waves * ((double)cdiv(nkb, sp) * t_kb + t_item0);
  if (sp > 1) cost += (double)M * rup8(N) * 4.0 * (2.0 * sp + 1.0) / 10.0e12 + 4e-6;
  return cost;
}

// tile shape + split-K with the lowest predicted time; pairs (cta_group::2)
// only for tiles >= 128 wide (thin tiles are bound by the A-operand smem
// reads, where pairs only add row padding)
int g_force_bn = 0, g_force_cl = 0, g_force_splits = 0;   // stz_set_tile (tests)
constexpr int TG_MAX_KB = 128;   // k-blocks (of 32) one work item may accumulate

// thin unpaired tile -> two 128-row halves per CTA when there are enough
// row tiles to fill the GPU (auto) or always (stz_set_mh(2)); splits re-chosen
template <class BS>
TgShape with_halves(TgShape sh, int M, BS& best_split) {
  if (sh.BN != 64 || sh.CL != 1 || g_mh_mode == 1) return sh;
  if (g_mh_mode == 0 && cdiv(M, 2 * TG_BM) < num_sms() / 2) return sh;
  double bc = 0.0;
  const int sp = best_split(64, 1, bc, 2);
  TgShape h{64, 1, sp, bc};
  h.MH = 2;
  return h;
}

TgShape tg_shape(int M, int N, int K, size_t ws_bytes) {
  const int nkb = cdiv(K, TG_BK);
  // accuracy: tcgen05 truncates the bits it shifts out when adding into an
  // accumulator, so the bias of the big b0*b0 accumulator
  // grows with the MMAs one tile accumulates: cap them at 256 (K <= 4096 per
  // split, worst case 2^-16 relative, typically a fifth of that)
  const int sp_min = cdiv(nkb, TG_MAX_KB);
  const size_t per = (size_t)M * rup8(N) * sizeof(float);
  const int fit = ws_bytes ? (int)(ws_bytes / per) : 1;
  // best split count for one tile shape
  auto best_split = [&](int BN, int CL, double& bc, int MH = 1) {
    const int smax = nkb / 2 < fit ? nkb / 2 : fit;
    int bsp = sp_min;
    bc = tg_cost(M, N, K, BN, CL, sp_min, MH);
    for (int sp = sp_min + 1; sp <= smax && sp <= 256; ++sp) {
      const double cst = tg_cost(M, N, K, BN, CL, sp, MH);
      if (cst < bc * 0.98) {   // more splits only for a real (> 2%) gain
        bc = cst;
        bsp = sp;
      }
    }
    return bsp;
  };
  if (g_force_bn) {
    const int cl = g_force_cl == 2 && cdiv(M, TG_BM) >= 2 ? 2 : 1;
    if (g_force_bn == 256 && cl == 1) {   // 256 wide needs a pair (TMEM)
      double bc = 0.0;
      return TgShape{128, 1, best_split(128, 1, bc), bc};
    }
    double bc = 0.0;
    const int sp = g_force_splits > 0 ? (g_force_splits > sp_min ? g_force_splits : sp_min)
                                      : best_split(g_force_bn, cl, bc);
    TgShape sh{g_force_bn, cl, sp, bc};
    if (g_mh_mode == 2 && sh.BN == 64 && sh.CL == 1) sh.MH = 2;
    return sh;
  }
  TgShape best{64, 1, sp_min, 1e30};
  const int cand[][2] = {{64, 1}, {96, 1}, {128, 1}, {192, 1}, {128, 2}, {192, 2}, {256, 2}};
  for (const auto& c : cand) {
    const int BN = c[0], CL = c[1];
    if (CL == 2 && (!g_use_cluster || cdiv(M, TG_BM) < 2)) continue;
    if (BN > 64 && N <= BN / 2) continue;   // mostly padding
    double bc;
    const int bsp = best_split(BN, CL, bc);
    if (bc < best.cost * 0.97) best = TgShape{BN, CL, bsp, bc};
  }
  return with_halves(best, M, best_split);
}

template <int BN, int NSETS, int CL, class EP, int MH = 1>
void launch_tg(const TgParams<EP>& prm, int splits, cudaStream_t st) {
  using Cfg = TgCfg<BN, NSETS, CL, MH>;
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(tgemm_kernel<BN, NSETS, CL, EP, MH>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM);
    attr_set = true;
  }
  const int items = cdiv(prm.M, TG_BM * CL * MH) * cdiv(prm.N, BN) * splits;
  const int max_ctas = num_sms() / CL * CL;
  const int grid = items * CL < max_ctas ? items * CL : max_ctas;
  if (CL == 1) {
    tgemm_kernel<BN, NSETS, CL, EP, MH><<<grid, TG_THREADS, Cfg::SMEM, st>>>(prm);
    return;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(TG_THREADS);
  cfg.dynamicSmemBytes = Cfg::SMEM;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CL;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, tgemm_kernel<BN, NSETS, CL, EP>, prm);
}

// ---- shifted-window (band) conv: stride-1 "valid" conv over an NHWC input ----------
int g_use_band = 1;     // stz_set_band
int g_band_padded = 0;  // 1: also padded convs (measured slower; tests keep the path covered)
// split-plane GEMM epilogue as 256-bit per-row stores (STZ_EPI_DIRECT=1)
// instead of the shared-memory staged row-contiguous stores
const int g_epi_direct = [] {
  const char* e = getenv("STZ_EPI_DIRECT");
  return e && *e == '1' ? 1 : 0;
}();
// band weights: a stage's three planes as one TMA box (STZ_BAND_B3=0: three)
const int g_band_b3 = [] {
  const char* e = getenv("STZ_BAND_B3");
  return e && *e == '0' ? 0 : 1;
}();
// thin outputs (O <= 64): one 128-row tile per work item with the 4-MMA thin
// schedule (weight planes b0 | b1 as one 128-wide operand, three
// accumulators, two TMEM sets) instead of two tiles on the 6-MMA schedule
// (STZ_BAND_THIN=1)
const int g_band_thin = [] {
  const char* e = getenv("STZ_BAND_THIN");
  return e && *e == '1' ? 1 : 0;
}();
// stacked band as exactly the raster rows a tile reads: 1 always, 0 only when
// whole padded rows do not fit (STZ_BAND_EXACT)
const int g_band_exact = [] {
  const char* e = getenv("STZ_BAND_EXACT");
  return e && *e == '1' ? 1 : 0;
}();

template <int BN, int MT, bool THIN = false, class EP>
int launch_band(BandParams<EP>& prm, int items, size_t smem, cudaStream_t st) {
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(bandconv_kernel<BN, MT, EP, THIN>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    attr_set = true;
  }
  const int grid = items < num_sms() ? items : num_sms();
  bandconv_kernel<BN, MT, EP, THIN><<<grid, BD_THREADS, smem, st>>>(prm);
  return STZ_OK;
}

// The band weight gradient (stz_bandw.cuh): 64 input / output channels,
// stride 1, no padding (the space-to-depth conv1).  Returns -1 when the shape
// or the switches do not allow it (the caller runs the im2col GEMM).
int run_band_wgrad(const bf16_t* x, size_t psx, const bf16_t* g, size_t psg,
                   const EpConvWgradS2D& ep, int N, int Hs, int Ws, int OH, int OW, int C8, int O,
                   int O8, int ks, void* ws, size_t ws_bytes, cudaStream_t st);

struct BandShape {
  int BN, MT, tiles, Hb;
  double junk;   // computed rows / output rows
};

BandShape band_shape(int BN, int MT, int Nimg, int OH, int OW, int Wp, int k) {
  BandShape b;
  b.BN = BN;
  b.MT = MT;
  const int TM = MT * TG_BM;
  b.tiles = cdiv(OH * Wp, TM);
  b.Hb = cdiv(Wp - 1 + TM + (k - 1) * (Wp + 1), Wp);
  b.junk = (double)b.tiles * TM / ((double)OH * OW);
  (void)Nimg;
  return b;
}

// Stride-1 conv of an NHWC split-plane input x [Nimg][H][W][C8] (C8 % 32 == 0),
// zero padding `pad`, with weights w [O][k*k*C8] (K-major split planes):
// out[(n, y, x)][o] for y < OH = H + 2 pad - k + 1, x < OW.  Returns -1 when
// the band path does not apply or would not pay (the caller uses the im2col
// GEMM): too much junk (computed rows outside the output), or too large.
template <class EP>
int run_band_conv(const char* what, const bf16_t* x, size_t psx, const bf16_t* w, size_t psw,
                  const EP& ep, int Nimg, int C8, int H, int W, int O, int k, int pad, void* ws,
                  size_t ws_bytes, cudaStream_t st, int creal = 0) {
  if (!g_use_band || !g_use_tma || !tma_ready() || C8 % 32 != 0 || k < 1 || pad < 0) return -1;
  // padded convs measured slower than the im2col GEMM (per-image tiling adds
  // junk rows and unaligned tap shifts double the A reads): pad 0 only, with
  // the images stacked into one raster
  if (pad != 0 && !g_band_padded) return -1;
  const int OH = H + 2 * pad - k + 1, OW = W + 2 * pad - k + 1, Wp = W + 2 * pad;
  if (OH <= 0 || OW <= 0 || Wp > 256) return -1;
  const bool stacked = pad == 0;
  const int vimg = stacked ? 1 : Nimg;              // images the kernel tiles
  const int vrows = stacked ? Nimg * H : OH;        // tiled rows per image
  BandShape sh;
  if (O <= 64) {
    // thin outputs: two 128-row tiles share each weight tile unless that adds junk
    BandShape s2 = band_shape(64, 2, Nimg, vrows, OW, Wp, k);
    BandShape s1 = band_shape(64, 1, Nimg, vrows, OW, Wp, k);
    if (stacked) {   // junk relative to the real output rows
      s2.junk *= (double)vrows / (Nimg * OH);
      s1.junk *= (double)vrows / (Nimg * OH);
    }
    sh = s2.junk <= s1.junk * 1.05 && !g_band_thin ? s2 : s1;
    if (sh.junk > 1.35) return -1;
  } else {
    sh = band_shape(O % 192 == 0 ? 192 : 128, 1, Nimg, vrows, OW, Wp, k);
    if (stacked) sh.junk *= (double)vrows / (Nimg * OH);
    if (sh.junk > 1.12) return -1;   // wide tiles are near MMA-bound: junk costs directly
  }
  auto smem_of = [&](const BandShape& b, int rows) -> size_t {
    if (b.BN == 64 && b.MT == 1 && g_band_thin) return band_smem<64, 1, true>(rows);
    if (b.BN == 64) return b.MT == 2 ? band_smem<64, 2>(rows) : band_smem<64, 1>(rows);
    if (b.BN == 192) return band_smem<192, 1>(rows);
    return band_smem<128, 1>(rows);
  };
  int rows_alloc = sh.Hb <= 256 ? band_rows_alloc(sh.Hb, Wp) : 1 << 20;
  size_t smem = sh.Hb <= 256 ? smem_of(sh, rows_alloc) : (size_t)1 << 30;
  int exact = 0, brows = 0, nbx = 0;
  if (stacked && (g_band_exact || smem > 227 * 1024)) {
    // the band as exactly the TM + (k-1)(Wp+1) raster rows a tile reads (2D
    // boxes over the stacked pixels): ResNet-50's 115-wide stem rows do not
    // fit as whole rows; fall back to one-tile (MT = 1) bands if needed
    for (int mt = sh.MT; mt >= 1 && !exact; --mt) {
      BandShape b = sh;
      if (mt != sh.MT) {
        b = band_shape(sh.BN, mt, Nimg, vrows, OW, Wp, k);
        b.junk *= (double)vrows / (Nimg * OH);
      }
      const int R = mt * TG_BM + (k - 1) * (Wp + 1);
      const int nb = cdiv(R, 256), br = (cdiv(R, nb) + 7) / 8 * 8;
      const size_t sm = smem_of(b, nb * br);
      if (sm <= 227 * 1024) {
        sh = b;
        exact = 1;
        nbx = nb;
        brows = br;
        rows_alloc = nb * br;
        smem = sm;
      }
    }
  }
  if (!exact && (sh.Hb > 256 || smem > 227 * 1024)) return -1;
  // split-K over channel blocks to keep K per work item <= TG_MAX_KB k-blocks;
  // blocks wholly past the real channels (a space-to-depth input padded to
  // 64) are neither loaded nor multiplied
  const int creal_eff = creal > 0 && creal <= C8 ? creal : C8;
  const int cblocks = cdiv(creal_eff, 32);
  const int kb_per_cb = k * k;
  int cb_per_split = TG_MAX_KB / kb_per_cb;
  if (cb_per_split < 1) cb_per_split = 1;
  if (cb_per_split > cblocks) cb_per_split = cblocks;
  const int splits = cdiv(cblocks, cb_per_split);
  const int M_out = Nimg * OH * OW, npad = rup8(O);
  if (splits > 1 && (!ws || (size_t)splits * M_out * npad * sizeof(float) > ws_bytes)) return -1;
  BandParams<EP> prm;
  for (int pl = 0; pl < 3; ++pl) {
    const bool ok = exact
        ? enc_band4d(&prm.band[pl], x + pl * psx, 1, 1, Nimg * H * W, C8, brows, 1)
        : enc_band4d(&prm.band[pl], x + pl * psx, vimg, stacked ? Nimg * H : H, W, C8, Wp, sh.Hb);
    if (!ok) return -1;
  }
  prm.exact = exact;
  prm.brows = brows;
  prm.nbx = nbx;
  if (!op_tiled_k(prm.b, w, psw, O, k * k * C8, k * k * C8, sh.BN)) return -1;
  prm.use_b3 = g_band_b3 && prm.b.nbox == 1 &&
               enc_planes3(&prm.b3, w, (uint64_t)k * k * C8, (uint64_t)O, (uint64_t)k * k * C8,
                           (uint64_t)psw, (uint32_t)sh.BN);
  prm.ep = ep;
  prm.partial = splits > 1 ? static_cast<float*>(ws) : nullptr;
  prm.N = O;
  prm.C8 = C8;
  prm.creal = creal_eff;
  prm.cblocks = cblocks;
  prm.Nimg = vimg;
  prm.Nreal = Nimg;
  prm.Hs = stacked ? H : (1 << 24);
  prm.d_hs = FastDiv((uint32_t)prm.Hs);
  prm.pad = pad;
  prm.Wp = Wp;
  prm.ksz = k;
  prm.OH = OH;
  prm.OW = OW;
  prm.tiles_per_img = sh.tiles;
  prm.Hb = sh.Hb;
  prm.cb_per_split = cb_per_split;
  prm.splits = splits;
  prm.d_wp = FastDiv((uint32_t)Wp);
  prm.debug = g_debug;
  const int items = vimg * sh.tiles * cdiv(O, sh.BN) * splits;
  if (g_trace)
    fprintf(stderr, "[stz] %-16s band N=%d OHxOW=%dx%d Wp=%d k=%d pad=%d C8=%d O=%d BN=%d MT=%d "
            "tiles/img=%d Hb=%d exact=%d(%dx%d) junk=%.2f splits=%d items=%d smem=%zu\n",
            what, Nimg, OH, OW, Wp, k, pad, C8, O, sh.BN, sh.MT, sh.tiles, sh.Hb, exact, nbx,
            brows, sh.junk, splits, items, smem);
  if (sh.BN == 64 && sh.MT == 2) launch_band<64, 2>(prm, items, smem, st);
  else if (sh.BN == 64 && g_band_thin) launch_band<64, 1, true>(prm, items, smem, st);
  else if (sh.BN == 64) launch_band<64, 1>(prm, items, smem, st);
  else if (sh.BN == 192) launch_band<192, 1>(prm, items, smem, st);
  else launch_band<128, 1>(prm, items, smem, st);
  int rc = check_launch(what);
  if (rc || splits == 1) return rc;
  launch_reduce(prm.partial, splits, M_out, O, ep, st);
  return check_launch("band_reduce");
}

// pixel rows of `ch` channels (64: SWIZZLE_128B, 32: SWIZZLE_64B), one box =
// bw pixels of one raster row
bool enc_sw128_rows(CUtensorMap* out, const void* base, int N, int H, int W, int bw,
                    int ch = 64) {
  const std::string key = cache_key(4, (uintptr_t)base, N, H, W, bw * 1000 + ch);
  auto it = g_map_cache.find(key);
  if (it != g_map_cache.end()) {
    *out = it->second;
    return true;
  }
  const cuuint64_t rb = (cuuint64_t)ch * 2;
  cuuint64_t dims[4] = {(cuuint64_t)ch, (cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)N};
  cuuint64_t strides[3] = {rb, (cuuint64_t)W * rb, (cuuint64_t)H * W * rb};
  cuuint32_t box[4] = {(cuuint32_t)ch, (cuuint32_t)bw, 1, 1};
  cuuint32_t es[4] = {1, 1, 1, 1};
  CUresult r = g_enc_tiled(out, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(base), dims,
                           strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                           ch == 64 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return false;
  g_map_cache.emplace(key, *out);
  return true;
}

int run_band_wgrad(const bf16_t* x, size_t psx, const bf16_t* g, size_t psg,
                   const EpConvWgradS2D& ep, int N, int Hs, int Ws, int OH, int OW, int C8, int O,
                   int O8, int ks, void* ws, size_t ws_bytes, cudaStream_t st) {
  if (!g_use_band || !g_use_tma || !tma_ready() || (C8 != 64 && C8 != 32) || O8 != 64 ||
      O > 64 || ks < 1 || ks > 4)
    return -1;
  const int Wv = (OW + 15) / 16 * 16;
  const int XW = Wv + 2 * ((ks + 1) / 2);
  if (Wv > 256 || XW > 256) return -1;
  const int rows_total = N * OH;
  int splits = 2 * num_sms() / ks;
  if (splits > rows_total) splits = rows_total;
  if (splits < 1) splits = 1;
  const int M = ks * ks * C8;
  if (!ws || (size_t)splits * M * 64 * sizeof(float) > ws_bytes) return -1;
  // as many stages as fit (wide rows fit fewer)
  int nst = BW_STAGES;
  while (nst > 2 && bw_smem(XW, Wv, nst, C8) > 227 * 1024) --nst;
  const size_t smem = bw_smem(XW, Wv, nst, C8);
  if (smem > 227 * 1024) return -1;
  BandWParams prm;
  prm.nst = nst;
  for (int pl = 0; pl < 3; ++pl) {
    if (!enc_sw128_rows(&prm.x[pl], x + pl * psx, N, Hs, Ws, XW, C8)) return -1;
    if (!enc_sw128_rows(&prm.g[pl], g + pl * psg, N, OH, OW, Wv)) return -1;
  }
  prm.partial = static_cast<float*>(ws);
  prm.N = N;
  prm.OH = OH;
  prm.ks = ks;
  prm.Wv = Wv;
  prm.XW = XW;
  prm.splits = splits;
  prm.rows_total = rows_total;
  prm.d_oh = FastDiv((uint32_t)OH);
  prm.debug = g_debug;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(bandwgrad_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         227 * 1024);
    cudaFuncSetAttribute(bandwgrad_kernel<32>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         227 * 1024);
    attr = true;
  }
  const int items = ks * splits;
  const int grid = items < num_sms() ? items : num_sms();
  if (g_trace)
    fprintf(stderr, "[stz] conv_wgrad[bandw] N=%d OHxOW=%dx%d ks=%d Wv=%d XW=%d splits=%d items=%d "
            "stages=%d smem=%zu\n", N, OH, OW, ks, Wv, XW, splits, items, nst, smem);
  if (C8 == 64) bandwgrad_kernel<64><<<grid, BW_THREADS, smem, st>>>(prm);
  else bandwgrad_kernel<32><<<grid, BW_THREADS, smem, st>>>(prm);
  int rc = check_launch("conv_wgrad[bandw]");
  if (rc) return rc;
  launch_reduce(prm.partial, splits, M, O, ep, st);
  return check_launch("bandw_reduce");
}

// Split-K fixup counters: one zeroed region per workspace (split GEMMs that
// may run concurrently never share a workspace -- their partials live in it),
// allocated on the workspace's first split GEMM outside stream capture and
// kept zero by the kernels between launches.  nullptr (-> separate reduce
// pass) when the region would be too small, the workspace is first seen
// while capturing, or stz_set_fixup(0).  Off by default: measured slower than
// the separate reduce pass on the model steps (AlexNet 3.67 vs 3.50 ms,
// ResNet-50 equal): the sums land on each tile's last CTA instead of the
// whole GPU.
int g_fixup = 0;
constexpr int kSemInts = 1 << 15;
int* split_sems(const void* ws, cudaStream_t st, int n) {
  if (n > kSemInts || !ws) return nullptr;
  static std::vector<std::pair<std::pair<int, const void*>, int*>> regions;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return nullptr;
  for (auto& r : regions)
    if (r.first.first == dev && r.first.second == ws) return r.second;
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(st, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone)
    return nullptr;
  int* p = nullptr;
  if (cudaMalloc(&p, kSemInts * sizeof(int)) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  if (cudaMemsetAsync(p, 0, kSemInts * sizeof(int), st) != cudaSuccess) {
    cudaFree(p);
    cudaGetLastError();
    return nullptr;
  }
  regions.push_back({{dev, ws}, p});
  return p;
}

// C[M,N] = A . B with TMA operands built for tile width BN
template <class EP>
int run_tgemm(const char* what, TgShape sh, const TgOperand& a, const TgOperand& b, const EP& ep,
              int M, int N, int K, void* ws, size_t ws_bytes, cudaStream_t st) {
  if (M <= 0 || N <= 0) return STZ_OK;
  const int BN = sh.BN, CL = sh.CL;
  const int tiles = cdiv(M, TG_BM * CL * sh.MH) * cdiv(N, BN);
  const int nkb = cdiv(K, TG_BK);
  const int npad = rup8(N);
  const size_t per = (size_t)M * npad * sizeof(float);
  const int fit = ws ? (int)(ws_bytes / per) : 1;
  int splits = sh.splits;
  const int sms = num_sms() / CL;   // work items run one per CTA pair
  if (g_max_kps > 0 && K > g_max_kps) splits = cdiv(K, g_max_kps);
  if (splits > fit) splits = fit;
  if (splits < 1) splits = 1;
  const int kps = cdiv(nkb, splits) * TG_BK;
  splits = cdiv(K, kps);
  TgParams<EP> prm;
  prm.epi_direct = g_epi_direct;
  prm.a = a;
  prm.b = b;
  prm.ep = ep;
  prm.partial = splits > 1 ? static_cast<float*>(ws) : nullptr;
  // in-kernel fixup only when the sums spread over the GPU: the last split of
  // each tile reads all its partials, so few tiles x many splits (weight
  // gradients: 7 tiles x 31 splits) would serialise on a few SMs
  const bool fix = splits > 1 && splits <= 4 && tiles * CL >= num_sms() && g_fixup;
  prm.sem = fix ? split_sems(ws, st, tiles * CL) : nullptr;
  prm.M = M;
  prm.N = N;
  prm.K = K;
  prm.k_per_split = kps;
  prm.debug = g_debug;
  if (g_trace) {
    const int items = tiles * splits;
    fprintf(stderr,
            "[stz] %-16s M=%6d N=%5d K=%6d BN=%3d CL=%d MH=%d tiles=%5d splits=%3d items=%5d "
            "slots=%3d waves=%.2f est=%.1fus\n",
            what, M, N, K, BN, CL, sh.MH, tiles, splits, items, sms, (double)items / sms,
            sh.cost * 1e6);
  }
  if (sh.MH == 2 && CL == 1 && BN == 64) launch_tg<64, 1, 1, EP, 2>(prm, splits, st);
  else if (sh.MH != 1) return fail(STZ_EINVAL, "%s: no two-half kernel for tile %d x %d", what, BN, CL);
  else if (CL == 2 && BN == 64) launch_tg<64, 2, 2>(prm, splits, st);
  else if (CL == 2 && BN == 128) launch_tg<128, 2, 2>(prm, splits, st);
  else if (CL == 2 && BN == 192) launch_tg<192, 1, 2>(prm, splits, st);
  else if (CL == 2 && BN == 256) launch_tg<256, 1, 2>(prm, splits, st);
  else if (CL == 1 && BN == 64) launch_tg<64, 2, 1>(prm, splits, st);
  else if (CL == 1 && BN == 96) launch_tg<96, 2, 1>(prm, splits, st);
  else if (CL == 1 && BN == 128) launch_tg<128, 2, 1>(prm, splits, st);
  else if (CL == 1 && BN == 192) launch_tg<192, 1, 1>(prm, splits, st);
  else return fail(STZ_EINVAL, "%s: no kernel for tile %d x %d", what, BN, CL);
  int rc = check_launch(what);
  if (rc) return rc;
  if (splits > 1 && !prm.sem) {
    launch_reduce(prm.partial, splits, M, N, ep, st);
    rc = check_launch("tgemm_reduce");
  }
  return rc;
}

bool tma_on() { return g_use_tma && tma_ready(); }

EpF32 ep_f32(float* out, int M, int N, uint32_t mdiv, long long ld_hi, long long ld_lo,
             long long ld_n, const float* bias, const float* mask, int relu) {
  EpF32 e;
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
  e.accumulate = 0;
  return e;
}

constexpr uint32_t kRowMajor = 1u << 30;  // m / kRowMajor == 0 for every row index

// ---- op bodies shared by both ABI levels --------------------------------------------

SvConvFwdA conv_fwd_A(const bf16_t* x, size_t ps, int N, int C8, int H, int W, int k, int s,
                      int p, int OH, int OW) {
  return SvConvFwdA{x, ps, N * OH * OW, k * k * C8, H, W, C8, OW, s, p,
                    FastDiv(OH * OW), FastDiv(OW), FastDiv(C8), FastDiv(k)};
}
SvConvDgradA conv_dgrad_A(const bf16_t* g, size_t ps, int N, int H, int W, int O8, int k, int s,
                          int p, int OH, int OW) {
  return SvConvDgradA{g, ps, N * H * W, k * k * O8, OH, OW, O8, s, p,
                      FastDiv(H * W), FastDiv(W), FastDiv(O8), FastDiv(k)};
}
SvConvWgradA conv_wgrad_A(const bf16_t* x, size_t ps, int N, int C8, int H, int W, int k, int s,
                          int p, int OH, int OW) {
  return SvConvWgradA{x, ps, k * k * C8, N * OH * OW, H, W, C8, OW, s, p,
                      FastDiv(C8), FastDiv(k), FastDiv(OH * OW), FastDiv(OW)};
}


// ---- GEMM-class ops: TMA kernel when the shapes allow, cp.async kernel otherwise ----

// Rectangular kernels (kh x kw, padding (ph, pw): Inception's 1xn / nx1)
// run only on the TMA im2col path -- per-dimension window corners, taps
// (th, tw) = divmod(tap, kw); the band and cp.async producers are square-only.
inline bool square_kp(int kh, int kw, int ph, int pw) { return kh == kw && ph == pw; }

template <class EP>
int gemm_conv_fwd(const bf16_t* x, size_t psx, const bf16_t* wf, size_t psw, const EP& ep, int N,
                  int C8, int H, int W, int O, int kh, int kw, int s, int ph, int pw, int OH,
                  int OW, void* ws, size_t ws_bytes, cudaStream_t st, int creal = 0) {
  const int M = N * OH * OW, K = kh * kw * C8;
  const bool sq = square_kp(kh, kw, ph, pw);
  if (kh == 1 && kw == 1 && s == 1 && ph == 0 && pw == 0 && tma_on() && C8 % 32 == 0) {
    // 1x1 conv = a plain GEMM over the NHWC pixel rows (ResNet bottlenecks):
    // tiled boxes for both operands, no im2col / band addressing
    const TgShape sh = tg_shape(M, O, K, ws_bytes);
    TgOperand a, b;
    if (op_tiled_k(a, x, psx, M, C8, C8, TG_BM * sh.MH) &&
        op_tiled_k(b, wf, psw, O, K, K, sh.BN / sh.CL))
      return run_tgemm("conv_fwd[1x1]", sh, a, b, ep, M, O, K, ws, ws_bytes, st);
  }
  if (s == 1 && sq) {
    const int rc = run_band_conv("conv_fwd[band]", x, psx, wf, psw, ep, N, C8, H, W, O, kh, ph, ws,
                                 ws_bytes, st, creal);
    if (rc >= 0) return rc;
  }
  if (tma_on() && C8 % 32 == 0 && ph - (kh - 1) >= -128 && pw - (kw - 1) >= -128 && ph <= 128 &&
      pw <= 128) {
    const TgShape sh = tg_shape(M, O, K, ws_bytes);
    TgOperand a, b;
    if (op_im2col(a, false, x, psx, N, H, W, C8, kw, s, -pw, pw - (kw - 1), OH, OW,
                  TG_BM * sh.MH, -ph, ph - (kh - 1)) &&
        op_tiled_k(b, wf, psw, O, K, K, sh.BN / sh.CL))
      return run_tgemm("conv_fwd[tma]", sh, a, b, ep, M, O, K, ws, ws_bytes, st);
  }
  if (!sq) return fail(STZ_EINVAL, "conv_fwd: a %dx%d kernel needs the TMA path (C8 %% 32 == 0)",
                       kh, kw);
  SvConvFwdA va = conv_fwd_A(x, psx, N, C8, H, W, kh, s, ph, OH, OW);
  SvRowsK vb{wf, psw, O, K, K};
  return run_sgemm("conv_fwd", va, vb, ep, M, O, K, ws, ws_bytes, st);
}

template <class EP>
int gemm_conv_dgrad(const bf16_t* g, size_t psg, const bf16_t* wd, size_t psw, const EP& ep,
                    int N, int C, int H, int W, int O8, int kh, int kw, int s, int ph, int pw,
                    int OH, int OW, void* ws, size_t ws_bytes, cudaStream_t st) {
  const int M = N * H * W, K = kh * kw * O8;
  const bool sq = square_kp(kh, kw, ph, pw);
  if (kh == 1 && kw == 1 && s == 1 && ph == 0 && pw == 0 && tma_on() && O8 % 32 == 0) {
    const TgShape sh = tg_shape(M, C, K, ws_bytes);   // 1x1: plain GEMM
    TgOperand a, b;
    if (op_tiled_k(a, g, psg, M, O8, O8, TG_BM * sh.MH) &&
        op_tiled_k(b, wd, psw, C, K, K, sh.BN / sh.CL))
      return run_tgemm("conv_dgrad[1x1]", sh, a, b, ep, M, C, K, ws, ws_bytes, st);
  }
  if (s == 1 && sq) {   // the same stride-1 conv over dY padded by k-1-p, flipped weights
    const int rc = run_band_conv("conv_dgrad[band]", g, psg, wd, psw, ep, N, O8, OH, OW, C, kh,
                                 kh - 1 - ph, ws, ws_bytes, st);
    if (rc >= 0) return rc;
  }
  if (tma_on() && O8 % 32 == 0 && s == 1 && ph - (kh - 1) >= -128 && pw - (kw - 1) >= -128 &&
      ph <= 127 && pw <= 127) {
    const TgShape sh = tg_shape(M, C, K, ws_bytes);
    TgOperand a, b;
    if (op_im2col(a, false, g, psg, N, OH, OW, O8, kw, 1, pw - (kw - 1), -pw, H, W,
                  TG_BM * sh.MH, ph - (kh - 1), -ph) &&
        op_tiled_k(b, wd, psw, C, K, K, sh.BN / sh.CL))
      return run_tgemm("conv_dgrad[tma]", sh, a, b, ep, M, C, K, ws, ws_bytes, st);
  }
  if (!sq) return fail(STZ_EINVAL, "conv_dgrad: a %dx%d kernel needs the TMA path (stride 1, "
                       "O8 %% 32 == 0)", kh, kw);
  SvConvDgradA va = conv_dgrad_A(g, psg, N, H, W, O8, kh, s, ph, OH, OW);
  SvRowsK vb{wd, psw, C, K, K};
  return run_sgemm("conv_dgrad", va, vb, ep, M, C, K, ws, ws_bytes, st);
}

template <class EP>
int gemm_conv_wgrad(const bf16_t* x, size_t psx, const bf16_t* g, size_t psg, const EP& ep, int N,
                    int C8, int H, int W, int O, int O8, int kh, int kw, int s, int ph, int pw,
                    int OH, int OW, void* ws, size_t ws_bytes, cudaStream_t st) {
  const int M = kh * kw * C8, P = N * OH * OW;
  if (tma_on() && C8 % 32 == 0 && ph - (kh - 1) >= -128 && pw - (kw - 1) >= -128) {
    const TgShape sh = tg_shape(M, O, P, ws_bytes);
    TgOperand a, b;
    if (op_im2col(a, true, x, psx, N, H, W, C8, kw, s, -pw, pw - (kw - 1), OH, OW,
                  TG_BM * sh.MH, -ph, ph - (kh - 1)) &&
        op_tiled_mn(b, g, psg, O, P, O8, sh.BN / sh.CL))
      return run_tgemm("conv_wgrad[tma]", sh, a, b, ep, M, O, P, ws, ws_bytes, st);
  }
  if (!square_kp(kh, kw, ph, pw))
    return fail(STZ_EINVAL, "conv_wgrad: a %dx%d kernel needs the TMA path (C8 %% 32 == 0)", kh,
                kw);
  SvConvWgradA va = conv_wgrad_A(x, psx, N, C8, H, W, kh, s, ph, OH, OW);
  SvRowsMN vb{g, psg, O, P, O8};
  return run_sgemm("conv_wgrad", va, vb, ep, M, O, P, ws, ws_bytes, st);
}

template <class EP>
int gemm_fc_fwd(const bf16_t* x, size_t psx, const bf16_t* w, size_t psw, const EP& ep, int M,
                int in_dim, int I8, int out_dim, int O8, void* ws, size_t ws_bytes,
                cudaStream_t st) {
  if (tma_on()) {
    const TgShape sh = tg_shape(M, out_dim, I8, ws_bytes);
    TgOperand a, b;
    if (op_tiled_k(a, x, psx, M, I8, I8, TG_BM * sh.MH) && op_tiled_mn(b, w, psw, out_dim, in_dim, O8, sh.BN / sh.CL))
      return run_tgemm("fc_fwd[tma]", sh, a, b, ep, M, out_dim, I8, ws, ws_bytes, st);
  }
  SvRowsK va{x, psx, M, I8, I8};
  SvRowsMN vb{w, psw, out_dim, in_dim, O8};
  return run_sgemm("fc_fwd", va, vb, ep, M, out_dim, I8, ws, ws_bytes, st);
}

template <class EP>
int gemm_fc_dgrad(const bf16_t* g, size_t psg, const bf16_t* w, size_t psw, const EP& ep, int M,
                  int in_dim, int O8, void* ws, size_t ws_bytes, cudaStream_t st) {
  if (tma_on()) {
    const TgShape sh = tg_shape(M, in_dim, O8, ws_bytes);
    TgOperand a, b;
    if (op_tiled_k(a, g, psg, M, O8, O8, TG_BM * sh.MH) && op_tiled_k(b, w, psw, in_dim, O8, O8, sh.BN / sh.CL))
      return run_tgemm("fc_dgrad[tma]", sh, a, b, ep, M, in_dim, O8, ws, ws_bytes, st);
  }
  SvRowsK va{g, psg, M, O8, O8};
  SvRowsK vb{w, psw, in_dim, O8, O8};
  return run_sgemm("fc_dgrad", va, vb, ep, M, in_dim, O8, ws, ws_bytes, st);
}

template <class EP>
int gemm_fc_wgrad(const bf16_t* x, size_t psx, const bf16_t* g, size_t psg, const EP& ep, int M,
                  int in_dim, int I8, int out_dim, int O8, void* ws, size_t ws_bytes,
                  cudaStream_t st) {
  if (tma_on()) {
    const TgShape sh = tg_shape(in_dim, out_dim, M, ws_bytes);
    TgOperand a, b;
    if (op_tiled_mn(a, x, psx, in_dim, M, I8, TG_BM * sh.MH) &&
        op_tiled_mn(b, g, psg, out_dim, M, O8, sh.BN / sh.CL))
      return run_tgemm("fc_wgrad[tma]", sh, a, b, ep, in_dim, out_dim, M, ws, ws_bytes, st);
  }
  SvRowsMN va{x, psx, in_dim, M, I8};
  SvRowsMN vb{g, psg, out_dim, M, O8};
  return run_sgemm("fc_wgrad", va, vb, ep, in_dim, out_dim, M, ws, ws_bytes, st);
}

int colsum_split(const bf16_t* g, size_t ps, int R, int N, int ld, float* out, void* ws,
                 size_t ws_bytes, cudaStream_t st, int accumulate = 0) {
  const int N8 = rup8(N);
  const int chunks = N8 / 8;
  const int lanes = chunks < 256 ? 256 / chunks : 1;
  int rpb = cdiv(R, 2 * num_sms());   // ~2 partial rows per SM: a short final
  rpb = cdiv(rpb < 4 * lanes ? 4 * lanes : rpb, lanes) * lanes;
  const int blocks = cdiv(R, rpb);
  Carve cv(ws, ws_bytes);
  double* part = cv.take<double>((size_t)blocks * N8);
  if (!part) return fail(STZ_EWORKSPACE, "colsum: workspace too small");
  colsum_partial_kernel<<<blocks, 256, 0, st>>>(g, ps, R, N8, ld, rpb, part);
  int rc = check_launch("colsum_partial");
  if (rc) return rc;
  colsum_final_kernel<<<cdiv(N, 8), 256, 0, st>>>(part, blocks, N, N8, out, accumulate);
  return check_launch("colsum_final");
}


// One-launch BatchNorm (stz_norm.cuh bn_fused_kernel): on unless STZ_BN_FUSED=0.
// Returns 1 when the grid cannot be co-resident (caller uses the three-launch
// path), else a status.
int g_bn_fused = -1;
bool bn_fused_on() {
  if (g_bn_fused < 0) {
    const char* e = getenv("STZ_BN_FUSED");
    g_bn_fused = (e && e[0] == '0') ? 0 : 1;
  }
  return g_bn_fused == 1;
}

template <bool BWD>
int bn_fused_launch(BnFusedParams& p, int nch, Carve& cv, bool want_bpart, cudaStream_t st,
                    const char* what) {
  constexpr int kMaxDyn = 200 * 1024;
  const int nops = BWD ? 2 : 1;
  const size_t per_k = (size_t)BNF_THREADS * 32 * nops;   // cache bytes per row step
  static bool attr = false;
  if (!attr) {
    if (cudaFuncSetAttribute(bn_fused_kernel<BWD>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             kMaxDyn) != cudaSuccess)
      return fail(STZ_ECUDA, "%s: smem attribute", what);
    attr = true;
  }
  const int tiles = p.tiles, G = p.G;
  const int r_min = BNF_THREADS / std::min(32, nch);   // row lanes of the widest tile
  int nb = 0, dyn = 0;
  for (int per_sm = 2; per_sm >= 1 && !nb; --per_sm) {
    const long cap = (long)per_sm * num_sms();
    if ((long)G * tiles > cap) continue;
    const long spg = std::max(1L, std::min(cap / ((long)G * tiles), (long)((p.grows + 15) / 16)));
    const int rps = (int)((p.grows + spg - 1) / spg);
    const int kneed = cdiv(rps, r_min);
    const int kcap = (int)std::min<size_t>((size_t)kneed, kMaxDyn / per_k);
    const int d = (int)(kcap * per_k);
    int occ = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, bn_fused_kernel<BWD>, BNF_THREADS, d) !=
        cudaSuccess)
      return fail(STZ_ECUDA, "%s: occupancy", what);
    if (occ < per_sm) continue;
    // the largest tensors (ResNet-50's stem and first stage at K = 32), mostly
    // beyond the cache, stream better through the three-launch path (its
    // passes run at higher occupancy; measured, profiles/r02/bn_fused)
    const double bytes = (double)p.grows * G * p.C8 * 6.0 * nops;
    if (kcap * 2 < kneed && bytes > 128e6) return 1;
    p.spg = (int)spg;
    p.rps = rps;
    p.kcap = kcap;
    nb = G * tiles * (int)spg;
    dyn = d;
  }
  if (!nb) return 1;
  if (!(p.partial = cv.take<double>((size_t)G * p.spg * p.C8 * 2)))
    return fail(STZ_EWORKSPACE, "%s: workspace too small", what);
  if (want_bpart && !(p.bpart = cv.take<double>((size_t)G * p.spg * p.C8)))
    return fail(STZ_EWORKSPACE, "%s: workspace too small", what);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(nb);
  cfg.blockDim = dim3(BNF_THREADS);
  cfg.dynamicSmemBytes = dyn;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeCooperative;
  at[0].val.cooperative = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  const cudaError_t e = cudaLaunchKernelEx(&cfg, bn_fused_kernel<BWD>, p);
  if (e != cudaSuccess) return fail(STZ_ECUDA, "%s: %s", what, cudaGetErrorString(e));
  return check_launch(what);
}
}  // namespace

// ===========================================================================
// exported C ABI
// ===========================================================================
extern "C" {

int stz_abi_version(void) { return 2; }

const char* stz_last_error(void) { return g_err.c_str(); }

unsigned long long stz_launch_count(void) { return g_launches; }

int stz_set_tma(int on) {
  g_use_tma = on ? 1 : 0;
  g_mn3d = on == 1 ? 1 : 0;
  return STZ_OK;
}

int stz_set_mh(int mode) {
  if (mode < 0 || mode > 2) return fail(STZ_EINVAL, "set_mh: mode %d (0 auto, 1 never, 2 always)", mode);
  g_mh_mode = mode;
  return STZ_OK;
}

int stz_set_cluster(int on) {
  g_use_cluster = on ? 1 : 0;
  return STZ_OK;
}

int stz_set_fixup(int on) {
  g_fixup = on ? 1 : 0;
  return STZ_OK;
}

int stz_set_band(int on) {
  g_use_band = on ? 1 : 0;
  g_band_padded = on == 2 ? 1 : 0;
  return STZ_OK;
}

int stz_set_tile(int bn, int cl, int splits) {
  if (bn != 0 && bn != 64 && bn != 96 && bn != 128 && bn != 192 && bn != 256)
    return fail(STZ_EINVAL, "stz_set_tile: width must be 0 (auto), 64, 96, 128, 192 or 256");
  if ((bn == 256 && cl != 2) || (bn == 96 && cl == 2))
    return fail(STZ_EINVAL, "stz_set_tile: widths 64 / 96 run unpaired, 256 only paired");
  g_force_bn = bn;
  g_force_cl = cl;
  g_force_splits = splits;
  return STZ_OK;
}

int stz_set_debug(int flags) {
  g_debug = flags;
  return STZ_OK;
}

int stz_set_max_k_per_split(int k) {
  if (k < 0) return fail(STZ_EINVAL, "max_k_per_split must be >= 0");
  g_max_kps = k;
  return STZ_OK;
}

// ---------------------------------------------------------------------------
// reference-layout operator contract
// ---------------------------------------------------------------------------

int stz_conv2d_fwd(const float* x, const float* w, const float* b, float* y, int N, int C, int H,
                   int W, int O, int k, int s, int p, int relu, void* ws, size_t ws_bytes,
                   void* stream) {
  const int OH = (H + 2 * p - k) / s + 1, OW = (W + 2 * p - k) / s + 1;
  if (N < 0 || C <= 0 || O <= 0 || k <= 0 || s <= 0 || p < 0 || OH <= 0 || OW <= 0)
    return fail(STZ_EINVAL, "conv2d_fwd: bad shape N=%d C=%d H=%d W=%d O=%d k=%d s=%d p=%d", N, C,
                H, W, O, k, s, p);
  if (N == 0) return STZ_OK;
  cudaStream_t st = as_stream(stream);
  const int C8 = rup8(C), kk = k * k;
  Carve cv(ws, ws_bytes);
  const size_t psx = (size_t)N * H * W * C8, psw = (size_t)O * kk * C8;
  bf16_t* xp = cv.take<bf16_t>(3 * psx);
  bf16_t* wf = cv.take<bf16_t>(3 * psw);
  if (!xp || !wf) return fail(STZ_EWORKSPACE, "conv2d_fwd: workspace too small");
  pack_nchw_kernel<<<grid_for((size_t)N * H * W * C8 / 8), 256, 0, st>>>(
      x, xp, psx, N, C, H, W, C8, FastDiv(C8 / 8), FastDiv(H * W));
  int rc = check_launch("pack_nchw");
  if (rc) return rc;
  pack_conv_w_kernel<<<grid_for(psw), 256, 0, st>>>(w, wf, psw, nullptr, 0, O, C, kk, C8, 0, k);
  if ((rc = check_launch("pack_conv_w"))) return rc;
  EpF32 e = ep_f32(y, N * OH * OW, O, OH * OW, (long long)O * OH * OW, 1, OH * OW, b, nullptr,
                   relu);
  return gemm_conv_fwd(xp, psx, wf, psw, e, N, C8, H, W, O, k, k, s, p, p, OH, OW, cv.p, cv.left,
                       st);
}

int stz_conv2d_bwd_data(const float* gy, const float* w, float* gx, const float* mask, int N,
                        int C, int H, int W, int O, int k, int s, int p, void* ws,
                        size_t ws_bytes, void* stream) {
  const int OH = (H + 2 * p - k) / s + 1, OW = (W + 2 * p - k) / s + 1;
  if (N < 0 || C <= 0 || O <= 0 || k <= 0 || s <= 0 || p < 0 || OH <= 0 || OW <= 0)
    return fail(STZ_EINVAL, "conv2d_bwd_data: bad shape");
  if (N == 0) return STZ_OK;
  cudaStream_t st = as_stream(stream);
  const int O8 = rup8(O), kk = k * k;
  Carve cv(ws, ws_bytes);
  const size_t psg = (size_t)N * OH * OW * O8, psw = (size_t)C * kk * O8;
  bf16_t* gp = cv.take<bf16_t>(3 * psg);
  bf16_t* wd = cv.take<bf16_t>(3 * psw);
  if (!gp || !wd) return fail(STZ_EWORKSPACE, "conv2d_bwd_data: workspace too small");
  pack_nchw_kernel<<<grid_for(psg / 8), 256, 0, st>>>(gy, gp, psg, N, O, OH, OW, O8,
                                                      FastDiv(O8 / 8), FastDiv(OH * OW));
  int rc = check_launch("pack_nchw");
  if (rc) return rc;
  pack_conv_w_kernel<<<grid_for(psw), 256, 0, st>>>(w, nullptr, 0, wd, psw, O, C, kk, 0, O8, k);
  if ((rc = check_launch("pack_conv_w"))) return rc;
  EpF32 e = ep_f32(gx, N * H * W, C, H * W, (long long)C * H * W, 1, H * W, nullptr, mask, 0);
  return gemm_conv_dgrad(gp, psg, wd, psw, e, N, C, H, W, O8, k, k, s, p, p, OH, OW, cv.p, cv.left,
                         st);
}

int stz_conv2d_bwd_filter(const float* x, const float* gy, float* gw, float* gb, int N, int C,
                          int H, int W, int O, int k, int s, int p, void* ws, size_t ws_bytes,
                          void* stream) {
  const int OH = (H + 2 * p - k) / s + 1, OW = (W + 2 * p - k) / s + 1;
  if (N <= 0 || C <= 0 || O <= 0 || k <= 0 || s <= 0 || p < 0 || OH <= 0 || OW <= 0)
    return fail(STZ_EINVAL, "conv2d_bwd_filter: bad shape");
  cudaStream_t st = as_stream(stream);
  const int C8 = rup8(C), O8 = rup8(O), kk = k * k;
  Carve cv(ws, ws_bytes);
  const size_t psx = (size_t)N * H * W * C8, psg = (size_t)N * OH * OW * O8;
  bf16_t* xp = cv.take<bf16_t>(3 * psx);
  bf16_t* gp = cv.take<bf16_t>(3 * psg);
  if (!xp || !gp) return fail(STZ_EWORKSPACE, "conv2d_bwd_filter: workspace too small");
  pack_nchw_kernel<<<grid_for(psx / 8), 256, 0, st>>>(x, xp, psx, N, C, H, W, C8,
                                                      FastDiv(C8 / 8), FastDiv(H * W));
  int rc = check_launch("pack_nchw");
  if (rc) return rc;
  pack_nchw_kernel<<<grid_for(psg / 8), 256, 0, st>>>(gy, gp, psg, N, O, OH, OW, O8,
                                                      FastDiv(O8 / 8), FastDiv(OH * OW));
  if ((rc = check_launch("pack_nchw"))) return rc;
  EpConvWgrad e{gw, kk * C8, O, C, kk, FastDiv(C8)};
  rc = gemm_conv_wgrad(xp, psx, gp, psg, e, N, C8, H, W, O, O8, k, k, s, p, p, OH, OW, cv.p,
                       cv.left, st);
  if (rc || !gb) return rc;
  conv_bias_grad_kernel<<<O, 256, 0, st>>>(gy, gb, N, O, OH * OW);
  return check_launch("conv_bias_grad");
}

int stz_fc_fwd(const float* x, const float* w, const float* b, float* y, int M, int in_dim,
               int out_dim, int relu, void* ws, size_t ws_bytes, void* stream) {
  if (M < 0 || in_dim <= 0 || out_dim <= 0) return fail(STZ_EINVAL, "fc_fwd: bad shape");
  if (M == 0) return STZ_OK;
  cudaStream_t st = as_stream(stream);
  const int I8 = rup8(in_dim), O8 = rup8(out_dim);
  Carve cv(ws, ws_bytes);
  const size_t psx = (size_t)M * I8, psw = (size_t)in_dim * O8;
  bf16_t* xp = cv.take<bf16_t>(3 * psx);
  bf16_t* wp = cv.take<bf16_t>(3 * psw);
  if (!xp || !wp) return fail(STZ_EWORKSPACE, "fc_fwd: workspace too small");
  pack_rows_kernel<<<grid_for(psx / 8), 256, 0, st>>>(x, xp, psx, M, in_dim, I8);
  int rc = check_launch("pack_rows");
  if (rc) return rc;
  pack_rows_kernel<<<grid_for(psw / 8), 256, 0, st>>>(w, wp, psw, in_dim, out_dim, O8);
  if ((rc = check_launch("pack_rows"))) return rc;
  EpF32 e = ep_f32(y, M, out_dim, kRowMajor, 0, out_dim, 1, b, nullptr, relu);
  return gemm_fc_fwd(xp, psx, wp, psw, e, M, in_dim, I8, out_dim, O8, cv.p, cv.left, st);
}

int stz_fc_bwd_data(const float* gy, const float* w, float* gx, const float* mask, int M,
                    int in_dim, int out_dim, void* ws, size_t ws_bytes, void* stream) {
  if (M < 0 || in_dim <= 0 || out_dim <= 0) return fail(STZ_EINVAL, "fc_bwd_data: bad shape");
  if (M == 0) return STZ_OK;
  cudaStream_t st = as_stream(stream);
  const int O8 = rup8(out_dim);
  Carve cv(ws, ws_bytes);
  const size_t psg = (size_t)M * O8, psw = (size_t)in_dim * O8;
  bf16_t* gp = cv.take<bf16_t>(3 * psg);
  bf16_t* wp = cv.take<bf16_t>(3 * psw);
  if (!gp || !wp) return fail(STZ_EWORKSPACE, "fc_bwd_data: workspace too small");
  pack_rows_kernel<<<grid_for(psg / 8), 256, 0, st>>>(gy, gp, psg, M, out_dim, O8);
  int rc = check_launch("pack_rows");
  if (rc) return rc;
  pack_rows_kernel<<<grid_for(psw / 8), 256, 0, st>>>(w, wp, psw, in_dim, out_dim, O8);
  if ((rc = check_launch("pack_rows"))) return rc;
  EpF32 e = ep_f32(gx, M, in_dim, kRowMajor, 0, in_dim, 1, nullptr, mask, 0);
  return gemm_fc_dgrad(gp, psg, wp, psw, e, M, in_dim, O8, cv.p, cv.left, st);
}

int stz_fc_bwd_weight(const float* x, const float* gy, float* gw, float* gb, int M, int in_dim,
                      int out_dim, void* ws, size_t ws_bytes, void* stream) {
  if (M <= 0 || in_dim <= 0 || out_dim <= 0) return fail(STZ_EINVAL, "fc_bwd_weight: bad shape");
  cudaStream_t st = as_stream(stream);
  const int I8 = rup8(in_dim), O8 = rup8(out_dim);
  Carve cv(ws, ws_bytes);
  const size_t psx = (size_t)M * I8, psg = (size_t)M * O8;
  bf16_t* xp = cv.take<bf16_t>(3 * psx);
  bf16_t* gp = cv.take<bf16_t>(3 * psg);
  if (!xp || !gp) return fail(STZ_EWORKSPACE, "fc_bwd_weight: workspace too small");
  pack_rows_kernel<<<grid_for(psx / 8), 256, 0, st>>>(x, xp, psx, M, in_dim, I8);
  int rc = check_launch("pack_rows");
  if (rc) return rc;
  pack_rows_kernel<<<grid_for(psg / 8), 256, 0, st>>>(gy, gp, psg, M, out_dim, O8);
  if ((rc = check_launch("pack_rows"))) return rc;
  EpF32 e = ep_f32(gw, in_dim, out_dim, kRowMajor, 0, out_dim, 1, nullptr, nullptr, 0);
  rc = gemm_fc_wgrad(xp, psx, gp, psg, e, M, in_dim, I8, out_dim, O8, cv.p, cv.left, st);
  if (rc || !gb) return rc;
  fc_bias_grad_kernel<<<cdiv(out_dim, 256), 256, 0, st>>>(gy, gb, M, out_dim);
  return check_launch("fc_bias_grad");
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

// ---------------------------------------------------------------------------
// hot path on split-plane tensors (p = plane 0, ps = plane stride in elements)
// ---------------------------------------------------------------------------

int stzx_pack_nchw(const float* x, void* xp, size_t ps, int N, int C, int H, int W, int C8,
                   void* stream) {
  if (C8 % 8 || C8 < C) return fail(STZ_EINVAL, "pack_nchw: C8 must be a multiple of 8 >= C");
  const size_t total = (size_t)N * H * W * C8 / 8;
  if (total == 0) return STZ_OK;
  pack_nchw_kernel<<<grid_for(total), 256, 0, as_stream(stream)>>>(
      x, mb(xp), ps, N, C, H, W, C8, FastDiv(C8 / 8), FastDiv(H * W));
  return check_launch("pack_nchw");
}

int stzx_unpack_nhwc(const void* xp, size_t ps, float* x, int N, int C, int H, int W, int C8,
                     void* stream) {
  const size_t total = (size_t)N * C * H * W;
  if (total == 0) return STZ_OK;
  unpack_nhwc_kernel<<<grid_for(total), 256, 0, as_stream(stream)>>>(cb(xp), ps, x, N, C, H, W,
                                                                      C8);
  return check_launch("unpack_nhwc");
}

int stzx_pack_rows(const float* x, void* xp, size_t ps, int M, int D, int D8, void* stream) {
  if (D8 % 8 || D8 < D) return fail(STZ_EINVAL, "pack_rows: D8 must be a multiple of 8 >= D");
  const size_t total = (size_t)M * D8 / 8;
  if (total == 0) return STZ_OK;
  pack_rows_kernel<<<grid_for(total), 256, 0, as_stream(stream)>>>(x, mb(xp), ps, M, D, D8);
  return check_launch("pack_rows");
}

int stzx_unpack_rows(const void* xp, size_t ps, float* x, int M, int D, int D8, void* stream) {
  const size_t total = (size_t)M * D;
  if (total == 0) return STZ_OK;
  unpack_rows_kernel<<<grid_for(total), 256, 0, as_stream(stream)>>>(cb(xp), ps, x, M, D, D8);
  return check_launch("unpack_rows");
}

int stzx_pack_conv2_w(const float* w, void* wf, size_t psf, void* wd, size_t psd, int O, int C,
                      int kh, int kw, int C8, int O8, void* stream) {
  const size_t kk = (size_t)kh * kw;
  const size_t nf = wf ? (size_t)O * kk * C8 : 0, nd = wd ? (size_t)C * kk * O8 : 0;
  if (nf + nd == 0) return STZ_OK;
  // the kernel walks [nf | nd); a null target contributes an empty range.
  // Flipping both tap axes of [kh][kw] is tap -> kk - 1 - tap.
  pack_conv_w_kernel<<<grid_for(nf + nd), 256, 0, as_stream(stream)>>>(
      w, mb(wf), psf, mb(wd), psd, O, C, (int)kk, wf ? C8 : 0, wd ? O8 : 0, kw);
  return check_launch("pack_conv_w");
}

int stzx_pack_conv_w_multi(const stz_conv_pack* jobs, int n, void* stream) {
  if (n < 0 || n > kMaxConvPack || (n && !jobs))
    return fail(STZ_EINVAL, "pack_conv_w_multi: %d jobs (<= %d)", n, kMaxConvPack);
  ConvPackTable t;
  memset(&t, 0, sizeof(t));
  long tiles = 0;
  for (int i = 0; i < n; ++i) {
    const stz_conv_pack& q = jobs[i];
    const int kk = q.kh * q.kw;
    if (!q.w || !q.wf || q.kh < 1 || q.kw < 1 || kk > kPackSpan / 2 || q.C8 % 8 || q.O8 % 8 ||
        q.C8 < q.C || q.O8 < q.O || q.psf % 2 || (q.wd && q.psd % 2) ||
        (reinterpret_cast<uintptr_t>(q.wf) & 3) || (reinterpret_cast<uintptr_t>(q.wd) & 3))
      return fail(STZ_EINVAL, "pack_conv_w_multi: job %d", i);
    // a multiple of 8 where the span allows (8-element stores), else even
    int cb = std::min(rup8(q.C8), (kPackSpan / kk) & ~7);
    if (cb == 0) cb = std::min(rup8(q.C8), (kPackSpan / kk) & ~1);   // even, >= 2
    const int vec = cb % 8 == 0 && aligned16(q.wf) && (!q.wd || aligned16(q.wd)) &&
                    q.psf % 8 == 0 && (!q.wd || q.psd % 8 == 0);
    const long jt = (long)cdiv(q.O8, 32) * cdiv(q.C8, cb);
    t.j[t.n++] = ConvPackJob{q.w, mb(q.wf), mb(q.wd), q.psf, q.psd, q.O, q.C, kk, q.C8, q.O8, cb,
                             (int)tiles, vec};
    tiles += jt;
  }
  if (tiles >= (1L << 31)) return fail(STZ_EINVAL, "pack_conv_w_multi: %ld tiles", tiles);
  t.tiles = (int)tiles;
  if (tiles == 0) return STZ_OK;
  pack_conv_w_multi_kernel<<<(unsigned)tiles, 256, 0, as_stream(stream)>>>(t);
  return check_launch("pack_conv_w_multi");
}

int stzx_pack_conv_w(const float* w, void* wf, size_t psf, void* wd, size_t psd, int O, int C,
                     int k, int C8, int O8, void* stream) {
  return stzx_pack_conv2_w(w, wf, psf, wd, psd, O, C, k, k, C8, O8, stream);
}

int stzx_conv2_fwd(const void* x, size_t psx, const void* wf, size_t psw, const float* bias,
                   void* y, size_t psy, int N, int C8, int H, int W, int O, int O8, int kh, int kw,
                   int s, int ph, int pw, int relu, void* ws, size_t ws_bytes, void* stream) {
  const int OH = (H + 2 * ph - kh) / s + 1, OW = (W + 2 * pw - kw) / s + 1;
  if (OH <= 0 || OW <= 0 || C8 % 8 || O8 % 8 || O8 < O) return fail(STZ_EINVAL, "conv_fwd: bad shape");
  EpSplit e{mb(y), psy, N * OH * OW, O, O8, bias, nullptr, relu};
  return gemm_conv_fwd(cb(x), psx, cb(wf), psw, e, N, C8, H, W, O, kh, kw, s, ph, pw, OH, OW, ws,
                       ws_bytes, as_stream(stream));
}

int stzx_conv_fwd(const void* x, size_t psx, const void* wf, size_t psw, const float* bias,
                  void* y, size_t psy, int N, int C8, int H, int W, int O, int O8, int k, int s,
                  int p, int relu, void* ws, size_t ws_bytes, void* stream) {
  return stzx_conv2_fwd(x, psx, wf, psw, bias, y, psy, N, C8, H, W, O, O8, k, k, s, p, p, relu, ws,
                        ws_bytes, stream);
}

int stzx_conv_fwd_s2d(const void* x, size_t psx, const void* wf, size_t psw, const float* bias,
                      void* y, size_t psy, int N, int Creal, int Cs8, int Hs, int Ws, int O, int O8,
                      int ks, int relu, void* ws, size_t ws_bytes, void* stream) {
  const int OH = Hs - ks + 1, OW = Ws - ks + 1;
  if (OH <= 0 || OW <= 0 || Cs8 % 8 || O8 % 8 || O8 < O || Creal < 1 || Creal > Cs8)
    return fail(STZ_EINVAL, "conv_fwd_s2d: bad shape");
  EpSplit e{mb(y), psy, N * OH * OW, O, O8, bias, nullptr, relu};
  return gemm_conv_fwd(cb(x), psx, cb(wf), psw, e, N, Cs8, Hs, Ws, O, ks, ks, 1, 0, 0, OH, OW, ws,
                       ws_bytes, as_stream(stream), Creal);
}

namespace {
// Input gradient of a stride-s conv as s*s phase sub-convolutions: input
// pixel (s i + a, s j + b) only receives the taps kh = kh0(a) + s t,
// kw = kw0(b) + s u, from output pixel (i + d_a - t, j + d_b - u).  Each
// phase is a stride-1 conv of dY with an nth x ntw sub-kernel over an
// Ha x Wa grid -- the TMA im2col GEMM, whose B operand reads the phase's
// taps out of the packed (flipped) weights by a tap remap and whose
// epilogue scatters row (n, i, j) to pixel (n, s i + a, s j + b).  Every
// pixel belongs to one phase; phases without taps are zeroed.  Returns -1
// when the geometry does not fit the TMA corners (caller falls back).
int conv_dgrad_phases(const bf16_t* g, size_t psg, const bf16_t* wd, size_t psw, bf16_t* gx,
                      size_t psgx, const bf16_t* mask, int N, int C, int C8, int H, int W, int O8,
                      int kh, int kw, int s, int ph, int pw, int OH, int OW, void* ws,
                      size_t ws_bytes, cudaStream_t st) {
  struct Phase { int a, b, Ha, Wa, nth, ntw, lo_h, lo_w, hi_h, hi_w, base; };
  std::vector<Phase> ph_list;
  bool empty_phase = false;
  for (int a = 0; a < s && a < H; ++a)
    for (int b = 0; b < s && b < W; ++b) {
      Phase q{a, b, (H - a + s - 1) / s, (W - b + s - 1) / s};
      const int kh0 = (a + ph) % s, kw0 = (b + pw) % s;
      q.nth = kh0 < kh ? (kh - kh0 + s - 1) / s : 0;
      q.ntw = kw0 < kw ? (kw - kw0 + s - 1) / s : 0;
      if (!q.nth || !q.ntw) {
        empty_phase = true;
        continue;
      }
      q.lo_h = (a + ph - kh0) / s - (q.nth - 1);
      q.lo_w = (b + pw - kw0) / s - (q.ntw - 1);
      q.hi_h = q.lo_h + q.Ha - OH;
      q.hi_w = q.lo_w + q.Wa - OW;
      for (int v : {q.lo_h, q.lo_w, q.hi_h, q.hi_w})
        if (v < -128 || v > 127) return -1;
      const int fh = (kh - 1) - kh0 - s * (q.nth - 1), fw = (kw - 1) - kw0 - s * (q.ntw - 1);
      q.base = fh * kw + fw;
      ph_list.push_back(q);
    }
  if (empty_phase) {
    const size_t plane = (size_t)N * H * W * C8 * sizeof(bf16_t);
    for (int q = 0; q < 3; ++q)
      if (cudaMemsetAsync(gx + q * psgx, 0, plane, st) != cudaSuccess)
        return fail(STZ_ECUDA, "conv_dgrad: memset");
  }
  for (const Phase& q : ph_list) {
    EpSplit e{gx, psgx, N * q.Ha * q.Wa, C, C8, nullptr, mask, 0};
    e.rs = s;
    e.rH = H;
    e.rW = W;
    e.ro_h = q.a;
    e.ro_w = q.b;
    e.rd_ow = FastDiv(q.Wa);
    e.rd_oh = FastDiv(q.Ha);
    const int M = N * q.Ha * q.Wa, K = q.nth * q.ntw * O8;
    const TgShape sh = tg_shape(M, C, K, ws_bytes);
    TgOperand A, B;
    if (!op_im2col(A, false, g, psg, N, OH, OW, O8, q.ntw, 1, q.lo_w, q.hi_w, q.Ha, q.Wa,
                   TG_BM * sh.MH, q.lo_h, q.hi_h) ||
        !op_tiled_k(B, wd, psw, C, kh * kw * O8, kh * kw * O8, sh.BN / sh.CL))
      return -1;
    B.remap = 1;
    B.r_base = q.base;
    B.r_sh = s * kw;
    B.r_sw = s;
    B.d_ro8 = FastDiv(O8);
    B.d_rtw = FastDiv(q.ntw);
    const int rc = run_tgemm("conv_dgrad[phase]", sh, A, B, e, M, C, K, ws, ws_bytes, st);
    if (rc != STZ_OK) return rc;
  }
  return STZ_OK;
}
}  // namespace

int stzx_conv2_dgrad(const void* g, size_t psg, const void* wd, size_t psw, void* gx, size_t psgx,
                     const void* mask, int N, int C, int C8, int H, int W, int O8, int kh, int kw,
                     int s, int ph, int pw, void* ws, size_t ws_bytes, void* stream) {
  const int OH = (H + 2 * ph - kh) / s + 1, OW = (W + 2 * pw - kw) / s + 1;
  if (OH <= 0 || OW <= 0 || C8 % 8 || O8 % 8) return fail(STZ_EINVAL, "conv_dgrad: bad shape");
  if (kh == 1 && kw == 1 && s > 1 && ph == 0 && pw == 0 && tma_on() && O8 % 32 == 0 &&
      (size_t)N * H * W < (1u << 31)) {
    // 1x1 stride-s (ResNet projection shortcut): input pixel (s*oh, s*ow)
    // receives g[oh, ow] . W and every other pixel 0 -- a plain GEMM over the
    // output rows whose epilogue scatters each row to its input pixel, after
    // zeroing gx
    cudaStream_t st = as_stream(stream);
    const size_t plane = (size_t)N * H * W * C8 * sizeof(bf16_t);
    for (int q = 0; q < 3; ++q)
      if (cudaMemsetAsync(mb(gx) + q * psgx, 0, plane, st) != cudaSuccess)
        return fail(STZ_ECUDA, "conv_dgrad: memset");
    EpSplit e{mb(gx), psgx, N * OH * OW, C, C8, nullptr, cb(mask), 0};
    e.rs = s;
    e.rH = H;
    e.rW = W;
    e.rd_ow = FastDiv(OW);
    e.rd_oh = FastDiv(OH);
    const int M = N * OH * OW;
    const TgShape sh = tg_shape(M, C, O8, ws_bytes);
    TgOperand a, b;
    if (op_tiled_k(a, cb(g), psg, M, O8, O8, TG_BM * sh.MH) &&
        op_tiled_k(b, cb(wd), psw, C, O8, O8, sh.BN / sh.CL))
      return run_tgemm("conv_dgrad[1x1s]", sh, a, b, e, M, C, O8, ws, ws_bytes, st);
  }
  if (s > 1 && (kh > 1 || kw > 1) && tma_on() && O8 % 32 == 0) {
    const int rc = conv_dgrad_phases(cb(g), psg, cb(wd), psw, mb(gx), psgx, cb(mask), N, C, C8, H,
                                     W, O8, kh, kw, s, ph, pw, OH, OW, ws, ws_bytes,
                                     as_stream(stream));
    if (rc >= 0) return rc;
  }
  EpSplit e{mb(gx), psgx, N * H * W, C, C8, nullptr, cb(mask), 0};
  return gemm_conv_dgrad(cb(g), psg, cb(wd), psw, e, N, C, H, W, O8, kh, kw, s, ph, pw, OH, OW,
                         ws, ws_bytes, as_stream(stream));
}

int stzx_conv_dgrad(const void* g, size_t psg, const void* wd, size_t psw, void* gx, size_t psgx,
                    const void* mask, int N, int C, int C8, int H, int W, int O8, int k, int s,
                    int p, void* ws, size_t ws_bytes, void* stream) {
  return stzx_conv2_dgrad(g, psg, wd, psw, gx, psgx, mask, N, C, C8, H, W, O8, k, k, s, p, p, ws,
                          ws_bytes, stream);
}

int stzx_conv2_wgrad(const void* x, size_t psx, const void* g, size_t psg, float* gw, float* gb,
                     int accumulate, int N, int C, int C8, int H, int W, int O, int O8, int kh,
                     int kw, int s, int ph, int pw, void* ws, size_t ws_bytes, void* stream) {
  const int OH = (H + 2 * ph - kh) / s + 1, OW = (W + 2 * pw - kw) / s + 1;
  if (OH <= 0 || OW <= 0 || C8 % 8 || O8 % 8) return fail(STZ_EINVAL, "conv_wgrad: bad shape");
  cudaStream_t st = as_stream(stream);
  EpConvWgrad e{gw, kh * kw * C8, O, C, kh * kw, FastDiv(C8), accumulate ? 1 : 0};
  int rc = gemm_conv_wgrad(cb(x), psx, cb(g), psg, e, N, C8, H, W, O, O8, kh, kw, s, ph, pw, OH,
                           OW, ws, ws_bytes, st);
  if (rc || !gb) return rc;
  return colsum_split(cb(g), psg, N * OH * OW, O, O8, gb, ws, ws_bytes, st, accumulate);
}

int stzx_conv_wgrad(const void* x, size_t psx, const void* g, size_t psg, float* gw, float* gb,
                    int accumulate, int N, int C, int C8, int H, int W, int O, int O8, int k,
                    int s, int p, void* ws, size_t ws_bytes, void* stream) {
  return stzx_conv2_wgrad(x, psx, g, psg, gw, gb, accumulate, N, C, C8, H, W, O, O8, k, k, s, p,
                          p, ws, ws_bytes, stream);
}

int stzx_fc_fwd(const void* x, size_t psx, const void* w, size_t psw, const float* bias, void* y,
                size_t psy, float* y_f32, int M, int in_dim, int in8, int out_dim, int out8,
                int relu, void* ws, size_t ws_bytes, void* stream) {
  if (in8 % 8 || out8 % 8 || in8 < in_dim || out8 < out_dim) return fail(STZ_EINVAL, "fc_fwd: bad shape");
  if (y) {
    EpSplit e{mb(y), psy, M, out_dim, out8, bias, nullptr, relu};
    return gemm_fc_fwd(cb(x), psx, cb(w), psw, e, M, in_dim, in8, out_dim, out8, ws, ws_bytes,
                       as_stream(stream));
  }
  EpF32 e = ep_f32(y_f32, M, out_dim, kRowMajor, 0, out_dim, 1, bias, nullptr, relu);
  return gemm_fc_fwd(cb(x), psx, cb(w), psw, e, M, in_dim, in8, out_dim, out8, ws, ws_bytes,
                     as_stream(stream));
}

int stzx_fc_dgrad(const void* g, size_t psg, const void* w, size_t psw, void* gx, size_t psgx,
                  const void* mask, int M, int in_dim, int in8, int out8, void* ws,
                  size_t ws_bytes, void* stream) {
  if (in8 % 8 || out8 % 8 || in8 < in_dim) return fail(STZ_EINVAL, "fc_dgrad: bad shape");
  EpSplit e{mb(gx), psgx, M, in_dim, in8, nullptr, cb(mask), 0};
  return gemm_fc_dgrad(cb(g), psg, cb(w), psw, e, M, in_dim, out8, ws, ws_bytes,
                       as_stream(stream));
}

int stzx_colsum(const void* g, size_t psg, int R, int N, int ld, float* out, int accumulate,
                void* ws, size_t ws_bytes, void* stream) {
  if (R < 0 || N <= 0 || ld < N || ld % 8 || !out) return fail(STZ_EINVAL, "colsum: bad shape");
  if (R == 0) return STZ_OK;
  return colsum_split(cb(g), psg, R, N, ld, out, ws, ws_bytes, as_stream(stream), accumulate);
}

int stzx_fc_wgrad_sgd(const void* x, size_t psx, const void* g, size_t psg, float* w, float* v,
                      void* planes, size_t psw, float* wb, float* vb, float* gw, float* gb,
                      int accumulate, int M, int in_dim, int in8, int out_dim, int out8, float lr,
                      float mu, float inv_n, void* ws, size_t ws_bytes, void* stream) {
  if (in8 % 8 || out8 % 8 || !w || !v || !planes || (accumulate && !gw) || (wb && (!vb || !gb)))
    return fail(STZ_EINVAL, "fc_wgrad_sgd: bad arguments");
  if (!aligned16(w) || !aligned16(v) || !aligned16(planes) || psw % 8)
    return fail(STZ_EINVAL, "fc_wgrad_sgd: w, v, planes must be 16-byte aligned");
  cudaStream_t st = as_stream(stream);
  EpSgd e{w, v, accumulate ? gw : nullptr, mb(planes), psw, in_dim, out_dim, out8, lr, mu, inv_n};
  int rc = gemm_fc_wgrad(cb(x), psx, cb(g), psg, e, M, in_dim, in8, out_dim, out8, ws, ws_bytes,
                         st);
  if (rc || !wb) return rc;
  // bias: fixed-order column sums of g, then the momentum step on (wb, vb)
  const int N8 = rup8(out_dim), chunks = N8 / 8;
  const int lanes = chunks < 256 ? 256 / chunks : 1;
  int rpb = cdiv(M, 2 * num_sms());
  rpb = cdiv(rpb < 4 * lanes ? 4 * lanes : rpb, lanes) * lanes;
  const int blocks = cdiv(M, rpb);
  Carve cv(ws, ws_bytes);
  double* part = cv.take<double>((size_t)blocks * N8);
  if (!part) return fail(STZ_EWORKSPACE, "fc_wgrad_sgd: workspace too small");
  colsum_partial_kernel<<<blocks, 256, 0, st>>>(cb(g), psg, M, N8, out8, rpb, part);
  if ((rc = check_launch("colsum_partial"))) return rc;
  colsum_sgd_final_kernel<<<cdiv(out_dim, 8), 256, 0, st>>>(part, blocks, out_dim, N8, gb,
                                                            accumulate ? gb : nullptr, wb, vb, lr,
                                                            mu, inv_n);
  return check_launch("colsum_sgd_final");
}

int stzx_fc_wgrad(const void* x, size_t psx, const void* g, size_t psg, float* gw, float* gb,
                  int accumulate, int M, int in_dim, int in8, int out_dim, int out8, void* ws,
                  size_t ws_bytes, void* stream) {
  if (in8 % 8 || out8 % 8) return fail(STZ_EINVAL, "fc_wgrad: bad shape");
  cudaStream_t st = as_stream(stream);
  EpF32 e = ep_f32(gw, in_dim, out_dim, kRowMajor, 0, out_dim, 1, nullptr, nullptr, 0);
  e.accumulate = accumulate ? 1 : 0;
  int rc = gemm_fc_wgrad(cb(x), psx, cb(g), psg, e, M, in_dim, in8, out_dim, out8, ws, ws_bytes,
                         st);
  if (rc || !gb) return rc;
  return colsum_split(cb(g), psg, M, out_dim, out8, gb, ws, ws_bytes, st, accumulate);
}

// row-tiled max-pool backward (maxpool_bwd_tiled_kernel; STZ_POOL_TILED=0:
// untiled) and forward (maxpool_fwd_tiled_kernel, STZ_POOL_FWD_TILED=1:
// measured slower than the untiled forward -- pool2 0.0556 vs 0.0439 ms --
// whose 9 loads per output hit L1, so it stays off)
const int g_pool_tiled = [] {
  const char* e = getenv("STZ_POOL_TILED");
  return e && *e == '0' ? 0 : 1;
}();
const int g_pool_fwd_tiled = [] {
  const char* e = getenv("STZ_POOL_FWD_TILED");
  return e && *e == '1' ? 1 : 0;
}();

int stzx_maxpool_fwd(const void* x, size_t psx, void* y, size_t psy, uint8_t* arg, int N, int C,
                     int C8, int H, int W, int k, int s, int flat_ld, void* stream) {
  const int OH = (H - k) / s + 1, OW = (W - k) / s + 1;
  if (k <= 0 || s <= 0 || OH <= 0 || OW <= 0 || k * k > 256)
    return fail(STZ_EINVAL, "maxpool_fwd: bad shape");
  cudaStream_t st = as_stream(stream);
  const size_t total = (size_t)N * OH * OW * C8 / 8;
  if (total == 0) return STZ_OK;
  const size_t flat_smem = (size_t)C * OH * OW * sizeof(float);
  if (flat_ld > 0 && flat_ld % 8 == 0 && flat_smem <= 200 * 1024) {
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(maxpool_fwd_flat_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           200 * 1024);
      attr = true;
    }
    maxpool_fwd_flat_kernel<<<N, 512, flat_smem, st>>>(cb(x), psx, mb(y), psy, arg, C, C8, H, W,
                                                        k, s, OH, OW, flat_ld);
    return check_launch("maxpool_fwd_flat");
  }
  // row-tiled NHWC form: the input rows of TOH output rows (+ k - s halo)
  // joined once into <= 96 KB of shared memory
  const long in_row = (long)W * C8 * (long)sizeof(float);
  const long tohf = k >= s ? (96L * 1024 / in_row - (k - s)) / s : 0;
  if (flat_ld == 0 && g_pool_fwd_tiled && k >= s && tohf >= 1) {
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(maxpool_fwd_tiled_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           96 * 1024);
      attr = true;
    }
    const int toh = (int)std::min((long)OH, tohf);
    const int tiles = cdiv(OH, toh);
    const size_t sm = (size_t)((toh - 1) * s + k) * (size_t)in_row;
    maxpool_fwd_tiled_kernel<<<N * tiles, 256, sm, st>>>(
        cb(x), psx, mb(y), psy, arg, C, C8, H, W, k, s, OH, OW, toh, FastDiv(C8 / 8),
        FastDiv(W), FastDiv(OW));
    return check_launch("maxpool_fwd_tiled");
  }
  if (flat_ld > C * OH * OW) {
    zero_flat_tail_kernel<<<grid_for((size_t)N * (flat_ld - C * OH * OW)), 256, 0, st>>>(
        mb(y), psy, N, C * OH * OW, flat_ld);
    int rc = check_launch("zero_flat_tail");
    if (rc) return rc;
  }
  maxpool_fwd_split_kernel<<<grid_for(total), 256, 0, st>>>(cb(x), psx, mb(y), psy, arg, N, C, C8,
                                                             H, W, k, s, OH, OW, flat_ld,
                                                             FastDiv(C8 / 8), FastDiv(OW),
                                                             FastDiv(OH));
  return check_launch("maxpool_fwd");
}

int stzx_maxpool_bwd(const void* gy, size_t psg, const uint8_t* arg, void* gx, size_t psx,
                     const void* mask, int N, int C, int C8, int H, int W, int k, int s,
                     int flat_ld, void* stream) {
  const int OH = (H - k) / s + 1, OW = (W - k) / s + 1;
  if (k <= 0 || s <= 0 || OH <= 0 || OW <= 0) return fail(STZ_EINVAL, "maxpool_bwd: bad shape");
  const size_t total = (size_t)N * H * W * C8 / 8;
  if (total == 0) return STZ_OK;
  cudaStream_t st = as_stream(stream);
  const size_t flat_smem = (size_t)C * OH * OW * sizeof(float);
  if (flat_ld > 0 && flat_ld % 8 == 0 && flat_smem <= 200 * 1024) {
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(maxpool_bwd_flat_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           200 * 1024);
      attr = true;
    }
    maxpool_bwd_flat_kernel<<<N, 512, flat_smem, st>>>(cb(gy), psg, arg, mb(gx), psx, cb(mask), C,
                                                        C8, H, W, k, s, OH, OW, flat_ld);
    return check_launch("maxpool_bwd_flat");
  }
  // row-tiled form: each tile's gradient windows joined once into shared
  // memory; TOH output rows per tile, their windows (+ the row above when
  // windows overlap) within 48 KB
  // shared-memory budget per block / block size (STZ_POOL_KB,
  // STZ_POOL_THREADS): 48 KB x 512 threads measured best over 24-160 KB x
  // 128-512 on AlexNet's pool2 + pool5 (0.121 ms against 0.124 at 256
  // threads; profiles/r02/pool_tiled/pool_sweep.log)
  static const int pool_kb = [] {
    const char* e = getenv("STZ_POOL_KB");
    return e ? atoi(e) : 48;
  }();
  static const int pool_thr = [] {
    const char* e = getenv("STZ_POOL_THREADS");
    return e ? atoi(e) : 512;
  }();
  const size_t row_smem = (size_t)OW * C8 * (sizeof(float) + 1);
  const int halo = k > s ? 1 : 0;
  const int toh = std::min(OH, (int)((size_t)pool_kb * 1024 / row_smem) - halo);
  if (flat_ld == 0 && g_pool_tiled && s == 2 && (k == 3 || k == 2) && toh >= 1) {
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(maxpool_bwd_tiled_kernel<3, 2>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
      cudaFuncSetAttribute(maxpool_bwd_tiled_kernel<2, 2>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
      attr = true;
    }
    const int tiles = cdiv(OH, toh);
    const size_t sm = (size_t)(toh + halo) * row_smem;
    if (k == 3)
      maxpool_bwd_tiled_kernel<3, 2><<<N * tiles, pool_thr, sm, st>>>(
          cb(gy), psg, arg, mb(gx), psx, cb(mask), C, C8, H, W, OH, OW, toh, FastDiv(C8 / 8),
          FastDiv(OW), FastDiv(W));
    else
      maxpool_bwd_tiled_kernel<2, 2><<<N * tiles, pool_thr, sm, st>>>(
          cb(gy), psg, arg, mb(gx), psx, cb(mask), C, C8, H, W, OH, OW, toh, FastDiv(C8 / 8),
          FastDiv(OW), FastDiv(W));
    return check_launch("maxpool_bwd_tiled");
  }
  if (flat_ld == 0 && k == 3 && s == 2) {
    maxpool_bwd_nhwc_kernel<3, 2><<<grid_for(total), 256, 0, st>>>(
        cb(gy), psg, arg, mb(gx), psx, cb(mask), N, C, C8, H, W, OH, OW, FastDiv(C8 / 8),
        FastDiv(W), FastDiv(H));
    return check_launch("maxpool_bwd_nhwc");
  }
  if (flat_ld == 0 && k == 2 && s == 2) {
    maxpool_bwd_nhwc_kernel<2, 2><<<grid_for(total), 256, 0, st>>>(
        cb(gy), psg, arg, mb(gx), psx, cb(mask), N, C, C8, H, W, OH, OW, FastDiv(C8 / 8),
        FastDiv(W), FastDiv(H));
    return check_launch("maxpool_bwd_nhwc");
  }
  maxpool_bwd_split_kernel<<<grid_for(total), 256, 0, st>>>(
      cb(gy), psg, arg, mb(gx), psx, cb(mask), N, C, C8, H, W, k, s, OH, OW, flat_ld,
      FastDiv(C8 / 8), FastDiv(W), FastDiv(H));
  return check_launch("maxpool_bwd");
}

int stzx_relu_fwd(const void* x, size_t psx, void* y, size_t psy, size_t n, void* stream) {
  if (n == 0) return STZ_OK;
  relu_fwd_split_kernel<<<grid_for(n), 256, 0, as_stream(stream)>>>(cb(x), psx, mb(y), psy, n);
  return check_launch("relu_fwd_split");
}

int stzx_relu_bwd(const void* gy, size_t psg, const void* src, void* gx, size_t psx, size_t n,
                  void* stream) {
  if (n == 0) return STZ_OK;
  relu_bwd_split_kernel<<<grid_for(n), 256, 0, as_stream(stream)>>>(cb(gy), psg, cb(src), mb(gx),
                                                                     psx, n);
  return check_launch("relu_bwd_split");
}

/* ---- ResNet-trunk kinds (semantics: oracle bn_* / gap_* / residual) ---- */

namespace {
// slices per group for the BatchNorm passes: one wave of resident blocks in
// total (`per_sm` from the kernel's occupancy), at least `min_rows` rows per
// slice (small late-stage layers still fill the GPU)
int resident_per_sm(const void* kernel) {
  int n = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kernel, 256, 0) != cudaSuccess || n < 1) n = 1;
  return n;
}
int bn_slices(size_t grows, int G, int tiles, int per_sm, int min_rows = 64) {
  const long want = std::max(1L, (long)(per_sm * num_sms()) / std::max(1, G * tiles));
  const long cap = std::max(1L, (long)((grows + min_rows - 1) / min_rows));
  return (int)std::min(want, cap);
}

}  // namespace

int stzx_bn_fwd(const void* x, size_t psx, const float* gamma, const float* beta, const void* res,
                size_t psr, void* y, size_t psy, double* stats, int N, int HW, int C, int C8,
                int group, float eps, int relu, void* ws, size_t ws_bytes, void* stream) {
  if (N <= 0 || HW <= 0 || C <= 0 || C8 < C || C8 % 8 || group <= 0 || N % group)
    return fail(STZ_EINVAL, "bn_fwd: bad shape N=%d HW=%d C=%d C8=%d group=%d", N, HW, C, C8, group);
  cudaStream_t st = as_stream(stream);
  const int G = N / group, tiles = cdiv(C8 / 8, 32);
  const size_t grows = (size_t)group * HW;
  static const int occ_r = resident_per_sm((const void*)bn_reduce_kernel<false>), occ_a = resident_per_sm((const void*)bn_apply_kernel);
  const int slices = bn_slices(grows, G, tiles, occ_r);
  const int rps = (int)((grows + slices - 1) / slices);
  const size_t total = (size_t)N * HW * (C8 / 8);
  if (total >= (1ull << 31)) return fail(STZ_EINVAL, "bn_fwd: %zu chunks exceed 2^31", total);
  if (bn_fused_on()) {
    Carve fcv(ws, ws_bytes);
    BnFusedParams fp{};
    fp.x = cb(x); fp.psx = psx; fp.res = cb(res); fp.psr = psr; fp.y = mb(y); fp.psy = psy;
    fp.stats = stats; fp.gamma = gamma; fp.beta = beta;
    fp.m = (double)grows; fp.eps = (double)eps; fp.grows = grows;
    fp.C = C; fp.C8 = C8; fp.G = G; fp.tiles = tiles; fp.relu = relu;
    const int rc = bn_fused_launch<false>(fp, C8 / 8, fcv, false, st, "bn_fwd_fused");
    if (rc != 1) return rc;
  }
  Carve cv(ws, ws_bytes);
  double* part = cv.take<double>((size_t)G * slices * C8 * 2);
  double2* coef = cv.take<double2>((size_t)G * C8);
  if (!part || !coef) return fail(STZ_EWORKSPACE, "bn_fwd: workspace too small");
  bn_reduce_kernel<false><<<dim3(slices, G, tiles), 256, 0, st>>>(cb(x), psx, nullptr, 0, nullptr,
                                                                 part, HW, C8, group, rps);
  bn_stats_final_kernel<<<cdiv(G * C8 * 32, 256), 256, 0, st>>>(part, stats, coef, gamma, beta, G,
                                                          slices, C, C8, (double)grows,
                                                          (double)eps);
  const uint32_t rows = (uint32_t)N * HW;
  const int aslices = std::max(G, bn_slices(rows, 1, tiles, occ_a, 16));   // slice <= group
  const uint32_t arps = (rows + aslices - 1) / aslices;
  bn_apply_kernel<<<dim3(aslices, tiles), 256, 0, st>>>(cb(x), psx, coef, cb(res), psr, mb(y), psy,
                                                        rows, arps, FastDiv((uint32_t)grows), C8,
                                                        relu);
  return check_launch("bn_fwd");
}

int stzx_bn_bwd(const void* g, size_t psg, const void* mask, const void* x, size_t psx,
                const double* stats,
                const float* gamma, float* ggamma, float* gbeta, float* gbias_in, int accumulate,
                void* gx, size_t psgx, int N, int HW, int C, int C8, int group, void* ws,
                size_t ws_bytes, void* stream) {
  if (N <= 0 || HW <= 0 || C <= 0 || C8 < C || C8 % 8 || group <= 0 || N % group)
    return fail(STZ_EINVAL, "bn_bwd: bad shape N=%d HW=%d C=%d C8=%d group=%d", N, HW, C, C8, group);
  if (gbias_in && !gx) return fail(STZ_EINVAL, "bn_bwd: gbias_in needs gx");
  cudaStream_t st = as_stream(stream);
  const int G = N / group, tiles = cdiv(C8 / 8, 32);
  const size_t grows = (size_t)group * HW;
  static const int occ_r = resident_per_sm((const void*)bn_reduce_kernel<true>), occ_a = resident_per_sm((const void*)bn_bwd_apply_kernel);
  const int slices = bn_slices(grows, G, tiles, occ_r);
  const int rps = (int)((grows + slices - 1) / slices);
  const size_t total = (size_t)N * HW * (C8 / 8);
  if (total >= (1ull << 31)) return fail(STZ_EINVAL, "bn_bwd: %zu chunks exceed 2^31", total);
  if (bn_fused_on()) {
    Carve fcv(ws, ws_bytes);
    BnFusedParams fp{};
    fp.x = cb(x); fp.psx = psx; fp.g = cb(g); fp.psg = psg; fp.mask = cb(mask);
    fp.y = mb(gx); fp.psy = psgx;
    fp.stats = const_cast<double*>(stats); fp.gamma = gamma;
    fp.ggamma = ggamma; fp.gbeta = gbeta; fp.gbias = gbias_in;
    fp.m = (double)grows; fp.grows = grows;
    fp.C = C; fp.C8 = C8; fp.G = G; fp.tiles = tiles; fp.accumulate = accumulate;
    const int rc = bn_fused_launch<true>(fp, C8 / 8, fcv, gbias_in != nullptr, st, "bn_bwd_fused");
    if (rc != 1) return rc;
  }
  Carve cv(ws, ws_bytes);
  double* part = cv.take<double>((size_t)G * slices * C8 * 2);
  double4* coef = cv.take<double4>((size_t)G * C8);
  if (!part || !coef) return fail(STZ_EWORKSPACE, "bn_bwd: workspace too small");
  bn_reduce_kernel<true><<<dim3(slices, G, tiles), 256, 0, st>>>(cb(x), psx, cb(g), psg, cb(mask),
                                                                part, HW, C8, group, rps);
  bn_bwd_final_kernel<<<cdiv(C8 * 32, 256), 256, 0, st>>>(part, stats, gamma, coef, ggamma, gbeta, G,
                                                    slices, C, C8, (double)grows, accumulate);
  if (gx) {
    const uint32_t rows = (uint32_t)N * HW;
    const int aslices = std::max(G, bn_slices(rows, 1, tiles, occ_a, 16));   // slice <= group
    const uint32_t arps = (rows + aslices - 1) / aslices;
    double* bpart = nullptr;
    if (gbias_in && !(bpart = cv.take<double>((size_t)aslices * C8)))
      return fail(STZ_EWORKSPACE, "bn_bwd: workspace too small");
    bn_bwd_apply_kernel<<<dim3(aslices, tiles), 256, 0, st>>>(
        cb(g), psg, cb(mask), cb(x), psx, coef, mb(gx), psgx, bpart, rows, arps,
        FastDiv((uint32_t)grows), C8);
    if (bpart)
      colsum_final_kernel<<<cdiv(C, 8), 256, 0, st>>>(bpart, aslices, C, C8, gbias_in,
                                                      accumulate);
  }
  return check_launch("bn_bwd");
}

int stzx_avgpool_fwd(const void* x, size_t psx, void* y, size_t psy, int N, int C8, int H,
                     int W, int k, int s, int p, void* stream) {
  const int OH = (H + 2 * p - k) / s + 1, OW = (W + 2 * p - k) / s + 1;
  if (OH <= 0 || OW <= 0 || C8 % 8 || k < 1 || s < 1 || p < 0 || 2 * p > k)
    return fail(STZ_EINVAL, "avgpool_fwd: k %d s %d p %d on %dx%d", k, s, p, H, W);
  avgpool_fwd_kernel<<<grid_for((size_t)N * OH * OW * (C8 / 8)), 256, 0, as_stream(stream)>>>(
      cb(x), psx, mb(y), psy, N, H, W, C8, OH, OW, k, s, p);
  return check_launch("avgpool_fwd");
}

int stzx_avgpool_bwd(const void* gy, size_t psg, void* gx, size_t psx, int N, int C8, int H, int W,
                     int k, int s, int p, void* stream) {
  const int OH = (H + 2 * p - k) / s + 1, OW = (W + 2 * p - k) / s + 1;
  if (OH <= 0 || OW <= 0 || C8 % 8 || k < 1 || s < 1 || p < 0 || 2 * p > k)
    return fail(STZ_EINVAL, "avgpool_bwd: k %d s %d p %d on %dx%d", k, s, p, H, W);
  avgpool_bwd_kernel<<<grid_for((size_t)N * H * W * (C8 / 8)), 256, 0, as_stream(stream)>>>(
      cb(gy), psg, mb(gx), psx, N, H, W, C8, OH, OW, k, s, p);
  return check_launch("avgpool_bwd");
}

int stzx_copy_channels(const void* src, size_t pss, int src8, int s0, void* dst, size_t psd,
                       int dst8, int d0, size_t rows, int C, const void* mask, int mask8, int m0,
                       void* stream) {
  if (C % 8 || s0 % 8 || d0 % 8 || src8 % 8 || dst8 % 8 || s0 + C > src8 || d0 + C > dst8 ||
      !aligned16(src) || !aligned16(dst) || pss % 8 || psd % 8 ||
      (mask && (mask8 % 8 || m0 % 8 || m0 + C > mask8 || !aligned16(mask))))
    return fail(STZ_EINVAL, "copy_channels: C %d from %d/%d to %d/%d (multiples of 8)", C, s0,
                src8, d0, dst8);
  if (rows == 0 || C == 0) return STZ_OK;
  copy_channels_kernel<<<grid_for(rows * (C / 8)), 256, 0, as_stream(stream)>>>(
      cb(src), pss, src8, s0, mb(dst), psd, dst8, d0, rows, C, cb(mask), mask8, m0);
  return check_launch("copy_channels");
}

int stzx_add_n(const void* const* xs, const size_t* ps, int nin, void* y, size_t psy, size_t n,
               void* stream) {
  if (nin < 2 || nin > 4 || n % 8 || !xs || !ps)
    return fail(STZ_EINVAL, "add_n: %d inputs (2..4), %zu elements (multiple of 8)", nin, n);
  if (n == 0) return STZ_OK;
  add_n_split_kernel<<<grid_for(n / 8), 256, 0, as_stream(stream)>>>(
      cb(xs[0]), cb(xs[1]), cb(nin > 2 ? xs[2] : xs[0]), cb(nin > 3 ? xs[3] : xs[0]), ps[0], ps[1],
      nin > 2 ? ps[2] : 0, nin > 3 ? ps[3] : 0, nin, mb(y), psy, n / 8);
  return check_launch("add_n");
}

int stzx_gap_fwd(const void* x, size_t psx, void* y, size_t psy, int N, int HW, int C8,
                 void* stream) {
  if (N <= 0 || HW <= 0 || C8 <= 0 || C8 % 8) return fail(STZ_EINVAL, "gap_fwd: bad shape");
  gap_fwd_kernel<<<grid_for((size_t)N * (C8 / 8)), 256, 0, as_stream(stream)>>>(cb(x), psx, mb(y),
                                                                               psy, N, HW, C8);
  return check_launch("gap_fwd");
}

int stzx_gap_bwd(const void* gy, size_t psg, void* gx, size_t psx, int N, int HW, int C8,
                 void* stream) {
  if (N <= 0 || HW <= 0 || C8 <= 0 || C8 % 8) return fail(STZ_EINVAL, "gap_bwd: bad shape");
  gap_bwd_kernel<<<grid_for((size_t)N * HW * (C8 / 8)), 256, 0, as_stream(stream)>>>(
      cb(gy), psg, mb(gx), psx, N, HW, C8);
  return check_launch("gap_bwd");
}

int stzx_add(const void* a, size_t psa, const void* b, size_t psb, const void* mask_b, void* y,
             size_t psy, size_t n, void* stream) {
  if (n % 8) return fail(STZ_EINVAL, "add: %zu elements is not a multiple of 8", n);
  if (n == 0) return STZ_OK;
  add_split_kernel<<<grid_for(n / 8), 256, 0, as_stream(stream)>>>(cb(a), psa, cb(b), psb,
                                                                   cb(mask_b), mb(y), psy, n / 8);
  return check_launch("add_split");
}

int stzx_softmax_ce(const float* logits, const int* labels, float* losses, void* dz, size_t psd,
                    int M, int C, int C8, void* stream) {
  if (M <= 0 || C <= 0 || C8 < C) return fail(STZ_EINVAL, "softmax_ce: bad shape");
  softmax_ce_split_kernel<<<M, 256, 0, as_stream(stream)>>>(logits, labels, losses, mb(dz), psd, C,
                                                             C8);
  return check_launch("softmax_ce_split");
}

int stzx_nhwc_to_flat(const void* x, size_t psx, void* y, size_t psy, int N, int C, int H, int W,
                      int C8, int D8, void* stream) {
  nhwc_to_flat_kernel<<<grid_for((size_t)N * D8), 256, 0, as_stream(stream)>>>(
      cb(x), psx, mb(y), psy, N, C, H, W, C8, D8);
  return check_launch("nhwc_to_flat");
}

int stzx_flat_to_nhwc(const void* y, size_t psy, void* x, size_t psx, int N, int C, int H, int W,
                      int C8, int D8, void* stream) {
  flat_to_nhwc_kernel<<<grid_for((size_t)N * H * W * C8), 256, 0, as_stream(stream)>>>(
      cb(y), psy, mb(x), psx, N, C, H, W, C8, D8);
  return check_launch("flat_to_nhwc");
}

// space-to-depth form of a strided first conv (AlexNet conv1)
int stzx_pack_s2d(const float* x, void* xp, size_t ps, int N, int C, int H, int W, int s, int p,
                  int Hs, int Ws, int Cs8, void* stream) {
  if (Cs8 % 8 || Cs8 < C * s * s) return fail(STZ_EINVAL, "pack_s2d: bad channel padding");
  const size_t total = (size_t)N * Hs * Ws * Cs8 / 8;
  if (total == 0) return STZ_OK;
  const size_t rows_smem = (size_t)C * s * s * Ws * sizeof(float);
  if (C == 3 && s == 4 && rows_smem <= 48 * 1024 && Cs8 % 8 == 0) {
    pack_s2d_rows_kernel<3, 4><<<N * Hs, 256, rows_smem, as_stream(stream)>>>(x, mb(xp), ps, H, W,
                                                                              p, Hs, Ws, Cs8);
    return check_launch("pack_s2d_rows");
  }
  pack_s2d_kernel<<<grid_for(total), 256, 0, as_stream(stream)>>>(
      x, mb(xp), ps, N, C, H, W, s, p, Hs, Ws, Cs8, FastDiv(Cs8 / 8), FastDiv(Ws), FastDiv(Hs));
  return check_launch("pack_s2d");
}

int stzx_pack_conv_w_s2d(const float* w, void* wf, size_t ps, int O, int C, int k, int s,
                         int Cs8, void* stream) {
  const int ks = (k + s - 1) / s;
  pack_s2d_w_kernel<<<grid_for((size_t)O * ks * ks * Cs8), 256, 0, as_stream(stream)>>>(
      w, mb(wf), ps, O, C, k, s, ks, Cs8);
  return check_launch("pack_s2d_w");
}

int stzx_conv_wgrad_s2d(const void* x, size_t psx, const void* g, size_t psg, float* gw,
                        float* gb, int accumulate, int N, int C, int Cs8, int Hs, int Ws, int O,
                        int O8, int k, int s, void* ws, size_t ws_bytes, void* stream) {
  const int ks = (k + s - 1) / s;
  const int OH = Hs - ks + 1, OW = Ws - ks + 1;
  if (OH <= 0 || OW <= 0 || Cs8 % 8 || O8 % 8) return fail(STZ_EINVAL, "conv_wgrad_s2d: bad shape");
  cudaStream_t st = as_stream(stream);
  EpConvWgradS2D e{gw, ks * ks * Cs8, O, C, k, s, ks, C * s * s, FastDiv(Cs8),
                   accumulate ? 1 : 0};
  int rc = run_band_wgrad(cb(x), psx, cb(g), psg, e, N, Hs, Ws, OH, OW, Cs8, O, O8, ks, ws,
                          ws_bytes, st);
  if (rc < 0)
    rc = gemm_conv_wgrad(cb(x), psx, cb(g), psg, e, N, Cs8, Hs, Ws, O, O8, ks, ks, 1, 0, 0, OH, OW,
                         ws, ws_bytes, st);
  if (rc || !gb) return rc;
  return colsum_split(cb(g), psg, N * OH * OW, O, O8, gb, ws, ws_bytes, st, accumulate);
}

}  // extern "C"

// ---------------------------------------------------------------------------
// exchange + update over NVLink peer memory (stz_peer.cuh)
// ---------------------------------------------------------------------------

namespace {
using AddrRangeFn = CUresult (*)(CUdeviceptr*, size_t*, CUdeviceptr);
AddrRangeFn g_addr_range = nullptr;
unsigned long long g_peer_timeout_ns = 60ull * 1000000000ull;

int fill_peers(PeerTable& t, const float* const* grads, float* const* red,
               unsigned* const* flags, int nranks, int me) {
  if (nranks < 1 || nranks > kMaxPeers || me < 0 || me >= nranks)
    return fail(STZ_EINVAL, "peer group: %d members, me=%d (1..%d members)", nranks, me,
                kMaxPeers);
  memset(&t, 0, sizeof(t));
  t.R = nranks;
  t.me = me;
  for (int j = 0; j < nranks; ++j) {
    if (grads) t.g[j] = grads[j];
    if (red) t.red[j] = red[j];
    if (flags) t.flags[j] = flags[j];
    if ((grads && !aligned16(t.g[j])) ||
        (red && (reinterpret_cast<uintptr_t>(t.red[j]) & 31)))
      return fail(STZ_EINVAL, "peer group: member %d gradient must be 16-byte aligned, reduced "
                  "buffer 32-byte aligned (256-bit stores)", j);
  }
  return STZ_OK;
}

int fill_ranges(PackTable& tab, size_t n, const stz_plane_range* ranges, int nranges) {
  memset(&tab, 0, sizeof(tab));
  size_t at = 0;
  auto add_plain = [&](size_t upto) {
    if (upto > at) {
      if (tab.n == kMaxPackRanges) return false;
      tab.r[tab.n++] = PackRange{at, upto - at, nullptr, 0, 1, 1};
      at = upto;
    }
    return true;
  };
  for (int i = 0; i < nranges; ++i) {
    const stz_plane_range& r = ranges[i];
    if (!r.planes && r.D == 0) {   // skip: updated in its weight-gradient epilogue
      if (r.off < at || r.off + r.len > n || !add_plain(r.off) || tab.n == kMaxPackRanges)
        return fail(STZ_EINVAL, "sgd pack skip range %d: off %zu len %zu", i, r.off, r.len);
      tab.r[tab.n++] = PackRange{r.off, r.len, nullptr, 0, 0, 0};
      at = r.off + r.len;
      continue;
    }
    if (r.off < at || r.off + r.len > n || r.off % 4 || !r.planes || r.D < 1 || r.D8 < r.D ||
        r.len % (size_t)r.D || r.ps % 4 || !aligned16(r.planes))
      return fail(STZ_EINVAL, "sgd pack range %d: off %zu len %zu D %d D8 %d (sorted, "
                  "disjoint, 16-byte aligned, whole rows)", i, r.off, r.len, r.D, r.D8);
    if (!add_plain(r.off) || tab.n == kMaxPackRanges)
      return fail(STZ_EINVAL, "sgd pack: more than %d ranges", kMaxPackRanges);
    tab.r[tab.n++] = PackRange{r.off, r.len, mb(r.planes), r.ps, r.D, r.D8};
    at = r.off + r.len;
  }
  if (!add_plain(n)) return fail(STZ_EINVAL, "sgd pack: more than %d ranges", kMaxPackRanges);
  return STZ_OK;
}

int launch_reduce_push(const PeerTable& t, size_t n, cudaStream_t st) {
  // chunk r of member r: 256-byte aligned, the last one ragged
  const size_t per = ((n + t.R - 1) / t.R + 63) / 64 * 64;
  const size_t c0 = std::min(n, per * t.me), c1 = std::min(n, c0 + per);
  const int grid = grid_for((c1 - c0) / 16 + 1);
  switch (t.R) {
#define STZ_RP(R) \
  case R: peer_reduce_push_kernel<R><<<grid, 256, 0, st>>>(t, c0, c1); break;
    STZ_RP(1) STZ_RP(2) STZ_RP(3) STZ_RP(4) STZ_RP(5) STZ_RP(6) STZ_RP(7) STZ_RP(8)
#undef STZ_RP
    default: return fail(STZ_EINVAL, "reduce_push: %d members", t.R);
  }
  return check_launch("peer_reduce_push");
}
}  // namespace

extern "C" {

int stz_ipc_handle(const void* dptr, void* handle, size_t* offset) {
  if (!dptr || !handle || !offset) return fail(STZ_EINVAL, "ipc_handle: null argument");
  if (!g_addr_range) {
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", reinterpret_cast<void**>(&g_addr_range),
                                cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess) {
      g_addr_range = nullptr;
      return fail(STZ_ECUDA, "ipc_handle: cuMemGetAddressRange unavailable");
    }
  }
  CUdeviceptr base = 0;
  size_t size = 0;
  if (g_addr_range(&base, &size, reinterpret_cast<CUdeviceptr>(dptr)) != CUDA_SUCCESS)
    return fail(STZ_ECUDA, "ipc_handle: %p is not device memory", dptr);
  cudaIpcMemHandle_t h;
  cudaError_t e = cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base));
  if (e != cudaSuccess) return fail(STZ_ECUDA, "ipc_handle: %s", cudaGetErrorString(e));
  static_assert(sizeof(h) == STZ_IPC_HANDLE_BYTES, "IPC handle size");
  memcpy(handle, &h, sizeof(h));
  *offset = reinterpret_cast<uintptr_t>(dptr) - (uintptr_t)base;
  return STZ_OK;
}

int stz_ipc_open(const void* handle, void** base) {
  if (!handle || !base) return fail(STZ_EINVAL, "ipc_open: null argument");
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof(h));
  cudaError_t e = cudaIpcOpenMemHandle(base, h, cudaIpcMemLazyEnablePeerAccess);
  if (e != cudaSuccess) return fail(STZ_ECUDA, "ipc_open: %s", cudaGetErrorString(e));
  return STZ_OK;
}

int stz_ipc_close(void* base) {
  cudaError_t e = cudaIpcCloseMemHandle(base);
  if (e != cudaSuccess) return fail(STZ_ECUDA, "ipc_close: %s", cudaGetErrorString(e));
  return STZ_OK;
}

int stz_set_peer_timeout_ms(unsigned long long ms) {
  g_peer_timeout_ns = (ms ? ms : 60000ull) * 1000000ull;
  return STZ_OK;
}

int stz_peer_barrier(unsigned* const* flags, int nranks, int me, void* stream) {
  PeerTable t;
  if (int rc = fill_peers(t, nullptr, nullptr, flags, nranks, me)) return rc;
  for (int j = 0; j < nranks; ++j)
    if (!t.flags[j]) return fail(STZ_EINVAL, "peer_barrier: member %d flags null", j);
  peer_barrier_kernel<<<1, 32, 0, as_stream(stream)>>>(t, g_peer_timeout_ns);
  return check_launch("peer_barrier");
}

int stz_peer_reduce_push(const float* const* grads, float* const* red, int nranks, int me,
                         size_t n, void* stream) {
  PeerTable t;
  if (int rc = fill_peers(t, grads, red, nullptr, nranks, me)) return rc;
  if (n == 0) return STZ_OK;
  return launch_reduce_push(t, n, as_stream(stream));
}

int stz_sgd_momentum_pack(float* w, float* v, const float* g, size_t n, float lr, float mu,
                          float inv_n, const stz_plane_range* ranges, int nranges, void* stream) {
  if (n == 0) return STZ_OK;
  if (!aligned16(w) || !aligned16(v) || !aligned16(g))
    return fail(STZ_EINVAL, "sgd_momentum_pack: buffers must be 16-byte aligned");
  PackTable tab;
  if (int rc = fill_ranges(tab, n, ranges, nranges)) return rc;
  sgd_pack_kernel<<<grid_for(n / 4 + 1), 256, 0, as_stream(stream)>>>(w, v, g, tab, lr, mu,
                                                                        inv_n);
  return check_launch("sgd_momentum_pack");
}

int stz_allreduce_sgd(const float* const* grads, float* const* red, unsigned* const* flags,
                      int nranks, int me, float* w, float* v, size_t n, float lr, float mu,
                      float inv_n, const stz_plane_range* ranges, int nranges, void* stream) {
  PeerTable t;
  if (int rc = fill_peers(t, grads, red, flags, nranks, me)) return rc;
  PackTable tab;
  if (int rc = fill_ranges(tab, n, ranges, nranges)) return rc;
  if (!aligned16(w) || !aligned16(v)) return fail(STZ_EINVAL, "allreduce_sgd: w, v alignment");
  cudaStream_t st = as_stream(stream);
  if (nranks > 1) {
    peer_barrier_kernel<<<1, 32, 0, st>>>(t, g_peer_timeout_ns);
    if (int rc = check_launch("allreduce_sgd barrier")) return rc;
    if (n) {
      if (int rc = launch_reduce_push(t, n, st)) return rc;
    }
    peer_barrier_kernel<<<1, 32, 0, st>>>(t, g_peer_timeout_ns);
    if (int rc = check_launch("allreduce_sgd barrier")) return rc;
  }
  if (n == 0) return STZ_OK;
  const float* g = nranks > 1 ? red[me] : grads[me];
  sgd_pack_kernel<<<grid_for(n / 4 + 1), 256, 0, st>>>(
      w, v, g, tab, lr, mu, inv_n, nranks > 1 ? t.flags[me] + kFlagStatus : nullptr);
  return check_launch("allreduce_sgd update");
}

static_assert(STZ_LINK_FLAG_WORDS == kLinkWords && STZ_LINK_SLOTS == kLinkSlots &&
                  STZ_LINK_EPOCH == kLinkEpoch && STZ_LINK_STATUS == kLinkStatus,
              "link flag layout");
static_assert(STZ_PEER_FLAG_WORDS == kFlagWords, "peer flag layout");

int stz_link_begin(unsigned* flags, void* stream) {
  if (!flags) return fail(STZ_EINVAL, "link_begin: null flags");
  link_begin_kernel<<<1, 32, 0, as_stream(stream)>>>(flags);
  return check_launch("link_begin");
}

int stz_link_put(const void* src, size_t ps, int rows, int D, int D8, float* dst,
                 const int* labels, int* labels_dst, unsigned* my_flags, unsigned* remote_slot,
                 void* stream) {
  if (!src || !dst || !my_flags || !remote_slot || rows < 0 || D < 1 || D8 < D || D8 % 8 ||
      ps % 8 || !aligned16(src) || (D % 8 == 0 && (reinterpret_cast<uintptr_t>(dst) & 31)) ||
      (labels != nullptr) != (labels_dst != nullptr))
    return fail(STZ_EINVAL, "link_put: rows %d D %d D8 %d (D8 %% 8 == 0, 16-byte aligned "
                "planes, labels and their destination together)", rows, D, D8);
  const int grid = grid_for((size_t)rows * (D8 / 8) + 1);
  link_put_kernel<<<grid, 256, 0, as_stream(stream)>>>(cb(src), ps, rows, D, D8, dst, labels,
                                                       labels_dst, my_flags, remote_slot);
  return check_launch("link_put");
}

int stz_link_get(const float* src, int rows, int D, void* dst, size_t ps, int D8,
                 unsigned* my_flags, int slot0, int nslots, int slot_stride, void* stream) {
  if (!src || !dst || !my_flags || rows < 0 || D < 1 || D8 < D || D8 % 8 || ps % 8 ||
      !aligned16(dst) || (D % 4 == 0 && !aligned16(src)) || nslots < 0 || nslots > 32 ||
      slot0 < 0 || slot0 + (nslots > 0 ? (nslots - 1) * slot_stride : 0) >= kLinkSlots)
    return fail(STZ_EINVAL, "link_get: rows %d D %d D8 %d slots %d+%d*%d (< %d)", rows, D, D8,
                slot0, nslots, slot_stride, kLinkSlots);
  const int grid = grid_for((size_t)rows * (D8 / 8) + 1);
  link_get_kernel<<<grid, 256, 0, as_stream(stream)>>>(src, rows, D, D8, mb(dst), ps, my_flags,
                                                       slot0, nslots, slot_stride,
                                                       g_peer_timeout_ns);
  return check_launch("link_get");
}

}  // extern "C"
