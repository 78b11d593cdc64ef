// Gradient exchange + momentum SGD over NVLink peer memory (no NCCL on the
// data path), and the fused SGD + split-plane weight repack.
//
// Replaces the reference's exchange and update phases,
//   _exchange_phase  stanza_runtime.py:309-338  (allreduce_sum of the flat
//                    block-gradient vector in the CONV group and, iff
//                    n_fc > 1, the FC group; collectives.py:117-157)
//   _update_phase    stanza_runtime.py:340-350  (unpack_vector + sgd_step,
//                    tensor_core.py:366-388, on every replica)
// for one role group of R ranks (one process per GPU) whose flat gradient
// vectors, reduced-gradient buffers and flag words are mapped into every
// member through CUDA IPC (stz_ipc_handle / stz_ipc_open):
//
//   barrier        every member's gradient vector is complete;
//   reduce-push    member r owns chunk r: it reads chunk r of every member's
//                  gradient over NVLink, sums them in group-rank order
//                  (g_0 + g_1 + ... + g_{R-1}, fp32 RN -- the same bits no
//                  matter which member computes them) and stores the sum into
//                  chunk r of EVERY member's reduced buffer (remote stores);
//   barrier        every chunk has landed everywhere;
//   sgd + pack     each member applies v = v*mu + g*inv_n; w = w - lr*v to
//                  its own replica from its local reduced buffer and, in the
//                  same pass, rewrites the GEMM-ready split-plane copy of the
//                  weights whose plane layout is row-major (FC W [in][out8]).
//
// Remote traffic per member is 2 (R-1)/R of the vector, as for a ring
// allreduce, and the update reads the reduced gradient from local HBM.  Every
// member ends with bit-identical (w, v) -- the replica invariant the reference
// asserts (tests/test_stanza_runtime.py:70-83) -- because every sum is formed
// once and copied.
//
// Safety across iterations: a member's gradient vector is rewritten only by
// its next backward, which follows its own second barrier, which no member
// passes before every member finished its reduce-push reads; the reduced
// buffer is rewritten only by the next reduce-push, which follows the next
// first barrier, which no member passes before every member finished its
// update.  So two barriers per iteration and no double buffering.
//
// Barrier: flags[t][me] = epoch (release, system scope) for every member t,
// then wait (acquire) until flags[me][t] >= epoch for every t.  The epoch is a
// device-resident counter so CUDA-graph replays advance it.  A member that
// never arrives does not hang the GPU: after the timeout the waiting kernel
// writes a status word (kFlagStatus) and returns; every later exchange kernel
// of that member sees the status and does nothing, and the host raises
// MissingSource when it reads the word (stanza_runtime.StanzaCluster.train).
#pragma once

#include "stz_split.cuh"

namespace stz {

constexpr int kMaxPeers = 8;
constexpr int kMaxPackRanges = 16;
// flag-word layout of one member's IPC-visible int32 block
constexpr int kFlagCounter = 16;   // local epoch counter
constexpr int kFlagStatus = 17;    // != 0: a wait timed out (code, see peer_barrier_kernel)
constexpr int kFlagWords = 32;

struct PeerTable {
  int R, me;
  const float* g[kMaxPeers];   // gradient vectors (index = group rank)
  float* red[kMaxPeers];       // reduced-gradient buffers
  unsigned* flags[kMaxPeers];  // flag blocks (kFlagWords words each)
};

// [off, off+len) of the flat parameter vector; planes != null: the values are
// also rewritten as split planes of a row-major [len/D][D8] matrix
struct PackRange {
  size_t off, len;
  bf16_t* planes;
  size_t ps;
  int D, D8;
};
struct PackTable {
  int n;
  PackRange r[kMaxPackRanges];
};

__device__ __forceinline__ void st_release_sys(unsigned* p, unsigned v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned ld_acquire_sys(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ unsigned ld_volatile(const unsigned* p) {
  return *reinterpret_cast<const volatile unsigned*>(p);
}

// status code of a barrier that timed out waiting for member j
constexpr unsigned kStatusBarrier = 0x10000u;

__global__ void peer_barrier_kernel(PeerTable t, unsigned long long timeout_ns) {
  __shared__ unsigned epoch;
  unsigned* mine = t.flags[t.me];
  if (ld_volatile(mine + kFlagStatus)) return;   // an earlier wait already failed
  if (threadIdx.x == 0) {
    epoch = mine[kFlagCounter] + 1;
    mine[kFlagCounter] = epoch;
  }
  __syncthreads();
  const int j = threadIdx.x;
  if (j < t.R) {
    __threadfence_system();  // this member's prior writes (kernels before us) first
    st_release_sys(t.flags[j] + t.me, epoch);
    const unsigned long long t0 = globaltimer_ns();
    while ((int)(ld_acquire_sys(mine + j) - epoch) < 0) {
      __nanosleep(64);
      if (globaltimer_ns() - t0 > timeout_ns) {
        printf("stz_peer_barrier: member %d waited %.1f s for member %d (epoch %u)\n", t.me,
               timeout_ns * 1e-9, j, epoch);
        atomicCAS(mine + kFlagStatus, 0u, kStatusBarrier | (unsigned)j);
        break;
      }
    }
  }
  __syncthreads();
}

__device__ __forceinline__ float4 add4(float4 a, float4 b) {
  return make_float4(__fadd_rn(a.x, b.x), __fadd_rn(a.y, b.y), __fadd_rn(a.z, b.z),
                     __fadd_rn(a.w, b.w));
}

// chunk [c0, c1) of the vector (c0 % 8 == 0): sum over members in rank order,
// store into every member's reduced buffer.  8 floats per item, two items
// per thread per trip keep 4R remote 16-byte loads in flight; each sum
// leaves as one 256-bit store per member (two 16-byte stores to the same
// sector halve the NVLink store rate, tools/p2p_bench.cu).
__device__ __forceinline__ void add8(float (&s)[8], float4 a, float4 b) {
  s[0] = __fadd_rn(s[0], a.x); s[1] = __fadd_rn(s[1], a.y);
  s[2] = __fadd_rn(s[2], a.z); s[3] = __fadd_rn(s[3], a.w);
  s[4] = __fadd_rn(s[4], b.x); s[5] = __fadd_rn(s[5], b.y);
  s[6] = __fadd_rn(s[6], b.z); s[7] = __fadd_rn(s[7], b.w);
}

template <int R>
__global__ void __launch_bounds__(256) peer_reduce_push_kernel(PeerTable t, size_t c0, size_t c1) {
  if (ld_volatile(t.flags[t.me] + kFlagStatus)) return;   // a peer is missing: touch nothing
  const size_t e0 = c0 / 8, e1 = c1 / 8;                  // 8-float items
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t q = e0 + blockIdx.x * (size_t)blockDim.x + threadIdx.x; q < e1; q += 2 * stride) {
    const size_t q2 = q + stride;
    const bool two = q2 < e1;
    float4 a[R][2], b[R][2];
#pragma unroll
    for (int j = 0; j < R; ++j) {
      const float4* g4 = reinterpret_cast<const float4*>(t.g[j]);
      a[j][0] = __ldcv(g4 + 2 * q);
      a[j][1] = __ldcv(g4 + 2 * q + 1);
      if (two) {
        b[j][0] = __ldcv(g4 + 2 * q2);
        b[j][1] = __ldcv(g4 + 2 * q2 + 1);
      }
    }
    float s[8] = {a[0][0].x, a[0][0].y, a[0][0].z, a[0][0].w,
                  a[0][1].x, a[0][1].y, a[0][1].z, a[0][1].w};
    float u[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    if (two) {
      u[0] = b[0][0].x; u[1] = b[0][0].y; u[2] = b[0][0].z; u[3] = b[0][0].w;
      u[4] = b[0][1].x; u[5] = b[0][1].y; u[6] = b[0][1].z; u[7] = b[0][1].w;
    }
#pragma unroll
    for (int j = 1; j < R; ++j) {
      add8(s, a[j][0], a[j][1]);
      if (two) add8(u, b[j][0], b[j][1]);
    }
#pragma unroll
    for (int j = 0; j < R; ++j) {
      stg256(t.red[j] + 8 * q, s);
      if (two) stg256(t.red[j] + 8 * q2, u);
    }
  }
  // scalar tail of the last chunk
  if (blockIdx.x == 0 && threadIdx.x < (c1 - e1 * 8) && e1 * 8 >= c0) {
    const size_t i = e1 * 8 + threadIdx.x;
    float s = __ldcv(t.g[0] + i);
#pragma unroll
    for (int j = 1; j < R; ++j) s = __fadd_rn(s, __ldcv(t.g[j] + i));
#pragma unroll
    for (int j = 0; j < R; ++j) t.red[j][i] = s;
  }
}

// tensor_core.py:366-388 in the exact fp32 op order (no contraction)
__device__ __forceinline__ void sgd_1(float& w, float& v, float g, float lr, float mu, float inv_n) {
  v = __fadd_rn(__fmul_rn(v, mu), __fmul_rn(g, inv_n));
  w = __fsub_rn(w, __fmul_rn(lr, v));
}

__device__ __forceinline__ uint2 pack4(bf16_t a, bf16_t b, bf16_t c, bf16_t d) {
  return make_uint2((uint32_t)a | ((uint32_t)b << 16), (uint32_t)c | ((uint32_t)d << 16));
}

// FC weight gradient fused with the momentum step (one FC worker):
// GEMM element (m, n) = the batch sum gW[m][n] of W [in][out] is never
// stored -- the epilogue applies sgd_1 (the reference's op order,
// tensor_core.py:366-388) to w / v at m*N + n and rewrites the split-plane
// GEMM copy at m*N8 + n, so the gradient makes no round trip through HBM.
// `accumulate`: the value is added to gw[m*N + n] first (micro-batch sums).
struct EpSgd {
  float* w;
  float* v;
  const float* gw;     // accumulate: earlier micro-batches' gradient sum (or null)
  bf16_t* planes;
  size_t ps;
  int M, N, N8;
  float lr, mu, inv_n;
  static constexpr bool HAS_BIAS = false;
  static constexpr bool STAGED = false;
  __device__ __forceinline__ void bias8(int, float (&)[8]) const {}
  __device__ __forceinline__ void store8_nb(int m, int n0, float (&g)[8]) const { store8(m, n0, g); }
  __device__ __forceinline__ void store8(int m, int n0, float (&g)[8]) const {
    if (m >= M || n0 >= N) return;
    const size_t row = (size_t)m * N;
    // the epilogue walks a row 32 columns per step: start this row's next two
    // steps of w / v towards L2 now (the loads below are latency-bound)
#pragma unroll
    for (int a = 32; a <= 64; a += 32)
      if (n0 + a < N) {
        asm volatile("prefetch.global.L2 [%0];" ::"l"(w + row + n0 + a));
        asm volatile("prefetch.global.L2 [%0];" ::"l"(v + row + n0 + a));
      }
    if (n0 + 8 <= N && ((row + n0) & 3) == 0) {
      float4* w4 = reinterpret_cast<float4*>(w + row + n0);
      float4* v4 = reinterpret_cast<float4*>(v + row + n0);
      const float4 a0 = w4[0], a1 = w4[1], b0 = v4[0], b1 = v4[1];
      float ww[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
      float vv[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
      if (gw) {
        const float4* g4 = reinterpret_cast<const float4*>(gw + row + n0);
        const float4 c0 = g4[0], c1 = g4[1];
        const float gg[8] = {c0.x, c0.y, c0.z, c0.w, c1.x, c1.y, c1.z, c1.w};
#pragma unroll
        for (int j = 0; j < 8; ++j) g[j] = __fadd_rn(gg[j], g[j]);
      }
#pragma unroll
      for (int j = 0; j < 8; ++j) sgd_1(ww[j], vv[j], g[j], lr, mu, inv_n);
      w4[0] = make_float4(ww[0], ww[1], ww[2], ww[3]);
      w4[1] = make_float4(ww[4], ww[5], ww[6], ww[7]);
      v4[0] = make_float4(vv[0], vv[1], vv[2], vv[3]);
      v4[1] = make_float4(vv[4], vv[5], vv[6], vv[7]);
      store_split8(planes + (size_t)m * N8 + n0, ps, ww);
      return;
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int n = n0 + j;
      if (n >= N) break;
      float a = w[row + n], b = v[row + n];
      const float gj = gw ? __fadd_rn(gw[row + n], g[j]) : g[j];
      sgd_1(a, b, gj, lr, mu, inv_n);
      w[row + n] = a;
      v[row + n] = b;
      store_split(planes, ps, (size_t)m * N8 + n, a);
    }
  }
};

// FC bias gradient (fixed-order column sums, as colsum_final_kernel) fused
// with its momentum step; the summed gradient is also stored in gb
__global__ void __launch_bounds__(256) colsum_sgd_final_kernel(const double* __restrict__ part,
                                                               int blocks, int N, int N8,
                                                               float* __restrict__ gb,
                                                               const float* __restrict__ gb_acc,
                                                               float* __restrict__ wb,
                                                               float* __restrict__ vb, float lr,
                                                               float mu, float inv_n) {
  const int c = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (c >= N) return;
  double s = 0.0;
  int b = lane;
  for (; b + 224 < blocks; b += 256) {
    double v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = part[(size_t)(b + 32 * u) * N8 + c];
#pragma unroll
    for (int u = 0; u < 8; ++u) s += v[u];
  }
  for (; b < blocks; b += 32) s += part[(size_t)b * N8 + c];
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane) return;
  const float g = gb_acc ? __fadd_rn(gb_acc[c], (float)s) : (float)s;
  if (gb) gb[c] = g;
  float a = wb[c], q = vb[c];
  sgd_1(a, q, g, lr, mu, inv_n);
  wb[c] = a;
  vb[c] = q;
}

// Momentum SGD over every range of the table (which partitions [0, n)); a
// range with planes also stores the new weights as split planes.  Range
// offsets are multiples of 4 (16-byte aligned tensor views).
__global__ void __launch_bounds__(256) sgd_pack_kernel(float* __restrict__ w, float* __restrict__ v,
                                                       const float* __restrict__ g, PackTable tab,
                                                       float lr, float mu, float inv_n,
                                                       const unsigned* status = nullptr) {
  if (status && ld_volatile(status)) return;   // the exchange before it failed
  const size_t tid = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (int r = 0; r < tab.n; ++r) {
    const PackRange rg = tab.r[r];
    if (rg.D == 0) continue;   // updated in its weight-gradient epilogue (EpSgd)
    const size_t n4 = rg.len / 4;
    float4* w4 = reinterpret_cast<float4*>(w + rg.off);
    float4* v4 = reinterpret_cast<float4*>(v + rg.off);
    const float4* g4 = reinterpret_cast<const float4*>(g + rg.off);
    const bool rowmajor = rg.planes != nullptr && rg.D == rg.D8;
    for (size_t i = tid; i < n4; i += stride) {
      float4 a = w4[i], b = v4[i];
      const float4 c = g4[i];
      sgd_1(a.x, b.x, c.x, lr, mu, inv_n);
      sgd_1(a.y, b.y, c.y, lr, mu, inv_n);
      sgd_1(a.z, b.z, c.z, lr, mu, inv_n);
      sgd_1(a.w, b.w, c.w, lr, mu, inv_n);
      w4[i] = a;
      v4[i] = b;
      if (rowmajor) {
        bf16_t p[4][3];
        split_bf16x3(a.x, p[0][0], p[0][1], p[0][2]);
        split_bf16x3(a.y, p[1][0], p[1][1], p[1][2]);
        split_bf16x3(a.z, p[2][0], p[2][1], p[2][2]);
        split_bf16x3(a.w, p[3][0], p[3][1], p[3][2]);
        uint2* dst = reinterpret_cast<uint2*>(rg.planes) + i;
        const size_t pq = rg.ps / 4;  // plane stride in uint2
#pragma unroll
        for (int k = 0; k < 3; ++k) dst[k * pq] = pack4(p[0][k], p[1][k], p[2][k], p[3][k]);
      } else if (rg.planes != nullptr) {
        const float vals[4] = {a.x, a.y, a.z, a.w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const size_t j = i * 4 + e;
          store_split(rg.planes, rg.ps, (j / rg.D) * rg.D8 + j % rg.D, vals[e]);
        }
      }
    }
    for (size_t j = n4 * 4 + tid; j < rg.len; j += stride) {
      float a = w[rg.off + j], b = v[rg.off + j];
      sgd_1(a, b, g[rg.off + j], lr, mu, inv_n);
      w[rg.off + j] = a;
      v[rg.off + j] = b;
      if (rg.planes != nullptr) store_split(rg.planes, rg.ps, (j / rg.D) * rg.D8 + j % rg.D, a);
    }
  }
}

// ---------------------------------------------------------------------------
// CONV <-> FC link over peer memory (the activation gather and the
// boundary-gradient scatter, stanza_runtime.py:228-307 in the reference)
//
// Each rank owns a link flag block (kLinkWords uint32, zeroed once, mapped
// by its link peers) and an fp32 staging buffer for what it receives (FC
// worker: [micro][member][kb][A] activations; CONV worker: [K][A] boundary
// gradients).  One iteration:
//
//   link_begin  epoch += 1 (every rank, once per step, first on its stream);
//   link_put    the sender reads its split-plane rows, joins them to fp32
//               (exact) and stores them straight into the receiver's staging
//               rows over NVLink -- 4 B per element on the link, one kernel
//               per (member, micro-batch) message -- plus the labels (int32)
//               into the receiver's label rows; the last CTA to finish
//               publishes the sender's epoch in the receiver's slot
//               (fence.sys + st.release.sys);
//   link_get    the receiver's CTAs each wait (ld.acquire.sys) until every
//               slot of the micro-batch carries the epoch, then split the
//               staged fp32 rows into its local split-plane buffer.
//
// No host synchronisation and no NCCL on the data path: the whole step is
// stream-ordered device work (a CUDA graph per rank).  Staging reuse is safe
// without credits: a sender's put of iteration t+1 follows (on its stream) its
// receipt of iteration t's answer, which the receiver sends only after its
// get of iteration t consumed the staging rows.
// ---------------------------------------------------------------------------
constexpr int kLinkWords = 256;
constexpr int kLinkSlots = 192;     // message slots [0, 192)
constexpr int kLinkEpoch = 240;     // local step epoch
constexpr int kLinkStatus = 241;    // != 0: a get timed out (kStatusLink | slot)
constexpr int kLinkDone = 242;      // CTA-completion counter of the running put
constexpr unsigned kStatusLink = 0x20000u;

__global__ void link_begin_kernel(unsigned* flags) {
  if (threadIdx.x == 0) flags[kLinkEpoch] += 1;
}

// src: split planes [rows][D8] (plane stride ps); dst: fp32 [rows][D] (remote)
__global__ void __launch_bounds__(256) link_put_kernel(const bf16_t* __restrict__ src, size_t ps,
                                                       int rows, int D, int D8, float* dst,
                                                       const int* __restrict__ lab_src,
                                                       int* lab_dst, unsigned* my_flags,
                                                       unsigned* remote_slot) {
  const unsigned epoch = ld_volatile(my_flags + kLinkEpoch);
  const int per_row = D8 / 8;
  const size_t n8 = (size_t)rows * per_row;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  const bool vec = (D % 8) == 0;
  for (size_t q = blockIdx.x * (size_t)blockDim.x + threadIdx.x; q < n8; q += stride) {
    const size_t r = q / per_row;
    const int c = (int)(q - r * per_row) * 8;
    const size_t s = r * D8 + c;
    const uint4 a = __ldg(reinterpret_cast<const uint4*>(src + s));
    const uint4 b = __ldg(reinterpret_cast<const uint4*>(src + s + ps));
    const uint4 d = __ldg(reinterpret_cast<const uint4*>(src + s + 2 * ps));
    const uint32_t aw[4] = {a.x, a.y, a.z, a.w}, bw[4] = {b.x, b.y, b.z, b.w},
                   dw[4] = {d.x, d.y, d.z, d.w};
    float v[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const int sh = (e & 1) * 16;
      v[e] = join3((bf16_t)(aw[e / 2] >> sh), (bf16_t)(bw[e / 2] >> sh), (bf16_t)(dw[e / 2] >> sh));
    }
    float* out = dst + r * D + c;
    if (vec) {
      // one 256-bit store per 8 elements: over NVLink two 16-byte stores to
      // the same 32-byte sector run at half the rate (tools/p2p_bench.cu:
      // 320 vs 680 GB/s GPU -> GPU)
      stg256(out, v);
    } else {
#pragma unroll
      for (int e = 0; e < 8; ++e)
        if (c + e < D) out[e] = v[e];
    }
  }
  if (lab_src)
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < (size_t)rows; i += stride)
      lab_dst[i] = lab_src[i];
  // publish: every thread's remote stores before the CTA's arrival, the last
  // CTA releases the receiver's slot
  __shared__ bool last;
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(my_flags + kLinkDone, 1u) == gridDim.x - 1;
  __syncthreads();
  if (last && threadIdx.x == 0) {
    my_flags[kLinkDone] = 0;
    __threadfence_system();
    st_release_sys(remote_slot, epoch);
  }
}

// wait for slots slot0 + i*slot_stride (i < nslots), then src fp32 [rows][D]
// (local staging, written by peers) -> split planes dst [rows][D8]
__global__ void __launch_bounds__(256) link_get_kernel(const float* src, int rows, int D, int D8,
                                                       bf16_t* __restrict__ dst, size_t ps,
                                                       unsigned* my_flags, int slot0, int nslots,
                                                       int slot_stride,
                                                       unsigned long long timeout_ns) {
  __shared__ int failed;
  const unsigned epoch = ld_volatile(my_flags + kLinkEpoch);
  if (threadIdx.x == 0) failed = ld_volatile(my_flags + kLinkStatus) != 0;
  __syncthreads();
  if (failed) return;
  if (threadIdx.x < nslots) {
    const int slot = slot0 + threadIdx.x * slot_stride;
    const unsigned long long t0 = globaltimer_ns();
    while ((int)(ld_acquire_sys(my_flags + slot) - epoch) < 0) {
      __nanosleep(128);
      if (globaltimer_ns() - t0 > timeout_ns) {
        if (atomicCAS(my_flags + kLinkStatus, 0u, kStatusLink | (unsigned)slot) == 0u)
          printf("stz_link_get: slot %d waited %.1f s (epoch %u)\n", slot, timeout_ns * 1e-9,
                 epoch);
        failed = 1;
        break;
      }
    }
  }
  __syncthreads();
  if (failed) return;
  const int per_row = D8 / 8;
  const size_t n8 = (size_t)rows * per_row;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  const bool vec = (D % 8) == 0;
  for (size_t q = blockIdx.x * (size_t)blockDim.x + threadIdx.x; q < n8; q += stride) {
    const size_t r = q / per_row;
    const int c = (int)(q - r * per_row) * 8;
    const float* in = src + r * D + c;
    float v[8];
    if (vec) {
      const float4 x = __ldcg(reinterpret_cast<const float4*>(in));
      const float4 y = __ldcg(reinterpret_cast<const float4*>(in) + 1);
      v[0] = x.x, v[1] = x.y, v[2] = x.z, v[3] = x.w, v[4] = y.x, v[5] = y.y, v[6] = y.z,
      v[7] = y.w;
    } else {
#pragma unroll
      for (int e = 0; e < 8; ++e) v[e] = c + e < D ? __ldcg(in + e) : 0.f;
    }
    store_split8(dst + r * D8 + c, ps, v);
  }
}

}  // namespace stz
