// Gather-GEMM cores for the Stanza hot path.
//
//   gemm_tc_kernel    tcgen05 (5th-gen tensor core): operands are gathered by
//                     8 producer warps straight from the reference layouts,
//                     split into BF16 (x6) or TF32 (x3) pieces and staged in
//                     shared memory in the UMMA K-major canonical layout; one
//                     thread issues tcgen05.mma (fp32 accumulate in TMEM);
//                     the epilogue warps read TMEM with tcgen05.ld and apply
//                     bias / ReLU / ReLU-mask.
//   gemm_simt_kernel  fp32 FFMA core over the same operand views; a
//                     validation kernel for the GPU tests (stz_set_gemm_impl).
//
// Split-K writes fp32 partials to a caller workspace; splitk_reduce sums
// them in fixed split order (deterministic) and applies the epilogue.
#pragma once

#include "stz_operands.cuh"

namespace stz {

constexpr int TC_BM = 128;
constexpr int TC_THREADS = 288;  // 8 producer warps + 1 MMA warp

// Operand-splitting schemes.  Each stages PIECES copies of every operand
// tile in shared memory and issues NMMA tcgen05.mma per 32-byte K step
// (smallest cross terms first).
//
//   TF32x3 : x = hi + lo (tf32);  hi*lo + lo*hi | hi*hi       (kind::tf32)
//   BF16x6 : x = b0 + b1 + b2 (bf16, 8 bits each);
//            b0*b2 + b2*b0 + b1*b1 + b0*b1 + b1*b0 | b0*b0   (kind::f16)
//
// The cross terms ("small") and the leading term ("big") accumulate in TWO
// TMEM accumulators that the epilogue adds in fp32 round-to-nearest.
// Measured on B200 (tools/precision_probe*.py): the tensor core sums
// same-exponent products exactly but truncates bits shifted out during
// alignment, i.e. every MMA into D costs a bias of up to ~1 ulp(D) toward
// zero.  With one accumulator the six MMAs per K step all pay ulp(D) of the
// full sum (-7e-7 relative bias on positive data); the separate small-term
// accumulator pays only ulp(small) ~ 2^-8 ulp(D).  BF16x6 runs at the same
// tensor-core time as TF32x3 (bf16 MMAs are 2x the tf32 rate) with exact
// 16-bit products and 25% less shared memory per stage.
struct SchemeTF32x3 {
  static constexpr int ES = 4, PIECES = 2, NMMA = 3;
  __host__ __device__ static constexpr int big(int i) { return i == 2; }
  static constexpr int EPC = 16 / ES;  // elements per 16-byte K chunk
  __host__ __device__ static constexpr int a_piece(int i) { return i == 1 ? 1 : 0; }
  __host__ __device__ static constexpr int b_piece(int i) { return i == 0 ? 1 : 0; }
  __host__ __device__ static constexpr uint32_t idesc(int m, int n) { return umma_idesc_tf32(m, n); }
  __device__ static void mma(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
    umma_tf32(d, a, b, id, acc);
  }
  // v: EPC fp32 values of one row's 16-byte chunk -> one 16-byte store per piece
  __device__ static void stage(const float (&v)[EPC], uint32_t dst, uint32_t piece_bytes) {
    float h[4], l[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) split_tf32(v[j], h[j], l[j]);
    sts128(dst, h[0], h[1], h[2], h[3]);
    sts128(dst + piece_bytes, l[0], l[1], l[2], l[3]);
  }
};

struct SchemeBF16x6 {
  static constexpr int ES = 2, PIECES = 3, NMMA = 6;
  __host__ __device__ static constexpr int big(int i) { return i == 5; }
  static constexpr int EPC = 16 / ES;
  __host__ __device__ static constexpr int a_piece(int i) {
    return i == 0 ? 0 : i == 1 ? 2 : i == 2 ? 1 : i == 3 ? 0 : i == 4 ? 1 : 0;
  }
  __host__ __device__ static constexpr int b_piece(int i) {
    return i == 0 ? 2 : i == 1 ? 0 : i == 2 ? 1 : i == 3 ? 1 : i == 4 ? 0 : 0;
  }
  __host__ __device__ static constexpr uint32_t idesc(int m, int n) { return umma_idesc_bf16(m, n); }
  __device__ static void mma(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
    umma_f16(d, a, b, id, acc);
  }
  __device__ static void stage(const float (&v)[EPC], uint32_t dst, uint32_t piece_bytes) {
    uint32_t p0[4], p1[4], p2[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      uint16_t a0, a1, a2, c0, c1, c2;
      split_bf16x3(v[2 * j], a0, a1, a2);
      split_bf16x3(v[2 * j + 1], c0, c1, c2);
      p0[j] = (uint32_t)a0 | ((uint32_t)c0 << 16);
      p1[j] = (uint32_t)a1 | ((uint32_t)c1 << 16);
      p2[j] = (uint32_t)a2 | ((uint32_t)c2 << 16);
    }
    sts128u(dst, p0[0], p0[1], p0[2], p0[3]);
    sts128u(dst + piece_bytes, p1[0], p1[1], p1[2], p1[3]);
    sts128u(dst + 2 * piece_bytes, p2[0], p2[1], p2[2], p2[3]);
  }
};

template <class S, int BN, int BK>
struct TcCfg {
  static constexpr int CH = BK * S::ES / 16;         // 16-byte K chunks per row
  static constexpr int A_BYTES = TC_BM * BK * S::ES; // one piece of the A tile
  static constexpr int B_BYTES = BN * BK * S::ES;
  static constexpr int STAGE_BYTES = S::PIECES * (A_BYTES + B_BYTES);
  static constexpr int STAGES = (200 * 1024) / STAGE_BYTES > 6 ? 6 : (200 * 1024) / STAGE_BYTES;
  static constexpr int SMEM = STAGES * STAGE_BYTES + 256;
  static constexpr int TPR = 8 * CH;                 // threads covering one 8-row group
  static constexpr int MG_STEP = 128 / TPR;          // row groups per pass of 128 threads
  static constexpr int A_IT = (TC_BM / 8) / MG_STEP;
  static constexpr int B_IT = (BN / 8) / MG_STEP;
  static constexpr int KSTEPS = BK * S::ES / 32;     // MMA K steps (32 bytes each) per stage
  // two accumulators (big, small) of BN fp32 columns each
  static constexpr int TMEM_COLS = BN <= 16 ? 32 : BN <= 32 ? 64 : BN <= 64 ? 128 : BN <= 128 ? 256 : 512;
  static constexpr uint32_t SBO = CH * 128;          // next 8-row core-matrix group
  static constexpr uint32_t LBO = 128;               // next 16-byte K chunk
  static_assert(STAGES >= 2, "tile too large");
  static_assert(TPR <= 128 && 128 % TPR == 0, "chunk mapping");
  static_assert((BN / 8) % MG_STEP == 0, "BN must cover whole producer passes");
};

template <class S, int BN, int BK, class VA, class VB>
__global__ void __launch_bounds__(TC_THREADS, 1)
    gemm_tc_kernel(VA va, VB vb, Epilogue epi, float* __restrict__ partial, int M, int N, int K,
                   int k_per_split) {
  using Cfg = TcCfg<S, BN, BK>;
  constexpr int STAGES = Cfg::STAGES;
  constexpr int EPC = S::EPC;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + STAGES * Cfg::STAGE_BYTES);
  uint64_t* empty_bar = full_bar + STAGES;
  uint64_t* done_bar = empty_bar + STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done_bar + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m0 = blockIdx.x * TC_BM, n0 = blockIdx.y * BN;
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
    // ---------------- producers: gather -> split -> st.shared ------------
    const int grp = warp >> 2;
    const int t = threadIdx.x & 127;
    const int mi = t & 7;
    const int ch = (t >> 3) % Cfg::CH;
    const int mg0 = t / Cfg::TPR;
    typename VA::Row ra[Cfg::A_IT];
    typename VB::Row rb[Cfg::B_IT];
#pragma unroll
    for (int i = 0; i < Cfg::A_IT; ++i) ra[i] = va.row(m0 + (mg0 + i * Cfg::MG_STEP) * 8 + mi);
#pragma unroll
    for (int i = 0; i < Cfg::B_IT; ++i) rb[i] = vb.row(n0 + (mg0 + i * Cfg::MG_STEP) * 8 + mi);

    for (int kb = grp; kb < nkb; kb += 2) {
      const int stage = kb % STAGES;
      mbar_wait(&empty_bar[stage], ((kb / STAGES) & 1) ^ 1);
      const int k0 = kbeg + kb * BK + ch * EPC;
      const uint32_t st = smem_base + stage * Cfg::STAGE_BYTES;
      float av[Cfg::A_IT][EPC], bv[Cfg::B_IT][EPC];
#pragma unroll
      for (int i = 0; i < Cfg::A_IT; ++i)
#pragma unroll
        for (int q = 0; q < EPC / 4; ++q) {
          const float4 v = va.load(ra[i], k0 + 4 * q);
          av[i][4 * q] = v.x; av[i][4 * q + 1] = v.y; av[i][4 * q + 2] = v.z; av[i][4 * q + 3] = v.w;
        }
#pragma unroll
      for (int i = 0; i < Cfg::B_IT; ++i)
#pragma unroll
        for (int q = 0; q < EPC / 4; ++q) {
          const float4 v = vb.load(rb[i], k0 + 4 * q);
          bv[i][4 * q] = v.x; bv[i][4 * q + 1] = v.y; bv[i][4 * q + 2] = v.z; bv[i][4 * q + 3] = v.w;
        }
#pragma unroll
      for (int i = 0; i < Cfg::A_IT; ++i) {
        const uint32_t off = ((mg0 + i * Cfg::MG_STEP) * Cfg::CH + ch) * 128 + mi * 16;
        S::stage(av[i], st + off, Cfg::A_BYTES);
      }
#pragma unroll
      for (int i = 0; i < Cfg::B_IT; ++i) {
        const uint32_t off = ((mg0 + i * Cfg::MG_STEP) * Cfg::CH + ch) * 128 + mi * 16;
        S::stage(bv[i], st + S::PIECES * Cfg::A_BYTES + off, Cfg::B_BYTES);
      }
      fence_proxy_async_smem();
      mbar_arrive(&full_bar[stage]);
    }

    if (grp == 0) {
      // ---------------- epilogue: TMEM -> registers -> global -------------
      mbar_wait(done_bar, 0);
      tc_fence_after();
      const int q = warp & 3;  // TMEM lane quadrant of this warp
      const int m = m0 + q * 32 + lane;
#pragma unroll 1
      for (int c = 0; c < BN; c += 16) {
        uint32_t r[16], rs[16];
        const uint32_t taddr = tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)c;
        tmem_ld16(taddr, r);
        tmem_ld16(taddr + BN, rs);
        tmem_ld_wait();
#pragma unroll
        for (int j = 0; j < 16; ++j)
          r[j] = __float_as_uint(__fadd_rn(__uint_as_float(r[j]), __uint_as_float(rs[j])));
        if (partial) {
          if (m < M) {
            float* dst = partial + ((size_t)blockIdx.z * M + m) * N;
#pragma unroll
            for (int j = 0; j < 16; ++j)
              if (n0 + c + j < N) dst[n0 + c + j] = __uint_as_float(r[j]);
          }
        } else {
#pragma unroll
          for (int j = 0; j < 16; ++j) epi.store(m, n0 + c + j, __uint_as_float(r[j]));
        }
      }
    }
  } else if (lane == 0) {
    // ---------------- MMA issuer (one thread) ---------------------------
    constexpr uint32_t idesc = S::idesc(TC_BM, BN);
    for (int kb = 0; kb < nkb; ++kb) {
      const int stage = kb % STAGES;
      mbar_wait(&full_bar[stage], (kb / STAGES) & 1);
      tc_fence_after();
      const uint32_t a0 = smem_base + stage * Cfg::STAGE_BYTES;
      const uint32_t b0 = a0 + S::PIECES * Cfg::A_BYTES;
#pragma unroll
      for (int j = 0; j < Cfg::KSTEPS; ++j) {
        const uint32_t off = j * 2 * Cfg::LBO;  // two 16-byte K chunks per MMA
#pragma unroll
        for (int i = 0; i < S::NMMA; ++i) {
          const uint64_t da =
              umma_desc_kmajor(a0 + S::a_piece(i) * Cfg::A_BYTES + off, Cfg::LBO, Cfg::SBO);
          const uint64_t db =
              umma_desc_kmajor(b0 + S::b_piece(i) * Cfg::B_BYTES + off, Cfg::LBO, Cfg::SBO);
          // first MMA into each accumulator overwrites it
          const bool first = (kb | j) == 0 && (S::big(i) ? true : i == 0);
          S::mma(tmem_base + (S::big(i) ? 0u : (uint32_t)BN), da, db, idesc, first ? 0u : 1u);
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

// ---------------------------------------------------------------------------
// SIMT fp32 core (validation): 128 x 64 tile, 256 threads, 8x4 per thread.
// ---------------------------------------------------------------------------

template <class VA, class VB>
__global__ void __launch_bounds__(256)
    gemm_simt_kernel(VA va, VB vb, Epilogue epi, float* __restrict__ partial, int M, int N, int K,
                     int k_per_split) {
  constexpr int BM = 128, BN = 64, BK = 16;
  __shared__ float As[BK][BM + 4];
  __shared__ float Bs[BK][BN + 4];
  const int t = threadIdx.x;
  const int m0 = blockIdx.x * BM, n0 = blockIdx.y * BN;
  const int kbeg = blockIdx.z * k_per_split;
  const int kend = min(K, kbeg + k_per_split);

  const int ar = t & 127, akc = t >> 7;  // rows 0..127, kc {0,1} (+2)
  const int br = t & 63, bkc = t >> 6;   // rows 0..63, kc 0..3
  typename VA::Row ra = va.row(m0 + ar);
  typename VB::Row rb = vb.row(n0 + br);
  const int tx = t & 15, ty = t >> 4;
  float acc[8][4];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;

  for (int k = kbeg; k < kend; k += BK) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int kc = akc + 2 * h;
      float4 v = va.load(ra, k + kc * 4);
      As[kc * 4 + 0][ar] = v.x;
      As[kc * 4 + 1][ar] = v.y;
      As[kc * 4 + 2][ar] = v.z;
      As[kc * 4 + 3][ar] = v.w;
    }
    {
      float4 v = vb.load(rb, k + bkc * 4);
      Bs[bkc * 4 + 0][br] = v.x;
      Bs[bkc * 4 + 1][br] = v.y;
      Bs[bkc * 4 + 2][br] = v.z;
      Bs[bkc * 4 + 3][br] = v.w;
    }
    __syncthreads();
    const int kmax = min(BK, kend - k);
    for (int kk = 0; kk < kmax; ++kk) {
      float a[8], b[4];
#pragma unroll
      for (int i = 0; i < 8; ++i) a[i] = As[kk][ty * 8 + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Bs[kk][tx * 4 + j];
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int m = m0 + ty * 8 + i;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int n = n0 + tx * 4 + j;
      if (partial) {
        if (m < M && n < N) partial[((size_t)blockIdx.z * M + m) * N + n] = acc[i][j];
      } else {
        epi.store(m, n, acc[i][j]);
      }
    }
  }
}

// Deterministic split-K reduction (fixed split order) + epilogue.
__global__ void splitk_reduce_kernel(const float* __restrict__ partial, int splits, int M, int N,
                                     Epilogue epi) {
  const size_t total = (size_t)M * N;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total;
       i += (size_t)gridDim.x * blockDim.x) {
    float s = partial[i];
    for (int z = 1; z < splits; ++z) s = __fadd_rn(s, partial[(size_t)z * total + i]);
    epi.store((int)(i / N), (int)(i % N), s);
  }
}

}  // namespace stz
