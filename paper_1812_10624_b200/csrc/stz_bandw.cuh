// Shifted-window ("band") weight gradient of a stride-1 conv with 64 or 32
// input channels and 64 outputs: AlexNet conv1 as space-to-depth (3x3 taps
// over 4x4 blocks, 48 -> 64 channels) and ResNet-50's stem (4x4 taps over
// 2x2 blocks, 12 -> 32 channels; CW = 32 puts four taps in one 128-row
// operand on SWIZZLE_64B rows), reference
// tensor_core.py:242-261.  The description below is the CW = 64 case.
//
//   dW[o][t][c] = sum_q dY[q][o] * X[q + off(t)][c]
//
// The im2col GEMM (stz_tma.cuh, IM2COL_MN) fetches the input once per tap:
// 9 boxes of the same pixels per k-block, which made this the least
// efficient GEMM of the step (profiles/r01/op/conv0_wgrad_*: 2.2 GB of TMA
// reads for 176 MB of operands).  Here every output raster row y of image n
// is one stage: dY row (n, y) -- Wv = rup16(OW) virtual pixels, TMA zero-fills
// the columns past OW -- and, for the stage's tap row dh, input row
// (n, y + dh) with Wv + ks - 1 (+ 1) pixels.  Both are SWIZZLE_128B rows of
// 64 channels (128 B).  In the MN-major view (M = channels, K = pixels) the
// taps (dh, dw) of one tap row are the input row shifted by dw rows, and two
// taps form one 128-row A operand: start = row dw, LBO = 128 B (the second
// 64-channel group starts one pixel later).  SWIZZLE_128B descriptors may
// start at any 128-byte row with base offset 0 (tools/swz_check.cu).
//
// Work item = (tap row dh, split z): split z covers the output raster rows
// [j0, j1) of the N*OH rows; all tap rows of one split run in the same wave
// (dY shared in L2).  Per item the CTA accumulates ceil(ks/2) tap-pair tiles
// over its rows, then the epilogue writes its tap rows of the split's
// partial [576][64]; the fixed-order split reduce applies EpConvWgradS2D
// (deterministic).  BF16x6 with the thin-tile schedule of stz_tma.cuh: the
// dY planes b0 | b1 are one 128-wide MN-major operand (LBO = plane stride),
// so each 16-deep step is 4 MMAs -- a0.b2 -> S2, a0.[b0|b1] -> [big|S1],
// a1.[b0|b1] -> [S1|S2], a2.b0 -> S1 (every accumulator's first write an
// overwrite) -- instead of 6, and the epilogue adds big + (S1 + S2).  The
// N = 64 MMAs are bound by their shared-memory operand reads, which this
// cuts by a fifth.  TMEM: 2 tiles x 192 columns.
#pragma once

#include "stz_band.cuh"

namespace stz {

struct alignas(64) BandWParams {
  CUtensorMap x[3];   // per plane: 4D [N][Hs][Ws][CW], box {CW, XW, 1, 1}, SWIZZLE_(2 CW)B
  CUtensorMap g[3];   // per plane: 4D [N][OH][OW][64], box {64, Wv, 1, 1}, SWIZZLE_128B
  float* partial;     // [splits][ks*ks*CW][64]
  int N, OH, ks, Wv, XW;
  int splits, rows_total;   // N * OH output raster rows
  int nst;                  // pipeline stages (2..BW_STAGES: wide rows fit fewer)
  FastDiv d_oh;
  int debug;  // diagnostics only (stz_set_debug): 1 skip partial stores, 2 skip MMAs, 4 skip TMA
};

constexpr int BW_THREADS = 256;
constexpr int BW_STAGES = 4;

// CW = input channels per pixel row: 64 (SWIZZLE_128B rows, two taps per
// 128-row A operand: AlexNet conv1) or 32 (SWIZZLE_64B rows, four taps per
// operand: ResNet-50's 7x7/2 stem as 4x4 taps over 12 of 32 channels)
__host__ __device__ inline int bw_xplane(int XW, int CW = 64) {
  return (XW * 2 * CW + 1023) / 1024 * 1024;
}
__host__ __device__ inline int bw_gplane(int Wv) { return Wv * 128; }
__host__ __device__ inline int bw_stage(int XW, int Wv, int CW = 64) {
  return 3 * (bw_xplane(XW, CW) + bw_gplane(Wv));
}
__host__ inline size_t bw_smem(int XW, int Wv, int nst = BW_STAGES, int CW = 64) {
  return 1024 + (size_t)nst * bw_stage(XW, Wv, CW) + 256;
}

template <int CW>
__global__ void __launch_bounds__(BW_THREADS, 1) bandwgrad_kernel(const __grid_constant__ BandWParams p) {
  constexpr int ACC = 192;                 // big | S1 | S2, 64 columns each
  constexpr int TPT = 128 / CW;            // taps per 128-row A operand
  constexpr int TILES = (4 + TPT - 1) / TPT;   // ceil(ks / TPT) for ks <= 4
  constexpr int SET = TILES * ACC;         // columns of one set
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  uint8_t* smem = smem_raw + (base - raw);
  const int XP = bw_xplane(p.XW, CW), GP = bw_gplane(p.Wv), STG = bw_stage(p.XW, p.Wv, CW);
  const int NST = p.nst;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + NST * STG);
  uint64_t* empty = full + NST;
  uint64_t* tfull = empty + NST;    // [2]
  uint64_t* tempty = tfull + 2;           // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ks = p.ks;
  const int items = ks * p.splits;
  auto rows_of = [&](int z, int& j0, int& j1) {
    j0 = (int)((long long)p.rows_total * z / p.splits);
    j1 = (int)((long long)p.rows_total * (z + 1) / p.splits);
  };

  if (threadIdx.x == 0) {
    for (int s = 0; s < NST; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(&tfull[0], 1);
    mbar_init(&tempty[0], 4);
    mbar_fence_init();
  }
  if (warp == 0 && lane < 3) {
    prefetch_tmap(&p.x[lane]);
    prefetch_tmap(&p.g[lane]);
  }
  if (warp == 2) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ---------------- TMA producer: one stage per output raster row ------------------
    const uint32_t tx = (uint32_t)(3 * (2 * CW * p.XW + 128 * p.Wv));
    int gs = 0;
    for (int w = blockIdx.x; w < items; w += gridDim.x) {
      const int z = w / ks, dh = w - z * ks;
      int j0, j1;
      rows_of(z, j0, j1);
      for (int j = j0; j < j1; ++j, ++gs) {
        const int s = gs % NST;
        mbar_wait(&empty[s], ((gs / NST) & 1) ^ 1);
        if (p.debug & 4) {
          if (lane == 0) mbar_arrive(&full[s]);
          __syncwarp();
          continue;
        }
        if (lane == 0) mbar_arrive_tx(&full[s], tx);
        __syncwarp();
        uint32_t n, y;
        p.d_oh.divmod((uint32_t)j, n, y);
        const uint32_t st = base + s * STG;
        if (lane < 6) {
          const bool isx = lane < 3;
          const int pl = isx ? lane : lane - 3;
          const uint32_t dst = st + (isx ? pl * XP : 3 * XP + pl * GP);
          const CUtensorMap* map = isx ? &p.x[pl] : &p.g[pl];
          const int row = isx ? (int)y + dh : (int)y;
          asm volatile(
              "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
              " [%0], [%1, {%3, %4, %5, %6}], [%2];" ::"r"(dst),
              "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(&full[s])), "r"(0), "r"(0),
              "r"(row), "r"((int)n)
              : "memory");
        }
      }
    }
  } else if (warp == 1 && lane == 0) {
    // ---------------- MMA issuer ---------------------------------------------------
    const uint32_t idesc64 = sg_idesc(TG_BM, 64, true, true);    // A, B MN-major
    const uint32_t idesc128 = sg_idesc(TG_BM, 128, true, true);  // B = [b0 | b1]
    const int ksteps = p.Wv / 16;
    int gs = 0, it = 0;
    for (int w = blockIdx.x; w < items; w += gridDim.x, ++it) {
      const int z = w / ks;
      int j0, j1;
      rows_of(z, j0, j1);
      mbar_wait(&tempty[0], (it & 1) ^ 1);
      tc_fence_after();
      for (int j = j0; j < j1; ++j, ++gs) {
        const int s = gs % NST;
        mbar_wait(&full[s], (gs / NST) & 1);
        tc_fence_after();
        const uint32_t st = base + s * STG;
        const uint32_t b0 = st + 3 * XP;
        for (int kq = 0; kq < ksteps && !(p.debug & 2); ++kq) {
          const uint32_t acc = (j == j0 && kq == 0) ? 0u : 1u;
          const uint64_t db0 = umma_desc_sw128(b0 + kq * 2048, GP, 1024);          // [b0|b1]
          const uint64_t db2 = umma_desc_sw128(b0 + 2 * GP + kq * 2048, GP, 1024);  // b2
#pragma unroll
          for (int tile = 0; tile < TILES; ++tile) {
            if (TPT * tile >= ks) break;
            // A plane a: input rows (TPT tile) + 16 kq ..; each further tap one row on
            const uint32_t arow = st + (uint32_t)(TPT * tile + 16 * kq) * (2 * CW);
            const uint64_t da0 = CW == 64 ? umma_desc_sw128(arow, 128, 1024)
                                          : umma_desc_sw64(arow, 64, 512);
            const uint64_t da1 = CW == 64 ? umma_desc_sw128(arow + XP, 128, 1024)
                                          : umma_desc_sw64(arow + XP, 64, 512);
            const uint64_t da2 = CW == 64 ? umma_desc_sw128(arow + 2 * XP, 128, 1024)
                                          : umma_desc_sw64(arow + 2 * XP, 64, 512);
            const uint32_t tbig = tmem_base + tile * ACC, ts1 = tbig + 64, ts2 = tbig + 128;
            umma_f16(ts2, da0, db2, idesc64, acc);     // a0.b2 -> S2
            umma_f16(tbig, da0, db0, idesc128, acc);   // a0.[b0|b1] -> big, S1
            umma_f16(ts1, da1, db0, idesc128, 1u);     // a1.[b0|b1] -> S1, S2
            umma_f16(ts1, da2, db0, idesc64, 1u);      // a2.b0 -> S1
          }
        }
        umma_commit(&empty[s]);
      }
      umma_commit(&tfull[0]);
    }
  } else if (warp >= 4) {
    // ---------------- epilogue: tap rows of the split's partial ---------------------
    const int q = warp & 3;
    const int r = q * 32 + lane;                 // accumulator row = (tap in tile, channel)
    const int mrows = ks * ks * CW;
    int it = 0;
    for (int w = blockIdx.x; w < items; w += gridDim.x, ++it) {
      const int z = w / ks, dh = w - z * ks;
      mbar_wait_backoff(&tfull[0], it & 1);
      tc_fence_after();
#pragma unroll 1
      for (int tile = 0; tile < TILES; ++tile) {
        if (TPT * tile >= ks) break;
        const int dw = TPT * tile + r / CW;
        const bool valid = dw < ks;
        const int m = (dh * ks + dw) * CW + (r % CW);
        const uint32_t tb = tmem_base + ((uint32_t)(q * 32) << 16) + tile * ACC;
#pragma unroll 1
        for (int c = 0; c < 64; c += 16) {
          uint32_t a[16], b[16], d[16];
          tmem_ld16(tb + (uint32_t)c, a);
          tmem_ld16(tb + 64 + (uint32_t)c, b);
          tmem_ld16(tb + 128 + (uint32_t)c, d);
          tmem_ld_wait();
          if (!valid || m >= mrows || (p.debug & 1)) continue;
          float4* dst = reinterpret_cast<float4*>(p.partial + ((size_t)z * mrows + m) * 64 + c);
#pragma unroll
          for (int h = 0; h < 4; ++h) {
            float v[4];
#pragma unroll
            for (int e = 0; e < 4; ++e)
              v[e] = __fadd_rn(__uint_as_float(a[4 * h + e]),
                               __fadd_rn(__uint_as_float(b[4 * h + e]), __uint_as_float(d[4 * h + e])));
            dst[h] = make_float4(v[0], v[1], v[2], v[3]);
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[0]);
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem_base, 512);
  }
}

}  // namespace stz
