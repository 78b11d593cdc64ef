// Shifted-window ("band") implicit GEMM for stride-1 convolutions.
//
// The im2col GEMM (stz_tma.cuh) loads its A tile once per (tap, channel
// block): a k x k conv re-fetches every input pixel k^2 times through L2,
// which makes the thin / small-tile conv GEMMs bound by the L2 -> SM operand
// feed (profiles/r01/SUMMARY.md).  Here the output rows are the input's own
// raster: virtual row q = (n, y, x) over the [N][Hi][Wi] input grid, and tap
// (th, tw) of output q reads input row q + th*Wi + tw.  So for MT x 128
// consecutive output rows one BAND of MT*128 + (k-1)*Wi + (k-1) input rows
// serves all k^2 taps of a 32-channel block: each tap is the same band
// addressed at a row offset.
//
// The band sits in shared memory non-swizzled and K-major, with the rows of
// each 8-channel chunk contiguous (16 B per row): core matrices of 8 rows x
// 16 B, SBO = 128 B, LBO = rows * 16 B.  A descriptor may then start at any
// 16-byte row offset (tools/band_check.cu verifies tcgen05.mma against a CPU
// reference at shifts 0..127).  TMA fills it with 16-byte-wide boxes of up to
// 256 rows per (plane, chunk).
//
// The convolution is "valid" over a (pre-padded) input: output (y, x) for
// y < Hi-k+1, x < Wi-k+1; the other virtual rows (the last k-1 columns and
// rows of each image) are computed and dropped by the epilogue.  Weights are
// the im2col GEMM's B operand ([N][k*k][C8] K-major, TILED_K boxes).
#pragma once

#include "stz_tma.cuh"

namespace stz {

template <class EP>
struct alignas(64) BandParams {
  CUtensorMap band[3];   // per plane: 2D [N*Hi*Wi rows][C8], box {8, box_rows}, no swizzle
  TgOperand b;           // weights, TILED_K
  EP ep;
  int M_virt;            // N * Hi * Wi
  int N;                 // GEMM N (output channels)
  int C8;                // input channels (multiple of 32)
  int Wi, ksz, OH, OW, Nimg;
  int box_rows, nrb, rows_alloc;   // band: nrb boxes of box_rows rows per (plane, chunk)
  FastDiv d_hw, d_w;
  int debug;
};

constexpr int BD_THREADS = 256;

template <int BN, int MT>
struct BandCfg {
  static constexpr int B_PLANE = BN * TG_BK * 2;          // one plane of a B tile
  static constexpr int B_STAGE = 3 * B_PLANE;
  static constexpr int STAGES = BN <= 64 ? 4 : 3;
  static constexpr int ACC_COLS = 2 * BN;                // big + small per M tile
  static constexpr int SET_COLS = MT * ACC_COLS;
  static constexpr int NSETS = 2 * SET_COLS <= 512 ? 2 : 1;
  static constexpr int TMEM_COLS = NSETS * SET_COLS <= 256 ? 256 : 512;
  static_assert(NSETS * SET_COLS <= 512, "band tile too wide for TMEM");
  static_assert(B_PLANE % 512 == 0, "B planes must stay 512-byte aligned");
};

// bytes of one band buffer (3 planes x 4 chunks x rows_alloc x 16 B)
__host__ __device__ inline int band_bytes(int rows_alloc) { return 3 * 4 * rows_alloc * 16; }

template <int BN, int MT>
__host__ inline int band_smem(int rows_alloc) {
  using Cfg = BandCfg<BN, MT>;
  return 1024 + 2 * band_bytes(rows_alloc) + Cfg::STAGES * Cfg::B_STAGE + 512;
}

// non-swizzled K-major descriptor (layout type 0)
__device__ __forceinline__ uint64_t umma_desc_none(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;
  return d;
}

template <int BN, int MT, class EP>
__global__ void __launch_bounds__(BD_THREADS, 1)
    bandconv_kernel(const __grid_constant__ BandParams<EP> p) {
  using Cfg = BandCfg<BN, MT>;
  constexpr int STAGES = Cfg::STAGES, NSETS = Cfg::NSETS;
  constexpr int TM = MT * TG_BM;   // virtual rows per work item
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t smem_base = (raw + 1023u) & ~1023u;
  uint8_t* smem = smem_raw + (smem_base - raw);
  const int BAND = band_bytes(p.rows_alloc);
  const int PLANE = 4 * p.rows_alloc * 16, CHUNK = p.rows_alloc * 16;
  const uint32_t band0 = smem_base;                          // [2] bands
  const uint32_t bst0 = band0 + 2 * BAND;                    // [STAGES] B tiles
  uint64_t* band_full = reinterpret_cast<uint64_t*>(smem + 2 * BAND + STAGES * Cfg::B_STAGE);
  uint64_t* band_empty = band_full + 2;
  uint64_t* b_full = band_empty + 2;
  uint64_t* b_empty = b_full + STAGES;
  uint64_t* tfull = b_empty + STAGES;    // [2]
  uint64_t* tempty = tfull + 2;          // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int mt_items = cdiv(p.M_virt, TM), nt = cdiv(p.N, BN);
  const int items = mt_items * nt;
  const int cblocks = p.C8 / 32, taps = p.ksz * p.ksz;

  if (threadIdx.x == 0) {
    for (int i = 0; i < 2; ++i) {
      mbar_init(&band_full[i], 1);
      mbar_init(&band_empty[i], 1);
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], 4);
    }
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&b_full[s], 1);
      mbar_init(&b_empty[s], 1);
    }
    mbar_fence_init();
  }
  if (warp == 0 && lane < 3) {
    prefetch_tmap(&p.band[lane]);
    prefetch_tmap(&p.b.map[lane]);
  }
  if (warp == 2) tmem_alloc(tmem_slot, Cfg::TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ---------------- TMA producer --------------------------------------------
    const int nbox = 3 * 4 * p.nrb;
    const uint32_t band_tx = (uint32_t)(nbox * p.box_rows * 16);
    int gb = 0, gs = 0;
    for (int w = blockIdx.x; w < items; w += gridDim.x) {
      const int q0 = (w / nt) * TM, n0 = (w % nt) * BN;
      for (int cb = 0; cb < cblocks; ++cb, ++gb) {
        const int bb = gb & 1;
        mbar_wait(&band_empty[bb], ((gb >> 1) & 1) ^ 1);
        if (lane == 0) mbar_arrive_tx(&band_full[bb], band_tx);
        __syncwarp();
        for (int i = lane; i < nbox; i += 32) {
          const int pl = i / (4 * p.nrb), c = (i / p.nrb) % 4, rb = i % p.nrb;
          const uint32_t dst = band0 + bb * BAND + pl * PLANE + c * CHUNK + rb * p.box_rows * 16;
          tma_2d<1>(&p.band[pl], dst, &band_full[bb], cb * 32 + c * 8, q0 + rb * p.box_rows);
        }
        for (int t = 0; t < taps; ++t, ++gs) {
          const int s = gs % STAGES;
          mbar_wait(&b_empty[s], ((gs / STAGES) & 1) ^ 1);
          if (lane == 0) mbar_arrive_tx(&b_full[s], Cfg::B_STAGE);
          __syncwarp();
          const uint32_t st = bst0 + s * Cfg::B_STAGE;
          for (int bi = lane; bi < 3 * p.b.nbox; bi += 32)
            tg_load_box<1>(p.b, bi, st, Cfg::B_PLANE, &b_full[s], n0, t * p.C8 + cb * 32);
        }
      }
    }
  } else if (warp == 1 && lane == 0) {
    // ---------------- MMA issuer --------------------------------------------------
    const uint32_t idesc = sg_idesc(TG_BM, BN, false, false);
    constexpr int AP[6] = {0, 2, 1, 0, 1, 0};
    constexpr int BP[6] = {2, 0, 1, 1, 0, 0};
    const uint64_t da0 = umma_desc_none(band0, (uint32_t)CHUNK, 128);
    const uint64_t db0 = tg_desc(TG_TILED_K, bst0, 0);
    int gb = 0, gs = 0, it = 0;
    for (int w = blockIdx.x; w < items; w += gridDim.x, ++it) {
      const int set = NSETS == 2 ? (it & 1) : 0;
      const int use = NSETS == 2 ? (it >> 1) : it;
      mbar_wait(&tempty[set], (use & 1) ^ 1);
      tc_fence_after();
      const uint32_t tset = tmem_base + set * Cfg::SET_COLS;
      for (int cb = 0; cb < cblocks; ++cb, ++gb) {
        const int bb = gb & 1;
        mbar_wait(&band_full[bb], (gb >> 1) & 1);
        tc_fence_after();
        for (int t = 0; t < taps; ++t, ++gs) {
          const int s = gs % STAGES;
          mbar_wait(&b_full[s], (gs / STAGES) & 1);
          tc_fence_after();
          const int th = t / p.ksz, tw = t - th * p.ksz;
          const uint32_t shift = (uint32_t)(th * p.Wi + tw);
          const uint32_t sb = (uint32_t)(s * Cfg::B_STAGE) >> 4;
#pragma unroll
          for (int j = 0; j < 2; ++j) {
            if (p.debug & 2) break;
#pragma unroll
            for (int mt = 0; mt < MT; ++mt) {
              const uint32_t arow = (uint32_t)(bb * BAND + 2 * j * CHUNK) / 16 + mt * TG_BM + shift;
              const uint32_t tbig = tset + mt * Cfg::ACC_COLS, tsmall = tbig + BN;
#pragma unroll
              for (int i = 0; i < 6; ++i) {
                const uint64_t da = da0 + (arow + (uint32_t)(AP[i] * PLANE) / 16);
                const uint64_t db = db0 + (sb + BP[i] * (Cfg::B_PLANE >> 4) + j * 2);
                const bool big = i == 5;
                const bool first = (cb | t | j) == 0 && (big || i == 0);
                umma_f16(big ? tbig : tsmall, da, db, idesc, first ? 0u : 1u);
              }
            }
          }
          umma_commit(&b_empty[s]);
        }
        umma_commit(&band_empty[bb]);
      }
      umma_commit(&tfull[set]);
    }
  } else if (warp >= 4) {
    // ---------------- epilogue: virtual rows -> output rows -----------------------
    const int q = warp & 3;
    const int npad = cdiv(p.N, 8) * 8;
    const int M_out = p.Nimg * p.OH * p.OW;
    int it = 0;
    for (int w = blockIdx.x; w < items; w += gridDim.x, ++it) {
      const int q0 = (w / nt) * TM, n0 = (w % nt) * BN;
      const int set = NSETS == 2 ? (it & 1) : 0;
      const int use = NSETS == 2 ? (it >> 1) : it;
      mbar_wait(&tfull[set], use & 1);
      tc_fence_after();
#pragma unroll 1
      for (int mt = 0; mt < MT; ++mt) {
        const int vq = q0 + mt * TG_BM + q * 32 + lane;
        uint32_t n, rem, y, x;
        p.d_hw.divmod((uint32_t)vq, n, rem);
        p.d_w.divmod(rem, y, x);
        const bool valid = vq < p.M_virt && (int)y < p.OH && (int)x < p.OW;
        const int m = valid ? ((int)n * p.OH + (int)y) * p.OW + (int)x : M_out;
        const uint32_t tbase = tmem_base + ((uint32_t)(q * 32) << 16) + set * Cfg::SET_COLS +
                               mt * Cfg::ACC_COLS;
#pragma unroll 1
        for (int c = 0; c < BN; c += 32) {
          if (n0 + c >= npad) break;
          float bb[4][8];
          if (EP::HAS_BIAS) {
#pragma unroll
            for (int q4 = 0; q4 < 4; ++q4) p.ep.bias8(n0 + c + 8 * q4, bb[q4]);
          }
          uint32_t r[32], rs[32];
          tmem_ld16(tbase + (uint32_t)c, *reinterpret_cast<uint32_t(*)[16]>(&r[0]));
          tmem_ld16(tbase + (uint32_t)c + 16, *reinterpret_cast<uint32_t(*)[16]>(&r[16]));
          tmem_ld16(tbase + BN + (uint32_t)c, *reinterpret_cast<uint32_t(*)[16]>(&rs[0]));
          tmem_ld16(tbase + BN + (uint32_t)c + 16, *reinterpret_cast<uint32_t(*)[16]>(&rs[16]));
          tmem_ld_wait();
#pragma unroll
          for (int h = 0; h < 4; ++h) {
            const int nb = n0 + c + 8 * h;
            if (nb >= npad) break;
            float v[8];
#pragma unroll
            for (int jj = 0; jj < 8; ++jj) {
              v[jj] = __fadd_rn(__uint_as_float(r[8 * h + jj]), __uint_as_float(rs[8 * h + jj]));
              if (EP::HAS_BIAS) v[jj] = __fadd_rn(v[jj], bb[h][jj]);
            }
            if (!(p.debug & 1)) p.ep.store8_nb(m, nb, v);
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[set]);
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem_base, Cfg::TMEM_COLS);
  }
}

}  // namespace stz
