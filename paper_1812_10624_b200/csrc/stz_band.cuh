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
// The band sits in shared memory K-major with the 64-byte SWIZZLE_64B
// pattern TMA writes for a {32 channels, Wp, Hb} box: one 64-byte row per
// virtual input row, 8-row atoms of 512 B.  The swizzle is a function of
// the absolute shared-memory address (descriptor base offset 0), so a
// descriptor may start at ANY 64-byte row: tap (th, tw) is the band at row
// offset th*Wi + tw, and every core matrix stays one aligned 16-byte chunk
// per row (tools/swz_check.cu checks tcgen05.mma on shifted SW64 / SW128
// views against a CPU reference; round 1's non-swizzled band paid a second
// shared-memory wavefront for every shift that was not a multiple of 8).
// TMA fills it with one 4D box per plane.

// Padding needs no padded copy: the band is loaded with a 4D TMA tiled box
// {8 channels, Wp = W + 2*pad columns, Hb rows, 1 image} at (-pad, y0 - pad);
// out-of-range coordinates are zero-filled, so shared memory holds exactly
// the padded image rows.  Work items tile each image's valid output rows
// (virtual rows q = y * Wp + x, y < OH); the junk columns x >= OW are
// computed and dropped by the epilogue.  Input gradients are the same conv
// over the output gradient padded by k-1-p, with flipped weights.  Weights
// are the im2col GEMM's B operand ([N][k*k][C8] K-major, TILED_K boxes).
// Split-K runs over channel blocks (fp32 partials + the fixed-order reduce).
//
// The band pays where the im2col GEMM is feed-bound and the junk rows are
// few: the unpadded space-to-depth conv1 (images stacked into one raster,
// ~7% junk).  Padded convs (per-image tiling, 23%+ junk) measured slower
// than im2col with the old non-swizzled band, so the host enables the band
// for pad == 0 unless stz_set_band(2).
#pragma once

#include "stz_tma.cuh"

namespace stz {

template <class EP>
struct alignas(64) BandParams {
  CUtensorMap band[3];   // per plane: 4D [N][H][W][C8], box {32, Wp, Hb, 1}, SWIZZLE_64B
  TgOperand b;           // weights, TILED_K
  CUtensorMap b3;        // weights as one 3D map {K, O, plane}: a stage's three planes in one box
  int use_b3;
  EP ep;
  float* partial;        // split-K partials [splits][M_out][npad] (nullptr: no split)
  int N;                 // GEMM N (output channels)
  int C8;                // input channels (multiple of 32)
  int exact;             // stacked raster only: the band is exactly the rows a tile reads,
  int brows, nbx;        //   nbx 2D boxes of brows pixels each (else whole padded rows)
  int creal;             // channels < creal are real: 16-deep k steps past it are skipped
  int cblocks;           // 32-channel blocks holding real channels (cdiv(creal, 32))
  int Nimg, pad, Wp, ksz, OH, OW;
  int Nreal, Hs;         // stacked mode (pad 0): Nimg = 1 image of Nreal * Hs rows
  FastDiv d_hs;
  int tiles_per_img;     // ceil(OH * Wp / (MT * 128))
  int Hb;                // padded rows per band
  int cb_per_split, splits;
  FastDiv d_wp;
  int debug;
};

constexpr int BD_THREADS = 256;

template <int BN, int MT, bool THIN_ = false>
struct BandCfg {
  static constexpr int B_PLANE = BN * TG_BK * 2;          // one plane of a B tile
  static constexpr int B_STAGE = 3 * B_PLANE;
  static constexpr int STAGES = (BN <= 64 && (MT == 2 || THIN_)) ? 4 : 3;
  // thin tiles: the 4-MMA schedule of stz_tma.cuh -- weight planes b0 | b1
  // (contiguous) as one 128-wide operand; accumulators big | S1 | S2.  Off:
  // with MT = 2 its 384 columns leave one TMEM set, and the serialised
  // epilogue cost more than the saved MMAs (conv1 forward 0.232 -> 0.287 ms,
  // measured); with MT = 1 the weight tile per 128 rows doubles the weight
  // feed (STZ_BAND_THIN=1 selects MT = 1 with the thin schedule).
  static constexpr bool THIN = THIN_;
  static constexpr int ACC_COLS = THIN ? 3 * BN : 2 * BN;
  static constexpr int SET_COLS = MT * ACC_COLS;
  static constexpr int NSETS = 2 * SET_COLS <= 512 ? 2 : 1;
  static constexpr int TMEM_COLS = NSETS * SET_COLS <= 256 ? 256 : 512;
  static_assert(NSETS * SET_COLS <= 512, "band tile too wide for TMEM");
  static_assert(B_PLANE % 512 == 0, "B planes must stay 512-byte aligned");
};

// band geometry: each plane holds Hb * Wp rows of 64 B (32 channels), padded
// to a multiple of 8 rows (planes stay 512-byte aligned: whole swizzle
// atoms); the two bands are followed by the 1024-byte aligned weight stages
__host__ __device__ inline int band_rows_alloc(int Hb, int Wp) { return (Hb * Wp + 7) / 8 * 8; }
__host__ __device__ inline int band_bytes(int rows_alloc) { return 3 * 4 * rows_alloc * 16; }
__host__ __device__ inline int band_region(int rows_alloc) {
  return (2 * band_bytes(rows_alloc) + 1023) / 1024 * 1024;
}

template <int BN, int MT, bool THIN = false>
__host__ inline int band_smem(int rows_alloc) {
  using Cfg = BandCfg<BN, MT, THIN>;
  return 1024 + band_region(rows_alloc) + Cfg::STAGES * Cfg::B_STAGE + 512;
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

template <int BN, int MT, class EP, bool THIN = false>
__global__ void __launch_bounds__(BD_THREADS, 1)
    bandconv_kernel(const __grid_constant__ BandParams<EP> p) {
  using Cfg = BandCfg<BN, MT, THIN>;
  constexpr int STAGES = Cfg::STAGES, NSETS = Cfg::NSETS;
  constexpr int TM = MT * TG_BM;   // virtual rows per work item
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t smem_base = (raw + 1023u) & ~1023u;
  uint8_t* smem = smem_raw + (smem_base - raw);
  const int rows_alloc = p.exact ? p.nbx * p.brows : band_rows_alloc(p.Hb, p.Wp);
  const int BAND = band_bytes(rows_alloc);
  const int PLANE = rows_alloc * 64;
  const int REGION = band_region(rows_alloc);
  const uint32_t band0 = smem_base;                          // [2] bands
  const uint32_t bst0 = band0 + REGION;                      // [STAGES] B tiles
  uint64_t* band_full = reinterpret_cast<uint64_t*>(smem + REGION + STAGES * Cfg::B_STAGE);
  uint64_t* band_empty = band_full + 2;
  uint64_t* b_full = band_empty + 2;
  uint64_t* b_empty = b_full + STAGES;
  uint64_t* tfull = b_empty + STAGES;    // [2]
  uint64_t* tempty = tfull + 2;          // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nt = cdiv(p.N, BN);
  const int per_split = p.Nimg * p.tiles_per_img * nt;
  const int items = per_split * p.splits;
  const int cblocks = p.cblocks, taps = p.ksz * p.ksz;
  // item w -> (split z, image n, tile t, n tile); n fastest so tiles share the band in L2
  auto decode = [&](int w, int& z, int& n, int& t, int& n0) {
    z = w / per_split;
    const int r = w - z * per_split;
    n0 = (r % nt) * BN;
    const int it = r / nt;
    n = it / p.tiles_per_img;
    t = it - n * p.tiles_per_img;
  };

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
    const uint32_t band_tx = (uint32_t)(p.exact ? 3 * p.nbx * p.brows * 64   // bytes the boxes land
                                                : 3 * p.Hb * p.Wp * 64);
    int gb = 0, gs = 0;
    for (int w = blockIdx.x; w < items; w += gridDim.x) {
      int z, n, t, n0;
      decode(w, z, n, t, n0);
      const int y0 = (t * TM) / p.Wp;
      const int cb0 = z * p.cb_per_split, cb1 = min(cblocks, cb0 + p.cb_per_split);
      for (int cb = cb0; cb < cb1; ++cb, ++gb) {
        const int bb = gb & 1;
        mbar_wait(&band_empty[bb], ((gb >> 1) & 1) ^ 1);
        if (p.debug & 4) {   // diagnostics: no data movement
          if (lane == 0) mbar_arrive(&band_full[bb]);
        } else if (lane == 0) {
          mbar_arrive_tx(&band_full[bb], band_tx);
        }
        __syncwarp();
        if (p.exact) {   // raster rows t*TM .. as nbx boxes per plane
          if (lane < 3 * p.nbx && !(p.debug & 4)) {
            const int pl = lane % 3, bi = lane / 3;
            const uint32_t dst = band0 + bb * BAND + pl * PLANE + bi * p.brows * 64;
            asm volatile(
                "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
                " [%0], [%1, {%3, %4, %5, %6}], [%2];" ::"r"(dst),
                "l"(reinterpret_cast<uint64_t>(&p.band[pl])), "r"(smem_u32(&band_full[bb])),
                "r"(cb * 32), "r"(t * TM + bi * p.brows), "r"(0), "r"(0)
                : "memory");
          }
        } else if (lane < 3 && !(p.debug & 4)) {   // one 4D box per plane: padded rows y0 .. y0+Hb-1
          const int pl = lane;
          const uint32_t dst = band0 + bb * BAND + pl * PLANE;
          asm volatile(
              "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
              " [%0], [%1, {%3, %4, %5, %6}], [%2];" ::"r"(dst),
              "l"(reinterpret_cast<uint64_t>(&p.band[pl])), "r"(smem_u32(&band_full[bb])),
              "r"(cb * 32), "r"(-p.pad), "r"(y0 - p.pad), "r"(n)
              : "memory");
        }
        for (int tp = 0; tp < taps; ++tp, ++gs) {
          const int s = gs % STAGES;
          mbar_wait(&b_empty[s], ((gs / STAGES) & 1) ^ 1);
          if (p.debug & 4) {
            if (lane == 0) mbar_arrive(&b_full[s]);
            __syncwarp();
            continue;
          }
          if (lane == 0) mbar_arrive_tx(&b_full[s], Cfg::B_STAGE);
          __syncwarp();
          const uint32_t st = bst0 + s * Cfg::B_STAGE;
          if (p.use_b3) {   // TMA cost is per box: the three planes as one {32, BN, 3} box
            if (lane == 0) tma_3d<1>(&p.b3, st, &b_full[s], tp * p.C8 + cb * 32, n0, 0);
          } else {
            for (int bi = lane; bi < 3 * p.b.nbox; bi += 32)
              tg_load_box<1>(p.b, bi, st, Cfg::B_PLANE, &b_full[s], n0, tp * p.C8 + cb * 32);
          }
        }
      }
    }
  } else if (warp == 1 && lane == 0) {
    // ---------------- MMA issuer --------------------------------------------------
    const uint32_t idesc = sg_idesc(TG_BM, BN, false, false);
    const uint32_t idesc2 = sg_idesc(TG_BM, 2 * BN, false, false);   // thin: B = [b0|b1]
    constexpr int AP[6] = {0, 2, 1, 0, 1, 0};
    constexpr int BP[6] = {2, 0, 1, 1, 0, 0};
    const uint64_t da0 = umma_desc_sw64(band0, 16, 512);
    const uint64_t db0 = tg_desc(TG_TILED_K, bst0, 0);
    int gb = 0, gs = 0, it = 0;
    for (int w = blockIdx.x; w < items; w += gridDim.x, ++it) {
      int z, n, t, n0;
      decode(w, z, n, t, n0);
      // band row of the tile's first output
      const uint32_t x0 = p.exact ? 0u : (uint32_t)((t * TM) % p.Wp);
      const int cb0 = z * p.cb_per_split, cb1 = min(cblocks, cb0 + p.cb_per_split);
      const int set = NSETS == 2 ? (it & 1) : 0;
      const int use = NSETS == 2 ? (it >> 1) : it;
      mbar_wait(&tempty[set], (use & 1) ^ 1);
      tc_fence_after();
      const uint32_t tset = tmem_base + set * Cfg::SET_COLS;
      for (int cb = cb0; cb < cb1; ++cb, ++gb) {
        const int bb = gb & 1;
        mbar_wait(&band_full[bb], (gb >> 1) & 1);
        tc_fence_after();
        for (int tp = 0; tp < taps; ++tp, ++gs) {
          const int s = gs % STAGES;
          mbar_wait(&b_full[s], (gs / STAGES) & 1);
          tc_fence_after();
          const int th = tp / p.ksz, tw = tp - th * p.ksz;
          const uint32_t shift = x0 + (uint32_t)(th * p.Wp + tw);
          const uint32_t sb = (uint32_t)(s * Cfg::B_STAGE) >> 4;
#pragma unroll
          for (int j = 0; j < 2; ++j) {
            if ((p.debug & 2) || cb * 32 + j * 16 >= p.creal) break;   // padded channels: zeros
#pragma unroll
            for (int mt = 0; mt < MT; ++mt) {
              // 16-byte units: 64-byte rows, the j-th 16-deep k step 32 B in
              const uint32_t arow = (uint32_t)(bb * BAND) / 16 + (mt * TG_BM + shift) * 4 + j * 2;
              const uint32_t tbig = tset + mt * Cfg::ACC_COLS, tsmall = tbig + BN;
              if constexpr (Cfg::THIN) {
                const uint32_t acc = (cb == cb0 && (tp | j) == 0) ? 0u : 1u;
                const uint64_t da_0 = da0 + arow;
                const uint64_t da_1 = da0 + (arow + (uint32_t)PLANE / 16);
                const uint64_t da_2 = da0 + (arow + (uint32_t)(2 * PLANE) / 16);
                const uint64_t db01 = db0 + (sb + j * 2);                             // [b0|b1]
                const uint64_t db_2 = db0 + (sb + 2 * (Cfg::B_PLANE >> 4) + j * 2);   // b2
                umma_f16(tsmall + BN, da_0, db_2, idesc, acc);   // a0.b2 -> S2
                umma_f16(tbig, da_0, db01, idesc2, acc);         // a0.[b0|b1] -> big, S1
                umma_f16(tsmall, da_1, db01, idesc2, 1u);        // a1.[b0|b1] -> S1, S2
                umma_f16(tsmall, da_2, db0 + (sb + j * 2), idesc, 1u);   // a2.b0 -> S1
              } else {
#pragma unroll
                for (int i = 0; i < 6; ++i) {
                  const uint64_t da = da0 + (arow + (uint32_t)(AP[i] * PLANE) / 16);
                  const uint64_t db = db0 + (sb + BP[i] * (Cfg::B_PLANE >> 4) + j * 2);
                  const bool big = i == 5;
                  const bool first = cb == cb0 && (tp | j) == 0 && (big || i == 0);
                  umma_f16(big ? tbig : tsmall, da, db, idesc, first ? 0u : 1u);
                }
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
    const int M_out = p.Nreal * p.OH * p.OW;
    int it = 0;
    for (int w = blockIdx.x; w < items; w += gridDim.x, ++it) {
      int z, n, t, n0;
      decode(w, z, n, t, n0);
      const int set = NSETS == 2 ? (it & 1) : 0;
      const int use = NSETS == 2 ? (it >> 1) : it;
      mbar_wait_backoff(&tfull[set], use & 1);
      tc_fence_after();
#pragma unroll 1
      for (int mt = 0; mt < MT; ++mt) {
        const int vq = t * TM + mt * TG_BM + q * 32 + lane;   // virtual row within image n
        uint32_t ya, x, ns, y;
        p.d_wp.divmod((uint32_t)vq, ya, x);
        p.d_hs.divmod(ya, ns, y);        // stacked images: (image, row); else ns = 0
        const int nr = n + (int)ns;
        const bool valid = nr < p.Nreal && (int)y < p.OH && (int)x < p.OW;
        const int m = valid ? (nr * p.OH + (int)y) * p.OW + (int)x : M_out;
        const uint32_t tbase = tmem_base + ((uint32_t)(q * 32) << 16) + set * Cfg::SET_COLS +
                               mt * Cfg::ACC_COLS;
#pragma unroll 1
        for (int c = 0; c < BN; c += 32) {
          if (n0 + c >= npad || (p.debug & 8)) break;
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
          if constexpr (Cfg::THIN) {     // small = S1 + S2
            uint32_t r2[32];
            tmem_ld16(tbase + 2 * BN + (uint32_t)c, *reinterpret_cast<uint32_t(*)[16]>(&r2[0]));
            tmem_ld16(tbase + 2 * BN + (uint32_t)c + 16, *reinterpret_cast<uint32_t(*)[16]>(&r2[16]));
            tmem_ld_wait();
#pragma unroll
            for (int e = 0; e < 32; ++e)
              rs[e] = __float_as_uint(__fadd_rn(__uint_as_float(rs[e]), __uint_as_float(r2[e])));
          }
          tmem_ld_wait();
          if constexpr (EP::STAGED) {
            // split-plane output: 16 columns per lane and plane as one 256-bit
            // store (whole sectors; the row-per-lane stores of 16 bytes kept
            // the LSU busy at half-sector granularity)
            if (!p.partial && !(p.debug & 1)) {
#pragma unroll
              for (int h2 = 0; h2 < 2; ++h2) {
                const int nb = n0 + c + 16 * h2;
                if (nb >= npad) break;
                float v[16];
#pragma unroll
                for (int jj = 0; jj < 16; ++jj) {
                  v[jj] = __fadd_rn(__uint_as_float(r[16 * h2 + jj]),
                                    __uint_as_float(rs[16 * h2 + jj]));
                  if (EP::HAS_BIAS) v[jj] = __fadd_rn(v[jj], bb[2 * h2 + jj / 8][jj % 8]);
                }
                if (valid) p.ep.store16_nb(m, nb, v);
              }
              continue;
            }
          }
#pragma unroll
          for (int h = 0; h < 4; ++h) {
            const int nb = n0 + c + 8 * h;
            if (nb >= npad) break;
            float v[8];
#pragma unroll
            for (int jj = 0; jj < 8; ++jj) {
              v[jj] = __fadd_rn(__uint_as_float(r[8 * h + jj]), __uint_as_float(rs[8 * h + jj]));
              if (EP::HAS_BIAS && !p.partial) v[jj] = __fadd_rn(v[jj], bb[h][jj]);
            }
            if (p.debug & 1) continue;
            if (p.partial) {
              if (valid) {
                float4* dst =
                    reinterpret_cast<float4*>(p.partial + ((size_t)z * M_out + m) * npad + nb);
                dst[0] = make_float4(v[0], v[1], v[2], v[3]);
                dst[1] = make_float4(v[4], v[5], v[6], v[7]);
              }
            } else {
              p.ep.store8_nb(m, nb, v);
            }
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
