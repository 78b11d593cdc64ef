// TMA-fed tcgen05 GEMM for split-plane operands (the main hot-path kernel).
//
// Round-1 profiling of the cp.async version (stz_split.cuh) showed the conv
// GEMMs L1tex-bound (82-95% of L1tex throughput, tensor pipe 14-27%): every
// 16-byte gather is an LSU request.  Here every operand tile moves L2 -> smem
// through the Tensor Memory Accelerator, one elected thread issuing
// cp.async.bulk.tensor per plane:
//
//   TILED_K   2D [rows][K] (K contiguous)       box {32 K, R rows}  -> K-major
//   TILED_MN  2D [K][rows] (rows contiguous)    box {32 rows, 32 K} -> MN-major
//   IM2COL_K  4D NHWC im2col, pixels = rows     32 channels x 128 pixels (conv fwd / dgrad A)
//   IM2COL_MN 4D NHWC im2col, pixels = K        32 channels x 32 pixels  (conv wgrad A)
//
// All boxes land with the 64-byte swizzle (BK = 32 bf16 = one 64-byte row);
// the UMMA shared-memory descriptors use the matching SWIZZLE_64B canonical
// layouts:
//   K-major : 8-row x 64 B atoms, SBO = 512 B, K step of 16 = +32 B
//   MN-major: 32-element x 8-k-row atoms, LBO = 2048 B between 32-element
//             MN groups, SBO = 512 B between 8-k-row groups, K step of 16 =
//             +1024 B.
// Out-of-range rows / pixels / channels are zero-filled by TMA.  The
// BF16x6 MMA schedule, the two TMEM accumulators and the epilogues are the
// ones of stz_split.cuh.
#pragma once

#include <cuda.h>

#include "stz_split.cuh"

namespace stz {

enum TgMode : int { TG_TILED_K = 0, TG_TILED_MN = 1, TG_IM2COL_K = 2, TG_IM2COL_MN = 3 };

struct alignas(64) TgOperand {
  CUtensorMap map[3];  // one per plane
  int mode;
  int nbox;            // boxes per plane per k-block
  int box_bytes;       // smem bytes per box (2048 for 32-wide MN boxes)
  int box_rows;        // TILED_K: rows per box (a B tile split between 2 CTAs)
  int mn3d;            // TILED_MN: the tile is one 3D box (rows % 32 == 0)
  int sw128;           // IM2COL_MN: 64-channel boxes with the 128-byte swizzle (C8 % 64 == 0)
  // im2col geometry: output pixel (n, oh, ow) -> window start (oh*s + lo_h, ow*s + lo);
  // taps (th, tw) = divmod(tap, ksz) with ksz = the kernel width
  int lo, s, C8, ksz, flip, lo_h;
  FastDiv d_ohw, d_ow, d_c8, d_k;
  // TILED_K tap remap (the weights of one phase of a strided conv's input
  // gradient): K index (tap', o) with tap' = (th', tw') over a sub-kernel of
  // width r_tw reads column (r_base + th' r_sh + tw' r_sw) * r_o8 + o
  int remap, r_base, r_sh, r_sw;
  FastDiv d_ro8, d_rtw;
};

template <class EP>
struct alignas(64) TgParams {
  TgOperand a, b;
  EP ep;
  float* partial;
  // split-K fixup counters (one per 128-row half tile, zero between launches):
  // the last split of a tile to finish sums every split's partial in split
  // order and applies the epilogue, so no separate reduce pass runs
  int* sem;
  int M, N, K, k_per_split;
  int debug;  // bench/diagnostics only: 1 skip epilogue stores, 2 skip MMAs, 4 skip TMA loads
  int epi_direct;   // split-plane epilogue: 256-bit per-row stores instead of smem staging
};

constexpr int TG_BM = 128, TG_BK = 32;
constexpr int TG_THREADS = 384;  // w0 TMA (32 lanes), w1 MMA, w2 TMEM alloc, w3 idle, w4-11 epilogue
constexpr int TG_EC = 16;        // epilogue columns per TMEM load round

// CL = 1: one CTA per 128 x BN tile.  CL = 2: a CTA pair computes a 256 x BN
// tile with cta_group::2 UMMA -- each CTA stages its own 128 A rows and HALF
// of B (BN / 2 rows), so per-SM operand traffic per MMA cycle drops by
// 1 - (128 + BN/2) / (128 + BN): the split-plane GEMMs are bound by the
// L2 -> SM operand feed (3 planes per operand), not by the tensor pipe.
// MH = 2 (unpaired only): one CTA computes TWO 128-row halves of a 256 x BN
// tile against the same B stage -- one 256-row A box per plane (TMA cost is
// per box: tools/tma_bench.cu) and B fetched once for both halves; each half
// has its own TMEM accumulators (MH * NSETS * ACC_COLS <= 512).
template <int BN, int NSETS = 2, int CL = 1, int MH = 1>
struct TgCfg {
  static_assert(MH == 1 || (CL == 1 && BN == 64), "two M halves: thin unpaired tiles only");
  static constexpr int A_BYTES = TG_BM * MH * TG_BK * 2;   // one plane, 8 KB per half
  static constexpr int B_ROWS = BN / CL;                    // B rows staged by this CTA
  static constexpr int B_BYTES = B_ROWS * TG_BK * 2;
  static constexpr int STAGE_BYTES = 3 * (A_BYTES + B_BYTES);
  static constexpr int STAGES = (200 * 1024) / STAGE_BYTES > 8 ? 8 : (200 * 1024) / STAGE_BYTES;
  // epilogue staging (STAGED epilogues): per epilogue warp, 32 rows x 16
  // columns of the three bf16 planes, so global stores go out row-contiguous
  static constexpr int EPI_WARP_BYTES = 3 * 32 * 32;
  static constexpr int EPI_BYTES = 8 * EPI_WARP_BYTES;
  static constexpr int SMEM = STAGES * STAGE_BYTES + EPI_BYTES + 1024 + 512;  // + slack + barriers
  // NSETS accumulator sets (2 = double-buffered across tiles), each = big + small.
  // PAIRB (thin unpaired tiles): the B planes b0 | b1 are contiguous, so they
  // act as one 128-wide operand -- 4 MMAs per 16-k (2 at N=128, 2 at N=64)
  // instead of 6 at N=64; the products land in big + two small accumulators.
  static constexpr bool PAIRB = BN == 64 && CL == 1;
  static constexpr int ACC_COLS = PAIRB ? 3 * BN : 2 * BN;
  static constexpr int TMEM_COLS = MH * NSETS * ACC_COLS <= 256 ? 256 : 512;
  static_assert(MH * NSETS * ACC_COLS <= 512, "BN too wide for the TMEM sets");
  static_assert(STAGES >= 3, "tile too large");
  static_assert(B_BYTES % 512 == 0, "B plane blocks must stay 512-byte aligned (SW64 atoms)");
};

__device__ __forceinline__ void mbar_arrive_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile(
      "{\n\t.reg .b64 st;\n\t"
      "mbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n\t}" ::"r"(smem_u32(bar)),
      "r"(bytes)
      : "memory");
}

// the leader (even) CTA's copy of a barrier of this CTA (shared::cluster address)
__device__ __forceinline__ uint32_t leader_bar(const uint64_t* bar) {
  return smem_u32(bar) & 0xFEFFFFFFu;
}

// CL = 2 loads complete on the LEADER's full barrier (cta_group::2 form)
template <int CL>
__device__ __forceinline__ void tma_2d(const CUtensorMap* map, uint32_t dst, uint64_t* bar,
                                       int c0, int c1) {
  if (CL == 2)
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4}], [%2];" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(leader_bar(bar)), "r"(c0), "r"(c1)
        : "memory");
  else
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4}], [%2];" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
        : "memory");
}

// 3D tiled box {32 elements, 32 K rows, g 32-element groups}: an MN-major tile
// of 32 g rows in ONE TMA instruction (the box lands as g consecutive 2 KB
// SW64 atoms -- the layout of g separate 2D boxes).  TMA cost is per box, so
// fewer, larger boxes feed faster (tools/tma_bench.cu: 2 KB boxes ~21
// B/cycle/SM, 8 KB ~41, 16 KB ~60 from L2).
template <int CL>
__device__ __forceinline__ void tma_3d(const CUtensorMap* map, uint32_t dst, uint64_t* bar,
                                       int c0, int c1, int c2) {
  if (CL == 2)
    asm volatile(
        "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(leader_bar(bar)), "r"(c0), "r"(c1), "r"(c2)
        : "memory");
  else
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
        : "memory");
}

__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}

__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;"
               ::: "memory");
}

// ---- cta_group::2 (CTA pair) tcgen05 forms --------------------------------------
__device__ __forceinline__ void umma_f16_pair(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                              uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

// arrive on the barrier at this offset in both CTAs of the pair once the
// pair's outstanding MMAs complete
__device__ __forceinline__ void umma_commit_pair(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
      " [%0], %1;" ::"r"(smem_u32(bar)),
      "h"((uint16_t)0x3)
      : "memory");
}

__device__ __forceinline__ void tmem_alloc_pair(uint32_t* slot, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                   smem_u32(slot)),
               "r"(ncols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
}

__device__ __forceinline__ void tmem_dealloc_pair(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols)
               : "memory");
}

// arrive on the leader CTA's copy of `bar`
__device__ __forceinline__ void mbar_arrive_leader(uint64_t* bar) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(
                   leader_bar(bar))
               : "memory");
}

template <int CL>
__device__ __forceinline__ void tma_im2col_4d(const CUtensorMap* map, uint32_t dst, uint64_t* bar,
                                              int c, int w, int h, int n, uint16_t ow,
                                              uint16_t oh) {
  if (CL == 2)
    asm volatile(
        "cp.async.bulk.tensor.4d.im2col.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4, %5, %6}], [%2], {%7, %8};" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(leader_bar(bar)), "r"(c), "r"(w), "r"(h),
        "r"(n), "h"(ow), "h"(oh)
        : "memory");
  else
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.im2col.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4, %5, %6}], [%2], {%7, %8};" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c), "r"(w), "r"(h),
        "r"(n), "h"(ow), "h"(oh)
        : "memory");
}

__device__ __forceinline__ void prefetch_tmap(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}

// SWIZZLE_64B UMMA descriptor (layout type 4)
__device__ __forceinline__ uint64_t umma_desc_sw64(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)4 << 61;
  return d;
}

// issue box `bi` (0 <= bi < 3*nbox) of one operand tile: plane = bi / nbox,
// box = bi % nbox (R rows starting at r0, K block starting at k0)
template <int CL>
__device__ __forceinline__ void tg_load_box(const TgOperand& op, int bi, uint32_t tile_base,
                                            uint32_t plane_bytes, uint64_t* bar, int r0, int k0) {
  const int plane = bi / op.nbox, box = bi - plane * op.nbox;
  const CUtensorMap* map = &op.map[plane];
  const uint32_t dst = tile_base + plane * plane_bytes + box * op.box_bytes;
  switch (op.mode) {
    case TG_TILED_K:
      if (op.remap) {
        uint32_t tap, o0, th, tw;
        op.d_ro8.divmod((uint32_t)k0, tap, o0);
        op.d_rtw.divmod(tap, th, tw);
        k0 = (op.r_base + (int)th * op.r_sh + (int)tw * op.r_sw) * (int)op.d_ro8.d + (int)o0;
      }
      tma_2d<CL>(map, dst, bar, k0, r0 + box * op.box_rows);
      break;
    case TG_TILED_MN:
      if (op.mn3d)   // one box for the whole tile: {32, 32 K, R/32 groups}
        tma_3d<CL>(map, dst, bar, 0, k0, r0 >> 5);
      else
        tma_2d<CL>(map, dst, bar, r0 + 32 * box, k0);
      break;
    case TG_IM2COL_K: {
      uint32_t n, j, oh, ow, tap, c0, th, tw;
      op.d_ohw.divmod((uint32_t)r0, n, j);
      op.d_ow.divmod(j, oh, ow);
      op.d_c8.divmod((uint32_t)k0, tap, c0);
      op.d_k.divmod(tap, th, tw);
      tma_im2col_4d<CL>(map, dst, bar, (int)c0, (int)(ow * op.s) + op.lo,
                        (int)(oh * op.s) + op.lo_h, (int)n, (uint16_t)tw, (uint16_t)th);
      break;
    }
    default: {  // TG_IM2COL_MN: k0 = first output pixel, rows = (tap, c)
      uint32_t n, j, oh, ow, tap, c0, th, tw;
      op.d_ohw.divmod((uint32_t)k0, n, j);
      op.d_ow.divmod(j, oh, ow);
      op.d_c8.divmod((uint32_t)(r0 + (op.sw128 ? 64 : 32) * box), tap, c0);
      op.d_k.divmod(tap, th, tw);
      tma_im2col_4d<CL>(map, dst, bar, (int)c0, (int)(ow * op.s) + op.lo,
                        (int)(oh * op.s) + op.lo_h, (int)n, (uint16_t)tw, (uint16_t)th);
    }
  }
}

// SWIZZLE_128B UMMA descriptor (layout type 2): MN-major 64-element x 8-k-row
// atoms of 1 KB; LBO = bytes between 64-element MN groups, SBO = 1 KB
__device__ __forceinline__ uint64_t umma_desc_sw128(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (umma_desc_sw64(saddr, lbo, sbo) & ~((uint64_t)7 << 61)) | ((uint64_t)2 << 61);
}

__device__ __forceinline__ uint64_t tg_desc(int mode, uint32_t plane_base, int kstep,
                                            int sw128 = 0) {
  const bool mn = mode == TG_TILED_MN || mode == TG_IM2COL_MN;
  if (mn && sw128) return umma_desc_sw128(plane_base + kstep * 2048, 4096, 1024);
  return mn ? umma_desc_sw64(plane_base + kstep * 1024, 2048, 512)
            : umma_desc_sw64(plane_base + kstep * 32, 16, 512);
}

// Persistent: grid = min(#work items, #SMs); work item w -> (split z, m tile,
// n tile), n fastest so consecutive items share the A tile in L2.  TMEM holds
// NSETS accumulator sets; with 2 the epilogue of item i overlaps the mainloop
// of item i+1.
// CL = 2 (cluster of 2 = one CTA pair per 256-row tile): rank r stages A rows
// m0 + 128 r and B rows n0 + r BN/2; both CTAs' loads complete on the leader's
// full barrier (expect_tx = both stages); the leader's single MMA thread
// issues cta_group::2 MMAs that read both CTAs' smem and write both CTAs'
// TMEM (each holds its 128 rows x BN); its commits arrive on the empty / tfull
// barriers of both CTAs; both epilogues release the set on the leader's
// tempty barrier (8 warp arrivals).
template <int BN, int NSETS, int CL, class EP, int MH = 1>
__global__ void __launch_bounds__(TG_THREADS, 1)
    tgemm_kernel(const __grid_constant__ TgParams<EP> p) {
  using Cfg = TgCfg<BN, NSETS, CL, MH>;
  constexpr int STAGES = Cfg::STAGES;
  constexpr int PM = TG_BM * CL * MH;   // rows per work item
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t smem_base = (raw + 1023u) & ~1023u;
  uint8_t* smem = smem_raw + (smem_base - raw);
  const uint32_t epi_smem = smem_base + STAGES * Cfg::STAGE_BYTES;
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + STAGES * Cfg::STAGE_BYTES + Cfg::EPI_BYTES);
  uint64_t* empty_bar = full_bar + STAGES;
  uint64_t* tfull_bar = empty_bar + STAGES;   // [2] accumulator set ready for the epilogue
  uint64_t* tempty_bar = tfull_bar + 2;       // [2] accumulator set drained
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty_bar + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int mt = cdiv(p.M, PM), nt = cdiv(p.N, BN);
  const int splits = cdiv(p.K, p.k_per_split);
  const int items = mt * nt * splits;
  const int rank = CL == 2 ? (int)cluster_ctarank() : 0;
  const int cid = blockIdx.x / CL, ncl = gridDim.x / CL;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull_bar[a], 1);
      mbar_init(&tempty_bar[a], 8 * CL);   // one arrival per epilogue warp of the pair
    }
    mbar_fence_init();
  }
  if (warp == 0 && lane < 3) {
    prefetch_tmap(&p.a.map[lane]);
    prefetch_tmap(&p.b.map[lane]);
  }
  if (warp == 2) {
    if (CL == 2) tmem_alloc_pair(tmem_slot, Cfg::TMEM_COLS);
    else tmem_alloc(tmem_slot, Cfg::TMEM_COLS);
  }
  tc_fence_before();
  __syncthreads();
  if (CL == 2) cluster_sync_all();   // the peer's barriers / TMEM exist before any traffic
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ---------------- TMA producer: the warp's lanes issue boxes in parallel --
    const int na = 3 * p.a.nbox, nbx = 3 * p.b.nbox;
    int g = 0;  // global k-block counter (stage / phase)
    for (int w = cid; w < items; w += ncl) {
      const int z = w / (mt * nt), rem = w % (mt * nt);
      const int m0 = (rem / nt) * PM + rank * TG_BM;
      const int n0 = (rem % nt) * BN + rank * Cfg::B_ROWS;
      const int kbeg = z * p.k_per_split, kend = min(p.K, kbeg + p.k_per_split);
      const int nkb = cdiv(kend - kbeg, TG_BK);
      for (int kb = 0; kb < nkb; ++kb, ++g) {
        const int stage = g % STAGES;
        mbar_wait(&empty_bar[stage], ((g / STAGES) & 1) ^ 1);
        if (p.debug & 4) {   // diagnostics: no data movement
          if (lane == 0 && rank == 0) mbar_arrive(&full_bar[stage]);
          __syncwarp();
          continue;
        }
        if (lane == 0 && rank == 0) mbar_arrive_tx(&full_bar[stage], CL * Cfg::STAGE_BYTES);
        __syncwarp();
        const int k0 = kbeg + kb * TG_BK;
        const uint32_t st = smem_base + stage * Cfg::STAGE_BYTES;
        for (int bi = lane; bi < na + nbx; bi += 32) {
          if (bi < na)
            tg_load_box<CL>(p.a, bi, st, Cfg::A_BYTES, &full_bar[stage], m0, k0);
          else
            tg_load_box<CL>(p.b, bi - na, st + 3 * Cfg::A_BYTES, Cfg::B_BYTES, &full_bar[stage],
                            n0, k0);
        }
      }
    }
    if (CL == 2 && lane == 0) {
      // drain: every multicast release of our stages has landed before exit
      for (int k = 0; k < STAGES; ++k, ++g) mbar_wait(&empty_bar[g % STAGES], ((g / STAGES) & 1) ^ 1);
    }
  } else if (warp == 1 && lane == 0 && rank == 0) {
    // ---------------- MMA issuer (the leader CTA for a pair) --------------------
    const bool amn = p.a.mode == TG_TILED_MN || p.a.mode == TG_IM2COL_MN;
    const bool bmn = p.b.mode == TG_TILED_MN || p.b.mode == TG_IM2COL_MN;
    const uint32_t idesc = sg_idesc(TG_BM * CL, BN, amn, bmn);
    constexpr int AP[6] = {0, 2, 1, 0, 1, 0};
    constexpr int BP[6] = {2, 0, 1, 1, 0, 0};
    // descriptors of stage 0 / plane 0 / k-step 0; every other (stage, plane,
    // k-step) only moves the 14-bit start-address field (addresses < 256 KB,
    // so the add never carries out of it): two integer adds per MMA
    const uint64_t da0 = tg_desc(p.a.mode, smem_base, 0, p.a.sw128);
    const uint64_t db0 = tg_desc(p.b.mode, smem_base + 3 * Cfg::A_BYTES, 0);
    const uint32_t ak = (amn ? (p.a.sw128 ? 2048u : 1024u) : 32u) >> 4,
                   bk = (bmn ? 1024u : 32u) >> 4;
    int g = 0, it = 0;
    for (int w = cid; w < items; w += ncl, ++it) {
      const int z = w / (mt * nt);
      const int kbeg = z * p.k_per_split, kend = min(p.K, kbeg + p.k_per_split);
      const int nkb = cdiv(kend - kbeg, TG_BK);
      const int acc = NSETS == 2 ? (it & 1) : 0;
      const int use = NSETS == 2 ? (it >> 1) : it;   // how often this set was used before
      mbar_wait(&tempty_bar[acc], (use & 1) ^ 1);
      tc_fence_after();
      const uint32_t tbig = tmem_base + acc * Cfg::ACC_COLS, tsmall = tbig + BN;
      for (int kb = 0; kb < nkb; ++kb, ++g) {
        const int stage = g % STAGES;
        mbar_wait(&full_bar[stage], (g / STAGES) & 1);
        tc_fence_after();
        const uint32_t so = (uint32_t)(stage * Cfg::STAGE_BYTES) >> 4;
        if constexpr (Cfg::PAIRB) {
          // big (cols 0..63) | S1 (64..127) | S2 (128..191):
          //   a0*b2 -> S2;  a0*[b0|b1] -> big, S1;  a1*[b0|b1] -> S1, S2;  a2*b0 -> S1
          // (ordered so that every accumulator's first write is an overwrite)
          const uint32_t idesc2 = sg_idesc(TG_BM, 2 * BN, amn, bmn);
#pragma unroll
          for (int j = 0; j < TG_BK / 16; ++j) {
            if (p.debug & 2) break;
            const uint32_t acc_in = (kb | j) == 0 ? 0u : 1u;
            const uint64_t b0d = db0 + (so + j * bk), b2d = b0d + 2 * (Cfg::B_BYTES >> 4);
#pragma unroll
            for (int h = 0; h < MH; ++h) {   // half h: A rows 128 h.., TMEM set h
              const uint32_t th = tbig + h * Cfg::ACC_COLS;
              const uint32_t tS1 = th + BN, tS2 = th + 2 * BN;
              const uint64_t a0d = da0 + (so + j * ak + h * ((TG_BM * TG_BK * 2) >> 4));
              const uint64_t a1d = a0d + (Cfg::A_BYTES >> 4), a2d = a0d + 2 * (Cfg::A_BYTES >> 4);
              umma_f16(tS2, a0d, b2d, idesc, acc_in);
              umma_f16(th, a0d, b0d, idesc2, acc_in);
              umma_f16(tS1, a1d, b0d, idesc2, 1u);
              umma_f16(tS1, a2d, b0d, idesc, 1u);
            }
          }
        } else {
#pragma unroll
        for (int j = 0; j < TG_BK / 16; ++j) {
          if (p.debug & 2) break;
#pragma unroll
          for (int i = 0; i < 6; ++i) {
            const uint64_t da = da0 + (so + AP[i] * (Cfg::A_BYTES >> 4) + j * ak);
            const uint64_t db = db0 + (so + BP[i] * (Cfg::B_BYTES >> 4) + j * bk);
            const bool big = i == 5;
            const bool first = (kb | j) == 0 && (big || i == 0);
            if (CL == 2) umma_f16_pair(big ? tbig : tsmall, da, db, idesc, first ? 0u : 1u);
            else umma_f16(big ? tbig : tsmall, da, db, idesc, first ? 0u : 1u);
          }
        }
        }
        if (CL == 2) umma_commit_pair(&empty_bar[stage]);
        else umma_commit(&empty_bar[stage]);
      }
      if (CL == 2) umma_commit_pair(&tfull_bar[acc]);
      else umma_commit(&tfull_bar[acc]);
    }
  } else if (warp >= 4) {
    // ---------------- epilogue: TMEM (big + small) -> registers -> ep ---------
    // 8 warps: warp w reads TMEM lanes 32 (w % 4) .. (its row quadrant) and
    // takes every other 16-column chunk (two warps per SM sub-partition, so
    // one's TMEM / memory latency hides behind the other's arithmetic)
    const int q = warp & 3, half = (warp - 4) >> 2;
    const int npad = cdiv(p.N, 8) * 8;
    int it = 0;
    for (int w = cid; w < items; w += ncl, ++it) {
      const int z = w / (mt * nt), rem = w % (mt * nt);
      const int m0 = (rem / nt) * PM + rank * TG_BM, n0 = (rem % nt) * BN;
      const int acc = NSETS == 2 ? (it & 1) : 0;
      const int use = NSETS == 2 ? (it >> 1) : it;
      mbar_wait_backoff(&tfull_bar[acc], use & 1);
      tc_fence_after();
#pragma unroll 1
      for (int h = 0; h < MH; ++h) {
      const int m = m0 + h * TG_BM + q * 32 + lane;
      const uint32_t tbase = tmem_base + ((uint32_t)(q * 32) << 16) + (acc + h) * Cfg::ACC_COLS;
#pragma unroll 1
      for (int c = half * TG_EC; c < BN; c += 2 * TG_EC) {
        if (n0 + c >= npad) break;
        // bias first (independent of TMEM), then 16 columns of big + small, one wait
        float bb[2][8];
        if (EP::HAS_BIAS && !p.partial) {
          p.ep.bias8(n0 + c, bb[0]);
          p.ep.bias8(n0 + c + 8, bb[1]);
        }
        uint32_t r[16], rs[16], rs2[16];
        tmem_ld16(tbase + (uint32_t)c, r);
        tmem_ld16(tbase + BN + (uint32_t)c, rs);
        if constexpr (Cfg::PAIRB) tmem_ld16(tbase + 2 * BN + (uint32_t)c, rs2);
        tmem_ld_wait();
        float v[2][8];
#pragma unroll
        for (int hh = 0; hh < 2; ++hh)
#pragma unroll
          for (int jj = 0; jj < 8; ++jj) {
            float sm = __uint_as_float(rs[8 * hh + jj]);
            if constexpr (Cfg::PAIRB) sm = __fadd_rn(sm, __uint_as_float(rs2[8 * hh + jj]));
            v[hh][jj] = __fadd_rn(__uint_as_float(r[8 * hh + jj]), sm);
          }
        if (p.debug & 1) continue;
        if (p.partial) {
#pragma unroll
          for (int hh = 0; hh < 2; ++hh) {
            const int nb = n0 + c + 8 * hh;
            if (m < p.M && nb < npad) {
              float* dst = p.partial + ((size_t)z * p.M + m) * npad + nb;
              if ((reinterpret_cast<uintptr_t>(dst) & 31) == 0) {
                stg256(dst, v[hh]);
              } else {
                reinterpret_cast<float4*>(dst)[0] = make_float4(v[hh][0], v[hh][1], v[hh][2], v[hh][3]);
                reinterpret_cast<float4*>(dst)[1] = make_float4(v[hh][4], v[hh][5], v[hh][6], v[hh][7]);
              }
            }
          }
          continue;
        }
        if (EP::HAS_BIAS) {
#pragma unroll
          for (int hh = 0; hh < 2; ++hh)
#pragma unroll
            for (int jj = 0; jj < 8; ++jj) v[hh][jj] = __fadd_rn(v[hh][jj], bb[hh][jj]);
        }
        if constexpr (EP::STAGED) {
          if (p.epi_direct) {   // each lane: its row's 16 columns, one 256-bit store per plane
            float v16[16];
#pragma unroll
            for (int jj = 0; jj < 8; ++jj) {
              v16[jj] = v[0][jj];
              v16[8 + jj] = v[1][jj];
            }
            p.ep.store16_nb(m, n0 + c, v16);
            continue;
          }
          // split planes of 32 rows x 16 columns through shared memory: each
          // lane writes its row's two 16-byte chunks per plane (slot XOR row
          // bit 2: conflict-free), then two lanes store one row's 32
          // contiguous bytes (one full sector) per plane, 16 rows per
          // instruction
          const uint32_t sb = epi_smem + (uint32_t)(warp - 4) * Cfg::EPI_WARP_BYTES;
#pragma unroll
          for (int hh = 0; hh < 2; ++hh) {
            p.ep.prep8(n0 + c + 8 * hh, v[hh]);
            uint32_t w0[4], w1[4], w2[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              bf16_t a0, a1, a2, c0, c1, c2;
              split_bf16x3(v[hh][2 * j], a0, a1, a2);
              split_bf16x3(v[hh][2 * j + 1], c0, c1, c2);
              w0[j] = (uint32_t)a0 | ((uint32_t)c0 << 16);
              w1[j] = (uint32_t)a1 | ((uint32_t)c1 << 16);
              w2[j] = (uint32_t)a2 | ((uint32_t)c2 << 16);
            }
            const uint32_t o = (uint32_t)lane * 32 + (uint32_t)((hh ^ (lane >> 2)) & 1) * 16;
            sts128u(sb + o, w0[0], w0[1], w0[2], w0[3]);
            sts128u(sb + 1024 + o, w1[0], w1[1], w1[2], w1[3]);
            sts128u(sb + 2048 + o, w2[0], w2[1], w2[2], w2[3]);
          }
          __syncwarp();
#pragma unroll
          for (int i = 0; i < 2; ++i) {
            const int rr = 16 * i + (lane >> 1), ch = lane & 1;
            const uint32_t o = (uint32_t)rr * 32 + (uint32_t)((ch ^ (rr >> 2)) & 1) * 16;
            const int mrow = m0 + h * TG_BM + q * 32 + rr, nb = n0 + c + 8 * ch;
            if (mrow < p.M && nb < npad) {
              uint4 pl[3];
              pl[0] = lds128(sb + o);
              pl[1] = lds128(sb + 1024 + o);
              pl[2] = lds128(sb + 2048 + o);
              p.ep.store_planes(mrow, nb, pl);
            }
          }
          __syncwarp();
        } else {
#pragma unroll
          for (int hh = 0; hh < 2; ++hh) {
            const int nb = n0 + c + 8 * hh;
            if (nb < npad) p.ep.store8_nb(m, nb, v[hh]);
          }
        }
      }
      }   // halves
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if (CL == 2) mbar_arrive_leader(&tempty_bar[acc]);
        else mbar_arrive(&tempty_bar[acc]);
      }
      if (p.partial && p.sem && !(p.debug & 1)) {
        // split-K fixup: publish this split's partial, count it; the tile's
        // last split reads all partials back (L2) and runs the epilogue
        __shared__ int s_last;
        const int splits = cdiv(p.K, p.k_per_split);
        int* cnt = p.sem + rem * CL + rank;
        __threadfence();
        asm volatile("bar.sync 1, 256;" ::: "memory");
        if (warp == 4 && lane == 0) s_last = atomicAdd(cnt, 1) == splits - 1;
        asm volatile("bar.sync 1, 256;" ::: "memory");
        if (s_last) {
          __threadfence();
          const size_t zs = (size_t)p.M * npad;
#pragma unroll 1
          for (int h = 0; h < MH; ++h) {
            const int m = m0 + h * TG_BM + q * 32 + lane;
#pragma unroll 1
            for (int c = half * TG_EC; c < BN; c += 2 * TG_EC) {
              if (n0 + c >= npad) break;
              // 16 columns x 4 splits of loads in flight per step, adds in split order
              const int nb = n0 + c;
              if (m >= p.M) continue;
              const bool two = nb + 8 < npad;
              const float* src = p.partial + (size_t)m * npad + nb;
              float v[2][8];
              for (int z0 = 0; z0 < splits; z0 += 4) {
                float4 ld[4][4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                  if (z0 + u < splits) {
                    const float4* q4 = reinterpret_cast<const float4*>(src + (size_t)(z0 + u) * zs);
                    ld[u][0] = __ldcg(q4);
                    ld[u][1] = __ldcg(q4 + 1);
                    ld[u][2] = two ? __ldcg(q4 + 2) : make_float4(0.f, 0.f, 0.f, 0.f);
                    ld[u][3] = two ? __ldcg(q4 + 3) : make_float4(0.f, 0.f, 0.f, 0.f);
                  }
                }
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                  if (z0 + u >= splits) break;
                  const float w[2][8] = {{ld[u][0].x, ld[u][0].y, ld[u][0].z, ld[u][0].w,
                                          ld[u][1].x, ld[u][1].y, ld[u][1].z, ld[u][1].w},
                                         {ld[u][2].x, ld[u][2].y, ld[u][2].z, ld[u][2].w,
                                          ld[u][3].x, ld[u][3].y, ld[u][3].z, ld[u][3].w}};
#pragma unroll
                  for (int hh = 0; hh < 2; ++hh)
#pragma unroll
                    for (int j = 0; j < 8; ++j)
                      v[hh][j] = (z0 + u == 0) ? w[hh][j] : __fadd_rn(v[hh][j], w[hh][j]);
                }
              }
              p.ep.store8(m, nb, v[0]);
              if (two) p.ep.store8(m, nb + 8, v[1]);
            }
          }
          if (warp == 4 && lane == 0) *cnt = 0;   // re-armed for the next launch
        }
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (CL == 2) cluster_sync_all();   // no pair traffic may target us after exit
  if (warp == 2) {
    tc_fence_after();
    if (CL == 2) tmem_dealloc_pair(tmem_base, Cfg::TMEM_COLS);
    else tmem_dealloc(tmem_base, Cfg::TMEM_COLS);
  }
}

}  // namespace stz
