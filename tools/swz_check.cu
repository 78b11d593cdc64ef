// Probe: can a SWIZZLE_128B UMMA operand start at any 128-byte row of a
// swizzled band (a conv tap as a shifted view), and what does the
// descriptor's base-offset field (bits 49-51) have to say?
//
// The band is R rows x 128 B (64 bf16) at a 1024-byte aligned base, written
// with the SW128 pattern (16-byte chunk j of row r at chunk j ^ (r & 7)) --
// what TMA writes for a {64, R} box.  Two views are checked against a CPU
// reference with tcgen05.mma kind::f16 (M=128, N=64, K=16):
//   KM: K-major A (rows = M, K = the 64 columns): start = base + s*128 (+ k0*2)
//       -- the forward conv band (pixels = rows of A);
//   MN: MN-major A (rows = K, M = the 64 columns, two 64-wide M groups
//       LBO = D*128 bytes apart): start = base + s*128 -- the weight-gradient
//       band (pixels = K, two taps D pixels apart as one 128-row A).
// For each shift s the base offset is tried as 0 and as s & 7.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -o swz_check tools/swz_check.cu
#include <cuda_bf16.h>
#include <cstdint>
#include <cstdio>
#include <vector>

constexpr int R = 256, N = 64, K = 16, M = 128;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ uint64_t desc_sw128(uint32_t saddr, uint32_t lbo, uint32_t sbo,
                                               uint32_t base_off) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;                    // sm100 descriptor version
  d |= (uint64_t)(base_off & 7) << 49;
  d |= (uint64_t)2 << 61;                    // SWIZZLE_128B
  return d;
}

__device__ __forceinline__ uint64_t desc_sw64(uint32_t saddr, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)1 << 16;                    // LBO (unused for swizzled K-major)
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)4 << 61;                    // SWIZZLE_64B
  return d;
}

__device__ __forceinline__ uint64_t desc_none(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;
  return d;
}

// mode 0: KM, mode 1: MN.  a_g: band [R][64] row-major (logical), b_g: [N][K]
__global__ void probe(const __nv_bfloat16* a_g, const __nv_bfloat16* b_g, int mode, int shift,
                      int k0, int dgap, int boff, float* d_g) {
  __shared__ __align__(1024) uint8_t sm[R * 128 + N * K * 2];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const uint32_t abase = smem_u32(sm), bbase = abase + R * 128;
  if (mode == 2) {   // SW64: rows of 32 bf16 (64 B); 16-byte chunk j at j ^ ((r >> 1) & 3)
    for (int i = threadIdx.x; i < R * 32; i += blockDim.x) {
      const int r = i / 32, c = i % 32;
      const int chunk = (c / 8) ^ ((r >> 1) & 3);
      *reinterpret_cast<__nv_bfloat16*>(sm + r * 64 + chunk * 16 + (c % 8) * 2) = a_g[r * 64 + c];
    }
  } else {
    for (int i = threadIdx.x; i < R * 64; i += blockDim.x) {
      const int r = i / 64, c = i % 64;
      const int chunk = (c / 8) ^ (r & 7);
      *reinterpret_cast<__nv_bfloat16*>(sm + r * 128 + chunk * 16 + (c % 8) * 2) = a_g[i];
    }
  }
  for (int i = threadIdx.x; i < N * K; i += blockDim.x) {
    const int n = i / K, k = i % K;
    *reinterpret_cast<__nv_bfloat16*>(sm + R * 128 + (k / 8) * (N * 16) + n * 16 + (k % 8) * 2) =
        b_g[i];
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 64;" ::"r"(
        smem_u32(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = slot;
  if (threadIdx.x == 0) {
    uint64_t da;
    uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) |
                     ((uint32_t)(M >> 4) << 24);
    if (mode == 0) {
      da = desc_sw128(abase + shift * 128 + k0 * 2, 16, 1024, boff);
    } else if (mode == 2) {
      da = desc_sw64(abase + shift * 64 + k0 * 2, 512);
    } else {
      da = desc_sw128(abase + shift * 128, dgap * 128, 1024, boff);
      idesc |= 1u << 15;                      // A is MN-major
    }
    const uint64_t db = desc_none(bbase, N * 16, 128);
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
        "l"(da), "l"(db), "r"(idesc), "r"(0));
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
        smem_u32(&bar)));
  }
  uint32_t done = 0;
  while (!done)
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\t"
                 "selp.u32 %0, 1, 0, p;\n\t}"
                 : "=r"(done)
                 : "r"(smem_u32(&bar)));
  asm volatile("tcgen05.fence::after_thread_sync;");
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int c = 0; c < N; c += 16) {
    uint32_t r[16];
    const uint32_t addr = tmem + ((uint32_t)(warp * 32) << 16) + c;
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
        "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
          "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
          "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(addr));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    for (int j = 0; j < 16; ++j) d_g[(warp * 32 + lane) * N + c + j] = __uint_as_float(r[j]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (threadIdx.x < 32)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 64;" ::"r"(tmem));
}

int main() {
  std::vector<__nv_bfloat16> a(R * 64), b(N * K);
  std::vector<float> af(R * 64), bf(N * K);
  for (int r = 0; r < R; ++r)
    for (int c = 0; c < 64; ++c) {
      af[r * 64 + c] = (float)((r * 7 + c * 3) % 19 - 9);
      a[r * 64 + c] = __float2bfloat16(af[r * 64 + c]);
    }
  for (int n = 0; n < N; ++n)
    for (int k = 0; k < K; ++k) {
      bf[n * K + k] = (float)((n + 2 * k) % 13 - 6);
      b[n * K + k] = __float2bfloat16(bf[n * K + k]);
    }
  __nv_bfloat16 *ag, *bg;
  float* dg;
  cudaMalloc(&ag, a.size() * 2);
  cudaMalloc(&bg, b.size() * 2);
  cudaMalloc(&dg, M * N * 4);
  cudaMemcpy(ag, a.data(), a.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(bg, b.data(), b.size() * 2, cudaMemcpyHostToDevice);
  for (int mode = 0; mode < 3; ++mode) {
    for (int shift : {0, 1, 3, 5, 8, 13, 57, 63}) {
      for (int k0 : {0, 16, 32}) {
        if (mode == 1 && k0) continue;
        if (mode == 2 && k0 > 16) continue;
        const int dgap = 57;
        int bad_by[2] = {0, 0};
        for (int bo = 0; bo < 2; ++bo) {
          const int boff = bo ? (shift & 7) : 0;
          cudaMemset(dg, 0, M * N * 4);
          probe<<<1, 128>>>(ag, bg, mode, shift, k0, dgap, boff, dg);
          cudaError_t e = cudaDeviceSynchronize();
          if (e != cudaSuccess) {
            printf("mode %d shift %d: %s\n", mode, shift, cudaGetErrorString(e));
            return 1;
          }
          std::vector<float> d(M * N);
          cudaMemcpy(d.data(), dg, M * N * 4, cudaMemcpyDeviceToHost);
          for (int m = 0; m < M; ++m)
            for (int n = 0; n < N; ++n) {
              float ref = 0.f;
              for (int k = 0; k < K; ++k) {
                float av;
                if (mode == 0 || mode == 2) av = af[(shift + m) * 64 + k0 + k];
                else av = af[(shift + (m >= 64 ? dgap : 0) + k) * 64 + (m % 64)];
                ref += av * bf[n * K + k];
              }
              if (d[m * N + n] != ref) ++bad_by[bo];
            }
        }
        printf("%s shift %3d k0 %2d: mismatches base_offset=0: %5d   base_offset=s&7: %5d\n",
               mode == 0 ? "KM128" : mode == 1 ? "MN128" : "KM64", shift, k0, bad_by[0],
               bad_by[1]);
      }
    }
  }
  return 0;
}
