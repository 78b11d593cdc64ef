// Correctness probe for shifted-window ("band") UMMA operands.
//
// A band of R rows x 16 k (bf16) is stored non-swizzled, K-major, with the
// rows of each 8-element K chunk contiguous (row stride 16 B):
//     addr(r, k) = (k / 8) * (R * 16) + r * 16 + (k % 8) * 2
// i.e. core matrices of 8 rows x 16 B with SBO = 128 B (next 8 rows) and
// LBO = R * 16 B (next K chunk).  A conv tap is then the view starting at
// row s: descriptor start = band + s * 16.  This checks tcgen05.mma
// (kind::f16, M=128, N=64, K=16) against a CPU reference for several s,
// including ones that are not multiples of 8.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -o band_check tools/band_check.cu
#include <cuda_bf16.h>
#include <cstdint>
#include <cstdio>
#include <vector>

constexpr int R = 256, M = 128, N = 64, K = 16;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ uint64_t desc_none(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;   // sm100 descriptor version
  return d;                 // layout type 0 = no swizzle
}

__global__ void probe(const __nv_bfloat16* a_g, const __nv_bfloat16* b_g, int shift, float* d_g) {
  __shared__ __align__(1024) uint8_t sm[R * K * 2 + N * K * 2];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const uint32_t abase = smem_u32(sm), bbase = abase + R * K * 2;
  // A band: element (r, k) at (k/8)*(R*16) + r*16 + (k%8)*2
  for (int i = threadIdx.x; i < R * K; i += blockDim.x) {
    const int r = i / K, k = i % K;
    *reinterpret_cast<__nv_bfloat16*>(sm + (k / 8) * (R * 16) + r * 16 + (k % 8) * 2) = a_g[i];
  }
  // B: N rows x 16 k, same interleaved form (LBO = N*16)
  for (int i = threadIdx.x; i < N * K; i += blockDim.x) {
    const int n = i / K, k = i % K;
    *reinterpret_cast<__nv_bfloat16*>(sm + R * K * 2 + (k / 8) * (N * 16) + n * 16 + (k % 8) * 2) =
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
    const uint64_t da = desc_none(abase + shift * 16, R * 16, 128);
    const uint64_t db = desc_none(bbase, N * 16, 128);
    const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) |
                           ((uint32_t)(M >> 4) << 24);
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
  // 4 warps x 32 lanes = 128 rows; 64 columns in 4 loads of 16
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
  std::vector<__nv_bfloat16> a(R * K), b(N * K);
  std::vector<float> af(R * K), bf(N * K);
  for (int r = 0; r < R; ++r)
    for (int k = 0; k < K; ++k) {
      af[r * K + k] = (float)((r * 3 + k * 5) % 17 - 8);
      a[r * K + k] = __float2bfloat16(af[r * K + k]);
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
  int bad_total = 0;
  for (int shift : {0, 1, 3, 7, 8, 13, 31, 64, 100, 127}) {
    cudaMemset(dg, 0, M * N * 4);
    probe<<<1, 128>>>(ag, bg, shift, dg);
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<float> d(M * N);
    cudaMemcpy(d.data(), dg, M * N * 4, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int r = 0; r < M; ++r)
      for (int n = 0; n < N; ++n) {
        float ref = 0.f;
        for (int k = 0; k < K; ++k) ref += af[(shift + r) * K + k] * bf[n * K + k];
        if (d[r * N + n] != ref) ++bad;
      }
    printf("shift %3d: %s, mismatches %d / %d\n", shift, e == cudaSuccess ? "ok" : cudaGetErrorString(e),
           bad, M * N);
    bad_total += bad;
  }
  printf("%s\n", bad_total == 0 ? "BAND LAYOUT OK" : "BAND LAYOUT MISMATCH");
  return bad_total != 0;
}
