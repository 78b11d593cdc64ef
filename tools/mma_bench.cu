// Microbenchmark: raw tcgen05.mma (kind::f16, SS operands) throughput per SM
// as a function of N, shared-memory swizzle mode and operand major-ness.
// One CTA per SM, one thread issues R MMAs back to back (operands = zeros in
// smem), then commits and waits; reports cycles per MMA.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o mma_bench tools/mma_bench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

// layout: 0 = none (interleave), 1 = SW128 (type 2), 2 = SW64 (type 4), 3 = SW32 (type 6)
__device__ __forceinline__ uint64_t desc(uint32_t saddr, uint32_t lbo, uint32_t sbo, int layout) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
  d |= (uint64_t)1 << 46;
  const uint64_t t = layout == 1 ? 2 : layout == 2 ? 4 : layout == 3 ? 6 : 0;
  d |= t << 61;
  return d;
}

__device__ __forceinline__ uint32_t idesc(int m, int n, bool amn, bool bmn) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((amn ? 1u : 0u) << 15) | ((bmn ? 1u : 0u) << 16) |
         ((uint32_t)(n >> 3) << 17) | ((uint32_t)(m >> 4) << 24);
}

template <int N>
__global__ void __launch_bounds__(128, 1) bench(int reps, int layout, int amn, int bmn, int accs,
                                                 unsigned long long* out, int mode = 0) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t bar;
  __shared__ uint64_t sbar[4];
  __shared__ uint32_t slot;
  const uint32_t base = (smem_u32(sm) + 1023u) & ~1023u;
  for (int i = threadIdx.x; i < 200 * 1024 / 4; i += blockDim.x)
    reinterpret_cast<uint32_t*>(sm)[i] = 0;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    for (int i = 0; i < 4; ++i)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&sbar[i])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
        smem_u32(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = slot;
  if (threadIdx.x == 0) {
    const uint32_t id = idesc(128, N, amn, bmn);
    // 3 A planes (16 KB each slot) + 3 B planes: distinct addresses like the GEMM
    uint32_t lbo_a = 16, sbo_a = 512, lbo_b = 16, sbo_b = 512;
    if (layout == 1) { sbo_a = sbo_b = 1024; }
    if (layout == 0) { lbo_a = lbo_b = 128 * 16; sbo_a = sbo_b = 128; }
    if (amn) { lbo_a = 2048; sbo_a = 512; }
    if (bmn) { lbo_b = 2048; sbo_b = 512; }
    uint64_t da[3], db[3];
    for (int p = 0; p < 3; ++p) {
      da[p] = desc(base + p * 16384, lbo_a, sbo_a, layout);
      db[p] = desc(base + 49152 + p * 16384, lbo_b, sbo_b, layout);
    }
    const int AP[6] = {0, 2, 1, 0, 1, 0};
    const int BP[6] = {2, 0, 1, 1, 0, 0};
    unsigned long long t0 = clock64();
    if (mode == 0) {
      for (int r = 0; r < reps; ++r) {
#pragma unroll
        for (int i = 0; i < 6; ++i) {
          const uint32_t acc = accs == 1 ? tmem : (i == 5 ? tmem : tmem + N);
          asm volatile(
              "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
              "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(acc),
              "l"(da[AP[i]]), "l"(db[BP[i]]), "r"(id), "r"(1));
        }
      }
    } else {
      // kernel-like: 4 stages x (3 A planes 8 KB + 3 B planes), 2 k-steps of 16 per
      // stage, commit per stage (mode & 2), fence::after + try_wait (mode & 4)
      const uint32_t ab = 8192, bb = N * 64, sb = 3 * (ab + bb);
      const uint64_t d0a = desc(base, lbo_a, sbo_a, layout), d0b = desc(base + 3 * ab, lbo_b, sbo_b, layout);
      int nst = (196608 / sb) < 4 ? (196608 / sb) : 4;
      for (int r = 0; r < reps / 2; ++r) {
        const int st = r % nst;
        const uint32_t so = (st * sb) >> 4;
        if (mode & 4) {
          asm volatile("tcgen05.fence::after_thread_sync;");
          uint32_t done = 0;
          while (!done)
            asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
                         "selp.u32 %0, 1, 0, p;\n\t}"
                         : "=r"(done)
                         : "r"(smem_u32(&sbar[st])), "r"(((r / nst) & 1) ^ 1));
        }
#pragma unroll
        for (int j = 0; j < 2; ++j)
#pragma unroll
          for (int i = 0; i < 6; ++i) {
            const uint32_t acc = i == 5 ? tmem : tmem + N;
            const uint32_t ka = amn ? 64 : 2, kb = bmn ? 64 : 2;
            const uint64_t a = d0a + (so + AP[i] * (ab >> 4) + j * ka);
            const uint64_t b = d0b + (so + BP[i] * (bb >> 4) + j * kb);
            asm volatile(
                "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(acc),
                "l"(a), "l"(b), "r"(id), "r"(1));
          }
        if (mode & 2)
          asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
              smem_u32(&sbar[st])));
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
        smem_u32(&bar)));
    uint32_t done = 0;
    while (!done)
      asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\t"
                   "selp.u32 %0, 1, 0, p;\n\t}"
                   : "=r"(done)
                   : "r"(smem_u32(&bar)));
    unsigned long long t1 = clock64();
    out[blockIdx.x] = t1 - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (threadIdx.x < 32)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

template <int N>
void run(int layout, int amn, int bmn, int accs, int mode = 0) {
  const int reps = 2000, sms = 148;
  unsigned long long* d;
  cudaMalloc(&d, sms * 8);
  cudaFuncSetAttribute(bench<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024 + 1024);
  bench<N><<<sms, 128, 200 * 1024 + 1024>>>(10, layout, amn, bmn, accs, d, mode);
  bench<N><<<sms, 128, 200 * 1024 + 1024>>>(reps, layout, amn, bmn, accs, d, mode);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h[148];
  cudaMemcpy(h, d, sms * 8, cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < sms; ++i) avg += h[i];
  avg /= sms;
  const double per = avg / (reps * 6.0);
  const double floor = 128.0 * N / 256.0;
  printf("mode=%d N=%3d layout=%s amn=%d bmn=%d accs=%d: %.1f cyc/MMA (floor %.0f, %.0f%%) %s\n",
         mode, N, layout == 0 ? "none " : layout == 1 ? "SW128" : layout == 2 ? "SW64 " : "SW32 ", amn, bmn,
         accs, per, floor, 100.0 * floor / per, e == cudaSuccess ? "" : cudaGetErrorString(e));
  cudaFree(d);
}

int main() {
  for (int mode : {0, 1, 3, 7}) {
    run<64>(2, 0, 0, 2, mode);
    run<128>(2, 0, 0, 2, mode);
    run<192>(2, 0, 0, 2, mode);
    run<256>(2, 0, 0, 2, mode);
    run<64>(2, 1, 1, 2, mode);
    run<192>(2, 1, 1, 2, mode);
  }
  run<64>(1, 0, 0, 2, 1);
  run<64>(1, 0, 0, 2, 7);
  run<192>(1, 0, 0, 2, 7);
  return 0;
}
