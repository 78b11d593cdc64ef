// NVLink store bandwidth of the peer-link put kernel's variants, GPU 0 -> GPU 1
// (one process, peer access enabled): what limits stz_link_put at ~330 GB/s?
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o p2p_bench tools/p2p_bench.cu
//
// src: three bf16 planes of R x 8192 elements on GPU 0; dst: fp32 on GPU 1.
//   join2x4 : the shipped form (3 x 16-byte plane loads, join, 2 x float4 stores)
//   join256 : the same with one 256-bit store (st.global.v8.f32)
//   join256x2 : two 8-element groups per step, all loads issued first
//   copy4   : fp32 -> fp32 float4 copy (no conversion), the SM-store ceiling
//   memcpy  : cudaMemcpyPeerAsync (copy engines)
#include <cuda_bf16.h>
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ float bf(uint16_t b) { return __uint_as_float((uint32_t)b << 16); }
__device__ __forceinline__ void join8(uint4 a, uint4 b, uint4 c, float (&v)[8]) {
  const uint32_t aw[4] = {a.x, a.y, a.z, a.w}, bw[4] = {b.x, b.y, b.z, b.w}, cw[4] = {c.x, c.y, c.z, c.w};
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    const int sh = (e & 1) * 16;
    v[e] = __fadd_rn(__fadd_rn(bf((uint16_t)(aw[e / 2] >> sh)), bf((uint16_t)(bw[e / 2] >> sh))),
                     bf((uint16_t)(cw[e / 2] >> sh)));
  }
}
__device__ __forceinline__ void st256(float* p, const float (&v)[8]) {
  asm volatile("st.global.v8.f32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(p), "f"(v[0]),
               "f"(v[1]), "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7])
               : "memory");
}

__global__ void join2x4(const uint16_t* src, size_t ps, float* dst, size_t n8) {
  for (size_t q = blockIdx.x * (size_t)blockDim.x + threadIdx.x; q < n8; q += (size_t)gridDim.x * blockDim.x) {
    float v[8];
    join8(__ldg((const uint4*)(src + q * 8)), __ldg((const uint4*)(src + q * 8 + ps)),
          __ldg((const uint4*)(src + q * 8 + 2 * ps)), v);
    ((float4*)(dst + q * 8))[0] = make_float4(v[0], v[1], v[2], v[3]);
    ((float4*)(dst + q * 8))[1] = make_float4(v[4], v[5], v[6], v[7]);
  }
  __threadfence_system();
}

__global__ void join256(const uint16_t* src, size_t ps, float* dst, size_t n8) {
  for (size_t q = blockIdx.x * (size_t)blockDim.x + threadIdx.x; q < n8; q += (size_t)gridDim.x * blockDim.x) {
    float v[8];
    join8(__ldg((const uint4*)(src + q * 8)), __ldg((const uint4*)(src + q * 8 + ps)),
          __ldg((const uint4*)(src + q * 8 + 2 * ps)), v);
    st256(dst + q * 8, v);
  }
  __threadfence_system();
}

__global__ void join256x2(const uint16_t* src, size_t ps, float* dst, size_t n8) {
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t q = blockIdx.x * (size_t)blockDim.x + threadIdx.x; q < n8; q += 2 * stride) {
    const size_t q2 = q + stride;
    const bool two = q2 < n8;
    uint4 a0 = __ldg((const uint4*)(src + q * 8)), b0 = __ldg((const uint4*)(src + q * 8 + ps)),
          c0 = __ldg((const uint4*)(src + q * 8 + 2 * ps));
    uint4 a1 = a0, b1 = b0, c1 = c0;
    if (two) {
      a1 = __ldg((const uint4*)(src + q2 * 8));
      b1 = __ldg((const uint4*)(src + q2 * 8 + ps));
      c1 = __ldg((const uint4*)(src + q2 * 8 + 2 * ps));
    }
    float v[8], w[8];
    join8(a0, b0, c0, v);
    st256(dst + q * 8, v);
    if (two) {
      join8(a1, b1, c1, w);
      st256(dst + q2 * 8, w);
    }
  }
  __threadfence_system();
}

__global__ void copy4(const float4* src, float4* dst, size_t n4) {
  for (size_t q = blockIdx.x * (size_t)blockDim.x + threadIdx.x; q < n4; q += (size_t)gridDim.x * blockDim.x)
    dst[q] = __ldg(src + q);
  __threadfence_system();
}

int main() {
  int ndev = 0;
  cudaGetDeviceCount(&ndev);
  if (ndev < 2) {
    printf("needs 2 GPUs\n");
    return 0;
  }
  int can = 0;
  cudaDeviceCanAccessPeer(&can, 0, 1);
  const size_t n = (size_t)32 << 20;   // 32 M elements: 128 MB fp32
  uint16_t* src;
  float *dst, *src32;
  cudaSetDevice(1);
  cudaMalloc(&dst, n * 4);
  cudaSetDevice(0);
  cudaDeviceEnablePeerAccess(1, 0);
  cudaMalloc(&src, n * 2 * 3);
  cudaMalloc(&src32, n * 4);
  cudaMemset(src, 0, n * 6);
  cudaMemset(src32, 0, n * 4);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  printf("peer access %d, %d SMs, %zu MB fp32 per transfer\n", can, sms, n * 4 >> 20);
  for (int mult : {2, 4, 8, 16}) {
    const int grid = sms * mult;
    for (int variant = 0; variant < 4; ++variant) {
      auto run = [&]() {
        if (variant == 0) join2x4<<<grid, 256>>>(src, n, dst, n / 8);
        if (variant == 1) join256<<<grid, 256>>>(src, n, dst, n / 8);
        if (variant == 2) join256x2<<<grid, 256>>>(src, n, dst, n / 8);
        if (variant == 3) copy4<<<grid, 256>>>((const float4*)src32, (float4*)dst, n / 4);
      };
      run();
      cudaEventRecord(e0);
      for (int r = 0; r < 5; ++r) run();
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      const char* names[4] = {"join2x4", "join256", "join256x2", "copy4"};
      printf("grid %4d (%2d/SM) %-10s %7.1f GB/s\n", grid, mult, names[variant],
             n * 4.0 / (ms / 5 / 1e3) / 1e9);
    }
  }
  cudaEventRecord(e0);
  for (int r = 0; r < 5; ++r) cudaMemcpyPeerAsync(dst, 1, src32, 0, n * 4);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  printf("cudaMemcpyPeerAsync %7.1f GB/s\n", n * 4.0 / (ms / 5 / 1e3) / 1e9);
  return 0;
}
