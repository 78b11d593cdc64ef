// Microbenchmark: L2 -> SM operand feed through TMA (cp.async.bulk.tensor)
// as a function of the box shape and swizzle, with every SM loading.  One
// CTA per SM; lane 0 of warp 0 keeps `stages` boxes-groups in flight on a
// ring of mbarriers; reports bytes per cycle per SM.  The source tensor is
// L2-resident (a few MB, re-read) or HBM-sized.
//
// Question it answers: is the ~30 B/cycle/SM operand feed of
// the split-plane GEMM a per-request limit of its 64-byte (SWIZZLE_64B) box
// rows, i.e. would 128-byte rows (SWIZZLE_128B) feed faster?
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/bin/tma_bench \
//        tools/tma_bench.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdint>
#include <vector>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

__global__ void __launch_bounds__(32, 1)
    feed(const __grid_constant__ CUtensorMap map, int box_inner, int box_rows, int boxes_per_group,
         int stages, int groups, int rows_total, unsigned long long* cycles) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ __align__(8) uint64_t bar[16];
  const uint32_t base = (smem_u32(sm) + 1023u) & ~1023u;
  const uint32_t box_bytes = box_inner * box_rows * 2;
  const uint32_t group_bytes = box_bytes * boxes_per_group;
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[s])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncwarp();
  if (threadIdx.x != 0) return;
  const int row_groups = rows_total / box_rows;
  int rg = (blockIdx.x * 7919) % row_groups;
  unsigned long long t0 = clock64();
  for (int g = 0; g < groups + stages; ++g) {
    const int s = g % stages;
    if (g >= stages) {  // wait for the group issued `stages` ago
      const uint32_t parity = ((g - stages) / stages) & 1;
      asm volatile(
          "{\n\t.reg .pred p;\n\tWAIT_%=:\n\t"
          "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
          "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(&bar[s])),
          "r"(parity)
          : "memory");
    }
    if (g >= groups) continue;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(
                     smem_u32(&bar[s])),
                 "r"(group_bytes)
                 : "memory");
    for (int b = 0; b < boxes_per_group; ++b) {
      const uint32_t dst = base + s * group_bytes + b * box_bytes;
      rg = rg + 1 == row_groups ? 0 : rg + 1;
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
          " [%0], [%1, {%3, %4}], [%2];" ::"r"(dst),
          "l"(reinterpret_cast<uint64_t>(&map)), "r"(smem_u32(&bar[s])), "r"(0),
          "r"(rg * box_rows)
          : "memory");
    }
  }
  cycles[blockIdx.x] = clock64() - t0;
}

using EncFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                           const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                           CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                           CUtensorMapFloatOOBfill);

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  EncFn enc = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&enc),
                          cudaEnableDefault, &q);
  unsigned long long* cyc;
  cudaMalloc(&cyc, sms * sizeof(unsigned long long));
  struct Case {
    const char* name;
    int inner, rows, boxes;
    CUtensorMapSwizzle sw;
  };
  const Case cases[] = {
      {"SW64  box 32x128 (K-major A tile, 8 KB)", 32, 128, 3, CU_TENSOR_MAP_SWIZZLE_64B},
      {"SW64  box 32x32  (MN-major 2 KB boxes)", 32, 32, 12, CU_TENSOR_MAP_SWIZZLE_64B},
      {"SW128 box 64x64  (8 KB, 128-B rows)", 64, 64, 3, CU_TENSOR_MAP_SWIZZLE_128B},
      {"SW128 box 64x32  (4 KB, 128-B rows)", 64, 32, 6, CU_TENSOR_MAP_SWIZZLE_128B},
      {"SW128 box 64x128 (16 KB, 128-B rows)", 64, 128, 2, CU_TENSOR_MAP_SWIZZLE_128B},
      {"SW32  box 16x128 (4 KB, 32-B rows)", 16, 128, 6, CU_TENSOR_MAP_SWIZZLE_32B},
  };
  for (size_t footprint : {size_t(8) << 20, size_t(2) << 30}) {
    void* src;
    cudaMalloc(&src, footprint);
    cudaMemset(src, 0, footprint);
    for (const Case& c : cases) {
      const int inner = c.inner;
      const cuuint64_t rows_total = footprint / (inner * 2);
      const cuuint64_t dims[2] = {(cuuint64_t)inner, rows_total};
      const cuuint64_t strides[1] = {(cuuint64_t)inner * 2};
      const cuuint32_t box[2] = {(cuuint32_t)inner, (cuuint32_t)c.rows};
      const cuuint32_t es[2] = {1, 1};
      CUtensorMap map;
      CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, src, dims, strides, box, es,
                       CU_TENSOR_MAP_INTERLEAVE_NONE, c.sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                       CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      if (r != CUDA_SUCCESS) {
        printf("%s: encode failed %d\n", c.name, (int)r);
        continue;
      }
      const int group_bytes = inner * c.rows * 2 * c.boxes;
      const int stages = (160 * 1024) / group_bytes > 8 ? 8 : (160 * 1024) / group_bytes;
      const int groups = 4000;
      const size_t smem = (size_t)stages * group_bytes + 1024;
      cudaFuncSetAttribute(feed, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      for (int rep = 0; rep < 2; ++rep)
        feed<<<sms, 32, smem>>>(map, inner, c.rows, c.boxes, stages, groups, (int)rows_total, cyc);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) {
        printf("%s: %s\n", c.name, cudaGetErrorString(e));
        return 1;
      }
      std::vector<unsigned long long> h(sms);
      cudaMemcpy(h.data(), cyc, sms * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
      double mx = 0;
      for (auto v : h) mx = v > mx ? v : mx;
      const double bytes = (double)groups * group_bytes;
      printf("%-42s src %5zu MB  stages %d  %6.1f B/cycle/SM (slowest SM)\n", c.name,
             footprint >> 20, stages, bytes / mx);
    }
    cudaFree(src);
  }
  return 0;
}
