// l2_bw.cu -- micro-benchmark: L2 -> SM TMA throughput when the data is L2-resident (debug tool).
// A 2-D bf16 tensor of ROWS x 64 (ROWS * 128 bytes, default 16 MB) is read by 148 persistent CTAs with TMA
// boxes of [128 rows][64] (16 KB, 128B swizzle), ST-stage ring, each CTA walking the rows from its own
// offset, NREP passes; also a DRAM-resident case (1 GB, read once). Reports TB/s and bytes/cycle/SM.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2404_02882_b200/csrc tools/l2_bw.cu -o /tmp/l2_bw -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <cstdint>
#include "sm100.cuh"
using namespace lasp::sm100;
template <int ST>
__global__ void __launch_bounds__(32, 1) rd(const __grid_constant__ CUtensorMap m, int nbox_total, int per_cta) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + ST * 16384);
  if (threadIdx.x == 0) {
    for (int s = 0; s < ST; ++s) mbar_init(&full[s], 1);
    fence_mbar_init();
    for (int J = 0; J < per_cta; ++J) {
      const int s = J % ST;
      if (J >= ST) mbar_wait(&full[s], ((J / ST) - 1) & 1);
      mbar_expect_tx(&full[s], 16384);
      const int box = (blockIdx.x * 7919 + J) % nbox_total;
      tma_load_2d(sm + s * 16384, &m, &full[s], 0, box * 128);
    }
    for (int J = per_cta > ST ? per_cta - ST : 0; J < per_cta; ++J) mbar_wait(&full[J % ST], (J / ST) & 1);
  }
}
int main() {
  PFN_cuTensorMapEncodeTiled_v12000 enc;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  int clk = 0; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  for (size_t mb : {16, 32, 64, 1024}) {
    const size_t bytes = mb << 20, rows = bytes / 128;
    void* buf; cudaMalloc(&buf, bytes); cudaMemset(buf, 1, bytes);
    CUtensorMap m;
    cuuint64_t dims[2] = {64, rows}; cuuint64_t str[1] = {128}; cuuint32_t box[2] = {64, 128}; cuuint32_t es[2] = {1, 1};
    enc(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    const int nbox = int(rows / 128);
    const int per_cta = mb >= 1024 ? nbox / 148 : 4096;
    auto run = [&](auto kern, int st) {
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, st * 16384 + 2048);
      kern<<<148, 32, st * 16384 + 2048>>>(m, nbox, per_cta);  // warm (L2-resident cases)
      cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
      cudaEventRecord(a);
      kern<<<148, 32, st * 16384 + 2048>>>(m, nbox, per_cta);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      const double tot = 148.0 * per_cta * 16384;
      printf("%5zu MB  stages %2d: %7.2f TB/s  %6.1f B/cycle/SM (at %d MHz)\n", mb, st, tot / ms / 1e9,
             tot / (ms * 1e-3 * clk * 1e3) / 148, clk / 1000);
    };
    run(rd<4>, 4); run(rd<8>, 8); run(rd<12>, 12);
    cudaFree(buf);
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
}
