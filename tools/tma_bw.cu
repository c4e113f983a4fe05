// tma_bw.cu -- micro-benchmark: achievable HBM read bandwidth of TMA tile streams over the
// [B][C][H][D] bf16 layout (head-sliced boxes [128 tokens][64] vs whole-row boxes), persistent grid.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2404_02882_b200/csrc tools/tma_bw.cu -o /tmp/tma_bw -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include "sm100.cuh"

using namespace lasp::sm100;

struct P { CUtensorMap m, m2; int H, C, nitems, blocks_per_item, box_h, ntens; };

template <int ST>
__global__ void __launch_bounds__(128, 1) stream_kernel(const __grid_constant__ P p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t stage_bytes = 128 * 128 * p.box_h * p.ntens;
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + ST * stage_bytes);
  if (threadIdx.x == 0) { for (int s = 0; s < ST; ++s) mbar_init(&full[s], 1); fence_mbar_init(); }
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t J = 0;
    // item = (head group, token segment); segment-major over heads like the LASP kernels
    for (int w = blockIdx.x; w < p.nitems; w += gridDim.x) {
      const int hg = w % (p.H / p.box_h), seg = w / (p.H / p.box_h);
      for (int j = 0; j < p.blocks_per_item; ++j, ++J) {
        const int s = J % ST;
        if (J >= ST) mbar_wait(&full[s], ((J / ST) - 1) & 1);
        mbar_expect_tx(&full[s], stage_bytes);
        tma_load_4d(sm + s * stage_bytes, &p.m, &full[s], 0, hg * p.box_h, (seg * p.blocks_per_item + j) * 128, 0);
        if (p.ntens == 2)
          tma_load_4d(sm + s * stage_bytes + stage_bytes / 2, &p.m2, &full[s], 0, hg * p.box_h, (seg * p.blocks_per_item + j) * 128, 0);
      }
    }
    for (uint32_t k = (J > ST ? J - ST : 0); k < J; ++k) mbar_wait(&full[k % ST], (k / ST) & 1);
  }
  __syncthreads();
}

// L2 flush by reading (a write flush would leave dirty lines whose write-back competes with the timed run)
__global__ void read_flush(const int4* p, size_t n, int* sink) {
  int4 acc = make_int4(0, 0, 0, 0);
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x) {
    const int4 v = p[i];
    acc.x ^= v.x; acc.y ^= v.y; acc.z ^= v.z; acc.w ^= v.w;
  }
  if ((acc.x ^ acc.y ^ acc.z ^ acc.w) == 0x12345678) *sink = 1;
}

int main(int argc, char** argv) {
  const int H = 16, D = 64, C = argc > 1 ? atoi(argv[1]) : 32768 * 4;
  size_t bytes = size_t(C) * H * D * 2;
  void* buf;
  cudaMalloc(&buf, bytes);
  cudaMemset(buf, 1, bytes);
  PFN_cuTensorMapEncodeTiled_v12000 enc;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  int nsm;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  void* buf2;
  cudaMalloc(&buf2, bytes);
  cudaMemset(buf2, 1, bytes);
  void* flush;  // read between timed runs so that no run starts with its data in L2 (126 MB)
  cudaMalloc(&flush, size_t(256) << 20);
  cudaMemset(flush, 0, size_t(256) << 20);
  int* sink;
  cudaMalloc(&sink, 4);
  struct Cfg { int box_h, st, ntens, ctas; };
  for (Cfg c : {Cfg{1, 3, 1, 1}, Cfg{1, 6, 1, 1}, Cfg{1, 3, 2, 1}, Cfg{1, 3, 2, 2}, Cfg{1, 6, 2, 1}, Cfg{1, 2, 2, 2},
                Cfg{2, 3, 2, 1}, Cfg{1, 1, 2, 2}}) {
    P p;
    cuuint64_t dims[4] = {cuuint64_t(D), cuuint64_t(H), cuuint64_t(C), 1};
    cuuint64_t strides[3] = {cuuint64_t(D * 2), cuuint64_t(H * D * 2), cuuint64_t(size_t(C) * H * D * 2)};
    cuuint32_t box[4] = {64, cuuint32_t(c.box_h), 128, 1};
    cuuint32_t es[4] = {1, 1, 1, 1};
    enc(&p.m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, buf, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    enc(&p.m2, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, buf2, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    p.H = H; p.C = C; p.box_h = c.box_h; p.ntens = c.ntens;
    p.blocks_per_item = 7;
    p.nitems = (C / 128 / p.blocks_per_item) * (H / c.box_h);
    const int smem = c.st * 128 * 128 * c.box_h * c.ntens + 1024 + 256;
    if (smem > 227 * 1024 / c.ctas) continue;
    auto k = c.st == 1 ? stream_kernel<1> : c.st == 2 ? stream_kernel<2> : c.st == 3 ? stream_kernel<3> : stream_kernel<6>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    float best = 1e9;
    for (int it = 0; it < 5; ++it) {
      read_flush<<<nsm * 4, 512>>>(static_cast<const int4*>(flush), (size_t(256) << 20) / 16, sink);
      cudaEventRecord(a);
      k<<<nsm * c.ctas, 128, smem>>>(p);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      if (it > 0 && ms < best) best = ms;
    }
    const double moved = double(p.nitems) * p.blocks_per_item * 128 * 128 * c.box_h * c.ntens;
    printf("box heads=%d stages=%d tensors=%d ctas/sm=%d: %.1f us, %.0f GB/s (err=%s)\n", c.box_h, c.st, c.ntens, c.ctas,
           best * 1e3, moved / (best * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
