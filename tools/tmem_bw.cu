// TMEM load / store bandwidth micro-benchmark (debug tool): NW warps of one CTA per SM each issue
// tcgen05.ld.32x32b.x16 (2 KB per warp-instruction) REPS times over their lane quadrant, MODE 0: wait after
// every load (latency-bound, like the mask's chunk loop), MODE 1: 4 loads then one wait, MODE 2: stores.
// Prints aggregate bytes per SM-cycle. Build: nvcc -gencode arch=compute_100a,code=sm_100a -I../paper_2404_02882_b200/csrc
#include <cstdio>
#include <cstdint>
#include "sm100.cuh"
using namespace lasp::sm100;
constexpr int REPS = 512;
template <int N>
__device__ __forceinline__ void ldN(uint32_t taddr, float* v);
template <>
__device__ __forceinline__ void ldN<32>(uint32_t taddr, float* v) {
  uint32_t r[32];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
               "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                 "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
                 "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
                 "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
               : "r"(taddr));
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}
// x32 loads, one wait each (MODE 3); 16x256b.x8 (MODE 4, 4 KB per warp instruction like x32)
template <int MODE>
__global__ void __launch_bounds__(512, 1) k(float* out, long long* cyc, int nw) {
  __shared__ uint32_t slot;
  const uint32_t warp = threadIdx.x >> 5;
  if (warp == 0) tmem_alloc<512>(&slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  float acc = 0.f;
  long long t0 = 0, t1 = 0;
  if (warp < uint32_t(nw)) {
    const uint32_t ta = tmem + (((warp & 3) * 32) << 16) + (warp >> 2) * 32;
    uint32_t z[16] = {};
    __syncwarp();
    t0 = clock64();
    for (int it = 0; it < REPS; ++it) {
      if (MODE == 3 || MODE == 4) {
        float v[32];
        if (MODE == 3) ldN<32>(ta + (it & 3) * 32, v);
        else tmem_ld_16x256b_x8(ta + (it & 3) * 32, *reinterpret_cast<float(*)[32]>(v));
        tmem_ld_wait();
#pragma unroll
        for (int u = 0; u < 32; ++u) acc += v[u];
      } else if (MODE == 2) {
        tmem_st16(ta + (it & 7) * 16, z);
        if ((it & 3) == 3) tmem_st_wait();
      } else if (MODE == 0) {
        float v[16];
        tmem_ld16(ta + (it & 7) * 16, v);
        tmem_ld_wait();
#pragma unroll
        for (int u = 0; u < 16; ++u) acc += v[u];
      } else {
        float v[4][16];
#pragma unroll
        for (int x = 0; x < 4; ++x) tmem_ld16(ta + ((it * 4 + x) & 7) * 16, v[x]);
        tmem_ld_wait();
#pragma unroll
        for (int x = 0; x < 4; ++x)
#pragma unroll
          for (int u = 0; u < 16; ++u) acc += v[x][u];
        it += 3;
      }
    }
    tmem_st_wait();
    t1 = clock64();
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x % 32 == 0 && warp < uint32_t(nw)) cyc[blockIdx.x * 16 + warp] = t1 - t0;
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(tmem);
}
template <int MODE>
void run(const char* name, int nw, float* o, long long* c) {
  k<MODE><<<148, 512>>>(o, c, nw);
  cudaDeviceSynchronize();
  long long h[148 * 16];
  cudaMemcpy(h, c, sizeof h, cudaMemcpyDeviceToHost);
  double mx = 0;
  for (int w = 0; w < nw; ++w) mx = h[w] > mx ? h[w] : mx;
  const double bytes = double(nw) * REPS * (MODE >= 3 ? 4096 : 2048);
  printf("%-22s warps %2d: %8.0f cycles, %6.1f B/cycle/SM, %5.1f cycles per warp-instruction\n", name, nw, mx,
         bytes / mx, mx / REPS);
}
int main() {
  float* o; long long* c;
  cudaMalloc(&o, 148 * 512 * 4); cudaMalloc(&c, 148 * 16 * 8);
  for (int nw : {1, 4, 8, 12, 16}) run<0>("ld x16 + wait each", nw, o, c);
  for (int nw : {1, 4, 8, 12, 16}) run<1>("4 x ld x16 + wait", nw, o, c);
  for (int nw : {1, 4, 8, 16}) run<2>("st x16", nw, o, c);
  for (int nw : {1, 4, 8, 16}) run<3>("ld x32 + wait each", nw, o, c);
  for (int nw : {1, 4, 8, 16}) run<4>("ld 16x256b.x8 + wait", nw, o, c);
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
}
