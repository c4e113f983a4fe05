// Issue-rate micro-benchmark (debug tool): cycles per warp-instruction of the mask warps' arithmetic
// (FMUL, FMUL2 = mul.rn.f32x2, F2FP = cvt.rn.bf16x2.f32, HMUL2.BF16 = mul.rn.bf16x2) with 8 independent
// chains, for 1 and 4 warps per SM sub-partition. Build: nvcc -gencode arch=compute_100a,code=sm_100a.
#include <cstdio>
#include <cstdint>
template <int MODE>
__global__ void k(uint32_t* out, long long* cyc) {
  uint32_t r[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) r[i] = __float_as_uint(1.0f + 1e-3f * (threadIdx.x + i));
  const uint32_t m = __float_as_uint(0.999f);
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < 1024; ++it) {
#pragma unroll
    for (int i = 0; i < 16; i += 2) {
      if (MODE == 0) {  // 2 scalar FMUL
        asm volatile("mul.rn.f32 %0, %0, %2;\n\tmul.rn.f32 %1, %1, %2;" : "+r"(r[i]), "+r"(r[i + 1]) : "r"(m));
      } else if (MODE == 1) {  // 1 FMUL2
        uint64_t x = (uint64_t(r[i + 1]) << 32) | r[i], y = (uint64_t(m) << 32) | m;
        asm volatile("mul.rn.f32x2 %0, %0, %1;" : "+l"(x) : "l"(y));
        r[i] = uint32_t(x); r[i + 1] = uint32_t(x >> 32);
      } else if (MODE == 2) {  // 1 F2FP (2 floats -> bf16x2), result fed back so the chain stays live
        uint32_t p;
        asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(p) : "r"(r[i]), "r"(r[i + 1]));
        r[i] = p;
      } else {  // 1 HMUL2.BF16
        asm volatile("mul.rn.bf16x2 %0, %0, %1;" : "+r"(r[i]) : "r"(0x3f803f80u));
      }
    }
  }
  long long t1 = clock64();
  uint32_t acc = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) acc ^= r[i];
  out[threadIdx.x] = acc;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
template <int MODE>
void run(const char* name, int warps, uint32_t* o, long long* c) {
  k<MODE><<<1, 32 * warps>>>(o, c);
  cudaDeviceSynchronize();
  long long h;
  cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  const double per_smsp = warps >= 4 ? warps / 4.0 : 1.0;
  printf("%-40s warps/SMSP %.0f: %.2f cycles per warp-instruction\n", name, per_smsp, double(h) / (per_smsp * 1024 * 8));
}
int main() {
  uint32_t* o; long long* c;
  cudaMalloc(&o, 1 << 16); cudaMalloc(&c, 64);
  for (int w : {4, 16}) {
    run<0>("FMUL x2 (per pair of elements)", w, o, c);
    run<1>("FMUL2 (mul.rn.f32x2)", w, o, c);
    run<2>("F2FP (cvt.rn.bf16x2.f32)", w, o, c);
    run<3>("HMUL2.BF16 (mul.rn.bf16x2)", w, o, c);
  }
  return 0;
}
