// kernels_simt.cu -- CUDA-core (FFMA) kernels of the LASP path.
//
// These serve the fp32 path (LASP_FP32, parity tolerance 1e-5: TF32 tensor cores cannot meet it,
// SURVEY.md V3) and any (dtype, head_dim) the tcgen05 kernels do not cover. They implement the
// same three stages as the tensor-core path (see lasp_common.cuh):
//   seg_state : decayed outer-product accumulation over one segment (F1 / B1, Eq. 12 / Eq. 21)
//   prefix    : fold of segment states along the rank, seeded with the received state (F2 / B2)
//   core      : fused intra + inter chunk pass with the running state (F3 / B3, Eq. 7-9, 15-22)
#include "lasp_common.cuh"

#include <cmath>

namespace lasp {
namespace {

template <typename T> __device__ __forceinline__ float ld(const T* p);
template <> __device__ __forceinline__ float ld<float>(const float* p) { return *p; }
template <> __device__ __forceinline__ float ld<__nv_bfloat16>(const __nv_bfloat16* p) {
  return __bfloat162float(*p);
}
template <typename T> __device__ __forceinline__ void st(T* p, float v);
template <> __device__ __forceinline__ void st<float>(float* p, float v) { *p = v; }
template <> __device__ __forceinline__ void st<__nv_bfloat16>(__nv_bfloat16* p, float v) {
  *p = __float2bfloat16_rn(v);
}

// lambda^k in fp64, rounded once to fp32 (reading A9: powers are never inverted).
__device__ __forceinline__ float powk(float lam, double k) { return (float)pow((double)lam, k); }

constexpr int kThreads = 256;

// ---------------------------------------------------------------------------------------------
// seg_state: out[b][h][p] = sum_{pos in seg p} w_pos x_pos y_pos^T  (D x D, fp32)
//   FWD: w = lam^(end-1-pos)  (Eq. 12's lambda^C Lambda^-1 weights, relative to the segment end)
//   REV: w = lam^(pos-begin+1) (Eq. 21's Lambda weights, relative to the segment begin)
template <typename T, int D, Dir DIR>
__global__ void __launch_bounds__(kThreads) seg_state_simt_kernel(Plan p, const T* __restrict__ x,
                                                                  const T* __restrict__ y,
                                                                  float* __restrict__ out) {
  pdl_wait();
  pdl_trigger();
  constexpr int TT = 32;        // tokens per smem tile
  constexpr int R = D / 16;     // per-thread register tile R x R
  __shared__ float xs[TT][D + 1];
  __shared__ float ys[TT][D + 1];
  const int64_t seg = blockIdx.x, h = blockIdx.y, b = blockIdx.z;
  const float lam = p.lam[h];
  const int64_t beg = seg_begin(DIR, seg, p.seg_len, p.C), end = seg_end(DIR, seg, p.seg_len, p.C);
  const int tr = threadIdx.x / 16, tc = threadIdx.x % 16;
  float acc[R][R];
#pragma unroll
  for (int i = 0; i < R; ++i)
#pragma unroll
    for (int j = 0; j < R; ++j) acc[i][j] = 0.f;
  const int64_t rs = p.H * D;  // row stride (elements) between consecutive tokens
  for (int64_t t0 = beg; t0 < end; t0 += TT) {
    for (int idx = threadIdx.x; idx < TT * D; idx += kThreads) {
      const int s = idx / D, d = idx % D;
      const int64_t pos = t0 + s;
      float xv = 0.f, yv = 0.f;
      if (pos < end) {
        const int64_t off = (b * p.C + pos) * rs + h * D + d;
        const double k = (DIR == Dir::FWD) ? double(end - 1 - pos) : double(pos - beg + 1);
        xv = ld(x + off) * powk(lam, k);
        yv = ld(y + off);
      }
      xs[s][d] = xv;
      ys[s][d] = yv;
    }
    __syncthreads();
#pragma unroll 4
    for (int s = 0; s < TT; ++s) {
      float xr[R], yr[R];
#pragma unroll
      for (int i = 0; i < R; ++i) xr[i] = xs[s][tr + 16 * i];
#pragma unroll
      for (int j = 0; j < R; ++j) yr[j] = ys[s][tc + 16 * j];
#pragma unroll
      for (int i = 0; i < R; ++i)
#pragma unroll
        for (int j = 0; j < R; ++j) acc[i][j] = fmaf(xr[i], yr[j], acc[i][j]);
    }
    __syncthreads();
  }
  float* o = out + ((b * p.H + h) * p.nseg + seg) * D * D;
#pragma unroll
  for (int i = 0; i < R; ++i)
#pragma unroll
    for (int j = 0; j < R; ++j) o[(tr + 16 * i) * D + tc + 16 * j] = acc[i][j];
}

// ---------------------------------------------------------------------------------------------
// prefix: per element, cur = init; for p: prefix[p] = cur; cur = lam^len_p cur + seg[p]; final = cur
// (Alg. 2 P:171 / Alg. 3 P:648 applied between segments). `prefix` may alias `seg_states`.
// U: segment loads in flight per thread, the smallest of {8, 16, 24, 40} that covers nseg (chosen by the host),
// D and DIR compile-time so the segment stride is an immediate offset (one base address per thread instead of
// one 64-bit address per load): TNL-1B's 24 segments took ~170-255 registers per thread with runtime strides,
// which left part of the launch to a second wave
template <int U, int D, Dir DIR>
__global__ void __launch_bounds__(64) prefix_kernel(Plan p, const float* __restrict__ init,
                                                    const float* seg_states, float* prefix,
                                                    float* __restrict__ final_out) {
  pdl_wait();
  pdl_trigger();
  // One thread per 4 consecutive state elements (float4); all (up to U) segment loads of a batch are
  // issued before the serial fold (nseg <= U: one L2 round trip). `prefix` may alias `seg_states`: a
  // thread loads every segment of a batch before it stores any of them.
  constexpr int64_t DD = int64_t(D) * D;
  constexpr int64_t step = DIR == Dir::FWD ? DD : -DD;  // floats between consecutive folded segments
  const int64_t idx4 = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;  // over B*H*D*D/4
  if (idx4 * 4 >= p.B * p.Hk * DD) return;
  const int64_t bh = (idx4 * 4) / DD, e = (idx4 * 4) % DD, h = bh % p.Hk;
  // every segment has seg_len tokens except possibly the last one (both directions)
  const int64_t last_len = p.C - (p.nseg - 1) * p.seg_len;
  // lam^len = exp2(len * log2(lam)) with log2(lam) from the host in fp64 (relative error ~1e-6 at len ~ 1e3)
  const float l2 = p.l2lam[h];
  const float dec_full = exp2f(float(p.seg_len) * l2);
  const float dec_last = exp2f(float(last_len > 0 ? last_len : 0) * l2);
  float4 cur = init ? *reinterpret_cast<const float4*>(init + idx4 * 4) : make_float4(0.f, 0.f, 0.f, 0.f);
  // first folded segment: 0 (FWD) or nseg - 1 (REV, folds from the rank end)
  const int64_t first = (bh * p.nseg + (DIR == Dir::FWD ? 0 : p.nseg - 1)) * DD + e;
  const float* src = seg_states ? seg_states + first : nullptr;
  float* dst = prefix ? prefix + first : nullptr;
  for (int64_t s0 = 0; s0 < p.nseg; s0 += U, src = src ? src + U * step : src, dst = dst ? dst + U * step : dst) {
    const int nb = int(p.nseg - s0);  // segments left
    float4 v[U];
#pragma unroll
    for (int t = 0; t < U; ++t)
      v[t] = (src && t < nb) ? __ldcg(reinterpret_cast<const float4*>(src + t * step)) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int t = 0; t < U; ++t) {
      if (t < nb) {
        if (dst) *reinterpret_cast<float4*>(dst + t * step) = cur;
        const int64_t sg = DIR == Dir::FWD ? s0 + t : p.nseg - 1 - (s0 + t);
        const float dcy = (sg == p.nseg - 1) ? dec_last : dec_full;
        cur.x = fmaf(dcy, cur.x, v[t].x); cur.y = fmaf(dcy, cur.y, v[t].y);
        cur.z = fmaf(dcy, cur.z, v[t].z); cur.w = fmaf(dcy, cur.w, v[t].w);
      }
    }
  }
  if (final_out) *reinterpret_cast<float4*>(final_out + idx4 * 4) = cur;
}

// kv_out = lam^C kv_in + local (the ring's combine step, Alg. 2 P:171 with the local part hoisted)
__global__ void combine_kernel(Plan p, const float* __restrict__ kv_in,
                               const float* __restrict__ local, float* __restrict__ kv_out) {
  pdl_wait();
  pdl_trigger();
  const int64_t DD = p.D * p.D;
  const int64_t idx = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx >= p.B * p.Hk * DD) return;
  const int64_t h = (idx / DD) % p.Hk;
  const float in = kv_in ? kv_in[idx] : 0.f;
  kv_out[idx] = fmaf(powk(p.lam[h], double(p.C)), in, local[idx]);
}

// ---------------------------------------------------------------------------------------------
// core: one CTA per (segment, head, batch); blocks of BT tokens in direction order with the running
// state S in shared memory (fp32).
template <typename T, int D, Dir DIR>
__global__ void __launch_bounds__(kThreads) core_simt_kernel(Plan p, SeqArgs a) {
  pdl_wait();
  pdl_trigger();
  constexpr int BT = 32;
  extern __shared__ float smem[];
  float* sa = smem;                  // [BT][D+1]
  float* sb = sa + BT * (D + 1);     // [BT][D+1]
  float* sc = sb + BT * (D + 1);     // [BT][D+1]
  float* S = sc + BT * (D + 1);      // [D][D+1]
  float* A = S + D * (D + 1);        // [BT][BT+1]
  float* pw = A + BT * (BT + 1);     // [BT+1]
  const int64_t seg = blockIdx.x, h = blockIdx.y, b = blockIdx.z;
  const float lam = p.lam[h];
  const int64_t beg = seg_begin(DIR, seg, p.seg_len, p.C), end = seg_end(DIR, seg, p.seg_len, p.C);
  const int tid = threadIdx.x;
  for (int k = tid; k <= BT; k += kThreads) pw[k] = powk(lam, double(k));
  const float* st0 = a.state + ((b * p.H + h) * p.nseg + seg) * D * D;
  const float poison = tag_poisoned(a.status) ? __int_as_float(0x7fc00000) : 0.f;  // cache tag mismatch: NaN
  for (int idx = tid; idx < D * D; idx += kThreads) {
    const int d = idx / D, e = idx % D;
    S[d * (D + 1) + e] = (a.trans_state ? st0[e * D + d] : st0[idx]) + poison;
  }
  const T* ga = static_cast<const T*>(a.a);
  const T* gb = static_cast<const T*>(a.b);
  const T* gc = static_cast<const T*>(a.c);
  T* go = static_cast<T*>(a.out);
  const int64_t rs = p.H * D;
  const int64_t nblk = (end - beg + BT - 1) / BT;
  __syncthreads();
  for (int64_t j = 0; j < nblk; ++j) {
    // block rows [t0, t0 + BT): FWD ascending from beg; REV descending, aligned to end
    const int64_t t0 = (DIR == Dir::FWD) ? beg + j * BT : end - (j + 1) * BT;
    for (int idx = tid; idx < BT * D; idx += kThreads) {
      const int s = idx / D, d = idx % D;
      const int64_t pos = t0 + s;
      float va = 0.f, vb = 0.f, vc = 0.f;
      if (pos >= beg && pos < end) {
        const int64_t off = (b * p.C + pos) * rs + h * D + d;
        va = ld(ga + off); vb = ld(gb + off); vc = ld(gc + off);
      }
      sa[s * (D + 1) + d] = va; sb[s * (D + 1) + d] = vb; sc[s * (D + 1) + d] = vc;
    }
    __syncthreads();
    // A_ij = (a_i . b_j) * M_ij
    for (int idx = tid; idx < BT * BT; idx += kThreads) {
      const int i = idx / BT, jj = idx % BT;
      const bool live = (DIR == Dir::FWD) ? (jj <= i) : (jj >= i);
      float s = 0.f;
      if (live) {
#pragma unroll 8
        for (int d = 0; d < D; ++d) s = fmaf(sa[i * (D + 1) + d], sb[jj * (D + 1) + d], s);
        s *= pw[(DIR == Dir::FWD) ? (i - jj) : (jj - i)];
      }
      A[i * (BT + 1) + jj] = s;
    }
    __syncthreads();
    // out_i = sum_j A_ij c_j + r_i a_i^T S
    for (int idx = tid; idx < BT * D; idx += kThreads) {
      const int i = idx / D, e = idx % D;
      const int64_t pos = t0 + i;
      float intra = 0.f, inter = 0.f;
#pragma unroll 8
      for (int jj = 0; jj < BT; ++jj) intra = fmaf(A[i * (BT + 1) + jj], sc[jj * (D + 1) + e], intra);
#pragma unroll 8
      for (int d = 0; d < D; ++d) inter = fmaf(sa[i * (D + 1) + d], S[d * (D + 1) + e], inter);
      const float r = (DIR == Dir::FWD) ? pw[i + 1] : pw[BT - 1 - i];
      if (pos >= beg && pos < end) st(go + (b * p.C + pos) * rs + h * D + e, fmaf(r, inter, intra));
    }
    __syncthreads();
    // S = lam^BT S + sum_s u_s b_s c_s^T
    if (j + 1 < nblk) {
      for (int idx = tid; idx < D * D; idx += kThreads) {
        const int d = idx / D, e = idx % D;
        float acc = 0.f;
#pragma unroll 8
        for (int s = 0; s < BT; ++s) {
          const float u = (DIR == Dir::FWD) ? pw[BT - 1 - s] : pw[s + 1];
          acc = fmaf(u * sb[s * (D + 1) + d], sc[s * (D + 1) + e], acc);
        }
        S[d * (D + 1) + e] = fmaf(pw[BT], S[d * (D + 1) + e], acc);
      }
    }
    __syncthreads();
  }
}

template <typename T, int D>
cudaError_t seg_state_dispatch_dir(const Plan& p, Dir dir, const void* x, const void* y, float* out,
                                   cudaStream_t st) {
  dim3 grid((unsigned)p.nseg, (unsigned)p.H, (unsigned)p.B);
  if (dir == Dir::FWD)
    return launch_k(seg_state_simt_kernel<T, D, Dir::FWD>, grid, dim3(kThreads), 0, st, p, (const T*)x, (const T*)y, out);
  else
    return launch_k(seg_state_simt_kernel<T, D, Dir::REV>, grid, dim3(kThreads), 0, st, p, (const T*)x, (const T*)y, out);
  return cudaGetLastError();
}

template <typename T, int D, Dir DIR>
cudaError_t core_launch(const Plan& p, const SeqArgs& a, cudaStream_t st) {
  constexpr int BT = 32;
  const size_t smem = sizeof(float) * (3 * BT * (D + 1) + D * (D + 1) + BT * (BT + 1) + BT + 1);
  auto kern = core_simt_kernel<T, D, DIR>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  dim3 grid((unsigned)p.nseg, (unsigned)p.H, (unsigned)p.B);
  return launch_k(kern, grid, dim3(kThreads), smem, st, p, a);
}

template <typename T>
cudaError_t seg_state_dispatch(const Plan& p, Dir dir, const void* x, const void* y, float* out,
                               cudaStream_t st) {
  switch (p.D) {
    case 32: return seg_state_dispatch_dir<T, 32>(p, dir, x, y, out, st);
    case 64: return seg_state_dispatch_dir<T, 64>(p, dir, x, y, out, st);
    case 128: return seg_state_dispatch_dir<T, 128>(p, dir, x, y, out, st);
  }
  return cudaErrorInvalidValue;
}

template <typename T>
cudaError_t core_dispatch(const Plan& p, Dir dir, const SeqArgs& a, cudaStream_t st) {
  const bool f = dir == Dir::FWD;
  switch (p.D) {
    case 32: return f ? core_launch<T, 32, Dir::FWD>(p, a, st) : core_launch<T, 32, Dir::REV>(p, a, st);
    case 64: return f ? core_launch<T, 64, Dir::FWD>(p, a, st) : core_launch<T, 64, Dir::REV>(p, a, st);
    case 128: return f ? core_launch<T, 128, Dir::FWD>(p, a, st) : core_launch<T, 128, Dir::REV>(p, a, st);
  }
  return cudaErrorInvalidValue;
}

}  // namespace

cudaError_t launch_seg_state_simt(const Plan& p, Dir dir, const void* x, const void* y, float* out,
                                  cudaStream_t st) {
  return p.dtype == 0 ? seg_state_dispatch<__nv_bfloat16>(p, dir, x, y, out, st)
                      : seg_state_dispatch<float>(p, dir, x, y, out, st);
}

cudaError_t launch_core_simt(const Plan& p, Dir dir, const SeqArgs& a, cudaStream_t st) {
  return p.dtype == 0 ? core_dispatch<__nv_bfloat16>(p, dir, a, st) : core_dispatch<float>(p, dir, a, st);
}

cudaError_t launch_prefix(const Plan& p, Dir dir, const float* init, const float* seg_states, float* prefix_out,
                          float* final_out, cudaStream_t st) {
  const int64_t n = p.B * p.Hk * p.D * p.D / 4;  // D*D is a multiple of 4
  const int threads = 64;
  const dim3 grid((unsigned)((n + threads - 1) / threads));
  auto go = [&](auto kern) { return launch_k(kern, grid, dim3(threads), 0, st, p, init, seg_states, prefix_out, final_out); };
  auto by_u = [&](auto d_tag, auto dir_tag) {
    constexpr int D = decltype(d_tag)::value;
    constexpr Dir R = decltype(dir_tag)::value;
    if (p.nseg <= 8) return go(prefix_kernel<8, D, R>);
    if (p.nseg <= 16) return go(prefix_kernel<16, D, R>);
    if (p.nseg <= 24) return go(prefix_kernel<24, D, R>);
    return go(prefix_kernel<40, D, R>);
  };
  auto by_dir = [&](auto d_tag) {
    return dir == Dir::FWD ? by_u(d_tag, std::integral_constant<Dir, Dir::FWD>{})
                           : by_u(d_tag, std::integral_constant<Dir, Dir::REV>{});
  };
  if (p.D == 32) return by_dir(std::integral_constant<int, 32>{});
  if (p.D == 64) return by_dir(std::integral_constant<int, 64>{});
  if (p.D == 128) return by_dir(std::integral_constant<int, 128>{});
  return cudaErrorInvalidValue;
}

// All-gather exchange: fold the gathered per-rank local states of ranks
// j0, j0 + step, ... (count of them) in that order: cur = lam^C cur + g[j], starting from 0. Forward:
// KV_in(r) = sum_{j<r} lam^(C (r-1-j)) L_j (j0 = 0, step +1, count r); backward: dKV_in(r) =
// sum_{j>r} lam^(C (j-r-1)) G_j (j0 = T-1, step -1, count T-1-r). Same decay as combine_kernel.
// Each rank's n_local travels with its state (ranks may hold different lengths, reading R3): folding rank j
// in is cur = lam^(C_j) cur + g_j, the combine step rank j itself would have applied (Alg. 2).
__global__ void fold_ranks_kernel(Plan p, const float* __restrict__ g, int64_t stride, int j0, int step, int count,
                                  float* __restrict__ out) {
  pdl_wait();
  pdl_trigger();
  const int64_t n = p.B * p.Hk * p.D * p.D;
  const int64_t idx = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx >= n) return;
  const int64_t h = (idx / (p.D * p.D)) % p.Hk;
  float cur = 0.f;
  for (int t = 0; t < count; ++t) {
    const float* gj = g + int64_t(j0 + t * step) * stride;
    const int64_t Cj = *reinterpret_cast<const int64_t*>(gj + n);
    cur = fmaf(powk(p.lam[h], double(Cj)), cur, gj[idx]);
  }
  out[idx] = cur;
}

cudaError_t launch_fold_ranks(const Plan& p, const float* gathered, int64_t stride, int j0, int step, int count,
                              float* out, cudaStream_t st) {
  const int64_t n = p.B * p.Hk * p.D * p.D;
  const int threads = 256;
  return launch_k(fold_ranks_kernel, dim3((unsigned)((n + threads - 1) / threads)), dim3(threads), 0, st, p, gathered,
                  stride, j0, step, count, out);
}

// all-gather message of one rank: its state (n floats) followed by its n_local as an int64
__global__ void pack_state_kernel(int64_t n, int64_t C, const float* __restrict__ src, float* __restrict__ dst) {
  pdl_wait();
  pdl_trigger();
  const int64_t idx = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx < n) dst[idx] = src[idx];
  if (idx == 0) *reinterpret_cast<int64_t*>(dst + n) = C;
}

cudaError_t launch_pack_state(const Plan& p, const float* src, float* dst, cudaStream_t st) {
  const int64_t n = p.B * p.Hk * p.D * p.D;
  const int threads = 256;
  return launch_k(pack_state_kernel, dim3((unsigned)((n + threads - 1) / threads)), dim3(threads), 0, st, n, p.C, src,
                  dst);
}

// Norm epilogue, second phase at head_dim 128 (the two 64-wide value slices of a head row are separate core
// items): r = (mean o^2 + eps)^-1/2 from the slices' sums of squares, y = o r in place, r stored for the
// backward. One thread per 8 elements (16 B), 16 threads per (token, head) row.
__global__ void norm_apply_kernel(int64_t rows, float eps, __nv_bfloat16* __restrict__ y, const float* __restrict__ nsum,
                                  float* __restrict__ rnorm) {
  pdl_wait();
  pdl_trigger();
  const int64_t idx = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t row = idx >> 4;
  if (row >= rows) return;
  const float rn = 1.f / sqrtf((nsum[2 * row] + nsum[2 * row + 1]) * (1.f / 128.f) + eps);
  uint4* ptr = reinterpret_cast<uint4*>(y) + idx;
  uint4 v = *ptr;
  uint32_t* w = reinterpret_cast<uint32_t*>(&v);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    __nv_bfloat162 h2 = *reinterpret_cast<__nv_bfloat162*>(&w[i]);
    float2 f = __bfloat1622float2(h2);
    h2 = __floats2bfloat162_rn(f.x * rn, f.y * rn);
    w[i] = *reinterpret_cast<uint32_t*>(&h2);
  }
  *ptr = v;
  if ((idx & 15) == 0) rnorm[row] = rn;
}

cudaError_t launch_norm_apply(const Plan& p, void* y, const NormArgs& n, cudaStream_t st) {
  const int64_t rows = p.B * p.C * p.H;
  const int64_t threads = rows * 16;
  return launch_k(norm_apply_kernel, dim3((unsigned)((threads + 255) / 256)), dim3(256), 0, st, rows, n.eps,
                  static_cast<__nv_bfloat16*>(y), (const float*)n.nsum, n.rnorm);
}

// Entry kernel of every call: waits until everything before the call has completed (griddepcontrol.wait),
// only then lets the call's next kernel start (lasp_common.cuh, PDL), writes (forward) or checks (backward)
// the cache tag into the call's status word ctrl[2], and zeroes the call's counters (ctrl[0..1]: fused
// prefix fold; ctrl[3..15]: work-claim counters of the persistent kernels).
__global__ void tag_kernel(CacheTag t, uint64_t* __restrict__ hdr, unsigned check_mask, unsigned* __restrict__ ctrl) {
  pdl_wait();
  entry_duty(t, hdr, check_mask, ctrl);
  // trigger only after the control block is zeroed: the next kernel's CTAs claim work items from it as they start
  __threadfence();
  pdl_trigger();
}

cudaError_t launch_tag(const CacheTag& t, uint64_t* hdr, unsigned check_mask, unsigned* ctrl, cudaStream_t st) {
  return launch_k(tag_kernel, dim3(1), dim3(32), 0, st, t, hdr, check_mask, ctrl);
}

// ---- P2P exchange (LASP_EXCHANGE_P2P): the ring hop as ONE kernel over peer memory -------------------------
// Rank r's hop in direction dir (0: forward, KV from r-1 to r+1; 1: backward, dKV from r+1 to r-1):
//   e = my epoch + 1; wait until the upstream has put epoch e into my receive buffer (flag, acquire.sys);
//   copy it to the rank's private KV_in (the fold reads that); wait until the downstream has copied my previous
//   message (ack >= e - 1); store lam^C KV_in + local straight into the downstream rank's receive buffer
//   (NVLink stores to peer memory: combine and send fused); the last CTA then publishes the data flag to the
//   downstream (release.sys), the ack to the upstream, and my epoch. Epochs live in device memory, so the launch
//   can be captured into a CUDA graph and replayed. Flag words: [dir] data epoch, [2 + dir] ack, [4 + dir] my
//   epoch, [6 + dir] CTA-done counter. A small grid (kP2PCtas) keeps the spinning CTAs off most SMs.
__device__ __forceinline__ uint64_t ld_acquire_sys(const uint64_t* a) {
  uint64_t v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(a) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(uint64_t* a, uint64_t v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(a), "l"(v) : "memory");
}
__device__ __forceinline__ void spin_until_ge(const uint64_t* a, uint64_t target) {
  uint32_t n = 0;
  while (ld_acquire_sys(a) < target) {
    __nanosleep(128);
    if (++n == (1u << 28)) __trap();  // a peer that never arrives: fail loudly instead of hanging
  }
}

__global__ void p2p_hop_kernel(Plan p, P2PHop h) {
  // no early trigger: the next kernel (a persistent core launch holding whole SMs) must not start while this
  // one waits for a peer -- with several ranks on one device its CTAs would starve the peer's kernels
  pdl_wait();
  const int dir = h.dir;
  __shared__ uint64_t e_s;
  if (threadIdx.x == 0) {
    const uint64_t e = *reinterpret_cast<volatile uint64_t*>(&h.my_flags[4 + dir]) + 1;
    if (h.has_up) spin_until_ge(&h.my_flags[dir], e);
    if (h.peer_recv != nullptr) spin_until_ge(&h.my_flags[2 + dir], e - 1);
    e_s = e;
  }
  __syncthreads();
  const uint64_t e = e_s;
  const int64_t DD = p.D * p.D;
  for (int64_t idx = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; idx < h.n; idx += int64_t(gridDim.x) * blockDim.x) {
    const float in = h.has_up ? __ldcg(h.my_recv + idx) : 0.f;
    h.in_priv[idx] = in;
    if (h.peer_recv != nullptr) {
      const int64_t hd = (idx / DD) % p.Hk;
      h.peer_recv[idx] = fmaf(powk(p.lam[hd], double(p.C)), in, h.local[idx]);
    }
  }
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned long long done = atomicAdd(reinterpret_cast<unsigned long long*>(&h.my_flags[6 + dir]), 1ull) + 1ull;
    if (done == gridDim.x) {  // every CTA's copies and peer stores are fenced
      __threadfence_system();
      if (h.has_up) st_release_sys(&h.up_flags[2 + dir], e);      // ack: epoch e has been copied
      if (h.peer_recv != nullptr) st_release_sys(&h.peer_flags[dir], e);
      h.my_flags[6 + dir] = 0;
      st_release_sys(&h.my_flags[4 + dir], e);
    }
  }
}

// ---- P2P all-gather exchange (LASP_EXCHANGE_P2P_ALLGATHER): ONE kernel per direction and rank ---------------
// Forward on rank r: store this rank's local state L_r (and its n_local) into slot r of every later rank's gather
// block (peer memory), publish a data flag there; wait for the data flags of every earlier rank in this rank's
// block and fold what arrived, KV_in(r) = sum_{i<r} lam^(C_{i+1} + ... + C_{r-1}) L_i (cur = lam^(C_i) cur + L_i
// in rank order, the ring's combine applied rank by rank); acknowledge each earlier rank. Backward mirrors it
// (to the earlier ranks, from the later ones). A sender overwrites a slot only after that receiver acknowledged the
// previous epoch. Gather-block words: data [dir][src] at dir 64 + src, ack [dir][dst] at 128 + dir 64 + dst,
// epoch [dir] at 256 + dir, CTA-done counters at 258 + dir (send) / 260 + dir (fold); slots follow the 4 KB flags.
__device__ __forceinline__ uint64_t* gflag(char* base, int w) { return reinterpret_cast<uint64_t*>(base) + w; }
__device__ __forceinline__ float* gslot(const P2PGather& g, char* base, int dir, int src) {
  return reinterpret_cast<float*>(base + kP2PFlagBytes + (size_t(dir) * g.world + src) * g.slot_bytes);
}

__global__ void p2p_gather_kernel(Plan p, P2PGather g) {
  pdl_wait();  // no early trigger (see p2p_hop_kernel)
  const int dir = g.dir, r = g.rank, T = g.world;
  const int dlo = dir == 0 ? r + 1 : 0, dhi = dir == 0 ? T : r;      // downstream ranks [dlo, dhi)
  const int ulo = dir == 0 ? 0 : r + 1, uhi = dir == 0 ? r : T;      // upstream ranks [ulo, uhi)
  char* mine = g.bases[r];
  __shared__ uint64_t e_s;
  if (threadIdx.x == 0) {
    const uint64_t e = *reinterpret_cast<volatile uint64_t*>(gflag(mine, 256 + dir)) + 1;
    for (int j = dlo; j < dhi; ++j) spin_until_ge(gflag(mine, 128 + dir * 64 + j), e - 1);
    e_s = e;
  }
  __syncthreads();
  const uint64_t e = e_s;
  // send: this rank's local state into slot r of every downstream rank
  for (int64_t idx = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; idx < g.n; idx += int64_t(gridDim.x) * blockDim.x) {
    const float v = g.local[idx];
    for (int j = dlo; j < dhi; ++j) gslot(g, g.bases[j], dir, r)[idx] = v;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0)
    for (int j = dlo; j < dhi; ++j) *reinterpret_cast<int64_t*>(gslot(g, g.bases[j], dir, r) + g.n) = p.C;
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned long long done = atomicAdd(reinterpret_cast<unsigned long long*>(gflag(mine, 258 + dir)), 1ull) + 1ull;
    if (done == gridDim.x) {
      __threadfence_system();
      for (int j = dlo; j < dhi; ++j) st_release_sys(gflag(g.bases[j], dir * 64 + r), e);
      *gflag(mine, 258 + dir) = 0;
    }
    for (int i = ulo; i < uhi; ++i) spin_until_ge(gflag(mine, dir * 64 + i), e);
  }
  __syncthreads();
  // fold what the upstream ranks sent, in rank order along the direction
  const int64_t DD = p.D * p.D;
  for (int64_t idx = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; idx < g.n; idx += int64_t(gridDim.x) * blockDim.x) {
    const int64_t hd = (idx / DD) % p.Hk;
    float cur = 0.f;
    for (int t = 0; t < uhi - ulo; ++t) {
      const int i = dir == 0 ? ulo + t : uhi - 1 - t;
      const float* sl = gslot(g, mine, dir, i);
      const int64_t Ci = __ldcg(reinterpret_cast<const long long*>(sl + g.n));
      cur = fmaf(powk(p.lam[hd], double(Ci)), cur, __ldcg(sl + idx));
    }
    g.in_priv[idx] = cur;
  }
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned long long done = atomicAdd(reinterpret_cast<unsigned long long*>(gflag(mine, 260 + dir)), 1ull) + 1ull;
    if (done == gridDim.x) {
      __threadfence_system();
      for (int i = ulo; i < uhi; ++i) st_release_sys(gflag(g.bases[i], 128 + dir * 64 + r), e);
      *gflag(mine, 260 + dir) = 0;
      st_release_sys(gflag(mine, 256 + dir), e);
    }
  }
}

cudaError_t launch_p2p_gather(const Plan& p, const P2PGather& g, cudaStream_t st) {
  return launch_k(p2p_gather_kernel, dim3(kP2PCtas), dim3(256), 0, st, p, g);
}

cudaError_t launch_p2p_hop(const Plan& p, const P2PHop& h, cudaStream_t st) {
  return launch_k(p2p_hop_kernel, dim3(kP2PCtas), dim3(256), 0, st, p, h);
}

cudaError_t launch_combine(const Plan& p, const float* kv_in, const float* local, float* kv_out, cudaStream_t st) {
  const int64_t n = p.B * p.Hk * p.D * p.D;
  const int threads = 256;
  return launch_k(combine_kernel, dim3((unsigned)((n + threads - 1) / threads)), dim3(threads), 0, st, p, kv_in, local,
                  kv_out);
}

}  // namespace lasp
