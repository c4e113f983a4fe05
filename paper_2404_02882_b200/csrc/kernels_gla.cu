// kernels_gla.cu -- generalised decay: the GLA / GateLoop row of Table 3 (App. A.4,
// P:671-713 general form m_t = o_t m_{t-1} + e_t i_t^T):
//
//   kv_t = Diag(g_t) kv_{t-1} + k_t v_t^T,   o_t = kv_t^T q_t,   g_t = exp(lg_t) in (0, 1]^D
//
// per token and key channel (a per-channel constant decay is lg_t = log lambda). fp32 in, fp32 out.
//
// LASP decomposition (the same Alg. 2 / 3 structure as the scalar path, with a diagonal decay per key row):
//   F1  L_p   = the recurrence from zero over segment p;      ls_p[d] = sum_{t in p} lg_t[d]
//   F2  P_0 = KV_in,  P_{p+1} = Diag(exp(ls_p)) P_p + L_p      (P_p = state entering segment p: the cache;
//                                                               P_nseg = KV_out, also kept in the cache)
//   F3  o_t: the recurrence over segment p started from P_p
//   B1  G'_p = Diag(g_{s_p}) (sum over segment p of the reverse recurrence dkv_t = q_t do_t^T +
//             Diag(g_{t+1}) dkv_{t+1}, from zero)
//   B2  R_{nseg-1} = dKV_in,  R_{p-1} = G'_p + Diag(exp(ls_p)) R_p   (R_p = dL/d kv_{e_p} from the tokens after
//       segment p, i.e. Diag(g_{e_p+1}) dkv_{e_p+1}; dKV_out = R_{-1}; the same definition of the message as the
//       scalar path: the gradient of the later ranks' loss w.r.t. the state leaving the rank)
//   B3  dQ (FWD, from P_p): dq_t = kv_t do_t;   dV (REV, from R_p): dv_t = dkv_t^T k_t;
//       dK (REV, from R_p): dk_t = dkv_t v_t and the decay gradient
//         dlg_t = sum_{u >= t} (q_u . dq_u - k_u . dk_u)          (elementwise products)
//       whose sum over the tokens after segment p is <R_p[d, :], P_{p+1}[d, :]> (the gradient through
//       kv_{e_p+1} = Diag(g_{e_p+1}) kv_{e_p} + ...), so no extra exchange is needed.
//
// Kernels run the recurrences token by token on CUDA cores (fp32 FFMA, exact: no decay is ever inverted, no
// exponent-range restriction). One CTA per (batch, head, segment) item; each thread owns one state column
// (F1, F3, B1, dV: the output / update index is the column) or one state row (dQ, dK), split over two
// threads at head_dim 128 (64 registers each, partial dot products combined with one shuffle). The tokens'
// vectors are staged in shared memory 16 at a time and read as warp-broadcasts.
#include "lasp_common.cuh"
#include "gla.cuh"

namespace lasp {
namespace {

constexpr int GT = 16;  // tokens per shared-memory tile (double-buffered with cp.async)

template <int D>
struct GlaCfg {
  static constexpr int RPT = D > 64 ? 64 : D;  // state elements per thread
  static constexpr int TPC = D / RPT;          // threads per state column / row (1 or 2)
  static constexpr int NT = D * TPC;           // threads per item
};

enum GlaMode : int { G_F1 = 0, G_F3 = 1, G_B1 = 2, G_DQ = 3, G_DV = 4, G_DK = 5 };

struct GlaArgs {
  GlaPlan p;
  const float* q; const float* k; const float* v; const float* lg; const float* d_o; const float* dq_in;
  float* out;          // o (F3), dq (DQ), dv (DV), dk (DK)
  float* dlg;          // DK
  float* seg;          // F1: L_p, B1: G'_p (write); DV / DK: R_p (read)
  float* ls;           // [B][H][nseg][D] segment log-decay sums (F1 / B1 write)
  const float* cache;  // [B][H][nseg + 1][D][D]: P_p (F3, DQ read; DK reads P_{p+1})
  const unsigned* status;  // backward cache-tag status (poison), or nullptr
};

__device__ __forceinline__ size_t row_off(const GlaPlan& p, int64_t b, int64_t t, int64_t h) {
  return size_t(((b * p.C + t) * p.H + h) * p.D);
}

// async copy of 16 bytes global -> shared (zero-filled when !valid)
__device__ __forceinline__ void cp16(float* dst, const float* src, bool valid) {
  const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(dst));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(d), "l"(src), "r"(valid ? 16 : 0) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_wait_prev() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }

// issue the async copies of tokens [t0, t0 + GT) of NX tensors into buf[NX][GT][D] (zeros outside [s0, s1))
template <int D, int NX>
__device__ __forceinline__ void stage_tile(const GlaPlan& p, int64_t b, int64_t h, int64_t t0, int64_t s0, int64_t s1,
                                           const float* const (&src)[NX], float* buf) {
  constexpr int NT = GlaCfg<D>::NT, V4 = D / 4;
  for (int i = threadIdx.x; i < NX * GT * V4; i += NT) {
    const int x = i / (GT * V4), r = (i / V4) % GT, c4 = i % V4;
    const int64_t t = t0 + r;
    const bool ok = t >= s0 && t < s1;
    cp16(buf + (size_t(x) * GT + r) * D + c4 * 4, ok ? src[x] + row_off(p, b, t, h) + c4 * 4 : src[x], ok);
  }
}

template <int TPC>
__device__ __forceinline__ float pair_sum(float x) {
  if constexpr (TPC == 2) x += __shfl_xor_sync(0xffffffffu, x, 1);
  return x;
}

// staged tensors per mode (the log decay is always index LGX; dK also stages dq and k)
template <int MODE> struct GlaTensors;
template <> struct GlaTensors<0> { static constexpr int NX = 3, LGX = 2; };  // F1: k, v, lg
template <> struct GlaTensors<1> { static constexpr int NX = 4, LGX = 3; };  // F3: q, k, v, lg
template <> struct GlaTensors<2> { static constexpr int NX = 3, LGX = 2; };  // B1: q, do, lg
template <> struct GlaTensors<3> { static constexpr int NX = 4, LGX = 3; };  // DQ: k, v, do, lg
template <> struct GlaTensors<4> { static constexpr int NX = 4, LGX = 3; };  // DV: q, do, k, lg
template <> struct GlaTensors<5> { static constexpr int NX = 6, LGX = 3; };  // DK: q, do, v, lg, dq, k

template <int D, int MODE>
constexpr size_t gla_smem_bytes() {
  return (2 * size_t(GlaTensors<MODE>::NX) + 1) * GT * D * sizeof(float);
}

template <int D, int MODE>
__global__ void __launch_bounds__(GlaCfg<D>::NT) gla_kernel(const GlaArgs a) {
  using Cfg = GlaCfg<D>;
  constexpr int RPT = Cfg::RPT, TPC = Cfg::TPC;
  constexpr bool REV = MODE == G_B1 || MODE == G_DV || MODE == G_DK;
  constexpr bool ROWS = MODE == G_DQ || MODE == G_DK;  // thread owns a state row (else a column)
  constexpr int NX = GlaTensors<MODE>::NX, LGX = GlaTensors<MODE>::LGX;
  extern __shared__ __align__(16) float smem[];
  float* raw = smem;                            // [2][NX][GT][D] double-buffered token tiles
  float* gb = smem + 2 * NX * GT * D;           // [GT][D] g = exp(lg) of the tile being computed

  pdl_wait();  // inputs and states come from the preceding kernels (never triggered early by this path)
  const GlaPlan& p = a.p;
  const int64_t item = blockIdx.x;
  const int64_t seg = item % p.nseg, bh = item / p.nseg, b = bh / p.H, h = bh % p.H;
  const int64_t s0 = seg * p.seg_len, s1 = (s0 + p.seg_len < p.C) ? s0 + p.seg_len : p.C;
  const int own = int(threadIdx.x) / TPC;             // owned column (or row) index
  const int part = int(threadIdx.x) % TPC;            // which RPT-slice of the other index
  const int base = part * RPT;
  const size_t seg_off = (size_t(bh) * size_t(p.nseg) + size_t(seg)) * size_t(p.D) * size_t(p.D);

  const float* srcs[NX];
  if constexpr (MODE == G_F1) { srcs[0] = a.k; srcs[1] = a.v; srcs[2] = a.lg; }
  if constexpr (MODE == G_F3) { srcs[0] = a.q; srcs[1] = a.k; srcs[2] = a.v; srcs[3] = a.lg; }
  if constexpr (MODE == G_B1) { srcs[0] = a.q; srcs[1] = a.d_o; srcs[2] = a.lg; }
  if constexpr (MODE == G_DQ) { srcs[0] = a.k; srcs[1] = a.v; srcs[2] = a.d_o; srcs[3] = a.lg; }
  if constexpr (MODE == G_DV) { srcs[0] = a.q; srcs[1] = a.d_o; srcs[2] = a.k; srcs[3] = a.lg; }
  if constexpr (MODE == G_DK) {
    srcs[0] = a.q; srcs[1] = a.d_o; srcs[2] = a.v; srcs[3] = a.lg; srcs[4] = a.dq_in; srcs[5] = a.k;
  }
  const int64_t ntile = (s1 - s0 + GT - 1) / GT;
  auto tile_t0 = [&](int64_t ti) { return REV ? s1 - (ti + 1) * GT : s0 + ti * GT; };  // REV tiles end at s1
  if (ntile > 0) stage_tile<D, NX>(p, b, h, tile_t0(0), s0, s1, srcs, raw);
  cp_commit();

  float st[RPT];
  // ---- initial state (loads overlap the first tile's copies)
  if constexpr (MODE == G_F1 || MODE == G_B1) {
#pragma unroll
    for (int r = 0; r < RPT; ++r) st[r] = 0.f;
  } else {
    const float* init;
    if constexpr (MODE == G_F3 || MODE == G_DQ)
      init = a.cache + (size_t(bh) * size_t(p.nseg + 1) + size_t(seg)) * size_t(p.D) * size_t(p.D);
    else
      init = a.seg + seg_off;  // R_p
#pragma unroll
    for (int r = 0; r < RPT; ++r)
      st[r] = ROWS ? init[size_t(own) * D + base + r] : init[size_t(base + r) * D + own];
    if (a.status != nullptr && tag_poisoned(a.status)) {
#pragma unroll
      for (int r = 0; r < RPT; ++r) st[r] = __int_as_float(0x7fc00000);
    }
  }
  float run = 0.f;  // DK: suffix sum of q . dq - k . dk (this row); F1 / B1: sum of lg (this column index)
  if constexpr (MODE == G_DK) {
    const float* pn = a.cache + (size_t(bh) * size_t(p.nseg + 1) + size_t(seg + 1)) * size_t(p.D) * size_t(p.D);
    float c = 0.f;
#pragma unroll
    for (int r = 0; r < RPT; ++r) c = fmaf(st[r], pn[size_t(own) * D + base + r], c);
    run = pair_sum<TPC>(c);  // <R_p[d, :], P_{p+1}[d, :]>: dlg summed over the tokens after this segment
  }

  for (int64_t ti = 0; ti < ntile; ++ti) {
    float* cur = raw + size_t(ti & 1) * NX * GT * D;
    __syncthreads();  // every thread is done with the other buffer (tile ti - 1) and with gb
    if (ti + 1 < ntile) stage_tile<D, NX>(p, b, h, tile_t0(ti + 1), s0, s1, srcs, raw + size_t((ti + 1) & 1) * NX * GT * D);
    cp_commit();
    cp_wait_prev();   // this thread's copies of tile ti have landed
    __syncthreads();  // ... and everybody's
    {
      const float* lgt = cur + size_t(LGX) * GT * D;
      for (int i = threadIdx.x; i < GT * D / 4; i += Cfg::NT) {
        const float4 l4 = reinterpret_cast<const float4*>(lgt)[i];
        reinterpret_cast<float4*>(gb)[i] = make_float4(__expf(l4.x), __expf(l4.y), __expf(l4.z), __expf(l4.w));
      }
    }
    __syncthreads();
    const int64_t t0 = tile_t0(ti);
    auto T = [&](int x, int r) -> const float* { return cur + (size_t(x) * GT + r) * D; };
    for (int rr = 0; rr < GT; ++rr) {
      const int r = REV ? GT - 1 - rr : rr;
      const int64_t t = t0 + r;
      if (t < s0 || t >= s1) continue;  // (uniform across the CTA)
      const float* g = gb + size_t(r) * D;
      if constexpr (MODE == G_F1 || MODE == G_F3) {
        // kv = Diag(g_t) kv + k_t v_t^T (column `own`), then (F3) o_t[own] = sum_d q_t[d] kv[d][own]
        const float* kk = T(MODE == G_F1 ? 0 : 1, r);
        const float vj = T(MODE == G_F1 ? 1 : 2, r)[own];
        float acc[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int i = 0; i < RPT; i += 4) {
          const float4 g4 = *reinterpret_cast<const float4*>(g + base + i);
          const float4 k4 = *reinterpret_cast<const float4*>(kk + base + i);
          st[i] = fmaf(g4.x, st[i], k4.x * vj);
          st[i + 1] = fmaf(g4.y, st[i + 1], k4.y * vj);
          st[i + 2] = fmaf(g4.z, st[i + 2], k4.z * vj);
          st[i + 3] = fmaf(g4.w, st[i + 3], k4.w * vj);
          if constexpr (MODE == G_F3) {
            const float4 q4 = *reinterpret_cast<const float4*>(T(0, r) + base + i);
            acc[0] = fmaf(q4.x, st[i], acc[0]);
            acc[1] = fmaf(q4.y, st[i + 1], acc[1]);
            acc[2] = fmaf(q4.z, st[i + 2], acc[2]);
            acc[3] = fmaf(q4.w, st[i + 3], acc[3]);
          }
        }
        if constexpr (MODE == G_F3) {
          const float o = pair_sum<TPC>((acc[0] + acc[1]) + (acc[2] + acc[3]));
          if (part == 0) a.out[row_off(p, b, t, h) + own] = o;
        }
        if constexpr (MODE == G_F1) if (part == 0) run += T(LGX, r)[own];
      } else if constexpr (MODE == G_DQ) {
        // row `own`: kv[own][:] = g_t[own] kv[own][:] + k_t[own] v_t[:], dq_t[own] = sum_e kv[own][e] do_t[e]
        const float gi = g[own], ki = T(0, r)[own];
        float acc[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int i = 0; i < RPT; i += 4) {
          const float4 v4 = *reinterpret_cast<const float4*>(T(1, r) + base + i);
          const float4 d4 = *reinterpret_cast<const float4*>(T(2, r) + base + i);
          st[i] = fmaf(gi, st[i], ki * v4.x);
          st[i + 1] = fmaf(gi, st[i + 1], ki * v4.y);
          st[i + 2] = fmaf(gi, st[i + 2], ki * v4.z);
          st[i + 3] = fmaf(gi, st[i + 3], ki * v4.w);
          acc[0] = fmaf(st[i], d4.x, acc[0]);
          acc[1] = fmaf(st[i + 1], d4.y, acc[1]);
          acc[2] = fmaf(st[i + 2], d4.z, acc[2]);
          acc[3] = fmaf(st[i + 3], d4.w, acc[3]);
        }
        const float o = pair_sum<TPC>((acc[0] + acc[1]) + (acc[2] + acc[3]));
        if (part == 0) a.out[row_off(p, b, t, h) + own] = o;
      } else if constexpr (MODE == G_B1 || MODE == G_DV) {
        // column `own`: dkv[:][own] += q_t[:] do_t[own]; (DV) dv_t[own] = sum_d dkv[d][own] k_t[d]; then
        // dkv *= g_t (the decay the next, earlier token sees: dkv_{t-1} = q do^T + Diag(g_t) dkv_t)
        const float dj = T(1, r)[own];
        float acc[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int i = 0; i < RPT; i += 4) {
          const float4 q4 = *reinterpret_cast<const float4*>(T(0, r) + base + i);
          const float4 g4 = *reinterpret_cast<const float4*>(g + base + i);
          st[i] = fmaf(q4.x, dj, st[i]);
          st[i + 1] = fmaf(q4.y, dj, st[i + 1]);
          st[i + 2] = fmaf(q4.z, dj, st[i + 2]);
          st[i + 3] = fmaf(q4.w, dj, st[i + 3]);
          if constexpr (MODE == G_DV) {
            const float4 k4 = *reinterpret_cast<const float4*>(T(2, r) + base + i);
            acc[0] = fmaf(st[i], k4.x, acc[0]);
            acc[1] = fmaf(st[i + 1], k4.y, acc[1]);
            acc[2] = fmaf(st[i + 2], k4.z, acc[2]);
            acc[3] = fmaf(st[i + 3], k4.w, acc[3]);
          }
          st[i] *= g4.x; st[i + 1] *= g4.y; st[i + 2] *= g4.z; st[i + 3] *= g4.w;
        }
        if constexpr (MODE == G_DV) {
          const float o = pair_sum<TPC>((acc[0] + acc[1]) + (acc[2] + acc[3]));
          if (part == 0) a.out[row_off(p, b, t, h) + own] = o;
        }
        if constexpr (MODE == G_B1) if (part == 0) run += T(LGX, r)[own];
      } else {  // G_DK
        // row `own`: dkv[own][:] += q_t[own] do_t[:]; dk_t[own] = sum_e dkv[own][e] v_t[e];
        // dlg_t[own] = (suffix) + q_t[own] dq_t[own] - k_t[own] dk_t[own]; dkv[own][:] *= g_t[own]
        const float qi = T(0, r)[own], gi = g[own];
        float acc[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int i = 0; i < RPT; i += 4) {
          const float4 d4 = *reinterpret_cast<const float4*>(T(1, r) + base + i);
          const float4 v4 = *reinterpret_cast<const float4*>(T(2, r) + base + i);
          st[i] = fmaf(qi, d4.x, st[i]);
          st[i + 1] = fmaf(qi, d4.y, st[i + 1]);
          st[i + 2] = fmaf(qi, d4.z, st[i + 2]);
          st[i + 3] = fmaf(qi, d4.w, st[i + 3]);
          acc[0] = fmaf(st[i], v4.x, acc[0]);
          acc[1] = fmaf(st[i + 1], v4.y, acc[1]);
          acc[2] = fmaf(st[i + 2], v4.z, acc[2]);
          acc[3] = fmaf(st[i + 3], v4.w, acc[3]);
          st[i] *= gi; st[i + 1] *= gi; st[i + 2] *= gi; st[i + 3] *= gi;
        }
        const float dk = pair_sum<TPC>((acc[0] + acc[1]) + (acc[2] + acc[3]));
        if (part == 0) {
          const size_t o = row_off(p, b, t, h) + own;
          run += fmaf(qi, T(4, r)[own], -T(5, r)[own] * dk);
          a.out[o] = dk;
          a.dlg[o] = run;
        }
      }
    }
  }
  // ---- segment results
  if constexpr (MODE == G_F1 || MODE == G_B1) {
    // F1: L_p column `own` (rows base..base+RPT); B1: G'_p = Diag(g_{s_p}) dkv_{s_p} (the loop already applied
    // g of every token down to s_p)
    float* dst = a.seg + seg_off;
#pragma unroll
    for (int r = 0; r < RPT; ++r) dst[size_t(base + r) * D + own] = st[r];
    if (part == 0) a.ls[(size_t(bh) * size_t(p.nseg) + size_t(seg)) * size_t(p.D) + own] = run;
  }
}

// F2 / B2 fold over segments, one thread per state element (b, h, d, e): see the file comment.
__global__ void gla_fold_kernel(GlaPlan p, int dir, const float* __restrict__ init, float* __restrict__ seg,
                                const float* __restrict__ ls, float* __restrict__ cache, float* __restrict__ fin,
                                float* __restrict__ lsum) {
  pdl_wait();
  const int64_t DD = p.D * p.D;
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= p.B * p.H * DD) return;
  const int64_t bh = i / DD, e = i % DD, d = e / p.D;
  float cur = init ? init[i] : 0.f;
  float tot = 0.f;
  if (dir == 0) {
    for (int64_t s = 0; s < p.nseg; ++s) {
      cache[(bh * (p.nseg + 1) + s) * DD + e] = cur;
      const float l = ls[(bh * p.nseg + s) * p.D + d];
      cur = fmaf(__expf(l), cur, seg[(bh * p.nseg + s) * DD + e]);
      tot += l;
    }
    cache[(bh * (p.nseg + 1) + p.nseg) * DD + e] = cur;  // P_nseg = KV_out (read by the dK pass)
  } else {
    for (int64_t s = p.nseg - 1; s >= 0; --s) {
      float* x = seg + (bh * p.nseg + s) * DD + e;
      const float gp = *x;
      *x = cur;  // R_s
      const float l = ls[(bh * p.nseg + s) * p.D + d];
      cur = fmaf(__expf(l), cur, gp);
      tot += l;
    }
  }
  if (fin) fin[i] = cur;
  if (lsum && e % p.D == 0) lsum[bh * p.D + d] = tot;
}

// ring hop: out = Diag(exp(lsum)) in + local (lsum: the rank's total log decay per key row)
__global__ void gla_combine_kernel(GlaPlan p, const float* __restrict__ in, const float* __restrict__ local,
                                   const float* __restrict__ lsum, float* __restrict__ out) {
  pdl_wait();
  const int64_t DD = p.D * p.D;
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= p.B * p.H * DD) return;
  const int64_t bh = i / DD, d = (i % DD) / p.D;
  out[i] = fmaf(__expf(lsum[bh * p.D + d]), in[i], local[i]);
}

template <int D, int MODE>
cudaError_t launch_mode(const GlaArgs& a, cudaStream_t st) {
  const int64_t items = a.p.B * a.p.H * a.p.nseg;
  constexpr size_t smem = gla_smem_bytes<D, MODE>();
  cudaError_t e = cudaFuncSetAttribute(gla_kernel<D, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  if (e != cudaSuccess) return e;
  return launch_k(gla_kernel<D, MODE>, dim3(unsigned(items)), dim3(GlaCfg<D>::NT), smem, st, a);
}

template <int MODE>
cudaError_t launch_d(const GlaArgs& a, cudaStream_t st) {
  switch (a.p.D) {
    case 32: return launch_mode<32, MODE>(a, st);
    case 64: return launch_mode<64, MODE>(a, st);
    case 128: return launch_mode<128, MODE>(a, st);
    default: return cudaErrorNotSupported;
  }
}

}  // namespace

cudaError_t gla_launch_state(const GlaPlan& p, int rev, const float* x, const float* y, const float* lg, float* seg,
                             float* ls, cudaStream_t st) {
  GlaArgs a{};
  a.p = p; a.lg = lg; a.seg = seg; a.ls = ls;
  if (rev) { a.q = x; a.d_o = y; return launch_d<G_B1>(a, st); }
  a.k = x; a.v = y;
  return launch_d<G_F1>(a, st);
}

cudaError_t gla_launch_fold(const GlaPlan& p, int rev, const float* init, float* seg, const float* ls, float* cache,
                            float* fin, float* lsum, cudaStream_t st) {
  const int64_t n = p.B * p.H * p.D * p.D;
  return launch_k(gla_fold_kernel, dim3(unsigned((n + 255) / 256)), dim3(256), 0, st, p, rev, init, seg, ls, cache,
                  fin, lsum);
}

cudaError_t gla_launch_combine(const GlaPlan& p, const float* in, const float* local, const float* lsum, float* out,
                               cudaStream_t st) {
  const int64_t n = p.B * p.H * p.D * p.D;
  return launch_k(gla_combine_kernel, dim3(unsigned((n + 255) / 256)), dim3(256), 0, st, p, in, local, lsum, out);
}

cudaError_t gla_launch_out(const GlaPlan& p, const float* q, const float* k, const float* v, const float* lg,
                           const float* cache, float* o, cudaStream_t st) {
  GlaArgs a{};
  a.p = p; a.q = q; a.k = k; a.v = v; a.lg = lg; a.cache = cache; a.out = o;
  return launch_d<G_F3>(a, st);
}

cudaError_t gla_launch_bwd(const GlaPlan& p, const float* q, const float* k, const float* v, const float* lg,
                           const float* d_o, const float* cache, float* rseg, float* dq, float* dk, float* dv,
                           float* dlg, const unsigned* status, cudaStream_t st) {
  GlaArgs a{};
  a.p = p; a.q = q; a.k = k; a.v = v; a.lg = lg; a.d_o = d_o; a.cache = cache; a.seg = rseg; a.status = status;
  a.out = dq;
  cudaError_t e = launch_d<G_DQ>(a, st);
  if (e != cudaSuccess) return e;
  a.out = dv;
  if ((e = launch_d<G_DV>(a, st)) != cudaSuccess) return e;
  a.out = dk; a.dlg = dlg; a.dq_in = dq;
  return launch_d<G_DK>(a, st);
}

}  // namespace lasp
