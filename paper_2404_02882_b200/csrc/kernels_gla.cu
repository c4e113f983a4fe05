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
// exponent-range restriction). One CTA per (batch, head, segment) item; each thread owns a 2-D tile of the state
// in registers (GlaCfg). The tokens' vectors are staged in shared memory 16 at a time (cp.async, double-buffered)
// and read as warp broadcasts.
#include "lasp_common.cuh"
#include "gla.cuh"

#include <algorithm>
#include <type_traits>

namespace lasp {
namespace {

// tokens per shared-memory tile (double-buffered with cp.async): smaller tiles leave room for more co-resident
// CTAs, which wins at head_dim <= 64 (same-box sweep, profiles/r3k / r3l: TNL-0.4B shape 4 / 8 / 16 / 32 tokens
// 16.4 / 14.5 / 12.1 / 8.5 M tokens/s) while head_dim 128 prefers 8 (3.82 / 3.96 / 3.62 / 3.0)
template <int D>
constexpr int gla_gt() { return D <= 64 ? 4 : 8; }

// Each thread owns an OSPAN x RSPAN tile of the D x D state: OSPAN output indices (the value column for the
// F1 / F3 / B1 / dV passes, the key row for dQ / dK) by RSPAN indices of the dimension the outputs reduce over.
// The NRED = D / RSPAN threads sharing the same outputs are adjacent lanes and combine their partial dot
// products with xor-shuffles. A thread's reduce indices are interleaved with its NRED partners' at float4
// granularity (chunk c of thread rg covers indices 4 (c NRED + rg) .. +3), so the partners' vector loads hit
// consecutive 16-byte words (no bank conflicts). Per token a thread reads 2-3 RSPAN-vectors and one OSPAN-vector from shared memory
// (warp broadcasts) for 2-3 x 64 FP32 instructions.
#ifndef LASP_GLA_OS64
#define LASP_GLA_OS64 4
#define LASP_GLA_RS64 16
#endif
template <int D>
struct GlaCfg {
  static constexpr int GT = gla_gt<D>();
  static constexpr int OSPAN = D == 128 ? 2 : D == 64 ? LASP_GLA_OS64 : 4;
  static constexpr int RSPAN = D == 32 ? 8 : D == 64 ? LASP_GLA_RS64 : 32;
  static constexpr int NRED = D / RSPAN;                 // 4
  static constexpr int NT = (D / OSPAN) * NRED;          // 32, 64, 256 threads per item
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
  constexpr int NT = GlaCfg<D>::NT, V4 = D / 4, GT = GlaCfg<D>::GT;
#pragma unroll
  for (int x = 0; x < NX; ++x)
    for (int i = threadIdx.x; i < GT * V4; i += NT) {
      const int r = i / V4, c4 = i % V4;
      const int64_t t = t0 + r;
      const bool ok = t >= s0 && t < s1;
      cp16(buf + (size_t(x) * GT + r) * D + c4 * 4, ok ? src[x] + row_off(p, b, t, h) + c4 * 4 : src[x], ok);
    }
}

template <int NRED>
__device__ __forceinline__ float red_sum(float x) {
#pragma unroll
  for (int m = 1; m < NRED; m <<= 1) x += __shfl_xor_sync(0xffffffffu, x, m);
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
  return (2 * size_t(GlaTensors<MODE>::NX) + 1) * GlaCfg<D>::GT * D * sizeof(float);
}

template <int D, int MODE>
__global__ void __launch_bounds__(GlaCfg<D>::NT) gla_kernel(const GlaArgs a) {
  using Cfg = GlaCfg<D>;
  constexpr int OS = Cfg::OSPAN, RS = Cfg::RSPAN, NRED = Cfg::NRED, GT = Cfg::GT;
  constexpr bool REV = MODE == G_B1 || MODE == G_DV || MODE == G_DK;
  constexpr bool ROWS = MODE == G_DQ || MODE == G_DK;  // outputs indexed by the key row (else the value column)
  constexpr int NX = GlaTensors<MODE>::NX, LGX = GlaTensors<MODE>::LGX;
  extern __shared__ __align__(16) float smem[];
  float* raw = smem;                            // [2][NX][GT][D] double-buffered token tiles
  float* gb = smem + 2 * NX * GT * D;           // [GT][D] g = exp(lg) of the tile being computed

  pdl_wait();  // inputs and states come from the preceding kernels (never triggered early by this path)
  const GlaPlan& p = a.p;
  const int64_t item = blockIdx.x;
  const int64_t seg = item % p.nseg, bh = item / p.nseg, b = bh / p.H, h = bh % p.H;
  const int64_t s0 = seg * p.seg_len, s1 = (s0 + p.seg_len < p.C) ? s0 + p.seg_len : p.C;
  const int tid = int(threadIdx.x);
  const int ob = (tid / NRED) * OS;      // first output index of this thread
  const int rg = tid % NRED;             // reduce group: indices 4 (c NRED + rg) + u, c < RS / 4, u < 4
  const bool lead = tid % NRED == 0;     // writes the reduced outputs
  const size_t seg_off = (size_t(bh) * size_t(p.nseg) + size_t(seg)) * size_t(p.D) * size_t(p.D);
  // state element (output j, reduce i) <-> S[d][e]: column modes d = ridx(i), e = ob + j; row modes d = ob + j,
  // e = ridx(i)
  auto ridx = [&](int i) -> int { return ((i >> 2) * NRED + rg) * 4 + (i & 3); };
  auto sidx = [&](int j, int i) -> size_t {
    return ROWS ? size_t(ob + j) * D + size_t(ridx(i)) : size_t(ridx(i)) * D + size_t(ob + j);
  };
  // RS consecutive reduce-index values of a [D] shared-memory vector into registers
  auto rvec = [&](float* dst, const float* src) {
#pragma unroll
    for (int i = 0; i < RS; i += 4)
      *reinterpret_cast<float4*>(dst + i) = *reinterpret_cast<const float4*>(src + ridx(i));
  };

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

  float st[OS][RS];
  // ---- initial state (loads overlap the first tile's copies)
  if constexpr (MODE == G_F1 || MODE == G_B1) {
#pragma unroll
    for (int j = 0; j < OS; ++j)
#pragma unroll
      for (int i = 0; i < RS; ++i) st[j][i] = 0.f;
  } else {
    const float* init;
    if constexpr (MODE == G_F3 || MODE == G_DQ)
      init = a.cache + (size_t(bh) * size_t(p.nseg + 1) + size_t(seg)) * size_t(p.D) * size_t(p.D);
    else
      init = a.seg + seg_off;  // R_p
    const bool poison = a.status != nullptr && tag_poisoned(a.status);
#pragma unroll
    for (int j = 0; j < OS; ++j)
#pragma unroll
      for (int i = 0; i < RS; ++i) st[j][i] = poison ? __int_as_float(0x7fc00000) : init[sidx(j, i)];
  }
  float run[OS];  // DK: suffix sums of q . dq - k . dk (rows ob..ob+OS); F1 / B1: sum of lg (index tid)
#pragma unroll
  for (int j = 0; j < OS; ++j) run[j] = 0.f;
  if constexpr (MODE == G_DK) {
    const float* pn = a.cache + (size_t(bh) * size_t(p.nseg + 1) + size_t(seg + 1)) * size_t(p.D) * size_t(p.D);
#pragma unroll
    for (int j = 0; j < OS; ++j) {
      float c = 0.f;
#pragma unroll
      for (int i = 0; i < RS; ++i) c = fmaf(st[j][i], pn[sidx(j, i)], c);
      run[j] = red_sum<NRED>(c);  // <R_p[d, :], P_{p+1}[d, :]>: dlg summed over the tokens after this segment
    }
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
      for (int i = tid; i < GT * D / 4; i += Cfg::NT) {
        const float4 l4 = reinterpret_cast<const float4*>(lgt)[i];
        reinterpret_cast<float4*>(gb)[i] = make_float4(__expf(l4.x), __expf(l4.y), __expf(l4.z), __expf(l4.w));
      }
    }
    __syncthreads();
    const int64_t t0 = tile_t0(ti);
    auto T = [&](int x, int r) -> const float* { return cur + (size_t(x) * GT + r) * D; };
    // vec<N>(ptr): N consecutive floats from shared memory (float4 broadcasts) into registers
    for (int rr = 0; rr < GT; ++rr) {
      const int r = REV ? GT - 1 - rr : rr;
      const int64_t t = t0 + r;
      if (t < s0 || t >= s1) continue;  // (uniform across the CTA)
      const float* g = gb + size_t(r) * D;
      float o[OS];
      if constexpr (MODE == G_F1 || MODE == G_F3) {
        // S[d][e] = g[d] S[d][e] + k[d] v[e]; (F3) o[e] = sum_d q[d] S[d][e]    (e outputs, d reduce)
        float gv[RS], kv[RS], vo[OS];
        rvec(gv, g);
        rvec(kv, T(MODE == G_F1 ? 0 : 1, r));
#pragma unroll
        for (int j = 0; j < OS; ++j) vo[j] = T(MODE == G_F1 ? 1 : 2, r)[ob + j];  // (consecutive: vectorized)
#pragma unroll
        for (int j = 0; j < OS; ++j)
#pragma unroll
          for (int i = 0; i < RS; ++i) st[j][i] = fmaf(gv[i], st[j][i], kv[i] * vo[j]);
        if constexpr (MODE == G_F3) {
          float qv[RS];
          rvec(qv, T(0, r));
#pragma unroll
          for (int j = 0; j < OS; ++j) {
            float x0 = 0.f, x1 = 0.f;
#pragma unroll
            for (int i = 0; i < RS; i += 2) {
              x0 = fmaf(qv[i], st[j][i], x0);
              x1 = fmaf(qv[i + 1], st[j][i + 1], x1);
            }
            o[j] = red_sum<NRED>(x0 + x1);
          }
          if (lead) {
            float* dst = a.out + row_off(p, b, t, h) + ob;
#pragma unroll
            for (int j = 0; j < OS; ++j) dst[j] = o[j];
          }
        }
      } else if constexpr (MODE == G_DQ) {
        // S[d][e] = g[d] S[d][e] + k[d] v[e]; dq[d] = sum_e S[d][e] do[e]    (d outputs, e reduce)
        float vv[RS], dv[RS], gd[OS], kd[OS];
        rvec(vv, T(1, r));
        rvec(dv, T(2, r));
#pragma unroll
        for (int j = 0; j < OS; ++j) { gd[j] = g[ob + j]; kd[j] = T(0, r)[ob + j]; }
#pragma unroll
        for (int j = 0; j < OS; ++j) {
          float x0 = 0.f, x1 = 0.f;
#pragma unroll
          for (int i = 0; i < RS; i += 2) {
            st[j][i] = fmaf(gd[j], st[j][i], kd[j] * vv[i]);
            st[j][i + 1] = fmaf(gd[j], st[j][i + 1], kd[j] * vv[i + 1]);
            x0 = fmaf(st[j][i], dv[i], x0);
            x1 = fmaf(st[j][i + 1], dv[i + 1], x1);
          }
          o[j] = red_sum<NRED>(x0 + x1);
        }
        if (lead) {
          float* dst = a.out + row_off(p, b, t, h) + ob;
#pragma unroll
          for (int j = 0; j < OS; ++j) dst[j] = o[j];
        }
      } else if constexpr (MODE == G_B1 || MODE == G_DV) {
        // S[d][e] += q[d] do[e]; (DV) dv[e] = sum_d S[d][e] k[d]; S[d][e] *= g[d]    (e outputs, d reduce)
        float qv[RS], gv[RS], dj[OS];
        rvec(qv, T(0, r));
        rvec(gv, g);
#pragma unroll
        for (int j = 0; j < OS; ++j) dj[j] = T(1, r)[ob + j];
#pragma unroll
        for (int j = 0; j < OS; ++j)
#pragma unroll
          for (int i = 0; i < RS; ++i) st[j][i] = fmaf(qv[i], dj[j], st[j][i]);
        if constexpr (MODE == G_DV) {
          float kv[RS];
          rvec(kv, T(2, r));
#pragma unroll
          for (int j = 0; j < OS; ++j) {
            float x0 = 0.f, x1 = 0.f;
#pragma unroll
            for (int i = 0; i < RS; i += 2) {
              x0 = fmaf(st[j][i], kv[i], x0);
              x1 = fmaf(st[j][i + 1], kv[i + 1], x1);
            }
            o[j] = red_sum<NRED>(x0 + x1);
          }
          if (lead) {
            float* dst = a.out + row_off(p, b, t, h) + ob;
#pragma unroll
            for (int j = 0; j < OS; ++j) dst[j] = o[j];
          }
        }
#pragma unroll
        for (int j = 0; j < OS; ++j)
#pragma unroll
          for (int i = 0; i < RS; ++i) st[j][i] *= gv[i];
      } else {  // G_DK
        // S[d][e] += q[d] do[e]; dk[d] = sum_e S[d][e] v[e]; dlg[d] = run + q[d] dq[d] - k[d] dk[d]; S *= g[d]
        float dv[RS], vv[RS], qd[OS];
        rvec(dv, T(1, r));
        rvec(vv, T(2, r));
#pragma unroll
        for (int j = 0; j < OS; ++j) qd[j] = T(0, r)[ob + j];
#pragma unroll
        for (int j = 0; j < OS; ++j) {
          float x0 = 0.f, x1 = 0.f;
          const float gj = g[ob + j];
#pragma unroll
          for (int i = 0; i < RS; i += 2) {
            st[j][i] = fmaf(qd[j], dv[i], st[j][i]);
            st[j][i + 1] = fmaf(qd[j], dv[i + 1], st[j][i + 1]);
            x0 = fmaf(st[j][i], vv[i], x0);
            x1 = fmaf(st[j][i + 1], vv[i + 1], x1);
            st[j][i] *= gj;
            st[j][i + 1] *= gj;
          }
          o[j] = red_sum<NRED>(x0 + x1);
        }
        if (lead) {
          const size_t off = row_off(p, b, t, h) + ob;
#pragma unroll
          for (int j = 0; j < OS; ++j) {
            run[j] += fmaf(qd[j], T(4, r)[ob + j], -T(5, r)[ob + j] * o[j]);
            a.out[off + j] = o[j];
            a.dlg[off + j] = run[j];
          }
        }
      }
      if constexpr (MODE == G_F1 || MODE == G_B1) {
        if (tid < D) run[0] += T(LGX, r)[tid];
      }
    }
  }
  // ---- segment results
  if constexpr (MODE == G_F1 || MODE == G_B1) {
    // F1: L_p; B1: G'_p = Diag(g_{s_p}) dkv_{s_p} (the loop already applied g of every token down to s_p)
    float* dst = a.seg + seg_off;
#pragma unroll
    for (int j = 0; j < OS; ++j)
#pragma unroll
      for (int i = 0; i < RS; ++i) dst[sidx(j, i)] = st[j][i];
    if (tid < D) a.ls[(size_t(bh) * size_t(p.nseg) + size_t(seg)) * size_t(p.D) + tid] = run[0];
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

int gla_slots_per_sm(int D) {
  // the fewest co-resident CTAs per SM over the passes (the segment count is common to all of them)
  auto occ = [](auto kern, size_t smem, int nt) {
    int n = 0;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kern, nt, smem) != cudaSuccess) n = 1;
    return n > 0 ? n : 1;
  };
  auto all = [&](auto dtag) {
    constexpr int DD = decltype(dtag)::value;
    constexpr int NT = GlaCfg<DD>::NT;
    int m = occ(gla_kernel<DD, G_F1>, gla_smem_bytes<DD, G_F1>(), NT);
    m = std::min(m, occ(gla_kernel<DD, G_F3>, gla_smem_bytes<DD, G_F3>(), NT));
    m = std::min(m, occ(gla_kernel<DD, G_DQ>, gla_smem_bytes<DD, G_DQ>(), NT));
    m = std::min(m, occ(gla_kernel<DD, G_DK>, gla_smem_bytes<DD, G_DK>(), NT));
    return m;
  };
  static int cache[3] = {0, 0, 0};
  const int k = D == 32 ? 0 : D == 64 ? 1 : 2;
  if (cache[k] == 0)
    cache[k] = D == 32 ? all(std::integral_constant<int, 32>{}) : D == 64 ? all(std::integral_constant<int, 64>{})
                                                                          : all(std::integral_constant<int, 128>{});
  return cache[k];
}

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
