// kernels_tc.cu -- tcgen05 / TMEM / TMA kernels (sm_100a) of the LASP path, bf16 in / fp32 accumulate.
//
// Two kernels (see lasp_common.cuh for the FWD/REV formulas):
//
//  seg_state_tc  (F1 / B1): L = sum_pos w_pos x_pos y_pos^T over one segment. Per 128-token block:
//                TMA loads X, Y tiles -> 4 scaler warps multiply X rows by w in place -> one thread
//                issues UMMA (M = N = D, K = 128, both operands MN-major) accumulating in TMEM.
//                Eq. 12 for the forward, Eq. 21 for the backward.
//
//  core_tc       (F3 / B3): per (segment, pass, batch x head, 64-wide value slice) item, blocks of 128
//                tokens in direction order, with warp roles
//                  warp 0       TMA producer (a, b, c tiles; 3-stage ring at D = 64, 2 at D = 128)
//                  warp 2       UMMA issuer  S = a b^T             (M=128, N=128, K=D)   [Eq. 7]
//                  warp 3       UMMA issuer  dS = b^T (u.c)        (M=D,   N=64,  K=128) [Eq. 12]
//                  warp 1       UMMA issuer  O_intra = P c         (M=128, N=64,  K=128) [Eq. 7]
//                                            O_inter = a S_j       (M=128, N=64,  K=D)   [Eq. 9]
//                  warps 4-7    mask: S (TMEM) -> (.) M_lambda -> bf16 P (TMEM, over the consumed S)
//                  warps 8-11   state: u.c (smem), S_{j+1} = lambda^128 S_j + dS in fp32 registers,
//                               bf16 hi/lo copy of S_{j+1} for the next block's inter MMA
//                  warps 12-15  epilogue: out = O_intra + r (.) O_inter -> bf16 -> TMA store
//                The running state is the paper's KV (dKV) state applied between GPU blocks; the
//                segment's initial state comes from the prefix fold (KV_in of the ring included): the
//                prefix kernel (ring path), or -- local path -- the same fold run by warps 8-15 of this
//                launch before their roles start (claimed chunks, a done counter the readers wait on).
#include "lasp_common.cuh"
#include "sm100.cuh"

#include <cudaTypedefs.h>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>

namespace lasp {
using namespace sm100;

namespace {

constexpr int BT = 128;                 // tokens per block (UMMA M of the query side)
constexpr uint32_t BOX = BT * 128;      // one [128 rows][64 bf16] 128B-swizzled box = 16 KB

// ------------------------------------------------------------------------------------------------
// host: TMA tensor maps over the [B][C][H][D] bf16 layout (4-D: D, H, C, B), box [64][1][128][1]
PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult q;
    void* f = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  });
  return fn;
}

thread_local char g_tc_err[256];
unsigned long long* g_trace = nullptr;  // debug timeline buffer (lasp_debug_trace)

// heads: the tensor's head count (H for q, o, do, dq; Hk for k, v, dk, dv)
cudaError_t make_seq_map(CUtensorMap* m, const void* base, const Plan& p, int64_t heads) {
  auto fn = encode_fn();
  if (!fn) {
    snprintf(g_tc_err, sizeof g_tc_err, "cuTensorMapEncodeTiled entry point unavailable");
    return cudaErrorNotSupported;
  }
  cuuint64_t dims[4] = {cuuint64_t(p.D), cuuint64_t(heads), cuuint64_t(p.C), cuuint64_t(p.B)};
  cuuint64_t strides[3] = {cuuint64_t(p.D * 2), cuuint64_t(heads * p.D * 2), cuuint64_t(p.C * heads * p.D * 2)};
  cuuint32_t box[4] = {64, 1, BT, 1};
  cuuint32_t es[4] = {1, 1, 1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(base), dims, strides, box, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    snprintf(g_tc_err, sizeof g_tc_err, "cuTensorMapEncodeTiled failed (CUresult %d) for ptr=%p dims=[%lld,%lld,%lld,%lld]",
             int(r), base, (long long)p.D, (long long)heads, (long long)p.C, (long long)p.B);
    return cudaErrorInvalidValue;
  }
  return cudaSuccess;
}


// scale the 8 bf16 of a 16-byte chunk by w (packed bf16x2 multiply; w is rounded to bf16 once)
__device__ __forceinline__ uint4 scale_chunk(uint4 v, uint32_t w2) {
  uint32_t* u = reinterpret_cast<uint32_t*>(&v);
#pragma unroll
  for (int i = 0; i < 4; ++i) asm("mul.rn.bf16x2 %0, %1, %2;" : "=r"(u[i]) : "r"(u[i]), "r"(w2));
  return v;
}
__device__ __forceinline__ uint32_t bf16x2_splat(float w) { return pack_bf16(w, w); }
__device__ __forceinline__ float fast_exp2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ uint4 lds128(uint32_t addr) {
  uint4 v;
  asm volatile("ld.shared.v4.b32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(addr));
  return v;
}
__device__ __forceinline__ void sts128(uint32_t addr, uint4 v) {
  asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};" ::"r"(addr), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
               : "memory");
}

// segment-state array [B][H][nseg][D][D] fp32 as 2-D rows of D floats, box [32 floats][D rows]
cudaError_t make_state_map(CUtensorMap* m, const float* base, const Plan& p) {
  auto fn = encode_fn();
  if (!fn) return cudaErrorNotSupported;
  cuuint64_t dims[2] = {cuuint64_t(p.D), cuuint64_t(p.B * p.Hk * p.nseg * p.D)};
  cuuint64_t strides[1] = {cuuint64_t(p.D * 4)};
  cuuint32_t box[2] = {32, cuuint32_t(p.D)};
  cuuint32_t es[2] = {1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims, strides, box, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    snprintf(g_tc_err, sizeof g_tc_err, "cuTensorMapEncodeTiled (state) failed (CUresult %d)", int(r));
    return cudaErrorInvalidValue;
  }
  return cudaSuccess;
}

__device__ __forceinline__ uint64_t desc_k(uint32_t addr) { return smem_desc(addr, 16, 1024); }
__device__ __forceinline__ uint64_t desc_mn(uint32_t addr, uint32_t lbo) { return smem_desc(addr, lbo, 1024); }

// ================================================================================================
// Dynamic work claiming (persistent kernels): the producer thread claims item indices in increasing
// order from a global counter (zeroed by the call's entry kernel) and hands them to the CTA's other roles
// through a 2-slot shared-memory queue. A CTA that starts late (its SM still busy with the previous kernel
// or a communication kernel on another stream) simply claims fewer items, instead of owning a fixed
// 1/grid share that stretches the launch. Items are independent (no cross-item reduction), so which CTA
// runs an item does not change any bit of the result.
struct ItemQueue {
  uint64_t full[2], empty[2];
  int64_t item[2];
};
__device__ __forceinline__ void q_init(ItemQueue& q, uint32_t consumers) {
  for (int s = 0; s < 2; ++s) { mbar_init(&q.full[s], 1); mbar_init(&q.empty[s], consumers); }
}
// producer: claim the k-th item of this CTA (>= W: no more work; still published, as the end marker).
// ctr == nullptr: the static round-robin assignment of round 1 (LASP_STATIC_ITEMS=1, A/B experiments)
__device__ __forceinline__ int64_t q_claim(ItemQueue& q, uint32_t k, unsigned* ctr) {
  const uint32_t s = k & 1u;
  mbar_wait(&q.empty[s], ((k >> 1) & 1u) ^ 1u);
  const int64_t w = ctr ? int64_t(atomicAdd(ctr, 1u)) : int64_t(blockIdx.x) + int64_t(k) * gridDim.x;
  q.item[s] = w;
  mbar_arrive(&q.full[s]);  // release: the item index is visible to the waiters
  return w;
}
// consumer: the k-th item of this CTA; then q_release once per consumer warp (or single-thread role)
__device__ __forceinline__ int64_t q_fetch(ItemQueue& q, uint32_t k) {
  mbar_wait(&q.full[k & 1u], (k >> 1) & 1u);
  return *reinterpret_cast<volatile int64_t*>(&q.item[k & 1u]);
}
__device__ __forceinline__ void q_release(ItemQueue& q, uint32_t k) { mbar_arrive(&q.empty[k & 1u]); }
// whole-warp consumer: fetch, then lane 0 releases the slot once every lane has read it
__device__ __forceinline__ int64_t q_fetch_warp(ItemQueue& q, uint32_t k) {
  const int64_t w = q_fetch(q, k);
  __syncwarp();
  if (lane_id() == 0) q_release(q, k);
  return w;
}

// ================================================================================================
// work items: (batch, state head, segment), claimed dynamically by a persistent grid
// ================================================================================================
struct Item {
  int64_t b, h, seg, beg, end;
  int nblk;
};

__device__ __noinline__ Item get_item(const Plan& p, Dir dir, int64_t w) {  // out of line: code size
  // Segment-major order: the CTAs in flight at any time cover the same token ranges for all
  // (batch, head) pairs, so the 128-byte head slices of each [H][D] token row are fetched together
  // (DRAM page locality, L2 sector promotion shared by neighbouring heads).
  Item it;  // 32-bit decode (the host guarantees B*H*nseg < 2^31): keeps the hot loops small
  const uint32_t wu = uint32_t(w), nbh = uint32_t(p.B * p.Hk), nh = uint32_t(p.Hk);
  it.seg = p.div_bhk.div(wu);
  const uint32_t bh = wu - uint32_t(it.seg) * nbh;
  it.b = p.div_hk.div(bh);
  it.h = bh - uint32_t(it.b) * nh;  // state (kv-) head
  it.beg = seg_begin(dir, it.seg, p.seg_len, p.C);
  it.end = seg_end(dir, it.seg, p.seg_len, p.C);
  it.nblk = int((it.end - it.beg + BT - 1) / BT);
  return it;
}

// first row of block j of an item: FWD blocks ascend from the segment begin, REV blocks descend
// from the segment end (so a ragged block only occurs where no state leaves it)
__device__ __forceinline__ int64_t block_row(Dir dir, const Item& it, int j) {
  return dir == Dir::FWD ? it.beg + int64_t(j) * BT : it.end - int64_t(j + 1) * BT;
}


// ================================================================================================
// seg_state_tc (persistent): warp 0 TMA, warp 1 UMMA, warps 4-7 scale X rows, warps 8-11 drain
// the (double-buffered) TMEM accumulator of finished items to global memory.
// ================================================================================================
// NORM (B1 with the Norm backward fused, NEXT-3): a third tile per stage holds the forward output y
template <int D, bool NORM = false>
struct SegLayout {
  static constexpr int NBOX = D / 64;
  static constexpr uint32_t TILE = NBOX * BOX;
  // VS = 2 (experiment, LASP_SEG_VSPLIT; head_dim 128 without the fused Norm backward): an item is one 64-wide
  // value slice of a segment's state, so the persistent grid gets twice the items (TNL-1B: 384 segment items are
  // 2.6 per SM) with 4 x 48 KB stages. Measured: F1 59.7 -> 74 us at TNL-1B, 347 -> 604 us at TNL-7B (the X tile
  // is fetched and row-scaled once per slice), so whole segments stay the default.
#ifdef LASP_SEG_VSPLIT
  static constexpr int VS = (D == 128 && !NORM) ? 2 : 1;
#else
  static constexpr int VS = 1;
#endif
  static constexpr int NBOXY = NBOX / VS;            // 64-wide boxes of the Y tile
  static constexpr int DN = D / VS;                  // state columns per item (UMMA N)
  static constexpr uint32_t TILEY = NBOXY * BOX;
  static constexpr uint32_t STG_BYTES = TILE + TILEY + (NORM ? TILE : 0);
#ifndef LASP_SEG_STAGES64
#define LASP_SEG_STAGES64 2  // 2 x 2 beat 3 x 2, 4 x 1 and 6 x 1 (stages x CTAs/SM) by ~1 % (round 1 sweep)
#define LASP_SEG_CTAS64 2
#endif
#ifndef LASP_SEG_STAGES128
#define LASP_SEG_STAGES128 3  // 3 x 64 KB stages, 1 CTA/SM: seg F 61.4 -> 58.0 us at TNL-1B
#endif
  static constexpr int STAGES = NORM ? 2 : D == 64 ? LASP_SEG_STAGES64 : VS > 1 ? 4 : LASP_SEG_STAGES128;
  static constexpr int CTAS_PER_SM = D == 64 ? LASP_SEG_CTAS64 : 1;  // 2 x (96 KB smem, 128 TMEM columns) per SM
  static constexpr uint32_t X(int s) { return uint32_t(s) * STG_BYTES; }
  static constexpr uint32_t Y(int s) { return uint32_t(s) * STG_BYTES + TILE; }
  static constexpr uint32_t Y2(int s) { return uint32_t(s) * STG_BYTES + TILE + TILEY; }
  static constexpr uint32_t BARS = STAGES * STG_BYTES;
  static constexpr uint32_t BYTES = BARS + 512 + 1024;  // barriers + item queue + tmem slot + alignment slack
  static constexpr uint32_t TCOLS = 2 * DN < 32 ? 32 : 2 * DN;  // two accumulators
  static_assert(BYTES <= 232448, "shared memory budget");
};

struct SegParams {
  CUtensorMap mx, my;
  Plan p;
  float* out;
  unsigned long long* trace;
  unsigned* claim;       // work-claim counter (ItemQueue), 0 at launch
  int sub;               // X, Y heads summed per state head (B1 with grouped queries: G; else 1)
  // fused Norm backward (NORM instantiation, B1 only): Y is dY, the third tile is the forward output y;
  // the scaler warps turn dY into dO = r (dY - y (y . dY) / D) in shared memory and write it to dout
  CUtensorMap my2;
  const float* rnorm;    // [B][C][H]
  __nv_bfloat16* dout;   // [B][C][H][D]
  EntryDuty entry;       // the call's entry duty (has_entry: this launch replaces tag_kernel)
  int has_entry;
};

// debug timeline: event ev (0..15) of block J (< 64) of CTA 0 -> trace[ev * 64 + J] = clock64()
#ifdef LASP_TRACE_BUILD
#define LASP_TRACE(ev, J)                                                                    \
  do {                                                                                       \
    if (prm.trace != nullptr && blockIdx.x == 0 && (J) < 64) prm.trace[(ev) * 64 + (J)] = clock64(); \
  } while (0)
#ifdef LASP_NO_TRACE2
#define LASP_TRACE2(ev, J) do { } while (0)
#else
#define LASP_TRACE2(ev, J)                                                                   \
  do {                                                                                       \
    if (prm.trace != nullptr && blockIdx.x == 0 && (J) < 64) prm.trace[1024 + (ev) * 64 + (J)] = clock64(); \
  } while (0)
#endif
#else
#define LASP_TRACE(ev, J) do { } while (0)
#define LASP_TRACE2(ev, J) do { } while (0)
#endif

template <int D, Dir DIR, bool NORM>
__global__ void __launch_bounds__(384, 2) seg_state_tc_kernel(const __grid_constant__ SegParams prm) {
  using L = SegLayout<D, NORM>;
  constexpr int ST = L::STAGES;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + L::BARS);
  uint64_t* scaled = full + ST;
  uint64_t* empty = scaled + ST;
  uint64_t* acc_full = empty + ST;     // [2]
  uint64_t* acc_empty = acc_full + 2;  // [2]
  ItemQueue* iq = reinterpret_cast<ItemQueue*>(acc_empty + 2);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(iq + 1);
  const uint32_t sbase = smem_u32(sm);

  const Plan& p = prm.p;
  constexpr int VS = L::VS;
  const int64_t W = p.B * p.Hk * p.nseg * VS;
  const int sub = prm.sub;
  const uint32_t warp = warp_id(), lane = lane_id();

  if (threadIdx.x == 0) {
    tma_prefetch(&prm.mx);
    tma_prefetch(&prm.my);
    if (NORM) tma_prefetch(&prm.my2);
    for (int s = 0; s < ST; ++s) { mbar_init(&full[s], 1); mbar_init(&scaled[s], 128); mbar_init(&empty[s], 1); }
    for (int s = 0; s < 2; ++s) { mbar_init(&acc_full[s], 1); mbar_init(&acc_empty[s], 128); }
    q_init(*iq, 1 + 4 + 4);  // consumers: the UMMA thread, 4 scaler warps, 4 drain warps
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc<L::TCOLS>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // Programmatic dependent launch: the producer, MMA and scaler roles only read this call's inputs, which
  // were complete before the preceding kernel started (every kernel of the library triggers its dependents
  // only after its own griddepcontrol.wait), so they start at once; the drain warps write the workspace,
  // which the preceding kernel may still read: they wait (and then trigger) before their first store.

  if (warp == 0) {
    if (elect_one()) {
      // first kernel of the call: nothing is read before all earlier work on the stream is complete (the
      // inputs may come from a kernel that triggered its dependents early)
      if (prm.has_entry) pdl_wait();
      uint32_t J = 0;
      for (uint32_t k = 0;; ++k) {
        const int64_t w = q_claim(*iq, k, prm.claim);
        if (w >= W) break;
        const Item it = get_item(p, DIR, w / VS);
        [[maybe_unused]] const int vs = int(w % VS);  // value slice of the item (head_dim 128)
        for (int jj = 0; jj < it.nblk * sub; ++jj, ++J) {  // block j = jj / sub, summed head u = jj % sub
          const int s = J % ST;
          mbar_wait(&empty[s], ((J / ST) & 1) ^ 1);
          LASP_TRACE(0, J);
          mbar_expect_tx(&full[s], L::STG_BYTES);
          const int t0 = int(block_row(DIR, it, jj / sub));
          const int hh = int(it.h) * sub + jj % sub;
#pragma unroll
          for (int x = 0; x < L::NBOX; ++x) {
            tma_load_4d(sm + L::X(s) + x * BOX, &prm.mx, &full[s], x * 64, hh, t0, int(it.b));
            if (x < L::NBOXY)
              tma_load_4d(sm + L::Y(s) + x * BOX, &prm.my, &full[s], (vs * L::NBOXY + x) * 64, hh, t0, int(it.b));
            if (NORM) tma_load_4d(sm + L::Y2(s) + x * BOX, &prm.my2, &full[s], x * 64, hh, t0, int(it.b));
          }
        }
      }
    }
  } else if (warp == 1) {
    if (elect_one()) {
      constexpr uint32_t idesc = idesc_bf16(D, L::DN, 1, 1);
      uint32_t J = 0;
      for (uint32_t k = 0;; ++k) {
        const int64_t w = q_fetch(*iq, k);
        q_release(*iq, k);
        if (w >= W) break;
        const Item it = get_item(p, DIR, w / VS);
        [[maybe_unused]] const int vs = int(w % VS);  // value slice of the item (head_dim 128)
        const uint32_t acc = tmem + (k & 1) * L::DN;
        mbar_wait(&acc_empty[k & 1], ((k >> 1) & 1) ^ 1);
        tc_fence_after();
        for (int jj = 0; jj < it.nblk * sub; ++jj, ++J) {
          const int s = J % ST;
          mbar_wait(&scaled[s], (J / ST) & 1);
          LASP_TRACE(3, J);
          tc_fence_after();
#ifdef LASP_EXPERIMENT_SEG_NOMMA  // timing experiment only: no accumulation
          if (false)
#endif
#pragma unroll
          for (int kk = 0; kk < BT / 16; ++kk)
            mma_bf16(acc, desc_mn(sbase + L::X(s) + kk * 2048, BOX), desc_mn(sbase + L::Y(s) + kk * 2048, BOX), idesc,
                     (jj | kk) != 0);
          mma_commit(&empty[s]);
        }
        mma_commit(&acc_full[k & 1]);
      }
    }
  } else if (warp >= 4 && warp < 8) {
    // scale X rows by the decay weight (Eq. 12 / Eq. 21 weights, relative to the segment end / begin)
    const int g = int(threadIdx.x) - 128;  // tile row
    uint32_t J = 0;
    for (uint32_t k = 0;; ++k) {
      const int64_t w = q_fetch_warp(*iq, k);
      if (w >= W) break;
      const Item it = get_item(p, DIR, w / VS);
        [[maybe_unused]] const int vs = int(w % VS);  // value slice of the item (head_dim 128)
      const float l2 = p.l2lam[it.h];
      for (int jj = 0; jj < it.nblk * sub; ++jj, ++J) {
        const int s = J % ST;
        mbar_wait(&full[s], (J / ST) & 1);
        if (g == 0) LASP_TRACE(1, J);
        const int64_t pos = block_row(DIR, it, jj / sub) + g;
        float wgt = 0.f;
        if (pos >= it.beg && pos < it.end)
          wgt = exp2f(float(DIR == Dir::FWD ? (it.end - 1 - pos) : (pos - it.beg + 1)) * l2);
        if constexpr (NORM) {
          // Norm backward of this row (reading N1): dO = r (dY - y (y . dY) / D) in fp32, rounded once to bf16,
          // into the Y tile (the MMA's operand) and to dout (read by the B3 passes)
          const int hh = int(it.h) * sub + jj % sub;
          const bool live = pos >= it.beg && pos < it.end;
          const int64_t row = (it.b * p.C + pos) * p.H + hh;
          const float rr = live ? prm.rnorm[row] : 0.f;
          float dot = 0.f;
#pragma unroll
          for (int x = 0; x < L::NBOX; ++x)
#pragma unroll
            for (int c = 0; c < 8; ++c) {
              const uint32_t o = x * BOX + uint32_t(g) * 128 + ((uint32_t(c) ^ (uint32_t(g) & 7)) << 4);
              const uint4 gy = lds128(sbase + L::Y(s) + o), yy = lds128(sbase + L::Y2(s) + o);
              const uint32_t* a = reinterpret_cast<const uint32_t*>(&gy);
              const uint32_t* b = reinterpret_cast<const uint32_t*>(&yy);
#pragma unroll
              for (int q = 0; q < 4; ++q) {
                dot = fmaf(__uint_as_float(a[q] << 16), __uint_as_float(b[q] << 16), dot);
                dot = fmaf(__uint_as_float(a[q] & 0xFFFF0000u), __uint_as_float(b[q] & 0xFFFF0000u), dot);
              }
            }
          const float coef = dot * (1.f / float(D));
          uint4* dst = reinterpret_cast<uint4*>(prm.dout + row * D);
#pragma unroll
          for (int x = 0; x < L::NBOX; ++x)
#pragma unroll
            for (int c = 0; c < 8; ++c) {
              const uint32_t o = x * BOX + uint32_t(g) * 128 + ((uint32_t(c) ^ (uint32_t(g) & 7)) << 4);
              uint4 gy = lds128(sbase + L::Y(s) + o);
              const uint4 yy = lds128(sbase + L::Y2(s) + o);
              uint32_t* a = reinterpret_cast<uint32_t*>(&gy);
              const uint32_t* b = reinterpret_cast<const uint32_t*>(&yy);
#pragma unroll
              for (int q = 0; q < 4; ++q) {
                const float lo = rr * fmaf(-__uint_as_float(b[q] << 16), coef, __uint_as_float(a[q] << 16));
                const float hi = rr * fmaf(-__uint_as_float(b[q] & 0xFFFF0000u), coef, __uint_as_float(a[q] & 0xFFFF0000u));
                a[q] = pack_bf16(lo, hi);
              }
              sts128(sbase + L::Y(s) + o, gy);
              if (live) dst[x * 8 + c] = gy;
            }
        }
#ifdef LASP_EXPERIMENT_SEG_NOSCALE  // timing experiment only (tools/cmp_variants.sh): unweighted X
        if (false)
#endif
#pragma unroll
        for (int x = 0; x < L::NBOX; ++x)
#pragma unroll
          for (int c = 0; c < 8; ++c) {  // swizzled chunk order: conflict-free across 8 rows
            const uint32_t a = sbase + L::X(s) + x * BOX + uint32_t(g) * 128 + ((uint32_t(c) ^ (uint32_t(g) & 7)) << 4);
            sts128(a, scale_chunk(lds128(a), bf16x2_splat(wgt)));
          }
        fence_async_smem();
        mbar_arrive(&scaled[s]);
        if (g == 0) LASP_TRACE(2, J);
      }
    }
  } else if (warp >= 8) {
    // drain finished accumulators: rows of L (TMEM layout of M = D), fp32 to [B][H][nseg][D][D]
    const uint32_t q4 = warp & 3;
    const bool valid = D == 128 || lane < 16;
    const int row = D == 128 ? int(q4 * 32 + lane) : int(q4 * 16 + lane);
    pdl_wait();
    if (prm.has_entry && blockIdx.x == 0) {
      // the call's entry duty before this CTA lets the next kernel launch: its CTAs claim items from the
      // control block as they start
      if (warp == 8) entry_duty(prm.entry.tag, prm.entry.hdr, prm.entry.check_mask, prm.entry.ctrl);
      __threadfence();
      named_bar_sync(3, 128);
    }
    pdl_trigger();
    for (uint32_t k = 0;; ++k) {
      const int64_t w = q_fetch_warp(*iq, k);
      if (w >= W) break;
      const Item it = get_item(p, DIR, w / VS);
        [[maybe_unused]] const int vs = int(w % VS);  // value slice of the item (head_dim 128)
      mbar_wait(&acc_full[k & 1], (k >> 1) & 1);
      tc_fence_after();
      float* o = prm.out + ((it.b * p.Hk + it.h) * p.nseg + it.seg) * D * D + int64_t(row) * D + vs * L::DN;
      const uint32_t ta = tmem + ((q4 * 32) << 16) + (k & 1) * L::DN;
#pragma unroll
      for (int c = 0; c < L::DN / 16; ++c) {
        float v[16];
        tmem_ld16(ta + c * 16, v);
        tmem_ld_wait();
        if (c == L::DN / 16 - 1) {
          tc_fence_before();
          mbar_arrive(&acc_empty[k & 1]);
        }
        if (valid) {
#pragma unroll
          for (int u = 0; u < 16; u += 4)
            *reinterpret_cast<float4*>(o + c * 16 + u) = make_float4(v[u], v[u + 1], v[u + 2], v[u + 3]);
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc<L::TCOLS>(tmem);
}

// ================================================================================================
// core_tc (persistent)
// ================================================================================================
template <int D>
struct CoreLayout {
  // Items work on one 64-wide slice of the value dimension (NV = D / 64 slices per head), with the
  // full key dimension DK = D: a, b tiles are [128][DK], c / u.c / out tiles are [128][64], the state
  // slice is [DK][64].
  static constexpr int DK = D, NBOX = D / 64, NV = D / 64;
  static constexpr uint32_t TA = NBOX * BOX;             // [128][DK] bf16 (a, b)
  static constexpr uint32_t TC = BOX;                    // [128][64] bf16 (c, u.c, out)
  static constexpr int STAGES = D == 64 ? 3 : 2;
  static constexpr int NSB = D == 64 ? 2 : 1;            // bf16 state copies (double-buffered if smem allows)
  static constexpr bool HAS_STG = D == 64;               // TMA-staged prefix state (else read directly); D = 64 only
  static_assert(!HAS_STG || D == 64, "the STG reader is the head_dim 64 split-state layout");
  static constexpr uint32_t STAGE = 2 * TA + TC;
  static constexpr uint32_t A(int s) { return uint32_t(s) * STAGE; }
  static constexpr uint32_t B_(int s) { return uint32_t(s) * STAGE + TA; }
  static constexpr uint32_t C_(int s) { return uint32_t(s) * STAGE + 2 * TA; }
  static constexpr uint32_t KU = STAGES * STAGE;         // u (.) c, [128][64]
  // state slice as bf16 hi part and lo part (S - hi), [DK][64] each, per buffer
  static constexpr uint32_t SBF(int b) { return KU + TC + uint32_t(b) * DK * 256; }
  static constexpr uint32_t SLO(int b) { return SBF(b) + DK * 128; }
  static constexpr uint32_t OST = KU + TC + NSB * DK * 256;  // [128][64] bf16 output staging
  static constexpr uint32_t STG = OST + TC;                  // [D][D] fp32 segment prefix state (TMA, SW128)
  static constexpr uint32_t BARS = STG + (HAS_STG ? 4 * D * D : 0);  // barriers and item queue (768 B)
  static constexpr uint32_t BYTES = BARS + 768 + 1024;
  // TMEM columns (P, bf16, overwrites the first 64 columns of its S buffer: FA4-style TS MMA)
  static constexpr uint32_t T_S0 = 0, T_S1 = 128, T_OI = 256, T_OX = 320, T_DS = 384;
  static_assert(BYTES <= 232448, "shared memory budget");
};

// One launch runs up to 3 passes of the core identity (e.g. dQ, dV and dK of the backward), with the
// passes of one segment interleaved so that their shared input tiles are re-read from L2.
struct CorePass {
  int dir;        // Dir::FWD / Dir::REV
  int trans;      // use S^T of the stored segment state
  int a, b, c;    // indices into CoreParams::min
  int out;        // index into CoreParams::mout / outp
  int state;      // index into CoreParams::mst
  int kvp;        // 1: kv-head pass (items over Hk, G query heads summed per block), 0: query-head pass
  int nh;         // item heads (H or Hk) = heads of a and out
  uint32_t off;   // first item of this pass inside a segment row
  FastDiv div_nh; // / nh
};

struct CoreParams {
  CUtensorMap min[4];  // distinct input sequence tensors
  CUtensorMap mout[3]; // outputs
  CUtensorMap mst[2];  // segment prefix states, fp32 2-D [rows = B*H*nseg*D][D], box [32][D], 128B swizzle
  const float* stp[2]; // the same states as plain pointers (D = 128: read directly by the state warps)
  Plan p;
  CorePass pass[3];
  __nv_bfloat16* outp[3];
  unsigned long long* trace;  // debug timeline (lasp_debug_trace), nullptr in production
  int npass;
  const unsigned* status;     // cache-tag status of a backward call (nonzero: NaN states), or nullptr
  unsigned* claim;            // work-claim counter (ItemQueue), 0 at launch
  FastDiv div_per;            // / (items per segment row) (work-item decode)
  uint32_t per;               // items per segment row (sum over the passes of B * nh * NV)
  FastDiv div_nbh, div_h;     // multi-head decode: / (B*H*NV), / H
  int uniform;                // every pass has the same item count (head_dim 128 interleaved order)
  PrefixFold fold;            // fold.gbar != nullptr: compute the prefix states first (fused F2 / B2)
  // Norm epilogue (NEXT-3, reading N1; the forward O pass of a NORM instantiation): head_dim 64 writes
  // y = o r and r = (mean o^2 + eps)^-1/2 into rnorm [B][C][H]; head_dim 128 (two value-slice items per
  // head row) writes o and each slice's sum of squares into nsum [B][C][H][2] for norm_apply_kernel.
  float* rnorm;
  float* nsum;
  float norm_eps;
  int seg_desc;               // 1: items in descending segment order (the segment-state launch before this one
                              // ascended, so its last-read tiles are still in L2)
  int short_last;             // with seg_desc: order nseg - 2, ..., 0, nseg - 1 (the last segment is ragged)
  int late_inputs;            // 1: an input tensor is written by the preceding kernel (fused Norm
                              // backward): the producer waits for it before the first load
};

// Fused F2 / B2 (Alg. 2, Alg. 3 P:648 between segments; the arithmetic of prefix_kernel): per
// element, cur = init; for each segment in fold order: prefix[p] = cur; cur = lam^len_p cur + seg[p];
// fin = cur, for float2 element i2 of the B*H*D*D / 2; all (up to U) segment loads of a batch are in
// flight before the serial fold, and a batch is loaded before any of it is stored (in place). One copy
// of the unrolled body serves both directions (code size: it sits in the core kernel).
template <int D>
__device__ __forceinline__ void fold_prefix(const Plan& p, const PrefixFold& f, int64_t i2) {
  constexpr int64_t D2 = int64_t(D) * D / 2;  // float2 elements per state
  constexpr int U = 40;
  const bool fwd = Dir(f.dir) == Dir::FWD;
  const int64_t step = fwd ? D2 : -D2;        // float2 elements between consecutive folded segments
  const int64_t last_len = p.C - (p.nseg - 1) * p.seg_len;
  const int64_t bh = i2 / D2, e2 = i2 - bh * D2;
  const float l2 = p.l2lam[bh % p.Hk];
  const float dec_full = exp2f(float(p.seg_len) * l2), dec_last = exp2f(float(last_len) * l2);
  float2 cur = f.init ? __ldcg(reinterpret_cast<const float2*>(f.init) + i2) : make_float2(0.f, 0.f);
  // segment 0 (FWD) or nseg - 1 (REV) of this element
  const int64_t first = (bh * p.nseg + (fwd ? 0 : p.nseg - 1)) * D2 + e2;
  const float2* src = reinterpret_cast<const float2*>(f.seg) + first;
  float2* dst = reinterpret_cast<float2*>(f.out) + first;
  for (int64_t s0 = 0; s0 < p.nseg; s0 += U, src += U * step, dst += U * step) {
    const int nb = int(p.nseg - s0);  // segments left
    // the segment nseg - 1 (length last_len) is folded last (FWD) or first (REV)
    const int last_u = fwd ? int(nb - 1) : (s0 == 0 ? 0 : -1);
    float2 v[U];
    const float2* ps = src;
#pragma unroll
    for (int u = 0; u < U; ++u, ps += step) v[u] = __ldcg(u < nb ? ps : src);  // past the end: a valid dummy
    float2* pd = dst;
#pragma unroll
    for (int u = 0; u < U; ++u, pd += step) {
      if (u < nb) {
        *pd = cur;
        const float dcy = u == last_u ? dec_last : dec_full;
        cur.x = fmaf(dcy, cur.x, v[u].x);
        cur.y = fmaf(dcy, cur.y, v[u].y);
      }
    }
  }
  if (f.fin) reinterpret_cast<float2*>(f.fin)[i2] = cur;
}

// wait (acquire) until *ctr >= target, then make the other CTAs' generic-proxy writes visible to this
// thread's TMA loads; traps instead of hanging if the count is never reached
__device__ __forceinline__ void grid_wait(const unsigned* ctr, unsigned target) {
  uint32_t n = 0;
  for (;;) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory");
    if (v >= target) break;
    __nanosleep(64);
    if (++n == (1u << 26)) __trap();
  }
  asm volatile("fence.proxy.async.global;" ::: "memory");
}

struct CItem {
  int32_t b, h, seg, beg, end;  // h: item head (of a and out); token indices < 2^30 (tc_supported)
  int nblk, pass, v;  // v: 64-wide value slice
  int sh, sub, bh0;   // state / decay head; query heads summed per block (1 or G); b, c head of sub-block 0
  Dir dir;
};

// item w -> (segment, pass, batch*head, value slice) at head_dim 64, (segment, batch*head, pass, value slice)
// at head_dim 128 when every pass has the same item count: segment-major, value slice innermost.
// Grouped queries: a query-head pass (O, dQ) reads b, c and the state of kv-head h / G; a kv-head pass
// (dV, dK) reads b, c of the G query heads h G + u, u = 0..G-1 (sub-blocks summed into one output block).
template <int NV, bool GQ>
__device__ __noinline__ CItem get_citem(const CoreParams& prm, int64_t w) {
  const Plan& p = prm.p;
  CItem it;
  const uint32_t wu = uint32_t(w);
  const uint32_t sg = prm.div_per.div(wu);
  const uint32_t rem = wu - sg * prm.per;
  // descending order; with short_last the ragged (shorter) last segment goes last instead of first, so the
  // launch's final claims are the short items (a smaller tail)
  it.seg = !prm.seg_desc ? int32_t(sg) : prm.short_last ? int32_t(sg + 1 < uint32_t(p.nseg) ? p.nseg - 2 - sg : p.nseg - 1)
                                                        : int32_t(p.nseg - 1 - sg);
  if constexpr (!GQ) {  // multi-head: every pass has B * H * NV items per segment row (round-1 decode)
    const uint32_t nbh = uint32_t(p.B * p.H) * uint32_t(NV), nh = uint32_t(p.H);
    uint32_t bhv;
    if constexpr (NV > 1) {
      const uint32_t pv = uint32_t(prm.npass) * uint32_t(NV), bh0 = rem / pv, r2 = rem - bh0 * pv;
      it.pass = int(r2 / uint32_t(NV));
      bhv = bh0 * uint32_t(NV) + (r2 - uint32_t(it.pass) * uint32_t(NV));
    } else {
      it.pass = int(prm.div_nbh.div(rem));
      bhv = rem - uint32_t(it.pass) * nbh;
    }
    const uint32_t bh = bhv / uint32_t(NV);
    it.v = int(bhv - bh * uint32_t(NV));
    it.b = prm.div_h.div(bh);
    it.h = bh - uint32_t(it.b) * nh;
    it.sh = int(it.h);
    it.sub = 1;
    it.bh0 = int(it.h);
    it.dir = Dir(prm.pass[it.pass].dir);
    it.beg = seg_begin(it.dir, it.seg, p.seg_len, p.C);
    it.end = seg_end(it.dir, it.seg, p.seg_len, p.C);
    it.nblk = int((it.end - it.beg + BT - 1) / BT);
    return it;
  }
  uint32_t bh;
  if (NV > 1 && prm.uniform) {
    // head_dim 128: (batch x head, pass, value slice) inside a segment row, so that the items re-reading one
    // (segment, batch x head)'s a / b tiles run on adjacent CTAs (fused backward 342 -> 336.5 us at TNL-1B;
    // at head_dim 64 the pass-major order is faster, 124.5 vs 125.8 us)
    const uint32_t pv = uint32_t(prm.npass) * uint32_t(NV), b0 = rem / pv, r2 = rem - b0 * pv;
    it.pass = int(r2 / uint32_t(NV));
    it.v = int(r2 - uint32_t(it.pass) * uint32_t(NV));
    bh = b0;
  } else {
    int ps = 0;
    while (ps + 1 < prm.npass && rem >= prm.pass[ps + 1].off) ++ps;
    it.pass = ps;
    const uint32_t bhv = rem - prm.pass[ps].off;
    bh = bhv / uint32_t(NV);
    it.v = int(bhv - bh * uint32_t(NV));
  }
  const CorePass& ps = prm.pass[it.pass];
  it.b = ps.div_nh.div(bh);
  it.h = bh - uint32_t(it.b) * uint32_t(ps.nh);
  if (ps.kvp) {
    it.sh = int(it.h);
    it.sub = int(p.G);
    it.bh0 = int(it.h * p.G);
  } else {
    it.sh = int(it.h / p.G);
    it.sub = 1;
    it.bh0 = it.sh;
  }
  it.dir = Dir(ps.dir);
  it.beg = seg_begin(it.dir, it.seg, p.seg_len, p.C);
  it.end = seg_end(it.dir, it.seg, p.seg_len, p.C);
  it.nblk = int((it.end - it.beg + BT - 1) / BT);
  return it;
}
__device__ __forceinline__ int64_t cblock_row(const CItem& it, int j) {
  return it.dir == Dir::FWD ? it.beg + int64_t(j) * BT : it.end - int64_t(j + 1) * BT;
}
struct CoreBars {
  uint64_t full[3], empty[3], s_full[2], s_empty[2];
  uint64_t fullc[3];  // ring slot: full = a, b tiles landed; fullc = c tile landed
  uint64_t p_full[2][4], ku_full, ku_empty, ds_full, ds_empty, st_full[2], st_empty[2], o_full, o_empty;
  uint64_t stg_full, stg_empty;
  ItemQueue iq;
  uint32_t tmem_slot;
  uint32_t fold_chunk;  // fused prefix fold: chunk claimed by this CTA's fold threads
};
static_assert(sizeof(CoreBars) <= 768, "CoreBars must fit its 768-byte slot");
constexpr int kFoldChunk = 256;  // float2 elements per claimed fold chunk (one per fold thread)
__device__ __forceinline__ unsigned fold_chunks(const Plan& p) {
  return unsigned((p.B * p.Hk * p.D * p.D / 2 + kFoldChunk - 1) / kFoldChunk);
}



// GQ: grouped queries (G > 1) -- a separate instantiation, so that the multi-head kernel keeps sub = 1 as a
// compile-time constant (no sub-block arithmetic, no u . c release barrier: measured -8 % otherwise)
template <int D, bool GQ, bool NORM>
__global__ void __launch_bounds__(512, 1) core_tc_kernel(const __grid_constant__ CoreParams prm) {
  using L = CoreLayout<D>;
  constexpr int ST = L::STAGES;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  CoreBars* bar = reinterpret_cast<CoreBars*>(sm + L::BARS);
  const uint32_t sbase = smem_u32(sm);

  const Plan& p = prm.p;
  const int64_t W = p.nseg * int64_t(prm.per);
  const uint32_t warp = warp_id(), lane = lane_id();
#ifdef LASP_TRACE_BUILD
  if (prm.trace != nullptr && threadIdx.x == 0) prm.trace[2 * 1024 + blockIdx.x * 2] = globaltimer();
#endif

  if (threadIdx.x == 0) {
    for (int x = 0; x < 4; ++x) tma_prefetch(&prm.min[x]);
    for (int x = 0; x < prm.npass; ++x) tma_prefetch(&prm.mout[x]);
    tma_prefetch(&prm.mst[0]); tma_prefetch(&prm.mst[1]);
    mbar_init(&bar->stg_full, 1); mbar_init(&bar->stg_empty, 128);
    for (int s = 0; s < ST; ++s) { mbar_init(&bar->full[s], 1); mbar_init(&bar->fullc[s], 1); mbar_init(&bar->empty[s], 2); }
    for (int s = 0; s < 2; ++s) { mbar_init(&bar->s_full[s], 1); mbar_init(&bar->s_empty[s], 1); }
    for (int b2 = 0; b2 < 2; ++b2)
      for (int c = 0; c < 4; ++c) mbar_init(&bar->p_full[b2][c], 128);
    mbar_init(&bar->ku_full, 128); mbar_init(&bar->ku_empty, 1);
    mbar_init(&bar->ds_full, 1); mbar_init(&bar->ds_empty, 128);
    for (int b2 = 0; b2 < L::NSB; ++b2) { mbar_init(&bar->st_full[b2], 128); mbar_init(&bar->st_empty[b2], 1); }
    mbar_init(&bar->o_full, 1); mbar_init(&bar->o_empty, 128);
    q_init(bar->iq, 3 + 12);  // consumers: 3 UMMA threads, 12 SIMT warps
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc<512>(&bar->tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = bar->tmem_slot;
  // Programmatic dependent launch: every kernel of the library triggers its dependents only after its
  // own griddepcontrol.wait, so when this kernel starts, the kernel two launches back (and everything
  // before it) has completed. The a, b, c tiles are inputs of that earlier work, so the producer fills
  // the ring before waiting; only the segment prefix states (written by the immediately preceding
  // kernel) are read after the wait (producer: STG; state warps at D = 128: direct loads).
  // Fused fold: the state and epilogue warps (idle until the first state is needed) wait for the
  // segment states, then claim chunks of kFoldChunk float2 elements from a global counter (fold.gbar[0])
  // and fold them, counting finished chunks in fold.gbar[1]; the readers of prefix states (producer STG /
  // D = 128 state warps) wait until every chunk is done. Chunks are claimed, not assigned, so the wait
  // completes whichever CTAs are resident (no co-residency requirement, no cooperative launch).
  if (prm.fold.gbar != nullptr && warp >= 8) {
    const unsigned n_chunks = fold_chunks(p);
    pdl_wait();
    const int64_t n2 = p.B * p.Hk * p.D * p.D / 2;
    for (;;) {
      if (threadIdx.x == 256) bar->fold_chunk = atomicAdd(&prm.fold.gbar[0], 1u);
      named_bar_sync(2, 256);
      const unsigned c = bar->fold_chunk;
      if (c >= n_chunks) break;
      const int64_t i2 = int64_t(c) * kFoldChunk + (threadIdx.x - 256);
      if (i2 < n2) fold_prefix<D>(p, prm.fold, i2);
      named_bar_sync(2, 256);  // chunk written (and fold_chunk read by every thread)
      if (threadIdx.x == 256) {
        asm volatile("fence.proxy.async.global;" ::: "memory");
        __threadfence();
        atomicAdd(&prm.fold.gbar[1], 1u);
      }
    }
  }

  if (warp == 0) {
    // ------------------------------------------------------------------ TMA producer
    if (elect_one()) {
      bool waited = false;
      if (prm.late_inputs) {  // the inputs are not complete before the preceding kernel has finished
        pdl_wait();
        pdl_trigger();
        waited = true;
      }
      uint32_t J = 0, k = 0;
      for (;; ++k) {
        const int64_t w = q_claim(bar->iq, k, prm.claim);
        if (w >= W) break;
        const CItem it = get_citem<L::NV, GQ>(prm, w);
        const CorePass& ps = prm.pass[it.pass];
        // the segment's prefix state -> STG (single buffer, released by the state warps)
        auto load_stg = [&]() {
          if constexpr (L::HAS_STG) {
            if (k == 0 && prm.fold.gbar != nullptr) grid_wait(&prm.fold.gbar[1], fold_chunks(p));
            mbar_wait(&bar->stg_empty, (k & 1) ^ 1);
            mbar_expect_tx(&bar->stg_full, 4 * D * D);
            const int srow = int(((it.b * p.Hk + it.sh) * p.nseg + it.seg) * D);
#pragma unroll
            for (int x = 0; x < D / 32; ++x)
              tma_load_2d(sm + L::STG + x * (D * 128), &prm.mst[ps.state], &bar->stg_full, x * 32, srow);
          }
        };
        if (waited) load_stg();
#ifndef LASP_NO_STATE_PREFETCH
        if constexpr (!L::HAS_STG) {
          // head_dim 128: the state warps read the item's prefix state with plain loads when the item starts;
          // pull it into L2 now, ~one ring depth ahead (a state written by the preceding kernel has usually left
          // L2 by the time the late items read it: the item-start load was ~3-5k cycles on the critical path)
          if (k > 0)
            l2_prefetch_bulk(prm.stp[ps.state] + ((int64_t(it.b) * p.Hk + it.sh) * p.nseg + it.seg) * D * D,
                             uint32_t(D * D * 4));
        }
#endif
        const CUtensorMap* ma = &prm.min[ps.a];
        const CUtensorMap* mb = &prm.min[ps.b];
        const CUtensorMap* mc = &prm.min[ps.c];
        const int isub = GQ ? it.sub : 1;
        const int nsb = it.nblk * isub;  // sub-blocks: block j = jj / sub, summed query head u = jj % sub
        for (int jj = 0; jj < nsb; ++jj, ++J) {
          if (!waited && jj == (nsb < ST ? nsb : ST)) {
            pdl_wait();
            pdl_trigger();
            waited = true;
            load_stg();
          }
          const int s = J % ST;
          mbar_wait(&bar->empty[s], ((J / ST) & 1) ^ 1);
          LASP_TRACE(0, J);
#ifdef LASP_FULL_WHOLE  // A/B experiment: one barrier for the whole stage
          mbar_expect_tx(&bar->full[s], L::STAGE);
          uint64_t* fc = &bar->full[s];
#else
          // a, b (S, O_inter, dS) and c (u . c, P c) on separate barriers, a and b issued first: S starts
          // before the c tile has landed
          mbar_expect_tx(&bar->full[s], 2 * L::TA);
          mbar_expect_tx(&bar->fullc[s], L::TC);
          uint64_t* fc = &bar->fullc[s];
#endif
          const int j = GQ ? jj / isub : jj;
          const int t0 = int(cblock_row(it, j)), hb = it.bh0 + (jj - j * isub);
#pragma unroll
          for (int x = 0; x < L::NBOX; ++x) {
            tma_load_4d(sm + L::A(s) + x * BOX, ma, &bar->full[s], x * 64, int(it.h), t0, int(it.b));
            tma_load_4d(sm + L::B_(s) + x * BOX, mb, &bar->full[s], x * 64, hb, t0, int(it.b));
          }
          tma_load_4d(sm + L::C_(s), mc, fc, it.v * 64, hb, t0, int(it.b));
#ifdef LASP_FULL_WHOLE
          mbar_arrive(&bar->fullc[s]);
#endif
        }
        if (!waited) {  // first item shorter than the ring
          pdl_wait();
          pdl_trigger();
          waited = true;
          load_stg();
        }
      }
    }
  } else if (warp >= 1 && warp <= 3) {
    // ------------------------------------------------------------------ UMMA issuers
    // Three single-thread issuers, each in program order with blocking waits (tcgen05.commit covers the
    // issuing thread's own MMAs): warp 2 issues S = a b^T, warp 3 the state chain dS = b^T (u . c),
    // warp 1 the outputs O_intra = P c (P read from TMEM) and O_inter = a (S_hi + S_lo). A stage is
    // released when both its dS and its output MMAs are done (empty count 2; a segment's last block
    // has no dS, so its output issuer arrives twice).
    if (elect_one()) {
      constexpr uint32_t id_qk = idesc_bf16(128, 128, 0, 0);
      constexpr uint32_t id_ds = idesc_bf16(L::DK, 64, 1, 1);
      constexpr uint32_t id_pv = idesc_bf16(128, 64, 0, 1);
      constexpr uint32_t id_x = idesc_bf16(128, 64, 0, 1);
      auto koff = [](int kk) -> uint32_t { return uint32_t(kk >> 2) * BOX + uint32_t(kk & 3) * 32; };
      uint32_t J = 0, Jb = 0, kd = 0, nku = 0;  // J: sub-blocks (ring, S buffers), Jb: blocks (outputs, state)
      for (uint32_t k = 0;; ++k) {
        const int64_t w = q_fetch(bar->iq, k);
        q_release(bar->iq, k);
        if (w >= W) break;
        const CItem itm = get_citem<L::NV, GQ>(prm, w);
        const int nblk = itm.nblk, sub = GQ ? itm.sub : 1;
        for (int jj = 0; jj < nblk * sub; ++jj, ++J) {
          const int j = GQ ? jj / sub : jj, u = jj - j * sub;
          const int s = int(J % ST);
          if (warp == 2) {
            // S = a b^T (double-buffered in TMEM; buffer J & 1 is free once out(J-2) has read its P)
            mbar_wait(&bar->full[s], (J / ST) & 1);
            LASP_TRACE(10, J);
            mbar_wait(&bar->s_empty[J & 1], ((J >> 1) & 1) ^ 1);
            tc_fence_after();
            const uint32_t dt = tmem + ((J & 1) ? L::T_S1 : L::T_S0);
            // (one N = 128 product: two N = 64 halves on separate barriers, so that the mask could start one half
            // earlier, measured TNL-1B fused bwd 325 -> 334 us -- each half re-reads the a tile from shared memory)
#pragma unroll
            for (int kk = 0; kk < L::DK / 16; ++kk)
              mma_bf16(dt, desc_k(sbase + L::A(s) + koff(kk)), desc_k(sbase + L::B_(s) + koff(kk)), id_qk, kk != 0);
            mma_commit(&bar->s_full[J & 1]);
            LASP_TRACE(1, J);
          } else if (warp == 3) {
            // dS = sum_u b_u^T (u . c_u), only for blocks that are not the last of their segment
            if (j + 1 < nblk) {
              mbar_wait(&bar->full[s], (J / ST) & 1);  // b (the u . c hand-off implies only the c tile)
              mbar_wait(&bar->ku_full, nku & 1);
              if (u == 0) mbar_wait(&bar->ds_empty, (kd & 1) ^ 1);
              tc_fence_after();
#pragma unroll
              for (int kk = 0; kk < BT / 16; ++kk)
                mma_bf16(tmem + L::T_DS, desc_mn(sbase + L::B_(s) + kk * 2048, BOX),
                         desc_mn(sbase + L::KU + kk * 2048, BOX), id_ds, (kk | u) != 0);
              if (GQ) mma_commit(&bar->ku_empty);  // the u . c buffer is free once this MMA has read it
              if (u + 1 == sub) {
                mma_commit(&bar->ds_full);
                ++kd;
              }
              mma_commit(&bar->empty[s]);
              LASP_TRACE(2, J);
              ++nku;
            }
          } else {
            // O_inter = a (S_hi + S_lo) first: it does not depend on the mask, so the tensor pipe runs it
            // while the mask warps build P; then O_intra = P c. (This issuer waits on the ring slot itself for
            // the a tile; it also releases the slot, so the parity wait stays within one phase.)
            mbar_wait(&bar->full[s], (J / ST) & 1);
            const int sb = int(Jb % L::NSB);
            if (u == 0) {  // once per block: the inter term of the block's rows
              mbar_wait(&bar->o_empty, (Jb & 1) ^ 1);
              LASP_TRACE(12, J);
              mbar_wait(&bar->st_full[sb], (Jb / L::NSB) & 1);
              tc_fence_after();
#pragma unroll
              for (int kk = 0; kk < L::DK / 16; ++kk)
                mma_bf16(tmem + L::T_OX, desc_k(sbase + L::A(s) + koff(kk)), desc_mn(sbase + L::SBF(sb) + kk * 2048, BOX),
                         id_x, kk != 0);
#pragma unroll
              for (int kk = 0; kk < L::DK / 16; ++kk)
                mma_bf16(tmem + L::T_OX, desc_k(sbase + L::A(s) + koff(kk)), desc_mn(sbase + L::SLO(sb) + kk * 2048, BOX),
                         id_x, 1);
              mma_commit(&bar->st_empty[sb]);  // the state copy is free once the inter MMAs have read it
            }
            const uint32_t pt = tmem + ((J & 1) ? L::T_S1 : L::T_S0);  // P in TMEM (2 bf16 / column)
            mbar_wait(&bar->fullc[s], (J / ST) & 1);  // the c tile
            // P c in four K steps of 32 tokens, each issued as soon as the mask warps have written that chunk of
            // P (the light row quadrants finish their chunks early; only the last K step waits for the
            // quadrant with the most live chunks), so P c ends ~one K step after the mask instead of four
#pragma unroll
            for (int c4 = 0; c4 < 4; ++c4) {
              mbar_wait(&bar->p_full[J & 1][c4], (J >> 1) & 1);
              if (c4 == 0) LASP_TRACE(11, J);
              tc_fence_after();
#pragma unroll
              for (int kk = 2 * c4; kk < 2 * c4 + 2; ++kk)
                mma_bf16_ts(tmem + L::T_OI, pt + kk * 8, desc_mn(sbase + L::C_(s) + kk * 2048, BOX), id_pv, (kk | u) != 0);
            }
            if (u + 1 == sub) {
              mma_commit(&bar->o_full);
              ++Jb;
            }
            mma_commit(&bar->s_empty[J & 1]);  // S/P buffer reusable once P c has been read
            mma_commit(&bar->empty[s]);
            if (j + 1 == nblk) mma_commit(&bar->empty[s]);  // no dS for the segment's last block
            LASP_TRACE(3, J);
          }
        }
      }
    }
  } else if (warp >= 4 && warp < 8) {
    // ------------------------------------------------------------------ mask warps: S -> P (bf16)
    const uint32_t q4 = warp & 3;  // rows [32 q4, 32 q4 + 32) of the block
    uint32_t J = 0;
    for (uint32_t k = 0;; ++k) {
      const int64_t w = q_fetch_warp(bar->iq, k);
      if (w >= W) break;
      const CItem it = get_citem<L::NV, GQ>(prm, w);
      const bool fwd = it.dir == Dir::FWD;
      const float l2 = p.l2lam[it.sh];
      // Per-thread decay factors of its row, kept in registers for the whole item. With e(u) = lane - u
      // (FWD) or u - lane (REV), column u of chunk c4 has M = lam^(32 |c4 - q4| + e(u)) on the live side:
      //   diagonal chunk (c4 = q4):  dm[u] = lam^e(u) for e(u) >= 0, else 0 (the causal cut)
      //   off-diagonal chunks:       t[u] = lam^(32 + e(u)), times lam^(32 (|c4 - q4| - 1))
      // All exponents are >= 0, so no factor overflows for any lam in (0, 1].
      // (ex2.approx.ftz: ~2^-22 relative, results below 2^-126 flush to 0 -- the exact limit, reading A9;
      // compact code: this setup runs once per item inside the warp's instruction stream)
      float dm[32], t[32];
      const float a2 = fwd ? l2 : -l2;             // e(u) * l2 = (lane - u) * a2
      const float x0 = float(int(lane)) * a2, x32 = 32.f * l2;
      const uint32_t lo = fwd ? 0u : lane, span = fwd ? lane : 31u - lane;  // live u in [lo, lo + span]
#pragma unroll
      for (int u = 0; u < 32; ++u) {
        const float x = fmaf(float(-u), a2, x0);
        dm[u] = uint32_t(u) - lo <= span ? fast_exp2(x) : 0.f;
        t[u] = fast_exp2(x + x32);
      }
      const float sc2 = fast_exp2(32.f * l2), sc3 = fast_exp2(64.f * l2);  // off-diagonal distance 2, 3
      for (int jj = 0; jj < it.nblk * (GQ ? it.sub : 1); ++jj, ++J) {  // every sub-block has its own S / P
        const int sb = J & 1;
        mbar_wait(&bar->s_full[sb], (J >> 1) & 1);
        if (lane == 0 && q4 == 3) LASP_TRACE(4, J);
        tc_fence_after();
        const uint32_t ts = tmem + ((q4 * 32) << 16) + (sb ? L::T_S1 : L::T_S0);
        // (software-pipelining the TMEM loads over half chunks -- next half loaded while the current one is
        // scaled -- measured TNL-0.4B fused bwd 121.3 -> 132 us: more spills, interleaved TMEM traffic; dropped)
#ifdef LASP_EXPERIMENT_NOMASK  // timing experiment only (tools/cmp_variants.sh): P = garbage
        if (false)
#endif
#pragma unroll 1
        for (int c4 = 0; c4 < 4; ++c4) {
          // chunk columns [32 c4, 32 c4 + 32) against warp rows [32 q4, 32 q4 + 32); dead chunks
          // (entirely on the non-causal side) are 0
          const int dist = fwd ? int(q4) - c4 : c4 - int(q4);
          uint32_t pk[16];
          if (lane == 0 && q4 == 3) LASP_TRACE2(c4 * 3, J);
          if (dist < 0) {
#pragma unroll
            for (int q = 0; q < 16; ++q) pk[q] = 0u;
          } else {
            float v[32];
            tmem_ld16(ts + c4 * 32, *reinterpret_cast<float(*)[16]>(&v[0]));
            tmem_ld16(ts + c4 * 32 + 16, *reinterpret_cast<float(*)[16]>(&v[16]));
            tmem_ld_wait();
            if (lane == 0 && q4 == 3) LASP_TRACE2(c4 * 3 + 1, J);
            if (dist == 0) {
#pragma unroll
              for (int u = 0; u < 32; u += 2) fmul2(v[u], v[u + 1], dm[u], dm[u + 1]);  // packed fp32x2
            } else {
#pragma unroll
              for (int u = 0; u < 32; u += 2) fmul2(v[u], v[u + 1], t[u], t[u + 1]);
              if (dist > 1) {
                const float sc = dist == 2 ? sc2 : sc3;
#pragma unroll
                for (int u = 0; u < 32; u += 2) fmul2(v[u], v[u + 1], sc, sc);
              }
            }
#pragma unroll
            for (int q = 0; q < 16; ++q) pk[q] = pack_bf16(v[2 * q], v[2 * q + 1]);
          }
          // P chunk -> TMEM columns [16 c4, 16 c4 + 16) of the same buffer (already consumed S columns); the
          // chunk is published on its own barrier (the P c MMA's K step c4 waits for it)
          tmem_st16(ts + c4 * 16, pk);
          if (lane == 0 && q4 == 3) LASP_TRACE2(c4 * 3 + 2, J);
          // (waiting for this store after the next chunk's load instead -- hiding its latency -- measured -0.4 %)
          tmem_st_wait();
          tc_fence_before();
          mbar_arrive(&bar->p_full[sb][c4]);  // per buffer: mask(J+1) may finish before out(J) is issued
        }
        if (lane == 0 && q4 == 3) LASP_TRACE(14, J);
#ifdef LASP_EXPERIMENT_NOMASK
        for (int c4 = 0; c4 < 4; ++c4) mbar_arrive(&bar->p_full[sb][c4]);
#endif
        if (lane == 0 && q4 == 3) LASP_TRACE(5, J);
      }
    }
  } else if (warp >= 8 && warp < 12) {
    // ------------------------------------------------------------------ state warps
    // Thread d owns row d (key index) of the [DK][64] state slice (TMEM layout of M = DK for dS).
    const uint32_t q4 = warp & 3;
    const int g = int(threadIdx.x) - 256;  // tile row for the u.c scaling
    // head_dim 64 (SPLIT): the M = 64 accumulator occupies lanes 0-15 of each quadrant, so each state row is
    // spread over 4 threads (tcgen05.ld.16x256b): thread (quadrant q4, lane l) holds rows q4 16 + l / 4 + 8 hr
    // (hr = 0, 1) at columns 8 r + 2 (l % 4) + f (r < 8, f = 0, 1) as S[4 r + 2 hr + f] -- all 32 lanes work,
    // 32 state values each. head_dim 128: thread q4 32 + l holds row d of the 64-wide value slice, S[64].
    constexpr bool SPLIT = L::DK == 64;
    constexpr int NS = SPLIT ? 32 : 64;
    const int d = int(q4 * 32 + lane);                               // (head_dim 128)
    const int r0 = int(q4 * 16) + int(lane >> 2), cq = int(lane & 3);  // (SPLIT)
    auto srow = [&](int i) { return r0 + 8 * ((i >> 1) & 1); };       // SPLIT: row / column of S[i]
    auto scol = [&](int i) { return 8 * (i >> 2) + 2 * cq + (i & 1); };
    float S[NS];
    auto load_state = [&](uint32_t k, const CItem& it, bool trans, int state) {
      if constexpr (SPLIT) {
        // segment prefix state from STG (TMA, 128B-swizzled fp32 rows of 32 floats)
        mbar_wait(&bar->stg_full, k & 1);
#pragma unroll
        for (int i = 0; i < NS; i += 2) {
          const uint32_t rr = uint32_t(srow(i)), cc = uint32_t(scol(i));
          if (trans) {  // S[rr][cc] = stored[cc][rr], [cc][rr + 1]
#pragma unroll
            for (int f = 0; f < 2; ++f) {
              const uint32_t e = cc + f, x = rr >> 5, c = (rr & 31) >> 2, wd = rr & 3;
              S[i + f] = *reinterpret_cast<const float*>(sm + L::STG + x * (D * 128) + e * 128 + ((c ^ (e & 7)) << 4) + wd * 4);
            }
          } else {
            const uint32_t x = cc >> 5, c = (cc & 31) >> 2;
            const float2 t = *reinterpret_cast<const float2*>(sm + L::STG + x * (D * 128) + rr * 128 +
                                                              ((c ^ (rr & 7)) << 4) + (cc & 3) * 4);
            S[i] = t.x; S[i + 1] = t.y;
          }
        }
        mbar_arrive(&bar->stg_empty);
      } else {
        // straight from the (L2-resident) prefix states: row d, columns [64 v, 64 v + 64) of S, or
        // column d, rows [64 v, 64 v + 64) for S^T (coalesced across the warp)
        if (k == 0) {  // the prefix states come from the preceding kernel, or from the fused fold
          if (prm.fold.gbar == nullptr) {
            pdl_wait();
          } else {
            if (lane == 0) grid_wait(&prm.fold.gbar[1], fold_chunks(p));
            __syncwarp();
          }
        }
        const float* st = prm.stp[state] + ((it.b * p.Hk + it.sh) * p.nseg + it.seg) * D * D;
        // states of the preceding kernel: read-only here (ld.global.nc); states folded by this launch: plain
        // (L1-allocating) loads after the acquire in grid_wait -- the fold read them with ld.global.cg, so
        // this SM's L1 holds no copy older than the fold's writes. (Each thread's 16 float4 row loads share
        // two 128-byte lines: L2-only loads would cost TNL-1B 4 %.)
        auto load = [&](auto ld) {
          if (trans) {
#pragma unroll
            for (int e = 0; e < 64; ++e) S[e] = ld(st + (it.v * 64 + e) * D + d);
          } else {
            const float4* row = reinterpret_cast<const float4*>(st + d * D + it.v * 64);
#pragma unroll
            for (int e = 0; e < 16; ++e) {
              const float4 t = ld(row + e);
              S[4 * e] = t.x; S[4 * e + 1] = t.y; S[4 * e + 2] = t.z; S[4 * e + 3] = t.w;
            }
          }
        };
        if (prm.fold.gbar == nullptr) load([](auto* ptr) { return __ldg(ptr); });
        else load([](auto* ptr) { return *ptr; });
      }
    };
    // after the loads are issued (the first block's u . c scaling runs while they are in flight)
    auto finish_state = [&]() {
      if (tag_poisoned(prm.status)) {  // the call's cache tag did not match: every output becomes NaN
#pragma unroll
        for (int e = 0; e < NS; ++e) S[e] = __int_as_float(0x7fc00000);
      }
    };
    uint32_t J = 0, Js = 0, kd = 0, nku = 0;  // J: blocks (state copies), Js: sub-blocks (ring), nku: u.c fills
    for (uint32_t k = 0;; ++k) {
      const int64_t w = q_fetch_warp(bar->iq, k);
      if (w >= W) break;
      const CItem it = get_citem<L::NV, GQ>(prm, w);
      const CorePass& ps = prm.pass[it.pass];
      if (g == 0) LASP_TRACE2(12, J);  // item fetched
      load_state(k, it, ps.trans != 0, ps.state);
#ifdef LASP_STATE_FINISH_EARLY  // A/B experiment: the round-2 order (state complete before the first u . c)
      finish_state();
#endif
      const float l2 = p.l2lam[it.sh];
      const uint32_t u2 = bf16x2_splat(exp2f(float(it.dir == Dir::FWD ? (BT - 1 - g) : (g + 1)) * l2));
      const float decay = exp2f(float(BT) * l2);
      // u (.) c for dS = b^T (u . c) of sub-block JJ (the Ku buffer is free once the dS MMA of the previous
      // sub-block has read it: ku_empty), done early so the dS MMA is never waiting on it
      auto scale_ku = [&](uint32_t JJ) {
        const int s = JJ % ST;
        if (GQ) {  // (one u . c per block: the ds_full wait before it already implies the buffer is free)
          mbar_wait(&bar->ku_empty, (nku & 1) ^ 1);
          ++nku;
        }
#ifdef LASP_FULL_WHOLE
        mbar_wait(&bar->full[s], (JJ / ST) & 1);
#else
        mbar_wait(&bar->fullc[s], (JJ / ST) & 1);  // the c tile
#endif
#if defined(LASP_EXPERIMENT_NOSTATE) || defined(LASP_EXPERIMENT_NOUC)
        if (false)
#endif
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          const uint32_t off = uint32_t(g) * 128 + ((uint32_t(c) ^ (uint32_t(g) & 7)) << 4);
          sts128(sbase + L::KU + off, scale_chunk(lds128(sbase + L::C_(s) + off), u2));
        }
        fence_async_smem();
        mbar_arrive(&bar->ku_full);
      };
      const int sub = GQ ? it.sub : 1;
#ifndef LASP_KU_EARLY
      const bool ku_late = !SPLIT && prm.npass == 1;
#else  // A/B experiment: the next block's u . c before its state copy in every launch
      constexpr bool ku_late = false;
#endif
      if (it.nblk > 1) scale_ku(Js);
#ifndef LASP_STATE_FINISH_EARLY
      finish_state();
#endif
      if (g == 0) LASP_TRACE(13, J);   // prefix state in registers
      for (int j = 0;; ++j, ++J) {
        // bf16 hi/lo copy of the state entering block J into buffer J % NSB (free once the output MMAs
        // of block J - NSB are done)
        const int sb = int(J % L::NSB);
        mbar_wait(&bar->st_empty[sb], ((J / L::NSB) & 1) ^ 1);
#if defined(LASP_EXPERIMENT_NOSTATE) || defined(LASP_EXPERIMENT_NOCOPY)  // timing experiments only
        if (false)
#endif
        if constexpr (SPLIT) {
          // one bf16 pair (4 bytes) per (row, 16-byte chunk): the 32 lanes of a store cover 8 rows x one chunk,
          // distinct banks under the 128B swizzle
#pragma unroll
          for (int i = 0; i < NS; i += 2) {
            const uint32_t hi = pack_bf16(S[i], S[i + 1]);
            const uint32_t lo = pack_bf16(S[i] - __uint_as_float(hi << 16), S[i + 1] - __uint_as_float(hi & 0xFFFF0000u));
            const uint32_t off = sw128_off(uint32_t(srow(i)), uint32_t(i >> 2)) + 4u * uint32_t(cq);
            asm volatile("st.shared.b32 [%0], %1;" ::"r"(sbase + L::SBF(sb) + off), "r"(hi) : "memory");
            asm volatile("st.shared.b32 [%0], %1;" ::"r"(sbase + L::SLO(sb) + off), "r"(lo) : "memory");
          }
        } else {
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            const float* v = &S[c * 8];
            uint32_t hi[4], lo[4];
#pragma unroll
            for (int t = 0; t < 4; ++t) {
              hi[t] = pack_bf16(v[2 * t], v[2 * t + 1]);
              lo[t] = pack_bf16(v[2 * t] - __uint_as_float(hi[t] << 16),
                                v[2 * t + 1] - __uint_as_float(hi[t] & 0xFFFF0000u));
            }
            const uint32_t off = sw128_off(uint32_t(d), uint32_t(c));
            sts128(sbase + L::SBF(sb) + off, make_uint4(hi[0], hi[1], hi[2], hi[3]));
            sts128(sbase + L::SLO(sb) + off, make_uint4(lo[0], lo[1], lo[2], lo[3]));
          }
        }
        fence_async_smem();
        mbar_arrive(&bar->st_full[sb]);
        if (g == 0) LASP_TRACE(7, J);
        // head_dim-128 forward (one pass): u . c of this block (after the first; not for the last block: no dS)
        // only now -- done before the copy above, it made the copy wait for this block's c tile, which the copy
        // does not need (forward core 130 -> 125 us at TNL-1B); in the backward the dS chain wants u . c early
        // (fused bwd 324 -> 346 us with the late order), so there it stays at the end of the previous block
        if (ku_late && j > 0 && j + 1 < it.nblk) scale_ku(Js);
        if (j + 1 == it.nblk) {  // no state leaves the last block of a segment
          Js += sub;
          break;
        }
        for (int u = 1; u < sub; ++u) scale_ku(Js + u);  // the block's other summed query heads
        // S_{J+1} = lam^128 S_J + dS_J
        mbar_wait(&bar->ds_full, kd & 1);
        if (g == 0) LASP_TRACE(6, J);
        tc_fence_after();
        const uint32_t td = tmem + ((q4 * 32) << 16) + L::T_DS;
#if defined(LASP_EXPERIMENT_NOSTATE) || defined(LASP_EXPERIMENT_NOUPD)
        if (false)
#endif
        if constexpr (SPLIT) {
          float v[32];
          tmem_ld_16x256b_x8(td, v);
          tmem_ld_wait();
#pragma unroll
          for (int t = 0; t < 32; ++t) S[t] = fmaf(decay, S[t], v[t]);
        } else {
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            float v[16];
            tmem_ld16(td + c * 16, v);
            tmem_ld_wait();
#pragma unroll
            for (int t = 0; t < 16; ++t) S[c * 16 + t] = fmaf(decay, S[c * 16 + t], v[t]);
          }
        }
        tc_fence_before();
        mbar_arrive(&bar->ds_empty);
        ++kd;
        Js += sub;
        if (!ku_late && j + 2 < it.nblk) scale_ku(Js);
      }
      ++J;  // the break skipped the increment of the last block
    }
  } else if (warp >= 12) {
    // ------------------------------------------------------------------ epilogue warps
    const uint32_t q4 = warp & 3;
    const int i = int(q4 * 32 + lane);
    const bool leader = threadIdx.x == 384;
    uint32_t J = 0;
    for (uint32_t k = 0;; ++k) {
      const int64_t w = q_fetch_warp(bar->iq, k);
      if (w >= W) break;
      const CItem it = get_citem<L::NV, GQ>(prm, w);
      const CUtensorMap* mo = &prm.mout[prm.pass[it.pass].out];
      __nv_bfloat16* outp = prm.outp[prm.pass[it.pass].out];
      const int64_t oh = prm.pass[it.pass].nh;  // heads of the output tensor
      const float r = exp2f(float(it.dir == Dir::FWD ? (i + 1) : (BT - 1 - i)) * p.l2lam[it.sh]);
      for (int j = 0; j < it.nblk; ++j, ++J) {
        mbar_wait(&bar->o_full, J & 1);
        if (i == 0) LASP_TRACE(8, J);
        tc_fence_after();
#ifdef LASP_EXPERIMENT_NOEPI  // timing experiment only: no output
        tc_fence_before();
        mbar_arrive(&bar->o_empty);
        continue;
#endif
        const uint32_t ti = tmem + ((q4 * 32) << 16) + L::T_OI;
        const uint32_t tx = tmem + ((q4 * 32) << 16) + L::T_OX;
        uint32_t pk[32];
        float rn = 1.f, ss = 0.f;
        if constexpr (NORM && L::NV == 1) {
          // Norm epilogue, whole head row in this thread: a first TMEM pass for the row's sum of squares
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            float a[16], x[16];
            tmem_ld16(ti + c * 16, a);
            tmem_ld16(tx + c * 16, x);
            tmem_ld_wait();
#pragma unroll
            for (int u = 0; u < 16; ++u) {
              const float o = fmaf(r, x[u], a[u]);
              ss = fmaf(o, o, ss);
            }
          }
          rn = 1.f / sqrtf(ss * (1.f / 64.f) + prm.norm_eps);
        }
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          float a[16], x[16];
          tmem_ld16(ti + c * 16, a);
          tmem_ld16(tx + c * 16, x);
          tmem_ld_wait();
          if (c == 3) {
            tc_fence_before();
            mbar_arrive(&bar->o_empty);
          }
#pragma unroll
          for (int u = 0; u < 16; u += 2) {
            float o0 = fmaf(r, x[u], a[u]), o1 = fmaf(r, x[u + 1], a[u + 1]);
            if constexpr (NORM && L::NV > 1) ss = fmaf(o0, o0, fmaf(o1, o1, ss));
            if constexpr (NORM && L::NV == 1) { o0 *= rn; o1 *= rn; }
            pk[c * 8 + u / 2] = pack_bf16(o0, o1);
          }
        }
        const int t0 = int(cblock_row(it, j));
        if constexpr (NORM) {  // per-row statistics of the forward O pass (rows of this segment only)
          const int64_t t = t0 + i;
          if (t >= it.beg && t < it.end) {
            const int64_t row = (it.b * p.C + t) * p.H + it.h;
            if constexpr (L::NV == 1) prm.rnorm[row] = rn;
            else prm.nsum[row * 2 + it.v] = ss;
          }
        }
        if (t0 < it.beg) {
          // ragged block of a REV pass, which starts before its segment: rows before the segment belong
          // to the previous segment's item (or precede the rank start, where TMA stores reject negative
          // coordinates), so only this segment's rows are written, directly from registers (ADVICE r1:
          // a full-tile store raced with the previous segment's store of the same rows)
          if (t0 + i >= it.beg) {
            uint4* dst = reinterpret_cast<uint4*>(outp + ((it.b * p.C + (t0 + i)) * oh + it.h) * D + it.v * 64);
#pragma unroll
            for (int c = 0; c < 8; ++c) dst[c] = make_uint4(pk[c * 4], pk[c * 4 + 1], pk[c * 4 + 2], pk[c * 4 + 3]);
          }
          continue;
        }
        const uint32_t ob = L::OST;
        if (leader) tma_store_wait_read<0>();
        named_bar_sync(1, 128);
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          const uint32_t* v = &pk[c * 4];
          sts128(sbase + ob + sw128_off(uint32_t(i), uint32_t(c)), make_uint4(v[0], v[1], v[2], v[3]));
        }
        fence_async_smem();
        named_bar_sync(1, 128);
        if (leader) {
          tma_store_4d(mo, sm + ob, it.v * 64, int(it.h), t0, int(it.b));
          tma_store_commit();
          LASP_TRACE(9, J);
        }
      }
    }
    if (leader) tma_store_wait_all<0>();
  }
  tc_fence_before();
  __syncthreads();
#ifdef LASP_TRACE_BUILD
  if (prm.trace != nullptr && threadIdx.x == 0) prm.trace[2 * 1024 + blockIdx.x * 2 + 1] = globaltimer();
#endif
  if (warp == 1) tmem_dealloc<512>(tmem);
}

bool static_items() {
  static const bool on = [] {
    const char* s = std::getenv("LASP_STATIC_ITEMS");
    return s && *s && *s != '0';
  }();
  return on;
}

int sm_count() {
  static int n = 0;
  if (n == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) n = 148;
  }
  return n;
}


template <int D, Dir DIR, bool NORM>
cudaError_t launch_seg(const Plan& p, const void* x, const void* y, float* out, cudaStream_t st,
                       unsigned* claim, const NormBwdArgs* nb, const EntryDuty* entry) {
  SegParams prm;
  std::memset(&prm, 0, sizeof prm);
  if (entry) {
    prm.entry = *entry;
    prm.has_entry = 1;
  }
  if (NORM) {
    if (nb == nullptr || DIR != Dir::REV) return cudaErrorInvalidValue;
    cudaError_t e2 = make_seq_map(&prm.my2, nb->y, p, p.H);
    if (e2 != cudaSuccess) return e2;
    prm.rnorm = nb->rnorm;
    prm.dout = static_cast<__nv_bfloat16*>(nb->dout);
  }
  prm.claim = static_items() || entry ? nullptr : claim;  // (the entry duty zeroes the counters only now)
  // F1 reads k, v (Hk heads); B1 reads q, do (H heads), summing the G query heads of each state head
  prm.sub = DIR == Dir::FWD ? 1 : int(p.G);
  const int64_t heads = DIR == Dir::FWD ? p.Hk : p.H;
  cudaError_t e;
  if ((e = make_seq_map(&prm.mx, x, p, heads)) != cudaSuccess) return e;
  if ((e = make_seq_map(&prm.my, y, p, heads)) != cudaSuccess) return e;
  prm.p = p;
  prm.out = out;
  prm.trace = g_trace ? g_trace + 16 * 64 : nullptr;  // second trace region: segment-state kernel
  auto kern = seg_state_tc_kernel<D, DIR, NORM>;
  const int smem = int(SegLayout<D, NORM>::BYTES);
  if ((e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem)) != cudaSuccess) return e;
  using SL = SegLayout<D, NORM>;
  const int64_t W = p.B * p.Hk * p.nseg * SL::VS, slots = int64_t(sm_count()) * SL::CTAS_PER_SM;
  return launch_k(kern, dim3(unsigned(W < slots ? W : slots)), dim3(384), smem, st, prm);
}

template <int D>
cudaError_t launch_core_multi(const Plan& p, int npass, const SeqArgs* a, const Dir* dirs, cudaStream_t st,
                              const PrefixFold* fold, unsigned* claim, int reserve_sms, const NormArgs* norm,
                              bool late_inputs) {
  CoreParams prm;
  std::memset(&prm, 0, sizeof prm);
  cudaError_t e;
  const void* ins[4];
  int nin = 0;
  auto in_index = [&](const void* ptr) -> int {
    for (int x = 0; x < nin; ++x)
      if (ins[x] == ptr) return x;
    ins[nin] = ptr;
    return nin++;
  };
  const float* sts[2];
  int nst = 0;
  int64_t in_heads[4] = {0, 0, 0, 0};
  uint32_t off = 0;
  constexpr int NV = CoreLayout<D>::NV;
  for (int x = 0; x < npass; ++x) {
    CorePass& ps = prm.pass[x];
    ps.dir = int(dirs[x]);
    ps.trans = a[x].trans_state;
    ps.kvp = a[x].kv_pass;
    // heads of a and out, and of b and c (grouped queries: a kv-head pass reads query-side b, c)
    const int64_t ha = ps.kvp ? p.Hk : p.H, hbc = ps.kvp ? p.H : p.Hk;
    ps.a = in_index(a[x].a);
    in_heads[ps.a] = ha;
    ps.b = in_index(a[x].b);
    in_heads[ps.b] = hbc;
    ps.c = in_index(a[x].c);
    in_heads[ps.c] = hbc;
    if (nin > 4) return cudaErrorInvalidValue;
    ps.nh = int(ha);
    ps.div_nh = FastDiv(uint32_t(ha));
    ps.off = off;
    off += uint32_t(p.B * ha * NV);
    ps.out = x;
    prm.outp[x] = static_cast<__nv_bfloat16*>(a[x].out);
    if ((e = make_seq_map(&prm.mout[x], a[x].out, p, ha)) != cudaSuccess) return e;
    ps.state = -1;
    for (int y = 0; y < nst; ++y)
      if (sts[y] == a[x].state) ps.state = y;
    if (ps.state < 0) {
      if (nst == 2) return cudaErrorInvalidValue;
      sts[nst] = a[x].state;
      if ((e = make_state_map(&prm.mst[nst], a[x].state, p)) != cudaSuccess) return e;
      prm.stp[nst] = a[x].state;
      ps.state = nst++;
    }
  }
  for (int x = 0; x < nin; ++x)
    if ((e = make_seq_map(&prm.min[x], ins[x], p, in_heads[x])) != cudaSuccess) return e;
  for (int x = nin; x < 4; ++x) prm.min[x] = prm.min[0];
  if (nst < 2) { prm.mst[1] = prm.mst[0]; prm.stp[1] = prm.stp[0]; }
  prm.p = p;
  prm.npass = npass;
  prm.status = a[0].status;
  prm.claim = claim;
  prm.trace = g_trace;
  if (fold) prm.fold = *fold;
  prm.per = off;
  prm.div_per = FastDiv(off);
  prm.div_nbh = FastDiv(uint32_t(p.B * p.H * NV));
  prm.div_h = FastDiv(uint32_t(p.H));
  prm.uniform = 1;
  for (int x = 1; x < npass; ++x) prm.uniform &= prm.pass[x].nh == prm.pass[0].nh;
  if (static_items()) prm.claim = nullptr;
  auto kern = norm != nullptr ? (p.G > 1 ? core_tc_kernel<D, true, true> : core_tc_kernel<D, false, true>)
                               : (p.G > 1 ? core_tc_kernel<D, true, false> : core_tc_kernel<D, false, false>);
  if (norm != nullptr) {
    if (npass != 1 || dirs[0] != Dir::FWD) return cudaErrorInvalidValue;
    prm.rnorm = norm->rnorm;
    prm.nsum = norm->nsum;
    prm.norm_eps = norm->eps;
  }
  prm.late_inputs = late_inputs ? 1 : 0;
  // descending segments: the preceding segment-state launch ascended, so the tiles it read last (K, V for
  // F3; Q, and for B3 also dO) are the first this launch needs, and this launch ends on the segments the next
  // ascending segment-state launch starts with (F3 -> B1 share Q). Same-box A/B: TNL-0.4B 228.0 -> 226.5 us
  // (B1 35.2 -> 33.4 us), TNL-1B 560.4 -> 559.7 us. LASP_CORE_SEG_DESC=0 restores ascending order.
  static const int seg_desc = [] {
    const char* e = std::getenv("LASP_CORE_SEG_DESC");
    return e && *e ? std::atoi(e) : 1;
  }();
  prm.seg_desc = seg_desc;
  // the ragged last segment's items are claimed last (tail of the persistent launch); LASP_SHORT_LAST=0: first
  static const int short_last = [] {
    const char* e = std::getenv("LASP_SHORT_LAST");
    return e && *e ? std::atoi(e) : 1;
  }();
  prm.short_last = short_last && p.nseg > 1 && p.C % p.seg_len != 0;
  const int smem = int(CoreLayout<D>::BYTES);
  if ((e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem)) != cudaSuccess) return e;
  const int64_t W = p.nseg * int64_t(off);
  // reserve_sms: SMs left free for kernels of another stream (the ring's NCCL kernels while a hop is in
  // flight): a persistent CTA holds an SM's whole register file and shared memory until the launch ends
  int64_t slots = sm_count() - (reserve_sms > 0 && reserve_sms < sm_count() ? reserve_sms : 0);
  const unsigned grid = unsigned(W < slots ? W : slots);
  return launch_k(kern, dim3(grid), dim3(512), smem, st, prm);
}

// Debug / experiments (lasp_debug_occupy): `ctas` CTAs that each hold most of an SM's shared memory and spin
// for `ns` nanoseconds -- a stand-in for kernels of another stream (NCCL) that occupy SMs while a persistent
// kernel of this library runs.
__global__ void occupy_kernel(unsigned long long ns) {
  extern __shared__ uint8_t sm_hog[];
  const unsigned long long t0 = globaltimer();
  while (globaltimer() - t0 < ns) {
    if (threadIdx.x == 0) sm_hog[0] = 1;
    __nanosleep(500);
  }
}

}  // namespace

cudaError_t launch_occupy(int ctas, int smem, double us, cudaStream_t st) {
  cudaError_t e = cudaFuncSetAttribute(occupy_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  occupy_kernel<<<ctas, 32, smem, st>>>((unsigned long long)(us * 1e3));
  return cudaGetLastError();
}

const char* tc_last_error() { return g_tc_err; }

bool tc_fold_fusable(const Plan& p) {
  // the fused fold runs on 256 threads per SM (a standalone prefix launch fills every SM): a win while
  // each fold thread has at most 2 elements (TNL-0.4B 16 x 64: 0.9; measured +1-1.7 %), a loss at 3.5
  // (TNL-1B 16 x 128: -0.4 %)
  static const int64_t rounds = [] {
    const char* s = std::getenv("LASP_FOLD_MAX_ROUNDS");
    return s && *s ? std::atoll(s) : int64_t(2);
  }();
  return tc_supported(p) && p.B * p.Hk * p.D * p.D / 2 <= rounds * sm_count() * kFoldChunk;
}

void tc_set_trace(unsigned long long* buf) { g_trace = buf; }

bool tc_supported(const Plan& p) {
  static const bool disabled = [] {
    const char* s = std::getenv("LASP_DISABLE_TC");
    return s && *s && *s != '0';
  }();
  // 32-bit token coordinates (TMA boxes, work items) and item indices (B * H * nseg * passes * slices)
  return !disabled && p.dtype == 0 && (p.D == 64 || p.D == 128) && p.C > 0 && p.C < (int64_t(1) << 30) &&
         p.B * p.H * p.nseg * 6 < (int64_t(1) << 31);
}

cudaError_t launch_seg_state_tc(const Plan& p, Dir dir, const void* x, const void* y, float* out, cudaStream_t st,
                                unsigned* r, const NormBwdArgs* nb, const EntryDuty* e) {
  if (r == nullptr) return cudaErrorInvalidValue;  // the work-claim counter is required
  if (nb != nullptr) {
    if (dir != Dir::REV) return cudaErrorInvalidValue;
    if (p.D == 64) return launch_seg<64, Dir::REV, true>(p, x, y, out, st, r, nb, e);
    if (p.D == 128) return launch_seg<128, Dir::REV, true>(p, x, y, out, st, r, nb, e);
    return cudaErrorNotSupported;
  }
  if (p.D == 64)
    return dir == Dir::FWD ? launch_seg<64, Dir::FWD, false>(p, x, y, out, st, r, nullptr, e)
                           : launch_seg<64, Dir::REV, false>(p, x, y, out, st, r, nullptr, e);
  if (p.D == 128)
    return dir == Dir::FWD ? launch_seg<128, Dir::FWD, false>(p, x, y, out, st, r, nullptr, e)
                           : launch_seg<128, Dir::REV, false>(p, x, y, out, st, r, nullptr, e);
  return cudaErrorNotSupported;
}

cudaError_t launch_core_tc(const Plan& p, Dir dir, const SeqArgs& a, cudaStream_t st, unsigned* claim,
                           int reserve_sms, const NormArgs* norm, bool late_inputs) {
  return launch_core_tc_multi(p, 1, &a, &dir, st, nullptr, claim, reserve_sms, norm, late_inputs);
}

cudaError_t launch_core_tc_multi(const Plan& p, int npass, const SeqArgs* a, const Dir* dirs, cudaStream_t st,
                                 const PrefixFold* fold, unsigned* claim, int reserve_sms, const NormArgs* norm,
                                 bool late_inputs) {
  if (npass < 1 || npass > 3 || claim == nullptr) return cudaErrorInvalidValue;
  if (p.D == 64) return launch_core_multi<64>(p, npass, a, dirs, st, fold, claim, reserve_sms, norm, late_inputs);
  if (p.D == 128) return launch_core_multi<128>(p, npass, a, dirs, st, fold, claim, reserve_sms, norm, late_inputs);
  return cudaErrorNotSupported;
}

}  // namespace lasp
