// lasp_common.cuh -- shared definitions of the LASP CUDA path (plan, launch interfaces).
//
// Notation (0-based, one (batch, head)):
//   C = n_local tokens of this rank, split into segments of Lseg tokens; segments are split into
//   GPU blocks of BT tokens. Every level applies the same LASP identity (Eq. 12):
//     FWD direction (O, dQ):   out_i = sum_{j<=i} lam^(i-j) (a_i.b_j) c_j + lam^(i+1) a_i^T S
//                              S'    = lam^BT S + sum_s lam^(BT-1-s) b_s c_s^T
//     REV direction (dK, dV):  out_i = sum_{j>=i} lam^(j-i) (a_i.b_j) c_j + lam^(BT-1-i) a_i^T S
//                              S'    = lam^BT S + sum_s lam^(s+1) b_s c_s^T
//   with (a,b,c,S) = (Q,K,V,KV) for O, (dO,V,K,KV^T) for dQ, (K,Q,dO,dKV) for dV and
//   (V,dO,Q,dKV^T) for dK (Eq. 4 and Eq. 13 rewritten; the REV state has exponent starting at 1,
//   reading A3). Segments are aligned to the rank start in both directions (see seg_begin), so a
//   ragged block only ever sits where no state leaves it.
#pragma once
#include <cstdint>
#include <cstdlib>
#include <utility>
#include <cuda_runtime.h>
#include <cuda_bf16.h>

namespace lasp {

// Programmatic dependent launch: every kernel of the path is launched with programmatic stream
// serialization, so a kernel's prologue (TMEM alloc, barrier init, descriptor prefetch) and its CTAs'
// start overlap the previous kernel's tail. The first kernel of every call (tag_kernel) executes
// griddepcontrol.wait -- which returns only once the preceding grid has COMPLETED, whether or not it
// triggered early -- before it triggers the call's next kernel; so every later kernel of the call starts
// after all work that preceded the call on the stream is complete and visible, whoever produced the
// inputs, and PDL edges that skip a wait exist only between kernels of one call, where the
// library controls both sides. LASP_NO_PDL=1 disables PDL (debugging).
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

inline bool pdl_enabled() {
  static const bool on = [] {
    const char* s = std::getenv("LASP_NO_PDL");
    return !(s && *s && *s != '0');
  }();
  return on;
}

template <typename... KArgs, typename... Args>
cudaError_t launch_k(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

enum class Dir : int { FWD = 0, REV = 1 };

// x / d for 0 <= x < 2^31 as one multiply-high and a shift (work-item decode in the persistent kernels:
// a runtime 32-bit division is a ~20-instruction dependent chain per call). Round-up multiplier
// m = ceil(2^p / d), p = 31 + ceil(log2 d) (the construction CUTLASS's FastDivmod uses).
struct FastDiv {
  uint32_t d = 1, m = 0, sh = 0;
  FastDiv() = default;
  explicit FastDiv(uint32_t div) : d(div) {
    if (d <= 1) return;
    uint32_t l = 0;
    while ((1u << l) < d) ++l;
    const uint32_t p = 31 + l;
    m = uint32_t(((uint64_t(1) << p) + d - 1) / d);
    sh = p - 32;
  }
  __host__ __device__ __forceinline__ uint32_t div(uint32_t x) const {
#ifdef __CUDA_ARCH__
    return d == 1 ? x : (__umulhi(x, m) >> sh);
#else
    return d == 1 ? x : uint32_t((uint64_t(x) * m) >> (32 + sh));
#endif
  }
};

struct Plan {
  int64_t B, C, H, D;  // batch, n_local, (query) heads, head_dim
  int64_t Hk, G;       // key/value heads = state heads, and query heads per kv-head (G = H / Hk; MHA: Hk = H)
  int dtype;           // 0 = bf16, 1 = fp32
  int64_t seg_len;     // multiple of kSegQuantum
  int64_t nseg;        // >= 1
  FastDiv div_bhk, div_hk;  // / (B*Hk), / Hk (work-item decode of the state kernels)
  float lam[256];      // per-state-head decay (fp32, the boundary's precision; reading A8), by value, [Hk]
  float l2lam[256];    // log2(lam) computed in fp64 on the host, rounded once (tcgen05 path: exp2 powers)
};
constexpr int64_t kMaxHeads = 256;

constexpr int64_t kSegQuantum = 128;  // every kernel's block size divides this

// Segment p geometry (both directions): [p*L, min((p+1)*L, C)). FWD blocks ascend from the segment
// begin, REV blocks descend from the segment end, so a ragged block is the last one processed in its
// segment (no state leaves it); REV folds segments from p = nseg-1 down to 0. Using the same token
// ranges in both directions lets the backward passes of one segment run side by side (L2 reuse).
__host__ __device__ inline int64_t seg_begin(Dir, int64_t p, int64_t L, int64_t) { return p * L; }
__host__ __device__ inline int64_t seg_end(Dir, int64_t p, int64_t L, int64_t C) {
  const int64_t e = (p + 1) * L;
  return e > C ? C : e;
}

// KV-cache tag (SURVEY §8(b) "cache header"; S:411 backward without a matching forward -> STATE): 16
// words stored in the cache itself, after the segment states. The forward's entry kernel writes it; the
// backward's entry kernel compares the words selected by a mask and writes the mismatch bits into the
// call's status word (workspace). A backward whose status is nonzero poisons every state it loads with
// NaN, so all its outputs are NaN (loud), and lasp_workspace_status() reports LASP_ERR_STATE.
enum TagWord { kTagMagic = 0, kTagB, kTagC, kTagH, kTagD, kTagSeg, kTagDtype, kTagLam, kTagRank, kTagWorld,
               kTagHk, kTagGen, kTagWords = 16 };
struct CacheTag { uint64_t w[kTagWords]; };
constexpr size_t kCacheTagBytes = 256;
constexpr uint64_t kTagMagicValue = 0x4c41535043414348ull;  // "LASPCACH"
// check_mask == 0: write the tag, else compare the masked words; the mismatch bits go to ctrl[2] (the
// call's status word) and the other 15 words of the call's control block (counters) are zeroed
cudaError_t launch_tag(const CacheTag& t, uint64_t* hdr, unsigned check_mask, unsigned* ctrl, cudaStream_t st);
// The entry duty of a call, run by one warp after griddepcontrol.wait (tag_kernel, or the first CTA of the call's
// first segment-state launch): write (check_mask == 0) or compare the cache tag and reset the call's 16-word
// control block (fold counters, status word = the tag mismatch bits, work-claim counters).
__device__ __forceinline__ void entry_duty(const CacheTag& t, uint64_t* hdr, unsigned check_mask, unsigned* ctrl) {
  const int i = int(threadIdx.x & 31);
  bool bad = false;
  if (check_mask == 0u) {
    if (i < kTagWords) hdr[i] = t.w[i];
  } else {
    bad = i < kTagWords && ((check_mask >> i) & 1u) && hdr[i] != t.w[i];
  }
  const unsigned bits = __ballot_sync(0xffffffffu, bad);
  if (i < 16) ctrl[i] = i == 2 ? bits : 0u;
}
struct EntryDuty {       // passed to the first launch of a call instead of a separate tag_kernel launch
  CacheTag tag;
  uint64_t* hdr;
  unsigned check_mask;
  unsigned* ctrl;
};
// true (on the device) when the call's entry kernel found a mismatching cache tag
__device__ __forceinline__ bool tag_poisoned(const unsigned* status) { return status != nullptr && __ldcg(status) != 0u; }

// Kernel launch interfaces (kernels_simt.cu, kernels_tc.cu). All return cudaGetLastError().
// Sequence tensors are [B][C][H][D] (queries-side: q, o, do, dq) or [B][C][Hk][D] (k, v, dk, dv); state
// arrays are [B][Hk][nseg][D][D] fp32.
struct SeqArgs {
  const void* a; const void* b; const void* c;  // core: out rows from a, keys b, values c
  void* out;
  const float* state;     // device [B][Hk][nseg][D][D] (state entering each segment)
  int trans_state;        // use S^T of the stored state
  const unsigned* status = nullptr;  // cache-tag status of the call (backward), nullptr = unchecked
  // grouped-query passes (NEXT-4): 0 = a query-head pass (O, dQ: items over the H query heads, a and out
  // have H heads, b, c and the state are those of kv-head h / G); 1 = a kv-head pass (dV, dK: items over
  // the Hk kv-heads, a and out have Hk heads, and every block sums the G query heads h = hk G + u of b, c)
  int kv_pass = 0;
};

cudaError_t launch_seg_state_simt(const Plan& p, Dir dir, const void* x, const void* y,
                                  float* out, cudaStream_t st);
cudaError_t launch_prefix(const Plan& p, Dir dir, const float* init, const float* seg_states,
                          float* prefix_out, float* final_out, cudaStream_t st);
cudaError_t launch_core_simt(const Plan& p, Dir dir, const SeqArgs& a, cudaStream_t st);
// dst[0..n) = src (n = B*H*D*D), then p.C as an int64 at dst + n (all-gather message)
cudaError_t launch_pack_state(const Plan& p, const float* src, float* dst, cudaStream_t st);
// gathered: [world][stride] fp32, rank j's state at j*stride, its n_local (int64) at j*stride + n
cudaError_t launch_fold_ranks(const Plan& p, const float* gathered, int64_t stride, int j0, int step, int count,
                              float* out, cudaStream_t st);
cudaError_t launch_combine(const Plan& p, const float* kv_in, const float* local, float* kv_out,
                           cudaStream_t st);
// P2P exchange hop (kernels_simt.cu p2p_hop_kernel): flags and buffers as in the kernel's comment
constexpr int kP2PCtas = 16;
struct P2PHop {
  const float* local;     // this rank's local state (L_r or G_r), n floats
  float* in_priv;         // out: the received state (KV_in / dKV_in), n floats (workspace)
  const float* my_recv;   // this rank's receive buffer for dir (written by the upstream rank)
  uint64_t* my_flags;     // this rank's 8 flag words
  float* peer_recv;       // the downstream rank's receive buffer for dir (peer memory), nullptr: no downstream
  uint64_t* peer_flags;   // the downstream rank's flag words
  uint64_t* up_flags;     // the upstream rank's flag words (ack), when has_up
  int has_up;             // an upstream rank exists (else KV_in = 0)
  int dir;                // 0 forward, 1 backward
  int64_t n;
};
cudaError_t launch_p2p_hop(const Plan& p, const P2PHop& h, cudaStream_t st);
// P2P all-gather exchange (kernels_simt.cu p2p_gather_kernel): bases[k] = rank k's gather block (peer memory)
constexpr int kP2PMaxWorld = 64;
constexpr size_t kP2PFlagBytes = 4096;
struct P2PGather {
  const float* local;            // this rank's local state, n floats
  float* in_priv;                // out: KV_in / dKV_in folded from the gathered states
  char* bases[kP2PMaxWorld];
  size_t slot_bytes;             // per (direction, source rank): n floats + the source's n_local (int64)
  int rank, world, dir;
  int64_t n;
};
cudaError_t launch_p2p_gather(const Plan& p, const P2PGather& g, cudaStream_t st);

// Segment-prefix fold (F2 / B2, same arithmetic as prefix_kernel) run by a core launch before its main
// loop: the 256 state + epilogue threads of each CTA claim chunks of elements (gbar[0]) and fold them;
// prefix states are read once every chunk is done (gbar[1]). Both counters are zeroed by the call's
// entry kernel (tag_kernel).
struct PrefixFold {
  const float* init;  // state entering the rank, or nullptr (zero)
  const float* seg;   // segment states [B][H][nseg][D][D]
  float* out;         // prefix states (may alias seg)
  float* fin;         // state leaving the rank, or nullptr
  unsigned* gbar;     // [2]: chunks claimed, chunks done; zeroed by the call's entry kernel
  int dir;            // Dir
};

// tcgen05 path (bf16 only); returns cudaErrorNotSupported when the shape is not covered.
bool tc_supported(const Plan& p);
bool tc_fold_fusable(const Plan& p);  // fuse the prefix fold into the core launch (small enough state)
const char* tc_last_error();
void tc_set_trace(unsigned long long* buf);  // debug: per-block clock64 timeline of CTA 0  // detail of the last tcgen05-path host failure on this thread
// Norm backward fused into B1 (NEXT-3): y here is dY; dO = r (dY - y_fwd (y_fwd . dY) / D) is formed per row
// in shared memory, used as the MMA operand and written to dout for the B3 passes
struct NormBwdArgs {
  const void* y;       // forward output Norm(O) [B][C][H][D] bf16
  const float* rnorm;  // [B][C][H]
  void* dout;          // [B][C][H][D] bf16, written
};
// claim: the launch's work-claim counter (a workspace word zeroed by the call's entry kernel)
// entry != nullptr: this launch is the call's first kernel and also runs the entry duty (no tag_kernel): its
// producer waits for all earlier work before loading, items are assigned statically (the claim counters are only
// zeroed by the duty), and CTA 0 triggers the next kernel only after the control block is reset
cudaError_t launch_seg_state_tc(const Plan& p, Dir dir, const void* x, const void* y, float* out,
                                cudaStream_t st, unsigned* claim, const NormBwdArgs* norm_bwd = nullptr,
                                const EntryDuty* entry = nullptr);
// Norm(.) of Eq. 2 (NEXT-3, reading N1: per-head RMS normalization) fused into the forward core's epilogue
constexpr float kNormEps = 1e-6f;  // reading N1
struct NormArgs {
  float* rnorm;   // [B][C][H] fp32: r = (mean_c o_c^2 + eps)^-1/2 (head_dim 64: written by the core epilogue)
  float* nsum;    // [B][C][H][2] fp32: per-value-slice sums of squares (head_dim 128; norm_apply finishes)
  float eps;
};
// reserve_sms: leave that many SMs free for another stream's kernels (ring hop in flight); norm: the
// forward O pass writes Norm(O) (NormArgs); late_inputs: an input is produced by the preceding kernel
cudaError_t launch_core_tc(const Plan& p, Dir dir, const SeqArgs& a, cudaStream_t st, unsigned* claim,
                           int reserve_sms = 0, const NormArgs* norm = nullptr, bool late_inputs = false);
// up to 3 core passes in one persistent launch (their segments interleaved: shared inputs hit L2);
// fold != nullptr: the launch first computes the prefix states its passes read (PrefixFold)
cudaError_t launch_core_tc_multi(const Plan& p, int npass, const SeqArgs* a, const Dir* dirs, cudaStream_t st,
                                 const PrefixFold* fold, unsigned* claim, int reserve_sms = 0,
                                 const NormArgs* norm = nullptr, bool late_inputs = false);
// head_dim 128 second phase of the Norm epilogue: y = o r in place from the two slice sums (nsum)
cudaError_t launch_norm_apply(const Plan& p, void* y, const NormArgs& n, cudaStream_t st);
cudaError_t launch_occupy(int ctas, int smem, double us, cudaStream_t st);  // debug: SM hog on another stream

}  // namespace lasp
