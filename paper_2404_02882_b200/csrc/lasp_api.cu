// lasp_api.cu -- the C ABI declared in include/lasp.h: validation, planning, the KV-cache tag
// registry, stage orchestration (Alg. 2 / Alg. 3 per rank) and the NCCL P2P ring.
//
// Stage order per rank:
//   forward : F1 seg_state(K,V) -> [ring: recv KV_in, combine, send] -> F2 prefix(KV_in) -> F3 core
//   backward: B1 seg_state(Q,dO) -> [ring: recv dKV_in, combine, send] || B3a core(dQ, cache)
//             -> B2 prefix(dKV_in) -> B3b core(dV), core(dK)
// The KV-independent local parts (F1/B1) are hoisted in front of the ring hop, so the hop carries
// lambda^C * received + local (Alg. 2, Alg. 3), and dQ overlaps the dKV ring.
#include "../../include/lasp.h"
#include "gla.cuh"
#include "lasp_common.cuh"

#include <cublas_v2.h>
#include <dlfcn.h>
#include <nccl.h>

#include <atomic>
#include <chrono>
#include <condition_variable>
#include <deque>
#include <map>
#include <memory>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <unordered_map>
#include <vector>

using namespace lasp;

namespace {

thread_local std::string g_err;

lasp_status_t fail(lasp_status_t st, const std::string& msg) {
  g_err = msg;
  return st;
}

lasp_status_t cuda_fail(cudaError_t e, const char* where) {
  std::string msg = std::string(where) + ": " + cudaGetErrorString(e);
  const char* tc = tc_last_error();
  if (tc && *tc) msg += std::string(" [") + tc + "]";
  return fail(LASP_ERR_CUDA, msg);
}

#define LASP_CUDA(call)                                       \
  do {                                                        \
    cudaError_t e_ = (call);                                  \
    if (e_ != cudaSuccess) return cuda_fail(e_, #call);       \
  } while (0)

// ---- planning --------------------------------------------------------------------------------
int64_t env_i64(const char* name, int64_t dflt) {
  const char* s = std::getenv(name);
  if (!s || !*s) return dflt;
  return std::atoll(s);
}

// Segments per (batch, head) such that the core launch has ~4 work items per SM: an item is one
// (segment, batch x head, 64-wide value slice), so head_dim 128 (2 value slices) takes half as many
// segments as head_dim 64 (measured: TNL-1B 56.9 -> 57.3 M tokens/s; TNL-0.4B is optimal at 4 x 148).
// Head_dim 128 takes ~5 items per SM (same-box sweep 296..888 with the (batch x head, pass, value slice)
// item order: TNL-1B 56.7 -> 57.0 M tokens/s, TNL-7B 27.42 -> 27.62 M; profiles/r1j_target_*.txt).
int64_t choose_seg_len(int64_t B, int64_t C, int64_t H, int64_t D) {
  const int64_t q = kSegQuantum;
  const int64_t forced = env_i64("LASP_SEG_LEN", 0);
  if (forced > 0) return ((forced + q - 1) / q) * q;
  if (C <= 0) return q;
  const int64_t nb = (C + q - 1) / q;
  const int64_t nv = D >= 128 ? D / 64 : 1;  // value slices per item (tensor-core core kernel)
  // head_dim 128 with enough work: segments of 28 blocks (3584 tokens), if the forward launch still gets at least
  // two items per SM. Same-box sweeps (profiles/r4q_*, r4p_*): TNL-1B 58.5 -> 59.9 M tokens/s (10 segments instead
  // of 24: the ragged last segment's short items, claimed last, fill the final wave of the long ones), TNL-7B
  // 30.0 -> 30.9 M (37 instead of 12: the 86-block items left the last wave's SMs idle); 22- and 19-block segments
  // lost at TNL-1B (56.0), so the block count is a measured value, not a model. LASP_LONG_SEG_BLOCKS=0: off.
  if (nv > 1) {
    const int64_t lb = env_i64("LASP_LONG_SEG_BLOCKS", 28);
    if (lb > 0 && B * H * nv * ((nb + lb - 1) / lb) >= 2 * 148) return lb * q;
  }
  const int64_t target = env_i64("LASP_TARGET_CTAS", (nv > 1 ? 5 : 4) * 148);
  int64_t nseg_t = (target + B * H * nv - 1) / (B * H * nv);
  if (nseg_t < 1) nseg_t = 1;
  if (nseg_t > nb) nseg_t = nb;
  int64_t seg_blocks = (nb + nseg_t - 1) / nseg_t;
  // short sequences: a segment of one or two blocks spends most of its item on pipeline fill and the fold;
  // at least 2 blocks (head_dim 64) / 4 blocks (head_dim 128) per segment (sweep profiles/r2x_short.txt: 2K
  // tokens 16 x 64 40.1 -> 44.3 M tokens/s, 16 x 128 20.9 -> 23.1 M; 32K unaffected: 7 / 11 blocks already)
  const int64_t min_blocks = env_i64("LASP_MIN_SEG_BLOCKS", nv > 1 ? 4 : 2);
  if (seg_blocks < min_blocks) seg_blocks = min_blocks < nb ? min_blocks : nb;
  return seg_blocks * q;
}

int64_t kv_heads(const lasp_shape_t* s) { return s->kv_heads > 0 ? s->kv_heads : s->heads; }

lasp_status_t validate_shape(const lasp_shape_t* s) {
  if (!s) return fail(LASP_ERR_SHAPE, "shape is NULL");
  if (s->batch < 1 || s->n_local < 0 || s->heads < 1 || s->kv_heads < 0)
    return fail(LASP_ERR_SHAPE, "need batch >= 1, n_local >= 0, heads >= 1, kv_heads >= 0");
  if (s->heads > kMaxHeads) return fail(LASP_ERR_UNSUPPORTED, "heads > 256 not supported");
  if (s->head_dim != 32 && s->head_dim != 64 && s->head_dim != 128)
    return fail(LASP_ERR_UNSUPPORTED, "head_dim must be 32, 64 or 128");
  if (s->dtype != LASP_BF16 && s->dtype != LASP_FP32) return fail(LASP_ERR_SHAPE, "bad dtype");
  if (s->heads % kv_heads(s) != 0) return fail(LASP_ERR_SHAPE, "kv_heads must divide heads (grouped-query attention)");
  if (kv_heads(s) != s->heads && !(s->dtype == LASP_BF16 && (s->head_dim == 64 || s->head_dim == 128)))
    return fail(LASP_ERR_UNSUPPORTED, "grouped-query attention (kv_heads < heads) needs bf16 and head_dim 64 or 128");
  return LASP_OK;
}

Plan make_plan(const lasp_shape_t* s) {
  Plan p{};
  p.B = s->batch; p.C = s->n_local; p.H = s->heads; p.D = s->head_dim;
  p.Hk = kv_heads(s);
  p.G = p.H / p.Hk;
  p.dtype = s->dtype == LASP_BF16 ? 0 : 1;
  p.seg_len = choose_seg_len(p.B, p.C, p.H, p.D);
  p.nseg = p.C > 0 ? (p.C + p.seg_len - 1) / p.seg_len : 1;
  p.div_bhk = FastDiv(uint32_t(p.B * p.Hk));
  p.div_hk = FastDiv(uint32_t(p.Hk));
  return p;
}

// one decay per state head (kv-head): the state of a query group is shared, so is its decay (reading G1)
lasp_status_t load_lambda(Plan& p, const float* lambda) {
  if (!lambda) return fail(LASP_ERR_SHAPE, "lambda is NULL");
  for (int64_t h = 0; h < p.Hk; ++h) {
    const float l = lambda[h];
    if (!(l > 0.f && l <= 1.f)) {
      char buf[96];
      std::snprintf(buf, sizeof buf, "lambda[%lld] = %g outside (0, 1]", (long long)h, (double)l);
      return fail(LASP_ERR_DOMAIN, buf);
    }
    p.lam[h] = l;
    p.l2lam[h] = float(std::log2(double(l)));
  }
  return LASP_OK;
}

size_t state_elems(const Plan& p) { return size_t(p.B * p.Hk * p.D * p.D); }
size_t seg_state_elems(const Plan& p) { return size_t(p.B * p.Hk * p.nseg * p.D * p.D); }
size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

struct Workspace {
  unsigned* gbar;   // control block (16 words, zeroed by the call's entry kernel): [0..1] fused prefix
                    // fold counters, [2] cache-tag status of the call, [3..5] work-claim counters
  float* seg;       // [B][H][nseg][D][D]
  float* local;     // [B][H][D][D] local total (ring)
  float* in;        // received state
  float* out;       // state to send
  unsigned* status() const { return gbar + 2; }
  unsigned* claim(int i) const { return gbar + 3 + i; }  // 0: segment states, 1: first core, 2: second core
};

// the 256-byte control block sits at the start, so lasp_workspace_status needs no shape
Workspace carve(const Plan& p, void* ws) {
  char* c = static_cast<char*>(ws);
  Workspace w;
  w.gbar = reinterpret_cast<unsigned*>(c);
  c += 256;
  w.seg = reinterpret_cast<float*>(c);
  c += align256(seg_state_elems(p) * 4);
  w.local = reinterpret_cast<float*>(c);
  c += align256(state_elems(p) * 4);
  w.in = reinterpret_cast<float*>(c);
  c += align256(state_elems(p) * 4);
  w.out = reinterpret_cast<float*>(c);
  return w;
}

size_t workspace_bytes(const Plan& p) {
  return 256 + align256(seg_state_elems(p) * 4) + 3 * align256(state_elems(p) * 4);
}

size_t cache_bytes(const Plan& p) { return align256(seg_state_elems(p) * 4) + kCacheTagBytes; }
uint64_t* cache_tag_ptr(const Plan& p, const void* cache) {
  return reinterpret_cast<uint64_t*>(static_cast<char*>(const_cast<void*>(cache)) + align256(seg_state_elems(p) * 4));
}

bool aligned16(const void* ptr) { return (reinterpret_cast<uintptr_t>(ptr) & 15) == 0; }

lasp_status_t check_ptrs(const Plan& p, std::initializer_list<const void*> seq, const void* cache,
                         const void* ws) {
  if (p.C > 0)
    for (const void* x : seq)
      if (!x || !aligned16(x)) return fail(LASP_ERR_SHAPE, "sequence tensor NULL or not 16-byte aligned");
  if (!cache || !aligned16(cache)) return fail(LASP_ERR_SHAPE, "cache NULL or not 16-byte aligned");
  if (!ws || !aligned16(ws)) return fail(LASP_ERR_SHAPE, "workspace NULL or not 16-byte aligned");
  return LASP_OK;
}

// ---- device check: the kernels are compiled for sm_100a only -----------------------------------
lasp_status_t check_device() {
  static std::mutex mu;
  static std::unordered_map<int, bool> ok;
  int dev = 0;
  LASP_CUDA(cudaGetDevice(&dev));
  // make the primary context current on this thread (driver-API calls such as the TMA descriptor
  // encode need it; e.g. torch's autograd worker threads may not have bound it yet)
  thread_local int bound_dev = -1;
  if (bound_dev != dev) {
    LASP_CUDA(cudaSetDevice(dev));
    LASP_CUDA(cudaFree(nullptr));
    bound_dev = dev;
  }
  std::lock_guard<std::mutex> g(mu);
  auto it = ok.find(dev);
  if (it == ok.end()) {
    int maj = 0, min = 0;
    LASP_CUDA(cudaDeviceGetAttribute(&maj, cudaDevAttrComputeCapabilityMajor, dev));
    LASP_CUDA(cudaDeviceGetAttribute(&min, cudaDevAttrComputeCapabilityMinor, dev));
    it = ok.emplace(dev, maj == 10 && min == 0).first;
  }
  if (!it->second) return fail(LASP_ERR_UNSUPPORTED, "device is not sm_100 (B200); kernels are sm_100a only");
  return LASP_OK;
}

// ---- KV-cache tag (backward before/without a matching forward -> STATE) ---------------------
// The tag lives in the cache (after the segment states): the forward's entry kernel writes it, the
// backward's entry kernel compares it on the device (no host-side registry: a reused or foreign buffer is
// judged by its contents) and records mismatching words in the call's status word.
uint64_t hash_lam(const Plan& p) {
  uint64_t h = 1469598103934665603ull;
  for (int64_t i = 0; i < p.Hk; ++i) {
    uint32_t bits;
    std::memcpy(&bits, &p.lam[i], 4);
    h = (h ^ bits) * 1099511628211ull;
  }
  return h;
}

std::atomic<uint64_t> g_generation{0};

CacheTag make_tag(const Plan& p, int rank, int world) {
  CacheTag t{};
  t.w[kTagMagic] = kTagMagicValue;
  t.w[kTagB] = uint64_t(p.B); t.w[kTagC] = uint64_t(p.C); t.w[kTagH] = uint64_t(p.H); t.w[kTagD] = uint64_t(p.D);
  t.w[kTagSeg] = uint64_t(p.seg_len);
  t.w[kTagDtype] = uint64_t(p.dtype);
  t.w[kTagLam] = hash_lam(p);
  t.w[kTagRank] = uint64_t(int64_t(rank));
  t.w[kTagWorld] = uint64_t(int64_t(world));
  t.w[kTagHk] = uint64_t(p.Hk);
  t.w[kTagGen] = ++g_generation;  // diagnostics only (not compared)
  return t;
}

unsigned tag_mask(bool check_rank) {
  unsigned m = 0;
  for (int i = kTagMagic; i <= kTagLam; ++i) m |= 1u << i;
  m |= 1u << kTagHk;
  if (check_rank) m |= (1u << kTagRank) | (1u << kTagWorld);
  return m;
}

// ---- launch accounting and optional per-stage CUDA-event profiling -----------------------------
std::atomic<uint64_t> g_launches{0};
std::atomic<int> g_profile{0};
struct ProfRec { const char* name; cudaEvent_t a, b; };
std::mutex g_prof_mu;
std::vector<ProfRec> g_prof_recs;
std::vector<cudaEvent_t> g_prof_pool;

cudaEvent_t prof_event() {
  cudaEvent_t e = nullptr;
  if (!g_prof_pool.empty()) { e = g_prof_pool.back(); g_prof_pool.pop_back(); return e; }
  cudaEventCreate(&e);
  return e;
}

template <class F>
cudaError_t staged(const char* name, cudaStream_t st, F&& launch) {
  ProfRec rec{name, nullptr, nullptr};
  const bool prof = g_profile.load(std::memory_order_relaxed) != 0;
  if (prof) {
    std::lock_guard<std::mutex> g(g_prof_mu);
    rec.a = prof_event();
    rec.b = prof_event();
  }
  if (prof) cudaEventRecord(rec.a, st);
  cudaError_t e = launch();
  if (prof) {
    cudaEventRecord(rec.b, st);
    std::lock_guard<std::mutex> g(g_prof_mu);
    g_prof_recs.push_back(rec);
  }
  if (e == cudaSuccess) g_launches.fetch_add(1, std::memory_order_relaxed);
  return e;
}

// entry kernel of a call: write (forward) or check (backward) the cache tag; it waits for the completion of
// all preceding work before it triggers, so the call's later kernels (PDL) only ever overlap kernels of the
// same call
cudaError_t entry_tag(const Plan& p, const void* cache, const Workspace& w, int rank, int world, bool check,
                      bool check_rank, cudaStream_t st) {
  const CacheTag t = make_tag(p, rank, world);
  return staged(check ? "tag_check" : "tag_write", st, [&] {
    return launch_tag(t, cache_tag_ptr(p, cache), check ? tag_mask(check_rank) : 0u, w.gbar, st);
  });
}

// The first kernel of a call: on the tensor-core path with tokens, the segment-state launch carries the entry duty
// (one kernel boundary less per call; LASP_SEPARATE_ENTRY=1 keeps tag_kernel); otherwise tag_kernel runs it.
bool entry_in_seg_state(const Plan& p) {
  static const bool sep = [] {
    const char* s = std::getenv("LASP_SEPARATE_ENTRY");
    return s && *s && *s != '0';
  }();
  return !sep && p.C > 0 && tc_supported(p);
}
EntryDuty make_entry(const Plan& p, const void* cache, const Workspace& w, int rank, int world, bool check,
                     bool check_rank) {
  EntryDuty e{};
  e.tag = make_tag(p, rank, world);
  e.hdr = cache_tag_ptr(p, cache);
  e.check_mask = check ? tag_mask(check_rank) : 0u;
  e.ctrl = w.gbar;
  return e;
}

// a profiled span that is not one launch (the ring hop / state exchange: receive ... send on one stream,
// including the wait for the upstream rank): events recorded only while profiling is enabled
struct ProfSpan {
  ProfRec rec{nullptr, nullptr, nullptr};
  ProfSpan(const char* name, cudaStream_t st) {
    if (g_profile.load(std::memory_order_relaxed) == 0) return;
    std::lock_guard<std::mutex> g(g_prof_mu);
    rec = ProfRec{name, prof_event(), prof_event()};
    cudaEventRecord(rec.a, st);
  }
  void stop(cudaStream_t st) {
    if (!rec.a) return;
    cudaEventRecord(rec.b, st);
    std::lock_guard<std::mutex> g(g_prof_mu);
    g_prof_recs.push_back(rec);
    rec.a = nullptr;
  }
};

// ---- stage dispatch: tcgen05 for covered bf16 shapes, CUDA cores otherwise ---------------------
cudaError_t seg_state(const Plan& p, Dir dir, const void* x, const void* y, float* out, cudaStream_t st,
                      unsigned* claim, const NormBwdArgs* nb = nullptr, const EntryDuty* entry = nullptr) {
  const bool tc = tc_supported(p);
  if ((nb || entry) && !tc) return cudaErrorNotSupported;
  return staged(dir == Dir::FWD ? (tc ? "seg_state_fwd_tc" : "seg_state_fwd_simt")
                                : (tc ? (nb ? "seg_state_rev_norm_tc" : "seg_state_rev_tc") : "seg_state_rev_simt"), st, [&] {
    return tc ? launch_seg_state_tc(p, dir, x, y, out, st, claim, nb, entry)
              : launch_seg_state_simt(p, dir, x, y, out, st);
  });
}

// Local path on the tensor cores: the F2 / B2 prefix fold runs inside the following core launch (one
// launch less per direction; PrefixFold) when the states are small enough (tc_fold_fusable).
// LASP_NO_FUSED_FOLD=1 keeps the separate prefix kernel.
bool fused_fold(const Plan& p) {
  static const bool off = [] {
    const char* s = std::getenv("LASP_NO_FUSED_FOLD");
    return s && *s && *s != '0';
  }();
  return !off && tc_fold_fusable(p);
}

cudaError_t core(const Plan& p, Dir dir, const void* a, const void* b, const void* c, void* out,
                 const float* state, int trans, cudaStream_t st, unsigned* claim, const unsigned* status = nullptr,
                 int reserve_sms = 0, const NormArgs* norm = nullptr, bool late_inputs = false) {
  SeqArgs args{a, b, c, out, state, trans, status};
  const bool tc = tc_supported(p);
  if (norm && !tc) return cudaErrorNotSupported;
  return staged(dir == Dir::FWD ? (tc ? "core_fwd_tc" : "core_fwd_simt") : (tc ? "core_rev_tc" : "core_rev_simt"),
                st, [&] {
                  return tc ? launch_core_tc(p, dir, args, st, claim, reserve_sms, norm, late_inputs)
                            : launch_core_simt(p, dir, args, st);
                });
}

// SMs the ring's dQ launch leaves free for the dKV hop's NCCL kernels on the comm stream (P:296 overlap):
// a persistent core CTA holds an SM's whole register file and shared memory, so without free SMs the hop
// could only start once dQ has finished. LASP_COMM_SMS overrides (0 disables).
int comm_sms() {
  static const int n = int(env_i64("LASP_COMM_SMS", 4));
  return n;
}

cudaError_t prefix(const Plan& p, Dir dir, const float* init, const float* seg, float* out, float* fin,
                   cudaStream_t st) {
  return staged(dir == Dir::FWD ? "prefix_fwd" : "prefix_rev", st,
                [&] { return launch_prefix(p, dir, init, seg, out, fin, st); });
}

cudaError_t combine(const Plan& p, const float* in, const float* local, float* out, cudaStream_t st) {
  return staged("combine", st, [&] { return launch_combine(p, in, local, out, st); });
}

// several core passes: one persistent tensor-core launch (passes of a segment interleaved, their
// shared inputs re-read from L2), or one CUDA-core launch per pass
cudaError_t core_multi(const Plan& p, int npass, const SeqArgs* a, const Dir* dirs, cudaStream_t st,
                       unsigned* claim, const PrefixFold* fold = nullptr, const NormArgs* norm = nullptr,
                       bool late_inputs = false) {
  if (tc_supported(p))
    return staged(npass == 3 ? "core_bwd3_tc" : npass == 1 && dirs[0] == Dir::FWD ? "core_fwd_tc" : "core_multi_tc", st,
                  [&] { return launch_core_tc_multi(p, npass, a, dirs, st, fold, claim, 0, norm, late_inputs); });
  if (norm) return cudaErrorNotSupported;
  for (int x = 0; x < npass; ++x) {
    cudaError_t e = staged(dirs[x] == Dir::FWD ? "core_fwd_simt" : "core_rev_simt", st,
                           [&] { return launch_core_simt(p, dirs[x], a[x], st); });
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

// ---- common prologue -------------------------------------------------------------------------
lasp_status_t prologue(const lasp_shape_t* shape, const float* lambda, Plan& p) {
  lasp_status_t s = validate_shape(shape);
  if (s != LASP_OK) return s;
  p = make_plan(shape);
  return load_lambda(p, lambda);
}

// Forward compute after KV_in is known (F2 prefix + F3 core). `seg` already holds F1's states. gbar:
// fused-fold counters (zeroed by F1's launch) or nullptr for the separate prefix kernel.
lasp_status_t fwd_tail(const Plan& p, const void* q, const void* k, const void* v, const float* kv_in,
                       void* o, float* kv_out, void* cache, float* seg, unsigned* gbar, unsigned* claim,
                       cudaStream_t st, const NormArgs* norm = nullptr) {
  float* P = static_cast<float*>(cache);
  if (p.C == 0) {
    LASP_CUDA(prefix(p, Dir::FWD, kv_in, nullptr, P, kv_out, st));
    return LASP_OK;
  }
  if (gbar) {
    const PrefixFold fold{kv_in, seg, P, kv_out, gbar, int(Dir::FWD)};
    const SeqArgs a{q, k, v, o, P, 0};
    const Dir dir = Dir::FWD;
    LASP_CUDA(core_multi(p, 1, &a, &dir, st, claim, &fold, norm));
  } else {
    LASP_CUDA(prefix(p, Dir::FWD, kv_in, seg, P, kv_out, st));
    LASP_CUDA(core(p, Dir::FWD, q, k, v, o, P, 0, st, claim, nullptr, 0, norm));
  }
  if (norm && p.D == 128)  // two value-slice items per head row: the row statistics meet in a second phase
    LASP_CUDA(staged("norm_apply", st, [&] { return launch_norm_apply(p, o, *norm, st); }));
  return LASP_OK;
}

// ---- NCCL, loaded lazily so that the library works without it (local path) -------------------
struct NcclApi {
  bool loaded = false;
  std::string why;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    // LASP_NCCL_LIB (the Python binding points it at torch's bundled NCCL), else the loader's search path
    const char* cands[] = {std::getenv("LASP_NCCL_LIB"), "libnccl.so.2"};
    void* h = nullptr;
    for (const char* c : cands)
      if (c && (h = dlopen(c, RTLD_NOW | RTLD_GLOBAL))) break;
    if (!h) { api.why = "libnccl.so.2 not found (set LASP_NCCL_LIB)"; return; }
    api.GetUniqueId = (decltype(api.GetUniqueId))dlsym(h, "ncclGetUniqueId");
    api.CommInitRank = (decltype(api.CommInitRank))dlsym(h, "ncclCommInitRank");
    api.CommDestroy = (decltype(api.CommDestroy))dlsym(h, "ncclCommDestroy");
    api.Send = (decltype(api.Send))dlsym(h, "ncclSend");
    api.Recv = (decltype(api.Recv))dlsym(h, "ncclRecv");
    api.AllGather = (decltype(api.AllGather))dlsym(h, "ncclAllGather");
    api.GetErrorString = (decltype(api.GetErrorString))dlsym(h, "ncclGetErrorString");
    api.loaded = api.GetUniqueId && api.CommInitRank && api.CommDestroy && api.Send && api.Recv &&
                 api.GetErrorString;
    if (!api.loaded) api.why = "libnccl.so.2 lacks the point-to-point API";
  });
  return api;
}

lasp_status_t nccl_fail(ncclResult_t r, const char* what, int rank, int peer) {
  char buf[256];
  std::snprintf(buf, sizeof buf, "%s failed on rank %d (peer %d): %s", what, rank, peer,
                nccl().GetErrorString ? nccl().GetErrorString(r) : "?");
  return fail(LASP_ERR_COMM, buf);
}

// ---- cuBLAS, loaded lazily (the projection GEMMs of the NEXT-3 layer entry points only) -------------
// The Q / K / V projections and their gradients are plain dense GEMMs (M = B*C tokens, K or N = d_model):
// tensor-core bound, nothing of LASP to fuse into them, so they run on the library GEMM (the task's rule for
// plain GEMMs); every LASP step around them stays in this library's kernels.
struct CublasApi {
  bool loaded = false;
  std::string why;
  cublasStatus_t (*Create)(cublasHandle_t*) = nullptr;
  cublasStatus_t (*SetStream)(cublasHandle_t, cudaStream_t) = nullptr;
  cublasStatus_t (*GemmEx)(cublasHandle_t, cublasOperation_t, cublasOperation_t, int, int, int, const void*,
                           const void*, cudaDataType, int, const void*, cudaDataType, int, const void*, void*,
                           cudaDataType, int, cublasComputeType_t, cublasGemmAlgo_t) = nullptr;
};

CublasApi& cublas() {
  static CublasApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    const char* cands[] = {std::getenv("LASP_CUBLAS_LIB"), "libcublas.so.12"};
    void* h = nullptr;
    for (const char* c : cands)
      if (c && (h = dlopen(c, RTLD_NOW | RTLD_GLOBAL))) break;
    if (!h) { api.why = "libcublas.so.12 not found (set LASP_CUBLAS_LIB)"; return; }
    api.Create = (decltype(api.Create))dlsym(h, "cublasCreate_v2");
    api.SetStream = (decltype(api.SetStream))dlsym(h, "cublasSetStream_v2");
    api.GemmEx = (decltype(api.GemmEx))dlsym(h, "cublasGemmEx");
    api.loaded = api.Create && api.SetStream && api.GemmEx;
    if (!api.loaded) api.why = "libcublas.so.12 lacks cublasGemmEx";
  });
  return api;
}

// one handle per (thread, device)
lasp_status_t cublas_handle(cudaStream_t st, cublasHandle_t* out) {
  CublasApi& cb = cublas();
  if (!cb.loaded) return fail(LASP_ERR_UNSUPPORTED, cb.why);
  thread_local std::unordered_map<int, cublasHandle_t> handles;
  int dev = 0;
  LASP_CUDA(cudaGetDevice(&dev));
  auto it = handles.find(dev);
  if (it == handles.end()) {
    cublasHandle_t h = nullptr;
    if (cb.Create(&h) != CUBLAS_STATUS_SUCCESS) return fail(LASP_ERR_CUDA, "cublasCreate failed");
    it = handles.emplace(dev, h).first;
  }
  if (cb.SetStream(it->second, st) != CUBLAS_STATUS_SUCCESS) return fail(LASP_ERR_CUDA, "cublasSetStream failed");
  *out = it->second;
  return LASP_OK;
}

// Row-major C[M][N] (=|+=) op(A) op(B), bf16 operands, fp32 accumulation; C bf16 or fp32. In cuBLAS's
// column-major terms this is C^T = op(B)^T op(A)^T.
//   ta == false: A is [M][K] row-major; true: A is [K][M] row-major (A^T used).
//   tb == false: B is [K][N] row-major; true: B is [N][K] row-major (B^T used).
lasp_status_t gemm_rm(cublasHandle_t h, int64_t M, int64_t N, int64_t K, const void* A, bool ta, const void* B, bool tb,
                      void* C, bool c_fp32, float beta) {
  const float alpha = 1.f;
  const cublasOperation_t opa = tb ? CUBLAS_OP_T : CUBLAS_OP_N;  // first cuBLAS operand = B^T (N x K col-major)
  const cublasOperation_t opb = ta ? CUBLAS_OP_T : CUBLAS_OP_N;
  const int lda = int(tb ? K : N), ldb = int(ta ? M : K);
  cublasStatus_t r = cublas().GemmEx(h, opa, opb, int(N), int(M), int(K), &alpha, B, CUDA_R_16BF, lda, A, CUDA_R_16BF,
                                     ldb, &beta, C, c_fp32 ? CUDA_R_32F : CUDA_R_16BF, int(N), CUBLAS_COMPUTE_32F,
                                     CUBLAS_GEMM_DEFAULT);
  if (r != CUBLAS_STATUS_SUCCESS) {
    char b[96];
    std::snprintf(b, sizeof b, "cublasGemmEx failed (status %d)", int(r));
    return fail(LASP_ERR_CUDA, b);
  }
  return LASP_OK;
}

// ---- loopback transport: the ring's ranks as threads of one process on one GPU (testing) ------
// A message is staged in a stream-ordered allocation: the sender copies into it and records an event,
// the receiver's stream waits on that event, copies out and frees it. Same ordering contract as
// ncclSend/ncclRecv on the given streams; the receiving host thread blocks until the send is posted.
struct LoopMsg {
  void* buf = nullptr;
  cudaEvent_t ev = nullptr;
  size_t bytes = 0;
};
struct LoopGroup {
  int world = 0;
  std::mutex mu;
  std::condition_variable cv;
  std::map<std::pair<int, int>, std::deque<LoopMsg>> q;  // (src, dst) -> messages in send order
  std::map<int, char*> p2p;                                // P2P exchange: rank -> its flag / buffer block
};
std::mutex g_loop_mu;
std::unordered_map<std::string, std::weak_ptr<LoopGroup>> g_loops;

std::shared_ptr<LoopGroup> loop_group(const std::string& name, int world) {
  std::lock_guard<std::mutex> g(g_loop_mu);
  auto it = g_loops.find(name);
  if (it != g_loops.end())
    if (auto sp = it->second.lock()) return sp->world == world ? sp : nullptr;
  auto sp = std::make_shared<LoopGroup>();
  sp->world = world;
  g_loops[name] = sp;
  return sp;
}

}  // namespace

struct lasp_ctx {
  ncclComm_t comm = nullptr;
  std::shared_ptr<LoopGroup> loop;  // non-null: loopback transport instead of NCCL
  int rank = 0, world = 1, device = 0;
  int exchange = LASP_EXCHANGE_RING;
  cudaStream_t comm_stream = nullptr;
  cudaEvent_t ev_ready = nullptr, ev_done = nullptr;
  float* gather = nullptr;  // all-gather exchange: [world + 1][B*H*D*D + 64] fp32 (ctx-owned, grown on demand)
  size_t gather_elems = 0;
  // P2P exchange: this rank's block [8 flag words | pad to 256 B | recv fwd (p2p_elems) | recv bwd], and the
  // blocks of ranks r - 1 and r + 1 (opened CUDA IPC handles, or the loopback group's pointers)
  char* p2p = nullptr;
  size_t p2p_elems = 0;
  char* p2p_prev = nullptr;
  char* p2p_next = nullptr;
  std::vector<char*> p2p_peers;  // every rank's block (this rank's own at [rank]); the all-gather needs them all
  bool p2p_ipc = false;  // the peer pointers are opened IPC handles (closed on destroy)
};

namespace {

lasp_status_t ring_send(lasp_ctx* c, const float* buf, size_t n, int peer, cudaStream_t st, const char* what) {
  if (!c->loop) {
    ncclResult_t r = nccl().Send(buf, n, ncclFloat32, peer, c->comm, st);
    return r == ncclSuccess ? LASP_OK : nccl_fail(r, what, c->rank, peer);
  }
  LoopMsg m;
  m.bytes = n * sizeof(float);
  LASP_CUDA(cudaMallocAsync(&m.buf, m.bytes, st));
  LASP_CUDA(cudaMemcpyAsync(m.buf, buf, m.bytes, cudaMemcpyDeviceToDevice, st));
  LASP_CUDA(cudaEventCreateWithFlags(&m.ev, cudaEventDisableTiming));
  LASP_CUDA(cudaEventRecord(m.ev, st));
  {
    std::lock_guard<std::mutex> g(c->loop->mu);
    c->loop->q[{c->rank, peer}].push_back(m);
  }
  c->loop->cv.notify_all();
  return LASP_OK;
}

lasp_status_t ring_recv(lasp_ctx* c, float* buf, size_t n, int peer, cudaStream_t st, const char* what) {
  if (!c->loop) {
    ncclResult_t r = nccl().Recv(buf, n, ncclFloat32, peer, c->comm, st);
    return r == ncclSuccess ? LASP_OK : nccl_fail(r, what, c->rank, peer);
  }
  LoopMsg m;
  {
    std::unique_lock<std::mutex> g(c->loop->mu);
    auto& dq = c->loop->q[{peer, c->rank}];
    if (!c->loop->cv.wait_for(g, std::chrono::seconds(120), [&] { return !dq.empty(); })) {
      char b[160];
      std::snprintf(b, sizeof b, "%s: loopback receive from rank %d timed out on rank %d", what, peer, c->rank);
      return fail(LASP_ERR_COMM, b);
    }
    m = dq.front();
    dq.pop_front();
  }
  if (m.bytes != n * sizeof(float)) return fail(LASP_ERR_COMM, "loopback message size mismatch");
  LASP_CUDA(cudaStreamWaitEvent(st, m.ev, 0));
  LASP_CUDA(cudaMemcpyAsync(buf, m.buf, m.bytes, cudaMemcpyDeviceToDevice, st));
  LASP_CUDA(cudaFreeAsync(m.buf, st));
  LASP_CUDA(cudaEventDestroy(m.ev));
  return LASP_OK;
}

// All-gather exchange (NEXT-2): every rank's local state into ctx->gather[world][n], then the state this
// rank would have received over the ring is folded from the gathered ones (fold_ranks_kernel).
lasp_status_t exchange_allgather(lasp_ctx* c, const Plan& p, const float* local, float* in, bool backward,
                                 cudaStream_t st) {
  // each rank contributes [state (n floats) | its n_local (int64) | pad] so that ranks of different lengths
  // fold correctly (fold_ranks_kernel decays rank j's contribution with its own lam^(C_j))
  const size_t n = state_elems(p);
  const size_t stride = n + 64;  // 256-byte trailer
  if (c->gather_elems < stride * size_t(c->world + 1)) {
    if (c->gather) LASP_CUDA(cudaFree(c->gather));
    c->gather = nullptr;
    c->gather_elems = 0;
    LASP_CUDA(cudaMalloc(&c->gather, stride * size_t(c->world + 1) * sizeof(float)));
    c->gather_elems = stride * size_t(c->world + 1);
  }
  float* mine = c->gather + size_t(c->world) * stride;  // send buffer: this rank's state + trailer
  LASP_CUDA(launch_pack_state(p, local, mine, st));  // state + this rank's n_local
  if (!c->loop) {
    if (!nccl().AllGather) return fail(LASP_ERR_COMM, "libnccl.so.2 lacks ncclAllGather");
    ncclResult_t r = nccl().AllGather(mine, c->gather, stride, ncclFloat32, c->comm, st);
    if (r != ncclSuccess) return nccl_fail(r, "ncclAllGather(state)", c->rank, -1);
  } else {
    lasp_status_t s;
    for (int j = 0; j < c->world; ++j)
      if (j != c->rank && (s = ring_send(c, mine, stride, j, st, "allgather send")) != LASP_OK) return s;
    for (int j = 0; j < c->world; ++j)
      if (j != c->rank && (s = ring_recv(c, c->gather + size_t(j) * stride, stride, j, st, "allgather recv")) != LASP_OK)
        return s;
    LASP_CUDA(cudaMemcpyAsync(c->gather + size_t(c->rank) * stride, mine, stride * sizeof(float),
                              cudaMemcpyDeviceToDevice, st));
  }
  const int j0 = backward ? c->world - 1 : 0, step = backward ? -1 : 1;
  const int count = backward ? c->world - 1 - c->rank : c->rank;
  return launch_fold_ranks(p, c->gather, int64_t(stride), j0, step, count, in, st) == cudaSuccess
             ? LASP_OK : cuda_fail(cudaGetLastError(), "fold_ranks");
}

// P2P exchange (LASP_EXCHANGE_P2P): the ring hop as one kernel that receives (flag wait on this rank's buffer),
// combines and stores the result into the downstream rank's buffer over peer memory (kernels_simt.cu).
size_t p2p_off_recv(const lasp_ctx* c, int dir) { return 256 + size_t(dir) * align256(c->p2p_elems * 4); }
// the all-gather part of a rank's block follows the ring part: 4 KB of flags, then [2 directions][world] slots
size_t p2p_off_gather(size_t elems) { return 256 + 2 * align256(elems * 4); }
size_t p2p_slot_bytes(size_t elems) { return align256((elems + 64) * 4); }
size_t p2p_block_bytes(size_t elems, int world) {
  return p2p_off_gather(elems) + kP2PFlagBytes + 2 * size_t(world) * p2p_slot_bytes(elems);
}
lasp_status_t p2p_gather(lasp_ctx* c, const Plan& p, const float* local, float* in, bool backward, cudaStream_t st) {
  const size_t n = state_elems(p);
  if (!c->p2p || int(c->p2p_peers.size()) != c->world)
    return fail(LASP_ERR_COMM, "P2P all-gather: lasp_ctx_p2p_setup / lasp_ctx_p2p_connect not done");
  if (n > c->p2p_elems) return fail(LASP_ERR_SHAPE, "P2P exchange: state larger than the setup's max_state_elems");
  P2PGather g{};
  g.local = local;
  g.in_priv = in;
  for (int k = 0; k < c->world; ++k) g.bases[k] = c->p2p_peers[k] + p2p_off_gather(c->p2p_elems);
  g.slot_bytes = p2p_slot_bytes(c->p2p_elems);
  g.rank = c->rank;
  g.world = c->world;
  g.dir = backward ? 1 : 0;
  g.n = int64_t(n);
  LASP_CUDA(staged(backward ? "p2p_gather_bwd" : "p2p_gather_fwd", st, [&] { return launch_p2p_gather(p, g, st); }));
  return LASP_OK;
}
lasp_status_t p2p_hop(lasp_ctx* c, const Plan& p, const float* local, float* in, bool backward, cudaStream_t st) {
  const size_t n = state_elems(p);
  if (!c->p2p || (c->world > 1 && !c->p2p_prev && !c->p2p_next))
    return fail(LASP_ERR_COMM, "P2P exchange: lasp_ctx_p2p_setup / lasp_ctx_p2p_connect not done");
  if (n > c->p2p_elems) return fail(LASP_ERR_SHAPE, "P2P exchange: state larger than the setup's max_state_elems");
  const int dir = backward ? 1 : 0;
  char* up = backward ? c->p2p_next : c->p2p_prev;     // the rank this one receives from
  char* down = backward ? c->p2p_prev : c->p2p_next;   // the rank this one sends to
  P2PHop h{};
  h.local = local;
  h.in_priv = in;
  h.my_recv = reinterpret_cast<const float*>(c->p2p + p2p_off_recv(c, dir));
  h.my_flags = reinterpret_cast<uint64_t*>(c->p2p);
  h.peer_recv = down ? reinterpret_cast<float*>(down + p2p_off_recv(c, dir)) : nullptr;
  h.peer_flags = down ? reinterpret_cast<uint64_t*>(down) : nullptr;
  h.up_flags = up ? reinterpret_cast<uint64_t*>(up) : nullptr;
  h.has_up = up != nullptr;
  h.dir = dir;
  h.n = int64_t(n);
  LASP_CUDA(staged(backward ? "p2p_hop_bwd" : "p2p_hop_fwd", st, [&] { return launch_p2p_hop(p, h, st); }));
  return LASP_OK;
}

// Alg. 2 for one rank after validation. c == nullptr: the communication-free local path (kv_in given, kv_out
// optional); otherwise the ring / all-gather of ctx c (KV_in received). norm: the Norm epilogue (NEXT-3).
lasp_status_t fwd_body(lasp_ctx* c, const Plan& p, const void* q, const void* k, const void* v, const float* kv_in,
                       void* o, float* kv_out, void* cache, void* workspace, cudaStream_t st, const NormArgs* norm) {
  Workspace w = carve(p, workspace);
  lasp_status_t s;
  unsigned* gbar = p.C > 0 && fused_fold(p) ? w.gbar : nullptr;
  if (entry_in_seg_state(p)) {  // F1, with the call's entry duty (cache tag, control block)
    const EntryDuty e = make_entry(p, cache, w, c ? c->rank : -1, c ? c->world : -1, false, false);
    LASP_CUDA(seg_state(p, Dir::FWD, k, v, w.seg, st, w.claim(0), nullptr, &e));
  } else {
    LASP_CUDA(entry_tag(p, cache, w, c ? c->rank : -1, c ? c->world : -1, false, false, st));   // cache tag
    if (p.C > 0) LASP_CUDA(seg_state(p, Dir::FWD, k, v, w.seg, st, w.claim(0)));                // F1
  }
  if (c == nullptr)
    return fwd_tail(p, q, k, v, kv_in, o, kv_out, cache, w.seg, gbar, w.claim(1), st, norm);  // F2 + F3
  const size_t n = state_elems(p);
  int from = -1, to = -1;
  lasp_ring_peers(c->rank, c->world, 0, &from, &to);
  LASP_CUDA(prefix(p, Dir::FWD, nullptr, p.C > 0 ? w.seg : nullptr, nullptr, w.local, st));
  ProfSpan hop("exchange_fwd", st);
  if (c->exchange == LASP_EXCHANGE_P2P) {
    if ((s = p2p_hop(c, p, w.local, w.in, false, st)) != LASP_OK) return s;
  } else if (c->exchange == LASP_EXCHANGE_P2P_ALLGATHER) {
    if ((s = p2p_gather(c, p, w.local, w.in, false, st)) != LASP_OK) return s;
  } else if (c->exchange == LASP_EXCHANGE_ALLGATHER && c->world > 1) {
    if ((s = exchange_allgather(c, p, w.local, w.in, false, st)) != LASP_OK) return s;
  } else {
    // F2 ring hop: Recv KV_in from r-1 (Alg. 2), combine, Send to r+1
    if (from >= 0) {
      if ((s = ring_recv(c, w.in, n, from, st, "ncclRecv(KV)")) != LASP_OK) return s;
    } else {
      LASP_CUDA(cudaMemsetAsync(w.in, 0, n * sizeof(float), st));
    }
    if (to >= 0) {
      LASP_CUDA(combine(p, w.in, w.local, w.out, st));
      if ((s = ring_send(c, w.out, n, to, st, "ncclSend(KV)")) != LASP_OK) return s;
    }
  }
  hop.stop(st);
  return fwd_tail(p, q, k, v, w.in, o, nullptr, cache, w.seg, gbar, w.claim(1), st, norm);     // F2 + F3
}

// Alg. 3 for one rank after validation (c == nullptr: local path). nb: the Norm backward fused into B1 --
// d_o is then dY, and dO = Norm'(dY) is written to nb->dout, which the B3 passes read.
lasp_status_t bwd_body(lasp_ctx* c, const Plan& p, const void* q, const void* k, const void* v, const void* d_o,
                       const void* cache, const float* dkv_in, void* dq, void* dk, void* dv, float* dkv_out,
                       void* workspace, cudaStream_t st, const NormBwdArgs* nb) {
  Workspace w = carve(p, workspace);
  lasp_status_t s;
  const float* P = static_cast<const float*>(cache);
  const bool fuse = p.C > 0 && fused_fold(p);
  const void* g = nb ? nb->dout : d_o;  // the dO the B3 passes read
  // B1 carries the call's entry duty (tag check, control block) on the tensor-core path, else tag_kernel
  const bool entry_b1 = entry_in_seg_state(p);
  const EntryDuty e = make_entry(p, cache, w, c ? c->rank : -1, c ? c->world : -1, true, c != nullptr);
  if (!entry_b1) LASP_CUDA(entry_tag(p, cache, w, c ? c->rank : -1, c ? c->world : -1, true, c != nullptr, st));
  if (c == nullptr) {
    if (p.C == 0) {
      LASP_CUDA(prefix(p, Dir::REV, dkv_in, nullptr, nullptr, dkv_out, st));
      return LASP_OK;
    }
    LASP_CUDA(seg_state(p, Dir::REV, q, d_o, w.seg, st, w.claim(0), nb, entry_b1 ? &e : nullptr));  // B1
    const PrefixFold fold{dkv_in, w.seg, w.seg, dkv_out, w.gbar, int(Dir::REV)};
    if (!fuse) LASP_CUDA(prefix(p, Dir::REV, dkv_in, w.seg, w.seg, dkv_out, st));          // B2 (in place)
    // B3: dQ (needs only the cache), dV and dK in one launch (with B2 folded in when fused)
    const SeqArgs passes[3] = {{g, v, k, dq, P, 1, w.status(), 0}, {k, q, g, dv, w.seg, 0, w.status(), 1},
                               {v, g, q, dk, w.seg, 1, w.status(), 1}};
    const Dir dirs[3] = {Dir::FWD, Dir::REV, Dir::REV};
    // with the fused fold B1 immediately precedes this launch: dO (written by B1) must be waited for
    LASP_CUDA(core_multi(p, 3, passes, dirs, st, w.claim(1), fuse ? &fold : nullptr, nullptr, nb && fuse));
    return LASP_OK;
  }
  const size_t n = state_elems(p);
  if (p.C > 0) LASP_CUDA(seg_state(p, Dir::REV, q, d_o, w.seg, st, w.claim(0), nb, entry_b1 ? &e : nullptr));  // B1
  LASP_CUDA(prefix(p, Dir::REV, nullptr, p.C > 0 ? w.seg : nullptr, nullptr, w.local, st));
  // B2 ring hop on the comm stream: Recv dKV_in from r+1 (Alg. 3), combine, Send to r-1
  LASP_CUDA(cudaEventRecord(c->ev_ready, st));
  LASP_CUDA(cudaStreamWaitEvent(c->comm_stream, c->ev_ready, 0));
  ProfSpan hop("exchange_bwd", c->comm_stream);
  int from = -1, to = -1;
  lasp_ring_peers(c->rank, c->world, 1, &from, &to);
  const bool hop_pending = c->world > 1;  // a receive, send or all-gather runs on the comm stream under dQ
  if (c->exchange == LASP_EXCHANGE_P2P) {
    if ((s = p2p_hop(c, p, w.local, w.in, true, c->comm_stream)) != LASP_OK) return s;
  } else if (c->exchange == LASP_EXCHANGE_P2P_ALLGATHER) {
    if ((s = p2p_gather(c, p, w.local, w.in, true, c->comm_stream)) != LASP_OK) return s;
  } else if (c->exchange == LASP_EXCHANGE_ALLGATHER && c->world > 1) {
    if ((s = exchange_allgather(c, p, w.local, w.in, true, c->comm_stream)) != LASP_OK) return s;
  } else if (from >= 0) {
    if ((s = ring_recv(c, w.in, n, from, c->comm_stream, "ncclRecv(dKV)")) != LASP_OK) return s;
  } else {
    LASP_CUDA(cudaMemsetAsync(w.in, 0, n * sizeof(float), c->comm_stream));
  }
  if (to >= 0 && c->exchange == LASP_EXCHANGE_RING) {
    LASP_CUDA(combine(p, w.in, w.local, w.out, c->comm_stream));
    if ((s = ring_send(c, w.out, n, to, c->comm_stream, "ncclSend(dKV)")) != LASP_OK) return s;
  }
  hop.stop(c->comm_stream);
  LASP_CUDA(cudaEventRecord(c->ev_done, c->comm_stream));
  // dQ needs only the cache: it runs while the dKV hop is in flight, on all SMs but comm_sms()
  if (p.C > 0)
    LASP_CUDA(core(p, Dir::FWD, g, v, k, dq, P, 1, st, w.claim(1), w.status(), hop_pending ? comm_sms() : 0));
  LASP_CUDA(cudaStreamWaitEvent(st, c->ev_done, 0));
  if (p.C == 0) return LASP_OK;
  if (!fuse) LASP_CUDA(prefix(p, Dir::REV, w.in, w.seg, w.seg, nullptr, st));   // B2
  {  // dV and dK in one launch (with B2 folded in when fused)
    const SeqArgs passes[2] = {{k, q, g, dv, w.seg, 0, w.status(), 1}, {v, g, q, dk, w.seg, 1, w.status(), 1}};
    const Dir dirs[2] = {Dir::REV, Dir::REV};
    const PrefixFold fold{w.in, w.seg, w.seg, nullptr, w.gbar, int(Dir::REV)};
    LASP_CUDA(core_multi(p, 2, passes, dirs, st, w.claim(2), fuse ? &fold : nullptr));
  }
  return LASP_OK;
}

}  // namespace

// ---- NEXT-4: generalised decay (kernels_gla.cu) --------------------------------------------------------
namespace {

constexpr uint64_t kGlaTagMagic = 0x4c415350474c4121ull;  // "LASPGLA!": a GLA cache, never a scalar-path one

lasp_status_t gla_plan(const lasp_shape_t* s, GlaPlan& g) {
  if (!s) return fail(LASP_ERR_SHAPE, "shape is NULL");
  if (s->batch < 1 || s->n_local < 0 || s->heads < 1 || s->kv_heads < 0)
    return fail(LASP_ERR_SHAPE, "need batch >= 1, n_local >= 0, heads >= 1, kv_heads >= 0");
  if (s->dtype != LASP_FP32) return fail(LASP_ERR_UNSUPPORTED, "generalised decay: fp32 tensors only");
  if (s->head_dim != 32 && s->head_dim != 64 && s->head_dim != 128)
    return fail(LASP_ERR_UNSUPPORTED, "head_dim must be 32, 64 or 128");
  if (s->kv_heads != 0 && s->kv_heads != s->heads)
    return fail(LASP_ERR_UNSUPPORTED, "generalised decay: kv_heads must equal heads");
  g.B = s->batch; g.C = s->n_local; g.H = s->heads; g.D = s->head_dim;
  // segments a multiple of the 8-token tile
  const int64_t forced = env_i64("LASP_GLA_SEG_LEN", 0);
  int64_t L;
  if (forced > 0) {
    L = (forced + 7) / 8 * 8;
  } else {
    // whole waves: the items (one CTA per (batch, head, segment), each a long sequential recurrence) are sized
    // to a multiple of the co-resident CTA slots, so no wave runs partly empty (1184 items on 1036 slots ran
    // as 2 waves)
    int dev = 0, sms = 148;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t slots = int64_t(sms) * gla_slots_per_sm(int(g.D));
    const int64_t waves = env_i64("LASP_GLA_WAVES", 1);  // 1 wave measured best (profiles/r2t_gla_waves.txt)
    int64_t nseg = (waves * slots) / (g.B * g.H);
    if (nseg < 1) nseg = 1;
    L = g.C > 0 ? ((g.C + nseg - 1) / nseg + 7) / 8 * 8 : 8;
    if (L < 32) L = 32;
  }
  g.seg_len = L;
  g.nseg = g.C > 0 ? (g.C + L - 1) / L : 1;
  if (g.B * g.H * g.nseg >= (int64_t(1) << 31)) return fail(LASP_ERR_UNSUPPORTED, "too many segments");
  return LASP_OK;
}

size_t gla_state_elems(const GlaPlan& g) { return size_t(g.B * g.H * g.D * g.D); }
size_t gla_cache_bytes(const GlaPlan& g) {
  return align256(size_t(g.B * g.H * (g.nseg + 1) * g.D * g.D) * 4) + kCacheTagBytes;
}
struct GlaWs {
  unsigned* ctrl;  // 16 words (entry kernel zeroes; [2] = cache-tag status)
  float* seg;      // [B][H][nseg][D][D]
  float* ls;       // [B][H][nseg][D]
  float* local;    // [B][H][D][D]
  float* in;
  float* out;
  float* lsum;     // [B][H][D]
};
GlaWs gla_carve(const GlaPlan& g, void* ws) {
  char* c = static_cast<char*>(ws);
  GlaWs w;
  w.ctrl = reinterpret_cast<unsigned*>(c); c += 256;
  w.seg = reinterpret_cast<float*>(c); c += align256(size_t(g.B * g.H * g.nseg * g.D * g.D) * 4);
  w.ls = reinterpret_cast<float*>(c); c += align256(size_t(g.B * g.H * g.nseg * g.D) * 4);
  w.local = reinterpret_cast<float*>(c); c += align256(gla_state_elems(g) * 4);
  w.in = reinterpret_cast<float*>(c); c += align256(gla_state_elems(g) * 4);
  w.out = reinterpret_cast<float*>(c); c += align256(gla_state_elems(g) * 4);
  w.lsum = reinterpret_cast<float*>(c);
  return w;
}
size_t gla_ws_bytes(const GlaPlan& g) {
  return 256 + align256(size_t(g.B * g.H * g.nseg * g.D * g.D) * 4) + align256(size_t(g.B * g.H * g.nseg * g.D) * 4) +
         3 * align256(gla_state_elems(g) * 4) + align256(size_t(g.B * g.H * g.D) * 4);
}

cudaError_t gla_entry(const GlaPlan& g, const void* cache, const GlaWs& w, int rank, int world, bool check,
                      cudaStream_t st) {
  CacheTag t{};
  t.w[kTagMagic] = kGlaTagMagic;
  t.w[kTagB] = uint64_t(g.B); t.w[kTagC] = uint64_t(g.C); t.w[kTagH] = uint64_t(g.H); t.w[kTagD] = uint64_t(g.D);
  t.w[kTagSeg] = uint64_t(g.seg_len);
  t.w[kTagDtype] = 1;
  t.w[kTagRank] = uint64_t(int64_t(rank));
  t.w[kTagWorld] = uint64_t(int64_t(world));
  t.w[kTagHk] = uint64_t(g.H);
  t.w[kTagGen] = ++g_generation;
  unsigned mask = 0;
  if (check) {
    for (int i = kTagMagic; i <= kTagDtype; ++i) mask |= 1u << i;
    if (rank >= 0) mask |= (1u << kTagRank) | (1u << kTagWorld);
  }
  uint64_t* hdr = reinterpret_cast<uint64_t*>(static_cast<char*>(const_cast<void*>(cache)) +
                                              align256(size_t(g.B * g.H * (g.nseg + 1) * g.D * g.D) * 4));
  return staged(check ? "gla_tag_check" : "gla_tag_write", st,
                [&] { return launch_tag(t, hdr, mask, w.ctrl, st); });
}

lasp_status_t gla_check(const GlaPlan& g, std::initializer_list<const void*> seq, const void* cache, const void* ws) {
  if (g.C > 0)
    for (const void* x : seq)
      if (!x || !aligned16(x)) return fail(LASP_ERR_SHAPE, "sequence tensor NULL or not 16-byte aligned");
  if (!cache || !aligned16(cache)) return fail(LASP_ERR_SHAPE, "cache NULL or not 16-byte aligned");
  if (!ws || !aligned16(ws)) return fail(LASP_ERR_SHAPE, "workspace NULL or not 16-byte aligned");
  return check_device();
}

// Alg. 2 / Alg. 3 with the generalised decay, one rank (c == nullptr: the local path with kv_in / kv_out).
// Ring: receive the neighbour's state, fold this rank's segments with it (the fold's final value is the
// message for the next rank: KV_out = Diag(prod_t g_t) KV_in + L_rank; dKV_out = G'_rank + Diag(...) dKV_in),
// send, then the per-token passes.
lasp_status_t gla_hop_in(lasp_ctx* c, const GlaPlan& g, float* in, bool backward, cudaStream_t st) {
  if (c->exchange == LASP_EXCHANGE_P2P || c->exchange == LASP_EXCHANGE_P2P_ALLGATHER || (!c->comm && !c->loop))
    return fail(LASP_ERR_UNSUPPORTED, "generalised decay: the ring exchange only (the P2P hop applies a scalar decay)");
  int from = -1, to = -1;
  lasp_ring_peers(c->rank, c->world, backward ? 1 : 0, &from, &to);
  const size_t n = gla_state_elems(g);
  if (from >= 0) return ring_recv(c, in, n, from, st, backward ? "ncclRecv(dKV, gla)" : "ncclRecv(KV, gla)");
  LASP_CUDA(cudaMemsetAsync(in, 0, n * sizeof(float), st));
  return LASP_OK;
}
lasp_status_t gla_hop_out(lasp_ctx* c, const GlaPlan& g, const float* out, bool backward, cudaStream_t st) {
  int from = -1, to = -1;
  lasp_ring_peers(c->rank, c->world, backward ? 1 : 0, &from, &to);
  if (to < 0) return LASP_OK;
  return ring_send(c, out, gla_state_elems(g), to, st, backward ? "ncclSend(dKV, gla)" : "ncclSend(KV, gla)");
}

lasp_status_t gla_fwd_body(lasp_ctx* c, const GlaPlan& g, const float* q, const float* k, const float* v,
                           const float* lg, const float* kv_in, float* o, float* kv_out, void* cache, void* ws,
                           cudaStream_t st) {
  GlaWs w = gla_carve(g, ws);
  float* P = static_cast<float*>(cache);
  lasp_status_t s;
  LASP_CUDA(gla_entry(g, cache, w, c ? c->rank : -1, c ? c->world : -1, false, st));
  if (g.C > 0) LASP_CUDA(staged("gla_state_fwd", st, [&] { return gla_launch_state(g, 0, k, v, lg, w.seg, w.ls, st); }));
  const float* init = kv_in;
  float* fin = kv_out;
  ProfSpan hop("exchange_fwd", st);
  if (c != nullptr) {
    if ((s = gla_hop_in(c, g, w.in, false, st)) != LASP_OK) return s;
    init = w.in;
    fin = w.out;
  }
  LASP_CUDA(staged("gla_fold_fwd", st, [&] { return gla_launch_fold(g, 0, init, w.seg, w.ls, P, fin, nullptr, st); }));
  if (c != nullptr && (s = gla_hop_out(c, g, w.out, false, st)) != LASP_OK) return s;
  hop.stop(st);
  if (g.C > 0) LASP_CUDA(staged("gla_out", st, [&] { return gla_launch_out(g, q, k, v, lg, P, o, st); }));
  return LASP_OK;
}

lasp_status_t gla_bwd_body(lasp_ctx* c, const GlaPlan& g, const float* q, const float* k, const float* v,
                           const float* lg, const float* d_o, const void* cache, const float* dkv_in, float* dq,
                           float* dk, float* dv, float* dlg, float* dkv_out, void* ws, cudaStream_t st) {
  GlaWs w = gla_carve(g, ws);
  const float* P = static_cast<const float*>(cache);
  lasp_status_t s;
  LASP_CUDA(gla_entry(g, cache, w, c ? c->rank : -1, c ? c->world : -1, true, st));
  if (g.C > 0) LASP_CUDA(staged("gla_state_rev", st, [&] { return gla_launch_state(g, 1, q, d_o, lg, w.seg, w.ls, st); }));
  const float* init = dkv_in;
  float* fin = dkv_out;
  ProfSpan hop("exchange_bwd", st);
  if (c != nullptr) {
    if ((s = gla_hop_in(c, g, w.in, true, st)) != LASP_OK) return s;
    init = w.in;
    fin = w.out;
  }
  LASP_CUDA(staged("gla_fold_rev", st, [&] { return gla_launch_fold(g, 1, init, w.seg, w.ls, nullptr, fin, nullptr, st); }));
  if (c != nullptr && (s = gla_hop_out(c, g, w.out, true, st)) != LASP_OK) return s;
  hop.stop(st);
  if (g.C > 0)
    LASP_CUDA(staged("gla_bwd", st, [&] {
      return gla_launch_bwd(g, q, k, v, lg, d_o, P, w.seg, dq, dk, dv, dlg, w.ctrl + 2, st);
    }));
  return LASP_OK;
}

}  // namespace

extern "C" {

const char* lasp_last_error(void) { return g_err.c_str(); }

uint64_t lasp_launch_count(void) { return g_launches.load(); }

void lasp_debug_trace(unsigned long long* device_buf) { tc_set_trace(device_buf); }

void lasp_profile_enable(int on) { g_profile.store(on ? 1 : 0); }

int lasp_profile_read(char* buf, size_t cap) {
  std::lock_guard<std::mutex> g(g_prof_mu);
  struct Acc { int64_t n = 0; double ms = 0; };
  std::vector<std::pair<std::string, Acc>> acc;
  int rc = 0;
  for (ProfRec& r : g_prof_recs) {
    float ms = 0.f;
    if (cudaEventSynchronize(r.b) != cudaSuccess || cudaEventElapsedTime(&ms, r.a, r.b) != cudaSuccess) rc = -1;
    auto it = acc.begin();
    for (; it != acc.end(); ++it) if (it->first == r.name) break;
    if (it == acc.end()) { acc.emplace_back(r.name, Acc{}); it = acc.end() - 1; }
    it->second.n += 1;
    it->second.ms += ms;
    g_prof_pool.push_back(r.a);
    g_prof_pool.push_back(r.b);
  }
  g_prof_recs.clear();
  std::string js = "{";
  for (size_t i = 0; i < acc.size(); ++i) {
    char item[160];
    std::snprintf(item, sizeof item, "%s\"%s\": [%lld, %.6f]", i ? ", " : "", acc[i].first.c_str(),
                  (long long)acc[i].second.n, acc[i].second.ms);
    js += item;
  }
  js += "}";
  if (buf && cap) { std::strncpy(buf, js.c_str(), cap - 1); buf[cap - 1] = 0; }
  return rc != 0 ? rc : (int)js.size();
}

const char* lasp_version(void) { return "lasp-b200 0.1 (sm_100a; tcgen05 + CUDA-core paths)"; }

size_t lasp_cache_bytes(const lasp_shape_t* shape) {
  if (validate_shape(shape) != LASP_OK) return 0;
  return cache_bytes(make_plan(shape));
}

lasp_status_t lasp_debug_occupy(int ctas, int smem_bytes, double microseconds, void* stream) {
  if (ctas < 1 || smem_bytes < 0 || !(microseconds >= 0)) return fail(LASP_ERR_SHAPE, "bad occupy arguments");
  LASP_CUDA(launch_occupy(ctas, smem_bytes, microseconds, static_cast<cudaStream_t>(stream)));
  return LASP_OK;
}

lasp_status_t lasp_workspace_status(const void* workspace, void* stream) {
  if (!workspace || !aligned16(workspace)) return fail(LASP_ERR_SHAPE, "workspace NULL or not 16-byte aligned");
  unsigned bits = 0;
  LASP_CUDA(cudaStreamSynchronize(static_cast<cudaStream_t>(stream)));
  LASP_CUDA(cudaMemcpy(&bits, static_cast<const unsigned*>(workspace) + 2, sizeof bits, cudaMemcpyDeviceToHost));
  if (bits == 0) return LASP_OK;
  static const char* names[kTagWords] = {"magic (not a cache written by lasp_fwd*)", "batch", "n_local", "heads",
                                         "head_dim", "segment length", "dtype", "lambda", "rank", "world",
                                         "kv_heads"};
  std::string msg = "cache tag mismatch (backward without a matching forward, S:411):";
  for (int i = 0; i < kTagWords; ++i)
    if ((bits >> i) & 1u) msg += std::string(" ") + (names[i] ? names[i] : "?");
  return fail(LASP_ERR_STATE, msg);
}

size_t lasp_workspace_bytes(const lasp_shape_t* shape) {
  if (validate_shape(shape) != LASP_OK) return 0;
  return workspace_bytes(make_plan(shape));
}

int64_t lasp_segment_len(const lasp_shape_t* shape) {
  if (validate_shape(shape) != LASP_OK) return 0;
  return make_plan(shape).seg_len;
}

lasp_status_t lasp_fwd_local(const lasp_shape_t* shape, const void* q, const void* k, const void* v,
                             const float* lambda, const float* kv_in, void* o, float* kv_out, void* cache,
                             void* workspace, void* stream) {
  Plan p;
  lasp_status_t s = prologue(shape, lambda, p);
  if (s != LASP_OK) return s;
  if ((s = check_ptrs(p, {q, k, v, o}, cache, workspace)) != LASP_OK) return s;
  if ((s = check_device()) != LASP_OK) return s;
  return fwd_body(nullptr, p, q, k, v, kv_in, o, kv_out, cache, workspace, static_cast<cudaStream_t>(stream), nullptr);
}

lasp_status_t lasp_bwd_local(const lasp_shape_t* shape, const void* q, const void* k, const void* v,
                             const float* lambda, const void* d_o, const void* cache, const float* dkv_in,
                             void* dq, void* dk, void* dv, float* dkv_out, void* workspace, void* stream) {
  Plan p;
  lasp_status_t s = prologue(shape, lambda, p);
  if (s != LASP_OK) return s;
  if ((s = check_ptrs(p, {q, k, v, d_o, dq, dk, dv}, cache, workspace)) != LASP_OK) return s;
  if ((s = check_device()) != LASP_OK) return s;
  return bwd_body(nullptr, p, q, k, v, d_o, cache, dkv_in, dq, dk, dv, dkv_out, workspace,
                  static_cast<cudaStream_t>(stream), nullptr);
}

lasp_status_t lasp_unique_id(uint8_t id[128]) {
  if (!id) return fail(LASP_ERR_SHAPE, "id is NULL");
  NcclApi& n = nccl();
  if (!n.loaded) return fail(LASP_ERR_COMM, n.why);
  ncclUniqueId uid;
  ncclResult_t r = n.GetUniqueId(&uid);
  if (r != ncclSuccess) return nccl_fail(r, "ncclGetUniqueId", -1, -1);
  static_assert(sizeof(uid.internal) == 128, "ncclUniqueId is 128 bytes");
  std::memcpy(id, uid.internal, 128);
  return LASP_OK;
}

lasp_status_t lasp_ctx_create(int rank, int world, const uint8_t id[128], int device, lasp_ctx_t* out) {
  if (!out || !id) return fail(LASP_ERR_SHAPE, "NULL argument");
  if (world < 1 || rank < 0 || rank >= world) return fail(LASP_ERR_PARTITION, "rank outside [0, world)");
  NcclApi& n = nccl();
  if (!n.loaded) return fail(LASP_ERR_COMM, n.why);
  LASP_CUDA(cudaSetDevice(device));
  lasp_ctx* c = new lasp_ctx;
  c->rank = rank; c->world = world; c->device = device;
  ncclUniqueId uid;
  std::memcpy(uid.internal, id, 128);
  ncclResult_t r = n.CommInitRank(&c->comm, world, uid, rank);
  if (r != ncclSuccess) { delete c; return nccl_fail(r, "ncclCommInitRank", rank, -1); }
  cudaError_t e = cudaStreamCreateWithFlags(&c->comm_stream, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->ev_ready, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->ev_done, cudaEventDisableTiming);
  if (e != cudaSuccess) { n.CommDestroy(c->comm); delete c; return cuda_fail(e, "ctx stream/event"); }
  *out = c;
  return LASP_OK;
}

lasp_status_t lasp_ctx_create_loopback(int rank, int world, const char* group, int device, lasp_ctx_t* out) {
  if (!out || !group) return fail(LASP_ERR_SHAPE, "NULL argument");
  if (world < 1 || rank < 0 || rank >= world) return fail(LASP_ERR_PARTITION, "rank outside [0, world)");
  LASP_CUDA(cudaSetDevice(device));
  auto grp = loop_group(group, world);
  if (!grp) return fail(LASP_ERR_PARTITION, "loopback group exists with a different world size");
  lasp_ctx* c = new lasp_ctx;
  c->rank = rank; c->world = world; c->device = device;
  c->loop = grp;
  cudaError_t e = cudaStreamCreateWithFlags(&c->comm_stream, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->ev_ready, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->ev_done, cudaEventDisableTiming);
  if (e != cudaSuccess) { delete c; return cuda_fail(e, "ctx stream/event"); }
  *out = c;
  return LASP_OK;
}

lasp_status_t lasp_ctx_set_exchange(lasp_ctx_t c, int exchange) {
  if (!c) return fail(LASP_ERR_SHAPE, "ctx is NULL");
  if (exchange != LASP_EXCHANGE_RING && exchange != LASP_EXCHANGE_ALLGATHER && exchange != LASP_EXCHANGE_P2P &&
      exchange != LASP_EXCHANGE_P2P_ALLGATHER)
    return fail(LASP_ERR_DOMAIN, "exchange must be LASP_EXCHANGE_RING, _ALLGATHER, _P2P or _P2P_ALLGATHER");
  const bool p2p_mode = exchange == LASP_EXCHANGE_P2P || exchange == LASP_EXCHANGE_P2P_ALLGATHER;
  if (!p2p_mode && !c->comm && !c->loop)
    return fail(LASP_ERR_COMM, "a P2P-only ctx (lasp_ctx_create_p2p) supports only the P2P exchanges");
  c->exchange = exchange;
  return LASP_OK;
}

lasp_status_t lasp_ctx_create_p2p(int rank, int world, int device, lasp_ctx_t* out) {
  if (!out) return fail(LASP_ERR_SHAPE, "NULL argument");
  if (world < 1 || rank < 0 || rank >= world) return fail(LASP_ERR_PARTITION, "rank outside [0, world)");
  LASP_CUDA(cudaSetDevice(device));
  lasp_ctx* c = new lasp_ctx;
  c->rank = rank; c->world = world; c->device = device;
  c->exchange = LASP_EXCHANGE_P2P;
  cudaError_t e = cudaStreamCreateWithFlags(&c->comm_stream, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->ev_ready, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->ev_done, cudaEventDisableTiming);
  if (e != cudaSuccess) { delete c; return cuda_fail(e, "ctx stream/event"); }
  *out = c;
  return LASP_OK;
}

lasp_status_t lasp_ctx_p2p_setup(lasp_ctx_t c, size_t max_state_elems, uint8_t handle[64]) {
  if (!c || !handle || max_state_elems == 0) return fail(LASP_ERR_SHAPE, "NULL ctx / handle or zero size");
  if (c->p2p) return fail(LASP_ERR_STATE, "P2P exchange already set up on this ctx");
  LASP_CUDA(cudaSetDevice(c->device));
  if (c->world > kP2PMaxWorld) return fail(LASP_ERR_UNSUPPORTED, "P2P exchange: world > 64");
  c->p2p_elems = max_state_elems;
  const size_t bytes = p2p_block_bytes(max_state_elems, c->world);
  LASP_CUDA(cudaMalloc(&c->p2p, bytes));
  // epochs, acks and counters start at 0 on every rank (ring flags and the all-gather's flag page)
  LASP_CUDA(cudaMemset(c->p2p, 0, 256));
  LASP_CUDA(cudaMemset(c->p2p + p2p_off_gather(max_state_elems), 0, kP2PFlagBytes));
  cudaIpcMemHandle_t h;
  static_assert(sizeof(h) == 64, "cudaIpcMemHandle_t is 64 bytes");
  LASP_CUDA(cudaIpcGetMemHandle(&h, c->p2p));
  std::memcpy(handle, &h, 64);
  if (c->loop) {
    {
      std::lock_guard<std::mutex> g(c->loop->mu);
      c->loop->p2p[c->rank] = c->p2p;
    }
    c->loop->cv.notify_all();
  }
  return LASP_OK;
}

lasp_status_t lasp_ctx_p2p_connect(lasp_ctx_t c, const uint8_t* handles) {
  if (!c || !c->p2p) return fail(LASP_ERR_STATE, "lasp_ctx_p2p_setup first");
  LASP_CUDA(cudaSetDevice(c->device));
  auto open = [&](int peer, char** dst) -> lasp_status_t {
    if (peer < 0 || peer >= c->world) return LASP_OK;
    if (handles == nullptr) {  // loopback group: the ranks are threads of this process
      if (!c->loop) return fail(LASP_ERR_SHAPE, "handles NULL outside a loopback group");
      std::unique_lock<std::mutex> g(c->loop->mu);
      if (!c->loop->cv.wait_for(g, std::chrono::seconds(120), [&] { return c->loop->p2p.count(peer) != 0; }))
        return fail(LASP_ERR_COMM, "P2P connect: loopback peer never set up");
      *dst = c->loop->p2p[peer];
      return LASP_OK;
    }
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handles + size_t(peer) * 64, 64);
    void* ptr = nullptr;
    cudaError_t e = cudaIpcOpenMemHandle(&ptr, h, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) {
      char b[160];
      std::snprintf(b, sizeof b, "cudaIpcOpenMemHandle(rank %d) on rank %d: %s", peer, c->rank, cudaGetErrorString(e));
      return fail(LASP_ERR_COMM, b);
    }
    *dst = static_cast<char*>(ptr);
    c->p2p_ipc = true;
    return LASP_OK;
  };
  if (c->loop) c->loop->cv.notify_all();
  lasp_status_t s;
  c->p2p_peers.assign(size_t(c->world), nullptr);
  for (int k = 0; k < c->world; ++k) {
    if (k == c->rank) {
      c->p2p_peers[size_t(k)] = c->p2p;
    } else if ((s = open(k, &c->p2p_peers[size_t(k)])) != LASP_OK) {
      return s;
    }
  }
  c->p2p_prev = c->rank > 0 ? c->p2p_peers[size_t(c->rank - 1)] : nullptr;
  c->p2p_next = c->rank + 1 < c->world ? c->p2p_peers[size_t(c->rank + 1)] : nullptr;
  return LASP_OK;
}

lasp_status_t lasp_ctx_destroy(lasp_ctx_t c) {
  if (!c) return LASP_OK;
  if (c->gather) cudaFree(c->gather);
  if (c->p2p_ipc)
    for (int k = 0; k < int(c->p2p_peers.size()); ++k)
      if (k != c->rank && c->p2p_peers[size_t(k)]) cudaIpcCloseMemHandle(c->p2p_peers[size_t(k)]);
  if (c->p2p) {
    if (c->loop) {
      std::lock_guard<std::mutex> g(c->loop->mu);
      c->loop->p2p.erase(c->rank);
    }
    cudaFree(c->p2p);
  }
  if (c->comm) nccl().CommDestroy(c->comm);
  if (c->ev_ready) cudaEventDestroy(c->ev_ready);
  if (c->ev_done) cudaEventDestroy(c->ev_done);
  if (c->comm_stream) cudaStreamDestroy(c->comm_stream);
  delete c;
  return LASP_OK;
}

lasp_status_t lasp_ring_peers(int rank, int world, int backward, int* recv_from, int* send_to) {
  if (!recv_from || !send_to) return fail(LASP_ERR_SHAPE, "NULL argument");
  if (world < 1 || rank < 0 || rank >= world) return fail(LASP_ERR_PARTITION, "rank outside [0, world)");
  if (!backward) {  // Alg. 2: Recv KV_{t-1} from i-1, Send KV_t to i+1
    *recv_from = rank > 0 ? rank - 1 : -1;
    *send_to = rank < world - 1 ? rank + 1 : -1;
  } else {          // Alg. 3: Recv dKV_{t+1} from i+1, Send dKV_t to i-1 (reading A2)
    *recv_from = rank < world - 1 ? rank + 1 : -1;
    *send_to = rank > 0 ? rank - 1 : -1;
  }
  return LASP_OK;
}

lasp_status_t lasp_topology(int rank, int world, int sp_size, int* group, int* group_rank, int* src_rank) {
  if (sp_size < 1 || world < 1 || world % sp_size != 0) {
    char b[128];
    std::snprintf(b, sizeof b, "sequence parallel size %d does not divide world size %d", sp_size, world);
    return fail(LASP_ERR_PARTITION, b);
  }
  if (rank < 0 || rank >= world) return fail(LASP_ERR_PARTITION, "rank outside [0, world)");
  if (group) *group = rank / sp_size;                 // Alg. 1: groups of T consecutive ranks
  if (group_rank) *group_rank = rank % sp_size;       // chunk index inside the group
  if (src_rank) *src_rank = (rank / sp_size) * sp_size;  // R_src = floor(R/T) * T (Alg. 1 line 5)
  return LASP_OK;
}

lasp_status_t lasp_ctx_protocol(lasp_ctx_t c, const lasp_shape_t* shape, int64_t* sends_fwd, int64_t* sends_bwd,
                                int64_t* elems_per_msg) {
  if (!c) return fail(LASP_ERR_SHAPE, "ctx is NULL");
  lasp_status_t s = validate_shape(shape);
  if (s != LASP_OK) return s;
  int f = -1, t = -1;
  lasp_ring_peers(c->rank, c->world, 0, &f, &t);
  if (sends_fwd) *sends_fwd = t >= 0 ? 1 : 0;  // Alg. 2: send to i+1
  lasp_ring_peers(c->rank, c->world, 1, &f, &t);
  if (sends_bwd) *sends_bwd = t >= 0 ? 1 : 0;  // Alg. 3 P:649 (reading A2): to i-1
  if (c->exchange == LASP_EXCHANGE_ALLGATHER) {  // one all-gather contribution per direction
    if (sends_fwd) *sends_fwd = c->world > 1 ? 1 : 0;
    if (sends_bwd) *sends_bwd = c->world > 1 ? 1 : 0;
  }
  if (elems_per_msg) *elems_per_msg = shape->batch * kv_heads(shape) * shape->head_dim * shape->head_dim;
  return LASP_OK;
}

lasp_status_t lasp_fwd(lasp_ctx_t c, const lasp_shape_t* shape, const void* q, const void* k, const void* v,
                       const float* lambda, void* o, void* cache, void* workspace, void* stream) {
  if (!c) return fail(LASP_ERR_SHAPE, "ctx is NULL");
  Plan p;
  lasp_status_t s = prologue(shape, lambda, p);
  if (s != LASP_OK) return s;
  if ((s = check_ptrs(p, {q, k, v, o}, cache, workspace)) != LASP_OK) return s;
  if ((s = check_device()) != LASP_OK) return s;
  return fwd_body(c, p, q, k, v, nullptr, o, nullptr, cache, workspace, static_cast<cudaStream_t>(stream), nullptr);
}

lasp_status_t lasp_bwd(lasp_ctx_t c, const lasp_shape_t* shape, const void* q, const void* k, const void* v,
                       const float* lambda, const void* d_o, const void* cache, void* dq, void* dk, void* dv,
                       void* workspace, void* stream) {
  if (!c) return fail(LASP_ERR_SHAPE, "ctx is NULL");
  Plan p;
  lasp_status_t s = prologue(shape, lambda, p);
  if (s != LASP_OK) return s;
  if ((s = check_ptrs(p, {q, k, v, d_o, dq, dk, dv}, cache, workspace)) != LASP_OK) return s;
  if ((s = check_device()) != LASP_OK) return s;
  return bwd_body(c, p, q, k, v, d_o, cache, nullptr, dq, dk, dv, nullptr, workspace,
                  static_cast<cudaStream_t>(stream), nullptr);
}

// ---- NEXT-3: the layer around the path (projection prologue, Norm epilogue) --------------------------------
size_t lasp_layer_workspace_bytes(const lasp_shape_t* shape) {
  if (validate_shape(shape) != LASP_OK) return 0;
  const Plan p = make_plan(shape);
  return workspace_bytes(p) + align256(size_t(p.B * p.C * p.H) * 2 * sizeof(float));  // + Norm slice sums
}

lasp_status_t lasp_layer_fwd(lasp_ctx_t c, const lasp_shape_t* shape, int64_t d_model, const void* x,
                             const void* w_q, const void* w_k, const void* w_v, const float* lambda, void* q, void* k,
                             void* v, void* y, float* rnorm, void* cache, void* workspace, void* stream) {
  Plan p;
  lasp_status_t s = prologue(shape, lambda, p);
  if (s != LASP_OK) return s;
  if (d_model < 1 || (p.C > 0 && (!x || !w_q || !w_k || !w_v || !rnorm)))
    return fail(LASP_ERR_SHAPE, "layer: d_model >= 1 and non-NULL x, w_q, w_k, w_v, rnorm required");
  if (!tc_supported(p)) return fail(LASP_ERR_UNSUPPORTED, "layer: the Norm epilogue needs bf16 and head_dim 64 or 128");
  if ((s = check_ptrs(p, {q, k, v, y}, cache, workspace)) != LASP_OK) return s;
  if ((s = check_device()) != LASP_OK) return s;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (p.C > 0) {  // Alg. 2: Q = X W_Q, K = X W_K, V = X W_V (the rank's own chunk)
    cublasHandle_t h;
    if ((s = cublas_handle(st, &h)) != LASP_OK) return s;
    const int64_t M = p.B * p.C;
    if ((s = gemm_rm(h, M, p.H * p.D, d_model, x, false, w_q, false, q, false, 0.f)) != LASP_OK) return s;
    if ((s = gemm_rm(h, M, p.Hk * p.D, d_model, x, false, w_k, false, k, false, 0.f)) != LASP_OK) return s;
    if ((s = gemm_rm(h, M, p.Hk * p.D, d_model, x, false, w_v, false, v, false, 0.f)) != LASP_OK) return s;
  }
  const NormArgs norm{rnorm, reinterpret_cast<float*>(static_cast<char*>(workspace) + workspace_bytes(p)),
                      kNormEps};
  return fwd_body(c, p, q, k, v, nullptr, y, nullptr, cache, workspace, st, &norm);
}

lasp_status_t lasp_layer_bwd(lasp_ctx_t c, const lasp_shape_t* shape, int64_t d_model, const void* x,
                             const void* w_q, const void* w_k, const void* w_v, const float* lambda, const void* q,
                             const void* k, const void* v, const void* y, const float* rnorm, const void* dy,
                             const void* cache, void* d_o, void* dq, void* dk, void* dv, void* dx, float* dw_q,
                             float* dw_k, float* dw_v, void* workspace, void* stream) {
  Plan p;
  lasp_status_t s = prologue(shape, lambda, p);
  if (s != LASP_OK) return s;
  if (d_model < 1 || (p.C > 0 && (!x || !w_q || !w_k || !w_v || !rnorm || !dx || !dw_q || !dw_k || !dw_v)))
    return fail(LASP_ERR_SHAPE, "layer: d_model >= 1 and non-NULL x, w_*, rnorm, dx, dw_* required");
  if (!tc_supported(p)) return fail(LASP_ERR_UNSUPPORTED, "layer: the Norm backward needs bf16 and head_dim 64 or 128");
  if ((s = check_ptrs(p, {q, k, v, y, dy, d_o, dq, dk, dv}, cache, workspace)) != LASP_OK) return s;
  if ((s = check_device()) != LASP_OK) return s;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const NormBwdArgs nb{y, rnorm, d_o};
  if ((s = bwd_body(c, p, q, k, v, dy, cache, nullptr, dq, dk, dv, nullptr, workspace, st, &nb)) != LASP_OK) return s;
  if (p.C > 0) {  // dX = dQ W_Q^T + dK W_K^T + dV W_V^T; dW_* = X^T d* (fp32)
    cublasHandle_t h;
    if ((s = cublas_handle(st, &h)) != LASP_OK) return s;
    const int64_t M = p.B * p.C, NQ = p.H * p.D, NK = p.Hk * p.D;
    if ((s = gemm_rm(h, M, d_model, NQ, dq, false, w_q, true, dx, false, 0.f)) != LASP_OK) return s;
    if ((s = gemm_rm(h, M, d_model, NK, dk, false, w_k, true, dx, false, 1.f)) != LASP_OK) return s;
    if ((s = gemm_rm(h, M, d_model, NK, dv, false, w_v, true, dx, false, 1.f)) != LASP_OK) return s;
    if ((s = gemm_rm(h, d_model, NQ, M, x, true, dq, false, dw_q, true, 0.f)) != LASP_OK) return s;
    if ((s = gemm_rm(h, d_model, NK, M, x, true, dk, false, dw_k, true, 0.f)) != LASP_OK) return s;
    if ((s = gemm_rm(h, d_model, NK, M, x, true, dv, false, dw_v, true, 0.f)) != LASP_OK) return s;
  }
  return LASP_OK;
}

// ---- NEXT-4: generalised decay (the GLA / GateLoop row of Table 3) ---------------------------------------
size_t lasp_gla_cache_bytes(const lasp_shape_t* shape) {
  GlaPlan g;
  return gla_plan(shape, g) == LASP_OK ? gla_cache_bytes(g) : 0;
}

size_t lasp_gla_workspace_bytes(const lasp_shape_t* shape) {
  GlaPlan g;
  return gla_plan(shape, g) == LASP_OK ? gla_ws_bytes(g) : 0;
}

int64_t lasp_gla_segment_len(const lasp_shape_t* shape) {
  GlaPlan g;
  return gla_plan(shape, g) == LASP_OK ? g.seg_len : 0;
}

lasp_status_t lasp_gla_fwd_local(const lasp_shape_t* shape, const float* q, const float* k, const float* v,
                                 const float* log_g, const float* kv_in, float* o, float* kv_out, void* cache,
                                 void* workspace, void* stream) {
  GlaPlan g;
  lasp_status_t s = gla_plan(shape, g);
  if (s != LASP_OK) return s;
  if ((s = gla_check(g, {q, k, v, log_g, o}, cache, workspace)) != LASP_OK) return s;
  return gla_fwd_body(nullptr, g, q, k, v, log_g, kv_in, o, kv_out, cache, workspace, static_cast<cudaStream_t>(stream));
}

lasp_status_t lasp_gla_bwd_local(const lasp_shape_t* shape, const float* q, const float* k, const float* v,
                                 const float* log_g, const float* d_o, const void* cache, const float* dkv_in,
                                 float* dq, float* dk, float* dv, float* dlog_g, float* dkv_out, void* workspace,
                                 void* stream) {
  GlaPlan g;
  lasp_status_t s = gla_plan(shape, g);
  if (s != LASP_OK) return s;
  if ((s = gla_check(g, {q, k, v, log_g, d_o, dq, dk, dv, dlog_g}, cache, workspace)) != LASP_OK) return s;
  return gla_bwd_body(nullptr, g, q, k, v, log_g, d_o, cache, dkv_in, dq, dk, dv, dlog_g, dkv_out, workspace,
                      static_cast<cudaStream_t>(stream));
}

lasp_status_t lasp_gla_fwd(lasp_ctx_t c, const lasp_shape_t* shape, const float* q, const float* k, const float* v,
                           const float* log_g, float* o, void* cache, void* workspace, void* stream) {
  if (!c) return fail(LASP_ERR_SHAPE, "ctx is NULL");
  GlaPlan g;
  lasp_status_t s = gla_plan(shape, g);
  if (s != LASP_OK) return s;
  if ((s = gla_check(g, {q, k, v, log_g, o}, cache, workspace)) != LASP_OK) return s;
  return gla_fwd_body(c, g, q, k, v, log_g, nullptr, o, nullptr, cache, workspace, static_cast<cudaStream_t>(stream));
}

lasp_status_t lasp_gla_bwd(lasp_ctx_t c, const lasp_shape_t* shape, const float* q, const float* k, const float* v,
                           const float* log_g, const float* d_o, const void* cache, float* dq, float* dk, float* dv,
                           float* dlog_g, void* workspace, void* stream) {
  if (!c) return fail(LASP_ERR_SHAPE, "ctx is NULL");
  GlaPlan g;
  lasp_status_t s = gla_plan(shape, g);
  if (s != LASP_OK) return s;
  if ((s = gla_check(g, {q, k, v, log_g, d_o, dq, dk, dv, dlog_g}, cache, workspace)) != LASP_OK) return s;
  return gla_bwd_body(c, g, q, k, v, log_g, d_o, cache, nullptr, dq, dk, dv, dlog_g, nullptr, workspace,
                      static_cast<cudaStream_t>(stream));
}

}  // extern "C"
