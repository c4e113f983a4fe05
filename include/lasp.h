/*
 * lasp.h -- C ABI of the B200-native LASP hot path (Linear Attention Sequence Parallelism,
 * arXiv 2404.02882): chunked causal linear attention with per-head decay lambda, sequence
 * split across ranks, one d x d KV state per head passed forward around a P2P ring and a
 * dKV state passed backward.
 *
 * Citations: "P:n" = line n of the paper text; "S:n" = line n of SPEC.md.
 *
 * ------------------------------------------------------------------------------------------
 * What is computed (per batch row b, head h; rank r owns tokens [r*C, (r+1)*C), C = n_local,
 * P:106-111 with T = W):
 *
 *   O    : o_s^T = q_s^T sum_{i<=s} lambda_h^(s-i) k_i v_i^T          (Eq. 4)
 *          evaluated per rank as Alg. 2:
 *            O_r = [(Q_r K_r^T) (.) M] V_r + Lambda Q_r KV_in(r)        (Eq. 7, 9)
 *            KV_out(r) = lambda^C KV_in(r) + (lambda^C Lambda^-1 K_r)^T V_r   (Eq. 12)
 *          M_ij = lambda^(i-j) (i >= j), Lambda = diag(lambda^1..lambda^C). No Norm(.)
 *          and no 1/sqrt(d).
 *   dQ, dK, dV : gradients of L = sum(O (.) dO) (Eq. 13-14), evaluated per rank as
 *          Alg. 3:
 *            dQ_r = [(dO V^T) (.) M] K + Lambda dO KV_in(r)^T
 *            dK_r = [(dO V^T) (.) M]^T Q + lambda^C Lambda^-1 V dKV_in(r)^T
 *            dV_r = [(Q K^T) (.) M]^T dO + lambda^C Lambda^-1 K dKV_in(r)
 *            dKV_out(r) = lambda^C dKV_in(r) + (Lambda Q_r)^T dO_r
 *          where dKV_in(r) = sum_{g >= (r+1)C} lambda^(g-(r+1)C+1) q_g do_g^T (exponent starts at
 *          1; reading A3) arrives from rank r+1 and dKV_out(r) goes to r-1 (reading A2).
 *
 * KV-state caching: lasp_fwd* writes into a caller-owned cache the state
 * ENTERING the rank, KV_in(r) (reading A4), plus the in-rank segment states derived from it;
 * lasp_bwd* reads them and never re-communicates KV.
 *
 * ------------------------------------------------------------------------------------------
 * Conventions
 *   Layout   : every sequence tensor is [batch][n_local][heads][head_dim], contiguous, row-major,
 *              device memory owned by the caller, base address 16-byte aligned. Element type is
 *              bf16 (LASP_BF16) or fp32 (LASP_FP32) for q, k, v, o, d_o, dq, dk, dv alike.
 *   States   : kv_in / kv_out / dkv_in / dkv_out are fp32 [batch][kv_heads][head_dim][head_dim],
 *              row index = the first factor's dimension (KV = sum k v^T: rows index k, columns v;
 *              dKV = sum q do^T: rows index q, columns do). Device memory, caller-owned.
 *   lambda   : HOST pointer to `kv_heads` (= `heads` unless grouped-query) fp32 decay rates, each in
 *              (0, 1] (P:145 gives a single lambda, heads are independent, P:18 -- reading A7).
 *              lambda = 1 is plain linear attention.
 *   Streams  : all device work is enqueued on the caller's stream; calls return after enqueue.
 *              The kernels of a call use programmatic dependent launch among themselves; the first
 *              one waits until all earlier work on the stream has completed before any other kernel of
 *              the call may start, so inputs produced by any earlier kernel (early-triggering or not)
 *              are complete when they are read.
 *   Graphs   : lasp_fwd_local / lasp_bwd_local and the NCCL entry points can be captured into CUDA
 *              graphs (the programmatic launch edges are kept; bench.py replays its step from a
 *              graph). Contexts made by lasp_ctx_create_loopback use host threads and cannot.
 *   Errors   : argument validation is synchronous and enqueues nothing. On a non-OK status
 *              lasp_last_error() returns a thread-local message. LASP_ERR_CUDA / LASP_ERR_COMM
 *              report launch / NCCL failures (with rank and peer for COMM). The KV-cache check
 *              (LASP_ERR_STATE) runs on the device, see lasp_workspace_status.
 *   Sizes    : n_local may be any value >= 0 (a ragged last GPU block is zero-padded on load and
 *              clipped on store); n_local = 0 is a no-op that forwards the state (kv_out = kv_in).
 *              head_dim must be 32, 64 or 128 (else LASP_ERR_UNSUPPORTED).
 *   Determinism: results are bitwise reproducible run to run for fixed inputs and shape (no
 *              order-dependent atomics; segment states are folded in a fixed order).
 *   Protocol : per direction and per call exactly world-1 messages of batch*heads*head_dim^2 fp32
 *              elements cross the ring, independent of n_local (Table 1 LASP row).
 *              Forward goes r -> r+1, backward r+1 -> r.
 */
#ifndef LASP_H_
#define LASP_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  LASP_OK = 0,
  LASP_ERR_SHAPE = 1,       /* null/misaligned pointer, negative or inconsistent sizes          */
  LASP_ERR_DOMAIN = 2,      /* lambda outside (0, 1]                                    */
  LASP_ERR_PARTITION = 3,   /* world/rank inconsistent (rank outside [0, world))                */
  LASP_ERR_STATE = 4,       /* cache not written by a matching lasp_fwd*                 */
  LASP_ERR_COMM = 5,        /* NCCL failure or NCCL unavailable                                  */
  LASP_ERR_CUDA = 6,        /* CUDA launch / driver failure                                      */
  LASP_ERR_UNSUPPORTED = 7  /* head_dim not in {32, 64, 128} or device is not sm_100            */
} lasp_status_t;

typedef enum { LASP_BF16 = 0, LASP_FP32 = 1 } lasp_dtype_t;

typedef struct {
  int64_t batch;     /* B >= 1                                   */
  int64_t n_local;   /* C = tokens owned by this rank, >= 0       */
  int64_t heads;     /* H >= 1 (query heads)                     */
  int64_t head_dim;  /* D = d_k = d_v, one of 32, 64, 128 */
  lasp_dtype_t dtype;
  int64_t kv_heads;  /* Hk: key/value heads, 0 = H (multi-head). Hk < H is grouped-query (multi-query for
                      * Hk = 1) attention: H % Hk == 0, query head h reads
                      * kv-head h / (H/Hk), and each kv-head has ONE shared state (and decay). k, v, dk, dv are
                      * [B][C][Hk][D]; lambda, the states, the cache and the ring messages are per kv-head.
                      * Needs bf16 and head_dim 64 or 128 (else LASP_ERR_UNSUPPORTED).          */
} lasp_shape_t;

/* Opaque ring context: owns the NCCL communicator and nothing else. */
typedef struct lasp_ctx* lasp_ctx_t;

/* Message for the last non-OK status on the calling thread ("" if none). */
const char* lasp_last_error(void);

/* Library version string and whether the tcgen05 (sm_100a) path is compiled in. */
const char* lasp_version(void);

/* Number of CUDA kernels this library has launched since it was loaded (all entry points). */
uint64_t lasp_launch_count(void);

/* Measurement hooks (bench.py): when enabled, every kernel launch is bracketed by CUDA events
 * recorded on the launching stream. lasp_profile_read synchronizes on them, writes a JSON object
 * {"stage": [launches, total_ms], ...} into buf (NUL-terminated, truncated to cap) and clears the
 * records; returns the JSON length, or -1 if an event could not be read. */
void lasp_profile_enable(int on);
/* Debug only: when non-NULL, tcgen05 core kernels record a clock64 timeline of CTA 0 into the
 * device buffer (2 regions of 16 events x 64 blocks, unsigned 64-bit: core kernel, then segment-state
 * kernel). Pass NULL to disable. */
void lasp_debug_trace(unsigned long long* device_buf);
int lasp_profile_read(char* buf, size_t cap);
/* Experiments only: launches `ctas` CTAs on `stream`, each holding `smem_bytes` of shared memory (with
 * >= 120 KB, one per SM and no co-resident 224 KB core CTA) and spinning for `microseconds` -- a stand-in
 * for another stream's kernels (e.g. NCCL's) occupying SMs while a persistent LASP kernel runs. */
lasp_status_t lasp_debug_occupy(int ctas, int smem_bytes, double microseconds, void* stream);

/* Bytes of the caller-owned per-layer KV cache for `shape`: fp32 segment states [B][H][nseg][D][D] (entry
 * 0 = the state entering the rank, KV_in(r), reading A4; entry p = the state entering in-rank segment p),
 * followed by a 256-byte tag (shape, segment length, dtype, lambda hash, rank, world, generation) that
 * lasp_fwd* writes and lasp_bwd* checks on the device. 16-byte aligned base. */
size_t lasp_cache_bytes(const lasp_shape_t* shape);

/* Result of the cache-tag check of the last lasp_bwd / lasp_bwd_local call that used `workspace` on
 * `stream` (synchronizes the stream). LASP_OK, or LASP_ERR_STATE when the cache was not written by a
 * lasp_fwd* call with the same shape, lambda and (ring calls) rank and world -- a buffer never written by
 * a forward, a freed-and-reused allocation now holding another forward's cache, a different lambda, ...
 * lasp_last_error() then names the mismatching fields. A backward whose check fails still runs, but every
 * state it loads is NaN, so dq, dk and dv are NaN: the mismatch cannot go unnoticed. (The
 * check is on the device so that calls stay asynchronous and capturable into CUDA graphs, and no host
 * registry keyed by pointers can be fooled by address reuse.) dkv_out is computed from q and d_o only
 * (not from the cache) and is not poisoned. */
lasp_status_t lasp_workspace_status(const void* workspace, void* stream /* cudaStream_t */);

/* Bytes of the caller-owned scratch workspace used by lasp_fwd, lasp_fwd_local, lasp_bwd and lasp_bwd_local (reusable across
 * calls on the same stream; contents are not preserved). */
size_t lasp_workspace_bytes(const lasp_shape_t* shape);

/* In-rank segment length (tokens) the library uses for `shape` (reported for tests/bench). */
int64_t lasp_segment_len(const lasp_shape_t* shape);

/* ---- communication-free halves (one rank's compute; a ring can be simulated on one GPU by
 *      chaining kv_out -> kv_in, exactly the Recv/Send of Alg. 2/3 without a transport) ---- */

/* Alg. 2 for one rank. kv_in: state entering the rank (NULL = zero, rank 0). kv_out
 * (nullable): KV_out(r) = lambda^C KV_in + (lambda^C Lambda^-1 K)^T V. Writes o and cache. */
lasp_status_t lasp_fwd_local(const lasp_shape_t* shape, const void* q, const void* k, const void* v,
                             const float* lambda, const float* kv_in, void* o, float* kv_out,
                             void* cache, void* workspace, void* stream /* cudaStream_t */);

/* Alg. 3 for one rank. dkv_in: dKV_in(r) from rank r+1 (NULL = zero, last rank).
 * dkv_out (nullable): lambda^C dKV_in + (Lambda Q)^T dO. `cache` must come from lasp_fwd_local or
 * lasp_fwd with the same shape and lambda; otherwise the outputs are NaN and lasp_workspace_status()
 * returns LASP_ERR_STATE. */
lasp_status_t lasp_bwd_local(const lasp_shape_t* shape, const void* q, const void* k, const void* v,
                             const float* lambda, const void* d_o, const void* cache,
                             const float* dkv_in, void* dq, void* dk, void* dv, float* dkv_out,
                             void* workspace, void* stream);

/* ---- the ring (NCCL point-to-point over NVLink; one process per GPU) ---- */

/* Writes a 128-byte NCCL unique id (rank 0 calls it; broadcast it with torch.distributed). */
lasp_status_t lasp_unique_id(uint8_t id[128]);

/* Creates the ring context for (rank, world) on CUDA device `device` (collective over the world). */
lasp_status_t lasp_ctx_create(int rank, int world, const uint8_t id[128], int device, lasp_ctx_t* out);
lasp_status_t lasp_ctx_destroy(lasp_ctx_t ctx);

/* Same ring context with an in-process loopback transport instead of NCCL: the `world` ranks are
 * threads of one process sharing CUDA device `device`, joined by the group name `group` (NUL-terminated,
 * owned by the caller). A send stages the message in a stream-ordered device allocation and records an
 * event on the sender's stream; the matching receive makes the receiver's stream wait on that event and
 * copies the message out, the receiving host thread blocking (up to 120 s, then LASP_ERR_COMM) until the
 * send is posted. Exists so that lasp_fwd / lasp_bwd with world > 1 can be exercised on a single GPU
 * (NCCL refuses two ranks on one device). LASP_ERR_PARTITION for a rank outside [0, world) or a group
 * name already in use with another world size. Destroy with lasp_ctx_destroy. */
lasp_status_t lasp_ctx_create_loopback(int rank, int world, const char* group, int device, lasp_ctx_t* out);

/* State exchange of lasp_fwd / lasp_bwd (not in the paper, which only has the ring).
 *   LASP_EXCHANGE_RING (default): the paper's T-1 dependent hops, Alg. 2 P:167-172 / Alg. 3 P:629-649.
 *   LASP_EXCHANGE_ALLGATHER: one all-gather of the T local states (B*H*D*D fp32 each; ncclAllGather, or
 *     pairwise sends on a loopback ctx) into a ctx-owned buffer, then each rank folds the states it would
 *     have received: KV_in(r) = sum_{j<r} lam^(C(r-1-j)) L_j, dKV_in(r) = sum_{j>r} lam^(C(j-r-1)) G_j.
 *     Same results up to fp32 summation order. Each rank's n_local travels with its state, so ranks of
 *     different lengths fold correctly (rank j's contribution is decayed with lam^(C_j)).
 *   LASP_EXCHANGE_P2P: the paper's ring, each hop ONE kernel over peer memory (NVLink): it waits for the
 *     upstream rank's data flag on this rank's receive buffer, copies KV_in out, and stores
 *     lam^C KV_in + L_r straight into the downstream rank's receive buffer (combine and send fused), then
 *     publishes a data flag to the downstream and an ack to the upstream (a sender waits for the ack of its
 *     previous message before overwriting). Flags are epoch counters in device memory, so steps can be
 *     graph-captured and replayed. Needs lasp_ctx_p2p_setup + lasp_ctx_p2p_connect; scalar-decay path only.
 *     The waits are on the device: with several ranks on ONE device (a loopback ctx, or processes sharing a
 *     GPU) no rank may block in a device-wide synchronize before the other ranks have submitted their calls
 *     (synchronize the rank's own stream instead), and no rank may launch a kernel for the first time in the
 *     process while a peer's hop kernel waits (lazy module loading synchronizes the context): run one step
 *     over another exchange first, or set CUDA_MODULE_LOADING=EAGER; across GPUs the ranks are independent.
 * LASP_ERR_DOMAIN for any other value; LASP_ERR_COMM for RING / ALLGATHER on a P2P-only ctx. */
#define LASP_EXCHANGE_RING 0
#define LASP_EXCHANGE_ALLGATHER 1
#define LASP_EXCHANGE_P2P 2
/*   LASP_EXCHANGE_P2P_ALLGATHER: the all-gather exchange as ONE kernel per direction over peer memory: each rank
 *     stores its local state (and n_local) into its slot of every downstream rank's block, publishes a data flag
 *     there, waits for the flags of every upstream rank and folds what arrived (the same fold as
 *     LASP_EXCHANGE_ALLGATHER); acks and epochs as LASP_EXCHANGE_P2P. One step instead of T - 1 dependent hops,
 *     no NCCL. Same setup (lasp_ctx_p2p_setup / _connect; world <= 64). */
#define LASP_EXCHANGE_P2P_ALLGATHER 3
lasp_status_t lasp_ctx_set_exchange(lasp_ctx_t ctx, int exchange);

/* A ring ctx without NCCL whose only exchanges are the P2P ones (peer buffers through CUDA IPC): rank r of
 * world ranks on `device` (several processes may share one GPU). Destroy with lasp_ctx_destroy. */
lasp_status_t lasp_ctx_create_p2p(int rank, int world, int device, lasp_ctx_t* out);
/* Collective P2P setup, step 1 (every rank): allocate this rank's flag / receive block for states of up to
 * max_state_elems (= batch * kv_heads * head_dim^2; the same value on every rank) and write its CUDA IPC handle
 * (64 bytes) to `handle`. The caller gathers the world's handles in rank order (e.g. torch.distributed
 * all_gather_object). LASP_ERR_STATE if already set up. */
lasp_status_t lasp_ctx_p2p_setup(lasp_ctx_t ctx, size_t max_state_elems, uint8_t handle[64]);
/* Step 2: open the blocks of the other ranks from `handles` (world x 64 bytes, rank order), or, on a
 * loopback ctx, handles = NULL: take them from the loopback group (waits up to 120 s for the peers' setup).
 * LASP_ERR_COMM if a handle cannot be opened. */
lasp_status_t lasp_ctx_p2p_connect(lasp_ctx_t ctx, const uint8_t* handles);

/* Ring schedule (host-only, no GPU): the peer this rank receives its state from and sends its state to
 * (-1 = none). Forward (backward = 0): from r-1, to r+1 (Alg. 2); backward: from r+1, to r-1
 * (Alg. 3, reading A2 of P:649). Used by lasp_fwd/lasp_bwd; exposed for protocol tests. */
lasp_status_t lasp_ring_peers(int rank, int world, int backward, int* recv_from, int* send_to);

/* Data-sequence hybrid topology (host-only, no GPU): Alg. 1
 * with W = world ranks and sequence-parallel size T = sp_size: G = W/T groups; global rank R belongs to
 * group floor(R/T), holds chunk R mod T of that group's sequence (tokens [(R mod T) C, (R mod T + 1) C)),
 * and the group's source rank is floor(R/T)*T (R_src, Alg. 1 line 5). Each group runs its own ring: create
 * one ctx per group with lasp_ctx_create(group_rank, T, <the group's id>, ...); no message crosses a group.
 * Any output pointer may be NULL. LASP_ERR_PARTITION if sp_size < 1, world % sp_size != 0 (reading A6: T
 * divides W) or rank outside [0, world). */
lasp_status_t lasp_topology(int rank, int world, int sp_size, int* group, int* group_rank, int* src_rank);

/* Messages and fp32 elements per message this ctx will send per direction per call (protocol
 * introspection for tests: ring exchange: world-1 hops in total, this rank sends 0 or 1; all-gather
 * exchange: one contribution per rank when world > 1). */
lasp_status_t lasp_ctx_protocol(lasp_ctx_t ctx, const lasp_shape_t* shape, int64_t* sends_fwd,
                                int64_t* sends_bwd, int64_t* elems_per_msg);

/* Alg. 2 across the ring: every rank calls it with identical shape and lambda. Rank r receives
 * KV_in(r) from r-1, stores it in its cache, sends KV_out(r) to r+1, and writes O_r. */
lasp_status_t lasp_fwd(lasp_ctx_t ctx, const lasp_shape_t* shape, const void* q, const void* k,
                       const void* v, const float* lambda, void* o, void* cache, void* workspace,
                       void* stream);

/* Alg. 3 across the ring: receives dKV_in(r) from r+1, sends dKV_out(r) to r-1, writes dQ, dK, dV.
 * The cache's tag must match (shape, lambda, rank, world), else NaN outputs + lasp_workspace_status. */
lasp_status_t lasp_bwd(lasp_ctx_t ctx, const lasp_shape_t* shape, const void* q, const void* k,
                       const void* v, const float* lambda, const void* d_o, const void* cache,
                       void* dq, void* dk, void* dv, void* workspace, void* stream);

/* ---- the steps either side of the path: one attention layer ----
 *
 *   Q = X W_Q, K = X W_K, V = X W_V          (Alg. 2; X is this rank's chunk, [B][C][d_model])
 *   O = LASP(Q, K, V; lambda)                (as lasp_fwd_local / lasp_fwd)
 *   Y = Norm(O)                              (Eq. 2; the paper leaves Norm undefined, P:180 --
 *                                             DESIGN.md reading N1: per-head RMS normalization
 *                                             y = o r, r = (mean_c o_c^2 + 1e-6)^(-1/2) per (b, s, h))
 * ctx == NULL: a single rank (no ring; the state entering the rank is zero); else the ring of ctx.
 * Layouts: x [B][C][d_model] bf16; w_q [d_model][H*D], w_k, w_v [d_model][Hk*D] bf16 (row-major, so
 * X W_Q is the [B][C][H][D] layout of q); q, y, d_o, dq [B][C][H][D] bf16; k, v, dk, dv [B][C][Hk][D]
 * bf16; rnorm [B][C][H] fp32; dx bf16 like x; dw_* fp32 like w_*. Needs bf16 and head_dim 64 or 128.
 * Fusion: the projections are plain tensor-core GEMMs (cuBLAS, loaded at first use; LASP_CUBLAS_LIB
 * overrides the library path); the Norm runs in the epilogue of the forward core kernel (head_dim 64:
 * y and r written directly; head_dim 128: the two value-slice items of a row meet in a second, elementwise
 * phase), and its backward dO = r (dY - y (y . dY) / D) runs inside the B1 kernel (dKV-state
 * accumulation), which writes dO to d_o for the B3 passes. workspace: lasp_layer_workspace_bytes. */
size_t lasp_layer_workspace_bytes(const lasp_shape_t* shape);
lasp_status_t lasp_layer_fwd(lasp_ctx_t ctx, const lasp_shape_t* shape, int64_t d_model, const void* x,
                             const void* w_q, const void* w_k, const void* w_v, const float* lambda,
                             void* q, void* k, void* v, void* y, float* rnorm, void* cache, void* workspace,
                             void* stream);
/* Gradients of sum(Y * dY): dx, dw_q, dw_k, dw_v (and the intermediates d_o = dL/dO, dq, dk, dv, which
 * the caller provides as scratch). q, k, v, y, rnorm and cache come from lasp_layer_fwd. */
lasp_status_t lasp_layer_bwd(lasp_ctx_t ctx, const lasp_shape_t* shape, int64_t d_model, const void* x,
                             const void* w_q, const void* w_k, const void* w_v, const float* lambda,
                             const void* q, const void* k, const void* v, const void* y, const float* rnorm,
                             const void* dy, const void* cache, void* d_o, void* dq, void* dk, void* dv,
                             void* dx, float* dw_q, float* dw_k, float* dw_v, void* workspace, void* stream);

/* ---- generalised decay: the GLA / GateLoop row of Table 3 ----
 *
 *   kv_t = Diag(g_t) kv_{t-1} + k_t v_t^T,   o_t = kv_t^T q_t,   g_t = exp(log_g_t) in (0, 1]^head_dim
 *
 * (App. A.4, the general form m_t = o_t m_{t-1} + e_t i_t^T with o_t = g_t 1^T, GLA / GateLoop
 * P:735; readings D1-D3). The decay is data-dependent: one value per token, head and key channel;
 * a per-channel constant decay is log_g_t = log(lambda) for every t, and lambda = exp(log_g) per head is the
 * scalar path. The paper claims LASP covers this row without giving the chunk form; this path
 * uses: segment state L_p (recurrence from zero), segment decay exp(sum log_g) per key row, the fold
 * P_{p+1} = Diag(exp(ls_p)) P_p + L_p, and the same one-state-per-head ring messages as Alg. 2 / 3 (KV r -> r+1,
 * dKV r+1 -> r; dKV = gradient of the later ranks' loss w.r.t. the state leaving the rank).
 * Tensors: fp32 (shape->dtype = LASP_FP32), kv_heads = heads (or 0), head_dim 32, 64 or 128; q, k, v, log_g,
 * o, d_o, dq, dk, dv, dlog_g are [batch][n_local][heads][head_dim]; states fp32 [batch][heads][head_dim]^2.
 * log_g must be <= 0 (not checked on the device). dlog_g = dL/dlog_g, L = sum(O * dO).
 * Cache / workspace: caller-owned, lasp_gla_cache_bytes / lasp_gla_workspace_bytes; the cache holds the state
 * entering every segment and the state leaving the rank, plus a tag (a backward whose cache was not written by
 * a matching lasp_gla_fwd* gets NaN outputs and lasp_workspace_status = LASP_ERR_STATE). Errors: LASP_ERR_SHAPE
 * (NULL / misaligned pointers, bad sizes), LASP_ERR_UNSUPPORTED (dtype, head_dim, kv_heads), LASP_ERR_COMM. */
size_t lasp_gla_cache_bytes(const lasp_shape_t* shape);
size_t lasp_gla_workspace_bytes(const lasp_shape_t* shape);
int64_t lasp_gla_segment_len(const lasp_shape_t* shape);
lasp_status_t lasp_gla_fwd_local(const lasp_shape_t* shape, const float* q, const float* k, const float* v,
                                 const float* log_g, const float* kv_in, float* o, float* kv_out, void* cache,
                                 void* workspace, void* stream);
lasp_status_t lasp_gla_bwd_local(const lasp_shape_t* shape, const float* q, const float* k, const float* v,
                                 const float* log_g, const float* d_o, const void* cache, const float* dkv_in,
                                 float* dq, float* dk, float* dv, float* dlog_g, float* dkv_out, void* workspace,
                                 void* stream);
lasp_status_t lasp_gla_fwd(lasp_ctx_t ctx, const lasp_shape_t* shape, const float* q, const float* k,
                           const float* v, const float* log_g, float* o, void* cache, void* workspace, void* stream);
lasp_status_t lasp_gla_bwd(lasp_ctx_t ctx, const lasp_shape_t* shape, const float* q, const float* k,
                           const float* v, const float* log_g, const float* d_o, const void* cache, float* dq,
                           float* dk, float* dv, float* dlog_g, void* workspace, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* LASP_H_ */
