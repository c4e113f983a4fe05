/*
 * lasp_oracle.c -- plain, slow, fp64 CPU oracle for the LASP hot path (arXiv 2404.02882).
 *
 * TEST INFRASTRUCTURE ONLY. Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library. It shares no code, header,
 * table or constant generator with the CUDA path (paper_2404_02882_b200/csrc, include/).
 *
 * Citations: "P:n" = line n of the paper text, "S:n" = line n of SPEC.md.
 * Notation follows the paper: q_s, k_s, v_s, o_s rows; kv_s / dkv_s states (d x d);
 * chunk size C = N/T; M_ij = lambda^(i-j) (i >= j); Lambda = diag(lambda, ..., lambda^C).
 *
 * Layout of every sequence tensor: [B][N][H][D] row-major doubles (token-major, heads
 * interleaved), the same logical layout as the C-ABI boundary. States: [B][H][D][D].
 *
 * lambda is passed as float and promoted with (double)(float)lambda -- DESIGN.md reading A8:
 * the boundary carries fp32 lambda, so the oracle computes with exactly that value.
 * Powers of lambda are formed by repeated multiplication; nothing is divided by a
 * power of lambda and Lambda^-1 is never formed (reading A9, P:230 read as
 * lambda^C Lambda^-1 = diag(lambda^(C-1), ..., 1)).
 *
 * Parity pins: every exported function is pinned by tests/test_oracle_*.py against the
 * dense masked form, fp64 autograd, finite differences, closed forms and the SPEC worked
 * examples.
 */
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>

#define ORACLE_OK 0
#define ORACLE_ERR_SHAPE 1
#define ORACLE_ERR_DOMAIN 2
#define ORACLE_ERR_PARTITION 3
#define ORACLE_ERR_NOMEM 8

static int check_lams(int64_t H, const float* lam) {
    for (int64_t h = 0; h < H; ++h) {
        double l = (double)lam[h];
        if (!(l > 0.0 && l <= 1.0)) return ORACLE_ERR_DOMAIN; /* S:159, lambda in (0,1] */
    }
    return ORACLE_OK;
}

/* ---------------------------------------------------------------------------------- */
/* Work distribution: one work item per (b, h); plain pthreads with a shared counter.   */
/* ---------------------------------------------------------------------------------- */
typedef void (*item_fn)(void* ctx, int64_t item);
typedef struct {
    item_fn fn;
    void* ctx;
    int64_t n_items;
    int64_t next;
    pthread_mutex_t mu;
} pool_t;

static void* pool_worker(void* arg) {
    pool_t* p = (pool_t*)arg;
    for (;;) {
        pthread_mutex_lock(&p->mu);
        int64_t it = p->next++;
        pthread_mutex_unlock(&p->mu);
        if (it >= p->n_items) break;
        p->fn(p->ctx, it);
    }
    return NULL;
}

static void run_items(item_fn fn, void* ctx, int64_t n_items, int nthreads) {
    if (nthreads < 1) nthreads = 1;
    if (nthreads > n_items) nthreads = (int)(n_items > 0 ? n_items : 1);
    pool_t p;
    p.fn = fn; p.ctx = ctx; p.n_items = n_items; p.next = 0;
    pthread_mutex_init(&p.mu, NULL);
    if (nthreads == 1) {
        pool_worker(&p);
    } else {
        pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)nthreads);
        for (int i = 0; i < nthreads; ++i) pthread_create(&th[i], NULL, pool_worker, &p);
        for (int i = 0; i < nthreads; ++i) pthread_join(th[i], NULL);
        free(th);
    }
    pthread_mutex_destroy(&p.mu);
}

/* ---------------------------------------------------------------------------------- */
/* Definition mode: the recurrence of Eq. 5 and Eq. 13-14.       */
/* ---------------------------------------------------------------------------------- */
typedef struct {
    int64_t B, N, H, D;
    const double *q, *k, *v, *dout;
    const float* lam;
    double *o, *dq, *dk, *dv;
} rec_ctx_t;

#define ROW(p, c, b, s, h) ((p) + ((((b) * (c)->N + (s)) * (c)->H + (h)) * (c)->D))

/* Forward, Eq. 5: kv_0 = 0; kv_s = lambda kv_{s-1} + k_s v_s^T; o_s^T = q_s^T kv_s. */
static void rec_fwd_item(void* vctx, int64_t item) {
    rec_ctx_t* c = (rec_ctx_t*)vctx;
    const int64_t b = item / c->H, h = item % c->H, D = c->D;
    const double lam = (double)c->lam[h];
    double* kv = (double*)calloc((size_t)(D * D), sizeof(double));
    for (int64_t s = 0; s < c->N; ++s) {
        const double* qs = ROW(c->q, c, b, s, h);
        const double* ks = ROW(c->k, c, b, s, h);
        const double* vs = ROW(c->v, c, b, s, h);
        double* os = ROW(c->o, c, b, s, h);
        for (int64_t d = 0; d < D; ++d)
            for (int64_t e = 0; e < D; ++e) kv[d * D + e] = lam * kv[d * D + e] + ks[d] * vs[e];
        for (int64_t e = 0; e < D; ++e) os[e] = 0.0;
        for (int64_t d = 0; d < D; ++d)
            for (int64_t e = 0; e < D; ++e) os[e] += qs[d] * kv[d * D + e];
    }
    free(kv);
}

/* Backward, Eq. 13: dq_s^T = do_s^T kv_s^T (kv_s inclusive of s, reading A16);
 * dkv_s = sum_{i>=s} lambda^(i-s) q_i do_i^T via the reverse recurrence of Eq. 14
 * (dkv_{N+1} = 0; dkv_s = lambda dkv_{s+1} + q_s do_s^T);
 * dk_s^T = v_s^T dkv_s^T; dv_s^T = k_s^T dkv_s. */
static void rec_bwd_item(void* vctx, int64_t item) {
    rec_ctx_t* c = (rec_ctx_t*)vctx;
    const int64_t b = item / c->H, h = item % c->H, D = c->D;
    const double lam = (double)c->lam[h];
    double* kv = (double*)calloc((size_t)(D * D), sizeof(double));
    /* sweep 1: recompute kv_s forward, dq_s[d] = sum_e kv_s[d][e] do_s[e] */
    for (int64_t s = 0; s < c->N; ++s) {
        const double* ks = ROW(c->k, c, b, s, h);
        const double* vs = ROW(c->v, c, b, s, h);
        const double* dos = ROW(c->dout, c, b, s, h);
        double* dqs = ROW(c->dq, c, b, s, h);
        for (int64_t d = 0; d < D; ++d)
            for (int64_t e = 0; e < D; ++e) kv[d * D + e] = lam * kv[d * D + e] + ks[d] * vs[e];
        for (int64_t d = 0; d < D; ++d) {
            double acc = 0.0;
            for (int64_t e = 0; e < D; ++e) acc += kv[d * D + e] * dos[e];
            dqs[d] = acc;
        }
    }
    /* sweep 2: reverse, dkv (d x d, rows indexed by q's dim, cols by do's dim) */
    double* dkv = kv;
    memset(dkv, 0, sizeof(double) * (size_t)(D * D));
    for (int64_t s = c->N - 1; s >= 0; --s) {
        const double* qs = ROW(c->q, c, b, s, h);
        const double* ks = ROW(c->k, c, b, s, h);
        const double* vs = ROW(c->v, c, b, s, h);
        const double* dos = ROW(c->dout, c, b, s, h);
        double* dks = ROW(c->dk, c, b, s, h);
        double* dvs = ROW(c->dv, c, b, s, h);
        for (int64_t d = 0; d < D; ++d)
            for (int64_t e = 0; e < D; ++e) dkv[d * D + e] = lam * dkv[d * D + e] + qs[d] * dos[e];
        /* dk_s[d] = sum_e dkv[d][e] v_s[e] */
        for (int64_t d = 0; d < D; ++d) {
            double acc = 0.0;
            for (int64_t e = 0; e < D; ++e) acc += dkv[d * D + e] * vs[e];
            dks[d] = acc;
        }
        /* dv_s[e] = sum_d k_s[d] dkv[d][e] */
        for (int64_t e = 0; e < D; ++e) dvs[e] = 0.0;
        for (int64_t d = 0; d < D; ++d)
            for (int64_t e = 0; e < D; ++e) dvs[e] += ks[d] * dkv[d * D + e];
    }
    free(kv);
}

int oracle_fwd(int64_t B, int64_t N, int64_t H, int64_t D, const double* q, const double* k,
               const double* v, const float* lam, double* o, int nthreads) {
    if (B < 0 || N < 0 || H < 1 || D < 1 || !q || !k || !v || !lam || !o) return ORACLE_ERR_SHAPE;
    int st = check_lams(H, lam);
    if (st) return st;
    rec_ctx_t c = {B, N, H, D, q, k, v, NULL, lam, o, NULL, NULL, NULL};
    run_items(rec_fwd_item, &c, B * H, nthreads);
    return ORACLE_OK;
}

int oracle_bwd(int64_t B, int64_t N, int64_t H, int64_t D, const double* q, const double* k,
               const double* v, const float* lam, const double* dout, double* dq, double* dk,
               double* dv, int nthreads) {
    if (B < 0 || N < 0 || H < 1 || D < 1 || !q || !k || !v || !lam || !dout || !dq || !dk || !dv)
        return ORACLE_ERR_SHAPE;
    int st = check_lams(H, lam);
    if (st) return st;
    rec_ctx_t c = {B, N, H, D, q, k, v, dout, lam, NULL, dq, dk, dv};
    run_items(rec_bwd_item, &c, B * H, nthreads);
    return ORACLE_OK;
}

/* ---------------------------------------------------------------------------------- */
/* Grouped-query / multi-query attention ("multi-query, and    */
/* grouped-query attentions"): H query heads share Hk = H/G key/value heads; q-head h    */
/* reads kv-head h/G. The recurrence Eq. 5 runs once per kv-head (the memory state is   */
/* shared by the group, so its decay lambda is one per kv-head -- DESIGN.md reading G1): */
/*   kv_s = lambda kv_{s-1} + k_s v_s^T,  o_{h,s}^T = q_{h,s}^T kv_s  (h in the group).  */
/* Gradients of L = sum_h sum_s o_{h,s} . do_{h,s}: dq_{h,s} = kv_s do_{h,s}; the       */
/* reverse state collects every head of the group, dkv_s = lambda dkv_{s+1} +            */
/* sum_h q_{h,s} do_{h,s}^T, and dk_s = dkv_s v_s, dv_s = dkv_s^T k_s (Eq. 13-14 with    */
/* the group's sum). Layout: q, o, do, dq [B][N][H][D]; k, v, dk, dv [B][N][Hk][D];     */
/* lam [Hk].                                                                             */
/* ---------------------------------------------------------------------------------- */
typedef struct {
    int64_t B, N, H, Hk, D;
    const double *q, *k, *v, *dout;
    const float* lam;
    double *o, *dq, *dk, *dv;
} gqa_ctx_t;

#define QROW(p, c, b, s, h) ((p) + ((((b) * (c)->N + (s)) * (c)->H + (h)) * (c)->D))
#define KROW(p, c, b, s, h) ((p) + ((((b) * (c)->N + (s)) * (c)->Hk + (h)) * (c)->D))

static void gqa_fwd_item(void* vctx, int64_t item) {
    gqa_ctx_t* c = (gqa_ctx_t*)vctx;
    const int64_t b = item / c->Hk, hk = item % c->Hk, D = c->D, G = c->H / c->Hk;
    const double lam = (double)c->lam[hk];
    double* kv = (double*)calloc((size_t)(D * D), sizeof(double));
    for (int64_t s = 0; s < c->N; ++s) {
        const double* ks = KROW(c->k, c, b, s, hk);
        const double* vs = KROW(c->v, c, b, s, hk);
        for (int64_t d = 0; d < D; ++d)
            for (int64_t e = 0; e < D; ++e) kv[d * D + e] = lam * kv[d * D + e] + ks[d] * vs[e];
        for (int64_t h = hk * G; h < (hk + 1) * G; ++h) {
            const double* qs = QROW(c->q, c, b, s, h);
            double* os = QROW(c->o, c, b, s, h);
            for (int64_t e = 0; e < D; ++e) os[e] = 0.0;
            for (int64_t d = 0; d < D; ++d)
                for (int64_t e = 0; e < D; ++e) os[e] += qs[d] * kv[d * D + e];
        }
    }
    free(kv);
}

static void gqa_bwd_item(void* vctx, int64_t item) {
    gqa_ctx_t* c = (gqa_ctx_t*)vctx;
    const int64_t b = item / c->Hk, hk = item % c->Hk, D = c->D, G = c->H / c->Hk;
    const double lam = (double)c->lam[hk];
    double* kv = (double*)calloc((size_t)(D * D), sizeof(double));
    for (int64_t s = 0; s < c->N; ++s) {          /* sweep 1: kv_s forward, dq_{h,s} = kv_s do_{h,s} */
        const double* ks = KROW(c->k, c, b, s, hk);
        const double* vs = KROW(c->v, c, b, s, hk);
        for (int64_t d = 0; d < D; ++d)
            for (int64_t e = 0; e < D; ++e) kv[d * D + e] = lam * kv[d * D + e] + ks[d] * vs[e];
        for (int64_t h = hk * G; h < (hk + 1) * G; ++h) {
            const double* dos = QROW(c->dout, c, b, s, h);
            double* dqs = QROW(c->dq, c, b, s, h);
            for (int64_t d = 0; d < D; ++d) {
                double acc = 0.0;
                for (int64_t e = 0; e < D; ++e) acc += kv[d * D + e] * dos[e];
                dqs[d] = acc;
            }
        }
    }
    double* dkv = kv;                             /* sweep 2: reverse, the group's shared dkv */
    memset(dkv, 0, sizeof(double) * (size_t)(D * D));
    for (int64_t s = c->N - 1; s >= 0; --s) {
        const double* ks = KROW(c->k, c, b, s, hk);
        const double* vs = KROW(c->v, c, b, s, hk);
        double* dks = KROW(c->dk, c, b, s, hk);
        double* dvs = KROW(c->dv, c, b, s, hk);
        for (int64_t d = 0; d < D; ++d)
            for (int64_t e = 0; e < D; ++e) dkv[d * D + e] = lam * dkv[d * D + e];
        for (int64_t h = hk * G; h < (hk + 1) * G; ++h) {
            const double* qs = QROW(c->q, c, b, s, h);
            const double* dos = QROW(c->dout, c, b, s, h);
            for (int64_t d = 0; d < D; ++d)
                for (int64_t e = 0; e < D; ++e) dkv[d * D + e] += qs[d] * dos[e];
        }
        for (int64_t d = 0; d < D; ++d) {
            double acc = 0.0;
            for (int64_t e = 0; e < D; ++e) acc += dkv[d * D + e] * vs[e];
            dks[d] = acc;
        }
        for (int64_t e = 0; e < D; ++e) dvs[e] = 0.0;
        for (int64_t d = 0; d < D; ++d)
            for (int64_t e = 0; e < D; ++e) dvs[e] += ks[d] * dkv[d * D + e];
    }
    free(kv);
}

int oracle_fwd_gqa(int64_t B, int64_t N, int64_t H, int64_t Hk, int64_t D, const double* q, const double* k,
                   const double* v, const float* lam, double* o, int nthreads) {
    if (B < 0 || N < 0 || H < 1 || Hk < 1 || H % Hk != 0 || D < 1 || !q || !k || !v || !lam || !o)
        return ORACLE_ERR_SHAPE;
    int st = check_lams(Hk, lam);
    if (st) return st;
    gqa_ctx_t c = {B, N, H, Hk, D, q, k, v, NULL, lam, o, NULL, NULL, NULL};
    run_items(gqa_fwd_item, &c, B * Hk, nthreads);
    return ORACLE_OK;
}

int oracle_bwd_gqa(int64_t B, int64_t N, int64_t H, int64_t Hk, int64_t D, const double* q, const double* k,
                   const double* v, const float* lam, const double* dout, double* dq, double* dk, double* dv,
                   int nthreads) {
    if (B < 0 || N < 0 || H < 1 || Hk < 1 || H % Hk != 0 || D < 1 || !q || !k || !v || !lam || !dout || !dq ||
        !dk || !dv)
        return ORACLE_ERR_SHAPE;
    int st = check_lams(Hk, lam);
    if (st) return st;
    gqa_ctx_t c = {B, N, H, Hk, D, q, k, v, dout, lam, NULL, dq, dk, dv};
    run_items(gqa_bwd_item, &c, B * Hk, nthreads);
    return ORACLE_OK;
}

/* ---------------------------------------------------------------------------------- */
/* Norm(.) of Eq. 2 (the paper omits it from the derivation, and does not   */
/* define it). DESIGN.md reading N1: per-head RMS normalization (TransNormerLLM's        */
/* SRMSNorm applied to each head's d-vector, no learnable gain -- a gain folds into the  */
/* output projection):  y = o * r,  r = (sum_c o_c^2 / D + eps)^(-1/2), per (b, s, h).   */
/* Backward: do = r * (dy - y * (y . dy) / D).                                            */
/* o, y, dy, do: [B][N][H][D]; r: [B][N][H].                                              */
/* ---------------------------------------------------------------------------------- */
int oracle_norm_fwd(int64_t rows, int64_t D, double eps, const double* o, double* y, double* r) {
    if (rows < 0 || D < 1 || !(eps >= 0.0) || !o || !y || !r) return ORACLE_ERR_SHAPE;
    for (int64_t i = 0; i < rows; ++i) {
        const double* oi = o + i * D;
        double ss = 0.0;
        for (int64_t c = 0; c < D; ++c) ss += oi[c] * oi[c];
        const double ri = 1.0 / sqrt(ss / (double)D + eps);
        for (int64_t c = 0; c < D; ++c) y[i * D + c] = oi[c] * ri;
        r[i] = ri;
    }
    return ORACLE_OK;
}

int oracle_norm_bwd(int64_t rows, int64_t D, const double* y, const double* r, const double* dy, double* dout) {
    if (rows < 0 || D < 1 || !y || !r || !dy || !dout) return ORACLE_ERR_SHAPE;
    for (int64_t i = 0; i < rows; ++i) {
        const double* yi = y + i * D;
        const double* gi = dy + i * D;
        double dot = 0.0;
        for (int64_t c = 0; c < D; ++c) dot += yi[c] * gi[c];
        for (int64_t c = 0; c < D; ++c) dout[i * D + c] = r[i] * (gi[c] - yi[c] * dot / (double)D);
    }
    return ORACLE_OK;
}

/* ---------------------------------------------------------------------------------- */
/* Chunk operations of Alg. 2 / Alg. 3, one head, C x D row-major matrices.              */
/* ---------------------------------------------------------------------------------- */

/* Alg. 2 lines "Initialize mask M" and "Initialize Lambda", plus the
 * diagonal of lambda^C Lambda^-1 used in Eq. 12 written as lambda^(C-1-i):
 *   mask[i*C+j] = lambda^(i-j) for i >= j else 0;  lam_fwd[i] = lambda^(i+1);
 *   lam_rev[i] = lambda^(C-1-i);  *lam_C = lambda^C.  Powers by repeated multiplication. */
int oracle_build_decay(int64_t C, float lambda_f, double* mask, double* lam_fwd, double* lam_rev,
                       double* lam_C) {
    const double lam = (double)lambda_f;
    if (C < 1) return ORACLE_ERR_DOMAIN;
    if (!(lam > 0.0 && lam <= 1.0)) return ORACLE_ERR_DOMAIN;
    double* pw = (double*)malloc(sizeof(double) * (size_t)(C + 1));
    pw[0] = 1.0;
    for (int64_t i = 1; i <= C; ++i) pw[i] = pw[i - 1] * lam;
    if (mask)
        for (int64_t i = 0; i < C; ++i)
            for (int64_t j = 0; j < C; ++j) mask[i * C + j] = (i >= j) ? pw[i - j] : 0.0;
    if (lam_fwd)
        for (int64_t i = 0; i < C; ++i) lam_fwd[i] = pw[i + 1];
    if (lam_rev)
        for (int64_t i = 0; i < C; ++i) lam_rev[i] = pw[C - 1 - i];
    if (lam_C) *lam_C = pw[C];
    free(pw);
    return ORACLE_OK;
}

/* Eq. 7: O_intra = [(Q K^T) (.) M] V. */
void oracle_intra_fwd(int64_t C, int64_t D, const double* Q, const double* K, const double* V,
                      const double* mask, double* out) {
    double* A = (double*)malloc(sizeof(double) * (size_t)(C * C));
    for (int64_t i = 0; i < C; ++i)
        for (int64_t j = 0; j < C; ++j) {
            double s = 0.0;
            for (int64_t d = 0; d < D; ++d) s += Q[i * D + d] * K[j * D + d];
            A[i * C + j] = s * mask[i * C + j];
        }
    for (int64_t i = 0; i < C; ++i)
        for (int64_t e = 0; e < D; ++e) {
            double s = 0.0;
            for (int64_t j = 0; j < C; ++j) s += A[i * C + j] * V[j * D + e];
            out[i * D + e] = s;
        }
    free(A);
}

/* Eq. 9 read as Alg. 2 P:169 (reading A1): O_inter = Lambda Q KV_{t-1}. */
void oracle_inter_fwd(int64_t C, int64_t D, const double* Q, const double* kv_prev,
                      const double* lam_fwd, double* out) {
    for (int64_t i = 0; i < C; ++i)
        for (int64_t e = 0; e < D; ++e) {
            double s = 0.0;
            for (int64_t d = 0; d < D; ++d) s += Q[i * D + d] * kv_prev[d * D + e];
            out[i * D + e] = lam_fwd[i] * s;
        }
}

/* Eq. 12: KV_t = lambda^C KV_{t-1} + (lambda^C Lambda^-1 K_t)^T V_t. */
void oracle_kv_update(int64_t C, int64_t D, const double* kv_prev, const double* K, const double* V,
                      const double* lam_rev, double lam_C, double* kv_out) {
    for (int64_t d = 0; d < D; ++d)
        for (int64_t e = 0; e < D; ++e) {
            double s = 0.0;
            for (int64_t i = 0; i < C; ++i) s += lam_rev[i] * K[i * D + d] * V[i * D + e];
            kv_out[d * D + e] = lam_C * (kv_prev ? kv_prev[d * D + e] : 0.0) + s;
        }
}

/* Alg. 3 loop 1, Eq. 15, 18 and the dV_intra line:
 * dQ_intra = [(dO V^T) (.) M] K;  dK_intra = [(dO V^T) (.) M]^T Q;
 * dV_intra = [(Q K^T) (.) M]^T dO. */
void oracle_intra_bwd(int64_t C, int64_t D, const double* Q, const double* K, const double* V,
                      const double* dO, const double* mask, double* dQ, double* dK, double* dV) {
    double* A = (double*)malloc(sizeof(double) * (size_t)(C * C)); /* (dO V^T) (.) M */
    double* S = (double*)malloc(sizeof(double) * (size_t)(C * C)); /* (Q K^T) (.) M */
    for (int64_t i = 0; i < C; ++i)
        for (int64_t j = 0; j < C; ++j) {
            double a = 0.0, s = 0.0;
            for (int64_t d = 0; d < D; ++d) {
                a += dO[i * D + d] * V[j * D + d];
                s += Q[i * D + d] * K[j * D + d];
            }
            A[i * C + j] = a * mask[i * C + j];
            S[i * C + j] = s * mask[i * C + j];
        }
    for (int64_t i = 0; i < C; ++i)
        for (int64_t d = 0; d < D; ++d) {
            double sq = 0.0, sk = 0.0, sv = 0.0;
            for (int64_t j = 0; j < C; ++j) {
                sq += A[i * C + j] * K[j * D + d];
                sk += A[j * C + i] * Q[j * D + d];
                sv += S[j * C + i] * dO[j * D + d];
            }
            dQ[i * D + d] = sq;
            dK[i * D + d] = sk;
            dV[i * D + d] = sv;
        }
    free(A);
    free(S);
}

/* Eq. 17: dQ_inter = Lambda dO KV_{t-1}^T (KV_{t-1} from the forward cache). */
void oracle_inter_bwd_q(int64_t C, int64_t D, const double* dO, const double* kv_prev,
                        const double* lam_fwd, double* out) {
    for (int64_t i = 0; i < C; ++i)
        for (int64_t d = 0; d < D; ++d) {
            double s = 0.0;
            for (int64_t e = 0; e < D; ++e) s += dO[i * D + e] * kv_prev[d * D + e];
            out[i * D + d] = lam_fwd[i] * s;
        }
}

/* Eq. 20: dK_inter = lambda^C Lambda^-1 V dKV_{t+1}^T. */
void oracle_inter_bwd_k(int64_t C, int64_t D, const double* V, const double* dkv_next,
                        const double* lam_rev, double* out) {
    for (int64_t i = 0; i < C; ++i)
        for (int64_t d = 0; d < D; ++d) {
            double s = 0.0;
            for (int64_t e = 0; e < D; ++e) s += V[i * D + e] * dkv_next[d * D + e];
            out[i * D + d] = lam_rev[i] * s;
        }
}

/* Eq. 22: dV_inter = lambda^C Lambda^-1 K dKV_{t+1}. */
void oracle_inter_bwd_v(int64_t C, int64_t D, const double* K, const double* dkv_next,
                        const double* lam_rev, double* out) {
    for (int64_t i = 0; i < C; ++i)
        for (int64_t e = 0; e < D; ++e) {
            double s = 0.0;
            for (int64_t d = 0; d < D; ++d) s += K[i * D + d] * dkv_next[d * D + e];
            out[i * D + e] = lam_rev[i] * s;
        }
}

/* Eq. 21 with the indices of Alg. 3 P:648 (reading A3):
 * dKV_t = lambda^C dKV_{t+1} + (Lambda Q_t)^T dO_t. */
void oracle_dkv_update(int64_t C, int64_t D, const double* dkv_next, const double* Q,
                       const double* dO, const double* lam_fwd, double lam_C, double* dkv_out) {
    for (int64_t d = 0; d < D; ++d)
        for (int64_t e = 0; e < D; ++e) {
            double s = 0.0;
            for (int64_t i = 0; i < C; ++i) s += lam_fwd[i] * Q[i * D + d] * dO[i * D + e];
            dkv_out[d * D + e] = lam_C * (dkv_next ? dkv_next[d * D + e] : 0.0) + s;
        }
}

/* ---------------------------------------------------------------------------------- */
/* Rank-simulated mode: Alg. 2 and Alg. 3 run literally with T   */
/* ranks, explicit message buffers (one d x d state per head per hop) and a KV cache     */
/* holding the state ENTERING each rank (reading A4).                                    */
/* ---------------------------------------------------------------------------------- */
typedef struct {
    int64_t B, N, H, D, T;
    const double *q, *k, *v, *dout;
    const float* lam;
    double *o, *dq, *dk, *dv;
    double* cache; /* [T][B][H][D][D] */
    int64_t msgs, msg_elems; /* per-head counts, summed by the caller */
} sim_ctx_t;

static void gather_chunk(const sim_ctx_t* c, const double* src, int64_t b, int64_t h, int64_t t,
                         double* dst) {
    const int64_t C = c->N / c->T, D = c->D;
    for (int64_t s = 0; s < C; ++s)
        memcpy(dst + s * D, src + (((b * c->N) + t * C + s) * c->H + h) * D, sizeof(double) * (size_t)D);
}
static void scatter_chunk(const sim_ctx_t* c, double* dst, int64_t b, int64_t h, int64_t t,
                          const double* src) {
    const int64_t C = c->N / c->T, D = c->D;
    for (int64_t s = 0; s < C; ++s)
        memcpy(dst + (((b * c->N) + t * C + s) * c->H + h) * D, src + s * D, sizeof(double) * (size_t)D);
}

static void sim_fwd_item(void* vctx, int64_t item) {
    sim_ctx_t* c = (sim_ctx_t*)vctx;
    const int64_t b = item / c->H, h = item % c->H, D = c->D, T = c->T, C = c->N / T;
    const size_t CD = (size_t)(C * D), DD = (size_t)(D * D);
    double *mask = malloc(sizeof(double) * (size_t)(C * C)), *lf = malloc(sizeof(double) * (size_t)C),
           *lr = malloc(sizeof(double) * (size_t)C), lC;
    oracle_build_decay(C, c->lam[h], mask, lf, lr, &lC);
    double *Q = malloc(sizeof(double) * CD), *K = malloc(sizeof(double) * CD),
           *V = malloc(sizeof(double) * CD), *Oin = malloc(sizeof(double) * CD * (size_t)T),
           *Oint = malloc(sizeof(double) * CD);
    double* mailbox = calloc(DD * (size_t)(T + 1), sizeof(double)); /* mailbox[t] = KV sent to rank t */
    /* loop 1, "in parallel" over ranks: O_intra (Alg. 2) */
    for (int64_t t = 0; t < T; ++t) {
        gather_chunk(c, c->q, b, h, t, Q);
        gather_chunk(c, c->k, b, h, t, K);
        gather_chunk(c, c->v, b, h, t, V);
        oracle_intra_fwd(C, D, Q, K, V, mask, Oin + (size_t)t * CD);
    }
    /* loop 2, sequential ring */
    int64_t msgs = 0;
    for (int64_t t = 0; t < T; ++t) {
        const double* kv_prev = mailbox + (size_t)t * DD;             /* Recv from t-1 (t=0: 0) */
        memcpy(c->cache + ((t * c->B + b) * c->H + h) * DD, kv_prev, sizeof(double) * DD); /* Save */
        gather_chunk(c, c->q, b, h, t, Q);
        gather_chunk(c, c->k, b, h, t, K);
        gather_chunk(c, c->v, b, h, t, V);
        oracle_inter_fwd(C, D, Q, kv_prev, lf, Oint);
        for (size_t i = 0; i < CD; ++i) Oint[i] += Oin[(size_t)t * CD + i];
        scatter_chunk(c, c->o, b, h, t, Oint);
        double* kv_next = mailbox + (size_t)(t + 1) * DD;
        oracle_kv_update(C, D, kv_prev, K, V, lr, lC, kv_next);
        if (t < T - 1) msgs++;                                       /* Send to t+1 */
    }
    c->msgs = msgs; /* identical for every item; D*D elements each */
    c->msg_elems = (int64_t)DD;
    free(mask); free(lf); free(lr); free(Q); free(K); free(V); free(Oin); free(Oint); free(mailbox);
}

static void sim_bwd_item(void* vctx, int64_t item) {
    sim_ctx_t* c = (sim_ctx_t*)vctx;
    const int64_t b = item / c->H, h = item % c->H, D = c->D, T = c->T, C = c->N / T;
    const size_t CD = (size_t)(C * D), DD = (size_t)(D * D);
    double *mask = malloc(sizeof(double) * (size_t)(C * C)), *lf = malloc(sizeof(double) * (size_t)C),
           *lr = malloc(sizeof(double) * (size_t)C), lC;
    oracle_build_decay(C, c->lam[h], mask, lf, lr, &lC);
    double *Q = malloc(sizeof(double) * CD), *K = malloc(sizeof(double) * CD),
           *V = malloc(sizeof(double) * CD), *dO = malloc(sizeof(double) * CD);
    double *dQ = malloc(sizeof(double) * CD * (size_t)T), *dK = malloc(sizeof(double) * CD * (size_t)T),
           *dV = malloc(sizeof(double) * CD * (size_t)T), *tmp = malloc(sizeof(double) * CD);
    double* mailbox = calloc(DD * (size_t)(T + 1), sizeof(double)); /* mailbox[t+1] = dKV_{t+1} */
    /* loop 1, in parallel */
    for (int64_t t = 0; t < T; ++t) {
        gather_chunk(c, c->q, b, h, t, Q);
        gather_chunk(c, c->k, b, h, t, K);
        gather_chunk(c, c->v, b, h, t, V);
        gather_chunk(c, c->dout, b, h, t, dO);
        oracle_intra_bwd(C, D, Q, K, V, dO, mask, dQ + (size_t)t * CD, dK + (size_t)t * CD,
                         dV + (size_t)t * CD);
        const double* kv_prev = c->cache + ((t * c->B + b) * c->H + h) * DD; /* cached KV_{t-1} */
        oracle_inter_bwd_q(C, D, dO, kv_prev, lf, tmp);                     /* P:607, Eq. 17 */
        for (size_t i = 0; i < CD; ++i) dQ[(size_t)t * CD + i] += tmp[i];
    }
    /* loop 2, reverse ring (send target read as rank i-1, reading A2) */
    int64_t msgs = 0;
    for (int64_t t = T - 1; t >= 0; --t) {
        const double* dkv_next = mailbox + (size_t)(t + 1) * DD; /* Recv from t+1 (last: 0) */
        gather_chunk(c, c->q, b, h, t, Q);
        gather_chunk(c, c->k, b, h, t, K);
        gather_chunk(c, c->v, b, h, t, V);
        gather_chunk(c, c->dout, b, h, t, dO);
        oracle_inter_bwd_k(C, D, V, dkv_next, lr, tmp);
        for (size_t i = 0; i < CD; ++i) dK[(size_t)t * CD + i] += tmp[i];
        oracle_inter_bwd_v(C, D, K, dkv_next, lr, tmp);
        for (size_t i = 0; i < CD; ++i) dV[(size_t)t * CD + i] += tmp[i];
        scatter_chunk(c, c->dq, b, h, t, dQ + (size_t)t * CD);
        scatter_chunk(c, c->dk, b, h, t, dK + (size_t)t * CD);
        scatter_chunk(c, c->dv, b, h, t, dV + (size_t)t * CD);
        oracle_dkv_update(C, D, dkv_next, Q, dO, lf, lC, mailbox + (size_t)t * DD);
        if (t > 0) msgs++;                                                       /* Send to t-1 */
    }
    c->msgs = msgs;
    c->msg_elems = (int64_t)DD;
    free(mask); free(lf); free(lr); free(Q); free(K); free(V); free(dO);
    free(dQ); free(dK); free(dV); free(tmp); free(mailbox);
}

/* The item function writes per-item counters into a private copy of the context so that
 * items can run concurrently; these wrappers give each item its own ctx. */
typedef struct { sim_ctx_t base; int bwd; int64_t* msgs; } sim_outer_t;
static void sim_item(void* vctx, int64_t item) {
    sim_outer_t* so = (sim_outer_t*)vctx;
    sim_ctx_t local = so->base;
    if (so->bwd) sim_bwd_item(&local, item); else sim_fwd_item(&local, item);
    so->msgs[item] = local.msgs;
}

/* Alg. 2 with T simulated ranks. cache: [T][B][H][D][D] (state entering each rank).
 * msg_count / msg_elems (nullable): messages sent per direction and elements per message
 * summed over (b, h) -- one hop carries B*H*D*D elements (Table 1 LASP row). */
int oracle_lasp_fwd_sim(int64_t B, int64_t N, int64_t H, int64_t D, int64_t T, const double* q,
                        const double* k, const double* v, const float* lam, double* o, double* cache,
                        int64_t* msg_count, int64_t* msg_elems, int nthreads) {
    if (B < 0 || N < 0 || H < 1 || D < 1 || T < 1 || !q || !k || !v || !lam || !o || !cache)
        return ORACLE_ERR_SHAPE;
    if (N % T != 0 || N / T < 1) return ORACLE_ERR_PARTITION; /* C = N/T exactly */
    int st = check_lams(H, lam);
    if (st) return st;
    int64_t* m = calloc((size_t)(B * H > 0 ? B * H : 1), sizeof(int64_t));
    sim_outer_t so = {{B, N, H, D, T, q, k, v, NULL, lam, o, NULL, NULL, NULL, cache, 0, 0}, 0, m};
    run_items(sim_item, &so, B * H, nthreads);
    if (msg_count) *msg_count = (B * H > 0) ? m[0] : 0; /* hops per direction */
    if (msg_elems) *msg_elems = B * H * D * D;          /* elements per hop, all heads */
    free(m);
    return ORACLE_OK;
}

/* Alg. 3 with T simulated ranks, consuming the cache written by oracle_lasp_fwd_sim. */
int oracle_lasp_bwd_sim(int64_t B, int64_t N, int64_t H, int64_t D, int64_t T, const double* q,
                        const double* k, const double* v, const float* lam, const double* dout,
                        const double* cache, double* dq, double* dk, double* dv, int64_t* msg_count,
                        int64_t* msg_elems, int nthreads) {
    if (B < 0 || N < 0 || H < 1 || D < 1 || T < 1 || !q || !k || !v || !lam || !dout || !cache ||
        !dq || !dk || !dv)
        return ORACLE_ERR_SHAPE;
    if (N % T != 0 || N / T < 1) return ORACLE_ERR_PARTITION;
    int st = check_lams(H, lam);
    if (st) return st;
    int64_t* m = calloc((size_t)(B * H > 0 ? B * H : 1), sizeof(int64_t));
    sim_outer_t so = {{B, N, H, D, T, q, k, v, dout, lam, NULL, dq, dk, dv, (double*)cache, 0, 0}, 1, m};
    run_items(sim_item, &so, B * H, nthreads);
    if (msg_count) *msg_count = (B * H > 0) ? m[0] : 0;
    if (msg_elems) *msg_elems = B * H * D * D;
    free(m);
    return ORACLE_OK;
}

/* ---------------------------------------------------------------------------------- */
/* Generalised decay: the GLA / GateLoop row of Table 3 (App. A.4,   */
/* P:671-713 general form m_t = o_t m_{t-1} + e_t i_t^T; GLA/GateLoop P:735):              */
/*   kv_t = Diag(g_t) kv_{t-1} + k_t v_t^T,  o_t^T = q_t^T kv_t,  g_t = exp(lg_t) in (0,1]^D  */
/* per token and key channel (data-dependent decay; a per-channel constant decay is        */
/* lg_t = log lambda for every t). Definition mode: the recurrence, token by token.          */
/* Backward of L = sum(O * dO): dkv_t = q_t do_t^T + Diag(g_{t+1}) dkv_{t+1} (dkv_N = 0),    */
/* dq_t = kv_t do_t, dk_t = dkv_t v_t, dv_t = dkv_t^T k_t, and the decay gradient from its    */
/* definition dL/dlg_t[d] = g_t[d] sum_e dkv_t[d][e] kv_{t-1}[d][e] (kv_{-1} = 0). The        */
/* reverse sweep needs kv_{t-1}: the forward states are recomputed per 64-token chunk from   */
/* checkpoints (kv entering each chunk), nothing is divided by a decay.                      */
/* ---------------------------------------------------------------------------------- */
typedef struct {
    int64_t B, N, H, D;
    const double *q, *k, *v, *lg, *dout;
    double *o, *dq, *dk, *dv, *dlg;
} gla_ctx_t;

#define GROW(p, c, b, s, h) ((p) + ((((b) * (c)->N + (s)) * (c)->H + (h)) * (c)->D))

/* kv <- Diag(exp(lg_s)) kv + k_s v_s^T */
static void gla_step(int64_t D, double* kv, const double* lgs, const double* ks, const double* vs) {
    for (int64_t d = 0; d < D; ++d) {
        const double g = exp(lgs[d]);
        for (int64_t e = 0; e < D; ++e) kv[d * D + e] = g * kv[d * D + e] + ks[d] * vs[e];
    }
}

static void gla_fwd_item(void* vctx, int64_t item) {
    gla_ctx_t* c = (gla_ctx_t*)vctx;
    const int64_t b = item / c->H, h = item % c->H, D = c->D;
    double* kv = (double*)calloc((size_t)(D * D), sizeof(double));
    for (int64_t s = 0; s < c->N; ++s) {
        gla_step(D, kv, GROW(c->lg, c, b, s, h), GROW(c->k, c, b, s, h), GROW(c->v, c, b, s, h));
        const double* qs = GROW(c->q, c, b, s, h);
        double* os = GROW(c->o, c, b, s, h);
        for (int64_t e = 0; e < D; ++e) os[e] = 0.0;
        for (int64_t d = 0; d < D; ++d)
            for (int64_t e = 0; e < D; ++e) os[e] += qs[d] * kv[d * D + e];
    }
    free(kv);
}

#define GLA_CK 64
static void gla_bwd_item(void* vctx, int64_t item) {
    gla_ctx_t* c = (gla_ctx_t*)vctx;
    const int64_t b = item / c->H, h = item % c->H, D = c->D, N = c->N, DD = D * D;
    const int64_t nck = (N + GLA_CK - 1) / GLA_CK;
    double* ck = (double*)calloc((size_t)((nck > 0 ? nck : 1) * DD), sizeof(double)); /* kv entering chunk j */
    double* st = (double*)malloc(sizeof(double) * (size_t)((GLA_CK + 1) * DD));       /* kv_{t-1}, kv_t, ... */
    double* kv = (double*)calloc((size_t)DD, sizeof(double));
    double* dkv = (double*)calloc((size_t)DD, sizeof(double));
    for (int64_t s = 0; s < N; ++s) {
        if (s % GLA_CK == 0) memcpy(ck + (s / GLA_CK) * DD, kv, sizeof(double) * (size_t)DD);
        gla_step(D, kv, GROW(c->lg, c, b, s, h), GROW(c->k, c, b, s, h), GROW(c->v, c, b, s, h));
    }
    for (int64_t j = nck - 1; j >= 0; --j) {
        const int64_t s0 = j * GLA_CK, s1 = (s0 + GLA_CK < N) ? s0 + GLA_CK : N;
        /* st[i] = kv_{s0 + i - 1} for i = 0 .. s1 - s0 */
        memcpy(st, ck + j * DD, sizeof(double) * (size_t)DD);
        for (int64_t s = s0; s < s1; ++s) {
            memcpy(st + (s - s0 + 1) * DD, st + (s - s0) * DD, sizeof(double) * (size_t)DD);
            gla_step(D, st + (s - s0 + 1) * DD, GROW(c->lg, c, b, s, h), GROW(c->k, c, b, s, h),
                     GROW(c->v, c, b, s, h));
        }
        for (int64_t s = s1 - 1; s >= s0; --s) {
            const double* qs = GROW(c->q, c, b, s, h);
            const double* ks = GROW(c->k, c, b, s, h);
            const double* vs = GROW(c->v, c, b, s, h);
            const double* dos = GROW(c->dout, c, b, s, h);
            const double* kvs = st + (s - s0 + 1) * DD;  /* kv_s */
            const double* kvp = st + (s - s0) * DD;      /* kv_{s-1} */
            /* dkv_s = q_s do_s^T + Diag(g_{s+1}) dkv_{s+1} */
            if (s + 1 < N) {
                const double* lgn = GROW(c->lg, c, b, s + 1, h);
                for (int64_t d = 0; d < D; ++d) {
                    const double g = exp(lgn[d]);
                    for (int64_t e = 0; e < D; ++e) dkv[d * D + e] *= g;
                }
            }
            for (int64_t d = 0; d < D; ++d)
                for (int64_t e = 0; e < D; ++e) dkv[d * D + e] += qs[d] * dos[e];
            double* dqs = GROW(c->dq, c, b, s, h);
            double* dks = GROW(c->dk, c, b, s, h);
            double* dvs = GROW(c->dv, c, b, s, h);
            double* dls = GROW(c->dlg, c, b, s, h);
            const double* lgs = GROW(c->lg, c, b, s, h);
            for (int64_t d = 0; d < D; ++d) {
                double aq = 0.0, ak = 0.0, al = 0.0;
                for (int64_t e = 0; e < D; ++e) {
                    aq += kvs[d * D + e] * dos[e];
                    ak += dkv[d * D + e] * vs[e];
                    al += dkv[d * D + e] * kvp[d * D + e];
                }
                dqs[d] = aq;
                dks[d] = ak;
                dls[d] = exp(lgs[d]) * al;
            }
            for (int64_t e = 0; e < D; ++e) {
                double av = 0.0;
                for (int64_t d = 0; d < D; ++d) av += dkv[d * D + e] * ks[d];
                dvs[e] = av;
            }
        }
    }
    free(ck); free(st); free(kv); free(dkv);
}

static int check_lg(int64_t n, const double* lg) {
    for (int64_t i = 0; i < n; ++i)
        if (!(lg[i] <= 0.0)) return ORACLE_ERR_DOMAIN; /* g = exp(lg) in (0, 1] */
    return ORACLE_OK;
}

int oracle_gla_fwd(int64_t B, int64_t N, int64_t H, int64_t D, const double* q, const double* k, const double* v,
                   const double* lg, double* o, int nthreads) {
    if (B < 0 || N < 0 || H < 1 || D < 1) return ORACLE_ERR_SHAPE;
    int st = check_lg(B * N * H * D, lg);
    if (st) return st;
    gla_ctx_t c = {B, N, H, D, q, k, v, lg, NULL, o, NULL, NULL, NULL, NULL};
    run_items(gla_fwd_item, &c, B * H, nthreads);
    return ORACLE_OK;
}

int oracle_gla_bwd(int64_t B, int64_t N, int64_t H, int64_t D, const double* q, const double* k, const double* v,
                   const double* lg, const double* dout, double* dq, double* dk, double* dv, double* dlg,
                   int nthreads) {
    if (B < 0 || N < 0 || H < 1 || D < 1) return ORACLE_ERR_SHAPE;
    int st = check_lg(B * N * H * D, lg);
    if (st) return st;
    gla_ctx_t c = {B, N, H, D, q, k, v, lg, dout, NULL, dq, dk, dv, dlg};
    run_items(gla_bwd_item, &c, B * H, nthreads);
    return ORACLE_OK;
}
