/*
 * vista_oracle.c -- float64 CPU oracle for VISTA stage-1 user-history summarization.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * `--impl reference` leg may load this library.  The product path (paper_2510_22049_b200) never
 * links, imports or executes it, and shares no source with it.
 *
 * What it computes (PAPER.md = /root/reference/PAPER.md, the VISTA paper, arXiv 2510.22049):
 *
 *  Softmax summarization -- the seed rows of self-attention over the user history.
 *    SoftmaxAttn(S =>full S) = RowSoftmax(Q K^T) V        (Sec. 3.2.1)
 *    with the queries being the k virtual seeds, "initialized randomly as shared parameters
 *    across users" (Sec. 3.2) and the keys/values the user's history items.
 *    Per user u, head h, seed row i, over keys j in [off_u, off_{u+1}):
 *      s_j = scale * sum_c q_{i,h,c} k_{j,h,c};  m = max_j s_j;  l = sum_j e^{s_j - m}
 *      o_{i,h,:} = sum_j e^{s_j - m} v_{j,h,:} / l;   lse_{h,i} = m + ln l
 *    Empty history: o = 0, lse = -inf (reading R6).  Two passes, sequential sums.
 *
 *  Quasi-linear attention (QLA), source part (Sec. 3.2.2; two-activation form
 *  PAPER.md:831-836, App. B.2):
 *      O[S] = phi1(Q[S]) phi2( phi1(K[S])^T V[S] )
 *    evaluated at the seed-row queries:  Z = sum_j phi1(k_j)^T v_j  (d x d),
 *    Zbar = Z / N_u when normalizing (the "1/N factor", App. B; N_u = L_u,
 *    DESIGN.md reading R10), O = phi1(Q) phi2(Zbar).
 *    phi: identity, SiLU ("we use SiLU"), shifted ELU (App. B.1.5:
 *    phi(x) = x if x >= 1 else e^{x-1}).
 *
 *  Merges used only to test split invariants: LSE merge of softmax partials and plain sum of
 *  QLA states.
 *
 *  NEXT-3 / NEXT-4: QLA at arbitrary per-user query rows (history rows of a deeper layer, or
 *  target rows with the Delta self term), vo_qla_rows.
 *
 *  NEXT-3: the multi-layer summarizer (projections, QLA over [seeds; history], SGLU gate, output
 *  projection, residual), vo_summarize_layers.
 *
 *  NEXT-4: stage-2 target-aware attention of candidates over the cached (int8-exported) summary
 *  tokens, vo_target_attend.
 *
 *  NEXT-2 (training): the QLA backward (vo_qla_backward) by the chain rule through
 *  O = phi1(Q) phi2(Z / N), Z = phi1(K)^T V.
 *
 * Inputs are float32 arrays whose values are exact (bf16 / f32 grid values from synth/); every
 * element is converted exactly to double and all arithmetic is double.  No blocking, no
 * reordering beyond the definitions above.  Compile: gcc -O2 -fopenmp (no -ffast-math).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define VO_ACT_IDENTITY 0
#define VO_ACT_SILU 1
#define VO_ACT_SHIFTED_ELU 2

/* phi, PAPER.md:795-800 (shifted ELU, "x >= 1" takes the x branch) and PAPER.md:219 (SiLU). */
double vo_act(int kind, double x) {
    switch (kind) {
        case VO_ACT_IDENTITY: return x;
        case VO_ACT_SILU: return x / (1.0 + exp(-x));
        case VO_ACT_SHIFTED_ELU: return x >= 1.0 ? x : exp(x - 1.0);
        default: return NAN;
    }
}

int vo_num_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

static void set_threads(int threads) {
#ifdef _OPENMP
    if (threads > 0) omp_set_num_threads(threads);
#else
    (void)threads;
#endif
}

/*
 * Softmax summarization for the query rows rows[0..n_rows) of every (user, head).
 *   q:   [S, H, d] when q_user_stride == 0 (shared seeds), else user u's block starts at
 *        q + u * q_user_stride (elements) and is laid out [S, H, d].
 *   k,v: [total_len, H, d];  offsets: [B+1] (offsets[0] = 0, non-decreasing).
 *   out: [B, n_rows, H, d];  lse: [B, H, n_rows].
 * Returns 0, or -1 on bad arguments / allocation failure.
 */
int vo_softmax(int64_t B, int64_t S, int64_t H, int64_t d, const float* q, int64_t q_user_stride,
               const float* k, const float* v, const int64_t* offsets, double scale,
               const int64_t* rows, int64_t n_rows, double* out, double* lse, int threads) {
    if (B < 0 || S < 1 || H < 1 || d < 1 || n_rows < 0) return -1;
    for (int64_t r = 0; r < n_rows; ++r)
        if (rows[r] < 0 || rows[r] >= S) return -1;
    set_threads(threads);
    int err = 0;
    const int64_t total = B * H * n_rows;
#pragma omp parallel
    {
        double* s = NULL;
        int64_t cap = 0;
#pragma omp for schedule(dynamic, 1)
        for (int64_t t = 0; t < total; ++t) {
            const int64_t u = t / (H * n_rows);
            const int64_t h = (t / n_rows) % H;
            const int64_t r = t % n_rows;
            const int64_t i = rows[r];
            const int64_t j0 = offsets[u], L = offsets[u + 1] - offsets[u];
            const float* qi = q + u * q_user_stride + (i * H + h) * d;
            double* o = out + ((u * n_rows + r) * H + h) * d;
            double* ls = lse + (u * H + h) * n_rows + r;
            if (L <= 0) {
                for (int64_t c = 0; c < d; ++c) o[c] = 0.0;
                *ls = -INFINITY;
                continue;
            }
            if (L > cap) {
                free(s);
                s = (double*)malloc((size_t)L * sizeof(double));
                cap = s ? L : 0;
                if (!s) {
#pragma omp atomic write
                    err = 1;
                    continue;
                }
            }
            /* pass 1: scores and their maximum */
            double m = -INFINITY;
            for (int64_t j = 0; j < L; ++j) {
                const float* kj = k + ((j0 + j) * H + h) * d;
                double acc = 0.0;
                for (int64_t c = 0; c < d; ++c) acc += (double)qi[c] * (double)kj[c];
                s[j] = scale * acc;
                if (s[j] > m) m = s[j];
            }
            /* pass 2: weights, their sum, weighted values */
            double l = 0.0;
            for (int64_t c = 0; c < d; ++c) o[c] = 0.0;
            for (int64_t j = 0; j < L; ++j) {
                const double p = exp(s[j] - m);
                const float* vj = v + ((j0 + j) * H + h) * d;
                l += p;
                for (int64_t c = 0; c < d; ++c) o[c] += p * (double)vj[c];
            }
            for (int64_t c = 0; c < d; ++c) o[c] /= l;
            *ls = m + log(l);
        }
        free(s);
    }
    return err ? -1 : 0;
}

/*
 * QLA state of every (user, head):  z[u,h,c1,c2] = sum_j phi1(k_{j,h,c1}) v_{j,h,c2}
 * ("phi(K[S])^T V[S]"; App. B "sum_j K[S]_j^T V[S]_j ... computed first",
 * PAPER.md:680).  z: [B, H, d, d].
 */
int vo_qla_state(int64_t B, int64_t H, int64_t d, const float* k, const float* v,
                 const int64_t* offsets, int phi1, double* z, int threads) {
    if (B < 0 || H < 1 || d < 1) return -1;
    set_threads(threads);
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t t = 0; t < B * H; ++t) {
        const int64_t u = t / H, h = t % H;
        double* zu = z + t * d * d;
        for (int64_t e = 0; e < d * d; ++e) zu[e] = 0.0;
        for (int64_t j = offsets[u]; j < offsets[u + 1]; ++j) {
            const float* kj = k + (j * H + h) * d;
            const float* vj = v + (j * H + h) * d;
            for (int64_t c1 = 0; c1 < d; ++c1) {
                const double a = vo_act(phi1, (double)kj[c1]);
                for (int64_t c2 = 0; c2 < d; ++c2) zu[c1 * d + c2] += a * (double)vj[c2];
            }
        }
    }
    return 0;
}

/*
 * QLA output from a state:  Zbar = Z / N_u (if normalize and N_u > 0; Z itself is 0 when
 * N_u = 0), O[u,i,h,:] = phi1(q_i) phi2(Zbar)   (B.2 PAPER.md:834;
 * 1/N PAPER.md:646-649).  z: [B, H, d, d]; n_items: [B]; out: [B, S, H, d].
 */
int vo_qla_finalize(int64_t B, int64_t S, int64_t H, int64_t d, const float* q,
                    int64_t q_user_stride, const double* z, const int64_t* n_items, int phi1,
                    int phi2, int normalize, double* out, int threads) {
    if (B < 0 || S < 1 || H < 1 || d < 1) return -1;
    set_threads(threads);
#pragma omp parallel
    {
        double* w = (double*)malloc((size_t)(d * d) * sizeof(double));
#pragma omp for schedule(dynamic, 1)
        for (int64_t t = 0; t < B * H; ++t) {
            const int64_t u = t / H, h = t % H;
            const double* zu = z + t * d * d;
            const double inv = (normalize && n_items[u] > 0) ? 1.0 / (double)n_items[u] : 1.0;
            for (int64_t e = 0; e < d * d; ++e) w[e] = vo_act(phi2, zu[e] * inv);
            for (int64_t i = 0; i < S; ++i) {
                const float* qi = q + u * q_user_stride + (i * H + h) * d;
                double* o = out + ((u * S + i) * H + h) * d;
                for (int64_t c2 = 0; c2 < d; ++c2) o[c2] = 0.0;
                for (int64_t c1 = 0; c1 < d; ++c1) {
                    const double a = vo_act(phi1, (double)qi[c1]);
                    for (int64_t c2 = 0; c2 < d; ++c2) o[c2] += a * w[c1 * d + c2];
                }
            }
        }
        free(w);
    }
    return 0;
}

/*
 * QLA at arbitrary per-user query rows (NEXT-3 / NEXT-4):
 *   history rows  O[S] = phi(Q[S]) phi(phi(K[S])^T V[S])
 *   target rows   O[T] = phi(Q[T]) phi(phi(K[S])^T V[S])
 *                        + Delta(phi(Q[T]), phi(K[T])) V[T]
 * with Delta(X, Y)_ij = sum_k X_ik Y_ik delta_ij, i.e. row r gains
 * (phi1(q_r) . phi1(k_self_r)) v_self_r.  Rows r in [row_offsets[u], row_offsets[u+1]) belong to
 * user u and use its state Zbar_u (as in vo_qla_finalize: Z / N_u when normalizing, DESIGN.md
 * reading R10).  When normalizing, the Delta term is divided by the SAME N_u: App. B writes the
 * mixed form as one product under one scalar, O = (Q K^T (.) M) V / N with M = [[1,0],[1,I_m]]
 * (PAPER.md:644-654), so the target's own diagonal term sits under the same /N as its source
 * term (reading R20).  N_u = 0 (no history): no division, as for the state.
 * k_self = v_self = NULL: no Delta term.
 * q_rows, k_self, v_self: [R, H, d]; z: [B, H, d, d]; out: [R, H, d].
 */
int vo_qla_rows(int64_t B, int64_t H, int64_t d, const double* z, const int64_t* n_items,
                const float* q_rows, const int64_t* row_offsets, const float* k_self,
                const float* v_self, int phi1, int phi2, int normalize, double* out, int threads) {
    if (B < 0 || H < 1 || d < 1) return -1;
    set_threads(threads);
#pragma omp parallel
    {
        double* w = (double*)malloc((size_t)(d * d) * sizeof(double));
#pragma omp for schedule(dynamic, 1)
        for (int64_t t = 0; t < B * H; ++t) {
            const int64_t u = t / H, h = t % H;
            const double* zu = z + t * d * d;
            const double inv = (normalize && n_items[u] > 0) ? 1.0 / (double)n_items[u] : 1.0;
            for (int64_t e = 0; e < d * d; ++e) w[e] = vo_act(phi2, zu[e] * inv);
            for (int64_t r = row_offsets[u]; r < row_offsets[u + 1]; ++r) {
                const float* qr = q_rows + (r * H + h) * d;
                double* o = out + (r * H + h) * d;
                for (int64_t c2 = 0; c2 < d; ++c2) o[c2] = 0.0;
                for (int64_t c1 = 0; c1 < d; ++c1) {
                    const double a = vo_act(phi1, (double)qr[c1]);
                    for (int64_t c2 = 0; c2 < d; ++c2) o[c2] += a * w[c1 * d + c2];
                }
                if (k_self) {
                    const float* kr = k_self + (r * H + h) * d;
                    const float* vr = v_self + (r * H + h) * d;
                    double dot = 0.0;
                    for (int64_t c = 0; c < d; ++c) dot += vo_act(phi1, (double)qr[c]) * vo_act(phi1, (double)kr[c]);
                    dot *= inv; /* App. B: the diagonal term under the same 1/N */
                    for (int64_t c = 0; c < d; ++c) o[c] += dot * (double)vr[c];
                }
            }
        }
        free(w);
    }
    return 0;
}

/* phi' (derivatives of the activations above; shifted ELU: PAPER.md:795-809 gives
 * phi'(x) = 1 if x >= 1 else e^{x-1}; SiLU: sigma(x) (1 + x (1 - sigma(x)))). */
double vo_act_prime(int kind, double x) {
    switch (kind) {
        case VO_ACT_IDENTITY: return 1.0;
        case VO_ACT_SILU: {
            const double s = 1.0 / (1.0 + exp(-x));
            return s * (1.0 + x * (1.0 - s));
        }
        case VO_ACT_SHIFTED_ELU: return x >= 1.0 ? 1.0 : exp(x - 1.0);
        default: return NAN;
    }
}

/*
 * QLA backward (NEXT-2), source part at the seed rows.  Forward per (user u, head h):
 *   A = phi1(Q) [S x d], Z = sum_j phi1(k_j)^T v_j [d x d], Zbar = Z / N_u (if normalize and
 *   N_u > 0), W = phi2(Zbar), O = A W.
 * Chain rule (the appendix derives the phi2 = identity, no-1/N case, PAPER.md:776-783 and the
 * activated forms PAPER.md:817-829; phi2 and 1/N are composed around Z, reading R19):
 *   dW = A^T dO;  dZ = (dW . phi2'(Zbar)) / N_u;  dA = dO W^T;  dQ = dA . phi1'(Q)
 *   dV_j = phi1(k_j) dZ;  dK_j = (v_j dZ^T) . phi1'(k_j)
 * dout: [B, S, H, d]; dq: [B, S, H, d] (per user, before any sum over users of shared seeds);
 * dk, dv: [total, H, d].  All float64.
 */
int vo_qla_backward(int64_t B, int64_t S, int64_t H, int64_t d, const float* q, int64_t q_user_stride,
                    const float* k, const float* v, const int64_t* offsets, const float* dout, int phi1,
                    int phi2, int normalize, double* dq, double* dk, double* dv, int threads) {
    if (B < 0 || S < 1 || H < 1 || d < 1) return -1;
    set_threads(threads);
#pragma omp parallel
    {
        double* z = (double*)malloc((size_t)(d * d) * sizeof(double));
        double* w = (double*)malloc((size_t)(d * d) * sizeof(double));
        double* dz = (double*)malloc((size_t)(d * d) * sizeof(double));
#pragma omp for schedule(dynamic, 1)
        for (int64_t t = 0; t < B * H; ++t) {
            const int64_t u = t / H, h = t % H;
            const int64_t N = offsets[u + 1] - offsets[u];
            const double inv = (normalize && N > 0) ? 1.0 / (double)N : 1.0;
            for (int64_t e = 0; e < d * d; ++e) z[e] = 0.0;
            for (int64_t j = offsets[u]; j < offsets[u + 1]; ++j) {
                const float* kj = k + (j * H + h) * d;
                const float* vj = v + (j * H + h) * d;
                for (int64_t c1 = 0; c1 < d; ++c1) {
                    const double a = vo_act(phi1, (double)kj[c1]);
                    for (int64_t c2 = 0; c2 < d; ++c2) z[c1 * d + c2] += a * (double)vj[c2];
                }
            }
            for (int64_t e = 0; e < d * d; ++e) w[e] = vo_act(phi2, z[e] * inv);
            /* dW = A^T dO, then dZ */
            for (int64_t e = 0; e < d * d; ++e) dz[e] = 0.0;
            for (int64_t i = 0; i < S; ++i) {
                const float* qi = q + u * q_user_stride + (i * H + h) * d;
                const float* go = dout + ((u * S + i) * H + h) * d;
                for (int64_t c1 = 0; c1 < d; ++c1) {
                    const double a = vo_act(phi1, (double)qi[c1]);
                    for (int64_t c2 = 0; c2 < d; ++c2) dz[c1 * d + c2] += a * (double)go[c2];
                }
            }
            for (int64_t e = 0; e < d * d; ++e) dz[e] = dz[e] * vo_act_prime(phi2, z[e] * inv) * inv;
            /* dQ = (dO W^T) . phi1'(Q) */
            for (int64_t i = 0; i < S; ++i) {
                const float* qi = q + u * q_user_stride + (i * H + h) * d;
                const float* go = dout + ((u * S + i) * H + h) * d;
                double* g = dq + ((u * S + i) * H + h) * d;
                for (int64_t c1 = 0; c1 < d; ++c1) {
                    double acc = 0.0;
                    for (int64_t c2 = 0; c2 < d; ++c2) acc += (double)go[c2] * w[c1 * d + c2];
                    g[c1] = acc * vo_act_prime(phi1, (double)qi[c1]);
                }
            }
            /* dV_j = phi1(k_j) dZ;  dK_j = (v_j dZ^T) . phi1'(k_j) */
            for (int64_t j = offsets[u]; j < offsets[u + 1]; ++j) {
                const float* kj = k + (j * H + h) * d;
                const float* vj = v + (j * H + h) * d;
                double* gv = dv + (j * H + h) * d;
                double* gk = dk + (j * H + h) * d;
                for (int64_t c2 = 0; c2 < d; ++c2) gv[c2] = 0.0;
                for (int64_t c1 = 0; c1 < d; ++c1) {
                    const double a = vo_act(phi1, (double)kj[c1]);
                    double acc = 0.0;
                    for (int64_t c2 = 0; c2 < d; ++c2) {
                        gv[c2] += a * dz[c1 * d + c2];
                        acc += (double)vj[c2] * dz[c1 * d + c2];
                    }
                    gk[c1] = acc * vo_act_prime(phi1, (double)kj[c1]);
                }
            }
        }
        free(z);
        free(w);
        free(dz);
    }
    return 0;
}

/*
 * Softmax backward (NEXT-2; "FA-style dQ/dK/dV for the S-query softmax"), the plain
 * gradient of o_i = sum_j p_ij v_j, p_ij = softmax_j(s_ij), s_ij = scale q_i . k_j
 * (PAPER.md:158-163), per user u, head h:
 *   P = softmax rows;  dV_j = sum_i p_ij dO_i;  dP_ij = dO_i . v_j;  D_i = sum_j p_ij dP_ij
 *   dS_ij = p_ij (dP_ij - D_i);  dQ_i = scale sum_j dS_ij k_j;  dK_j = scale sum_i dS_ij q_i.
 * Two passes per row (max, then exp), sequential sums, float64.  dq [B,S,H,d] per user.
 */
int vo_softmax_backward(int64_t B, int64_t S, int64_t H, int64_t d, const float* q, int64_t q_user_stride,
                        const float* k, const float* v, const int64_t* offsets, double scale, const float* dout,
                        double* dq, double* dk, double* dv, int threads) {
    if (B < 0 || S < 1 || H < 1 || d < 1) return -1;
    set_threads(threads);
    int64_t total = offsets[B];
    for (int64_t e = 0; e < total * H * d; ++e) {
        dk[e] = 0.0;
        dv[e] = 0.0;
    }
    /* parallel over (u, h): each owns disjoint dk/dv rows and dq entries */
#pragma omp parallel
    {
        int64_t maxL = 0;
        for (int64_t u = 0; u < B; ++u) maxL = offsets[u + 1] - offsets[u] > maxL ? offsets[u + 1] - offsets[u] : maxL;
        double* p = (double*)malloc((size_t)(maxL > 0 ? maxL : 1) * sizeof(double));
        double* dp = (double*)malloc((size_t)(maxL > 0 ? maxL : 1) * sizeof(double));
#pragma omp for schedule(dynamic, 1)
        for (int64_t t = 0; t < B * H; ++t) {
            const int64_t u = t / H, h = t % H;
            const int64_t j0 = offsets[u], L = offsets[u + 1] - offsets[u];
            for (int64_t i = 0; i < S; ++i) {
                const float* qi = q + u * q_user_stride + (i * H + h) * d;
                const float* go = dout + ((u * S + i) * H + h) * d;
                double* gq = dq + ((u * S + i) * H + h) * d;
                for (int64_t c = 0; c < d; ++c) gq[c] = 0.0;
                if (L == 0) continue;
                double m = -INFINITY;
                for (int64_t j = 0; j < L; ++j) {
                    const float* kj = k + ((j0 + j) * H + h) * d;
                    double s = 0.0;
                    for (int64_t c = 0; c < d; ++c) s += (double)qi[c] * (double)kj[c];
                    p[j] = scale * s;
                    if (p[j] > m) m = p[j];
                }
                double l = 0.0;
                for (int64_t j = 0; j < L; ++j) {
                    p[j] = exp(p[j] - m);
                    l += p[j];
                }
                double D = 0.0;
                for (int64_t j = 0; j < L; ++j) {
                    p[j] /= l;
                    const float* vj = v + ((j0 + j) * H + h) * d;
                    double s = 0.0;
                    for (int64_t c = 0; c < d; ++c) s += (double)go[c] * (double)vj[c];
                    dp[j] = s;
                    D += p[j] * s;
                }
                for (int64_t j = 0; j < L; ++j) {
                    const float* kj = k + ((j0 + j) * H + h) * d;
                    double* gk = dk + ((j0 + j) * H + h) * d;
                    double* gv = dv + ((j0 + j) * H + h) * d;
                    const double ds = p[j] * (dp[j] - D);
                    for (int64_t c = 0; c < d; ++c) {
                        gv[c] += p[j] * (double)go[c];
                        gk[c] += scale * ds * (double)qi[c];
                        gq[c] += scale * ds * (double)kj[c];
                    }
                }
            }
        }
        free(p);
        free(dp);
    }
    return 0;
}

/*
 * LSE merge of P softmax partials over disjoint key sets, for n rows of width d
 * (flash-decoding style combination; the exact identity
 *   softmax over A u B = e^{lse_A - lse} O_A + e^{lse_B - lse} O_B,  lse = ln(e^{lse_A}+e^{lse_B})).
 *   part_o: [P, n, d]; part_lse: [P, n]; out: [n, d]; lse: [n].  Parts with lse = -inf weigh 0.
 */
int vo_merge_lse(int64_t P, int64_t n, int64_t d, const double* part_o, const double* part_lse,
                 double* out, double* lse) {
    for (int64_t r = 0; r < n; ++r) {
        double m = -INFINITY;
        for (int64_t p = 0; p < P; ++p)
            if (part_lse[p * n + r] > m) m = part_lse[p * n + r];
        double* o = out + r * d;
        for (int64_t c = 0; c < d; ++c) o[c] = 0.0;
        if (m == -INFINITY) {
            lse[r] = -INFINITY;
            continue;
        }
        double l = 0.0;
        for (int64_t p = 0; p < P; ++p) l += exp(part_lse[p * n + r] - m);
        const double L = m + log(l);
        for (int64_t p = 0; p < P; ++p) {
            const double w = exp(part_lse[p * n + r] - L);
            for (int64_t c = 0; c < d; ++c) o[c] += w * part_o[(p * n + r) * d + c];
        }
        lse[r] = L;
    }
    return 0;
}

/* Plain sum of P QLA states (split == sum of states, the associativity of sum_j). */
int vo_merge_sum(int64_t P, int64_t n, const double* parts, double* out) {
    for (int64_t e = 0; e < n; ++e) {
        double acc = 0.0;
        for (int64_t p = 0; p < P; ++p) acc += parts[p * n + e];
        out[e] = acc;
    }
    return 0;
}

/*
 * Int8 export of summary tokens (NEXT-1): "quantized and exported to a large key-value cache ...
 * dequantized with minimal distortion" (Sec. 3.1).  The scheme is SPEC.md:339-347
 * (the paper gives none): per token row of d values, symmetric-range affine quantization
 *   scale = max((max - min) / 254, 1e-12),  zero_point = (max + min) / 2,
 *   code  = clamp(round_half_even((x - zero_point) / scale), -127, 127),  x^ = code * scale + zp.
 * Reading R21: the codes are an integer decision taken from floating point, so they
 * are decided in float32 -- the precision of the stored scale and zero point, the only values a
 * consumer ever dequantizes with -- with no FMA contraction (-std=c11 => -ffp-contract=off):
 * t = (x - zp) / s with the stored s, zp.  SPEC.md:342 says only "round"; an exact tie
 * t = k + 1/2 goes to the even k (round-half-to-even, rintf, the IEEE default).  Both choices are
 * pinned by tests/test_oracle_pins.py (exact .5 ties; |code s + zp - x| <= s/2 with the stored s).
 */
int vo_quantize_rows_f32(int64_t n, int64_t d, const float* x, signed char* codes, float* scale, float* zp) {
    for (int64_t r = 0; r < n; ++r) {
        const float* xr = x + r * d;
        float mx = xr[0], mn = xr[0];
        for (int64_t c = 1; c < d; ++c) {
            if (xr[c] > mx) mx = xr[c];
            if (xr[c] < mn) mn = xr[c];
        }
        float s = (mx - mn) / 254.0f;
        if (!(s > 1e-12f)) s = 1e-12f;
        const float z = 0.5f * (mx + mn);
        scale[r] = s;
        zp[r] = z;
        for (int64_t c = 0; c < d; ++c) {
            float q = rintf((xr[c] - z) / s);
            if (q > 127.0f) q = 127.0f;
            if (q < -127.0f) q = -127.0f;
            codes[r * d + c] = (signed char)q;
        }
    }
    return 0;
}

/*
 * Stage-2 target-aware attention (NEXT-4): "any attention network can technically be used for the
 * target-aware attention stage ... we selected a standard O(N^2) transformer block, which delivers
 * excellent performance on the compact summary sequences" (Sec. 3.3), over the
 * summary tokens "retrieved from the cache and dequantized" (Sec. 3.1), with
 * candidates never attending each other ("the candidates cannot attend each other").
 * Reading R22: each candidate attends to [the S tokens of its user; itself]
 * (SPEC.md:264-272 target_attend), keys = values = the dequantized tokens (a block's W_k / W_v fold
 * into the query and the output by linearity), the candidate's own key / value given.
 * For candidate c in [row_offsets[u], row_offsets[u+1]) and head h:
 *   t_i    = codes[u,i,h,:] * tscale[u,i,h] + tzp[u,i,h]            (dequantization)
 *   s_i    = scale q_c . t_i,   s_self = scale q_c . k_c,   m = max(s_i, s_self)
 *   o_c    = (sum_i e^{s_i - m} t_i + e^{s_self - m} v_c) / (sum_i e^{s_i - m} + e^{s_self - m})
 *   out_c  = o_c + resid_c (resid may be NULL);   lse_c = m + ln(sum ...)  (lse may be NULL)
 * codes [B,S,H,d] int8; tscale, tzp [B,S,H]; q, k_self, v_self, resid, out [R,H,d]; lse [R,H].
 */
int vo_target_attend(int64_t B, int64_t S, int64_t H, int64_t d, const signed char* codes, const float* tscale,
                     const float* tzp, const float* q, const float* k_self, const float* v_self, const float* resid,
                     const int64_t* row_offsets, double scale, double* out, double* lse, int threads) {
    if (B < 0 || S < 1 || H < 1 || d < 1) return -1;
    set_threads(threads);
    const int64_t R = row_offsets[B];
#pragma omp parallel
    {
        double* t = (double*)malloc((size_t)(S * d) * sizeof(double));
        double* sc = (double*)malloc((size_t)(S + 1) * sizeof(double));
#pragma omp for schedule(dynamic, 1)
        for (int64_t x = 0; x < R * H; ++x) {
            const int64_t c = x / H, h = x % H;
            int64_t u = 0;
            while (row_offsets[u + 1] <= c) ++u;
            for (int64_t i = 0; i < S; ++i) {
                const double a = (double)tscale[(u * S + i) * H + h], b = (double)tzp[(u * S + i) * H + h];
                for (int64_t e = 0; e < d; ++e) t[i * d + e] = (double)codes[((u * S + i) * H + h) * d + e] * a + b;
            }
            const float* qc = q + (c * H + h) * d;
            const float* kc = k_self + (c * H + h) * d;
            const float* vc = v_self + (c * H + h) * d;
            double m = -INFINITY;
            for (int64_t i = 0; i <= S; ++i) {
                double acc = 0.0;
                for (int64_t e = 0; e < d; ++e) acc += (double)qc[e] * (i < S ? t[i * d + e] : (double)kc[e]);
                sc[i] = scale * acc;
                if (sc[i] > m) m = sc[i];
            }
            double l = 0.0;
            double* o = out + (c * H + h) * d;
            for (int64_t e = 0; e < d; ++e) o[e] = 0.0;
            for (int64_t i = 0; i <= S; ++i) {
                const double p = exp(sc[i] - m);
                l += p;
                for (int64_t e = 0; e < d; ++e) o[e] += p * (i < S ? t[i * d + e] : (double)vc[e]);
            }
            for (int64_t e = 0; e < d; ++e) o[e] = o[e] / l + (resid ? (double)resid[(c * H + h) * d + e] : 0.0);
            if (lse) lse[c * H + h] = m + log(l);
        }
        free(t);
        free(sc);
    }
    return 0;
}

/*
 * Multi-layer summarizer (NEXT-3).  "self-attention with virtual seed embeddings to summarize
 * ultra-long UIH sequences" (Sec. 3.2) with "the QLU module and the SGLU module"
 * (Sec. 3.2.2), full (not causal) self-attention, 3 -> 5 layers in
 * production.  Reading R23: user u's sequence
 * X = [S seed rows; L_u history rows] (rows [offsets[u], offsets[u+1]) of x, width D = H d); per layer
 *   Q = X Wq^T, K = X Wk^T, V = X Wv^T, G = X Wg^T                     (W* [D][D], row = output)
 *   per head h (columns [h d, h d + d)):  Z = sum_{rows j of u} phi1(K_jh)^T V_jh,
 *        W_h = phi2(Z / N_u) (N_u = S + L_u when normalizing),  O_rh = phi1(Q_rh) W_h
 *   Y = (O (.) sigmoid(G)) Wo^T,   X <- X + Y
 * After the layers, the summary tokens are the first S rows of every user.
 * weights: [L][5][D][D] (q, k, v, g, o); x: [R][D] input; x_out: [R][D] after the layers (float64).
 */
int vo_summarize_layers(int64_t B, int64_t S, int64_t H, int64_t d, int64_t n_layers, const float* weights,
                        const float* x, const int64_t* offsets, int phi1, int phi2, int normalize, double* x_out,
                        int threads) {
    if (B < 0 || S < 1 || H < 1 || d < 1 || n_layers < 0) return -1;
    set_threads(threads);
    const int64_t D = H * d, R = offsets[B];
    for (int64_t e = 0; e < R * D; ++e) x_out[e] = (double)x[e];
    double* qkvg = (double*)malloc((size_t)(R * 4 * D) * sizeof(double));
    double* o = (double*)malloc((size_t)(R * D) * sizeof(double));
    if (!qkvg || !o) {
        free(qkvg);
        free(o);
        return -1;
    }
    for (int64_t layer = 0; layer < n_layers; ++layer) {
        const float* W = weights + layer * 5 * D * D;
        /* projections: qkvg[r][t*D + c] = sum_i x[r][i] W_t[c][i] */
#pragma omp parallel for schedule(static)
        for (int64_t r = 0; r < R; ++r)
            for (int64_t t = 0; t < 4; ++t)
                for (int64_t c = 0; c < D; ++c) {
                    double acc = 0.0;
                    for (int64_t i = 0; i < D; ++i) acc += x_out[r * D + i] * (double)W[(t * D + c) * D + i];
                    qkvg[r * 4 * D + t * D + c] = acc;
                }
        /* QLA over all rows of the user, per head */
#pragma omp parallel
        {
            double* z = (double*)malloc((size_t)(d * d) * sizeof(double));
#pragma omp for schedule(dynamic, 1)
            for (int64_t t = 0; t < B * H; ++t) {
                const int64_t u = t / H, h = t % H;
                const int64_t N = offsets[u + 1] - offsets[u];
                const double inv = (normalize && N > 0) ? 1.0 / (double)N : 1.0;
                for (int64_t e = 0; e < d * d; ++e) z[e] = 0.0;
                for (int64_t j = offsets[u]; j < offsets[u + 1]; ++j)
                    for (int64_t c1 = 0; c1 < d; ++c1) {
                        const double a = vo_act(phi1, qkvg[j * 4 * D + D + h * d + c1]);
                        for (int64_t c2 = 0; c2 < d; ++c2) z[c1 * d + c2] += a * qkvg[j * 4 * D + 2 * D + h * d + c2];
                    }
                for (int64_t e = 0; e < d * d; ++e) z[e] = vo_act(phi2, z[e] * inv);
                for (int64_t r = offsets[u]; r < offsets[u + 1]; ++r)
                    for (int64_t c2 = 0; c2 < d; ++c2) {
                        double acc = 0.0;
                        for (int64_t c1 = 0; c1 < d; ++c1) acc += vo_act(phi1, qkvg[r * 4 * D + h * d + c1]) * z[c1 * d + c2];
                        o[r * D + h * d + c2] = acc;
                    }
            }
            free(z);
        }
        /* SGLU gate, output projection, residual */
        const float* Wo = W + 4 * D * D;
#pragma omp parallel
        {
            double* gated = (double*)malloc((size_t)D * sizeof(double));
#pragma omp for schedule(static)
            for (int64_t r = 0; r < R; ++r) {
                for (int64_t i = 0; i < D; ++i)
                    gated[i] = o[r * D + i] / (1.0 + exp(-qkvg[r * 4 * D + 3 * D + i]));
                for (int64_t c = 0; c < D; ++c) {
                    double acc = 0.0;
                    for (int64_t i = 0; i < D; ++i) acc += gated[i] * (double)Wo[c * D + i];
                    x_out[r * D + c] += acc;
                }
            }
            free(gated);
        }
    }
    free(qkvg);
    free(o);
    return 0;
}
