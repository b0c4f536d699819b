/*
 * vsp_oracle.c — TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C, f64, single-threaded restatement of the reference VS-prefill hot path
 * (/root/reference/proj/include/vsprefill/ headers). It is the CHECKER for the sm_100a
 * kernels: only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may call it. The product path never links it.
 *
 * Parity pinning: tests/test_oracle.py checks every function here against
 *   (1) the reference's own known-answer tests (restated, with file:line), and
 *   (2) golden vectors produced by the reference itself (oracle/_ref, built from
 *       /root/reference headers by oracle/Makefile; tests/golden/make_golden.py).
 *
 * Every matrix argument is (base, row_stride): element (t, c) is base[t*stride + c],
 * so heads of a [n, H, d] tensor are addressed in place (stride = H*d).
 * Functions return 0 on success, or VSO_EINVAL with the reference's message copied
 * into err (the reference throws std::invalid_argument with the same text).
 */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#define VSO_OK 0
#define VSO_EINVAL 1

static int fail(char* err, size_t errlen, const char* msg) {
    if (err && errlen) {
        strncpy(err, msg, errlen - 1);
        err[errlen - 1] = '\0';
    }
    return VSO_EINVAL;
}

/* ------------------------------------------------------------------ numerics */

/* numerics.hpp:17-24 — overflow-safe SiLU */
double vso_silu(double x) {
    if (x >= 0.0) return x / (1.0 + exp(-x));
    const double e = exp(x);
    return x * e / (1.0 + e);
}

/* numerics.hpp:34-52 (softmax_row_inplace with no mask) */
static int softmax_inplace(double* row, int64_t n, char* err, size_t errlen) {
    double m = -INFINITY;
    for (int64_t j = 0; j < n; ++j) m = row[j] > m ? row[j] : m;
    if (m == -INFINITY) return fail(err, errlen, "empty softmax row");
    double denom = 0.0;
    for (int64_t j = 0; j < n; ++j) {
        row[j] = exp(row[j] - m);
        denom += row[j];
    }
    for (int64_t j = 0; j < n; ++j) row[j] /= denom;
    return VSO_OK;
}

/* ------------------------------------------------------------------ merge */

/* merge.hpp:18-56 — ascending union of {j in iv : j <= i} and {i - o : o in is, o <= i}.
 * out must hold kv + ks entries. Returns the count, or -1 on unsorted input. */
int64_t vso_merge_row_columns(const int64_t* iv, int64_t kv, const int64_t* is, int64_t ks,
                              int64_t i, int64_t* out, char* err, size_t errlen) {
    for (int64_t t = 1; t < kv; ++t)
        if (!(iv[t - 1] < iv[t])) {
            fail(err, errlen, "merge_row_columns: i_v not strictly ascending");
            return -1;
        }
    for (int64_t t = 1; t < ks; ++t)
        if (!(is[t - 1] < is[t])) {
            fail(err, errlen, "merge_row_columns: i_s not strictly ascending");
            return -1;
        }
    int64_t s = ks;
    while (s > 0 && is[s - 1] > i) --s; /* merge.hpp:30-31 */
    int64_t cnt = 0, v = 0, si = s;
    for (;;) {
        const int has_v = v < kv && iv[v] <= i;
        const int has_s = si > 0;
        if (!has_v && !has_s) break;
        const int64_t cv = has_v ? iv[v] : 0;
        const int64_t cs = has_s ? i - is[si - 1] : 0;
        if (has_v && (!has_s || cv < cs)) {
            out[cnt++] = cv;
            ++v;
        } else if (has_s && (!has_v || cs < cv)) {
            out[cnt++] = cs;
            --si;
        } else {
            out[cnt++] = cv;
            ++v;
            --si;
        }
    }
    return cnt;
}

/* merge.hpp:69-95 — p-way merge-path cut points (a-first on ties). cuts: 2*(p+1) entries
 * (a_idx, b_idx) pairs. */
int vso_merge_path_partition(const int64_t* a, int64_t na, const int64_t* b, int64_t nb, int64_t p,
                             int64_t* cuts, char* err, size_t errlen) {
    if (p < 1) return fail(err, errlen, "merge_path_partition: p must be >= 1");
    const int64_t total = na + nb;
    cuts[0] = 0;
    cuts[1] = 0;
    cuts[2 * p] = na;
    cuts[2 * p + 1] = nb;
    for (int64_t s = 1; s < p; ++s) {
        const int64_t diag = s * total / p;
        int64_t lo = diag > nb ? diag - nb : 0;
        int64_t hi = diag < na ? diag : na;
        while (lo < hi) {
            const int64_t mid = lo + (hi - lo) / 2;
            if (a[mid] <= b[diag - mid - 1])
                lo = mid + 1;
            else
                hi = mid;
        }
        cuts[2 * s] = lo;
        cuts[2 * s + 1] = diag - lo;
    }
    return VSO_OK;
}

/* ------------------------------------------------------------------ attention */

static double dot(const double* x, const double* y, int64_t d) {
    double s = 0.0;
    for (int64_t c = 0; c < d; ++c) s += x[c] * y[c];
    return s;
}

/* attention.hpp:96-145 — blockwise (flash-style) dense causal attention, one head.
 * lse (optional) receives m_i + log(l_i) in natural-log units of the scaled logits. */
int vso_blockwise_attention(int64_t n, int64_t d, const double* q, int64_t qs, const double* k,
                            int64_t ks, const double* v, int64_t vs, int64_t block, double* o,
                            int64_t os, double* lse, char* err, size_t errlen) {
    if (block < 1) return fail(err, errlen, "blockwise_attention: block must be >= 1");
    if (n < 1) return fail(err, errlen, "attention inputs: empty sequence");
    const double scale = 1.0 / sqrt((double)d);
    const int64_t bs = block < n ? block : n;
    double* acc = (double*)calloc((size_t)(n * d), sizeof(double));
    double* mx = (double*)malloc(sizeof(double) * n);
    double* den = (double*)calloc((size_t)n, sizeof(double));
    double* tile = (double*)malloc(sizeof(double) * bs);
    for (int64_t i = 0; i < n; ++i) mx[i] = -INFINITY;
    for (int64_t i0 = 0; i0 < n; i0 += bs) {
        const int64_t i1 = i0 + bs < n ? i0 + bs : n;
        for (int64_t j0 = 0; j0 < i1; j0 += bs) {
            const int64_t j1 = j0 + bs < n ? j0 + bs : n;
            for (int64_t i = (i0 > j0 ? i0 : j0); i < i1; ++i) {
                const int64_t jend = j1 < i + 1 ? j1 : i + 1;
                double tmax = -INFINITY;
                for (int64_t j = j0; j < jend; ++j) {
                    tile[j - j0] = dot(q + i * qs, k + j * ks, d) * scale;
                    if (tile[j - j0] > tmax) tmax = tile[j - j0];
                }
                double* ai = acc + i * d;
                if (tmax > mx[i]) {
                    const double r = exp(mx[i] - tmax);
                    den[i] *= r;
                    for (int64_t c = 0; c < d; ++c) ai[c] *= r;
                    mx[i] = tmax;
                }
                for (int64_t j = j0; j < jend; ++j) {
                    const double w = exp(tile[j - j0] - mx[i]);
                    den[i] += w;
                    const double* vj = v + j * vs;
                    for (int64_t c = 0; c < d; ++c) ai[c] += w * vj[c];
                }
            }
        }
    }
    for (int64_t i = 0; i < n; ++i) {
        for (int64_t c = 0; c < d; ++c) o[i * os + c] = acc[i * d + c] / den[i];
        if (lse) lse[i] = mx[i] + log(den[i]);
    }
    free(acc);
    free(mx);
    free(den);
    free(tile);
    return VSO_OK;
}

/* attention.hpp:150-194 — VS sparse attention over the per-row merged column set
 * (merge.hpp:18-56), chunks of `block` columns with online max/denominator.
 * Throws "uncovered query row i" (attention.hpp:161-163). */
int vso_sparse_attention(int64_t n, int64_t d, const double* q, int64_t qs, const double* k,
                         int64_t ks, const double* v, int64_t vs, const int64_t* iv, int64_t kv,
                         const int64_t* is, int64_t ksl, int64_t block, double* o, int64_t os,
                         double* lse, char* err, size_t errlen) {
    if (block < 1) return fail(err, errlen, "sparse_attention: block must be >= 1");
    if (n < 1) return fail(err, errlen, "attention inputs: empty sequence");
    const double scale = 1.0 / sqrt((double)d);
    int64_t* cols = (int64_t*)malloc(sizeof(int64_t) * (size_t)(kv + ksl + 1));
    double* acc = (double*)malloc(sizeof(double) * d);
    double* lg = (double*)malloc(sizeof(double) * block);
    int rc = VSO_OK;
    for (int64_t i = 0; i < n; ++i) {
        const int64_t nc = vso_merge_row_columns(iv, kv, is, ksl, i, cols, err, errlen);
        if (nc < 0) {
            rc = VSO_EINVAL;
            break;
        }
        if (nc == 0) {
            char msg[64];
            snprintf(msg, sizeof msg, "uncovered query row %lld", (long long)i);
            rc = fail(err, errlen, msg);
            break;
        }
        double m = -INFINITY, den = 0.0;
        for (int64_t c = 0; c < d; ++c) acc[c] = 0.0;
        for (int64_t st = 0; st < nc; st += block) {
            const int64_t en = st + block < nc ? st + block : nc;
            double bmax = -INFINITY;
            for (int64_t t = st; t < en; ++t) {
                lg[t - st] = dot(q + i * qs, k + cols[t] * ks, d) * scale;
                if (lg[t - st] > bmax) bmax = lg[t - st];
            }
            if (bmax > m) {
                const double r = exp(m - bmax);
                den *= r;
                for (int64_t c = 0; c < d; ++c) acc[c] *= r;
                m = bmax;
            }
            for (int64_t t = st; t < en; ++t) {
                const double w = exp(lg[t - st] - m);
                den += w;
                const double* vj = v + cols[t] * vs;
                for (int64_t c = 0; c < d; ++c) acc[c] += w * vj[c];
            }
        }
        for (int64_t c = 0; c < d; ++c) o[i * os + c] = acc[c] / den;
        if (lse) lse[i] = m + log(den);
    }
    free(cols);
    free(acc);
    free(lg);
    return rc;
}

/* attention.hpp:198-215 via the LSE identity: sum_{j in cols(i)} A[i,j] =
 * exp(lse_sparse_i - lse_dense_i). Returns mean over rows. */
double vso_recall_from_lse(int64_t n, const double* lse_sparse, const double* lse_dense) {
    double t = 0.0;
    for (int64_t i = 0; i < n; ++i) t += exp(lse_sparse[i] - lse_dense[i]);
    return t / (double)n;
}

/* ------------------------------------------------------------------ selection */

static int cmp_desc(const void* a, const void* b) {
    const double x = *(const double*)a, y = *(const double*)b;
    return (x < y) - (x > y);
}

/* sparsity.hpp:22-36 BudgetConfig::check */
static int budget_check(double tau_v, double tau_s, int64_t min_b, int64_t max_b, char* err,
                        size_t errlen) {
    if (!(tau_v > 0.0 && tau_v <= 1.0)) return fail(err, errlen, "budget config: tau_v must be in (0, 1]");
    if (!(tau_s > 0.0 && tau_s <= 1.0)) return fail(err, errlen, "budget config: tau_s must be in (0, 1]");
    if (min_b < 1) return fail(err, errlen, "budget config: min_budget must be >= 1");
    if (max_b >= 0 && min_b > max_b)
        return fail(err, errlen, "budget config: min_budget exceeds max_budget");
    return VSO_OK;
}

/* sparsity.hpp:51-79 — smallest k whose sorted-desc cumulative mass >= tau - 1e-12,
 * clamped to [min_budget, max_budget ^ n]. max_b < 0 means "no max". */
int vso_cumulative_budget(const double* scores, int64_t n, double tau, double tau_v, double tau_s,
                          int64_t min_b, int64_t max_b, int64_t* k_out, char* err, size_t errlen) {
    int rc = budget_check(tau_v, tau_s, min_b, max_b, err, errlen);
    if (rc) return rc;
    if (!(tau > 0.0 && tau <= 1.0)) return fail(err, errlen, "cumulative_budget: tau must be in (0, 1]");
    if (n < 1) return fail(err, errlen, "cumulative_budget: empty scores");
    double total = 0.0;
    for (int64_t i = 0; i < n; ++i) {
        if (!(scores[i] >= 0.0)) return fail(err, errlen, "cumulative_budget: negative score");
        total += scores[i];
    }
    if (fabs(total - 1.0) > 1e-6) return fail(err, errlen, "cumulative_budget: scores do not sum to 1");
    double* sorted = (double*)malloc(sizeof(double) * n);
    memcpy(sorted, scores, sizeof(double) * n);
    qsort(sorted, (size_t)n, sizeof(double), cmp_desc);
    int64_t k = n;
    double cum = 0.0;
    for (int64_t i = 0; i < n; ++i) {
        cum += sorted[i];
        if (cum >= tau - 1e-12) {
            k = i + 1;
            break;
        }
    }
    free(sorted);
    const int64_t lo = min_b < n ? min_b : n;
    if (k < lo) k = lo;
    int64_t upper = n;
    if (max_b >= 0 && max_b < upper) upper = max_b;
    *k_out = k < upper ? k : upper;
    return VSO_OK;
}

static const double* g_scores;
static int cmp_topk(const void* a, const void* b) {
    const int64_t x = *(const int64_t*)a, y = *(const int64_t*)b;
    if (g_scores[x] != g_scores[y]) return g_scores[x] > g_scores[y] ? -1 : 1;
    return (x > y) - (x < y);
}
static int cmp_i64(const void* a, const void* b) {
    const int64_t x = *(const int64_t*)a, y = *(const int64_t*)b;
    return (x > y) - (x < y);
}

/* sparsity.hpp:83-97 — k largest, value desc then index asc, output ascending. */
int vso_topk_indices(const double* scores, int64_t n, int64_t k, int64_t* out, char* err,
                     size_t errlen) {
    if (k < 1) return fail(err, errlen, "topk_indices: k must be >= 1");
    if (k > n) return fail(err, errlen, "topk_indices: k exceeds score count");
    int64_t* order = (int64_t*)malloc(sizeof(int64_t) * n);
    for (int64_t i = 0; i < n; ++i) order[i] = i;
    g_scores = scores; /* single-threaded checker */
    qsort(order, (size_t)n, sizeof(int64_t), cmp_topk);
    qsort(order, (size_t)k, sizeof(int64_t), cmp_i64);
    memcpy(out, order, sizeof(int64_t) * k);
    free(order);
    return VSO_OK;
}

/* sparsity.hpp:105-114 (+ inject_offset_zero :99-101). iv/is must hold n (+1) entries. */
int vso_select_pattern(const double* sv, const double* ss, int64_t n, double tau_v, double tau_s,
                       int64_t min_b, int64_t max_b, int64_t* iv, int64_t* kv, int64_t* is,
                       int64_t* ks, char* err, size_t errlen) {
    int64_t k_v = 0, k_s = 0;
    int rc = vso_cumulative_budget(sv, n, tau_v, tau_v, tau_s, min_b, max_b, &k_v, err, errlen);
    if (rc) return rc;
    rc = vso_cumulative_budget(ss, n, tau_s, tau_v, tau_s, min_b, max_b, &k_s, err, errlen);
    if (rc) return rc;
    rc = vso_topk_indices(sv, n, k_v, iv, err, errlen);
    if (rc) return rc;
    rc = vso_topk_indices(ss, n, k_s, is, err, errlen);
    if (rc) return rc;
    if (is[0] != 0) {
        memmove(is + 1, is, sizeof(int64_t) * k_s);
        is[0] = 0;
        ++k_s;
    }
    *kv = k_v;
    *ks = k_s;
    return VSO_OK;
}

/* ------------------------------------------------------------------ indexer */

/* indexer.hpp:77-120 — X = [K | V] (hconcat :119), Y = X W_U + b_U, Z = SiLU(Y),
 * logit_v = Z w_v + b_v, raw_s = Z w_s + b_s, logit_s[o] = raw_s[n-1-o] (Reverse,
 * :26-28) or raw_s[o] (Identity), pred = softmax over n. w_u is [2d, d_h] row-major. */
int vso_indexer_forward(int64_t n, int64_t d, const double* k, int64_t ks, const double* v,
                        int64_t vs, int64_t d_h, const double* w_u, const double* b_u,
                        const double* w_v, double b_v, const double* w_s, double b_s,
                        int reverse, double* logits_v, double* logits_s, double* pred_v,
                        double* pred_s, char* err, size_t errlen) {
    if (n < 1) return fail(err, errlen, "indexer_forward: empty input");
    double* y = (double*)malloc(sizeof(double) * d_h);
    double* raw_s = (double*)malloc(sizeof(double) * n);
    for (int64_t t = 0; t < n; ++t) {
        for (int64_t h = 0; h < d_h; ++h) y[h] = 0.0;
        /* matrix.hpp:56-71 i-k-j order: y[h] += x[c] * W[c][h] */
        for (int64_t c = 0; c < 2 * d; ++c) {
            const double xc = c < d ? k[t * ks + c] : v[t * vs + (c - d)];
            const double* wr = w_u + c * d_h;
            for (int64_t h = 0; h < d_h; ++h) y[h] += xc * wr[h];
        }
        double lv = b_v, ls = b_s;
        for (int64_t h = 0; h < d_h; ++h) {
            const double z = vso_silu(y[h] + b_u[h]);
            lv += z * w_v[h];
            ls += z * w_s[h];
        }
        logits_v[t] = lv;
        raw_s[t] = ls;
    }
    for (int64_t o = 0; o < n; ++o) logits_s[o] = raw_s[reverse ? n - 1 - o : o];
    memcpy(pred_v, logits_v, sizeof(double) * n);
    memcpy(pred_s, logits_s, sizeof(double) * n);
    int rc = softmax_inplace(pred_v, n, err, errlen);
    if (!rc) rc = softmax_inplace(pred_s, n, err, errlen);
    free(y);
    free(raw_s);
    return rc;
}

/* ------------------------------------------------------------------ aggregation */

/* vsaggregate.hpp:62-127 — two-pass streaming aggregation of one head; adds
 * vertical[j] += A[i,j], slash[i-j] += A[i,j] (raw, i.e. summing to n), then
 * normalize_scores (:27-33) divides by n when normalized != 0. */
int vso_aggregate_streaming(int64_t n, int64_t d, const double* q, int64_t qs, const double* k,
                            int64_t ks, int64_t block, int normalized, double* vertical,
                            double* slash, char* err, size_t errlen) {
    if (block < 1) return fail(err, errlen, "aggregate_streaming: block must be >= 1");
    const double scale = 1.0 / sqrt((double)d);
    const int64_t bs = block < n ? block : n;
    double* mx = (double*)malloc(sizeof(double) * n);
    double* den = (double*)calloc((size_t)n, sizeof(double));
    double* tile = (double*)malloc(sizeof(double) * bs * bs);
    for (int64_t i = 0; i < n; ++i) {
        mx[i] = -INFINITY;
        vertical[i] = 0.0;
        slash[i] = 0.0;
    }
    for (int pass = 0; pass < 2; ++pass) {
        for (int64_t i0 = 0; i0 < n; i0 += bs) {
            const int64_t i1 = i0 + bs < n ? i0 + bs : n;
            for (int64_t j0 = 0; j0 < i1; j0 += bs) {
                const int64_t j1 = j0 + bs < n ? j0 + bs : n;
                for (int64_t i = (i0 > j0 ? i0 : j0); i < i1; ++i) {
                    const int64_t jend = j1 < i + 1 ? j1 : i + 1;
                    for (int64_t j = j0; j < jend; ++j)
                        tile[(i - i0) * bs + (j - j0)] = dot(q + i * qs, k + j * ks, d) * scale;
                }
                for (int64_t i = (i0 > j0 ? i0 : j0); i < i1; ++i) {
                    const int64_t jend = j1 < i + 1 ? j1 : i + 1;
                    if (pass == 0) {
                        double tmax = -INFINITY;
                        for (int64_t j = j0; j < jend; ++j) {
                            const double s = tile[(i - i0) * bs + (j - j0)];
                            tmax = s > tmax ? s : tmax;
                        }
                        if (tmax > mx[i]) {
                            den[i] *= exp(mx[i] - tmax);
                            mx[i] = tmax;
                        }
                        for (int64_t j = j0; j < jend; ++j)
                            den[i] += exp(tile[(i - i0) * bs + (j - j0)] - mx[i]);
                    } else {
                        for (int64_t j = j0; j < jend; ++j) {
                            const double w = exp(tile[(i - i0) * bs + (j - j0)] - mx[i]) / den[i];
                            vertical[j] += w;
                            slash[i - j] += w;
                        }
                    }
                }
            }
        }
    }
    if (normalized) {
        const double inv = 1.0 / (double)n;
        for (int64_t i = 0; i < n; ++i) {
            vertical[i] *= inv;
            slash[i] *= inv;
        }
    }
    free(mx);
    free(den);
    free(tile);
    return VSO_OK;
}

/* vsaggregate.hpp:133-157 — combine_scores over `heads` score vectors laid out
 * [heads][n]; mean != 0 selects GroupReduce::Mean. */
void vso_combine_scores(int64_t heads, int64_t n, const double* v_in, const double* s_in, int mean,
                        double* v_out, double* s_out) {
    for (int64_t i = 0; i < n; ++i) {
        v_out[i] = 0.0;
        s_out[i] = 0.0;
    }
    for (int64_t h = 0; h < heads; ++h)
        for (int64_t i = 0; i < n; ++i) {
            v_out[i] += v_in[h * n + i];
            s_out[i] += s_in[h * n + i];
        }
    if (mean) {
        const double inv = 1.0 / (double)heads;
        for (int64_t i = 0; i < n; ++i) {
            v_out[i] *= inv;
            s_out[i] *= inv;
        }
    }
}

/* ------------------------------------------------------------------ RoPE */

/* RopeConfig (rope.hpp:13-39) + apply_rope (rope.hpp:63-79) for one head: row t of x
 * (n x d, row stride xs) rotated by R(positions[t]) (positions NULL: t), plane p pairs
 * (2p, 2p+1) and rotates by t * base^(-2p/d). out may alias x. */
int vso_apply_rope(int64_t n, int64_t d, const double* x, int64_t xs, const int64_t* positions, double base,
                   double* out, int64_t os, char* err, size_t errlen) {
    if (d < 2 || d % 2 != 0) return fail(err, errlen, "rope head_dim must be even and >= 2");
    if (!(base > 0.0)) return fail(err, errlen, "rope base must be positive");
    for (int64_t i = 0; i < n; ++i) {
        const double t = positions ? (double)positions[i] : (double)i;
        const double* src = x + i * xs;
        double* dst = out + i * os;
        for (int64_t p = 0; p < d / 2; ++p) {
            const double angle = t * pow(base, -2.0 * (double)p / (double)d);
            const double c = cos(angle), s = sin(angle);
            const double a = src[2 * p], b = src[2 * p + 1];
            dst[2 * p] = c * a - s * b;
            dst[2 * p + 1] = s * a + c * b;
        }
    }
    return VSO_OK;
}

/* ------------------------------------------------------------------ distillation (training half) */

/* kl_loss_grad Forward (indexer.hpp:158-185) + softmax_backward (numerics.hpp:62-72) +
 * indexer_backward_from_upstream (indexer.hpp:222-262) for one KV head, fused:
 *   loss = KL(pred_v || t_v + eps) + KL(pred_s || t_s + eps)        (kl_loss :138-149)
 *   dpred = log(pred) + 1 - log(t + eps)   (log(1e-300) for pred == 0)
 *   dlogit = pred * (dpred - <pred, dpred>)
 *   dlogit_s is mapped back to tokens: token slash_token_for_offset(o) gets dlogit_s[o]
 *   g.w_v[h] = sum_i dlogit_v[i] z[i][h]; g.w_s likewise; g.b_v = sum dlogit_v; g.b_s likewise
 *   dy = (dlogit_v[i] w_v[h] + dlogit_s[i] w_s[h]) * silu'(y[i][h]);  g.w_u = X^T dy; g.b_u = sum dy
 * The forward is recomputed here (indexer_forward_features :77-113). Validation as kl_loss:
 * pred/target non-negative and summing to 1 within 1e-6 (check_distribution :125-135). */
static double silu_deriv(double x) {
    const double s = x >= 0.0 ? 1.0 / (1.0 + exp(-x)) : exp(x) / (1.0 + exp(x));
    return s + x * s * (1.0 - s);
}

static int check_dist(const double* v, int64_t n, const char* what, char* err, size_t errlen) {
    double sum = 0.0;
    char msg[96];
    for (int64_t i = 0; i < n; ++i) {
        if (v[i] < 0.0) {
            snprintf(msg, sizeof msg, "%s has negative entries", what);
            return fail(err, errlen, msg);
        }
        sum += v[i];
    }
    if (fabs(sum - 1.0) > 1e-6) {
        snprintf(msg, sizeof msg, "%s does not sum to 1", what);
        return fail(err, errlen, msg);
    }
    return VSO_OK;
}

static double kl_grad(const double* pred, const double* target, int64_t n, double eps, double* dlogit) {
    double loss = 0.0, inner = 0.0;
    for (int64_t i = 0; i < n; ++i) {
        if (pred[i] > 0.0) loss += pred[i] * (log(pred[i]) - log(target[i] + eps));
        const double dp = (pred[i] > 0.0 ? log(pred[i]) : log(1e-300)) + 1.0 - log(target[i] + eps);
        dlogit[i] = dp;
        inner += dp * pred[i];
    }
    for (int64_t i = 0; i < n; ++i) dlogit[i] = pred[i] * (dlogit[i] - inner);
    return loss;
}

int vso_indexer_backward(int64_t n, int64_t d, const double* k, int64_t ks, const double* v, int64_t vs,
                         int64_t d_h, const double* w_u, const double* b_u, const double* w_v, double b_v,
                         const double* w_s, double b_s, int reverse, const double* target_v,
                         const double* target_s, double eps, double* loss_out, double* g_w_u, double* g_b_u,
                         double* g_w_v, double* g_b_v, double* g_w_s, double* g_b_s, char* err, size_t errlen) {
    if (eps <= 0.0) return fail(err, errlen, "kl_loss: eps must be positive");
    double* lv = (double*)malloc(sizeof(double) * n);
    double* ls = (double*)malloc(sizeof(double) * n);
    double* pv = (double*)malloc(sizeof(double) * n);
    double* ps = (double*)malloc(sizeof(double) * n);
    double* dv = (double*)malloc(sizeof(double) * n);
    double* dso = (double*)malloc(sizeof(double) * n);
    double* y = (double*)malloc(sizeof(double) * d_h);
    int rc = vso_indexer_forward(n, d, k, ks, v, vs, d_h, w_u, b_u, w_v, b_v, w_s, b_s, reverse, lv, ls, pv, ps,
                                 err, errlen);
    if (!rc) rc = check_dist(pv, n, "kl_loss pred", err, errlen);
    if (!rc) rc = check_dist(target_v, n, "kl_loss target", err, errlen);
    if (!rc) rc = check_dist(ps, n, "kl_loss pred", err, errlen);
    if (!rc) rc = check_dist(target_s, n, "kl_loss target", err, errlen);
    if (!rc) {
        *loss_out = kl_grad(pv, target_v, n, eps, dv) + kl_grad(ps, target_s, n, eps, dso);
        memset(g_w_u, 0, sizeof(double) * 2 * d * d_h);
        memset(g_b_u, 0, sizeof(double) * d_h);
        memset(g_w_v, 0, sizeof(double) * d_h);
        memset(g_w_s, 0, sizeof(double) * d_h);
        *g_b_v = 0.0;
        *g_b_s = 0.0;
        for (int64_t t = 0; t < n; ++t) {
            const double dlv = dv[t];
            const double dls = dso[reverse ? n - 1 - t : t]; /* token t fed offset slot o(t) */
            /* y = X W_U (matrix.hpp:56-71 order) then + b_U, as indexer_forward_features :86-90 */
            for (int64_t h = 0; h < d_h; ++h) y[h] = 0.0;
            for (int64_t c = 0; c < 2 * d; ++c) {
                const double xc = c < d ? k[t * ks + c] : v[t * vs + (c - d)];
                const double* wr = w_u + c * d_h;
                for (int64_t h = 0; h < d_h; ++h) y[h] += xc * wr[h];
            }
            for (int64_t h = 0; h < d_h; ++h) y[h] += b_u[h];
            for (int64_t h = 0; h < d_h; ++h) {
                const double z = vso_silu(y[h]);
                g_w_v[h] += dlv * z;
                g_w_s[h] += dls * z;
                const double dy = (dlv * w_v[h] + dls * w_s[h]) * silu_deriv(y[h]);
                g_b_u[h] += dy;
                y[h] = dy;
            }
            *g_b_v += dlv;
            *g_b_s += dls;
            for (int64_t c = 0; c < 2 * d; ++c) {
                const double xc = c < d ? k[t * ks + c] : v[t * vs + (c - d)];
                double* gr = g_w_u + c * d_h;
                for (int64_t h = 0; h < d_h; ++h) gr[h] += xc * y[h];
            }
        }
    }
    free(lv); free(ls); free(pv); free(ps); free(dv); free(dso); free(y);
    return rc;
}

/* optimizer_step (indexer.hpp:347-363) over a flat parameter vector; lr from learning_rate
 * (:322-329) is passed in. */
void vso_adamw_step(int64_t count, double* p, const double* g, double* m, double* v, int64_t step_index, double lr,
                    double beta1, double beta2, double adam_eps, double weight_decay) {
    const double t = (double)(step_index + 1);
    const double bc1 = 1.0 - pow(beta1, t), bc2 = 1.0 - pow(beta2, t);
    for (int64_t i = 0; i < count; ++i) {
        m[i] = beta1 * m[i] + (1.0 - beta1) * g[i];
        v[i] = beta2 * v[i] + (1.0 - beta2) * g[i] * g[i];
        const double mhat = m[i] / bc1, vhat = v[i] / bc2;
        p[i] -= lr * (mhat / (sqrt(vhat) + adam_eps) + weight_decay * p[i]);
    }
}
