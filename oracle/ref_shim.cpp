// ref_shim.cpp — TEST INFRASTRUCTURE ONLY.
//
// extern "C" wrappers that call the UNMODIFIED reference library, compiled straight
// from /root/reference/proj/include (header-only C++20; nothing is copied into this
// repo). Built by oracle/Makefile into oracle/_ref/libvspref.so. Used to pin the C
// oracle (tests/golden/make_golden.py) and as the reference CPU arm of bench.py.
//
// Argument conventions match oracle/vsp_oracle.c: matrices are (base, row_stride)
// f64, index lists are int64, errors return 1 with the exception text in err.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <thread>
#include <vector>

#include "vsprefill/attention.hpp"
#include "vsprefill/indexer.hpp"
#include "vsprefill/merge.hpp"
#include "vsprefill/rope.hpp"
#include "vsprefill/sparsity.hpp"
#include "vsprefill/tensor_io.hpp"
#include "vsprefill/vsaggregate.hpp"

namespace {

int set_err(char* err, size_t errlen, const char* msg) {
    if (err && errlen) {
        std::strncpy(err, msg, errlen - 1);
        err[errlen - 1] = '\0';
    }
    return 1;
}

vsp::Matrix gather(const double* base, int64_t stride, int64_t rows, int64_t cols) {
    vsp::Matrix m(static_cast<size_t>(rows), static_cast<size_t>(cols));
    for (int64_t t = 0; t < rows; ++t)
        std::memcpy(m.row_ptr(t), base + t * stride, sizeof(double) * cols);
    return m;
}

std::vector<size_t> idx(const int64_t* p, int64_t n) {
    std::vector<size_t> v(static_cast<size_t>(n));
    for (int64_t i = 0; i < n; ++i) v[i] = static_cast<size_t>(p[i]);
    return v;
}

template <class F>
int guarded(char* err, size_t errlen, F&& f) {
    try {
        f();
        return 0;
    } catch (const std::exception& e) {
        return set_err(err, errlen, e.what());
    }
}

// Formats: 1 = std::invalid_argument, 2 = std::runtime_error (the types the tests assert).
template <class F>
int typed(char* err, size_t errlen, F&& f) {
    try {
        f();
        return 0;
    } catch (const std::invalid_argument& e) {
        return set_err(err, errlen, e.what());
    } catch (const std::runtime_error& e) {
        set_err(err, errlen, e.what());
        return 2;
    }
}

}  // namespace

extern "C" {

int64_t vspref_merge_row_columns(const int64_t* iv, int64_t kv, const int64_t* is, int64_t ks,
                                 int64_t i, int64_t* out, char* err, size_t errlen) {
    int64_t cnt = -1;
    guarded(err, errlen, [&] {
        auto cols = vsp::merge_row_columns(idx(iv, kv), idx(is, ks), static_cast<size_t>(i));
        for (size_t t = 0; t < cols.size(); ++t) out[t] = static_cast<int64_t>(cols[t]);
        cnt = static_cast<int64_t>(cols.size());
    });
    return cnt;
}

int vspref_merge_path_partition(const int64_t* a, int64_t na, const int64_t* b, int64_t nb,
                                int64_t p, int64_t* cuts, char* err, size_t errlen) {
    return guarded(err, errlen, [&] {
        auto c = vsp::merge_path_partition(idx(a, na), idx(b, nb), static_cast<size_t>(p));
        for (size_t s = 0; s < c.size(); ++s) {
            cuts[2 * s] = static_cast<int64_t>(c[s].a);
            cuts[2 * s + 1] = static_cast<int64_t>(c[s].b);
        }
    });
}

int vspref_blockwise_attention(int64_t n, int64_t d, const double* q, int64_t qs, const double* k,
                               int64_t ks, const double* v, int64_t vs, int64_t block, double* o,
                               int64_t os, char* err, size_t errlen) {
    return guarded(err, errlen, [&] {
        vsp::AttentionInputs in(gather(q, qs, n, d), gather(k, ks, n, d), gather(v, vs, n, d));
        auto out = vsp::blockwise_attention(in, static_cast<size_t>(block));
        for (int64_t t = 0; t < n; ++t) std::memcpy(o + t * os, out.o.row_ptr(t), sizeof(double) * d);
    });
}

int vspref_sparse_attention(int64_t n, int64_t d, const double* q, int64_t qs, const double* k,
                            int64_t ks, const double* v, int64_t vs, const int64_t* iv, int64_t kv,
                            const int64_t* is, int64_t ksl, int64_t block, double* o, int64_t os,
                            char* err, size_t errlen) {
    return guarded(err, errlen, [&] {
        vsp::AttentionInputs in(gather(q, qs, n, d), gather(k, ks, n, d), gather(v, vs, n, d));
        vsp::SparsePattern pat{idx(iv, kv), idx(is, ksl)};
        auto out = vsp::sparse_attention(in, pat, static_cast<size_t>(block));
        for (int64_t t = 0; t < n; ++t) std::memcpy(o + t * os, out.o.row_ptr(t), sizeof(double) * d);
    });
}

// attention.hpp:52-75 + :198-215 (materialises n x n; small n only)
int vspref_attention_recall(int64_t n, int64_t d, const double* q, int64_t qs, const double* k,
                            int64_t ks, const int64_t* iv, int64_t kv, const int64_t* is,
                            int64_t ksl, double* recall, char* err, size_t errlen) {
    return guarded(err, errlen, [&] {
        auto a = vsp::attention_matrix(gather(q, qs, n, d), gather(k, ks, n, d));
        *recall = vsp::attention_recall(a, vsp::SparsePattern{idx(iv, kv), idx(is, ksl)});
    });
}

static vsp::BudgetConfig budget(double tau_v, double tau_s, int64_t min_b, int64_t max_b) {
    vsp::BudgetConfig c;
    c.tau_v = tau_v;
    c.tau_s = tau_s;
    c.min_budget = static_cast<size_t>(min_b < 0 ? 0 : min_b);
    if (max_b >= 0) c.max_budget = static_cast<size_t>(max_b);
    return c;
}

int vspref_cumulative_budget(const double* scores, int64_t n, double tau, double tau_v,
                             double tau_s, int64_t min_b, int64_t max_b, int64_t* k_out, char* err,
                             size_t errlen) {
    return guarded(err, errlen, [&] {
        std::vector<double> s(scores, scores + n);
        *k_out = static_cast<int64_t>(vsp::cumulative_budget(s, tau, budget(tau_v, tau_s, min_b, max_b)));
    });
}

int vspref_topk_indices(const double* scores, int64_t n, int64_t k, int64_t* out, char* err,
                        size_t errlen) {
    return guarded(err, errlen, [&] {
        std::vector<double> s(scores, scores + n);
        auto r = vsp::topk_indices(s, static_cast<size_t>(k));
        for (size_t t = 0; t < r.size(); ++t) out[t] = static_cast<int64_t>(r[t]);
    });
}

int vspref_select_pattern(const double* sv, const double* ss, int64_t n, double tau_v, double tau_s,
                          int64_t min_b, int64_t max_b, int64_t* iv, int64_t* kv, int64_t* is,
                          int64_t* ks, char* err, size_t errlen) {
    return guarded(err, errlen, [&] {
        vsp::VSScores sc;
        sc.vertical.assign(sv, sv + n);
        sc.slash.assign(ss, ss + n);
        sc.normalized = true;
        auto sel = vsp::select_pattern(sc, budget(tau_v, tau_s, min_b, max_b));
        for (size_t t = 0; t < sel.i_v.size(); ++t) iv[t] = static_cast<int64_t>(sel.i_v[t]);
        for (size_t t = 0; t < sel.i_s.size(); ++t) is[t] = static_cast<int64_t>(sel.i_s[t]);
        *kv = static_cast<int64_t>(sel.i_v.size());
        *ks = static_cast<int64_t>(sel.i_s.size());
    });
}

static vsp::IndexerParams params(int64_t d, int64_t d_h, const double* w_u, const double* b_u,
                                 const double* w_v, double b_v, const double* w_s, double b_s) {
    vsp::IndexerParams p;
    p.d_h = static_cast<size_t>(d_h);
    p.w_u = vsp::Matrix(static_cast<size_t>(2 * d), static_cast<size_t>(d_h),
                        std::vector<double>(w_u, w_u + 2 * d * d_h));
    p.b_u.assign(b_u, b_u + d_h);
    p.w_v.assign(w_v, w_v + d_h);
    p.b_v = b_v;
    p.w_s.assign(w_s, w_s + d_h);
    p.b_s = b_s;
    return p;
}

int vspref_indexer_forward(int64_t n, int64_t d, const double* k, int64_t ks, const double* v,
                           int64_t vs, int64_t d_h, const double* w_u, const double* b_u,
                           const double* w_v, double b_v, const double* w_s, double b_s,
                           int reverse, double* logits_v, double* logits_s, double* pred_v,
                           double* pred_s, char* err, size_t errlen) {
    return guarded(err, errlen, [&] {
        auto acts = vsp::indexer_forward(params(d, d_h, w_u, b_u, w_v, b_v, w_s, b_s),
                                         gather(k, ks, n, d), gather(v, vs, n, d),
                                         reverse ? vsp::SlashMapping::Reverse : vsp::SlashMapping::Identity);
        std::copy(acts.logits_v.begin(), acts.logits_v.end(), logits_v);
        std::copy(acts.logits_s.begin(), acts.logits_s.end(), logits_s);
        std::copy(acts.pred_v.begin(), acts.pred_v.end(), pred_v);
        std::copy(acts.pred_s.begin(), acts.pred_s.end(), pred_s);
    });
}

int vspref_aggregate_streaming(int64_t n, int64_t d, const double* q, int64_t qs, const double* k,
                               int64_t ks, int64_t block, int normalized, double* vertical,
                               double* slash, char* err, size_t errlen) {
    return guarded(err, errlen, [&] {
        vsp::Matrix qm = gather(q, qs, n, d), km = gather(k, ks, n, d);
        vsp::AttentionInputs in(qm, km, km);  // V is unused by aggregation
        auto s = vsp::aggregate_streaming(in, static_cast<size_t>(block), normalized != 0);
        std::copy(s.vertical.begin(), s.vertical.end(), vertical);
        std::copy(s.slash.begin(), s.slash.end(), slash);
    });
}

int vspref_combine_scores(int64_t heads, int64_t n, const double* v_in, const double* s_in, int mean,
                          double* v_out, double* s_out, char* err, size_t errlen) {
    return guarded(err, errlen, [&] {
        std::vector<vsp::VSScores> hs(static_cast<size_t>(heads));
        for (int64_t h = 0; h < heads; ++h) {
            hs[h].vertical.assign(v_in + h * n, v_in + (h + 1) * n);
            hs[h].slash.assign(s_in + h * n, s_in + (h + 1) * n);
            hs[h].normalized = true;
        }
        auto c = vsp::combine_scores(hs, mean ? vsp::GroupReduce::Mean : vsp::GroupReduce::Sum);
        std::copy(c.vertical.begin(), c.vertical.end(), v_out);
        std::copy(c.slash.begin(), c.slash.end(), s_out);
    });
}

// Whole-layer VS prefill through the reference API, threaded over heads with
// std::thread (each reference call is a pure per-head function).
// Tensors are token-major f64: q [n, hq, d], k/v [n, hkv, d]; indexer params per KV
// head: w_u [hkv, 2d, d_h], b_u/w_v/w_s [hkv, d_h], b_v/b_s [hkv]. Output o [n, hq, d].
// k_v/k_s (out, [hkv]) report the selected budgets.
int vspref_layer_vs_prefill(int64_t n, int64_t hq, int64_t hkv, int64_t d, const double* q,
                            const double* k, const double* v, int64_t d_h, const double* w_u,
                            const double* b_u, const double* w_v, const double* b_v,
                            const double* w_s, const double* b_s, const double* tau_v, const double* tau_s,
                            int64_t min_b, int64_t max_b, int64_t block, int n_threads, double* o,
                            int64_t* k_v, int64_t* k_s, char* err, size_t errlen) {
    const int64_t group = hq / hkv;
    std::vector<vsp::SparsePattern> pats(static_cast<size_t>(hkv));
    std::vector<std::string> errs;
    std::atomic<int64_t> next{0};
    std::atomic<int> failed{0};
    std::string first_err;
    auto run_pool = [&](int64_t items, auto&& body) {
        next = 0;
        std::vector<std::thread> pool;
        const int nt = std::max(1, std::min<int>(n_threads, static_cast<int>(items)));
        for (int t = 0; t < nt; ++t)
            pool.emplace_back([&] {
                for (int64_t it; (it = next.fetch_add(1)) < items;) {
                    try {
                        body(it);
                    } catch (const std::exception& e) {
                        if (failed.exchange(1) == 0) first_err = e.what();
                    }
                }
            });
        for (auto& th : pool) th.join();
    };
    run_pool(hkv, [&](int64_t g) {
        auto p = params(d, d_h, w_u + g * 2 * d * d_h, b_u + g * d_h, w_v + g * d_h, b_v[g],
                        w_s + g * d_h, b_s[g]);
        auto acts = vsp::indexer_forward(p, gather(k + g * d, hkv * d, n, d),
                                         gather(v + g * d, hkv * d, n, d));
        vsp::VSScores sc{acts.pred_v, acts.pred_s, true};
        auto sel = vsp::select_pattern(sc, budget(tau_v[g], tau_s[g], min_b, max_b));
        k_v[g] = static_cast<int64_t>(sel.k_v());
        k_s[g] = static_cast<int64_t>(sel.k_s());
        pats[g] = sel.pattern();
    });
    if (failed) return set_err(err, errlen, first_err.c_str());
    run_pool(hq, [&](int64_t h) {
        const int64_t g = h / group;
        vsp::AttentionInputs in(gather(q + h * d, hq * d, n, d), gather(k + g * d, hkv * d, n, d),
                                gather(v + g * d, hkv * d, n, d));
        auto out = vsp::sparse_attention(in, pats[g], static_cast<size_t>(block));
        for (int64_t t = 0; t < n; ++t)
            std::memcpy(o + (t * hq + h) * d, out.o.row_ptr(t), sizeof(double) * d);
    });
    if (failed) return set_err(err, errlen, first_err.c_str());
    return 0;
}

// ---- the layer in stages, for the bench's reference arm (bounded samples of one layer) ----
// Each stage calls the reference per head exactly as the reference's own callers do
// (indexer_forward -> select_pattern -> sparse_attention, tools/vsprefill.cpp:154-185), threaded
// over heads with std::thread. Tensors are token-major f64 ([tokens, heads, d]).

}  // extern "C"

namespace {
// item_s (optional, [items]): wall seconds of each item's call on its worker thread.
template <class Body>
int parallel_heads(int64_t items, int n_threads, char* err, size_t errlen, Body&& body, double* item_s = nullptr) {
    std::atomic<int64_t> next{0};
    std::atomic<int> failed{0};
    std::string first_err;
    std::vector<std::thread> pool;
    const int nt = std::max(1, std::min<int>(n_threads, static_cast<int>(items)));
    for (int t = 0; t < nt; ++t)
        pool.emplace_back([&] {
            for (int64_t it; (it = next.fetch_add(1)) < items;) {
                const auto t0 = std::chrono::steady_clock::now();
                try {
                    body(it);
                } catch (const std::exception& e) {
                    if (failed.exchange(1) == 0) first_err = e.what();
                }
                if (item_s)
                    item_s[it] = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
            }
        });
    for (auto& th : pool) th.join();
    return failed ? set_err(err, errlen, first_err.c_str()) : 0;
}
}  // namespace

extern "C" {

// indexer_forward (indexer.hpp:116-120) of every KV head over `len` tokens: pred/logits [hkv, len].
int vspref_layer_indexer(int64_t len, int64_t hkv, int64_t d, const double* k, const double* v, int64_t d_h,
                         const double* w_u, const double* b_u, const double* w_v, const double* b_v,
                         const double* w_s, const double* b_s, int n_threads, double* pred_v, double* pred_s,
                         double* head_s, char* err, size_t errlen) {
    return parallel_heads(hkv, n_threads, err, errlen, [&](int64_t g) {
        auto p = params(d, d_h, w_u + g * 2 * d * d_h, b_u + g * d_h, w_v + g * d_h, b_v[g], w_s + g * d_h, b_s[g]);
        auto acts = vsp::indexer_forward(p, gather(k + g * d, hkv * d, len, d), gather(v + g * d, hkv * d, len, d));
        std::copy(acts.pred_v.begin(), acts.pred_v.end(), pred_v + g * len);
        std::copy(acts.pred_s.begin(), acts.pred_s.end(), pred_s + g * len);
    }, head_s);
}

// select_pattern (sparsity.hpp:105-114) of every KV head: lists [hkv, cap] int64 + counts.
int vspref_layer_select(int64_t n, int64_t hkv, const double* pred_v, const double* pred_s, const double* tau_v,
                        const double* tau_s, int64_t min_b, int64_t max_b, int64_t cap, int n_threads,
                        int64_t* iv, int64_t* kv, int64_t* is, int64_t* ks, char* err, size_t errlen) {
    return parallel_heads(hkv, n_threads, err, errlen, [&](int64_t g) {
        vsp::VSScores sc{std::vector<double>(pred_v + g * n, pred_v + (g + 1) * n),
                         std::vector<double>(pred_s + g * n, pred_s + (g + 1) * n), true};
        auto sel = vsp::select_pattern(sc, budget(tau_v[g], tau_s[g], min_b, max_b));
        if (static_cast<int64_t>(sel.i_v.size()) > cap || static_cast<int64_t>(sel.i_s.size()) > cap)
            throw std::invalid_argument("layer_select: cap too small");
        kv[g] = static_cast<int64_t>(sel.i_v.size());
        ks[g] = static_cast<int64_t>(sel.i_s.size());
        for (size_t t = 0; t < sel.i_v.size(); ++t) iv[g * cap + t] = static_cast<int64_t>(sel.i_v[t]);
        for (size_t t = 0; t < sel.i_s.size(); ++t) is[g * cap + t] = static_cast<int64_t>(sel.i_s[t]);
    });
}

// sparse_attention (attention.hpp:150-194) of every Q head over the first `rows` tokens with the
// given per-KV-head patterns (selected on the full sequence): causality makes these rows of the
// output identical to the full layer's. o [rows, hq, d].
int vspref_layer_sparse(int64_t rows, int64_t hq, int64_t hkv, int64_t d, const double* q, const double* k,
                        const double* v, const int64_t* iv, const int64_t* kv, const int64_t* is,
                        const int64_t* ks, int64_t cap, int64_t block, int n_threads, double* o, double* head_s,
                        char* err, size_t errlen) {
    const int64_t group = hq / hkv;
    std::vector<vsp::SparsePattern> pats(static_cast<size_t>(hkv));
    for (int64_t g = 0; g < hkv; ++g) {
        pats[g].i_v = idx(iv + g * cap, kv[g]);
        pats[g].i_s = idx(is + g * cap, ks[g]);
    }
    return parallel_heads(hq, n_threads, err, errlen, [&](int64_t h) {
        const int64_t g = h / group;
        vsp::AttentionInputs in(gather(q + h * d, hq * d, rows, d), gather(k + g * d, hkv * d, rows, d),
                                gather(v + g * d, hkv * d, rows, d));
        auto out = vsp::sparse_attention(in, pats[g], static_cast<size_t>(block));
        for (int64_t t = 0; t < rows; ++t) std::memcpy(o + (t * hq + h) * d, out.o.row_ptr(t), sizeof(double) * d);
    }, head_s);
}

// Dense causal layer through blockwise_attention (attention.hpp:96-145), threaded.
int vspref_layer_dense(int64_t n, int64_t hq, int64_t hkv, int64_t d, const double* q,
                       const double* k, const double* v, int64_t block, int n_threads, double* o,
                       char* err, size_t errlen) {
    const int64_t group = hq / hkv;
    std::atomic<int64_t> next{0};
    std::atomic<int> failed{0};
    std::string first_err;
    std::vector<std::thread> pool;
    const int nt = std::max(1, std::min<int>(n_threads, static_cast<int>(hq)));
    for (int t = 0; t < nt; ++t)
        pool.emplace_back([&] {
            for (int64_t h; (h = next.fetch_add(1)) < hq;) {
                try {
                    const int64_t g = h / group;
                    vsp::AttentionInputs in(gather(q + h * d, hq * d, n, d),
                                            gather(k + g * d, hkv * d, n, d),
                                            gather(v + g * d, hkv * d, n, d));
                    auto out = vsp::blockwise_attention(in, static_cast<size_t>(block));
                    for (int64_t r = 0; r < n; ++r)
                        std::memcpy(o + (r * hq + h) * d, out.o.row_ptr(r), sizeof(double) * d);
                } catch (const std::exception& e) {
                    if (failed.exchange(1) == 0) first_err = e.what();
                }
            }
        });
    for (auto& th : pool) th.join();
    if (failed) return set_err(err, errlen, first_err.c_str());
    return 0;
}

// ---- interchange formats (tensor_io.hpp, indexer.hpp:450-499, sparsity.hpp:187-245) ----

int vspref_write_matrix(const char* path, int64_t rows, int64_t cols, const double* data, char* err,
                        size_t errlen) {
    return typed(err, errlen, [&] { vsp::write_tensor(path, gather(data, cols, rows, cols)); });
}

int vspref_write_vector(const char* path, int64_t n, const double* data, char* err, size_t errlen) {
    return typed(err, errlen, [&] { vsp::write_tensor(path, std::vector<double>(data, data + n)); });
}

// rank 2 -> read_tensor, rank 1 -> read_vector; shape_out[0..1] and data (cap values)
int vspref_read_tensor(const char* path, int rank, int64_t* shape_out, double* data, int64_t cap, char* err,
                       size_t errlen) {
    return typed(err, errlen, [&] {
        std::vector<double> v;
        if (rank == 2) {
            vsp::Matrix m = vsp::read_tensor(path);
            shape_out[0] = static_cast<int64_t>(m.rows);
            shape_out[1] = static_cast<int64_t>(m.cols);
            v = std::move(m.data);
        } else {
            v = vsp::read_vector(path);
            shape_out[0] = static_cast<int64_t>(v.size());
        }
        std::memcpy(data, v.data(), sizeof(double) * std::min<int64_t>(cap, static_cast<int64_t>(v.size())));
    });
}

int vspref_save_checkpoint(const char* path, int64_t in_dim, int64_t d_h, const double* w_u, const double* b_u,
                           const double* w_v, double b_v, const double* w_s, double b_s, char* err, size_t errlen) {
    return typed(err, errlen, [&] {
        vsp::IndexerParams p;
        p.d_h = static_cast<size_t>(d_h);
        p.w_u = gather(w_u, d_h, in_dim, d_h);
        p.b_u.assign(b_u, b_u + d_h);
        p.w_v.assign(w_v, w_v + d_h);
        p.w_s.assign(w_s, w_s + d_h);
        p.b_v = b_v;
        p.b_s = b_s;
        vsp::save_checkpoint(p, path);
    });
}

// dims_out = {in_dim, d_h}; buffers sized by the caller (query with a first call, cap 0)
int vspref_load_checkpoint(const char* path, int64_t* dims_out, int64_t cap_dh, double* w_u, double* b_u,
                           double* w_v, double* b_v, double* w_s, double* b_s, char* err, size_t errlen) {
    return typed(err, errlen, [&] {
        vsp::IndexerParams p = vsp::load_checkpoint(path);
        dims_out[0] = static_cast<int64_t>(p.in_dim());
        dims_out[1] = static_cast<int64_t>(p.d_h);
        if (cap_dh < static_cast<int64_t>(p.d_h)) return;
        std::memcpy(w_u, p.w_u.data.data(), sizeof(double) * p.w_u.data.size());
        std::memcpy(b_u, p.b_u.data(), sizeof(double) * p.d_h);
        std::memcpy(w_v, p.w_v.data(), sizeof(double) * p.d_h);
        std::memcpy(w_s, p.w_s.data(), sizeof(double) * p.d_h);
        *b_v = p.b_v;
        *b_s = p.b_s;
    });
}

int vspref_write_indices(const char* path, const int64_t* iv, int64_t kv, const int64_t* is, int64_t ks, char* err,
                         size_t errlen) {
    return typed(err, errlen, [&] {
        vsp::SelectedIndices sel;
        sel.i_v = idx(iv, kv);
        sel.i_s = idx(is, ks);
        vsp::write_indices(path, sel);
    });
}

int vspref_read_indices(const char* path, int64_t* iv, int64_t* kv, int64_t* is, int64_t* ks, int64_t cap,
                        char* err, size_t errlen) {
    return typed(err, errlen, [&] {
        vsp::SelectedIndices sel = vsp::read_indices(std::string(path));
        *kv = static_cast<int64_t>(sel.i_v.size());
        *ks = static_cast<int64_t>(sel.i_s.size());
        for (int64_t t = 0; t < std::min<int64_t>(cap, *kv); ++t) iv[t] = static_cast<int64_t>(sel.i_v[t]);
        for (int64_t t = 0; t < std::min<int64_t>(cap, *ks); ++t) is[t] = static_cast<int64_t>(sel.i_s[t]);
    });
}

// ---- RoPE (rope.hpp:63-79): same argument convention as vso_apply_rope
int vspref_apply_rope(int64_t n, int64_t d, const double* x, int64_t xs, const int64_t* positions, double base,
                      double* out, int64_t os, char* err, size_t errlen) {
    return guarded(err, errlen, [&] {
        const vsp::RopeConfig cfg(static_cast<size_t>(d), base);
        const vsp::Matrix m = gather(x, xs, n, d);
        vsp::Matrix r = positions ? vsp::apply_rope(m, idx(positions, n), cfg) : vsp::apply_rope(m, cfg);
        for (int64_t t = 0; t < n; ++t) std::memcpy(out + t * os, r.row_ptr(t), sizeof(double) * d);
    });
}

// ---- distillation: indexer_backward_loss (indexer.hpp:265-272) with the product-path KL loss,
// gradients flattened like vso_indexer_backward
int vspref_indexer_backward(int64_t n, int64_t d, const double* k, int64_t ks, const double* v, int64_t vs,
                            int64_t d_h, const double* w_u, const double* b_u, const double* w_v, double b_v,
                            const double* w_s, double b_s, int reverse, const double* target_v,
                            const double* target_s, double eps, double* loss_out, double* g_w_u, double* g_b_u,
                            double* g_w_v, double* g_b_v, double* g_w_s, double* g_b_s, char* err, size_t errlen) {
    return guarded(err, errlen, [&] {
        const vsp::IndexerParams p = params(d, d_h, w_u, b_u, w_v, b_v, w_s, b_s);
        const auto acts = vsp::indexer_forward(p, gather(k, ks, n, d), gather(v, vs, n, d),
                                               reverse ? vsp::SlashMapping::Reverse : vsp::SlashMapping::Identity);
        const std::vector<double> tv(target_v, target_v + n), ts(target_s, target_s + n);
        double loss = 0.0;
        const vsp::IndexerGrads g = vsp::indexer_backward_loss(p, acts, tv, ts, vsp::make_kl_loss(eps), &loss);
        *loss_out = loss;
        std::copy(g.w_u.data.begin(), g.w_u.data.end(), g_w_u);
        std::copy(g.b_u.begin(), g.b_u.end(), g_b_u);
        std::copy(g.w_v.begin(), g.w_v.end(), g_w_v);
        std::copy(g.w_s.begin(), g.w_s.end(), g_w_s);
        *g_b_v = g.b_v;
        *g_b_s = g.b_s;
    });
}

// ---- optimizer_step (indexer.hpp:347-363) on one head's parameters; params and the Adam
// moments are updated in place (flattened as W_U | b_U | w_v | b_v | w_s | b_s)
int vspref_optimizer_step(int64_t d, int64_t d_h, double* flat_p, const double* flat_g, double* flat_m,
                          double* flat_v, int64_t step, int64_t steps, int64_t warmup, double lr_peak, char* err,
                          size_t errlen) {
    return guarded(err, errlen, [&] {
        const int64_t nw = 2 * d * d_h;
        auto unflat = [&](const double* f) {
            vsp::IndexerParams p = params(d, d_h, f, f + nw, f + nw + d_h, f[nw + 2 * d_h], f + nw + 2 * d_h + 1,
                                          f[nw + 3 * d_h + 1]);
            return p;
        };
        auto grads = [&](const double* f) {
            vsp::IndexerGrads g;
            vsp::IndexerParams q = unflat(f);
            g.w_u = q.w_u; g.b_u = q.b_u; g.w_v = q.w_v; g.b_v = q.b_v; g.w_s = q.w_s; g.b_s = q.b_s;
            return g;
        };
        vsp::IndexerParams p = unflat(flat_p);
        vsp::OptState st{grads(flat_m), grads(flat_v)};
        vsp::TrainConfig cfg;
        cfg.steps = static_cast<size_t>(steps);
        cfg.warmup_steps = static_cast<size_t>(warmup);
        cfg.lr_peak = lr_peak;
        vsp::optimizer_step(p, grads(flat_g), st, static_cast<size_t>(step), cfg);
        auto flat = [&](const vsp::IndexerParams& q, double* f) {
            std::copy(q.w_u.data.begin(), q.w_u.data.end(), f);
            std::copy(q.b_u.begin(), q.b_u.end(), f + nw);
            std::copy(q.w_v.begin(), q.w_v.end(), f + nw + d_h);
            f[nw + 2 * d_h] = q.b_v;
            std::copy(q.w_s.begin(), q.w_s.end(), f + nw + 2 * d_h + 1);
            f[nw + 3 * d_h + 1] = q.b_s;
        };
        flat(p, flat_p);
        auto flat_g2 = [&](const vsp::IndexerGrads& q, double* f) {
            std::copy(q.w_u.data.begin(), q.w_u.data.end(), f);
            std::copy(q.b_u.begin(), q.b_u.end(), f + nw);
            std::copy(q.w_v.begin(), q.w_v.end(), f + nw + d_h);
            f[nw + 2 * d_h] = q.b_v;
            std::copy(q.w_s.begin(), q.w_s.end(), f + nw + 2 * d_h + 1);
            f[nw + 3 * d_h + 1] = q.b_s;
        };
        flat_g2(st.m, flat_m);
        flat_g2(st.v, flat_v);
    });
}

// learning_rate (indexer.hpp:322-329)
double vspref_learning_rate(int64_t step, int64_t steps, int64_t warmup, double lr_peak) {
    vsp::TrainConfig cfg;
    cfg.steps = static_cast<size_t>(steps);
    cfg.warmup_steps = static_cast<size_t>(warmup);
    cfg.lr_peak = lr_peak;
    return vsp::learning_rate(static_cast<size_t>(step), cfg);
}

}  // extern "C"
