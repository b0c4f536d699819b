// vsprefill_gpu.hpp — C++ drop-in shim: the reference's hot-path signatures on the B200.
//
// Include AFTER the reference headers (it uses vsp::Matrix, vsp::AttentionInputs, ... from
// /root/reference/proj/include/vsprefill) and link libvsp_gpu.so + cudart. Each function has
// the signature of the reference function it replaces, so reference call sites and test
// bodies can be re-pointed from `vsp::` to `vsp::gpu::` unchanged:
//
//   vsp::gpu::indexer_forward      <- vsp::indexer_forward      indexer.hpp:116
//   vsp::gpu::select_pattern       <- vsp::select_pattern       sparsity.hpp:105
//   vsp::gpu::cumulative_budget    <- vsp::cumulative_budget    sparsity.hpp:51
//   vsp::gpu::topk_indices         <- vsp::topk_indices         sparsity.hpp:83
//   vsp::gpu::merge_row_columns    <- vsp::merge_row_columns    merge.hpp:18
//   vsp::gpu::merge_path_partition <- vsp::merge_path_partition merge.hpp:69 (host)
//   vsp::gpu::combine_scores       <- vsp::combine_scores       vsaggregate.hpp:133
//   vsp::gpu::sparse_attention     <- vsp::sparse_attention     attention.hpp:150
//   vsp::gpu::blockwise_attention  <- vsp::blockwise_attention  attention.hpp:96
//   vsp::gpu::attention_recall     <- vsp::attention_recall     attention.hpp:198 (from inputs)
//   vsp::gpu::aggregate_streaming  <- vsp::aggregate_streaming  vsaggregate.hpp:62
//   vsp::gpu::apply_rope           <- vsp::apply_rope           rope.hpp:63-79
//   vsp::gpu::indexer_backward     <- vsp::indexer_backward     indexer.hpp:275 (Forward KL)
//   vsp::gpu::optimizer_step       <- vsp::optimizer_step       indexer.hpp:347
//   vsp::gpu::{write,read}_tensor, read_vector, save/load_checkpoint, write/read_indices
//                                  <- tensor_io.hpp, indexer.hpp:450-499, sparsity.hpp:187-245
//
// Host f64 data is converted to the device formats (bf16 Q/K/V/W_U, fp32 scores) on the way
// in and widened back to f64 on the way out, so results carry the GPU path's stated
// tolerances; index sets from select_pattern are bit-exact for scores that
// are exactly representable in fp32. Errors: VSP_EINVAL -> std::invalid_argument with the
// reference's message, anything else -> std::runtime_error. `block` arguments are accepted
// for signature compatibility; the GPU tiling is fixed (results do not depend on it, as in
// the reference, test_attention.cpp:145-155). The single-head API runs on the batched
// kernels as one-head groups (one KV head, one Q head).
#pragma once

#include <cuda_runtime.h>
#include <cuda_bf16.h>

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "vsp_gpu.h"

namespace vsp::gpu {

namespace detail {

inline void check(int rc) {
    if (rc == VSP_OK) return;
    if (rc == VSP_EINVAL) throw std::invalid_argument(vsp_last_error());
    throw std::runtime_error(vsp_last_error());
}
inline void cuda(cudaError_t e) {
    if (e != cudaSuccess) throw std::runtime_error(std::string("vsp::gpu: ") + cudaGetErrorString(e));
}

inline vsp_ctx* context() {
    static vsp_ctx* ctx = [] {
        vsp_ctx* c = nullptr;
        int dev = 0;
        cudaGetDevice(&dev);
        check(vsp_create(&c, dev));
        return c;
    }();
    return ctx;
}

struct Buf {
    void* p = nullptr;
    explicit Buf(size_t bytes) { cuda(cudaMalloc(&p, bytes ? bytes : 16)); }
    ~Buf() { cudaFree(p); }
    Buf(const Buf&) = delete;
    Buf& operator=(const Buf&) = delete;
    template <class T>
    T* as() const { return static_cast<T*>(p); }
};

// rows x cols f64 -> device bf16 laid out [rows, copies, cols] (head dimension `copies`)
inline std::unique_ptr<Buf> upload_bf16(const Matrix& m, int copies = 1) {
    std::vector<__nv_bfloat16> h(m.rows * copies * m.cols);
    for (size_t t = 0; t < m.rows; ++t)
        for (int c = 0; c < copies; ++c)
            for (size_t x = 0; x < m.cols; ++x) h[(t * copies + c) * m.cols + x] = __float2bfloat16(static_cast<float>(m(t, x)));
    auto b = std::make_unique<Buf>(h.size() * sizeof(__nv_bfloat16));
    cuda(cudaMemcpy(b->p, h.data(), h.size() * sizeof(__nv_bfloat16), cudaMemcpyHostToDevice));
    return b;
}
inline std::unique_ptr<Buf> upload_f32(const std::vector<double>& v) {
    std::vector<float> h(v.begin(), v.end());
    auto b = std::make_unique<Buf>(h.size() * sizeof(float));
    cuda(cudaMemcpy(b->p, h.data(), h.size() * sizeof(float), cudaMemcpyHostToDevice));
    return b;
}
inline std::vector<double> download_f32(const Buf& b, size_t n) {
    std::vector<float> h(n);
    cuda(cudaMemcpy(h.data(), b.p, n * sizeof(float), cudaMemcpyDeviceToHost));
    return std::vector<double>(h.begin(), h.end());
}
inline Matrix download_head0(const Buf& o, size_t n, size_t d, int heads) {
    std::vector<__nv_bfloat16> h(n * heads * d);
    cuda(cudaMemcpy(h.data(), o.p, h.size() * sizeof(__nv_bfloat16), cudaMemcpyDeviceToHost));
    Matrix m(n, d);
    for (size_t t = 0; t < n; ++t)
        for (size_t x = 0; x < d; ++x) m(t, x) = static_cast<double>(__bfloat162float(h[t * heads * d + x]));
    return m;
}

}  // namespace detail

// indexer.hpp:116-120. Activations x/y/z are not materialised (they never leave the SM);
// logits and predictions are filled.
inline IndexerActivations indexer_forward(const IndexerParams& p, const Matrix& k, const Matrix& v,
                                          SlashMapping mapping = SlashMapping::Reverse) {
    require(k.same_shape(v), "indexer_forward: K/V shape mismatch");
    p.check_shapes();
    require(k.cols * 2 == p.in_dim(), "indexer_forward: feature width != in_dim");
    require(k.rows >= 1, "indexer_forward: empty input");
    const int n = static_cast<int>(k.rows), d = static_cast<int>(k.cols), dh = static_cast<int>(p.d_h);
    auto dk = detail::upload_bf16(k), dv = detail::upload_bf16(v), dw = detail::upload_bf16(p.w_u);
    auto bu = detail::upload_f32(p.b_u), wv = detail::upload_f32(p.w_v), ws = detail::upload_f32(p.w_s);
    auto bv = detail::upload_f32({p.b_v}), bs = detail::upload_f32({p.b_s});
    detail::Buf av(n * 4), as(n * 4), lv(n * 4), ls(n * 4), wsp(vsp_indexer_workspace_size(n, 1, dh));
    detail::check(vsp_indexer_scores(detail::context(), dk->p, dv->p, n, 1, d, dh, dw->p, bu->as<float>(),
                                     wv->as<float>(), bv->as<float>(), ws->as<float>(), bs->as<float>(),
                                     mapping == SlashMapping::Reverse ? VSP_SLASH_REVERSE : VSP_SLASH_IDENTITY,
                                     av.as<float>(), as.as<float>(), lv.as<float>(), ls.as<float>(), wsp.p, nullptr));
    IndexerActivations a;
    a.mapping = mapping;
    a.logits_v = detail::download_f32(lv, n);
    a.logits_s = detail::download_f32(ls, n);
    a.pred_v = detail::download_f32(av, n);
    a.pred_s = detail::download_f32(as, n);
    return a;
}

// sparsity.hpp:105-114
inline SelectedIndices select_pattern(const VSScores& scores, const BudgetConfig& cfg) {
    require(scores.normalized, "select_pattern: scores must be normalized");
    cfg.check();
    const int n = static_cast<int>(scores.n());
    require(n >= 1, "cumulative_budget: empty scores");
    auto a_v = detail::upload_f32(scores.vertical), a_s = detail::upload_f32(scores.slash);
    detail::Buf iv((n + 1) * 4), is((n + 1) * 4), kv(4), ks(4), wsp(vsp_select_workspace_size(n, 1));
    vsp_budget b{cfg.tau_v, cfg.tau_s, static_cast<int64_t>(cfg.min_budget),
                 cfg.max_budget ? static_cast<int64_t>(*cfg.max_budget) : -1};
    detail::check(vsp_select(detail::context(), a_v->as<float>(), a_s->as<float>(), n, 1, &b, iv.as<int>(),
                             kv.as<int>(), is.as<int>(), ks.as<int>(), n + 1, wsp.p, VSP_VALIDATE, nullptr));
    int hk[2];
    detail::cuda(cudaMemcpy(&hk[0], kv.p, 4, cudaMemcpyDeviceToHost));
    detail::cuda(cudaMemcpy(&hk[1], ks.p, 4, cudaMemcpyDeviceToHost));
    std::vector<int> a(hk[0]), c(hk[1]);
    detail::cuda(cudaMemcpy(a.data(), iv.p, 4 * a.size(), cudaMemcpyDeviceToHost));
    detail::cuda(cudaMemcpy(c.data(), is.p, 4 * c.size(), cudaMemcpyDeviceToHost));
    SelectedIndices sel;
    sel.i_v.assign(a.begin(), a.end());
    sel.i_s.assign(c.begin(), c.end());
    return sel;
}

// sparsity.hpp:51-79: k of one score vector under the cumulative threshold, computed by the
// selection kernel (its vertical direction; the same exactness guard, so bit-identical k
// for scores exactly representable in fp32). The slash direction is fed the same vector.
inline std::size_t cumulative_budget(const std::vector<double>& scores, double tau, const BudgetConfig& cfg) {
    cfg.check();
    require(tau > 0.0 && tau <= 1.0, "cumulative_budget: tau must be in (0, 1]");
    require(!scores.empty(), "cumulative_budget: empty scores");
    const int n = static_cast<int>(scores.size());
    auto a = detail::upload_f32(scores);
    detail::Buf iv((n + 1) * 4), is((n + 1) * 4), kv(4), ks(4), wsp(vsp_select_workspace_size(n, 1));
    vsp_budget b{tau, tau, static_cast<int64_t>(cfg.min_budget), cfg.max_budget ? static_cast<int64_t>(*cfg.max_budget) : -1};
    detail::check(vsp_select(detail::context(), a->as<float>(), a->as<float>(), n, 1, &b, iv.as<int>(), kv.as<int>(),
                             is.as<int>(), ks.as<int>(), n + 1, wsp.p, VSP_VALIDATE, nullptr));
    int k = 0;
    detail::cuda(cudaMemcpy(&k, kv.p, 4, cudaMemcpyDeviceToHost));
    return static_cast<std::size_t>(k);
}

// sparsity.hpp:83-97 (values as fp32 on the device; -0.0 == 0.0 as in the reference)
inline std::vector<std::size_t> topk_indices(const std::vector<double>& scores, std::size_t k) {
    const std::size_t n = scores.size();
    require(k >= 1, "topk_indices: k must be >= 1");
    require(k <= n, "topk_indices: k exceeds score count");
    auto s = detail::upload_f32(scores);
    const int kk = static_cast<int>(k);
    detail::Buf out(k * 4), wsp(vsp_topk_workspace_size(1));
    detail::check(vsp_topk_indices(detail::context(), s->as<float>(), static_cast<int>(n), 1, &kk, out.as<int>(), kk,
                                   wsp.p, nullptr));
    std::vector<int> h(k);
    detail::cuda(cudaMemcpy(h.data(), out.p, 4 * k, cudaMemcpyDeviceToHost));
    return std::vector<std::size_t>(h.begin(), h.end());
}

// merge.hpp:18-56 (one row; the device kernel validates both lists like the reference)
inline std::vector<std::size_t> merge_row_columns(const std::vector<std::size_t>& i_v,
                                                  const std::vector<std::size_t>& i_s, std::size_t i) {
    std::vector<int> a(i_v.begin(), i_v.end()), b(i_s.begin(), i_s.end());
    const int row = static_cast<int>(i), cap = static_cast<int>(a.size() + b.size());
    detail::Buf da(a.size() * 4), db(b.size() * 4), dr(4), out(cap * 4), len(4);
    if (!a.empty()) detail::cuda(cudaMemcpy(da.p, a.data(), a.size() * 4, cudaMemcpyHostToDevice));
    if (!b.empty()) detail::cuda(cudaMemcpy(db.p, b.data(), b.size() * 4, cudaMemcpyHostToDevice));
    detail::cuda(cudaMemcpy(dr.p, &row, 4, cudaMemcpyHostToDevice));
    detail::check(vsp_merge_row_columns(detail::context(), da.as<int>(), static_cast<int>(a.size()), db.as<int>(),
                                        static_cast<int>(b.size()), dr.as<int>(), 1, out.as<int>(), len.as<int>(),
                                        cap, VSP_VALIDATE, nullptr));
    int m = 0;
    detail::cuda(cudaMemcpy(&m, len.p, 4, cudaMemcpyDeviceToHost));
    std::vector<int> h(m);
    if (m) detail::cuda(cudaMemcpy(h.data(), out.p, 4 * m, cudaMemcpyDeviceToHost));
    return std::vector<std::size_t>(h.begin(), h.end());
}

// merge.hpp:69-95 (host code of the C ABI; the device row merge runs the same search)
inline std::vector<MergeCut> merge_path_partition(const std::vector<std::size_t>& a, const std::vector<std::size_t>& b,
                                                  std::size_t p) {
    require(p >= 1, "merge_path_partition: p must be >= 1");
    std::vector<int64_t> x(a.begin(), a.end()), y(b.begin(), b.end()), cuts(2 * (p + 1));
    detail::check(vsp_merge_path_partition(x.data(), static_cast<int64_t>(x.size()), y.data(),
                                           static_cast<int64_t>(y.size()), static_cast<int64_t>(p), cuts.data()));
    std::vector<MergeCut> out(p + 1);
    for (std::size_t s = 0; s <= p; ++s)
        out[s] = {static_cast<std::size_t>(cuts[2 * s]), static_cast<std::size_t>(cuts[2 * s + 1])};
    return out;
}

// vsaggregate.hpp:133-157 (fp32 scores on the device, f64 accumulation in head order)
inline VSScores combine_scores(const std::vector<VSScores>& heads, GroupReduce reduce = GroupReduce::Mean) {
    require(!heads.empty(), "combine_scores: no heads");
    const std::size_t n = heads.front().n();
    const bool normalized = heads.front().normalized;
    std::vector<double> v, s;
    for (const VSScores& h : heads) {
        require(h.n() == n && h.slash.size() == n, "combine_scores: length mismatch");
        require(h.normalized == normalized, "combine_scores: mixed raw/normalized inputs");
        v.insert(v.end(), h.vertical.begin(), h.vertical.end());
        s.insert(s.end(), h.slash.begin(), h.slash.end());
    }
    auto dv = detail::upload_f32(v), ds = detail::upload_f32(s);
    detail::Buf ov(n * 4), os(n * 4);
    detail::check(vsp_combine_scores(detail::context(), dv->as<float>(), ds->as<float>(), static_cast<int>(heads.size()),
                                     static_cast<int>(n), reduce == GroupReduce::Mean ? VSP_REDUCE_MEAN : VSP_REDUCE_SUM,
                                     ov.as<float>(), os.as<float>(), nullptr));
    VSScores out;
    out.vertical = detail::download_f32(ov, n);
    out.slash = detail::download_f32(os, n);
    out.normalized = reduce == GroupReduce::Mean ? normalized : false;
    return out;
}

namespace detail {
// Runs K4 (pat null) or K3 on one head; the row LSEs stay on the device in `lse_out` when given.
inline AttentionOutput attend(const AttentionInputs& in, const SparsePattern* pat,
                              std::unique_ptr<Buf>* lse_out = nullptr) {
    const int n = static_cast<int>(in.n()), d = static_cast<int>(in.d());
    // one head: a single-head group (the kernels pair Q heads; an odd group's last pair holds one)
    auto q = upload_bf16(in.q), k = upload_bf16(in.k), v = upload_bf16(in.v);
    Buf o(static_cast<size_t>(n) * d * 2);
    auto lse_buf = std::make_unique<Buf>(static_cast<size_t>(n) * 4);
    Buf& lse = *lse_buf;
    const float scale = static_cast<float>(in.scale);
    if (!pat) {
        check(vsp_dense_attn_fwd(context(), q->p, k->p, v->p, n, 1, 1, d, scale, o.p, lse.as<float>(), nullptr));
    } else {
        const int cap = static_cast<int>(std::max(pat->i_v.size(), pat->i_s.size())) + 1;
        std::vector<int> hv(cap, 0), hs(cap, 0);
        for (size_t t = 0; t < pat->i_v.size(); ++t) hv[t] = static_cast<int>(pat->i_v[t]);
        for (size_t t = 0; t < pat->i_s.size(); ++t) hs[t] = static_cast<int>(pat->i_s[t]);
        const int cnt[2] = {static_cast<int>(pat->i_v.size()), static_cast<int>(pat->i_s.size())};
        Buf iv(cap * 4), is(cap * 4), kv(4), ks(4), wsp(vsp_vs_attn_workspace_size(n, 1, cap));
        cuda(cudaMemcpy(iv.p, hv.data(), cap * 4, cudaMemcpyHostToDevice));
        cuda(cudaMemcpy(is.p, hs.data(), cap * 4, cudaMemcpyHostToDevice));
        cuda(cudaMemcpy(kv.p, &cnt[0], 4, cudaMemcpyHostToDevice));
        cuda(cudaMemcpy(ks.p, &cnt[1], 4, cudaMemcpyHostToDevice));
        check(vsp_vs_attn_fwd(context(), q->p, k->p, v->p, n, 1, 1, d, iv.as<int>(), kv.as<int>(), is.as<int>(),
                              ks.as<int>(), cap, scale, o.p, lse.as<float>(), wsp.p, VSP_VALIDATE, nullptr));
    }
    cuda(cudaDeviceSynchronize());
    AttentionOutput out;
    out.o = download_head0(o, n, d, 1);
    if (lse_out) *lse_out = std::move(lse_buf);
    return out;
}
}  // namespace detail

// attention.hpp:150-194 (uncovered rows and unsorted lists throw the reference's messages)
inline AttentionOutput sparse_attention(const AttentionInputs& in, const SparsePattern& pat,
                                        std::size_t block = 32) {
    require(block >= 1, "sparse_attention: block must be >= 1");
    return detail::attend(in, &pat);
}

// attention.hpp:96-145
inline AttentionOutput blockwise_attention(const AttentionInputs& in, std::size_t block) {
    require(block >= 1, "blockwise_attention: block must be >= 1");
    return detail::attend(in, nullptr);
}

// attention.hpp:198-215 without the n x n matrix: the reference takes the dense attention
// weights A; on the device the covered mass of row i is exp(LSE_sparse_i - LSE_dense_i), so
// this overload takes the inputs A was formed from and returns the same mean over rows
// (vsp_recall_from_lse, exact up to the kernels' LSE tolerance).
inline double attention_recall(const AttentionInputs& in, const SparsePattern& pat) {
    const int n = static_cast<int>(in.n());
    std::unique_ptr<detail::Buf> lse_s, lse_d;
    detail::attend(in, &pat, &lse_s);
    detail::attend(in, nullptr, &lse_d);
    detail::Buf r(4);
    detail::check(vsp_recall_from_lse(detail::context(), lse_s->as<float>(), lse_d->as<float>(), n, 1, r.as<float>(),
                                      nullptr));
    float h = 0.f;
    detail::cuda(cudaMemcpy(&h, r.p, 4, cudaMemcpyDeviceToHost));
    return h;
}

// vsaggregate.hpp:62-127 (one head; the group combine of the batched API is the identity)
inline VSScores aggregate_streaming(const AttentionInputs& in, std::size_t block, bool normalized = true) {
    require(block >= 1, "aggregate_streaming: block must be >= 1");
    const int n = static_cast<int>(in.n()), d = static_cast<int>(in.d());
    auto q = detail::upload_bf16(in.q), k = detail::upload_bf16(in.k);
    detail::Buf av(n * 4), as(n * 4), wsp(vsp_aggregate_workspace_size(n, 1));
    detail::check(vsp_vs_aggregate(detail::context(), q->p, k->p, n, 1, 1, d, static_cast<float>(in.scale), nullptr,
                                   VSP_REDUCE_MEAN, normalized ? 1 : 0, av.as<float>(), as.as<float>(), wsp.p,
                                   nullptr));
    VSScores s;
    s.vertical = detail::download_f32(av, n);
    s.slash = detail::download_f32(as, n);
    s.normalized = normalized;
    return s;
}

// rope.hpp:63-79 (interleaved planes, as the reference)
inline Matrix apply_rope(const Matrix& x, const std::vector<std::size_t>& positions, const RopeConfig& cfg) {
    require(x.cols == cfg.head_dim, "apply_rope: column count != head_dim");
    require(positions.size() == x.rows, "apply_rope: positions length != row count");
    const int n = static_cast<int>(x.rows), d = static_cast<int>(x.cols);
    Matrix out(x.rows, x.cols);
    if (n == 0) return out;
    auto in = detail::upload_bf16(x);
    detail::Buf o(static_cast<size_t>(n) * d * 2), pos(static_cast<size_t>(n) * 8);
    std::vector<int64_t> hp(positions.begin(), positions.end());
    detail::cuda(cudaMemcpy(pos.p, hp.data(), hp.size() * 8, cudaMemcpyHostToDevice));
    detail::check(vsp_apply_rope(detail::context(), in->p, nullptr, o.p, nullptr, n, 1, 0, d, pos.as<int64_t>(),
                                 cfg.base, VSP_ROPE_INTERLEAVED, nullptr));
    return detail::download_head0(o, x.rows, x.cols, 1);
}
inline Matrix apply_rope(const Matrix& x, const RopeConfig& cfg) {
    std::vector<std::size_t> positions(x.rows);
    for (std::size_t i = 0; i < positions.size(); ++i) positions[i] = i;
    return vsp::gpu::apply_rope(x, positions, cfg);
}

// indexer.hpp:275-282 with the product-path loss. The GPU recomputes the forward from acts.x
// (= [K | V]); only the forward KL direction is implemented.
inline IndexerGrads indexer_backward(const IndexerParams& p, const IndexerActivations& acts,
                                     const std::vector<double>& target_v, const std::vector<double>& target_s,
                                     double eps = 1e-8, KlDirection dir = KlDirection::Forward) {
    require(dir == KlDirection::Forward, "vsp::gpu::indexer_backward: only the forward KL direction");
    require(p.in_dim() == acts.x.cols && p.in_dim() % 2 == 0, "indexer_backward: feature width != in_dim");
    const int n = static_cast<int>(acts.x.rows), d = static_cast<int>(p.in_dim() / 2), dh = static_cast<int>(p.d_h);
    Matrix k(n, d), v(n, d);
    for (int t = 0; t < n; ++t)
        for (int c = 0; c < d; ++c) {
            k(t, c) = acts.x(t, c);
            v(t, c) = acts.x(t, d + c);
        }
    auto kb = detail::upload_bf16(k), vb = detail::upload_bf16(v), wu = detail::upload_bf16(p.w_u);
    auto bu = detail::upload_f32(p.b_u), wv = detail::upload_f32(p.w_v), ws = detail::upload_f32(p.w_s);
    auto bv = detail::upload_f32({p.b_v}), bs = detail::upload_f32({p.b_s});
    auto tv = detail::upload_f32(target_v), ts = detail::upload_f32(target_s);
    const size_t count = 2 * static_cast<size_t>(d) * dh + 3 * static_cast<size_t>(dh) + 2;
    detail::Buf grads(count * 4), wsp(vsp_indexer_grad_workspace_size(n, 1, dh));
    detail::check(vsp_indexer_loss_grad(detail::context(), kb->p, vb->p, n, 1, d, dh, wu->p, bu->as<float>(),
                                        wv->as<float>(), bv->as<float>(), ws->as<float>(), bs->as<float>(),
                                        acts.mapping == SlashMapping::Reverse ? VSP_SLASH_REVERSE : VSP_SLASH_IDENTITY,
                                        tv->as<float>(), ts->as<float>(), eps, nullptr, grads.as<float>(), wsp.p,
                                        nullptr));
    const std::vector<double> g = detail::download_f32(grads, count);
    IndexerGrads out = IndexerGrads::zeros_like(p);
    const size_t nw = 2 * static_cast<size_t>(d) * dh;
    std::copy(g.begin(), g.begin() + nw, out.w_u.data.begin());
    std::copy(g.begin() + nw, g.begin() + nw + dh, out.b_u.begin());
    std::copy(g.begin() + nw + dh, g.begin() + nw + 2 * dh, out.w_v.begin());
    std::copy(g.begin() + nw + 2 * dh, g.begin() + nw + 3 * dh, out.w_s.begin());
    out.b_v = g[nw + 3 * dh];
    out.b_s = g[nw + 3 * dh + 1];
    return out;
}

// indexer.hpp:347-363, fp32 state on the device (parameters and moments round-trip as f64)
inline void optimizer_step(IndexerParams& p, const IndexerGrads& grads, OptState& state, std::size_t step_index,
                           const TrainConfig& cfg) {
    auto flat = [](const Matrix& w, const std::vector<double>& b, const std::vector<double>& wv, double bv,
                   const std::vector<double>& ws, double bs) {
        std::vector<double> f(w.data);
        f.insert(f.end(), b.begin(), b.end());
        f.insert(f.end(), wv.begin(), wv.end());
        f.insert(f.end(), ws.begin(), ws.end());
        f.push_back(bv);
        f.push_back(bs);
        return f;
    };
    auto unflat = [](const std::vector<double>& f, Matrix& w, std::vector<double>& b, std::vector<double>& wv,
                     double& bv, std::vector<double>& ws, double& bs) {
        size_t o = 0;
        for (double& x : w.data) x = f[o++];
        for (double& x : b) x = f[o++];
        for (double& x : wv) x = f[o++];
        for (double& x : ws) x = f[o++];
        bv = f[o++];
        bs = f[o++];
    };
    const auto fp = flat(p.w_u, p.b_u, p.w_v, p.b_v, p.w_s, p.b_s);
    const auto fg = flat(grads.w_u, grads.b_u, grads.w_v, grads.b_v, grads.w_s, grads.b_s);
    const auto fm = flat(state.m.w_u, state.m.b_u, state.m.w_v, state.m.b_v, state.m.w_s, state.m.b_s);
    const auto fv = flat(state.v.w_u, state.v.b_u, state.v.w_v, state.v.b_v, state.v.w_s, state.v.b_s);
    auto bp = detail::upload_f32(fp), bg = detail::upload_f32(fg), bm = detail::upload_f32(fm), bvv = detail::upload_f32(fv);
    const vsp_adamw a{learning_rate(step_index, cfg), cfg.beta1, cfg.beta2, cfg.adam_eps, cfg.weight_decay};
    detail::check(vsp_adamw_step(detail::context(), bp->as<float>(), bg->as<float>(), bm->as<float>(), bvv->as<float>(),
                                 static_cast<int64_t>(fp.size()), static_cast<int64_t>(step_index), &a, nullptr, 0,
                                 nullptr));
    unflat(detail::download_f32(*bp, fp.size()), p.w_u, p.b_u, p.w_v, p.b_v, p.w_s, p.b_s);
    unflat(detail::download_f32(*bm, fp.size()), state.m.w_u, state.m.b_u, state.m.w_v, state.m.b_v, state.m.w_s,
           state.m.b_s);
    unflat(detail::download_f32(*bvv, fp.size()), state.v.w_u, state.v.b_u, state.v.w_v, state.v.b_v, state.v.w_s,
           state.v.b_s);
}

// ---- interchange formats through the C ABI (same bytes and error texts as the reference)
inline void write_tensor(const std::string& path, const Matrix& m) {
    const uint64_t dims[2] = {m.rows, m.cols};
    detail::check(vsp_write_tensor(path.c_str(), 2, dims, m.data.data()));
}
inline void write_tensor(const std::string& path, const std::vector<double>& v) {
    const uint64_t dims[1] = {v.size()};
    detail::check(vsp_write_tensor(path.c_str(), 1, dims, v.data()));
}
inline Matrix read_tensor(const std::string& path) {
    int nd = 0;
    uint64_t dims[8] = {};
    detail::check(vsp_tensor_header(path.c_str(), &nd, dims, 8));
    Matrix m(nd == 2 ? dims[0] : 0, nd == 2 ? dims[1] : 0);
    detail::check(vsp_read_tensor(path.c_str(), 2, m.data.data(), m.data.size()));
    return m;
}
inline std::vector<double> read_vector(const std::string& path) {
    int nd = 0;
    uint64_t dims[8] = {};
    detail::check(vsp_tensor_header(path.c_str(), &nd, dims, 8));
    std::vector<double> v(nd == 1 ? dims[0] : 0);
    detail::check(vsp_read_tensor(path.c_str(), 1, v.data(), v.size()));
    return v;
}
inline void save_checkpoint(const IndexerParams& p, const std::string& path) {
    p.check_shapes();
    require(p.in_dim() % 2 == 0, "save_checkpoint: in_dim must be 2d");
    detail::check(vsp_save_checkpoint(path.c_str(), static_cast<int>(p.in_dim() / 2), static_cast<int>(p.d_h),
                                      p.w_u.data.data(), p.b_u.data(), p.w_v.data(), p.b_v, p.w_s.data(), p.b_s));
}
inline IndexerParams load_checkpoint(const std::string& path) {
    int d = 0, dh = 0;
    detail::check(vsp_checkpoint_header(path.c_str(), &d, &dh));
    IndexerParams p;
    p.d_h = static_cast<size_t>(dh);
    p.w_u = Matrix(2 * static_cast<size_t>(d), p.d_h);
    p.b_u.resize(p.d_h);
    p.w_v.resize(p.d_h);
    p.w_s.resize(p.d_h);
    detail::check(vsp_load_checkpoint(path.c_str(), d, dh, p.w_u.data.data(), p.b_u.data(), p.w_v.data(), &p.b_v,
                                      p.w_s.data(), &p.b_s));
    return p;
}
inline void write_indices(const std::string& path, const SelectedIndices& sel) {
    std::vector<int64_t> a(sel.i_v.begin(), sel.i_v.end()), b(sel.i_s.begin(), sel.i_s.end());
    detail::check(vsp_write_indices(path.c_str(), a.data(), static_cast<int64_t>(a.size()), b.data(),
                                    static_cast<int64_t>(b.size())));
}
inline SelectedIndices read_indices(const std::string& path) {
    FILE* f = std::fopen(path.c_str(), "rb");
    long size = 1;
    if (f) {
        std::fseek(f, 0, SEEK_END);
        size = std::max(1L, std::ftell(f));
        std::fclose(f);
    }
    std::vector<int64_t> a(size), b(size);
    int64_t kv = 0, ks = 0;
    detail::check(vsp_read_indices(path.c_str(), a.data(), &kv, b.data(), &ks, size));
    SelectedIndices sel;
    sel.i_v.assign(a.begin(), a.begin() + kv);
    sel.i_s.assign(b.begin(), b.begin() + ks);
    return sel;
}

}  // namespace vsp::gpu
