// vsprefill_gpu.hpp — C++ drop-in shim: the reference's hot-path signatures on the B200.
//
// Include AFTER the reference headers (it uses vsp::Matrix, vsp::AttentionInputs, ... from
// /root/reference/proj/include/vsprefill) and link libvsp_gpu.so + cudart. Each function has
// the signature of the reference function it replaces, so reference call sites and test
// bodies can be re-pointed from `vsp::` to `vsp::gpu::` unchanged:
//
//   vsp::gpu::indexer_forward      <- vsp::indexer_forward      indexer.hpp:116
//   vsp::gpu::select_pattern       <- vsp::select_pattern       sparsity.hpp:105
//   vsp::gpu::sparse_attention     <- vsp::sparse_attention     attention.hpp:150
//   vsp::gpu::blockwise_attention  <- vsp::blockwise_attention  attention.hpp:96
//   vsp::gpu::aggregate_streaming  <- vsp::aggregate_streaming  vsaggregate.hpp:62
//
// Host f64 data is converted to the device formats (bf16 Q/K/V/W_U, fp32 scores) on the way
// in and widened back to f64 on the way out, so results carry the GPU path's stated
// tolerances; index sets from select_pattern are bit-exact for scores that
// are exactly representable in fp32. Errors: VSP_EINVAL -> std::invalid_argument with the
// reference's message, anything else -> std::runtime_error. `block` arguments are accepted
// for signature compatibility; the GPU tiling is fixed (results do not depend on it, as in
// the reference, test_attention.cpp:145-155). The single-head API runs on the batched
// kernels with one KV head and the Q head duplicated (the CTA processes Q-head pairs).
#pragma once

#include <cuda_runtime.h>
#include <cuda_bf16.h>

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

namespace detail {
inline AttentionOutput attend(const AttentionInputs& in, const SparsePattern* pat) {
    const int n = static_cast<int>(in.n()), d = static_cast<int>(in.d());
    auto q = upload_bf16(in.q, 2), k = upload_bf16(in.k), v = upload_bf16(in.v);
    Buf o(static_cast<size_t>(n) * 2 * d * 2), lse(static_cast<size_t>(n) * 2 * 4);
    const float scale = static_cast<float>(in.scale);
    if (!pat) {
        check(vsp_dense_attn_fwd(context(), q->p, k->p, v->p, n, 2, 1, d, scale, o.p, lse.as<float>(), nullptr));
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
        check(vsp_vs_attn_fwd(context(), q->p, k->p, v->p, n, 2, 1, d, iv.as<int>(), kv.as<int>(), is.as<int>(),
                              ks.as<int>(), cap, scale, o.p, lse.as<float>(), wsp.p, VSP_VALIDATE, nullptr));
    }
    cuda(cudaDeviceSynchronize());
    AttentionOutput out;
    out.o = download_head0(o, n, d, 2);
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

// vsaggregate.hpp:62-127 (one head; the group combine of the batched API is the identity)
inline VSScores aggregate_streaming(const AttentionInputs& in, std::size_t block, bool normalized = true) {
    require(block >= 1, "aggregate_streaming: block must be >= 1");
    const int n = static_cast<int>(in.n()), d = static_cast<int>(in.d());
    auto q = detail::upload_bf16(in.q, 2), k = detail::upload_bf16(in.k);
    detail::Buf av(n * 4), as(n * 4), wsp(vsp_aggregate_workspace_size(n, 2));
    detail::check(vsp_vs_aggregate(detail::context(), q->p, k->p, n, 2, 1, d, static_cast<float>(in.scale), nullptr,
                                   VSP_REDUCE_MEAN, normalized ? 1 : 0, av.as<float>(), as.as<float>(), wsp.p,
                                   nullptr));
    VSScores s;
    s.vertical = detail::download_f32(av, n);
    s.slash = detail::download_f32(as, n);
    s.normalized = normalized;
    return s;
}

}  // namespace vsp::gpu
