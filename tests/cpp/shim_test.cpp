// Reference test bodies re-pointed from vsp:: to vsp::gpu:: through include/vsprefill_gpu.hpp.
// Built where the reference headers exist (tests/cpp/Makefile); the binary travels to the GPU
// box and runs under tests/test_gpu_cpp_shim.py. Prints one PASS/FAIL line per case.
#include <cmath>
#include <cstdio>
#include <functional>
#include <string>

#include "oracles.hpp"
#include "vsprefill/vsprefill.hpp"
#include "vsprefill_gpu.hpp"

using namespace vsp;
static int failures = 0;

static void check(const char* name, const std::function<bool(std::string&)>& fn) {
    std::string detail;
    bool ok = false;
    try {
        ok = fn(detail);
    } catch (const std::exception& e) {
        detail = std::string("exception: ") + e.what();
    }
    std::printf("[%s] %s %s\n", ok ? "PASS" : "FAIL", name, detail.c_str());
    if (!ok) ++failures;
}

int main() {
    // SparseAttention.MatchesMaskedSoftmaxOracle (test_attention.cpp:129-143), d = 128
    check("sparse_attention_matches_masked_oracle", [](std::string& det) {
        Rng rng(4242);
        double worst = 0.0;
        for (int trial = 0; trial < 4; ++trial) {
            const size_t n = 40 + 37 * trial;
            const AttentionInputs in(oracle::random_matrix(rng, n, 128), oracle::random_matrix(rng, n, 128),
                                     oracle::random_matrix(rng, n, 128));
            SparsePattern pat;
            for (size_t j = 0; j < n; j += 3 + trial) pat.i_v.push_back(j);
            pat.i_s = {0, 1, 5, 9};
            const Matrix want = oracle::masked_attention(in.q, in.k, in.v, oracle::pattern_mask(n, pat.i_v, pat.i_s));
            const Matrix got = vsp::gpu::sparse_attention(in, pat).o;
            worst = std::max(worst, max_abs_diff(got, want));
        }
        det = "max|d|=" + std::to_string(worst);
        return worst <= 2e-2;
    });
    // FullVerticalEqualsFull / BlockwiseAttention.EquivalentToFullAcrossSizes
    check("blockwise_attention_matches_full", [](std::string& det) {
        Rng rng(7);
        double worst = 0.0;
        for (size_t n : {1, 7, 128, 300}) {
            const AttentionInputs in(oracle::random_matrix(rng, n, 128), oracle::random_matrix(rng, n, 128),
                                     oracle::random_matrix(rng, n, 128));
            worst = std::max(worst, max_abs_diff(vsp::gpu::blockwise_attention(in, 64).o,
                                                 oracle::dense_attention(in.q, in.k, in.v)));
        }
        det = "max|d|=" + std::to_string(worst);
        return worst <= 2e-2;
    });
    // SparseAttention.UncoveredRowThrows (test_attention.cpp:157-170)
    check("uncovered_row_throws", [](std::string& det) {
        Rng rng(1);
        const AttentionInputs in(oracle::random_matrix(rng, 8, 128), oracle::random_matrix(rng, 8, 128),
                                 oracle::random_matrix(rng, 8, 128));
        try {
            vsp::gpu::sparse_attention(in, SparsePattern{{5}, {3}});
        } catch (const std::invalid_argument& e) {
            det = e.what();
            return std::string(e.what()) == "uncovered query row 0";
        }
        return false;
    });
    // CumulativeBudget.DyadicHandValues + SelectPattern hand cases (test_sparsity.cpp:22-32, 133-159)
    check("select_pattern_hand_cases", [](std::string& det) {
        VSScores s;
        s.vertical.assign(8, 1.0 / 8.0);
        s.slash.assign(8, 1.0 / 8.0);
        BudgetConfig cfg;
        cfg.tau_v = 0.5;
        cfg.tau_s = 0.25;
        const SelectedIndices a = vsp::gpu::select_pattern(s, cfg), b = vsp::select_pattern(s, cfg);
        VSScores t;
        t.vertical = {0.0, 0.0, 1.0, 0.0};
        t.slash = {0.0, 0.0, 0.0, 1.0};
        BudgetConfig c2;
        const SelectedIndices x = vsp::gpu::select_pattern(t, c2), y = vsp::select_pattern(t, c2);
        det = "k_v=" + std::to_string(a.k_v()) + " k_s=" + std::to_string(a.k_s());
        return a.i_v == b.i_v && a.i_s == b.i_s && x.i_v == y.i_v && x.i_s == y.i_s;
    });
    // select_pattern on fp32-exact random scores: bit-exact vs the reference
    check("select_pattern_matches_reference", [](std::string& det) {
        Rng rng(93);
        int trials = 0;
        for (int trial = 0; trial < 30; ++trial) {
            const size_t n = 1 + rng.next_below(3000);
            VSScores s;
            s.vertical.resize(n);
            s.slash.resize(n);
            double tv = 0, ts = 0;
            for (size_t i = 0; i < n; ++i) {
                s.vertical[i] = static_cast<double>(1 + rng.next_below(64));
                s.slash[i] = static_cast<double>(1 + rng.next_below(64));
                tv += s.vertical[i];
                ts += s.slash[i];
            }
            for (size_t i = 0; i < n; ++i) {  // fp32-representable normalised scores
                s.vertical[i] = static_cast<double>(static_cast<float>(s.vertical[i] / tv));
                s.slash[i] = static_cast<double>(static_cast<float>(s.slash[i] / ts));
            }
            BudgetConfig cfg;
            cfg.tau_v = 0.05 + 0.9 * rng.next_uniform();
            cfg.tau_s = 0.05 + 0.9 * rng.next_uniform();
            const SelectedIndices a = vsp::gpu::select_pattern(s, cfg), b = vsp::select_pattern(s, cfg);
            if (a.i_v != b.i_v || a.i_s != b.i_s) {
                det = "mismatch at trial " + std::to_string(trial);
                return false;
            }
            ++trials;
        }
        det = std::to_string(trials) + " trials bit-exact";
        return true;
    });
    // IndexerForward vs the reference on the same bf16-representable inputs, d=128, d_h=256
    check("indexer_forward_matches_reference", [](std::string& det) {
        Rng rng(73);
        IndexerParams p = make_indexer_params(256, 256, rng);
        for (double& w : p.w_v) w = 0.2 * rng.next_normal();
        for (double& w : p.w_s) w = 0.2 * rng.next_normal();
        auto bf = [](Matrix m) {
            for (double& x : m.data) x = static_cast<double>(__bfloat162float(__float2bfloat16(static_cast<float>(x))));
            return m;
        };
        p.w_u = bf(p.w_u);
        const Matrix k = bf(oracle::random_matrix(rng, 300, 128)), v = bf(oracle::random_matrix(rng, 300, 128));
        const IndexerActivations a = vsp::gpu::indexer_forward(p, k, v), b = vsp::indexer_forward(p, k, v);
        double worst = 0.0;
        for (size_t i = 0; i < a.logits_v.size(); ++i) {
            worst = std::max(worst, std::fabs(a.logits_v[i] - b.logits_v[i]));
            worst = std::max(worst, std::fabs(a.logits_s[i] - b.logits_s[i]));
        }
        det = "logits max|d|=" + std::to_string(worst);
        return worst <= 3e-2;
    });
    // AggregateStreaming.EqualsNaive (test_vsaggregate.cpp:86-98) at d = 128
    check("aggregate_streaming_matches_reference", [](std::string& det) {
        Rng rng(11);
        const size_t n = 333;
        const AttentionInputs in(oracle::random_matrix(rng, n, 128, 0.5), oracle::random_matrix(rng, n, 128, 0.5),
                                 oracle::random_matrix(rng, n, 128));
        const VSScores a = vsp::gpu::aggregate_streaming(in, 64), b = vsp::aggregate_streaming(in, 64);
        double worst = 0.0;
        for (size_t i = 0; i < n; ++i) {
            worst = std::max(worst, std::fabs(a.vertical[i] - b.vertical[i]) / (b.vertical[i] + 1e-4));
            worst = std::max(worst, std::fabs(a.slash[i] - b.slash[i]) / (b.slash[i] + 1e-4));
        }
        det = "max rel=" + std::to_string(worst);
        return worst <= 2e-2;
    });
    std::printf("%s: %d failure(s)\n", failures ? "FAIL" : "OK", failures);
    return failures ? 1 : 0;
}
