// Reference test bodies re-pointed from vsp:: to vsp::gpu:: through include/vsprefill_gpu.hpp.
// Built where the reference headers exist (tests/cpp/Makefile); the binary travels to the GPU
// box and runs under tests/test_gpu_cpp_shim.py. Prints one PASS/FAIL line per case.
#include <algorithm>
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
    // AttentionRecall (test_attention.cpp:172-235): the reference's recall over the dense
    // weights A = attention_matrix(q, k) vs the device recall from the two LSEs
    check("attention_recall_from_lse", [](std::string& det) {
        Rng rng(99);
        double worst = 0.0;
        for (size_t n : {64, 257}) {
            const AttentionInputs in(oracle::random_matrix(rng, n, 128), oracle::random_matrix(rng, n, 128),
                                     oracle::random_matrix(rng, n, 128));
            SparsePattern pat;
            for (size_t j = 0; j < n; j += 5) pat.i_v.push_back(j);
            pat.i_s = {0, 2, 7};
            const double want = vsp::attention_recall(vsp::attention_matrix(in.q, in.k), pat);
            const double got = vsp::gpu::attention_recall(in, pat);
            worst = std::max(worst, std::fabs(got - want));
        }
        det = "max|d recall|=" + std::to_string(worst);
        return worst <= 2e-3;
    });
    // CumulativeBudget.DyadicHandValues (test_sparsity.cpp:22-32) + random distributions
    check("cumulative_budget_matches_reference", [](std::string& det) {
        const std::vector<double> dy = {0.5, 0.25, 0.125, 0.125};
        BudgetConfig cfg;
        int bad = 0, trials = 0;
        for (double tau : {0.1, 0.5, 0.6, 0.75, 0.8, 0.875, 0.9, 1.0}) {
            ++trials;
            if (vsp::gpu::cumulative_budget(dy, tau, cfg) != vsp::cumulative_budget(dy, tau, cfg)) ++bad;
        }
        Rng rng(17);
        for (int t = 0; t < 12; ++t) {
            std::vector<double> s = oracle::random_distribution(rng, 100 + 97 * t);
            for (double& x : s) x = static_cast<double>(static_cast<float>(x));  // fp32-exact scores
            double sum = 0.0;
            for (double x : s) sum += x;
            for (double& x : s) x /= sum;
            for (double& x : s) x = static_cast<double>(static_cast<float>(x));
            for (double tau : {0.3, 0.9}) {
                BudgetConfig c2;
                c2.min_budget = 2;
                ++trials;
                try {
                    if (vsp::gpu::cumulative_budget(s, tau, c2) != vsp::cumulative_budget(s, tau, c2)) ++bad;
                } catch (const std::invalid_argument&) {  // both must reject the same inputs
                    try { vsp::cumulative_budget(s, tau, c2); ++bad; } catch (const std::invalid_argument&) {}
                }
            }
        }
        det = std::to_string(trials - bad) + "/" + std::to_string(trials) + " equal";
        return bad == 0;
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
    // Rope.MatchesExplicitRotationMatrix / ApplyRope.* (test_rope.cpp), d = 128, long positions
    check("apply_rope_matches_reference", [](std::string& det) {
        Rng rng(25);
        const RopeConfig cfg(128, 10000.0);
        const Matrix x = oracle::random_matrix(rng, 9, 128);
        const std::vector<std::size_t> pos = {0, 1, 7, 4095, 32768, 65537, 100000, 131071, 3};
        const double err = max_abs_diff(vsp::gpu::apply_rope(x, pos, cfg), vsp::apply_rope(x, pos, cfg));
        const double err2 = max_abs_diff(vsp::gpu::apply_rope(x, cfg), vsp::apply_rope(x, cfg));
        det = "max|d|=" + std::to_string(std::max(err, err2));
        return err <= 3e-2 && err2 <= 3e-2;  // bf16 in and out
    });
    // IndexerBackward vs the reference (gradients within bf16-operand tolerance)
    check("indexer_backward_matches_reference", [](std::string& det) {
        Rng rng(31);
        const size_t n = 200, d = 128, dh = 256;
        IndexerParams p = make_indexer_params(2 * d, dh, rng);
        for (double& w : p.w_v) w = 0.3 * rng.next_normal();
        for (double& w : p.w_s) w = 0.3 * rng.next_normal();
        // W_U, K, V exactly bf16-representable so both sides see the same inputs
        auto bf = [](double x) { return static_cast<double>(__bfloat162float(__float2bfloat16(static_cast<float>(x)))); };
        for (double& w : p.w_u.data) w = bf(w);
        Matrix k = oracle::random_matrix(rng, n, d), v = oracle::random_matrix(rng, n, d);
        for (double& x : k.data) x = bf(x);
        for (double& x : v.data) x = bf(x);
        std::vector<double> tv(n), ts(n);
        double sv = 0, ss = 0;
        for (size_t i = 0; i < n; ++i) {
            tv[i] = rng.next_uniform() + 0.01;
            ts[i] = rng.next_uniform() + 0.01;
            sv += tv[i];
            ss += ts[i];
        }
        for (size_t i = 0; i < n; ++i) {
            tv[i] /= sv;
            ts[i] /= ss;
        }
        const IndexerActivations acts = vsp::indexer_forward(p, k, v);
        const IndexerGrads want = vsp::indexer_backward(p, acts, tv, ts);
        const IndexerGrads got = vsp::gpu::indexer_backward(p, acts, tv, ts);
        auto rel = [](const std::vector<double>& a, const std::vector<double>& b) {
            double num = 0, den = 0;
            for (size_t i = 0; i < a.size(); ++i) {
                num += (a[i] - b[i]) * (a[i] - b[i]);
                den += b[i] * b[i];
            }
            return std::sqrt(num / std::max(den, 1e-300));
        };
        const double e = std::max({rel(got.w_u.data, want.w_u.data), rel(got.b_u, want.b_u), rel(got.w_v, want.w_v),
                                   rel(got.w_s, want.w_s)});
        det = "max rel=" + std::to_string(e);
        return e <= 3e-2 && std::fabs(got.b_v - want.b_v) <= 1e-4 && std::fabs(got.b_s - want.b_s) <= 1e-4;
    });
    // Optimizer.MatchesScalarAdamWOracle (test_indexer.cpp:346-380) on the device
    check("optimizer_step_matches_reference", [](std::string& det) {
        Rng rng(33);
        IndexerParams p = make_indexer_params(8, 5, rng);
        IndexerGrads g = IndexerGrads::zeros_like(p);
        for (double& x : g.w_u.data) x = rng.next_normal();
        for (double& x : g.w_v) x = rng.next_normal();
        g.b_s = 0.5;
        OptState s1 = OptState::zeros_like(p), s2 = OptState::zeros_like(p);
        IndexerParams p1 = p, p2 = p;
        TrainConfig cfg;
        cfg.steps = 10;
        cfg.warmup_steps = 2;
        for (size_t step = 0; step < 3; ++step) {
            vsp::optimizer_step(p1, g, s1, step, cfg);
            vsp::gpu::optimizer_step(p2, g, s2, step, cfg);
        }
        double e = std::fabs(p1.b_s - p2.b_s);
        for (size_t i = 0; i < p1.w_u.data.size(); ++i) e = std::max(e, std::fabs(p1.w_u.data[i] - p2.w_u.data[i]));
        det = "max|d|=" + std::to_string(e);
        return e <= 1e-6;
    });
    // TensorIo / Checkpoint / IndicesText: the GPU library writes the reference's bytes
    check("formats_match_reference", [](std::string& det) {
        Rng rng(35);
        const Matrix m = oracle::random_matrix(rng, 5, 3);
        vsp::write_tensor("/tmp/vsp_shim_ref.vstn", m);
        vsp::gpu::write_tensor("/tmp/vsp_shim_gpu.vstn", m);
        auto slurp = [](const char* f) {
            FILE* h = std::fopen(f, "rb");
            std::string s;
            int c;
            while (h && (c = std::fgetc(h)) != EOF) s.push_back(static_cast<char>(c));
            if (h) std::fclose(h);
            return s;
        };
        bool ok = slurp("/tmp/vsp_shim_ref.vstn") == slurp("/tmp/vsp_shim_gpu.vstn");
        ok = ok && vsp::gpu::read_tensor("/tmp/vsp_shim_ref.vstn").data == m.data;
        IndexerParams p = make_indexer_params(8, 5, rng);
        vsp::save_checkpoint(p, "/tmp/vsp_shim_ref.vsck");
        vsp::gpu::save_checkpoint(p, "/tmp/vsp_shim_gpu.vsck");
        ok = ok && slurp("/tmp/vsp_shim_ref.vsck") == slurp("/tmp/vsp_shim_gpu.vsck");
        ok = ok && vsp::gpu::load_checkpoint("/tmp/vsp_shim_ref.vsck").w_u.data == p.w_u.data;
        SelectedIndices sel;
        sel.i_v = {1, 3, 17};
        sel.i_s = {0, 5};
        vsp::write_indices("/tmp/vsp_shim_ref.txt", sel);
        vsp::gpu::write_indices("/tmp/vsp_shim_gpu.txt", sel);
        ok = ok && slurp("/tmp/vsp_shim_ref.txt") == slurp("/tmp/vsp_shim_gpu.txt");
        ok = ok && vsp::gpu::read_indices("/tmp/vsp_shim_ref.txt").i_v == sel.i_v;
        try {
            vsp::gpu::read_tensor("/nonexistent/x.vstn");
            ok = false;
        } catch (const std::runtime_error& e) {
            ok = ok && std::string(e.what()) == "cannot open tensor: /nonexistent/x.vstn";
        }
        det = ok ? "bytes and texts identical" : "mismatch";
        return ok;
    });
    // TopK.HandValuesWithTies / DeterministicUnderPermutedTies / MatchesFullSortOracle /
    // RejectsBadK (test_sparsity.cpp:93-131)
    check("topk_indices_reference_bodies", [](std::string& det) {
        using V = std::vector<std::size_t>;
        const std::vector<double> s = {0.2, 0.5, 0.2, 0.1};
        bool ok = vsp::gpu::topk_indices(s, 1) == V{1} && vsp::gpu::topk_indices(s, 2) == V{0, 1} &&
                  vsp::gpu::topk_indices(s, 3) == V{0, 1, 2} && vsp::gpu::topk_indices(s, 4) == V{0, 1, 2, 3};
        const std::vector<double> twin = {0.3, 0.2, 0.2, 0.3};
        ok = ok && vsp::gpu::topk_indices(twin, 2) == V{0, 3} && vsp::gpu::topk_indices(twin, 3) == V{0, 1, 3};
        ok = ok && vsp::gpu::topk_indices({0.4, 0.1, 0.1, 0.4}, 2) == V{0, 3} &&
             vsp::gpu::topk_indices({0.1, 0.4, 0.4, 0.1}, 2) == V{1, 2};
        Rng rng(93);
        int bad = 0;
        for (int trial = 0; trial < 200; ++trial) {
            const std::size_t n = 1 + static_cast<std::size_t>(rng.next_below(50));
            std::vector<double> sc(n);
            for (double& x : sc) x = static_cast<double>(rng.next_below(8)) / 8.0;
            const std::size_t k = 1 + static_cast<std::size_t>(rng.next_below(n));
            bad += vsp::gpu::topk_indices(sc, k) != oracle::topk(sc, k);
        }
        int thrown = 0;
        for (std::size_t k : {std::size_t{0}, std::size_t{3}}) {
            try {
                vsp::gpu::topk_indices({0.5, 0.5}, k);
            } catch (const std::invalid_argument&) {
                ++thrown;
            }
        }
        det = "oracle mismatches=" + std::to_string(bad) + " bad-k throws=" + std::to_string(thrown);
        return ok && bad == 0 && thrown == 2;
    });
    // MergeRowColumns.HandCases / RejectsUnsortedInput / MatchesSetUnionOracle
    // (test_attention.cpp:274-302)
    check("merge_row_columns_reference_bodies", [](std::string& det) {
        using V = std::vector<std::size_t>;
        bool ok = vsp::gpu::merge_row_columns({0, 5}, {0, 2}, 4) == V{0, 2, 4} &&
                  vsp::gpu::merge_row_columns({}, {0}, 7) == V{7} && vsp::gpu::merge_row_columns({1, 9}, {}, 3) == V{1} &&
                  vsp::gpu::merge_row_columns({2}, {3}, 5) == V{2} && vsp::gpu::merge_row_columns({}, {}, 4).empty();
        int thrown = 0;
        try {
            vsp::gpu::merge_row_columns({3, 1}, {}, 5);
        } catch (const std::invalid_argument& e) {
            thrown += std::string(e.what()) == "merge_row_columns: i_v not strictly ascending";
        }
        try {
            vsp::gpu::merge_row_columns({}, {2, 2}, 5);
        } catch (const std::invalid_argument& e) {
            thrown += std::string(e.what()) == "merge_row_columns: i_s not strictly ascending";
        }
        Rng rng(44);
        auto subset = [&](std::size_t n, std::size_t k) {
            std::vector<std::size_t> pool(n);
            for (std::size_t i = 0; i < n; ++i) pool[i] = i;
            for (std::size_t i = 0; i < k; ++i) std::swap(pool[i], pool[i + rng.next_below(n - i)]);
            pool.resize(k);
            std::sort(pool.begin(), pool.end());
            return pool;
        };
        int bad = 0;
        for (int trial = 0; trial < 300; ++trial) {
            const std::size_t n = 1 + static_cast<std::size_t>(rng.next_below(40));
            const V i_v = subset(n, 1 + static_cast<std::size_t>(rng.next_below(n)));
            const V i_s = subset(n, 1 + static_cast<std::size_t>(rng.next_below(n)));
            const std::size_t i = static_cast<std::size_t>(rng.next_below(n));
            bad += vsp::gpu::merge_row_columns(i_v, i_s, i) != oracle::merge_union(i_v, i_s, i);
        }
        det = "union mismatches=" + std::to_string(bad) + " messages=" + std::to_string(thrown);
        return ok && bad == 0 && thrown == 2;
    });
    // MergePath.HandCase / BalancedSliceSizes-style property (test_attention.cpp:328-350)
    check("merge_path_partition_reference_bodies", [](std::string& det) {
        const std::vector<std::size_t> a = {1, 3, 5}, b = {2, 4, 6};
        const auto cuts = vsp::gpu::merge_path_partition(a, b, 2);
        bool ok = cuts.size() == 3 && cuts[0] == (MergeCut{0, 0}) && cuts[1] == (MergeCut{2, 1}) &&
                  cuts[2] == (MergeCut{3, 3});
        Rng rng(45);
        int bad = 0;
        for (int trial = 0; trial < 100; ++trial) {
            std::vector<std::size_t> x(rng.next_below(40)), y(rng.next_below(40));
            for (auto& t : x) t = rng.next_below(60);
            for (auto& t : y) t = rng.next_below(60);
            std::sort(x.begin(), x.end());
            std::sort(y.begin(), y.end());
            const std::size_t p = 1 + rng.next_below(7);
            bad += vsp::gpu::merge_path_partition(x, y, p) != vsp::merge_path_partition(x, y, p);
        }
        det = "cut mismatches=" + std::to_string(bad);
        return ok && bad == 0;
    });
    // CombineScores.MeanAndSum / RejectsEmptyOrMismatched (test_vsaggregate.cpp:144-162), at
    // fp32: |d| <= 1e-7 instead of 1e-15
    check("combine_scores_reference_bodies", [](std::string& det) {
        VSScores a{{0.6, 0.4}, {1.0, 0.0}, true};
        VSScores b{{0.2, 0.8}, {0.4, 0.6}, true};
        const VSScores mean = vsp::gpu::combine_scores({a, b});
        const VSScores sum = vsp::gpu::combine_scores({a, b}, GroupReduce::Sum);
        bool ok = mean.normalized && std::fabs(mean.vertical[0] - 0.4) <= 1e-7 && std::fabs(mean.slash[1] - 0.3) <= 1e-7 &&
                  !sum.normalized && std::fabs(sum.vertical[0] - 0.8) <= 1e-7 && std::fabs(sum.slash[0] - 1.4) <= 1e-7;
        int thrown = 0;
        try {
            vsp::gpu::combine_scores({});
        } catch (const std::invalid_argument&) {
            ++thrown;
        }
        try {
            VSScores c{{1.0}, {1.0}, true};
            vsp::gpu::combine_scores({a, c});
        } catch (const std::invalid_argument&) {
            ++thrown;
        }
        det = "throws=" + std::to_string(thrown);
        return ok && thrown == 2;
    });
    std::printf("%s: %d failure(s)\n", failures ? "FAIL" : "OK", failures);
    return failures ? 1 : 0;
}
