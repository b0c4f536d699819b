// train.cu — the training half of the paper on sm_100a: VSIndexer
// distillation against K5's ground-truth aggregates, with the reference's objective and
// optimiser (reference indexer.hpp):
//   loss     = KL(pred_v || t_v + eps) + KL(pred_s || t_s + eps)        kl_loss :138-149
//   dlogit   = pred * (dpred - <pred, dpred>), dpred = log pred + 1 - log(t + eps)
//                                                                        kl_loss_grad :158-185,
//                                                                        softmax_backward
//   backward = indexer_backward_from_upstream :222-262 (dlogit_s mapped back to tokens)
//   update   = optimizer_step :347-363 (AdamW, bias-corrected, decoupled decay)
//
// Kernels:
//   kl_grad_kernel   one CTA per (KV head, direction): max / sum-exp / KL / dlogit over n in
//                    fp64 (the softmax over all n tokens), plus the bias gradient sum(dlogit).
//   backward_kernel  tcgen05: per (KV head, 128-wide hidden chunk, token split) the CTA keeps
//                    its W_U chunk resident and, per 128-token tile, recomputes Y^T = W_U^T X^T
//                    in TMEM (hidden units on lanes, double-buffered), forms
//                    dY = (dlv w_v + dls w_s) * silu'(Y) as bf16 K-major rows in smem and
//                    accumulates dW_U^T += dY^T X (M = 128 hidden, N = 256 features) in TMEM;
//                    dw_v, dw_s and db_U are per-thread fp32 sums (a thread owns a hidden unit).
//                    Partials per token split are summed in a fixed order (deterministic).
//   adamw_kernel     optimizer_step over the flat fp32 master parameters; refreshes the bf16
//                    W_U copy the K1 forward reads.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>

#include "vsp_launch.h"
#include "indexer.h"
#include "sm100.cuh"
#include "tma_host.h"
#include "train.h"

using namespace vsp_sm100;

namespace vsp_train {

// ------------------------------------------------------------------ KL loss + dlogit

// grid (hkv * kKlCluster, 2) in clusters of kKlCluster CTAs along x: one cluster per (KV
// head, direction), y = 0 vertical, 1 slash (offset order), 1024 threads per CTA. Each CTA
// strides over its share of the n tokens; the four fp64 reductions (max, sum-exp, KL and
// <p, dpred>, sum dlogit) are block sums published to shared memory and combined by every
// CTA over DSMEM in rank order, so all CTAs hold bit-identical totals (deterministic).
constexpr int kKlCluster = 8;

VSP_DEVICE double ld_cluster_f64(uint32_t cluster_addr) {
    double v;
    asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(v) : "r"(cluster_addr) : "memory");
    return v;
}

__global__ void __cluster_dims__(kKlCluster, 1, 1) __launch_bounds__(1024)
    kl_grad_kernel(const float* __restrict__ logits_v, const float* __restrict__ logits_s,
                   const float* __restrict__ target_v, const float* __restrict__ target_s, int n, double eps,
                   float* dlogit_v, float* dlogit_s, double* loss, double* dbias) {
    const int rank = static_cast<int>(cluster_ctarank());
    const int g = blockIdx.x / kKlCluster, dir = blockIdx.y, heads = gridDim.x / kKlCluster;
    const float* l = (dir ? logits_s : logits_v) + static_cast<size_t>(g) * n;
    const float* t = (dir ? target_s : target_v) + static_cast<size_t>(g) * n;
    float* dl = (dir ? dlogit_s : dlogit_v) + static_cast<size_t>(g) * n;
    __shared__ double red[32];
    __shared__ double xch[5];  // one slot per exchange: max, z, kl, inner, db
    const int i0 = rank * 1024 + static_cast<int>(threadIdx.x), step = kKlCluster * 1024;
    auto block_red = [&](double x, bool is_max) {
        for (int o = 16; o > 0; o >>= 1) {
            const double y = __shfl_xor_sync(0xffffffffu, x, o);
            x = is_max ? fmax(x, y) : x + y;
        }
        __syncthreads();
        if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = x;
        __syncthreads();
        double s = is_max ? -INFINITY : 0.0;
        for (int w = 0; w < 32; ++w) s = is_max ? fmax(s, red[w]) : s + red[w];
        return s;
    };
    // block value -> cluster total (slot k), identical in every CTA
    auto cluster_red = [&](double x, int k, bool is_max) {
        x = block_red(x, is_max);
        if (threadIdx.x == 0) xch[k] = x;
        cluster_sync();
        const uint32_t a = smem_u32(&xch[k]);
        double s = is_max ? -INFINITY : 0.0;
        for (int r = 0; r < kKlCluster; ++r) {
            const double y = ld_cluster_f64(mapa_shared(a, static_cast<uint32_t>(r)));
            s = is_max ? fmax(s, y) : s + y;
        }
        return s;
    };
    double m = -INFINITY;
    for (int i = i0; i < n; i += step) m = fmax(m, static_cast<double>(l[i]));
    m = cluster_red(m, 0, true);
    double z = 0.0;
    for (int i = i0; i < n; i += step) z += exp(static_cast<double>(l[i]) - m);
    const double log_z = log(cluster_red(z, 1, false));
    // loss = sum p (log p - log(t + eps)); inner = sum p * dpred (dpred = log p + 1 - log(t + eps))
    double kl = 0.0, inner = 0.0;
    for (int i = i0; i < n; i += step) {
        const double lp = static_cast<double>(l[i]) - m - log_z;
        const double p = exp(lp);
        const double lt = log(static_cast<double>(t[i]) + eps);
        if (p > 0.0) kl += p * (lp - lt);
        inner += p * ((p > 0.0 ? lp : log(1e-300)) + 1.0 - lt);
    }
    kl = cluster_red(kl, 2, false);
    inner = cluster_red(inner, 3, false);
    double db = 0.0;
    for (int i = i0; i < n; i += step) {
        const double lp = static_cast<double>(l[i]) - m - log_z;
        const double p = exp(lp);
        const double dp = (p > 0.0 ? lp : log(1e-300)) + 1.0 - log(static_cast<double>(t[i]) + eps);
        const double d = p * (dp - inner);
        dl[i] = static_cast<float>(d);
        db += d;
    }
    db = cluster_red(db, 4, false);
    if (rank == 0 && threadIdx.x == 0) {
        loss[dir * heads + g] = kl;
        dbias[dir * heads + g] = db;
    }
    cluster_sync();  // no CTA exits while a peer may still read its xch
}

// ------------------------------------------------------------------ backward GEMM (tcgen05)

// Transposed form (hidden units on TMEM lanes): per 128-token tile
//   Y^T  = W_U^T X^T      A = W_U chunk (smem, MN-major, M = 128 hidden), B = X (K-major, N = 128 tokens),
//                         K = 256 features; double-buffered in TMEM (cols 0 / 128)
//   dY^T = (dlv w_v + dls w_s) * silu'(Y)   epilogue, thread = hidden unit, bf16 K-major rows in smem
//   dW^T += dY^T X        A = dY^T (smem, K-major, M = 128 hidden), B = X (MN-major, N = 256 features),
//                         K = 128 tokens; fp32 in TMEM cols 256..511
// and, since a thread owns one hidden unit, dw_v = sum_t silu(y) dlv, dw_s = sum_t silu(y) dls and
// db_U = sum_t dY accumulate in fp32 registers (no N = 8 MMAs, no Z tile). X is double-buffered
// (two 64 KB slots, each in K / V halves) so Y^T(i+1) runs on the tensor core while the
// epilogue of tile i computes; the epilogue does its math before waiting for dW(i-1) to
// release the single dY tile.
constexpr int kTok = 128;
constexpr int kHid = 128;                   // hidden chunk per CTA
constexpr int kXBytes = kTok * 256 * 2;     // 64 KB per X slot: 4 SW128 boxes [128 tok x 64 feat] (K0 K1 V0 V1)
constexpr int kWBytes = 256 * kHid * 2;     // 64 KB: 2 blocks [256 feat x 64 hid]
constexpr int kTBytes = kHid * kTok * 2;    // 32 KB: dY^T, 2 boxes [128 hid x 64 tok]
constexpr int kOffX = 0;                    // slots at 0 / kXBytes
constexpr int kOffW = 2 * kXBytes;
constexpr int kOffDY = kOffW + kWBytes;
constexpr int kOffDL = kOffDY + kTBytes;    // float2 {dlv, dls} per token of the current tile
constexpr int kOffBar = kOffDL + kTok * 8;
constexpr int kSmemBytes = kOffBar + 256 + 1024;
constexpr int kThreads = 640;               // warp0 TMA, warp1 MMA, warps 4-19 epilogue
constexpr int kEpiWarps = 16;               // 4 lane quarters x 4 token quarters
constexpr uint32_t kEpiBar = 1;             // named barrier of the epilogue warps
static_assert(kSmemBytes <= 227 * 1024, "train smem");

struct __align__(64) BwdParams {
    CUtensorMap map_k, map_v, map_w;
    const float* dlogit_v;  // [hkv, n] token order
    const float* dlogit_s;  // [hkv, n] offset order
    const float* b_u;       // [hkv, d_h]
    const float* w_v;
    const float* w_s;
    float* part_wu;         // [S, hkv, 256, d_h]
    float* part_bu;         // [S, hkv, d_h]
    float* part_wv;
    float* part_ws;
    int n, hkv, d_h, nsplit, tiles, reverse;
};

struct BwdSmem {
    uint64_t w_full, x_full[2][2], x_empty[2][2], y_full[2], y_free[2], ep_done, dy_free, all_done;
    uint32_t tmem_base;
};

VSP_DEVICE uint32_t sw128(int row, int chunk) { return static_cast<uint32_t>(row * 128 + (((chunk ^ (row & 7)) & 7) << 4)); }

__global__ void __launch_bounds__(kThreads, 1) backward_kernel(const __grid_constant__ BwdParams p) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* base = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    BwdSmem& sm = *reinterpret_cast<BwdSmem*>(base + kOffBar);
    const int nchunks = p.d_h / kHid;
    const int sp = blockIdx.x % p.nsplit;
    const int rest = blockIdx.x / p.nsplit;
    const int hc = rest % nchunks;
    const int g = rest / nchunks;
    const int tile_lo = static_cast<int>(static_cast<long long>(p.tiles) * sp / p.nsplit);
    const int tile_hi = static_cast<int>(static_cast<long long>(p.tiles) * (sp + 1) / p.nsplit);
    const int ntiles = tile_hi - tile_lo;
    const uint32_t warp = warp_id(), lane = lane_id();

    if (warp == 0 && lane == 0) {
        mbar_init(&sm.w_full, 1);
        for (int s = 0; s < 2; ++s) {
            mbar_init(&sm.x_full[s][0], 1);
            mbar_init(&sm.x_full[s][1], 1);
            mbar_init(&sm.x_empty[s][0], 1);
            mbar_init(&sm.x_empty[s][1], 1);
            mbar_init(&sm.y_full[s], 1);
            mbar_init(&sm.y_free[s], kEpiWarps);
        }
        mbar_init(&sm.ep_done, kEpiWarps);
        mbar_init(&sm.dy_free, 1);
        mbar_init(&sm.all_done, 1);
        fence_barrier_init();
    }
    if (warp == 1) tmem_alloc<512>(&sm.tmem_base);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = sm.tmem_base;
    const uint32_t t_y = tmem;         // Y^T slots [128 hid x 128 tok] at +0 / +128
    const uint32_t t_dw = tmem + 256;  // dW^T [128 hid x 256 feat]

    if (warp == 0) {
        if (elect_one()) {
            tma_prefetch_desc(&p.map_k);
            tma_prefetch_desc(&p.map_v);
            tma_prefetch_desc(&p.map_w);
            mbar_arrive_expect_tx(&sm.w_full, kWBytes);
            for (int nb = 0; nb < 2; ++nb)
                tma_load_3d(base + kOffW + nb * (kWBytes / 2), &p.map_w, &sm.w_full, hc * kHid + nb * 64, 0, g);
        }
        __syncwarp();
        for (int i = 0; i < ntiles; ++i) {
            const int t0 = (tile_lo + i) * kTok, s = i & 1;
#pragma unroll 1
            for (int h = 0; h < 2; ++h) {
                if (i >= 2) mbar_wait(&sm.x_empty[s][h], ((i >> 1) - 1) & 1);
                if (elect_one()) {
                    mbar_arrive_expect_tx(&sm.x_full[s][h], kXBytes / 2);
                    for (int hf = 0; hf < 2; ++hf)
                        tma_load_3d(base + kOffX + s * kXBytes + (2 * h + hf) * 16384, h ? &p.map_v : &p.map_k,
                                    &sm.x_full[s][h], hf * 64, g, t0);
                }
                __syncwarp();
            }
        }
    } else if (warp == 1) {
        const uint32_t idesc_y = umma_idesc_bf16(128, kTok, true, false);  // A MN-major, B K-major
        const uint32_t idesc_dw = umma_idesc_bf16(128, 256, false, true);  // A K-major, B MN-major
        const uint64_t w_mn = umma_desc_sw128(smem_u32(base + kOffW), kWBytes / 2, 1024);
        const uint64_t dy_k = umma_desc_sw128(smem_u32(base + kOffDY), 16, 1024);
        mbar_wait(&sm.w_full, 0);
        for (int i = 0; i <= ntiles; ++i) {
            if (i < ntiles) {
                const int s = i & 1;
                const uint64_t x_k = umma_desc_sw128(smem_u32(base + kOffX + s * kXBytes), 16, 1024);
                if (i >= 2) mbar_wait(&sm.y_free[s], ((i >> 1) - 1) & 1);  // Y(i-2) read out of slot s
#pragma unroll 1
                for (int h = 0; h < 2; ++h) {
                    mbar_wait(&sm.x_full[s][h], (i >> 1) & 1);
                    tc_fence_after();
                    if (elect_one()) {
#pragma unroll
                        for (int kg = 128 * h; kg < 128 * h + 128; kg += 16)
                            umma_ss(t_y + s * 128, w_mn + static_cast<uint64_t>((kg * 128) >> 4),
                                    x_k + static_cast<uint64_t>(((kg >> 6) * 16384 + (kg & 63) * 2) >> 4), idesc_y,
                                    kg > 0 ? 1u : 0u);
                        if (h == 1) umma_commit(&sm.y_full[s]);
                    }
                    __syncwarp();
                }
            }
            if (i >= 1) {
                const int j = i - 1, sj = j & 1;
                const uint64_t x_mn = umma_desc_sw128(smem_u32(base + kOffX + sj * kXBytes), 16384, 1024);
                mbar_wait(&sm.ep_done, j & 1);  // dY^T of tile j is in smem
                tc_fence_after();
                if (elect_one()) {
#pragma unroll
                    for (int kk = 0; kk < 8; ++kk)  // 16 tokens per MMA
                        umma_ss(t_dw, dy_k + static_cast<uint64_t>(((kk >> 2) * 16384 + (kk & 3) * 32) >> 4),
                                x_mn + static_cast<uint64_t>((kk * 2048) >> 4), idesc_dw, (j > 0 || kk > 0) ? 1u : 0u);
                    umma_commit(&sm.x_empty[sj][0]);
                    umma_commit(&sm.x_empty[sj][1]);
                    umma_commit(&sm.dy_free);
                    if (j == ntiles - 1) umma_commit(&sm.all_done);
                }
                __syncwarp();
            }
        }
    } else if (warp >= 4) {
        const int quarter = warp & 3;
        const int part = (warp - 4) >> 2;  // tokens [32 part, 32 part + 32) of each tile
        const int r = quarter * 32 + lane;  // hidden unit (TMEM lane)
        const int e = (warp - 4) * 32 + lane;  // 0..511: e < 256 loads dlv (e < 128) / dls of token e & 127
        const uint32_t lane_base = static_cast<uint32_t>(quarter * 32) << 16;
        const size_t ho = static_cast<size_t>(g) * p.d_h + hc * kHid + r;
        const float bu = p.b_u[ho], wv = p.w_v[ho], ws = p.w_s[ho];
        uint8_t* dyb = base + kOffDY + (part >> 1) * 16384;  // the 64-token box holding these tokens
        float* dl = reinterpret_cast<float*>(base + kOffDL);  // [tok][2]
        auto load_dl = [&](int i) {
            const int t = (tile_lo + i) * kTok + (e & 127);
            if (e >= 256 || i >= ntiles || t >= p.n) return 0.f;
            return e < 128 ? p.dlogit_v[static_cast<size_t>(g) * p.n + t]
                           : p.dlogit_s[static_cast<size_t>(g) * p.n + (p.reverse ? p.n - 1 - t : t)];
        };
        float dwv = 0.f, dws = 0.f, db = 0.f;
        float nxt = load_dl(0);
        for (int i = 0; i < ntiles; ++i) {
            const int s = i & 1;
            named_bar_sync(kEpiBar, 32 * kEpiWarps);  // every epilogue thread is done with tile i-1's dl
            if (e < 256) dl[(e & 127) * 2 + (e >> 7)] = nxt;
            named_bar_sync(kEpiBar, 32 * kEpiWarps);
            nxt = load_dl(i + 1);
            mbar_wait(&sm.y_full[s], (i >> 1) & 1);
            tc_fence_after();
            uint32_t u[32];
            tmem_ld32(t_y + s * 128 + lane_base + part * 32, u);
            tmem_wait_ld(u);
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&sm.y_free[s]);
            uint32_t dyw[16];
#pragma unroll
            for (int c2 = 0; c2 < 16; ++c2) {
                float dy2[2];
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int col = 2 * c2 + h;  // token within this part
                    const float2 d = *reinterpret_cast<const float2*>(dl + (part * 32 + col) * 2);
                    const float y = __uint_as_float(u[col]) + bu;
                    const float hh = 0.5f * y;
                    float th;
                    asm("tanh.approx.f32 %0, %1;" : "=f"(th) : "f"(hh));
                    const float sg = 0.5f + 0.5f * th;  // sigmoid(y)
                    const float z = hh + hh * th;       // y * sigmoid(y)
                    const float dsilu = sg * (1.f + y * (1.f - sg));
                    dy2[h] = (d.x * wv + d.y * ws) * dsilu;
                    dwv += z * d.x;
                    dws += z * d.y;
                    db += dy2[h];
                }
                dyw[c2] = pack_bf16x2(dy2[0], dy2[1]);
            }
            if (i >= 1) mbar_wait(&sm.dy_free, (i - 1) & 1);  // dW(i-1) has read the dY^T tile
#pragma unroll
            for (int ch = 0; ch < 4; ++ch)
                *reinterpret_cast<uint4*>(dyb + sw128(r, (part & 1) * 4 + ch)) =
                    make_uint4(dyw[4 * ch], dyw[4 * ch + 1], dyw[4 * ch + 2], dyw[4 * ch + 3]);
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) mbar_arrive(&sm.ep_done);
        }
        // ---- partial gradients of this token split (summed over splits in a fixed order)
        float* red = reinterpret_cast<float*>(base + kOffW);  // [part][3][128]: W is free once the last Y^T landed
        mbar_wait(&sm.w_full, 0);  // (a split without tiles: the W load must not land on red)
        named_bar_sync(kEpiBar, 32 * kEpiWarps);
        red[(part * 3 + 0) * 128 + r] = dwv;
        red[(part * 3 + 1) * 128 + r] = dws;
        red[(part * 3 + 2) * 128 + r] = db;
        if (ntiles > 0) {
            mbar_wait(&sm.all_done, 0);
            tc_fence_after();
            const size_t hid = static_cast<size_t>(hc) * kHid + r;
            float* dst = p.part_wu + (static_cast<size_t>(sp) * p.hkv + g) * 256 * p.d_h + hid;
#pragma unroll 1
            for (int c = 0; c < 2; ++c) {
                const int f0 = part * 64 + c * 32;
                uint32_t w[32];
                tmem_ld32(t_dw + lane_base + f0, w);
                tmem_wait_ld(w);
#pragma unroll
                for (int q = 0; q < 32; ++q) dst[static_cast<size_t>(f0 + q) * p.d_h] = __uint_as_float(w[q]);
            }
        }
        named_bar_sync(kEpiBar, 32 * kEpiWarps);
        if (part == 0) {  // token quarters summed in order
            const size_t vo = (static_cast<size_t>(sp) * p.hkv + g) * p.d_h + static_cast<size_t>(hc) * kHid + r;
            float a[3];
#pragma unroll
            for (int k = 0; k < 3; ++k)
                a[k] = ((red[k * 128 + r] + red[(3 + k) * 128 + r]) + red[(6 + k) * 128 + r]) + red[(9 + k) * 128 + r];
            p.part_wv[vo] = a[0];
            p.part_ws[vo] = a[1];
            p.part_bu[vo] = a[2];
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) tmem_free<512>(tmem);
}

// Flat gradient in the parameter layout W_U [hkv,256,d_h] | b_U | w_v | w_s [hkv,d_h] |
// b_v | b_s [hkv]: partials summed over the token splits in a fixed order.
__global__ void reduce_grads_kernel(const float* __restrict__ part_wu, const float* __restrict__ part_bu,
                                    const float* __restrict__ part_wv, const float* __restrict__ part_ws,
                                    const double* __restrict__ dbias, int hkv, int d_h, int nsplit, float* grads) {
    const long long nw = static_cast<long long>(hkv) * 256 * d_h;  // multiple of 4 (d_h % 256 == 0)
    const long long nv = static_cast<long long>(hkv) * d_h;
    const long long total = nw + 3 * nv + 2 * hkv;
    const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
    const long long t0 = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    // W_U: float4 lanes, all nsplit loads issued before the in-order sum (HBM-latency bound otherwise)
    const float4* pw = reinterpret_cast<const float4*>(part_wu);
    const long long nw4 = nw / 4;
    for (long long i = t0; i < nw4; i += stride) {
        float4 v[16];
        float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
        for (int k0 = 0; k0 < nsplit; k0 += 16) {
            const int kn = min(16, nsplit - k0);
#pragma unroll
            for (int k = 0; k < 16; ++k)
                if (k < kn) v[k] = __ldcs(pw + (k0 + k) * nw4 + i);
#pragma unroll
            for (int k = 0; k < 16; ++k)
                if (k < kn) {
                    s.x += v[k].x;
                    s.y += v[k].y;
                    s.z += v[k].z;
                    s.w += v[k].w;
                }
        }
        reinterpret_cast<float4*>(grads)[i] = s;
    }
    for (long long i = nw + t0; i < total; i += stride) {
        float s = 0.f;
        if (i < nw + 3 * nv) {
            const long long j = i - nw;
            const int which = static_cast<int>(j / nv);
            const long long o = j % nv;
            const float* src = which == 0 ? part_bu : (which == 1 ? part_wv : part_ws);
            for (int k = 0; k < nsplit; ++k) s += src[k * nv + o];
        } else {
            s = static_cast<float>(dbias[i - nw - 3 * nv]);  // [b_v heads | b_s heads]
        }
        grads[i] = s;
    }
}

__global__ void adamw_kernel(float* __restrict__ params, const float* __restrict__ grads, float* __restrict__ m,
                             float* __restrict__ v, long long count, float lr, float beta1, float beta2, float bc1,
                             float bc2, float adam_eps, float weight_decay, __nv_bfloat16* shadow,
                             long long shadow_count) {
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < count;
         i += static_cast<long long>(gridDim.x) * blockDim.x) {
        const float g = grads[i];
        const float mi = beta1 * m[i] + (1.f - beta1) * g;
        const float vi = beta2 * v[i] + (1.f - beta2) * g * g;
        m[i] = mi;
        v[i] = vi;
        const float mhat = mi / bc1, vhat = vi / bc2;
        float pi = params[i];
        pi -= lr * (mhat / (sqrtf(vhat) + adam_eps) + weight_decay * pi);
        params[i] = pi;
        if (i < shadow_count) shadow[i] = __float2bfloat16_rn(pi);
    }
}

__global__ void sum_loss_kernel(const double* loss2, int hkv, float* loss) {
    for (int g = threadIdx.x; g < hkv; g += blockDim.x) loss[g] = static_cast<float>(loss2[g] + loss2[hkv + g]);
}

// ------------------------------------------------------------------ host

// Token splits per (KV head, hidden chunk) unit: minimise waves x tiles per CTA (one CTA
// per SM) plus a per-CTA prologue and a per-split reduction cost, in tile units. 128k x 8
// heads (64 units, 1024 tiles): 9 splits = 576 CTAs in 4 full-ish waves of 114 tiles,
// against 5 splits = 320 CTAs in 3 waves (the last 16 % full) of 205 tiles.
static int splits_for(int hkv, int d_h, int tiles) {
    const int sms = vsp_detail::current_sm_count();
    const int units = hkv * (d_h / kHid);
    int best = 1;
    double best_cost = 1e300;
    for (int s = 1; s <= std::min(64, std::max(1, tiles)); ++s) {
        const int waves = (units * s + sms - 1) / sms;
        const int per = (tiles + s - 1) / s;
        const double cost = static_cast<double>(waves) * (per + 2) + 0.5 * s;
        if (cost < best_cost) {
            best_cost = cost;
            best = s;
        }
    }
    return best;
}

size_t workspace_bytes(int n, int hkv, int d_h) {
    const int tiles = (n + kTok - 1) / kTok;
    const int s = std::min(64, std::max(1, tiles));  // upper bound of splits_for
    auto al = [](size_t b) { return (b + 255) & ~size_t(255); };
    return al(2 * static_cast<size_t>(hkv) * n * 4)                       // logits v, s
           + al(2 * static_cast<size_t>(hkv) * n * 4)                     // dlogit v, s
           + al(4 * static_cast<size_t>(hkv) * 8)                         // loss, dbias (double)
           + al(static_cast<size_t>(s) * hkv * 256 * d_h * 4)             // part_wu
           + 3 * al(static_cast<size_t>(s) * hkv * d_h * 4)               // part_bu / wv / ws
           + vsp_indexer::workspace_bytes(n, hkv, d_h) + 256;
}

cudaError_t loss_grad(const GradArgs& a, void* workspace, cudaStream_t stream) {
    if (a.d_h % kHid != 0) return cudaErrorInvalidValue;
    const int tiles = (a.n + kTok - 1) / kTok;
    const int nsplit = std::min(64, splits_for(a.hkv, a.d_h, tiles));
    uint8_t* ws = static_cast<uint8_t*>(workspace);
    auto take = [&](size_t b) {
        uint8_t* r = ws;
        ws += (b + 255) & ~size_t(255);
        return r;
    };
    float* lv = reinterpret_cast<float*>(take(2 * static_cast<size_t>(a.hkv) * a.n * 4));
    float* ls = lv + static_cast<size_t>(a.hkv) * a.n;
    float* dv = reinterpret_cast<float*>(take(2 * static_cast<size_t>(a.hkv) * a.n * 4));
    float* ds = dv + static_cast<size_t>(a.hkv) * a.n;
    double* loss2 = reinterpret_cast<double*>(take(4 * static_cast<size_t>(a.hkv) * 8));
    double* dbias = loss2 + 2 * a.hkv;
    float* part_wu = reinterpret_cast<float*>(take(static_cast<size_t>(nsplit) * a.hkv * 256 * a.d_h * 4));
    float* part_bu = reinterpret_cast<float*>(take(static_cast<size_t>(nsplit) * a.hkv * a.d_h * 4));
    float* part_wv = reinterpret_cast<float*>(take(static_cast<size_t>(nsplit) * a.hkv * a.d_h * 4));
    float* part_ws = reinterpret_cast<float*>(take(static_cast<size_t>(nsplit) * a.hkv * a.d_h * 4));
    void* ws_ix = ws;

    // 1. forward logits with the bf16 weights (K1)
    vsp_indexer::Args ia{a.k, a.v, a.n, a.hkv, a.d_h, a.w_u_bf16, a.b_u, a.w_v, a.b_v, a.w_s, a.b_s, a.reverse,
                         nullptr, nullptr, lv, ls};
    cudaError_t e = vsp_indexer::launch(ia, ws_ix, stream);
    if (e != cudaSuccess) return e;
    // 2. loss and dlogit (fp64 softmax over n)
    vsp_detail::count_launch();
    kl_grad_kernel<<<dim3(a.hkv * kKlCluster, 2), 1024, 0, stream>>>(lv, ls, a.target_v, a.target_s, a.n, a.kl_eps, dv, ds,
                                                        loss2, dbias);
    // 3. backward GEMMs
    BwdParams p{};
    const uint32_t box[3] = {64, 1, kTok};
    const uint64_t dk[3] = {128, (uint64_t)a.hkv, (uint64_t)a.n};
    const uint64_t sk[2] = {128 * 2, (uint64_t)a.hkv * 128 * 2};
    const uint32_t wbox[3] = {64, 256, 1};
    const uint64_t dw[3] = {(uint64_t)a.d_h, 256, (uint64_t)a.hkv};
    const uint64_t sw[2] = {(uint64_t)a.d_h * 2, (uint64_t)a.d_h * 256 * 2};
    if (!vsp_host::make_map_bf16(&p.map_k, a.k, 3, dk, sk, box) ||
        !vsp_host::make_map_bf16(&p.map_v, a.v, 3, dk, sk, box) ||
        !vsp_host::make_map_bf16(&p.map_w, a.w_u_bf16, 3, dw, sw, wbox))
        return cudaErrorInvalidValue;
    p.dlogit_v = dv;
    p.dlogit_s = ds;
    p.b_u = a.b_u;
    p.w_v = a.w_v;
    p.w_s = a.w_s;
    p.part_wu = part_wu;
    p.part_bu = part_bu;
    p.part_wv = part_wv;
    p.part_ws = part_ws;
    p.n = a.n;
    p.hkv = a.hkv;
    p.d_h = a.d_h;
    p.nsplit = nsplit;
    p.tiles = tiles;
    p.reverse = a.reverse ? 1 : 0;
    static std::once_flag attr[vsp_detail::kMaxDevices];
    vsp_detail::once_per_device(attr, [] {
        cudaFuncSetAttribute(backward_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes);
    });
    vsp_detail::count_launch();
    backward_kernel<<<a.hkv * (a.d_h / kHid) * nsplit, kThreads, kSmemBytes, stream>>>(p);
    // 4. fixed-order reduction into the flat gradient; per-head loss = KL_v + KL_s
    vsp_detail::count_launch();
    reduce_grads_kernel<<<592, 256, 0, stream>>>(part_wu, part_bu, part_wv, part_ws, dbias, a.hkv, a.d_h, nsplit,
                                                 a.grads);
    e = cudaGetLastError();
    if (e == cudaSuccess && a.loss) {
        vsp_detail::count_launch();
        sum_loss_kernel<<<1, 128, 0, stream>>>(loss2, a.hkv, a.loss);
        e = cudaGetLastError();
    }
    return e;
}

cudaError_t adamw(const AdamArgs& a, cudaStream_t stream) {
    const double t = static_cast<double>(a.step_index + 1);
    const float bc1 = static_cast<float>(1.0 - std::pow(a.beta1, t));
    const float bc2 = static_cast<float>(1.0 - std::pow(a.beta2, t));
    vsp_detail::count_launch();
    adamw_kernel<<<592, 256, 0, stream>>>(a.params, a.grads, a.m, a.v, a.count, static_cast<float>(a.lr),
                                          static_cast<float>(a.beta1), static_cast<float>(a.beta2), bc1, bc2,
                                          static_cast<float>(a.adam_eps), static_cast<float>(a.weight_decay),
                                          static_cast<__nv_bfloat16*>(a.shadow), a.shadow_count);
    return cudaGetLastError();
}

}  // namespace vsp_train
