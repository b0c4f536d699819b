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
//                    its W_U chunk resident, recomputes Y = X W_U for each 128-token tile in
//                    TMEM (never stored), turns it into dY = (dlv w_v + dls w_s) * silu'(Y)
//                    and Z = silu(Y) (bf16 tiles in smem), and accumulates in TMEM
//                      dW_U += X^T dY   (M = 2 x 128 features, N = 128, K = 128 tokens)
//                      [dw_v dw_s] += Z^T [dlv dls]   and   db_U += dY^T 1   (N = 8)
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

constexpr int kTok = 128;
constexpr int kHid = 128;                   // hidden chunk per CTA
constexpr int kXBytes = kTok * 256 * 2;     // 64 KB: 4 SW128 boxes [128 tok x 64 feat]
constexpr int kWBytes = 256 * kHid * 2;     // 64 KB: 2 N-blocks [256 feat x 64 hid]
constexpr int kTBytes = kTok * kHid * 2;    // 32 KB: dY / Z tiles, 2 blocks [128 tok x 64 hid]
constexpr int kNBytes = 2048;               // [8 x 128] K-major B operands (DL, ones)
constexpr int kOffX = 0;
constexpr int kOffW = kOffX + kXBytes;
constexpr int kOffDY = kOffW + kWBytes;
constexpr int kOffZ = kOffDY + kTBytes;
constexpr int kOffDL = kOffZ + kTBytes;
constexpr int kOffOnes = kOffDL + kNBytes;
constexpr int kOffVec = kOffOnes + kNBytes;  // b_U, w_v, w_s of the chunk: 3 x 128 floats
constexpr int kSmemBytes = kOffVec + 3 * kHid * 4 + 1024;
constexpr int kThreads = 384;               // warp0 TMA, warp1 MMA, warps 4-11 epilogue
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
    uint64_t w_full, x_full[2], x_empty[2], y_full, ep_done, bw_done, all_done;  // x_*[h]: K / V half of X
    uint32_t tmem_base;
};

VSP_DEVICE uint32_t sw128(int row, int chunk) { return static_cast<uint32_t>(row * 128 + (((chunk ^ (row & 7)) & 7) << 4)); }

__global__ void __launch_bounds__(kThreads, 1) backward_kernel(const __grid_constant__ BwdParams p) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* base = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    __shared__ BwdSmem sm;
    const int nchunks = p.d_h / kHid;
    const int sp = blockIdx.x % p.nsplit;
    const int rest = blockIdx.x / p.nsplit;
    const int hc = rest % nchunks;
    const int g = rest / nchunks;
    const int tile_lo = static_cast<int>(static_cast<long long>(p.tiles) * sp / p.nsplit);
    const int tile_hi = static_cast<int>(static_cast<long long>(p.tiles) * (sp + 1) / p.nsplit);
    const int ntiles = tile_hi - tile_lo;
    const uint32_t warp = warp_id(), lane = lane_id();
    float* vec = reinterpret_cast<float*>(base + kOffVec);  // [b_U | w_v | w_s] of the chunk

    if (warp == 0 && lane == 0) {
        mbar_init(&sm.w_full, 1);
        mbar_init(&sm.x_full[0], 1);
        mbar_init(&sm.x_full[1], 1);
        mbar_init(&sm.x_empty[0], 1);
        mbar_init(&sm.x_empty[1], 1);
        mbar_init(&sm.y_full, 1);
        mbar_init(&sm.ep_done, 8);
        mbar_init(&sm.bw_done, 1);
        mbar_init(&sm.all_done, 1);
        fence_barrier_init();
    }
    if (warp == 1) tmem_alloc<512>(&sm.tmem_base);
    {
        // DL rows 2..7 and the ones operand (row 0 = 1) are constant; DL rows 0/1 are rewritten
        uint32_t* dl = reinterpret_cast<uint32_t*>(base + kOffDL);
        for (int i = threadIdx.x; i < kNBytes / 4; i += kThreads) dl[i] = 0u;
        uint16_t* ones = reinterpret_cast<uint16_t*>(base + kOffOnes);
        for (int i = threadIdx.x; i < 8 * 128; i += kThreads) {
            const int nrow = i >> 7, tok = i & 127;
            const uint32_t off = (tok >> 6) * 1024 + sw128(nrow, (tok & 63) >> 3) + ((tok & 7) << 1);
            ones[off >> 1] = nrow == 0 ? 0x3f80u : 0u;
        }
        for (int i = threadIdx.x; i < kHid; i += kThreads) {
            const size_t o = static_cast<size_t>(g) * p.d_h + hc * kHid + i;
            vec[i] = p.b_u[o];
            vec[kHid + i] = p.w_v[o];
            vec[2 * kHid + i] = p.w_s[o];
        }
        fence_proxy_async_smem();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = sm.tmem_base;
    const uint32_t t_y = tmem;            // Y chunk [128 tok x 128 hid]
    const uint32_t t_dw = tmem + 128;     // dW_U: feature halves at +0 / +128, [128 feat x 128 hid]
    const uint32_t t_dwv = tmem + 384;    // [128 hid x 8]: col 0 dw_v, col 1 dw_s
    const uint32_t t_db = tmem + 392;     // [128 hid x 8]: col 0 db_U

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
        // X in two halves (K features -> boxes 0-1, V features -> boxes 2-3), each with its own
        // full/empty pair: the K half of tile i+1 loads while the MMAs of tile i still read the V
        // half, and the first half of Y(i+1) runs while the V half is in flight.
        for (int i = 0; i < ntiles; ++i) {
            const int t0 = (tile_lo + i) * kTok;
#pragma unroll 1
            for (int h = 0; h < 2; ++h) {
                if (i >= 1) mbar_wait(&sm.x_empty[h], (i - 1) & 1);
                if (elect_one()) {
                    mbar_arrive_expect_tx(&sm.x_full[h], kXBytes / 2);
                    for (int hf = 0; hf < 2; ++hf)
                        tma_load_3d(base + kOffX + (2 * h + hf) * 16384, h ? &p.map_v : &p.map_k, &sm.x_full[h],
                                    hf * 64, g, t0);
                }
                __syncwarp();
            }
        }
    } else if (warp == 1) {
        const uint32_t idesc_y = umma_idesc_bf16(128, kHid, false, true);
        const uint32_t idesc_dw = umma_idesc_bf16(128, kHid, true, true);
        const uint32_t idesc_n8 = umma_idesc_bf16(128, 8, true, false);
        const uint64_t x_k = umma_desc_sw128(smem_u32(base + kOffX), 16, 1024);          // X, K-major
        const uint64_t w_mn = umma_desc_sw128(smem_u32(base + kOffW), kWBytes / 2, 1024);  // W chunk, MN-major
        const uint64_t x_mn0 = umma_desc_sw128(smem_u32(base + kOffX), 16384, 1024);       // X^T, features 0..127
        const uint64_t x_mn1 = umma_desc_sw128(smem_u32(base + kOffX + 32768), 16384, 1024);
        const uint64_t dy_mn = umma_desc_sw128(smem_u32(base + kOffDY), 16384, 1024);
        const uint64_t z_mn = umma_desc_sw128(smem_u32(base + kOffZ), 16384, 1024);
        const uint64_t dl_k = umma_desc_sw128(smem_u32(base + kOffDL), 16, 1024);
        const uint64_t ones_k = umma_desc_sw128(smem_u32(base + kOffOnes), 16, 1024);
        mbar_wait(&sm.w_full, 0);
        for (int i = 0; i < ntiles; ++i) {
            // Y = X W_U: K-feature half, then V-feature half as it lands
#pragma unroll 1
            for (int h = 0; h < 2; ++h) {
                mbar_wait(&sm.x_full[h], i & 1);
                if (h == 0 && i >= 1) mbar_wait(&sm.ep_done, (i - 1) & 1);  // Y(i-1) has been read out of TMEM
                tc_fence_after();
                if (elect_one()) {
#pragma unroll
                    for (int kg = 128 * h; kg < 128 * h + 128; kg += 16)
                        umma_ss(t_y, x_k + static_cast<uint64_t>(((kg >> 6) * 16384 + (kg & 63) * 2) >> 4),
                                w_mn + static_cast<uint64_t>((kg * 128) >> 4), idesc_y, kg > 0 ? 1u : 0u);
                    if (h == 1) umma_commit(&sm.y_full);
                }
                __syncwarp();
            }
            mbar_wait(&sm.ep_done, i & 1);  // dY, Z, DL of tile i are in smem
            tc_fence_after();
            if (elect_one()) {
                const uint32_t acc0 = i > 0 ? 1u : 0u;
                // dW_U rows of the K half first so its X boxes are released before the V half's
#pragma unroll
                for (int kk = 0; kk < 8; ++kk) {
                    const uint64_t off = static_cast<uint64_t>((kk * 2048) >> 4);  // 16 tokens
                    umma_ss(t_dw, x_mn0 + off, dy_mn + off, idesc_dw, (acc0 || kk > 0) ? 1u : 0u);
                }
                umma_commit(&sm.x_empty[0]);
#pragma unroll
                for (int kk = 0; kk < 8; ++kk) {
                    const uint64_t off = static_cast<uint64_t>((kk * 2048) >> 4);
                    const uint32_t acc = (acc0 || kk > 0) ? 1u : 0u;
                    const uint64_t koff = static_cast<uint64_t>(((kk >> 2) * 1024 + (kk & 3) * 32) >> 4);
                    umma_ss(t_dwv, z_mn + off, dl_k + koff, idesc_n8, acc);
                    umma_ss(t_db, dy_mn + off, ones_k + koff, idesc_n8, acc);
                }
#pragma unroll
                for (int kk = 0; kk < 8; ++kk) {
                    const uint64_t off = static_cast<uint64_t>((kk * 2048) >> 4);
                    umma_ss(t_dw + 128, x_mn1 + off, dy_mn + off, idesc_dw, (acc0 || kk > 0) ? 1u : 0u);
                }
                umma_commit(&sm.x_empty[1]);
                umma_commit(&sm.bw_done);
                if (i == ntiles - 1) umma_commit(&sm.all_done);
            }
            __syncwarp();
        }
    } else if (warp >= 4) {
        const int quarter = warp & 3;
        const int part = (warp - 4) >> 2;  // hidden columns [64 part, 64 part + 64)
        const int r = quarter * 32 + lane;
        const uint32_t lane_base = static_cast<uint32_t>(quarter * 32) << 16;
        uint8_t* dyb = base + kOffDY + part * 16384;
        uint8_t* zb = base + kOffZ + part * 16384;
        uint16_t* dlb = reinterpret_cast<uint16_t*>(base + kOffDL);
        for (int i = 0; i < ntiles; ++i) {
            const int t = (tile_lo + i) * kTok + r;
            float dlv = 0.f, dls = 0.f;
            if (t < p.n) {
                dlv = p.dlogit_v[static_cast<size_t>(g) * p.n + t];
                dls = p.dlogit_s[static_cast<size_t>(g) * p.n + (p.reverse ? p.n - 1 - t : t)];
            }
            mbar_wait(&sm.y_full, i & 1);
            tc_fence_after();
            uint32_t u[2][32];
            tmem_ld32(t_y + lane_base + part * 64, u[0]);
            tmem_ld32(t_y + lane_base + part * 64 + 32, u[1]);
            tmem_wait_ld(u[0]);
            tmem_reg_fence(u[1]);
            if (i >= 1) mbar_wait(&sm.bw_done, (i - 1) & 1);  // tile i-1's MMAs have read dY / Z / DL
#pragma unroll
            for (int ch = 0; ch < 8; ++ch) {
                uint32_t dyw[4], zw[4];
#pragma unroll
                for (int e2 = 0; e2 < 4; ++e2) {
                    float dy2[2], z2[2];
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        const int col = ch * 8 + e2 * 2 + h;  // 0..63 within this part
                        const int j = part * 64 + col;
                        const float y = __uint_as_float(u[col >> 5][col & 31]) + vec[j];
                        const float hh = 0.5f * y;
                        float th;
                        asm("tanh.approx.f32 %0, %1;" : "=f"(th) : "f"(hh));
                        const float sg = 0.5f + 0.5f * th;           // sigmoid(y)
                        z2[h] = hh + hh * th;                       // y * sigmoid(y)
                        const float dsilu = sg * (1.f + y * (1.f - sg));
                        dy2[h] = (dlv * vec[kHid + j] + dls * vec[2 * kHid + j]) * dsilu;
                    }
                    dyw[e2] = pack_bf16x2(dy2[0], dy2[1]);
                    zw[e2] = pack_bf16x2(z2[0], z2[1]);
                }
                *reinterpret_cast<uint4*>(dyb + sw128(r, ch)) = make_uint4(dyw[0], dyw[1], dyw[2], dyw[3]);
                *reinterpret_cast<uint4*>(zb + sw128(r, ch)) = make_uint4(zw[0], zw[1], zw[2], zw[3]);
            }
            if (part == 0) {  // DL[0][tok] = dlv, DL[1][tok] = dls (K-major [8 x 128])
                const uint32_t o0 = (r >> 6) * 1024 + sw128(0, (r & 63) >> 3) + ((r & 7) << 1);
                const uint32_t o1 = (r >> 6) * 1024 + sw128(1, (r & 63) >> 3) + ((r & 7) << 1);
                dlb[o0 >> 1] = __bfloat16_as_ushort(__float2bfloat16_rn(dlv));
                dlb[o1 >> 1] = __bfloat16_as_ushort(__float2bfloat16_rn(dls));
            }
            fence_proxy_async_smem();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&sm.ep_done);
        }
        // ---- write the partial gradients of this token split (fixed-order sum in adamw)
        if (ntiles > 0) {
            mbar_wait(&sm.all_done, 0);
            tc_fence_after();
            const size_t hbase = static_cast<size_t>(hc) * kHid + part * 64;
            for (int mh = 0; mh < 2; ++mh) {
                const int f = mh * 128 + r;  // feature row (TMEM lane)
                float* dst = p.part_wu + ((static_cast<size_t>(sp) * p.hkv + g) * 256 + f) * p.d_h + hbase;
#pragma unroll
                for (int h2 = 0; h2 < 2; ++h2) {
                    uint32_t w[32];
                    tmem_ld32(t_dw + mh * 128 + part * 64 + h2 * 32 + lane_base, w);
                    tmem_wait_ld(w);
#pragma unroll
                    for (int q = 0; q < 8; ++q)
                        reinterpret_cast<float4*>(dst + h2 * 32)[q] =
                            make_float4(__uint_as_float(w[4 * q]), __uint_as_float(w[4 * q + 1]),
                                        __uint_as_float(w[4 * q + 2]), __uint_as_float(w[4 * q + 3]));
                }
            }
            uint32_t e[8];
            const size_t vo = (static_cast<size_t>(sp) * p.hkv + g) * p.d_h + static_cast<size_t>(hc) * kHid + r;
            if (part == 0) {
                asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                             : "=r"(e[0]), "=r"(e[1]), "=r"(e[2]), "=r"(e[3]), "=r"(e[4]), "=r"(e[5]), "=r"(e[6]),
                               "=r"(e[7])
                             : "r"(t_dwv + lane_base));
                tmem_wait_ld(e);
                p.part_wv[vo] = __uint_as_float(e[0]);
                p.part_ws[vo] = __uint_as_float(e[1]);
            } else {
                asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                             : "=r"(e[0]), "=r"(e[1]), "=r"(e[2]), "=r"(e[3]), "=r"(e[4]), "=r"(e[5]), "=r"(e[6]),
                               "=r"(e[7])
                             : "r"(t_db + lane_base));
                tmem_wait_ld(e);
                p.part_bu[vo] = __uint_as_float(e[0]);
            }
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
    const long long nw = static_cast<long long>(hkv) * 256 * d_h;
    const long long nv = static_cast<long long>(hkv) * d_h;
    const long long total = nw + 3 * nv + 2 * hkv;
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
         i += static_cast<long long>(gridDim.x) * blockDim.x) {
        float s = 0.f;
        if (i < nw) {
            for (int k = 0; k < nsplit; ++k) s += part_wu[k * nw + i];
        } else if (i < nw + 3 * nv) {
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
