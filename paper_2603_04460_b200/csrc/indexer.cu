// indexer.cu — K1: VSIndexer scoring on sm_100a.
//
// Replaces vsp::indexer_forward (reference indexer.hpp:116-120 -> :77-113), per KV head g:
//   X_t = [K_t | V_t]                      (hconcat, indexer.hpp:119)
//   Y   = X W_U + b_U ; Z = SiLU(Y)        (:84-92)
//   logit_v[t] = Z_t w_v + b_v ; raw_s[t] = Z_t w_s + b_s      (:93-105)
//   logit_s[o] = raw_s[n-1-o] (Reverse) | raw_s[o] (Identity)   (:106-109, :26-28)
//   A_v = softmax(logit_v), A_s = softmax(logit_s) over all n   (:110-111)
//
// GEMM kernel (persistent, one CTA per SM): work item = 128 tokens x one KV head, walked
// head-major so concurrent CTAs share W_U in L2. A = X tile (K-major, 4 x [128 x 64] SW128
// boxes straight from the K and V tensors: the concatenation is free), double-buffered
// across work items. B = W_U streamed in [32 K-rows x 256 N] MN-major stages (the
// reference's [2d, d_h] row-major layout, no transpose). tcgen05.mma M=128 N=256 into two
// TMEM accumulators (double-buffered over 256-wide hidden chunks, continuing across work
// items) so the SiLU / two-head epilogue of chunk c overlaps the MMA of chunk c+1 (16
// epilogue warps, four per TMEM lane quarter, 64 columns each: 8 warps left the MUFU and
// tensor pipes ~60 % busy, latency-bound; 16: 466 -> 453 us at 128k x 8 heads). The
// [n, d_h] activation never leaves the SM: only two fp32 logits per token are written.
// The softmax over n runs in the selection clusters (select.cu, fp64 normaliser).
#include <cuda_bf16.h>

#include "vsp_launch.h"
#include "indexer.h"
#include "select.h"
#include "sm100.cuh"
#include "tma_host.h"

using namespace vsp_sm100;

namespace vsp_indexer {

constexpr int kTok = 128;
constexpr int kChunkN = 256;
constexpr int kDefaultStageK = 32;                  // W_U K-rows per ring stage (VSP_K1_STAGEK)
constexpr int kABytes = kTok * 256 * 2;             // 64 KB per token tile
constexpr int kRingBytes = 64 * 1024;               // W_U ring: 4 x 16 KB (one CTA) / 8 x 8 KB (pair)
constexpr int kSplitRingBytes = 128 * 1024;         // split-X mode: one X tile, 8 x 16 KB W_U stages
constexpr int kMaxStages = 8;
constexpr int kMaxDh = 2048;
constexpr int kEpiParts = 4;                        // epilogue warps per TMEM lane quarter
constexpr int kEpiWarps = 4 * kEpiParts;
constexpr int kEpiThreads = 32 * kEpiWarps;
constexpr int kThreads = 64 + kEpiThreads;          // warp0 TMA, warp1 MMA, then the epilogue
constexpr int kDefaultSplit = 1;                    // split-X layout (VSP_K1_SPLIT)
constexpr int kDefaultMc = 1;                       // 1: one CTA per tile; 2: CTA pairs (cta_group::2)

struct __align__(64) Params {
    CUtensorMap map_k, map_v, map_w;
    const float* b_u;
    const float* w_v;
    const float* w_s;
    const float* b_v;
    const float* b_s;
    float* logit_v;  // [hkv, n]
    float* logit_s;  // [hkv, n] (mapping applied)
    int n, hkv, d_h;
    int g0, count;   // KV heads [g0, g0 + count)
    int tiles;       // token tiles per head
    int reverse;
};

struct Smem {
    uint64_t a_full[4], a_empty[4];  // per X buffer (2), or per 64-feature X box (split mode, 4)
    uint64_t full[kMaxStages], empty[kMaxStages];
    uint64_t acc_full[2], acc_empty[2];
    uint32_t tmem_base;
};

// SiLU via one MUFU op: y * sigmoid(y) = h + h * tanh(h), h = y / 2 (overflow-free for any y)
VSP_DEVICE float tanh_f(float h) {
    float t;
    asm("tanh.approx.f32 %0, %1;" : "=f"(t) : "f"(h));
    return t;
}

// Persistent: one CTA per SM walks work items w = blockIdx.x + i * gridDim.x, head-major
// (w / tiles = head, w % tiles = 128-token tile), so the CTAs of one wave stream the same
// W_U from L2. The X tile is double-buffered across work items and the W_U stream and the
// TMEM accumulators run continuously across them, so loads, MMAs and the epilogue of
// consecutive tiles overlap.
//
// Default layout kSplit (VSP_K1_SPLIT = 1): ONE X tile in four 16 KB boxes with per-box
// barriers (the next item's box b loads as soon as the last chunk has consumed it), which
// frees 64 KB for a 128 KB W_U ring: 462 -> 429 us at 128k x 8 heads (the W_U bytes in flight
// per SM, not L2 bandwidth, bound the stream; see the probe numbers below).
// Opt-in variants (parity-green and bit-identical to the default, measured slower):
//   kPair (VSP_K1_MC = 2): CTA pairs (one cluster, one TPC) take two consecutive token tiles of
//   one head and run M = 256 tcgen05.mma.cta_group::2 MMAs issued by the leader: each CTA holds
//   its own 128-token X tile and HALF of every W_U stage (128 of the chunk's 256 columns), so
//   each SM receives half the W_U bytes per unit of MMA work. The peer's TMA loads complete on
//   the leader's barriers (cta_group::2 TMA), its epilogue warps release the accumulators on
//   the leader's acc_empty, and the leader's commits arrive on both CTAs' barriers. Tiles past
//   a head's end (odd tile counts) load tile 0 again and store nothing.
//   kStageK (VSP_K1_STAGEK = 32 / 64): W_U K-rows per ring stage (the ring stays 64 KB).
// Measured at 128k x 8 heads (ncu, two rounds each, tools/dev/gpu_k1pair.sh): one CTA 32 / 64
// K-rows 466 / 472 us, pairs 556 / 548 us. The bound probe (tools/dev/gpu_k1probe2.sh): 454 us;
// epilogue off 388; half the MMAs 391; both 329 — the W_U/X stream pace sets a ~330 us floor,
// but neither halving the W_U bytes per SM (pairs), nor halving the L2 reads (an earlier
// multicast variant: 481 us), nor fewer, larger stages moves it; the pair's lockstep (both
// epilogues must release an accumulator) costs more than it saves.
template <bool kPair, int kStageK, bool kSplit>
__global__ void __launch_bounds__(kThreads, 1) indexer_gemm_kernel(const __grid_constant__ Params p) {
    static_assert(!kSplit || (!kPair && kStageK == 32), "split-X mode: one CTA, 32-row stages");
    constexpr int kMc = kPair ? 2 : 1;
    constexpr int kNCta = kChunkN / kMc;      // W_U columns of a stage held by this CTA
    constexpr int kSB = kStageK * kNCta * 2;  // stage bytes per CTA: 16 KB / 8 KB
    constexpr int kRing = kSplit ? kSplitRingBytes : kRingBytes;
    constexpr int kNS = kRing / kSB;          // stages: 4 / 8 (pairs, split-X)
    static_assert(kNS <= kMaxStages, "indexer ring");
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    // offset from smem_raw (not a cast through an integer) so the compiler keeps the
    // shared state space and emits LDS/STS rather than generic LD/ST
    uint8_t* base = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    uint8_t* sA = base;                        // 2 x 64 KB (split-X: 1 x 64 KB)
    uint8_t* sB = base + (kSplit ? 1 : 2) * kABytes;  // W_U ring
    float* s_bh = reinterpret_cast<float*>(sB + kRing);  // b_U / 2
    float* s_wv = s_bh + kMaxDh;
    float* s_ws = s_wv + kMaxDh;
    float* s_xch = s_ws + kMaxDh;              // 2 x (kEpiParts - 1) x 256 floats (tile parity)
    __shared__ Smem sm;

    const int num_chunks = p.d_h / kChunkN;
    const int groups_per_head = (p.tiles + kMc - 1) / kMc;
    const int total = groups_per_head * p.count;  // tile groups, one per cluster at a time
    const int cl = static_cast<int>(blockIdx.x) / kMc;
    const int ncl = static_cast<int>(gridDim.x) / kMc;
    const int rank = kPair ? static_cast<int>(cluster_ctarank()) : 0;
    const bool leader = rank == 0;
    const uint32_t warp = warp_id();
    const uint32_t lane = lane_id();

    if (warp == 0 && lane == 0) {
        for (int b = 0; b < 4; ++b) {
            mbar_init(&sm.a_full[b], 1);
            mbar_init(&sm.a_empty[b], 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&sm.acc_full[b], 1);
            mbar_init(&sm.acc_empty[b], kEpiWarps * kMc);  // both CTAs' epilogues (leader's copy)
        }
        for (int s = 0; s < kNS; ++s) {
            mbar_init(&sm.full[s], 1);
            mbar_init(&sm.empty[s], 1);
        }
        fence_barrier_init();
    }
    if (warp == 1) {
        if constexpr (kPair)
            tmem_alloc_pair<512>(&sm.tmem_base);
        else
            tmem_alloc<512>(&sm.tmem_base);
    }
    tc_fence_before();
    __syncthreads();
    if constexpr (kPair) cluster_sync();  // the peer's barriers exist before any remote arrive / commit
    tc_fence_after();
    const uint32_t tmem = sm.tmem_base;

    if (warp == 0) {
        // TMA producer: warp-uniform loop, one elected lane issues
        if (elect_one()) {
            tma_prefetch_desc(&p.map_k);
            tma_prefetch_desc(&p.map_v);
            tma_prefetch_desc(&p.map_w);
        }
        __syncwarp();
        int it = 0, j = 0;
        if constexpr (kSplit) {
            // One X tile in four 16 KB boxes (features 0-63 / 64-127 of K, then of V), each with
            // its own full/empty barrier: the MMA releases box b of item j as soon as the last
            // chunk's stages over features [64b, 64b + 64) have run, and box b of item j + 1 is
            // loaded then, while the rest of the last chunk runs. The freed 64 KB doubles the
            // W_U ring. Boxes are polled without blocking between W_U stages; all four must be
            // issued before any stage that only the item's later chunks (or the next item) need.
            uint32_t pend = 0;
            int jp = 0, gp = 0, t0p = 0;
            auto issue_x = [&](bool block) {
                for (int b = 0; b < 4; ++b) {
                    if (!((pend >> b) & 1u)) continue;
                    if (jp >= 1) {
                        const uint32_t par = static_cast<uint32_t>((jp - 1) & 1);
                        if (block)
                            mbar_wait(&sm.a_empty[b], par);
                        else if (!__all_sync(0xffffffffu, mbar_test(&sm.a_empty[b], par)))
                            break;  // released in box order
                    }
                    if (elect_one()) {
                        mbar_arrive_expect_tx(&sm.a_full[b], 16384);
                        tma_load_3d(sA + b * 16384, b < 2 ? &p.map_k : &p.map_v, &sm.a_full[b], (b & 1) * 64, gp, t0p);
                    }
                    __syncwarp();
                    pend &= ~(1u << b);
                }
            };
            for (int w = cl; w < total; w += ncl, ++j) {
                const int g = p.g0 + w / groups_per_head;
                const int t0 = (w % groups_per_head) * kTok;
                issue_x(true);  // the previous item's boxes (single-chunk items)
                jp = j, gp = g, t0p = t0, pend = 0xFu;
                issue_x(false);
                for (int c = 0; c < num_chunks; ++c) {
                    for (int ks = 0; ks < 256 / kStageK; ++ks, ++it) {
                        if (pend) issue_x(c >= 1);
                        const int s = it % kNS;
                        if (it >= kNS) mbar_wait(&sm.empty[s], ((it / kNS) & 1) ^ 1);
                        if (elect_one()) {
                            mbar_arrive_expect_tx(&sm.full[s], kSB);
                            for (int nb = 0; nb < kChunkN / 64; ++nb)
                                tma_load_3d(sB + s * kSB + nb * (kStageK * 128), &p.map_w, &sm.full[s],
                                            c * kChunkN + nb * 64, ks * kStageK, g);
                        }
                        __syncwarp();
                    }
                }
            }
            issue_x(true);
        } else
        for (int w = cl; w < total; w += ncl, ++j) {
            const int g = p.g0 + w / groups_per_head;
            const int tile = (w % groups_per_head) * kMc + rank;
            const int t0 = (tile < p.tiles ? tile : 0) * kTok;  // past the end: any valid tile, no store
            const int buf = j & 1;
            if (j >= 2) mbar_wait(&sm.a_empty[buf], ((j >> 1) & 1) ^ 1);
            if (elect_one()) {
                uint8_t* a = sA + buf * kABytes;
                if (leader) {
                    mbar_arrive_expect_tx(&sm.a_full[buf], kMc * kABytes);  // the pair's tiles land on the leader's barrier
                    for (int hf = 0; hf < 2; ++hf) {
                        tma_load_3d(a + hf * 16384, &p.map_k, &sm.a_full[buf], hf * 64, g, t0);
                        tma_load_3d(a + (2 + hf) * 16384, &p.map_v, &sm.a_full[buf], hf * 64, g, t0);
                    }
                } else if constexpr (kPair) {
                    const uint32_t bar = mapa_shared(smem_u32(&sm.a_full[buf]), 0);
                    for (int hf = 0; hf < 2; ++hf) {
                        tma_load_3d_pair(a + hf * 16384, &p.map_k, bar, hf * 64, g, t0);
                        tma_load_3d_pair(a + (2 + hf) * 16384, &p.map_v, bar, hf * 64, g, t0);
                    }
                }
            }
            __syncwarp();
            for (int c = 0; c < num_chunks; ++c) {
                for (int ks = 0; ks < 256 / kStageK; ++ks, ++it) {
                    const int s = it % kNS;
                    if (it >= kNS) mbar_wait(&sm.empty[s], ((it / kNS) & 1) ^ 1);
                    if (elect_one()) {
                        uint8_t* dst = sB + s * kSB;
                        const int n0 = c * kChunkN + rank * kNCta;  // this CTA's columns of the chunk
                        if (leader) {
                            mbar_arrive_expect_tx(&sm.full[s], kMc * kSB);
                            for (int nb = 0; nb < kNCta / 64; ++nb)
                                tma_load_3d(dst + nb * (kStageK * 128), &p.map_w, &sm.full[s], n0 + nb * 64,
                                            ks * kStageK, g);
                        } else if constexpr (kPair) {
                            const uint32_t bar = mapa_shared(smem_u32(&sm.full[s]), 0);
                            for (int nb = 0; nb < kNCta / 64; ++nb)
                                tma_load_3d_pair(dst + nb * (kStageK * 128), &p.map_w, bar, n0 + nb * 64, ks * kStageK, g);
                        }
                    }
                    __syncwarp();
                }
            }
        }
        if constexpr (kPair) {
            // drain: the leader's commits for the last uses of every ring slot and X buffer have
            // arrived here before the pair may exit (no remote arrive left in flight)
            for (int i = it; i < it + kNS; ++i)
                if (i >= kNS) mbar_wait(&sm.empty[i % kNS], ((i / kNS) & 1) ^ 1);
            for (int jj = j; jj < j + 2; ++jj)
                if (jj >= 2) mbar_wait(&sm.a_empty[jj & 1], ((jj >> 1) & 1) ^ 1);
        }
    } else if (warp == 1) {
        // MMA issuer (the pair's leader only): warp-uniform loop, one elected lane issues each batch
        if (leader) {
            const uint32_t idesc = umma_idesc_bf16(128 * kMc, kChunkN, false, true);
            const uint64_t b_desc0 = umma_desc_sw128(smem_u32(sB), kStageK * 128, 1024);
            int it = 0, cc = 0, j = 0;
            for (int w = cl; w < total; w += ncl, ++j) {
                const int buf = kSplit ? 0 : (j & 1);
                const uint64_t a_desc0 = umma_desc_sw128(smem_u32(sA + buf * kABytes), 16, 1024);
                if constexpr (!kSplit) mbar_wait(&sm.a_full[buf], (j >> 1) & 1);
                for (int c = 0; c < num_chunks; ++c, ++cc) {
                    const int acc = cc & 1;
                    if (cc >= 2) mbar_wait(&sm.acc_empty[acc], ((cc >> 1) & 1) ^ 1);
                    tc_fence_after();
                    for (int ks = 0; ks < 256 / kStageK; ++ks, ++it) {
                        const int s = it % kNS;
                        mbar_wait(&sm.full[s], (it / kNS) & 1);
                        if constexpr (kSplit)  // first stage over X box b in this item
                            if (c == 0 && ((ks * kStageK) & 63) == 0) mbar_wait(&sm.a_full[(ks * kStageK) >> 6], j & 1);
                        tc_fence_after();
                        if (elect_one()) {
#pragma unroll
                            for (int kk = 0; kk < kStageK / 16; ++kk) {
#ifdef VSP_K1_HALF_MMA  // probe (tools/dev/gpu_k1probe2.sh): half the MMAs, same W/X stream
                                if (kk & 1) continue;
#endif
                                const int kg = ks * kStageK + kk * 16;  // global K index (feature)
                                const uint64_t adesc =
                                    a_desc0 + static_cast<uint64_t>(((kg >> 6) * 16384 + (kg & 63) * 2) >> 4);
                                const uint64_t bdesc = b_desc0 + static_cast<uint64_t>((s * kSB + kk * 2048) >> 4);
                                const uint32_t accum = (ks > 0 || kk > 0) ? 1u : 0u;
                                if constexpr (kPair)
                                    umma_ss_pair(tmem + acc * kChunkN, adesc, bdesc, idesc, accum);
                                else
                                    umma_ss(tmem + acc * kChunkN, adesc, bdesc, idesc, accum);
                            }
                            if constexpr (kPair) {
                                umma_commit_pair_mc(&sm.empty[s], 3);
                                if (ks == 256 / kStageK - 1) {
                                    umma_commit_pair_mc(&sm.acc_full[acc], 3);
                                    if (c == num_chunks - 1) umma_commit_pair_mc(&sm.a_empty[buf], 3);
                                }
                            } else {
                                umma_commit(&sm.empty[s]);
                                if constexpr (kSplit)  // last chunk done with X box b: release it
                                    if (c == num_chunks - 1 && ((ks * kStageK + kStageK) & 63) == 0)
                                        umma_commit(&sm.a_empty[(ks * kStageK) >> 6]);
                                if (ks == 256 / kStageK - 1) {
                                    umma_commit(&sm.acc_full[acc]);
                                    if (!kSplit && c == num_chunks - 1) umma_commit(&sm.a_empty[buf]);
                                }
                            }
                        }
                        __syncwarp();
                    }
                }
            }
            if constexpr (kPair) {
                // drain: both epilogues' releases of the last two accumulators have arrived
                for (int c2 = cc; c2 < cc + 2; ++c2)
                    if (c2 >= 2) mbar_wait(&sm.acc_empty[c2 & 1], ((c2 >> 1) & 1) ^ 1);
            }
        }
    } else {
        // epilogue warps 2..9: TMEM lane quarter = warp % 4; part = which 128-column half of
        // each 256-wide accumulator chunk this warp reduces (two warps per lane quarter)
        const int quarter = warp & 3;
        const int part = (warp - 2) >> 2;
        const int r = quarter * 32 + lane;
        const uint32_t lane_base = tmem + (static_cast<uint32_t>(quarter * 32) << 16);
        const int et = threadIdx.x - 64;  // 0..kEpiThreads-1
        int cc = 0, j = 0, cur_g = -1;
        for (int w = cl; w < total; w += ncl, ++j) {
            const int g = p.g0 + w / groups_per_head;
            const int t = ((w % groups_per_head) * kMc + rank) * kTok + r;  // >= n past the end: no store
            if (g != cur_g) {  // head change: everyone is past the previous tile's exchange
                for (int i = et; i < p.d_h; i += kEpiThreads) {
                    s_bh[i] = 0.5f * p.b_u[static_cast<size_t>(g) * p.d_h + i];
                    s_wv[i] = p.w_v[static_cast<size_t>(g) * p.d_h + i];
                    s_ws[i] = p.w_s[static_cast<size_t>(g) * p.d_h + i];
                }
                named_bar_sync(1, kEpiThreads);
                cur_g = g;
            }
            float2 lv = make_float2(0.f, 0.f), ls = make_float2(0.f, 0.f);
            float2 lv1 = lv, ls1 = ls;  // two independent chains per dot
            for (int c = 0; c < num_chunks; ++c, ++cc) {
                const int acc = cc & 1;
                mbar_wait(&sm.acc_full[acc], (cc >> 1) & 1);
                tc_fence_after();
                uint32_t ub[2][32];  // ping-pong: the next 32 columns load while these compute
                tmem_ld32(lane_base + acc * kChunkN + part * (kChunkN / kEpiParts), ub[0]);
                tmem_wait_ld(ub[0]);
#pragma unroll
                for (int q = 0; q < kChunkN / (32 * kEpiParts); ++q) {
                    uint32_t* u = ub[q & 1];
                    const int col = part * (kChunkN / kEpiParts) + q * 32;
                    if (q + 1 < kChunkN / (32 * kEpiParts)) tmem_ld32(lane_base + acc * kChunkN + col + 32, ub[(q + 1) & 1]);
                    const int col0 = c * kChunkN + col;
                    const float4* bh4 = reinterpret_cast<const float4*>(s_bh + col0);
                    const float4* wv4 = reinterpret_cast<const float4*>(s_wv + col0);
                    const float4* ws4 = reinterpret_cast<const float4*>(s_ws + col0);
#ifdef VSP_K1_NOEPI  // probe (tools/dev/gpu_k1probe.sh): accumulator hand-off only, no SiLU / dots
                    lv.x += __uint_as_float(u[0]);
                    if (false)
#endif
#pragma unroll
                    for (int x4 = 0; x4 < 8; ++x4) {
                        const float4 b = bh4[x4], wv = wv4[x4], ws = ws4[x4];
                        // h = y/2 + b/2 ; z = h + h tanh(h) ; packed f32x2 for everything but MUFU
                        const float2 h0 = ffma2(make_float2(__uint_as_float(u[4 * x4]), __uint_as_float(u[4 * x4 + 1])),
                                                make_float2(0.5f, 0.5f), make_float2(b.x, b.y));
                        const float2 h1 = ffma2(make_float2(__uint_as_float(u[4 * x4 + 2]), __uint_as_float(u[4 * x4 + 3])),
                                                make_float2(0.5f, 0.5f), make_float2(b.z, b.w));
                        const float2 z0 = ffma2(h0, make_float2(tanh_f(h0.x), tanh_f(h0.y)), h0);
                        const float2 z1 = ffma2(h1, make_float2(tanh_f(h1.x), tanh_f(h1.y)), h1);
                        lv = ffma2(z0, make_float2(wv.x, wv.y), lv);
                        ls = ffma2(z0, make_float2(ws.x, ws.y), ls);
                        lv1 = ffma2(z1, make_float2(wv.z, wv.w), lv1);
                        ls1 = ffma2(z1, make_float2(ws.z, ws.w), ls1);
                    }
                    if (q + 1 < kChunkN / (32 * kEpiParts)) tmem_wait_ld(ub[(q + 1) & 1]);
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) {
                    if constexpr (kPair)
                        mbar_arrive_cluster(mapa_shared(smem_u32(&sm.acc_empty[acc]), 0));  // the leader's
                    else
                        mbar_arrive(&sm.acc_empty[acc]);
                }
            }
            const float sv = (lv.x + lv.y) + (lv1.x + lv1.y);
            const float ss = (ls.x + ls.y) + (ls1.x + ls1.y);
            float* xch = s_xch + (j & 1) * (kEpiParts - 1) * 256;
            if (part > 0) {
                xch[(part - 1) * 256 + r] = sv;
                xch[(part - 1) * 256 + 128 + r] = ss;
            }
            named_bar_sync(1, kEpiThreads);
            if (part == 0 && t < p.n) {
                float tv = sv, ts = ss;
#pragma unroll
                for (int q = 0; q < kEpiParts - 1; ++q) {  // fixed order: deterministic sums
                    tv += xch[q * 256 + r];
                    ts += xch[q * 256 + 128 + r];
                }
                p.logit_v[static_cast<size_t>(g) * p.n + t] = tv + p.b_v[g];
                const int o = p.reverse ? p.n - 1 - t : t;
                p.logit_s[static_cast<size_t>(g) * p.n + o] = ts + p.b_s[g];
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if constexpr (kPair) {
        cluster_sync();  // both CTAs are done with the pair's TMEM and barriers
        if (warp == 1) tmem_free_pair<512>(tmem);
    } else {
        if (warp == 1) tmem_free<512>(tmem);
    }
}

constexpr int kSmemBytes = 2 * kABytes + kRingBytes + 3 * kMaxDh * 4 + 2 * (kEpiParts - 1) * 256 * 4 + 1024;
static_assert(2 * kABytes + kRingBytes == kABytes + kSplitRingBytes, "both X/W_U layouts fill the same bytes");

size_t workspace_bytes(int n, int hkv, int /*d_h*/) {
    return 2 * static_cast<size_t>(hkv) * n * sizeof(float) + 256;
}

cudaError_t launch(const Args& a, void* workspace, cudaStream_t stream) {
    if (a.d_h > kMaxDh || a.d_h % kChunkN != 0) return cudaErrorInvalidValue;
    Params p{};
    const uint32_t box[3] = {64, 1, kTok};
    static_assert(kSmemBytes <= 227 * 1024, "indexer smem");
    const uint64_t dk[3] = {128, (uint64_t)a.hkv, (uint64_t)a.n};
    const uint64_t sk[2] = {128 * 2, (uint64_t)a.hkv * 128 * 2};
    const uint64_t dw[3] = {(uint64_t)a.d_h, 256, (uint64_t)a.hkv};
    const uint64_t sw[2] = {(uint64_t)a.d_h * 2, (uint64_t)a.d_h * 256 * 2};
    if (!vsp_host::make_map_bf16(&p.map_k, a.k, 3, dk, sk, box) ||
        !vsp_host::make_map_bf16(&p.map_v, a.v, 3, dk, sk, box))
        return cudaErrorInvalidValue;
    float* lv = a.logits_v ? a.logits_v : static_cast<float*>(workspace);
    float* ls = a.logits_s ? a.logits_s : static_cast<float*>(workspace) + static_cast<size_t>(a.hkv) * a.n;
    p.b_u = a.b_u;
    p.w_v = a.w_v;
    p.w_s = a.w_s;
    p.b_v = a.b_v;
    p.b_s = a.b_s;
    p.logit_v = lv;
    p.logit_s = ls;
    p.n = a.n;
    p.hkv = a.hkv;
    p.d_h = a.d_h;
    p.reverse = a.reverse ? 1 : 0;
    static std::once_flag attr[vsp_detail::kMaxDevices];
    vsp_detail::once_per_device(attr, [] {
        cudaFuncSetAttribute(indexer_gemm_kernel<false, 32, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes);
        cudaFuncSetAttribute(indexer_gemm_kernel<false, 64, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes);
        cudaFuncSetAttribute(indexer_gemm_kernel<true, 32, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes);
        cudaFuncSetAttribute(indexer_gemm_kernel<true, 64, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes);
        cudaFuncSetAttribute(indexer_gemm_kernel<false, 32, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes);
    });
    const int count = a.count < 0 ? a.hkv - a.g0 : a.count;
    p.g0 = a.g0;
    p.count = count;
    p.tiles = (a.n + kTok - 1) / kTok;
    const int sms = vsp_detail::current_sm_count();
    // VSP_K1_MC = 1: one CTA per tile; 2: CTA pairs (cta_group::2); single tiles need no pair.
    // VSP_K1_STAGEK = 32 / 64: W_U K-rows per ring stage (the ring stays 64 KB)
    int mc = kDefaultMc, stage_k = kDefaultStageK, split = kDefaultSplit;
    if (const char* s = getenv("VSP_K1_MC")) mc = atoi(s);
    if (const char* s = getenv("VSP_K1_SPLIT")) split = atoi(s) != 0;
    if (const char* s = getenv("VSP_K1_STAGEK")) stage_k = atoi(s);
    if (mc != 1 && mc != 2) mc = kDefaultMc;
    if (stage_k != 32 && stage_k != 64) stage_k = kDefaultStageK;
    if (p.tiles < 2) mc = 1;
    if (mc != 1 || stage_k != 32) split = 0;  // split-X: one CTA per tile, 32-row stages
    const uint32_t wbox[3] = {64, static_cast<uint32_t>(stage_k), 1};
    if (!vsp_host::make_map_bf16(&p.map_w, a.w_u, 3, dw, sw, wbox)) return cudaErrorInvalidValue;
    const int groups = ((p.tiles + mc - 1) / mc) * count;
    const int clusters = std::max(1, std::min(groups, sms / mc));
    vsp_detail::count_launch();
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(clusters * mc);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = kSmemBytes;
    cfg.stream = stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = mc;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaError_t e = split         ? cudaLaunchKernelEx(&cfg, indexer_gemm_kernel<false, 32, true>, p)
                    : mc == 2     ? (stage_k == 64 ? cudaLaunchKernelEx(&cfg, indexer_gemm_kernel<true, 64, false>, p)
                                                   : cudaLaunchKernelEx(&cfg, indexer_gemm_kernel<true, 32, false>, p))
                    : stage_k == 64 ? cudaLaunchKernelEx(&cfg, indexer_gemm_kernel<false, 64, false>, p)
                                    : cudaLaunchKernelEx(&cfg, indexer_gemm_kernel<false, 32, false>, p);
    if (e == cudaSuccess) e = cudaGetLastError();
    // A_v / A_s: the cluster softmax shared with the selection kernel (a_v null: logits only,
    // the layer path softmaxes inside selection)
    if (e == cudaSuccess && a.a_v) e = vsp_select_k::launch_softmax(lv, ls, a.a_v, a.a_s, a.n, a.g0, count, stream);
    return e;
}

}  // namespace vsp_indexer
