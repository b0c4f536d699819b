// aggregate.cu — K5: ground-truth vertical/slash aggregation on sm_100a.
//
// Replaces vsp::aggregate_streaming (reference vsaggregate.hpp:62-127) for every Q head,
// fused with combine_scores (vsaggregate.hpp:133-157) over each KV group:
//   pass 1: LSE_i of every row (online softmax; vsaggregate.hpp:83-103) — K4's LSE output
//   pass 2: w = exp(s_ij - LSE_i); vertical[j] += w; slash[i - j] += w (:109-124)
//   normalize by n (:27-33), then group Mean (or Sum).
// The n x n weights never exist.
//
// Pass 2 works on TRANSPOSED tiles: S^T = K_J Q_I^T (tcgen05, M = 128 keys, N = 128 query
// rows, TMEM), so the softmax thread that owns TMEM lane c holds key j = 128J + c against
// all 128 query rows of the tile:
//   * vertical[j] = sum over rows of P^T[c][.] — a running fp32 register sum per thread, for
//     every query block and head the CTA visits; one atomic per key at the end.
//   * slash: offset o = i - j = 128(t-1) + cc' - (c & 7) with t = I - J and the COARSE
//     column cc' = r + 128 - 8*floor(c/8). The thread writes its 128 weights as bf16 to row c
//     of a [128 x 256] shared buffer starting at cc' (a 16-byte aligned chunk: 16 plain
//     vector stores, no per-element skew), and the tensor core reduces the columns against a
//     SELECTOR B[c][f] = (f == c & 7) (M=128 coarse columns, N=8, K=128 keys): D[x][f] =
//     sum over keys with c & 7 == f. The true diagonal is slash[o] = sum_f E[o + f][f], with
//     E the coarse accumulator; that 8-term combination runs once per CTA in the flush.
// CTA = one 128-key block J (K tile resident), one KV group, a chunk of up to 14 query
// blocks, all Q heads of the group (two softmax warpgroups take alternate heads and
// ping-pong against the tensor core). Every coarse offset block the CTA touches keeps its own
// TMEM accumulator (15 x 8 columns), so nothing is flushed until the CTA ends. CTAs are
// ordered (query chunk, group, key block) so concurrently resident CTAs stream the same Q
// tiles from L2.
#include <cuda_bf16.h>

#include <algorithm>
#include <cmath>
#include <type_traits>

#include "vsp_launch.h"
#include "aggregate.h"
#include "attn.h"
#include "sm100.cuh"
#include "tma_host.h"

using namespace vsp_sm100;

namespace vsp_aggregate {

#ifndef VSP_K5_TS
#define VSP_K5_TS 0      // S^T as a TS MMA: the CTA's K tile resident in TMEM (A operand)
#endif
#ifndef VSP_K5_SBUFS
#define VSP_K5_SBUFS 3
#endif
#ifndef VSP_K5_CHUNK
#define VSP_K5_CHUNK 14
#endif
#ifndef VSP_K5_PBUFS
#define VSP_K5_PBUFS 1   // 2: one coarse P buffer per softmax warpgroup (TS form only)
#endif

constexpr int kBlock = 128;
constexpr int kTile = kBlock * 128 * 2;  // 32 KB bf16 tile
constexpr int kHalf = kTile / 2;
constexpr int kChunk = VSP_K5_CHUNK;     // query blocks per CTA (kChunk + 1 coarse blocks in TMEM)
constexpr int kPBufs = VSP_K5_PBUFS;
static_assert(kPBufs == 1 || (kPBufs == 2 && VSP_K5_TS), "two P buffers reuse the K tile's smem");
constexpr int kQStages = kPBufs == 2 ? 2 : 3;
constexpr int kLStages = 6;              // LSE rows: released late (after the exps), so deeper
constexpr int kThreads = 384;            // warp0 TMA, warp1 MMA, warps 4-11 two softmax groups
constexpr int kAccCols = 8;              // N = 8 selector columns per coarse accumulator
constexpr int kSBufs = VSP_K5_SBUFS;     // S^T TMEM buffers (items rotate through them)
constexpr bool kTsS = VSP_K5_TS != 0;
constexpr int kKCol = 448;               // TS form: K tile as packed bf16 pairs, columns [448, 512)
static_assert(kSBufs * 128 + (kChunk + 1) * kAccCols <= (kTsS ? kKCol : 512), "aggregate TMEM budget");
constexpr float kLog2e = 1.4426950408889634f;

struct __align__(64) Params {
    CUtensorMap map_q, map_k;
    const float* lse;  // [hq, n]
    unsigned long long* acc_v;  // [hkv, n] fixed-point (2^52) accumulators: integer atomics are
    unsigned long long* acc_s;  // order-independent, so the aggregates are bit-reproducible
    int n, hq, hkv, num_qb, num_qc;
    float scale;       // 1/sqrt(d)
    float out_scale;   // (normalized ? 1/n : 1) * (mean ? 1/group : 1)
    double fix_scale;  // 2^52 / (power of two >= the expected total of one profile)
};

struct Smem {
    uint64_t bar_k;
    uint64_t q_full[kQStages], q_empty[kQStages];
    uint64_t l_full[kLStages], l_empty[kLStages];
    uint64_t s_full[kSBufs], s_free[kSBufs];
    uint64_t p_full[2], p_free[2], all_done;  // [b]: items with k & 1 == b (P written / reduced)
    uint64_t k_tmem;                        // TS form: the K tile is in TMEM
    uint32_t tmem_base;
};

// smem: K 32K | Q ring 3 x 32K | P coarse 64K (4 x [128 x 64] SW128 blocks) | selector 4K |
//       lse ring 6 x 512 B | vertical exchange 512 B | flush staging 2 x 136 x 8 floats
// two P buffers: P1 = [0, 64K) takes over the K tile once it is in TMEM; the Q ring has 2 stages
constexpr int kOffK = 0;
constexpr int kOffQ = kPBufs == 2 ? 2 * kTile : kTile;
constexpr int kOffP = kOffQ + kQStages * kTile;
constexpr int kOffP1 = kPBufs == 2 ? 0 : kOffP;
constexpr int kOffSel = kOffP + 2 * kTile;
constexpr int kOffLse = kOffSel + 4096;
constexpr int kOffVx = kOffLse + kLStages * 512;
constexpr int kOffStage = kOffVx + 512;
constexpr int kStageFloats = 136 * 8;
constexpr int kSmemBytes = kOffStage + 2 * kStageFloats * 4 + 1024;
static_assert(kSmemBytes <= 227 * 1024, "aggregate smem");

VSP_DEVICE unsigned long long to_fixed(float x, double scale) {
    return static_cast<unsigned long long>(__double2ll_rn(static_cast<double>(x) * scale));
}

// (query chunk, group, key block) of this CTA; chunk qc covers query blocks
// [kChunk*qc, kChunk*qc + kChunk) and pairs with key blocks J < min(num_qb, kChunk*(qc+1)).
VSP_DEVICE void decode_cta(const Params& p, int& qc, int& g, int& jb) {
    int b = blockIdx.x;
    for (qc = 0; qc < p.num_qc; ++qc) {
        const int per = min(p.num_qb, kChunk * (qc + 1)) * p.hkv;
        if (b < per) break;
        b -= per;
    }
    const int nj = min(p.num_qb, kChunk * (qc + 1));
    g = b / nj;
    jb = b % nj;
}

__global__ void __launch_bounds__(kThreads, 1) aggregate_kernel(const __grid_constant__ Params p) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* base = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    __shared__ Smem sm;
    const int grp = p.hq / p.hkv;
    int qc, g, jb;
    decode_cta(p, qc, g, jb);
    const int i_first = max(jb, kChunk * qc);
    const int i_end = min(p.num_qb, kChunk * (qc + 1));
    const int t0 = i_first - jb;              // first t = I - J of this CTA
    const int nblk = i_end - i_first;         // query blocks (>= 1)
    const int num_items = nblk * grp;
    const int j0 = jb * kBlock;
    const uint32_t warp = warp_id(), lane = lane_id();
    float* lse_ring = reinterpret_cast<float*>(base + kOffLse);

    if (warp == 0 && lane == 0) {
        mbar_init(&sm.bar_k, 1);
        for (int s = 0; s < kQStages; ++s) {
            mbar_init(&sm.q_full[s], 1);
            mbar_init(&sm.q_empty[s], 1);
        }
        for (int s = 0; s < kLStages; ++s) {
            mbar_init(&sm.l_full[s], 1);
            mbar_init(&sm.l_empty[s], 4);
        }
        for (int b = 0; b < kSBufs; ++b) {
            mbar_init(&sm.s_full[b], 1);
            mbar_init(&sm.s_free[b], 4);
        }
        mbar_init(&sm.p_full[0], 4);
        mbar_init(&sm.p_full[1], 4);
        mbar_init(&sm.p_free[0], 1);
        mbar_init(&sm.p_free[1], 1);
        mbar_init(&sm.all_done, 1);
        mbar_init(&sm.k_tmem, 4);
        fence_barrier_init();
    }
    if (warp == 1) tmem_alloc<512>(&sm.tmem_base);
    // zero the coarse P buffer once (each row's band is fixed, the rest stays zero) and
    // build the selector B[c][f] = (f == c & 7): K-major [16 x 128], two SW128 K-halves
    {
        uint4* pz = reinterpret_cast<uint4*>(base + kOffP);
        for (int i = threadIdx.x; i < 2 * kTile / 16; i += kThreads) pz[i] = make_uint4(0, 0, 0, 0);
        if (kPBufs == 2) {  // the upper half of P1 (the lower half holds K until it is in TMEM)
            uint4* pz1 = reinterpret_cast<uint4*>(base + kOffP1 + kTile);
            for (int i = threadIdx.x; i < kTile / 16; i += kThreads) pz1[i] = make_uint4(0, 0, 0, 0);
        }
        uint16_t* sel = reinterpret_cast<uint16_t*>(base + kOffSel);
        for (int i = threadIdx.x; i < 16 * 128; i += kThreads) {
            const int f = i >> 7, c = i & 127;
            const int cl = c & 63;
            const uint32_t off = (c >> 6) * 2048 + f * 128 + ((((cl >> 3) ^ (f & 7)) << 4) | ((cl & 7) << 1));
            sel[off >> 1] = (f < 8 && f == (c & 7)) ? 0x3f80u : 0u;  // bf16 1.0
        }
        fence_proxy_async_smem();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = sm.tmem_base;
    // TMEM: S^T buffers [0, 128 kSBufs); coarse accumulators: slot s at columns 128 kSBufs + 8 s
    // (kChunk + 1 slots); TS form: K (A operand, lane = key, column = packed d pair) at [448, 512)
    const uint32_t t_acc = tmem + kSBufs * 128;
    const uint32_t t_k = tmem + kKCol;

    if (warp == 0) {
        // =========================== producer: K once; per item the Q tile (TMA) + LSE row
        if (elect_one()) {
            tma_prefetch_desc(&p.map_q);
            tma_prefetch_desc(&p.map_k);
            mbar_arrive_expect_tx(&sm.bar_k, kTile);
            for (int hf = 0; hf < 2; ++hf)
                tma_load_3d(base + kOffK + hf * kHalf, &p.map_k, &sm.bar_k, hf * 64, g, j0);
        }
        __syncwarp();
        for (int k = 0; k < num_items; ++k) {
            const int ib = i_first + k / grp;
            const int h = g * grp + k % grp;
            const int s = k % kQStages;
            if (k >= kQStages) mbar_wait(&sm.q_empty[s], ((k / kQStages) - 1) & 1);
            if (elect_one()) {
                mbar_arrive_expect_tx(&sm.q_full[s], kTile);
                for (int hf = 0; hf < 2; ++hf)
                    tma_load_3d(base + kOffQ + s * kTile + hf * kHalf, &p.map_q, &sm.q_full[s], hf * 64, h,
                                ib * kBlock);
            }
            __syncwarp();
            // LSE of the tile's rows in log2 units; rows past n get +inf (weight exactly 0)
            const int ls = k % kLStages;
            if (k >= kLStages) mbar_wait(&sm.l_empty[ls], ((k / kLStages) - 1) & 1);
            float4 l4;
            const int i = ib * kBlock + 4 * lane;
            const float* src = p.lse + static_cast<size_t>(h) * p.n;
            l4.x = i + 0 < p.n ? __ldg(src + i + 0) * kLog2e : INFINITY;
            l4.y = i + 1 < p.n ? __ldg(src + i + 1) * kLog2e : INFINITY;
            l4.z = i + 2 < p.n ? __ldg(src + i + 2) * kLog2e : INFINITY;
            l4.w = i + 3 < p.n ? __ldg(src + i + 3) * kLog2e : INFINITY;
            reinterpret_cast<float4*>(lse_ring + ls * kBlock)[lane] = l4;
            __syncwarp();
            if (elect_one()) mbar_arrive(&sm.l_full[ls]);
            __syncwarp();
        }
    } else if (warp == 1) {
        // =========================== MMA issuer (warp-uniform loop, elected lane issues)
        const uint32_t idesc_s = umma_idesc_bf16(128, 128, false, false);
        const uint32_t idesc_red = umma_idesc_bf16(128, kAccCols, true, false);
        const uint64_t k_desc0 = umma_desc_sw128(smem_u32(base + kOffK), 16, 1024);
        const uint64_t q_desc0 = umma_desc_sw128(smem_u32(base + kOffQ), 16, 1024);
        const uint64_t sel_desc0 = umma_desc_sw128(smem_u32(base + kOffSel), 16, 1024);
        const uint32_t p_addr = smem_u32(base + kOffP);
        const uint32_t p_addr1 = smem_u32(base + kOffP1);
        auto issue_s = [&](int k) {  // S^T = K Q^T into TMEM buffer k % 3
            const int s = k % kQStages;
            const int b = k % kSBufs;
            mbar_wait(&sm.q_full[s], (k / kQStages) & 1);
            if (k >= kSBufs) mbar_wait(&sm.s_free[b], ((k / kSBufs) - 1) & 1);
            tc_fence_after();
            if (elect_one()) {
#pragma unroll
                for (int kk = 0; kk < 8; ++kk) {
                    const uint64_t off = static_cast<uint64_t>(((kk >> 2) * kHalf + (kk & 3) * 32) >> 4);
                    if constexpr (kTsS)
                        umma_ts(tmem + b * 128, t_k + kk * 8, q_desc0 + static_cast<uint64_t>((s * kTile) >> 4) + off,
                                idesc_s, kk > 0 ? 1u : 0u);
                    else
                        umma_ss(tmem + b * 128, k_desc0 + off, q_desc0 + static_cast<uint64_t>((s * kTile) >> 4) + off,
                                idesc_s, kk > 0 ? 1u : 0u);
                }
                umma_commit(&sm.s_full[b]);
                umma_commit(&sm.q_empty[s]);
            }
            __syncwarp();
        };
        // D[slot] (+)= Pc[:, half]^T . Sel   (M = 128 coarse columns, K = 128 keys)
        auto issue_red = [&](uint32_t pa, int slot, int half, bool acc) {
            const uint64_t a0 = umma_desc_sw128(pa + half * 2 * kHalf, kHalf, 1024);
#pragma unroll
            for (int kk = 0; kk < 8; ++kk)
                umma_ss(t_acc + slot * kAccCols, a0 + static_cast<uint64_t>((kk * 2048) >> 4),
                        sel_desc0 + static_cast<uint64_t>(((kk >> 2) * 2048 + (kk & 3) * 32) >> 4), idesc_red,
                        (acc || kk > 0) ? 1u : 0u);
        };
        mbar_wait(&sm.bar_k, 0);
        if constexpr (kTsS) mbar_wait(&sm.k_tmem, 0);
        for (int k = 0; k < kSBufs && k < num_items; ++k) issue_s(k);
        for (int k = 0; k < num_items; ++k) {
            const int tl = k / grp, hh = k % grp;
            const int t = t0 + tl;
            // tcgen05.mma runs in issue order, so the reduction of item k goes in right after
            // its P is written (the next warpgroup waits for p_free), and S(k+3) — needed only
            // after the other warpgroup's next item — goes in behind it
            mbar_wait(&sm.p_full[k & 1], (k >> 1) & 1);
            tc_fence_after();
            if (elect_one()) {
                const uint32_t pa = (kPBufs == 2 && (k & 1)) ? p_addr1 : p_addr;
                // lower half -> coarse block t-1 (slot tl), upper half -> block t (slot tl+1)
                if (t >= 1) issue_red(pa, tl, 0, tl > 0 || hh > 0);
                issue_red(pa, tl + 1, 1, hh > 0);
                umma_commit(&sm.p_free[k & 1]);
                if (k == num_items - 1) umma_commit(&sm.all_done);
            }
            __syncwarp();
            if (k + kSBufs < num_items) issue_s(k + kSBufs);
        }
    } else if (warp >= 4) {
        // =========================== softmax groups: WG w takes items k with k & 1 == w
        const int w = (warp - 4) >> 2;
        const int quarter = warp & 3;
        const int c = quarter * 32 + lane;  // key row (TMEM lane) within block J
        const uint32_t lane_base = static_cast<uint32_t>(quarter * 32) << 16;
        const float sl2 = p.scale * kLog2e;
        // this thread's row of the coarse buffer starts at chunk 16 - c/8 (column 128 - 8 floor(c/8))
        uint8_t* prow = base + (kPBufs == 2 && w == 1 ? kOffP1 : kOffP) + c * 128;
        const int a0 = 16 - (c >> 3);
        float2 vacc = make_float2(0.f, 0.f);
        if (kTsS && w == 0) {
            // K row c (SW128: 16-byte chunk q of d-half hf at chunk q ^ (c & 7)) -> TMEM lane c,
            // column hf * 32 + 4 q + e = packed (d, d + 1) pairs, the TS A-operand layout
            mbar_wait(&sm.bar_k, 0);
#pragma unroll
            for (int hf = 0; hf < 2; ++hf) {
                uint32_t u[32];
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    const uint4 x = *reinterpret_cast<const uint4*>(base + kOffK + hf * kHalf + c * 128 + ((q ^ (c & 7)) << 4));
                    u[4 * q] = x.x;
                    u[4 * q + 1] = x.y;
                    u[4 * q + 2] = x.z;
                    u[4 * q + 3] = x.w;
                }
                tmem_st32(t_k + lane_base + hf * 32, u);
            }
            tmem_wait_st();
            if constexpr (kPBufs == 2) {  // the K tile's smem becomes the lower half of P1
                __syncwarp();
                named_bar_sync(4, 128);
                uint4* pz1 = reinterpret_cast<uint4*>(base + kOffP1);
                for (int i = c; i < kTile / 16; i += 128) pz1[i] = make_uint4(0, 0, 0, 0);
                fence_proxy_async_smem();
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&sm.k_tmem);
        }
        if (kPBufs == 2 && w == 1) mbar_wait(&sm.k_tmem, 0);
        for (int k = w; k < num_items; k += 2) {
            const int tl = k / grp;
            const int t = t0 + tl;
            const int ls = k % kLStages;
            const bool plain = t > 0 && (i_first + tl + 1) * kBlock <= p.n;  // no causal mask, full rows
            mbar_wait(&sm.l_full[ls], (k / kLStages) & 1);
            const int sb = k % kSBufs;
            mbar_wait(&sm.s_full[sb], (k / kSBufs) & 1);
            tc_fence_after();
            const float4* l4 = reinterpret_cast<const float4*>(lse_ring + ls * kBlock);
            // The exp pass is straight-line code per 32-column chunk (no per-element branches:
            // the two variants are separate instantiations), so the scheduler can interleave
            // the MUFU / FMA chains of 32 independent elements. Packed bf16 weights of chunk cq
            // go back into TMEM columns [16 cq, 16 cq + 16) of the same S^T buffer (already
            // consumed), so the row is not held in registers while waiting for the P buffer.
            const uint32_t s_t = tmem + lane_base + sb * 128;
            auto exp_pass = [&](auto plain_tag) {
                constexpr bool kPlain = decltype(plain_tag)::value;
                // diagonal tile: keep r >= c; elsewhere nothing is masked (ragged rows carry
                // lse = +inf and come out exactly 0 on the MUFU path)
                const int lim = t == 0 ? c : 0;
                float2 acc[4] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f),
                                 make_float2(0.f, 0.f)};
                uint32_t u[2][32];
                tmem_ld32(s_t, u[0]);
                tmem_wait_ld(u[0]);
#pragma unroll
                for (int cq = 0; cq < 4; ++cq) {
                    if (cq < 3) tmem_ld32(s_t + (cq + 1) * 32, u[(cq + 1) & 1]);
                    const uint32_t* x = u[cq & 1];
                    uint32_t pk[16];
#pragma unroll
                    for (int e4 = 0; e4 < 8; ++e4) {
                        const float4 l = l4[cq * 8 + e4];
                        const int r = cq * 32 + e4 * 4;
                        float2 y0 = ffma2(make_float2(__uint_as_float(x[4 * e4]), __uint_as_float(x[4 * e4 + 1])),
                                          make_float2(sl2, sl2), make_float2(-l.x, -l.y));
                        float2 y1 = ffma2(make_float2(__uint_as_float(x[4 * e4 + 2]), __uint_as_float(x[4 * e4 + 3])),
                                          make_float2(sl2, sl2), make_float2(-l.z, -l.w));
                        float2 e0, e1;
                        if constexpr (kPlain) {
                            // 3 pairs in 8 on the FMA pipe, the rest on MUFU (the K4 balance)
                            if ((0x54u >> e4) & 1u) {
                                e0 = exp2_poly2(y0);
                                e1 = exp2_poly2(y1);
                            } else {
                                e0 = make_float2(ex2_approx(y0.x), ex2_approx(y0.y));
                                e1 = make_float2(ex2_approx(y1.x), ex2_approx(y1.y));
                            }
                        } else {
                            y0.x = r + 0 >= lim ? y0.x : -INFINITY;
                            y0.y = r + 1 >= lim ? y0.y : -INFINITY;
                            y1.x = r + 2 >= lim ? y1.x : -INFINITY;
                            y1.y = r + 3 >= lim ? y1.y : -INFINITY;
                            e0 = make_float2(ex2_approx(y0.x), ex2_approx(y0.y));
                            e1 = make_float2(ex2_approx(y1.x), ex2_approx(y1.y));
                        }
                        acc[(2 * e4) & 3] = fadd2(acc[(2 * e4) & 3], e0);
                        acc[(2 * e4 + 1) & 3] = fadd2(acc[(2 * e4 + 1) & 3], e1);
                        pk[2 * e4] = pack_bf16x2(e0.x, e0.y);
                        pk[2 * e4 + 1] = pack_bf16x2(e1.x, e1.y);
                    }
                    tmem_st16(s_t + cq * 16, pk);
                    if (cq < 3) tmem_wait_ld(u[(cq + 1) & 1]);
                }
                vacc = fadd2(vacc, fadd2(fadd2(acc[0], acc[1]), fadd2(acc[2], acc[3])));
            };
            if (plain) exp_pass(std::true_type{});
            else exp_pass(std::false_type{});
            tmem_wait_st();
            __syncwarp();
            if (lane == 0) mbar_arrive(&sm.l_empty[ls]);
            // the reduction of item k-1 (the other warpgroup's) must have read the P buffer.
            // One barrier per item parity: a single barrier would let this warpgroup, one item
            // ahead, match the parity of item k-3's completion and overwrite P too early.
            if constexpr (kPBufs == 2) {
                if (k >= 2) mbar_wait(&sm.p_free[k & 1], ((k - 2) >> 1) & 1);  // own buffer, item k-2
            } else {
                if (k >= 1) mbar_wait(&sm.p_free[(k - 1) & 1], ((k - 1) >> 1) & 1);
            }
            // row c of the coarse buffer: 16 aligned 16-byte chunks, chunk q -> coarse column
            // 128 - 8 floor(c/8) + 8q
#pragma unroll
            for (int h2 = 0; h2 < 2; ++h2) {
                uint32_t pk[32];
                tmem_ld32(s_t + h2 * 32, pk);
                tmem_wait_ld(pk);
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    const int a = a0 + h2 * 8 + q;  // absolute 8-column chunk, 1..31
                    *reinterpret_cast<uint4*>(prow + (a >> 3) * kHalf + (((a & 7) ^ (c & 7)) << 4)) =
                        make_uint4(pk[4 * q], pk[4 * q + 1], pk[4 * q + 2], pk[4 * q + 3]);
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&sm.s_free[sb]);
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) mbar_arrive(&sm.p_full[k & 1]);
        }

        // ---- flush (once per CTA)
        float* vx = reinterpret_cast<float*>(base + kOffVx);
        if (w == 1) vx[c] = vacc.x + vacc.y;
        mbar_wait(&sm.all_done, 0);
        tc_fence_after();
        named_bar_sync(1, 256);
        if (w == 0) {
            const int j = j0 + c;
            if (j < p.n && num_items > 0)
                atomicAdd(p.acc_v + static_cast<size_t>(g) * p.n + j, to_fixed((vacc.x + vacc.y + vx[c]) * p.out_scale, p.fix_scale));
        }
        // slash block b = sum_f E[128 b + x + f][f]; E block b lives in slot b - t0 + 1 (slot 0
        // only when t0 >= 1). WG w flushes blocks with (b - b_lo) % 2 == w.
        float* stage = reinterpret_cast<float*>(base + kOffStage) + w * kStageFloats;
        const int nslots = nblk + 1;
        const int b_lo = max(0, t0 - 2);
        const int b_hi = t0 + nblk - 1;
        for (int b = b_lo + w; b <= b_hi; b += 2) {
            const int s0 = b - t0 + 1;
            const bool v0 = s0 >= 0 && s0 < nslots && !(s0 == 0 && t0 == 0);
            const bool v1 = s0 + 1 >= 0 && s0 + 1 < nslots && !(s0 + 1 == 0 && t0 == 0);
            uint32_t e[16];
            if (v0) {
                tmem_ld16(t_acc + s0 * kAccCols + lane_base, e);
                tmem_wait_ld(e);
            }
#pragma unroll
            for (int f = 0; f < 8; ++f) stage[c * 8 + f] = v0 ? __uint_as_float(e[f]) : 0.f;
            if (quarter == 0) {  // rows 128..135 of the window: first rows of block b+1
                if (v1) {
                    tmem_ld16(t_acc + (s0 + 1) * kAccCols + lane_base, e);
                    tmem_wait_ld(e);
                }
                if (lane < 8) {
#pragma unroll
                    for (int f = 0; f < 8; ++f) stage[(128 + lane) * 8 + f] = v1 ? __uint_as_float(e[f]) : 0.f;
                }
            }
            named_bar_sync(2 + w, 128);
            float sum = 0.f;
#pragma unroll
            for (int f = 0; f < 8; ++f) sum += stage[(c + f) * 8 + f];
            const int o = b * kBlock + c;
            if (o < p.n && sum != 0.f) atomicAdd(p.acc_s + static_cast<size_t>(g) * p.n + o, to_fixed(sum * p.out_scale, p.fix_scale));
            named_bar_sync(2 + w, 128);
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) tmem_free<512>(tmem);
}

// Fixed-point accumulators -> fp32 profiles rescaled to their exact expected total (1 per
// normalised head, averaged or summed over the group): the bf16 tensor-core reductions leave
// ~1e-4 of drift, and select_pattern requires |sum - 1| <= 1e-6 (sparsity.hpp:61). The sum
// is an exact integer, so the result does not depend on the order of the atomics. grid (hkv, 2).
__global__ void finalize_kernel(const unsigned long long* acc_v, const unsigned long long* acc_s, float* a_v,
                                float* a_s, int n, double total) {
    const unsigned long long* x = (blockIdx.y == 0 ? acc_v : acc_s) + static_cast<size_t>(blockIdx.x) * n;
    float* y = (blockIdx.y == 0 ? a_v : a_s) + static_cast<size_t>(blockIdx.x) * n;
    unsigned long long s = 0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) s += x[i];
    __shared__ unsigned long long red[32];
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long t = 0;
        for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) t += red[w];
        red[0] = t;
    }
    __syncthreads();
    const double f = red[0] > 0 ? total / static_cast<double>(red[0]) : 0.0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) y[i] = static_cast<float>(static_cast<double>(x[i]) * f);
}

size_t workspace_bytes(int n, int hq) {
    // fixed-point accumulators (2 x [hq >= hkv, n] u64), then the pass-1 scratch when the
    // caller has no LSE: O [n, hq, 128] bf16 + LSE [hq, n]
    return 2 * static_cast<size_t>(hq) * n * 8 + static_cast<size_t>(n) * hq * 128 * 2 +
           static_cast<size_t>(hq) * n * 4 + 1024;
}

cudaError_t launch(const Args& a, void* workspace, cudaStream_t stream) {
    const float* lse = a.lse;
    auto* acc = static_cast<unsigned long long*>(workspace);
    uint8_t* scratch = static_cast<uint8_t*>(workspace) + 2 * static_cast<size_t>(a.hq) * a.n * 8;
    if (lse == nullptr) {
        auto* o = reinterpret_cast<__nv_bfloat16*>(scratch);
        float* l = reinterpret_cast<float*>(scratch + static_cast<size_t>(a.n) * a.hq * 128 * 2);
        vsp_attn::AttnArgs d{a.q, a.k, a.k, o, l, a.n, a.hq, a.hkv, a.scale};
        cudaError_t e = vsp_attn::launch_dense(d, stream);
        if (e != cudaSuccess) return e;
        lse = l;
    }
    Params p{};
    const uint32_t box[3] = {64, 1, kBlock};
    const uint64_t dq[3] = {128, (uint64_t)a.hq, (uint64_t)a.n};
    const uint64_t sq[2] = {128 * 2, (uint64_t)a.hq * 128 * 2};
    const uint64_t dk[3] = {128, (uint64_t)a.hkv, (uint64_t)a.n};
    const uint64_t sk[2] = {128 * 2, (uint64_t)a.hkv * 128 * 2};
    if (!vsp_host::make_map_bf16(&p.map_q, a.q, 3, dq, sq, box) ||
        !vsp_host::make_map_bf16(&p.map_k, a.k, 3, dk, sk, box))
        return cudaErrorInvalidValue;
    p.lse = lse;
    p.acc_v = acc;
    p.acc_s = acc + static_cast<size_t>(a.hkv) * a.n;
    p.n = a.n;
    p.hq = a.hq;
    p.hkv = a.hkv;
    p.num_qb = (a.n + kBlock - 1) / kBlock;
    p.num_qc = (p.num_qb + kChunk - 1) / kChunk;
    p.scale = a.scale;
    p.out_scale = (a.normalized ? 1.0f / static_cast<float>(a.n) : 1.0f) *
                  (a.mean ? 1.0f / static_cast<float>(a.hq / a.hkv) : 1.0f);
    {
        const double tot = (a.normalized ? 1.0 : static_cast<double>(a.n)) *
                           (a.mean ? 1.0 : static_cast<double>(a.hq / a.hkv));
        p.fix_scale = std::ldexp(1.0, 52 - static_cast<int>(std::ceil(std::log2(std::max(tot, 1.0)))));
    }
    cudaError_t e = cudaMemsetAsync(acc, 0, 2 * sizeof(unsigned long long) * a.hkv * a.n, stream);
    if (e != cudaSuccess) return e;
    static std::once_flag attr[vsp_detail::kMaxDevices];
    vsp_detail::once_per_device(attr, [] {
        cudaFuncSetAttribute(aggregate_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes);
    });
    long long ctas = 0;
    for (int qc = 0; qc < p.num_qc; ++qc) ctas += static_cast<long long>(std::min(p.num_qb, kChunk * (qc + 1))) * a.hkv;
    vsp_detail::count_launch();
    aggregate_kernel<<<static_cast<unsigned>(ctas), kThreads, kSmemBytes, stream>>>(p);
    const int grp = a.hq / a.hkv;
    const double total = (a.normalized ? 1.0 : static_cast<double>(a.n)) * (a.mean ? 1.0 : static_cast<double>(grp));
    vsp_detail::count_launch();
    finalize_kernel<<<dim3(a.hkv, 2), 1024, 0, stream>>>(p.acc_v, p.acc_s, a.a_v, a.a_s, a.n, total);
    return cudaGetLastError();
}

}  // namespace vsp_aggregate
