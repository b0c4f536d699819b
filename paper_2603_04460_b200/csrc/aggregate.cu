// aggregate.cu — K5: ground-truth vertical/slash aggregation on sm_100a.
//
// Replaces vsp::aggregate_streaming (reference vsaggregate.hpp:62-127) for every Q head,
// fused with combine_scores (vsaggregate.hpp:133-157) over each KV group:
//   pass 1: LSE_i of every row (online softmax; vsaggregate.hpp:83-103) — K4's LSE output
//   pass 2: w = exp(s_ij - LSE_i); vertical[j] += w; slash[i - j] += w (:109-124)
//   normalize by n (:27-33), then group Mean (or Sum).
// The n x n weights never exist: each 128 x 128 tile of P lives in shared memory for the
// two reductions, and both reductions run on the TENSOR cores:
//   column sums   D_col[j] += sum_i P[i][j]      = (P^T . 1)   (A = P^T, MN-major smem view)
//   diagonal sums D_dia[c] += sum_i P'[i][c]     = (P'^T . 1)  with the skewed copy
//                 P'[r][c] = P[r][r - c + 128], so column c of P' is diagonal o = 128t + c - 128
//                 (t = query block - key block); the two 128-wide halves of P' feed the
//                 accumulators of offset blocks t-1 and t, which complete in order.
// CTA = one 128-key block (K tile resident), one KV group, a chunk of query blocks; it walks
// (query block, Q head) items in order. Per item: S = Q K^T (tcgen05, TMEM), softmax warps
// turn S into P (bf16) in two smem layouts, the MMA warp issues the three reduction MMAs
// (M=128, N=16, K=128) into TMEM accumulators. Completed offset blocks and, at the end, the
// column sums are added to the [hkv, n] fp32 outputs (global atomics across CTAs).
#include <cuda_bf16.h>

#include "aggregate.h"
#include "attn.h"
#include "sm100.cuh"
#include "tma_host.h"

using namespace vsp_sm100;

namespace vsp_aggregate {

constexpr int kBlock = 128;
constexpr int kTile = kBlock * 128 * 2;  // 32 KB bf16 tile
constexpr int kHalf = kTile / 2;
constexpr int kChunk = 16;               // query blocks per CTA
constexpr int kThreads = 256;            // warp0 TMA, warp1 MMA, warps 4-7 softmax
constexpr float kLog2e = 1.4426950408889634f;

struct __align__(64) Params {
    CUtensorMap map_q, map_k;
    const float* lse;  // [hq, n]
    float* a_v;        // [hkv, n]
    float* a_s;
    int n, hq, hkv, num_qb, chunks_per_kb;
    float scale;       // 1/sqrt(d)
    float out_scale;   // (normalized ? 1/n : 1) * (mean ? 1/group : 1)
};

struct Smem {
    uint64_t bar_k;
    uint64_t q_full[2], q_empty[2];
    uint64_t s_full[2], s_free[2];
    uint64_t p_full, p_free;
    uint64_t d_done, flush_done;
    uint32_t tmem_base;
};

// smem: K 32K | Q ring 2 x 32K | P row-major 32K | P skew 64K | ones 4K
constexpr int kOffK = 0;
constexpr int kOffQ = kTile;
constexpr int kOffP = 3 * kTile;
constexpr int kOffPS = 4 * kTile;
constexpr int kOffOnes = 6 * kTile;
constexpr int kSmemBytes = 6 * kTile + 4096 + 1024;

// byte offset of element (row r, col c) in a [128 x 64]-bf16 SW128 K-major/MN-major block
VSP_DEVICE uint32_t sw128_off(int r, int c) {
    const int chunk = (c * 2) >> 4;
    return static_cast<uint32_t>(r * 128 + (((chunk ^ (r & 7)) << 4) | ((c * 2) & 15)));
}

__global__ void __launch_bounds__(kThreads, 1) aggregate_kernel(const __grid_constant__ Params p) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    // offset from smem_raw (not a cast through an integer) so the compiler keeps the
    // shared state space and emits LDS/STS rather than generic LD/ST
    uint8_t* base = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    __shared__ Smem sm;
    const int grp = p.hq / p.hkv;

    // block -> (key block jb, group g, chunk): heavy key blocks (small jb) first
    const int per_g = p.num_qb * p.chunks_per_kb;
    const int g = blockIdx.x % p.hkv;
    const int rest = blockIdx.x / p.hkv;
    const int jb = rest / p.chunks_per_kb;
    const int chunk = rest % p.chunks_per_kb;
    (void)per_g;
    const int t_first = chunk * kChunk;                   // t = ib - jb
    const int t_end = min(t_first + kChunk, p.num_qb - jb);
    const uint32_t warp = warp_id(), lane = lane_id();
    if (t_first >= t_end) return;
    const int num_items = (t_end - t_first) * grp;
    const int j0 = jb * kBlock;

    if (warp == 0 && lane == 0) {
        mbar_init(&sm.bar_k, 1);
        for (int s = 0; s < 2; ++s) {
            mbar_init(&sm.q_full[s], 1);
            mbar_init(&sm.q_empty[s], 1);
            mbar_init(&sm.s_full[s], 1);
            mbar_init(&sm.s_free[s], 4);
        }
        mbar_init(&sm.p_full, 4);
        mbar_init(&sm.p_free, 1);
        mbar_init(&sm.d_done, 1);
        mbar_init(&sm.flush_done, 4);
        fence_barrier_init();
    }
    if (warp == 1) tmem_alloc<512>(&sm.tmem_base);
    // ones operand for the reduction MMAs
    {
        uint32_t* ones = reinterpret_cast<uint32_t*>(base + kOffOnes);
        for (int i = threadIdx.x; i < 1024; i += blockDim.x) ones[i] = 0x3f803f80u;  // bf16 1.0 x2
        fence_proxy_async_smem();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = sm.tmem_base;
    const uint32_t t_col = tmem + 256;             // column sums   [128 x 16]
    const uint32_t t_dia[2] = {tmem + 288, tmem + 320};

    if (warp == 0) {
        if (elect_one()) {
            tma_prefetch_desc(&p.map_q);
            tma_prefetch_desc(&p.map_k);
            mbar_arrive_expect_tx(&sm.bar_k, kTile);
            for (int hf = 0; hf < 2; ++hf)
                tma_load_3d(base + kOffK + hf * kHalf, &p.map_k, &sm.bar_k, hf * 64, g, j0);
        }
        __syncwarp();
        for (int it = 0; it < num_items; ++it) {
            const int t = t_first + it / grp;
            const int h = g * grp + it % grp;
            const int s = it & 1;
            if (it >= 2) mbar_wait(&sm.q_empty[s], ((it >> 1) & 1) ^ 1);
            if (elect_one()) {
                mbar_arrive_expect_tx(&sm.q_full[s], kTile);
                for (int hf = 0; hf < 2; ++hf)
                    tma_load_3d(base + kOffQ + s * kTile + hf * kHalf, &p.map_q, &sm.q_full[s], hf * 64, h,
                                (jb + t) * kBlock);
            }
            __syncwarp();
        }
    } else if (warp == 1) {
        // MMA issuer: warp-uniform loop, one elected lane issues each batch
        const uint32_t idesc_qk = umma_idesc_bf16(128, 128, false, false);
        const uint32_t idesc_red = umma_idesc_bf16(128, 16, true, false);
        const uint64_t k_desc0 = umma_desc_sw128(smem_u32(base + kOffK), 16, 1024);
        const uint64_t q_desc0 = umma_desc_sw128(smem_u32(base + kOffQ), 16, 1024);
        const uint64_t ones_desc0 = umma_desc_sw128(smem_u32(base + kOffOnes), 16, 1024);
        const uint32_t p_addr = smem_u32(base + kOffP);
        const uint32_t ps_addr = smem_u32(base + kOffPS);
        auto issue_s = [&](int it) {
            const int s = it & 1;
            mbar_wait(&sm.q_full[s], (it >> 1) & 1);
            if (it >= 2) mbar_wait(&sm.s_free[s], ((it >> 1) & 1) ^ 1);
            tc_fence_after();
            if (elect_one()) {
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    const uint64_t off = static_cast<uint64_t>(((k >> 2) * kHalf + (k & 3) * 32) >> 4);
                    umma_ss(tmem + s * 128, q_desc0 + static_cast<uint64_t>((s * kTile) >> 4) + off, k_desc0 + off,
                            idesc_qk, k > 0 ? 1u : 0u);
                }
                umma_commit(&sm.s_full[s]);
                umma_commit(&sm.q_empty[s]);
            }
            __syncwarp();
        };
        // reduction: D[tm] (+)= A^T . 1, A = [128 rows x 128 cols] bf16 (two 16 KB halves)
        auto issue_red = [&](uint32_t d_t, uint32_t a_base, bool acc) {
            const uint64_t a0 = umma_desc_sw128(a_base, kHalf, 1024);
#pragma unroll
            for (int k = 0; k < 8; ++k)
                umma_ss(d_t, a0 + static_cast<uint64_t>((k * 2048) >> 4),
                        ones_desc0 + static_cast<uint64_t>(((k >> 2) * 2048 + (k & 3) * 32) >> 4), idesc_red,
                        (acc || k > 0) ? 1u : 0u);
        };
        mbar_wait(&sm.bar_k, 0);
        issue_s(0);
        if (num_items > 1) issue_s(1);
        for (int it = 0; it < num_items; ++it) {
            const int tl = it / grp;            // local t index
            const int t = t_first + tl;
            const int hi = it % grp;
            mbar_wait(&sm.p_full, it & 1);
            tc_fence_after();
            if (elect_one()) {
                issue_red(t_col, p_addr, it > 0);
                if (t >= 1) issue_red(t_dia[(t - 1) & 1], ps_addr, !(tl == 0 && hi == 0));
            }
            __syncwarp();
            if (hi == 0 && tl >= 1) {
                // the accumulator of block t last held block t-2, flushed after the
                // previous query block (flush arrival tl-1)
                mbar_wait(&sm.flush_done, (tl - 1) & 1);
                tc_fence_after();
            }
            if (elect_one()) {
                issue_red(t_dia[t & 1], ps_addr + 2 * kHalf, hi != 0);
                umma_commit(&sm.p_free);
                if (hi == grp - 1) umma_commit(&sm.d_done);
            }
            __syncwarp();
            if (it + 2 < num_items) issue_s(it + 2);
        }
    } else if (warp >= 4) {
        const int quarter = warp & 3;
        const int r = quarter * 32 + lane;
        const uint32_t lane_base = static_cast<uint32_t>(quarter * 32) << 16;
        const float sl2 = p.scale * kLog2e;
        uint8_t* sp = base + kOffP;
        uint8_t* sps = base + kOffPS;
        for (int it = 0; it < num_items; ++it) {
            const int tl = it / grp;
            const int t = t_first + tl;
            const int h = g * grp + it % grp;
            const int i = (jb + t) * kBlock + r;
            const int s = it & 1;
            const float lse2 = i < p.n ? __ldg(p.lse + static_cast<size_t>(h) * p.n + i) * kLog2e : INFINITY;
            mbar_wait(&sm.s_full[s], (it >> 1) & 1);
            tc_fence_after();
            float x[128];
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                uint32_t u[32];
                tmem_ld32(tmem + lane_base + s * 128 + c * 32, u);
                tmem_wait_ld();
#pragma unroll
                for (int e = 0; e < 32; ++e) x[c * 32 + e] = __uint_as_float(u[e]);
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&sm.s_free[s]);
#pragma unroll
            for (int c = 0; c < 128; ++c) {
                const bool ok = (t > 0 || c <= r) && i < p.n;  // causal on the diagonal tile
                x[c] = ok ? ex2_approx(fmaf(x[c], sl2, -lse2)) : 0.f;
            }
            if (it > 0) mbar_wait(&sm.p_free, (it - 1) & 1);
            // row-major P (two 64-column SW128 halves)
#pragma unroll
            for (int hf = 0; hf < 2; ++hf)
#pragma unroll
                for (int ch = 0; ch < 8; ++ch) {
                    const int c0 = hf * 64 + ch * 8;
                    uint4 v;
                    v.x = pack_bf16x2(x[c0 + 0], x[c0 + 1]);
                    v.y = pack_bf16x2(x[c0 + 2], x[c0 + 3]);
                    v.z = pack_bf16x2(x[c0 + 4], x[c0 + 5]);
                    v.w = pack_bf16x2(x[c0 + 6], x[c0 + 7]);
                    *reinterpret_cast<uint4*>(sp + hf * kHalf + r * 128 + (((ch ^ (r & 7)) << 4))) = v;
                }
            // skewed P': zero the row, then P'[r][r - c + 128] = P[r][c]
#pragma unroll
            for (int q4 = 0; q4 < 4; ++q4)
#pragma unroll
                for (int ch = 0; ch < 8; ++ch)
                    *reinterpret_cast<uint4*>(sps + q4 * kHalf + r * 128 + (ch << 4)) = make_uint4(0, 0, 0, 0);
            __syncwarp();
#pragma unroll
            for (int c = 0; c < 128; ++c) {
                const int cc = r - c + 128;  // 1..255
                __nv_bfloat16 b = __float2bfloat16_rn(x[c]);
                *reinterpret_cast<__nv_bfloat16*>(sps + (cc >> 6) * kHalf + sw128_off(r, cc & 63)) = b;
            }
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) mbar_arrive(&sm.p_full);

            if (it % grp == grp - 1) {
                // all heads of this query block are in: offset block t-1 is complete
                mbar_wait(&sm.d_done, tl & 1);
                tc_fence_after();
                if (t >= 1) {
                    uint32_t u[32];
                    // only column 0 is needed (all 16 columns hold the same sums)
                    tmem_ld32(t_dia[(t - 1) & 1] + lane_base, u);
                    tmem_wait_ld();
                    const int o = (t - 1) * kBlock + r;
                    if (o < p.n) atomicAdd(p.a_s + static_cast<size_t>(g) * p.n + o, __uint_as_float(u[0]) * p.out_scale);
                }
                if (t == t_end - 1) {
                    uint32_t u[32];
                    tmem_ld32(t_dia[t & 1] + lane_base, u);
                    tmem_wait_ld();
                    const int o = t * kBlock + r;
                    if (o < p.n) atomicAdd(p.a_s + static_cast<size_t>(g) * p.n + o, __uint_as_float(u[0]) * p.out_scale);
                    tmem_ld32(t_col + lane_base, u);
                    tmem_wait_ld();
                    const int j = j0 + r;
                    if (j < p.n) atomicAdd(p.a_v + static_cast<size_t>(g) * p.n + j, __uint_as_float(u[0]) * p.out_scale);
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&sm.flush_done);
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) tmem_free<512>(tmem);
}

// Rescale each [n] profile to its exact expected total (1 per normalised head, averaged or
// summed over the group): the bf16 tensor-core reductions leave ~1e-4 of drift, and
// select_pattern requires |sum - 1| <= 1e-6 (sparsity.hpp:61). grid (hkv, 2).
__global__ void renormalize_kernel(float* a_v, float* a_s, int n, double total) {
    float* x = (blockIdx.y == 0 ? a_v : a_s) + static_cast<size_t>(blockIdx.x) * n;
    double s = 0.0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) s += x[i];
    __shared__ double red[32];
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) t += red[w];
        red[0] = t;
    }
    __syncthreads();
    const double f = red[0] > 0.0 ? total / red[0] : 0.0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) x[i] = static_cast<float>(x[i] * f);
}

size_t workspace_bytes(int n, int hq) {
    // pass-1 scratch when the caller has no LSE: O [n, hq, 128] bf16 + LSE [hq, n]
    return static_cast<size_t>(n) * hq * 128 * 2 + static_cast<size_t>(hq) * n * 4 + 1024;
}

cudaError_t launch(const Args& a, void* workspace, cudaStream_t stream) {
    const float* lse = a.lse;
    if (lse == nullptr) {
        auto* o = static_cast<__nv_bfloat16*>(workspace);
        float* l = reinterpret_cast<float*>(static_cast<uint8_t*>(workspace) + static_cast<size_t>(a.n) * a.hq * 128 * 2);
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
    p.a_v = a.a_v;
    p.a_s = a.a_s;
    p.n = a.n;
    p.hq = a.hq;
    p.hkv = a.hkv;
    p.num_qb = (a.n + kBlock - 1) / kBlock;
    p.chunks_per_kb = (p.num_qb + kChunk - 1) / kChunk;
    p.scale = a.scale;
    p.out_scale = (a.normalized ? 1.0f / static_cast<float>(a.n) : 1.0f) *
                  (a.mean ? 1.0f / static_cast<float>(a.hq / a.hkv) : 1.0f);
    cudaError_t e = cudaMemsetAsync(a.a_v, 0, sizeof(float) * a.hkv * a.n, stream);
    if (e == cudaSuccess) e = cudaMemsetAsync(a.a_s, 0, sizeof(float) * a.hkv * a.n, stream);
    if (e != cudaSuccess) return e;
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(aggregate_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes);
        attr = true;
    }
    dim3 grid(p.num_qb * p.chunks_per_kb * a.hkv);
    aggregate_kernel<<<grid, kThreads, kSmemBytes, stream>>>(p);
    const int grp = a.hq / a.hkv;
    const double total = (a.normalized ? 1.0 : static_cast<double>(a.n)) * (a.mean ? 1.0 : static_cast<double>(grp));
    renormalize_kernel<<<dim3(a.hkv, 2), 1024, 0, stream>>>(a.a_v, a.a_s, a.n, total);
    return cudaGetLastError();
}

}  // namespace vsp_aggregate
