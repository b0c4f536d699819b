// attn_fwd.cu — K4 dense causal attention and K3 vertical-slash sparse attention on
// sm_100a (tcgen05 + TMEM + TMA), one shared pipeline.
//
// Replaces, per Q head:
//   vsp::blockwise_attention  (reference attention.hpp:96-145)   -> dense mode
//   vsp::sparse_attention     (reference attention.hpp:150-194) + merge_row_columns
//                             (merge.hpp:18-56)                  -> sparse mode
//
// Work item = one 128-row query block x TWO Q heads of the same KV group (GQA: both Q
// tiles share every K/V tile). Persistent grid (one CTA per SM) pulling items heaviest
// first from a global counter. 12 warps:
//   warp 0      TMA producer (item fetch, Q per item, then K/V tiles through a ring)
//   warp 1      MMA issuer: S_h = Q_h K^T (SS), O_h += P_h V (TS, P read from TMEM)
//   warps 4-7   softmax/epilogue for Q tile 0 (thread = query row = TMEM lane)
//   warps 8-11  softmax/epilogue for Q tile 1
// TMEM (512 cols): S0 [0,128) S1 [128,256) O0 [256,384) O1 [384,512); P_h (bf16) aliases
// the first 64 columns of S_h. The MMA order PV_h(j-1) -> S_h(j) keeps the alias safe
// because tcgen05.mma executes in issue order; the S_full commit after S_h(j) therefore
// also proves PV_h(j-1) finished, which is when the softmax warps may rescale O_h. P is
// published in two halves (p_half: keys 0-63, p_full: keys 64-127), so the first half of
// PV_h(j-1) runs while the softmax still computes the second half's exponentials.
// Cross-item barriers: q_full/q_free (the Q tiles of the current item), o_free (the
// epilogue has read O_h, so the next item's first PV may overwrite it), and a two-slot smem
// ring that carries each fetched item index from the producer to the other warps.
// Online softmax runs in the exp2 domain with lazy rescaling (only when the running max
// grows by more than 2^8), exactly the same math as the reference's per-row rescale.
//
// Sparse mode: per (KV head, query block) a tile list built by vs_prep_kernel. An entry is
// (value, gathered flag, width): a "slash span" tile covers K/V rows [value, value+width) of
// the original tensors with element mask (i-j) in I_s AND j not in I_v AND j <= i (from n-bit
// bitmaps); a gathered vertical tile t = value covers rows [128t, 128t+width) of K[I_v], V[I_v]
// (gathered once per head), mask r < #{I_v <= i}. Every covered (i, j) pair is visited exactly
// once, which is the reference's duplicate-free per-row union. The last tile of a vertical run
// or of a merged slash range is narrow (width = its used columns rounded up to 16): the S MMA
// runs with N = width and PV with width/16 K-steps, so a 9-column remainder costs ~0.3 of a
// full tile on the tensor core instead of 1.
#include <cuda_bf16.h>

#include <algorithm>
#include <cstdlib>
#include <atomic>
#include <type_traits>
#include <vector>

#include "vsp_launch.h"
#include "attn.h"
#include "sm100.cuh"

using namespace vsp_sm100;

namespace vsp_attn {

constexpr int kBlock = 128;     // query rows per tile and key rows per tile
constexpr int kHeadDim = 128;
constexpr int kNumK = 2;        // K smem stages
constexpr int kNumV = 2;        // V smem stages
constexpr int kTileBytes = kBlock * kHeadDim * 2;   // 32 KB (two 16 KB d-halves)
constexpr int kHalfBytes = kTileBytes / 2;
constexpr int kOStage = kHalfBytes;  // per Q tile: O staging for the TMA store, one 64-column half
constexpr int kSmemBytes = (2 + kNumK + kNumV) * kTileBytes + 2 * kOStage + 1024;
constexpr int kThreads = 384;
// per-thread registers after setmaxnreg: launch cap 168 (65536 / 384); the producer/MMA
// warpgroup gives back (168 - 64) x 128, the softmax warps take (216 - 168) x 256 of it
constexpr uint32_t kRegsOther = 64;
constexpr uint32_t kRegsSoftmax = 216;
constexpr float kRescaleThreshold = 8.0f;  // log2 units
constexpr float kLog2e = 1.4426950408889634f;
constexpr float kLn2 = 0.6931471805599453f;

#ifndef VSP_POLY_MASK
#define VSP_POLY_MASK 0x5454u  // exp2 pairs (of 16 per 32-column chunk) evaluated by the FMA-pipe polynomial
#endif

constexpr int kItemRing = 2;
constexpr int kItemConsumers = 9;  // MMA warp + 8 softmax warps

struct Smem {
    uint64_t q_full, q_free;                  // Q tiles of the current work item
    uint64_t k_full[kNumK], k_empty[kNumK];
    uint64_t v_full[kNumV], v_empty[kNumV];
    uint64_t s_full[2], p_half[2], p_full[2], o_done[2];  // p_half: P columns [0, 64) written
    uint64_t o_free[2];                       // epilogue has read O_w (next item may PV into it)
    uint64_t item_full[kItemRing], item_empty[kItemRing];
    int item[kItemRing];                      // work item index, -1 = no more work
    int item_nt[kItemRing], item_vc[kItemRing];  // sparse: the item's tile-list header (the
                                                 // producer reads it one item ahead)
    uint32_t tmem_base;
};

// Tile-list entry: bits [0, 27) value, bit 27 gathered, bits [28, 31) width / 16 - 1.
constexpr int kEntValueBits = 27;
constexpr int kEntGathered = 1 << kEntValueBits;
__host__ __device__ constexpr int ent_make(int value, bool gathered, int width) {
    return value | (gathered ? kEntGathered : 0) | (((width >> 4) - 1) << 28);
}
VSP_DEVICE int ent_value(int e) { return e & (kEntGathered - 1); }
VSP_DEVICE bool ent_gathered(int e) { return (e & kEntGathered) != 0; }
VSP_DEVICE int ent_width(int e) { return ((e >> 28) + 1) << 4; }
VSP_DEVICE int round16(int x) { return (x + 15) & ~15; }

// Work item it (heaviest query blocks first: causal work grows with the block index).
struct Item {
    int qb, h0, h1, g, num_tiles, vcnt0;  // Q heads h0, h1 (h1 == h0: odd group, one head)
    const int* tiles;
};

// Bits [start, start+128) of a bitmap as four words, word k bit b <-> bit start+32k+b.
// Bits below 0 and at/above nbits are zero (bitmaps are padded by one zero word).
VSP_DEVICE void window128(const uint32_t* __restrict__ bm, int start, int nwords, uint32_t (&w)[4]) {
    const int ws = start >> 5;  // floor division (arithmetic shift)
    const uint32_t sh = static_cast<uint32_t>(start) & 31u;
    uint32_t raw[5];
#pragma unroll
    for (int k = 0; k < 5; ++k) {
        const int idx = ws + k;
        raw[k] = (idx >= 0 && idx < nwords) ? __ldg(bm + idx) : 0u;
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) w[k] = __funnelshift_r(raw[k], raw[k + 1], sh);
}

#ifndef VSP_NOINLINE_SLASH_MASK
#define VSP_NOINLINE_SLASH_MASK 1  // A/B on the bench, 20 steps: 4.41 -> 4.34 ms/step
#endif
// Element mask of a slash-span tile starting at original column e for query row i (see the
// softmax loop); out of line under VSP_NOINLINE_SLASH_MASK so the hot loop stays compact.
__device__ __noinline__ uint4 slash_tile_mask(const uint32_t* __restrict__ vb, const uint32_t* __restrict__ sb,
                                              int bm_words, int e, int i, int width, int vcnt0) {
    auto prefix_word = [](int b) { return b <= 0 ? 0u : (b >= 32 ? 0xffffffffu : (0xffffffffu >> (32 - b))); };
    uint32_t vw[4], sw[4], mk[4];
    window128(vb, e, bm_words, vw);
    window128(sb, i - e - 127, bm_words, sw);
    if (vcnt0 >= 0) {
#pragma unroll
        for (int k = 0; k < 4; ++k) mk[k] = __brev(sw[3 - k]) & ~vw[k];
    } else {
        const int lim = i - e + 1;
#pragma unroll
        for (int k = 0; k < 4; ++k) mk[k] = __brev(sw[3 - k]) | (vw[k] & prefix_word(lim - 32 * k));
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) mk[k] &= prefix_word(width - 32 * k);
    return make_uint4(mk[0], mk[1], mk[2], mk[3]);
}

#ifdef VSP_K3_TRACE
// Timeline probe (tools/k3_trace.py builds a separate library with -DVSP_K3_TRACE): clock64
// stamps of CTA 0's pipeline events per (event, head w, global tile G).
constexpr int kTraceTiles = 8192;
__device__ unsigned long long g_k3_trace[12 * 2 * kTraceTiles];
#define VSP_TRACE(ev, w, G)                                                                              \
    do {                                                                                                 \
        if (blockIdx.x == 0 && (G) < kTraceTiles && lane_id() == 0)                                      \
            g_k3_trace[((ev) * 2 + (w)) * kTraceTiles + (G)] = clock64();                                \
    } while (0)
#else
#define VSP_TRACE(ev, w, G) \
    do {                    \
    } while (0)
#endif

// One tile of the online softmax for one warp (thread = query row): read S from TMEM, mask,
// row max, lazy rescale of O, exponentials -> bf16 P written back over S, p_half after the
// first 64 columns. kM = the warp has masked columns (per-chunk modes dead/part, see caller).
template <bool kM>
VSP_DEVICE void softmax_tile(uint32_t s_t, uint32_t o_t, uint32_t dead, uint32_t part, uint4 mk4,
                             int width, int j, float sl2, float& m_used, float& l, uint64_t* p_half_bar,
                             int quarter, int w, int gtj) {
    const uint32_t lane = lane_id();
    const uint32_t mk[4] = {mk4.x, mk4.y, mk4.z, mk4.w};
    (void)quarter;
    (void)w;
    (void)gtj;
    // the S row is read from TMEM once and stays in registers (the softmax warps run with
    // more registers, see setmaxnreg above)
    uint32_t u[4][32];
#pragma unroll
    for (int c = 0; c < 4; ++c) tmem_ld32(s_t + c * 32, u[c]);
    tmem_wait_ld();
#pragma unroll
    for (int c = 0; c < 4; ++c) tmem_reg_fence(u[c]);
    float mx;
    {
        // eight independent max chains (a single chain is 64 dependent 3-input maxes)
        float mxa[8];
#pragma unroll
        for (int t = 0; t < 8; ++t) mxa[t] = -INFINITY;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            if (kM && ((dead >> c) & 1u)) continue;
            if (kM && ((part >> c) & 1u)) {
#pragma unroll
                for (int t = 0; t < 32; ++t)
                    if (!((mk[c] >> t) & 1u)) u[c][t] = 0xff800000u;  // -inf
            }
#pragma unroll
            for (int t = 0; t < 32; t += 2)
                mxa[(t >> 1) & 7] = fmaxf(mxa[(t >> 1) & 7], fmaxf(__uint_as_float(u[c][t]), __uint_as_float(u[c][t + 1])));
        }
        mx = fmaxf(fmaxf(fmaxf(mxa[0], mxa[1]), fmaxf(mxa[2], mxa[3])),
                   fmaxf(fmaxf(mxa[4], mxa[5]), fmaxf(mxa[6], mxa[7])));
    }
    const float m_new = fmaxf(m_used, mx * sl2);
    const bool need = (m_used == -INFINITY) ? (m_new > -INFINITY) : (m_new > m_used + kRescaleThreshold);
    if (__any_sync(0xffffffffu, need)) {
        const float m_next = need ? m_new : m_used;
        const float f = (m_used == -INFINITY) ? 0.f : ex2_approx(m_used - m_next);
        l *= f;
        m_used = m_next;
        if (j > 0) {  // O holds PV(0..j-1); PV(j-1) is complete (see header)
#pragma unroll 1
            for (int c = 0; c < 4; ++c) {
                uint32_t v[32];
                tmem_ld32(o_t + c * 32, v);
                tmem_wait_ld(v);
#pragma unroll
                for (int t = 0; t < 32; ++t) v[t] = __float_as_uint(__uint_as_float(v[t]) * f);
                tmem_st32(o_t + c * 32, v);
            }
        }
    }
    if (quarter == 0) VSP_TRACE(3, w, gtj);
    const float m_eff = (m_used == -INFINITY) ? 0.f : m_used;
    const float2 scl = make_float2(sl2, sl2);
    const float2 neg_m = make_float2(-m_eff, -m_eff);
    float2 lsum[4] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f),
                      make_float2(0.f, 0.f)};
    // p = 2^(s * scale * log2e - m), packed to bf16 pairs and written over the consumed
    // S columns (chunk c's P lands in [16c, 16c+16))
#pragma unroll
    for (int c = 0; c < 4; ++c) {
        if (!kM || c * 32 < width) {  // chunks past a narrow tile are never read by PV
            uint32_t pk[16];
            if (kM && ((dead >> c) & 1u)) {
#pragma unroll
                for (int t = 0; t < 16; ++t) pk[t] = 0u;
            } else {
#pragma unroll
                for (int t = 0; t < 16; ++t) {
                    const float2 y = ffma2(make_float2(__uint_as_float(u[c][2 * t]),
                                                       __uint_as_float(u[c][2 * t + 1])),
                                           scl, neg_m);
                    float2 e;
                    if ((VSP_POLY_MASK >> t) & 1u) {  // 3 pairs in 8 on the FMA pipe (MUFU/FMA balance)
                        e = exp2_poly2(y);
                    } else {
                        e.x = ex2_approx(y.x);
                        e.y = ex2_approx(y.y);
                    }
                    lsum[t & 3] = fadd2(lsum[t & 3], e);
                    pk[t] = pack_bf16x2(e.x, e.y);
                }
            }
            tmem_st16(s_t + c * 16, pk);
        }
        if (c == 1) {  // P columns [0, 64) are in TMEM: the first PV half may start
            tmem_wait_st();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(p_half_bar);
            if (quarter == 0) VSP_TRACE(4, w, gtj);
        }
    }
    l += ((lsum[0].x + lsum[0].y) + (lsum[1].x + lsum[1].y)) + ((lsum[2].x + lsum[2].y) + (lsum[3].x + lsum[3].y));
}

// kMc = 2: a two-CTA cluster runs the two Q-head pairs of a 4-head group on the same query
// block in lockstep (identical tile lists); each CTA TMA-loads one half of every K/V tile and
// multicasts it to both, halving the L2 -> SMEM traffic. Ring slots are released by both
// CTAs' MMA commits (multicast tcgen05.commit), the item index travels from the leader's
// producer to the peer through distributed shared memory.
template <bool kSparse, int kMc>
__global__ void __launch_bounds__(kThreads, 1) attn_fwd_kernel(const __grid_constant__ AttnParams p) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    // offset from smem_raw (not a cast through an integer) so the compiler keeps the
    // shared state space and emits LDS/STS rather than generic LD/ST
    uint8_t* base = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    uint8_t* sQ = base;                                  // 2 tiles
    uint8_t* sK = base + 2 * kTileBytes;                 // kNumK tiles
    uint8_t* sV = sK + kNumK * kTileBytes;               // kNumV tiles
    uint8_t* sO = sV + kNumV * kTileBytes;               // 2 x kOStage: O staging per Q tile
    __shared__ Smem sm;

    const int num_qb = (p.n + kBlock - 1) / kBlock;
    // Persistent: one CTA per SM pulls work items (heavy first) from a global counter; the
    // producer publishes each item index through a two-slot smem ring, so the next item's Q
    // load and first S MMA overlap this item's last PV and epilogue, and the fetch order keeps
    // the dynamic load balance of a one-CTA-per-item grid.
    const uint32_t crank = kMc > 1 ? cluster_ctarank() : 0u;
    const int cpairs = p.npairs / kMc;  // pair groups per query block (one per cluster item)
    auto item = [&](int it, int hdr_nt, int hdr_vc) {
        Item x;
        // pair index -> (KV group, pair within the group); an odd group's last pair carries
        // one head (both Q tiles load it, only tile 0 writes)
        const int grp = p.hq / p.hkv, ppg = (grp + 1) >> 1;
        int pi;
        if (p.nunits > 0) {  // units mode: query-block runs of single KV heads, pairs = the group's
            const int itq = it / cpairs;
            int u = 0;
            while (u + 1 < p.nunits && __ldg(p.units + 4 * (u + 1) + 3) <= itq) ++u;
            const int g = __ldg(p.units + 4 * u);
            x.qb = __ldg(p.units + 4 * u + 2) - 1 - (itq - __ldg(p.units + 4 * u + 3));
            pi = g * ppg + kMc * (it % cpairs) + static_cast<int>(crank);
        } else {
            x.qb = p.qb_hi - 1 - it / cpairs;
            pi = p.pair0 + kMc * (it % cpairs) + static_cast<int>(crank);
        }
        x.g = pi / ppg;
        x.h0 = x.g * grp + 2 * (pi % ppg);
        x.h1 = min(x.h0 + 1, x.g * grp + grp - 1);
        x.vcnt0 = 0;
        x.tiles = nullptr;
        if constexpr (kSparse) {
            x.num_tiles = hdr_nt;
            x.vcnt0 = hdr_vc;
            x.tiles = p.tile_lists + (static_cast<size_t>(x.g) * num_qb + x.qb) * p.list_stride + 2;
        } else {
            x.num_tiles = x.qb + 1;
        }
        return x;
    };

    const uint32_t warp = warp_id();
    const uint32_t lane = lane_id();
    // consumer side of the item ring (MMA warp and softmax warps): item of round n_it, or -1
    auto next_item = [&](int n_it, int& nt, int& vc) {
        const int slot = n_it % kItemRing;
#ifdef VSP_K3_TRACE
        if (warp == 1) VSP_TRACE(11, 0, n_it);
#endif
        mbar_wait(&sm.item_full[slot], (n_it / kItemRing) & 1);
#ifdef VSP_K3_TRACE
        if (warp == 1) VSP_TRACE(11, 1, n_it);
#endif
        const int it = *reinterpret_cast<volatile int*>(&sm.item[slot]);
        nt = *reinterpret_cast<volatile int*>(&sm.item_nt[slot]);
        vc = *reinterpret_cast<volatile int*>(&sm.item_vc[slot]);
        __syncwarp();
        if (lane == 0) {
            if (crank == 0) mbar_arrive(&sm.item_empty[slot]);
            else mbar_arrive_cluster(mapa_shared(smem_u32(&sm.item_empty[slot]), 0));  // the leader's ring
        }
        return it;
    };

    if (warp == 0 && lane == 0) {
        mbar_init(&sm.q_full, 1);
        mbar_init(&sm.q_free, 1);
        for (int s = 0; s < kNumK; ++s) {
            mbar_init(&sm.k_full[s], 1);
            mbar_init(&sm.k_empty[s], kMc);  // every CTA's MMA releases the (multicast) slot
        }
        for (int s = 0; s < kNumV; ++s) {
            mbar_init(&sm.v_full[s], 1);
            mbar_init(&sm.v_empty[s], kMc);
        }
        for (int s = 0; s < kItemRing; ++s) {
            mbar_init(&sm.item_full[s], 1);
            // the leader's slots are also consumed by the peer's warps and producer
            mbar_init(&sm.item_empty[s], kItemConsumers + (kMc - 1) * (kItemConsumers + 1));
        }
        for (int w = 0; w < 2; ++w) {
            mbar_init(&sm.s_full[w], 1);
            mbar_init(&sm.p_half[w], 4);
            mbar_init(&sm.p_full[w], 4);
            mbar_init(&sm.o_done[w], 1);
            mbar_init(&sm.o_free[w], 4);
        }
        fence_barrier_init();
    }
    if (warp == 1) tmem_alloc<512>(&sm.tmem_base);
    tc_fence_before();
    __syncthreads();
    if constexpr (kMc > 1) cluster_sync();  // peers' barriers exist before any remote arrive / multicast
    tc_fence_after();
    // launched as a programmatic dependent of the planning grid: everything above overlapped
    // its tail; the tile lists, bitmaps, gathered rows and work counters are read below
    griddep_wait();
    const uint32_t tmem = sm.tmem_base;
    // register split (per warpgroup, at the top of each role's branch so the allocator sees
    // it): the producer / MMA warpgroup needs few, the softmax warps hold a whole S row (128
    // fp32) in registers. setmaxnreg.inc waits for registers released by .dec inside the CTA:
    // (168 - kRegsOther) x 128 >= (kRegsSoftmax - 168) x 256
    if (warp < 4) {
    setmaxnreg_dec<kRegsOther>();
    if (warp == 0) {
        // =========================== TMA producer (warp-uniform loop, elected issuer)
        if (elect_one()) {
            tma_prefetch_desc(&p.map_q);
            tma_prefetch_desc(&p.map_k);
            tma_prefetch_desc(&p.map_v);
            if constexpr (kSparse) {
                tma_prefetch_desc(&p.map_kv);
                tma_prefetch_desc(&p.map_vv);
            }
        }
        __syncwarp();
        int gj = 0;  // K/V ring position, continuous across items
        // Producer side of the item ring, one round ahead of the item being loaded: the next
        // item's Q tiles are prefetched into L2 while this item streams its K/V tiles, so the
        // Q load at the item boundary (single-buffered, it waits for the last S MMA) hits L2.
        // The leader also reads the item's tile-list header here, so the consumers take it
        // from shared memory instead of each paying an L2 round trip at the item boundary
        // (both CTAs of a cluster run the same (KV head, query block): same header).
        auto fetch = [&](int n_it, int& nt, int& vc) {
            const int slot = n_it % kItemRing;
            int it = 0;
            if (crank == 0) {
                if (n_it >= kItemRing) mbar_wait(&sm.item_empty[slot], ((n_it / kItemRing) - 1) & 1);
                if (lane == 0) {
                    const int nclusters = static_cast<int>(gridDim.x) / kMc;
                    it = n_it == 0 ? static_cast<int>(blockIdx.x) / kMc : atomicAdd(p.work + 0, 1) + nclusters;
                    if (it >= p.items) it = -1;
                    nt = 0;
                    vc = 0;
                    if (kSparse && it >= 0) {
                        const int* hdr = item(it, 0, 0).tiles - 2;
                        nt = __ldcg(hdr);
                        vc = __ldcg(hdr + 1);
                    }
                    sm.item[slot] = it;
                    sm.item_nt[slot] = nt;
                    sm.item_vc[slot] = vc;
                    mbar_arrive(&sm.item_full[slot]);  // release: the item is visible to waiters
                    if constexpr (kMc > 1) {
                        st_cluster_u32(mapa_shared(smem_u32(&sm.item[slot]), 1), static_cast<uint32_t>(it));
                        st_cluster_u32(mapa_shared(smem_u32(&sm.item_nt[slot]), 1), static_cast<uint32_t>(nt));
                        st_cluster_u32(mapa_shared(smem_u32(&sm.item_vc[slot]), 1), static_cast<uint32_t>(vc));
                        mbar_arrive_cluster(mapa_shared(smem_u32(&sm.item_full[slot]), 1));
                    }
                }
                it = __shfl_sync(0xffffffffu, it, 0);
                nt = __shfl_sync(0xffffffffu, nt, 0);
                vc = __shfl_sync(0xffffffffu, vc, 0);
            } else {
                it = next_item(n_it, nt, vc);  // the peer's producer consumes the leader's fetch
            }
            return it;
        };
        int nt_next = 0, vc_next = 0;
        int it_next = fetch(0, nt_next, vc_next);
        for (int n_it = 0;; ++n_it) {
            const int it = it_next, it_nt = nt_next, it_vc = vc_next;
            if (it < 0) break;
            it_next = fetch(n_it + 1, nt_next, vc_next);
            VSP_TRACE(9, 0, gj);
            if (it_next >= 0 && p.prefetch_q) {
                const Item xn = item(it_next, nt_next, vc_next);
                if (elect_one())
                    for (int w = 0; w < 2; ++w)
                        for (int hf = 0; hf < 2; ++hf) tma_prefetch_3d(&p.map_q, hf * 64, w ? xn.h1 : xn.h0, xn.qb * kBlock);
                __syncwarp();
            }
            const Item x = item(it, it_nt, it_vc);
            // the previous item's last S MMA has read its Q tiles
            if (n_it > 0) mbar_wait(&sm.q_free, (n_it - 1) & 1);
            VSP_TRACE(7, 0, gj);
            if (elect_one()) {
                mbar_arrive_expect_tx(&sm.q_full, 2 * kTileBytes);
                for (int w = 0; w < 2; ++w)
                    for (int hf = 0; hf < 2; ++hf)
                        tma_load_3d(sQ + w * kTileBytes + hf * kHalfBytes, &p.map_q, &sm.q_full, hf * 64,
                                    w ? x.h1 : x.h0, x.qb * kBlock);
            }
            __syncwarp();
            VSP_TRACE(9, 1, gj);
            for (int j = 0; j < x.num_tiles; ++j, ++gj) {
                // dense-mode blocks (vcnt0 < 0) list tiles 0..qb in order: no entry load
                const int e = (kSparse && x.vcnt0 >= 0) ? __ldg(x.tiles + j) : ent_make(j * kBlock, false, kBlock);
                const bool gathered = kSparse && ent_gathered(e);
                const int row = kSparse ? (gathered ? ent_value(e) * kBlock : ent_value(e)) : j * kBlock;
                const CUtensorMap* mk_ = gathered ? &p.map_kv : &p.map_k;
                const CUtensorMap* mv_ = gathered ? &p.map_vv : &p.map_v;
                const int c1 = gathered ? row : x.g, c2 = gathered ? x.g : row;
                const int ks = gj % kNumK;
                if (gj >= kNumK) mbar_wait(&sm.k_empty[ks], ((gj / kNumK) & 1) ^ 1);
                VSP_TRACE(10, 0, gj);
                if (elect_one()) {
                    mbar_arrive_expect_tx(&sm.k_full[ks], kTileBytes);
                    if constexpr (kMc > 1)  // this CTA's half, multicast; the peer sends the other
                        tma_load_3d_mc(sK + ks * kTileBytes + crank * kHalfBytes, mk_, &sm.k_full[ks],
                                       static_cast<int>(crank) * 64, c1, c2, 0x3);
                    else
                        for (int hf = 0; hf < 2; ++hf)
                            tma_load_3d(sK + ks * kTileBytes + hf * kHalfBytes, mk_, &sm.k_full[ks], hf * 64, c1, c2);
                }
                __syncwarp();
                const int vs = gj % kNumV;
                if (gj >= kNumV) mbar_wait(&sm.v_empty[vs], ((gj / kNumV) & 1) ^ 1);
                if (elect_one()) {
                    mbar_arrive_expect_tx(&sm.v_full[vs], kTileBytes);
                    if constexpr (kMc > 1)
                        tma_load_3d_mc(sV + vs * kTileBytes + crank * kHalfBytes, mv_, &sm.v_full[vs],
                                       static_cast<int>(crank) * 64, c1, c2, 0x3);
                    else
                        for (int hf = 0; hf < 2; ++hf)
                            tma_load_3d(sV + vs * kTileBytes + hf * kHalfBytes, mv_, &sm.v_full[vs], hf * 64, c1, c2);
                }
                __syncwarp();
            }
        }
    } else if (warp == 1) {
        // =========================== MMA issuer
        // The whole warp walks the schedule (warp-uniform control flow keeps descriptors in
        // uniform registers); one elected lane issues each batch of tcgen05.mma / commit.
        const uint32_t idesc_qk = umma_idesc_bf16(128, 128, false, false);
        // K/V ring slots are filled by both CTAs of a cluster: release to both
        auto release = [&](uint64_t* bar) {
            if constexpr (kMc > 1) umma_commit_mc(bar, 0x3);
            else umma_commit(bar);
        };
        const uint32_t idesc_pv = umma_idesc_bf16(128, 128, false, true);
        // descriptor bases; per-k offsets are added to the 14-bit start-address field
        const uint64_t q_desc0 = umma_desc_sw128(smem_u32(sQ), 16, 1024);
        const uint64_t k_desc0 = umma_desc_sw128(smem_u32(sK), 16, 1024);
        const uint64_t v_desc0 = umma_desc_sw128(smem_u32(sV), kHalfBytes, 1024);
        // gj: global tile index (ring slots and s/p barrier phases continue across items);
        // first: the item's first PV overwrites O (accumulate = 0)
        // half h of PV: K-steps [4h, 4h + 4), i.e. P columns [64h, 64h + 64) (TMEM [32h, 32h + 32))
        // against V rows [64h, 64h + 64); the softmax publishes the two halves separately
        // nk: K-steps of the tile (width / 16; 8 for a full tile)
        auto issue_pv = [&](int w, int gjj, bool first, int h, int nk) {
            const uint64_t vd = v_desc0 + static_cast<uint64_t>(((gjj % kNumV) * kTileBytes) >> 4);
            const uint32_t o_t = tmem + 256 + w * 128;
            const uint32_t p_t = tmem + w * 128;
            if (nk == 8) {  // full tile (every dense tile, most sparse ones): straight-line issue
#pragma unroll
                for (int k = 4 * h; k < 4 * h + 4; ++k)
                    umma_ts(o_t, p_t + k * 8, vd + static_cast<uint64_t>((k * 2048) >> 4), idesc_pv,
                            (!first || k > 0) ? 1u : 0u);
            } else {
#pragma unroll
                for (int k = 4 * h; k < 4 * h + 4; ++k)
                    if (k < nk)
                        umma_ts(o_t, p_t + k * 8, vd + static_cast<uint64_t>((k * 2048) >> 4), idesc_pv,
                                (!first || k > 0) ? 1u : 0u);
            }
        };
        // S_w = Q_w K^T over the tile's first `width` keys (N = width)
        auto issue_s = [&](int w, int gjj, int width) {
            const uint32_t idesc =
                width == kBlock ? idesc_qk : (idesc_qk & ~(0x3Fu << 17)) | (static_cast<uint32_t>(width >> 3) << 17);
            const uint64_t qd = q_desc0 + static_cast<uint64_t>((w * kTileBytes) >> 4);
            const uint64_t kd = k_desc0 + static_cast<uint64_t>(((gjj % kNumK) * kTileBytes) >> 4);
            const uint32_t s_t = tmem + w * 128;
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const uint64_t off = static_cast<uint64_t>(((k >> 2) * kHalfBytes + (k & 3) * 32) >> 4);
                umma_ss(s_t, qd + off, kd + off, idesc, k > 0 ? 1u : 0u);
            }
        };
        int gj = 0;
        for (int n_it = 0;; ++n_it) {
            VSP_TRACE(8, 0, gj);
            int it_nt, it_vc;
            const int it = next_item(n_it, it_nt, it_vc);
            VSP_TRACE(8, 1, gj);
            if (it < 0) break;
            const Item x = item(it, it_nt, it_vc);
            const int nt = x.num_tiles;
            mbar_wait(&sm.q_full, n_it & 1);
            VSP_TRACE(7, 1, gj);
            tc_fence_after();
            if (nt == 0) {  // nothing covered: release the epilogue (O is not touched)
                // keep o_free's phases in lock-step with the items (no parity aliasing)
                if (n_it > 0) {
                    mbar_wait(&sm.o_free[0], (n_it - 1) & 1);
                    mbar_wait(&sm.o_free[1], (n_it - 1) & 1);
                }
                if (elect_one()) {
                    umma_commit(&sm.q_free);
                    umma_commit(&sm.o_done[0]);
                    umma_commit(&sm.o_done[1]);
                }
                __syncwarp();
                continue;
            }
            int nk_prev = 8;  // K-steps of tile j-1
            for (int j = 0; j < nt; ++j) {
                const int G = gj + j;
                const int ks = G % kNumK;
                const int width = (kSparse && x.vcnt0 >= 0) ? ent_width(__ldg(x.tiles + j)) : kBlock;
                mbar_wait(&sm.k_full[ks], (G / kNumK) & 1);
                VSP_TRACE(1, 0, G);
                tc_fence_after();
                for (int w = 0; w < 2; ++w) {
                    if (j > 0) {
                        // first half of P(j-1): its PV overlaps the softmax's second half
                        mbar_wait(&sm.p_half[w], (G - 1) & 1);
                        VSP_TRACE(6, w, G - 1);
                        if (w == 0) mbar_wait(&sm.v_full[(G - 1) % kNumV], ((G - 1) / kNumV) & 1);
                        // the item's first PV writes O_w: the previous item's epilogue must be done
                        if (j == 1 && n_it > 0) mbar_wait(&sm.o_free[w], (n_it - 1) & 1);
                        tc_fence_after();
                        if (elect_one()) issue_pv(w, G - 1, j == 1, 0, nk_prev);
                        __syncwarp();
                        mbar_wait(&sm.p_full[w], (G - 1) & 1);
                        tc_fence_after();
                    }
                    VSP_TRACE(0, w, G);
                    if (elect_one()) {
                        if (j > 0) {
                            issue_pv(w, G - 1, false, 1, nk_prev);
                            if (w == 1) release(&sm.v_empty[(G - 1) % kNumV]);
                        }
                        issue_s(w, G, width);
                        umma_commit(&sm.s_full[w]);
                        if (w == 1) {
                            release(&sm.k_empty[ks]);
                            if (j == nt - 1) umma_commit(&sm.q_free);  // Q of this item no longer read
                        }
                    }
                    __syncwarp();
                }
                nk_prev = width >> 4;
            }
            const int GL = gj + nt - 1;
            for (int w = 0; w < 2; ++w) {
                mbar_wait(&sm.p_half[w], GL & 1);
                if (w == 0) mbar_wait(&sm.v_full[GL % kNumV], (GL / kNumV) & 1);
                if (nt == 1 && n_it > 0) mbar_wait(&sm.o_free[w], (n_it - 1) & 1);
                tc_fence_after();
                if (elect_one()) issue_pv(w, GL, nt == 1, 0, nk_prev);
                __syncwarp();
                mbar_wait(&sm.p_full[w], GL & 1);
                tc_fence_after();
                if (elect_one()) {
                    issue_pv(w, GL, false, 1, nk_prev);
                    umma_commit(&sm.o_done[w]);
                    if (w == 1) release(&sm.v_empty[GL % kNumV]);
                }
                __syncwarp();
            }
            gj += nt;
        }
    }
    } else {
        setmaxnreg_inc<kRegsSoftmax>();
        // =========================== softmax + epilogue
        const int w = (warp - 4) >> 2;             // Q tile / head within the pair
        const int quarter = warp & 3;              // TMEM lane quarter
        const int r = quarter * 32 + lane;         // row within the block
        const uint32_t lane_base = tmem + (static_cast<uint32_t>(quarter * 32) << 16);
        const uint32_t s_t = lane_base + w * 128;
        const uint32_t o_t = lane_base + 256 + w * 128;
        const float sl2 = p.scale * kLog2e;
        int gt = 0;  // global tile index: s_full / p_full phases continue across items
        for (int n_it = 0;; ++n_it) {
        int it_nt, it_vc;
        const int it = next_item(n_it, it_nt, it_vc);
        if (it < 0) break;
        const Item x = item(it, it_nt, it_vc);
        const int qb = x.qb, g = x.g, num_tiles = x.num_tiles, vcnt0 = x.vcnt0;
        const int* tiles = x.tiles;
        (void)tiles;
        (void)vcnt0;
        const int i0 = qb * kBlock;
        const int i = i0 + r;                      // query row

        // sparse: #{I_v <= i} = vcnt0 + popcount(vbits over [i0, i])
        int vcnt_i = 0;
        if (kSparse && vcnt0 >= 0) {
            uint32_t vw[4];
            window128(p.vbits + static_cast<size_t>(g) * p.bm_words, i0, p.bm_words, vw);
            int c = 0;
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const int lo = 32 * k;
                if (r >= lo + 31) c += __popc(vw[k]);
                else if (r >= lo) c += __popc(vw[k] & (0xffffffffu >> (31 - (r - lo))));
            }
            vcnt_i = vcnt0 + c;
        }

        float m_used = -INFINITY;
        float l = 0.f;
        for (int j = 0; j < num_tiles; ++j) {
            // ---- mask for this tile: bit c of mk[c>>5] = column allowed
            uint32_t mk[4] = {0xffffffffu, 0xffffffffu, 0xffffffffu, 0xffffffffu};
            bool masked = false;
            int width = kBlock;  // columns the S MMA wrote (the rest of S is stale)
            auto prefix_word = [](int b) { return b <= 0 ? 0u : (b >= 32 ? 0xffffffffu : (0xffffffffu >> (32 - b))); };
            if constexpr (kSparse) {
                const int ee = vcnt0 >= 0 ? __ldg(tiles + j) : ent_make(j * kBlock, false, kBlock);
                const int e = ent_value(ee);
                width = ent_width(ee);
                if (ent_gathered(ee)) {
                    // allowed gathered rows: c < lim (lim <= the tile's width by construction)
                    const int lim = vcnt_i - e * kBlock;
                    if (lim < kBlock) {
                        masked = true;
#pragma unroll
                        for (int k = 0; k < 4; ++k) mk[k] = prefix_word(lim - 32 * k);
                    }
                } else if (vcnt0 == -2) {  // dense switch: unmasked causal block
                    if (e == i0) {
                        masked = true;
#pragma unroll
                        for (int k = 0; k < 4; ++k) mk[k] = prefix_word(r - 32 * k + 1);
                    }
                } else {
                    masked = true;
#if VSP_NOINLINE_SLASH_MASK
                    const uint4 m4 = slash_tile_mask(p.vbits + static_cast<size_t>(g) * p.bm_words,
                                                     p.sbits + static_cast<size_t>(g) * p.bm_words, p.bm_words, e, i,
                                                     width, vcnt0);
                    mk[0] = m4.x;
                    mk[1] = m4.y;
                    mk[2] = m4.z;
                    mk[3] = m4.w;
#else
                    uint32_t vw[4], sw[4];
                    window128(p.vbits + static_cast<size_t>(g) * p.bm_words, e, p.bm_words, vw);
                    window128(p.sbits + static_cast<size_t>(g) * p.bm_words, i - e - 127, p.bm_words, sw);
                    if (vcnt0 >= 0) {
#pragma unroll
                        for (int k = 0; k < 4; ++k) mk[k] = __brev(sw[3 - k]) & ~vw[k];
                    } else {  // dense-masked block: verticals come from this tile too (j <= i)
                        const int lim = i - e + 1;
#pragma unroll
                        for (int k = 0; k < 4; ++k) mk[k] = __brev(sw[3 - k]) | (vw[k] & prefix_word(lim - 32 * k));
                    }
                    // columns past a narrow tile belong to the next tile of the range
#pragma unroll
                    for (int k = 0; k < 4; ++k) mk[k] &= prefix_word(width - 32 * k);
#endif
                }
            } else {
                if (j == qb) {  // diagonal tile: c <= r
                    masked = true;
#pragma unroll
                    for (int k = 0; k < 4; ++k) mk[k] = prefix_word(r - 32 * k + 1);
                }
            }

            masked = __any_sync(0xffffffffu, masked || width < kBlock);
            // Masked tiles work per 32-column chunk with warp-uniform modes: a chunk masked for
            // all 32 rows of the warp is skipped (no max, no exponentials; its P is written as
            // zeros) — most of a slash tile, the tail of a vertical run; a partially masked chunk
            // gets element selects; a fully allowed one neither. Unmasked tiles take a
            // branch-free path.
            uint32_t dead = 0u, part = 0u;
            if (masked) {
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    if (!__any_sync(0xffffffffu, mk[k] != 0u)) dead |= 1u << k;
                    else if (__any_sync(0xffffffffu, mk[k] != 0xffffffffu)) part |= 1u << k;
                }
            }
            mbar_wait(&sm.s_full[w], (gt + j) & 1);
            if (quarter == 0) VSP_TRACE(2, w, gt + j);
            tc_fence_after();
            if (masked)
                softmax_tile<true>(s_t, o_t, dead, part, make_uint4(mk[0], mk[1], mk[2], mk[3]), width, j, sl2, m_used, l, &sm.p_half[w], quarter, w, gt + j);
            else
                softmax_tile<false>(s_t, o_t, dead, part, make_uint4(mk[0], mk[1], mk[2], mk[3]), width, j, sl2, m_used, l, &sm.p_half[w], quarter, w, gt + j);
            tmem_wait_st();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&sm.p_full[w]);
            if (quarter == 0) VSP_TRACE(5, w, gt + j);
        }

        // ---- epilogue: O / l -> bf16 [n, Hq, d]; LSE (natural log of sum exp(scaled logits))
        mbar_wait(&sm.o_done[w], n_it & 1);
        tc_fence_after();
        const int h = w ? x.h1 : x.h0;
        const bool store = w == 0 || x.h1 != x.h0;  // a duplicated head is written once
        const float inv_l = l > 0.f ? 1.f / l : 0.f;
        // O -> bf16 through a swizzled 16 KB staging half per Q tile and TMA stores (one 64-column
        // half at a time): per-thread row stores (rows 256 B apart) clogged the LSU/MIO pipe for
        // thousands of cycles at every item end. Rows past n are clipped by the TMA unit.
        uint8_t* stage = sO + w * kOStage;
        const bool issuer = quarter == 0 && lane == 0;
#pragma unroll
        for (int hf = 0; hf < 2; ++hf) {
            uint32_t v[2][32];
            tmem_ld32(o_t + hf * 64, v[0]);
            tmem_ld32(o_t + hf * 64 + 32, v[1]);
            tmem_wait_ld();
            tmem_reg_fence(v[0]);
            tmem_reg_fence(v[1]);
            if (hf == 1) {  // O_w has been read: the next item's first PV may overwrite it
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&sm.o_free[w]);
            }
            if (store) {
                // the previous TMA store from this buffer has finished reading it
                if (issuer) bulk_wait_read0();
                named_bar_sync(1 + w, 128);
#pragma unroll
                for (int u8 = 0; u8 < 8; ++u8) {  // 16-byte unit u8 of the row's 128-byte half
                    uint4 q4;
                    const uint32_t* src = &v[u8 >> 2][(u8 & 3) * 8];
                    q4.x = num_tiles ? pack_bf16x2(__uint_as_float(src[0]) * inv_l, __uint_as_float(src[1]) * inv_l) : 0u;
                    q4.y = num_tiles ? pack_bf16x2(__uint_as_float(src[2]) * inv_l, __uint_as_float(src[3]) * inv_l) : 0u;
                    q4.z = num_tiles ? pack_bf16x2(__uint_as_float(src[4]) * inv_l, __uint_as_float(src[5]) * inv_l) : 0u;
                    q4.w = num_tiles ? pack_bf16x2(__uint_as_float(src[6]) * inv_l, __uint_as_float(src[7]) * inv_l) : 0u;
                    *reinterpret_cast<uint4*>(stage + r * 128 + ((u8 ^ (r & 7)) << 4)) = q4;  // SWIZZLE_128B
                }
                fence_proxy_async_smem();
                named_bar_sync(1 + w, 128);
                if (issuer && !(p.prefetch_q & 2)) {
                    tma_store_3d(&p.map_o, stage, hf * 64, h, i0);
                    for (int m = 0; m < p.n_mirrors; ++m)  // the same tile into every mirror (peer HBM over NVLink)
                        tma_store_3d(&p.map_o_mirror[m], stage, hf * 64, h, i0);
                    bulk_commit_group();
                }
            }
        }
        if (i < p.n && store) {
            const float lse_i = l > 0.f ? (m_used + __log2f(l)) * kLn2 : -INFINITY;
            if (p.lse != nullptr) p.lse[static_cast<size_t>(h) * p.n + i] = lse_i;
            for (int m = 0; m < p.n_mirrors; ++m)
                if (p.lse_mirror[m] != nullptr) p.lse_mirror[m][static_cast<size_t>(h) * p.n + i] = lse_i;
        }
        gt += num_tiles;
        }
        if (quarter == 0 && lane == 0) bulk_wait0();  // this tile's O stores are complete
    }

    // mirrored outputs live in other GPUs' memory: make this CTA's stores (the TMA stores have
    // completed, bulk_wait0 above) visible system-wide before the launch can be seen as done
    if (p.n_mirrors > 0) __threadfence_system();
    tc_fence_before();
    __syncthreads();
    if (warp == 1) tmem_free<512>(tmem);
    // no CTA of a cluster leaves while its peer may still multicast into it or arrive on it
    if constexpr (kMc > 1) cluster_sync();
    // the last CTA out resets the work counter for the next launch on this stream
    if (threadIdx.x == 0) {
        __threadfence();
        if (atomicAdd(p.work + 1, 1) == static_cast<int>(gridDim.x) - 1) {
            p.work[0] = 0;
            p.work[1] = 0;
            __threadfence();
        }
    }
}

// ------------------------------------------------------------------ sparse planning

// #{a[t] <= x} for ascending a[0, n), by the whole warp: a 32-ary search (one pivot per lane,
// a ballot narrows the range 32x per step), so 4 dependent L2 round trips at n = 128k
// instead of the 17 of a binary search. Warp-uniform arguments.
VSP_DEVICE int warp_upper_bound(const int* a, int n, int x) {
    const int lane = threadIdx.x & 31;
    int lo = 0, hi = n;  // answer in [lo, hi]
    while (lo < hi) {
        const int step = (hi - lo + 31) >> 5;
        const int pv = lo + (lane + 1) * step - 1;
        const bool t = pv < hi && __ldg(a + pv) <= x;
        const int nlo = lo + __popc(__ballot_sync(0xffffffffu, t)) * step;
        hi = min(hi, nlo + step - 1);
        lo = nlo;
    }
    return lo;
}

// Sparse planning in ONE launch (it replaced two memsets and three kernels): blockIdx.x
// selects the role, blockIdx.y the KV head, 128 threads.
//   [0, 2 nbw)            bitmaps: block c of direction d owns bitmap words [128c, 128c+128)
//                         (bit j of vbits[g] <=> j in I_v[g]; bit o of sbits[g] <=> o in I_s[g]);
//                         the words are built in shared memory from the sorted index run
//                         that falls into them and stored whole, so no memset is needed
//   [2 nbw, 2 nbw + ngb)  vertical gather (gather_vertical below)
//   [.., + nplan)         tile lists, four query blocks per block (plan_block below); the
//                         first plan block also zeroes the head's attention work counters
// The attention kernel is launched as a programmatic dependent of this grid: every block
// triggers at entry, so K3's CTAs take over the SMs as this grid drains and run their
// prologue before their griddepcontrol.wait.
struct PrepArgs {
    const int* iv;
    const int* kv;
    const int* is;
    const int* ks;
    int cap, n, bm_words, hkv, kvcap, num_qb, list_stride, g0;
    int nbw, ngb;  // bitmap blocks per direction, gather blocks
    int dense_switch;
    uint32_t* vbits;
    uint32_t* sbits;
    const __nv_bfloat16* k;
    const __nv_bfloat16* v;
    __nv_bfloat16* kg;
    __nv_bfloat16* vg;
    int* lists;
    int* work;
};

VSP_DEVICE void build_bitmap_block(const int* __restrict__ idx, int count, int n, int bm_words, int c,
                                   uint32_t* __restrict__ bits, uint32_t* sw) {
    const int w0 = c * 128;
    sw[threadIdx.x] = 0u;
    __shared__ int range[2];
    const int wid = threadIdx.x >> 5;
    if (wid < 2) {
        // index run [lo, hi) of the sorted list inside columns [32 w0, 32 (w0 + 128)) and < n
        const int col = min(32 * (w0 + 128 * wid), n);
        const int lo = warp_upper_bound(idx, count, col - 1);  // #{idx < col}
        if ((threadIdx.x & 31) == 0) range[wid] = lo;
    }
    __syncthreads();
#pragma unroll 4
    for (int t = range[0] + static_cast<int>(threadIdx.x); t < range[1]; t += blockDim.x) {
        const int j = __ldg(idx + t);
        if (j >= 0) atomicOr(sw + ((j >> 5) - w0), 1u << (j & 31));  // columns >= n never set
    }
    __syncthreads();
    if (w0 + static_cast<int>(threadIdx.x) < bm_words) bits[w0 + threadIdx.x] = sw[threadIdx.x];
}

// Kv[g][r] = K[I_v[g][r]][g] for r < k_v; rows [k_v, round_up(k_v, 128)) zero (the last
// gathered tile is read whole: finite V rows keep 0 * V out of NaN); rows past that tile are
// never read, so they are not written. 16 threads x 16 B per 256 B row, 8 rows per step.
VSP_DEVICE void gather_vertical(const PrepArgs& a, int g, int b, int nb) {
    const int t = threadIdx.x & 15;
    const int cnt = min(a.kv[g], a.kvcap);
    const int rows = min((cnt + kBlock - 1) / kBlock * kBlock, a.kvcap);
    for (int r = b * 8 + (threadIdx.x >> 4); r < rows; r += nb * 8) {
        uint4 x = make_uint4(0, 0, 0, 0), y = make_uint4(0, 0, 0, 0);
        if (r < cnt) {
            const int j = min(max(__ldg(a.iv + static_cast<size_t>(g) * a.cap + r), 0), a.n - 1);
            x = __ldg(reinterpret_cast<const uint4*>(a.k + (static_cast<size_t>(j) * a.hkv + g) * kHeadDim) + t);
            y = __ldg(reinterpret_cast<const uint4*>(a.v + (static_cast<size_t>(j) * a.hkv + g) * kHeadDim) + t);
        }
        reinterpret_cast<uint4*>(a.kg + (static_cast<size_t>(g) * a.kvcap + r) * kHeadDim)[t] = x;
        reinterpret_cast<uint4*>(a.vg + (static_cast<size_t>(g) * a.kvcap + r) * kHeadDim)[t] = y;
    }
}


// Per (KV head g, query block qb): header {num_tiles, vcnt0} then entries (see file
// header). Slash spans: for offsets o <= i_last (ascending I_s walked from the largest
// offset down, i.e. ascending column start) the column intervals [max(0,i0-o), i_last-o]
// are merged and covered greedily by disjoint 128-row tiles.
// One warp per (KV head, query block). Walking the offsets from the largest down gives
// intervals [lo, hi] = [max(0, i0-o), i_last-o] with lo and hi both non-decreasing, so a
// merged range is [lo of its first interval, hi of its last] and a range breaks exactly where
// lo_next > hi_prev + 1. 32 offsets are classified per step (coalesced loads, ballot of the
// breaks); lane 0 emits the finished ranges' tiles in order. grid (ceil(num_qb/4), hkv), 128.
VSP_DEVICE void plan_block(const int* __restrict__ iv, const int* __restrict__ kv, const int* __restrict__ is,
                           const int* __restrict__ ks, int cap, int n, int num_qb, int list_stride,
                           int* __restrict__ lists, int g, int qb, int dense_switch) {
    const int lane = threadIdx.x & 31;
    if (qb >= num_qb) return;
    const int i0 = qb * kBlock;
    const int ilast = min(i0 + kBlock - 1, n - 1);
    const int* ivg = iv + static_cast<size_t>(g) * cap;
    const int* isg = is + static_cast<size_t>(g) * cap;
    const int k_v = kv[g], k_s = ks[g];
    int* out = lists + (static_cast<size_t>(g) * num_qb + qb) * list_stride;
    const int cv = warp_upper_bound(ivg, k_v, ilast);
    const int vc0 = warp_upper_bound(ivg, k_v, i0 - 1);
    const int ntv = (cv + kBlock - 1) / kBlock;
    // the run's last gathered tile is narrow: its used rows rounded up to 16
    for (int t = lane; t < ntv; t += 32)
        out[2 + t] = ent_make(t, true, t == ntv - 1 ? round16(cv - t * kBlock) : kBlock);
    int cnt = ntv;
    const int s = warp_upper_bound(isg, k_s, ilast);
    int cur = 0, a = -1, b = -1;  // open range [a, b] (lane-uniform state)
    auto emit = [&](int lo, int hi) {  // lane-uniform: every lane computes, lanes write
        const int st0 = max(lo, cur);
        const int m = st0 <= hi ? (hi - st0) / kBlock + 1 : 0;
        const int wl = round16(hi - (st0 + (m - 1) * kBlock) + 1);  // narrow last tile of the range
        for (int x = lane; x < m; x += 32) out[2 + cnt + x] = ent_make(st0 + x * kBlock, false, x == m - 1 ? wl : kBlock);
        cnt += m;
        if (m) cur = st0 + (m - 1) * kBlock + wl;
    };
    const int limit = qb + 1;  // stop as soon as dense-masked mode is certain
    {
        // m offsets <= i0 give m length-128 intervals with distinct starts: their union spans
        // >= m + 127 columns, so the slash tiles alone number >= ceil(m / 128)
        const int m = warp_upper_bound(isg, k_s, i0);
        if (cnt + (m + 127) / kBlock >= limit) cnt = limit;
    }
    // four 32-offset chunks per round: their loads are issued together (one L2 round trip per
    // 128 offsets instead of per 32), then the chunks are merged in order
    for (int base4 = s - 1; base4 >= 0 && cnt < limit; base4 -= 128) {
        int ov[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int t = base4 - 32 * q - lane;
            ov[q] = t >= 0 ? __ldg(isg + t) : 0;
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int base = base4 - 32 * q;
            if (base < 0 || cnt >= limit) break;
            const bool valid = base - lane >= 0;
            const int o = ov[q];
            const int lo = max(0, i0 - o), hi = ilast - o;
            const int prev_hi = __shfl_up_sync(0xffffffffu, hi, 1);
            bool brk = valid && (lane == 0 ? (a >= 0 && lo > b + 1) : (lo > prev_hi + 1));
            const unsigned bm = __ballot_sync(0xffffffffu, brk);
            const unsigned vm = __ballot_sync(0xffffffffu, valid);
            if (a < 0) a = __shfl_sync(0xffffffffu, lo, 0);  // first interval opens the first range
            unsigned rem = bm;
            while (rem) {  // close the open range at each break, open the next one
                const int e = __ffs(rem) - 1;
                rem &= rem - 1;
                const int b_close = e == 0 ? b : __shfl_sync(0xffffffffu, hi, e - 1);
                emit(a, b_close);
                a = __shfl_sync(0xffffffffu, lo, e);
            }
            const int last = 31 - __clz(vm);
            b = __shfl_sync(0xffffffffu, hi, last);
            // the open range only grows: once it alone would reach the limit, the block is
            // dense (long runs of consecutive offsets otherwise walk the whole list)
            const int st0 = max(a, cur);
            if (b >= st0 && cnt + (b - st0) / kBlock + 1 >= limit) cnt = limit;
        }
    }
    if (a >= 0 && cnt < limit) emit(a, b);
    const bool dense_mode = cnt >= limit;
    if (dense_mode) {
        // the VS tiles would visit at least as many tiles as the dense causal row of tiles:
        // switch this block to dense-masked mode (header vcnt0 = -1), columns [0, i0+127]
        // with mask (j in I_v OR i-j in I_s) AND j <= i. With the dense switch (opt-in,
        // VSP_DENSE_SWITCH) the block runs unmasked causal attention instead (vcnt0 = -2):
        // the same tiles, no mask work, every causal pair of its rows covered.
        __syncwarp();
        for (int t = lane; t < limit; t += 32) out[2 + t] = ent_make(t * kBlock, false, kBlock);
        cnt = limit;
    }
    if (lane == 0) {
        out[0] = cnt;
        out[1] = dense_mode ? (dense_switch ? -2 : -1) : vc0;
    }
}

__global__ void __launch_bounds__(128) vs_prep_kernel(const __grid_constant__ PrepArgs a) {
    griddep_launch_dependents();
    const int g = a.g0 + static_cast<int>(blockIdx.y);
    const int b = blockIdx.x;
    __shared__ uint32_t sw[128];
    if (b < 2 * a.nbw) {
        const bool slash = b >= a.nbw;
        build_bitmap_block(slash ? a.is + static_cast<size_t>(g) * a.cap : a.iv + static_cast<size_t>(g) * a.cap,
                           slash ? a.ks[g] : a.kv[g], a.n, a.bm_words, slash ? b - a.nbw : b,
                           (slash ? a.sbits : a.vbits) + static_cast<size_t>(g) * a.bm_words, sw);
    } else if (b < 2 * a.nbw + a.ngb) {
        gather_vertical(a, g, b - 2 * a.nbw, a.ngb);
    } else {
        const int pb = b - 2 * a.nbw - a.ngb;
        if (pb == 0 && threadIdx.x < 2) a.work[2 * g + threadIdx.x] = 0;
        plan_block(a.iv, a.kv, a.is, a.ks, a.cap, a.n, a.num_qb, a.list_stride, a.lists, g, pb * 4 + (threadIdx.x >> 5),
                   a.dense_switch);
    }
}

// ------------------------------------------------------------------ host launchers

static bool set_o_layout(AttnParams& p, const AttnArgs& a) {
    p.o_tok_stride = a.o_head_major ? kHeadDim : static_cast<long long>(a.hq) * kHeadDim;
    p.o_head_stride = a.o_head_major ? static_cast<long long>(a.n) * kHeadDim : kHeadDim;
    const uint32_t box[3] = {64, 1, kBlock};
    const uint64_t dims[3] = {kHeadDim, (uint64_t)a.hq, (uint64_t)a.n};
    const uint64_t strides[2] = {static_cast<uint64_t>(p.o_head_stride) * 2, static_cast<uint64_t>(p.o_tok_stride) * 2};
    if (a.n_mirrors < 0 || a.n_mirrors > kMaxMirrors || (a.n_mirrors > 0 && a.o_mirrors == nullptr)) return false;
    p.n_mirrors = a.n_mirrors;
    for (int m = 0; m < a.n_mirrors; ++m) {
        if (a.o_mirrors[m] == nullptr ||
            !vsp_host::make_map_bf16(&p.map_o_mirror[m], a.o_mirrors[m], 3, dims, strides, box))
            return false;
        p.lse_mirror[m] = a.lse_mirrors ? a.lse_mirrors[m] : nullptr;
    }
    return vsp_host::make_map_bf16(&p.map_o, a.o, 3, dims, strides, box);
}

static bool make_qkv_maps(AttnParams& p, const void* q, const void* k, const void* v) {
    const uint32_t box[3] = {64, 1, kBlock};
    const uint64_t dq[3] = {kHeadDim, (uint64_t)p.hq, (uint64_t)p.n};
    const uint64_t sq[2] = {kHeadDim * 2, (uint64_t)p.hq * kHeadDim * 2};
    const uint64_t dk[3] = {kHeadDim, (uint64_t)p.hkv, (uint64_t)p.n};
    const uint64_t sk[2] = {kHeadDim * 2, (uint64_t)p.hkv * kHeadDim * 2};
    return vsp_host::make_map_bf16(&p.map_q, q, 3, dq, sq, box) &&
           vsp_host::make_map_bf16(&p.map_k, k, 3, dk, sk, box) &&
           vsp_host::make_map_bf16(&p.map_v, v, 3, dk, sk, box);
}

// work counters of the dense kernel (zero at module load, reset by each launch's last CTA);
// every launch takes the next of kDenseSlots pairs, so launches in flight on different
// streams (up to kDenseSlots of them) never share a counter
constexpr int kDenseSlots = 256;
__device__ int g_dense_work[2 * kDenseSlots];
std::atomic<unsigned> g_dense_slot{0};

bool getenv_flag(const char* name) {
    const char* v = std::getenv(name);
    return v != nullptr && v[0] != '\0' && v[0] != '0';
}

// persistent grid: one CTA per SM (the kernel's smem allows one), never more than the items
int persistent_grid(int items) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    return std::max(1, std::min(items, sms));
}

// Launch the attention kernel: pairs of Q-head pairs in two-CTA clusters (K/V multicast) when
// every KV group has an even number of pairs (group size a multiple of 4), else one CTA per
// item. Grid: one CTA per SM, never more CTAs than items need.
template <bool kSparse>
cudaError_t launch_attn(AttnParams& p, int nqb, cudaStream_t stream) {
    static std::once_flag attr[vsp_detail::kMaxDevices];
    vsp_detail::once_per_device(attr, [] {
        cudaFuncSetAttribute(attn_fwd_kernel<kSparse, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes);
        cudaFuncSetAttribute(attn_fwd_kernel<kSparse, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes);
    });
    const int grp = p.hq / p.hkv;
    const bool mc = ((grp + 1) / 2) % 2 == 0 && p.pair0 % 2 == 0 && p.npairs % 2 == 0 && !getenv_flag("VSP_NO_MULTICAST");
    p.prefetch_q = (getenv_flag("VSP_NO_Q_PREFETCH") ? 0 : 1) | (getenv_flag("VSP_DEBUG_NO_O_STORE") ? 2 : 0);
    vsp_detail::count_launch();
    if (!mc) {
        p.items = nqb * p.npairs;
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(persistent_grid(p.items));
        cfg.blockDim = dim3(kThreads);
        cfg.dynamicSmemBytes = kSmemBytes;
        cfg.stream = stream;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = kSparse ? 1 : 0;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        return cudaLaunchKernelEx(&cfg, attn_fwd_kernel<kSparse, 1>, p);
    }
    p.items = nqb * (p.npairs / 2);
    const int clusters = std::max(1, std::min(p.items, persistent_grid(1 << 30) / 2));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(2 * clusters);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = kSmemBytes;
    cfg.stream = stream;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[1].val.programmaticStreamSerializationAllowed = kSparse ? 1 : 0;
    cfg.attrs = at;
    cfg.numAttrs = 2;
    return cudaLaunchKernelEx(&cfg, attn_fwd_kernel<kSparse, 2>, p);
}

cudaError_t launch_dense(const AttnArgs& a, cudaStream_t stream) {
    AttnParams p{};
    p.n = a.n;
    p.hq = a.hq;
    p.hkv = a.hkv;
    p.scale = a.scale;
    p.o = static_cast<__nv_bfloat16*>(a.o);
    p.lse = a.lse;
    if (!set_o_layout(p, a) || !make_qkv_maps(p, a.q, a.k, a.v)) return cudaErrorInvalidValue;
    const int num_qb = (a.n + kBlock - 1) / kBlock;
    p.pair0 = 0;
    p.npairs = a.hkv * ((a.hq / a.hkv + 1) / 2);
    p.qb_hi = num_qb;
    void* work = nullptr;
    cudaGetSymbolAddress(&work, g_dense_work);
    p.work = static_cast<int*>(work) + 2 * (g_dense_slot.fetch_add(1, std::memory_order_relaxed) % kDenseSlots);
    return launch_attn<false>(p, num_qb, stream);
}

size_t sparse_workspace_bytes(int n, int hkv, int cap) {
    const int num_qb = (n + kBlock - 1) / kBlock;
    const int kvcap = ((cap + kBlock - 1) / kBlock) * kBlock;
    const int bm_words = (n + 31) / 32 + 1;
    const int list_stride = 2 + kvcap / kBlock + num_qb + 3;
    size_t bytes = 0;
    auto add = [&](size_t b) { bytes += (b + 255) & ~size_t(255); };
    add(static_cast<size_t>(hkv) * kvcap * kHeadDim * 2);  // Kv
    add(static_cast<size_t>(hkv) * kvcap * kHeadDim * 2);  // Vv
    add(static_cast<size_t>(hkv) * bm_words * 4 * 2);      // bitmaps
    add(static_cast<size_t>(hkv) * num_qb * list_stride * 4);
    add(static_cast<size_t>(hkv) * 2 * 4);                 // per-KV-head work counters
    add(2 * 4 + static_cast<size_t>(kMaxUnits) * 4 * 4);  // units launch: counters + unit table
    return bytes;
}

// phase: 1 = plan (bitmaps, vertical gather, tile lists), 2 = attention kernel, 3 = both;
// only KV heads [g0, g0 + count) are touched, so head ranges can be pipelined on streams.
namespace {
cudaError_t launch_sparse_impl(const AttnArgs& a, const SparseArgs& s, void* workspace, cudaStream_t stream, int g0,
                               int count, int phase, int qb_lo, int qb_hi, const int* host_units, int nunits) {
    if (count < 0) count = a.hkv - g0;
    if (a.n >= kEntGathered) return cudaErrorInvalidValue;  // tile-list entries hold rows in 27 bits
    AttnParams p{};
    p.n = a.n;
    p.hq = a.hq;
    p.hkv = a.hkv;
    p.scale = a.scale;
    p.o = static_cast<__nv_bfloat16*>(a.o);
    p.lse = a.lse;
    if (!set_o_layout(p, a) || !make_qkv_maps(p, a.q, a.k, a.v)) return cudaErrorInvalidValue;
    const int num_qb = (a.n + kBlock - 1) / kBlock;
    const int kvcap = ((s.cap + kBlock - 1) / kBlock) * kBlock;
    const int bm_words = (a.n + 31) / 32 + 1;
    const int list_stride = 2 + kvcap / kBlock + num_qb + 3;
    uint8_t* ws = static_cast<uint8_t*>(workspace);
    auto take = [&](size_t b) {
        uint8_t* r = ws;
        ws += (b + 255) & ~size_t(255);
        return r;
    };
    auto* kg = reinterpret_cast<__nv_bfloat16*>(take(static_cast<size_t>(a.hkv) * kvcap * kHeadDim * 2));
    auto* vg = reinterpret_cast<__nv_bfloat16*>(take(static_cast<size_t>(a.hkv) * kvcap * kHeadDim * 2));
    auto* bits = reinterpret_cast<uint32_t*>(take(static_cast<size_t>(a.hkv) * bm_words * 4 * 2));
    auto* lists = reinterpret_cast<int*>(take(static_cast<size_t>(a.hkv) * num_qb * list_stride * 4));
    int* work = reinterpret_cast<int*>(take(static_cast<size_t>(a.hkv) * 2 * 4));
    int* uwork = reinterpret_cast<int*>(take(2 * 4 + static_cast<size_t>(kMaxUnits) * 4 * 4));
    p.vbits = bits;
    p.sbits = bits + static_cast<size_t>(a.hkv) * bm_words;
    p.bm_words = bm_words;
    p.tile_lists = lists;
    p.list_stride = list_stride;

    const uint32_t box[3] = {64, kBlock, 1};
    const uint64_t dg[3] = {kHeadDim, (uint64_t)kvcap, (uint64_t)a.hkv};
    const uint64_t sg[2] = {kHeadDim * 2, (uint64_t)kvcap * kHeadDim * 2};
    if (!vsp_host::make_map_bf16(&p.map_kv, kg, 3, dg, sg, box) ||
        !vsp_host::make_map_bf16(&p.map_vv, vg, 3, dg, sg, box))
        return cudaErrorInvalidValue;

    if (phase & 1) {
        PrepArgs pa{};
        pa.iv = s.iv;
        pa.kv = s.kv;
        pa.is = s.is;
        pa.ks = s.ks;
        pa.cap = s.cap;
        pa.n = a.n;
        pa.bm_words = bm_words;
        pa.hkv = a.hkv;
        pa.kvcap = kvcap;
        pa.num_qb = num_qb;
        pa.list_stride = list_stride;
        pa.g0 = g0;
        pa.nbw = (bm_words + 127) / 128;
        pa.ngb = std::max(1, std::min(kvcap / 8, 256));
        pa.dense_switch = s.dense_switch ? 1 : 0;
        pa.vbits = bits;
        pa.sbits = bits + static_cast<size_t>(a.hkv) * bm_words;
        pa.k = static_cast<const __nv_bfloat16*>(a.k);
        pa.v = static_cast<const __nv_bfloat16*>(a.v);
        pa.kg = kg;
        pa.vg = vg;
        pa.lists = lists;
        pa.work = work;
        vsp_detail::count_launch();
        vs_prep_kernel<<<dim3(2 * pa.nbw + pa.ngb + (num_qb + 3) / 4, count), 128, 0, stream>>>(pa);
    }
    if ((phase & 2) && nunits > 0) {
        // one launch over all units: table (KV head, qb_lo, qb_hi, qb prefix) in the workspace
        if (nunits > kMaxUnits) return cudaErrorInvalidValue;
        std::vector<int> tab(static_cast<size_t>(nunits) * 4);
        int total = 0;
        for (int u = 0; u < nunits; ++u) {
            const int lo = std::max(host_units[3 * u + 1], 0), hi = std::min(host_units[3 * u + 2], num_qb);
            tab[4 * u] = host_units[3 * u];
            tab[4 * u + 1] = lo;
            tab[4 * u + 2] = hi;
            tab[4 * u + 3] = total;
            total += std::max(hi - lo, 0);
        }
        if (total == 0) return cudaGetLastError();
        cudaError_t e = cudaMemcpyAsync(uwork + 2, tab.data(), tab.size() * sizeof(int), cudaMemcpyHostToDevice, stream);
        if (e == cudaSuccess) e = cudaMemsetAsync(uwork, 0, 2 * sizeof(int), stream);
        if (e != cudaSuccess) return e;
        p.units = uwork + 2;
        p.nunits = nunits;
        p.pair0 = 0;
        p.npairs = (a.hq / a.hkv + 1) / 2;  // the pairs of one KV group
        p.qb_hi = 0;
        p.work = uwork;
        return launch_attn<true>(p, total, stream);
    }
    if (phase & 2) {
        const int pairs_per_group = (a.hq / a.hkv + 1) / 2;
        p.pair0 = g0 * pairs_per_group;
        p.npairs = count * pairs_per_group;
        // query blocks [qb_lo, qb_hi) only (a balanced work unit of a multi-GPU split)
        p.qb_hi = qb_hi < 0 ? num_qb : std::min(qb_hi, num_qb);
        const int nqb = p.qb_hi - std::max(qb_lo, 0);
        if (nqb <= 0) return cudaGetLastError();
        p.work = work + 2 * g0;  // launches on different KV-head ranges never share a counter
        cudaError_t e = launch_attn<true>(p, nqb, stream);
        if (e != cudaSuccess) return e;
    }
    return cudaGetLastError();
}
}  // namespace

cudaError_t launch_sparse(const AttnArgs& a, const SparseArgs& s, void* workspace, cudaStream_t stream, int g0,
                          int count, int phase, int qb_lo, int qb_hi) {
    return launch_sparse_impl(a, s, workspace, stream, g0, count, phase, qb_lo, qb_hi, nullptr, 0);
}

cudaError_t launch_sparse_units(const AttnArgs& a, const SparseArgs& s, void* workspace, cudaStream_t stream,
                                const int* host_units, int nunits) {
    return launch_sparse_impl(a, s, workspace, stream, 0, a.hkv, 2, 0, -1, host_units, nunits);
}

}  // namespace vsp_attn

#ifdef VSP_K3_TRACE
extern "C" __attribute__((visibility("default"))) int vsp_k3_trace_read(void* host, size_t bytes) {
    return static_cast<int>(cudaMemcpyFromSymbol(host, vsp_attn::g_k3_trace, bytes));
}
#endif

namespace vsp_attn {

// per-KV-head sums of the tile-list lengths; grid (hkv), out[g] += count
__global__ void tile_stats_kernel(const int* lists, int num_qb, int list_stride, unsigned long long* out) {
    const int g = blockIdx.x;
    unsigned long long s = 0;
    for (int t = threadIdx.x; t < num_qb; t += blockDim.x)
        s += static_cast<unsigned long long>(lists[(static_cast<size_t>(g) * num_qb + t) * list_stride]);
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0) atomicAdd(out + g, s);
}

// tiles_out: [0] total tiles, [1] dense tiles, [2 + g] tiles of KV head g
cudaError_t sparse_tile_stats(int n, int hkv, int cap, const void* workspace, long long* tiles_out,
                              cudaStream_t stream) {
    const int num_qb = (n + kBlock - 1) / kBlock;
    const int kvcap = ((cap + kBlock - 1) / kBlock) * kBlock;
    const int bm_words = (n + 31) / 32 + 1;
    const int list_stride = 2 + kvcap / kBlock + num_qb + 3;
    size_t off = 0;
    auto skip = [&](size_t b) { off += (b + 255) & ~size_t(255); };
    skip(static_cast<size_t>(hkv) * kvcap * kHeadDim * 2);
    skip(static_cast<size_t>(hkv) * kvcap * kHeadDim * 2);
    skip(static_cast<size_t>(hkv) * bm_words * 4 * 2);
    const int* lists = reinterpret_cast<const int*>(static_cast<const uint8_t*>(workspace) + off);
    unsigned long long* d = nullptr;
    cudaError_t e = cudaMallocAsync(&d, sizeof(unsigned long long) * hkv, stream);
    if (e != cudaSuccess) return e;
    cudaMemsetAsync(d, 0, sizeof(unsigned long long) * hkv, stream);
    vsp_detail::count_launch();
    tile_stats_kernel<<<hkv, 256, 0, stream>>>(lists, num_qb, list_stride, d);
    std::vector<unsigned long long> h(hkv);
    cudaMemcpyAsync(h.data(), d, sizeof(unsigned long long) * hkv, cudaMemcpyDeviceToHost, stream);
    cudaFreeAsync(d, stream);
    e = cudaStreamSynchronize(stream);
    long long total = 0;
    for (int g = 0; g < hkv; ++g) {
        tiles_out[2 + g] = static_cast<long long>(h[g]);
        total += static_cast<long long>(h[g]);
    }
    tiles_out[0] = total;
    tiles_out[1] = static_cast<long long>(hkv) * num_qb * (num_qb + 1) / 2;
    return e;
}

}  // namespace vsp_attn
