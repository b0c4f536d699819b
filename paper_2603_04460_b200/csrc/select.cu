// select.cu — K2: adaptive cumulative-threshold budget + top-k selection on sm_100a.
//
// Replaces vsp::select_pattern (reference sparsity.hpp:105-114) per KV head:
//   k_d = cumulative_budget(A_d, tau_d)   (:51-79)  smallest k whose sorted-descending
//         prefix mass reaches tau - 1e-12, clamped to [min_budget, max_budget ^ n]
//   I_d = topk_indices(A_d, k_d)          (:83-97)  value desc, ties to the lower index,
//         output ascending
//   inject_offset_zero(I_s)               (:99-101)
//
// One 6-CTA thread-block cluster per (head, direction) (8-CTA clusters did not all fit on the
// GPCs at once — half of them ran in a second wave; 6 fit three per GPC, and 4 leave SMs idle:
// 128k select 83 / 58 / 72 us for 8 / 6 / 4); each CTA owns a contiguous sixth of
// the n scores, keeps it in shared memory for all passes, the CTAs exchange their radix
// histograms through distributed shared memory and every CTA takes the same decisions.
// On the layer path the kernel starts from the indexer's logits and performs the softmax
// itself (cluster-wide max and fp64 normaliser, indexer.hpp:110-111), writing A_v / A_s as
// it goes; the standalone softmax kernel for vsp_indexer_scores runs the same code, so both
// paths produce bit-identical scores. No sort on the fast path:
//   1. mass radix-select: 4 MSB-first passes over the fp32 bit pattern (non-negative floats
//      order like their bits). Per-warp private histograms of (count, mass) where mass is
//      u64 fixed point x*2^62 (exact to 2^-62 per element, deterministic integer sums);
//      the lanes of a warp that share the warp's most common buckets are merged with
//      full-warp reductions first, so the concentrated score distributions of real layers
//      do not serialise on one bucket (match.any grouping measured 2x slower).
//      The crossing value v*, the count and mass strictly above it give k. The first pass
//      also performs the reference's score validation.
//   2. exactness guard: the reference sums the sorted doubles sequentially in f64. If our
//      exact prefix masses at k-1 and k sit farther from the threshold than the worst-case
//      f64 rounding of that sequential sum, k is provably identical. Otherwise (rare: the
//      crossing lands within ~1e-11 of tau) the CTA falls back to the reference algorithm
//      verbatim: bitonic sort of the scores in scratch, then a sequential f64 sum.
//   3. only when min/max clamping or the fallback moved k: count radix-select for the k-th
//      largest value T (otherwise T = v* and the ties to take follow from pass 1).
//   4. ordered compaction: per-CTA and per-warp counts of elements above T and equal to T
//      are known from the radix passes (the histogram loops walk the same warp-contiguous
//      runs), so each warp writes its run's indices ascending at its own offset with ballot
//      prefixes, ties to T lowest index first; offset 0 is injected for slash.
#include <cuda_runtime.h>

#include <cooperative_groups.h>
#include <cstdint>

#include "vsp_launch.h"
#include "select.h"

namespace vsp_select_k {

namespace cg = cooperative_groups;

#ifndef VSP_SELECT_CLUSTER
#define VSP_SELECT_CLUSTER 6  // 6-CTA clusters: all 16 co-resident (3 per GPC); 8 did not fit
#endif
constexpr int kCluster = VSP_SELECT_CLUSTER;
constexpr int kThreads = 512;
constexpr int kWarps = kThreads / 32;
constexpr int kMergeRounds = 2;
constexpr int kMaxHeads = 128;
constexpr uint32_t kNoBucket = 256u;
constexpr double kFixScale = 4611686018427387904.0;  // 2^62
constexpr int kMaxCachedSlice = 36864;                 // floats of one CTA's slice kept in smem

struct Params {
    const float* a[2];       // a_v, a_s  [hkv, n] (scores; written here when from logits)
    const float* logits[2];  // null, or logits_v / logits_s [hkv, n] to softmax first
    int* idx[2];             // i_v, i_s  [hkv, cap]
    int* cnt[2];             // k_v, k_s  [hkv]
    uint32_t* scratch;       // [2*hkv, 2 * npow2]
    int* status;             // [2*hkv]: 0 ok, 1 negative score, 2 sum != 1
    int n, hkv, cap, npow2;
    int g0;  // first KV head of this launch
    double tau[2][kMaxHeads];
    long long min_b[kMaxHeads];
    long long max_b[kMaxHeads];
};

// What one CTA publishes to its cluster per exchange step (double-buffered by step parity).
struct Exchange {
    uint32_t c[256];
    unsigned long long m[256];
    double sum;
    float mx;
    int bad, big;
    long long k;  // fallback result (rank 0)
};

struct Shared {
    uint32_t hc[kWarps][256];
    unsigned long long hm[kWarps][256];
    Exchange ex[2];
    uint32_t tc[256];            // cluster-wide histogram of the current pass
    unsigned long long tm[256];
    uint32_t loc[kCluster][256]; // per-rank counts of the current pass
    uint32_t rank_above[kCluster];
    uint32_t rank_eq[kCluster];
    uint32_t warp_gt[kWarps], warp_eq[kWarps];  // compaction: per-warp counts > T and == T
    unsigned long long red[kWarps];
    double red_d[kWarps];
    float red_f[kWarps];
    int found;
    int bad, big;
    uint32_t x0;  // bits of score 0 (slash offset 0)
    long long base_pos, eq_base;
};

#ifdef VSP_SELECT_TRACE
// Phase probe (tools/k2_trace.py builds a separate library with -DVSP_SELECT_TRACE): globaltimer
// stamps of every CTA's phase boundaries, [cta][event].
constexpr int kTraceEvents = 18;  // events: clock64; 16, 17: globaltimer at start / end
__device__ unsigned long long g_k2_trace[4096 * kTraceEvents];
#define VSP_K2_TRACE(ev)                                                                                 \
    do {                                                                                                 \
        if (threadIdx.x == 0) {                                                                          \
            const unsigned long long t_ = clock64();                                                     \
            g_k2_trace[((blockIdx.y * gridDim.x) + blockIdx.x) * kTraceEvents + (ev)] = t_;              \
        }                                                                                                \
    } while (0)
__device__ unsigned long long g_k2_scan[4096 * 8];
#define VSP_K2_SCAN(ev)                                                                                  \
    do {                                                                                                 \
        if (threadIdx.x == 0) g_k2_scan[((blockIdx.y * gridDim.x) + blockIdx.x) * 8 + (ev)] = clock64();  \
    } while (0)
#else
#define VSP_K2_SCAN(ev) \
    do {                \
    } while (0)
#define VSP_K2_TRACE(ev) \
    do {                 \
    } while (0)
#endif

__device__ __forceinline__ unsigned long long to_fix(float x) {
    // inputs are validated scores in [0, 1]; clamp keeps invalid ones from overflowing 2^64
    // (an integer-shift version from the bit pattern measured slower: branchy on this part)
    return static_cast<unsigned long long>(__float2ull_rz(fminf(x, 2.0f) * 4611686018427387904.0f));
}

__device__ __forceinline__ int slice_of(int n, int rank, int& lo, int& hi) {
    const int slice = (n + kCluster - 1) / kCluster;
    lo = min(n, rank * slice);
    hi = min(n, lo + slice);
    return slice;
}

// Cluster-wide softmax of one logit row (indexer.hpp:110-111): max, fp64 sum of exp, and
// the normalised fp32 scores, written to `out` (global) and, when cached, to xs (this CTA's
// slice in shared memory, which also holds the logits on entry). The reduction order is a
// function of (n, thread and cluster shape) only, so every caller gets identical bits.
template <bool kCached>
__device__ void cluster_softmax(Shared& sh, cg::cluster_group& cluster, const float* __restrict__ logits, float* xs,
                                int lo, int hi, float* __restrict__ out, int& parity) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int len = hi - lo;
    auto src = [&](int i) { return kCached ? xs[i] : __ldg(logits + lo + i); };
    // ONE cluster exchange: each CTA publishes its slice's max m_r and fp64 sum
    // s_r = sum exp(x - m_r); the global max is M = max m_r and the normaliser
    // sum_r s_r * exp(m_r - M) (fp64) — the same terms as sum exp(x - M), regrouped per CTA
    float mx = -INFINITY;
    if (kCached) {  // fill this CTA's slice cache from global while taking the max (one pass)
        int i = threadIdx.x;
        for (; i + 3 * kThreads < len; i += 4 * kThreads) {
            const float a = __ldg(logits + lo + i), b = __ldg(logits + lo + i + kThreads),
                        c = __ldg(logits + lo + i + 2 * kThreads), d = __ldg(logits + lo + i + 3 * kThreads);
            xs[i] = a;
            xs[i + kThreads] = b;
            xs[i + 2 * kThreads] = c;
            xs[i + 3 * kThreads] = d;
            mx = fmaxf(mx, fmaxf(fmaxf(a, b), fmaxf(c, d)));
        }
        for (; i < len; i += kThreads) {
            const float a = __ldg(logits + lo + i);
            xs[i] = a;
            mx = fmaxf(mx, a);
        }
        // the next pass reads back only this thread's own elements (same i pattern)
    } else {
        for (int i = threadIdx.x; i < len; i += kThreads) mx = fmaxf(mx, src(i));
    }
    for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if (lane == 0) sh.red_f[warp] = mx;
    __syncthreads();
    float mloc = -INFINITY;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) mloc = fmaxf(mloc, sh.red_f[w]);
    double s = 0.0;
    for (int i = threadIdx.x; i < len; i += kThreads) s += static_cast<double>(expf(src(i) - mloc));
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) sh.red_d[warp] = s;
    __syncthreads();
    Exchange& e1 = sh.ex[parity];
    if (threadIdx.x == 0) {
        double v = 0.0;
        for (int w = 0; w < kWarps; ++w) v += sh.red_d[w];
        e1.mx = mloc;
        e1.sum = v;
    }
    cluster.sync();
    float m = -INFINITY;
    float mr[kCluster];
    double sr[kCluster];
#pragma unroll
    for (int r = 0; r < kCluster; ++r) {
        const Exchange* e = cluster.map_shared_rank(&e1, r);
        mr[r] = e->mx;
        sr[r] = e->sum;
        m = fmaxf(m, mr[r]);
    }
    double tot = 0.0;
#pragma unroll
    for (int r = 0; r < kCluster; ++r)  // fixed rank order: every CTA (and both callers) agree
        if (sr[r] > 0.0) tot += sr[r] * exp(static_cast<double>(mr[r]) - static_cast<double>(m));
    parity ^= 1;
    const double inv = 1.0 / tot;
    if (threadIdx.x == 0) sh.x0 = __float_as_uint(static_cast<float>(static_cast<double>(expf(__ldg(logits) - m)) * inv));
    for (int i = threadIdx.x; i < len; i += kThreads) {
        const float v = static_cast<float>(static_cast<double>(expf(src(i) - m)) * inv);
        if (kCached) xs[i] = v;
        out[lo + i] = v;
    }
    __syncthreads();
}

template <bool kCached>
__device__ void load_slice(float* xs, const float* __restrict__ x, int lo, int hi) {
    const int len = hi - lo;
    int i = threadIdx.x;
    for (; i + 3 * kThreads < len; i += 4 * kThreads) {
        const float a = __ldg(x + lo + i), b = __ldg(x + lo + i + kThreads), c = __ldg(x + lo + i + 2 * kThreads),
                    d = __ldg(x + lo + i + 3 * kThreads);
        xs[i] = a;
        xs[i + kThreads] = b;
        xs[i + 2 * kThreads] = c;
        xs[i + 3 * kThreads] = d;
    }
    for (; i < len; i += kThreads) xs[i] = __ldg(x + lo + i);
    __syncthreads();
}

// Contiguous element run of warp w in a slice of len elements (a multiple of 32 per warp):
// the histogram loops and the compaction use the same runs, so per-warp bucket counts are
// the compaction's per-warp counts.
__device__ __forceinline__ void warp_range(int len, int w, int& w_lo, int& w_hi) {
    const int per_warp = ((len + kWarps - 1) / kWarps + 31) & ~31;
    w_lo = min(len, w * per_warp);
    w_hi = min(len, w_lo + per_warp);
}

// Ordering key of a (validated, non-negative) score: its fp32 bit pattern, with -0.0 folded
// onto +0.0. The reference compares values (sparsity.hpp:83-97), where -0.0 == 0.0 and both
// rank below every positive score; the raw pattern 0x80000000 would rank above them all.
__device__ __forceinline__ uint32_t score_bits(float v) {
    const uint32_t b = __float_as_uint(v);
    return b == 0x80000000u ? 0u : b;
}

// Local histogram of digit (bits >> shift) & 255 over this CTA's slice xs[0, len), restricted
// to elements whose bits above (shift + 8) equal `prefix`, published to ex[parity]; then
// the cluster-wide histogram (tc, tm) and the per-rank counts (loc) are gathered over DSMEM.
// `validate` also records negative/NaN (bad) and > 1.5 (big) scores.
__device__ void cluster_histogram(Shared& sh, cg::cluster_group& cluster, const float* xs, int len, uint32_t prefix,
                                  int shift, bool with_mass, bool validate, int& parity) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int b = lane; b < 256; b += 32) {
        sh.hc[warp][b] = 0;
        sh.hm[warp][b] = 0ull;
    }
    __syncwarp();
    const uint32_t hi_mask = (shift + 8 >= 32) ? 0u : (0xffffffffu << (shift + 8));
    int bad = 0, big = 0;
    // Per-thread two-slot cache of (bucket, count, mass): the elements of one thread mostly
    // fall into a few buckets (scores concentrate in a few exponents), so the loop is
    // lane-independent register work; a miss flushes the oldest slot with shared-memory
    // atomics, and the slots are merged across the warp once at the end.
    auto flush_atomic = [&](uint32_t key, uint32_t cnt, unsigned long long m) {
        atomicAdd(&sh.hc[warp][key], cnt);
        if (with_mass) {
            // 64-bit add as two native 32-bit adds, the carry from the returned low word (a
            // 64-bit shared atomic add is a CAS spin loop on this part)
            uint32_t* h32 = reinterpret_cast<uint32_t*>(&sh.hm[warp][key]);
            const uint32_t lo = static_cast<uint32_t>(m);
            const uint32_t old = atomicAdd(h32, lo);
            const uint32_t hi = static_cast<uint32_t>(m >> 32) + (old + lo < old ? 1u : 0u);
            if (hi) atomicAdd(h32 + 1, hi);
        }
    };
    // lanes sharing the first remaining lane's bucket are merged with full-warp reductions
    // (mass exact: three 21/21/22-bit pieces summed in u32), at most kMergeRounds times; the
    // rest go through flush_atomic
    auto merge_slot = [&](uint32_t key, uint32_t cnt, unsigned long long f) {
        uint32_t rem = __ballot_sync(0xffffffffu, key != kNoBucket);
#pragma unroll
        for (int round = 0; round < kMergeRounds; ++round) {
            if (!rem) break;
            const int src = __ffs(rem) - 1;
            const uint32_t k0 = __shfl_sync(0xffffffffu, key, src);
            const bool mine = key == k0;
            const uint32_t grp = __ballot_sync(0xffffffffu, mine);
            const uint32_t c = __reduce_add_sync(0xffffffffu, mine ? cnt : 0u);
            if (with_mass) {
                const uint32_t s0 = __reduce_add_sync(0xffffffffu, mine ? static_cast<uint32_t>(f & 0x1fffffu) : 0u);
                const uint32_t s1 =
                    __reduce_add_sync(0xffffffffu, mine ? static_cast<uint32_t>((f >> 21) & 0x1fffffu) : 0u);
                const uint32_t s2 = __reduce_add_sync(0xffffffffu, mine ? static_cast<uint32_t>(f >> 42) : 0u);
                if (lane == src)
                    sh.hm[warp][k0] += static_cast<unsigned long long>(s0) + (static_cast<unsigned long long>(s1) << 21) +
                                       (static_cast<unsigned long long>(s2) << 42);
            }
            if (lane == src) sh.hc[warp][k0] += c;
            rem &= ~grp;
            __syncwarp();
        }
        if ((rem >> lane) & 1u) flush_atomic(key, cnt, f);
        __syncwarp();
    };
    constexpr int kSlots = 2;
    constexpr int kBatch = 4;  // elements loaded and keyed together (independent chains), then
                               // folded into the slots
    uint32_t ks[kSlots], cs[kSlots];
    unsigned long long ms[kSlots];
#pragma unroll
    for (int q = 0; q < kSlots; ++q) {
        ks[q] = kNoBucket;
        cs[q] = 0;
        ms[q] = 0;
    }
    // each warp owns a contiguous run of the slice (the compaction's order), lanes interleaved
    int w_lo, w_hi;
    warp_range(len, warp, w_lo, w_hi);
    for (int i0 = w_lo + lane; i0 < w_hi; i0 += kBatch * 32) {
        uint32_t key[kBatch];
        unsigned long long f[kBatch];
#pragma unroll
        for (int u = 0; u < kBatch; ++u) {
            const int i = i0 + u * 32;
            const float v = i < w_hi ? xs[i] : 0.f;
            const uint32_t bits = score_bits(v);
            if (validate && i < w_hi) {
                if (!(v >= 0.f)) bad = 1;
                else if (v > 1.5f) big = 1;
            }
            key[u] = (i < w_hi && (bits & hi_mask) == (prefix & hi_mask)) ? (bits >> shift) & 255u : kNoBucket;
            f[u] = (with_mass && key[u] != kNoBucket) ? to_fix(v) : 0ull;
        }
#pragma unroll
        for (int u = 0; u < kBatch; ++u) {
            if (key[u] == kNoBucket) continue;
            bool hit = false;
#pragma unroll
            for (int q = 0; q < kSlots; ++q) {  // branch-free hit update
                const bool h = key[u] == ks[q];
                cs[q] += h ? 1u : 0u;
                ms[q] += h ? f[u] : 0ull;
                hit |= h;
            }
            if (!hit) {  // miss: flush the oldest slot, shift, take slot 0
                if (ks[kSlots - 1] != kNoBucket) flush_atomic(ks[kSlots - 1], cs[kSlots - 1], ms[kSlots - 1]);
#pragma unroll
                for (int q = kSlots - 1; q > 0; --q) {
                    ks[q] = ks[q - 1];
                    cs[q] = cs[q - 1];
                    ms[q] = ms[q - 1];
                }
                ks[0] = key[u];
                cs[0] = 1;
                ms[0] = f[u];
            }
        }
    }
    if (validate) VSP_K2_TRACE(14);
    __syncwarp();
#pragma unroll
    for (int q = 0; q < kSlots; ++q) merge_slot(ks[q], cs[q], ms[q]);
    if (validate) VSP_K2_TRACE(15);
    if (validate) {
        bad = __syncthreads_or(bad);
        big = __syncthreads_or(big);
    } else {
        __syncthreads();
    }
    if (validate) VSP_K2_TRACE(13);
    Exchange& mine = sh.ex[parity];
    if (threadIdx.x < 256) {
        uint32_t c = 0;
        unsigned long long m = 0;
        for (int w = 0; w < kWarps; ++w) {
            c += sh.hc[w][threadIdx.x];
            m += sh.hm[w][threadIdx.x];
        }
        mine.c[threadIdx.x] = c;
        mine.m[threadIdx.x] = m;
    }
    if (threadIdx.x == 0) {
        mine.bad = bad;
        mine.big = big;
    }
    cluster.sync();
    if (threadIdx.x < 256) {
        uint32_t c = 0;
        unsigned long long m = 0;
#pragma unroll
        for (int r = 0; r < kCluster; ++r) {
            const Exchange* e = cluster.map_shared_rank(&mine, r);
            const uint32_t cr = e->c[threadIdx.x];
            sh.loc[r][threadIdx.x] = cr;
            c += cr;
            if (with_mass) m += e->m[threadIdx.x];
        }
        sh.tc[threadIdx.x] = c;
        sh.tm[threadIdx.x] = m;
    }
    if (validate && threadIdx.x == 0) {
        int b = 0, g = 0;
        for (int r = 0; r < kCluster; ++r) {
            const Exchange* e = cluster.map_shared_rank(&mine, r);
            b |= e->bad;
            g |= e->big;
        }
        sh.bad = b;
        sh.big = g;
    }
    parity ^= 1;
    __syncthreads();
}

// Warp 0 scans buckets from 255 down and finds the first bucket where
// base + cumulative(key) >= target (key = mass if use_mass else count). Returns the bucket
// (or -1) and the totals strictly above it.
__device__ void scan_top(Shared& sh, unsigned long long base, unsigned long long target, bool use_mass,
                         int& bucket, uint32_t& above_cnt, unsigned long long& above_mass) {
    VSP_K2_SCAN(0);
    if (threadIdx.x < 32) {
        const int lane = threadIdx.x;
        // lane L owns buckets 255-8L ... 248-8L (descending)
        unsigned long long seg = 0, segm = 0;
        uint32_t segc = 0;
        for (int t = 0; t < 8; ++t) {
            const int b = 255 - 8 * lane - t;
            seg += use_mass ? sh.tm[b] : sh.tc[b];
            segc += sh.tc[b];
            segm += sh.tm[b];
        }
        unsigned long long pre = seg, prec = segc, prem = segm;
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned long long a = __shfl_up_sync(0xffffffffu, pre, o);
            const unsigned long long ac = __shfl_up_sync(0xffffffffu, prec, o);
            const unsigned long long am = __shfl_up_sync(0xffffffffu, prem, o);
            if (lane >= o) {
                pre += a;
                prec += ac;
                prem += am;
            }
        }
        VSP_K2_SCAN(1);
        pre -= seg;
        prec -= segc;
        prem -= segm;
        int hit = -1;
        unsigned long long run = base + pre, runc = prec, runm = prem;
        unsigned long long hc = 0, hm = 0;
        for (int t = 0; t < 8; ++t) {
            const int b = 255 - 8 * lane - t;
            const unsigned long long key = use_mass ? sh.tm[b] : sh.tc[b];
            if (hit < 0 && run + key >= target && sh.tc[b] > 0) {
                hit = b;
                hc = runc;
                hm = runm;
            }
            run += key;
            runc += sh.tc[b];
            runm += sh.tm[b];
        }
        const unsigned ballot = __ballot_sync(0xffffffffu, hit >= 0);
        const int first = ballot ? __ffs(ballot) - 1 : 0;
        hit = __shfl_sync(0xffffffffu, hit, first);
        hc = __shfl_sync(0xffffffffu, hc, first);
        hm = __shfl_sync(0xffffffffu, hm, first);
        if (lane == 0) {
            sh.found = ballot ? hit : -1;
            sh.red[1] = hc;
            sh.red[2] = hm;
        }
        __syncwarp();
    }
    VSP_K2_SCAN(2);
    __syncthreads();
    VSP_K2_SCAN(3);
    bucket = sh.found;
    above_cnt = bucket >= 0 ? static_cast<uint32_t>(sh.red[1]) : 0;
    above_mass = bucket >= 0 ? sh.red[2] : 0;
    // per-rank counts strictly above the chosen bucket, and (last pass) equal to it; per warp
    // the same from its private histogram (this pass's elements of its run)
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (bucket >= 0) {
        uint32_t s = 0;
        for (int b = bucket + 1 + lane; b < 256; b += 32) s += sh.hc[warp][b];
        s = __reduce_add_sync(0xffffffffu, s);
        if (lane == 0) {
            sh.warp_gt[warp] += s;
            sh.warp_eq[warp] = sh.hc[warp][bucket];
        }
    }
    if (bucket >= 0 && warp < kCluster) {
        uint32_t s = 0;
        for (int b = bucket + 1 + lane; b < 256; b += 32) s += sh.loc[warp][b];
        s = __reduce_add_sync(0xffffffffu, s);
        if (lane == 0) {
            sh.rank_above[warp] += s;
            sh.rank_eq[warp] = sh.loc[warp][bucket];
        }
    }
    VSP_K2_SCAN(4);
    __syncthreads();
    VSP_K2_SCAN(5);
}

template <bool kCached>
__global__ void __cluster_dims__(kCluster, 1, 1) __launch_bounds__(kThreads, 1)
    select_kernel(const __grid_constant__ Params p) {
    extern __shared__ __align__(16) uint8_t smem_raw[];
    Shared& sh = *reinterpret_cast<Shared*>(smem_raw);
    float* cache = reinterpret_cast<float*>(smem_raw + sizeof(Shared));
    cg::cluster_group cluster = cg::this_cluster();
    const int rank = static_cast<int>(cluster.block_rank());

    const int dir = blockIdx.y;
    const int g = p.g0 + static_cast<int>(blockIdx.x) / kCluster;
    const int n = p.n;
    const float* x = p.a[dir] + static_cast<size_t>(g) * n;
    const double tau = p.tau[dir][g];
    int lo, hi;
    slice_of(n, rank, lo, hi);
    VSP_K2_TRACE(0);
#ifdef VSP_SELECT_TRACE
    if (threadIdx.x == 0) {
        unsigned long long t_;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));
        g_k2_trace[((blockIdx.y * gridDim.x) + blockIdx.x) * kTraceEvents + 16] = t_;
    }
#endif
    if (threadIdx.x < kCluster) {
        sh.rank_above[threadIdx.x] = 0;
        sh.rank_eq[threadIdx.x] = 0;
    }
    if (threadIdx.x == 0) {
        sh.bad = 0;
        sh.big = 0;
    }
    if (threadIdx.x < kWarps) {
        sh.warp_gt[threadIdx.x] = 0;
        sh.warp_eq[threadIdx.x] = 0;
    }
    __syncthreads();
    int parity = 0;
    // this CTA's slice of the scores: shared memory when it fits, else global (L2)
    if (p.logits[dir]) {
        const float* lg = p.logits[dir] + static_cast<size_t>(g) * n;
        VSP_K2_TRACE(1);
        cluster_softmax<kCached>(sh, cluster, lg, cache, lo, hi, const_cast<float*>(x), parity);
    } else {
        if (kCached) load_slice<true>(cache, x, lo, hi);
        if (threadIdx.x == 0) sh.x0 = score_bits(__ldg(x));
        __syncthreads();
    }
    const float* xs = kCached ? cache : x + lo;
    const int len = hi - lo;
    VSP_K2_TRACE(2);

    // ---- 1. mass radix-select; pass 0 also validates (sparsity.hpp:60-61)
    const double thr = tau - 1e-12;
    const unsigned long long thr_fx = thr <= 0.0 ? 0ull : static_cast<unsigned long long>(thr * kFixScale);
    uint32_t prefix = 0, cnt_above = 0;
    unsigned long long mass_above = 0, total_fx = 0;
    bool never = false;
    // min >= max clamps k to max whatever the mass says (fixed top-k, sparsity.hpp:75-78): only
    // pass 0 runs (the reference's score checks); the count select reuses its histogram
    long long up0 = n;
    if (p.max_b[g] >= 0 && p.max_b[g] < up0) up0 = p.max_b[g];
    const bool fixed_k = (p.min_b[g] < n ? p.min_b[g] : static_cast<long long>(n)) >= up0;
    for (int pass = 0; pass < 4; ++pass) {
        const int shift = 24 - 8 * pass;
        // per-element score checks only for caller-supplied scores: the logits path's scores
        // come from the softmax above (non-negative, <= 1 by construction); the sum check
        // below uses the histogram's exact total either way
        cluster_histogram(sh, cluster, xs, len, prefix, shift, true, pass == 0 && !p.logits[dir], parity);
        VSP_K2_TRACE(3 + 2 * pass);
        if (pass == 0) {
            if (threadIdx.x < 32) {
                unsigned long long t = 0;
                for (int b = threadIdx.x; b < 256; b += 32) t += sh.tm[b];
                for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
                if (threadIdx.x == 0) sh.red[0] = t;
            }
            __syncthreads();
            total_fx = sh.red[0];
            const double total = static_cast<double>(total_fx) / kFixScale;
            const int st = sh.bad ? 1 : ((sh.big || fabs(total - 1.0) > 1e-6) ? 2 : 0);
            if (rank == 0 && threadIdx.x == 0 && p.status) p.status[dir * p.hkv + g] = st;
            // Invalid scores are reported through `status` (the C ABI raises the reference's
            // error under VSP_VALIDATE); negative/NaN entries have no bit order: empty set.
            if (st == 1) {
                if (rank == 0 && threadIdx.x == 0) p.cnt[dir][g] = 0;
                cluster.sync();  // no CTA leaves while others may still read its histograms
                return;
            }
            if (fixed_k) break;
        }
        int bucket;
        unsigned long long am;
        uint32_t ac;
        scan_top(sh, mass_above, thr_fx, true, bucket, ac, am);
        VSP_K2_TRACE(4 + 2 * pass);
        if (bucket < 0) {
            never = true;
            break;
        }
        prefix |= static_cast<uint32_t>(bucket) << shift;
        cnt_above += ac;
        mass_above += am;
    }
    long long k, need_eq = 0;
    bool ambiguous = false;
    // worst-case |reference sequential f64 sum - our exact fixed-point sum|, doubled
    const double k_err = 2.0 * static_cast<double>(n) * (1.1102230246251565e-16 + 2.168404344971009e-19);
    if (fixed_k) {
        k = up0;
    } else if (never) {
        // the whole vector's mass stays below the threshold: k = n unless that is within
        // rounding of the reference's sequential sum (then the exact fallback decides)
        k = n;
        ambiguous = !(thr - static_cast<double>(total_fx) / kFixScale > k_err);
    } else {
        const float vstar = __uint_as_float(prefix);
        const unsigned long long fv = to_fix(vstar);
        const uint32_t c_eq = sh.tc[prefix & 255u];
        unsigned long long m = 1;
        if (thr_fx > mass_above && fv > 0) m = (thr_fx - mass_above + fv - 1) / fv;
        if (m < 1) m = 1;
        if (m > c_eq) m = c_eq;
        k = static_cast<long long>(cnt_above) + static_cast<long long>(m);
        need_eq = static_cast<long long>(m);
        const double pk = (static_cast<double>(mass_above) + static_cast<double>(m) * static_cast<double>(fv)) / kFixScale;
        const double pk1 = (static_cast<double>(mass_above) + static_cast<double>(m - 1) * static_cast<double>(fv)) / kFixScale;
        ambiguous = !(pk - thr > k_err) || !(k == 1 || thr - pk1 > k_err);
    }

    // ---- 2. exact fallback: the reference algorithm verbatim (sort desc, sequential f64
    // sum), run by rank 0 and broadcast over DSMEM
    if (ambiguous) {
        if (rank == 0) {
            uint32_t* s = p.scratch + static_cast<size_t>(dir * p.hkv + g) * 2 * p.npow2;
            const int np2 = p.npow2;
            // plain loads: on the logits path x was written by this cluster (no .nc cache)
            for (int i = threadIdx.x; i < np2; i += kThreads) s[i] = i < n ? score_bits(x[i]) : 0u;
            __syncthreads();
            for (int size = 2; size <= np2; size <<= 1) {
                for (int stride = size >> 1; stride > 0; stride >>= 1) {
                    for (int t = threadIdx.x; t < np2 / 2; t += kThreads) {
                        const int a_i = 2 * t - (t & (stride - 1));
                        const int b_i = a_i + stride;
                        const bool desc = ((a_i & size) == 0);
                        const uint32_t a = s[a_i], b = s[b_i];
                        if (desc ? (a < b) : (a > b)) {
                            s[a_i] = b;
                            s[b_i] = a;
                        }
                    }
                    __syncthreads();
                }
            }
            if (threadIdx.x == 0) {
                long long kk = n;
                double cum = 0.0;
                for (int i = 0; i < n; ++i) {
                    cum += static_cast<double>(__uint_as_float(s[i]));
                    if (cum >= thr) {
                        kk = i + 1;
                        break;
                    }
                }
                sh.ex[0].k = kk;
            }
        }
        cluster.sync();
        k = cluster.map_shared_rank(&sh.ex[0], 0)->k;
        cluster.sync();
    }

    // clamp (sparsity.hpp:75-78)
    const long long k_mass = k;
    const long long mn = p.min_b[g] < n ? p.min_b[g] : n;
    if (k < mn) k = mn;
    long long upper = n;
    if (p.max_b[g] >= 0 && p.max_b[g] < upper) upper = p.max_b[g];
    if (k > upper) k = upper;

    // ---- 3. count radix-select for the k-th largest value (only if pass 1 does not give it)
    if (fixed_k || never || ambiguous || k != k_mass) {
        if (threadIdx.x < kCluster) sh.rank_above[threadIdx.x] = 0;
        if (threadIdx.x < kWarps) sh.warp_gt[threadIdx.x] = 0;
        __syncthreads();
        prefix = 0;
        uint32_t gt = 0;
        for (int pass = 0; pass < 4; ++pass) {
            const int shift = 24 - 8 * pass;
            // pass 0 of a fixed k: the mass pass's histogram (prefix 0, same digit) is in place
            if (!(fixed_k && pass == 0)) cluster_histogram(sh, cluster, xs, len, prefix, shift, false, false, parity);
            int bucket;
            unsigned long long am;
            uint32_t ac;
            scan_top(sh, gt, static_cast<unsigned long long>(k), false, bucket, ac, am);
            prefix |= static_cast<uint32_t>(bucket) << shift;
            gt += ac;
        }
        need_eq = k - gt;
    }
    const uint32_t tbits = prefix;

    VSP_K2_TRACE(11);
    // ---- 4. ordered compaction: this CTA's offset from the per-rank counts
    if (threadIdx.x == 0) {
        long long pos = 0, eqb = 0;
        for (int r = 0; r < rank; ++r) {
            const long long take = min(static_cast<long long>(sh.rank_eq[r]), max(0ll, need_eq - eqb));
            pos += sh.rank_above[r] + take;
            eqb += sh.rank_eq[r];
        }
        sh.base_pos = pos;
        sh.eq_base = eqb;
    }
    __syncthreads();
    int* out = p.idx[dir] + static_cast<size_t>(g) * p.cap;
    const bool inject = (dir == 1);
    int zero_sel;
    {
        const uint32_t b0 = sh.x0;
        zero_sel = (b0 > tbits) || (b0 == tbits && need_eq > 0);
    }
    const int shift_out = (inject && !zero_sel) ? 1 : 0;
    // Each warp owns a contiguous run of the slice (warp_range) and walks it 32 elements at a
    // time (lane order = index order, conflict-free shared loads); its counts above / equal to
    // T came with the radix passes (scan_top), so positions follow from ballot prefixes.
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t lanes_lt = (1u << lane) - 1u;
    int w_lo, w_hi;
    warp_range(hi - lo, warp, w_lo, w_hi);
    long long eq_run = sh.eq_base, sel_run = sh.base_pos + shift_out;
    for (int w = 0; w < warp; ++w) {  // ties are taken lowest index first across the warps
        const long long take = min(static_cast<long long>(sh.warp_eq[w]), max(0ll, need_eq - eq_run));
        sel_run += sh.warp_gt[w] + take;
        eq_run += sh.warp_eq[w];
    }
    for (int b = w_lo; b < w_hi; b += 32) {
        const int j = b + lane;
        const uint32_t bits = j < w_hi ? score_bits(xs[j]) : 0u;
        const bool gt = j < w_hi && bits > tbits;
        const bool eq = j < w_hi && bits == tbits;
        const uint32_t eqm = __ballot_sync(0xffffffffu, eq);
        const bool take = eq && eq_run + __popc(eqm & lanes_lt) < need_eq;
        const uint32_t selm = __ballot_sync(0xffffffffu, gt || take);
        if (gt || take) out[sel_run + __popc(selm & lanes_lt)] = lo + j;
        eq_run += __popc(eqm);
        sel_run += __popc(selm);
    }
    if (rank == 0 && threadIdx.x == 0) {
        if (shift_out) out[0] = 0;
        p.cnt[dir][g] = static_cast<int>(k) + shift_out;
    }
    VSP_K2_TRACE(12);
    cluster.sync();  // keep this CTA's shared memory alive until the cluster is done with it
    VSP_K2_TRACE(13);
#ifdef VSP_SELECT_TRACE
    if (threadIdx.x == 0) {
        unsigned long long t_;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));
        g_k2_trace[((blockIdx.y * gridDim.x) + blockIdx.x) * kTraceEvents + 17] = t_;
    }
#endif
}

// Standalone cluster softmax of logit rows (vsp_indexer_scores): the same code as the
// layer path's fused softmax, so both produce identical scores. grid (count * 8, 2).
template <bool kCached>
__global__ void __cluster_dims__(kCluster, 1, 1) __launch_bounds__(kThreads, 1)
    softmax_kernel(const float* __restrict__ lv, const float* __restrict__ ls, float* av, float* as, int n, int g0) {
    extern __shared__ __align__(16) uint8_t smem_raw[];
    Shared& sh = *reinterpret_cast<Shared*>(smem_raw);
    float* cache = reinterpret_cast<float*>(smem_raw + sizeof(Shared));
    cg::cluster_group cluster = cg::this_cluster();
    const int rank = static_cast<int>(cluster.block_rank());
    const int g = g0 + static_cast<int>(blockIdx.x) / kCluster;
    const size_t row = static_cast<size_t>(g) * n;
    const float* lg = (blockIdx.y == 0 ? lv : ls) + row;
    float* out = (blockIdx.y == 0 ? av : as) + row;
    int lo, hi;
    slice_of(n, rank, lo, hi);
    int parity = 0;
    cluster_softmax<kCached>(sh, cluster, lg, cache, lo, hi, out, parity);
    cluster.sync();  // keep this CTA's shared memory alive until the cluster is done with it
}

static int next_pow2(int n) {
    int p = 1;
    while (p < n) p <<= 1;
    return p;
}

size_t workspace_bytes(int n, int hkv) {
    return static_cast<size_t>(2 * hkv) * 2 * next_pow2(n) * sizeof(uint32_t) + 2 * hkv * sizeof(int) + 512;
}

namespace {
bool cached_slice(int n) { return (n + kCluster - 1) / kCluster <= kMaxCachedSlice; }
int smem_bytes(int n) {
    return static_cast<int>(sizeof(Shared)) + (cached_slice(n) ? ((n + kCluster - 1) / kCluster) * 4 : 0);
}
template <typename K>
void allow_smem(K kernel) {
    cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(sizeof(Shared)) + kMaxCachedSlice * 4);
}
}  // namespace

cudaError_t launch_impl(const float* lv, const float* ls, const float* a_v, const float* a_s, int n, int hkv,
                        const vsp_budget* budgets, int* i_v, int* k_v, int* i_s, int* k_s, int cap, void* workspace,
                        cudaStream_t stream, int g0, int count) {
    if (hkv > kMaxHeads) return cudaErrorInvalidValue;
    if (count < 0) count = hkv - g0;
    Params p{};  // ~3 KB parameter block, copied into the launch
    p.a[0] = a_v;
    p.a[1] = a_s;
    p.logits[0] = lv;
    p.logits[1] = ls;
    p.idx[0] = i_v;
    p.idx[1] = i_s;
    p.cnt[0] = k_v;
    p.cnt[1] = k_s;
    p.npow2 = next_pow2(n);
    p.scratch = static_cast<uint32_t*>(workspace);
    p.status = reinterpret_cast<int*>(static_cast<uint8_t*>(workspace) +
                                      static_cast<size_t>(2 * hkv) * 2 * p.npow2 * sizeof(uint32_t));
    p.n = n;
    p.hkv = hkv;
    p.cap = cap;
    for (int g = 0; g < hkv; ++g) {
        p.tau[0][g] = budgets[g].tau_v;
        p.tau[1][g] = budgets[g].tau_s;
        p.min_b[g] = budgets[g].min_budget;
        p.max_b[g] = budgets[g].max_budget;
    }
    static std::once_flag attr[vsp_detail::kMaxDevices];
    vsp_detail::once_per_device(attr, [] {
        allow_smem(select_kernel<true>);
        allow_smem(select_kernel<false>);
    });
    p.g0 = g0;
    const dim3 grid(count * kCluster, 2);
    vsp_detail::count_launch();
    if (cached_slice(n))
        select_kernel<true><<<grid, kThreads, smem_bytes(n), stream>>>(p);
    else
        select_kernel<false><<<grid, kThreads, smem_bytes(n), stream>>>(p);
    return cudaGetLastError();
}

cudaError_t launch(const float* a_v, const float* a_s, int n, int hkv, const vsp_budget* budgets, int* i_v,
                   int* k_v, int* i_s, int* k_s, int cap, void* workspace, cudaStream_t stream, int g0, int count) {
    return launch_impl(nullptr, nullptr, a_v, a_s, n, hkv, budgets, i_v, k_v, i_s, k_s, cap, workspace, stream, g0,
                       count);
}

cudaError_t launch_from_logits(const float* lv, const float* ls, float* a_v, float* a_s, int n, int hkv,
                               const vsp_budget* budgets, int* i_v, int* k_v, int* i_s, int* k_s, int cap,
                               void* workspace, cudaStream_t stream, int g0, int count) {
    return launch_impl(lv, ls, a_v, a_s, n, hkv, budgets, i_v, k_v, i_s, k_s, cap, workspace, stream, g0, count);
}

cudaError_t launch_softmax(const float* lv, const float* ls, float* a_v, float* a_s, int n, int g0, int count,
                           cudaStream_t stream) {
    static std::once_flag attr[vsp_detail::kMaxDevices];
    vsp_detail::once_per_device(attr, [] {
        allow_smem(softmax_kernel<true>);
        allow_smem(softmax_kernel<false>);
    });
    const dim3 grid(count * kCluster, 2);
    vsp_detail::count_launch();
    if (cached_slice(n))
        softmax_kernel<true><<<grid, kThreads, smem_bytes(n), stream>>>(lv, ls, a_v, a_s, n, g0);
    else
        softmax_kernel<false><<<grid, kThreads, smem_bytes(n), stream>>>(lv, ls, a_v, a_s, n, g0);
    return cudaGetLastError();
}

const int* status_ptr(void* workspace, int n, int hkv) {
    return reinterpret_cast<const int*>(static_cast<uint8_t*>(workspace) +
                                        static_cast<size_t>(2 * hkv) * 2 * next_pow2(n) * sizeof(uint32_t));
}

}  // namespace vsp_select_k

#ifdef VSP_SELECT_TRACE
extern "C" __attribute__((visibility("default"))) int vsp_k2_trace_read(void* host, size_t bytes) {
    return static_cast<int>(cudaMemcpyFromSymbol(host, vsp_select_k::g_k2_trace, bytes));
}
extern "C" __attribute__((visibility("default"))) int vsp_k2_scan_read(void* host, size_t bytes) {
    return static_cast<int>(cudaMemcpyFromSymbol(host, vsp_select_k::g_k2_scan, bytes));
}
#endif
