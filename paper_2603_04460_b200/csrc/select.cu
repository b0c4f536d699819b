// select.cu — K2: adaptive cumulative-threshold budget + top-k selection on sm_100a.
//
// Replaces vsp::select_pattern (reference sparsity.hpp:105-114) per KV head:
//   k_d = cumulative_budget(A_d, tau_d)   (:51-79)  smallest k whose sorted-descending
//         prefix mass reaches tau - 1e-12, clamped to [min_budget, max_budget ^ n]
//   I_d = topk_indices(A_d, k_d)          (:83-97)  value desc, ties to the lower index,
//         output ascending
//   inject_offset_zero(I_s)               (:99-101)
//
// One CTA (1024 threads) per (head, direction); no sort on the fast path:
//   1. mass radix-select: 4 MSB-first passes over the fp32 bit pattern (non-negative floats
//      order like their bits). Per-warp private histograms of (count, mass) where mass is
//      u64 fixed point x*2^62 (exact to 2^-62 per element, deterministic integer atomics).
//      The crossing value v*, the count and mass strictly above it give k.
//   2. exactness guard: the reference sums the sorted doubles sequentially in f64. If our
//      exact prefix masses at k-1 and k sit farther from the threshold than the worst-case
//      f64 rounding of that sequential sum, k is provably identical. Otherwise (rare: the
//      crossing lands within ~1e-11 of tau) the CTA falls back to the reference algorithm
//      verbatim: bitonic sort of the scores in scratch, then a sequential f64 sum.
//   3. count radix-select for the k-th largest value T and the number of ties to take.
//   4. ordered compaction (two block scans per 8192-element chunk) writes indices ascending,
//      taking equal-to-T elements lowest index first; offset 0 is injected for slash.
#include <cuda_runtime.h>

#include <cstdint>

#include "select.h"

namespace vsp_select_k {

constexpr int kThreads = 1024;
constexpr int kWarps = kThreads / 32;
constexpr int kItems = 8;
constexpr int kMaxHeads = 128;
constexpr double kFixScale = 4611686018427387904.0;  // 2^62

struct Params {
    const float* a[2];  // a_v, a_s  [hkv, n]
    int* idx[2];        // i_v, i_s  [hkv, cap]
    int* cnt[2];        // k_v, k_s  [hkv]
    uint32_t* scratch;  // [2*hkv, 2 * npow2]
    int* status;        // [2*hkv]: 0 ok, 1 negative score, 2 sum != 1
    int n, hkv, cap, npow2;
    int g0;  // first KV head of this launch
    double tau[2][kMaxHeads];
    long long min_b[kMaxHeads];
    long long max_b[kMaxHeads];
};

struct Shared {
    uint32_t hc[kWarps][256];
    unsigned long long hm[kWarps][256];
    uint32_t tc[256];
    unsigned long long tm[256];
    uint32_t scan_a[kWarps];
    uint32_t scan_b[kWarps];
    unsigned long long red[kWarps];
    int flag;
    uint32_t prefix;
    uint32_t cnt_above;
    unsigned long long mass_above;
    int found;
    int ambiguous;
    long long k;
};

__device__ __forceinline__ unsigned long long to_fix(float x) {
    // inputs are validated scores in [0, 1]; clamp keeps invalid ones from overflowing 2^64
    return static_cast<unsigned long long>(__float2ull_rz(fminf(x, 2.0f) * 4611686018427387904.0f));
}

// Fill tc/tm with the histogram of digit (bits >> shift) & 255 over elements whose bits
// above (shift + 8) equal `prefix`. with_mass = false skips the mass atomics.
__device__ void histogram(Shared& sh, const float* __restrict__ x, int n, uint32_t prefix, int shift, bool with_mass) {
    const int warp = threadIdx.x >> 5;
    for (int b = threadIdx.x & 31; b < 256; b += 32) {
        sh.hc[warp][b] = 0;
        sh.hm[warp][b] = 0ull;
    }
    __syncthreads();
    const uint32_t hi_mask = (shift + 8 >= 32) ? 0u : (0xffffffffu << (shift + 8));
    for (int i = threadIdx.x; i < n; i += kThreads) {
        const float v = __ldg(x + i);
        const uint32_t bits = __float_as_uint(v);
        if ((bits & hi_mask) == (prefix & hi_mask)) {
            const uint32_t b = (bits >> shift) & 255u;
            atomicAdd(&sh.hc[warp][b], 1u);
            if (with_mass) atomicAdd(&sh.hm[warp][b], to_fix(v));
        }
    }
    __syncthreads();
    if (threadIdx.x < 256) {
        uint32_t c = 0;
        unsigned long long m = 0;
        for (int w = 0; w < kWarps; ++w) {
            c += sh.hc[w][threadIdx.x];
            m += sh.hm[w][threadIdx.x];
        }
        sh.tc[threadIdx.x] = c;
        sh.tm[threadIdx.x] = m;
    }
    __syncthreads();
}

// Warp 0 scans buckets from 255 down and finds the first bucket where
// base + cumulative(key) >= target (key = mass if use_mass else count). Writes found bucket
// (or -1) and the totals strictly above it into sh.
__device__ void scan_top(Shared& sh, unsigned long long base, unsigned long long target, bool use_mass,
                         int& bucket, unsigned long long& above_key, uint32_t& above_cnt, unsigned long long& above_mass) {
    if (threadIdx.x < 32) {
        const int lane = threadIdx.x;
        // lane L owns buckets 255-8L ... 248-8L (descending)
        unsigned long long seg = 0;
        uint32_t segc = 0;
        unsigned long long segm = 0;
        for (int t = 0; t < 8; ++t) {
            const int b = 255 - 8 * lane - t;
            seg += use_mass ? sh.tm[b] : sh.tc[b];
            segc += sh.tc[b];
            segm += sh.tm[b];
        }
        // exclusive prefix over lanes
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
        pre -= seg;
        prec -= segc;
        prem -= segm;
        int hit = -1;
        unsigned long long run = base + pre, runc = prec, runm = prem;
        unsigned long long hk = 0, hc = 0, hm = 0;
        for (int t = 0; t < 8; ++t) {
            const int b = 255 - 8 * lane - t;
            const unsigned long long key = use_mass ? sh.tm[b] : sh.tc[b];
            if (hit < 0 && run + key >= target && sh.tc[b] > 0) {
                hit = b;
                hk = run - base;
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
        hk = __shfl_sync(0xffffffffu, hk, first);
        hc = __shfl_sync(0xffffffffu, hc, first);
        hm = __shfl_sync(0xffffffffu, hm, first);
        if (lane == 0) {
            sh.found = ballot ? hit : -1;
            sh.red[0] = hk;
            sh.red[1] = hc;
            sh.red[2] = hm;
        }
        __syncwarp();
    }
    __syncthreads();
    bucket = sh.found;
    above_key = bucket >= 0 ? sh.red[0] : 0;
    above_cnt = bucket >= 0 ? static_cast<uint32_t>(sh.red[1]) : 0;
    above_mass = bucket >= 0 ? sh.red[2] : 0;
    __syncthreads();
}

// Block-wide exclusive scan of one u32 per thread; returns exclusive prefix, total via ref.
__device__ uint32_t block_scan(uint32_t v, uint32_t* buf, uint32_t& total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t inc = v;
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t a = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += a;
    }
    if (lane == 31) buf[warp] = inc;
    __syncthreads();
    if (warp == 0) {
        uint32_t w = buf[lane];
        uint32_t wi = w;
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t a = __shfl_up_sync(0xffffffffu, wi, o);
            if (lane >= o) wi += a;
        }
        buf[lane] = wi - w;
        if (lane == 31) buf[32 + 0] = wi;  // stash total just past the warp slots (buf has >= 33)
    }
    __syncthreads();
    const uint32_t res = buf[warp] + inc - v;
    total = buf[32];
    __syncthreads();
    return res;
}

__global__ void __launch_bounds__(kThreads, 1) select_kernel(const __grid_constant__ Params p) {
    extern __shared__ __align__(16) uint8_t smem_raw[];
    Shared& sh = *reinterpret_cast<Shared*>(smem_raw);
    uint32_t* scanbuf = reinterpret_cast<uint32_t*>(smem_raw + sizeof(Shared));  // 64 words

    const int dir = blockIdx.y;
    const int g = p.g0 + static_cast<int>(blockIdx.x);
    const int n = p.n;
    const float* x = p.a[dir] + static_cast<size_t>(g) * n;
    const double tau = p.tau[dir][g];

    // ---- validation (sparsity.hpp:60-61): non-negative, sum within 1e-6 of 1
    {
        int bad = 0, big = 0;
        unsigned long long s = 0;
        for (int i = threadIdx.x; i < n; i += kThreads) {
            const float v = __ldg(x + i);
            if (!(v >= 0.f)) bad = 1;       // negative or NaN
            else if (v > 1.5f) big = 1;     // cannot sum to 1 without negatives
            else s += to_fix(v);
        }
        bad = __syncthreads_or(bad);
        big = __syncthreads_or(big);
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if ((threadIdx.x & 31) == 0) sh.red[threadIdx.x >> 5] = s;
        __syncthreads();
        if (threadIdx.x == 0) {
            unsigned long long t = 0;
            for (int w = 0; w < kWarps; ++w) t += sh.red[w];
            const double total = static_cast<double>(t) / kFixScale;
            int st = 0;
            if (bad) st = 1;
            else if (big || fabs(total - 1.0) > 1e-6) st = 2;
            sh.flag = st;
            if (p.status) p.status[dir * p.hkv + g] = st;
        }
        __syncthreads();
        // Invalid scores are reported through `status` (the C ABI raises the reference's
        // error under VSP_VALIDATE); without validation the selection still runs on them.
        if (sh.flag == 1) {  // negative/NaN entries have no meaningful bit order: empty set
            if (threadIdx.x == 0) p.cnt[dir][g] = 0;
            return;
        }
    }

    // ---- 1. mass radix-select
    const double thr = tau - 1e-12;
    const unsigned long long thr_fx =
        thr <= 0.0 ? 0ull : static_cast<unsigned long long>(thr * kFixScale);
    uint32_t prefix = 0, cnt_above = 0;
    unsigned long long mass_above = 0;
    bool never = false;
    for (int pass = 0; pass < 4; ++pass) {
        const int shift = 24 - 8 * pass;
        histogram(sh, x, n, prefix, shift, true);
        int bucket;
        unsigned long long ak, am;
        uint32_t ac;
        scan_top(sh, mass_above, thr_fx, true, bucket, ak, ac, am);
        if (bucket < 0) {
            never = true;
            break;
        }
        prefix |= static_cast<uint32_t>(bucket) << shift;
        cnt_above += ac;
        mass_above += am;
    }
    long long k;
    bool ambiguous = false;
    // worst-case |reference sequential f64 sum - our exact fixed-point sum|, doubled
    const double k_err = 2.0 * static_cast<double>(n) * (1.1102230246251565e-16 + 2.168404344971009e-19);
    if (never) {
        // the whole vector's mass stays below the threshold: k = n unless that is within
        // rounding of the reference's sequential sum (then the exact fallback decides)
        k = n;
        unsigned long long t = 0;
        for (int i = threadIdx.x; i < n; i += kThreads) t += to_fix(__ldg(x + i));
        for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
        if ((threadIdx.x & 31) == 0) sh.red[threadIdx.x >> 5] = t;
        __syncthreads();
        unsigned long long tt = 0;
        for (int w = 0; w < kWarps; ++w) tt += sh.red[w];
        __syncthreads();
        const double total = static_cast<double>(tt) / kFixScale;
        ambiguous = !(thr - total > k_err);
    } else {
        const float vstar = __uint_as_float(prefix);
        const unsigned long long fv = to_fix(vstar);
        const uint32_t c_eq = sh.tc[prefix & 255u];
        unsigned long long m = 1;
        if (thr_fx > mass_above && fv > 0) m = (thr_fx - mass_above + fv - 1) / fv;
        if (m < 1) m = 1;
        if (m > c_eq) m = c_eq;
        k = static_cast<long long>(cnt_above) + static_cast<long long>(m);
        const double pk = (static_cast<double>(mass_above) + static_cast<double>(m) * static_cast<double>(fv)) / kFixScale;
        const double pk1 = (static_cast<double>(mass_above) + static_cast<double>(m - 1) * static_cast<double>(fv)) / kFixScale;
        ambiguous = !(pk - thr > k_err) || !(k == 1 || thr - pk1 > k_err);
    }

    // ---- 2. exact fallback: the reference algorithm verbatim (sort desc, sequential f64 sum)
    if (ambiguous) {
        uint32_t* s = p.scratch + static_cast<size_t>(dir * p.hkv + g) * 2 * p.npow2;
        const int np2 = p.npow2;
        for (int i = threadIdx.x; i < np2; i += kThreads) s[i] = i < n ? __float_as_uint(__ldg(x + i)) : 0u;
        __syncthreads();
        // bitonic sort, descending (non-negative float bits order like values)
        for (int size = 2; size <= np2; size <<= 1) {
            for (int stride = size >> 1; stride > 0; stride >>= 1) {
                for (int t = threadIdx.x; t < np2 / 2; t += kThreads) {
                    const int lo = 2 * t - (t & (stride - 1));
                    const int hi = lo + stride;
                    const bool desc = ((lo & size) == 0);
                    const uint32_t a = s[lo], b = s[hi];
                    if (desc ? (a < b) : (a > b)) {
                        s[lo] = b;
                        s[hi] = a;
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
            sh.k = kk;
        }
        __syncthreads();
        k = sh.k;
    }

    // clamp (sparsity.hpp:75-78)
    const long long mn = p.min_b[g] < n ? p.min_b[g] : n;
    if (k < mn) k = mn;
    long long upper = n;
    if (p.max_b[g] >= 0 && p.max_b[g] < upper) upper = p.max_b[g];
    if (k > upper) k = upper;

    // ---- 3. count radix-select for the k-th largest value
    prefix = 0;
    uint32_t gt = 0;  // count strictly greater than the current prefix range
    for (int pass = 0; pass < 4; ++pass) {
        const int shift = 24 - 8 * pass;
        histogram(sh, x, n, prefix, shift, false);
        int bucket;
        unsigned long long ak, am;
        uint32_t ac;
        scan_top(sh, gt, static_cast<unsigned long long>(k), false, bucket, ak, ac, am);
        prefix |= static_cast<uint32_t>(bucket) << shift;
        gt += ac;
    }
    const uint32_t tbits = prefix;
    const long long need_eq = k - gt;

    // ---- 4. ordered compaction
    int* out = p.idx[dir] + static_cast<size_t>(g) * p.cap;
    const bool inject = (dir == 1);
    // is index 0 selected? (needed up front to shift the slash list by one)
    int zero_sel;
    {
        const uint32_t b0 = __float_as_uint(__ldg(x));
        zero_sel = (b0 > tbits) || (b0 == tbits && need_eq > 0);
    }
    const int shift_out = (inject && !zero_sel) ? 1 : 0;
    uint32_t sel_base = 0, eq_base = 0;
    const int chunk = kThreads * kItems;
    for (int c0 = 0; c0 < n; c0 += chunk) {
        const int i0 = c0 + threadIdx.x * kItems;
        uint32_t bits[kItems];
        uint32_t n_eq = 0;
#pragma unroll
        for (int t = 0; t < kItems; ++t) {
            const int i = i0 + t;
            bits[t] = i < n ? __float_as_uint(__ldg(x + i)) : 0u;
            n_eq += (i < n && bits[t] == tbits) ? 1u : 0u;
        }
        uint32_t eq_tot;
        uint32_t eq_pre = block_scan(n_eq, scanbuf, eq_tot) + eq_base;
        uint32_t n_sel = 0;
        uint32_t flags = 0;
#pragma unroll
        for (int t = 0; t < kItems; ++t) {
            const int i = i0 + t;
            bool s = false;
            if (i < n) {
                if (bits[t] > tbits) s = true;
                else if (bits[t] == tbits) {
                    s = static_cast<long long>(eq_pre) < need_eq;
                    ++eq_pre;
                }
            }
            flags |= (s ? 1u : 0u) << t;
            n_sel += s ? 1u : 0u;
        }
        uint32_t sel_tot;
        uint32_t pos = block_scan(n_sel, scanbuf, sel_tot) + sel_base + shift_out;
#pragma unroll
        for (int t = 0; t < kItems; ++t)
            if ((flags >> t) & 1u) out[pos++] = i0 + t;
        sel_base += sel_tot;
        eq_base += eq_tot;
    }
    if (threadIdx.x == 0) {
        if (shift_out) out[0] = 0;
        p.cnt[dir][g] = static_cast<int>(k) + shift_out;
    }
}

static int next_pow2(int n) {
    int p = 1;
    while (p < n) p <<= 1;
    return p;
}

size_t workspace_bytes(int n, int hkv) {
    return static_cast<size_t>(2 * hkv) * 2 * next_pow2(n) * sizeof(uint32_t) + 2 * hkv * sizeof(int) + 512;
}

cudaError_t launch(const float* a_v, const float* a_s, int n, int hkv, const vsp_budget* budgets, int* i_v,
                   int* k_v, int* i_s, int* k_s, int cap, void* workspace, cudaStream_t stream, int g0, int count) {
    if (hkv > kMaxHeads) return cudaErrorInvalidValue;
    if (count < 0) count = hkv - g0;
    Params p{};  // ~3 KB parameter block, copied into the launch
    p.a[0] = a_v;
    p.a[1] = a_s;
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
    const int smem = static_cast<int>(sizeof(Shared)) + 64 * sizeof(uint32_t);
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(select_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        attr = true;
    }
    p.g0 = g0;
    select_kernel<<<dim3(count, 2), kThreads, smem, stream>>>(p);
    return cudaGetLastError();
}

const int* status_ptr(void* workspace, int n, int hkv) {
    return reinterpret_cast<const int*>(static_cast<uint8_t*>(workspace) +
                                        static_cast<size_t>(2 * hkv) * 2 * next_pow2(n) * sizeof(uint32_t));
}

}  // namespace vsp_select_k
