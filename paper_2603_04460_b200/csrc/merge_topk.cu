// merge_topk.cu — the standalone operators of the reference's selection/merge layer that the
// fused layer path (K2 select, K3 plan) does not expose on their own:
//
//   * merge_path_partition (merge.hpp:69-95)  -> vsp_misc::merge_path_search, host + device
//   * merge_row_columns    (merge.hpp:18-56)  -> merge_rows_kernel: one CTA per query row; the
//     row's two ascending lists (verticals <= i, slash columns i - o for offsets o <= i) are
//     cut into per-thread slices by merge path (the spec the reference gives for a parallel
//     merge), each thread merges its slice, and a block scan places the
//     duplicate-free union
//   * topk_indices         (sparsity.hpp:83-97) -> topk_kernel: general-value top-k per row
//     (any sign), MSB-first radix select on an order-preserving key, ties to the lower index,
//     ascending output
//   * combine_scores       (vsaggregate.hpp:133-157) -> combine_kernel: group mean / sum
//
// None of these is on the timed layer path; they make the reference's free functions
// callable on device data with the reference's semantics (tests: test_gpu_misc_ops.py,
// tests/cpp/shim_test.cpp).
#include <cuda_runtime.h>

#include <cstdint>

#include "misc_ops.h"
#include "vsp_launch.h"

namespace vsp_misc {
namespace {

constexpr int kMergeThreads = 256;
constexpr int kTopkThreads = 1024;

// Exclusive block scan of one int per thread; returns the prefix, writes the block total.
// `warp_sums` holds blockDim.x / 32 ints of shared memory. Ends with a __syncthreads.
__device__ int block_exclusive_scan(int x, int* warp_sums, int& total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
    int incl = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
    }
    if (lane == 31) warp_sums[warp] = incl;
    __syncthreads();
    if (warp == 0) {
        int w = lane < nwarps ? warp_sums[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, w, o);
            if (lane >= o) w += y;
        }
        if (lane < nwarps) warp_sums[lane] = w;  // inclusive over warps
    }
    __syncthreads();
    const int before = warp ? warp_sums[warp - 1] : 0;
    total = warp_sums[nwarps - 1];
    __syncthreads();
    return before + incl - x;
}

// Number of entries <= x in an ascending list.
__device__ int upper_bound(const int* a, int len, int x) {
    int lo = 0, hi = len;
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (a[mid] <= x) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

struct RowLists {
    const int* iv;  // verticals, ascending; A[t] = iv[t], t < na (the verticals <= i)
    const int* is;  // offsets, ascending; B[t] = i - is[nb - 1 - t], t < nb (offsets <= i)
    int na, nb, i;
    __device__ int a(long long t) const { return iv[t]; }
    __device__ int b(long long t) const { return i - is[nb - 1 - t]; }
};

// merge_path_search over the row's virtual B list (same search as merge.hpp:69-95).
__device__ int row_search(const RowLists& L, int diag) {
    int lo = diag > L.nb ? diag - L.nb : 0, hi = diag < L.na ? diag : L.na;
    while (lo < hi) {
        const int mid = lo + ((hi - lo) >> 1);
        if (L.a(mid) <= L.b(diag - mid - 1)) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

// Walks merged positions [d0, d1) (a-first ties); emit(col) for every column of the union:
// an A entry always, a B entry only when it is not also a vertical (the collapse of
// merge.hpp:49-53 — with a-first ties the equal A entry precedes it).
template <class F>
__device__ void walk(const RowLists& L, int d0, int d1, F&& emit) {
    int ai = row_search(L, d0), bi = d0 - ai;
    for (int d = d0; d < d1; ++d) {
        const bool take_a = bi >= L.nb || (ai < L.na && L.a(ai) <= L.b(bi));
        if (take_a) {
            emit(L.a(ai));
            ++ai;
        } else {
            const int c = L.b(bi);
            if (!(ai > 0 && L.a(ai - 1) == c)) emit(c);
            ++bi;
        }
    }
}

__global__ void __launch_bounds__(kMergeThreads) merge_rows_kernel(const int* i_v, int k_v, const int* i_s, int k_s,
                                                                  const int* rows, int* out, int* out_len,
                                                                  int out_cap, int validate) {
    __shared__ int warp_sums[kMergeThreads / 32];
    const int r = blockIdx.x;
    const int i = rows[r];
    if (validate) {  // the reference re-validates both lists on every call (merge.hpp:21-26)
        int bad_v = 0, bad_s = 0;
        for (int t = threadIdx.x + 1; t < k_v; t += blockDim.x) bad_v |= !(i_v[t - 1] < i_v[t]);
        for (int t = threadIdx.x + 1; t < k_s; t += blockDim.x) bad_s |= !(i_s[t - 1] < i_s[t]);
        bad_v = __syncthreads_or(bad_v);
        bad_s = __syncthreads_or(bad_s);
        if (bad_v || bad_s) {
            if (threadIdx.x == 0) out_len[r] = bad_v ? -1 : -2;
            return;
        }
    }
    RowLists L{i_v, i_s, upper_bound(i_v, k_v, i), upper_bound(i_s, k_s, i), i};
    const int total = L.na + L.nb;
    const int d0 = static_cast<int>(static_cast<long long>(total) * threadIdx.x / blockDim.x);
    const int d1 = static_cast<int>(static_cast<long long>(total) * (threadIdx.x + 1) / blockDim.x);
    int cnt = 0;
    walk(L, d0, d1, [&](int) { ++cnt; });
    int kept = 0;
    int pos = block_exclusive_scan(cnt, warp_sums, kept);
    if (kept > out_cap) {
        if (threadIdx.x == 0) out_len[r] = -3;
        return;
    }
    int* o = out + static_cast<size_t>(r) * out_cap;
    walk(L, d0, d1, [&](int c) { o[pos++] = c; });
    if (threadIdx.x == 0) out_len[r] = kept;
}

// Order-preserving key of an fp32 value (value compare of sparsity.hpp:89-92): -0.0 folds
// onto +0.0, negatives reverse.
__device__ __forceinline__ uint32_t order_key(float x) {
    uint32_t b = __float_as_uint(x);
    if (b == 0x80000000u) b = 0u;
    return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}

__global__ void __launch_bounds__(kTopkThreads) topk_kernel(const float* scores, int n, const int* kk, int* out,
                                                           int cap) {
    __shared__ int hist[256];
    __shared__ int warp_sums[kTopkThreads / 32];
    __shared__ uint32_t sh_prefix;
    __shared__ int sh_remaining;
    const int r = blockIdx.x;
    const float* x = scores + static_cast<size_t>(r) * n;
    const int k = kk[r];
    uint32_t prefix = 0u, mask = 0u;
    int remaining = k;  // how many of the elements matching `prefix` still belong to the top k
    for (int shift = 24; shift >= 0; shift -= 8) {
        for (int b = threadIdx.x; b < 256; b += blockDim.x) hist[b] = 0;
        __syncthreads();
        for (int t = threadIdx.x; t < n; t += blockDim.x) {
            const uint32_t key = order_key(__ldg(x + t));
            if ((key & mask) == prefix) atomicAdd(&hist[(key >> shift) & 255u], 1);
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            int b = 255, rem = remaining;
            for (; b > 0 && hist[b] < rem; --b) rem -= hist[b];
            sh_prefix = prefix | (static_cast<uint32_t>(b) << shift);
            sh_remaining = rem;
        }
        __syncthreads();
        prefix = sh_prefix;
        remaining = sh_remaining;
        mask |= 255u << shift;
        __syncthreads();
    }
    // prefix = key of the k-th largest value; take every larger key and the first
    // `remaining` equal keys in index order (ties to the lower index), ascending
    int base = 0, eq_base = 0;
    int* o = out + static_cast<size_t>(r) * cap;
    for (int c0 = 0; c0 < n; c0 += blockDim.x) {
        const int t = c0 + threadIdx.x;
        const uint32_t key = t < n ? order_key(__ldg(x + t)) : 0u;
        const int gt = t < n && key > prefix, eq = t < n && key == prefix;
        int eq_tot = 0;
        const int eq_rank = block_exclusive_scan(eq, warp_sums, eq_tot) + eq_base;
        const int take = gt || (eq && eq_rank < remaining);
        int take_tot = 0;
        const int p = block_exclusive_scan(take, warp_sums, take_tot) + base;
        if (take) o[p] = t;
        base += take_tot;
        eq_base += eq_tot;
        if (base >= k) break;  // uniform across the CTA
    }
}

__global__ void combine_kernel(const float* v_in, const float* s_in, int heads, int n, int mean, float* v_out,
                               float* s_out) {
    const double inv = 1.0 / static_cast<double>(heads);
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        double v = 0.0, s = 0.0;  // head order, as combine_scores sums
        for (int h = 0; h < heads; ++h) {
            v += static_cast<double>(v_in[static_cast<size_t>(h) * n + i]);
            s += static_cast<double>(s_in[static_cast<size_t>(h) * n + i]);
        }
        if (mean) {
            v *= inv;
            s *= inv;
        }
        v_out[i] = static_cast<float>(v);
        s_out[i] = static_cast<float>(s);
    }
}

}  // namespace

void merge_path_partition_host(const int64_t* a, int64_t na, const int64_t* b, int64_t nb, int64_t p,
                               int64_t* cuts) {
    const int64_t total = na + nb;
    cuts[0] = 0;
    cuts[1] = 0;
    for (int64_t s = 1; s < p; ++s) {
        const int64_t diag = s * total / p;
        const int64_t ai = merge_path_search(a, na, b, nb, diag);
        cuts[2 * s] = ai;
        cuts[2 * s + 1] = diag - ai;
    }
    cuts[2 * p] = na;
    cuts[2 * p + 1] = nb;
}

cudaError_t launch_merge_rows(const int* i_v, int k_v, const int* i_s, int k_s, const int* rows, int count, int* out,
                              int* out_len, int out_cap, bool validate, cudaStream_t stream) {
    if (count <= 0) return cudaSuccess;
    vsp_detail::count_launch();
    merge_rows_kernel<<<count, kMergeThreads, 0, stream>>>(i_v, k_v, i_s, k_s, rows, out, out_len, out_cap,
                                                           validate ? 1 : 0);
    return cudaGetLastError();
}

cudaError_t launch_topk(const float* scores, int n, int rows, const int* k_dev, int* out, int cap,
                        cudaStream_t stream) {
    if (rows <= 0) return cudaSuccess;
    vsp_detail::count_launch();
    topk_kernel<<<rows, kTopkThreads, 0, stream>>>(scores, n, k_dev, out, cap);
    return cudaGetLastError();
}

cudaError_t launch_combine(const float* v_in, const float* s_in, int heads, int n, bool mean, float* v_out,
                           float* s_out, cudaStream_t stream) {
    const int sms = vsp_detail::current_sm_count();
    int grid = (n + 255) / 256;
    if (grid > 4 * sms) grid = 4 * sms;
    vsp_detail::count_launch();
    combine_kernel<<<grid > 0 ? grid : 1, 256, 0, stream>>>(v_in, s_in, heads, n, mean ? 1 : 0, v_out, s_out);
    return cudaGetLastError();
}

}  // namespace vsp_misc
