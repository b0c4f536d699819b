// misc_ops.h — standalone reference operators on the device (merge_topk.cu).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

namespace vsp_misc {

// merge.hpp:69-95: the a-first crossing of merge-path diagonal `diag` of two ascending
// sequences — the smallest ai in [max(0, diag - nb), min(diag, na)] with a[ai] > b[diag-ai-1].
template <class T>
__host__ __device__ inline int64_t merge_path_search(const T* a, int64_t na, const T* b, int64_t nb, int64_t diag) {
    int64_t lo = diag > nb ? diag - nb : 0, hi = diag < na ? diag : na;
    while (lo < hi) {
        const int64_t mid = lo + (hi - lo) / 2;
        if (a[mid] <= b[diag - mid - 1]) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

// cuts int64 [(p + 1) x 2]: (a_idx, b_idx) of the p + 1 cut points (p >= 1).
void merge_path_partition_host(const int64_t* a, int64_t na, const int64_t* b, int64_t nb, int64_t p, int64_t* cuts);

cudaError_t launch_merge_rows(const int* i_v, int k_v, const int* i_s, int k_s, const int* rows, int count, int* out,
                              int* out_len, int out_cap, bool validate, cudaStream_t stream);
cudaError_t launch_topk(const float* scores, int n, int rows, const int* k_dev, int* out, int cap, cudaStream_t stream);
cudaError_t launch_combine(const float* v_in, const float* s_in, int heads, int n, bool mean, float* v_out,
                           float* s_out, cudaStream_t stream);

}  // namespace vsp_misc
