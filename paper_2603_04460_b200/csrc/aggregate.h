// aggregate.h — internal launch interface of K5 (ground-truth VS aggregation).
#pragma once
#include <cuda_runtime.h>
#include <cstddef>

namespace vsp_aggregate {

struct Args {
    const void* q;  // [n, hq, 128] bf16
    const void* k;  // [n, hkv, 128] bf16
    int n, hq, hkv;
    float scale;
    const float* lse;  // [hq, n] or null (computed in pass 1)
    bool mean;
    bool normalized;
    float* a_v;  // [hkv, n]
    float* a_s;  // [hkv, n]
};

size_t workspace_bytes(int n, int hq);
cudaError_t launch(const Args& a, void* workspace, cudaStream_t stream);

}  // namespace vsp_aggregate
