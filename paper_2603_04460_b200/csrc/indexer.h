// indexer.h — internal launch interface of K1 (VSIndexer scoring).
#pragma once
#include <cuda_runtime.h>
#include <cstddef>

namespace vsp_indexer {

struct Args {
    const void* k;    // [n, hkv, 128] bf16
    const void* v;    // [n, hkv, 128] bf16
    int n, hkv, d_h;
    const void* w_u;  // [hkv, 256, d_h] bf16
    const float* b_u; // [hkv, d_h]
    const float* w_v; // [hkv, d_h]
    const float* b_v; // [hkv]
    const float* w_s; // [hkv, d_h]
    const float* b_s; // [hkv]
    bool reverse;
    float* a_v;       // [hkv, n]
    float* a_s;       // [hkv, n]
    float* logits_v;  // [hkv, n] or null
    float* logits_s;  // [hkv, n] or null
    int g0 = 0;       // first KV head of this launch (head-range launches for pipelining)
    int count = -1;   // number of KV heads (-1: all from g0)
};

size_t workspace_bytes(int n, int hkv, int d_h);
cudaError_t launch(const Args& a, void* workspace, cudaStream_t stream);

}  // namespace vsp_indexer
