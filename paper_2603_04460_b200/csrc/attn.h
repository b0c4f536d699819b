// attn.h — internal launch interface of the attention kernels (K3 sparse, K4 dense).
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "tma_host.h"

namespace vsp_attn {

// Output mirrors: every O tile / LSE row is also stored, at the same offsets, into up to
// kMaxMirrors other buffers of the same layout (peer GPUs' outputs mapped over NVLink, so the
// heads split needs no all-gather after the layer).
constexpr int kMaxMirrors = 7;

struct __align__(64) AttnParams {
    CUtensorMap map_q;   // [n, hq, 128] bf16, box {64, 1, 128}
    CUtensorMap map_k;   // [n, hkv, 128]
    CUtensorMap map_v;
    CUtensorMap map_kv;  // gathered verticals [hkv, kvcap, 128], box {64, 128, 1}
    CUtensorMap map_vv;
    CUtensorMap map_o;   // O for the epilogue's TMA stores: dims (128, hq, n) with the layout's strides
    CUtensorMap map_o_mirror[kMaxMirrors];  // the same map over each mirror buffer
    float* lse_mirror[kMaxMirrors];
    int n_mirrors;
    __nv_bfloat16* o;    // row i of head h at o + i * o_tok_stride + h * o_head_stride
    float* lse;          // [hq, n] or null
    long long o_tok_stride, o_head_stride;  // elements: [n, hq, 128] -> (hq*128, 128); head-major -> (128, n*128)
    const int* tile_lists;
    const uint32_t* vbits;
    const uint32_t* sbits;
    int list_stride;
    int pair0, npairs;   // Q-head pairs [pair0, pair0 + npairs) handled by this launch
    int qb_hi;           // query blocks [qb_hi - items / npairs, qb_hi) handled by this launch
    int items;           // work items (query block, head pair), pulled by persistent CTAs
    const int* units;    // units mode (nunits > 0): [nunits][4] = (KV head, qb_lo, qb_hi, qb prefix)
    int nunits;
    int* work;           // {next item - gridDim.x, CTAs done}: zero at launch, reset by the last CTA
    int bm_words;
    int prefetch_q;      // L2-prefetch the next work item's Q tiles (VSP_NO_Q_PREFETCH=1 disables)
    int n, hq, hkv;
    float scale;
};

struct AttnArgs {
    const void* q;  // [n, hq, 128] bf16
    const void* k;  // [n, hkv, 128] bf16
    const void* v;  // [n, hkv, 128] bf16
    void* o;        // [n, hq, 128] bf16 (token-major) or [hq, n, 128] (o_head_major)
    float* lse;     // [hq, n] fp32, may be null
    int n, hq, hkv;
    float scale;
    bool o_head_major = false;
    int n_mirrors = 0;                      // <= kMaxMirrors
    void* const* o_mirrors = nullptr;       // [n_mirrors] buffers shaped like o
    float* const* lse_mirrors = nullptr;    // [n_mirrors] like lse (entries may be null)
};

struct SparseArgs {
    const int* iv;  // [hkv, cap] ascending column indices
    const int* kv;  // [hkv] counts
    const int* is;  // [hkv, cap] ascending slash offsets
    const int* ks;  // [hkv]
    int cap;
    bool dense_switch = false;  // blocks whose VS tiles reach the dense count run unmasked causal
};

cudaError_t launch_dense(const AttnArgs& a, cudaStream_t stream);
size_t sparse_workspace_bytes(int n, int hkv, int cap);
cudaError_t launch_sparse(const AttnArgs& a, const SparseArgs& s, void* workspace, cudaStream_t stream,
                          int g0 = 0, int count = -1, int phase = 3, int qb_lo = 0, int qb_hi = -1);
// Attention phase over a list of (KV head, qb_lo, qb_hi) units in ONE persistent launch (the
// plans of their heads must exist in `workspace`); host_units: nunits x 3 ints.
constexpr int kMaxUnits = 512;
cudaError_t launch_sparse_units(const AttnArgs& a, const SparseArgs& s, void* workspace, cudaStream_t stream,
                                const int* host_units, int nunits);

}  // namespace vsp_attn

namespace vsp_attn {
cudaError_t sparse_tile_stats(int n, int hkv, int cap, const void* workspace, long long* tiles_out,
                              cudaStream_t stream);
}
