// select.h — internal launch interface of K2 (cumulative-threshold top-k selection).
#pragma once
#include <cuda_runtime.h>
#include <cstddef>

#include "../../include/vsp_gpu.h"

namespace vsp_select_k {

size_t workspace_bytes(int n, int hkv);
cudaError_t launch(const float* a_v, const float* a_s, int n, int hkv, const vsp_budget* budgets,
                   int* i_v, int* k_v, int* i_s, int* k_s, int cap, void* workspace,
                   cudaStream_t stream, int g0 = 0, int count = -1);
// Layer path: softmax the indexer's logits inside the selection clusters (A_v / A_s are
// written as outputs), then select. Scores are bit-identical to launch_softmax's.
cudaError_t launch_from_logits(const float* lv, const float* ls, float* a_v, float* a_s, int n, int hkv,
                               const vsp_budget* budgets, int* i_v, int* k_v, int* i_s, int* k_s, int cap,
                               void* workspace, cudaStream_t stream, int g0 = 0, int count = -1);
// Softmax of logit rows [g0, g0 + count) of both directions (indexer.hpp:110-111).
cudaError_t launch_softmax(const float* lv, const float* ls, float* a_v, float* a_s, int n, int g0, int count,
                           cudaStream_t stream);
// Per-(direction, head) validation status written by the last launch on this workspace:
// [2*hkv] ints, dir-major: 0 ok, 1 negative score, 2 scores do not sum to 1.
const int* status_ptr(void* workspace, int n, int hkv);

}  // namespace vsp_select_k
