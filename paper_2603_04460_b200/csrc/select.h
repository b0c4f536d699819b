// select.h — internal launch interface of K2 (cumulative-threshold top-k selection).
#pragma once
#include <cuda_runtime.h>
#include <cstddef>

#include "../../include/vsp_gpu.h"

namespace vsp_select_k {

size_t workspace_bytes(int n, int hkv);
cudaError_t launch(const float* a_v, const float* a_s, int n, int hkv, const vsp_budget* budgets,
                   int* i_v, int* k_v, int* i_s, int* k_s, int cap, void* workspace,
                   cudaStream_t stream);

}  // namespace vsp_select_k
