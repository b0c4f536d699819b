// train.h — internal launch interface of the distillation kernels (csrc/train.cu).
#pragma once
#include <cuda_runtime.h>

#include <cstddef>

namespace vsp_train {

struct GradArgs {
    const void* k;         // [n, hkv, 128] bf16
    const void* v;
    int n, hkv, d_h;
    const void* w_u_bf16;  // [hkv, 256, d_h] bf16 (the forward's copy of the master weights)
    const float* b_u;      // [hkv, d_h]
    const float* w_v;
    const float* b_v;      // [hkv]
    const float* w_s;
    const float* b_s;
    bool reverse;
    const float* target_v; // [hkv, n] distributions (K5 output)
    const float* target_s;
    double kl_eps;
    float* loss;           // [hkv] device (KL_v + KL_s per head), may be null
    float* grads;          // flat, parameter layout W_U | b_U | w_v | w_s | b_v | b_s
};

struct AdamArgs {
    float* params;         // flat fp32 master parameters
    const float* grads;
    float* m;
    float* v;
    long long count;
    long long step_index;
    double lr, beta1, beta2, adam_eps, weight_decay;
    void* shadow;          // bf16 copy of the first shadow_count parameters (W_U) or null
    long long shadow_count;
};

size_t workspace_bytes(int n, int hkv, int d_h);
cudaError_t loss_grad(const GradArgs& a, void* workspace, cudaStream_t stream);
cudaError_t adamw(const AdamArgs& a, cudaStream_t stream);

}  // namespace vsp_train
