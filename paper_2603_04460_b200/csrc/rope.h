// rope.h — internal launch interface of the RoPE feed kernel (csrc/rope.cu).
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

namespace vsp_rope {

struct Args {
    const __nv_bfloat16* q_in;  // [n, hq, d] (hq may be 0)
    const __nv_bfloat16* k_in;  // [n, hkv, d] (hkv may be 0)
    __nv_bfloat16* q_out;       // may alias q_in (in place)
    __nv_bfloat16* k_out;
    const int64_t* positions;   // [n] or null (position t = row t, rope.hpp:73-79)
    int n, hq, hkv, d;
    double base;
    bool half_split;            // planes (p, p + d/2) instead of (2p, 2p+1)
};

cudaError_t launch(const Args& a, cudaStream_t stream);

}  // namespace vsp_rope
