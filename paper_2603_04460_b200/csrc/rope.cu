// rope.cu — the step before the path: rotary embedding of Q and K,
// the "post-RoPE K" the indexer consumes (§3, indexer.hpp:116) and the Q/K the
// attention kernels read.
//
// Replaces vsp::apply_rope (reference rope.hpp:63-79) + rope_rotate_inplace (:42-52):
// plane p of head vector x at position t is rotated by t * theta_p, theta_p =
// base^(-2p/D). Interleaved planes (2p, 2p+1) are the reference's convention; the
// half-split planes (p, p + D/2) of HF LLaMA/Qwen checkpoints are an option.
//
// HBM-bound: every element is read and written once, so the kernel is one streaming pass
// over Q and K together (one launch). The angle work is per (token, plane) and shared by
// all Hq + Hkv heads of a token: each thread owns one 16-byte chunk of planes of a token,
// evaluates its cos/sin ONCE in fp64 (t * theta_p reaches ~1e5 rad at 128k; fp64 keeps the
// reference's f64 angle, and the cost is amortised over 40 heads), then walks the heads,
// rotating in fp32 and rounding to bf16 once. Consecutive threads cover consecutive 16-byte
// chunks of one head row, so every warp access is fully coalesced.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cmath>

#include "vsp_launch.h"
#include "rope.h"

namespace vsp_rope {

namespace {

constexpr int kThreads = 256;
constexpr int kMaxPlanes = 128;  // d <= 256

// theta_p per plane, passed by value (kernel parameter space): no global state shared by
// concurrent launches with different bases
struct Theta {
    double v[kMaxPlanes];
};

__device__ __forceinline__ void rot(float& x, float& y, float c, float s) {
    const float a = c * x - s * y;
    const float b = s * x + c * y;
    x = a;
    y = b;
}

// plain (coherent) 16-byte accesses: q_out may alias q_in (in-place rotation); each
// element is read and written by the same thread only
__device__ __forceinline__ uint4 ld16(const __nv_bfloat16* p) { return *reinterpret_cast<const uint4*>(p); }
__device__ __forceinline__ void st16(__nv_bfloat16* p, uint4 v) { *reinterpret_cast<uint4*>(p) = v; }

__device__ __forceinline__ void unpack8(const uint4& u, float (&f)[8]) {
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
    for (int t = 0; t < 4; ++t) {
        const float2 v = __bfloat1622float2(h[t]);
        f[2 * t] = v.x;
        f[2 * t + 1] = v.y;
    }
}

__device__ __forceinline__ uint4 pack8(const float (&f)[8]) {
    uint4 u;
    __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&u);
#pragma unroll
    for (int t = 0; t < 4; ++t) h[t] = __floats2bfloat162_rn(f[2 * t], f[2 * t + 1]);
    return u;
}

// Interleaved: thread c of a token owns elements [8c, 8c+8) = planes 4c .. 4c+3 of every head.
// grid-stride over (token, chunk) with tpt = d/8 chunks per token.
__global__ void __launch_bounds__(kThreads) rope_interleaved_kernel(const Args a, const Theta th) {
    const int tpt = a.d / 8;
    const long long total = static_cast<long long>(a.n) * tpt;
    for (long long w = blockIdx.x * static_cast<long long>(kThreads) + threadIdx.x; w < total;
         w += static_cast<long long>(gridDim.x) * kThreads) {
        const long long tok = w / tpt;
        const int c = static_cast<int>(w - tok * tpt);
        const double pos = a.positions ? static_cast<double>(a.positions[tok]) : static_cast<double>(tok);
        float cs[4], sn[4];
#pragma unroll
        for (int t = 0; t < 4; ++t) {
            double s, co;
            sincos(pos * th.v[4 * c + t], &s, &co);
            cs[t] = static_cast<float>(co);
            sn[t] = static_cast<float>(s);
        }
        for (int part = 0; part < 2; ++part) {
            const int heads = part ? a.hkv : a.hq;
            if (heads == 0) continue;
            const __nv_bfloat16* src = part ? a.k_in : a.q_in;
            __nv_bfloat16* dst = part ? a.k_out : a.q_out;
            const size_t row = static_cast<size_t>(tok) * heads * a.d + 8 * c;
            // batches of 4 heads: four independent 16-byte loads in flight per thread
            for (int h0 = 0; h0 < heads; h0 += 4) {
                const int nb = min(4, heads - h0);
                uint4 u[4];
#pragma unroll
                for (int b = 0; b < 4; ++b)
                    if (b < nb) u[b] = ld16(src + row + static_cast<size_t>(h0 + b) * a.d);
#pragma unroll
                for (int b = 0; b < 4; ++b) {
                    if (b >= nb) break;
                    float f[8];
                    unpack8(u[b], f);
#pragma unroll
                    for (int t = 0; t < 4; ++t) rot(f[2 * t], f[2 * t + 1], cs[t], sn[t]);
                    st16(dst + row + static_cast<size_t>(h0 + b) * a.d, pack8(f));
                }
            }
        }
    }
}

// Half-split: plane p pairs elements (p, p + d/2). Thread c owns elements [8c, 8c+8) and
// their partners [d/2 + 8c, d/2 + 8c + 8): planes 8c .. 8c+7; tpt = d/16.
__global__ void __launch_bounds__(kThreads) rope_half_kernel(const Args a, const Theta th) {
    const int tpt = a.d / 16;
    const int half = a.d / 2;
    const long long total = static_cast<long long>(a.n) * tpt;
    for (long long w = blockIdx.x * static_cast<long long>(kThreads) + threadIdx.x; w < total;
         w += static_cast<long long>(gridDim.x) * kThreads) {
        const long long tok = w / tpt;
        const int c = static_cast<int>(w - tok * tpt);
        const double pos = a.positions ? static_cast<double>(a.positions[tok]) : static_cast<double>(tok);
        float cs[8], sn[8];
#pragma unroll
        for (int t = 0; t < 8; ++t) {
            double s, co;
            sincos(pos * th.v[8 * c + t], &s, &co);
            cs[t] = static_cast<float>(co);
            sn[t] = static_cast<float>(s);
        }
        for (int part = 0; part < 2; ++part) {
            const int heads = part ? a.hkv : a.hq;
            if (heads == 0) continue;
            const __nv_bfloat16* src = part ? a.k_in : a.q_in;
            __nv_bfloat16* dst = part ? a.k_out : a.q_out;
            const size_t row = static_cast<size_t>(tok) * heads * a.d + 8 * c;
            for (int h0 = 0; h0 < heads; h0 += 2) {
                const int nb = min(2, heads - h0);
                uint4 ux[2], uy[2];
#pragma unroll
                for (int b = 0; b < 2; ++b)
                    if (b < nb) {
                        const size_t off = row + static_cast<size_t>(h0 + b) * a.d;
                        ux[b] = ld16(src + off);
                        uy[b] = ld16(src + off + half);
                    }
#pragma unroll
                for (int b = 0; b < 2; ++b) {
                    if (b >= nb) break;
                    const size_t off = row + static_cast<size_t>(h0 + b) * a.d;
                    float x[8], y[8];
                    unpack8(ux[b], x);
                    unpack8(uy[b], y);
#pragma unroll
                    for (int t = 0; t < 8; ++t) rot(x[t], y[t], cs[t], sn[t]);
                    st16(dst + off, pack8(x));
                    st16(dst + off + half, pack8(y));
                }
            }
        }
    }
}

}  // namespace

cudaError_t launch(const Args& a, cudaStream_t stream) {
    // theta_p = base^(-2p/D) in f64 exactly as RopeConfig::theta (rope.hpp:30-32)
    Theta th{};
    for (int p = 0; p < a.d / 2; ++p) th.v[p] = std::pow(a.base, -2.0 * p / static_cast<double>(a.d));
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int tpt = a.half_split ? a.d / 16 : a.d / 8;
    const long long work = static_cast<long long>(a.n) * tpt;
    // enough resident warps to cover HBM latency: 8 CTAs of 256 threads per SM, grid-stride
    const long long want = (work + kThreads - 1) / kThreads;
    const int grid = static_cast<int>(want < 8LL * sms ? (want > 0 ? want : 1) : 8LL * sms);
    vsp_detail::count_launch();
    if (a.half_split) rope_half_kernel<<<grid, kThreads, 0, stream>>>(a, th);
    else rope_interleaved_kernel<<<grid, kThreads, 0, stream>>>(a, th);
    return cudaGetLastError();
}

}  // namespace vsp_rope
