// capi.cu — the C ABI (include/vsp_gpu.h): argument checks with the reference's error
// texts, workspace sizing, and dispatch to the sm_100a kernels. No CPU fallback.
#include <cuda_runtime.h>
#include <cstring>

#include <cstdio>
#include <algorithm>
#include <cmath>
#include <string>
#include <initializer_list>
#include <atomic>
#include <vector>

#include "vsp_launch.h"
#include "../../include/vsp_gpu.h"
#include "aggregate.h"
#include "attn.h"
#include "indexer.h"
#include "misc_ops.h"
#include "rope.h"
#include "select.h"
#include "train.h"
#include "vsp_error.h"

namespace vsp_detail {
thread_local std::string g_err;
int set_err(int code, const std::string& msg) {
    g_err = msg;
    return code;
}
std::atomic<long long> g_launches{0};
void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
}  // namespace vsp_detail

extern "C" long long vsp_kernel_launches(void) { return vsp_detail::g_launches.load(std::memory_order_relaxed); }

struct vsp_ctx {
    int device = 0;
    int sm_count = 0;
    // vsp_vs_prefill pipelining: high-priority side stream and per-chunk events
    static constexpr int kMaxChunks = 64;
    cudaStream_t side = nullptr;
    cudaEvent_t ev_start = nullptr;
    cudaEvent_t ev_chunk[kMaxChunks] = {};
    // vsp_vs_prefill_host: copy-engine streams and their events
    cudaStream_t h2d = nullptr, d2h = nullptr;
    cudaEvent_t ev_host0 = nullptr, ev_host1 = nullptr;
    cudaEvent_t ev_kv[kMaxChunks] = {}, ev_q[kMaxChunks] = {}, ev_attn[kMaxChunks] = {};
    // optional live timing of the K3 launches of the layer entry points (vsp_attn_timing):
    // an event pair around every attention launch, summed by vsp_attn_timing_read
    static constexpr int kTimingSlots = 512;
    bool timing = false;
    int timed = 0;
    cudaEvent_t t_beg[kTimingSlots] = {}, t_end[kTimingSlots] = {};
};

namespace {

using vsp_detail::set_err;
int cuda_err(cudaError_t e, const char* where) {
    return set_err(VSP_ECUDA, std::string(where) + ": " + cudaGetErrorString(e));
}
#define VSP_CHECK_CTX(ctx)                                                         \
    do {                                                                           \
        if (!(ctx)) return set_err(VSP_EINVAL, "vsp: null context");               \
        if (cudaSetDevice((ctx)->device) != cudaSuccess)                           \
            return set_err(VSP_ECUDA, "vsp: cannot select device");                \
    } while (0)

cudaStream_t as_stream(void* s) { return static_cast<cudaStream_t>(s); }

// Strict ascending order, non-negative entries, and row-0 coverage, per KV head.
__global__ void validate_pattern_kernel(const int* iv, const int* kv, const int* is, const int* ks,
                                        int cap, int* flags) {
    const int g = blockIdx.x;
    const int nv = kv[g], ns = ks[g];
    // the list scans stay inside the row even when a count is out of range (flag 16)
    const int nv_c = nv < 0 ? 0 : (nv > cap ? cap : nv), ns_c = ns < 0 ? 0 : (ns > cap ? cap : ns);
    const int* a = iv + static_cast<size_t>(g) * cap;
    const int* b = is + static_cast<size_t>(g) * cap;
    int f = 0;
    for (int t = threadIdx.x; t < nv_c; t += blockDim.x) {
        if (a[t] < 0) f |= 8;
        if (t > 0 && !(a[t - 1] < a[t])) f |= 1;
    }
    for (int t = threadIdx.x; t < ns_c; t += blockDim.x) {
        if (b[t] < 0) f |= 8;
        if (t > 0 && !(b[t - 1] < b[t])) f |= 2;
    }
    if (threadIdx.x == 0) {
        const bool covered0 = (nv_c > 0 && a[0] == 0) || (ns_c > 0 && b[0] == 0);
        if (!covered0) f |= 4;
        if (nv < 0 || ns < 0 || nv > cap || ns > cap) f |= 16;
    }
    f = __reduce_or_sync(0xffffffffu, f);
    __shared__ int acc;
    if (threadIdx.x == 0) acc = 0;
    __syncthreads();
    if ((threadIdx.x & 31) == 0 && f) atomicOr(&acc, f);
    __syncthreads();
    if (threadIdx.x == 0) flags[g] = acc;
}

// Exact recall per head (attention.hpp:198-215 without the n x n matrix): mean_i
// exp(LSE_sparse_i - LSE_dense_i). One 8-CTA cluster per head (a single 512-thread block per
// head left the 33.5 MB read at 5.7 % of HBM bandwidth at 128k x 32 heads): each CTA sums a
// fixed contiguous eighth of the row in fp64, and CTA 0 adds the eight partials in rank order
// over DSMEM, so the result does not depend on scheduling.
constexpr int kRecallCluster = 8;
__global__ void __cluster_dims__(kRecallCluster, 1, 1) __launch_bounds__(512)
    recall_kernel(const float* ls, const float* ld, int n, float* out) {
    const int h = blockIdx.x / kRecallCluster;
    const int part = blockIdx.x % kRecallCluster;  // == cluster rank (1-D cluster along x)
    const int per = (n + kRecallCluster - 1) / kRecallCluster;
    const int lo = part * per, hi = min(n, lo + per);
    double acc = 0.0;
    for (int i = lo + static_cast<int>(threadIdx.x); i < hi; i += blockDim.x) {
        const size_t x = static_cast<size_t>(h) * n + i;
        acc += exp(static_cast<double>(ls[x]) - static_cast<double>(ld[x]));
    }
    __shared__ double red[32];
    __shared__ double part_sum;
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
        part_sum = t;
    }
    // every CTA's partial is written before CTA 0 reads them; no CTA leaves before the read
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    if (part == 0 && threadIdx.x == 0) {
        double t = 0.0;
        const uint32_t local = static_cast<uint32_t>(__cvta_generic_to_shared(&part_sum));
        for (int r = 0; r < kRecallCluster; ++r) {
            uint32_t remote;
            asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(local), "r"(r));
            double v;
            asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(v) : "r"(remote) : "memory");
            t += v;
        }
        out[h] = static_cast<float>(t / n);
    }
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

int check_attn_shapes(int n, int hq, int hkv, int d) {
    if (n < 1) return set_err(VSP_EINVAL, "attention inputs: empty sequence");
    if (hkv < 1 || hq < hkv || hq % hkv != 0)
        return set_err(VSP_EINVAL, "attention inputs: hq must be a positive multiple of hkv");
    if (d != 128) return set_err(VSP_EINVAL, "vsp: head dim must be 128");
    return VSP_OK;
}

}  // namespace

extern "C" {

const char* vsp_last_error(void) { return vsp_detail::g_err.c_str(); }
const char* vsp_version(void) { return "vsp-b200 0.1 (sm_100a)"; }

int vsp_create(vsp_ctx** out, int device) {
    if (!out) return set_err(VSP_EINVAL, "vsp_create: null output");
    int count = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0)
        return set_err(VSP_ECUDA, "vsp_create: no CUDA device (the VS-prefill path has no CPU fallback)");
    if (device < 0 || device >= count) return set_err(VSP_EINVAL, "vsp_create: bad device ordinal");
    cudaDeviceProp prop;
    cudaError_t e = cudaGetDeviceProperties(&prop, device);
    if (e != cudaSuccess) return cuda_err(e, "vsp_create");
    if (prop.major != 10)
        return set_err(VSP_ECUDA, "vsp_create: an sm_100 (B200) device is required, got sm_" +
                                      std::to_string(prop.major) + std::to_string(prop.minor));
    auto* ctx = new vsp_ctx();
    ctx->device = device;
    ctx->sm_count = prop.multiProcessorCount;
    cudaSetDevice(device);
    {
        int lo = 0, hi = 0;
        cudaDeviceGetStreamPriorityRange(&lo, &hi);
        e = cudaStreamCreateWithPriority(&ctx->side, cudaStreamNonBlocking, hi);
    }
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&ctx->h2d, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&ctx->d2h, cudaStreamNonBlocking);
    for (cudaEvent_t* ev : {&ctx->ev_start, &ctx->ev_host0, &ctx->ev_host1})
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(ev, cudaEventDisableTiming);
    for (int c = 0; c < vsp_ctx::kMaxChunks && e == cudaSuccess; ++c) {
        for (cudaEvent_t* ev : {&ctx->ev_chunk[c], &ctx->ev_kv[c], &ctx->ev_q[c], &ctx->ev_attn[c]})
            if (e == cudaSuccess) e = cudaEventCreateWithFlags(ev, cudaEventDisableTiming);
    }
    if (e != cudaSuccess) {
        delete ctx;
        return cuda_err(e, "vsp_create");
    }
    *out = ctx;
    return VSP_OK;
}

int vsp_destroy(vsp_ctx* ctx) {
    if (!ctx) return VSP_OK;
    cudaSetDevice(ctx->device);
    for (int i = 0; i < vsp_ctx::kTimingSlots; ++i)
        for (cudaEvent_t ev : {ctx->t_beg[i], ctx->t_end[i]})
            if (ev) cudaEventDestroy(ev);
    for (cudaStream_t st : {ctx->side, ctx->h2d, ctx->d2h})
        if (st) cudaStreamDestroy(st);
    for (cudaEvent_t ev : {ctx->ev_start, ctx->ev_host0, ctx->ev_host1})
        if (ev) cudaEventDestroy(ev);
    for (int c = 0; c < vsp_ctx::kMaxChunks; ++c)
        for (cudaEvent_t ev : {ctx->ev_chunk[c], ctx->ev_kv[c], ctx->ev_q[c], ctx->ev_attn[c]})
            if (ev) cudaEventDestroy(ev);
    delete ctx;
    return VSP_OK;
}

// ------------------------------------------------------------------ attention
int vsp_dense_attn_fwd(vsp_ctx* ctx, const void* q, const void* k, const void* v, int n, int hq,
                       int hkv, int d, float scale, void* o, float* lse, void* stream) {
    VSP_CHECK_CTX(ctx);
    int rc = check_attn_shapes(n, hq, hkv, d);
    if (rc) return rc;
    vsp_attn::AttnArgs a{q, k, v, o, lse, n, hq, hkv, scale};
    cudaError_t e = vsp_attn::launch_dense(a, as_stream(stream));
    return e == cudaSuccess ? VSP_OK : cuda_err(e, "vsp_dense_attn_fwd");
}

// The caller's workspace ends with this call's validation flags ([hkv] ints), so concurrent
// validating calls on different streams never share device state.
static size_t validate_flags_offset(int n, int hkv, int cap) {
    return (vsp_attn::sparse_workspace_bytes(n, hkv, cap) + 255) / 256 * 256;
}

size_t vsp_vs_attn_workspace_size(int n, int hkv, int cap) {
    return validate_flags_offset(n, hkv, cap) + 1024 * sizeof(int);
}

int vsp_vs_attn_fwd(vsp_ctx* ctx, const void* q, const void* k, const void* v, int n, int hq,
                    int hkv, int d, const int* i_v, const int* k_v, const int* i_s, const int* k_s,
                    int cap, float scale, void* o, float* lse, void* workspace, int flags,
                    void* stream) {
    VSP_CHECK_CTX(ctx);
    int rc = check_attn_shapes(n, hq, hkv, d);
    if (rc) return rc;
    if (cap < 1) return set_err(VSP_EINVAL, "vsp_vs_attn_fwd: cap must be >= 1");
    if (!workspace) return set_err(VSP_EINVAL, "vsp_vs_attn_fwd: workspace required");
    cudaStream_t st = as_stream(stream);
    if (flags & VSP_VALIDATE) {
        if (hkv > 1024) return set_err(VSP_EINVAL, "vsp_vs_attn_fwd: too many heads to validate");
        vsp_detail::count_launch();
        int* d_flags = reinterpret_cast<int*>(static_cast<uint8_t*>(workspace) + validate_flags_offset(n, hkv, cap));
        validate_pattern_kernel<<<hkv, 256, 0, st>>>(i_v, k_v, i_s, k_s, cap, d_flags);
        int hflags[1024];
        cudaError_t e = cudaMemcpyAsync(hflags, d_flags, sizeof(int) * hkv, cudaMemcpyDeviceToHost, st);
        if (e == cudaSuccess) e = cudaStreamSynchronize(st);
        if (e != cudaSuccess) return cuda_err(e, "vsp_vs_attn_fwd(validate)");
        for (int g = 0; g < hkv; ++g) {
            // same precedence as the reference: merge_row_columns validates i_v, then i_s
            // (merge.hpp:21-26), then sparse_attention reports the uncovered row (:161-163)
            if (hflags[g] & 16) return set_err(VSP_EINVAL, "vsp_vs_attn_fwd: index count exceeds cap");
            if (hflags[g] & 8) return set_err(VSP_EINVAL, "vsp_vs_attn_fwd: negative index");
            if (hflags[g] & 1) return set_err(VSP_EINVAL, "merge_row_columns: i_v not strictly ascending");
            if (hflags[g] & 2) return set_err(VSP_EINVAL, "merge_row_columns: i_s not strictly ascending");
            if (hflags[g] & 4) return set_err(VSP_EINVAL, "uncovered query row 0");
        }
    }
    if (flags & ~(VSP_VALIDATE | VSP_O_HEAD_MAJOR | VSP_DENSE_SWITCH))
        return set_err(VSP_EINVAL, "vsp_vs_attn_fwd: unknown flags");
    vsp_attn::AttnArgs a{q, k, v, o, lse, n, hq, hkv, scale, (flags & VSP_O_HEAD_MAJOR) != 0};
    vsp_attn::SparseArgs s{i_v, k_v, i_s, k_s, cap, (flags & VSP_DENSE_SWITCH) != 0};
    cudaError_t e = vsp_attn::launch_sparse(a, s, workspace, st);
    return e == cudaSuccess ? VSP_OK : cuda_err(e, "vsp_vs_attn_fwd");
}

int vsp_merge_path_partition(const int64_t* a, int64_t na, const int64_t* b, int64_t nb, int64_t p, int64_t* cuts) {
    if (p < 1) return set_err(VSP_EINVAL, "merge_path_partition: p must be >= 1");
    if (na < 0 || nb < 0 || !cuts || (na && !a) || (nb && !b))
        return set_err(VSP_EINVAL, "merge_path_partition: bad arguments");
    vsp_misc::merge_path_partition_host(a, na, b, nb, p, cuts);
    return VSP_OK;
}

int vsp_merge_row_columns(vsp_ctx* ctx, const int* i_v, int k_v, const int* i_s, int k_s, const int* rows,
                          int count, int* out, int* out_len, int out_cap, int flags, void* stream) {
    VSP_CHECK_CTX(ctx);
    if (k_v < 0 || k_s < 0 || count < 0 || out_cap < 0 || (count && (!rows || !out_len)))
        return set_err(VSP_EINVAL, "merge_row_columns: bad arguments");
    if (flags & ~VSP_VALIDATE) return set_err(VSP_EINVAL, "merge_row_columns: unknown flags");
    cudaStream_t st = as_stream(stream);
    cudaError_t e = vsp_misc::launch_merge_rows(i_v, k_v, i_s, k_s, rows, count, out, out_len, out_cap,
                                                (flags & VSP_VALIDATE) != 0, st);
    if (e != cudaSuccess) return cuda_err(e, "vsp_merge_row_columns");
    if (flags & VSP_VALIDATE) {
        std::vector<int> len(count);
        e = cudaMemcpyAsync(len.data(), out_len, sizeof(int) * count, cudaMemcpyDeviceToHost, st);
        if (e == cudaSuccess) e = cudaStreamSynchronize(st);
        if (e != cudaSuccess) return cuda_err(e, "vsp_merge_row_columns(validate)");
        for (int r = 0; r < count; ++r) {
            if (len[r] == -1) return set_err(VSP_EINVAL, "merge_row_columns: i_v not strictly ascending");
            if (len[r] == -2) return set_err(VSP_EINVAL, "merge_row_columns: i_s not strictly ascending");
            if (len[r] == -3) return set_err(VSP_EINVAL, "merge_row_columns: out_cap too small");
        }
    }
    return VSP_OK;
}

size_t vsp_topk_workspace_size(int rows) { return static_cast<size_t>(rows > 0 ? rows : 1) * sizeof(int); }

int vsp_topk_indices(vsp_ctx* ctx, const float* scores, int n, int rows, const int* k, int* out, int cap,
                     void* workspace, void* stream) {
    VSP_CHECK_CTX(ctx);
    if (rows < 0 || (rows && (!scores || !k || !out || !workspace)))
        return set_err(VSP_EINVAL, "topk_indices: bad arguments");
    for (int r = 0; r < rows; ++r) {
        if (k[r] < 1) return set_err(VSP_EINVAL, "topk_indices: k must be >= 1");
        if (k[r] > n) return set_err(VSP_EINVAL, "topk_indices: k exceeds score count");
        if (k[r] > cap) return set_err(VSP_EINVAL, "topk_indices: k exceeds cap");
    }
    cudaStream_t st = as_stream(stream);
    int* kd = static_cast<int*>(workspace);
    cudaError_t e = rows ? cudaMemcpyAsync(kd, k, sizeof(int) * rows, cudaMemcpyHostToDevice, st) : cudaSuccess;
    if (e == cudaSuccess) e = vsp_misc::launch_topk(scores, n, rows, kd, out, cap, st);
    return e == cudaSuccess ? VSP_OK : cuda_err(e, "vsp_topk_indices");
}

int vsp_combine_scores(vsp_ctx* ctx, const float* v_in, const float* s_in, int heads, int n, int reduce,
                       float* v_out, float* s_out, void* stream) {
    VSP_CHECK_CTX(ctx);
    if (heads < 1) return set_err(VSP_EINVAL, "combine_scores: no heads");
    if (n < 0 || (n && (!v_in || !s_in || !v_out || !s_out)))
        return set_err(VSP_EINVAL, "combine_scores: bad arguments");
    if (reduce != VSP_REDUCE_MEAN && reduce != VSP_REDUCE_SUM)
        return set_err(VSP_EINVAL, "combine_scores: unknown reduce");
    if (n == 0) return VSP_OK;
    cudaError_t e = vsp_misc::launch_combine(v_in, s_in, heads, n, reduce == VSP_REDUCE_MEAN, v_out, s_out,
                                             as_stream(stream));
    return e == cudaSuccess ? VSP_OK : cuda_err(e, "vsp_combine_scores");
}

int vsp_recall_from_lse(vsp_ctx* ctx, const float* lse_sparse, const float* lse_dense, int n, int hq,
                        float* recall_per_head, void* stream) {
    VSP_CHECK_CTX(ctx);
    if (n < 1 || hq < 1) return set_err(VSP_EINVAL, "vsp_recall_from_lse: bad shape");
    vsp_detail::count_launch();
    recall_kernel<<<hq * kRecallCluster, 512, 0, as_stream(stream)>>>(lse_sparse, lse_dense, n, recall_per_head);
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? VSP_OK : cuda_err(e, "vsp_recall_from_lse");
}

// ------------------------------------------------------------------ RoPE feed
int vsp_apply_rope(vsp_ctx* ctx, const void* q_in, const void* k_in, void* q_out, void* k_out, int n, int hq,
                   int hkv, int d, const int64_t* positions, double base, int style, void* stream) {
    VSP_CHECK_CTX(ctx);
    // RopeConfig's own checks first (rope.hpp:19-26), then this kernel's layout limits
    if (d < 2 || d % 2 != 0) return set_err(VSP_EINVAL, "rope head_dim must be even and >= 2");
    if (!(base > 0.0)) return set_err(VSP_EINVAL, "rope base must be positive");
    if (style != VSP_ROPE_INTERLEAVED && style != VSP_ROPE_HALF_SPLIT)
        return set_err(VSP_EINVAL, "vsp_apply_rope: bad style");
    const int unit = style == VSP_ROPE_HALF_SPLIT ? 16 : 8;
    if (d % unit != 0 || d > 256)
        return set_err(VSP_EINVAL, "vsp_apply_rope: head dim must be a multiple of " + std::to_string(unit) +
                                       " and <= 256");
    if (n < 0 || hq < 0 || hkv < 0) return set_err(VSP_EINVAL, "vsp_apply_rope: bad shape");
    if ((hq > 0 && (!q_in || !q_out)) || (hkv > 0 && (!k_in || !k_out)))
        return set_err(VSP_EINVAL, "vsp_apply_rope: null tensor");
    if (n == 0 || (hq == 0 && hkv == 0)) return VSP_OK;
    vsp_rope::Args a{static_cast<const __nv_bfloat16*>(q_in), static_cast<const __nv_bfloat16*>(k_in),
                     static_cast<__nv_bfloat16*>(q_out), static_cast<__nv_bfloat16*>(k_out), positions, n, hq, hkv, d,
                     base, style == VSP_ROPE_HALF_SPLIT};
    cudaError_t e = vsp_rope::launch(a, as_stream(stream));
    return e == cudaSuccess ? VSP_OK : cuda_err(e, "vsp_apply_rope");
}

// ------------------------------------------------------------------ distillation
size_t vsp_indexer_grad_workspace_size(int n, int hkv, int d_h) { return vsp_train::workspace_bytes(n, hkv, d_h); }

int vsp_indexer_loss_grad(vsp_ctx* ctx, const void* k, const void* v, int n, int hkv, int d, int d_h,
                          const void* w_u_bf16, const float* b_u, const float* w_v, const float* b_v,
                          const float* w_s, const float* b_s, int slash_mapping, const float* target_v,
                          const float* target_s, double kl_eps, float* loss, float* grads, void* workspace,
                          void* stream) {
    VSP_CHECK_CTX(ctx);
    if (n < 1) return set_err(VSP_EINVAL, "indexer_forward: empty input");
    if (d != 128) return set_err(VSP_EINVAL, "vsp: head dim must be 128");
    if (d_h < 1 || d_h % 256 != 0) return set_err(VSP_EINVAL, "vsp_indexer_loss_grad: d_h must be a multiple of 256");
    if (!(kl_eps > 0.0)) return set_err(VSP_EINVAL, "kl_loss: eps must be positive");
    if (slash_mapping != VSP_SLASH_REVERSE && slash_mapping != VSP_SLASH_IDENTITY)
        return set_err(VSP_EINVAL, "vsp_indexer_loss_grad: bad slash mapping");
    if (!workspace || !grads || !target_v || !target_s)
        return set_err(VSP_EINVAL, "vsp_indexer_loss_grad: null argument");
    vsp_train::GradArgs a{k, v, n, hkv, d_h, w_u_bf16, b_u, w_v, b_v, w_s, b_s,
                          slash_mapping == VSP_SLASH_REVERSE, target_v, target_s, kl_eps, loss, grads};
    cudaError_t e = vsp_train::loss_grad(a, workspace, as_stream(stream));
    return e == cudaSuccess ? VSP_OK : cuda_err(e, "vsp_indexer_loss_grad");
}

int vsp_adamw_step(vsp_ctx* ctx, float* params, const float* grads, float* m, float* v, int64_t count,
                   int64_t step_index, const vsp_adamw* cfg, void* shadow_bf16, int64_t shadow_count, void* stream) {
    VSP_CHECK_CTX(ctx);
    if (!params || !grads || !m || !v || !cfg || count < 0 || step_index < 0)
        return set_err(VSP_EINVAL, "vsp_adamw_step: bad arguments");
    if (shadow_count < 0 || shadow_count > count || (shadow_count > 0 && !shadow_bf16))
        return set_err(VSP_EINVAL, "vsp_adamw_step: bad shadow range");
    vsp_train::AdamArgs a{params, grads, m, v, count, step_index, cfg->lr, cfg->beta1, cfg->beta2, cfg->adam_eps,
                          cfg->weight_decay, shadow_bf16, shadow_count};
    cudaError_t e = vsp_train::adamw(a, as_stream(stream));
    return e == cudaSuccess ? VSP_OK : cuda_err(e, "vsp_adamw_step");
}

// ------------------------------------------------------------------ indexer
size_t vsp_indexer_workspace_size(int n, int hkv, int d_h) { return vsp_indexer::workspace_bytes(n, hkv, d_h); }

int vsp_indexer_scores(vsp_ctx* ctx, const void* k, const void* v, int n, int hkv, int d, int d_h,
                       const void* w_u, const float* b_u, const float* w_v, const float* b_v,
                       const float* w_s, const float* b_s, int slash_mapping, float* a_v, float* a_s,
                       float* logits_v, float* logits_s, void* workspace, void* stream) {
    VSP_CHECK_CTX(ctx);
    if (n < 1) return set_err(VSP_EINVAL, "indexer_forward: empty input");
    if (d != 128) return set_err(VSP_EINVAL, "vsp: head dim must be 128");
    if (d_h < 1 || d_h % 256 != 0) return set_err(VSP_EINVAL, "vsp_indexer_scores: d_h must be a multiple of 256");
    if (slash_mapping != VSP_SLASH_REVERSE && slash_mapping != VSP_SLASH_IDENTITY)
        return set_err(VSP_EINVAL, "vsp_indexer_scores: bad slash mapping");
    if (!workspace) return set_err(VSP_EINVAL, "vsp_indexer_scores: workspace required");
    vsp_indexer::Args a{k, v, n, hkv, d_h, w_u, b_u, w_v, b_v, w_s, b_s,
                        slash_mapping == VSP_SLASH_REVERSE, a_v, a_s, logits_v, logits_s};
    cudaError_t e = vsp_indexer::launch(a, workspace, as_stream(stream));
    return e == cudaSuccess ? VSP_OK : cuda_err(e, "vsp_indexer_scores");
}

// ------------------------------------------------------------------ selection
size_t vsp_select_workspace_size(int n, int hkv) { return vsp_select_k::workspace_bytes(n, hkv); }

int vsp_select(vsp_ctx* ctx, const float* a_v, const float* a_s, int n, int hkv, const vsp_budget* budgets,
               int* i_v, int* k_v, int* i_s, int* k_s, int cap, void* workspace, int flags, void* stream) {
    VSP_CHECK_CTX(ctx);
    if (n < 1) return set_err(VSP_EINVAL, "cumulative_budget: empty scores");
    if (cap < n + 1) return set_err(VSP_EINVAL, "vsp_select: cap must be >= n + 1");
    if (!budgets) return set_err(VSP_EINVAL, "vsp_select: null budgets");
    for (int g = 0; g < hkv; ++g) {  // BudgetConfig::check (sparsity.hpp:27-35)
        const vsp_budget& b = budgets[g];
        if (!(b.tau_v > 0.0 && b.tau_v <= 1.0)) return set_err(VSP_EINVAL, "budget config: tau_v must be in (0, 1]");
        if (!(b.tau_s > 0.0 && b.tau_s <= 1.0)) return set_err(VSP_EINVAL, "budget config: tau_s must be in (0, 1]");
        if (b.min_budget < 1) return set_err(VSP_EINVAL, "budget config: min_budget must be >= 1");
        if (b.max_budget >= 0 && b.min_budget > b.max_budget)
            return set_err(VSP_EINVAL, "budget config: min_budget exceeds max_budget");
    }
    if (!workspace) return set_err(VSP_EINVAL, "vsp_select: workspace required");
    if (hkv > 128) return set_err(VSP_EINVAL, "vsp_select: at most 128 KV heads per call");
    cudaStream_t st = as_stream(stream);
    cudaError_t e = vsp_select_k::launch(a_v, a_s, n, hkv, budgets, i_v, k_v, i_s, k_s, cap, workspace, st);
    if (e != cudaSuccess) return cuda_err(e, "vsp_select");
    if (flags & VSP_VALIDATE) {
        int hs[256];
        e = cudaMemcpyAsync(hs, vsp_select_k::status_ptr(workspace, n, hkv), sizeof(int) * 2 * hkv,
                            cudaMemcpyDeviceToHost, st);
        if (e == cudaSuccess) e = cudaStreamSynchronize(st);
        if (e != cudaSuccess) return cuda_err(e, "vsp_select(validate)");
        for (int g = 0; g < hkv; ++g)
            for (int dir = 0; dir < 2; ++dir) {  // vertical budget is computed first (sparsity.hpp:108-109)
                const int code = hs[dir * hkv + g];
                if (code == 1) return set_err(VSP_EINVAL, "cumulative_budget: negative score");
                if (code == 2) return set_err(VSP_EINVAL, "cumulative_budget: scores do not sum to 1");
            }
    }
    return VSP_OK;
}

// ------------------------------------------------------------------ aggregation
size_t vsp_aggregate_workspace_size(int n, int hq) { return vsp_aggregate::workspace_bytes(n, hq); }

int vsp_vs_aggregate(vsp_ctx* ctx, const void* q, const void* k, int n, int hq, int hkv, int d, float scale,
                     const float* lse, int reduce, int normalized, float* a_v, float* a_s, void* workspace,
                     void* stream) {
    VSP_CHECK_CTX(ctx);
    int rc = check_attn_shapes(n, hq, hkv, d);
    if (rc) return rc;
    if (reduce != VSP_REDUCE_MEAN && reduce != VSP_REDUCE_SUM)
        return set_err(VSP_EINVAL, "vsp_vs_aggregate: bad reduce");
    if (!workspace) return set_err(VSP_EINVAL, "vsp_vs_aggregate: workspace required");
    vsp_aggregate::Args a{q, k, n, hq, hkv, scale, lse, reduce == VSP_REDUCE_MEAN, normalized != 0, a_v, a_s};
    cudaError_t e = vsp_aggregate::launch(a, workspace, as_stream(stream));
    return e == cudaSuccess ? VSP_OK : cuda_err(e, "vsp_vs_aggregate");
}

}  // extern "C"

extern "C" int vsp_vs_attn_tile_stats(vsp_ctx* ctx, int n, int hkv, int cap, const void* workspace,
                                      int64_t* tiles_out, void* stream) {
    VSP_CHECK_CTX(ctx);
    if (!workspace || !tiles_out) return set_err(VSP_EINVAL, "vsp_vs_attn_tile_stats: null argument");
    std::vector<long long> t(2 + hkv);
    cudaError_t e = vsp_attn::sparse_tile_stats(n, hkv, cap, workspace, t.data(), as_stream(stream));
    if (e != cudaSuccess) return cuda_err(e, "vsp_vs_attn_tile_stats");
    for (int x = 0; x < 2 + hkv; ++x) tiles_out[x] = t[x];
    return VSP_OK;
}

// ------------------------------------------------------------------ fused layer
namespace {
size_t align256(size_t b) { return (b + 255) & ~size_t(255); }

// KV-head chunk schedule of the pipelined layer: hpc > 0 gives uniform chunks of hpc heads;
// hpc == 0 (automatic) uses two halves: the second half's scoring and selection overlap
// the first half's attention, and each attention launch still spans enough heads to
// balance its long and short CTAs (tools/sched_sweep.py: profiles/r01_schedule_sweep.json).
// Automatic schedule: one chunk. K3 is a persistent kernel that holds every SM, so the
// side-stream scoring of a later chunk (cluster launches need free SMs) could not overlap it
// anyway; chunking pays only where copies overlap compute (the host-buffer entry).
int auto_hpc(int hkv) { return hkv; }
// hpc < 0: a lead chunk of -hpc heads (its scoring is the only exposed part), then the rest
// as one chunk whose scoring overlaps the lead chunk's attention.
int num_chunks(int hkv, int hpc) {
    if (hpc < 0) return -hpc >= hkv ? 1 : 2;
    if (hpc == 0) hpc = auto_hpc(hkv);
    return (hkv + hpc - 1) / hpc;
}
void chunk_range(int c, int hkv, int hpc, int& g0, int& cnt) {
    if (hpc < 0) {
        const int lead = std::min(-hpc, hkv);
        g0 = c == 0 ? 0 : lead;
        cnt = c == 0 ? lead : hkv - lead;
        return;
    }
    if (hpc == 0) hpc = auto_hpc(hkv);
    g0 = c * hpc;
    cnt = std::min(hpc, hkv - g0);
}

struct PrefillDev {
    const void *q, *k, *v;
    const void* w_u;
    const float *b_u, *w_v, *b_v, *w_s, *b_s;
    float *a_v, *a_s;
    int *i_v, *k_v, *i_s, *k_s;
    void* o;
    float* lse;
    bool o_head_major;
    bool dense_switch = false;
    int n_mirrors = 0;                    // vsp_vs_prefill_mirrored: O / LSE also written here
    void* const* o_mirrors = nullptr;
    float* const* lse_mirrors = nullptr;
};

int check_prefill(int n, int hq, int hkv, int d, int d_h, int cap, int slash_mapping, const vsp_budget* budgets,
                  const void* workspace, int heads_per_chunk, const char* who) {
    int rc = check_attn_shapes(n, hq, hkv, d);
    if (rc) return rc;
    const std::string w(who);
    if (d_h < 1 || d_h % 256 != 0) return set_err(VSP_EINVAL, w + ": d_h must be a multiple of 256");
    if (cap < n + 1) return set_err(VSP_EINVAL, w + ": cap must be >= n + 1");
    if (!workspace || !budgets) return set_err(VSP_EINVAL, w + ": null workspace or budgets");
    if (hkv > 128) return set_err(VSP_EINVAL, w + ": at most 128 KV heads per call");
    if (slash_mapping != VSP_SLASH_REVERSE && slash_mapping != VSP_SLASH_IDENTITY)
        return set_err(VSP_EINVAL, w + ": bad slash mapping");
    for (int g = 0; g < hkv; ++g) {
        const vsp_budget& b = budgets[g];
        if (!(b.tau_v > 0.0 && b.tau_v <= 1.0)) return set_err(VSP_EINVAL, "budget config: tau_v must be in (0, 1]");
        if (!(b.tau_s > 0.0 && b.tau_s <= 1.0)) return set_err(VSP_EINVAL, "budget config: tau_s must be in (0, 1]");
        if (b.min_budget < 1) return set_err(VSP_EINVAL, "budget config: min_budget must be >= 1");
        if (b.max_budget >= 0 && b.min_budget > b.max_budget)
            return set_err(VSP_EINVAL, "budget config: min_budget exceeds max_budget");
    }
    if (num_chunks(hkv, heads_per_chunk) > vsp_ctx::kMaxChunks) return set_err(VSP_EINVAL, w + ": too many chunks");
    return VSP_OK;
}

// Query-block boundaries of the host-buffer entry's automatic schedule: 7/8 of the blocks in
// 14 equal ranges, the last 1/8 in halving ranges (1/16, 1/32, ... down to one block), so
// the exposed tail — the last range's attention and the D2H of its O rows — is one block.
std::vector<int> row_chunk_bounds(int num_qb) {
    std::vector<int> b{0};
    const int tail = num_qb / 8;
    const int head = num_qb - tail;
    const int heads = std::min(14, head);
    for (int c = 1; c <= heads; ++c) b.push_back(static_cast<int>(static_cast<long long>(head) * c / heads));
    int left = tail;
    while (left > 0) {
        const int piece = std::max(1, left / 2);
        b.push_back(b.back() + piece);
        left -= piece;
    }
    return b;  // at most 14 + log2(num_qb / 8) + 1 ranges
}

void* attn_workspace(void* workspace, int n, int hkv, int d_h) {
    uint8_t* ws = static_cast<uint8_t*>(workspace);
    ws += align256(vsp_indexer::workspace_bytes(n, hkv, d_h));
    ws += align256(vsp_select_k::workspace_bytes(n, hkv));
    return ws;
}

// K3 (attention phase) launch, bracketed by a timing event pair when vsp_attn_timing is on.
cudaError_t timed_attention(vsp_ctx* ctx, const vsp_attn::AttnArgs& aa, const vsp_attn::SparseArgs& sa, void* ws,
                            cudaStream_t st, int g0, int cnt, int qb_lo = 0, int qb_hi = -1) {
    const bool t = ctx->timing && ctx->timed < vsp_ctx::kTimingSlots;
    cudaError_t e = cudaSuccess;
    if (t) e = cudaEventRecord(ctx->t_beg[ctx->timed], st);
    if (e == cudaSuccess) e = vsp_attn::launch_sparse(aa, sa, ws, st, g0, cnt, 2, qb_lo, qb_hi);
    if (t && e == cudaSuccess) e = cudaEventRecord(ctx->t_end[ctx->timed++], st);
    return e;
}

// The attention of a list of units in one persistent launch, timed like timed_attention.
cudaError_t timed_attention_units(vsp_ctx* ctx, const vsp_attn::AttnArgs& aa, const vsp_attn::SparseArgs& sa,
                                  void* ws, cudaStream_t st, const vsp_unit* units, int nunits) {
    std::vector<int> tab(static_cast<size_t>(nunits) * 3);
    for (int u = 0; u < nunits; ++u) {
        tab[3 * u] = units[u].g;
        tab[3 * u + 1] = units[u].qb_lo;
        tab[3 * u + 2] = units[u].qb_hi;
    }
    const bool t = ctx->timing && ctx->timed < vsp_ctx::kTimingSlots;
    cudaError_t e = cudaSuccess;
    if (t) e = cudaEventRecord(ctx->t_beg[ctx->timed], st);
    if (e == cudaSuccess) e = vsp_attn::launch_sparse_units(aa, sa, ws, st, tab.data(), nunits);
    if (t && e == cudaSuccess) e = cudaEventRecord(ctx->t_end[ctx->timed++], st);
    return e;
}

// K1 (logits) -> K2 (softmax + selection) -> K3 plan for KV heads [g0, g0 + cnt) on `st`.
cudaError_t enqueue_scoring(const PrefillDev& p, int n, int hq, int hkv, int d, int d_h, int cap, int slash_mapping,
                            const vsp_budget* budgets, void* workspace, int g0, int cnt, cudaStream_t st) {
    uint8_t* ws = static_cast<uint8_t*>(workspace);
    void* ws_ix = ws;
    void* ws_sel = ws + align256(vsp_indexer::workspace_bytes(n, hkv, d_h));
    void* ws_attn = attn_workspace(workspace, n, hkv, d_h);
    float* lv = static_cast<float*>(ws_ix);  // logits [hkv, n] x 2 in the indexer workspace
    float* ls = lv + static_cast<size_t>(hkv) * n;
    // logits only (a_v null); the selection clusters softmax them and write A_v / A_s
    vsp_indexer::Args ia{p.k, p.v, n, hkv, d_h, p.w_u, p.b_u, p.w_v, p.b_v, p.w_s, p.b_s,
                         slash_mapping == VSP_SLASH_REVERSE, nullptr, nullptr, lv, ls, g0, cnt};
    cudaError_t e = vsp_indexer::launch(ia, ws_ix, st);
    if (e == cudaSuccess)
        e = vsp_select_k::launch_from_logits(lv, ls, p.a_v, p.a_s, n, hkv, budgets, p.i_v, p.k_v, p.i_s, p.k_s, cap,
                                             ws_sel, st, g0, cnt);
    vsp_attn::AttnArgs aa{p.q, p.k, p.v, p.o, p.lse, n, hq, hkv, 1.0f / sqrtf(static_cast<float>(d)), p.o_head_major};
    vsp_attn::SparseArgs sa{p.i_v, p.k_v, p.i_s, p.k_s, cap, p.dense_switch};
    if (e == cudaSuccess) e = vsp_attn::launch_sparse(aa, sa, ws_attn, st, g0, cnt, 1);
    return e;
}

// Enqueue K1 -> K2 -> plan on the side stream and K3 on `main`, chunk by chunk. Chunk c's
// scoring waits for kv_ready[c] and its attention for q_ready[c] (copy-engine events of
// the host-buffer entry; null = inputs already resident); attn_done[c] is recorded after
// chunk c's attention when non-null.
cudaError_t enqueue_prefill(vsp_ctx* ctx, const PrefillDev& p, int n, int hq, int hkv, int d, int d_h, int cap,
                            int slash_mapping, const vsp_budget* budgets, void* workspace, int hpc,
                            cudaStream_t main, const cudaEvent_t* kv_ready, const cudaEvent_t* q_ready,
                            const cudaEvent_t* attn_done) {
    const int chunks = num_chunks(hkv, hpc);
    void* ws_attn = attn_workspace(workspace, n, hkv, d_h);
    // One chunk on resident inputs: nothing to overlap (K3 is persistent and fills every SM),
    // so the whole layer runs in order on the caller's stream without the event hops.
    const bool serial = chunks == 1 && kv_ready == nullptr && q_ready == nullptr;
    cudaStream_t side = serial ? main : ctx->side;
    cudaError_t e = cudaSuccess;
    if (!serial) {
        e = cudaEventRecord(ctx->ev_start, main);
        if (e == cudaSuccess) e = cudaStreamWaitEvent(side, ctx->ev_start, 0);
    }
    vsp_attn::AttnArgs aa{p.q, p.k, p.v, p.o, p.lse, n, hq, hkv, 1.0f / sqrtf(static_cast<float>(d)), p.o_head_major};
    aa.n_mirrors = p.n_mirrors;
    aa.o_mirrors = p.o_mirrors;
    aa.lse_mirrors = p.lse_mirrors;
    vsp_attn::SparseArgs sa{p.i_v, p.k_v, p.i_s, p.k_s, cap, p.dense_switch};
    for (int c = 0; c < chunks && e == cudaSuccess; ++c) {
        int g0, cnt;
        chunk_range(c, hkv, hpc, g0, cnt);
        if (kv_ready) e = cudaStreamWaitEvent(side, kv_ready[c], 0);
        if (e == cudaSuccess)
            e = enqueue_scoring(p, n, hq, hkv, d, d_h, cap, slash_mapping, budgets, workspace, g0, cnt, side);
        if (e == cudaSuccess && !serial) e = cudaEventRecord(ctx->ev_chunk[c], side);
    }
    for (int c = 0; c < chunks && e == cudaSuccess; ++c) {
        int g0, cnt;
        chunk_range(c, hkv, hpc, g0, cnt);
        if (!serial) e = cudaStreamWaitEvent(main, ctx->ev_chunk[c], 0);
        if (e == cudaSuccess && q_ready) e = cudaStreamWaitEvent(main, q_ready[c], 0);
        if (e == cudaSuccess) e = timed_attention(ctx, aa, sa, ws_attn, main, g0, cnt);
        if (e == cudaSuccess && attn_done) e = cudaEventRecord(attn_done[c], main);
    }
    return e;
}

size_t host_staging_bytes(int n, int hq, int hkv, int cap) {
    const size_t row = 128 * 2;
    return align256(size_t(n) * hq * row) * 2 + align256(size_t(n) * hkv * row) * 2 +
           align256(size_t(hq) * n * 4) + align256(size_t(hkv) * n * 4) * 2 + align256(size_t(hkv) * cap * 4) * 2 +
           align256(size_t(hkv) * 4) * 2;
}
}  // namespace

extern "C" size_t vsp_vs_prefill_workspace_size(int n, int hkv, int d_h, int cap) {
    return align256(vsp_indexer::workspace_bytes(n, hkv, d_h)) + align256(vsp_select_k::workspace_bytes(n, hkv)) +
           align256(vsp_attn::sparse_workspace_bytes(n, hkv, cap));
}

extern "C" int vsp_vs_prefill(vsp_ctx* ctx, const void* q, const void* k, const void* v, int n, int hq, int hkv,
                              int d, int d_h, const void* w_u, const float* b_u, const float* w_v, const float* b_v,
                              const float* w_s, const float* b_s, int slash_mapping, const vsp_budget* budgets,
                              float* a_v, float* a_s, int* i_v, int* k_v, int* i_s, int* k_s, int cap, void* o,
                              float* lse, void* workspace, int heads_per_chunk, int flags, void* stream) {
    VSP_CHECK_CTX(ctx);
    int rc = check_prefill(n, hq, hkv, d, d_h, cap, slash_mapping, budgets, workspace, heads_per_chunk,
                           "vsp_vs_prefill");
    if (rc) return rc;
    if (flags & ~(VSP_O_HEAD_MAJOR | VSP_DENSE_SWITCH)) return set_err(VSP_EINVAL, "vsp_vs_prefill: unknown flags");
    PrefillDev p{q, k, v, w_u, b_u, w_v, b_v, w_s, b_s, a_v, a_s, i_v, k_v, i_s, k_s, o, lse,
                 (flags & VSP_O_HEAD_MAJOR) != 0, (flags & VSP_DENSE_SWITCH) != 0};
    cudaError_t e = enqueue_prefill(ctx, p, n, hq, hkv, d, d_h, cap, slash_mapping, budgets, workspace,
                                    heads_per_chunk, as_stream(stream), nullptr, nullptr,
                                    nullptr);
    return e == cudaSuccess ? VSP_OK : cuda_err(e, "vsp_vs_prefill");
}

extern "C" int vsp_vs_prefill_mirrored(vsp_ctx* ctx, const void* q, const void* k, const void* v, int n, int hq,
                                       int hkv, int d, int d_h, const void* w_u, const float* b_u, const float* w_v,
                                       const float* b_v, const float* w_s, const float* b_s, int slash_mapping,
                                       const vsp_budget* budgets, float* a_v, float* a_s, int* i_v, int* k_v,
                                       int* i_s, int* k_s, int cap, void* o, float* lse, void* workspace,
                                       int heads_per_chunk, int flags, int n_mirrors, void* const* o_mirrors,
                                       float* const* lse_mirrors, void* stream) {
    VSP_CHECK_CTX(ctx);
    int rc = check_prefill(n, hq, hkv, d, d_h, cap, slash_mapping, budgets, workspace, heads_per_chunk,
                           "vsp_vs_prefill_mirrored");
    if (rc) return rc;
    if (flags & ~(VSP_O_HEAD_MAJOR | VSP_DENSE_SWITCH))
        return set_err(VSP_EINVAL, "vsp_vs_prefill_mirrored: unknown flags");
    if (n_mirrors < 0 || n_mirrors > vsp_attn::kMaxMirrors)
        return set_err(VSP_EINVAL, "vsp_vs_prefill_mirrored: at most 7 mirrors");
    if (n_mirrors > 0 && o_mirrors == nullptr) return set_err(VSP_EINVAL, "vsp_vs_prefill_mirrored: null mirror list");
    for (int m = 0; m < n_mirrors; ++m) {
        if (o_mirrors[m] == nullptr) return set_err(VSP_EINVAL, "vsp_vs_prefill_mirrored: null O mirror");
        if ((lse == nullptr) != (lse_mirrors == nullptr || lse_mirrors[m] == nullptr))
            return set_err(VSP_EINVAL, "vsp_vs_prefill_mirrored: LSE mirrors must match lse");
    }
    PrefillDev p{q, k, v, w_u, b_u, w_v, b_v, w_s, b_s, a_v, a_s, i_v, k_v, i_s, k_s, o, lse,
                 (flags & VSP_O_HEAD_MAJOR) != 0, (flags & VSP_DENSE_SWITCH) != 0};
    p.n_mirrors = n_mirrors;
    p.o_mirrors = o_mirrors;
    p.lse_mirrors = lse_mirrors;
    cudaError_t e = enqueue_prefill(ctx, p, n, hq, hkv, d, d_h, cap, slash_mapping, budgets, workspace,
                                    heads_per_chunk, as_stream(stream), nullptr, nullptr, nullptr);
    return e == cudaSuccess ? VSP_OK : cuda_err(e, "vsp_vs_prefill_mirrored");
}

// ---- CUDA IPC: device buffers another process (a peer GPU's rank) can map
extern "C" int vsp_ipc_alloc(vsp_ctx* ctx, size_t bytes, void** ptr, unsigned char* handle) {
    VSP_CHECK_CTX(ctx);
    if (!ptr || !handle || bytes == 0) return set_err(VSP_EINVAL, "vsp_ipc_alloc: bad arguments");
    cudaError_t e = cudaSetDevice(ctx->device);
    if (e == cudaSuccess) e = cudaMalloc(ptr, bytes);
    cudaIpcMemHandle_t h;
    if (e == cudaSuccess) e = cudaIpcGetMemHandle(&h, *ptr);
    if (e != cudaSuccess) return cuda_err(e, "vsp_ipc_alloc");
    std::memcpy(handle, &h, sizeof(h));
    return VSP_OK;
}

extern "C" int vsp_ipc_open(vsp_ctx* ctx, const unsigned char* handle, void** ptr) {
    VSP_CHECK_CTX(ctx);
    if (!ptr || !handle) return set_err(VSP_EINVAL, "vsp_ipc_open: bad arguments");
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle, sizeof(h));
    cudaError_t e = cudaSetDevice(ctx->device);
    if (e == cudaSuccess) e = cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess);
    return e == cudaSuccess ? VSP_OK : cuda_err(e, "vsp_ipc_open");
}

extern "C" int vsp_ipc_close(void* ptr) {
    const cudaError_t e = cudaIpcCloseMemHandle(ptr);
    return e == cudaSuccess ? VSP_OK : cuda_err(e, "vsp_ipc_close");
}

extern "C" int vsp_ipc_free(void* ptr) {
    const cudaError_t e = cudaFree(ptr);
    return e == cudaSuccess ? VSP_OK : cuda_err(e, "vsp_ipc_free");
}

// per (KV head, query block) tile counts of the last plan on `workspace` -> host [hkv, num_qb]
namespace {
__global__ void tile_counts_kernel(const int* lists, int total, int list_stride, int* out) {
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < total; t += gridDim.x * blockDim.x)
        out[t] = lists[static_cast<size_t>(t) * list_stride];
}
}  // namespace

extern "C" int vsp_vs_attn_tile_counts(vsp_ctx* ctx, int n, int hkv, int cap, const void* workspace, int32_t* counts,
                                       void* stream) {
    VSP_CHECK_CTX(ctx);
    if (!workspace || !counts || n < 1 || hkv < 1) return set_err(VSP_EINVAL, "vsp_vs_attn_tile_counts: bad arguments");
    const int num_qb = (n + 127) / 128;
    const int kvcap = ((cap + 127) / 128) * 128;
    const int bm_words = (n + 31) / 32 + 1;
    const int list_stride = 2 + kvcap / 128 + num_qb + 3;
    size_t off = 0;
    auto skip = [&](size_t b) { off += (b + 255) & ~size_t(255); };
    skip(static_cast<size_t>(hkv) * kvcap * 128 * 2);
    skip(static_cast<size_t>(hkv) * kvcap * 128 * 2);
    skip(static_cast<size_t>(hkv) * bm_words * 4 * 2);
    const int* lists = reinterpret_cast<const int*>(static_cast<const uint8_t*>(workspace) + off);
    cudaStream_t st = as_stream(stream);
    int* d = nullptr;
    const int total = hkv * num_qb;
    cudaError_t e = cudaMallocAsync(&d, sizeof(int) * total, st);
    if (e != cudaSuccess) return cuda_err(e, "vsp_vs_attn_tile_counts");
    vsp_detail::count_launch();
    tile_counts_kernel<<<(total + 255) / 256, 256, 0, st>>>(lists, total, list_stride, d);
    e = cudaMemcpyAsync(counts, d, sizeof(int) * total, cudaMemcpyDeviceToHost, st);
    cudaFreeAsync(d, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    return e == cudaSuccess ? VSP_OK : cuda_err(e, "vsp_vs_attn_tile_counts");
}

// Balanced multi-GPU split (SURVEY.md §8e refinement): score + select + plan the distinct KV
// heads of `units`, then attend each unit's query-block range. Collective-free; units of
// different ranks write disjoint (head, row) regions of O / LSE.
extern "C" int vsp_vs_prefill_units(vsp_ctx* ctx, const void* q, const void* k, const void* v, int n, int hq, int hkv,
                                    int d, int d_h, const void* w_u, const float* b_u, const float* w_v,
                                    const float* b_v, const float* w_s, const float* b_s, int slash_mapping,
                                    const vsp_budget* budgets, float* a_v, float* a_s, int* i_v, int* k_v, int* i_s,
                                    int* k_s, int cap, void* o, float* lse, void* workspace, const vsp_unit* units,
                                    int nunits, int flags, void* stream) {
    VSP_CHECK_CTX(ctx);
    int rc = check_prefill(n, hq, hkv, d, d_h, cap, slash_mapping, budgets, workspace, 0, "vsp_vs_prefill_units");
    if (rc) return rc;
    if (flags & ~(VSP_O_HEAD_MAJOR | VSP_DENSE_SWITCH))
        return set_err(VSP_EINVAL, "vsp_vs_prefill_units: unknown flags");
    if (nunits < 0 || (nunits > 0 && !units)) return set_err(VSP_EINVAL, "vsp_vs_prefill_units: bad units");
    if (nunits > vsp_attn::kMaxUnits) return set_err(VSP_EINVAL, "vsp_vs_prefill_units: at most 512 units per call");
    const int num_qb = (n + 127) / 128;
    std::vector<char> touched(hkv, 0);
    for (int u = 0; u < nunits; ++u) {
        const vsp_unit& x = units[u];
        if (x.g < 0 || x.g >= hkv || x.qb_lo < 0 || x.qb_hi > num_qb || x.qb_lo > x.qb_hi)
            return set_err(VSP_EINVAL, "vsp_vs_prefill_units: unit out of range");
        touched[x.g] = 1;
    }
    uint8_t* ws = static_cast<uint8_t*>(workspace);
    void* ws_ix = ws;
    ws += align256(vsp_indexer::workspace_bytes(n, hkv, d_h));
    void* ws_sel = ws;
    ws += align256(vsp_select_k::workspace_bytes(n, hkv));
    void* ws_attn = ws;
    float* lv = static_cast<float*>(ws_ix);
    float* ls = lv + static_cast<size_t>(hkv) * n;
    cudaStream_t st = as_stream(stream);
    vsp_attn::AttnArgs aa{q, k, v, o, lse, n, hq, hkv, 1.0f / sqrtf(static_cast<float>(d)),
                          (flags & VSP_O_HEAD_MAJOR) != 0};
    vsp_attn::SparseArgs sa{i_v, k_v, i_s, k_s, cap, (flags & VSP_DENSE_SWITCH) != 0};
    cudaError_t e = cudaSuccess;
    // score, select and plan each contiguous run of touched heads with one launch per kernel
    for (int g = 0; g < hkv && e == cudaSuccess;) {
        if (!touched[g]) {
            ++g;
            continue;
        }
        int cnt = 1;
        while (g + cnt < hkv && touched[g + cnt]) ++cnt;
        vsp_indexer::Args ia{k, v, n, hkv, d_h, w_u, b_u, w_v, b_v, w_s, b_s, slash_mapping == VSP_SLASH_REVERSE,
                             nullptr, nullptr, lv, ls, g, cnt};
        e = vsp_indexer::launch(ia, ws_ix, st);
        if (e == cudaSuccess)
            e = vsp_select_k::launch_from_logits(lv, ls, a_v, a_s, n, hkv, budgets, i_v, k_v, i_s, k_s, cap, ws_sel,
                                                 st, g, cnt);
        if (e == cudaSuccess) e = vsp_attn::launch_sparse(aa, sa, ws_attn, st, g, cnt, 1);
        g += cnt;
    }
    // all units' attention in one persistent launch (one work queue across the units)
    if (e == cudaSuccess && nunits > 0) e = timed_attention_units(ctx, aa, sa, ws_attn, st, units, nunits);
    return e == cudaSuccess ? VSP_OK : cuda_err(e, "vsp_vs_prefill_units");
}

extern "C" size_t vsp_vs_prefill_host_workspace_size(int n, int hq, int hkv, int d_h) {
    const int cap = n + 1;
    return vsp_vs_prefill_workspace_size(n, hkv, d_h, cap) + host_staging_bytes(n, hq, hkv, cap);
}

extern "C" int vsp_vs_prefill_host(vsp_ctx* ctx, const void* q_h, const void* k_h, const void* v_h, int n, int hq,
                                   int hkv, int d, int d_h, const void* w_u, const float* b_u, const float* w_v,
                                   const float* b_v, const float* w_s, const float* b_s, int slash_mapping,
                                   const vsp_budget* budgets, void* o_h, float* lse_h, int* k_v_h, int* k_s_h,
                                   void* workspace, int heads_per_chunk, void* stream) {
    VSP_CHECK_CTX(ctx);
    const int cap = n + 1;
    int rc = check_prefill(n, hq, hkv, d, d_h, cap, slash_mapping, budgets, workspace, heads_per_chunk,
                           "vsp_vs_prefill_host");
    if (rc) return rc;
    if (!q_h || !k_h || !v_h || !o_h) return set_err(VSP_EINVAL, "vsp_vs_prefill_host: null host buffer");
    const int hpc = heads_per_chunk;
    const int chunks = num_chunks(hkv, hpc), grp = hq / hkv;
    const size_t row = 128 * 2;
    // device staging after the prefill workspace
    uint8_t* base = static_cast<uint8_t*>(workspace);
    uint8_t* s = base + vsp_vs_prefill_workspace_size(n, hkv, d_h, cap);
    auto take = [&](size_t bytes) {
        uint8_t* r = s;
        s += align256(bytes);
        return r;
    };
    uint8_t* q_d = take(size_t(n) * hq * row);
    uint8_t* o_d = take(size_t(n) * hq * row);
    uint8_t* k_d = take(size_t(n) * hkv * row);
    uint8_t* v_d = take(size_t(n) * hkv * row);
    float* lse_d = reinterpret_cast<float*>(take(size_t(hq) * n * 4));
    float* av_d = reinterpret_cast<float*>(take(size_t(hkv) * n * 4));
    float* as_d = reinterpret_cast<float*>(take(size_t(hkv) * n * 4));
    int* iv_d = reinterpret_cast<int*>(take(size_t(hkv) * cap * 4));
    int* is_d = reinterpret_cast<int*>(take(size_t(hkv) * cap * 4));
    int* kv_d = reinterpret_cast<int*>(take(size_t(hkv) * 4));
    int* ks_d = reinterpret_cast<int*>(take(size_t(hkv) * 4));

    cudaStream_t main = as_stream(stream);
    cudaError_t e = cudaEventRecord(ctx->ev_host0, main);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(ctx->h2d, ctx->ev_host0, 0);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(ctx->d2h, ctx->ev_host0, 0);
    PrefillDev p{q_d, k_d, v_d, w_u, b_u, w_v, b_v, w_s, b_s, av_d, as_d, iv_d, kv_d, is_d, ks_d, o_d, lse_d, false};
    if (hpc == 0) {
        // Query-row pipeline (automatic schedule): K and V go first as two contiguous copies
        // (the scoring softmaxes over all n rows), then Q in row ranges; the attention of a
        // range runs as soon as its Q rows land and its O rows / LSE columns go back while
        // later Q ranges are still in flight. Every copy is a long contiguous run.
        const std::vector<int> bounds = row_chunk_bounds((n + 127) / 128);
        const int rc_chunks = static_cast<int>(bounds.size()) - 1;
        auto rows_of = [&](int c, int& qb_lo, int& qb_hi) {
            qb_lo = bounds[c];
            qb_hi = bounds[c + 1];
        };
        const size_t kv_bytes = size_t(n) * hkv * row, q_row = size_t(hq) * row;
        e = cudaMemcpyAsync(k_d, k_h, kv_bytes, cudaMemcpyHostToDevice, ctx->h2d);
        if (e == cudaSuccess) e = cudaMemcpyAsync(v_d, v_h, kv_bytes, cudaMemcpyHostToDevice, ctx->h2d);
        if (e == cudaSuccess) e = cudaEventRecord(ctx->ev_kv[0], ctx->h2d);
        for (int c = 0; c < rc_chunks && e == cudaSuccess; ++c) {
            int lo, hi;
            rows_of(c, lo, hi);
            const size_t r0 = size_t(lo) * 128, r1 = std::min(size_t(hi) * 128, size_t(n));
            e = cudaMemcpyAsync(q_d + r0 * q_row, static_cast<const uint8_t*>(q_h) + r0 * q_row, (r1 - r0) * q_row,
                                cudaMemcpyHostToDevice, ctx->h2d);
            if (e == cudaSuccess) e = cudaEventRecord(ctx->ev_q[c], ctx->h2d);
        }
        if (e == cudaSuccess) e = cudaStreamWaitEvent(main, ctx->ev_kv[0], 0);
        if (e == cudaSuccess)
            e = enqueue_scoring(p, n, hq, hkv, d, d_h, cap, slash_mapping, budgets, workspace, 0, hkv, main);
        vsp_attn::AttnArgs aa{p.q, p.k, p.v, p.o, p.lse, n, hq, hkv, 1.0f / sqrtf(static_cast<float>(d)), false};
        vsp_attn::SparseArgs sa{p.i_v, p.k_v, p.i_s, p.k_s, cap, p.dense_switch};
        void* ws_attn = attn_workspace(workspace, n, hkv, d_h);
        for (int c = 0; c < rc_chunks && e == cudaSuccess; ++c) {
            int lo, hi;
            rows_of(c, lo, hi);
            e = cudaStreamWaitEvent(main, ctx->ev_q[c], 0);
            if (e == cudaSuccess) e = timed_attention(ctx, aa, sa, ws_attn, main, 0, hkv, lo, hi);
            if (e == cudaSuccess) e = cudaEventRecord(ctx->ev_attn[c], main);
        }
        for (int c = 0; c < rc_chunks && e == cudaSuccess; ++c) {
            int lo, hi;
            rows_of(c, lo, hi);
            const size_t r0 = size_t(lo) * 128, r1 = std::min(size_t(hi) * 128, size_t(n));
            e = cudaStreamWaitEvent(ctx->d2h, ctx->ev_attn[c], 0);
            if (e == cudaSuccess)
                e = cudaMemcpyAsync(static_cast<uint8_t*>(o_h) + r0 * q_row, o_d + r0 * q_row, (r1 - r0) * q_row,
                                    cudaMemcpyDeviceToHost, ctx->d2h);
            if (e == cudaSuccess && lse_h)  // LSE [hq, n]: columns [r0, r1) of every head row
                e = cudaMemcpy2DAsync(lse_h + r0, size_t(n) * 4, lse_d + r0, size_t(n) * 4, (r1 - r0) * 4, hq,
                                      cudaMemcpyDeviceToHost, ctx->d2h);
        }
    } else {
    // H2D per chunk: this chunk's K and V columns (strided rows of cnt heads), then its Q heads
    const uint8_t* qh = static_cast<const uint8_t*>(q_h);
    const uint8_t* kh = static_cast<const uint8_t*>(k_h);
    const uint8_t* vh = static_cast<const uint8_t*>(v_h);
    for (int c = 0; c < chunks && e == cudaSuccess; ++c) {
        int g0, cnt;
        chunk_range(c, hkv, hpc, g0, cnt);
        const size_t kvoff = size_t(g0) * row, kvw = size_t(cnt) * row, kvp = size_t(hkv) * row;
        e = cudaMemcpy2DAsync(k_d + kvoff, kvp, kh + kvoff, kvp, kvw, n, cudaMemcpyHostToDevice, ctx->h2d);
        if (e == cudaSuccess)
            e = cudaMemcpy2DAsync(v_d + kvoff, kvp, vh + kvoff, kvp, kvw, n, cudaMemcpyHostToDevice, ctx->h2d);
        if (e == cudaSuccess) e = cudaEventRecord(ctx->ev_kv[c], ctx->h2d);
        const size_t qoff = size_t(g0) * grp * row, qw = size_t(cnt) * grp * row, qp = size_t(hq) * row;
        if (e == cudaSuccess)
            e = cudaMemcpy2DAsync(q_d + qoff, qp, qh + qoff, qp, qw, n, cudaMemcpyHostToDevice, ctx->h2d);
        if (e == cudaSuccess) e = cudaEventRecord(ctx->ev_q[c], ctx->h2d);
    }
    if (e == cudaSuccess)
        e = enqueue_prefill(ctx, p, n, hq, hkv, d, d_h, cap, slash_mapping, budgets, workspace, hpc, main, ctx->ev_kv,
                            ctx->ev_q, ctx->ev_attn);
    // D2H per chunk as its attention lands: O columns, LSE rows
    uint8_t* oh = static_cast<uint8_t*>(o_h);
    for (int c = 0; c < chunks && e == cudaSuccess; ++c) {
        int g0, cnt;
        chunk_range(c, hkv, hpc, g0, cnt);
        const size_t qoff = size_t(g0) * grp * row, qw = size_t(cnt) * grp * row, qp = size_t(hq) * row;
        e = cudaStreamWaitEvent(ctx->d2h, ctx->ev_attn[c], 0);
        if (e == cudaSuccess)
            e = cudaMemcpy2DAsync(oh + qoff, qp, o_d + qoff, qp, qw, n, cudaMemcpyDeviceToHost, ctx->d2h);
        if (e == cudaSuccess && lse_h)
            e = cudaMemcpyAsync(lse_h + size_t(g0) * grp * n, lse_d + size_t(g0) * grp * n,
                                size_t(cnt) * grp * n * 4, cudaMemcpyDeviceToHost, ctx->d2h);
    }
    }
    if (e == cudaSuccess && k_v_h) e = cudaMemcpyAsync(k_v_h, kv_d, size_t(hkv) * 4, cudaMemcpyDeviceToHost, ctx->d2h);
    if (e == cudaSuccess && k_s_h) e = cudaMemcpyAsync(k_s_h, ks_d, size_t(hkv) * 4, cudaMemcpyDeviceToHost, ctx->d2h);
    if (e == cudaSuccess) e = cudaEventRecord(ctx->ev_host1, ctx->d2h);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(main, ctx->ev_host1, 0);
    return e == cudaSuccess ? VSP_OK : cuda_err(e, "vsp_vs_prefill_host");
}

// ------------------------------------------------------------------ live K3 timing
extern "C" int vsp_attn_timing(vsp_ctx* ctx, int enable) {
    VSP_CHECK_CTX(ctx);
    for (int i = 0; enable && i < vsp_ctx::kTimingSlots; ++i) {
        for (cudaEvent_t* ev : {&ctx->t_beg[i], &ctx->t_end[i]}) {
            if (*ev) continue;
            const cudaError_t e = cudaEventCreate(ev);
            if (e != cudaSuccess) return cuda_err(e, "vsp_attn_timing");
        }
    }
    ctx->timing = enable != 0;
    ctx->timed = 0;
    return VSP_OK;
}

extern "C" int vsp_attn_timing_read(vsp_ctx* ctx, double* total_ms, int* launches) {
    VSP_CHECK_CTX(ctx);
    if (!total_ms || !launches) return set_err(VSP_EINVAL, "vsp_attn_timing_read: null output");
    double sum = 0.0;
    for (int i = 0; i < ctx->timed; ++i) {
        cudaError_t e = cudaEventSynchronize(ctx->t_end[i]);
        float ms = 0.f;
        if (e == cudaSuccess) e = cudaEventElapsedTime(&ms, ctx->t_beg[i], ctx->t_end[i]);
        if (e != cudaSuccess) return cuda_err(e, "vsp_attn_timing_read");
        sum += ms;
    }
    *total_ms = sum;
    *launches = ctx->timed;
    ctx->timed = 0;
    return VSP_OK;
}
