// mma_rate2.cu — tcgen05.mma issue rate with cta_group::2 (M = 256 over a CTA pair, each SM
// holds 128 rows of A and half of B's N columns) vs the cta_group::1 numbers of mma_rate.cu.
// Per-SM work per instruction is the same 128 x N x 16 as the 1-CTA probe, so clocks per
// instruction compare directly. Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/mma_rate2.cu -o tools/mma_rate2
#include "../paper_2603_04460_b200/csrc/sm100.cuh"

#include <cstdio>

using namespace vsp_sm100;

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1)
    rate2_kernel(int n_mma, int N, int ts, unsigned long long* out) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t bar;
    __shared__ uint32_t tmem_base_s;
    const uint32_t warp = warp_id();
    const uint32_t rank = cluster_ctarank();
    for (int i = threadIdx.x; i < 96 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;
    fence_proxy_async_smem();
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tmem_base_s)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
    if (threadIdx.x == 32) {
        mbar_init(&bar, 1);
        fence_barrier_init();
    }
    tc_fence_before();
    __syncthreads();
    cluster_sync();
    tc_fence_after();
    const uint32_t tmem = tmem_base_s;
    if (warp == 0 && rank == 0) {
        const uint32_t idesc = umma_idesc_bf16(256, N, false, false);
        const uint64_t a = umma_desc_sw128(smem_u32(smem), 16, 1024);
        const uint64_t b = umma_desc_sw128(smem_u32(smem + 32768), 16, 1024);
        unsigned long long t0 = 0, t1 = 0;
        if (elect_one()) {
            t0 = clock64();
            for (int i = 0; i < n_mma; ++i) {
                const uint64_t off = static_cast<uint64_t>(((i & 3) * 32) >> 4);
                if (ts)
                    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                                 "tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem + 256),
                                 "r"(tmem + (i & 7) * 8), "l"(b + off), "r"(idesc), "r"(1u));
                else
                    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                                 "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem + 256),
                                 "l"(a + off), "l"(b + off), "r"(idesc), "r"(1u));
            }
            asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
                         ::"r"(smem_u32(&bar)), "h"(static_cast<uint16_t>(1)) : "memory");
            mbar_wait(&bar, 0);
            t1 = clock64();
            out[blockIdx.x / 2] = t1 - t0;
        }
        __syncwarp();
    }
    tc_fence_before();
    __syncthreads();
    cluster_sync();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

int main() {
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int pairs = sms / 2;
    unsigned long long* d;
    cudaMalloc(&d, sizeof(unsigned long long) * pairs);
    const int smem = 96 * 1024 + 1024;
    cudaFuncSetAttribute(rate2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int n_mma = 20000;
    printf("{\"probe\": \"tcgen05.mma M=256 cta_group::2 bf16 (per SM: 128 x N x 16), %d instr, %d pairs\", \"rows\": [",
           n_mma, pairs);
    bool first = true;
    for (int ts = 0; ts < 2; ++ts)
        for (int N : {64, 128, 256}) {
            rate2_kernel<<<2 * pairs, 128, smem>>>(n_mma, N, ts, d);
            rate2_kernel<<<2 * pairs, 128, smem>>>(n_mma, N, ts, d);
            cudaError_t e = cudaDeviceSynchronize();
            unsigned long long h[1024];
            cudaMemcpy(h, d, sizeof(unsigned long long) * pairs, cudaMemcpyDeviceToHost);
            unsigned long long mx = 0;
            for (int i = 0; i < pairs; ++i) mx = h[i] > mx ? h[i] : mx;
            printf("%s{\"form\": \"%s\", \"N\": %d, \"clk_per_mma\": %.2f, \"floor_per_sm\": %.1f, \"err\": \"%s\"}",
                   first ? "" : ", ", ts ? "TS" : "SS", N, double(mx) / n_mma, 128.0 * N / 256.0, cudaGetErrorString(e));
            first = false;
        }
    printf("]}\n");
    return 0;
}
