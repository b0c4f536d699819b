// mma_rate.cu — tcgen05.mma issue-rate probe (M = 128, cta_group::1, bf16 -> fp32):
// clocks per instruction for SS (A and B from shared memory) and TS (A from TMEM) at
// N = 16 ... 256, one CTA per SM, one elected thread issuing back-to-back MMAs into one
// accumulator. Decides whether narrow (N < 128) tiles save tensor time in K3.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/mma_rate.cu -o mma_rate
#include "../paper_2603_04460_b200/csrc/sm100.cuh"

#include <cstdio>

using namespace vsp_sm100;

__global__ void __launch_bounds__(128, 1) rate_kernel(int n_mma, int N, int ts, unsigned long long* out, int bmn = 0) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t bar;
    __shared__ uint32_t tmem_base_s;
    const uint32_t warp = warp_id();
    // deterministic finite operands (timing does not depend on the values)
    for (int i = threadIdx.x; i < 96 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;
    fence_proxy_async_smem();
    if (warp == 0) tmem_alloc<512>(&tmem_base_s);
    if (threadIdx.x == 32) {
        mbar_init(&bar, 1);
        fence_barrier_init();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tmem_base_s;
    if (warp == 0) {
        const uint32_t idesc = umma_idesc_bf16(128, N, false, bmn != 0);
        const uint64_t a = umma_desc_sw128(smem_u32(smem), 16, 1024);
        const uint64_t b = umma_desc_sw128(smem_u32(smem + 32768), 16, 1024);
        unsigned long long t0 = 0, t1 = 0;
        if (elect_one()) {
            t0 = clock64();
            for (int i = 0; i < n_mma; ++i) {
                const uint64_t off = static_cast<uint64_t>(((i & 3) * 32) >> 4);
                if (ts) umma_ts(tmem + 256, tmem + 0 + (i & 7) * 8, b + off, idesc, 1u);
                else umma_ss(tmem + 256, a + off, b + off, idesc, 1u);
            }
            umma_commit(&bar);
            mbar_wait(&bar, 0);
            t1 = clock64();
            out[blockIdx.x] = t1 - t0;
        }
        __syncwarp();
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_free<512>(tmem);
}

int main() {
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    unsigned long long* d;
    cudaMalloc(&d, sizeof(unsigned long long) * sms);
    const int smem = 96 * 1024 + 1024;
    cudaFuncSetAttribute(rate_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int n_mma = 20000;
    printf("{\"probe\": \"tcgen05.mma M=128 cta_group::1 bf16, back-to-back into one accumulator, %d instr, %d CTAs\", \"rows\": [", n_mma, sms);
    bool first = true;
    for (int mode = 0; mode < 4; ++mode)
        for (int N : {16, 32, 64, 96, 128, 192, 256}) {
            const int ts = mode & 1, bmn = mode >> 1;
            rate_kernel<<<sms, 128, smem>>>(n_mma, N, ts, d, bmn);
            rate_kernel<<<sms, 128, smem>>>(n_mma, N, ts, d, bmn);
            cudaError_t e = cudaDeviceSynchronize();
            unsigned long long h[1024];
            cudaMemcpy(h, d, sizeof(unsigned long long) * sms, cudaMemcpyDeviceToHost);
            unsigned long long mx = 0;
            for (int i = 0; i < sms; ++i) mx = h[i] > mx ? h[i] : mx;
            printf("%s{\"form\": \"%s%s\", \"N\": %d, \"clk_per_mma\": %.2f, \"floor_formula\": %.1f, \"err\": \"%s\"}",
                   first ? "" : ", ", ts ? "TS" : "SS", bmn ? "-Bmn" : "", N, double(mx) / n_mma, 128.0 * N / 256.0, cudaGetErrorString(e));
            first = false;
        }
    printf("]}\n");
    return 0;
}
