// Probe: validates the hand-written UMMA/TMA/TMEM conventions in sm100.cuh on one tile.
//   S = Q K^T   (SS MMA, K-major both, SWIZZLE_128B, 3-D TMA over [n, H, d])
//   P = bf16(S * pscale) written to TMEM, O = P V (TS MMA, V MN-major)
#include "../paper_2603_04460_b200/csrc/sm100.cuh"
#include "../paper_2603_04460_b200/csrc/tma_host.h"

#include <cstdio>

using namespace vsp_sm100;

struct __align__(64) ProbeMaps {
    CUtensorMap q, k, v;
};

__global__ void __launch_bounds__(128, 1)
    probe_kernel(const __grid_constant__ ProbeMaps maps, int q_head, float pscale, float* s_out,
                 float* o_out) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sQ = smem;
    uint8_t* sK = smem + 32768;
    uint8_t* sV = smem + 65536;
    __shared__ uint64_t bar_load, bar_mma1, bar_mma2;
    __shared__ uint32_t tmem_base_s;

    const uint32_t warp = warp_id();
    if (warp == 0) tmem_alloc<512>(&tmem_base_s);
    if (threadIdx.x == 32) {
        mbar_init(&bar_load, 1);
        mbar_init(&bar_mma1, 1);
        mbar_init(&bar_mma2, 1);
        fence_barrier_init();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tmem_base_s;

    if (threadIdx.x == 0) {
        mbar_arrive_expect_tx(&bar_load, 3 * 32768);
        for (int h = 0; h < 2; ++h) {
            tma_load_3d(sQ + h * 16384, &maps.q, &bar_load, h * 64, q_head, 0);
            tma_load_3d(sK + h * 16384, &maps.k, &bar_load, h * 64, 0, 0);
            tma_load_3d(sV + h * 16384, &maps.v, &bar_load, h * 64, 0, 0);
        }
    }
    mbar_wait(&bar_load, 0);

    if (threadIdx.x == 0) {
        tc_fence_after();
        const uint32_t idesc = umma_idesc_bf16(128, 128, false, false);
        for (int k = 0; k < 8; ++k) {
            const uint32_t off = (k >> 2) * 16384 + (k & 3) * 32;
            uint64_t a = umma_desc_sw128(smem_u32(sQ) + off, 16, 1024);
            uint64_t b = umma_desc_sw128(smem_u32(sK) + off, 16, 1024);
            umma_ss(tmem + 0, a, b, idesc, k > 0);
        }
        umma_commit(&bar_mma1);
    }
    mbar_wait(&bar_mma1, 0);
    tc_fence_after();

    const uint32_t row = warp * 32 + lane_id();
    const uint32_t lane_addr = tmem + ((warp * 32u) << 16);
    for (int c = 0; c < 4; ++c) {
        uint32_t r[32];
        tmem_ld32(lane_addr + c * 32, r);
        tmem_wait_ld();
        uint32_t p[16];
        for (int i = 0; i < 32; ++i) s_out[row * 128 + c * 32 + i] = __uint_as_float(r[i]);
        for (int i = 0; i < 16; ++i)
            p[i] = pack_bf16x2(__uint_as_float(r[2 * i]) * pscale, __uint_as_float(r[2 * i + 1]) * pscale);
        tmem_st16(lane_addr + 256 + c * 16, p);
    }
    tmem_wait_st();
    tc_fence_before();
    __syncthreads();

    if (threadIdx.x == 0) {
        tc_fence_after();
        const uint32_t idesc = umma_idesc_bf16(128, 128, false, true);
        for (int k = 0; k < 8; ++k) {
            uint64_t b = umma_desc_sw128(smem_u32(sV) + k * 2048, 16384, 1024);
            umma_ts(tmem + 128, tmem + 256 + k * 8, b, idesc, k > 0);
        }
        umma_commit(&bar_mma2);
    }
    mbar_wait(&bar_mma2, 0);
    tc_fence_after();
    for (int c = 0; c < 4; ++c) {
        uint32_t r[32];
        tmem_ld32(lane_addr + 128 + c * 32, r);
        tmem_wait_ld();
        for (int i = 0; i < 32; ++i) o_out[row * 128 + c * 32 + i] = __uint_as_float(r[i]);
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_free<512>(tmem);
}

// q: [128, Hq, 128] bf16, k/v: [128, 1, 128] bf16 (device). Returns cudaError as int.
extern "C" int probe_run(const void* q, int hq, int q_head, const void* k, const void* v,
                         float pscale, float* s_out, float* o_out) {
    ProbeMaps maps;
    uint64_t dq[3] = {128, (uint64_t)hq, 128};
    uint64_t sq[2] = {128 * 2, (uint64_t)hq * 128 * 2};
    uint64_t dk[3] = {128, 1, 128};
    uint64_t sk[2] = {128 * 2, 128 * 2};
    uint32_t box[3] = {64, 1, 128};
    if (!vsp_host::make_map_bf16(&maps.q, q, 3, dq, sq, box)) return -1;
    if (!vsp_host::make_map_bf16(&maps.k, k, 3, dk, sk, box)) return -2;
    if (!vsp_host::make_map_bf16(&maps.v, v, 3, dk, sk, box)) return -3;
    const int smem = 3 * 32768 + 1024;
    cudaFuncSetAttribute(probe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    probe_kernel<<<1, 128, smem>>>(maps, q_head, pscale, s_out, o_out);
    cudaError_t e = cudaDeviceSynchronize();
    return (int)e;
}
