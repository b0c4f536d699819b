// MUFU throughput probe: clocks per warp instruction per SM sub-partition for tanh.approx.f32,
// ex2.approx.f32, rcp.approx.f32 and tanh.approx.bf16x2 (16 warps per SM, 8 independent chains
// per thread). nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/mufu_rate.cu -o mufu_rate
#include <cstdio>
#include <cuda_bf16.h>

template <int OP>
__global__ void probe(float* out, long long* clk, int iters) {
    float x[8];
    for (int j = 0; j < 8; ++j) x[j] = 0.001f * (threadIdx.x + j);
    __syncthreads();
    const long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            float y;
            if (OP == 0) asm volatile("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x[j]));
            if (OP == 1) asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x[j]));
            if (OP == 2) asm volatile("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x[j]));
            if (OP == 3) {
                unsigned u = __float_as_uint(x[j]), v;
                asm volatile("tanh.approx.bf16x2 %0, %1;" : "=r"(v) : "r"(u));
                y = __uint_as_float(v);
            }
            x[j] = y;
        }
    }
    __syncthreads();
    const long long t1 = clock64();
    float s = 0.f;
    for (int j = 0; j < 8; ++j) s += x[j];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
}

template <int OP>
void run(const char* name, int sms) {
    float* out;
    long long* clk;
    cudaMalloc(&out, sms * 512 * sizeof(float));
    cudaMalloc(&clk, sms * sizeof(long long));
    const int iters = 4096;
    probe<OP><<<sms, 512>>>(out, clk, iters);
    probe<OP><<<sms, 512>>>(out, clk, iters);
    cudaDeviceSynchronize();
    long long h[1024];
    cudaMemcpy(h, clk, sms * sizeof(long long), cudaMemcpyDeviceToHost);
    long long mx = 0;
    for (int i = 0; i < sms; ++i) mx = h[i] > mx ? h[i] : mx;
    // 16 warps x iters x 8 instructions per SM, 4 sub-partitions
    const double per_smsp = 16.0 * iters * 8 / 4;
    printf("%-20s %.2f clk per warp instruction per SMSP (%.1f lanes/clk/SM)\n", name, mx / per_smsp,
           32.0 * 4 / (mx / per_smsp));
    cudaFree(out);
    cudaFree(clk);
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    run<0>("tanh.approx.f32", sms);
    run<1>("ex2.approx.ftz.f32", sms);
    run<2>("rcp.approx.ftz.f32", sms);
    run<3>("tanh.approx.bf16x2", sms);
    return 0;
}
