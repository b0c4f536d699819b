#include <cstdio>
#include <cstdint>
#include <cstring>
__device__ __forceinline__ unsigned long long old_fix(float x) {
    return static_cast<unsigned long long>(__float2ull_rz(fminf(x, 2.0f) * 4611686018427387904.0f));
}
__device__ __forceinline__ unsigned long long to_fix(float x) {
    const uint32_t b = __float_as_uint(fminf(x, 2.0f));
    if (b >> 31) return 0ull;
    const uint32_t e = b >> 23;
    const unsigned long long m = (b & 0x7fffffu) | (e ? 0x800000u : 0u);
    const int sh = static_cast<int>(e ? e : 1u) - 88;
    return sh >= 0 ? (m << sh) : (sh > -64 ? (m >> -sh) : 0ull);
}
__global__ void k(unsigned long long* bad, unsigned int* first) {
    for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < (1ull << 32);
         i += (unsigned long long)gridDim.x * blockDim.x) {
        const float x = __uint_as_float((uint32_t)i);
        if (old_fix(x) != to_fix(x)) { if (atomicAdd(bad, 1ull) == 0) *first = (uint32_t)i; }
    }
}
int main() {
    unsigned long long* bad; unsigned int* first;
    cudaMallocManaged(&bad, 8); cudaMallocManaged(&first, 4); *bad = 0; *first = 0;
    k<<<148 * 8, 256>>>(bad, first);
    cudaDeviceSynchronize();
    printf("to_fix mismatches over all 2^32 patterns: %llu (first 0x%08x)\n", *bad, *first);
    return 0;
}
