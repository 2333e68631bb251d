// tcgen05.st -> tcgen05.ld round trip check (debug tool).
#include <cstdio>
#include <cstdint>
#include "../../paper_2110_11199_b200/csrc/tc_ptx.cuh"
using namespace ab;
__global__ void k(int* bad, int col0) {
    __shared__ uint32_t slot;
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    if (warp == 0) ptx::tmem_alloc(&slot, 512);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t base = slot;
    const uint32_t q = warp % 4;
    const uint32_t a = base + ((q * 32) << 16) + col0;
    uint32_t v[16], r[16];
    for (int i = 0; i < 16; ++i) v[i] = (q * 32 + lane) * 1000 + i + col0;
    ptx::tmem_st_32x32b_x16(a, v);
    ptx::tmem_st_wait();
    ptx::tmem_ld_32x32b_x16_(a, r);
    ptx::tmem_ld_wait();
    for (int i = 0; i < 16; ++i) if (r[i] != v[i]) atomicAdd(bad, 1);
    if (threadIdx.x == 0) printf("base=0x%08x\n", base);
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 0) ptx::tmem_dealloc(base, 512);
}
int main() {
    int* bad; cudaMallocManaged(&bad, 4);
    for (int col : {0, 16, 256, 320, 448}) {
        *bad = 0;
        k<<<1, 128>>>(bad, col);
        cudaDeviceSynchronize();
        printf("col %d: mismatches %d (%s)\n", col, *bad, cudaGetErrorString(cudaGetLastError()));
    }
}
