// L2 -> SM delivery probe: how many bytes per second can TMA land in shared memory across the
// whole chip, and does sharing (unicast of the same tile by G CTAs) or cluster multicast (each of
// G CTAs loads 1/G of the tile and multicasts it to all G) lift the chip-wide cap?
// No MMA: one producer thread per CTA streams 16 KB boxes (128 rows x 64 bf16, 128B swizzle)
// through an 8-stage mbarrier ring; one consumer thread frees the stages.
//   build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tma_mc_probe tools/tma_mc_probe.cu
//   run:   tools/tma_mc_probe            (prints one line per (mode, G))
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                          \
    do {                                                                               \
        cudaError_t e_ = (x);                                                          \
        if (e_ != cudaSuccess) {                                                       \
            std::fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); \
            std::exit(1);                                                              \
        }                                                                              \
    } while (0)

constexpr int STAGES = 8;
constexpr int BOX = 16384;

__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void wait_par(uint64_t* b, uint32_t par) {
    asm volatile("{\n.reg .pred P;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n@!P bra W_%=;\n}\n" ::"r"(su32(b)),
                 "r"(par)
                 : "memory");
}
__device__ __forceinline__ uint32_t ctarank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ uint32_t clusterid() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%clusterid.x;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void csync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// mode 0: every CTA reads its own rows; 1: groups of G consecutive CTAs read the same rows (unicast);
// 2: clusters of G CTAs, CTA r loads rows [r 128/G, +128/G) of the group's tile and multicasts them to all G.
__global__ void __launch_bounds__(64) probe(const __grid_constant__ CUtensorMap m, int mode, int G, int kblocks, int iters) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    __shared__ __align__(8) uint64_t full[STAGES], empty[STAGES];
    const bool mc = mode == 2;
    const uint32_t rank = mc ? ctarank() : 0;
    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&full[s])), "r"(1));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&empty[s])), "r"(mc ? G : 1));
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (mc) csync();
    const int group = mc ? static_cast<int>(clusterid()) : (mode == 1 ? blockIdx.x / G : blockIdx.x);
    const int total = kblocks * iters;
    if (threadIdx.x == 0) {  // producer
        const int rows = mc ? 128 / G : 128;
        const uint16_t mask = static_cast<uint16_t>((1u << G) - 1u);
        for (int i = 0; i < total; ++i) {
            const int s = i % STAGES;
            if (i >= STAGES) wait_par(&empty[s], ((i / STAGES) - 1) & 1);
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&full[s])), "r"(BOX) : "memory");
            const int c0 = (i % kblocks) * 64, c1 = group * 128 + static_cast<int>(rank) * rows;
            uint8_t* dst = sm + s * BOX + rank * rows * 128;
            if (mc)
                asm volatile(
                    "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster "
                    "[%0], [%1, {%2, %3}], [%4], %5;" ::"r"(su32(dst)),
                    "l"(reinterpret_cast<uint64_t>(&m)), "r"(c0), "r"(c1), "r"(su32(&full[s])), "h"(mask)
                    : "memory");
            else
                asm volatile(
                    "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
                        su32(dst)),
                    "l"(reinterpret_cast<uint64_t>(&m)), "r"(c0), "r"(c1), "r"(su32(&full[s]))
                    : "memory");
        }
    } else if (threadIdx.x == 32) {  // consumer: frees each stage in every CTA that writes into it
        for (int i = 0; i < total; ++i) {
            const int s = i % STAGES;
            wait_par(&full[s], (i / STAGES) & 1);
            if (mc) {
                for (int r = 0; r < G; ++r) {
                    uint32_t a;
                    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(a) : "r"(su32(&empty[s])), "r"(r));
                    asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(a) : "memory");
                }
            } else {
                asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&empty[s])) : "memory");
            }
        }
    }
    __syncthreads();
    if (mc) csync();
}


// Recurrent-kernel access patterns without MMA (one CTA pair = 2 CTAs, 64 pairs):
//   pat 3 (BPTT): A = dz [1024 x 4096] K-major 128-row boxes (m-tile, rank), B = W_hh [4096 x 1024]
//                 MN-major 64-unit x 64-K boxes (n-tile of 128 units, rank half), K halves: 32 k-blocks
//   pat 4 (forward): A = [x|h] [1024 x 3072] K-major, B = W [4096 x 3072] K-major, two 64-row gate
//                 boxes per CTA (64 units x 4 gates per pair): 48 k-blocks
__global__ void __launch_bounds__(64) probe2(const __grid_constant__ CUtensorMap mA, const __grid_constant__ CUtensorMap mB,
                                             int pat, int stages, int iters, int split) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    __shared__ __align__(8) uint64_t full[8], empty[8];
    if (threadIdx.x == 0) {
        for (int s = 0; s < stages; ++s) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&full[s])), "r"(1));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&empty[s])), "r"(1));
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const int pair = blockIdx.x / 2, r = blockIdx.x % 2;
    const int kbs = pat == 3 ? 32 : 48;
    const int SB = pat == 3 ? 24576 : 32768;
    const int total = kbs * iters;
    if (threadIdx.x == 0) {
        for (int i = 0; i < total; ++i) {
            const int s = i % stages;
            if (i >= stages) wait_par(&empty[s], ((i / stages) - 1) & 1);
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&full[s])), "r"(SB) : "memory");
            const int kb = i % kbs;
            uint8_t* dst = sm + s * SB;
            int a0, a1;
            if (pat == 3) {
                const int mt = pair % 4, nt = (pair / 4) % 8, kh = pair / 32;
                const int k0 = kh * 2048 + kb * 64;
                a0 = k0; a1 = mt * 256 + r * 128;
                asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
                                 su32(dst + 16384)), "l"(reinterpret_cast<uint64_t>(&mB)), "r"(nt * 128 + r * 64), "r"(k0),
                             "r"(su32(&full[s])) : "memory");
            } else {
                const int mt = pair % 4, nt = pair / 4;
                const int k0 = kb * 64;
                a0 = k0; a1 = mt * 256 + r * 128;
                const int br = 64 / split;  // split: B boxes of 64 / split rows (same bytes, more TMA ops)
                for (int j = 0; j < 2; ++j)
                    for (int q = 0; q < split; ++q)
                        asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
                                         su32(dst + 16384 + (j * split + q) * (8192 / split))), "l"(reinterpret_cast<uint64_t>(&mB)), "r"(k0),
                                     "r"((2 * r + j) * 1024 + nt * 64 + q * br), "r"(su32(&full[s])) : "memory");
            }
            asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
                             su32(dst)), "l"(reinterpret_cast<uint64_t>(&mA)), "r"(a0), "r"(a1), "r"(su32(&full[s])) : "memory");
        }
    } else if (threadIdx.x == 32) {
        for (int i = 0; i < total; ++i) {
            const int s = i % stages;
            wait_par(&full[s], (i / stages) & 1);
            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&empty[s])) : "memory");
        }
    }
    __syncthreads();
}

// CTA-pair pipeline (as persistent_kernel_2cta, no MMA): clusters of 2, both CTAs' TMA loads
// (.cta_group::2) complete on the leader's full barrier; the leader frees each stage in both CTAs
// by rel = 0: remote mbarrier arrives, rel = 1: tcgen05.commit.cta_group::2 multicast (mask 3).
// Forward pattern (pat 4 above).
__global__ void __launch_bounds__(64) probe3(const __grid_constant__ CUtensorMap mA, const __grid_constant__ CUtensorMap mB,
                                             int rel, int stages, int iters) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    __shared__ __align__(8) uint64_t full[8], empty[8];
    __shared__ uint32_t tslot;
    const uint32_t rank = ctarank();
    if (threadIdx.x == 0) {
        for (int s = 0; s < stages; ++s) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&full[s])), "r"(1));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&empty[s])), "r"(1));
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (threadIdx.x < 32 && rel == 1) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&tslot)), "r"(32) : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    }
    __syncthreads();
    csync();
    const int pair = blockIdx.x / 2;
    const int SB = 32768, kbs = 48;
    const int total = kbs * iters;
    if (threadIdx.x == 0) {
        for (int i = 0; i < total; ++i) {
            const int s = i % stages;
            if (i >= stages) wait_par(&empty[s], ((i / stages) - 1) & 1);
            if (rank == 0)
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&full[s])), "r"(2 * SB) : "memory");
            uint32_t bar;
            asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(bar) : "r"(su32(&full[s])), "r"(0));
            const int kb = i % kbs, mt = pair % 4, nt = pair / 4, k0 = kb * 64;
            uint8_t* dst = sm + s * SB;
            asm volatile("cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
                             su32(dst)), "l"(reinterpret_cast<uint64_t>(&mA)), "r"(k0), "r"(mt * 256 + (int)rank * 128), "r"(bar) : "memory");
            for (int j = 0; j < 2; ++j)
                asm volatile("cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
                                 su32(dst + 16384 + j * 8192)), "l"(reinterpret_cast<uint64_t>(&mB)), "r"(k0),
                             "r"((2 * (int)rank + j) * 1024 + nt * 64), "r"(bar) : "memory");
        }
    } else if (threadIdx.x == 32 && rank == 0) {
        for (int i = 0; i < total; ++i) {
            const int s = i % stages;
            wait_par(&full[s], (i / stages) & 1);
            if (rel == 1) {
                asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                                 su32(&empty[s])), "h"((uint16_t)3) : "memory");
            } else {
                for (int r = 0; r < 2; ++r) {
                    uint32_t a;
                    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(a) : "r"(su32(&empty[s])), "r"(r));
                    asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(a) : "memory");
                }
            }
        }
    }
    __syncthreads();
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    csync();
    if (threadIdx.x < 32 && rel == 1)
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tslot), "r"(32) : "memory");
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main(int argc, char** argv) {
    int nsm = 0;
    CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
    void* fp = nullptr;
    cudaDriverEntryPointQueryResult q;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q));
    EncodeFn enc = reinterpret_cast<EncodeFn>(fp);
    const int kblocks = argc > 1 ? std::atoi(argv[1]) : 32;  // K = 64 * kblocks per row block (L2-resident)
    const int iters = argc > 2 ? std::atoi(argv[2]) : 40;
    const uint64_t K = 64ull * kblocks, R = 128ull * nsm;
    void* buf;
    CK(cudaMalloc(&buf, K * R * 2));
    CK(cudaMemset(buf, 1, K * R * 2));
    const int smem = STAGES * BOX + 1024;
    CK(cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    CK(cudaFuncSetAttribute(probe, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    struct Cfg { int mode, G; };
    std::vector<Cfg> cfgs = {{0, 1}, {1, 2}, {1, 4}, {1, 8}, {1, 16}, {2, 2}, {2, 4}, {2, 8}, {2, 16}};
    for (const Cfg& c : cfgs) {
        CUtensorMap m;
        cuuint64_t dims[2] = {K, R};
        cuuint64_t str[1] = {K * 2};
        cuuint32_t box[2] = {64, static_cast<cuuint32_t>(c.mode == 2 ? 128 / c.G : 128)};
        cuuint32_t es[2] = {1, 1};
        if (enc(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
            std::printf("encode failed\n");
            return 1;
        }
        cudaLaunchConfig_t lc = {};
        cudaLaunchAttribute at[1];
        int grid = nsm;
        if (c.mode == 2) {
            at[0].id = cudaLaunchAttributeClusterDimension;
            at[0].val.clusterDim.x = c.G;
            at[0].val.clusterDim.y = 1;
            at[0].val.clusterDim.z = 1;
            lc.attrs = at;
            lc.numAttrs = 1;
            lc.gridDim = dim3(c.G);
            lc.blockDim = dim3(64);
            lc.dynamicSmemBytes = smem;
            int ncl = 0;
            if (cudaOccupancyMaxActiveClusters(&ncl, probe, &lc) != cudaSuccess || ncl == 0) {
                std::printf("mode=%d G=%2d: cluster not schedulable\n", c.mode, c.G);
                cudaGetLastError();
                continue;
            }
            grid = ncl * c.G;
        } else {
            grid = nsm / c.G * c.G;
        }
        lc.gridDim = dim3(grid);
        lc.blockDim = dim3(64);
        lc.dynamicSmemBytes = smem;
        cudaEvent_t e0, e1;
        CK(cudaEventCreate(&e0));
        CK(cudaEventCreate(&e1));
        float best = 1e30f;
        for (int rep = 0; rep < 4; ++rep) {
            CK(cudaEventRecord(e0));
            CK(cudaLaunchKernelEx(&lc, probe, m, c.mode, c.G, kblocks, iters));
            CK(cudaEventRecord(e1));
            CK(cudaEventSynchronize(e1));
            float ms;
            CK(cudaEventElapsedTime(&ms, e0, e1));
            if (rep > 0 && ms < best) best = ms;
        }
        CK(cudaGetLastError());
        const double delivered = double(grid) * kblocks * iters * BOX;
        const double unique = c.mode == 0 ? delivered : delivered / c.G;
        std::printf("mode=%d G=%2d grid=%3d: %8.1f us  delivered %6.2f TB/s (%5.1f GB/s per SM)  L2-unique %6.2f TB/s\n",
                    c.mode, c.G, grid, best * 1e3, delivered / best / 1e9, delivered / best / 1e6 / grid, unique / best / 1e9);
    }

    {  // recurrent patterns
        auto mk = [&](CUtensorMap* m, void* base, uint64_t inner, uint64_t outer, uint32_t bi, uint32_t bo) {
            cuuint64_t dims[2] = {inner, outer};
            cuuint64_t str[1] = {inner * 2};
            cuuint32_t box[2] = {bi, bo};
            cuuint32_t es[2] = {1, 1};
            return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, base, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                       CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        };
        void *A, *B;
        CK(cudaMalloc(&A, 1024ull * 4096 * 2));
        CK(cudaMalloc(&B, 4096ull * 3072 * 2));
        CK(cudaMemset(A, 1, 1024ull * 4096 * 2));
        CK(cudaMemset(B, 1, 4096ull * 3072 * 2));
        CK(cudaFuncSetAttribute(probe2, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
        for (int pat = 3; pat <= 4; ++pat)
            for (int split : {1, 2, 4, 8})
            for (int stages : {5}) {
                if (stages * (pat == 3 ? 24576 : 32768) + 1024 > 220 * 1024) continue;
                if (pat == 3 && split > 1) continue;
                CUtensorMap ma, mb;
                if (pat == 3) { mk(&ma, A, 4096, 1024, 64, 128); mk(&mb, B, 1024, 4096, 64, 64); }
                else { mk(&ma, A, 3072, 1024, 64, 128); mk(&mb, B, 3072, 4096, 64, 64 / split); }
                const int SB = pat == 3 ? 24576 : 32768;
                const int iters = 200;
                cudaEvent_t e0, e1;
                CK(cudaEventCreate(&e0));
                CK(cudaEventCreate(&e1));
                float best = 1e30f;
                for (int rep = 0; rep < 4; ++rep) {
                    CK(cudaEventRecord(e0));
                    probe2<<<128, 64, stages * SB + 1024>>>(ma, mb, pat, stages, iters, split);
                    CK(cudaEventRecord(e1));
                    CK(cudaEventSynchronize(e1));
                    float ms;
                    CK(cudaEventElapsedTime(&ms, e0, e1));
                    if (rep > 0 && ms < best) best = ms;
                }
                CK(cudaGetLastError());
                const int kbs = pat == 3 ? 32 : 48;
                const double delivered = 128.0 * kbs * iters * SB;
                std::printf("pat=%d (%s) B boxes of %d rows, stages=%d: %8.1f us  %6.2f TB/s delivered (%5.1f GB/s per SM), %.2f us per item\n", pat,
                            pat == 3 ? "BPTT" : "fwd", 64 / split, stages, best * 1e3, delivered / best / 1e9, delivered / best / 1e6 / 128,
                            best * 1e3 / iters);
            }

        {  // CTA-pair pipeline, forward pattern
            CUtensorMap ma, mb;
            mk(&ma, A, 3072, 1024, 64, 128);
            mk(&mb, B, 3072, 4096, 64, 64);
            CK(cudaFuncSetAttribute(probe3, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
            for (int rel = 0; rel < 2; ++rel)
                for (int stages : {3, 5, 6}) {
                    cudaLaunchConfig_t lc = {};
                    cudaLaunchAttribute at[1];
                    at[0].id = cudaLaunchAttributeClusterDimension;
                    at[0].val.clusterDim.x = 2; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
                    lc.attrs = at; lc.numAttrs = 1;
                    lc.gridDim = dim3(128); lc.blockDim = dim3(64); lc.dynamicSmemBytes = stages * 32768 + 1024;
                    const int iters = 200;
                    cudaEvent_t e0, e1;
                    CK(cudaEventCreate(&e0));
                    CK(cudaEventCreate(&e1));
                    float best = 1e30f;
                    for (int rep = 0; rep < 4; ++rep) {
                        CK(cudaEventRecord(e0));
                        CK(cudaLaunchKernelEx(&lc, probe3, ma, mb, rel, stages, iters));
                        CK(cudaEventRecord(e1));
                        CK(cudaEventSynchronize(e1));
                        float ms;
                        CK(cudaEventElapsedTime(&ms, e0, e1));
                        if (rep > 0 && ms < best) best = ms;
                    }
                    CK(cudaGetLastError());
                    const double delivered = 128.0 * 48 * iters * 32768;
                    std::printf("pair pipeline (%s release) stages=%d: %8.1f us  %6.2f TB/s (%5.1f GB/s per SM), %.2f us per item\n",
                                rel ? "tcgen05.commit" : "remote-arrive", stages, best * 1e3, delivered / best / 1e9,
                                delivered / best / 1e6 / 128, best * 1e3 / iters);
                }
        }
    }
    return 0;
}
