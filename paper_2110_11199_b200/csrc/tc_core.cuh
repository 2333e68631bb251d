// Persistent warp-specialised tcgen05 GEMM skeleton shared by the fused LSTM kernels.
//
//   warp 0     TMA producer (lane 0): Traits::load(p, tile, kb, sA, sB, bar)
//   warp 1     MMA issuer (lane 0) + TMEM owner; 2 accumulator stages of BN fp32 columns
//   warps 2-5  epilogue: Traits::epilogue(p, tile, tmem_col_base, quarter, lane)
// 128 x BN x 64 tiles, UMMA 128 x BN x 16, bf16 operands (K-major A; B K-major or MN-major
// per Traits::B_MN), fp32 accumulate in TMEM.
#pragma once

#include "common.cuh"
#include "tc_ptx.cuh"

namespace ab::tc {

constexpr int kBM = 128, kBK = 64, kThreads = 192;

template <int BN>
struct Shape {
    static constexpr int STAGES = BN >= 256 ? 4 : (BN >= 128 ? 6 : 8);
    static constexpr int A_BYTES = kBM * kBK * 2;
    static constexpr int B_BYTES = BN * kBK * 2;
    static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
    static constexpr int TMEM_COLS = 2 * BN < 32 ? 32 : 2 * BN;
    static constexpr int SMEM = STAGES * STAGE_BYTES + 1024 + 256;
};

template <class Traits, class Params>
__global__ void __launch_bounds__(kThreads, 1) persistent_kernel(const __grid_constant__ Params p) {
    constexpr int BN = Traits::BN;
    using S = Shape<BN>;
    constexpr int STAGES = S::STAGES;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sA = smem;
    uint8_t* sB = smem + STAGES * S::A_BYTES;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * S::STAGE_BYTES);
    uint64_t* empty = full + STAGES;
    uint64_t* tfull = empty + STAGES;
    uint64_t* tempty = tfull + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int num_tiles = Traits::num_tiles(p);

    if (warp == 0 && lane == 0) {
        for (int i = 0; i < STAGES; ++i) { ptx::mbar_init(&full[i], 1); ptx::mbar_init(&empty[i], 1); }
        for (int i = 0; i < 2; ++i) { ptx::mbar_init(&tfull[i], 1); ptx::mbar_init(&tempty[i], 4); }
        ptx::fence_barrier_init();
        Traits::prefetch(p);
    }
    if (warp == 1) ptx::tmem_alloc(tmem_slot, S::TMEM_COLS);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
                const int nkb = Traits::kblocks(p, tile);
                for (int kb = 0; kb < nkb; ++kb) {
                    ptx::mbar_wait(&empty[stage], phase ^ 1);
                    ptx::mbar_arrive_expect_tx(&full[stage], S::STAGE_BYTES);
                    Traits::load(p, tile, kb, sA + stage * S::A_BYTES, sB + stage * S::B_BYTES, &full[stage]);
                    if (++stage == STAGES) { stage = 0; phase ^= 1; }
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            constexpr uint32_t idesc = ptx::idesc_bf16_f32(kBM, BN, false, Traits::B_MN);
            int stage = 0;
            uint32_t phase = 0;
            int acc = 0;
            uint32_t aphase = 0;
            for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
                const int nkb = Traits::kblocks(p, tile);
                ptx::mbar_wait(&tempty[acc], aphase ^ 1);
                ptx::tc_fence_after();
                const uint32_t tmem_d = tmem_base + acc * BN;
                for (int kb = 0; kb < nkb; ++kb) {
                    ptx::mbar_wait(&full[stage], phase);
                    ptx::tc_fence_after();
                    const uint32_t a_addr = ptx::smem_u32(sA + stage * S::A_BYTES);
                    const uint32_t b_addr = ptx::smem_u32(sB + stage * S::B_BYTES);
#pragma unroll
                    for (int kk = 0; kk < kBK / 16; ++kk) {
                        const uint64_t ad = ptx::umma_desc_sw128(a_addr + kk * 32, 16, 1024);
                        const uint64_t bd = Traits::B_MN ? ptx::umma_desc_sw128(b_addr + kk * 2048, 64 * kBK * 2, 1024)
                                                         : ptx::umma_desc_sw128(b_addr + kk * 32, 16, 1024);
                        ptx::mma_bf16(tmem_d, ad, bd, idesc, (kb | kk) != 0);
                    }
                    ptx::mma_commit(&empty[stage]);
                    if (++stage == STAGES) { stage = 0; phase ^= 1; }
                }
                ptx::mma_commit(&tfull[acc]);
                if (++acc == 2) { acc = 0; aphase ^= 1; }
            }
        }
    } else {
        const int q = warp % 4;
        int acc = 0;
        uint32_t aphase = 0;
        for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
            ptx::mbar_wait(&tfull[acc], aphase);
            ptx::tc_fence_after();
            const uint32_t tbase = tmem_base + (static_cast<uint32_t>(q * 32) << 16) + acc * BN;
            Traits::epilogue(p, tile, tbase, q, lane, &tempty[acc]);
            if (++acc == 2) { acc = 0; aphase ^= 1; }
        }
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 1) ptx::tmem_dealloc(tmem_base, S::TMEM_COLS);
}

// Epilogue helper: after the last tcgen05.ld of an accumulator stage, hand it back to the MMA warp.
__device__ __forceinline__ void release_acc(uint64_t* tempty, int lane) {
    ptx::tc_fence_before();
    __syncwarp();
    if (lane == 0) ptx::mbar_arrive(tempty);
}

}  // namespace ab::tc
