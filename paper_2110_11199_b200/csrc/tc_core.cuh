// Persistent warp-specialised tcgen05 GEMM skeleton shared by the fused LSTM kernels.
//
//   warp 0     TMA producer (lane 0): Traits::load(p, tile, kb, sA, sB, bar)
//   warp 1     MMA issuer (lane 0) + TMEM owner; 2 accumulator stages of BN fp32 columns
//   warps 2-5  epilogue: Traits::epilogue(p, tile, tmem_col_base, quarter, lane)
// 128 x BN x 64 tiles, UMMA 128 x BN x 16, bf16 operands (K-major A; B K-major or MN-major
// per Traits::B_MN), fp32 accumulate in TMEM.
#pragma once

#include <type_traits>

#include "common.cuh"
#include "knobs.hpp"
#include "tc_ptx.cuh"

namespace ab::tc {

// Debug timeline (adpsgd_debug_trace): per-CTA globaltimer stamps written by the MMA and
// epilogue warps of persistent_kernel_2cta into p.trace (nullptr = off).
// Slot layout: [cta][event] u64, event = 4 * tile_iter + kind.
constexpr int kTraceCtas = 160, kTraceEv = 48;  // events: 4 per item (items 0..9), 40..45 free, 46 start, 47 end
__device__ __forceinline__ void trace(unsigned long long* buf, int ev) {
    if (buf && blockIdx.x < kTraceCtas && ev < 40 || (buf && blockIdx.x < kTraceCtas && ev >= kTraceEv - 2 && ev < kTraceEv)) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        buf[blockIdx.x * kTraceEv + ev] = t;
    }
}

// Per-item timeline (tools/trace_items.py), after the block above: [cta][item < 64][12 slots]
// 0 producer: first load issued, 1 producer: mid-item dependency passed, 2 producer: last load issued,
// 3 MMA: first stage landed, 4 MMA: last MMA committed, 5 epilogue: accumulator full, 6 epilogue done,
// 7 producer: item reached (before its cross-CTA dependency wait); durations (ns, summed over the
// item's k-blocks): 8 MMA warp waiting for full stages, 9 producer waiting for empty stages
constexpr int kTraceItems = 64, kTraceItemEv = 12;  // 10 / 11: clock64 at MMA start / last MMA
__device__ __forceinline__ void trace_item(unsigned long long* buf, int item, int ev) {
#ifndef ADPSGD_ITEM_TRACE
    return;
#endif
    if (buf && blockIdx.x < kTraceCtas && item < kTraceItems) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        buf[kTraceCtas * kTraceEv + (blockIdx.x * kTraceItems + item) * kTraceItemEv + ev] = t;
    }
}
// per-k-block detail of CTAs 0 and 1, items < 8 (after the item block): [cta][item][kb < 64][3]
// 0 = producer issued the k-block's loads, 1 = the MMA warp saw the stage full (leader CTA only),
// 2 = producer got the empty stage (before issuing)
constexpr int kTraceDetailItems = 8, kTraceDetailKb = 64;
__device__ __forceinline__ void trace_kb(unsigned long long* buf, int item, int kb, int ev) {
#ifndef ADPSGD_ITEM_TRACE
    return;
#endif
    if (buf && blockIdx.x < 2 && item < kTraceDetailItems && kb < kTraceDetailKb) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        buf[kTraceCtas * kTraceEv + kTraceCtas * kTraceItems * kTraceItemEv +
            ((blockIdx.x * kTraceDetailItems + item) * kTraceDetailKb + kb) * 3 + ev] = t;
    }
}
// per-item / per-k-block instrumentation (trace_item*, wait durations, trace_kb): only in ADPSGD_ITEM_TRACE builds
// (tools/trace_items.py); the product build keeps the per-k-block loops free of it
__device__ __forceinline__ unsigned long long gclock(const void* buf) {
#ifdef ADPSGD_ITEM_TRACE
    if (buf) return clock64();
#endif
    return 0;
}
__device__ __forceinline__ unsigned long long gtimer(const void* buf) {
    unsigned long long t = 0;
#ifdef ADPSGD_ITEM_TRACE
    if (buf) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
#endif
    return t;
}
__device__ __forceinline__ void trace_item_put(unsigned long long* buf, int item, int ev, unsigned long long v) {
#ifndef ADPSGD_ITEM_TRACE
    return;
#endif
    if (buf && blockIdx.x < kTraceCtas && item < kTraceItems)
        buf[kTraceCtas * kTraceEv + (blockIdx.x * kTraceItems + item) * kTraceItemEv + ev] = v;
}

constexpr int kBM = 128, kBK = 64, kThreads = 192;

// Which column chunks of the accumulator an epilogue warp owns: with EPI_WARPS = 8 two warps
// share each TMEM lane quarter and take alternate chunks (index % n == sub).
struct EpiSlot {
    int sub, n;
};

constexpr int kSmemBudget = 225 * 1024;
#ifndef ADPSGD_STAGE_CAP
#define ADPSGD_STAGE_CAP 8  // A/B experiments only: cap on the CTA-pair mainloop stages
#endif

// Default hooks: Traits inherit from TraitsBase and may shadow these.
// epi_begin / epi_begin2 run on every epilogue warp BEFORE it waits for the tile's accumulator:
// epilogue inputs that do not depend on the GEMM (cell state, upstream gradients) can be
// loaded or L2-prefetched there, overlapping the mainloop. Each epilogue warp owns two
// mbarriers (ebar[0], ebar[1]) and the bits of ephase.
struct TraitsBase {
    static constexpr int ACC_STAGES = 2;      // TMEM accumulator stages (ACC_STAGES * BN <= 512 columns)
    static constexpr int MMA_N = 0;           // N of one MMA instruction (0: = BN); BN / MMA_N MMAs per k-step
    static constexpr bool EPI_OVERLAY = false; // epilogue smem overlays the pipeline stages (one tile per CTA only)
    static constexpr bool STREAMK = false;     // work items from Traits::sk_item / epilogue via Traits::epilogue_sk
    static constexpr int EXTRA_COLS = 0;       // extra TMEM columns: row sums of A (all-ones N = 16 MMA) on extra_tile()s
    static constexpr int CLUSTER = 2;          // 4: two CTA pairs per cluster sharing B by TMA multicast (load2_mc)
    static constexpr int TMEM_EXTRA = 0;       // TMEM columns past the accumulators for the epilogue's own state
    // > 0: the extra N = 16 MMA reads a per-stage K-major B tile of XB_BYTES per CTA loaded by
    // Traits::load_x (real operand columns past the main tile) instead of the all-ones tile
    static constexpr int XB_BYTES = 0;
    // STREAMK-style item kernels: the producer lane calls item_ready(p, w, cid, rank) before the
    // first TMA load of every item (cross-CTA dependencies of the A operand).
    template <class P, class W>
    __device__ static void item_ready(const P&, const W&, int, uint32_t) {}
    // ... and kb_ready(p, w, kb, cid, rank) before the load of k-block kb (mid-item dependencies).
    template <class P, class W>
    __device__ static void kb_ready(const P&, const W&, int, int, uint32_t) {}
    template <class P, class S>
    __device__ static void epi_begin(const P&, int, int, int, uint8_t*, uint64_t*, S) {}
    template <class P, class S>
    __device__ static void epi_begin2(const P&, int, uint32_t, int, int, uint8_t*, uint64_t*, S) {}
};

template <int BN, int EPI = 0>
struct Shape {
    static constexpr int A_BYTES = kBM * kBK * 2;
    static constexpr int B_BYTES = BN * kBK * 2;
    static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
    static constexpr int FIT = (kSmemBudget - EPI - 2048) / STAGE_BYTES;
    static constexpr int STAGES = FIT > 8 ? 8 : FIT;
    static constexpr int TMEM_COLS = 2 * BN < 32 ? 32 : 2 * BN;
    static constexpr int SMEM = STAGES * STAGE_BYTES + EPI + 2048;
};

template <class Traits>
constexpr int threads_of() { return 64 + 32 * Traits::EPI_WARPS; }

template <class Traits, class Params>
__global__ void __launch_bounds__(64 + 32 * Traits::EPI_WARPS, 1) persistent_kernel(const __grid_constant__ Params p) {
    constexpr int BN = Traits::BN;
    using S = Shape<BN, Traits::EPI_SMEM>;
    constexpr int STAGES = S::STAGES;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sA = smem;
    uint8_t* sB = smem + STAGES * S::A_BYTES;
    // 1 KB barrier block: full[<=8] @0, empty[<=8] @64, tfull[2] @128, tempty[2] @144,
    // TMEM slot @160, per-epilogue-warp barrier pairs[<=16] @256
    uint8_t* bblk = smem + STAGES * S::STAGE_BYTES;
    uint64_t* full = reinterpret_cast<uint64_t*>(bblk);
    uint64_t* empty = reinterpret_cast<uint64_t*>(bblk + 64);
    uint64_t* tfull = reinterpret_cast<uint64_t*>(bblk + 128);
    uint64_t* tempty = reinterpret_cast<uint64_t*>(bblk + 144);
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bblk + 160);
    uint64_t* epi_bar = reinterpret_cast<uint64_t*>(bblk + 256);
    uint8_t* epi_smem = bblk + 1024;  // 1024-aligned (TMA swizzle atoms)
    static_assert(STAGES <= 8 && Traits::EPI_WARPS <= 8, "barrier block layout");

    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int num_tiles = Traits::num_tiles(p);

    if (warp == 0 && lane == 0) {
        for (int i = 0; i < STAGES; ++i) { ptx::mbar_init(&full[i], 1); ptx::mbar_init(&empty[i], 1); }
        for (int i = 0; i < 2; ++i) { ptx::mbar_init(&tfull[i], 1); ptx::mbar_init(&tempty[i], Traits::EPI_WARPS); }
        for (int i = 0; i < 2 * Traits::EPI_WARPS; ++i) ptx::mbar_init(&epi_bar[i], 1);
        ptx::fence_barrier_init();
        Traits::prefetch(p);
    }
    if (warp == 1) ptx::tmem_alloc(tmem_slot, S::TMEM_COLS);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    // prologue done: dependents may launch; inputs of the previous kernel must be complete
    ptx::griddep_launch();
    ptx::griddep_wait();

    if (warp == 0) {
        // whole warp walks the loop (lane 0 issues); after the first tile's first STAGES loads
        // it releases the epilogue warps' epi_begin (their TMA traffic queues behind the operands)
        int stage = 0;
        uint32_t phase = 0;
        bool released = false;
        for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
            const int nkb = Traits::kblocks(p, tile);
            for (int kb = 0; kb < nkb; ++kb) {
                if (lane == 0) {
                    ptx::mbar_wait(&empty[stage], phase ^ 1);
                    ptx::mbar_arrive_expect_tx(&full[stage], S::STAGE_BYTES);
                    Traits::load(p, tile, kb, sA + stage * S::A_BYTES, sB + stage * S::B_BYTES, &full[stage]);
                }
                if (++stage == STAGES) { stage = 0; phase ^= 1; }
                if (!released && (kb + 1 == STAGES || kb + 1 == nkb)) {
                    __syncwarp();
                    ptx::named_arrive(1, 32 + 32 * Traits::EPI_WARPS);
                    released = true;
                }
            }
        }
        if (!released) ptx::named_arrive(1, 32 + 32 * Traits::EPI_WARPS);
    } else if (warp == 1) {
        if (lane == 0) {
            constexpr uint32_t idesc = ptx::idesc_bf16_f32(kBM, BN, Traits::A_MN, Traits::B_MN);
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
                        const uint64_t ad = Traits::A_MN ? ptx::umma_desc_sw128(a_addr + kk * 2048, 64 * kBK * 2, 1024)
                                                         : ptx::umma_desc_sw128(a_addr + kk * 32, 16, 1024);
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
        const int q = warp % 4;          // TMEM lane quarter this warp may access
        const int e = warp - 2;          // epilogue warp index
        const EpiSlot slot{(e / 4), Traits::EPI_WARPS / 4};
        int acc = 0;
        uint32_t aphase = 0, ephase = 0;
        uint8_t* est = epi_smem + e * (Traits::EPI_WARPS ? Traits::EPI_SMEM / Traits::EPI_WARPS : 0);
        ptx::named_sync(1, 32 + 32 * Traits::EPI_WARPS);
        for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
            Traits::epi_begin(p, tile, q, lane, est, &epi_bar[2 * e], slot);
            ptx::mbar_wait_sleep(&tfull[acc], aphase);
            ptx::tc_fence_after();
            const uint32_t tbase = tmem_base + (static_cast<uint32_t>(q * 32) << 16) + acc * BN;
            Traits::epilogue(p, tile, tbase, q, lane, &tempty[acc], est, &epi_bar[2 * e], ephase, slot);
            if (++acc == 2) { acc = 0; aphase ^= 1; }
        }
        if (lane == 0) ptx::bulk_wait0();
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 1) ptx::tmem_dealloc(tmem_base, S::TMEM_COLS);
}

// ---------------------------------------------------------------------------
// CTA-pair variant (cta_group::2): a cluster of 2 CTAs computes a 256 x BN tile; CTA rank r
// loads A rows [m0 + 128 r, +128) and B rows [n0 + r BN/2, +BN/2) into its own smem, both
// TMAs complete on the leader's barrier, the leader alone issues
// tcgen05.mma.cta_group::2 (M = 256), and each CTA's TMEM holds its 128 rows x BN fp32.
// Per-SM operand bytes per FLOP drop by a third vs 128 x BN single-CTA tiles.
// Traits: BN, B_MN, num_tiles (pair tiles), kblocks, prefetch,
//         load2(p, tile, kb, rank, sA, sB, bar_cluster_addr), epilogue2(p, tile, rank, tbase, q, lane, tempty_leader)
// ---------------------------------------------------------------------------
template <int BN, int EPI = 0, bool OVERLAY = false, int ACC = 2, int EXTRA = 0, int TX = 0, int XB = 0>
struct Shape2 {
    static constexpr int BNH = BN / 2;  // B rows held per CTA
    static constexpr int A_BYTES = kBM * kBK * 2;
    static constexpr int B_BYTES = BNH * kBK * 2;
    static constexpr int X_BYTES = XB;  // per-stage extra B tile (after the A and B regions)
    static constexpr int STAGE_BYTES = A_BYTES + B_BYTES + X_BYTES;
    static constexpr int ONES_BYTES = (EXTRA && !XB) ? 2048 : 0;  // all-ones bf16 B operand of the extra MMA
    static constexpr int FIT = (kSmemBudget - (OVERLAY ? 0 : EPI) - ONES_BYTES - 2048) / STAGE_BYTES;
    static constexpr int CAP = OVERLAY ? 8 : ADPSGD_STAGE_CAP;
    static constexpr int STAGES = FIT > CAP ? CAP : FIT;
    static constexpr int COLS = ACC * BN + EXTRA + TX;
    static constexpr int TMEM_COLS = COLS <= 32 ? 32 : COLS <= 64 ? 64 : COLS <= 128 ? 128 : COLS <= 256 ? 256 : 512;
    static constexpr int SMEM = STAGES * STAGE_BYTES + (OVERLAY ? 0 : EPI) + ONES_BYTES + 2048;
    static_assert(!OVERLAY || EPI <= STAGES * STAGE_BYTES, "overlaid epilogue smem must fit in the stages");
    static_assert(COLS <= 512, "TMEM has 512 columns");
};
template <class T>
using ShapeOf2 = Shape2<T::BN, T::EPI_SMEM, T::EPI_OVERLAY, T::ACC_STAGES, T::EXTRA_COLS, T::TMEM_EXTRA, T::XB_BYTES>;

// One unit of work of a CTA pair: k-blocks [kb0, kb1) of a tile. role: 0 = whole tile,
// 1 = stream-K owner (holds k-block 0, adds the later segments' partials), 2 = stream-K
// contributor (exports its partial). Default traits: whole tiles strided over the pairs.
struct Item {
    int tile, kb0, kb1, role;
};
template <class Traits, class Params>
__device__ __forceinline__ bool next_item(const Params& p, int cid, int ncl, int it, Item& w) {
    if constexpr (Traits::STREAMK) {
        return Traits::sk_item(p, cid, ncl, it, w);
    } else {
        w.tile = cid + it * ncl;
        if (w.tile >= Traits::num_tiles(p)) return false;
        w.kb0 = 0;
        w.kb1 = Traits::kblocks(p, w.tile);
        w.role = 0;
        return true;
    }
}

// Optional per-item load context: Traits with a LoadCtx type compute every item-invariant part of
// the TMA coordinates (tile rows, tensor-map pointers, cache policy) once per item in
// load_ctx(p, tile, rank); the producer's per-k-block work is then load2c(ctx, kb, sA, sB, bar):
// a handful of adds and the TMA issues. (The per-k-block path is a single thread's dependent
// instruction chain -- divisions by runtime tile counts there made the producer, not the memory
// system, the limit of the persistent recurrent kernels.)
template <class T, class = void>
struct HasLoadCtx : std::false_type {};
template <class T>
struct HasLoadCtx<T, std::void_t<typename T::LoadCtx>> : std::true_type {};
template <class T, bool = HasLoadCtx<T>::value>
struct LoadCtxOf {
    struct type {};
};
template <class T>
struct LoadCtxOf<T, true> {
    using type = typename T::LoadCtx;
};

template <class Traits, class Params>
__global__ void __launch_bounds__(64 + 32 * Traits::EPI_WARPS, 1) persistent_kernel_2cta(const __grid_constant__ Params p) {
    constexpr int BN = Traits::BN;
    using S = ShapeOf2<Traits>;
    constexpr int STAGES = S::STAGES;
    constexpr int ACC = Traits::ACC_STAGES;
    constexpr int MN = Traits::MMA_N ? Traits::MMA_N : BN;  // N per MMA instruction
    constexpr int NSUB = BN / MN;                             // MMAs per k-step (B sub-tiles of MN/2 rows per CTA)
    // (sub-MMA u's B sub-tile sits at u * (MN/2) * kBK * 2 bytes for K-major and MN-major B alike)
    static_assert(!Traits::EXTRA_COLS || ACC == 1, "extra accumulator columns need a single accumulator stage");
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sA = smem;
    uint8_t* sB = smem + STAGES * S::A_BYTES;
    uint8_t* sX = sB + STAGES * S::B_BYTES;  // XB_BYTES per stage (1024-aligned when XB_BYTES is)
    // 1 KB barrier block: full[<=8] @0, empty[<=8] @64, tfull[2] @128, tempty[2] @144,
    // TMEM slot @160, per-epilogue-warp barrier pairs[<=16] @256
    uint8_t* bblk = smem + STAGES * S::STAGE_BYTES;
    uint64_t* full = reinterpret_cast<uint64_t*>(bblk);
    uint64_t* empty = reinterpret_cast<uint64_t*>(bblk + 64);
    uint64_t* tfull = reinterpret_cast<uint64_t*>(bblk + 128);
    uint64_t* tempty = reinterpret_cast<uint64_t*>(bblk + 144);
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bblk + 160);
    uint64_t* epi_bar = reinterpret_cast<uint64_t*>(bblk + 256);
    uint8_t* epi_smem = Traits::EPI_OVERLAY ? smem : bblk + 1024;  // 1024-aligned (TMA swizzle atoms)
    uint8_t* ones = bblk + 1024 + (Traits::EPI_OVERLAY ? 0 : Traits::EPI_SMEM);  // S::ONES_BYTES, 1024-aligned
    static_assert(STAGES <= 8 && Traits::EPI_WARPS <= 8, "barrier block layout");

    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    constexpr bool MC = Traits::CLUSTER == 4;
    const uint32_t crank = ptx::cluster_ctarank();  // rank in the cluster (2 or 4 CTAs)
    const uint32_t rank = crank & 1;                // rank in the CTA pair
    const uint32_t leader = crank & ~1u;            // the pair's MMA-issuing CTA
    const uint16_t pair_mask = static_cast<uint16_t>(3u << leader);
    const int cid = blockIdx.x >> 1, ncl = gridDim.x >> 1;
    if (threadIdx.x == 0) trace(p.trace, kTraceEv - 2);

    if (warp == 0 && lane == 0) {
        // MC: a stage is written by both pairs' TMA multicasts, so both pairs' MMAs must free it
        for (int i = 0; i < STAGES; ++i) { ptx::mbar_init(&full[i], 1); ptx::mbar_init(&empty[i], MC ? 2 : 1); }
        for (int i = 0; i < 2; ++i) { ptx::mbar_init(&tfull[i], 1); ptx::mbar_init(&tempty[i], 2 * Traits::EPI_WARPS); }
        for (int i = 0; i < 2 * Traits::EPI_WARPS; ++i) ptx::mbar_init(&epi_bar[i], 1);
        ptx::fence_barrier_init();
        Traits::prefetch(p);
    }
    if constexpr (S::ONES_BYTES > 0) {
        for (int i = threadIdx.x; i < S::ONES_BYTES / 16; i += blockDim.x)
            ptx::st_shared_v4(ptx::smem_u32(ones) + 16 * i, 0x3F803F80u, 0x3F803F80u, 0x3F803F80u, 0x3F803F80u);
        ptx::fence_proxy_async_smem();  // generic-proxy writes -> visible to the tensor core
    }
    if (warp == 1) ptx::tmem_alloc_2sm(tmem_slot, S::TMEM_COLS);
    ptx::tc_fence_before();
    ptx::cluster_sync();
    ptx::tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    ptx::griddep_launch();
    ptx::griddep_wait();

    if (warp == 0) {
        int stage = 0;
        uint32_t phase = 0;
        bool released = false;
        Item w;
        const uint32_t full0 = ptx::mapa(ptx::smem_u32(&full[0]), leader);  // the leader's full[stage] = full0 + 8 stage
        for (int it = 0; next_item<Traits>(p, cid, ncl, it, w); ++it) {
            if constexpr (Traits::STREAMK) {
                if (lane == 0) { trace_item(p.trace, it, 7); Traits::item_ready(p, w, cid, rank); }
            }
            unsigned long long ewait = 0;
            typename LoadCtxOf<Traits>::type ctx;
            if constexpr (HasLoadCtx<Traits>::value) ctx = Traits::load_ctx(p, w.tile, rank);
            for (int kb = w.kb0; kb < w.kb1; ++kb) {
                if (lane == 0) {
                    if constexpr (Traits::STREAMK) Traits::kb_ready(p, w, kb, cid, rank);
                    const unsigned long long tw0 = gtimer(p.trace);
                    ptx::mbar_wait(&empty[stage], phase ^ 1);
                    ewait += gtimer(p.trace) - tw0;
                    trace_kb(p.trace, it, kb - w.kb0, 2);
                    if (kb == w.kb0) trace_item(p.trace, it, 0);
                    if (kb == w.kb0 + 32) trace_item(p.trace, it, 1);
                    if (kb + 1 == w.kb1) trace_item(p.trace, it, 2);
                    const uint32_t bar0 = full0 + 8 * stage;
                    if (rank == 0) ptx::mbar_arrive_expect_tx(&full[stage], 2 * S::STAGE_BYTES);
                    if constexpr (MC)
                        Traits::load2_mc(p, w.tile, kb, crank, sA + stage * S::A_BYTES, sB + stage * S::B_BYTES, bar0);
                    else if constexpr (HasLoadCtx<Traits>::value)
                        Traits::load2c(ctx, kb, sA + stage * S::A_BYTES, sB + stage * S::B_BYTES, bar0);
                    else
                        Traits::load2(p, w.tile, kb, rank, sA + stage * S::A_BYTES, sB + stage * S::B_BYTES, bar0);
                    trace_kb(p.trace, it, kb - w.kb0, 0);
                    if constexpr (S::X_BYTES > 0) Traits::load_x(p, w.tile, kb, rank, sX + stage * S::X_BYTES, bar0);
                }
                if (++stage == STAGES) { stage = 0; phase ^= 1; }
                if (!released && (kb + 1 - w.kb0 == STAGES || kb + 1 == w.kb1)) {
                    __syncwarp();
                    ptx::named_arrive(1, 32 + 32 * Traits::EPI_WARPS);
                    released = true;
                }
            }
            if (lane == 0) trace_item_put(p.trace, it, 9, ewait);
        }
        if (!released) ptx::named_arrive(1, 32 + 32 * Traits::EPI_WARPS);
    } else if (warp == 1) {
        if (lane == 0 && rank == 0) {
            constexpr uint32_t idesc = ptx::idesc_bf16_f32(2 * kBM, MN, Traits::A_MN, Traits::B_MN);
            constexpr uint32_t idesc_x = ptx::idesc_bf16_f32(2 * kBM, 16, Traits::A_MN, false);
            int stage = 0;
            uint32_t phase = 0;
            int acc = 0;
            uint32_t aphase = 0;
            Item w;
            for (int it = 0; next_item<Traits>(p, cid, ncl, it, w); ++it) {
                ptx::mbar_wait(&tempty[acc], aphase ^ 1);
                ptx::tc_fence_after();
                trace(p.trace, 4 * it + 0);
                const uint32_t tmem_d = tmem_base + acc * BN;
                bool extra = false;
                if constexpr (Traits::EXTRA_COLS > 0) extra = Traits::extra_tile(p, w.tile);
                unsigned long long fwait = 0;
                for (int kb = w.kb0; kb < w.kb1; ++kb) {
                    const unsigned long long tw0 = gtimer(p.trace);
                    ptx::mbar_wait(&full[stage], phase);
                    fwait += gtimer(p.trace) - tw0;
                    trace_kb(p.trace, it, kb - w.kb0, 1);
                    if (kb == w.kb0) { trace(p.trace, 4 * it + 1); trace_item(p.trace, it, 3); trace_item_put(p.trace, it, 10, gclock(p.trace)); }
                    ptx::tc_fence_after();
                    const uint32_t a_addr = ptx::smem_u32(sA + stage * S::A_BYTES);
                    const uint32_t b_addr = ptx::smem_u32(sB + stage * S::B_BYTES);
#pragma unroll
                    for (int kk = 0; kk < kBK / 16; ++kk) {
                        const uint64_t ad = Traits::A_MN ? ptx::umma_desc_sw128(a_addr + kk * 2048, 64 * kBK * 2, 1024)
                                                         : ptx::umma_desc_sw128(a_addr + kk * 32, 16, 1024);
                        const uint64_t bd = Traits::B_MN ? ptx::umma_desc_sw128(b_addr + kk * 2048, 64 * kBK * 2, 1024)
                                                         : ptx::umma_desc_sw128(b_addr + kk * 32, 16, 1024);
                        const bool accum = kb != w.kb0 || kk != 0;
#pragma unroll
                        for (int sub = 0; sub < NSUB; ++sub) {
                            // sub-MMA sub: B rows [sub MN/2, +MN/2) of this CTA's stage -> TMEM cols [sub MN, +MN)
                            const uint64_t bds = bd + static_cast<uint64_t>((sub * (MN / 2) * kBK * 2) >> 4);
#ifndef ADPSGD_DBG_NOMMA  // timing experiments only: the pipeline without tensor work
                            ptx::mma_bf16_2sm(tmem_d + sub * MN, ad, bds, idesc, accum);
#endif
                        }
                        if constexpr (Traits::EXTRA_COLS > 0) {
                            // row sums of A: an N = 16 MMA against an all-ones K-major B -> TMEM cols [BN, BN + 16)
                            const uint32_t xb = S::X_BYTES > 0 ? ptx::smem_u32(sX + stage * S::X_BYTES) : ptx::smem_u32(ones);
                            if (extra)
                                ptx::mma_bf16_2sm(tmem_d + BN, ad, ptx::umma_desc_sw128(xb + kk * 32, 16, 1024), idesc_x, accum);
                        }
                    }
                    ptx::mma_commit_2sm(&empty[stage], MC ? static_cast<uint16_t>(0xF) : pair_mask);
                    if (++stage == STAGES) { stage = 0; phase ^= 1; }
                }
                ptx::mma_commit_2sm(&tfull[acc], pair_mask);
                trace(p.trace, 4 * it + 2);
                trace_item(p.trace, it, 4);
                trace_item_put(p.trace, it, 8, fwait);
                trace_item_put(p.trace, it, 11, gclock(p.trace));
                if (++acc == ACC) { acc = 0; aphase ^= 1; }
            }
        }
    } else {
        const int q = warp % 4;
        const int e = warp - 2;
        const EpiSlot slot{(e / 4), Traits::EPI_WARPS / 4};
        const uint32_t tempty0 = ptx::mapa(ptx::smem_u32(&tempty[0]), leader);
        int acc = 0;
        uint32_t aphase = 0, ephase = 0;
        uint8_t* est = epi_smem + e * (Traits::EPI_WARPS ? Traits::EPI_SMEM / Traits::EPI_WARPS : 0);
        ptx::named_sync(1, 32 + 32 * Traits::EPI_WARPS);
        Item w;
        for (int it = 0; next_item<Traits>(p, cid, ncl, it, w); ++it) {
            Traits::epi_begin2(p, w.tile, rank, q, lane, est, &epi_bar[2 * e], slot);
            ptx::mbar_wait_sleep(&tfull[acc], aphase);
            ptx::tc_fence_after();
            if (e == 0 && lane == 0) trace_item(p.trace, it, 5);
            const uint32_t tbase = tmem_base + (static_cast<uint32_t>(q * 32) << 16) + acc * BN;
            if constexpr (Traits::STREAMK)
                Traits::epilogue_sk(p, w, cid, rank, tbase, q, lane, tempty0 + acc * 8, slot, est, &epi_bar[2 * e], ephase);
            else
                Traits::epilogue2(p, w.tile, rank, tbase, q, lane, tempty0 + acc * 8, est, &epi_bar[2 * e], ephase, slot);
            if (e == 0 && lane == 0) { trace(p.trace, 4 * it + 3); trace_item(p.trace, it, 6); }
            if (++acc == ACC) { acc = 0; aphase ^= 1; }
        }
        if (lane == 0) ptx::bulk_wait0();
    }
    ptx::tc_fence_before();
    ptx::cluster_sync();
    if (threadIdx.x == 0) trace(p.trace, kTraceEv - 1);
    if (warp == 1) ptx::tmem_dealloc_2sm(tmem_base, S::TMEM_COLS);
}

// CTA-pair epilogue helper: release the accumulator stage on the leader's tempty barrier.
__device__ __forceinline__ void release_acc_2sm(uint32_t tempty_leader, int lane) {
    ptx::tc_fence_before();
    __syncwarp();
    if (lane == 0) ptx::mbar_arrive_cluster(tempty_leader);
}

// Per-warp staging of a 32-row x NC-column fp32 accumulator chunk: thread `lane` holds row
// `lane` (tcgen05.ld 32x32b layout); after stage_rows + __syncwarp, element (row, col) sits at
// st[row * (NC + 1) + col] (padded: conflict-free both ways), so the warp can sweep rows with
// lanes along columns (coalesced global access).
template <int NC>
__device__ __forceinline__ void stage_rows(float* st, int lane, const uint32_t* v) {
    // (row-major padded staging; used by epilogues that sweep rows)
#pragma unroll
    for (int i = 0; i < NC; ++i) st[lane * (NC + 1) + i] = __uint_as_float(v[i]);
}

// Swizzled smem tiles for TMA boxes (row = this thread's lane).
// fp32 row of 32 values (128 B) in a SWIZZLE_128B box: 16-B chunk c at c ^ (row & 7).
__device__ __forceinline__ void st_row_f32_sw128(uint8_t* box, int row, const float* v) {
    const uint32_t base = ptx::smem_u32(box) + row * 128;
#pragma unroll
    for (int c = 0; c < 8; ++c)
        ptx::st_shared_v4(base + ((c ^ (row & 7)) << 4), __float_as_uint(v[4 * c]), __float_as_uint(v[4 * c + 1]),
                          __float_as_uint(v[4 * c + 2]), __float_as_uint(v[4 * c + 3]));
}
__device__ __forceinline__ void ld_row_f32_sw128(const uint8_t* box, int row, float* v) {
    const uint32_t base = ptx::smem_u32(box) + row * 128;
#pragma unroll
    for (int c = 0; c < 8; ++c) {
        const float4 f = ptx::ld_shared_v4f(base + ((c ^ (row & 7)) << 4));
        v[4 * c] = f.x; v[4 * c + 1] = f.y; v[4 * c + 2] = f.z; v[4 * c + 3] = f.w;
    }
}
// bf16 row of 32 values (64 B) in a SWIZZLE_64B box: 16-B chunk c at c ^ ((row >> 1) & 3).
__device__ __forceinline__ void st_row_bf16_sw64(uint8_t* box, int row, const float* v) {
    const uint32_t base = ptx::smem_u32(box) + row * 64;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
        uint32_t w[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            __nv_bfloat162 b2 = __floats2bfloat162_rn(v[8 * c + 2 * k], v[8 * c + 2 * k + 1]);
            w[k] = *reinterpret_cast<uint32_t*>(&b2);
        }
        ptx::st_shared_v4(base + ((c ^ ((row >> 1) & 3)) << 4), w[0], w[1], w[2], w[3]);
    }
}

// Half rows (16 values) of the 32-value swizzled rows above: half h = chunks [h*n, (h+1)*n).
__device__ __forceinline__ void st_half_bf16_sw64(uint8_t* box, int row, int h, const float* v) {
    const uint32_t base = ptx::smem_u32(box) + row * 64;
#pragma unroll
    for (int k = 0; k < 2; ++k) {
        const int c = 2 * h + k;
        uint32_t w[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            __nv_bfloat162 b2 = __floats2bfloat162_rn(v[8 * k + 2 * j], v[8 * k + 2 * j + 1]);
            w[j] = *reinterpret_cast<uint32_t*>(&b2);
        }
        ptx::st_shared_v4(base + ((c ^ ((row >> 1) & 3)) << 4), w[0], w[1], w[2], w[3]);
    }
}
__device__ __forceinline__ void st_half_f32_sw128(uint8_t* box, int row, int h, const float* v) {
    const uint32_t base = ptx::smem_u32(box) + row * 128;
#pragma unroll
    for (int k = 0; k < 4; ++k)
        ptx::st_shared_v4(base + (((4 * h + k) ^ (row & 7)) << 4), __float_as_uint(v[4 * k]), __float_as_uint(v[4 * k + 1]),
                          __float_as_uint(v[4 * k + 2]), __float_as_uint(v[4 * k + 3]));
}
__device__ __forceinline__ void ld_half_f32_sw128(const uint8_t* box, int row, int h, float* v) {
    const uint32_t base = ptx::smem_u32(box) + row * 128;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const float4 f = ptx::ld_shared_v4f(base + (((4 * h + k) ^ (row & 7)) << 4));
        v[4 * k] = f.x; v[4 * k + 1] = f.y; v[4 * k + 2] = f.z; v[4 * k + 3] = f.w;
    }
}

// first-write-wins stamp (sub-phases of the first tile's epilogue)
__device__ __forceinline__ void trace_once(unsigned long long* buf, int ev) {
    if (buf && blockIdx.x < kTraceCtas && ev < kTraceEv && buf[blockIdx.x * kTraceEv + ev] == 0) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        buf[blockIdx.x * kTraceEv + ev] = t;
    }
}

// Generic swizzled-row access for TMA boxes whose rows are ROWB bytes (32, 64 or 128):
// 16-B chunk c of row r sits at chunk position c ^ swz(r) (SWIZZLE_32B / 64B / 128B).
template <int ROWB>
__device__ __forceinline__ int swz(int r) {
    return ROWB == 128 ? (r & 7) : (ROWB == 64 ? ((r >> 1) & 3) : ((r >> 2) & 1));
}
template <int ROWB>
__device__ __forceinline__ void st_row_words(uint8_t* box, int row, const uint32_t* w) {
    const uint32_t base = ptx::smem_u32(box) + row * ROWB;
#pragma unroll
    for (int c = 0; c < ROWB / 16; ++c)
        ptx::st_shared_v4(base + ((c ^ swz<ROWB>(row)) << 4), w[4 * c], w[4 * c + 1], w[4 * c + 2], w[4 * c + 3]);
}
template <int ROWB>
__device__ __forceinline__ void ld_row_words(const uint8_t* box, int row, uint32_t* w) {
    const uint32_t base = ptx::smem_u32(box) + row * ROWB;
#pragma unroll
    for (int c = 0; c < ROWB / 16; ++c) {
        const float4 f = ptx::ld_shared_v4f(base + ((c ^ swz<ROWB>(row)) << 4));
        w[4 * c] = __float_as_uint(f.x); w[4 * c + 1] = __float_as_uint(f.y);
        w[4 * c + 2] = __float_as_uint(f.z); w[4 * c + 3] = __float_as_uint(f.w);
    }
}
__device__ __forceinline__ uint32_t pack_bf16x2(float a, float b) {
    __nv_bfloat162 v = __floats2bfloat162_rn(a, b);
    return *reinterpret_cast<uint32_t*>(&v);
}
__device__ __forceinline__ float bf16_lo(uint32_t w) { return __uint_as_float(w << 16); }
__device__ __forceinline__ float bf16_hi(uint32_t w) { return __uint_as_float(w & 0xffff0000u); }

// Epilogue helper: after the last tcgen05.ld of an accumulator stage, hand it back to the MMA warp.
__device__ __forceinline__ void release_acc(uint64_t* tempty, int lane) {
    ptx::tc_fence_before();
    __syncwarp();
    if (lane == 0) ptx::mbar_arrive(tempty);
}

// Host: launch a persistent tcgen05 kernel (optionally as 2-CTA clusters) with programmatic
// dependent launch, so its prologue (barrier init, TMEM alloc, tensor-map prefetch) overlaps
// the previous kernel's tail; the kernel griddep_wait()s before touching dependent data.
template <class P>
inline void launch_tc(void (*kern)(P), const P& p, int grid, int threads, int smem, bool pair, cudaStream_t s,
                      int cluster = 2, const cudaAccessPolicyWindow* l2win = nullptr) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(threads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attrs[3];
    int n = 0;
    if (pair) {
        attrs[n].id = cudaLaunchAttributeClusterDimension;
        attrs[n].val.clusterDim.x = cluster;
        attrs[n].val.clusterDim.y = 1;
        attrs[n].val.clusterDim.z = 1;
        ++n;
    }
    if (knobs().pdl) {
        attrs[n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attrs[n].val.programmaticStreamSerializationAllowed = 1;
        ++n;
    }
    if (l2win) {  // L2 persisting window (e.g. the recurrent weights of a persistent layer kernel)
        attrs[n].id = cudaLaunchAttributeAccessPolicyWindow;
        attrs[n].val.accessPolicyWindow = *l2win;
        ++n;
    }
    cfg.attrs = attrs;
    cfg.numAttrs = n;
    AB_CUDA(cudaLaunchKernelEx(&cfg, kern, p));
}

}  // namespace ab::tc
