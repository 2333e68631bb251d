// tcgen05 bf16 GEMM for sm_100a: TMA-fed, mbarrier-pipelined, accumulators in TMEM.
//
// Persistent warp-specialised kernel, one CTA per SM:
//   warp 0     TMA producer (one elected lane), STAGES-deep smem ring
//   warp 1     MMA issuer (one lane) + TMEM allocator; 2 accumulator stages in TMEM
//   warps 2-5  epilogue: tcgen05.ld -> alpha/bias/accumulate -> global
// Tile 128 x BN (BN = 256 or 128) x 64, UMMA 128 x BN x 16. Either operand may be K-major
// or MN-major (instruction-descriptor transpose bits; SW128 canonical layouts), so the
// LSTM's dgrad / wgrad contractions run without explicit transposes.
#include <cuda.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <unordered_map>

#include "gemm.hpp"
#include "gemm_lstm.hpp"
#include "tc_core.cuh"
#include "tc_ptx.cuh"
#include "prof.hpp"

namespace ab {

namespace {

constexpr int BM = 128, BK = 64;

struct TcParams {
    CUtensorMap ta[2];
    CUtensorMap tb[2];
    // MN-major operands as 3-D views {64, K, M/64 (or N/64)} (when the extent is a multiple of 64):
    // a CTA's two 64-wide blocks of a k-block in ONE TMA op (see tma_load_3d_2sm)
    CUtensorMap ta3[2];
    CUtensorMap tb3[2];
    int a3d, b3d;
    int kblocks[2];
    int nseg;
    int M, N;
    int m_tiles, n_tiles;
    void* C;
    int64_t ldc;
    float alpha;
    int accumulate;
    const float* bias;
    int vec_ok;
    unsigned long long* trace;
    int n_main;    // columns >= n_main are redirected to extra[row]
    float* extra;
    // stream-K (GenTraits SK): pair cid owns iterations [cid * total / pairs, (cid + 1) * total / pairs)
    // of the tile-major (tile, k-block) space; partials of split tiles meet in sk_ws.
    float* sk_ws;              // [pair * 2 + rank][chunk][128 rows][32] fp32
    unsigned int* sk_flags;    // [pair * 2 + rank], zeroed between launches by the owners
    int64_t sk_total;          // tiles * k-blocks per tile
    int sk_split;              // > 0: one-wave split-K instead -- pair c < sk_split * tiles takes K slice
                               //      c / tiles of tile c % tiles (slice 0 owns the tile)
    CUtensorMap tx;            // XTRA = 2: K-major tail columns [16 rows x K] (B columns n_tail0 + row)
    int n_tail0;
    // fused SGD update (GemmArgs::upd_*): C / extra element x -> o = w - lr x into o and bf16 shadow
    const float* upd_w;
    float* upd_o;
    bf16* upd_sh;
    const float* upd_xw;
    float* upd_xo;
    bf16* upd_xsh;
    const float* upd_lr;
};

// Final store of one fp32 output element (gradient or, fused, the SGD-updated weight + shadow).
__device__ __forceinline__ void put_c(const TcParams& p, int64_t idx, float x, float lr) {
    if (p.upd_o) {
        const float o = p.upd_w[idx] - lr * x;
        p.upd_o[idx] = o;
        p.upd_sh[idx] = __float2bfloat16_rn(o);
    } else {
        float* C = reinterpret_cast<float*>(p.C);
        C[idx] = p.accumulate ? C[idx] + x : x;
    }
}
__device__ __forceinline__ void put_x(const TcParams& p, int gm, float x, float lr) {
    if (p.upd_xo) {
        const float o = p.upd_xw[gm] - lr * x;
        p.upd_xo[gm] = o;
        p.upd_xsh[gm] = __float2bfloat16_rn(o);
    } else {
        p.extra[gm] = p.accumulate ? p.extra[gm] + x : x;
    }
}


// Generic GEMM traits for the persistent skeletons in tc_core.cuh (single CTA and CTA pair).
// XTRA: an extra N = 16 MMA per k-step on the tiles of the last n-tile (TMEM cols [BN, BN+16)),
//       so N stays a multiple of the tile width (CTA pairs, single accumulator stage).
//       1: against an all-ones smem tile -- the B operand's "ones column" (bias gradient = row
//          sums of A) without a ragged n-tile;
//       2: against B columns [n_tail0, n_tail0 + 16) loaded per stage from a K-major copy of
//          them (p.tx): a few real columns past the last full tile (layer-1 input features
//          256..259 + the ones column of a 260-feature input) ride on the last tile.
// SK:   stream-K work split (tc::Item): every CTA pair gets the same number of k-block iterations;
//       a tile split between pairs is finished by the pair holding its k-block 0, which adds the
//       other segments' partials in pair order (deterministic).
template <int BN_, bool AMN, bool BMN, bool CBF16, int XTRA = 0, bool SK = false, bool MCB = false>
struct GenTraits : tc::TraitsBase {
    static constexpr int BN = BN_;
    static constexpr int CLUSTER = MCB ? 4 : 2;  // MCB: two pairs (same n-tile) share B by TMA multicast
    static constexpr int EPI_SMEM = 0;
    static constexpr int EPI_WARPS = 8;
    static constexpr bool A_MN = AMN;
    static constexpr bool B_MN = BMN;
    static constexpr int EXTRA_COLS = XTRA ? 32 : 0;
    static constexpr int XB_BYTES = XTRA == 2 ? 1024 : 0;  // per CTA: 8 tail rows x 64 k, K-major SW128
    static constexpr int ACC_STAGES = (XTRA || BN_ > 256) ? 1 : 2;
    static constexpr int MMA_N = BN_ > 256 ? 256 : 0;
    static constexpr bool STREAMK = SK;
    static constexpr int NCH = BN / 32 + (XTRA ? 1 : 0);  // 32-column chunks of a partial (incl. the extra)
    __device__ static bool extra_tile(const TcParams& p, int tile) { return XTRA && tile / p.m_tiles == p.n_tiles - 1; }
    // XTRA = 2: rank r loads tail rows [8 r, +8) of k-block kb (single K segment)
    __device__ static void load_x(const TcParams& p, int, int kb, uint32_t rank, uint8_t* sX, uint32_t bar) {
        ptx::tma_load_2d_2sm(sX, &p.tx, bar, kb * BK, 8 * static_cast<int>(rank));
    }
    __device__ static int64_t sk_start(const TcParams& p, int c, int ncl) { return p.sk_total * c / ncl; }
    __device__ static bool sk_item(const TcParams& p, int cid, int ncl, int it, tc::Item& w) {
        const int kbt = kblocks(p, 0);
        if (p.sk_split > 0) {  // split-K: concurrent pairs walk the same K range (DRAM row locality)
            const int tiles = num_tiles(p), S = p.sk_split;
            if (it > 0 || cid >= S * tiles) return false;
            const int slice = cid / tiles;
            w.tile = cid % tiles;
            w.kb0 = static_cast<int>(static_cast<int64_t>(slice) * kbt / S);
            w.kb1 = static_cast<int>(static_cast<int64_t>(slice + 1) * kbt / S);
            w.role = S == 1 ? 0 : (slice == 0 ? 1 : 2);
            return true;
        }
        int64_t pos = sk_start(p, cid, ncl);
        const int64_t end = sk_start(p, cid + 1, ncl);
        for (int i = 0;; ++i) {
            if (pos >= end) return false;
            const int tile = static_cast<int>(pos / kbt), kb0 = static_cast<int>(pos % kbt);
            const int kb1 = static_cast<int>(kb0 + (end - pos) < kbt ? kb0 + (end - pos) : kbt);
            if (i == it) {
                w.tile = tile; w.kb0 = kb0; w.kb1 = kb1;
                w.role = (kb0 == 0 && kb1 == kbt) ? 0 : (kb0 == 0 ? 1 : 2);
                return true;
            }
            pos += kb1 - kb0;
        }
    }
    __device__ static int num_tiles(const TcParams& p) { return p.m_tiles * p.n_tiles; }
    __device__ static void prefetch(const TcParams& p) {
        for (int s = 0; s < p.nseg; ++s) { ptx::tma_prefetch(&p.ta[s]); ptx::tma_prefetch(&p.tb[s]); }
    }
    __device__ static int kblocks(const TcParams& p, int) { return p.kblocks[0] + (p.nseg > 1 ? p.kblocks[1] : 0); }
    __device__ static void seg_of(const TcParams& p, int kb, int& s, int& k0) {
        s = kb < p.kblocks[0] ? 0 : 1;
        k0 = (s == 0 ? kb : kb - p.kblocks[0]) * BK;
    }
    // ---- single CTA: 128 x BN tiles ----
    __device__ static void load(const TcParams& p, int tile, int kb, uint8_t* sA, uint8_t* sB, uint64_t* bar) {
        const int m0 = (tile % p.m_tiles) * BM, n0 = (tile / p.m_tiles) * BN;
        int s, k0;
        seg_of(p, kb, s, k0);
        if (AMN) {
#pragma unroll
            for (int j = 0; j < BM / 64; ++j) ptx::tma_load_2d(sA + j * 64 * BK * 2, &p.ta[s], bar, m0 + 64 * j, k0);
        } else {
            ptx::tma_load_2d(sA, &p.ta[s], bar, k0, m0);
        }
        if (BMN) {
#pragma unroll
            for (int j = 0; j < BN / 64; ++j) ptx::tma_load_2d(sB + j * 64 * BK * 2, &p.tb[s], bar, n0 + 64 * j, k0);
        } else {
            ptx::tma_load_2d(sB, &p.tb[s], bar, k0, n0);
        }
    }
    __device__ static void epilogue(const TcParams& p, int tile, uint32_t tbase, int q, int lane, uint64_t* tempty,
                                    uint8_t*, uint64_t*, uint32_t&, tc::EpiSlot sl) {
        const int m0 = (tile % p.m_tiles) * BM, n0 = (tile / p.m_tiles) * BN;
        body(p, m0 + q * 32, n0, tbase, lane, [&] { tc::release_acc(tempty, lane); }, sl, false, [](int, uint32_t*) {});
    }
    // ---- CTA pair: 256 x BN tiles, rank r holds A rows [m0 + 128 r, +128) and B rows [n0 + r BN/2, +BN/2) ----
    // BN = 512: two N = 256 sub-MMAs per k-step; for sub-MMA u CTA r holds B columns
    // [n_base + 256 u + 128 r, +128) at smem offset u * 16 KB (TMEM cols [256 u, +256) = tile cols).
    __device__ static void load2(const TcParams& p, int tile, int kb, uint32_t rank, uint8_t* sA, uint8_t* sB,
                                 uint32_t bar) {
        const int m0 = (tile % p.m_tiles) * 2 * BM + BM * rank;
        const int nb = (tile / p.m_tiles) * BN;
        int s, k0;
        seg_of(p, kb, s, k0);
        if (AMN) {
#pragma unroll
            for (int j = 0; j < BM / 64; ++j) ptx::tma_load_2d_2sm(sA + j * 64 * BK * 2, &p.ta[s], bar, m0 + 64 * j, k0);
        } else {
            ptx::tma_load_2d_2sm(sA, &p.ta[s], bar, k0, m0);
        }
        constexpr int SUBN = BN > 256 ? 256 : BN;  // N of one sub-MMA
#pragma unroll
        for (int u = 0; u < BN / SUBN; ++u) {
            const int n0 = nb + u * SUBN + (SUBN / 2) * static_cast<int>(rank);
            uint8_t* dst = sB + u * (SUBN / 2) * BK * 2;
            if (BMN) {
#pragma unroll
                for (int j = 0; j < SUBN / 128; ++j) ptx::tma_load_2d_2sm(dst + j * 64 * BK * 2, &p.tb[s], bar, n0 + 64 * j, k0);
            } else {
                ptx::tma_load_2d_2sm(dst, &p.tb[s], bar, k0, n0);
            }
        }
    }
    // Per-item TMA context (tc_core.cuh HasLoadCtx): the tile's row / column bases and the segment
    // boundary once per item; load2c is load2 without the per-k-block divisions by the tile counts.
    struct LoadCtx {
        const CUtensorMap* a[2];
        const CUtensorMap* b[2];
        int m0, nb, kbs;
        bool a3, b3;  // MN-major A / B through the 3-D views (one op for the CTA's two 64-wide blocks)
    };
    __device__ static LoadCtx load_ctx(const TcParams& p, int tile, uint32_t rank) {
        constexpr int SUBN = BN > 256 ? 256 : BN;
        LoadCtx c;
        c.a3 = AMN && p.a3d;
        c.b3 = BMN && SUBN == 256 && p.b3d;
        for (int s = 0; s < 2; ++s) {
            c.a[s] = c.a3 ? &p.ta3[s] : &p.ta[s];
            c.b[s] = c.b3 ? &p.tb3[s] : &p.tb[s];
        }
        c.m0 = (tile % p.m_tiles) * 2 * BM + BM * static_cast<int>(rank);
        c.nb = (tile / p.m_tiles) * BN + (SUBN / 2) * static_cast<int>(rank);
        c.kbs = p.kblocks[0];
        return c;
    }
    __device__ static void load2c(const LoadCtx& c, int kb, uint8_t* sA, uint8_t* sB, uint32_t bar) {
        const int s = kb < c.kbs ? 0 : 1;
        const int k0 = (kb - s * c.kbs) * BK;
        if (AMN) {
            if (c.a3) {
                ptx::tma_load_3d_2sm(sA, c.a[s], bar, 0, k0, c.m0 / 64);
            } else {
#pragma unroll
                for (int j = 0; j < BM / 64; ++j) ptx::tma_load_2d_2sm(sA + j * 64 * BK * 2, c.a[s], bar, c.m0 + 64 * j, k0);
            }
        } else {
            ptx::tma_load_2d_2sm(sA, c.a[s], bar, k0, c.m0);
        }
        constexpr int SUBN = BN > 256 ? 256 : BN;
#pragma unroll
        for (int u = 0; u < BN / SUBN; ++u) {
            const int n0 = c.nb + u * SUBN;
            uint8_t* dst = sB + u * (SUBN / 2) * BK * 2;
            if (BMN) {
                if (c.b3) {
                    ptx::tma_load_3d_2sm(dst, c.b[s], bar, 0, k0, n0 / 64);
                } else {
#pragma unroll
                    for (int j = 0; j < SUBN / 128; ++j) ptx::tma_load_2d_2sm(dst + j * 64 * BK * 2, c.b[s], bar, n0 + 64 * j, k0);
                }
            } else {
                ptx::tma_load_2d_2sm(dst, c.b[s], bar, k0, n0);
            }
        }
    }
    // MCB (MN-major B, BN = 256): cluster CTA c = 2 pc + r loads A rows as usual and B chunk pc of
    // its pair-rank half, multicast to CTA c and CTA c ^ 2 (the other pair's same-rank CTA).
    __device__ static void load2_mc(const TcParams& p, int tile, int kb, uint32_t crank, uint8_t* sA, uint8_t* sB,
                                    uint32_t bar) {
        const uint32_t rank = crank & 1, pc = crank >> 1;
        const int m0 = (tile % p.m_tiles) * 2 * BM + BM * rank;
        const int nb = (tile / p.m_tiles) * BN;
        int s, k0;
        seg_of(p, kb, s, k0);
        if (AMN) {
#pragma unroll
            for (int j = 0; j < BM / 64; ++j) ptx::tma_load_2d_2sm(sA + j * 64 * BK * 2, &p.ta[s], bar, m0 + 64 * j, k0);
        } else {
            ptx::tma_load_2d_2sm(sA, &p.ta[s], bar, k0, m0);
        }
        static_assert(!MCB || (BMN && BN == 256), "B multicast: MN-major B, 256-wide tiles");
        const int n0 = nb + (BN / 2) * static_cast<int>(rank);
        const uint16_t mask = static_cast<uint16_t>((1u << crank) | (1u << (crank ^ 2)));
        ptx::tma_load_2d_2sm_mc(sB + pc * 64 * BK * 2, &p.tb[s], bar, n0 + 64 * static_cast<int>(pc), k0, mask);
    }
    __device__ static void epilogue2(const TcParams& p, int tile, uint32_t rank, uint32_t tbase, int q, int lane,
                                     uint32_t tempty_leader, uint8_t*, uint64_t*, uint32_t&, tc::EpiSlot sl) {
        const int m0 = (tile % p.m_tiles) * 2 * BM + BM * rank, n0 = (tile / p.m_tiles) * BN;
        body(p, m0 + q * 32, n0, tbase, lane, [&] { tc::release_acc_2sm(tempty_leader, lane); }, sl,
             extra_tile(p, tile), [](int, uint32_t*) {});
    }
    // One-wave split-K epilogue as a reduce-scatter: the S units of a tile (K slices, pairs
    // j * tiles + tile) each finalise one group of its 32-column chunks (chunk c -> slice c * S / NCH)
    // and export the others. Every output element is summed in slice order 0..S-1 whichever unit
    // finalises it (deterministic). The last unit through re-arms the tile's flags.
    template <class Rel>
    __device__ static void split_epilogue(const TcParams& p, const tc::Item& w, int cid, uint32_t rank, uint32_t tbase,
                                          int q, int lane, tc::EpiSlot sl, Rel release) {
        const int tiles = num_tiles(p), S = p.sk_split;
        const int m0 = (w.tile % p.m_tiles) * 2 * BM + BM * static_cast<int>(rank), n0 = (w.tile / p.m_tiles) * BN;
        const int row = q * 32 + lane;
        const bool xt = extra_tile(p, w.tile);
        const int slice = cid / tiles;
        constexpr int kSlot = NCH * 128 * 32;
        auto group = [&](int c) { return c * S / NCH; };
        auto slot = [&](int j) { return p.sk_ws + static_cast<int64_t>((j * tiles + w.tile) * 2 + static_cast<int>(rank)) * kSlot; };
        const bool leader = q == 0 && sl.sub == 0 && lane == 0;
        if (S > 1) {
            // 1) export the chunks the other units finalise
#pragma unroll 1
            for (int c = sl.sub; c < NCH; c += sl.n) {
                if (group(c) == slice) continue;
                const bool xc = c >= BN / 32;
                if (xc && !xt) continue;
                uint32_t r[32];
                if (!xc) ptx::tmem_ld_32x32b_x32(tbase + 32 * c, r);
                else ptx::tmem_ld_32x32b_x16_(tbase + BN, r);
                ptx::tmem_ld_wait();
                float4* dst = reinterpret_cast<float4*>(slot(slice) + (static_cast<int64_t>(c) * 128 + row) * 32);
#pragma unroll
                for (int i = 0; i < 8; ++i)
                    __stcg(dst + i, make_float4(__uint_as_float(r[4 * i]), __uint_as_float(r[4 * i + 1]),
                                                __uint_as_float(r[4 * i + 2]), __uint_as_float(r[4 * i + 3])));
            }
            // 2) handshake with the other S - 1 units of the tile
            ptx::named_sync(2, 32 * EPI_WARPS);
            if (leader) {
                __threadfence();
                asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p.sk_flags + cid * 2 + rank), "r"(1u) : "memory");
                for (int j = 0; j < S; ++j)
                    if (j != slice) ptx::spin_until_geq(p.sk_flags + (j * tiles + w.tile) * 2 + rank, 1u);
                __threadfence();
            }
            ptx::named_sync(2, 32 * EPI_WARPS);
        }
        // 3) finalise this unit's chunks: sum over slices in order, own TMEM value at position `slice`
        body(p, m0 + q * 32, n0, tbase, lane, release, sl, xt, [&](int c, uint32_t* r) {
            if (S == 1) return;
            float acc[32];
#pragma unroll
            for (int i = 0; i < 32; ++i) acc[i] = 0.f;
            for (int j = 0; j < S; ++j) {
                if (j == slice) {
#pragma unroll
                    for (int i = 0; i < 32; ++i) acc[i] = j == 0 ? __uint_as_float(r[i]) : acc[i] + __uint_as_float(r[i]);
                } else {
                    const float4* src = reinterpret_cast<const float4*>(slot(j) + (static_cast<int64_t>(c) * 128 + row) * 32);
#pragma unroll
                    for (int i = 0; i < 8; ++i) {
                        const float4 f = __ldcg(src + i);
                        acc[4 * i] = j == 0 ? f.x : acc[4 * i] + f.x;
                        acc[4 * i + 1] = j == 0 ? f.y : acc[4 * i + 1] + f.y;
                        acc[4 * i + 2] = j == 0 ? f.z : acc[4 * i + 2] + f.z;
                        acc[4 * i + 3] = j == 0 ? f.w : acc[4 * i + 3] + f.w;
                    }
                }
            }
#pragma unroll
            for (int i = 0; i < 32; ++i) r[i] = __float_as_uint(acc[i]);
        }, [&](int c) { return S == 1 || group(c) == slice; });
        if (S > 1) {  // 4) every unit has read the tile's partials: the last one re-arms the flags
            ptx::named_sync(2, 32 * EPI_WARPS);
            if (leader) {
                unsigned int* ctr = p.sk_flags + gridDim.x + w.tile * 2 + rank;
                __threadfence();
                if (atomicAdd(ctr, 1u) == static_cast<unsigned>(S - 1)) {
                    for (int j = 0; j < S; ++j) p.sk_flags[(j * tiles + w.tile) * 2 + rank] = 0u;
                    *ctr = 0u;
                    __threadfence();
                }
            }
        }
    }
    // stream-K epilogue: role 0 = plain tile; 2 = export the partial (all chunks incl. the extra)
    // and flag it; 1 = wait for the later segments' pairs, add their partials, finish the tile.
    __device__ static void epilogue_sk(const TcParams& p, const tc::Item& w, int cid, uint32_t rank, uint32_t tbase,
                                       int q, int lane, uint32_t tempty_leader, tc::EpiSlot sl, uint8_t*, uint64_t*,
                                       uint32_t&) {
        const int m0 = (w.tile % p.m_tiles) * 2 * BM + BM * static_cast<int>(rank), n0 = (w.tile / p.m_tiles) * BN;
        const int row = q * 32 + lane;
        const bool xt = extra_tile(p, w.tile);
        auto release = [&] { tc::release_acc_2sm(tempty_leader, lane); };
        constexpr int kSlot = NCH * 128 * 32;  // floats per CTA slot
        const int ncl = gridDim.x >> 1;
        if (p.sk_split > 0) {
            split_epilogue(p, w, cid, rank, tbase, q, lane, sl, release);
            return;
        }
        if (w.role == 2) {
            float* ws = p.sk_ws + static_cast<int64_t>(cid * 2 + static_cast<int>(rank)) * kSlot;
#pragma unroll 1
            for (int c = sl.sub; c < NCH; c += sl.n) {
                uint32_t r[32];
                if (c < BN / 32) ptx::tmem_ld_32x32b_x32(tbase + 32 * c, r);
                else if (xt) ptx::tmem_ld_32x32b_x16_(tbase + BN, r);
                ptx::tmem_ld_wait();
                if (c >= BN / 32 && !xt) continue;
                float4* dst = reinterpret_cast<float4*>(ws + (static_cast<int64_t>(c) * 128 + row) * 32);
#pragma unroll
                for (int i = 0; i < 8; ++i)
                    __stcg(dst + i, make_float4(__uint_as_float(r[4 * i]), __uint_as_float(r[4 * i + 1]),
                                                __uint_as_float(r[4 * i + 2]), __uint_as_float(r[4 * i + 3])));
            }
            release();
            ptx::named_sync(2, 32 * EPI_WARPS);
            if (q == 0 && sl.sub == 0 && lane == 0) {
                __threadfence();
                asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p.sk_flags + cid * 2 + rank), "r"(1u) : "memory");
            }
            return;
        }
        int c_last = cid;  // owner: later pairs whose ranges start inside this tile contributed
        if (w.role == 1) {
            const int64_t tile_end = static_cast<int64_t>(w.tile + 1) * kblocks(p, 0);
            while (c_last + 1 < ncl && sk_start(p, c_last + 1, ncl) < tile_end) ++c_last;
            if (q == 0 && sl.sub == 0 && lane == 0) {
                for (int j = cid + 1; j <= c_last; ++j) {
                    if (sk_start(p, j, ncl) == sk_start(p, j + 1, ncl)) continue;  // empty range: no partial
                    ptx::spin_until_geq(p.sk_flags + j * 2 + rank, 1u);
                }
                __threadfence();
            }
            ptx::named_sync(2, 32 * EPI_WARPS);
        }
        body(p, m0 + q * 32, n0, tbase, lane, release, sl, xt, [&](int c, uint32_t* r) {
            for (int j = cid + 1; j <= c_last; ++j) {
                if (sk_start(p, j, ncl) == sk_start(p, j + 1, ncl)) continue;
                const float4* src = reinterpret_cast<const float4*>(
                    p.sk_ws + static_cast<int64_t>(j * 2 + static_cast<int>(rank)) * kSlot + (static_cast<int64_t>(c) * 128 + row) * 32);
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    const float4 f = __ldcg(src + i);
                    r[4 * i] = __float_as_uint(__uint_as_float(r[4 * i]) + f.x);
                    r[4 * i + 1] = __float_as_uint(__uint_as_float(r[4 * i + 1]) + f.y);
                    r[4 * i + 2] = __float_as_uint(__uint_as_float(r[4 * i + 2]) + f.z);
                    r[4 * i + 3] = __float_as_uint(__uint_as_float(r[4 * i + 3]) + f.w);
                }
            }
        });
        if (w.role == 1) {  // every warp has read the partials: re-arm the contributors' flags
            ptx::named_sync(2, 32 * EPI_WARPS);
            if (q == 0 && sl.sub == 0 && lane == 0)
                for (int j = cid + 1; j <= c_last; ++j)
                    if (sk_start(p, j, ncl) != sk_start(p, j + 1, ncl)) p.sk_flags[j * 2 + rank] = 0u;
        }
    }
    // TMEM accumulator (thread = row, 32-column chunks in registers) -> alpha / bias / accumulate
    // -> vectorised row-segment stores. fix(c, r) adds stream-K partials to chunk c; xt: also
    // write the extra row-sum column (TMEM col BN) to extra[row].
    struct KeepAll {
        __device__ bool operator()(int) const { return true; }
    };
    template <class Rel, class Fix, class Keep = KeepAll>
    __device__ static void body(const TcParams& p, int rowbase, int n0, uint32_t tbase, int lane, Rel release,
                                tc::EpiSlot sl, bool xt, Fix fix, Keep keep = Keep()) {
        const int gm = rowbase + lane;
        const bool row_ok = gm < p.M;
        const float lr = p.upd_lr ? *p.upd_lr : 0.f;
        if (XTRA && xt && sl.sub == 0 && keep(BN / 32)) {
            uint32_t r[32];
            ptx::tmem_ld_32x32b_x16_(tbase + BN, r);
            ptx::tmem_ld_wait();
            fix(BN / 32, r);
            if (row_ok && XTRA == 1) put_x(p, gm, p.alpha * __uint_as_float(r[0]), lr);
            if (row_ok && XTRA == 2) {  // tail columns n_tail0 + f: the C row below n_main, extra[] at n_main
#pragma unroll
                for (int f = 0; f < 16; ++f) {
                    const int gn = p.n_tail0 + f;
                    const float x = p.alpha * __uint_as_float(r[f]);
                    if (gn < p.n_main) put_c(p, static_cast<int64_t>(gm) * p.ldc + gn, x, lr);
                    else if (gn == p.n_main) put_x(p, gm, x, lr);
                }
            }
        }
#pragma unroll 1
        for (int c = 32 * sl.sub; c < BN; c += 32 * sl.n) {
            if (!keep(c / 32)) {
                if (c + 32 * sl.n >= BN) release();
                continue;
            }
            uint32_t r[32];
            ptx::tmem_ld_32x32b_x32(tbase + c, r);
            ptx::tmem_ld_wait();
            if (c + 32 * sl.n >= BN) release();
            fix(c / 32, r);
            if (!row_ok) continue;
            const int gn0 = n0 + c;
            if (gn0 >= p.N) continue;
            if (!XTRA && p.extra && gn0 + 32 > p.n_main) {
                // tail chunk containing redirected columns (fp32 output only)
                for (int i = 0; i < 32; ++i) {
                    const int gn = gn0 + i;
                    if (gn >= p.N) break;
                    const float x = p.alpha * __uint_as_float(r[i]) + (p.bias ? p.bias[gn] : 0.f);
                    if (gn < p.n_main) put_c(p, static_cast<int64_t>(gm) * p.ldc + gn, x, lr);
                    else if (gn == p.n_main) put_x(p, gm, x, lr);
                }
                continue;
            }
            float v[32];
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] = p.alpha * __uint_as_float(r[i]);
            if (p.bias) {
#pragma unroll
                for (int i = 0; i < 32; ++i)
                    if (gn0 + i < p.N) v[i] += p.bias[gn0 + i];
            }
            if constexpr (CBF16) {
                bf16* crow = reinterpret_cast<bf16*>(p.C) + static_cast<int64_t>(gm) * p.ldc + gn0;
                if (p.vec_ok && gn0 + 32 <= p.N) {
#pragma unroll
                    for (int i = 0; i < 32; i += 8) {
                        uint4 u;
                        if (p.accumulate) {
                            const uint4 o = *reinterpret_cast<const uint4*>(crow + i);
                            const bf16* ob = reinterpret_cast<const bf16*>(&o);
#pragma unroll
                            for (int j = 0; j < 8; ++j) v[i + j] += __bfloat162float(ob[j]);
                        }
                        bf16* ub = reinterpret_cast<bf16*>(&u);
#pragma unroll
                        for (int j = 0; j < 8; ++j) ub[j] = __float2bfloat16_rn(v[i + j]);
                        *reinterpret_cast<uint4*>(crow + i) = u;
                    }
                } else {
                    for (int i = 0; i < 32 && gn0 + i < p.N; ++i) {
                        float x = v[i];
                        if (p.accumulate) x += __bfloat162float(crow[i]);
                        crow[i] = __float2bfloat16_rn(x);
                    }
                }
            } else if (p.upd_o) {  // fused SGD update: w' = w - lr g (+ bf16 shadow), the gradient never stored
                const int64_t i0 = static_cast<int64_t>(gm) * p.ldc + gn0;
                if (p.vec_ok && gn0 + 32 <= p.N) {
#pragma unroll
                    for (int i = 0; i < 32; i += 4) {
                        const float4 wv = *reinterpret_cast<const float4*>(p.upd_w + i0 + i);
                        const float4 o = make_float4(wv.x - lr * v[i], wv.y - lr * v[i + 1], wv.z - lr * v[i + 2],
                                                     wv.w - lr * v[i + 3]);
                        *reinterpret_cast<float4*>(p.upd_o + i0 + i) = o;
                        uint2 sh;
                        sh.x = tc::pack_bf16x2(o.x, o.y);
                        sh.y = tc::pack_bf16x2(o.z, o.w);
                        *reinterpret_cast<uint2*>(p.upd_sh + i0 + i) = sh;
                    }
                } else {
                    for (int i = 0; i < 32 && gn0 + i < p.N; ++i) put_c(p, i0 + i, v[i], lr);
                }
            } else {
                float* crow = reinterpret_cast<float*>(p.C) + static_cast<int64_t>(gm) * p.ldc + gn0;
                if (p.vec_ok && gn0 + 32 <= p.N) {
#pragma unroll
                    for (int i = 0; i < 32; i += 4) {
                        float4 u = make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]);
                        if (p.accumulate) {
                            const float4 o = *reinterpret_cast<const float4*>(crow + i);
                            u.x += o.x; u.y += o.y; u.z += o.z; u.w += o.w;
                        }
                        *reinterpret_cast<float4*>(crow + i) = u;
                    }
                } else {
                    for (int i = 0; i < 32 && gn0 + i < p.N; ++i) {
                        float x = v[i];
                        if (p.accumulate) x += crow[i];
                        crow[i] = x;
                    }
                }
            }
        }
    }
};

// ---- host side -------------------------------------------------------------


}  // namespace

unsigned long long* trace_take();  // prof.cu

EncodeFnT get_encode_fn() {
    static EncodeFnT fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeFnT>(p);
    });
    AB_CHECK(fn != nullptr, ADPSGD_E_CUDA, "cuTensorMapEncodeTiled unavailable");
    return fn;
}

namespace {

// bf16 2-D tensor map, SWIZZLE_128B, box {64, box_outer}.
void make_map(CUtensorMap* m, const void* base, uint64_t inner, uint64_t outer, int64_t ld_elems, uint32_t box_outer) {
    AB_CHECK((reinterpret_cast<uintptr_t>(base) & 15) == 0, ADPSGD_E_DIMENSION, "TMA base must be 16B aligned");
    AB_CHECK(((ld_elems * 2) & 15) == 0, ADPSGD_E_DIMENSION, "TMA row pitch must be a multiple of 16 bytes");
    log_map_alignment(__FILE__, base, inner, outer, ld_elems * 2);
    cuuint64_t dims[2] = {inner, outer};
    cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld_elems) * 2};
    cuuint32_t box[2] = {64, box_outer};
    cuuint32_t es[2] = {1, 1};
    CUresult r = get_encode_fn()(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, es,
                             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                             ADPSGD_L2PROMO, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    AB_CHECK(r == CUDA_SUCCESS, ADPSGD_E_CUDA, "cuTensorMapEncodeTiled failed: " + std::to_string(r));
}

// MN-major bf16 operand [K rows x extent] (pitch ld) as a 3-D view {64, K, extent / 64}: block b of
// row k at column 64 b; box {64, 64, 2} = a CTA's two 64-wide blocks of one k-block.
void make_map3_mn(CUtensorMap* m, const void* base, uint64_t extent, uint64_t K, int64_t ld_elems) {
    AB_CHECK((reinterpret_cast<uintptr_t>(base) & 15) == 0, ADPSGD_E_DIMENSION, "TMA base must be 16B aligned");
    cuuint64_t dims[3] = {64, K, extent / 64};
    cuuint64_t strides[2] = {static_cast<cuuint64_t>(ld_elems) * 2, 128};
    cuuint32_t box[3] = {64, 64, 2};
    cuuint32_t es[3] = {1, 1, 1};
    CUresult r = get_encode_fn()(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides, box, es,
                                 CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                 ADPSGD_L2PROMO, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    AB_CHECK(r == CUDA_SUCCESS, ADPSGD_E_CUDA, "cuTensorMapEncodeTiled (3-D MN) failed: " + std::to_string(r));
}

template <class Traits>
void launch_single(const TcParams& p, cudaStream_t s) {
    auto k = tc::persistent_kernel<Traits, TcParams>;
    note_kernel<cta_single<Traits>>();
    static bool attr = false;
    if (!attr) {
        AB_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, tc::Shape<Traits::BN, Traits::EPI_SMEM>::SMEM));
        attr = true;
    }
    const int tiles = p.m_tiles * p.n_tiles;
    const int grid = tiles < num_sms() ? tiles : num_sms();
    tc::launch_tc(k, p, grid, tc::threads_of<Traits>(), tc::Shape<Traits::BN, Traits::EPI_SMEM>::SMEM, false, s);
    count_launch();
    AB_CUDA(cudaGetLastError());
}

template <class Traits>
void launch_pair(const TcParams& p, cudaStream_t s) {
    auto k = tc::persistent_kernel_2cta<Traits, TcParams>;
    note_kernel<cta_pair<Traits>>();
    static bool attr = false;
    if (!attr) {
        AB_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, tc::ShapeOf2<Traits>::SMEM));
        attr = true;
    }
    const int tiles = p.m_tiles * p.n_tiles;
    // stream-K spreads the k-block iterations over every pair; plain tiles use at most one pair per tile
    const int pairs = Traits::STREAMK ? num_sms() / 2 : (tiles < num_sms() / 2 ? tiles : num_sms() / 2);
    tc::launch_tc(k, p, 2 * pairs, tc::threads_of<Traits>(), tc::ShapeOf2<Traits>::SMEM, true, s, Traits::CLUSTER);
    count_launch();
}

template <int BN, bool AMN, bool BMN, bool CBF16>
void launch_cfg(const TcParams& p, bool pair, cudaStream_t s) {
    if (pair) launch_pair<GenTraits<BN, AMN, BMN, CBF16>>(p, s);
    else launch_single<GenTraits<BN, AMN, BMN, CBF16>>(p, s);
}

// CTA-pair 256-wide variants with the extra row-sum MMA (xtra) and / or stream-K (sk).
// Returns false for operand layouts that have no such instantiation.
template <int BN>
bool dispatch_ext(const TcParams& p, bool amn, bool bmn, bool cbf16, int xtra, bool sk, cudaStream_t s) {
    if (BN == 512 && !sk && !xtra) {  // one-round weight-gradient GEMMs (gemm_wgrad_wide)
        if (!(amn && bmn && !cbf16)) return false;
        launch_pair<GenTraits<512, true, true, false, false, false>>(p, s);
        return true;
    }
    if (xtra) {  // 1: ones column, 2: tail columns (p.tx)
        if (!(amn && bmn && !cbf16)) return false;
        if constexpr (BN == 256) {
            if (xtra == 2) {
                if (sk) launch_pair<GenTraits<256, true, true, false, 2, true>>(p, s);
                else launch_pair<GenTraits<256, true, true, false, 2, false>>(p, s);
            } else {
                if (sk) launch_pair<GenTraits<256, true, true, false, 1, true>>(p, s);
                else launch_pair<GenTraits<256, true, true, false, 1, false>>(p, s);
            }
            return true;
        }
        return false;
    }
    if (!sk) return false;
    const int key = (amn ? 4 : 0) | (bmn ? 2 : 0) | (cbf16 ? 1 : 0);
    switch (key) {
        case 6:
            if constexpr (BN == 256) {  // small weight gradients (dW_proj)
                launch_pair<GenTraits<256, true, true, false, false, true>>(p, s);
                return true;
            }
            return false;
        case 2: launch_pair<GenTraits<BN, false, true, false, false, true>>(p, s); return true;  // dgrad, fp32 out
        case 3: launch_pair<GenTraits<BN, false, true, true, false, true>>(p, s); return true;   // dgrad, bf16 out
        default: return false;
    }
}

template <int BN>
void dispatch(const TcParams& p, bool amn, bool bmn, bool cbf16, bool pair, cudaStream_t s) {
    const int key = (amn ? 4 : 0) | (bmn ? 2 : 0) | (cbf16 ? 1 : 0);
    if constexpr (BN == 256) {
        // B multicast across two CTA pairs (experiment / where tiles pair up along M)
        const int tiles = p.m_tiles * p.n_tiles;
        const int pairs = tiles < num_sms() / 2 ? tiles : num_sms() / 2;
        if (knobs().mcb && pair && bmn && p.m_tiles % 2 == 0 && tiles % 2 == 0 && pairs % 2 == 0) {
            if (key == 6) { launch_pair<GenTraits<256, true, true, false, false, false, true>>(p, s); return; }
            if (key == 2) { launch_pair<GenTraits<256, false, true, false, false, false, true>>(p, s); return; }
        }
    }
    switch (key) {
        case 0: launch_cfg<BN, false, false, false>(p, pair, s); break;
        case 1: launch_cfg<BN, false, false, true>(p, pair, s); break;
        case 2: launch_cfg<BN, false, true, false>(p, pair, s); break;
        case 3: launch_cfg<BN, false, true, true>(p, pair, s); break;
        case 4: launch_cfg<BN, true, false, false>(p, pair, s); break;
        case 5: launch_cfg<BN, true, false, true>(p, pair, s); break;
        case 6: launch_cfg<BN, true, true, false>(p, pair, s); break;
        default: launch_cfg<BN, true, true, true>(p, pair, s); break;
    }
}

struct PlanKey {
    const void* a[2]; const void* b[2]; const void* tail;
    int64_t lda[2], ldb[2];
    int K[2], M, N, nseg, bn, mode;
    bool amn, bmn;
    bool operator==(const PlanKey& o) const { return std::memcmp(this, &o, sizeof(PlanKey)) == 0; }
};
struct PlanHash {
    size_t operator()(const PlanKey& k) const {
        const uint64_t* w = reinterpret_cast<const uint64_t*>(&k);
        uint64_t h = 1469598103934665603ULL;
        for (size_t i = 0; i < sizeof(PlanKey) / 8; ++i) { h ^= w[i]; h *= 1099511628211ULL; }
        return h;
    }
};

}  // namespace

// Weight-gradient GEMMs [M gates x N inputs] whose 256 x 512 pair tiles fit one wave while the
// 256-wide tiles (+ the bias column) need two: the caller then computes the bias separately.
// Off by default: measured on B200 (6x1024 BLSTM) the one-wave 512-wide dW_ih ran 0.65 ms/step
// slower than two waves of 256-wide tiles, before the extra bias column sums (+0.65 ms).
// ADPSGD_FORCE_EXT=1 (tests) still takes it.
bool gemm_wgrad_wide(int M, int N) {
    const int npairs = num_sms() / 2;
    const int mt = (M + 255) / 256;
    return (knobs().force_ext || knobs().wide_wgrad) && knobs().wide_gemm && M > 128 && N >= 1024 && N % 512 == 0 && mt * (N / 512) <= npairs;
}

namespace {
thread_local GemmWorkspace t_ws;
}
void set_gemm_workspace(const GemmWorkspace& w) { t_ws = w; }
const GemmWorkspace& gemm_workspace() { return t_ws; }

void gemm_tc(const GemmArgs& g, cudaStream_t s) {
    if (g.M <= 0 || g.N <= 0) return;
    AB_CHECK(g.nseg >= 1 && g.nseg <= 2, ADPSGD_E_DIMENSION, "gemm_tc: 1 or 2 K segments");
    const bool amn = g.seg[0].a.mn, bmn = g.seg[0].b.mn;
    for (int i = 1; i < g.nseg; ++i)
        AB_CHECK(g.seg[i].a.mn == amn && g.seg[i].b.mn == bmn, ADPSGD_E_DIMENSION,
                 "gemm_tc: segments must share operand majorness");
    // CTA pairs (256-row tiles) whenever there are at least two row blocks
    const bool pair = knobs().pair_mma && g.M > BM;
    const int rows = pair ? 2 * BM : BM;
    const int m_tiles = (g.M + rows - 1) / rows;
    int kbt_all = 0;
    for (int i = 0; i < g.nseg; ++i) kbt_all += (g.seg[i].K + BK - 1) / BK;
    // few-tile, long-K weight gradients (dW_proj) go 256-wide and stream-K over every pair
    const bool tiny_wgrad = knobs().streamk && pair && amn && bmn && !g.c_bf16 && g.N > 128 && kbt_all >= 64 &&
                            m_tiles * ((g.N + 255) / 256) * 4 <= num_sms() / 2 && gemm_workspace().ws;
    const int force_bn = knobs().force_bn;  // probes
    const int bn0 = force_bn == 128 || force_bn == 256
                        ? force_bn
                        : (g.N > 128 && (knobs().force_ext || tiny_wgrad ||
                                         m_tiles * ((g.N + 255) / 256) >= (pair ? num_sms() / 4 : num_sms() / 2)))
                              ? 256 : 128;
    // bias column (g.extra, one column past n_main) by the extra row-sum MMA instead of a ragged n-tile
    // (only when it saves a round of CTA-pair waves: the extra MMA costs a single accumulator stage)
    const int npairs = num_sms() / 2;
    const int rounds_plain = (m_tiles * ((g.N + bn0 - 1) / bn0) + npairs - 1) / npairs;
    const int rounds_xtra = (m_tiles * (g.n_main / 256) + npairs - 1) / npairs;
    // a few columns past the last full 256-wide tile (+ the bias column) from the K-major tail copy
    const int n_tail0 = g.n_main > 0 ? (g.n_main / 256) * 256 : 0;
    const bool xb = knobs().xtra && g.b_tail && g.extra && pair && !g.c_bf16 && amn && bmn && g.nseg == 1 &&
                    g.n_main == g.N - 1 && n_tail0 >= 256 && g.N - n_tail0 <= 8;
    // ... or when dropping the bias tile brings the weight gradient within one-wave split-K reach
    // (tiles <= pairs / 2: every pair busy instead of one tile per pair)
    const int tiles_plain = m_tiles * ((g.N + bn0 - 1) / bn0), tiles_xtra = m_tiles * (g.n_main / 256);
    const bool xtra_splits = knobs().streamk && tiles_xtra * 2 <= npairs && tiles_plain * 2 > npairs;
    const bool xtra = xb || (knobs().xtra && g.extra && pair && bn0 == 256 && !g.c_bf16 && amn && bmn && g.n_main == g.N - 1 &&
                             g.n_main % 256 == 0 && (rounds_xtra < rounds_plain || xtra_splits || knobs().force_ext));
    const int xmode = xb ? 2 : (xtra ? 1 : 0);
    const int n_eff = xb ? n_tail0 : (xtra ? g.n_main : g.N);
    int kbt = 0;
    for (int i = 0; i < g.nseg; ++i) kbt += (g.seg[i].K + BK - 1) / BK;
    const GemmWorkspace& wsp = gemm_workspace();
    // stream-K when the tiles do not fill whole waves of CTA pairs -- dgrad layouts only (A K-major
    // activations, B MN-major weights that stay L2-resident): for the long-K weight-gradient
    // GEMMs (both operands streamed) pairs drifting apart along K lose the L2 reuse of the
    // lockstep wave order and run slower (measured). Large dgrads take 256 x 512 pair tiles
    // (two N = 256 MMAs per k-step: a quarter less L2->SM operand traffic per FLOP).
    auto sk_ok = [&](int bnx) {
        const int t = m_tiles * ((n_eff + bnx - 1) / bnx);
        // weight-gradient layout (both operands MN-major, long K) only when the tiles fill at most
        // half the pairs (dW_proj: 9 tiles, layer-1 dW_ih: 16): those run one-wave split-K with
        // every pair of a K slice in lockstep (p.sk_split); stream-K's pairs drift apart along K and
        // read scattered 512-byte pieces of the MN-major rows (measured slower for dW_out)
        const bool layout_ok = (!amn && bmn) || (amn && bmn && !g.c_bf16 && bnx == 256 && t * 2 <= npairs);
        return knobs().streamk && pair && bnx >= 256 && wsp.ws && (!xtra || bnx == 256) && layout_ok &&
               (t % npairs != 0 || knobs().force_ext) &&
               kbt >= 8 && wsp.floats >= static_cast<size_t>(npairs) * 2 * (bnx / 32 + 1) * 128 * 32 &&
               wsp.flag_count >= static_cast<size_t>(npairs) * 2;
    };
    const bool wide_wgrad = knobs().wide_gemm && amn && bmn && !g.c_bf16 && !g.extra && gemm_wgrad_wide(g.M, g.N);
    // 256 x 512 tiles have one accumulator stage (the epilogue is exposed once per tile): worth it
    // from ~3 waves of tiles on (H = 1024 dgrads: 4.5 waves, -6 % vs 256-wide; H = 512: 2.3 waves,
    // +6 %)
    const bool wide = (!xtra && wide_wgrad) || (!xtra && knobs().wide_gemm && bn0 == 256 && g.N >= 1024 && g.N % 512 == 0 &&
                                     (m_tiles * (g.N / 512) >= 3 * npairs || knobs().force_ext) && sk_ok(512));
    const int bn = wide ? 512 : (xb ? 256 : bn0);
    const int tiles = m_tiles * ((n_eff + bn - 1) / bn);
    const bool sk = !wide_wgrad && sk_ok(bn);
    static const bool log_gemm = std::getenv("ADPSGD_LOG_GEMM") != nullptr;  // diagnosis
    if (log_gemm)
        std::fprintf(stderr, "gemm M=%d N=%d K=%d nseg=%d amn=%d bmn=%d cbf16=%d pair=%d bn=%d xtra=%d xb=%d sk=%d tag=%d\n", g.M,
                     g.N, g.seg[0].K, g.nseg, amn, bmn, g.c_bf16, pair, bn, xtra, xb, sk, g.tag);

    static std::unordered_map<PlanKey, TcParams, PlanHash> cache;
    static std::mutex mu;
    PlanKey key;
    std::memset(&key, 0, sizeof(key));
    for (int i = 0; i < g.nseg; ++i) {
        key.a[i] = g.seg[i].a.ptr; key.b[i] = g.seg[i].b.ptr;
        key.lda[i] = g.seg[i].a.ld; key.ldb[i] = g.seg[i].b.ld; key.K[i] = g.seg[i].K;
    }
    key.tail = xb ? g.b_tail : nullptr;
    key.M = g.M; key.N = g.N; key.nseg = g.nseg; key.bn = bn * (pair ? 2 : 1); key.amn = amn; key.bmn = bmn;
    key.mode = (xtra ? 1 : 0) | (sk ? 2 : 0) | (xb ? 4 : 0) | (knobs().no_tma3d ? 8 : 0);

    TcParams p;
    {
        std::lock_guard<std::mutex> lk(mu);
        static const bool no_cache = std::getenv("ADPSGD_NO_PLAN_CACHE") != nullptr;  // diagnosis
        auto it = no_cache ? cache.end() : cache.find(key);
        if (it != cache.end()) {
            p = it->second;
        } else {
            std::memset(&p, 0, sizeof(p));
            for (int i = 0; i < g.nseg; ++i) {
                const GemmSeg& sg = g.seg[i];
                AB_CHECK(sg.K > 0, ADPSGD_E_DIMENSION, "gemm_tc: K must be > 0");
                if (amn) make_map(&p.ta[i], sg.a.ptr, g.M, sg.K, sg.a.ld, BK);
                else make_map(&p.ta[i], sg.a.ptr, sg.K, g.M, sg.a.ld, BM);
                if (bmn) make_map(&p.tb[i], sg.b.ptr, g.N, sg.K, sg.b.ld, BK);
                else make_map(&p.tb[i], sg.b.ptr, sg.K, g.N, sg.b.ld, pair ? (bn > 256 ? 128 : bn / 2) : bn);
                p.kblocks[i] = (sg.K + BK - 1) / BK;
            }
            // 3-D views of MN-major operands (CTA pairs; same extent as the 2-D maps, whole 64-wide
            // blocks only, so both views read and zero-fill exactly the same elements)
            p.a3d = amn && pair && g.M % 64 == 0 && !knobs().no_tma3d;
            p.b3d = bmn && pair && bn >= 256 && g.N % 64 == 0 && !knobs().no_tma3d;
            for (int i = 0; i < g.nseg; ++i) {
                const GemmSeg& sg = g.seg[i];
                if (p.a3d) make_map3_mn(&p.ta3[i], sg.a.ptr, g.M, sg.K, sg.a.ld);
                if (p.b3d) make_map3_mn(&p.tb3[i], sg.b.ptr, g.N, sg.K, sg.b.ld);
            }
            if (xb) {
                make_map(&p.tx, g.b_tail, g.seg[0].K, 16, g.ld_tail, 8);
                p.n_tail0 = n_tail0;
            }
            p.nseg = g.nseg;
            p.M = g.M; p.N = n_eff;
            p.m_tiles = m_tiles;
            p.n_tiles = (n_eff + bn - 1) / bn;
            if (cache.size() > 4096) cache.clear();
            cache.emplace(key, p);
        }
    }
    p.C = g.C;
    p.ldc = g.ldc;
    p.alpha = g.alpha;
    p.accumulate = g.accumulate;
    p.bias = g.bias;
    const int esz = g.c_bf16 ? 2 : 4;
    double ksum = 0;
    for (int i = 0; i < g.nseg; ++i) ksum += g.seg[i].K;
    ProfScope ps_(s, g.tag, 2.0 * g.M * g.N * ksum,
                  2.0 * (static_cast<double>(g.M) + g.N) * ksum + static_cast<double>(g.M) * g.N * esz * (g.accumulate ? 2 : 1));
    p.trace = trace_take();
    p.n_main = g.n_main < 0 ? g.N : g.n_main;
    p.extra = g.extra;
    AB_CHECK(!g.extra || (!g.c_bf16 && g.N == p.n_main + 1), ADPSGD_E_DIMENSION,
             "column redirect: fp32 output, exactly one extra column");
    p.vec_ok = ((reinterpret_cast<uintptr_t>(g.C) & 15) == 0) && ((g.ldc * esz) % 16 == 0);
    p.upd_w = g.upd_w; p.upd_o = g.upd_o; p.upd_sh = g.upd_sh;
    p.upd_xw = g.upd_xw; p.upd_xo = g.upd_xo; p.upd_xsh = g.upd_xsh;
    p.upd_lr = g.upd_lr;
    if (g.upd_o) {
        AB_CHECK(!g.c_bf16 && !g.accumulate && g.upd_w && g.upd_sh && g.upd_lr && (!g.extra || (g.upd_xw && g.upd_xo && g.upd_xsh)),
                 ADPSGD_E_INVALID_STATE, "fused update: fp32 output, no accumulate, complete pointers");
        p.vec_ok = p.vec_ok && ((reinterpret_cast<uintptr_t>(g.upd_w) & 15) == 0) &&
                   ((reinterpret_cast<uintptr_t>(g.upd_o) & 15) == 0) && ((reinterpret_cast<uintptr_t>(g.upd_sh) & 7) == 0);
    }
    p.sk_ws = wsp.ws;
    p.sk_flags = wsp.flags;
    p.sk_total = static_cast<int64_t>(tiles) * kbt;
    // slices of >= 16 k-blocks, at most 4 (the owner adds S - 1 partials on its own)
    if (sk && amn && bmn && wsp.flag_count >= static_cast<size_t>(2 * npairs + 2 * tiles)) {
        int S = npairs / tiles;
        if (S > knobs().split_max) S = knobs().split_max;
        if (S < 1) S = 1;
        while (S > 1 && kbt / S < 16) --S;
        p.sk_split = S;
    } else {
        p.sk_split = 0;
    }
    if (bn == 512) {
        AB_CHECK(dispatch_ext<512>(p, amn, bmn, g.c_bf16, xmode, sk, s), ADPSGD_E_INVALID_STATE,
                 "gemm_tc: no 512-wide kernel for this layout");
        return;
    }
    if ((xtra || sk) && dispatch_ext<256>(p, amn, bmn, g.c_bf16, xmode, sk, s)) return;
    AB_CHECK(!xtra, ADPSGD_E_INVALID_STATE, "gemm_tc: no plain kernel for the extra-column layout");
    if (bn == 256) dispatch<256>(p, amn, bmn, g.c_bf16, pair, s);
    else dispatch<128>(p, amn, bmn, g.c_bf16, pair, s);
}

}  // namespace ab
