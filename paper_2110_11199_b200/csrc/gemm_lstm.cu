// Fused LSTM recurrent-step kernels on tcgen05 (bf16 operands, fp32 TMEM accumulators).
//
// lstm_fwd_step: for each direction d (one launch covers both),
//     z = [x_t | h_{t-1}] [W_ih | W_hh]^T + b                       (K = I + H)
//     i,f,g,o = sig/sig/tanh/sig(z); c_t = f c_{t-1} + i g; h_t = o tanh(c_t)
//   A 128 x 256 tile spans 64 hidden units x the 4 gates (four 64-row TMA boxes of the
//   gate blocks of W), so the whole cell runs in the epilogue straight out of TMEM:
//   z never touches HBM.
// lstm_bwd_step: BPTT step, for each direction d,
//     dh_rec = dz_t W_hh                       (the recurrent dgrad, K = 4H, W_hh MN-major)
//   and in the epilogue the cell backward of the next BPTT time t':
//     dh = dH[t'] + dh_rec; dc = dc_rec + dh o (1 - tanh^2 c); dz_{t'} = ...; dc_rec = dc f
#include <cuda.h>

#include <cstdio>
#include <cstdlib>

#include "gemm_lstm.hpp"
#include "prof.hpp"
#include "tc_core.cuh"

namespace ab {

EncodeFnT get_encode_fn();  // gemm_tc.cu
unsigned long long* trace_take();  // prof.cu

void make_map_gen(CUtensorMap* m, const void* base, bool f32, uint64_t inner, uint64_t outer, int64_t ld,
                  uint32_t box_inner, uint32_t box_outer, CUtensorMapSwizzle sw) {
    const int esz = f32 ? 4 : 2;
    AB_CHECK((reinterpret_cast<uintptr_t>(base) & 15) == 0, ADPSGD_E_DIMENSION, "TMA base must be 16B aligned");
    log_map_alignment(__FILE__, base, inner, outer, ld * esz);
    AB_CHECK(((ld * esz) & 15) == 0, ADPSGD_E_DIMENSION, "TMA row pitch must be a multiple of 16 bytes");
    cuuint64_t dims[2] = {inner, outer};
    cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld) * esz};
    cuuint32_t box[2] = {box_inner, box_outer};
    cuuint32_t es[2] = {1, 1};
    CUresult r = get_encode_fn()(m, f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2,
                                 const_cast<void*>(base), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
                                 ADPSGD_L2PROMO, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    AB_CHECK(r == CUDA_SUCCESS, ADPSGD_E_CUDA, "cuTensorMapEncodeTiled failed: " + std::to_string(r));
}

// 3-D bf16 view [outer2][outer1][inner] (SWIZZLE_128B, 64-element inner box): rows of `ld`
// elements, blocks of `blk_stride` elements; box {64, box1, box2}. Lands in smem exactly as box2
// consecutive 2-D boxes of 64 x box1, i.e. the layout the MMA descriptors already expect.
void make_map_3d(CUtensorMap* m, const void* base, uint64_t inner, uint64_t outer1, uint64_t outer2, int64_t ld,
                 int64_t blk_stride, uint32_t box1, uint32_t box2) {
    AB_CHECK((reinterpret_cast<uintptr_t>(base) & 15) == 0, ADPSGD_E_DIMENSION, "TMA base must be 16B aligned");
    AB_CHECK(((ld * 2) & 15) == 0 && ((blk_stride * 2) & 15) == 0, ADPSGD_E_DIMENSION, "TMA strides must be multiples of 16 bytes");
    cuuint64_t dims[3] = {inner, outer1, outer2};
    cuuint64_t strides[2] = {static_cast<cuuint64_t>(ld) * 2, static_cast<cuuint64_t>(blk_stride) * 2};
    cuuint32_t box[3] = {64, box1, box2};
    cuuint32_t es[3] = {1, 1, 1};
    CUresult r = get_encode_fn()(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides, box, es,
                                 CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, ADPSGD_L2PROMO,
                                 CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    AB_CHECK(r == CUDA_SUCCESS, ADPSGD_E_CUDA, "cuTensorMapEncodeTiled (3-D) failed: " + std::to_string(r));
}

namespace {

using tc::kBK;
using tc::kBM;

void make_map_box(CUtensorMap* m, const void* base, uint64_t inner, uint64_t outer, int64_t ld, uint32_t box_outer) {
    make_map_gen(m, base, false, inner, outer, ld, 64, box_outer, CU_TENSOR_MAP_SWIZZLE_128B);
}


// One MUFU.TANH each (max rel. err ~2^-11, below the bf16 rounding of the stored activations);
// an IEEE-division sigmoid/tanh compiles to branchy slow paths that serialise the unrolled
// per-row element chains of the epilogue (measured ~15 us per 32-unit chunk).
__device__ __forceinline__ float tanhf_fast(float x) {
    float y;
    asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ float sigf(float x) { return fmaf(0.5f, tanhf_fast(0.5f * x), 0.5f); }

// ---------------- forward ----------------
struct FwdGroup {
    CUtensorMap ta[2];
    CUtensorMap tb[2];
    CUtensorMap m_cprev, m_gates, m_c, m_h;  // epilogue I/O (TMA)
    int kb0, kb1, nseg;
    const float* bias;
    const float* c_prev;
    bf16* gates;
    float* c;
    bf16* h;
};
struct FwdParams {
    FwdGroup g[2];
    int ngroups, m_tiles, n_tiles, B, H, ldg, ldc, ldh;
    int epi_skip;  // debug: timing experiments only
    unsigned long long* trace;
};

// U = hidden units per tile (x 4 gates = BN accumulator columns).
//   U = 64:  256-column pair tiles, 2 accumulator stages, 4 epilogue warps (tiles > CTA pairs).
//   U = 128: 512-column pair tiles (two N = 256 MMAs per k-step), one accumulator stage, 8
//            epilogue warps whose staging overlays the (then idle) pipeline stages; used when
//            every CTA pair owns exactly one tile (one wave, ~25% less L2->SM operand traffic).
template <int U>
struct FwdT : tc::TraitsBase {
    static constexpr bool WIDE = U == 128;
    static constexpr int BN = 4 * U;
    static constexpr int EPI_WARP = 22 * 1024;  // see body()
    static constexpr int EPI_WARPS = WIDE ? 8 : 4;
    static constexpr int EPI_SMEM = EPI_WARPS * EPI_WARP;
    static constexpr int ACC_STAGES = WIDE ? 1 : 2;
    static constexpr int MMA_N = WIDE ? 256 : 0;
    static constexpr bool EPI_OVERLAY = WIDE;
    static constexpr bool B_MN = false;
    __device__ static int num_tiles(const FwdParams& p) { return p.ngroups * p.m_tiles * p.n_tiles; }
    __device__ static void prefetch(const FwdParams& p) {
        for (int i = 0; i < p.ngroups; ++i)
            for (int s = 0; s < p.g[i].nseg; ++s) { ptx::tma_prefetch(&p.g[i].ta[s]); ptx::tma_prefetch(&p.g[i].tb[s]); }
    }
    __device__ static void coords(const FwdParams& p, int tile, int& grp, int& m0, int& u0) {
        const int per = p.m_tiles * p.n_tiles;
        grp = tile / per;
        const int r = tile % per;
        m0 = (r % p.m_tiles) * kBM;
        u0 = (r / p.m_tiles) * U;
    }
    __device__ static int kblocks(const FwdParams& p, int tile) {
        const FwdGroup& g = p.g[tile / (p.m_tiles * p.n_tiles)];
        return g.kb0 + (g.nseg > 1 ? g.kb1 : 0);
    }
    __device__ static void load(const FwdParams& p, int tile, int kb, uint8_t* sA, uint8_t* sB, uint64_t* bar) {
        int grp, m0, u0;
        coords(p, tile, grp, m0, u0);
        const FwdGroup& g = p.g[grp];
        const int s = kb < g.kb0 ? 0 : 1;
        const int k0 = (s == 0 ? kb : kb - g.kb0) * kBK;
        ptx::tma_load_2d_hint(sA, &g.ta[s], bar, k0, m0, ptx::policy_evict_first());
        const uint64_t keep = ptx::policy_evict_last();
#pragma unroll
        for (int gate = 0; gate < 4; ++gate)
            ptx::tma_load_2d_hint(sB + gate * 64 * kBK * 2, &g.tb[s], bar, k0, gate * p.H + u0, keep);
    }
    // CTA pair: rank r loads rows [m0 + 128 r, +128) of A and gates {2r, 2r+1} of B
    static constexpr bool A_MN = false;
    __device__ static void coords2(const FwdParams& p, int tile, int& grp, int& m0, int& u0) {
        const int per = p.m_tiles * p.n_tiles;
        grp = tile / per;
        const int r = tile % per;
        m0 = (r % p.m_tiles) * 2 * kBM;
        u0 = (r / p.m_tiles) * U;
    }
    __device__ static void load2(const FwdParams& p, int tile, int kb, uint32_t rank, uint8_t* sA, uint8_t* sB,
                                 uint32_t bar) {
        int grp, m0, u0;
        coords2(p, tile, grp, m0, u0);
        const FwdGroup& g = p.g[grp];
        const int s = kb < g.kb0 ? 0 : 1;
        const int k0 = (s == 0 ? kb : kb - g.kb0) * kBK;
        ptx::tma_load_2d_2sm_hint(sA, &g.ta[s], bar, k0, m0 + kBM * rank, ptx::policy_evict_first());
        const uint64_t keep = ptx::policy_evict_last();
        // U = 64: CTA r holds gates {2r, 2r+1} (64 rows each) of the one N = 256 MMA.
        // U = 128: CTA r holds gate r (sub-MMA 0 -> cols [0,256)) and gate 2+r (sub-MMA 1).
#pragma unroll
        for (int j = 0; j < 2; ++j)
            ptx::tma_load_2d_2sm_hint(sB + j * U * kBK * 2, &g.tb[s], bar, k0,
                                      (WIDE ? 2 * j + static_cast<int>(rank) : 2 * static_cast<int>(rank) + j) * p.H + u0, keep);
    }
    // WIDE: the whole tile's c_{t-1} goes to L2 while the mainloop runs (epilogue smem is the
    // pipeline's, so no early smem loads)
    template <class S>
    __device__ static void epi_begin2(const FwdParams& p, int tile, uint32_t rank, int q, int lane, uint8_t*, uint64_t*,
                                      S sl) {
        if (!WIDE) return;
        int grp, m0, u0;
        coords2(p, tile, grp, m0, u0);
        const FwdGroup& g = p.g[grp];
        if (g.c_prev == nullptr) return;
        const int uc = 32 * sl.sub + 32 * sl.n * (lane & 1);
        if (lane < 2 && uc < U) ptx::tma_prefetch_l2_2d(&g.m_cprev, u0 + uc, m0 + kBM * static_cast<int>(rank) + q * 32);
    }
    __device__ static void epilogue2(const FwdParams& p, int tile, uint32_t rank, uint32_t tbase, int q, int lane,
                                     uint32_t tempty_leader, uint8_t* st, uint64_t* ebar, uint32_t& ephase,
                                     tc::EpiSlot sl) {
        int grp, m0, u0;
        coords2(p, tile, grp, m0, u0);
        body(p, grp, m0 + kBM * rank, u0, tbase, q, lane, [&] { tc::release_acc_2sm(tempty_leader, lane); }, st, ebar,
             ephase, sl);
    }
    __device__ static void epilogue(const FwdParams& p, int tile, uint32_t tbase, int q, int lane, uint64_t* tempty,
                                    uint8_t* st, uint64_t* ebar, uint32_t& ephase, tc::EpiSlot sl) {
        int grp, m0, u0;
        coords(p, tile, grp, m0, u0);
        body(p, grp, m0, u0, tbase, q, lane, [&] { tc::release_acc(tempty, lane); }, st, ebar, ephase, sl);
    }
    // epilogue (thread = row): per 32-unit chunk, c_{t-1} arrives by TMA into swizzled smem
    // (double-buffered: chunk j+1's load is issued when chunk j starts); the 4 gate columns
    // leave TMEM in two 16-unit halves (bounding register pressure); the cell runs in registers;
    // each half's gates (bf16), c (fp32) and h (bf16) are staged in one of two swizzled output
    // sets and leave by TMA bulk stores that overlap the next half's math (rows >= B clipped).
    // smem per warp (22 KB): c_{t-1} 2 x 4 KB | out 2 x 7 KB (c 2 KB | gates 4 x 1 KB | h 1 KB)
    template <class Rel>
    __device__ static void body(const FwdParams& p, int grp, int m0, int u0, uint32_t tbase, int q, int lane,
                                Rel release, uint8_t* st, uint64_t* ebar, uint32_t& ephase, tc::EpiSlot sl) {
        body_g(p.g[grp], p.H, m0, u0, tbase, q, lane, release, st, ebar, ephase, sl, p.trace, 0, 0,
               p.g[grp].c_prev != nullptr);
    }
    // row_out / row_cp: row offsets of the outputs and of c_{t-1} (maps spanning all time steps)
    // NSETS: output staging sets per warp (2: a half's stores overlap the next half's math;
    // 1: 15 KB per warp instead of 22, so the persistent forward fits one more mainloop stage)
    template <class Rel, int NSETS = 2>
    __device__ static void body_g(const FwdGroup& g, int H, int m0, int u0, uint32_t tbase, int q, int lane,
                                  Rel release, uint8_t* st, uint64_t* ebar, uint32_t& ephase, tc::EpiSlot sl,
                                  unsigned long long* trace, int row_out, int row_cp, bool has_prev) {
        const int rowbase = m0 + q * 32;
        const bool tr = trace && q == 2 && lane == 0;
        const int step = 32 * sl.n;
        auto issue_cprev = [&](int uc, int b) {
            ptx::mbar_arrive_expect_tx(ebar + b, 32 * 32 * 4);
            ptx::tma_load_2d(st + b * 4096, &g.m_cprev, ebar + b, u0 + uc, rowbase + row_cp);
        };
        if (has_prev && lane == 0) issue_cprev(32 * sl.sub, 0);
        int ob = 0;
        int cb = 0;
#pragma unroll 1
        for (int uc = 32 * sl.sub; uc < U; uc += step, cb ^= 1) {
            const int j0 = u0 + uc;
            if (has_prev && lane == 0 && uc + step < U) issue_cprev(uc + step, cb ^ 1);
            if (tr) tc::trace_once(trace, 12 + (uc / 32) * 4 + 0);
            const uint8_t* cin = st + cb * 4096;
#pragma unroll
            for (int h = 0; h < 2; ++h, ob ^= 1) {
                const int c16 = uc + 16 * h;  // first unit of this half (tile-relative)
                uint32_t zi[16], zf[16], zg[16], zo[16];
                ptx::tmem_ld_32x32b_x16_(tbase + 0 * U + c16, zi);
                ptx::tmem_ld_32x32b_x16_(tbase + 1 * U + c16, zf);
                ptx::tmem_ld_32x32b_x16_(tbase + 2 * U + c16, zg);
                ptx::tmem_ld_32x32b_x16_(tbase + 3 * U + c16, zo);
                ptx::tmem_ld_wait();
                if (h == 1 && uc + step >= U) release();
                float cp[16];
                if (has_prev) {
                    if (h == 0) {
                        ptx::mbar_wait(ebar + cb, (ephase >> cb) & 1u);
                        ephase ^= 1u << cb;
                    }
                    tc::ld_half_f32_sw128(cin, lane, h, cp);
                } else {
#pragma unroll
                    for (int i = 0; i < 16; ++i) cp[i] = 0.f;
                }
                if (tr && h == 0) tc::trace_once(trace, 12 + (uc / 32) * 4 + 1);
                uint8_t* out = st + 8192 + (NSETS == 2 ? ob * 7168 : 0);
                // the store that last used this output set (NSETS halves ago) has read it
                if (lane == 0) {
                    if constexpr (NSETS == 2) ptx::bulk_wait_read1();
                    else ptx::bulk_wait_read0();
                }
                __syncwarp();
                const int jb = j0 + 16 * h;
                float a[16], gv[16];
                uint32_t w[8];
                // i
#pragma unroll
                for (int i = 0; i < 16; i += 4) {
                    const float4 b4 = __ldg(reinterpret_cast<const float4*>(g.bias + jb + i));
                    a[i] = sigf(__uint_as_float(zi[i]) + b4.x); a[i + 1] = sigf(__uint_as_float(zi[i + 1]) + b4.y);
                    a[i + 2] = sigf(__uint_as_float(zi[i + 2]) + b4.z); a[i + 3] = sigf(__uint_as_float(zi[i + 3]) + b4.w);
                }
#pragma unroll
                for (int i = 0; i < 8; ++i) w[i] = tc::pack_bf16x2(a[2 * i], a[2 * i + 1]);
                tc::st_row_words<32>(out + 2048 + 0 * 1024, lane, w);
                // g, and i*g (c_t = f c_{t-1} + i g, accumulated in two parts)
#pragma unroll
                for (int i = 0; i < 16; i += 4) {
                    const float4 b4 = __ldg(reinterpret_cast<const float4*>(g.bias + 2 * H + jb + i));
                    gv[i] = tanhf_fast(__uint_as_float(zg[i]) + b4.x);
                    gv[i + 1] = tanhf_fast(__uint_as_float(zg[i + 1]) + b4.y);
                    gv[i + 2] = tanhf_fast(__uint_as_float(zg[i + 2]) + b4.z);
                    gv[i + 3] = tanhf_fast(__uint_as_float(zg[i + 3]) + b4.w);
                }
#pragma unroll
                for (int i = 0; i < 8; ++i) w[i] = tc::pack_bf16x2(gv[2 * i], gv[2 * i + 1]);
                tc::st_row_words<32>(out + 2048 + 2 * 1024, lane, w);
#pragma unroll
                for (int i = 0; i < 16; ++i) gv[i] *= a[i];  // i * g
                // f
#pragma unroll
                for (int i = 0; i < 16; i += 4) {
                    const float4 b4 = __ldg(reinterpret_cast<const float4*>(g.bias + H + jb + i));
                    a[i] = sigf(__uint_as_float(zf[i]) + b4.x); a[i + 1] = sigf(__uint_as_float(zf[i + 1]) + b4.y);
                    a[i + 2] = sigf(__uint_as_float(zf[i + 2]) + b4.z); a[i + 3] = sigf(__uint_as_float(zf[i + 3]) + b4.w);
                }
#pragma unroll
                for (int i = 0; i < 8; ++i) w[i] = tc::pack_bf16x2(a[2 * i], a[2 * i + 1]);
                tc::st_row_words<32>(out + 2048 + 1 * 1024, lane, w);
#pragma unroll
                for (int i = 0; i < 16; ++i) cp[i] = a[i] * cp[i] + gv[i];  // c_t
                {
                    uint32_t cw[16];
#pragma unroll
                    for (int i = 0; i < 16; ++i) cw[i] = __float_as_uint(cp[i]);
                    tc::st_row_words<64>(out, lane, cw);
                }
                // o, h
#pragma unroll
                for (int i = 0; i < 16; i += 4) {
                    const float4 b4 = __ldg(reinterpret_cast<const float4*>(g.bias + 3 * H + jb + i));
                    a[i] = sigf(__uint_as_float(zo[i]) + b4.x); a[i + 1] = sigf(__uint_as_float(zo[i + 1]) + b4.y);
                    a[i + 2] = sigf(__uint_as_float(zo[i + 2]) + b4.z); a[i + 3] = sigf(__uint_as_float(zo[i + 3]) + b4.w);
                }
#pragma unroll
                for (int i = 0; i < 8; ++i) w[i] = tc::pack_bf16x2(a[2 * i], a[2 * i + 1]);
                tc::st_row_words<32>(out + 2048 + 3 * 1024, lane, w);
#pragma unroll
                for (int i = 0; i < 8; ++i)
                    w[i] = tc::pack_bf16x2(a[2 * i] * tanhf_fast(cp[2 * i]), a[2 * i + 1] * tanhf_fast(cp[2 * i + 1]));
                tc::st_row_words<32>(out + 6144, lane, w);
                ptx::fence_proxy_async_smem();
                __syncwarp();
                if (lane == 0) {
#ifndef ADPSGD_DBG_NOSTORE  // timing experiments only: no gate stores (h, c still stored)
                    const uint64_t stream = ptx::policy_evict_first();
#pragma unroll
                    for (int gi = 0; gi < 4; ++gi)
                        ptx::tma_store_2d_hint(&g.m_gates, out + 2048 + gi * 1024, gi * H + jb, rowbase + row_out, stream);
#endif
                    ptx::tma_store_2d(&g.m_c, out, jb, rowbase + row_out);
                    ptx::tma_store_2d(&g.m_h, out + 6144, jb, rowbase + row_out);
                    ptx::bulk_commit();
                }
            }
            if (tr) tc::trace_once(trace, 12 + (uc / 32) * 4 + 2);
        }
    }
};

using FwdTraits = FwdT<64>;
using FwdWideTraits = FwdT<128>;

// ---------------- backward ----------------
struct BwdGroup {
    CUtensorMap ta;
    CUtensorMap tb;
    CUtensorMap m_dH, m_dc, m_gates, m_c, m_cp, m_dz;  // epilogue I/O (TMA), 16-unit x 32-row boxes
    int kb;
    const float* dH;
    float* dc_rec;
    const bf16* gates;
    const float* c;
    const float* c_prev;
    bf16* dz;
};
struct BwdParams {
    BwdGroup g[2];
    int ngroups, m_tiles, n_tiles, B, H, lddh, ldg, ldc, lddz;
    int epi_skip;  // debug: timing experiments only
    unsigned long long* trace;
    float* sk_scratch;        // split-K partial exchange (BwdSplitTraits)
    unsigned int* sk_flags;   // split-K epoch counters, one per CTA slot (zeroed once)
};

// BPTT cell-backward epilogue shared by the plain and the split-K recurrent dgrad kernels.
// Row coordinates of the epilogue I/O relative to the warp's local row: tensor maps spanning all
// time steps (persistent BPTT) put dH / c / gates / dz at t*B + row, c_{t-1} at t'*B + row and
// dc_rec at row; the per-step kernels use zero offsets.
struct EpiRows {
    int data = 0, cp = 0, dc = 0;
    bool has_prev = false;
    // persistent BPTT: dc_rec lives in TMEM (column base, per-warp lane quarter) after the first
    // step, and c_t is the c_{t-1} the same CTA loaded one step earlier (also kept in TMEM)
    bool dc_tmem = false;    // read dc_rec from TMEM (else TMA) -- written to TMEM whenever tdc != 0
    bool c_tmem = false;     // read c from TMEM (else TMA); c_{t-1} is written to TMEM whenever tc != 0
    bool tstate = false;     // TMEM state addresses present (TMEM address 0 is a valid lane-quarter-0 address)
    bool tdc_valid = false, tc_valid = false;
    uint32_t tdc = 0, tc_ = 0;
    // compact (8 KB per chunk): dc_rec and c always come from TMEM, so the chunk buffer holds only
    // dH | c_{t-1} | gates (else 12 KB: dH | dc | c | c_{t-1} | gates)
    bool compact = false;
    __device__ int o_cp() const { return compact ? 2048 : 6144; }
    __device__ int o_g() const { return compact ? 4096 : 8192; }
};

struct BwdEpi {
    // The epilogue inputs (dH, dc_rec, c, c_{t-1}, gates) do not depend on the GEMM: epi_begin
    // issues the TMA loads of this warp's first two 16-unit chunks into smem and L2-prefetches
    // the rest while the mainloop runs; body then consumes chunk c from buffer c&1 and refills
    // that buffer with chunk c+2 (two chunks in flight per warp).
    static constexpr int IN_BYTES = 12 * 1024;
    __device__ static EpiRows rows0(const BwdGroup& g) {
        EpiRows r;
        r.has_prev = g.c_prev != nullptr;
        return r;
    }
    __device__ static void issue(const BwdGroup& g, int H, int j0, int rowbase, uint8_t* in, uint64_t* bar, const EpiRows& r) {
        ptx::mbar_arrive_expect_tx(bar, (1 + (r.dc_tmem ? 0 : 1) + (r.c_tmem ? 0 : 1) + (r.has_prev ? 1 : 0)) * 2048 + 4 * 1024);
        const uint64_t stream = ptx::policy_evict_first();
        ptx::tma_load_2d_hint(in, &g.m_dH, bar, j0, rowbase + r.data, stream);
        if (!r.dc_tmem) ptx::tma_load_2d(in + 2048, &g.m_dc, bar, j0, rowbase + r.dc);
        if (!r.c_tmem) ptx::tma_load_2d_hint(in + 4096, &g.m_c, bar, j0, rowbase + r.data, stream);
        if (r.has_prev) ptx::tma_load_2d_hint(in + r.o_cp(), &g.m_cp, bar, j0, rowbase + r.cp, stream);
#pragma unroll
        for (int gi = 0; gi < 4; ++gi)
            ptx::tma_load_2d_hint(in + r.o_g() + gi * 1024, &g.m_gates, bar, gi * H + j0, rowbase + r.data, stream);
    }
    // SMEM: issue the first two chunks into the warp's staging smem (not with an overlaid
    // epilogue: the stages are busy during the mainloop) and L2-prefetch the rest; else
    // L2-prefetch every chunk and let body() issue the first two.
    template <int SPAN, bool SMEM = true>
    __device__ static void begin(const BwdParams& p, int grp, int m0, int u0, int q, int lane, uint8_t* st, uint64_t* ebar,
                                 tc::EpiSlot sl) {
        begin_g<SPAN, SMEM>(p.g[grp], p.H, m0, u0, q, lane, st, ebar, sl, rows0(p.g[grp]));
    }
    template <int SPAN, bool SMEM = true, int NBUF = 2>
    __device__ static void begin_g(const BwdGroup& g, int H, int m0, int u0, int q, int lane, uint8_t* st, uint64_t* ebar,
                                   tc::EpiSlot sl, const EpiRows& r) {
        const int rowbase = m0 + q * 32;
        const int step = 16 * sl.n;
        if (SMEM && lane == 0) {
            int b = 0;
            for (int uc = 16 * sl.sub; uc < SPAN && b < NBUF; uc += step, ++b) issue(g, H, u0 + uc, rowbase, st + b * IN_BYTES, ebar + b, r);
        }
        // L2 prefetch of the remaining chunks: one box per lane
        const bool has_prev = r.has_prev;
        for (int uc = 16 * sl.sub + (SMEM ? NBUF * step : 0), i = 0; uc < SPAN; uc += step, ++i) {
            const int j0 = u0 + uc;
            const int box = lane & 7;
            if ((lane >> 3) != (i & 3)) continue;
            if (box == 0) ptx::tma_prefetch_l2_2d(&g.m_dH, j0, rowbase + r.data);
            else if (box == 1) { if (!r.dc_tmem) ptx::tma_prefetch_l2_2d(&g.m_dc, j0, rowbase + r.dc); }
            else if (box == 2) { if (!r.c_tmem) ptx::tma_prefetch_l2_2d(&g.m_c, j0, rowbase + r.data); }
            else if (box == 3) { if (has_prev) ptx::tma_prefetch_l2_2d(&g.m_cp, j0, rowbase + r.cp); }
            else ptx::tma_prefetch_l2_2d(&g.m_gates, (box - 4) * H + j0, rowbase + r.data);
        }
    }
    // epilogue (thread = row), per 16-unit chunk: dh_rec leaves TMEM; the cell backward runs in
    // registers on the chunk's prefetched inputs; dz (4 x bf16) and dc_rec leave by TMA stores.
    // peer (split-K only): the partner CTA's fp32 partial of this CTA's units, [chunk][row][16]
    // INPLACE: outputs are staged in the consumed input buffer (24 KB per warp instead of 30);
    // the buffer is refilled with chunk c+2 once the chunk's stores have read it.
    template <int SPAN, bool INPLACE = false, class Rel>
    __device__ static void body(const BwdParams& p, int grp, int m0, int u0, uint32_t tbase, int q, int lane,
                                Rel release, uint8_t* st, uint64_t* ebar, uint32_t& ephase, tc::EpiSlot sl,
                                const float* peer, bool preissued = true) {
        body_g<SPAN, INPLACE>(p.g[grp], p.H, m0, u0, tbase, q, lane, release, st, ebar, ephase, sl, peer, preissued,
                              rows0(p.g[grp]));
    }
    // NBUF: input buffers per warp (chunks in flight); INPLACE with NBUF = 1 needs 12 KB per warp.
    template <int SPAN, bool INPLACE, class Rel, int NBUF = 2>
    __device__ static void body_g(const BwdGroup& g, int H, int m0, int u0, uint32_t tbase, int q, int lane,
                                  Rel release, uint8_t* st, uint64_t* ebar, uint32_t& ephase, tc::EpiSlot sl,
                                  const float* peer, bool preissued, const EpiRows& r, const float* peer2 = nullptr,
                                  const float* peer3 = nullptr) {
        static_assert(NBUF == 2 || INPLACE, "a single input buffer needs in-place outputs");
        const int rowbase = m0 + q * 32;
        uint8_t* bdz = st + 2 * IN_BYTES;         // 4 x 1 KB (INPLACE: in the chunk's input buffer)
        uint8_t* bdco = st + 2 * IN_BYTES + 4096;  // 2 KB
        const bool has_prev = r.has_prev;
        const int step = 16 * sl.n;
        if (!preissued && lane == 0) {
            int bb = 0;
            for (int uc = 16 * sl.sub; uc < SPAN && bb < NBUF; uc += step, ++bb) issue(g, H, u0 + uc, rowbase, st + bb * IN_BYTES, ebar + bb, r);
        }
        int b = 0;
#pragma unroll 1
        for (int uc = 16 * sl.sub; uc < SPAN; uc += step, b = (b + 1) % NBUF) {
            const int j0 = u0 + uc;
            uint8_t* in = st + b * IN_BYTES;
            uint32_t acc[16];
            ptx::tmem_ld_32x32b_x16_(tbase + uc, acc);
            ptx::tmem_ld_wait_regs(acc);
            if (uc + step >= SPAN) release();
            // split-K partners' partials of these units, added in a fixed order (deterministic)
            const float* peers[3] = {peer, peer2, peer3};
#pragma unroll
            for (int pi = 0; pi < 3; ++pi) {
                if (!peers[pi]) continue;
                const float4* pp = reinterpret_cast<const float4*>(peers[pi] + ((uc / 16) * 128 + q * 32 + lane) * 16);
                float4 f[4];
#pragma unroll
                for (int v = 0; v < 4; ++v) f[v] = __ldcg(pp + v);
#pragma unroll
                for (int v = 0; v < 4; ++v) {
                    acc[4 * v] = __float_as_uint(__uint_as_float(acc[4 * v]) + f[v].x);
                    acc[4 * v + 1] = __float_as_uint(__uint_as_float(acc[4 * v + 1]) + f[v].y);
                    acc[4 * v + 2] = __float_as_uint(__uint_as_float(acc[4 * v + 2]) + f[v].z);
                    acc[4 * v + 3] = __float_as_uint(__uint_as_float(acc[4 * v + 3]) + f[v].w);
                }
            }
            ptx::mbar_wait(ebar + b, (ephase >> b) & 1u);
            ephase ^= 1u << b;
            uint32_t wdh[16], wdc[16], wc[16], wcp[16], wi[8], wf[8], wg[8], wo[8];
            if (r.dc_tmem || r.c_tmem) {  // (same lane quarter as the accumulator; uc = the chunk's column)
                __syncwarp();  // tcgen05.ld is .sync.aligned: reconverge after the per-thread mbarrier spin
                if (r.dc_tmem) ptx::tmem_ld_32x32b_x16_(r.tdc + uc, wdc);
                if (r.c_tmem) ptx::tmem_ld_32x32b_x16_(r.tc_ + uc, wc);
                if (r.dc_tmem) ptx::tmem_ld_wait_regs(wdc);
                if (r.c_tmem) ptx::tmem_ld_wait_regs(wc);
            }
            tc::ld_row_words<64>(in, lane, wdh);
            if (!r.dc_tmem) tc::ld_row_words<64>(in + 2048, lane, wdc);
            if (!r.c_tmem) tc::ld_row_words<64>(in + 4096, lane, wc);
            if (has_prev) tc::ld_row_words<64>(in + r.o_cp(), lane, wcp);
            if (r.tstate && r.tc_valid && has_prev) {  // c_{t-1} is the next step's c
                __syncwarp();
                ptx::tmem_st_32x32b_x16(r.tc_ + uc, wcp);
            }
            tc::ld_row_words<32>(in + r.o_g() + 0 * 1024, lane, wi);
            tc::ld_row_words<32>(in + r.o_g() + 1 * 1024, lane, wf);
            tc::ld_row_words<32>(in + r.o_g() + 2 * 1024, lane, wg);
            tc::ld_row_words<32>(in + r.o_g() + 3 * 1024, lane, wo);
            uint32_t zi[8], zf[8], zg[8], zo[8], dco[16];
#pragma unroll
            for (int e = 0; e < 16; ++e) {
                const int w = e >> 1;
                const bool hi = e & 1;
                const float ig = hi ? tc::bf16_hi(wi[w]) : tc::bf16_lo(wi[w]);
                const float fg = hi ? tc::bf16_hi(wf[w]) : tc::bf16_lo(wf[w]);
                const float gg = hi ? tc::bf16_hi(wg[w]) : tc::bf16_lo(wg[w]);
                const float og = hi ? tc::bf16_hi(wo[w]) : tc::bf16_lo(wo[w]);
                const float dh = __uint_as_float(wdh[e]) + __uint_as_float(acc[e]);
                const float tc = tanhf_fast(__uint_as_float(wc[e]));
                const float cp = has_prev ? __uint_as_float(wcp[e]) : 0.f;
                const float dc = __uint_as_float(wdc[e]) + dh * og * (1.f - tc * tc);
                const float vi = dc * gg * ig * (1.f - ig);
                const float vf = dc * cp * fg * (1.f - fg);
                const float vg = dc * ig * (1.f - gg * gg);
                const float vo = dh * tc * og * (1.f - og);
                dco[e] = __float_as_uint(dc * fg);
                if (hi) {
                    zi[w] = tc::pack_bf16x2(__uint_as_float(zi[w]), vi);
                    zf[w] = tc::pack_bf16x2(__uint_as_float(zf[w]), vf);
                    zg[w] = tc::pack_bf16x2(__uint_as_float(zg[w]), vg);
                    zo[w] = tc::pack_bf16x2(__uint_as_float(zo[w]), vo);
                } else {
                    zi[w] = __float_as_uint(vi); zf[w] = __float_as_uint(vf);
                    zg[w] = __float_as_uint(vg); zo[w] = __float_as_uint(vo);
                }
            }
            if (INPLACE) {
                bdz = in;  // dz over the consumed dH | dc boxes, dc_rec over the c box
                bdco = in + 4096;
                __syncwarp();  // every lane has read its inputs
            } else {
                // every lane has consumed its inputs: refill this buffer with chunk c + 2; and the
                // previous chunk's stores must have read the output boxes before they are rewritten
                if (lane == 0) ptx::bulk_wait_read0();
                __syncwarp();
                if (lane == 0 && uc + 2 * step < SPAN) issue(g, H, j0 + 2 * step, rowbase, in, ebar + b, r);
            }
            tc::st_row_words<32>(bdz + 0 * 1024, lane, zi);
            tc::st_row_words<32>(bdz + 1 * 1024, lane, zf);
            tc::st_row_words<32>(bdz + 2 * 1024, lane, zg);
            tc::st_row_words<32>(bdz + 3 * 1024, lane, zo);
            if (r.tstate && r.tdc_valid) {
                __syncwarp();
                ptx::tmem_st_32x32b_x16(r.tdc + uc, dco);
                ptx::tmem_st_wait();
            } else {
                tc::st_row_words<64>(bdco, lane, dco);
            }
            ptx::fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) {
#ifndef ADPSGD_DBG_BWD_NOSTORE  // timing experiments only: dz not stored
#pragma unroll
                for (int gi = 0; gi < 4; ++gi) ptx::tma_store_2d(&g.m_dz, bdz + gi * 1024, gi * H + j0, rowbase + r.data);
#endif
                if (!(r.tstate && r.tdc_valid)) ptx::tma_store_2d(&g.m_dc, bdco, j0, rowbase + r.dc);
                ptx::bulk_commit();
                if (INPLACE && uc + NBUF * step < SPAN) {
                    ptx::bulk_wait_read0();  // the stores have read the buffer: refill it with chunk c + NBUF
                    issue(g, H, j0 + NBUF * step, rowbase, in, ebar + b, r);
                }
            }
        }
    }
};

template <int BN_>
struct BwdTraits : tc::TraitsBase, BwdEpi {
    static constexpr int BN = BN_;
    // per warp (30 KB): two input sets (12 KB each: dH | dc | c | c_prev fp32 16x32 SW64 2 KB each,
    // gates 4 x bf16 16x32 SW32 1 KB) | dz out 4 x 1 KB | dc out 2 KB
    static constexpr int EPI_WARPS = 4;
    static constexpr int EPI_SMEM = EPI_WARPS * 30 * 1024;
    static constexpr bool B_MN = true;
    __device__ static int num_tiles(const BwdParams& p) { return p.ngroups * p.m_tiles * p.n_tiles; }
    __device__ static void prefetch(const BwdParams& p) {
        for (int i = 0; i < p.ngroups; ++i) { ptx::tma_prefetch(&p.g[i].ta); ptx::tma_prefetch(&p.g[i].tb); }
    }
    __device__ static void coords(const BwdParams& p, int tile, int& grp, int& m0, int& u0) {
        const int per = p.m_tiles * p.n_tiles;
        grp = tile / per;
        const int r = tile % per;
        m0 = (r % p.m_tiles) * kBM;
        u0 = (r / p.m_tiles) * BN;
    }
    __device__ static int kblocks(const BwdParams& p, int tile) { return p.g[tile / (p.m_tiles * p.n_tiles)].kb; }
    __device__ static void load(const BwdParams& p, int tile, int kb, uint8_t* sA, uint8_t* sB, uint64_t* bar) {
        int grp, m0, u0;
        coords(p, tile, grp, m0, u0);
        const BwdGroup& g = p.g[grp];
        const int k0 = kb * kBK;
        ptx::tma_load_2d_hint(sA, &g.ta, bar, k0, m0, ptx::policy_evict_first());
        const uint64_t keep = ptx::policy_evict_last();
#pragma unroll
        for (int j = 0; j < BN / 64; ++j)
            ptx::tma_load_2d_hint(sB + j * 64 * kBK * 2, &g.tb, bar, u0 + 64 * j, k0, keep);
    }
    // CTA pair (BN = pair tile width): rank r loads A rows [m0 + 128 r, +128) and units
    // [u0 + r BN/2, +BN/2) of W_hh (MN-major)
    static constexpr bool A_MN = false;
    __device__ static void coords2(const BwdParams& p, int tile, int& grp, int& m0, int& u0) {
        const int per = p.m_tiles * p.n_tiles;
        grp = tile / per;
        const int r = tile % per;
        m0 = (r % p.m_tiles) * 2 * kBM;
        u0 = (r / p.m_tiles) * BN;
    }
    __device__ static void load2(const BwdParams& p, int tile, int kb, uint32_t rank, uint8_t* sA, uint8_t* sB,
                                 uint32_t bar) {
        int grp, m0, u0;
        coords2(p, tile, grp, m0, u0);
        const BwdGroup& g = p.g[grp];
        const int k0 = kb * kBK;
        ptx::tma_load_2d_2sm_hint(sA, &g.ta, bar, k0, m0 + kBM * rank, ptx::policy_evict_first());
        const uint64_t keep = ptx::policy_evict_last();
#pragma unroll
        for (int j = 0; j < BN / 128; ++j)
            ptx::tma_load_2d_2sm_hint(sB + j * 64 * kBK * 2, &g.tb, bar, u0 + rank * (BN / 2) + 64 * j, k0, keep);
    }
    template <class S>
    __device__ static void epi_begin2(const BwdParams& p, int tile, uint32_t rank, int q, int lane, uint8_t* st,
                                      uint64_t* ebar, S sl) {
        int grp, m0, u0;
        coords2(p, tile, grp, m0, u0);
        begin<BN>(p, grp, m0 + kBM * rank, u0, q, lane, st, ebar, sl);
    }
    template <class S>
    __device__ static void epi_begin(const BwdParams& p, int tile, int q, int lane, uint8_t* st, uint64_t* ebar, S sl) {
        int grp, m0, u0;
        coords(p, tile, grp, m0, u0);
        begin<BN>(p, grp, m0, u0, q, lane, st, ebar, sl);
    }
    __device__ static void epilogue2(const BwdParams& p, int tile, uint32_t rank, uint32_t tbase, int q, int lane,
                                     uint32_t tempty_leader, uint8_t* st, uint64_t* ebar, uint32_t& ephase,
                                     tc::EpiSlot sl) {
        int grp, m0, u0;
        coords2(p, tile, grp, m0, u0);
        body<BN>(p, grp, m0 + kBM * rank, u0, tbase, q, lane, [&] { tc::release_acc_2sm(tempty_leader, lane); }, st,
                 ebar, ephase, sl, nullptr);
    }
    __device__ static void epilogue(const BwdParams& p, int tile, uint32_t tbase, int q, int lane, uint64_t* tempty,
                                    uint8_t* st, uint64_t* ebar, uint32_t& ephase, tc::EpiSlot sl) {
        int grp, m0, u0;
        coords(p, tile, grp, m0, u0);
        body<BN>(p, grp, m0, u0, tbase, q, lane, [&] { tc::release_acc(tempty, lane); }, st, ebar, ephase, sl, nullptr);
    }
};

// Split-K BPTT dgrad (CTA pairs, 256 x 256 tiles, K = 4H halved): work unit w = (dir, m, n, kh)
// computes a K-half partial of a 256-row x 256-unit tile; the two halves exchange the half of
// the partial the other one finalises through a global scratch (64 KB per CTA, L2-resident) and
// an epoch-counter handshake, then each CTA runs the cell backward on 128 rows x 128 units.
// Operand traffic drops by a third vs 256 x 128 tiles. Requires every work unit resident at
// once (host checks 2 x tiles <= 148 CTAs; one unit per CTA).
struct BwdSplitTraits : tc::TraitsBase, BwdEpi {
    static constexpr int BN = 256;
    static constexpr int EPI_WARPS = 8;
    static constexpr int EPI_SMEM = EPI_WARPS * 24 * 1024;  // BwdEpi::body<.., INPLACE>
    static constexpr int ACC_STAGES = 1;
    static constexpr bool EPI_OVERLAY = true;  // one unit per CTA: all smem to the mainloop stages
    static constexpr bool A_MN = false;
    static constexpr bool B_MN = true;
    __device__ static int num_tiles(const BwdParams& p) { return p.ngroups * p.m_tiles * p.n_tiles * 2; }
    __device__ static void prefetch(const BwdParams& p) {
        for (int i = 0; i < p.ngroups; ++i) { ptx::tma_prefetch(&p.g[i].ta); ptx::tma_prefetch(&p.g[i].tb); }
    }
    // tile = ((grp * n_tiles + nt) * m_tiles + mt) * 2 + kh
    __device__ static void coords2(const BwdParams& p, int tile, int& grp, int& m0, int& u0, int& kh) {
        kh = tile & 1;
        const int r = tile >> 1;
        const int mt = r % p.m_tiles, rn = r / p.m_tiles;
        m0 = mt * 2 * kBM;
        u0 = (rn % p.n_tiles) * BN;
        grp = rn / p.n_tiles;
    }
    __device__ static int kblocks(const BwdParams& p, int tile) {
        int grp, m0, u0, kh;
        coords2(p, tile, grp, m0, u0, kh);
        const int kb = p.g[grp].kb;
        return kh == 0 ? kb / 2 : kb - kb / 2;
    }
    __device__ static void load2(const BwdParams& p, int tile, int kb, uint32_t rank, uint8_t* sA, uint8_t* sB,
                                 uint32_t bar) {
        int grp, m0, u0, kh;
        coords2(p, tile, grp, m0, u0, kh);
        const BwdGroup& g = p.g[grp];
        const int k0 = (kh * (g.kb / 2) + kb) * kBK;
        ptx::tma_load_2d_2sm_hint(sA, &g.ta, bar, k0, m0 + kBM * rank, ptx::policy_evict_first());
        const uint64_t keep = ptx::policy_evict_last();
#pragma unroll
        for (int j = 0; j < BN / 128; ++j)
            ptx::tma_load_2d_2sm_hint(sB + j * 64 * kBK * 2, &g.tb, bar, u0 + rank * (BN / 2) + 64 * j, k0, keep);
    }
    template <class S>
    __device__ static void epi_begin2(const BwdParams& p, int tile, uint32_t rank, int q, int lane, uint8_t* st,
                                      uint64_t* ebar, S sl) {
        int grp, m0, u0, kh;
        coords2(p, tile, grp, m0, u0, kh);
        begin<128, false>(p, grp, m0 + kBM * rank, u0 + 128 * kh, q, lane, st, ebar, sl);
    }
    __device__ static void epilogue2(const BwdParams& p, int tile, uint32_t rank, uint32_t tbase, int q, int lane,
                                     uint32_t tempty_leader, uint8_t* st, uint64_t* ebar, uint32_t& ephase,
                                     tc::EpiSlot sl) {
        int grp, m0, u0, kh;
        coords2(p, tile, grp, m0, u0, kh);
        const int slot = tile * 2 + static_cast<int>(rank), peer_slot = (tile ^ 1) * 2 + static_cast<int>(rank);
        constexpr int kSlot = 128 * 128;  // floats
        // 1) export the half the partner finalises: [chunk][row][16] fp32 (coalesced 2 KB per warp chunk)
        float* mine = p.sk_scratch + static_cast<int64_t>(slot) * kSlot;
        const int row = q * 32 + lane;
#pragma unroll 1
        for (int c = sl.sub; c < 8; c += sl.n) {
            uint32_t v[16];
            ptx::tmem_ld_32x32b_x16_(tbase + (1 - kh) * 128 + 16 * c, v);
            ptx::tmem_ld_wait();
            float4* dst = reinterpret_cast<float4*>(mine + (c * 128 + row) * 16);
#pragma unroll
            for (int k = 0; k < 4; ++k)
                __stcg(dst + k, make_float4(__uint_as_float(v[4 * k]), __uint_as_float(v[4 * k + 1]),
                                            __uint_as_float(v[4 * k + 2]), __uint_as_float(v[4 * k + 3])));
        }
        // 2) handshake: epoch counters (one increment per launch per slot; no reset needed)
        if (q == 2 && lane == 0) tc::trace_once(p.trace, 12);
        ptx::named_sync(2, 32 * EPI_WARPS);
        if (q == 0 && sl.sub == 0 && lane == 0) {
            __threadfence();  // (8 epilogue warps: (q, sub) = (0, 0) is warp 2)
            const unsigned mine_epoch = atomicAdd(p.sk_flags + slot, 1u) + 1u;
            ptx::spin_until_geq(p.sk_flags + peer_slot, mine_epoch);
            __threadfence();
        }
        ptx::named_sync(2, 32 * EPI_WARPS);
        if (q == 2 && lane == 0) tc::trace_once(p.trace, 13);
        // 3) cell backward on the owned 128 units with the partner's partial added
        body<128, true>(p, grp, m0 + kBM * rank, u0 + 128 * kh, tbase + 128 * kh, q, lane,
                  [&] { tc::release_acc_2sm(tempty_leader, lane); }, st, ebar, ephase, sl,
                  p.sk_scratch + static_cast<int64_t>(peer_slot) * kSlot, false);
    }
};

// ---------------- persistent forward recurrence (one launch per layer) ----------------
// All T steps of both directions in one kernel: CTA pair c owns (m-tile, 64-unit tile) for both
// directions and walks items (step s, direction d) = d0(s0) d1(s0) d0(s1) ...; 256 x 256 tiles
// (64 units x 4 gates, FwdT<64> layout) with two TMEM accumulator stages, so one direction's
// cell epilogue runs under the other direction's mainloop. Each item's k-blocks run x_t first
// (no dependency) and h_{t-1} last: only the recurrent k-blocks wait for the previous step's
// h rows of the m-tile (per (d, m-tile, rank) counters of finished epilogues).
struct FwdPParams {
    FwdGroup g[2];  // ta[0] = X (T*B rows), tb[0] = W_ih(d); ta[1] = Hout(d) (T*B rows), tb[1] = W_hh(d);
                    // m_cprev / m_gates / m_c / m_h span T*B rows; bias per direction
    int B, H, T, m_tiles, n_tiles, units, kbx, kbh;
    unsigned int* dep;       // [dir][m_tile][rank] finished epilogues
    unsigned int* exit_ctr;
    unsigned long long* trace;
};

// UW = hidden units per tile (x 4 gates = BN): 64 by default; 32 when 64-unit tiles would leave
// most CTA pairs idle (H = 512: 4 row blocks x 8 unit blocks = 32 tiles for 74 pairs).
template <int UW>
struct FwdPersistT : tc::TraitsBase {
    using F = FwdT<UW>;
    static constexpr int BN = 4 * UW;
#ifdef ADPSGD_FWD_TWO_SETS
    static constexpr int OUT_SETS = 2;
#else
    static constexpr int OUT_SETS = 1;  // one output staging set per warp: 15 KB, 5 mainloop stages instead of 4
#endif
    static constexpr int EPI_WARP = OUT_SETS == 2 ? F::EPI_WARP : 15 * 1024;
    static constexpr int EPI_WARPS = 4;
    static constexpr int EPI_SMEM = EPI_WARPS * EPI_WARP;
    static constexpr int ACC_STAGES = 2;
    static constexpr bool A_MN = false;
    static constexpr bool B_MN = false;
    static constexpr bool STREAMK = true;
    struct U {
        int mt, nt, s, d, t, tp;
    };
    __device__ static U unit(const FwdPParams& p, int cid, int it) {
        U u;
        u.mt = cid % p.m_tiles;
        u.nt = cid / p.m_tiles;
        u.s = it >> 1;
        u.d = it & 1;
        u.t = u.d == 0 ? u.s : p.T - 1 - u.s;
        u.tp = u.d == 0 ? u.t - 1 : u.t + 1;
        return u;
    }
    __device__ static int num_tiles(const FwdPParams& p) { return 2 * p.T; }
    __device__ static int kblocks(const FwdPParams& p, int it) { return p.kbx + ((it >> 1) > 0 ? p.kbh : 0); }
    __device__ static void prefetch(const FwdPParams& p) {
        for (int i = 0; i < 2; ++i)
            for (int s = 0; s < 2; ++s) { ptx::tma_prefetch(&p.g[i].ta[s]); ptx::tma_prefetch(&p.g[i].tb[s]); }
    }
    __device__ static bool sk_item(const FwdPParams& p, int cid, int, int it, tc::Item& w) {
        if (cid >= p.units || it >= 2 * p.T) return false;
        w.tile = it; w.kb0 = 0; w.kb1 = kblocks(p, it); w.role = 0;
        return true;
    }
    __device__ static void kb_ready(const FwdPParams& p, const tc::Item& w, int kb, int cid, uint32_t rank) {
#ifdef ADPSGD_DBG_NODEP  // timing experiments only: no cross-CTA step dependency
        return;
#endif
        if (kb != p.kbx) return;  // first recurrent k-block: h_{t-1} of every unit tile of this m-tile
        const U u = unit(p, cid, w.tile);
        const unsigned need = static_cast<unsigned>(u.s) * p.n_tiles;
        const unsigned* f = p.dep + (u.d * p.m_tiles + u.mt) * 2 + rank;
        // trace (tools/trace_fwd.py): producer reaches / passes the h-part dependency of items 4, 5, 8
        const int tev = w.tile == 4 ? 40 : w.tile == 5 ? 42 : w.tile == 8 ? 44 : -1;
        if (tev >= 0) tc::trace_once(p.trace, tev);
        ptx::spin_until_geq(f, need);
        if (tev >= 0) tc::trace_once(p.trace, tev + 1);
        asm volatile("fence.proxy.async.global;" ::: "memory");
    }
    // per-item TMA context (tc_core.cuh HasLoadCtx): segment 0 = x-part (X, W_ih), 1 = h-part (Hout, W_hh)
    struct LoadCtx {
        const CUtensorMap* a[2];
        const CUtensorMap* b[2];
        int row[2], brow, bgate, H, kbx;
        uint64_t keep;
    };
    __device__ static LoadCtx load_ctx(const FwdPParams& p, int it, uint32_t rank) {
        const U u = unit(p, blockIdx.x >> 1, it);
        const FwdGroup& g = p.g[u.d];
        LoadCtx c;
        const int r0 = u.mt * 2 * kBM + kBM * static_cast<int>(rank);
        for (int sgm = 0; sgm < 2; ++sgm) { c.a[sgm] = &g.ta[sgm]; c.b[sgm] = &g.tb[sgm]; }
#ifdef ADPSGD_DBG_FIXROWS  // timing experiments only: every step reads the rows of t = 0
        c.row[0] = r0;
        c.row[1] = r0;
#else
        c.row[0] = u.t * p.B + r0;
        c.row[1] = u.tp * p.B + r0;
#endif
        c.brow = u.nt * UW;  // units of the 3-D gate-block view; gate blocks 2r, 2r + 1
        c.bgate = 2 * static_cast<int>(rank);
        c.H = p.H;
        c.kbx = p.kbx;
        c.keep = ptx::policy_evict_last();
        return c;
    }
    // A rows are read by every unit tile of the m-tile, at different times in the persistent
    // schedule: default L2 policy (evict_first cost DRAM re-reads); B (weights) evict_last
    __device__ static void load2c(const LoadCtx& c, int kb, uint8_t* sA, uint8_t* sB, uint32_t bar) {
        const int seg = kb < c.kbx ? 0 : 1;
        const int k0 = (kb - seg * c.kbx) * kBK;
        ptx::tma_load_2d_2sm(sA, c.a[seg], bar, k0, c.row[seg]);
        ptx::tma_load_3d_2sm_hint(sB, c.b[seg], bar, k0, c.brow, c.bgate, c.keep);
    }
    template <class S>
    __device__ static void epi_begin2(const FwdPParams& p, int it, uint32_t rank, int q, int lane, uint8_t*, uint64_t*,
                                      S sl) {
        const U u = unit(p, blockIdx.x >> 1, it);
#ifdef ADPSGD_DBG_NOEPI
        return;
#endif
        if (u.s == 0) return;
        const int uc = 32 * sl.sub + 32 * sl.n * (lane & 1);
        if (lane < 2 && uc < UW)
            ptx::tma_prefetch_l2_2d(&p.g[u.d].m_cprev, u.nt * UW + uc,
                                    u.tp * p.B + u.mt * 2 * kBM + kBM * static_cast<int>(rank) + q * 32);
    }
    __device__ static void epilogue_sk(const FwdPParams& p, const tc::Item& w, int cid, uint32_t rank, uint32_t tbase,
                                       int q, int lane, uint32_t tempty_leader, tc::EpiSlot sl, uint8_t* st,
                                       uint64_t* ebar, uint32_t& ephase) {
        const U u = unit(p, cid, w.tile);
#ifdef ADPSGD_DBG_NOEPI  // timing experiments only: release the accumulator, publish, no cell
        tc::release_acc_2sm(tempty_leader, lane);
#else
        auto rel = [&] { tc::release_acc_2sm(tempty_leader, lane); };
        F::template body_g<decltype(rel), OUT_SETS>(p.g[u.d], p.H, u.mt * 2 * kBM + kBM * static_cast<int>(rank), u.nt * UW,
                                                    tbase, q, lane, rel, st, ebar, ephase, sl, nullptr, u.t * p.B,
                                                    u.s > 0 ? u.tp * p.B : 0, u.s > 0);
#endif
        // publish: this CTA's h_t (and c_t) block is in memory
#ifdef ADPSGD_DBG_NOPUB  // timing experiments only (with ADPSGD_DBG_NODEP): no publication at all
        if (true) return;
#endif
        if (lane == 0) {
            ptx::bulk_wait0();
            asm volatile("fence.proxy.async.global;" ::: "memory");
        }
        ptx::named_sync(2, 32 * EPI_WARPS);
        if (q == 0 && sl.sub == 0 && lane == 0) {
#ifndef ADPSGD_DBG_NOFENCE
            __threadfence();
#endif
            atomicAdd(p.dep + (u.d * p.m_tiles + u.mt) * 2 + rank, 1u);
            if (w.tile == 2 * p.T - 1) {
                __threadfence();
                if (atomicAdd(p.exit_ctr, 1u) == gridDim.x - 1) {
                    for (int i = 0; i < 2 * p.m_tiles * 2; ++i) p.dep[i] = 0u;
                    __threadfence();
                    *p.exit_ctr = 0u;
                }
            }
        }
    }
};

using FwdPersistTraits = FwdPersistT<64>;

// ---------------- persistent BPTT (one launch per layer) ----------------
// All T-1 recurrent steps of both directions in one kernel. CTA pair c owns work unit
// (m-tile, n-tile, K-half) for BOTH directions and walks items (step s, direction d) in the order
// (0,0) (1,0)... i.e. d0(s0) d1(s0) d0(s1) d1(s1): with two TMEM accumulator stages the cell-
// backward epilogue of one direction runs while the tensor cores work on the other direction,
// so the epilogue hides behind the mainloop. Step s+1 of direction d needs dz_{t}(d) rows of its
// m-tile from every (n-tile, K-half) unit: per (d, m-tile, rank) counters of finished
// epilogues (release / acquire, proxy fences around the TMA traffic) replace kernel boundaries.
// Split-K partials meet in a parity-double-buffered global scratch (see BwdSplitTraits).
struct BwdPParams {
    BwdGroup g[2];  // maps span all T*B rows: ta = dZ(d), tb = W_hh(d), m_dH / m_c / m_cp / m_gates / m_dz; m_dc = dc_rec(d)
    int B, H, T, m_tiles, n_tiles, units, kbh;
    int64_t ldc;             // row pitch of c (first_step_state)
    float* sk_scratch;       // [pair * 2 + rank][parity][4 chunks][128 rows][16] fp32
    unsigned int* sk_flags;  // [pair * 2 + rank] exchange epochs
    unsigned int* dep;       // [dir][m_tile][rank] finished epilogues
    unsigned int* exit_ctr;
    int epi_skip;
    unsigned long long* trace;
};

// KQ = K splits per tile: KQ = 2 -> 256 x 128 pair tiles (K halves); KQ = 4 -> 256 x 256 tiles
// (K quarters: a third less operand ingress per FLOP, three partials per owned block).
// UC = units each CTA finalises: 64, or 32 (H <= 512: twice the CTA pairs, half the epilogue per
// item). UC = 32 reads B = W_hh^T (a K-major transposed copy, [H x 4H]) so 32-unit B tiles
// stay in the 128-byte-swizzle layout.
template <int KQ, int UC = 64, bool KMAJ = false>
struct BwdPersistTraits : tc::TraitsBase, BwdEpi {
    static constexpr int BN = UC * KQ;  // pair tile width
    static constexpr int NCHK = UC / 16;  // 16-unit chunks per finalised block
#ifdef ADPSGD_NO_TSTATE
    static constexpr bool TSTATE_ = false;
#else
    static constexpr bool TSTATE_ = KQ == 2;
#endif
#ifdef ADPSGD_BWD_EPI_WARPS
    static constexpr int EPI_WARPS = ADPSGD_BWD_EPI_WARPS;  // A/B experiments
#else
    static constexpr int EPI_WARPS = 8;
#endif
    // BwdEpi::body_g<64, INPLACE, .., NBUF = 1>: 12 KB per warp, or 8 KB (compact chunk buffer) when
    // dc_rec / c live in TMEM from the first step on -- the saved 32 KB buy a 6th mainloop stage
    static constexpr int EPI_SMEM = EPI_WARPS * (TSTATE_ ? 8 : 12) * 1024;
    static constexpr int ACC_STAGES = 2;
    static constexpr bool A_MN = false;
    static constexpr bool B_MN = UC == 64 && !KMAJ;  // KMAJ: K-major W_hh^T for the 64-unit tiles too
    static constexpr bool STREAMK = true;
    // TMEM past the accumulators (KQ = 2 only: 2 BN + 4 UC <= 512 columns): per direction d,
    // dc_rec at [2 BN + UC d, +UC) and the carried c at [2 BN + 2 UC + UC d, +UC)
#ifdef ADPSGD_NO_TSTATE
    static constexpr bool TSTATE = false;
#else
    static constexpr bool TSTATE = KQ == 2;
#endif
    static constexpr int TMEM_EXTRA = TSTATE ? 4 * UC : 0;
    static constexpr int kBlock = NCHK * 128 * 16;  // floats of one exported block: [chunks][128 rows][16]
    struct U {
        int mt, nt, kh, s, d;
    };
    __device__ static U unit(const BwdPParams& p, int cid, int it) {
        U u;
        u.mt = cid % p.m_tiles;
        u.nt = (cid / p.m_tiles) % p.n_tiles;
        u.kh = cid / (p.m_tiles * p.n_tiles);
        u.s = it >> 1;
        u.d = it & 1;
        return u;
    }
    // time rows: A = dz_{t_src}; the cell backward runs at tn with c_{tnp}
    __device__ static int t_src(const BwdPParams& p, const U& u) { return u.d == 0 ? p.T - 1 - u.s : u.s; }
    __device__ static EpiRows rows(const BwdPParams& p, const U& u, uint32_t tmem_q = 0, bool have_q = false) {
        const int tn = u.d == 0 ? p.T - 2 - u.s : u.s + 1;
        const int tnp = u.d == 0 ? tn - 1 : tn + 1;
        EpiRows r;
        r.data = tn * p.B;
        r.has_prev = tnp >= 0 && tnp < p.T;
        r.cp = r.has_prev ? tnp * p.B : 0;
        r.dc = 0;
        if (TSTATE) {
            // dc_rec and c_t always from TMEM: the first step's (the first cell backward's dc_rec and
            // c_{T-2} / c_1) are put there by first_step_state() before that step's cell backward;
            // after it, c_t is the c_{t-1} this CTA loaded one step earlier
            r.dc_tmem = true;
            r.c_tmem = true;
            r.compact = true;
            if (have_q) {         // tmem_q: TMEM base of this warp's lane quarter (epilogue only)
                r.tstate = true;
                r.tdc = tmem_q + 2 * BN + UC * u.d;
                r.tc_ = tmem_q + 2 * BN + 2 * UC + UC * u.d;
                r.tdc_valid = true;
                r.tc_valid = true;
            }
        }
        return r;
    }
    // First BPTT step of each direction: load this thread's row of dc_rec (the first cell backward's
    // output) and of c at tn into the TMEM state columns, for the chunks this warp owns.
    __device__ static void first_step_state(const BwdPParams& p, const U& u, int m0, int u0, int q, int lane, tc::EpiSlot sl,
                                            const EpiRows& r) {
        const BwdGroup& g = p.g[u.d];
        const int64_t row = m0 + q * 32 + lane;
        const float* dcrow = g.dc_rec + row * p.H;
        const float* crow = g.c + (r.data + row) * p.ldc;
#pragma unroll 1
        for (int uc = 16 * sl.sub; uc < UC; uc += 16 * sl.n) {
            uint32_t vdc[16], vc[16];
            const float4* a = reinterpret_cast<const float4*>(dcrow + u0 + uc);
            const float4* b = reinterpret_cast<const float4*>(crow + u0 + uc);
#pragma unroll
            for (int v = 0; v < 4; ++v) {
                const float4 x = __ldcg(a + v), y = __ldcg(b + v);
                vdc[4 * v] = __float_as_uint(x.x); vdc[4 * v + 1] = __float_as_uint(x.y);
                vdc[4 * v + 2] = __float_as_uint(x.z); vdc[4 * v + 3] = __float_as_uint(x.w);
                vc[4 * v] = __float_as_uint(y.x); vc[4 * v + 1] = __float_as_uint(y.y);
                vc[4 * v + 2] = __float_as_uint(y.z); vc[4 * v + 3] = __float_as_uint(y.w);
            }
            __syncwarp();
            ptx::tmem_st_32x32b_x16(r.tdc + uc, vdc);
            ptx::tmem_st_32x32b_x16(r.tc_ + uc, vc);
        }
        ptx::tmem_st_wait();
    }
    __device__ static int num_tiles(const BwdPParams& p) { return 2 * (p.T - 1); }
    __device__ static int kblocks(const BwdPParams& p, int) { return p.kbh; }
    __device__ static void prefetch(const BwdPParams& p) {
        for (int i = 0; i < 2; ++i) { ptx::tma_prefetch(&p.g[i].ta); ptx::tma_prefetch(&p.g[i].tb); }
    }
    __device__ static bool sk_item(const BwdPParams& p, int cid, int, int it, tc::Item& w) {
        if (cid >= p.units || it >= 2 * (p.T - 1)) return false;
        w.tile = it; w.kb0 = 0; w.kb1 = p.kbh; w.role = 0;
        return true;
    }
    __device__ static void item_ready(const BwdPParams& p, const tc::Item& w, int cid, uint32_t rank) {
        const U u = unit(p, cid, w.tile);
#ifdef ADPSGD_DBG_NODEP
        return;
#endif
        if (u.s == 0) return;  // dz of the first BPTT step comes from the previous kernel
        const unsigned need = static_cast<unsigned>(u.s) * p.n_tiles * KQ;
        ptx::spin_until_geq(p.dep + (u.d * p.m_tiles + u.mt) * 2 + rank, need);
        asm volatile("fence.proxy.async.global;" ::: "memory");  // generic acquire -> async-proxy (TMA) reads
    }
    // per-item TMA context (tc_core.cuh HasLoadCtx): A = dz_{t_src} rows of this m-tile, B = W_hh
    // (UC = 64: MN-major [4H x H] 64-unit boxes; UC = 32: K-major W_hh^T [H x 4H])
    struct LoadCtx {
        const CUtensorMap* a;
        const CUtensorMap* b;
        int rowA, kbase, bcol;
        uint64_t keep;
    };
    __device__ static LoadCtx load_ctx(const BwdPParams& p, int it, uint32_t rank) {
        const U u = unit(p, blockIdx.x >> 1, it);
        const BwdGroup& g = p.g[u.d];
        LoadCtx c;
        c.a = &g.ta;
        c.b = &g.tb;
#ifdef ADPSGD_DBG_FIXROWS
        c.rowA = u.mt * 2 * kBM + kBM * static_cast<int>(rank);
#else
        c.rowA = t_src(p, u) * p.B + u.mt * 2 * kBM + kBM * static_cast<int>(rank);
#endif
        c.kbase = u.kh * p.kbh;
        c.bcol = u.nt * BN + static_cast<int>(rank) * (BN / 2);
        c.keep = ptx::policy_evict_last();
        return c;
    }
    __device__ static void load2c(const LoadCtx& c, int kb, uint8_t* sA, uint8_t* sB, uint32_t bar) {
        const int k0 = (c.kbase + kb) * kBK;
        ptx::tma_load_2d_2sm(sA, c.a, bar, k0, c.rowA);
        if constexpr (B_MN) {
#pragma unroll
            for (int j = 0; j < BN / 128; ++j) ptx::tma_load_2d_2sm_hint(sB + j * 64 * kBK * 2, c.b, bar, c.bcol + 64 * j, k0, c.keep);
        } else {
            ptx::tma_load_2d_2sm_hint(sB, c.b, bar, k0, c.bcol, c.keep);
        }
    }
    template <class S>
    __device__ static void epi_begin2(const BwdPParams& p, int it, uint32_t rank, int q, int lane, uint8_t* st,
                                      uint64_t* ebar, S sl) {
        const U u = unit(p, blockIdx.x >> 1, it);
#ifdef ADPSGD_DBG_NOEPI
        return;
#endif
        begin_g<UC, true, 1>(p.g[u.d], p.H, u.mt * 2 * kBM + kBM * static_cast<int>(rank), u.nt * BN + UC * u.kh, q, lane,
                             st, ebar, sl, rows(p, u));
    }
    __device__ static void epilogue_sk(const BwdPParams& p, const tc::Item& w, int cid, uint32_t rank, uint32_t tbase,
                                       int q, int lane, uint32_t tempty_leader, tc::EpiSlot sl, uint8_t* st,
                                       uint64_t* ebar, uint32_t& ephase) {
        const U u = unit(p, cid, w.tile);
        const int per = p.m_tiles * p.n_tiles;
        const int base = cid % per;  // partners: base + j * per, j = K split
        const int par = w.tile & 1;
        const int row = q * 32 + lane;
        // slot layout: [cta slot][parity][destination split j][kBlock]
        auto block = [&](int c_id, int j) {
            return p.sk_scratch + ((static_cast<int64_t>(c_id * 2 + static_cast<int>(rank)) * 2 + par) * KQ + j) * kBlock;
        };
        const bool leader = q == 0 && sl.sub == 0 && lane == 0;
#ifdef ADPSGD_DBG_NOEPI  // timing experiments only: release the accumulator, publish, no exchange / cell
        tc::release_acc_2sm(tempty_leader, lane);
        if (true) goto publish;
#endif
        {
        // 1) export the blocks the partners finalise (TMEM cols [UC j, +UC) for j != kh)
        //    (p.epi_skip: diagnosis only -- 1 skips the TMEM loads, 2 skips the stores)
#pragma unroll 1
        for (int x = sl.sub; x < NCHK * KQ; x += sl.n) {
            const int j = x / NCHK, c = x % NCHK;
            if (j == u.kh) continue;
            uint32_t v[16];
            if (p.epi_skip != 1) {
                ptx::tmem_ld_32x32b_x16_(tbase + UC * j + 16 * c, v);
                ptx::tmem_ld_wait();
            } else {
#pragma unroll
                for (int k = 0; k < 16; ++k) v[k] = 0u;
            }
            if (p.epi_skip == 2) continue;
            float4* dst = reinterpret_cast<float4*>(block(cid, j) + (c * 128 + row) * 16);
#pragma unroll
            for (int k = 0; k < 4; ++k)
                __stcg(dst + k, make_float4(__uint_as_float(v[4 * k]), __uint_as_float(v[4 * k + 1]),
                                            __uint_as_float(v[4 * k + 2]), __uint_as_float(v[4 * k + 3])));
        }
        // 2) handshake (epoch counters, one increment per item)
        if (leader && w.tile == 2) tc::trace_once(p.trace, 42);  // this warp's export done
        ptx::named_sync(2, 32 * EPI_WARPS);
        if (leader && w.tile == 2) tc::trace_once(p.trace, 40);  // export done (all warps)
        if (leader) {
            __threadfence();
            const unsigned mine_epoch = atomicAdd(p.sk_flags + cid * 2 + rank, 1u) + 1u;
            for (int j = 0; j < KQ; ++j)
                if (j != u.kh) ptx::spin_until_geq(p.sk_flags + (base + j * per) * 2 + rank, mine_epoch);
            __threadfence();
        }
        ptx::named_sync(2, 32 * EPI_WARPS);
        if (leader && w.tile == 2) tc::trace_once(p.trace, 41);  // handshake done
        // 3) cell backward on the owned 64 units (inputs pre-issued by epi_begin2), partners' partials added
        const float* pr[3] = {nullptr, nullptr, nullptr};
        for (int j = 0, n = 0; j < KQ; ++j)
            if (j != u.kh) pr[n++] = block(base + j * per, u.kh);
        auto rel = [&] { tc::release_acc_2sm(tempty_leader, lane); };
        const EpiRows rr = rows(p, u, tbase - (tbase & 0xFFFFu) % (2 * BN), true);
        if (TSTATE && u.s == 0)
            first_step_state(p, u, u.mt * 2 * kBM + kBM * static_cast<int>(rank), u.nt * BN + UC * u.kh, q, lane, sl, rr);
        body_g<UC, true, decltype(rel), 1>(p.g[u.d], p.H, u.mt * 2 * kBM + kBM * static_cast<int>(rank),
                                          u.nt * BN + UC * u.kh, tbase + UC * u.kh, q, lane, rel, st, ebar, ephase, sl,
                                          pr[0], true, rr, pr[1], pr[2]);
        }
        // 4) publish: this CTA's dz block of step tn is in memory (TMA stores complete)
#ifdef ADPSGD_DBG_NOEPI
    publish:
#endif
        if (lane == 0) {
            ptx::bulk_wait0();
            asm volatile("fence.proxy.async.global;" ::: "memory");
        }
        ptx::named_sync(2, 32 * EPI_WARPS);
        if (leader) {
            __threadfence();
            atomicAdd(p.dep + (u.d * p.m_tiles + u.mt) * 2 + rank, 1u);
            if (w.tile == 2 * (p.T - 1) - 1) {  // last item: the last CTA out re-arms every counter
                __threadfence();
                if (atomicAdd(p.exit_ctr, 1u) == gridDim.x - 1) {
                    for (int i = 0; i < 2 * p.m_tiles * 2; ++i) p.dep[i] = 0u;
                    for (int i = 0; i < static_cast<int>(gridDim.x); ++i) p.sk_flags[i] = 0u;
                    __threadfence();
                    *p.exit_ctr = 0u;
                }
            }
        }
    }
};

template <class Traits, class Params>
void launch_persistent(const Params& p, int tiles, cudaStream_t s) {
    auto k = tc::persistent_kernel<Traits, Params>;
    note_kernel<cta_single<Traits>>();
    static bool attr = false;
    if (!attr) {
        AB_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, tc::Shape<Traits::BN, Traits::EPI_SMEM>::SMEM));
        attr = true;
    }
    const int grid = tiles < num_sms() ? tiles : num_sms();
    tc::launch_tc(k, p, grid, tc::threads_of<Traits>(), tc::Shape<Traits::BN, Traits::EPI_SMEM>::SMEM, false, s);
    count_launch();
    AB_CUDA(cudaGetLastError());
}

template <class Traits, class Params>
void launch_pair(const Params& p, int pair_tiles, cudaStream_t s) {
    auto k = tc::persistent_kernel_2cta<Traits, Params>;
    note_kernel<cta_pair<Traits>>();
    static bool attr = false;
    if (!attr) {
        AB_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, tc::ShapeOf2<Traits>::SMEM));
        attr = true;
    }
    int pairs = num_sms() / 2;
    if (pair_tiles < pairs) pairs = pair_tiles;
    tc::launch_tc(k, p, 2 * pairs, tc::threads_of<Traits>(), tc::ShapeOf2<Traits>::SMEM, true, s);
    count_launch();
}

}  // namespace


void lstm_fwd_step(const LstmFwdDir* dirs, int ndirs, int B, int H, int ldg, int ldc, int ldh, cudaStream_t s) {
    AB_CHECK(H % 64 == 0 && ndirs >= 1 && ndirs <= 2, ADPSGD_E_DIMENSION, "fused LSTM step needs H % 64 == 0");
    FwdParams p;
    std::memset(&p, 0, sizeof(p));
    const bool pair = knobs().pair_mma && B > kBM;
    // one wave of 256 x 512 pair tiles when every CTA pair gets exactly one tile
    const bool wide = pair && knobs().wide_fwd && H % 128 == 0 &&
                      ndirs * ((B + 2 * kBM - 1) / (2 * kBM)) * (H / 128) <= num_sms() / 2;
    const uint32_t wbox = wide ? 128 : 64;
    double flops = 0, bytes = 0;
    for (int d = 0; d < ndirs; ++d) {
        const LstmFwdDir& a = dirs[d];
        FwdGroup& g = p.g[d];
        make_map_box(&g.ta[0], a.x, a.Kx, B, a.ldx, kBM);
        make_map_box(&g.tb[0], a.w_ih, a.Kx, 4 * H, a.ld_wih, wbox);
        g.kb0 = (a.Kx + kBK - 1) / kBK;
        g.nseg = 1;
        double K = a.Kx;
        if (a.h_prev) {
            make_map_box(&g.ta[1], a.h_prev, H, B, a.ld_hprev, kBM);
            make_map_box(&g.tb[1], a.w_hh, H, 4 * H, H, wbox);
            g.kb1 = (H + kBK - 1) / kBK;
            g.nseg = 2;
            K += H;
        }
        g.bias = a.bias; g.c_prev = a.c_prev; g.gates = a.gates; g.c = a.c; g.h = a.h;
        if (a.c_prev) make_map_gen(&g.m_cprev, a.c_prev, true, H, B, ldc, 32, 32, CU_TENSOR_MAP_SWIZZLE_128B);
        // epilogue stores: 16-unit x 32-row half boxes
        make_map_gen(&g.m_gates, a.gates, false, 4 * H, B, ldg, 16, 32, CU_TENSOR_MAP_SWIZZLE_32B);
        make_map_gen(&g.m_c, a.c, true, H, B, ldc, 16, 32, CU_TENSOR_MAP_SWIZZLE_64B);
        make_map_gen(&g.m_h, a.h, false, H, B, ldh, 16, 32, CU_TENSOR_MAP_SWIZZLE_32B);
        flops += 2.0 * B * 4.0 * H * K;
        bytes += 2.0 * (B + 4.0 * H) * K + B * H * (8.0 + 4 + 2 + (a.c_prev ? 4 : 0));
    }
    p.ngroups = ndirs; p.B = B; p.H = H; p.ldg = ldg; p.ldc = ldc; p.ldh = ldh;
    p.epi_skip = knobs().epi_skip;
    p.trace = trace_take();
    p.n_tiles = H / (wide ? 128 : 64);
    ProfScope ps_(s, PROF_GEMM_REC_FWD, flops, bytes);
    if (wide) {
        p.m_tiles = (B + 2 * kBM - 1) / (2 * kBM);
        launch_pair<FwdWideTraits>(p, ndirs * p.m_tiles * p.n_tiles, s);
    } else if (pair) {
        p.m_tiles = (B + 2 * kBM - 1) / (2 * kBM);
        launch_pair<FwdTraits>(p, ndirs * p.m_tiles * p.n_tiles, s);
    } else {
        p.m_tiles = (B + kBM - 1) / kBM;
        launch_persistent<FwdTraits>(p, ndirs * p.m_tiles * p.n_tiles, s);
    }
}

int64_t lstm_bwd_splitk_slots(int ndirs, int B, int H) {
    return static_cast<int64_t>(ndirs) * ((B + 2 * kBM - 1) / (2 * kBM)) * (H / 256 > 0 ? H / 256 : 1) * 2 * 2;
}

void lstm_bwd_step(const LstmBwdDir* dirs, int ndirs, int B, int H, int lddh, int ldg, int ldc, int lddz,
                   cudaStream_t s, float* sk_scratch, unsigned int* sk_flags) {
    AB_CHECK(H % 64 == 0 && ndirs >= 1 && ndirs <= 2, ADPSGD_E_DIMENSION, "fused BPTT step needs H % 64 == 0");
    BwdParams p;
    std::memset(&p, 0, sizeof(p));
    // 128 x 64 tiles: a 1024 x 1024 dgrad per direction is only 64 tiles at BN = 128
    const bool pair = knobs().pair_mma && B > kBM && H % 128 == 0;
    const int m_tiles = pair ? (B + 2 * kBM - 1) / (2 * kBM) : (B + kBM - 1) / kBM;
    // split-K 256 x 256 tiles when every (tile, K-half) work unit is resident at once
    const bool split = pair && knobs().splitk_bwd && sk_scratch && sk_flags && H % 256 == 0 &&
                       2 * ndirs * m_tiles * (H / 256) <= num_sms() / 2;
    const int bn = split ? 256 : pair ? 128 : ((ndirs * m_tiles * (H / 128) >= num_sms()) ? 128 : 64);
    double flops = 0, bytes = 0;
    for (int d = 0; d < ndirs; ++d) {
        const LstmBwdDir& a = dirs[d];
        BwdGroup& g = p.g[d];
        make_map_box(&g.ta, a.dz_src, 4 * H, B, a.ld_dz_src, kBM);
        make_map_box(&g.tb, a.w_hh, H, 4 * H, H, 64);
        g.kb = (4 * H + kBK - 1) / kBK;
        g.dH = a.dH; g.dc_rec = a.dc_rec; g.gates = a.gates; g.c = a.c; g.c_prev = a.c_prev; g.dz = a.dz_dst;
        make_map_gen(&g.m_dH, a.dH, true, H, B, lddh, 16, 32, CU_TENSOR_MAP_SWIZZLE_64B);
        make_map_gen(&g.m_dc, a.dc_rec, true, H, B, H, 16, 32, CU_TENSOR_MAP_SWIZZLE_64B);
        make_map_gen(&g.m_c, a.c, true, H, B, ldc, 16, 32, CU_TENSOR_MAP_SWIZZLE_64B);
        if (a.c_prev) make_map_gen(&g.m_cp, a.c_prev, true, H, B, ldc, 16, 32, CU_TENSOR_MAP_SWIZZLE_64B);
        make_map_gen(&g.m_gates, a.gates, false, 4 * H, B, ldg, 16, 32, CU_TENSOR_MAP_SWIZZLE_32B);
        make_map_gen(&g.m_dz, a.dz_dst, false, 4 * H, B, lddz, 16, 32, CU_TENSOR_MAP_SWIZZLE_32B);
        flops += 2.0 * B * H * 4.0 * H;
        bytes += 2.0 * (B + H) * 4.0 * H + B * H * (4 + 8 + 8 + 4 + (a.c_prev ? 4 : 0) + 8);
    }
    p.ngroups = ndirs; p.B = B; p.H = H; p.lddh = lddh; p.ldg = ldg; p.ldc = ldc; p.lddz = lddz;
    p.epi_skip = knobs().epi_skip;
    p.trace = trace_take();
    p.m_tiles = m_tiles;
    p.n_tiles = H / bn;
    p.sk_scratch = sk_scratch;
    p.sk_flags = sk_flags;
    ProfScope ps_(s, PROF_GEMM_REC_BWD, flops, bytes);
    if (split) launch_pair<BwdSplitTraits>(p, 2 * ndirs * p.m_tiles * p.n_tiles, s);
    else if (pair) launch_pair<BwdTraits<128>>(p, ndirs * p.m_tiles * p.n_tiles, s);
    else if (bn == 128) launch_persistent<BwdTraits<128>>(p, ndirs * p.m_tiles * p.n_tiles, s);
    else launch_persistent<BwdTraits<64>>(p, ndirs * p.m_tiles * p.n_tiles, s);
}

#ifdef ADPSGD_DBG_PROBE
#include "dbg_fwd_probe.inc"  // timing experiments only
#endif

bool lstm_fwd_layer_persistent(const LstmFwdLayer& L, int ndirs, int B, int H, int T, cudaStream_t s, unsigned int* dep,
                               unsigned int* exit_ctr) {
    // 32-unit tiles when 64-unit ones would leave more than half of the CTA pairs idle
    const int m_tiles = B / (2 * kBM);
    const int uw = (knobs().fwd_u32 && H % 32 == 0 && m_tiles * (H / 64) * 2 <= num_sms() / 2) ? 32 : 64;
    const int n_tiles = H / uw;
    const int units = m_tiles * n_tiles;
    if (!(knobs().persist_fwd && knobs().pair_mma && ndirs == 2 && B % (2 * kBM) == 0 && H % 64 == 0 &&
          units <= num_sms() / 2 && dep && exit_ctr && 4 * m_tiles <= kFwdDepSlots))
        return false;
    FwdPParams p;
    std::memset(&p, 0, sizeof(p));
    const int64_t TB = static_cast<int64_t>(T) * B;
    double flops = 0;
    for (int d = 0; d < 2; ++d) {
        FwdGroup& g = p.g[d];
        make_map_box(&g.ta[0], L.x, L.Kx, TB, L.ldx, kBM);
        // B: one 3-D box per k-block = the CTA's two gate blocks (rows 2r H + u0 .. and (2r+1) H + u0 ..)
        make_map_3d(&g.tb[0], L.w_ih[d], L.Kx, H, 4, L.ld_wih, static_cast<int64_t>(H) * L.ld_wih, uw, 2);
        make_map_box(&g.ta[1], L.h + d * H, H, TB, L.ldh, kBM);
        make_map_3d(&g.tb[1], L.w_hh[d], H, H, 4, H, static_cast<int64_t>(H) * H, uw, 2);
        make_map_gen(&g.m_cprev, L.c + d * H, true, H, TB, L.ldc, 32, 32, CU_TENSOR_MAP_SWIZZLE_128B);
        make_map_gen(&g.m_gates, L.gates + d * 4 * H, false, 4 * H, TB, L.ldg, 16, 32, CU_TENSOR_MAP_SWIZZLE_32B);
        make_map_gen(&g.m_c, L.c + d * H, true, H, TB, L.ldc, 16, 32, CU_TENSOR_MAP_SWIZZLE_64B);
        make_map_gen(&g.m_h, L.h + d * H, false, H, TB, L.ldh, 16, 32, CU_TENSOR_MAP_SWIZZLE_32B);
        g.bias = L.bias[d];
        g.kb0 = (L.Kx + kBK - 1) / kBK; g.kb1 = (H + kBK - 1) / kBK; g.nseg = 2;
        flops += 2.0 * TB * 4.0 * H * (L.Kx + H) - 2.0 * B * 4.0 * H * H;
    }
    p.B = B; p.H = H; p.T = T; p.m_tiles = m_tiles; p.n_tiles = n_tiles; p.units = units;
    p.kbx = (L.Kx + kBK - 1) / kBK; p.kbh = (H + kBK - 1) / kBK;
    p.dep = dep; p.exit_ctr = exit_ctr;
    p.trace = trace_take();
    const double bytes = 2.0 * T * (2.0 * (B + 4.0 * H) * (L.Kx + H) + static_cast<double>(B) * H * 22);
    // ADPSGD_FWD_L2WIN=1: keep the layer's recurrent-kernel weights (read every step by the m-tiles)
    // in the persisting L2 set-aside (the streaming gate / c / h stores otherwise evict them)
    cudaAccessPolicyWindow win = {};
    if (knobs().fwd_l2win && l2_persist_bytes() > 0) {
        uintptr_t lo = UINTPTR_MAX, hi = 0;
        for (int d = 0; d < 2; ++d) {
            const uintptr_t a = reinterpret_cast<uintptr_t>(L.w_ih[d]), b = reinterpret_cast<uintptr_t>(L.w_hh[d]);
            lo = std::min(lo, std::min(a, b));
            hi = std::max(hi, std::max(a + static_cast<uintptr_t>(4 * H) * L.ld_wih * 2, b + static_cast<uintptr_t>(4 * H) * H * 2));
        }
        const size_t span = hi - lo, need = static_cast<size_t>(2) * 4 * H * (L.ld_wih + H) * 2;
        if (span <= need + need / 4 && span <= l2_window_max()) {  // contiguous enough (layer 1's padded W_ih is not)
            win.base_ptr = reinterpret_cast<void*>(lo);
            win.num_bytes = span;
            win.hitRatio = std::min(1.0f, static_cast<float>(l2_persist_bytes()) / static_cast<float>(span));
            win.hitProp = cudaAccessPropertyPersisting;
            win.missProp = cudaAccessPropertyStreaming;
        }
    }
    ProfScope ps_(s, PROF_GEMM_REC_FWD, flops, bytes);
    auto launch = [&](auto tr) {
        using Tr = decltype(tr);
        auto k = tc::persistent_kernel_2cta<Tr, FwdPParams>;
        note_kernel<cta_pair<Tr>>();
        static bool attr = false;
        if (!attr) {
            AB_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, tc::ShapeOf2<Tr>::SMEM));
            attr = true;
        }
        tc::launch_tc(k, p, 2 * units, tc::threads_of<Tr>(), tc::ShapeOf2<Tr>::SMEM, true, s, 2,
                      win.num_bytes ? &win : nullptr);
    };
#ifdef ADPSGD_DBG_PROBE
    if (uw == 64 && std::getenv("ADPSGD_DBG_PROBE_STAGES")) {
        fwd_probe(p, units, s);
        cudaEvent_t e0, e1;
        AB_CUDA(cudaEventCreate(&e0));
        AB_CUDA(cudaEventCreate(&e1));
        float best = 1e30f;
        for (int rep = 0; rep < 5; ++rep) {
            AB_CUDA(cudaEventRecord(e0, s));
            launch(FwdPersistT<64>{});
            AB_CUDA(cudaEventRecord(e1, s));
            AB_CUDA(cudaEventSynchronize(e1));
            float ms;
            AB_CUDA(cudaEventElapsedTime(&ms, e0, e1));
            if (rep > 0) best = ms < best ? ms : best;
        }
        std::fprintf(stderr, "[fwd_probe] K=%d stages=%d %-16s %.1f us per launch\n", p.kbx * 64,
                     tc::ShapeOf2<FwdPersistT<64>>::STAGES, "skeleton", best * 1e3);
    }
#endif
    if (uw == 32) launch(FwdPersistT<32>{});
    else launch(FwdPersistT<64>{});
    count_launch();
    return true;
}


bool lstm_bwd_wants_whh_t(int ndirs, int B, int H) {
    if (!(knobs().persist_bwd && knobs().pair_mma && !knobs().bwd_kq4 && ndirs == 2 && B % (2 * kBM) == 0 && H % 128 == 0))
        return false;
    return knobs().bwd_kmajor || (knobs().bwd_u32 && (B / (2 * kBM)) * (H / 128) * 2 * 2 <= num_sms() / 2);
}

bool lstm_bwd_layer_persistent(const LstmBwdLayer& L, int ndirs, int B, int H, int T, cudaStream_t s, float* sk_scratch,
                               unsigned int* sk_flags, unsigned int* dep, unsigned int* exit_ctr) {
    // 256 x 256 tiles in K quarters when H allows and the units fit, else 256 x 128 in K halves
    const int kq = (knobs().bwd_kq4 && H % 256 == 0 && (B / (2 * kBM)) * (H / 256) * 4 <= num_sms() / 2) ? 4 : 2;
    // 32 units per CTA when 64-unit blocks would leave more than half of the pairs idle (needs W_hh^T)
    const int uc = (kq == 2 && knobs().bwd_u32 && L.w_hh_t[0] && L.w_hh_t[1] && H % 64 == 0 &&
                    (B / (2 * kBM)) * (H / 128) * 2 * 2 <= num_sms() / 2) ? 32 : 64;
    const bool kmaj = uc == 64 && kq == 2 && knobs().bwd_kmajor && L.w_hh_t[0] && L.w_hh_t[1];
    const int m_tiles = B / (2 * kBM), n_tiles = H / (uc * kq);
    const int units = m_tiles * n_tiles * kq;
    if (!(knobs().persist_bwd && knobs().pair_mma && ndirs == 2 && T >= 2 && B % (2 * kBM) == 0 && H % 128 == 0 &&
          units <= num_sms() / 2 && sk_scratch && sk_flags && dep && exit_ctr && 4 * m_tiles <= kBwdDepSlots))
        return false;
    BwdPParams p;
    std::memset(&p, 0, sizeof(p));
    const int G4 = 4 * H;
    for (int d = 0; d < 2; ++d) {
        BwdGroup& g = p.g[d];
        const int64_t TB = static_cast<int64_t>(T) * B;
        make_map_box(&g.ta, L.dZ + d * G4, G4, TB, L.ld_dz, kBM);
        if (uc == 32 || kmaj) make_map_box(&g.tb, L.w_hh_t[d], G4, H, G4, uc * kq / 2);  // K-major W_hh^T [H x 4H]
        else make_map_box(&g.tb, L.w_hh[d], H, G4, H, 64);
        make_map_gen(&g.m_dH, L.dH + d * H, true, H, TB, L.lddh, 16, 32, CU_TENSOR_MAP_SWIZZLE_64B);
        make_map_gen(&g.m_dc, L.dc_rec[d], true, H, B, H, 16, 32, CU_TENSOR_MAP_SWIZZLE_64B);
        make_map_gen(&g.m_c, L.c + d * H, true, H, TB, L.ldc, 16, 32, CU_TENSOR_MAP_SWIZZLE_64B);
        g.m_cp = g.m_c;
        make_map_gen(&g.m_gates, L.gates + d * G4, false, G4, TB, L.ldg, 16, 32, CU_TENSOR_MAP_SWIZZLE_32B);
        make_map_gen(&g.m_dz, L.dZ + d * G4, false, G4, TB, L.ld_dz, 16, 32, CU_TENSOR_MAP_SWIZZLE_32B);
        g.dc_rec = L.dc_rec[d];
        g.c = L.c + d * H;
        g.kb = G4 / kBK;
    }
    p.B = B; p.H = H; p.T = T; p.m_tiles = m_tiles; p.n_tiles = n_tiles; p.units = units; p.kbh = G4 / kBK / kq;
    p.ldc = L.ldc;
    p.sk_scratch = sk_scratch; p.sk_flags = sk_flags; p.dep = dep; p.exit_ctr = exit_ctr;
    p.epi_skip = knobs().export_dbg;
    p.trace = trace_take();
    const double flops = 2.0 * 2 * (T - 1) * static_cast<double>(B) * H * G4;
    const double bytes = 2.0 * (T - 1) * (2.0 * (B + H) * G4 + static_cast<double>(B) * H * (4 + 8 + 8 + 4 + 4 + 8));
    ProfScope ps_(s, PROF_GEMM_REC_BWD, flops, bytes);
    auto launch = [&](auto tr) {
        using Tr = decltype(tr);
        auto k = tc::persistent_kernel_2cta<Tr, BwdPParams>;
        note_kernel<cta_pair<Tr>>();
        static bool attr = false;
        if (!attr) {
            AB_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, tc::ShapeOf2<Tr>::SMEM));
            attr = true;
        }
        tc::launch_tc(k, p, 2 * units, tc::threads_of<Tr>(), tc::ShapeOf2<Tr>::SMEM, true, s);
    };
    if (kq == 4) launch(BwdPersistTraits<4>{});
    else if (uc == 32) launch(BwdPersistTraits<2, 32>{});
    else if (kmaj) launch(BwdPersistTraits<2, 64, true>{});
    else launch(BwdPersistTraits<2>{});
    count_launch();
    return true;
}

}  // namespace ab
