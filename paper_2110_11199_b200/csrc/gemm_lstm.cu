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

#include "gemm_lstm.hpp"
#include "prof.hpp"
#include "tc_core.cuh"

namespace ab {

EncodeFnT get_encode_fn();  // gemm_tc.cu

namespace {

using tc::kBK;
using tc::kBM;

__device__ __forceinline__ float sigf(float x) { return 1.f / (1.f + __expf(-x)); }
__device__ __forceinline__ float tanhf_fast(float x) {
    // tanh via exp; accurate to ~1e-6 relative in fp32 for the ranges of an LSTM cell
    const float e = __expf(-2.f * fabsf(x));
    const float t = (1.f - e) / (1.f + e);
    return copysignf(t, x);
}

// ---------------- forward ----------------
struct FwdGroup {
    CUtensorMap ta[2];
    CUtensorMap tb[2];
    int kb0, kb1, nseg;
    const float* bias;
    const float* c_prev;
    float* gates;
    float* c;
    bf16* h;
};
struct FwdParams {
    FwdGroup g[2];
    int ngroups, m_tiles, n_tiles, B, H, ldg, ldc, ldh;
};

struct FwdTraits {
    static constexpr int BN = 256;
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
        u0 = (r / p.m_tiles) * 64;
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
        ptx::tma_load_2d(sA, &g.ta[s], bar, k0, m0);
#pragma unroll
        for (int gate = 0; gate < 4; ++gate)
            ptx::tma_load_2d(sB + gate * 64 * kBK * 2, &g.tb[s], bar, k0, gate * p.H + u0);
    }
    __device__ static void epilogue(const FwdParams& p, int tile, uint32_t tbase, int q, int lane, uint64_t* tempty) {
        int grp, m0, u0;
        coords(p, tile, grp, m0, u0);
        const FwdGroup& g = p.g[grp];
        const int r = m0 + q * 32 + lane;
        const bool ok = r < p.B;
        const int H = p.H;
#pragma unroll 1
        for (int uc = 0; uc < 64; uc += 32) {
            uint32_t zi[32], zf[32], zg[32], zo[32];
            ptx::tmem_ld_32x32b_x32(tbase + 0 * 64 + uc, zi);
            ptx::tmem_ld_32x32b_x32(tbase + 1 * 64 + uc, zf);
            ptx::tmem_ld_32x32b_x32(tbase + 2 * 64 + uc, zg);
            ptx::tmem_ld_32x32b_x32(tbase + 3 * 64 + uc, zo);
            ptx::tmem_ld_wait();
            if (uc == 32) tc::release_acc(tempty, lane);
            if (!ok) continue;
            const int j0 = u0 + uc;
            const float* bi = g.bias + j0;
            float* grow = g.gates + static_cast<int64_t>(r) * p.ldg + j0;
            float* crow = g.c + static_cast<int64_t>(r) * p.ldc + j0;
            const float* cprow = g.c_prev ? g.c_prev + static_cast<int64_t>(r) * p.ldc + j0 : nullptr;
            bf16* hrow = g.h + static_cast<int64_t>(r) * p.ldh + j0;
#pragma unroll
            for (int i0 = 0; i0 < 32; i0 += 4) {
                const float4 bI = __ldg(reinterpret_cast<const float4*>(bi + i0));
                const float4 bF = __ldg(reinterpret_cast<const float4*>(bi + H + i0));
                const float4 bG = __ldg(reinterpret_cast<const float4*>(bi + 2 * H + i0));
                const float4 bO = __ldg(reinterpret_cast<const float4*>(bi + 3 * H + i0));
                const float4 cp4 = cprow ? *reinterpret_cast<const float4*>(cprow + i0) : make_float4(0.f, 0.f, 0.f, 0.f);
                const float bIa[4] = {bI.x, bI.y, bI.z, bI.w}, bFa[4] = {bF.x, bF.y, bF.z, bF.w};
                const float bGa[4] = {bG.x, bG.y, bG.z, bG.w}, bOa[4] = {bO.x, bO.y, bO.z, bO.w};
                const float cpa[4] = {cp4.x, cp4.y, cp4.z, cp4.w};
                float ig[4], fg[4], gg[4], og[4], cn[4], hn[4];
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const int i = i0 + e;
                    ig[e] = sigf(__uint_as_float(zi[i]) + bIa[e]);
                    fg[e] = sigf(__uint_as_float(zf[i]) + bFa[e]);
                    gg[e] = tanhf_fast(__uint_as_float(zg[i]) + bGa[e]);
                    og[e] = sigf(__uint_as_float(zo[i]) + bOa[e]);
                    cn[e] = fg[e] * cpa[e] + ig[e] * gg[e];
                    hn[e] = og[e] * tanhf_fast(cn[e]);
                }
                *reinterpret_cast<float4*>(grow + i0) = make_float4(ig[0], ig[1], ig[2], ig[3]);
                *reinterpret_cast<float4*>(grow + H + i0) = make_float4(fg[0], fg[1], fg[2], fg[3]);
                *reinterpret_cast<float4*>(grow + 2 * H + i0) = make_float4(gg[0], gg[1], gg[2], gg[3]);
                *reinterpret_cast<float4*>(grow + 3 * H + i0) = make_float4(og[0], og[1], og[2], og[3]);
                *reinterpret_cast<float4*>(crow + i0) = make_float4(cn[0], cn[1], cn[2], cn[3]);
                __nv_bfloat162 h01 = __floats2bfloat162_rn(hn[0], hn[1]), h23 = __floats2bfloat162_rn(hn[2], hn[3]);
                uint2 hv;
                hv.x = *reinterpret_cast<uint32_t*>(&h01);
                hv.y = *reinterpret_cast<uint32_t*>(&h23);
                *reinterpret_cast<uint2*>(hrow + i0) = hv;
            }
        }
    }
};

// ---------------- backward ----------------
struct BwdGroup {
    CUtensorMap ta;
    CUtensorMap tb;
    int kb;
    const float* dH;
    float* dc_rec;
    const float* gates;
    const float* c;
    const float* c_prev;
    bf16* dz;
};
struct BwdParams {
    BwdGroup g[2];
    int ngroups, m_tiles, n_tiles, B, H, lddh, ldg, ldc, lddz;
};

template <int BN_>
struct BwdTraits {
    static constexpr int BN = BN_;
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
        ptx::tma_load_2d(sA, &g.ta, bar, k0, m0);
#pragma unroll
        for (int j = 0; j < BN / 64; ++j) ptx::tma_load_2d(sB + j * 64 * kBK * 2, &g.tb, bar, u0 + 64 * j, k0);
    }
    __device__ static void epilogue(const BwdParams& p, int tile, uint32_t tbase, int q, int lane, uint64_t* tempty) {
        int grp, m0, u0;
        coords(p, tile, grp, m0, u0);
        const BwdGroup& g = p.g[grp];
        const int r = m0 + q * 32 + lane;
        const bool ok = r < p.B;
        const int H = p.H;
#pragma unroll 1
        for (int uc = 0; uc < BN; uc += 32) {
            uint32_t acc[32];
            ptx::tmem_ld_32x32b_x32(tbase + uc, acc);
            ptx::tmem_ld_wait();
            if (uc + 32 >= BN) tc::release_acc(tempty, lane);
            if (!ok) continue;
            const int j0 = u0 + uc;
            const float* dHr = g.dH + static_cast<int64_t>(r) * p.lddh + j0;
            float* dcr = g.dc_rec + static_cast<int64_t>(r) * H + j0;
            const float* gr = g.gates + static_cast<int64_t>(r) * p.ldg + j0;
            const float* cr = g.c + static_cast<int64_t>(r) * p.ldc + j0;
            const float* cpr = g.c_prev ? g.c_prev + static_cast<int64_t>(r) * p.ldc + j0 : nullptr;
            bf16* dzr = g.dz + static_cast<int64_t>(r) * p.lddz + j0;
#pragma unroll
            for (int i0 = 0; i0 < 32; i0 += 4) {
                const float4 dh4 = *reinterpret_cast<const float4*>(dHr + i0);
                const float4 dc4 = *reinterpret_cast<const float4*>(dcr + i0);
                const float4 i4 = *reinterpret_cast<const float4*>(gr + i0);
                const float4 f4 = *reinterpret_cast<const float4*>(gr + H + i0);
                const float4 g4 = *reinterpret_cast<const float4*>(gr + 2 * H + i0);
                const float4 o4 = *reinterpret_cast<const float4*>(gr + 3 * H + i0);
                const float4 c4 = *reinterpret_cast<const float4*>(cr + i0);
                const float4 cp4 = cpr ? *reinterpret_cast<const float4*>(cpr + i0) : make_float4(0.f, 0.f, 0.f, 0.f);
                const float dha[4] = {dh4.x, dh4.y, dh4.z, dh4.w}, dca[4] = {dc4.x, dc4.y, dc4.z, dc4.w};
                const float ia[4] = {i4.x, i4.y, i4.z, i4.w}, fa[4] = {f4.x, f4.y, f4.z, f4.w};
                const float ga[4] = {g4.x, g4.y, g4.z, g4.w}, oa[4] = {o4.x, o4.y, o4.z, o4.w};
                const float ca[4] = {c4.x, c4.y, c4.z, c4.w}, cpa[4] = {cp4.x, cp4.y, cp4.z, cp4.w};
                float zi[4], zf[4], zg[4], zo[4], dco[4];
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const float dh = dha[e] + __uint_as_float(acc[i0 + e]);
                    const float tc = tanhf_fast(ca[e]);
                    const float dc = dca[e] + dh * oa[e] * (1.f - tc * tc);
                    zi[e] = dc * ga[e] * ia[e] * (1.f - ia[e]);
                    zf[e] = dc * cpa[e] * fa[e] * (1.f - fa[e]);
                    zg[e] = dc * ia[e] * (1.f - ga[e] * ga[e]);
                    zo[e] = dh * tc * oa[e] * (1.f - oa[e]);
                    dco[e] = dc * fa[e];
                }
                *reinterpret_cast<float4*>(dcr + i0) = make_float4(dco[0], dco[1], dco[2], dco[3]);
                auto st4 = [](bf16* dst, const float* v) {
                    __nv_bfloat162 a = __floats2bfloat162_rn(v[0], v[1]), b = __floats2bfloat162_rn(v[2], v[3]);
                    uint2 u;
                    u.x = *reinterpret_cast<uint32_t*>(&a);
                    u.y = *reinterpret_cast<uint32_t*>(&b);
                    *reinterpret_cast<uint2*>(dst) = u;
                };
                st4(dzr + i0, zi);
                st4(dzr + H + i0, zf);
                st4(dzr + 2 * H + i0, zg);
                st4(dzr + 3 * H + i0, zo);
            }
        }
    }
};

void make_map_box(CUtensorMap* m, const void* base, uint64_t inner, uint64_t outer, int64_t ld, uint32_t box_outer) {
    AB_CHECK((reinterpret_cast<uintptr_t>(base) & 15) == 0, ADPSGD_E_DIMENSION, "TMA base must be 16B aligned");
    AB_CHECK(((ld * 2) & 15) == 0, ADPSGD_E_DIMENSION, "TMA row pitch must be a multiple of 16 bytes");
    cuuint64_t dims[2] = {inner, outer};
    cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld) * 2};
    cuuint32_t box[2] = {64, box_outer};
    cuuint32_t es[2] = {1, 1};
    CUresult r = get_encode_fn()(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box,
                                 es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                 CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    AB_CHECK(r == CUDA_SUCCESS, ADPSGD_E_CUDA, "cuTensorMapEncodeTiled failed: " + std::to_string(r));
}

template <class Traits, class Params>
void launch_persistent(const Params& p, int tiles, cudaStream_t s) {
    auto k = tc::persistent_kernel<Traits, Params>;
    static bool attr = false;
    if (!attr) {
        AB_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, tc::Shape<Traits::BN>::SMEM));
        attr = true;
    }
    const int grid = tiles < num_sms() ? tiles : num_sms();
    k<<<grid, tc::kThreads, tc::Shape<Traits::BN>::SMEM, s>>>(p);
    count_launch();
    AB_CUDA(cudaGetLastError());
}

}  // namespace

void lstm_fwd_step(const LstmFwdDir* dirs, int ndirs, int B, int H, int ldg, int ldc, int ldh, cudaStream_t s) {
    AB_CHECK(H % 64 == 0 && ndirs >= 1 && ndirs <= 2, ADPSGD_E_DIMENSION, "fused LSTM step needs H % 64 == 0");
    FwdParams p;
    std::memset(&p, 0, sizeof(p));
    double flops = 0, bytes = 0;
    for (int d = 0; d < ndirs; ++d) {
        const LstmFwdDir& a = dirs[d];
        FwdGroup& g = p.g[d];
        make_map_box(&g.ta[0], a.x, a.Kx, B, a.ldx, kBM);
        make_map_box(&g.tb[0], a.w_ih, a.Kx, 4 * H, a.ld_wih, 64);
        g.kb0 = (a.Kx + kBK - 1) / kBK;
        g.nseg = 1;
        double K = a.Kx;
        if (a.h_prev) {
            make_map_box(&g.ta[1], a.h_prev, H, B, a.ld_hprev, kBM);
            make_map_box(&g.tb[1], a.w_hh, H, 4 * H, H, 64);
            g.kb1 = (H + kBK - 1) / kBK;
            g.nseg = 2;
            K += H;
        }
        g.bias = a.bias; g.c_prev = a.c_prev; g.gates = a.gates; g.c = a.c; g.h = a.h;
        flops += 2.0 * B * 4.0 * H * K;
        bytes += 2.0 * (B + 4.0 * H) * K + B * H * (16.0 + 4 + 2 + (a.c_prev ? 4 : 0));
    }
    p.ngroups = ndirs; p.B = B; p.H = H; p.ldg = ldg; p.ldc = ldc; p.ldh = ldh;
    p.m_tiles = (B + kBM - 1) / kBM;
    p.n_tiles = H / 64;
    ProfScope ps_(s, PROF_GEMM_REC_FWD, flops, bytes);
    launch_persistent<FwdTraits>(p, ndirs * p.m_tiles * p.n_tiles, s);
}

void lstm_bwd_step(const LstmBwdDir* dirs, int ndirs, int B, int H, int lddh, int ldg, int ldc, int lddz,
                   cudaStream_t s) {
    AB_CHECK(H % 64 == 0 && ndirs >= 1 && ndirs <= 2, ADPSGD_E_DIMENSION, "fused BPTT step needs H % 64 == 0");
    BwdParams p;
    std::memset(&p, 0, sizeof(p));
    // 128 x 64 tiles: a 1024 x 1024 dgrad per direction is only 64 tiles at BN = 128
    const int m_tiles = (B + kBM - 1) / kBM;
    const int bn = (ndirs * m_tiles * (H / 128) >= num_sms()) ? 128 : 64;
    double flops = 0, bytes = 0;
    for (int d = 0; d < ndirs; ++d) {
        const LstmBwdDir& a = dirs[d];
        BwdGroup& g = p.g[d];
        make_map_box(&g.ta, a.dz_src, 4 * H, B, a.ld_dz_src, kBM);
        make_map_box(&g.tb, a.w_hh, H, 4 * H, H, 64);
        g.kb = (4 * H + kBK - 1) / kBK;
        g.dH = a.dH; g.dc_rec = a.dc_rec; g.gates = a.gates; g.c = a.c; g.c_prev = a.c_prev; g.dz = a.dz_dst;
        flops += 2.0 * B * H * 4.0 * H;
        bytes += 2.0 * (B + H) * 4.0 * H + B * H * (4 + 8 + 16 + 4 + (a.c_prev ? 4 : 0) + 8);
    }
    p.ngroups = ndirs; p.B = B; p.H = H; p.lddh = lddh; p.ldg = ldg; p.ldc = ldc; p.lddz = lddz;
    p.m_tiles = m_tiles;
    p.n_tiles = H / bn;
    ProfScope ps_(s, PROF_GEMM_REC_BWD, flops, bytes);
    if (bn == 128) launch_persistent<BwdTraits<128>>(p, ndirs * p.m_tiles * p.n_tiles, s);
    else launch_persistent<BwdTraits<64>>(p, ndirs * p.m_tiles * p.n_tiles, s);
}

}  // namespace ab
