// Output layer + softmax cross-entropy fused into the tcgen05 output GEMM (bf16 mode).
//
//   logits = Y W_out^T + b_out        [M = T*B frames, N = C classes, K = P]
//   pass 1: per 256-column tile, each frame's running max / sum-exp (thread = frame row, the
//           32-column TMEM chunks stay in registers) -> part[r][tile].
//   reduce: per frame, lse = combine(part), logit[label] = Y[r] . W_out[label] + b (a warp dot
//           product), loss_r = lse - logit[label].
//   pass 2: the logits tile is recomputed and dlogits = (softmax - onehot) / (T*B) leaves as
//           bf16 through swizzled smem + TMA bulk stores.
// The 21,504 x 32,000 logits (2.75 GB fp32) never reach HBM; the recompute costs one more
// K = 256 GEMM (~0.35 TFLOP) instead of ~7 GB of logit traffic.
#include <cuda.h>

#include <cstdlib>

#include "gemm_ce.hpp"
#include "prof.hpp"
#include "tc_core.cuh"

namespace ab {

EncodeFnT get_encode_fn();                // gemm_tc.cu
unsigned long long* trace_take();         // prof.cu
void make_map_gen(CUtensorMap* m, const void* base, bool f32, uint64_t inner, uint64_t outer, int64_t ld,
                  uint32_t box_inner, uint32_t box_outer, CUtensorMapSwizzle sw);  // gemm_lstm.cu

namespace {

using tc::kBK;
using tc::kBM;

struct CeParams {
    CUtensorMap ta, tb, m_dl;
    int kb, M, N, m_tiles, n_tiles, mode;
    const float* bias;
    const int32_t* labels;
    float2* part;
    float* zlab;
    const float* lse;
    float scale;
    unsigned long long* trace;
    int epi_skip;  // debug timing experiments (ADPSGD_EPI_SKIP=2): drain TMEM only
};

struct CeTraits : tc::TraitsBase {
    static constexpr int BN = 256;
    static constexpr bool A_MN = false;
    static constexpr bool B_MN = false;
    static constexpr int EPI_WARPS = 8;
    static constexpr int EPI_SMEM = EPI_WARPS * 2 * 4096;  // per warp: 2 x (bf16 64 cols x 32 rows, SW128)
    __device__ static int num_tiles(const CeParams& p) { return p.m_tiles * p.n_tiles; }
    __device__ static void prefetch(const CeParams& p) {
        ptx::tma_prefetch(&p.ta);
        ptx::tma_prefetch(&p.tb);
    }
    __device__ static int kblocks(const CeParams& p, int) { return p.kb; }
    __device__ static void load(const CeParams& p, int tile, int kb, uint8_t* sA, uint8_t* sB, uint64_t* bar) {
        const int m0 = (tile % p.m_tiles) * kBM, n0 = (tile / p.m_tiles) * BN;
        ptx::tma_load_2d(sA, &p.ta, bar, kb * kBK, m0);
        ptx::tma_load_2d_hint(sB, &p.tb, bar, kb * kBK, n0, ptx::policy_evict_last());
    }
    __device__ static void load2(const CeParams& p, int tile, int kb, uint32_t rank, uint8_t* sA, uint8_t* sB,
                                 uint32_t bar) {
        const int m0 = (tile % p.m_tiles) * 2 * kBM + kBM * rank;
        const int n0 = (tile / p.m_tiles) * BN + (BN / 2) * rank;
        ptx::tma_load_2d_2sm(sA, &p.ta, bar, kb * kBK, m0);
        ptx::tma_load_2d_2sm_hint(sB, &p.tb, bar, kb * kBK, n0, ptx::policy_evict_last());
    }
    // per-item TMA context (tc_core.cuh HasLoadCtx)
    struct LoadCtx {
        const CUtensorMap* a;
        const CUtensorMap* b;
        int m0, n0;
        uint64_t keep;
    };
    __device__ static LoadCtx load_ctx(const CeParams& p, int tile, uint32_t rank) {
        LoadCtx c;
        c.a = &p.ta;
        c.b = &p.tb;
        c.m0 = (tile % p.m_tiles) * 2 * kBM + kBM * static_cast<int>(rank);
        c.n0 = (tile / p.m_tiles) * BN + (BN / 2) * static_cast<int>(rank);
        c.keep = ptx::policy_evict_last();
        return c;
    }
    __device__ static void load2c(const LoadCtx& c, int kb, uint8_t* sA, uint8_t* sB, uint32_t bar) {
        ptx::tma_load_2d_2sm(sA, c.a, bar, kb * kBK, c.m0);
        ptx::tma_load_2d_2sm_hint(sB, c.b, bar, kb * kBK, c.n0, c.keep);
    }
    __device__ static void epilogue(const CeParams& p, int tile, uint32_t tbase, int q, int lane, uint64_t* tempty,
                                    uint8_t* st, uint64_t*, uint32_t&, tc::EpiSlot sl) {
        const int m0 = (tile % p.m_tiles) * kBM, nt = tile / p.m_tiles;
        body(p, m0 + q * 32, nt, tbase, lane, [&] { tc::release_acc(tempty, lane); }, st, sl);
    }
    __device__ static void epilogue2(const CeParams& p, int tile, uint32_t rank, uint32_t tbase, int q, int lane,
                                     uint32_t tempty_leader, uint8_t* st, uint64_t*, uint32_t&, tc::EpiSlot sl) {
        const int m0 = (tile % p.m_tiles) * 2 * kBM + kBM * rank, nt = tile / p.m_tiles;
        body(p, m0 + q * 32, nt, tbase, lane, [&] { tc::release_acc_2sm(tempty_leader, lane); }, st, sl);
    }
    // thread = frame row; two warps per TMEM lane quarter take alternate 32-column chunks
    // (EpiSlot), two chunks per TMEM wait. Per element: pass 1 = FADD2 (bias) + FMNMX3 (max) +
    // FFMA2 (scale, shift) + MUFU.EX2 + FADD2 (sum); pass 2 = FADD2 + FFMA2 + MUFU.EX2 + pack.
    // No per-element branches: the label's logit comes from ce_reduce (a dot product), and
    // pass 2 patches the one label element of a row in the staged smem box.
    __device__ static __forceinline__ float ex2(float x) {
        float y;
        asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
        return y;
    }
    __device__ static __forceinline__ float max3(float a, float b, float c) {
        float d;
        asm("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
        return d;
    }
    __device__ static __forceinline__ void add2(float& a0, float& a1, float b0, float b1) {
        uint64_t d;
        asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(pk(a0, a1)), "l"(pk(b0, b1)));
        a0 = __uint_as_float(static_cast<uint32_t>(d)); a1 = __uint_as_float(static_cast<uint32_t>(d >> 32));
    }
    __device__ static __forceinline__ void fma2(float& a0, float& a1, float m, float c) {
        uint64_t d;
        asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(pk(a0, a1)), "l"(pk(m, m)), "l"(pk(c, c)));
        a0 = __uint_as_float(static_cast<uint32_t>(d)); a1 = __uint_as_float(static_cast<uint32_t>(d >> 32));
    }
    __device__ static __forceinline__ uint64_t pk(float a, float b) {
        return static_cast<uint64_t>(__float_as_uint(a)) | (static_cast<uint64_t>(__float_as_uint(b)) << 32);
    }
    // z[i] = acc[i] + bias[col + i]; columns >= N -> -inf (non-full tiles only)
    template <bool FULL>
    __device__ static __forceinline__ void logits32(const CeParams& p, int col, const uint32_t* v, float* z) {
#pragma unroll
        for (int i = 0; i < 32; i += 4) {
            float b0, b1, b2, b3;
            if (FULL) {
                const float4 b4 = __ldg(reinterpret_cast<const float4*>(p.bias + col + i));
                b0 = b4.x; b1 = b4.y; b2 = b4.z; b3 = b4.w;
            } else {
                b0 = __ldg(p.bias + min(col + i, p.N - 1)); b1 = __ldg(p.bias + min(col + i + 1, p.N - 1));
                b2 = __ldg(p.bias + min(col + i + 2, p.N - 1)); b3 = __ldg(p.bias + min(col + i + 3, p.N - 1));
            }
            z[i] = __uint_as_float(v[i]); z[i + 1] = __uint_as_float(v[i + 1]);
            z[i + 2] = __uint_as_float(v[i + 2]); z[i + 3] = __uint_as_float(v[i + 3]);
            add2(z[i], z[i + 1], b0, b1);
            add2(z[i + 2], z[i + 3], b2, b3);
        }
        if (!FULL) {
#pragma unroll
            for (int i = 0; i < 32; ++i) z[i] = col + i < p.N ? z[i] : -INFINITY;
        }
    }
    // online (max, sum-exp) over one 32-column chunk, natural-log units
    __device__ static __forceinline__ void online32(float* z, float& m, float& s) {
        constexpr float kLog2e = 1.4426950408889634f;
        float t[11];
#pragma unroll
        for (int i = 0; i < 10; ++i) t[i] = max3(z[3 * i], z[3 * i + 1], z[3 * i + 2]);
        t[10] = fmaxf(z[30], z[31]);
        const float c0 = max3(t[0], t[1], t[2]), c1 = max3(t[3], t[4], t[5]), c2 = max3(t[6], t[7], t[8]);
        const float mn = max3(max3(c0, c1, c2), t[9], fmaxf(t[10], m));
        // all columns so far past N: keep m = -inf, subtract 0 instead of -inf
        const float mr = mn == -INFINITY ? 0.f : mn;
        const float sh = -mr * kLog2e;
#pragma unroll
        for (int i = 0; i < 32; i += 2) {
            fma2(z[i], z[i + 1], kLog2e, sh);
            z[i] = ex2(z[i]); z[i + 1] = ex2(z[i + 1]);
        }
#pragma unroll
        for (int w = 16; w >= 2; w >>= 1)
#pragma unroll
            for (int i = 0; i < w; i += 2) add2(z[i], z[i + 1], z[i + w], z[i + w + 1]);
        s = s * ex2((m - mr) * kLog2e) + (z[0] + z[1]);
        m = mn;
    }
    template <bool FULL, class Rel>
    __device__ static void body_t(const CeParams& p, int rowbase, int nt, uint32_t tbase, int lane, Rel release,
                                  uint8_t* st, tc::EpiSlot sl) {
        constexpr int PER = BN / 32;  // chunks per tile
        const int r = rowbase + lane;
        const bool ok = r < p.M;
        const int n0 = nt * BN;
        constexpr float kLog2e = 1.4426950408889634f;
        if (p.mode == 0) {
            float m = -INFINITY, s = 0.f;
#pragma unroll 1
            for (int jp = sl.sub; jp < PER / 2; jp += sl.n) {  // adjacent chunk pairs: 64 columns
                const int ca = 64 * jp, cb = ca + 32;
                uint32_t va[32], vb[32];
                ptx::tmem_ld_32x32b_x32(tbase + ca, va);
                ptx::tmem_ld_32x32b_x32(tbase + cb, vb);
                ptx::tmem_ld_wait();
                if (jp + sl.n >= PER / 2) release();
                float za[32], zb[32];
                logits32<FULL>(p, n0 + ca, va, za);
                logits32<FULL>(p, n0 + cb, vb, zb);
                online32(za, m, s);
                online32(zb, m, s);
            }
            // one partial per (tile, epilogue sub-slot)
            if (ok) p.part[(static_cast<int64_t>(r) * p.n_tiles + nt) * sl.n + sl.sub] = make_float2(m, s);
        } else {
            const float lse = ok ? p.lse[r] : 0.f;
            const float sc = p.scale;
            const float q = __log2f(sc) - lse * kLog2e;  // dlogit = exp(z - lse) * sc = ex2(z log2e + q)
            const int lab = ok ? p.labels[r] : -1;
            const float dlab = ok ? ex2(fmaf(p.zlab[r], kLog2e, q)) - sc : 0.f;
            int buf = 0;
#pragma unroll 1
            for (int jp = sl.sub; jp < PER / 2; jp += sl.n, buf ^= 1) {  // 64 adjacent columns per iteration
                const int col = n0 + 64 * jp;
                uint32_t v[2][32];
                ptx::tmem_ld_32x32b_x32(tbase + 64 * jp, v[0]);
                ptx::tmem_ld_32x32b_x32(tbase + 64 * jp + 32, v[1]);
                ptx::tmem_ld_wait();
                if (jp + sl.n >= PER / 2) release();
                uint32_t w[32];
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    float z[32];
                    logits32<FULL>(p, col + 32 * h, v[h], z);
#pragma unroll
                    for (int i = 0; i < 32; i += 2) {
                        fma2(z[i], z[i + 1], kLog2e, q);
                        w[16 * h + i / 2] = tc::pack_bf16x2(ex2(z[i]), ex2(z[i + 1]));
                    }
                }
                // one 32-row x 64-column bf16 box (SW128) per iteration: one fence and one TMA store
                uint8_t* box = st + buf * 4096;
                if (lane == 0) ptx::bulk_wait_read1();  // the store that last used this buffer has read it
                __syncwarp();
                tc::st_row_words<128>(box, lane, w);
                const int ll = lab - col;
                if (ll >= 0 && ll < 64) {  // softmax - onehot at the label column
                    const uint32_t a = ptx::smem_u32(box) + lane * 128 + (((ll >> 3) ^ (lane & 7)) << 4) + (ll & 7) * 2;
                    const __nv_bfloat16 hv = __float2bfloat16_rn(dlab);
                    asm volatile("st.shared.b16 [%0], %1;" ::"r"(a), "h"(*reinterpret_cast<const unsigned short*>(&hv)) : "memory");
                }
                ptx::fence_proxy_async_smem();
                __syncwarp();
                if (lane == 0) {
                    ptx::tma_store_2d_hint(&p.m_dl, box, col, rowbase, ptx::policy_evict_first());
                    ptx::bulk_commit();
                }
            }
        }
    }
    template <class Rel>
    __device__ static void body(const CeParams& p, int rowbase, int nt, uint32_t tbase, int lane, Rel release,
                                uint8_t* st, tc::EpiSlot sl) {
        if (p.epi_skip == 1) {
#pragma unroll 1
            for (int c = 32 * sl.sub; c < BN; c += 32 * sl.n) {
                uint32_t v[32];
                ptx::tmem_ld_32x32b_x32(tbase + c, v);
                ptx::tmem_ld_wait();
                if (c + 32 * sl.n >= BN) release();
            }
            return;
        }
        if ((nt + 1) * BN <= p.N) body_t<true>(p, rowbase, nt, tbase, lane, release, st, sl);
        else body_t<false>(p, rowbase, nt, tbase, lane, release, st, sl);
    }
};

template <class Traits, class Params>
void launch_any(const Params& p, int tiles, bool pair, cudaStream_t s) {
    if (pair) {
        auto k = tc::persistent_kernel_2cta<Traits, Params>;
        note_kernel<cta_pair<Traits>>();
        static bool attr = false;
        constexpr int SM = tc::ShapeOf2<Traits>::SMEM;
        if (!attr) {
            AB_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, SM));
            attr = true;
        }
        const int pairs = tiles < num_sms() / 2 ? tiles : num_sms() / 2;
        tc::launch_tc(k, p, 2 * pairs, tc::threads_of<Traits>(), SM, true, s);
    } else {
        auto k = tc::persistent_kernel<Traits, Params>;
        note_kernel<cta_single<Traits>>();
        static bool attr = false;
        constexpr int SM = tc::Shape<Traits::BN, Traits::EPI_SMEM>::SMEM;
        if (!attr) {
            AB_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, SM));
            attr = true;
        }
        const int grid = tiles < num_sms() ? tiles : num_sms();
        tc::launch_tc(k, p, grid, tc::threads_of<Traits>(), SM, false, s);
    }
    count_launch();
    AB_CUDA(cudaGetLastError());
}

// one warp per frame: lse = m* + log(sum_t s_t exp(m_t - m*)); the label's logit
// z_label = Y[r] . W_out[label] + b[label] (bf16 operands, fp32 accumulate, like the GEMM);
// loss = lse - z_label.
__global__ void ce_reduce_kernel(const float2* __restrict__ part, int n_tiles, const bf16* __restrict__ Y, int ldY,
                                 const bf16* __restrict__ W, int K, const float* __restrict__ bias,
                                 const int32_t* __restrict__ labels, int M, float* __restrict__ zlab,
                                 float* __restrict__ lse, float* __restrict__ row_loss) {
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (warp >= M) return;
    const float2* pr = part + static_cast<int64_t>(warp) * n_tiles;
    float m = -INFINITY;
    for (int t = lane; t < n_tiles; t += 32) m = fmaxf(m, pr[t].x);
    for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    float s = 0.f;
    for (int t = lane; t < n_tiles; t += 32) s += pr[t].y * __expf(pr[t].x - m);
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    const int lab = labels[warp];
    const bf16* y = Y + static_cast<int64_t>(warp) * ldY;
    const bf16* w = W + static_cast<int64_t>(lab) * K;
    float d = 0.f;
    for (int k = 2 * lane; k < K; k += 64) {
        const float2 a = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(y + k));
        const float2 b = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(w + k));
        d = fmaf(a.x, b.x, fmaf(a.y, b.y, d));
    }
    for (int o = 16; o; o >>= 1) d += __shfl_xor_sync(0xffffffffu, d, o);
    if (lane == 0) {
        const float l = m + __logf(s);
        const float z = d + bias[lab];
        lse[warp] = l;
        zlab[warp] = z;
        row_loss[warp] = l - z;
    }
}

}  // namespace

void ce_forward_backward(const CeArgs& a, cudaStream_t s) {
    AB_CHECK(a.N % 8 == 0 && a.K % 8 == 0, ADPSGD_E_DIMENSION, "fused CE needs C, P multiples of 8");
    CeParams p;
    std::memset(&p, 0, sizeof(p));
    const bool pair = knobs().pair_mma && a.M > kBM;
    make_map_gen(&p.ta, a.Y, false, a.K, a.M, a.ldY, 64, kBM, CU_TENSOR_MAP_SWIZZLE_128B);
    make_map_gen(&p.tb, a.W, false, a.K, a.N, a.K, 64, pair ? 128 : 256, CU_TENSOR_MAP_SWIZZLE_128B);
    make_map_gen(&p.m_dl, a.dlogits, false, a.N, a.M, a.N, 64, 32, CU_TENSOR_MAP_SWIZZLE_128B);
    p.kb = (a.K + kBK - 1) / kBK;
    p.M = a.M; p.N = a.N;
    p.m_tiles = pair ? (a.M + 2 * kBM - 1) / (2 * kBM) : (a.M + kBM - 1) / kBM;
    p.n_tiles = (a.N + 255) / 256;
    p.bias = a.bias; p.labels = a.labels; p.part = a.part; p.zlab = a.zlab; p.lse = a.lse; p.scale = a.scale;
    const int skip = knobs().epi_skip;
    p.epi_skip = skip == 2 ? 1 : (skip >= 3 ? skip : 0);
    const int tiles = p.m_tiles * p.n_tiles;
    const double gemm_flops = 2.0 * a.M * a.N * a.K;
    const double in_bytes = 2.0 * (static_cast<double>(a.M) + a.N) * a.K;
    {
        p.mode = 0;
        p.trace = trace_take();
        ProfScope ps_(s, PROF_GEMM_OUT, gemm_flops, in_bytes + static_cast<double>(a.M) * p.n_tiles * 8);
        launch_any<CeTraits>(p, tiles, pair, s);
    }
    {
        ProfScope ps_(s, PROF_CE, 0, static_cast<double>(a.M) * (p.n_tiles * 8 + 12));
        ce_reduce_kernel<<<(a.M * 32 + 255) / 256, 256, 0, s>>>(a.part, p.n_tiles * (CeTraits::EPI_WARPS / 4), a.Y,
                                                                a.ldY, a.W, a.K, a.bias, a.labels, a.M, a.zlab,
                                                                a.lse, a.row_loss);
        count_launch();
    }
    {
        p.mode = 1;
        p.trace = trace_take();
        // pass 2 recomputes the logits tile to write dlogits: time counted, FLOPs not (the
        // algorithmic output-layer work is the pass-1 GEMM plus dY / dW_out)
        ProfScope ps_(s, PROF_GEMM_OUT, 0.0, in_bytes + static_cast<double>(a.M) * a.N * 2);
        launch_any<CeTraits>(p, tiles, pair, s);
    }
}

int64_t ce_part_elems(int M, int N) { return static_cast<int64_t>(M) * ((N + 255) / 256) * (CeTraits::EPI_WARPS / 4); }

}  // namespace ab
