// Output layer + softmax cross-entropy fused into the tcgen05 output GEMM (bf16 mode).
//
//   logits = Y W_out^T + b_out        [M = T*B frames, N = C classes, K = P]
//   pass 1: per 256-column tile, each frame's running max / sum-exp (thread = frame row, the
//           32-column TMEM chunks stay in registers) -> part[r][tile]; the tile holding the
//           frame's label records its logit.
//   reduce: per frame, lse = combine(part), loss_r = lse - logit[label].
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
extern bool g_use_pair_mma;               // gemm_lstm.cu
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

struct CeTraits {
    static constexpr int BN = 256;
    static constexpr bool A_MN = false;
    static constexpr bool B_MN = false;
    static constexpr int EPI_WARPS = 8;
    static constexpr int EPI_SMEM = EPI_WARPS * 2 * 2048;  // per warp: 2 x (bf16 32 cols x 32 rows, SW64)
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
    // (EpiSlot); exponentials are single MUFU.EX2 on log2e-prescaled values; reductions are trees.
    __device__ static __forceinline__ float ex2(float x) {
        float y;
        asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
        return y;
    }
    __device__ static __forceinline__ void bias32(const CeParams& p, int col, bool full, float* b) {
#pragma unroll
        for (int i = 0; i < 32; i += 4) {
            if (full) {
                const float4 b4 = __ldg(reinterpret_cast<const float4*>(p.bias + col + i));
                b[i] = b4.x; b[i + 1] = b4.y; b[i + 2] = b4.z; b[i + 3] = b4.w;
            } else {
#pragma unroll
                for (int e = 0; e < 4; ++e) b[i + e] = col + i + e < p.N ? p.bias[col + i + e] : 0.f;
            }
        }
    }
    template <class Rel>
    __device__ static void body(const CeParams& p, int rowbase, int nt, uint32_t tbase, int lane, Rel release,
                                uint8_t* st, tc::EpiSlot sl) {
        const int r = rowbase + lane;
        const bool ok = r < p.M;
        const int n0 = nt * BN;
        const int lab = ok ? p.labels[r] : -1;
        constexpr float kLog2e = 1.4426950408889634f;
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
        if (p.mode == 0) {
            float m = -INFINITY, s = 0.f, zl = 0.f;
            bool has = false;
#pragma unroll 1
            for (int c = 32 * sl.sub; c < BN; c += 32 * sl.n) {
                const int col = n0 + c;
                const bool full = col + 32 <= p.N;
                float b[32];
                bias32(p, col, full, b);  // issued before the TMEM wait
                uint32_t v[32];
                ptx::tmem_ld_32x32b_x32(tbase + c, v);
                ptx::tmem_ld_wait();
                if (c + 32 * sl.n >= BN) release();
                float z[32];
#pragma unroll
                for (int i = 0; i < 32; ++i)
                    z[i] = (full || col + i < p.N) ? (__uint_as_float(v[i]) + b[i]) * kLog2e : -INFINITY;
                const int ll = lab - col;
                if (ll >= 0 && ll < 32) {
#pragma unroll
                    for (int i = 0; i < 32; ++i)
                        if (i == ll) zl = z[i];
                    has = true;
                }
                float t[16];
#pragma unroll
                for (int i = 0; i < 16; ++i) t[i] = fmaxf(z[i], z[i + 16]);
#pragma unroll
                for (int w = 8; w >= 1; w >>= 1)
#pragma unroll
                    for (int i = 0; i < w; ++i) t[i] = fmaxf(t[i], t[i + w]);
                const float mn = fmaxf(m, t[0]);
#pragma unroll
                for (int i = 0; i < 16; ++i) t[i] = ex2(z[i] - mn) + ex2(z[i + 16] - mn);
#pragma unroll
                for (int w = 8; w >= 1; w >>= 1)
#pragma unroll
                    for (int i = 0; i < w; ++i) t[i] += t[i + w];
                s = s * ex2(m - mn) + t[0];
                m = mn;
            }
            if (ok) {
                // natural-log units; one partial per (tile, epilogue sub-slot)
                p.part[(static_cast<int64_t>(r) * p.n_tiles + nt) * sl.n + sl.sub] = make_float2(m / kLog2e, s);
                if (has) p.zlab[r] = zl / kLog2e;
            }
        } else {
            const float lse2 = ok ? p.lse[r] * kLog2e : 0.f;
            const float sc = p.scale;
            int buf = 0;
#pragma unroll 1
            for (int c = 32 * sl.sub; c < BN; c += 32 * sl.n, buf ^= 1) {
                const int col = n0 + c;
                const bool full = col + 32 <= p.N;
                float b[32];
                bias32(p, col, full, b);
                uint32_t v[32];
                ptx::tmem_ld_32x32b_x32(tbase + c, v);
                ptx::tmem_ld_wait();
                if (c + 32 * sl.n >= BN) release();
                const int ll = lab - col;
                uint32_t w[16];
#pragma unroll
                for (int i = 0; i < 32; i += 2) {
                    float x0 = ex2(fmaf(__uint_as_float(v[i]) + b[i], kLog2e, -lse2)) * sc;
                    float x1 = ex2(fmaf(__uint_as_float(v[i + 1]) + b[i + 1], kLog2e, -lse2)) * sc;
                    if (i == ll) x0 -= sc;
                    if (i + 1 == ll) x1 -= sc;
                    w[i / 2] = tc::pack_bf16x2(x0, x1);
                }
                uint8_t* box = st + buf * 2048;
                if (lane == 0) ptx::bulk_wait_read1();  // the store that last used this buffer has read it
                __syncwarp();
                tc::st_row_words<64>(box, lane, w);
                ptx::fence_proxy_async_smem();
                __syncwarp();
                if (lane == 0) {
                    ptx::tma_store_2d_hint(&p.m_dl, box, col, rowbase, ptx::policy_evict_first());
                    ptx::bulk_commit();
                }
            }
        }
    }
};

template <class Traits, class Params>
void launch_any(const Params& p, int tiles, bool pair, cudaStream_t s) {
    if (pair) {
        auto k = tc::persistent_kernel_2cta<Traits, Params>;
        static bool attr = false;
        constexpr int SM = tc::Shape2<Traits::BN, Traits::EPI_SMEM>::SMEM;
        if (!attr) {
            AB_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, SM));
            attr = true;
        }
        const int pairs = tiles < num_sms() / 2 ? tiles : num_sms() / 2;
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(2 * pairs);
        cfg.blockDim = dim3(tc::threads_of<Traits>());
        cfg.dynamicSmemBytes = SM;
        cfg.stream = s;
        cudaLaunchAttribute attrs[1];
        attrs[0].id = cudaLaunchAttributeClusterDimension;
        attrs[0].val.clusterDim.x = 2;
        attrs[0].val.clusterDim.y = 1;
        attrs[0].val.clusterDim.z = 1;
        cfg.attrs = attrs;
        cfg.numAttrs = 1;
        AB_CUDA(cudaLaunchKernelEx(&cfg, k, p));
    } else {
        auto k = tc::persistent_kernel<Traits, Params>;
        static bool attr = false;
        constexpr int SM = tc::Shape<Traits::BN, Traits::EPI_SMEM>::SMEM;
        if (!attr) {
            AB_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, SM));
            attr = true;
        }
        const int grid = tiles < num_sms() ? tiles : num_sms();
        k<<<grid, tc::threads_of<Traits>(), SM, s>>>(p);
    }
    count_launch();
    AB_CUDA(cudaGetLastError());
}

// one warp per frame: lse = m* + log(sum_t s_t exp(m_t - m*)), loss = lse - z_label
__global__ void ce_reduce_kernel(const float2* __restrict__ part, int n_tiles, const float* __restrict__ zlab, int M,
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
    if (lane == 0) {
        const float l = m + __logf(s);
        lse[warp] = l;
        row_loss[warp] = l - zlab[warp];
    }
}

}  // namespace

void ce_forward_backward(const CeArgs& a, cudaStream_t s) {
    AB_CHECK(a.N % 8 == 0 && a.K % 8 == 0, ADPSGD_E_DIMENSION, "fused CE needs C, P multiples of 8");
    CeParams p;
    std::memset(&p, 0, sizeof(p));
    const bool pair = g_use_pair_mma && a.M > kBM;
    make_map_gen(&p.ta, a.Y, false, a.K, a.M, a.ldY, 64, kBM, CU_TENSOR_MAP_SWIZZLE_128B);
    make_map_gen(&p.tb, a.W, false, a.K, a.N, a.K, 64, pair ? 128 : 256, CU_TENSOR_MAP_SWIZZLE_128B);
    make_map_gen(&p.m_dl, a.dlogits, false, a.N, a.M, a.N, 32, 32, CU_TENSOR_MAP_SWIZZLE_64B);
    p.kb = (a.K + kBK - 1) / kBK;
    p.M = a.M; p.N = a.N;
    p.m_tiles = pair ? (a.M + 2 * kBM - 1) / (2 * kBM) : (a.M + kBM - 1) / kBM;
    p.n_tiles = (a.N + 255) / 256;
    p.bias = a.bias; p.labels = a.labels; p.part = a.part; p.zlab = a.zlab; p.lse = a.lse; p.scale = a.scale;
    static const int skip = std::getenv("ADPSGD_EPI_SKIP") ? std::atoi(std::getenv("ADPSGD_EPI_SKIP")) : 0;
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
        ce_reduce_kernel<<<(a.M * 32 + 255) / 256, 256, 0, s>>>(a.part, p.n_tiles * (CeTraits::EPI_WARPS / 4), a.zlab,
                                                                a.M, a.lse, a.row_loss);
        count_launch();
    }
    {
        p.mode = 1;
        p.trace = trace_take();
        ProfScope ps_(s, PROF_GEMM_OUT, gemm_flops, in_bytes + static_cast<double>(a.M) * a.N * 2);
        launch_any<CeTraits>(p, tiles, pair, s);
    }
}

int64_t ce_part_elems(int M, int N) { return static_cast<int64_t>(M) * ((N + 255) / 256) * (CeTraits::EPI_WARPS / 4); }

}  // namespace ab
