// fp32 SIMT GEMM — the "exact" parity-mode contraction (ADPSGD_PREC_FP32).
// Tiled 64x64x16, 256 threads, 4x4 register micro-tile, any operand majorness.
// Not the performance path: the bf16 tcgen05 kernel (gemm_tc.cu) is.
#include "gemm.hpp"
#include "prof.hpp"

namespace ab {

namespace {

constexpr int BM = 64, BN = 64, BK = 16;

struct SimtSeg {
    const float* a; int64_t lda; int amn;
    const float* b; int64_t ldb; int bmn;
    int K;
};

struct SimtParams {
    int M, N, nseg;
    SimtSeg seg[2];
    void* C; int64_t ldc; int cbf16;
    float alpha; int accumulate; const float* bias;
};

__global__ void __launch_bounds__(256) gemm_simt_kernel(const SimtParams p) {
    __shared__ float As[BK][BM + 4];
    __shared__ float Bs[BK][BN + 4];
    const int tid = threadIdx.x;
    const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
    const int tm = (tid / 16) * 4, tn = (tid % 16) * 4;
    float acc[4][4] = {};
    for (int s = 0; s < p.nseg; ++s) {
        const SimtSeg& sg = p.seg[s];
        for (int k0 = 0; k0 < sg.K; k0 += BK) {
            for (int e = tid; e < BM * BK; e += 256) {
                int m, k;
                if (sg.amn) { m = e % BM; k = e / BM; } else { k = e % BK; m = e / BK; }
                const int gm = m0 + m, gk = k0 + k;
                float v = 0.f;
                if (gm < p.M && gk < sg.K)
                    v = sg.amn ? sg.a[(int64_t)gk * sg.lda + gm] : sg.a[(int64_t)gm * sg.lda + gk];
                As[k][m] = v;
            }
            for (int e = tid; e < BN * BK; e += 256) {
                int n, k;
                if (sg.bmn) { n = e % BN; k = e / BN; } else { k = e % BK; n = e / BK; }
                const int gn = n0 + n, gk = k0 + k;
                float v = 0.f;
                if (gn < p.N && gk < sg.K)
                    v = sg.bmn ? sg.b[(int64_t)gk * sg.ldb + gn] : sg.b[(int64_t)gn * sg.ldb + gk];
                Bs[k][n] = v;
            }
            __syncthreads();
#pragma unroll
            for (int k = 0; k < BK; ++k) {
                float av[4], bv[4];
#pragma unroll
                for (int i = 0; i < 4; ++i) { av[i] = As[k][tm + i]; bv[i] = Bs[k][tn + i]; }
#pragma unroll
                for (int i = 0; i < 4; ++i)
#pragma unroll
                    for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
            }
            __syncthreads();
        }
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int gm = m0 + tm + i;
        if (gm >= p.M) continue;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int gn = n0 + tn + j;
            if (gn >= p.N) continue;
            float v = p.alpha * acc[i][j];
            if (p.bias) v += p.bias[gn];
            const int64_t off = (int64_t)gm * p.ldc + gn;
            if (p.cbf16) {
                bf16* c = reinterpret_cast<bf16*>(p.C);
                if (p.accumulate) v += __bfloat162float(c[off]);
                c[off] = __float2bfloat16_rn(v);
            } else {
                float* c = reinterpret_cast<float*>(p.C);
                if (p.accumulate) v += c[off];
                c[off] = v;
            }
        }
    }
}

}  // namespace

void gemm_simt(const GemmArgs& g, cudaStream_t s) {
    if (g.M <= 0 || g.N <= 0) return;
    AB_CHECK(g.extra == nullptr, ADPSGD_E_DIMENSION, "column redirect is a tcgen05-path feature");
    SimtParams p{};
    p.M = g.M; p.N = g.N; p.nseg = g.nseg;
    for (int i = 0; i < g.nseg; ++i) {
        p.seg[i].a = static_cast<const float*>(g.seg[i].a.ptr);
        p.seg[i].lda = g.seg[i].a.ld; p.seg[i].amn = g.seg[i].a.mn;
        p.seg[i].b = static_cast<const float*>(g.seg[i].b.ptr);
        p.seg[i].ldb = g.seg[i].b.ld; p.seg[i].bmn = g.seg[i].b.mn;
        p.seg[i].K = g.seg[i].K;
    }
    p.C = g.C; p.ldc = g.ldc; p.cbf16 = g.c_bf16;
    p.alpha = g.alpha; p.accumulate = g.accumulate; p.bias = g.bias;
    double ksum = 0;
    for (int i = 0; i < g.nseg; ++i) ksum += g.seg[i].K;
    ProfScope ps_(s, PROF_GEMM_SIMT, 2.0 * g.M * g.N * ksum,
                  4.0 * (static_cast<double>(g.M) + g.N) * ksum + static_cast<double>(g.M) * g.N * 4.0);
    dim3 grid((g.N + BN - 1) / BN, (g.M + BM - 1) / BM);
    gemm_simt_kernel<<<grid, 256, 0, s>>>(p);
    count_launch();
    AB_CUDA(cudaGetLastError());
}

}  // namespace ab
