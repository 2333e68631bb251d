// Pointwise, reduction and update kernels of the ADPSGD learner step (sm_100a).
// All are HBM-bound: vectorised, grid-stride, grids sized in multiples of the SM count.
#include "kernels.cuh"
#include "prof.hpp"

namespace ab {

int64_t g_launch_count = 0;

namespace {

constexpr int kMaxTab = 64;
struct PtrTab { const float* p[kMaxTab]; };
struct MutTab { float* p[kMaxTab]; };
struct BfTab { bf16* p[kMaxTab]; };

inline int grid_for(int64_t work, int threads = 256, int per_sm = 8) {
    int64_t g = (work + threads - 1) / threads;
    const int64_t cap = static_cast<int64_t>(num_sms()) * per_sm;
    if (g > cap) g = cap;
    return static_cast<int>(g < 1 ? 1 : g);
}

// ---- gather ----
template <typename AT>
__global__ void gather_kernel(const float* __restrict__ feats, const int32_t* __restrict__ labels,
                              const int32_t* __restrict__ idx, int B, int T, int I, int ldx, AT* __restrict__ X,
                              int32_t* __restrict__ lab, int ones_col, AT* __restrict__ tail, int tail_n0) {
    const int64_t total = static_cast<int64_t>(T) * B * ldx;
    for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int i = static_cast<int>(e % ldx);
        const int64_t r = e / ldx;  // r = t*B + b
        const int b = static_cast<int>(r % B), t = static_cast<int>(r / B);
        const int64_t n = idx[b];
        const float v = i < I ? feats[(n * T + t) * I + i] : ((ones_col && i == I) ? 1.f : 0.f);
        X[e] = from_f<AT>(v);
        // K-major copy of columns [tail_n0, tail_n0 + 8) for the tail-column weight-gradient MMA
        if (tail && i >= tail_n0 && i < tail_n0 + 8) tail[static_cast<int64_t>(i - tail_n0) * T * B + r] = from_f<AT>(v);
        if (i == 0) lab[r] = labels[n * T + t];
    }
}

// 4 columns per thread (I % 4 == 0, ldx % 4 == 0): one 16-byte feature load, one 8-byte bf16 /
// 16-byte fp32 store; the group holding column I also writes the ones column and the zero pad.
template <typename AT>
__global__ void gather4_kernel(const float* __restrict__ feats, const int32_t* __restrict__ labels,
                               const int32_t* __restrict__ idx, int B, int T, int I, int ldx, AT* __restrict__ X,
                               int32_t* __restrict__ lab, int ones_col, AT* __restrict__ tail, int tail_n0) {
    const int g4 = ldx / 4;
    const int64_t total = static_cast<int64_t>(T) * B * g4;
    for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int i0 = static_cast<int>(e % g4) * 4;
        const int64_t r = e / g4;  // r = t*B + b
        const int b = static_cast<int>(r % B), t = static_cast<int>(r / B);
        const int64_t n = idx[b];
        float v[4];
        if (i0 + 4 <= I) {
            const float4 f = __ldg(reinterpret_cast<const float4*>(feats + (n * T + t) * I + i0));
            v[0] = f.x; v[1] = f.y; v[2] = f.z; v[3] = f.w;
        } else {
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const int i = i0 + k;
                v[k] = i < I ? feats[(n * T + t) * I + i] : ((ones_col && i == I) ? 1.f : 0.f);
            }
        }
        AT* dst = X + r * ldx + i0;
#pragma unroll
        for (int k = 0; k < 4; ++k) dst[k] = from_f<AT>(v[k]);
        if (tail && i0 + 4 > tail_n0 && i0 < tail_n0 + 8) {
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const int i = i0 + k;
                if (i >= tail_n0 && i < tail_n0 + 8) tail[static_cast<int64_t>(i - tail_n0) * T * B + r] = from_f<AT>(v[k]);
            }
        }
        if (i0 == 0) lab[r] = labels[n * T + t];
    }
}

// ---- LSTM cell ----
template <typename AT>
__global__ void cell_fwd_kernel(const float* __restrict__ z, int ldz, const float* __restrict__ c_prev, int ldc,
                                AT* __restrict__ gates, int ldg, float* __restrict__ c, AT* __restrict__ h, int ldh,
                                int B, int H) {
    const int64_t total = static_cast<int64_t>(B) * H;
    for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int b = static_cast<int>(e / H), j = static_cast<int>(e % H);
        const float* zr = z + static_cast<int64_t>(b) * ldz;
        const float ig = 1.f / (1.f + expf(-zr[j]));
        const float fg = 1.f / (1.f + expf(-zr[H + j]));
        const float gg = tanhf(zr[2 * H + j]);
        const float og = 1.f / (1.f + expf(-zr[3 * H + j]));
        const float cp = c_prev ? c_prev[static_cast<int64_t>(b) * ldc + j] : 0.f;
        const float cn = fg * cp + ig * gg;
        AT* gr = gates + static_cast<int64_t>(b) * ldg;
        gr[j] = from_f<AT>(ig); gr[H + j] = from_f<AT>(fg); gr[2 * H + j] = from_f<AT>(gg); gr[3 * H + j] = from_f<AT>(og);
        c[static_cast<int64_t>(b) * ldc + j] = cn;
        h[static_cast<int64_t>(b) * ldh + j] = from_f<AT>(og * tanhf(cn));
    }
}

template <typename AT>
__global__ void cell_bwd_kernel(const float* __restrict__ dH, int lddh, const float* __restrict__ dh_rec,
                                float* __restrict__ dc_rec, int first, const AT* __restrict__ gates, int ldg,
                                const float* __restrict__ c, const float* __restrict__ c_prev, int ldc,
                                AT* __restrict__ dz, int lddz, int B, int H) {
    const int64_t total = static_cast<int64_t>(B) * H;
    for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int b = static_cast<int>(e / H), j = static_cast<int>(e % H);
        float dh = dH[static_cast<int64_t>(b) * lddh + j];
        float dcr = 0.f;
        if (!first) { dh += dh_rec[e]; dcr = dc_rec[e]; }
        const AT* gr = gates + static_cast<int64_t>(b) * ldg;
        const float ig = to_f<AT>(gr[j]), fg = to_f<AT>(gr[H + j]), gg = to_f<AT>(gr[2 * H + j]), og = to_f<AT>(gr[3 * H + j]);
        const float tc = tanhf(c[static_cast<int64_t>(b) * ldc + j]);
        const float cp = c_prev ? c_prev[static_cast<int64_t>(b) * ldc + j] : 0.f;
        const float dc = dcr + dh * og * (1.f - tc * tc);
        AT* dzr = dz + static_cast<int64_t>(b) * lddz;
        dzr[j] = from_f<AT>(dc * gg * ig * (1.f - ig));
        dzr[H + j] = from_f<AT>(dc * cp * fg * (1.f - fg));
        dzr[2 * H + j] = from_f<AT>(dc * ig * (1.f - gg * gg));
        dzr[3 * H + j] = from_f<AT>(dh * tc * og * (1.f - og));
        dc_rec[e] = dc * fg;
    }
}

// First BPTT cell backward (no recurrent term) of both directions in one launch, 8 units per
// thread with 16-byte accesses (bf16 gates / dz, fp32 dH / c / c_prev / dc_rec).
struct CellFirstDir {
    const float* dH; const bf16* gates; const float* c; const float* c_prev; bf16* dz; float* dc_rec;
};
struct CellFirstArgs {
    CellFirstDir d[2];
    int lddh, ldg, ldc, lddz, B, H;
};
__global__ void cell_bwd_first2_kernel(const __grid_constant__ CellFirstArgs a) {
    const CellFirstDir& D = a.d[blockIdx.y];
    const int hv = a.H / 8;
    const int64_t total = static_cast<int64_t>(a.B) * hv;
    for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int b = static_cast<int>(e / hv), j = static_cast<int>(e % hv) * 8;
        float dh[8], c[8], cp[8], gi[8], gf[8], gg[8], go[8];
        const float4* ph = reinterpret_cast<const float4*>(D.dH + static_cast<int64_t>(b) * a.lddh + j);
        const float4* pc = reinterpret_cast<const float4*>(D.c + static_cast<int64_t>(b) * a.ldc + j);
        for (int v = 0; v < 2; ++v) {
            const float4 x = __ldg(ph + v), y = __ldg(pc + v);
            dh[4 * v] = x.x; dh[4 * v + 1] = x.y; dh[4 * v + 2] = x.z; dh[4 * v + 3] = x.w;
            c[4 * v] = y.x; c[4 * v + 1] = y.y; c[4 * v + 2] = y.z; c[4 * v + 3] = y.w;
        }
        if (D.c_prev) {
            const float4* pp = reinterpret_cast<const float4*>(D.c_prev + static_cast<int64_t>(b) * a.ldc + j);
            for (int v = 0; v < 2; ++v) {
                const float4 z = __ldg(pp + v);
                cp[4 * v] = z.x; cp[4 * v + 1] = z.y; cp[4 * v + 2] = z.z; cp[4 * v + 3] = z.w;
            }
        } else {
            for (int i = 0; i < 8; ++i) cp[i] = 0.f;
        }
        const bf16* gr = D.gates + static_cast<int64_t>(b) * a.ldg + j;
        float* gsets[4] = {gi, gf, gg, go};
        for (int q = 0; q < 4; ++q) {
            const uint4 u = __ldg(reinterpret_cast<const uint4*>(gr + static_cast<int64_t>(q) * a.H));
            const bf16* ub = reinterpret_cast<const bf16*>(&u);
            for (int i = 0; i < 8; ++i) gsets[q][i] = __bfloat162float(ub[i]);
        }
        bf16 zi[8], zf[8], zg[8], zo[8];
        float dco[8];
        for (int i = 0; i < 8; ++i) {
            const float tc = tanhf(c[i]);
            const float dc = dh[i] * go[i] * (1.f - tc * tc);
            zi[i] = __float2bfloat16_rn(dc * gg[i] * gi[i] * (1.f - gi[i]));
            zf[i] = __float2bfloat16_rn(dc * cp[i] * gf[i] * (1.f - gf[i]));
            zg[i] = __float2bfloat16_rn(dc * gi[i] * (1.f - gg[i] * gg[i]));
            zo[i] = __float2bfloat16_rn(dh[i] * tc * go[i] * (1.f - go[i]));
            dco[i] = dc * gf[i];
        }
        bf16* dzr = D.dz + static_cast<int64_t>(b) * a.lddz + j;
        *reinterpret_cast<uint4*>(dzr) = *reinterpret_cast<const uint4*>(zi);
        *reinterpret_cast<uint4*>(dzr + a.H) = *reinterpret_cast<const uint4*>(zf);
        *reinterpret_cast<uint4*>(dzr + 2 * a.H) = *reinterpret_cast<const uint4*>(zg);
        *reinterpret_cast<uint4*>(dzr + 3 * a.H) = *reinterpret_cast<const uint4*>(zo);
        float4* pd = reinterpret_cast<float4*>(D.dc_rec + static_cast<int64_t>(b) * a.H + j);
        pd[0] = make_float4(dco[0], dco[1], dco[2], dco[3]);
        pd[1] = make_float4(dco[4], dco[5], dco[6], dco[7]);
    }
}

// ---- softmax cross-entropy (one block per row) ----
__device__ __forceinline__ float block_reduce(float v, bool is_max, float* sh) {
    const int lane = threadIdx.x % 32, w = threadIdx.x / 32;
    for (int o = 16; o; o >>= 1) {
        const float u = __shfl_xor_sync(0xffffffffu, v, o);
        v = is_max ? fmaxf(v, u) : v + u;
    }
    __syncthreads();
    if (lane == 0) sh[w] = v;
    __syncthreads();
    const int nw = blockDim.x / 32;
    v = threadIdx.x < nw ? sh[threadIdx.x] : (is_max ? -INFINITY : 0.f);
    if (w == 0)
        for (int o = 16; o; o >>= 1) {
            const float u = __shfl_xor_sync(0xffffffffu, v, o);
            v = is_max ? fmaxf(v, u) : v + u;
        }
    if (threadIdx.x == 0) sh[0] = v;
    __syncthreads();
    return sh[0];
}

template <typename AT>
__global__ void __launch_bounds__(256) softmax_ce_kernel(const float* __restrict__ logits,
                                                         const int32_t* __restrict__ labels, int C, float scale,
                                                         AT* __restrict__ dlogits, float* __restrict__ row_loss) {
    __shared__ float sh[32];
    const int64_t r = blockIdx.x;
    const float* x = logits + r * C;
    float mx = -INFINITY;
    for (int i = threadIdx.x; i < C; i += blockDim.x) mx = fmaxf(mx, x[i]);
    mx = block_reduce(mx, true, sh);
    float se = 0.f;
    for (int i = threadIdx.x; i < C; i += blockDim.x) se += expf(x[i] - mx);
    se = block_reduce(se, false, sh);
    const float lse = mx + logf(se);
    const int lab = labels[r];
    AT* d = dlogits + r * C;
    for (int i = threadIdx.x; i < C; i += blockDim.x) {
        float p = expf(x[i] - lse) * scale;
        if (i == lab) p -= scale;
        d[i] = from_f<AT>(p);
    }
    if (threadIdx.x == 0) row_loss[r] = lse - x[lab];
}

// ---- deterministic column sums ----
template <typename AT>
__global__ void colsum_partial_kernel(const AT* __restrict__ X, int64_t ld, int R, int N, int rows_per_chunk,
                                      float* __restrict__ part) {
    const int n = blockIdx.x * blockDim.x + threadIdx.x;
    const int chunk = blockIdx.y;
    if (n >= N) return;
    const int r0 = chunk * rows_per_chunk;
    const int r1 = min(R, r0 + rows_per_chunk);
    float s = 0.f;
    for (int r = r0; r < r1; ++r) s += to_f<AT>(X[static_cast<int64_t>(r) * ld + n]);
    part[static_cast<int64_t>(chunk) * N + n] = s;
}
// bf16 rows, 8 columns per thread (16-byte loads): the bias-gradient column sums of dZ / dY
__global__ void colsum_partial_bf16x8_kernel(const bf16* __restrict__ X, int64_t ld, int R, int N, int rows_per_chunk,
                                             float* __restrict__ part) {
    const int n0 = 8 * (blockIdx.x * blockDim.x + threadIdx.x);
    const int chunk = blockIdx.y;
    if (n0 >= N) return;
    const int r0 = chunk * rows_per_chunk;
    const int r1 = min(R, r0 + rows_per_chunk);
    float s[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll 4
    for (int r = r0; r < r1; ++r) {
        const uint4 v = __ldcs(reinterpret_cast<const uint4*>(X + static_cast<int64_t>(r) * ld + n0));
        const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&v);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const float2 f = __bfloat1622float2(h[i]);
            s[2 * i] += f.x;
            s[2 * i + 1] += f.y;
        }
    }
    float4* o = reinterpret_cast<float4*>(part + static_cast<int64_t>(chunk) * N + n0);
    o[0] = make_float4(s[0], s[1], s[2], s[3]);
    o[1] = make_float4(s[4], s[5], s[6], s[7]);
}
__global__ void colsum_final_kernel(const float* __restrict__ part, int chunks, int N, float* __restrict__ out) {
    const int n = blockIdx.x * blockDim.x + threadIdx.x;
    if (n >= N) return;
    float s = 0.f;
    for (int c = 0; c < chunks; ++c) s += part[static_cast<int64_t>(c) * N + n];
    out[n] = s;
}

__global__ void sum_kernel(const float* __restrict__ x, int n, float scale, float* __restrict__ out) {
    __shared__ float sh[32];
    float s = 0.f;
    const int n4 = (reinterpret_cast<uintptr_t>(x) & 15) == 0 ? n / 4 : 0;  // 16-byte loads, fixed order
    for (int i = threadIdx.x; i < n4; i += blockDim.x) {
        const float4 v = __ldg(reinterpret_cast<const float4*>(x) + i);
        s += (v.x + v.y) + (v.z + v.w);
    }
    for (int i = 4 * n4 + threadIdx.x; i < n; i += blockDim.x) s += x[i];
    s = block_reduce(s, false, sh);
    if (threadIdx.x == 0) out[0] = s * scale;
}

// sum of row_loss over rows r = t*B + b with b < valid (masked tail of a padded batch)
__global__ void sum_masked_kernel(const float* __restrict__ x, int T, int B, int valid, float* __restrict__ out) {
    __shared__ float sh[32];
    float s = 0.f;
    for (int i = threadIdx.x; i < T * B; i += blockDim.x)
        if (i % B < valid) s += x[i];
    s = block_reduce(s, false, sh);
    if (threadIdx.x == 0) out[0] = s;
}

__global__ void fill_col_kernel(bf16* __restrict__ p, int64_t rows, int64_t ld, int col, float v) {
    for (int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; r < rows;
         r += static_cast<int64_t>(gridDim.x) * blockDim.x)
        p[r * ld + col] = __float2bfloat16_rn(v);
}

__global__ void f32_to_bf16_kernel(const float* __restrict__ in, bf16* __restrict__ out, int64_t n) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        out[i] = __float2bfloat16_rn(in[i]);
}
__global__ void pad_rows_kernel(const float* __restrict__ in, int64_t ld_in, bf16* __restrict__ out, int64_t ld_out,
                                int rows, int cols) {
    const int64_t total = static_cast<int64_t>(rows) * ld_out;
    for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t r = e / ld_out, c = e % ld_out;
        out[e] = __float2bfloat16_rn(c < cols ? in[r * ld_in + c] : 0.f);
    }
}

// ---- mixing / update ----
__global__ void mix3_kernel(int64_t n, const float* __restrict__ w, const float* __restrict__ wl,
                            const float* __restrict__ wr, const float* __restrict__ g, float lr,
                            float* __restrict__ out, bf16* __restrict__ shadow) {
    const float third = 1.0f / 3.0f;
    const int64_t n4 = n / 4;
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n4; i += stride) {
        const float4 a = reinterpret_cast<const float4*>(w)[i];
        const float4 b = reinterpret_cast<const float4*>(wl)[i];
        const float4 c = reinterpret_cast<const float4*>(wr)[i];
        const float4 d = reinterpret_cast<const float4*>(g)[i];
        float4 o;
        o.x = (a.x + b.x + c.x) * third - lr * d.x;
        o.y = (a.y + b.y + c.y) * third - lr * d.y;
        o.z = (a.z + b.z + c.z) * third - lr * d.z;
        o.w = (a.w + b.w + c.w) * third - lr * d.w;
        reinterpret_cast<float4*>(out)[i] = o;
        if (shadow) {
            __nv_bfloat162 lo = __floats2bfloat162_rn(o.x, o.y), hi = __floats2bfloat162_rn(o.z, o.w);
            reinterpret_cast<__nv_bfloat162*>(shadow)[2 * i] = lo;
            reinterpret_cast<__nv_bfloat162*>(shadow)[2 * i + 1] = hi;
        }
    }
    for (int64_t i = n4 * 4 + blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n; i += stride) {
        const float o = (w[i] + wl[i] + wr[i]) * third - lr * g[i];
        out[i] = o;
        if (shadow) shadow[i] = __float2bfloat16_rn(o);
    }
}

__device__ __forceinline__ float4 f4add(float4 a, float4 b) { return make_float4(a.x + b.x, a.y + b.y, a.z + b.z, a.w + b.w); }
__device__ __forceinline__ void st_shadow4(bf16* sh, int64_t i4, float4 o) {
    __nv_bfloat162 lo = __floats2bfloat162_rn(o.x, o.y), hi = __floats2bfloat162_rn(o.z, o.w);
    uint2 u;
    u.x = *reinterpret_cast<uint32_t*>(&lo);
    u.y = *reinterpret_cast<uint32_t*>(&hi);
    reinterpret_cast<uint2*>(sh)[i4] = u;
}

// D1D update, float4-vectorised: one pass reads the L models (or their allreduced sum) and
// the local gradients, writes the new fp32 models and their bf16 shadows.
__global__ void d1d_kernel(int64_t n, int L, PtrTab w, const float* __restrict__ w_sum, int nloc, PtrTab g, float lr,
                           MutTab out, BfTab sh) {
    const float invL = 1.0f / static_cast<float>(L);
    const int64_t n4 = n / 4;
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n4; i += stride) {
        float4 s;
        if (w_sum) {
            s = reinterpret_cast<const float4*>(w_sum)[i];
        } else {
            s = reinterpret_cast<const float4*>(w.p[0])[i];
            for (int l = 1; l < L; ++l) s = f4add(s, reinterpret_cast<const float4*>(w.p[l])[i]);
        }
        for (int j = 0; j < nloc; ++j) {
            const float4 gg = reinterpret_cast<const float4*>(g.p[j])[i];
            const float4 o = make_float4(s.x * invL - lr * gg.x, s.y * invL - lr * gg.y, s.z * invL - lr * gg.z,
                                         s.w * invL - lr * gg.w);
            reinterpret_cast<float4*>(out.p[j])[i] = o;
            if (sh.p[j]) st_shadow4(sh.p[j], i, o);
        }
    }
    for (int64_t i = n4 * 4 + blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n; i += stride) {
        float s;
        if (w_sum) {
            s = w_sum[i];
        } else {
            s = 0.f;
            for (int l = 0; l < L; ++l) s += w.p[l][i];
        }
        for (int j = 0; j < nloc; ++j) {
            const float o = s * invL - lr * g.p[j][i];
            out.p[j][i] = o;
            if (sh.p[j]) sh.p[j][i] = __float2bfloat16_rn(o);
        }
    }
}

// SDPSGD update (engine.cpp:145-153), float4-vectorised.
// out = in[0] + in[1] + ... (learner order, the same summation order as d1d / sdpsgd kernels)
__global__ void sum_tab_kernel(int64_t n, int L, PtrTab in, float* __restrict__ out) {
    const int64_t n4 = n / 4;
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n4; i += stride) {
        float4 s = reinterpret_cast<const float4*>(in.p[0])[i];
        for (int l = 1; l < L; ++l) s = f4add(s, reinterpret_cast<const float4*>(in.p[l])[i]);
        reinterpret_cast<float4*>(out)[i] = s;
    }
    for (int64_t i = n4 * 4 + blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n; i += stride) {
        float s = in.p[0][i];
        for (int l = 1; l < L; ++l) s += in.p[l][i];
        out[i] = s;
    }
}

__global__ void sdpsgd_kernel(int64_t n, int L, const float* __restrict__ w, PtrTab g, const float* __restrict__ g_sum,
                              int nloc, float lr, MutTab out, BfTab sh) {
    const float invL = 1.0f / static_cast<float>(L);
    const int64_t n4 = n / 4;
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n4; i += stride) {
        float4 s;
        if (g_sum) {
            s = reinterpret_cast<const float4*>(g_sum)[i];
        } else {
            s = reinterpret_cast<const float4*>(g.p[0])[i];
            for (int l = 1; l < L; ++l) s = f4add(s, reinterpret_cast<const float4*>(g.p[l])[i]);
        }
        const float4 wv = reinterpret_cast<const float4*>(w)[i];
        const float4 o = make_float4(wv.x - lr * (s.x * invL), wv.y - lr * (s.y * invL), wv.z - lr * (s.z * invL),
                                     wv.w - lr * (s.w * invL));
        for (int j = 0; j < nloc; ++j) {
            reinterpret_cast<float4*>(out.p[j])[i] = o;
            if (sh.p[j]) st_shadow4(sh.p[j], i, o);
        }
    }
    for (int64_t i = n4 * 4 + blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n; i += stride) {
        float s;
        if (g_sum) {
            s = g_sum[i];
        } else {
            s = 0.f;
            for (int l = 0; l < L; ++l) s += g.p[l][i];
        }
        const float o = w[i] - lr * (s * invL);
        for (int j = 0; j < nloc; ++j) {
            out.p[j][i] = o;
            if (sh.p[j]) sh.p[j][i] = __float2bfloat16_rn(o);
        }
    }
}

struct DenseT { float t[kMaxTab]; int idx[kMaxTab]; int cnt; };
struct DenseArgs { DenseT col[16]; };

__global__ void dense_mix_kernel(int64_t n, PtrTab w, DenseArgs T, int nloc, PtrTab g, float lr, MutTab out,
                                 BfTab sh) {
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        for (int j = 0; j < nloc; ++j) {
            float s = 0.f;
            for (int q = 0; q < T.col[j].cnt; ++q) s += T.col[j].t[q] * w.p[T.col[j].idx[q]][i];
            const float o = s - lr * g.p[j][i];
            out.p[j][i] = o;
            if (sh.p[j]) sh.p[j][i] = __float2bfloat16_rn(o);
        }
    }
}

__global__ void maxdiff_kernel(int64_t n, const float* __restrict__ a, const float* __restrict__ b, float* out) {
    float m = 0.f;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        m = fmaxf(m, fabsf(a[i] - b[i]));
    for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0) atomicMax(reinterpret_cast<int*>(out), __float_as_int(m));
}

// Gram of the deviations from the learner mean, G[a][b] += sum_p (w_a - mean)(w_b - mean), for a
// list of up to 36 (a, b) pairs per launch (mixing.cpp:159-180 consensus_distance, on device).
struct PairList { int a[36], b[36]; int n; };
__global__ void gram_kernel(int64_t n, int L, PtrTab w, PairList pl, double* __restrict__ G) {
    double acc[36];
#pragma unroll
    for (int q = 0; q < 36; ++q) acc[q] = 0.0;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        float v[kMaxTab > 16 ? 16 : kMaxTab];
        float mean = 0.f;
        for (int l = 0; l < L; ++l) { v[l] = w.p[l][i]; mean += v[l]; }
        mean /= static_cast<float>(L);
#pragma unroll
        for (int q = 0; q < 36; ++q)
            if (q < pl.n) acc[q] += static_cast<double>(v[pl.a[q]] - mean) * static_cast<double>(v[pl.b[q]] - mean);
    }
    __shared__ double sh[36][8];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
    for (int q = 0; q < 36; ++q) {
        double x = acc[q];
        for (int o = 16; o; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
        if (lane == 0 && wid < 8) sh[q][wid] = x;
    }
    __syncthreads();
    if (threadIdx.x < pl.n) {  // this block's partial; gram_reduce_kernel sums blocks in order (deterministic)
        double x = 0.0;
        for (int j = 0; j < (blockDim.x >> 5) && j < 8; ++j) x += sh[threadIdx.x][j];
        G[static_cast<int64_t>(blockIdx.x) * 36 + threadIdx.x] = x;
    }
}

__global__ void gram_reduce_kernel(int nblocks, int L, PairList pl, const double* __restrict__ part,
                                   double* __restrict__ G) {
    const int q = threadIdx.x;
    if (q >= pl.n) return;
    double x = 0.0;
    for (int b = 0; b < nblocks; ++b) x += part[static_cast<int64_t>(b) * 36 + q];
    G[pl.a[q] * L + pl.b[q]] = x;
}

__device__ __forceinline__ uint64_t hash64(uint64_t x) {
    x += 0x9e3779b97f4a7c15ULL;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
    return x ^ (x >> 31);
}
__device__ __forceinline__ float u01(uint64_t h) { return (static_cast<float>(h >> 40) + 0.5f) * (1.0f / 16777216.0f); }

// Synthetic SWB-shaped frames: label ~ U[0,C) per frame with a slowly varying state
// (runs of frames share a label), features N(0,1) + 0.75 * class prototype (+/-1).
__global__ void synth_kernel(float* __restrict__ feats, int32_t* __restrict__ labels, int n_seg, int T, int I, int C,
                             uint64_t seed) {
    const int64_t total = static_cast<int64_t>(n_seg) * T * I;
    for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int i = static_cast<int>(e % I);
        const int64_t nt = e / I;
        const int t = static_cast<int>(nt % T);
        const int64_t n = nt / T;
        const uint64_t lh = hash64(seed ^ hash64(static_cast<uint64_t>(n) * 64 + t / 4));
        const int lab = static_cast<int>(lh % static_cast<uint64_t>(C));
        const uint64_t h1 = hash64(seed + 0x1234567ULL + static_cast<uint64_t>(e) * 2);
        const uint64_t h2 = hash64(seed + 0x89abcdefULL + static_cast<uint64_t>(e) * 2 + 1);
        const float r = sqrtf(-2.f * logf(u01(h1)));
        const float gsn = r * cospif(2.f * u01(h2));
        const float proto = (hash64(static_cast<uint64_t>(lab) * 1315423911ULL + i) & 1) ? 0.75f : -0.75f;
        feats[e] = gsn + proto;
        if (i == 0) labels[nt] = lab;
    }
}

__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ long long ld_acquire_sys(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return static_cast<long long>(v);
}
__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void st_relaxed_sys(unsigned long long* p, unsigned long long v) {
    asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

constexpr int kAsyncFree = 0, kAsyncLockstep = 1, kAsyncBounded = 2;

__global__ void async_select_kernel(AsyncPeers pe, int mode, long long k, long long lag, unsigned long long* my_ver,
                                    AsyncSel* sel, unsigned long long timeout_ns) {
    if (threadIdx.x != 0) return;
    const unsigned long long t0 = gtimer();
    sel->torn = 0;
    sel->err = 0;
    for (int side = 0; side < 2; ++side) {
        long long v = ld_acquire_sys(pe.ver[side]);
        const bool wait = mode == kAsyncLockstep || mode == kAsyncBounded;
        const long long need = mode == kAsyncLockstep ? k : k - lag;
        while (wait && v < need) {
            if (gtimer() - t0 > timeout_ns) {
                sel->err = 1;
                return;
            }
            __nanosleep(2000);
            v = ld_acquire_sys(pe.ver[side]);
        }
        const long long c = mode == kAsyncLockstep ? k : v;
        sel->ptr[side] = pe.slots[side][c & 3];
        sel->ver[side] = c;
    }
    sel->wait_ns = static_cast<long long>(gtimer() - t0);
    // slot (k + 1) % 4 is about to be overwritten: readers of version k - 3 must see it first
    st_relaxed_sys(my_ver + 1, static_cast<unsigned long long>(k + 1));
    __threadfence_system();
}

__global__ void mix3_sel_kernel(int64_t n, const float* __restrict__ w, const AsyncSel* __restrict__ sel,
                                const float* __restrict__ g, float lr, float* __restrict__ out, bf16* __restrict__ shadow) {
    if (sel->err) return;
    const float* __restrict__ wl = sel->ptr[0];
    const float* __restrict__ wr = sel->ptr[1];
    const float third = 1.0f / 3.0f;
    const int64_t n4 = n / 4;
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n4; i += stride) {
        const float4 a = reinterpret_cast<const float4*>(w)[i];
        const float4 b = reinterpret_cast<const float4*>(wl)[i];
        const float4 c = reinterpret_cast<const float4*>(wr)[i];
        const float4 d = reinterpret_cast<const float4*>(g)[i];
        float4 o;
        o.x = (a.x + b.x + c.x) * third - lr * d.x;
        o.y = (a.y + b.y + c.y) * third - lr * d.y;
        o.z = (a.z + b.z + c.z) * third - lr * d.z;
        o.w = (a.w + b.w + c.w) * third - lr * d.w;
        reinterpret_cast<float4*>(out)[i] = o;
        if (shadow) {
            reinterpret_cast<__nv_bfloat162*>(shadow)[2 * i] = __floats2bfloat162_rn(o.x, o.y);
            reinterpret_cast<__nv_bfloat162*>(shadow)[2 * i + 1] = __floats2bfloat162_rn(o.z, o.w);
        }
    }
    for (int64_t i = n4 * 4 + blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n; i += stride) {
        const float o = (w[i] + wl[i] + wr[i]) * third - lr * g[i];
        out[i] = o;
        if (shadow) shadow[i] = __float2bfloat16_rn(o);
    }
}

__global__ void async_publish_kernel(AsyncPeers pe, AsyncSel* sel, unsigned long long* my_ver, long long k) {
    if (threadIdx.x != 0 || sel->err) return;
    __threadfence_system();  // the mix (previous kernel) has read the neighbour slots
    const long long wl = ld_acquire_sys(pe.ver[0] + 1), wr = ld_acquire_sys(pe.ver[1] + 1);
    const int torn = (wl >= sel->ver[0] + 4) || (wr >= sel->ver[1] + 4);
    sel->torn = torn;
    if (!torn) st_release_sys(my_ver, static_cast<unsigned long long>(k + 1));
}

__global__ void delay_kernel(uint64_t ns) {
    uint64_t t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    for (;;) {
        uint64_t t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        if (t - t0 >= ns) break;
        __nanosleep(1000);
    }
}

}  // namespace

template <typename AT>
void launch_gather(const float* feats, const int32_t* labels, const int32_t* idx, int B, int T, int I, int ldx, AT* X,
                   int32_t* lab, cudaStream_t s, bool ones_col, AT* tail, int tail_n0) {
    ProfScope ps_(s, PROF_GATHER, 0, (double)T * B * ldx * (sizeof(AT) + 4.0) + (double)T * B * 8);
    const int64_t total = static_cast<int64_t>(T) * B * ldx;
    if (I % 4 == 0 && ldx % 4 == 0)
        gather4_kernel<AT><<<grid_for(total / 4), 256, 0, s>>>(feats, labels, idx, B, T, I, ldx, X, lab, ones_col ? 1 : 0,
                                                               tail, tail_n0);
    else
        gather_kernel<AT><<<grid_for(total), 256, 0, s>>>(feats, labels, idx, B, T, I, ldx, X, lab, ones_col ? 1 : 0, tail,
                                                          tail_n0);
    count_launch();
}

template <typename AT>
void launch_cell_fwd(const float* z, int ldz, const float* c_prev, int ldc, AT* gates, int ldg, float* c, AT* h,
                     int ldh, int B, int H, cudaStream_t s) {
    ProfScope ps_(s, PROF_CELL, 0, (double)B * H * (16 + 4 + 5 * sizeof(AT) + 4 + (c_prev ? 4 : 0)));
    cell_fwd_kernel<AT><<<grid_for(static_cast<int64_t>(B) * H), 256, 0, s>>>(z, ldz, c_prev, ldc, gates, ldg, c, h,
                                                                                ldh, B, H);
    count_launch();
}

template <typename AT>
void launch_cell_bwd(const float* dH, int lddh, const float* dh_rec, float* dc_rec, bool first, const AT* gates,
                     int ldg, const float* c, const float* c_prev, int ldc, AT* dz, int lddz, int B, int H,
                     cudaStream_t s) {
    ProfScope ps_(s, PROF_CELL, 0, (double)B * H * (4 + 4 * sizeof(AT) + 4 + 4 + 4 * sizeof(AT) + (first ? 0 : 8) + (c_prev ? 4 : 0)));
    cell_bwd_kernel<AT><<<grid_for(static_cast<int64_t>(B) * H), 256, 0, s>>>(
        dH, lddh, dh_rec, dc_rec, first ? 1 : 0, gates, ldg, c, c_prev, ldc, dz, lddz, B, H);
    count_launch();
}

template <typename AT>
void launch_softmax_ce(const float* logits, const int32_t* labels, int R, int C, float scale, AT* dlogits,
                       float* row_loss, cudaStream_t s) {
    ProfScope ps_(s, PROF_CE, 0, (double)R * C * (4 + sizeof(AT)) + (double)R * 8);
    softmax_ce_kernel<AT><<<R, 256, 0, s>>>(logits, labels, C, scale, dlogits, row_loss);
    count_launch();
}

template <typename AT>
void launch_colsum(const AT* X, int64_t ld, int R, int N, float* out, float* ws, int64_t ws_elems, cudaStream_t s) {
    ProfScope ps_(s, PROF_REDUCE, 0, (double)R * N * sizeof(AT) + (double)N * 4);
    int chunks = (R + 127) / 128;
    if (chunks > 128) chunks = 128;
    while (chunks > 1 && static_cast<int64_t>(chunks) * N > ws_elems) chunks /= 2;
    const int rpc = (R + chunks - 1) / chunks;
    const bool vec8 = sizeof(AT) == 2 && N % 8 == 0 && ld % 8 == 0 && (reinterpret_cast<uintptr_t>(X) & 15) == 0;
    if (vec8) {
        dim3 grid((N / 8 + 127) / 128, chunks);
        colsum_partial_bf16x8_kernel<<<grid, 128, 0, s>>>(reinterpret_cast<const bf16*>(X), ld, R, N, rpc, ws);
    } else {
        dim3 grid((N + 255) / 256, chunks);
        colsum_partial_kernel<AT><<<grid, 256, 0, s>>>(X, ld, R, N, rpc, ws);
    }
    colsum_final_kernel<<<(N + 255) / 256, 256, 0, s>>>(ws, chunks, N, out);
    count_launch(2);
}

void launch_sum(const float* x, int n, float scale, float* out, cudaStream_t s) {
    ProfScope ps_(s, PROF_REDUCE, 0, (double)n * 4);
    sum_kernel<<<1, 1024, 0, s>>>(x, n, scale, out);
    count_launch();
}

void launch_sum_masked(const float* x, int T, int B, int valid, float* out, cudaStream_t s) {
    ProfScope ps_(s, PROF_REDUCE, 0, static_cast<double>(T) * B * 4);
    sum_masked_kernel<<<1, 1024, 0, s>>>(x, T, B, valid, out);
    count_launch();
}

void launch_fill_col_bf16(bf16* p, int64_t rows, int64_t ld, int col, float v, cudaStream_t s) {
    fill_col_kernel<<<grid_for(rows), 256, 0, s>>>(p, rows, ld, col, v);
    count_launch();
}

void launch_f32_to_bf16(const float* in, bf16* out, int64_t n, cudaStream_t s) {
    ProfScope ps_(s, PROF_MIX, 0, (double)n * 6);
    f32_to_bf16_kernel<<<grid_for(n), 256, 0, s>>>(in, out, n);
    count_launch();
}
void launch_pad_rows_bf16(const float* in, int64_t ld_in, bf16* out, int64_t ld_out, int rows, int cols,
                          cudaStream_t s) {
    ProfScope ps_(s, PROF_MIX, 0, (double)rows * (cols * 4.0 + ld_out * 2.0));
    pad_rows_kernel<<<grid_for(static_cast<int64_t>(rows) * ld_out), 256, 0, s>>>(in, ld_in, out, ld_out, rows, cols);
    count_launch();
}

void launch_mix3(int64_t n, const float* w, const float* wl, const float* wr, const float* g, float lr, float* w_out,
                 bf16* shadow, cudaStream_t s) {
    ProfScope ps_(s, PROF_MIX, 0, (double)n * (20 + (shadow ? 2 : 0)));
    mix3_kernel<<<grid_for((n + 3) / 4, 256, 4), 256, 0, s>>>(n, w, wl, wr, g, lr, w_out, shadow);
    count_launch();
}

void launch_d1d(int64_t n, int L, const float* const* w_tab, const float* w_sum, int nloc, const float* const* g_tab,
                float lr, float* const* out_tab, bf16* const* shadow_tab, cudaStream_t s) {
    ProfScope ps_(s, PROF_MIX, 0, (double)n * ((w_sum ? 4 : 4 * L) + nloc * 10.0));
    AB_CHECK(L <= kMaxTab && nloc <= kMaxTab, ADPSGD_E_CONFIG, "too many learners for one device");
    PtrTab w{}, g{};
    MutTab o{};
    BfTab sh{};
    if (!w_sum)
        for (int i = 0; i < L; ++i) w.p[i] = w_tab[i];
    for (int j = 0; j < nloc; ++j) { g.p[j] = g_tab[j]; o.p[j] = out_tab[j]; sh.p[j] = shadow_tab[j]; }
    d1d_kernel<<<grid_for((n + 3) / 4, 256, 4), 256, 0, s>>>(n, L, w, w_sum, nloc, g, lr, o, sh);
    count_launch();
}

void launch_sum_tab(int64_t n, int L, const float* const* tab, float* out, cudaStream_t s) {
    ProfScope ps_(s, PROF_MIX, 0, (double)n * 4.0 * (L + 1));
    AB_CHECK(L >= 1 && L <= kMaxTab, ADPSGD_E_CONFIG, "sum_tab: 1..64 inputs");
    PtrTab t{};
    for (int i = 0; i < L; ++i) t.p[i] = tab[i];
    sum_tab_kernel<<<grid_for((n + 3) / 4, 256, 4), 256, 0, s>>>(n, L, t, out);
    count_launch();
}

void launch_sdpsgd(int64_t n, int L, const float* w, const float* const* g_tab, const float* g_sum, int nloc,
                   float lr, float* const* out_tab, bf16* const* shadow_tab, cudaStream_t s) {
    ProfScope ps_(s, PROF_MIX, 0, (double)n * ((g_sum ? 4 : 4 * L) + 4 + nloc * 6.0));
    AB_CHECK(L <= kMaxTab && nloc <= kMaxTab, ADPSGD_E_CONFIG, "too many learners for one device");
    PtrTab g{};
    MutTab o{};
    BfTab sh{};
    if (!g_sum)
        for (int i = 0; i < L; ++i) g.p[i] = g_tab[i];
    for (int j = 0; j < nloc; ++j) { o.p[j] = out_tab[j]; sh.p[j] = shadow_tab[j]; }
    sdpsgd_kernel<<<grid_for((n + 3) / 4, 256, 4), 256, 0, s>>>(n, L, w, g, g_sum, nloc, lr, o, sh);
    count_launch();
}

void launch_dense_mix(int64_t n, int L, const float* const* w_tab, const double* T, const int* cols, int nloc,
                      const float* const* g_tab, float lr, float* const* out_tab, bf16* const* shadow_tab,
                      cudaStream_t s) {
    ProfScope ps_(s, PROF_MIX, 0, (double)n * (4 * L + nloc * 10.0));
    AB_CHECK(L <= kMaxTab && nloc <= 16, ADPSGD_E_CONFIG, "too many learners for dense mixing");
    PtrTab w{}, g{};
    MutTab o{};
    BfTab sh{};
    DenseArgs da{};
    for (int i = 0; i < L; ++i) w.p[i] = w_tab[i];
    for (int j = 0; j < nloc; ++j) {
        g.p[j] = g_tab[j]; o.p[j] = out_tab[j]; sh.p[j] = shadow_tab[j];
        int cnt = 0;
        for (int i = 0; i < L; ++i) {
            const double t = T[i * L + cols[j]];
            if (t != 0.0) { da.col[j].t[cnt] = static_cast<float>(t); da.col[j].idx[cnt] = i; ++cnt; }
        }
        da.col[j].cnt = cnt;
    }
    dense_mix_kernel<<<grid_for(n, 256, 4), 256, 0, s>>>(n, w, da, nloc, g, lr, o, sh);
    count_launch();
}

void launch_gram(int64_t n, int L, const float* const* w_tab, double* G, double* partial, cudaStream_t s) {
    AB_CHECK(L >= 1 && L <= 16, ADPSGD_E_CONFIG, "device consensus distance supports up to 16 local learners");
    ProfScope ps_(s, PROF_OTHER, 0, static_cast<double>(n) * 4 * L);
    PtrTab w{};
    for (int l = 0; l < L; ++l) w.p[l] = w_tab[l];
    AB_CUDA(cudaMemsetAsync(G, 0, sizeof(double) * L * L, s));
    const int grid = grid_for(n, 256, 4);  // <= gram_partial_doubles() / 36 blocks
    PairList pl{};
    auto run = [&] {
        gram_kernel<<<grid, 256, 0, s>>>(n, L, w, pl, partial);
        gram_reduce_kernel<<<1, 64, 0, s>>>(grid, L, pl, partial, G);
        count_launch();
        count_launch();
        pl.n = 0;
    };
    for (int a = 0; a < L; ++a)
        for (int b = a; b < L; ++b) {
            pl.a[pl.n] = a;
            pl.b[pl.n] = b;
            if (++pl.n == 36) run();
        }
    if (pl.n) run();
}

size_t gram_partial_doubles() { return static_cast<size_t>(num_sms()) * 4 * 36; }

void launch_maxdiff(int64_t n, const float* a, const float* b, float* out, cudaStream_t s) {
    ProfScope ps_(s, PROF_OTHER, 0, (double)n * 8);
    maxdiff_kernel<<<grid_for(n, 256, 4), 256, 0, s>>>(n, a, b, out);
    count_launch();
}

void launch_synth(float* feats, int32_t* labels, int n_seg, int T, int I, int C, uint64_t seed, cudaStream_t s) {
    ProfScope ps_(s, PROF_OTHER, 0, (double)n_seg * T * I * 4);
    synth_kernel<<<grid_for(static_cast<int64_t>(n_seg) * T * I), 256, 0, s>>>(feats, labels, n_seg, T, I, C, seed);
    count_launch();
}

void launch_async_select(const AsyncPeers& pe, int mode, long long k, long long lag, unsigned long long* my_ver,
                         AsyncSel* sel, unsigned long long timeout_ns, cudaStream_t s) {
    ProfScope ps_(s, PROF_MIX, 0, 0);
    async_select_kernel<<<1, 32, 0, s>>>(pe, mode, k, lag, my_ver, sel, timeout_ns);
    count_launch();
}

void launch_mix3_sel(int64_t n, const float* w, const AsyncSel* sel, const float* g, float lr, float* w_out,
                     bf16* shadow, cudaStream_t s) {
    ProfScope ps_(s, PROF_MIX, 0, (double)n * (20.0 + (shadow ? 2.0 : 0.0)));
    AB_CHECK((reinterpret_cast<uintptr_t>(w) & 15) == 0 && (reinterpret_cast<uintptr_t>(w_out) & 15) == 0,
             ADPSGD_E_INVALID_STATE, "mix3_sel: 16-byte aligned weights required");
    mix3_sel_kernel<<<grid_for((n + 3) / 4, 256, 4), 256, 0, s>>>(n, w, sel, g, lr, w_out, shadow);
    count_launch();
}

void launch_async_publish(const AsyncPeers& pe, AsyncSel* sel, unsigned long long* my_ver, long long k,
                          cudaStream_t s) {
    ProfScope ps_(s, PROF_MIX, 0, 0);
    async_publish_kernel<<<1, 32, 0, s>>>(pe, sel, my_ver, k);
    count_launch();
}

void launch_delay(uint64_t ns, cudaStream_t s) {
    ProfScope ps_(s, PROF_OTHER, 0, 0);
    delay_kernel<<<1, 1, 0, s>>>(ns);
    count_launch();
}

// out[c * rows + r] = in[r * cols + c] (bf16, 32 x 32 smem tiles)
__global__ void transpose_bf16_kernel(const bf16* __restrict__ in, bf16* __restrict__ out, int rows, int cols) {
    __shared__ bf16 tile[32][33];
    const int c0 = blockIdx.x * 32, r0 = blockIdx.y * 32;
    for (int i = threadIdx.y; i < 32; i += blockDim.y) {
        const int r = r0 + i, c = c0 + threadIdx.x;
        if (r < rows && c < cols) tile[i][threadIdx.x] = in[static_cast<int64_t>(r) * cols + c];
    }
    __syncthreads();
    for (int i = threadIdx.y; i < 32; i += blockDim.y) {
        const int c = c0 + i, r = r0 + threadIdx.x;
        if (r < rows && c < cols) out[static_cast<int64_t>(c) * rows + r] = tile[threadIdx.x][i];
    }
}

void launch_transpose_bf16(const bf16* in, bf16* out, int rows, int cols, cudaStream_t s) {
    ProfScope ps_(s, PROF_REDUCE, 0, 4.0 * rows * cols);
    transpose_bf16_kernel<<<dim3((cols + 31) / 32, (rows + 31) / 32), dim3(32, 8), 0, s>>>(in, out, rows, cols);
    count_launch();
}

bool launch_cell_bwd_first2(const float* const dH[2], const bf16* const gates[2], const float* const c[2],
                            const float* const c_prev[2], bf16* const dz[2], float* const dc_rec[2], int lddh, int ldg,
                            int ldc, int lddz, int B, int H, cudaStream_t s) {
    auto al = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
    bool ok = H % 8 == 0 && lddh % 4 == 0 && ldc % 4 == 0 && ldg % 8 == 0 && lddz % 8 == 0;
    for (int d = 0; d < 2 && ok; ++d)
        ok = al(dH[d]) && al(gates[d]) && al(c[d]) && (!c_prev[d] || al(c_prev[d])) && al(dz[d]) && al(dc_rec[d]);
    if (!ok) return false;
    CellFirstArgs a;
    for (int d = 0; d < 2; ++d) a.d[d] = {dH[d], gates[d], c[d], c_prev[d], dz[d], dc_rec[d]};
    a.lddh = lddh; a.ldg = ldg; a.ldc = ldc; a.lddz = lddz; a.B = B; a.H = H;
    ProfScope ps_(s, PROF_CELL, 0, 2.0 * B * H * (4 + 8 + 4 + 4 + 8 + 4));
    const int64_t per = static_cast<int64_t>(B) * (H / 8);
    const int gx = static_cast<int>((per + 255) / 256 < 1184 ? (per + 255) / 256 : 1184);
    cell_bwd_first2_kernel<<<dim3(gx, 2), 256, 0, s>>>(a);
    count_launch();
    return true;
}

#define AB_INST(AT)                                                                                                  \
    template void launch_gather<AT>(const float*, const int32_t*, const int32_t*, int, int, int, int, AT*, int32_t*, \
                                    cudaStream_t, bool, AT*, int);                                                  \
    template void launch_cell_fwd<AT>(const float*, int, const float*, int, AT*, int, float*, AT*, int, int, int, \
                                      cudaStream_t);                                                                \
    template void launch_cell_bwd<AT>(const float*, int, const float*, float*, bool, const AT*, int, const float*, \
                                      const float*, int, AT*, int, int, int, cudaStream_t);                         \
    template void launch_softmax_ce<AT>(const float*, const int32_t*, int, int, float, AT*, float*, cudaStream_t);  \
    template void launch_colsum<AT>(const AT*, int64_t, int, int, float*, float*, int64_t, cudaStream_t);
AB_INST(float)
AB_INST(bf16)
#undef AB_INST

}  // namespace ab
