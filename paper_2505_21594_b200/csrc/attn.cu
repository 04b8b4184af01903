// attn.cu — K3: gamma-query causal attention over a paged bf16 KV cache.
//
// For request b, head h and query row j (position ctx_b + j) the kernel computes
//   a_j = softmax(q_j K^T / sqrt(Dh)) V   over keys 0 .. ctx_b + j      (Eq. 3 block)
// Split-KV ("flash-decoding"): one CTA per (request, head, 64-key page); each CTA
// stages its K and V page in shared memory (all 16-byte loads of the page issued
// before the first store, so a page costs one memory round trip), computes the
// G x 64 score block, a page-local max / sum (log2 domain) and the partial
// P.V, and writes (m, l, o) partials.  The last CTA of a (request, head)
// (atomic ticket) merges the pages in page order 0..n-1 — a fixed order, so the
// result does not depend on scheduling.  Memory bound (AI ~ G FLOP/B): CUDA
// cores, no tensor cores (K3).
#include <cfloat>

#include "common.cuh"
#include "kernels.h"

namespace sv {

constexpr int KPAGE = 64;     // keys per page (= page_tokens)
constexpr int GMAX = SV_MAX_GAMMA + 1;
constexpr int MAXCH = 64;     // pages per request (ctx <= 4096)

template <int D>
__global__ void __launch_bounds__(128) attn_kernel(const __grid_constant__ AttnArgs a) {
    constexpr int KST = D + 8;                 // padded K row (bf16) -> conflict-free 16 B reads
    constexpr int VPR = D / 8;                 // 16-byte vectors per row
    constexpr int NV = KPAGE * VPR / 128;      // vectors per thread for a full page
    __shared__ __align__(16) bf16 sK[KPAGE * KST];
    __shared__ __align__(16) bf16 sV[KPAGE * D];
    __shared__ __align__(16) float sQ[GMAX * D];
    __shared__ float sS[GMAX * KPAGE];
    __shared__ float sM[GMAX], sL[GMAX];
    __shared__ float sW[GMAX * MAXCH], sLc[GMAX * MAXCH];
    __shared__ int s_last;

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int bh = blockIdx.x, c = blockIdx.y;
    const int b = bh / a.n_heads, h = bh % a.n_heads;
    const int G = a.G;
    pdl_launch_dependents();   // the next GEMM may start streaming its weights now
    pdl_wait();
    const int ctx = a.ctx[b];
    const int T = ctx + G;
    const int nch_b = (T + KPAGE - 1) / KPAGE;
    if (c >= nch_b) return;
    const int k0 = c * KPAGE;
    const int nk = min(KPAGE, T - k0);
    const int blk = a.page_table[b * a.pt_stride + c];
    const size_t plane = (size_t)a.n_heads * a.page_tokens * D;
    const bf16* Kp = reinterpret_cast<const bf16*>(a.kv_pool) +
                     (((size_t)blk * a.n_layers + a.layer) * 2 + 0) * plane + (size_t)h * a.page_tokens * D;
    const bf16* Vp = Kp + plane;

    {
        uint4 kr[NV], vr[NV];
#pragma unroll
        for (int i = 0; i < NV; ++i) {
            const int v = tid + i * 128, key = v / VPR, part = v % VPR;
            if (key < nk) {
                kr[i] = __ldg(reinterpret_cast<const uint4*>(Kp + (size_t)key * D) + part);
                vr[i] = __ldg(reinterpret_cast<const uint4*>(Vp + (size_t)key * D) + part);
            }
        }
        constexpr int QN = (GMAX * D + 127) / 128;
        float qv[QN];
#pragma unroll
        for (int i = 0; i < QN; ++i) {
            const int e = tid + i * 128, j = e / D, dd = e % D;
            qv[i] = (j < G) ? a.q[(size_t)(b * G + j) * a.d_model + h * D + dd] : 0.f;
        }
#pragma unroll
        for (int i = 0; i < NV; ++i) {
            const int v = tid + i * 128, key = v / VPR, part = v % VPR;
            if (key < nk) {
                *reinterpret_cast<uint4*>(&sK[key * KST + part * 8]) = kr[i];
                *reinterpret_cast<uint4*>(&sV[key * D + part * 8]) = vr[i];
            }
        }
#pragma unroll
        for (int i = 0; i < QN; ++i) {
            const int e = tid + i * 128;
            if (e < GMAX * D) sQ[e] = qv[i] * a.scale_log2;
        }
    }
    __syncthreads();

    // scores (log2 domain), causal: key k0+key visible to row j iff k0+key <= ctx+j
    for (int p = tid; p < G * KPAGE; p += 128) {
        const int j = p / KPAGE, key = p % KPAGE;
        float s = -INFINITY;
        if (key < nk && k0 + key <= ctx + j) {
            const bf16* kr = &sK[key * KST];
            const float* qr = &sQ[j * D];
            float acc = 0.f;
#pragma unroll
            for (int dd = 0; dd < D; dd += 8) {
                const uint4 kv = *reinterpret_cast<const uint4*>(kr + dd);
                const __nv_bfloat162* k2 = reinterpret_cast<const __nv_bfloat162*>(&kv);
#pragma unroll
                for (int t = 0; t < 4; ++t) {
                    const float2 kf = __bfloat1622float2(k2[t]);
                    acc = fmaf(qr[dd + 2 * t], kf.x, acc);
                    acc = fmaf(qr[dd + 2 * t + 1], kf.y, acc);
                }
            }
            s = acc;
        }
        sS[j * KPAGE + key] = s;
    }
    __syncthreads();
    for (int j = warp; j < G; j += 4) {
        const float x0 = sS[j * KPAGE + lane], x1 = sS[j * KPAGE + lane + 32];
        float m = fmaxf(x0, x1);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
        const float e0 = (x0 == -INFINITY) ? 0.f : exp2f(x0 - m);
        const float e1 = (x1 == -INFINITY) ? 0.f : exp2f(x1 - m);
        const float l = warp_sum(e0 + e1);
        sS[j * KPAGE + lane] = e0;
        sS[j * KPAGE + lane + 32] = e1;
        if (lane == 0) {
            sM[j] = m;
            sL[j] = l;
        }
    }
    __syncthreads();
    constexpr int JG = 128 / D;                // query rows handled in parallel
    const int dd = tid % D, jg = tid / D;
    const size_t pbase = ((size_t)bh * a.nchunk + c) * G;
    for (int j = jg; j < G; j += JG) {
        float o = 0.f;
        for (int key = 0; key < nk; ++key) o = fmaf(sS[j * KPAGE + key], __bfloat162float(sV[key * D + dd]), o);
        a.part_o[(pbase + j) * D + dd] = o;
    }
    if (tid < G) {
        a.part_ml[(pbase + tid) * 2 + 0] = sM[tid];
        a.part_ml[(pbase + tid) * 2 + 1] = sL[tid];
    }
    __threadfence();
    __syncthreads();
    if (tid == 0) s_last = (atomicAdd(&a.counters[bh], 1) == nch_b - 1);
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    // merge the pages of (b, h) in page order: (1) all (m, l) pairs in parallel
    const size_t mbase = (size_t)bh * a.nchunk * G;
    for (int i = tid; i < nch_b * G; i += 128) {
        const int cc = i / G, j = i % G;
        const float2 ml = __ldcg(reinterpret_cast<const float2*>(&a.part_ml[(mbase + (size_t)cc * G + j) * 2]));
        sW[j * MAXCH + cc] = ml.x;
        sLc[j * MAXCH + cc] = ml.y;
    }
    __syncthreads();
    // (2) per row: M = max_c m_c, w_c = 2^(m_c - M), L = sum_c l_c w_c (page order)
    if (tid < G) {
        float M = -INFINITY;
        for (int cc = 0; cc < nch_b; ++cc) M = fmaxf(M, sW[tid * MAXCH + cc]);
        float L = 0.f;
        for (int cc = 0; cc < nch_b; ++cc) {
            const float m = sW[tid * MAXCH + cc];
            const float w = (m == -INFINITY) ? 0.f : exp2f(m - M);
            sW[tid * MAXCH + cc] = w;
            L = fmaf(sLc[tid * MAXCH + cc], w, L);
        }
        sL[tid] = L;
    }
    __syncthreads();
    // (3) O = sum_c w_c o_c / L, loads of 8 pages in flight
    for (int i = tid; i < G * D; i += 128) {
        const int j = i / D, e = i % D;
        const float* po = a.part_o + (mbase + j) * D + e;
        const size_t cs = (size_t)G * D;       // page stride in part_o
        float O = 0.f;
        int cc = 0;
        for (; cc + 8 <= nch_b; cc += 8) {
            float v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) v[u] = __ldcg(po + (cc + u) * cs);
#pragma unroll
            for (int u = 0; u < 8; ++u) O = fmaf(v[u], sW[j * MAXCH + cc + u], O);
        }
        for (; cc < nch_b; ++cc) O = fmaf(__ldcg(po + cc * cs), sW[j * MAXCH + cc], O);
        reinterpret_cast<bf16*>(a.out)[(size_t)(b * G + j) * a.d_model + h * D + e] = __float2bfloat16_rn(O / sL[j]);
    }
    if (tid == 0) a.counters[bh] = 0;
}

template <int D>
static cudaError_t launch_d(const AttnArgs& a, cudaStream_t st) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(a.B * a.n_heads, a.nchunk, 1);
    cfg.blockDim = dim3(128, 1, 1);
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = g_use_pdl ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, attn_kernel<D>, a);
}

cudaError_t attn_launch(const AttnArgs& a, cudaStream_t st) {
    if (a.page_tokens != KPAGE || a.G > GMAX || a.nchunk > MAXCH) return cudaErrorInvalidValue;
    switch (a.head_dim) {
        case 32: return launch_d<32>(a, st);
        case 64: return launch_d<64>(a, st);
        case 128: return launch_d<128>(a, st);
    }
    return cudaErrorInvalidValue;
}

}  // namespace sv
