// attn_dev.cuh — device body of K3 (gamma-query causal attention over one
// 64-key page of the paged bf16 KV cache, plus the in-order page merge by the
// last finisher), used by attn.cu (head_dim != 128).
//
//   a_j = softmax(q_j K^T / sqrt(Dh)) V   over keys 0 .. ctx_b + j      (Eq. 3)
#pragma once
#include <cfloat>

#include "common.cuh"
#include "kernels.h"

namespace sv {

constexpr int KPAGE = 64;     // keys per page (= page_tokens)
constexpr int GMAX = SV_MAX_GAMMA + 1;
constexpr int MAXCH = 64;     // pages per request (ctx <= 4096)

template <int D>
struct AttnSmem {
    static constexpr int KST = D + 8;          // padded K row -> conflict-free 16 B reads
    __align__(16) bf16 sK[KPAGE * KST];
    __align__(16) bf16 sV[KPAGE * D];
    __align__(16) float sQ[GMAX * D];
    float sS[GMAX * KPAGE];
    float sM[GMAX], sL[GMAX];
    float sW[GMAX * MAXCH], sLc[GMAX * MAXCH];
    int s_last;
};

// One (request b, head h, page c) unit with 128 threads (tid 0..127).  Returns
// true in all threads of the unit that merged (b, h) (the last page finisher).
template <int D, class Sync>
__device__ bool attn_page_body(const AttnArgs& a, int bh, int c, int tid, AttnSmem<D>& S, Sync sync) {
    constexpr int KST = AttnSmem<D>::KST;
    constexpr int VPR = D / 8;                 // 16-byte vectors per row
    constexpr int NV = KPAGE * VPR / 128;      // vectors per thread for a full page
    const int warp = tid >> 5, lane = tid & 31;
    const int b = bh / a.n_heads, h = bh % a.n_heads;
    const int G = a.G;
    const int ctx = a.ctx[b];                          // both loads issued together
    const int blk = a.page_table[b * a.pt_stride + c];  // (in bounds; unused if c is past the end)
    const int Gb = a.g_rows ? a.g_rows[b] : G;         // valid query rows (prefill blocks)
    const int T = ctx + Gb;
    const int nch_b = (T + KPAGE - 1) / KPAGE;
    if (c >= nch_b) return false;
    const int k0 = c * KPAGE;
    const int nk = min(KPAGE, T - k0);
    const size_t plane = (size_t)a.n_heads * a.page_tokens * D;
    const bf16* Kp = reinterpret_cast<const bf16*>(a.kv_pool) +
                     (((size_t)blk * a.n_layers + a.layer) * 2 + 0) * plane + (size_t)h * a.page_tokens * D;
    const bf16* Vp = Kp + plane;

    {   // all loads of the page in flight before the first store (one round trip)
        uint4 kr[NV], vr[NV];
#pragma unroll
        for (int i = 0; i < NV; ++i) {
            const int v = tid + i * 128, key = v / VPR, part = v % VPR;
            if (key < nk) {
                kr[i] = __ldcg(reinterpret_cast<const uint4*>(Kp + (size_t)key * D) + part);
                vr[i] = __ldcg(reinterpret_cast<const uint4*>(Vp + (size_t)key * D) + part);
            }
        }
        constexpr int QN = (GMAX * D + 127) / 128;
        float qv[QN];
#pragma unroll
        for (int i = 0; i < QN; ++i) {
            const int e = tid + i * 128, j = e / D, dd = e % D;
            qv[i] = (j < G) ? __ldcg(&a.q[(size_t)(b * G + j) * a.d_model + h * D + dd]) : 0.f;
        }
#pragma unroll
        for (int i = 0; i < NV; ++i) {
            const int v = tid + i * 128, key = v / VPR, part = v % VPR;
            if (key < nk) {
                *reinterpret_cast<uint4*>(&S.sK[key * KST + part * 8]) = kr[i];
                *reinterpret_cast<uint4*>(&S.sV[key * D + part * 8]) = vr[i];
            }
        }
#pragma unroll
        for (int i = 0; i < QN; ++i) {
            const int e = tid + i * 128;
            if (e < GMAX * D) S.sQ[e] = qv[i] * a.scale_log2;
        }
    }
    sync();

    // scores (log2 domain), causal: key k0+key visible to row j iff k0+key <= ctx+j
    for (int p = tid; p < G * KPAGE; p += 128) {
        const int j = p / KPAGE, key = p % KPAGE;
        float s = -INFINITY;
        if (key < nk && k0 + key <= ctx + j) {
            const bf16* kr = &S.sK[key * KST];
            const float* qr = &S.sQ[j * D];
            float acc[4] = {0.f, 0.f, 0.f, 0.f};       // 4 independent chains (ILP)
#pragma unroll
            for (int dd = 0; dd < D; dd += 8) {
                const uint4 kv = *reinterpret_cast<const uint4*>(kr + dd);
                const float4 q0 = *reinterpret_cast<const float4*>(qr + dd);
                const float4 q1 = *reinterpret_cast<const float4*>(qr + dd + 4);
                const __nv_bfloat162* k2 = reinterpret_cast<const __nv_bfloat162*>(&kv);
                const float2 f0 = __bfloat1622float2(k2[0]), f1 = __bfloat1622float2(k2[1]);
                const float2 f2 = __bfloat1622float2(k2[2]), f3 = __bfloat1622float2(k2[3]);
                acc[0] = fmaf(q0.x, f0.x, fmaf(q0.y, f0.y, acc[0]));
                acc[1] = fmaf(q0.z, f1.x, fmaf(q0.w, f1.y, acc[1]));
                acc[2] = fmaf(q1.x, f2.x, fmaf(q1.y, f2.y, acc[2]));
                acc[3] = fmaf(q1.z, f3.x, fmaf(q1.w, f3.y, acc[3]));
            }
            s = (acc[0] + acc[1]) + (acc[2] + acc[3]);
        }
        S.sS[j * KPAGE + key] = s;
    }
    sync();
    for (int j = warp; j < G; j += 4) {
        const float x0 = S.sS[j * KPAGE + lane], x1 = S.sS[j * KPAGE + lane + 32];
        float m = fmaxf(x0, x1);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
        const float e0 = (x0 == -INFINITY) ? 0.f : exp2f(x0 - m);
        const float e1 = (x1 == -INFINITY) ? 0.f : exp2f(x1 - m);
        const float l = warp_sum(e0 + e1);
        S.sS[j * KPAGE + lane] = e0;
        S.sS[j * KPAGE + lane + 32] = e1;
        if (lane == 0) {
            S.sM[j] = m;
            S.sL[j] = l;
        }
    }
    sync();
    constexpr int JG = 128 / D;                // query rows handled in parallel
    const int dd = tid % D, jg = tid / D;
    const size_t pbase = ((size_t)bh * a.nchunk + c) * G;
    for (int j = jg; j < G; j += JG) {
        float o[4] = {0.f, 0.f, 0.f, 0.f};
        int key = 0;
        for (; key + 4 <= nk; key += 4) {
#pragma unroll
            for (int u = 0; u < 4; ++u)
                o[u] = fmaf(S.sS[j * KPAGE + key + u], __bfloat162float(S.sV[(key + u) * D + dd]), o[u]);
        }
        for (; key < nk; ++key) o[0] = fmaf(S.sS[j * KPAGE + key], __bfloat162float(S.sV[key * D + dd]), o[0]);
        a.part_o[(pbase + j) * D + dd] = (o[0] + o[1]) + (o[2] + o[3]);
    }
    if (tid < G) {
        a.part_ml[(pbase + tid) * 2 + 0] = S.sM[tid];
        a.part_ml[(pbase + tid) * 2 + 1] = S.sL[tid];
    }
    sync();
    if (tid == 0) S.s_last = (atomic_add_acq_rel(&a.counters[bh], 1) == nch_b - 1);
    sync();
    if (!S.s_last) return false;
    // merge the pages of (b, h) in page order: (1) all (m, l) pairs in parallel
    const size_t mbase = (size_t)bh * a.nchunk * G;
    for (int i = tid; i < nch_b * G; i += 128) {
        const int cc = i / G, j = i % G;
        const float2 ml = __ldcg(reinterpret_cast<const float2*>(&a.part_ml[(mbase + (size_t)cc * G + j) * 2]));
        S.sW[j * MAXCH + cc] = ml.x;
        S.sLc[j * MAXCH + cc] = ml.y;
    }
    sync();
    // (2) per row: M = max_c m_c, w_c = 2^(m_c - M), L = sum_c l_c w_c (page order)
    if (tid < G) {
        float M = -INFINITY;
        for (int cc = 0; cc < nch_b; ++cc) M = fmaxf(M, S.sW[tid * MAXCH + cc]);
        float L = 0.f;
        for (int cc = 0; cc < nch_b; ++cc) {
            const float m = S.sW[tid * MAXCH + cc];
            const float w = (m == -INFINITY) ? 0.f : exp2f(m - M);
            S.sW[tid * MAXCH + cc] = w;
            L = fmaf(S.sLc[tid * MAXCH + cc], w, L);
        }
        S.sL[tid] = L;
    }
    sync();
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
            for (int u = 0; u < 8; ++u) O = fmaf(v[u], S.sW[j * MAXCH + cc + u], O);
        }
        for (; cc < nch_b; ++cc) O = fmaf(__ldcg(po + cc * cs), S.sW[j * MAXCH + cc], O);
        reinterpret_cast<bf16*>(a.out)[(size_t)(b * G + j) * a.d_model + h * D + e] = __float2bfloat16_rn(O / S.sL[j]);
    }
    if (tid == 0) a.counters[bh] = 0;
    return true;
}

}  // namespace sv
