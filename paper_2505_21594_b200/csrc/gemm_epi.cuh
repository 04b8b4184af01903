// gemm_epi.cuh — fused GEMM epilogues (shared by the small-tile GEMM kernel and the
// persistent large-tile kernel).  Input: an fp32 tile sOut[EPI_CHUNK tokens][128 rows] of
// out[m, n0 + r] = sum_k X[m, k] W[n0 + r, k] for tokens tok0 .. tok0+15, and
// rstd[m - m0] (RMSNorm folded: X = bf16(h * g), so out * rstd = RMSNorm(h) W^T).
//   EPI_QKV    : RoPE (rotate-half, cos/sin table) on q and k; q -> fp32 buffer,
//                k and v -> paged KV cache at pos[m]                  (Eq. 3)
//   EPI_RESID  : h += out (fp32 residual); u = bf16(h * g_next) (+ early-exit
//                copy with the final gain); sum(h^2) of the 128-column tile
//   EPI_SWIGLU : act = bf16(silu(gate * rstd) * (up * rstd)) (64-row interleave)
//   EPI_LOGITS : z = out * rstd (fp32 logits; LM head)
//   EPI_SILU   : act = bf16(silu(out * rstd)), row stride N (exit adapter W_dn)
// 128 threads, r = 0..127 (row of the tile); `sync` = barrier of those threads.
#pragma once
#include "common.cuh"
#include "kernels.h"

namespace sv {

constexpr int EPI_TM = 128;       // weight rows per tile
constexpr int EPI_CHUNK = 16;     // token columns per epilogue pass
constexpr int EPI_PAGE = 64;      // KV page size (sv_model_cfg.page_tokens is required to be 64)

// one step of a transposing warp butterfly: lanes with bit SH set keep the upper W of
// v[0..2W), the others the lower W, each adding the partner lane's copy of its half
template <int W, int SH>
__device__ __forceinline__ void butterfly_half(float* v, int lane) {
    const bool hi = (lane & SH) != 0;
#pragma unroll
    for (int i = 0; i < W; ++i) {
        const float keep = hi ? v[i + W] : v[i];
        const float send = hi ? v[i] : v[i + W];
        v[i] = keep + __shfl_xor_sync(0xffffffffu, send, SH);
    }
}

// Inputs of a single 16-token tile's epilogue that do not depend on the
// accumulator, loaded by every thread while the tensor core still runs (so the
// split-K reducer's tail has no load round trip of its own): the residual column
// and the norm gains (EPI_RESID), RoPE cos/sin of the thread's dimension (EPI_QKV).
struct EpiPre {
    float h[EPI_CHUNK];
    float g, g2;
    float2 cs[EPI_CHUNK];
};

// sPos / sBlk (optional, EPI_QKV): position and KV page of token m0 + t, staged in
// shared memory once per tile (epi_meta) instead of re-gathered per chunk.
template <int EPI, class Sync>
__device__ __forceinline__ void epi_apply(const GemmArgs& a, const float* sOut, const float* sR, float* sRed,
                                          int tok0, int m0, int n0, int nt, int r, Sync sync,
                                          const int* sPos = nullptr, const int* sBlk = nullptr,
                                          const EpiPre* pre = nullptr, bool dry = false) {
    // dry: the instruction-cache warm-up pass of gemm_kernel — the same code with
    // every global store predicated off
    constexpr int TM = EPI_TM;
    const int warp = r >> 5, lane = r & 31;
    if constexpr (EPI == EPI_QKV) {
        const int d = a.d_model, D = a.head_dim, half = D >> 1;
        const int sec = n0 / d;                // 0 = q, 1 = k, 2 = v
        const int col = (n0 % d) + r;
        const int hd = col / D, i = col % D;
        const int rp = r - i + ((i + half) % D);
        const int ih = i % half;
        // per-thread part of the KV offset (head, dim, K or V plane); per token:
        // (block, layer) plane base and slot (integer division by the runtime
        // sizes kept out of the token loop)
        const size_t plane = (size_t)a.n_heads * EPI_PAGE * D;
        const size_t kv_thread = (sec >= 1 ? (size_t)(sec - 1) * plane : 0) + (size_t)hd * EPI_PAGE * D + i;
        const size_t layer_planes = (size_t)a.layer * 2 * plane, block_stride = (size_t)a.n_layers * 2 * plane;
        const int nv = min(EPI_CHUNK, a.M - tok0);
        // every global load of the chunk is issued before the first store (the loop
        // below would otherwise serialise one memory round trip per token: the
        // compiler cannot move loads across the stores of the previous token)
        int pos[EPI_CHUNK], blk[EPI_CHUNK];
        float2 cs[EPI_CHUNK];
        if (sPos) {
#pragma unroll
            for (int j = 0; j < EPI_CHUNK; ++j) {
                pos[j] = (j < nv) ? sPos[tok0 - m0 + j] : 0;
                blk[j] = (j < nv) ? sBlk[tok0 - m0 + j] : 0;
            }
        } else {
#pragma unroll
            for (int j = 0; j < EPI_CHUNK; ++j) pos[j] = (j < nv) ? a.meta.pos[tok0 + j] : 0;
        }
        if (sec >= 1 && !sPos) {
            int req[EPI_CHUNK];
#pragma unroll
            for (int j = 0; j < EPI_CHUNK; ++j) req[j] = (j < nv) ? a.meta.row_req[tok0 + j] : 0;
#pragma unroll
            for (int j = 0; j < EPI_CHUNK; ++j)
                blk[j] = (j < nv) ? a.meta.page_table[req[j] * a.meta.pt_stride + pos[j] / EPI_PAGE] : 0;
        }
        if (sec < 2) {
#pragma unroll
            for (int j = 0; j < EPI_CHUNK; ++j)
                cs[j] = pre ? pre->cs[j]
                            : ((j < nv) ? reinterpret_cast<const float2*>(a.rope_cs)[(size_t)pos[j] * half + ih]
                                        : make_float2(1.f, 0.f));
        }
#pragma unroll
        for (int j = 0; j < EPI_CHUNK; ++j) {
            if (j >= nv) continue;
            const int tok = tok0 + j;
            const float rs = sR[tok - m0];
            float v = sOut[j * TM + r] * rs;
            if (sec < 2) {
                const float vp = sOut[j * TM + rp] * rs;
                v = (i < half) ? (v * cs[j].x - vp * cs[j].y) : (v * cs[j].x + vp * cs[j].y);
            }
            if (dry) {
            } else if (sec == 0) {
                a.qbuf[(size_t)tok * d + col] = v;
            } else {
                const int slot = pos[j] & (EPI_PAGE - 1);
                const size_t off = (size_t)blk[j] * block_stride + layer_planes + kv_thread + (size_t)slot * D;
                reinterpret_cast<bf16*>(a.kv_pool)[off] = __float2bfloat16_rn(v);
            }
        }
    } else if constexpr (EPI == EPI_RESID) {
        const int d = a.d_model;
        const float g = pre ? pre->g : __bfloat162float(reinterpret_cast<const bf16*>(a.g_out)[n0 + r]);
        const float g2 = pre ? pre->g2
                             : (a.u_out2 ? __bfloat162float(reinterpret_cast<const bf16*>(a.g_out2)[n0 + r]) : 0.f);
        const int nv = min(EPI_CHUNK, a.M - tok0);
        float hv[EPI_CHUNK];
#pragma unroll
        for (int j = 0; j < EPI_CHUNK; ++j)          // all residual loads in flight first
            hv[j] = pre ? pre->h[j] : ((j < nv) ? __ldcg(&a.h[(size_t)(tok0 + j) * d + n0 + r]) : 0.f);
#pragma unroll
        for (int j = 0; j < EPI_CHUNK; ++j) {
            if (j < nv) hv[j] += sOut[j * TM + r];
#ifdef SV_EXP_NO_RESID_STORES
            if (j < nv && !dry && a.M < 0) {
#else
            if (j < nv && !dry) {
#endif
                const size_t idx = (size_t)(tok0 + j) * d + n0 + r;
                a.h[idx] = hv[j];
                reinterpret_cast<bf16*>(a.u_out)[idx] = __float2bfloat16_rn(hv[j] * g);
                if (a.h_out2) a.h_out2[idx] = hv[j];
                if (a.u_out2) reinterpret_cast<bf16*>(a.u_out2)[idx] = __float2bfloat16_rn(hv[j] * g2);
            }
        }
        {   // sum of h^2 over the warp's 32 rows for all 16 tokens at once: a transposing
            // butterfly (8 + 4 + 2 + 1 + 1 independent shuffles instead of 16 x 5
            // dependent ones); lane pairs (2t, 2t+1) end with token t's sum
            float v[EPI_CHUNK];
#pragma unroll
            for (int j = 0; j < EPI_CHUNK; ++j) v[j] = hv[j] * hv[j];
            butterfly_half<8, 16>(v, lane);
            butterfly_half<4, 8>(v, lane);
            butterfly_half<2, 4>(v, lane);
            butterfly_half<1, 2>(v, lane);
            v[0] += __shfl_xor_sync(0xffffffffu, v[0], 1);
            const int t = ((lane >> 4) & 1) * 8 + ((lane >> 3) & 1) * 4 + ((lane >> 2) & 1) * 2 + ((lane >> 1) & 1);
            if ((lane & 1) == 0) sRed[warp * EPI_CHUNK + t] = v[0];
        }
        sync();
        if (r < EPI_CHUNK && tok0 + r < a.M && !dry) {
            const float s = (sRed[0 * EPI_CHUNK + r] + sRed[1 * EPI_CHUNK + r]) +
                            (sRed[2 * EPI_CHUNK + r] + sRed[3 * EPI_CHUNK + r]);
            a.ssq_out[(size_t)nt * a.MP + tok0 + r] = s;
        }
    } else if constexpr (EPI == EPI_SWIGLU) {
        const int rr = r & 63, jh = r >> 6;
        for (int j = jh * (EPI_CHUNK / 2); j < (jh + 1) * (EPI_CHUNK / 2); ++j) {
            const int tok = tok0 + j;
            if (tok >= a.M) break;
            const float rs = sR[tok - m0];
            const float g = sOut[j * TM + rr] * rs;
            const float u = sOut[j * TM + 64 + rr] * rs;
            const float y = g / (1.0f + expf(-g)) * u;
            if (!dry) reinterpret_cast<bf16*>(a.act)[(size_t)tok * a.d_ff + nt * 64 + rr] = __float2bfloat16_rn(y);
        }
    } else if constexpr (EPI == EPI_SILU) {
        for (int j = 0; j < EPI_CHUNK; ++j) {
            const int tok = tok0 + j;
            if (tok >= a.M) break;
            const float x = sOut[j * TM + r] * sR[tok - m0];
            if (!dry) reinterpret_cast<bf16*>(a.act)[(size_t)tok * a.N + n0 + r] = __float2bfloat16_rn(x / (1.0f + expf(-x)));
        }
    } else {  // EPI_LOGITS
        for (int j = 0; j < EPI_CHUNK; ++j) {
            const int tok = tok0 + j;
            if (tok >= a.M) break;
            if (!dry) a.logits[(size_t)tok * a.N + n0 + r] = sOut[j * TM + r] * sR[tok - m0];
        }
    }
}

// rstd[t] = 1/sqrt(sum_k ssq_in[k][m0+t] / d + eps), loads 8 tiles in flight,
// summed in tile order (deterministic); 1 when the GEMM has no folded norm.
__device__ __forceinline__ void epi_rstd(const GemmArgs& a, float* sR, int m0, int tn, int r, int nthreads) {
    for (int t = r; t < tn; t += nthreads) {
        const int tok = m0 + t;
        float rs = 1.0f;
        if (a.ssq_in && tok < a.M) {
            float s = 0.f;
            int k = 0;
            for (; k + 8 <= a.ssq_tiles; k += 8) {
                float v[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) v[u] = __ldcg(&a.ssq_in[(size_t)(k + u) * a.MP + tok]);
#pragma unroll
                for (int u = 0; u < 8; ++u) s += v[u];
            }
            for (; k < a.ssq_tiles; ++k) s += __ldcg(&a.ssq_in[(size_t)k * a.MP + tok]);
            rs = 1.0f / sqrtf(s * a.inv_d + a.eps);
        }
        sR[t] = rs;
    }
}

// position and KV page of tokens m0 .. m0+tn-1 (EPI_QKV metadata, see epi_apply)
__device__ __forceinline__ void epi_meta(const GemmArgs& a, int* sPos, int* sBlk, int m0, int tn, int r,
                                         int nthreads) {
    for (int t = r; t < tn; t += nthreads) {
        const int tok = m0 + t;
        int p = 0, b = 0;
        if (tok < a.M) {
            p = a.meta.pos[tok];
            b = a.meta.page_table[a.meta.row_req[tok] * a.meta.pt_stride + p / EPI_PAGE];
        }
        sPos[t] = p;
        sBlk[t] = b;
    }
}

}  // namespace sv
