// attn2.cu — K3 v2: gamma-query causal attention over the paged bf16 KV cache,
// built for the HBM roofline at any batch / context:
//
//   a_j = softmax(q_j K^T / sqrt(Dh)) V   over keys 0 .. ctx_b + j      (Eq. 3)
//
// * one CTA per (request b, head h, split r); split r owns a contiguous run of
//   64-key pages and streams them through an NST-deep shared-memory ring with
//   1D TMA bulk copies (a (layer, head) page of K or V is one contiguous
//   64 x Dh bf16 block in the head-major KV layout: 16 KB at Dh = 128);
// * per page: scores with a key-rotated chunk order (conflict-free shared
//   memory reads of the unpadded rows), online softmax in the log2 domain, P.V
//   accumulated in registers (one head dimension per thread);
// * the S splits of a (b, h) form one thread-block cluster; split partials
//   (m, l, o) are merged by rank 0 through distributed shared memory in rank
//   order (fixed order -> deterministic), no global partials / atomics.
// Memory bound (AI ~ G FLOP/B): CUDA cores.
#include <cfloat>

#include "common.cuh"
#include "kernels.h"

namespace sv {

constexpr int A2_PAGE = 64;
constexpr int A2_GMAX = SV_MAX_GAMMA + 1;
constexpr int A2_THREADS = 128;

template <int D>
struct A2Cfg {
    static constexpr int NST = D == 128 ? 3 : 4;             // pages in flight
    static constexpr int PAGE_BYTES = A2_PAGE * D * 2;       // one K (or V) page
    static constexpr int RING = NST * 2 * PAGE_BYTES;
    static constexpr int SMEM = 1024 + RING + A2_GMAX * D * 4 /*q*/ + 2 * A2_GMAX * A2_PAGE * 4 /*partial s*/ +
                                A2_GMAX * A2_PAGE * 4 /*p*/ + A2_GMAX * D * 4 /*o*/ + 4 * A2_GMAX * 4 + 256;
};

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ float ld_dsmem_f32(const void* local_ptr, uint32_t rank) {
    uint32_t raddr;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(raddr) : "r"(smem_u32(local_ptr)), "r"(rank));
    float v;
    asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(v) : "r"(raddr) : "memory");
    return v;
}

template <int D>
__global__ void __launch_bounds__(A2_THREADS) attn2_kernel(const __grid_constant__ AttnArgs a) {
    using C = A2Cfg<D>;
    constexpr int DH = D / 2;          // dims per half (two threads per key)
    constexpr int NC = DH / 8;         // 16-byte chunks per half row
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    bf16* ring = reinterpret_cast<bf16*>(smem);                                   // [NST][K|V][64][D]
    float* sQ = reinterpret_cast<float*>(smem + C::RING);                         // [G][D] (scaled, log2)
    float* sPart = sQ + A2_GMAX * D;                                              // [2][G][64]
    float* sP = sPart + 2 * A2_GMAX * A2_PAGE;                                    // [G][64]
    float* sO = sP + A2_GMAX * A2_PAGE;                                           // [G][D] (merge)
    float* sM = sO + A2_GMAX * D;                                                 // running max [G]
    float* sL = sM + A2_GMAX;                                                     // running sum [G]
    float* sAl = sL + A2_GMAX;                                                    // rescale [G]
    float* sRm = sAl + A2_GMAX;                                                   // [2 warps][G]
    uint64_t* full = reinterpret_cast<uint64_t*>(sRm + 2 * A2_GMAX + 2);          // 8-aligned below
    full = reinterpret_cast<uint64_t*>((reinterpret_cast<uintptr_t>(full) + 7) & ~uintptr_t(7));
    __shared__ int sBlk[64];

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int S = gridDim.x, r = blockIdx.x;                 // split (cluster rank when S > 1)
    const int bh = blockIdx.y;
    const int b = bh / a.n_heads, h = bh % a.n_heads;
    const int G = a.G;
    pdl_launch_dependents();
    if (tid == 0) {
        for (int s = 0; s < C::NST; ++s) mbar_init(&full[s], 1);
        fence_mbar_init();
    }
    pdl_wait();
    const int ctx = a.ctx[b];
    const int T = ctx + G;
    const int npg = (T + A2_PAGE - 1) / A2_PAGE;
    const int p0 = (int)((long long)npg * r / S), p1 = (int)((long long)npg * (r + 1) / S);
    const int np = p1 - p0;
    for (int i = tid; i < np; i += A2_THREADS) sBlk[i] = a.page_table[b * a.pt_stride + p0 + i];
    for (int i = tid; i < G * D; i += A2_THREADS) {
        const int j = i / D, d = i % D;
        sQ[i] = a.q[(size_t)(b * G + j) * a.d_model + h * D + d] * a.scale_log2;
    }
    if (tid < G) {
        sM[tid] = -INFINITY;
        sL[tid] = 0.f;
    }
    __syncthreads();
    const size_t plane = (size_t)a.n_heads * a.page_tokens * D;
    auto page_src = [&](int i, int kv) {
        return reinterpret_cast<const bf16*>(a.kv_pool) + (((size_t)sBlk[i] * a.n_layers + a.layer) * 2 + kv) * plane +
               (size_t)h * a.page_tokens * D;
    };
    if (tid == 0)
        for (int i = 0; i < np && i < C::NST; ++i) {
            mbar_arrive_expect_tx(&full[i], 2 * C::PAGE_BYTES);
            bulk_g2s(ring + (size_t)(i * 2 + 0) * A2_PAGE * D, page_src(i, 0), C::PAGE_BYTES, &full[i]);
            bulk_g2s(ring + (size_t)(i * 2 + 1) * A2_PAGE * D, page_src(i, 1), C::PAGE_BYTES, &full[i]);
        }

    const int key = tid & 63, half = tid >> 6;
    float o[A2_GMAX];                                         // O[j][d = tid] (D == 128) accumulators
#pragma unroll
    for (int j = 0; j < A2_GMAX; ++j) o[j] = 0.f;

    for (int i = 0; i < np; ++i) {
        const int s = i % C::NST;
        mbar_wait(&full[s], (i / C::NST) & 1);
        const bf16* Ks = ring + (size_t)(s * 2 + 0) * A2_PAGE * D;
        const bf16* Vs = ring + (size_t)(s * 2 + 1) * A2_PAGE * D;
        const int kabs0 = (p0 + i) * A2_PAGE;
        // ---- partial scores over this thread's half of the head dimension
        float acc[A2_GMAX];
#pragma unroll
        for (int j = 0; j < A2_GMAX; ++j) acc[j] = 0.f;
        const bf16* krow = Ks + (size_t)key * D + half * DH;
#pragma unroll
        for (int c = 0; c < NC; ++c) {
            const int ch = (c + key) % NC;                    // rotated: conflict-free across the warp
            const uint4 kv = *reinterpret_cast<const uint4*>(krow + ch * 8);
            const __nv_bfloat162* k2 = reinterpret_cast<const __nv_bfloat162*>(&kv);
            const float2 f0 = __bfloat1622float2(k2[0]), f1 = __bfloat1622float2(k2[1]);
            const float2 f2 = __bfloat1622float2(k2[2]), f3 = __bfloat1622float2(k2[3]);
#pragma unroll
            for (int j = 0; j < A2_GMAX; ++j) {
                if (j < G) {
                    const float* qr = sQ + j * D + half * DH + ch * 8;
                    const float4 q0 = *reinterpret_cast<const float4*>(qr);
                    const float4 q1 = *reinterpret_cast<const float4*>(qr + 4);
                    acc[j] = fmaf(q0.x, f0.x, fmaf(q0.y, f0.y, fmaf(q0.z, f1.x, fmaf(q0.w, f1.y,
                             fmaf(q1.x, f2.x, fmaf(q1.y, f2.y, fmaf(q1.z, f3.x, fmaf(q1.w, f3.y, acc[j]))))))));
                }
            }
        }
#pragma unroll
        for (int j = 0; j < A2_GMAX; ++j)
            if (j < G) sPart[(half * A2_GMAX + j) * A2_PAGE + key] = acc[j];
        __syncthreads();
        // ---- full scores, causal mask, page max per row (threads 0..63 = keys)
        if (tid < A2_PAGE) {
#pragma unroll
            for (int j = 0; j < A2_GMAX; ++j) {
                if (j < G) {
                    const int kabs = kabs0 + key;
                    float sc = sPart[j * A2_PAGE + key] + sPart[(A2_GMAX + j) * A2_PAGE + key];
                    if (kabs > ctx + j) sc = -INFINITY;
                    sP[j * A2_PAGE + key] = sc;
                    float m = sc;
#pragma unroll
                    for (int off = 16; off > 0; off >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, off));
                    if (lane == 0) sRm[warp * A2_GMAX + j] = m;
                }
            }
        }
        __syncthreads();
        if (tid < G) {
            const float mold = sM[tid];
            const float mnew = fmaxf(mold, fmaxf(sRm[tid], sRm[A2_GMAX + tid]));
            sAl[tid] = (mold == -INFINITY) ? 0.f : exp2f(mold - mnew);
            sM[tid] = mnew;
        }
        __syncthreads();
        // ---- p = 2^(s - m); page row sums
        if (tid < A2_PAGE) {
#pragma unroll
            for (int j = 0; j < A2_GMAX; ++j) {
                if (j < G) {
                    const float sc = sP[j * A2_PAGE + key];
                    const float m = sM[j];
                    const float p = (sc == -INFINITY || m == -INFINITY) ? 0.f : exp2f(sc - m);
                    sP[j * A2_PAGE + key] = p;
                    const float l = warp_sum(p);
                    if (lane == 0) sRm[warp * A2_GMAX + j] = l;
                }
            }
        }
        __syncthreads();
        if (tid < G) sL[tid] = sL[tid] * sAl[tid] + (sRm[tid] + sRm[A2_GMAX + tid]);
        // ---- O = O * alpha + P V  (thread = head dimension; D < 128: rows split)
        {
            constexpr int JG = A2_THREADS / D;
            const int d = tid % D, jg = tid / D;
#pragma unroll
            for (int j = 0; j < A2_GMAX; ++j) {
                if (j < G && (j % JG) == jg) {
                    float acc2[4] = {o[j] * sAl[j], 0.f, 0.f, 0.f};
#pragma unroll 4
                    for (int k = 0; k < A2_PAGE; k += 4) {
#pragma unroll
                        for (int u = 0; u < 4; ++u)
                            acc2[u] = fmaf(sP[j * A2_PAGE + k + u], __bfloat162float(Vs[(size_t)(k + u) * D + d]), acc2[u]);
                    }
                    o[j] = (acc2[0] + acc2[1]) + (acc2[2] + acc2[3]);
                }
            }
        }
        __syncthreads();                                       // page slot free
        if (tid == 0 && i + C::NST < np) {
            const int nx = i + C::NST;
            mbar_arrive_expect_tx(&full[s], 2 * C::PAGE_BYTES);
            bulk_g2s(ring + (size_t)(s * 2 + 0) * A2_PAGE * D, page_src(nx, 0), C::PAGE_BYTES, &full[s]);
            bulk_g2s(ring + (size_t)(s * 2 + 1) * A2_PAGE * D, page_src(nx, 1), C::PAGE_BYTES, &full[s]);
        }
    }

    // ---- output: single split writes directly; else merge the cluster in rank order
    constexpr int JG = A2_THREADS / D;
    const int d = tid % D, jg = tid / D;
    if (S == 1) {
#pragma unroll
        for (int j = 0; j < A2_GMAX; ++j)
            if (j < G && (j % JG) == jg)
                reinterpret_cast<bf16*>(a.out)[(size_t)(b * G + j) * a.d_model + h * D + d] =
                    __float2bfloat16_rn(o[j] / sL[j]);
        return;
    }
#pragma unroll
    for (int j = 0; j < A2_GMAX; ++j)
        if (j < G && (j % JG) == jg) sO[j * D + d] = o[j];
    cluster_sync_all();                                       // partials visible cluster-wide
    if (cluster_rank() == 0) {
        for (int j = jg; j < G; j += JG) {
            float mq[8], lq[8], oq[8];                        // all remote loads in flight
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                mq[q] = q < S ? ld_dsmem_f32(&sM[j], q) : -INFINITY;
                lq[q] = q < S ? ld_dsmem_f32(&sL[j], q) : 0.f;
                oq[q] = q < S ? ld_dsmem_f32(&sO[j * D + d], q) : 0.f;
            }
            float M = -INFINITY;
#pragma unroll
            for (int q = 0; q < 8; ++q) M = fmaxf(M, mq[q]);
            float L = 0.f, O = 0.f;
#pragma unroll
            for (int q = 0; q < 8; ++q) {                     // rank order
                if (mq[q] == -INFINITY) continue;
                const float w = exp2f(mq[q] - M);
                L = fmaf(lq[q], w, L);
                O = fmaf(oq[q], w, O);
            }
            reinterpret_cast<bf16*>(a.out)[(size_t)(b * G + j) * a.d_model + h * D + d] = __float2bfloat16_rn(O / L);
        }
    }
    cluster_sync_all();                                       // keep partials alive until merged
}

int attn2_splits(int B, int H, int max_pages, int num_sms) {
    const int units = B * H;
    int s = (2 * num_sms + units - 1) / units;                 // aim for ~2 CTAs per SM
    if (s > 8) s = 8;                                          // portable cluster size
    if (s > max_pages) s = max_pages;
    if (s < 1) s = 1;
    return s;
}

template <int D>
static cudaError_t launch2(const AttnArgs& a, int splits, cudaStream_t st) {
    using C = A2Cfg<D>;
    static bool attr = false;
    if (!attr) {
        cudaError_t e = cudaFuncSetAttribute(attn2_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
        if (e != cudaSuccess) return e;
        attr = true;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(splits, a.B * a.n_heads, 1);
    cfg.blockDim = dim3(A2_THREADS, 1, 1);
    cfg.dynamicSmemBytes = C::SMEM;
    cfg.stream = st;
    cudaLaunchAttribute attr2[2];
    int na = 0;
    attr2[na].id = cudaLaunchAttributeClusterDimension;
    attr2[na].val.clusterDim.x = splits;
    attr2[na].val.clusterDim.y = 1;
    attr2[na].val.clusterDim.z = 1;
    ++na;
    if (g_use_pdl) {
        attr2[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr2[na].val.programmaticStreamSerializationAllowed = 1;
        ++na;
    }
    cfg.attrs = attr2;
    cfg.numAttrs = na;
    return cudaLaunchKernelEx(&cfg, attn2_kernel<D>, a);
}

cudaError_t attn2_launch(const AttnArgs& a, int splits, cudaStream_t st) {
    if (a.page_tokens != A2_PAGE || a.G > A2_GMAX || splits < 1 || splits > 8) return cudaErrorInvalidValue;
    switch (a.head_dim) {
        case 32: return launch2<32>(a, splits, st);
        case 64: return launch2<64>(a, splits, st);
        case 128: return launch2<128>(a, splits, st);
    }
    return cudaErrorInvalidValue;
}

}  // namespace sv
