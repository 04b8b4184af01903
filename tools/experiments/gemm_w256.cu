// EXPERIMENT (not built): batch-1 GEMM with the weights as the N = 256 tcgen05.mma operand and
// cluster split-K; measured slower end to end than gemm.cu (C2 3.64 vs 3.37 ms), see DESIGN.md section 11.
// gemm_w256.cu — K1 for small token blocks (M <= 16 rows: batch-1..3 verify
// steps): weights as the wide (N = 256) operand of tcgen05.mma, split-K over a
// thread-block cluster with a distributed-shared-memory reduction.
//
//   out[m, n] = sum_k X[m, k] * W[n, k]      (X: activations [M, K], W: weights [N, K])
//
// Why this shape (tools/stream_bw.cu, one CTA per SM, B200):
// * tcgen05.mma issue cost is per instruction; with the weights as a 128-row A
//   operand and N = 16 tokens each instruction carries 4 KB of weights and the
//   tensor pipe capped weight streaming at 3.9-5.0 TB/s.  As the B operand with
//   N = 256 (M = 128 activation rows) each instruction carries 8 KB and the GEMM
//   streams at the TMA-only rate.
// * only BR = 8 (M <= 8) or 16 activation rows are loaded per 64-wide K block.
//   For BR = 8 the activation descriptor's 8-row-group stride is 0, so all 16
//   groups of the 128-row A operand alias the same 8 rows: every 32-lane quarter
//   of the accumulator holds tokens 0..7 and the 4 epilogue warps each drain 64
//   columns.  For BR = 16 rows >= 16 of D are garbage (never read).
// * shared memory <= 113 KB (3 x 32 KB weight slots): two CTAs per SM, so the
//   next launch's CTAs are resident during this one (programmatic dependent
//   launch) and stream their first weight slots before griddepcontrol.wait.
// * split-K: the S splits of a 256-row tile form one cluster (1 x 1 x S); every
//   split drains its fp32 partial to its own shared memory; the rank that owns a
//   128-row half (rank = half % S) sums the S partials over DSMEM in rank order
//   (deterministic, independent of M) and runs the fused epilogue on it.
#include <cudaTypedefs.h>

#include <algorithm>

#include "common.cuh"
#include "gemm_epi.cuh"
#include "kernels.h"

namespace sv {

constexpr int W2_BK = 64;                    // K elements per ring slot (128 B rows)
constexpr int W2_TW = 256;                   // weight rows per tile (UMMA N)
constexpr int W2_W = W2_TW * W2_BK * 2;      // 32 KB of weights per slot
constexpr int W2_THREADS = 192;
constexpr int W2_TCOLS = 256;
constexpr int W2_SMEM_LIMIT = 113 * 1024;    // two CTAs (+1 KB reserved each) per 228 KB SM

template <int BR>
struct W2Cfg {
    static constexpr int STAGES = BR == 8 ? 3 : 2;
    static constexpr int X = BR * 128;                                 // activation bytes per slot
    static constexpr int W_OFF = 0;                                    // [STAGES][32 KB] weights
    static constexpr int X_OFF = STAGES * W2_W;                        // [STAGES][X]
    static constexpr int T_OFF = X_OFF + STAGES * X;                  // (BR=16: the MMA's reads of A rows >= 16 land in sT)
    static constexpr int T_BYTES = 2 * BR * 128 * 4;                   // sT [2 halves][BR tok][128] fp32
    static constexpr int R_OFF = T_OFF + T_BYTES;                      // sR [16]
    static constexpr int RED_OFF = R_OFF + 64 * 4;                     // sRed [4][EPI_CHUNK]
    static constexpr int BAR_OFF = RED_OFF + 4 * EPI_CHUNK * 4;
    static constexpr int END = BAR_OFF + (2 * STAGES + 1) * 8 + 16;
    static constexpr int SMEM = 1024 + END;
    static_assert(SMEM <= W2_SMEM_LIMIT, "two grids must fit one SM");
};

struct W2NamedSync {
    __device__ void operator()() const { asm volatile("bar.sync 1, 128;" ::: "memory"); }
};

template <int BR>
__device__ __forceinline__ uint64_t w2_xdesc(uint32_t saddr) {
    uint64_t d = umma_sdesc_sw128(saddr);
    if (BR == 8) d &= ~(static_cast<uint64_t>(0x3FFF) << 32);   // 8-row-group stride 0
    return d;
}

// 32 lanes x 64 consecutive 32-bit TMEM columns
__device__ __forceinline__ void tmem_ld_x64(uint32_t taddr, uint32_t (&r)[64]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x64.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,"
        "%32,%33,%34,%35,%36,%37,%38,%39,%40,%41,%42,%43,%44,%45,%46,%47,"
        "%48,%49,%50,%51,%52,%53,%54,%55,%56,%57,%58,%59,%60,%61,%62,%63}, [%64];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
          "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
          "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31]),
          "=r"(r[32]), "=r"(r[33]), "=r"(r[34]), "=r"(r[35]), "=r"(r[36]), "=r"(r[37]), "=r"(r[38]), "=r"(r[39]),
          "=r"(r[40]), "=r"(r[41]), "=r"(r[42]), "=r"(r[43]), "=r"(r[44]), "=r"(r[45]), "=r"(r[46]), "=r"(r[47]),
          "=r"(r[48]), "=r"(r[49]), "=r"(r[50]), "=r"(r[51]), "=r"(r[52]), "=r"(r[53]), "=r"(r[54]), "=r"(r[55]),
          "=r"(r[56]), "=r"(r[57]), "=r"(r[58]), "=r"(r[59]), "=r"(r[60]), "=r"(r[61]), "=r"(r[62]), "=r"(r[63])
        : "r"(taddr));
}

template <int BR, int EPI>
__global__ void __launch_bounds__(W2_THREADS, 1)
    gemm_w256_kernel(const __grid_constant__ CUtensorMap tmW, const __grid_constant__ CUtensorMap tmX,
                     const __grid_constant__ GemmArgs a) {
    using C = W2Cfg<BR>;
    constexpr int STAGES = C::STAGES;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sW = smem + C::W_OFF;
    uint8_t* sX = smem + C::X_OFF;
    float* sT = reinterpret_cast<float*>(smem + C::T_OFF);
    float* sR = reinterpret_cast<float*>(smem + C::R_OFF);
    float* sRed = reinterpret_cast<float*>(smem + C::RED_OFF);
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::BAR_OFF);
    uint64_t* empty = full + STAGES;
    uint64_t* done = empty + STAGES;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done + 1);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    ktrace_mark(a.ktrace, a.ktrace_id, 0);
    const int t = blockIdx.x, split = blockIdx.z, S = gridDim.z;
    const int KB = a.K / W2_BK;
    const int kb0 = (int)((long long)KB * split / S), kb1 = (int)((long long)KB * (split + 1) / S);
    const int n = kb1 - kb0;
    const int n0 = t * W2_TW;
    constexpr uint32_t STAGE_TX = W2_W + BR * 128;

    if (warp == 0 && lane == 0) {
        tma_prefetch_desc(&tmW);
        tma_prefetch_desc(&tmX);
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        mbar_init(done, 1);
        fence_mbar_init();
    }
    if (warp == 1) tmem_alloc(tmem_slot, W2_TCOLS);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    pdl_launch_dependents();

    if (warp == 0) {
        if (lane == 0) {
            // ------------------------------------------------ TMA producer
            const uint64_t pol_w = policy_evict_first(), pol_x = policy_evict_last();
            const int pre = n < STAGES ? n : STAGES;
            for (int i = 0; i < pre; ++i) {          // weights never depend on the previous launch
                mbar_arrive_expect_tx(&full[i], STAGE_TX);
                tma_load_2d(&tmW, sW + i * W2_W, &full[i], (kb0 + i) * W2_BK, n0, pol_w);
            }
            pdl_wait();
            for (int i = 0; i < pre; ++i) tma_load_2d(&tmX, sX + i * C::X, &full[i], (kb0 + i) * W2_BK, 0, pol_x);
            for (int i = pre; i < n; ++i) {
                const int s = i % STAGES;
                mbar_wait(&empty[s], ((i / STAGES) - 1) & 1);
                mbar_arrive_expect_tx(&full[s], STAGE_TX);
                tma_load_2d(&tmW, sW + s * W2_W, &full[s], (kb0 + i) * W2_BK, n0, pol_w);
                tma_load_2d(&tmX, sX + s * C::X, &full[s], (kb0 + i) * W2_BK, 0, pol_x);
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            // ------------------------------------------------ MMA issuer
            constexpr uint32_t idesc = umma_idesc_bf16(128, W2_TW);   // D row r = TMEM lane r
            for (int i = 0; i < n; ++i) {
                const int s = i % STAGES;
                mbar_wait(&full[s], (i / STAGES) & 1);
                tc_fence_after();
                const uint64_t xd = w2_xdesc<BR>(smem_u32(sX + s * C::X));
                const uint64_t wd = umma_sdesc_sw128(smem_u32(sW + s * W2_W));
#pragma unroll
                for (int k = 0; k < W2_BK / 16; ++k)   // +32 B per K=16 step inside the swizzle atom
                    umma_bf16(tmem, xd + 2 * k, wd + 2 * k, idesc, (i == 0 && k == 0) ? 0u : 1u);
                umma_commit(&empty[s]);
            }
            umma_commit(done);
        }
    } else {
        // ------------------------------------- epilogue part 1: TMEM -> sT (128 threads)
        const int wt = threadIdx.x - 64;
        W2NamedSync sync;
        pdl_wait();                                     // rstd inputs come from earlier launches
        epi_rstd(a, sR, 0, 16, wt, 128);
        mbar_wait(done, 0);
        tc_fence_after();
        const int M = a.M;
        if constexpr (BR == 8) {                        // every lane quarter holds tokens 0..7
            const int q = warp & 3;
            uint32_t r[64];
            tmem_ld_x64(tmem + (static_cast<uint32_t>(q * 32) << 16) + q * 64, r);
            tmem_ld_wait();
            if (lane < M) {
                float* dst = sT + ((q >> 1) * BR + lane) * 128 + (q & 1) * 64;
#pragma unroll
                for (int j = 0; j < 64; ++j) dst[j] = __uint_as_float(r[j]);
            }
        } else if ((warp & 3) == 0) {                   // lanes 0..31 = rows 0..31
#pragma unroll 1
            for (int c0 = 0; c0 < W2_TW; c0 += 64) {
                uint32_t r[64];
                tmem_ld_x64(tmem + c0, r);
                tmem_ld_wait();
                if (lane < M) {
                    float* dst = sT + ((c0 >> 7) * BR + lane) * 128 + (c0 & 127);
#pragma unroll
                    for (int j = 0; j < 64; ++j) dst[j] = __uint_as_float(r[j]);
                }
            }
        }
        (void)sync;
    }
    tc_fence_before();
    __syncthreads();
    if (S > 1) cluster_sync_all();                      // every split's partial is in its sT
    if (warp >= 2) {
        // --------------------- epilogue part 2: reduce + fused op per 128-row half
        const int wt = threadIdx.x - 64;
        W2NamedSync sync;
        const int M = a.M;
#pragma unroll 1
        for (int h = 0; h < 2; ++h) {
            if (h % S != split || n0 + h * 128 >= a.N) continue;
            float* half = sT + h * BR * 128;
            if (S > 1) {
                for (int e = wt; e < M * 128; e += 128) {   // rank order 0..S-1 (deterministic)
                    float v[16];
#pragma unroll
                    for (int q = 0; q < 16; ++q) v[q] = (q < S) ? ld_dsmem_f32(&half[e], q) : 0.f;
                    float acc = 0.f;
#pragma unroll
                    for (int q = 0; q < 16; ++q)
                        if (q < S) acc += v[q];
                    half[e] = acc;
                }
                sync();
            }
            epi_apply<EPI>(a, half, sR, sRed, 0, 0, n0 + h * 128, 2 * t + h, wt, sync);
            sync();
        }
    }
    if (S > 1) cluster_sync_all();                      // partials stay alive until read
    if (warp == 1) tmem_dealloc(tmem, W2_TCOLS);
    ktrace_mark(a.ktrace, a.ktrace_id, 1);
}

// ------------------------------------------------------------------ host side
int gemm_w256_splits(int N, int K, int num_sms, int max_splits) {
    const int NT = (N + W2_TW - 1) / W2_TW, KB = K / W2_BK;
    int s = 1;
    while (s < max_splits && NT * s * 2 <= 2 * num_sms && KB / (2 * s) >= 2) s *= 2;
    return s;
}

template <int BR, int EPI>
static cudaError_t w2_launch_t(const CUtensorMap& tmW, const CUtensorMap& tmX, const GemmArgs& a, int splits,
                               cudaStream_t st) {
    static bool attr_done = false;
    if (!attr_done) {
        cudaError_t e = cudaFuncSetAttribute(gemm_w256_kernel<BR, EPI>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             W2Cfg<BR>::SMEM);
        if (e != cudaSuccess) return e;
        e = cudaFuncSetAttribute(gemm_w256_kernel<BR, EPI>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        if (e != cudaSuccess) return e;
        attr_done = true;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((a.N + W2_TW - 1) / W2_TW, 1, splits);
    cfg.blockDim = dim3(W2_THREADS, 1, 1);
    cfg.dynamicSmemBytes = W2Cfg<BR>::SMEM;
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    int na = 0;
    attr[na].id = cudaLaunchAttributeClusterDimension;
    attr[na].val.clusterDim.x = 1;
    attr[na].val.clusterDim.y = 1;
    attr[na].val.clusterDim.z = splits;
    ++na;
    if (g_use_pdl) {
        attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[na].val.programmaticStreamSerializationAllowed = 1;
        ++na;
    }
    cfg.attrs = attr;
    cfg.numAttrs = na;
    return cudaLaunchKernelEx(&cfg, gemm_w256_kernel<BR, EPI>, tmW, tmX, a);
}

template <int BR>
static cudaError_t w2_launch_epi(int epi, const CUtensorMap& tmW, const CUtensorMap& tmX, const GemmArgs& a,
                                 int splits, cudaStream_t st) {
    switch (epi) {
        case EPI_QKV: return w2_launch_t<BR, EPI_QKV>(tmW, tmX, a, splits, st);
        case EPI_RESID: return w2_launch_t<BR, EPI_RESID>(tmW, tmX, a, splits, st);
        case EPI_SWIGLU: return w2_launch_t<BR, EPI_SWIGLU>(tmW, tmX, a, splits, st);
        case EPI_LOGITS: return w2_launch_t<BR, EPI_LOGITS>(tmW, tmX, a, splits, st);
    }
    return cudaErrorInvalidValue;
}

// tmW: weights, box 64 x 256 rows; tmX: activations, box 64 x box_rows (8 if M <= 8,
// else 16); splits from gemm_w256_splits (<= 16).
cudaError_t gemm_w256_launch(int epi, int box_rows, const CUtensorMap& tmW, const CUtensorMap& tmX, const GemmArgs& a,
                             int splits, cudaStream_t st) {
    if (a.M > 16 || a.M > box_rows || a.N % 128 || a.K % W2_BK || splits < 1 || splits > 16 ||
        a.K / W2_BK < splits)
        return cudaErrorInvalidValue;
    if (box_rows == 8) return w2_launch_epi<8>(epi, tmW, tmX, a, splits, st);
    if (box_rows == 16) return w2_launch_epi<16>(epi, tmW, tmX, a, splits, st);
    return cudaErrorInvalidValue;
}

}  // namespace sv
