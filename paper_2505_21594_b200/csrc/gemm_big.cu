// gemm_big.cu — K1 for large token blocks (TILE_N = 128 / 256, i.e. batched
// verify steps where M = B*(gamma+1) > 64 and the projections turn compute-bound):
// a persistent tcgen05 GEMM, one CTA per SM, with the epilogue of tile i running
// on dedicated warps while the tensor core already accumulates tile i+1 into the
// second TMEM buffer.
//
//   warps 0-7  epilogue in two groups of four (group g = warps 4g..4g+3, TMEM lane
//              quarter = warp % 4) taking alternate 16-token chunks of the tile:
//              TMEM -> smem -> fused op (gemm_epi.cuh); per-tile metadata (rstd,
//              positions, KV pages) is staged in smem before the accumulator is
//              ready; the tile is released through tmem_empty[buf]
//   warp 8     TMA producer: continuous STAGES-deep ring over all (tile, k-block)
//              of this CTA (weights evict-first, activations evict-last)
//   warp 9     tcgen05.mma issuer (M = 128 weight rows, N = TILE_N tokens)
// Tiles are ordered n-major, m-minor (tile = n*MT + m) and dealt round-robin, so
// the m-tiles that share one weight tile run on neighbouring CTAs at the same time
// and the weight tile is read from HBM once (L2 serves the others).
#include "common.cuh"
#include "gemm_epi.cuh"
#include "kernels.h"

namespace sv {

constexpr int GB_BK = 64;
constexpr int GB_TM = 128;
constexpr int GB_A = GB_TM * GB_BK * 2;

template <int TN>
struct GBCfg {
    static constexpr int B_STAGE = TN * GB_BK * 2;
    static constexpr int STAGE = GB_A + B_STAGE;
    // two groups x (sOut [16][128] f32 + sRed [4][16]) + sR, sPos, sBlk [TN]
    static constexpr int EPI = 2 * (EPI_CHUNK * GB_TM * 4 + 4 * EPI_CHUNK * 4) + 3 * TN * 4;
    static constexpr int AUX = 512;
    static constexpr int RAW = (227 * 1024 - 1024 - EPI - AUX) / STAGE;
    static constexpr int STAGES = RAW > 8 ? 8 : RAW;
    static constexpr int SMEM = 1024 + STAGES * STAGE + EPI + AUX;
    static constexpr int TCOLS = 2 * TN <= 256 ? 256 : 512;   // two accumulators (alloc: power of two)
    static_assert(STAGES >= 3 && TCOLS <= 512, "config");
};

constexpr int GB_EPI_WARPS = 8, GB_THREADS = (GB_EPI_WARPS + 2) * 32;

struct EpiBar {   // one epilogue group (named barrier 1 + group)
    int id;
    __device__ void operator()() const { asm volatile("bar.sync %0, 128;" ::"r"(id) : "memory"); }
};
__device__ __forceinline__ void epi_all_bar() { asm volatile("bar.sync 3, 256;" ::: "memory"); }

template <int TN, int EPI>
__global__ void __launch_bounds__(GB_THREADS, 1)
    gemm_big_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                    const __grid_constant__ GemmArgs a) {
    using C = GBCfg<TN>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sA = smem;
    uint8_t* sB = smem + C::STAGES * GB_A;
    float* sOut0 = reinterpret_cast<float*>(smem + C::STAGES * C::STAGE);  // 2 x [EPI_CHUNK][128]
    float* sRed0 = sOut0 + 2 * EPI_CHUNK * GB_TM;                          // 2 x [4][EPI_CHUNK]
    float* sR = sRed0 + 2 * 4 * EPI_CHUNK;                                 // [TN]
    int* sPos = reinterpret_cast<int*>(sR + TN);                           // [TN]
    int* sBlk = sPos + TN;                                                 // [TN]
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::STAGES * C::STAGE + C::EPI);
    uint64_t* empty = full + C::STAGES;
    uint64_t* tfull = empty + C::STAGES;
    uint64_t* tempty = tfull + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int NT = a.N / GB_TM, MT = (a.M + TN - 1) / TN, T = NT * MT;
    const int KB = a.K / GB_BK;
    ktrace_mark(a.ktrace, a.ktrace_id, 0);
    if (warp == 8 && lane == 0) {
        tma_prefetch_desc(&tmA);
        tma_prefetch_desc(&tmB);
        for (int s = 0; s < C::STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&tfull[b], 1);
            mbar_init(&tempty[b], 1);
        }
        fence_mbar_init();
    }
    if (warp == 9) tmem_alloc(tmem_slot, C::TCOLS);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    pdl_launch_dependents();

    if (warp == 8) {
        if (lane == 0) {   // ------------------------------------------ producer
            const uint64_t pol_w = policy_evict_first(), pol_x = policy_evict_last();
            const uint32_t stage_tx = GB_A + (a.b_box ? a.b_box : TN) * GB_BK * 2;   // GemmArgs::b_box
            int it = 0;
            bool waited = false;
            for (int t = blockIdx.x; t < T; t += gridDim.x) {
                const int n0 = (t / MT) * GB_TM, m0 = (t % MT) * TN;
                for (int kb = 0; kb < KB; ++kb, ++it) {
                    const int s = it % C::STAGES;
                    if (it >= C::STAGES) mbar_wait(&empty[s], ((it / C::STAGES) - 1) & 1);
                    mbar_arrive_expect_tx(&full[s], stage_tx);
                    tma_load_2d(&tmA, sA + s * GB_A, &full[s], kb * GB_BK, n0, pol_w);
                    if (!waited) {     // weights above never depend on the previous kernel
                        pdl_wait();
                        waited = true;
                    }
                    tma_load_2d(&tmB, sB + s * C::B_STAGE, &full[s], kb * GB_BK, m0 + a.b_row0, pol_x);
                }
            }
        }
    } else if (warp == 9) {
        if (lane == 0) {   // ------------------------------------------ MMA issuer
            constexpr uint32_t idesc = umma_idesc_bf16(GB_TM, TN);
            int it = 0, seg = 0;
            for (int t = blockIdx.x; t < T; t += gridDim.x, ++seg) {
                const int buf = seg & 1;
                if (seg >= 2) mbar_wait(&tempty[buf], ((seg >> 1) - 1) & 1);
                tc_fence_after();
                const uint32_t dt = tmem + buf * TN;
                for (int kb = 0; kb < KB; ++kb, ++it) {
                    const int s = it % C::STAGES;
                    mbar_wait(&full[s], (it / C::STAGES) & 1);
                    tc_fence_after();
                    const uint64_t ad = umma_sdesc_sw128(smem_u32(sA + s * GB_A));
                    const uint64_t bd = umma_sdesc_sw128(smem_u32(sB + s * C::B_STAGE));
#pragma unroll
                    for (int k = 0; k < GB_BK / 16; ++k)
                        umma_bf16(dt, ad + 2 * k, bd + 2 * k, idesc, (kb | k) ? 1u : 0u);
                    umma_commit(&empty[s]);
                }
                umma_commit(&tfull[buf]);
            }
        }
    } else {               // ------------------------------------------ epilogue warps 0-7
        const int grp = warp >> 2, tid = threadIdx.x;     // tid 0..255
        const EpiBar bar{1 + grp};
        const int r = tid & 127;                           // tile row (TMEM lane)
        float* sOut = sOut0 + grp * EPI_CHUNK * GB_TM;
        float* sRed = sRed0 + grp * 4 * EPI_CHUNK;
        pdl_wait();                                        // epilogue inputs come from earlier kernels
        int seg = 0;
        for (int t = blockIdx.x; t < T; t += gridDim.x, ++seg) {
            const int buf = seg & 1;
            const int nt = t / MT, n0 = nt * GB_TM, m0 = (t % MT) * TN;
            epi_rstd(a, sR, m0, TN, tid, 256);             // overlaps the tile's MMA
            if constexpr (EPI == EPI_QKV) epi_meta(a, sPos, sBlk, m0, TN, tid, 256);
            epi_all_bar();
            mbar_wait(&tfull[buf], (seg >> 1) & 1);
            tc_fence_after();
            const uint32_t tb = tmem + (static_cast<uint32_t>((warp & 3) * 32) << 16) + buf * TN;
            for (int c0 = grp * EPI_CHUNK; c0 < TN; c0 += 2 * EPI_CHUNK) {
                if (m0 + c0 >= a.M) break;                 // uniform over the group
                uint32_t v[16];
                tmem_ld_32x32b_x16(tb + c0, v);
                tmem_ld_wait();
                bar();
#pragma unroll
                for (int j = 0; j < 16; ++j) sOut[j * GB_TM + r] = __uint_as_float(v[j]);
                bar();
                epi_apply<EPI>(a, sOut, sR, sRed, m0 + c0, m0, n0, nt, r, bar, sPos, sBlk);
            }
            tc_fence_before();
            epi_all_bar();                                 // also guards sR / sPos reuse
            if (tid == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&tempty[buf])) : "memory");
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 9) tmem_dealloc(tmem, C::TCOLS);
    ktrace_mark(a.ktrace, a.ktrace_id, 1);
}

template <int TN, int EPI>
static cudaError_t big_t(const CUtensorMap& tmA, const CUtensorMap& tmB, const GemmArgs& a, cudaStream_t st) {
    using C = GBCfg<TN>;
    static bool attr = false;
    static int sms = 0;
    if (!attr) {
        cudaError_t e = cudaFuncSetAttribute(gemm_big_kernel<TN, EPI>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             C::SMEM);
        if (e != cudaSuccess) return e;
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        attr = true;
    }
    const int T = (a.N / GB_TM) * ((a.M + TN - 1) / TN);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(T < sms ? T : sms, 1, 1);
    cfg.blockDim = dim3(GB_THREADS, 1, 1);
    cfg.dynamicSmemBytes = C::SMEM;
    cfg.stream = st;
    cudaLaunchAttribute attr1[1];
    attr1[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr1[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr1;
    cfg.numAttrs = g_use_pdl ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, gemm_big_kernel<TN, EPI>, tmA, tmB, a);
}

template <int TN>
static cudaError_t big_epi(int epi, const CUtensorMap& tmA, const CUtensorMap& tmB, const GemmArgs& a,
                           cudaStream_t st) {
    switch (epi) {
        case EPI_QKV: return big_t<TN, EPI_QKV>(tmA, tmB, a, st);
        case EPI_RESID: return big_t<TN, EPI_RESID>(tmA, tmB, a, st);
        case EPI_SWIGLU: return big_t<TN, EPI_SWIGLU>(tmA, tmB, a, st);
        case EPI_LOGITS: return big_t<TN, EPI_LOGITS>(tmA, tmB, a, st);
        case EPI_SILU: return big_t<TN, EPI_SILU>(tmA, tmB, a, st);
    }
    return cudaErrorInvalidValue;
}

cudaError_t gemm_big_launch(int epi, int tile_n, const CUtensorMap& tmA, const CUtensorMap& tmB, const GemmArgs& a,
                            cudaStream_t st) {
    if (tile_n == 128) return big_epi<128>(epi, tmA, tmB, a, st);
    if (tile_n == 256) return big_epi<256>(epi, tmA, tmB, a, st);
    if (tile_n == 160) return big_epi<160>(epi, tmA, tmB, a, st);
    return cudaErrorInvalidValue;
}

}  // namespace sv
