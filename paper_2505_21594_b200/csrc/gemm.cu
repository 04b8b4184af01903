// gemm.cu — K1: bf16 weight-streaming GEMM on 5th-generation tensor cores.
//
//   out[m, n] = sum_k X[m, k] * W[n, k]      (X: activations [M, K], W: weights [N, K])
//
// computed "swap-AB": the weight tile is the MMA A operand (M_mma = 128 weight
// rows = 128 output features) and the token block is the B operand
// (N_mma = TILE_N tokens, 16..256), so a batch-1 verify step (gamma+1 = 5 query
// rows) still fills the 128-row MMA and every weight byte is read exactly once.
//
// Per CTA: one 128-row weight tile x one TILE_N token tile x one K split.
//   warp 0 / lane 0 : TMA producer (weights evict-first, activations evict-last),
//                     STAGES-deep mbarrier ring of 64-wide K blocks (128 B rows,
//                     128B swizzle); weight loads are issued BEFORE
//                     griddepcontrol.wait so they overlap the previous kernel.
//   warp 1 / lane 0 : tcgen05.mma.cta_group::1.kind::f16 issuer, fp32 accumulator
//                     in TMEM (TILE_N columns), tcgen05.commit frees smem slots.
//   all 4 warps     : epilogue, TMEM -> registers (tcgen05.ld 32x32b) -> smem tile
//                     -> fused op, or -> split-K partials; the last CTA of a tile
//                     (atomic ticket) reduces the partials in split order 0..S-1,
//                     so results are deterministic and independent of the other
//                     token columns (row invariance used by the rollback pin).
//
// Fused epilogues:
//   EPI_QKV    : y = acc * rstd[m]; RoPE (rotate-half, table cos/sin) on q and k;
//                q -> fp32 buffer, k and v -> paged KV cache at pos[m]   (Eq. 3)
//   EPI_RESID  : h += acc (fp32 residual); u = bf16(h * g_next) for the next
//                RMSNorm; sum(h^2) per 128-column tile -> ssq partials
//   EPI_SWIGLU : act = bf16(silu(gate * rstd) * (up * rstd))
//   EPI_LOGITS : z = acc * rstd[m] (fp32 logits, LM head)
// RMSNorm is folded: the GEMM consumes u = bf16(h * g) and multiplies its
// accumulator by rstd[m] = 1/sqrt(sum(h^2)/d + eps) from the producer's partials.
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "common.cuh"
#include "gemm_epi.cuh"
#include "kernels.h"

namespace sv {

constexpr int BK = 64;                      // K elements per stage (one 128 B swizzle row)
constexpr int TM = 128;                     // weight rows per tile (UMMA M)
constexpr int A_STAGE = TM * BK * 2;        // 16 KB
// split-K partners a reducer polls in one batch (splits <= SK_MAXP + 1); 9 splits
// for O / down at batch 1 (288 CTAs) measured slower than 8 (O 10.0 vs 8.3 us)
#ifndef SV_SK_MAXP
#define SV_SK_MAXP 7
#endif
constexpr int SK_MAXP = SV_SK_MAXP;
#ifndef SV_GEMM_MAX_STAGES
#define SV_GEMM_MAX_STAGES 8
#endif
#ifndef SV_GEMM_CTAS_PER_SM
#define SV_GEMM_CTAS_PER_SM 2
#endif

template <int TN, int MAXST = SV_GEMM_MAX_STAGES>
struct GemmCfg {
    static constexpr int B_STAGE = TN * BK * 2;
    static constexpr int STAGE = A_STAGE + B_STAGE;
    // small token tiles: SV_GEMM_CTAS_PER_SM CTAs per SM (two grids co-resident
    // under programmatic dependent launch), else 1 CTA per SM
    static constexpr int AUX = 2304;        // barriers, tmem slot, rstd[TN], reductions, token metadata
    static constexpr int BUDGET =
        (TN <= 64 ? (228 * 1024) / SV_GEMM_CTAS_PER_SM - 1024 : 225 * 1024) - 1024 - AUX;
    static constexpr int STAGES_RAW = BUDGET / STAGE;
    static constexpr int STAGES = STAGES_RAW > MAXST ? MAXST : STAGES_RAW;
    static constexpr int TMEM_COLS = TN <= 32 ? 32 : TN <= 64 ? 64 : TN <= 128 ? 128 : 256;   // alloc: power of two
    static constexpr int SMEM = 1024 + STAGES * STAGE + AUX;
    static_assert(STAGES >= 2, "pipeline too shallow");
    static_assert(EPI_CHUNK * TM * 4 <= STAGES * STAGE, "epilogue tile must fit the ring");
    static_assert((TN + EPI_CHUNK) * TM * 4 <= STAGES * STAGE, "split partial + epilogue tile");
};

// barrier of the tail: all 128 threads (barrier 0) in the real pass, warps 2-3
// (barrier 1, 64 threads) in the warm-up pass
struct EpiBar {
    int id, cnt;
    __device__ void operator()() const { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(cnt) : "memory"); }
};

template <int TN, int EPI, int MAXST = SV_GEMM_MAX_STAGES>
__global__ void __launch_bounds__(128, 1)
    gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                const __grid_constant__ GemmArgs a) {
    using C = GemmCfg<TN, MAXST>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sA = smem;
    uint8_t* sB = smem + C::STAGES * A_STAGE;
    uint8_t* aux = smem + C::STAGES * C::STAGE;
    uint64_t* full = reinterpret_cast<uint64_t*>(aux);
    uint64_t* empty = full + C::STAGES;
    uint64_t* done = empty + C::STAGES;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done + 1);
    float* sR = reinterpret_cast<float*>(aux + 256);          // [TN]
    float* sRed = sR + 256;                                   // [4][EPI_CHUNK]
    float* sRedDry = reinterpret_cast<float*>(aux + 2048);    // [4][EPI_CHUNK] (warm-up pass)
    int* sPos = reinterpret_cast<int*>(aux + 1536);           // [TN <= 64] (EPI_QKV token metadata)
    int* sBlk = sPos + 64;
    float* sOut = reinterpret_cast<float*>(smem);             // [EPI_CHUNK][128], reuses the ring

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nt = blockIdx.x, mt = blockIdx.y, split = blockIdx.z;
    ktrace_mark(a.ktrace, a.ktrace_id, 0);
    unsigned long long* gtr = threadIdx.x == 0 ? a.gtrace : nullptr;
    gphase_mark(gtr, a.ktrace_id, 0);
    const int NT = gridDim.x, MT = gridDim.y;
    const int n0 = nt * TM, m0 = mt * TN;
    const int KB = a.K / BK;
    const int kb0 = (int)((long long)KB * split / a.splits);
    const int kb1 = (int)((long long)KB * (split + 1) / a.splits);
    const int nk = kb1 - kb0;

    if (warp == 0 && lane == 0) {
        tma_prefetch_desc(&tmA);
        tma_prefetch_desc(&tmB);
        for (int s = 0; s < C::STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        mbar_init(done, 1);
        fence_mbar_init();
    }
    if (warp == 2) tmem_alloc(tmem_slot, C::TMEM_COLS);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    // let the next kernel's CTAs become resident now: they set up and start
    // streaming their weights while this grid runs (their griddepcontrol.wait
    // still waits for this grid's completion before touching activations)
    pdl_launch_dependents();

    if (warp == 0 && lane == 0) {
        // ---------------- TMA producer
        const uint64_t pol_w = policy_evict_first(), pol_x = policy_evict_last();
        // the activation box holds only the tile's real token rows (GemmArgs::b_box);
        // the MMA's other B rows read stale smem into output columns never stored
        const uint32_t stage_tx = A_STAGE + (a.b_box ? a.b_box : TN) * BK * 2;
        const int pre = nk < C::STAGES ? nk : C::STAGES;
        for (int i = 0; i < pre; ++i) {   // weights do not depend on the previous kernel
            mbar_arrive_expect_tx(&full[i], stage_tx);
            tma_load_2d(&tmA, sA + i * A_STAGE, &full[i], (kb0 + i) * BK, n0, pol_w);
        }
        pdl_wait();
        gphase_mark(gtr, a.ktrace_id, 1);
        for (int i = 0; i < pre; ++i) tma_load_2d(&tmB, sB + i * C::B_STAGE, &full[i], (kb0 + i) * BK, m0 + a.b_row0, pol_x);
        for (int i = pre; i < nk; ++i) {
            const int s = i % C::STAGES;
            mbar_wait(&empty[s], ((i / C::STAGES) - 1) & 1);
            mbar_arrive_expect_tx(&full[s], stage_tx);
            tma_load_2d(&tmA, sA + s * A_STAGE, &full[s], (kb0 + i) * BK, n0, pol_w);
            tma_load_2d(&tmB, sB + s * C::B_STAGE, &full[s], (kb0 + i) * BK, m0 + a.b_row0, pol_x);
        }
    } else if (warp == 1 && lane == 0) {
        // ---------------- MMA issuer (single thread)
        constexpr uint32_t idesc = umma_idesc_bf16(TM, TN);
        for (int i = 0; i < nk; ++i) {
            const int s = i % C::STAGES;
            mbar_wait(&full[s], (i / C::STAGES) & 1);
            tc_fence_after();
            const uint64_t ad = umma_sdesc_sw128(smem_u32(sA + s * A_STAGE));
            const uint64_t bd = umma_sdesc_sw128(smem_u32(sB + s * C::B_STAGE));
#pragma unroll
            for (int k = 0; k < BK / 16; ++k)   // +32 B per K=16 step inside the swizzle atom
                umma_bf16(tmem, ad + 2 * k, bd + 2 * k, idesc, (i | k) ? 1u : 0u);
            umma_commit(&empty[s]);
        }
        umma_commit(done);
    }
    __syncwarp();

    // The tail below (TMEM -> partials / epilogue, split-K ticket and reduction)
    // runs once per CTA, so its instructions are cold in the SM's instruction cache
    // and it sits on the step's critical path.  Warps 2-3, idle until the
    // accumulator is ready, first run the very same code as a dry pass (pass 0:
    // every store and atomic predicated off, their own 64-thread barrier, before
    // griddepcontrol.wait), so the real pass (pass 1, all 128 threads) runs warm.
    constexpr bool kStageMeta = (EPI == EPI_QKV && TN <= 64);
    constexpr bool kPre = (EPI == EPI_RESID || EPI == EPI_QKV) && TN == 16;
    EpiPre pre;
    const int row = warp * 32 + lane;
    const uint32_t tbase = tmem + (static_cast<uint32_t>(warp * 32) << 16);
    const bool direct = (a.splits == 1);
    // tiles of more than one 16-token chunk reduce split-K through fp32 partials and one
    // release/acquire flag per (split, row); single-chunk tiles through tagged pairs
    constexpr bool kFlags = TN > EPI_CHUNK;
    const uint32_t tag = (a.meta.epoch ? (*a.meta.epoch << 10) : 0u) | (uint32_t)(a.ktrace_id & 1023);
    if (warp >= 2 && a.warm && TN <= 32 && kStageMeta)   // valid (zero) token metadata for the warm-up pass's loads
        for (int t = threadIdx.x - 64; t < TN; t += 64) sPos[t] = sBlk[t] = 0;
    for (int pass = (warp >= 2 && a.warm && TN <= 32) ? 0 : 1; pass < 2; ++pass) {
        const bool dry = pass == 0;
        const EpiBar bar{dry ? 1 : 0, dry ? 64 : 128};
        float* sRedP = dry ? sRedDry : sRed;
        if (dry && kStageMeta) bar();
        if (!dry) {
            pdl_wait();   // everything below reads data produced by the previous kernel
            gphase_mark(gtr, a.ktrace_id, 1);
            // warps 2-3 (idle during the mainloop) stage what the epilogue needs while the
            // tensor core still runs: rstd of the folded RMSNorm (fixed summation order) and,
            // for the QKV epilogue, each token's position and KV page
            if (warp >= 2) {
                epi_rstd(a, sR, m0, TN, threadIdx.x - 64, 64);
                if constexpr (kStageMeta) epi_meta(a, sPos, sBlk, m0, TN, threadIdx.x - 64, 64);
            }
            // single 16-token tile: every input of the epilogue that does not depend on the
            // accumulator is loaded before it is ready (EpiPre), so the tail — the split-K
            // reducer's in particular — has no load round trip of its own
            if constexpr (kPre && EPI == EPI_RESID) {
                const int r = threadIdx.x;
#pragma unroll
                for (int j = 0; j < 16; ++j)
                    pre.h[j] = (m0 + j < a.M) ? __ldcg(&a.h[(size_t)(m0 + j) * a.d_model + n0 + r]) : 0.f;
                pre.g = __bfloat162float(reinterpret_cast<const bf16*>(a.g_out)[n0 + r]);
                pre.g2 = a.u_out2 ? __bfloat162float(reinterpret_cast<const bf16*>(a.g_out2)[n0 + r]) : 0.f;
            }
            if constexpr (kPre && EPI == EPI_QKV) {
                const int D = a.head_dim, half = D >> 1, i = ((n0 % a.d_model) + (int)threadIdx.x) % D;
                const bool rot = n0 / a.d_model < 2;    // q and k sections
#pragma unroll
                for (int j = 0; j < 16; ++j)
                    pre.cs[j] = (rot && m0 + j < a.M)
                                    ? reinterpret_cast<const float2*>(a.rope_cs)[(size_t)a.meta.pos[m0 + j] * half + i % half]
                                    : make_float2(1.f, 0.f);
            }
            mbar_wait(done, 0);
            tc_fence_after();
            gphase_mark(gtr, a.ktrace_id, 2);
        }

        // split-K: every split but 0 stores its partial as (value, tag) pairs with single
        // 64-bit relaxed stores and is done; split 0 adds the others' pairs to its own
        // partial (TMEM) in split order 0..S-1 (deterministic), polling until they carry
        // this launch's tag (host step epoch, launch index): no fence, no ticket, one
        // round trip when the partials are already there.  One epilogue call site, so
        // the tail's code is small (it runs cold once per CTA).
        const bool writer = !direct && split != 0 && !dry;
        const size_t sstride = (size_t)NT * a.MP * TM;
        for (int c0 = 0; c0 < TN; c0 += EPI_CHUNK) {
            if (m0 + c0 >= a.M) break;                       // CTA-uniform
            const int nv = min(EPI_CHUNK, a.M - (m0 + c0));
            uint32_t r[16];
            if (!dry) {
                tmem_ld_32x32b_x16(tbase + c0, r);
                tmem_ld_wait();
            } else {
#pragma unroll
                for (int j = 0; j < 16; ++j) r[j] = 0u;
            }
            if (writer) {
                if constexpr (kFlags) {   // fp32 partial; the row's flag follows the last chunk
                    float* wsp = a.ws + (((size_t)split * NT + nt) * a.MP + m0 + c0) * TM + row;
#pragma unroll
                    for (int j = 0; j < 16; ++j)
                        if (j < nv) __stcg(&wsp[(size_t)j * TM], __uint_as_float(r[j]));
                } else {
                    uint64_t* wsp = reinterpret_cast<uint64_t*>(a.ws) + (((size_t)split * NT + nt) * a.MP + m0 + c0) * TM + row;
#pragma unroll
                    for (int j = 0; j < 16; ++j)
                        if (j < nv) st_relaxed_b64(&wsp[(size_t)j * TM], ((uint64_t)tag << 32) | r[j]);
                }
                continue;
            }
            // the chunk's fp32 tile goes through sOut[token][row]; each thread owns its
            // row's column, so the split-K accumulation below needs no barrier
            bar();                                           // sR visible / previous chunk consumed
            if (!dry)
#pragma unroll
                for (int j = 0; j < EPI_CHUNK; ++j)
                    sOut[j * TM + row] = direct ? __uint_as_float(r[j]) : 0.f + __uint_as_float(r[j]);
            if (!direct && kFlags) {
                // multi-chunk tile: one acquire of each writer's flag for this row (before
                // the first chunk), then every chunk's partial loads pipeline freely
                if (c0 == 0 && !dry)
                    for (int u = 1; u < a.splits; ++u) {
                        const uint32_t* f = a.sk_flags + (((size_t)u * NT + nt) * MT + mt) * TM + row;
                        for (uint32_t n = 0; ld_acquire_u32(f) != tag; ++n)
                            if (n > SV_SPIN_LIMIT) __trap();
                    }
                const float* base = a.ws + ((size_t)nt * a.MP + m0 + c0) * TM + row;
                float acc[EPI_CHUNK];
#pragma unroll
                for (int j = 0; j < EPI_CHUNK; ++j) acc[j] = 0.f + __uint_as_float(r[j]);
#pragma unroll
                for (int u = 1; u <= SK_MAXP; ++u)
                    if (u < a.splits) {
                        float v[EPI_CHUNK];
#pragma unroll
                        for (int j = 0; j < EPI_CHUNK; ++j) v[j] = j < nv ? __ldcg(base + u * sstride + j * TM) : 0.f;
#pragma unroll
                        for (int j = 0; j < EPI_CHUNK; ++j) acc[j] += v[j];
                    }
                if (!dry)
#pragma unroll
                    for (int j = 0; j < EPI_CHUNK; ++j) sOut[j * TM + row] = acc[j];
            } else if (!direct) {
                const uint64_t* base = reinterpret_cast<const uint64_t*>(a.ws) + ((size_t)nt * a.MP + m0 + c0) * TM + row;
#pragma unroll 1
                for (int g = 0; g * 8 < nv; ++g) {    // 8 tokens x 7 splits per round trip
                    uint64_t x[SK_MAXP][8];
                    bool ok;
                    uint32_t n = 0;
                    do {   // all pairs in flight; again (L2 hits) until every pair carries this launch's tag
                        ok = true;
#pragma unroll
                        for (int u = 0; u < SK_MAXP; ++u)
#pragma unroll
                            for (int j = 0; j < 8; ++j) {
                                const bool live = u + 1 < a.splits && g * 8 + j < nv;
                                x[u][j] = live ? ld_relaxed_b64(base + (u + 1) * sstride + (g * 8 + j) * TM)
                                               : ((uint64_t)tag << 32);
                            }
#pragma unroll
                        for (int u = 0; u < SK_MAXP; ++u)
#pragma unroll
                            for (int j = 0; j < 8; ++j) ok = ok && (uint32_t)(x[u][j] >> 32) == tag;
                        if (dry) break;
                        if (++n > SV_SPIN_LIMIT) __trap();
                    } while (!ok);
                    if (dry) continue;
#pragma unroll
                    for (int j = 0; j < 8; ++j) {
                        float v = sOut[(g * 8 + j) * TM + row];
#pragma unroll
                        for (int u = 0; u < SK_MAXP; ++u)
                            if (u + 1 < a.splits && g * 8 + j < nv) v += __uint_as_float((uint32_t)x[u][j]);
                        sOut[(g * 8 + j) * TM + row] = v;
                    }
                }
                if (!dry && c0 == 0) gphase_mark(gtr, a.ktrace_id, 7);
            }
            bar();
            if (!dry && c0 == 0) gphase_mark(gtr, a.ktrace_id, 8);
            epi_apply<EPI>(a, sOut, sR, sRedP, m0 + c0, m0, n0, nt, row, bar, kStageMeta ? sPos : nullptr,
                           kStageMeta ? sBlk : nullptr, kPre ? &pre : nullptr, dry);
            if (!dry && c0 == 0) gphase_mark(gtr, a.ktrace_id, 9);
        }
        if constexpr (kFlags)
            if (writer)   // release: this thread's partial stores of every chunk precede the flag
                st_release_u32(a.sk_flags + (((size_t)split * NT + nt) * MT + mt) * TM + row, tag);
        if (dry) bar();   // the warm-up pass's smem reads end before pass 1 rewrites sR / sPos / sBlk
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 2) tmem_dealloc(tmem, C::TMEM_COLS);
    gphase_mark(gtr, a.ktrace_id, 5);
    ktrace_mark(a.ktrace, a.ktrace_id, 1);
}

// ------------------------------------------------------------------ host side
static PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;

bool make_tmap_bf16(CUtensorMap* map, const void* base, uint64_t rows, uint64_t K, uint32_t box_rows) {
    if (!g_encode) {
        cudaDriverEntryPointQueryResult q;
        void* fn = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess || !fn)
            return false;
        g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    }
    cuuint64_t gdim[2] = {K, rows};
    cuuint64_t gstride[1] = {K * 2};
    cuuint32_t box[2] = {(cuuint32_t)BK, box_rows};
    cuuint32_t estride[2] = {1, 1};
    CUresult r = g_encode(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), gdim, gstride, box,
                          estride, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                          CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

int gemm_pick_tile_n(int M) {
    if (M <= 16) return 16;
    if (M <= 32) return 32;
    if (M <= 64) return 64;
    if (M <= 128) return 128;
    return 256;
}

// Split-K factor <= 8, only for small token tiles (TN <= 64; larger tiles have
// enough tiles to fill the GPU), with all CTAs resident in one wave (2 per SM) and
// >= 2 K blocks each: a power of two, or (g_split_fill) the largest count that
// still fits the wave (QKV at batch 1: 3 splits = 288 CTAs on 296 slots).
bool g_split_fill = true;   // env SV_SPLIT_POW2: powers of two only

int gemm_pick_splits(int N, int K, int M, int tile_n, int num_sms) {
    const int ntiles = (N / TM) * ((M + tile_n - 1) / tile_n);
    const int slots = num_sms * (tile_n <= 64 ? SV_GEMM_CTAS_PER_SM : 1);
    const int KB = K / BK;
    int s = 1;
    if (g_split_fill && tile_n <= 64) {
        s = std::max(1, std::min({SK_MAXP + 1, slots / ntiles, KB / 2}));
        return s;
    }
    while (s < 8 && ntiles * (2 * s) <= slots && 2 * (2 * s) <= KB) s *= 2;
    return s;
}

template <int TN, int EPI, int MAXST = SV_GEMM_MAX_STAGES>
static cudaError_t launch_t(const CUtensorMap& tmA, const CUtensorMap& tmB, const GemmArgs& a, cudaStream_t st) {
    using C = GemmCfg<TN, MAXST>;
    static bool attr_done = false;
    if (!attr_done) {
        cudaError_t e = cudaFuncSetAttribute(gemm_kernel<TN, EPI, MAXST>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             C::SMEM);
        if (e != cudaSuccess) return e;
        if (!getenv("SV_NO_CARVEOUT")) {   // let two grids' CTAs share an SM (PDL co-residency)
            e = cudaFuncSetAttribute(gemm_kernel<TN, EPI, MAXST>, cudaFuncAttributePreferredSharedMemoryCarveout,
                                     cudaSharedmemCarveoutMaxShared);
            if (e != cudaSuccess) return e;
        }
        if (getenv("SV_GEMM_DEBUG")) {
            int nb = 0;
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, gemm_kernel<TN, EPI, MAXST>, 128, C::SMEM);
            cudaFuncAttributes fa;
            cudaFuncGetAttributes(&fa, gemm_kernel<TN, EPI, MAXST>);
            int dev = 0, smsm = 0, rsv = 0, optin = 0;
            cudaGetDevice(&dev);
            cudaDeviceGetAttribute(&smsm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev);
            cudaDeviceGetAttribute(&rsv, cudaDevAttrReservedSharedMemoryPerBlock, dev);
            cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
            fprintf(stderr, "gemm_kernel<%d,%d>: smem %d static %zu regs %d local %zu -> %d blocks/SM "
                    "(SM smem %d, reserved/block %d, opt-in max %d)\n", TN, EPI, C::SMEM, fa.sharedSizeBytes,
                    fa.numRegs, fa.localSizeBytes, nb, smsm, rsv, optin);
        }
        attr_done = true;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(a.N / TM, (a.M + TN - 1) / TN, a.splits);
    cfg.blockDim = dim3(128, 1, 1);
    cfg.dynamicSmemBytes = C::SMEM;
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    int na = 0;
    if (g_use_pdl) {
        attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[na].val.programmaticStreamSerializationAllowed = 1;
        ++na;
    }
    cfg.attrs = attr;
    cfg.numAttrs = na;
    return cudaLaunchKernelEx(&cfg, gemm_kernel<TN, EPI, MAXST>, tmA, tmB, a);
}

template <int TN>
static cudaError_t launch_epi(int epi, const CUtensorMap& tmA, const CUtensorMap& tmB, const GemmArgs& a,
                              cudaStream_t st) {
    switch (epi) {
        case EPI_QKV: return launch_t<TN, EPI_QKV>(tmA, tmB, a, st);
        case EPI_RESID: return launch_t<TN, EPI_RESID>(tmA, tmB, a, st);
        case EPI_SWIGLU: return launch_t<TN, EPI_SWIGLU>(tmA, tmB, a, st);
        case EPI_LOGITS: return launch_t<TN, EPI_LOGITS>(tmA, tmB, a, st);
        case EPI_SILU: return launch_t<TN, EPI_SILU>(tmA, tmB, a, st);
    }
    return cudaErrorInvalidValue;
}

cudaError_t gemm_big_launch(int epi, int tile_n, const CUtensorMap& tmA, const CUtensorMap& tmB, const GemmArgs& a,
                            cudaStream_t st);

cudaError_t gemm_launch(int epi, int tile_n, const CUtensorMap& tmA, const CUtensorMap& tmB, const GemmArgs& a,
                        cudaStream_t st) {
    // large token tiles without split-K: persistent kernel with overlapped epilogue
    if (tile_n > 64 && (a.splits == 1 || a.stream_k) && !getenv("SV_NO_BIG_GEMM"))
        return gemm_big_launch(epi, tile_n, tmA, tmB, a, st);
    switch (tile_n) {
        case 16: return launch_epi<16>(epi, tmA, tmB, a, st);
        case 32: return launch_epi<32>(epi, tmA, tmB, a, st);
        case 64: return launch_epi<64>(epi, tmA, tmB, a, st);
        case 80: return launch_epi<80>(epi, tmA, tmB, a, st);
        case 128: return launch_epi<128>(epi, tmA, tmB, a, st);
        case 256: return launch_epi<256>(epi, tmA, tmB, a, st);
    }
    return cudaErrorInvalidValue;
}

}  // namespace sv
