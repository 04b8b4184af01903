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

#ifndef SV_GB_GROUPS
#define SV_GB_GROUPS 3
#endif
constexpr int GB_GROUPS = SV_GB_GROUPS;
// SV_GB_TRACE (compile-time): per-launch phase stamps of the persistent GEMM in the
// SV_GTRACE buffer (tools/trace_step.py); off in the product build
#ifdef SV_GB_TRACE
#define GB_MARK(ph) gphase_mark(a.gtrace, a.ktrace_id, ph)
// wait-time accounting (ns, summed over the launch's CTAs into slot (id, ph).first,
// which starts at ~0: the stored value is sum - 1)
#define GB_T0() const unsigned long long _gbt0 = gb_now()
#define GB_ACC(var) var += gb_now() - _gbt0
#define GB_FLUSH(ph, var) do { if (a.gtrace) atomicAdd(&a.gtrace[(a.ktrace_id * 16 + (ph)) * 2], var); } while (0)
#else
#define GB_MARK(ph) ((void)0)
#define GB_T0() ((void)0)
#define GB_ACC(var) ((void)0)
#define GB_FLUSH(ph, var) ((void)0)
#endif
__device__ __forceinline__ unsigned long long gb_now() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
constexpr int GB_BK = 64;
constexpr int GB_TM = 128;
constexpr int GB_A = GB_TM * GB_BK * 2;

template <int TN>
struct GBCfg {
    static constexpr int B_STAGE = TN * GB_BK * 2;
    static constexpr int STAGE = GB_A + B_STAGE;
    // two groups x (sOut [16][128] f32 + sRed [4][16]) + sR, sPos, sBlk [TN]
    static constexpr int EPI = GB_GROUPS * (EPI_CHUNK * GB_TM * 4 + 4 * EPI_CHUNK * 4) + 3 * TN * 4;
    static constexpr int AUX = 512;
    static constexpr int RAW = (227 * 1024 - 1024 - EPI - AUX) / STAGE;
    static constexpr int STAGES = RAW > 8 ? 8 : RAW;
    static constexpr int SMEM = 1024 + STAGES * STAGE + EPI + AUX;
    static constexpr int TCOLS = 2 * TN <= 256 ? 256 : 512;   // two accumulators (alloc: power of two)
    static_assert(STAGES >= 3 && TCOLS <= 512, "config");
};

// epilogue groups of 4 warps (one TMEM lane quarter each) taking every GB_GROUPS-th
// 16-token chunk: three groups cut the tail epilogue of a 5-chunk tile (C5) from
// 3 to 2 chunks and keep up with the tensor core at 256-token tiles (C4)
constexpr int GB_EPI_WARPS = 4 * GB_GROUPS, GB_THREADS = (GB_EPI_WARPS + 2) * 32;
constexpr int GB_PROD_WARP = GB_EPI_WARPS, GB_MMA_WARP = GB_EPI_WARPS + 1;

struct EpiBar {   // one epilogue group (named barrier 1 + group)
    int id;
    __device__ void operator()() const { asm volatile("bar.sync %0, 128;" ::"r"(id) : "memory"); }
};
__device__ __forceinline__ void epi_all_bar() {   // all epilogue warps (barrier 15)
    asm volatile("bar.sync 15, %0;" ::"n"(GB_EPI_WARPS * 32) : "memory");
}

// Stream-K (SK): the T x KB (tile, K block) units are dealt to the P CTAs as equal
// contiguous ranges, so every SM streams the same number of weight bytes whatever
// T mod P is.  A CTA's range is a sequence of pieces (tile, kb0, kb1): a piece that
// covers its whole tile runs the normal epilogue; a piece that starts mid-tile is
// always the first piece of its CTA's range ("writer": fp32 partial -> ws[cta],
// then one release flag per thread); the piece holding a tile's first K block
// ("reducer", the last piece of its CTA) adds the later pieces' partials in CTA
// (= K) order after acquiring their flags — deterministic, and a reducer only ever
// waits for writers, which wait for nothing (all P <= #SMs CTAs are resident).
struct SkPiece {
    int t, kb0, kb1;
};
__device__ __forceinline__ long long sk_bound(long long U, int P, int c) { return U * c / P; }
__device__ __forceinline__ int sk_cta_of(long long u, long long U, int P) {   // CTA whose range holds unit u
    int c = (int)((u * P) / U);
    while (c + 1 < P && sk_bound(U, P, c + 1) <= u) ++c;
    while (c > 0 && sk_bound(U, P, c) > u) --c;
    return c;
}

template <int TN, int EPI, bool SK = false>
__global__ void __launch_bounds__(GB_THREADS, 1)
    gemm_big_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                    const __grid_constant__ GemmArgs a) {
    using C = GBCfg<TN>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sA = smem;
    uint8_t* sB = smem + C::STAGES * GB_A;
    float* sOut0 = reinterpret_cast<float*>(smem + C::STAGES * C::STAGE);  // 2 x [EPI_CHUNK][128]
    float* sRed0 = sOut0 + GB_GROUPS * EPI_CHUNK * GB_TM;                  // groups x [4][EPI_CHUNK]
    float* sR = sRed0 + GB_GROUPS * 4 * EPI_CHUNK;                         // [TN]
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
    // the CTA's work: plain = whole tiles blockIdx.x, +P, ...; SK = unit range [u0, u1)
    const int P = gridDim.x;
    const long long U = (long long)T * KB;
    const long long u0 = SK ? sk_bound(U, P, blockIdx.x) : 0, u1 = SK ? sk_bound(U, P, blockIdx.x + 1) : 0;
    auto first_piece = [&](SkPiece& pc, long long& u) -> bool {
        if (SK) {
            u = u0;
            if (u >= u1) return false;
            pc.t = (int)(u / KB);
            pc.kb0 = (int)(u % KB);
            pc.kb1 = (int)min((long long)KB, pc.kb0 + (u1 - u));
            return true;
        }
        pc.t = blockIdx.x;
        pc.kb0 = 0;
        pc.kb1 = KB;
        return pc.t < T;
    };
    auto next_piece = [&](SkPiece& pc, long long& u) -> bool {
        if (SK) {
            u += pc.kb1 - pc.kb0;
            if (u >= u1) return false;
            pc.t = (int)(u / KB);
            pc.kb0 = 0;
            pc.kb1 = (int)min((long long)KB, u1 - u);
            return true;
        }
        pc.t += P;
        return pc.t < T;
    };
    ktrace_mark(a.ktrace, a.ktrace_id, 0);
    if (threadIdx.x == 0) GB_MARK(0);
    if (warp == GB_PROD_WARP && lane == 0) {
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
    if (warp == GB_MMA_WARP) tmem_alloc(tmem_slot, C::TCOLS);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    pdl_launch_dependents();

    if (warp == GB_PROD_WARP) {
        if (lane == 0) {   // ------------------------------------------ producer
            const uint64_t pol_w = policy_evict_first(), pol_x = policy_evict_last();
            const uint32_t stage_tx = GB_A + (a.b_box ? a.b_box : TN) * GB_BK * 2;   // GemmArgs::b_box
            // weights never depend on the previous kernel: the first ring's worth of weight
            // blocks is requested before griddepcontrol.wait (streams during its tail)
            unsigned long long w_empty = 0;
            (void)w_empty;
            int pre = 0;
            {
                SkPiece pc;
                long long u;
                for (bool ok = first_piece(pc, u); ok && pre < C::STAGES; ok = next_piece(pc, u)) {
                    const int n0 = (pc.t / MT) * GB_TM;
                    for (int kb = pc.kb0; kb < pc.kb1 && pre < C::STAGES; ++kb, ++pre) {
                        mbar_arrive_expect_tx(&full[pre], stage_tx);
                        tma_load_2d(&tmA, sA + pre * GB_A, &full[pre], kb * GB_BK, n0, pol_w);
                    }
                }
            }
            pdl_wait();
            GB_MARK(1);
            int it = 0;
            SkPiece pc;
            long long u;
            for (bool ok = first_piece(pc, u); ok; ok = next_piece(pc, u)) {
                const int n0 = (pc.t / MT) * GB_TM, m0 = (pc.t % MT) * TN;
                for (int kb = pc.kb0; kb < pc.kb1; ++kb, ++it) {
                    const int s = it % C::STAGES;
                    if (it >= pre) {
                        if (it >= C::STAGES) {
                            GB_T0();
                            mbar_wait(&empty[s], ((it / C::STAGES) - 1) & 1);
                            GB_ACC(w_empty);
                        }
                        mbar_arrive_expect_tx(&full[s], stage_tx);
                        tma_load_2d(&tmA, sA + s * GB_A, &full[s], kb * GB_BK, n0, pol_w);
                    }
                    tma_load_2d(&tmB, sB + s * C::B_STAGE, &full[s], kb * GB_BK, m0 + a.b_row0, pol_x);
                }
            }
            GB_FLUSH(6, w_empty);
            GB_FLUSH(10, 1ull);
            if constexpr (EPI == EPI_QKV) {   // GemmArgs::kv_pf_blocks
                const size_t plane = (size_t)a.n_heads * EPI_PAGE * a.head_dim;   // elements per K (or V) plane
                int item = 0;
                for (int b = 0; b < a.kv_pf_B && item < a.kv_pf_blocks; ++b) {
                    const int npg = (a.meta.ctx[b] + EPI_PAGE - 1) / EPI_PAGE;
                    for (int p = 0; p < npg && item < a.kv_pf_blocks; ++p, ++item) {
                        if (item % P != (int)blockIdx.x) continue;
                        const int blk = a.meta.page_table[b * a.meta.pt_stride + p];
                        const uint8_t* base = reinterpret_cast<const uint8_t*>(a.kv_pool) +
                                              (((size_t)blk * a.n_layers + a.layer) * 2 * plane) * 2;
                        for (size_t o = 0; o < 2 * plane * 2; o += 65536)
                            bulk_prefetch_l2(base + o, (uint32_t)min((size_t)65536, 2 * plane * 2 - o));
                    }
                }
            }
        }
    } else if (warp == GB_MMA_WARP) {
        if (lane == 0) {   // ------------------------------------------ MMA issuer
            constexpr uint32_t idesc = umma_idesc_bf16(GB_TM, TN);
            int it = 0, seg = 0;
            unsigned long long w_full = 0, w_tempty = 0;
            (void)w_full; (void)w_tempty;
            SkPiece pc;
            long long u;
            for (bool ok = first_piece(pc, u); ok; ok = next_piece(pc, u), ++seg) {
                const int buf = seg & 1;
                if (seg >= 2) {
                    GB_T0();
                    mbar_wait(&tempty[buf], ((seg >> 1) - 1) & 1);
                    GB_ACC(w_tempty);
                }
                tc_fence_after();
                const uint32_t dt = tmem + buf * TN;
                for (int kb = pc.kb0; kb < pc.kb1; ++kb, ++it) {
                    const int s = it % C::STAGES;
                    {
                        GB_T0();
                        mbar_wait(&full[s], (it / C::STAGES) & 1);
                        if (it > 0) GB_ACC(w_full);
                    }
                    if (it == 0) GB_MARK(2);
                    tc_fence_after();
                    const uint64_t ad = umma_sdesc_sw128(smem_u32(sA + s * GB_A));
                    const uint64_t bd = umma_sdesc_sw128(smem_u32(sB + s * C::B_STAGE));
#pragma unroll
                    for (int k = 0; k < GB_BK / 16; ++k)
                        umma_bf16(dt, ad + 2 * k, bd + 2 * k, idesc, (kb > pc.kb0 || k) ? 1u : 0u);
                    umma_commit(&empty[s]);
                }
                umma_commit(&tfull[buf]);
            }
            GB_MARK(3);
            GB_FLUSH(7, w_full);
            GB_FLUSH(8, w_tempty);
        }
    } else {               // ------------------------------------------ epilogue warps
        const int grp = warp >> 2, tid = threadIdx.x;     // tid 0 .. 32 * GB_EPI_WARPS - 1
        const EpiBar bar{1 + grp};
        const int r = tid & 127;                           // tile row (TMEM lane)
        float* sOut = sOut0 + grp * EPI_CHUNK * GB_TM;
        float* sRed = sRed0 + grp * 4 * EPI_CHUNK;
        pdl_wait();                                        // epilogue inputs come from earlier kernels
        const uint32_t tag = SK ? ((*a.meta.epoch << 10) | (uint32_t)(a.ktrace_id & 1023)) : 0u;
        int seg = 0;
        unsigned long long w_tfull = 0;
        (void)w_tfull;
        SkPiece pc;
        long long u;
        for (bool ok = first_piece(pc, u); ok; ok = next_piece(pc, u), ++seg) {
            const int buf = seg & 1;
            const int t = pc.t, nt = t / MT, n0 = nt * GB_TM, m0 = (t % MT) * TN;
            const bool writer = SK && pc.kb0 > 0;                    // later K blocks of a split tile
            const bool reducer = SK && pc.kb0 == 0 && pc.kb1 < KB;   // first K blocks: adds the others
            const int cl = reducer ? sk_cta_of((long long)(t + 1) * KB - 1, U, P) : 0;
            if (!writer) {
                epi_rstd(a, sR, m0, TN, tid, GB_EPI_WARPS * 32);         // overlaps the tile's MMA
                if constexpr (EPI == EPI_QKV) epi_meta(a, sPos, sBlk, m0, TN, tid, GB_EPI_WARPS * 32);
            }
            epi_all_bar();
            if (tid == 0) GB_MARK(11);
            {
                GB_T0();
                mbar_wait(&tfull[buf], (seg >> 1) & 1);
                if (tid == 0 && seg > 0) GB_ACC(w_tfull);
            }
            if (tid == 0) GB_MARK(13);
            tc_fence_after();
            const uint32_t tb = tmem + (static_cast<uint32_t>((warp & 3) * 32) << 16) + buf * TN;
            if (reducer) {   // the writers of this tile: CTAs blockIdx.x + 1 .. cl (their first pieces)
                for (int c = blockIdx.x + 1; c <= cl; ++c) {
                    const uint32_t* f = a.sk_flags + ((size_t)c * GB_GROUPS + grp) * GB_TM + r;
                    for (uint32_t n = 0; ld_acquire_u32(f) != tag; ++n)
                        if (n > SV_SPIN_LIMIT) __trap();
                }
                if (tid == 0) GB_MARK(4);
            }
            for (int c0 = grp * EPI_CHUNK; c0 < TN; c0 += GB_GROUPS * EPI_CHUNK) {
                if (m0 + c0 >= a.M) break;                 // uniform over the group
                const int nv = min(EPI_CHUNK, a.M - (m0 + c0));
                // the chunk's epilogue inputs that do not depend on the accumulator, issued
                // with (before) the partial loads: one round trip per chunk
                EpiPre pre;
                if (!writer) {
                    if constexpr (EPI == EPI_RESID) {
#pragma unroll
                        for (int j = 0; j < 16; ++j)
                            pre.h[j] = j < nv ? __ldcg(&a.h[(size_t)(m0 + c0 + j) * a.d_model + n0 + r]) : 0.f;
                        pre.g = __bfloat162float(reinterpret_cast<const bf16*>(a.g_out)[n0 + r]);
                        pre.g2 = a.u_out2 ? __bfloat162float(reinterpret_cast<const bf16*>(a.g_out2)[n0 + r]) : 0.f;
                    }
                }
                uint32_t v[16];
                tmem_ld_32x32b_x16(tb + c0, v);
                tmem_ld_wait();
                if (writer) {
                    float* w = a.ws + ((size_t)blockIdx.x * TN + c0) * GB_TM + r;
#pragma unroll
                    for (int j = 0; j < 16; ++j)
                        if (j < nv) __stcg(&w[(size_t)j * GB_TM], __uint_as_float(v[j]));
                    continue;
                }
                float acc[16];
#pragma unroll
                for (int j = 0; j < 16; ++j) acc[j] = reducer ? 0.f + __uint_as_float(v[j]) : __uint_as_float(v[j]);
                if (reducer)
                    for (int c = blockIdx.x + 1; c <= cl; c += 3) {   // K order, 3 partners' loads in flight
                        float x[3][16];
#pragma unroll
                        for (int q = 0; q < 3; ++q) {
                            const float* w = a.ws + ((size_t)(c + q) * TN + c0) * GB_TM + r;
#pragma unroll
                            for (int j = 0; j < 16; ++j) x[q][j] = (j < nv && c + q <= cl) ? __ldcg(&w[(size_t)j * GB_TM]) : 0.f;
                        }
#pragma unroll
                        for (int q = 0; q < 3; ++q)
                            if (c + q <= cl)
#pragma unroll
                                for (int j = 0; j < 16; ++j) acc[j] += x[q][j];
                    }
                bar();
#pragma unroll
                for (int j = 0; j < 16; ++j) sOut[j * GB_TM + r] = acc[j];
                bar();
                epi_apply<EPI>(a, sOut, sR, sRed, m0 + c0, m0, n0, nt, r, bar, sPos, sBlk,
                               EPI == EPI_RESID ? &pre : nullptr);
            }
            if (writer)   // release: this thread's partial stores precede its flag
                st_release_u32(a.sk_flags + ((size_t)blockIdx.x * GB_GROUPS + grp) * GB_TM + r, tag);
            tc_fence_before();
            epi_all_bar();                                 // also guards sR / sPos reuse
            if (tid == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&tempty[buf])) : "memory");
            if (tid == 0) GB_MARK(14);
        }
        if (tid == 0) GB_FLUSH(9, w_tfull);
    }
    tc_fence_before();
    __syncthreads();
    if (warp == GB_MMA_WARP) tmem_dealloc(tmem, C::TCOLS);
    if (threadIdx.x == 0) GB_MARK(5);
    ktrace_mark(a.ktrace, a.ktrace_id, 1);
}

template <int TN, int EPI, bool SK>
static cudaError_t big_t(const CUtensorMap& tmA, const CUtensorMap& tmB, const GemmArgs& a, cudaStream_t st) {
    using C = GBCfg<TN>;
    static bool attr = false;
    static int sms = 0;
    if (!attr) {
        cudaError_t e = cudaFuncSetAttribute(gemm_big_kernel<TN, EPI, SK>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             C::SMEM);
        if (e != cudaSuccess) return e;
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        attr = true;
    }
    const int T = (a.N / GB_TM) * ((a.M + TN - 1) / TN);
    const long long U = (long long)T * (a.K / GB_BK);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(SK ? (int)(U < sms ? U : sms) : (T < sms ? T : sms), 1, 1);
    cfg.blockDim = dim3(GB_THREADS, 1, 1);
    cfg.dynamicSmemBytes = C::SMEM;
    cfg.stream = st;
    cudaLaunchAttribute attr1[1];
    attr1[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr1[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr1;
    cfg.numAttrs = g_use_pdl ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, gemm_big_kernel<TN, EPI, SK>, tmA, tmB, a);
}

template <int TN>
static cudaError_t big_epi(int epi, const CUtensorMap& tmA, const CUtensorMap& tmB, const GemmArgs& a,
                           cudaStream_t st) {
    switch (epi) {
        case EPI_QKV: return a.stream_k ? big_t<TN, EPI_QKV, true>(tmA, tmB, a, st) : big_t<TN, EPI_QKV, false>(tmA, tmB, a, st);
        case EPI_RESID: return a.stream_k ? big_t<TN, EPI_RESID, true>(tmA, tmB, a, st) : big_t<TN, EPI_RESID, false>(tmA, tmB, a, st);
        case EPI_SWIGLU: return a.stream_k ? big_t<TN, EPI_SWIGLU, true>(tmA, tmB, a, st) : big_t<TN, EPI_SWIGLU, false>(tmA, tmB, a, st);
        case EPI_LOGITS: return big_t<TN, EPI_LOGITS, false>(tmA, tmB, a, st);
        case EPI_SILU: return big_t<TN, EPI_SILU, false>(tmA, tmB, a, st);
    }
    return cudaErrorInvalidValue;
}

cudaError_t gemm_big_launch(int epi, int tile_n, const CUtensorMap& tmA, const CUtensorMap& tmB, const GemmArgs& a,
                            cudaStream_t st) {
    if (tile_n == 128) return big_epi<128>(epi, tmA, tmB, a, st);
    if (tile_n == 256) return big_epi<256>(epi, tmA, tmB, a, st);
    if (tile_n == 160) return big_epi<160>(epi, tmA, tmB, a, st);
    if (tile_n == 80) return big_epi<80>(epi, tmA, tmB, a, st);
    return cudaErrorInvalidValue;
}

}  // namespace sv
