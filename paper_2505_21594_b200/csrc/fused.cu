// fused.cu — the whole verify step as ONE persistent kernel (one CTA per SM).
//
// Why: at batch 1 the step streams 13.5 GB of weights through ~130 GEMMs of
// 5-28 us each; as separate kernels every op pays launch ramp, pipeline fill,
// split-K tail and a dependency bubble.  Here each CTA walks a precomputed list
// of work items (stage order) with three warp roles:
//   warp 0 (1 thread)  TMA producer: streams the 128x64 weight tiles of its GEMM
//                      segments into a STAGES-deep smem ring AHEAD of dependencies
//                      (weights never depend on the step's data); the activation
//                      tile of a stage is loaded only once the producing stage has
//                      completed (device-scope counter, acquire), so the HBM weight
//                      stream continues across op boundaries.
//   warp 1 (1 thread)  tcgen05.mma issuer (kind::f16, M=128, N=TILE_N, fp32 accum)
//                      into a double-buffered TMEM accumulator.
//   warps 2-5          workers: GEMM epilogues (TMEM -> fused op, or split
//                      partial + in-order reduction by the last segment), attention
//                      pages, vocabulary statistics, acceptance, embedding.
// GEMMs are split stream-K style: the (tile, k-block) units of each GEMM are
// divided into equal contiguous ranges, one per CTA, so every SM streams the same
// number of weight bytes per op; a tile cut by a range boundary is reduced by
// its last-arriving segment in k order (deterministic).
// Dependencies: every stage waits only on an earlier stage and every CTA's list is
// in stage order, so the persistent grid (co-resident, cooperative launch) cannot
// deadlock; all spins are bounded (trap).
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "accept_dev.cuh"
#include "attn_dev.cuh"
#include "fused.h"
#include "gemm_epi.cuh"

namespace sv {

constexpr int F_BK = 64;
constexpr int F_TM = 128;
constexpr int F_A_STAGE = F_TM * F_BK * 2;   // 16 KB of weights per stage
constexpr int F_THREADS = 192;
#ifndef SV_FUSED_SMEM
#define SV_FUSED_SMEM 232448                 // 227 KB opt-in dynamic shared memory (one CTA per SM)
#endif
constexpr int F_SMEM_MAX = SV_FUSED_SMEM;

template <int TN>
struct EpiSmem {
    float sOut[EPI_CHUNK * F_TM];
    float sR[TN < 16 ? 16 : TN];
    float sRed[4 * EPI_CHUNK];
    int flag;
};

template <int TN, int D>
struct FCfg {
    static constexpr int B_STAGE = TN * F_BK * 2;
    static constexpr int STAGE = F_A_STAGE + B_STAGE;
    static constexpr int U1 = (int)sizeof(AttnSmem<D>);
    static constexpr int U2 = (int)sizeof(EpiSmem<TN>);
    static constexpr int U3 = (int)sizeof(AcceptSmem);
    static constexpr int UNION = ((U1 > U2 ? (U1 > U3 ? U1 : U3) : (U2 > U3 ? U2 : U3)) + 127) / 128 * 128;
    static constexpr int BAR = 512;
    static constexpr int SCACHE = 1024;      // per-item copy of the stage descriptor
    static constexpr int STAGES_RAW = (F_SMEM_MAX - 1024 - UNION - BAR - SCACHE) / STAGE;
    static constexpr int STAGES = STAGES_RAW < 2 ? 2 : (STAGES_RAW > 12 ? 12 : STAGES_RAW);   // (a shallow-smem
                                                     // build cannot launch the largest tiles: launch error)
    static constexpr int SMEM = 1024 + STAGES * STAGE + UNION + BAR + SCACHE;
    static_assert(sizeof(FStage) <= SCACHE && sizeof(FStage) % 16 == 0, "stage descriptor cache");
    static constexpr int TBUF = TN < 32 ? 32 : TN;                 // TMEM columns per accumulator
    static constexpr int TCOLS = 2 * TBUF <= 32 ? 32 : (2 * TBUF <= 64 ? 64 : (2 * TBUF <= 128 ? 128 : (2 * TBUF <= 256 ? 256 : 512)));
};

struct FArgs {
    const FStage* stages;
    const FItem* items;
    const int* item_start;
    const int* seg_slots;
    int* cnt;
    int* tile_cnt;
    float* ws_main;
    float* ws_exit;
    sv_exit_result* early_host;
    uint64_t* early_flag;
    const uint64_t* seq;
    unsigned long long* trace;   // optional timeline [item][4] (globaltimer ns), nullptr = off
};

__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

__device__ __forceinline__ int ld_acquire(const int* p) {
    int v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void fence_proxy_async_global() {
    asm volatile("fence.proxy.async.global;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
struct WorkerSync {
    __device__ void operator()() const { asm volatile("bar.sync 1, 128;" ::: "memory"); }
};

template <class Sync>
__device__ __forceinline__ void wait_stage(const FArgs& f, const FStage& S, int wt, Sync sync) {
    if (S.dep >= 0) {
        if (wt == 0) {
            uint32_t n = 0;
            while (ld_acquire(&f.cnt[S.dep]) < S.dep_target) {
                if (++n > SV_SPIN_LIMIT) __trap();
            }
        }
        sync();
    }
}

template <int EPI, class Sync>
__device__ __forceinline__ void epi_dispatch_t(const GemmArgs& g, const float* sOut, const float* sR, float* sRed,
                                               int tok0, int m0, int n0, int nt, int r, Sync sync) {
    epi_apply<EPI>(g, sOut, sR, sRed, tok0, m0, n0, nt, r, sync);
}
template <class Sync>
__device__ __forceinline__ void epi_dispatch(int epi, const GemmArgs& g, const float* sOut, const float* sR,
                                             float* sRed, int tok0, int m0, int n0, int nt, int r, Sync sync) {
    switch (epi) {
        case EPI_QKV: epi_dispatch_t<EPI_QKV>(g, sOut, sR, sRed, tok0, m0, n0, nt, r, sync); break;
        case EPI_RESID: epi_dispatch_t<EPI_RESID>(g, sOut, sR, sRed, tok0, m0, n0, nt, r, sync); break;
        case EPI_SWIGLU: epi_dispatch_t<EPI_SWIGLU>(g, sOut, sR, sRed, tok0, m0, n0, nt, r, sync); break;
        default: epi_dispatch_t<EPI_LOGITS>(g, sOut, sR, sRed, tok0, m0, n0, nt, r, sync); break;
    }
}

// rstd[t] = 1/sqrt(sum_k ssq[k][m0+t] / d + eps) with every load of the step in
// flight at once: for TN <= 16, 8 groups x 16 tokens, each group sums a contiguous
// run of tiles in order, then the 8 group sums are added in order (fixed tree).
template <int TN, class Sync>
__device__ __forceinline__ void fused_rstd(const GemmArgs& g, float* sR, float* scratch, int m0, int wt, Sync sync) {
    if (!g.ssq_in) {
        for (int t = wt; t < TN; t += 128) sR[t] = 1.0f;
        sync();
        return;
    }
    if constexpr (TN <= 16) {
        const int grp = wt >> 4, t = wt & 15, tok = m0 + t;
        const int per = (g.ssq_tiles + 7) / 8, k0 = grp * per;
        float v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int k = k0 + u;
            v[u] = (u < per && k < g.ssq_tiles && tok < g.M) ? __ldcg(&g.ssq_in[(size_t)k * g.MP + tok]) : 0.f;
        }
        float s = 0.f;
        for (int u = 0; u < per && u < 8; ++u) s += v[u];
        for (int k = k0 + 8; k < k0 + per && k < g.ssq_tiles; ++k)       // (d > 8192 only)
            s += (tok < g.M) ? __ldcg(&g.ssq_in[(size_t)k * g.MP + tok]) : 0.f;
        scratch[grp * 16 + t] = s;
        sync();
        if (wt < 16) {
            float a = 0.f;
#pragma unroll
            for (int q = 0; q < 8; ++q) a += scratch[q * 16 + wt];
            sR[wt] = 1.0f / sqrtf(a * g.inv_d + g.eps);
        }
        sync();
    } else {
        for (int t = wt; t < TN; t += 128) {
            const int tok = m0 + t;
            float s = 0.f;
            if (tok < g.M) {
                int k = 0;
                for (; k + 16 <= g.ssq_tiles; k += 16) {
                    float v[16];
#pragma unroll
                    for (int u = 0; u < 16; ++u) v[u] = __ldcg(&g.ssq_in[(size_t)(k + u) * g.MP + tok]);
#pragma unroll
                    for (int u = 0; u < 16; ++u) s += v[u];
                }
                for (; k < g.ssq_tiles; ++k) s += __ldcg(&g.ssq_in[(size_t)k * g.MP + tok]);
            }
            sR[t] = 1.0f / sqrtf(s * g.inv_d + g.eps);
        }
        sync();
    }
}

template <int TN, int D>
__global__ void __launch_bounds__(F_THREADS, F_SMEM_MAX < 120 * 1024 ? 2 : 1) fused_step_kernel(const __grid_constant__ FArgs f) {
    using C = FCfg<TN, D>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sA = smem;
    uint8_t* sB = smem + C::STAGES * F_A_STAGE;
    uint8_t* uni = smem + C::STAGES * C::STAGE;
    uint64_t* full = reinterpret_cast<uint64_t*>(uni + C::UNION);
    uint64_t* empty = full + C::STAGES;
    uint64_t* tfull = empty + C::STAGES;
    uint64_t* tempty = tfull + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
    FStage* sStage = reinterpret_cast<FStage*>(uni + C::UNION + C::BAR);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int beg = f.item_start[blockIdx.x], end = f.item_start[blockIdx.x + 1];

    if (warp == 0 && lane == 0) {
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
    if (warp == 1) tmem_alloc(tmem_slot, C::TCOLS);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {
            // ------------------------------------------------ TMA producer
            const uint64_t pol_w = policy_evict_first(), pol_x = policy_evict_last();
            int qs[C::STAGES], qst[C::STAGES], qkb[C::STAGES], qm0[C::STAGES], qit[C::STAGES];
            int qh = 0, qt = 0, a_cnt = 0, sat = -1;
            uint32_t spins = 0;
            auto dep_ok = [&](int st) -> bool {
                if (st == sat) return true;
                const FStage& S = f.stages[st];
                if (S.dep < 0 || ld_acquire(&f.cnt[S.dep]) >= S.dep_target) {
                    // once per newly satisfied dependency: make the producers' generic
                    // stores (acquired above) visible to this thread's async-proxy reads
                    fence_proxy_async_global();
                    sat = st;
                    return true;
                }
                return false;
            };
            auto service = [&]() {
                while (qh != qt) {
                    const int k = qh % C::STAGES;
                    if (!dep_ok(qst[k])) break;
                    tma_load_2d(f.stages[qst[k]].tmB, sB + qs[k] * C::B_STAGE, &full[qs[k]], qkb[k] * F_BK, qm0[k],
                                pol_x);
                    if (f.trace && qit[k] >= 0) f.trace[(size_t)qit[k] * 4 + 1] = gtimer();
                    ++qh;
                }
            };
            for (int it = beg; it < end; ++it) {
                const FItem I = f.items[it];
                if (I.type != IT_GEMM) continue;
                const FStage& S = f.stages[I.stage];
                const int n0 = (I.tile / S.nt_m) * F_TM, m0 = (I.tile % S.nt_m) * TN;
                for (int kb = I.kb0; kb < I.kb1; ++kb) {
                    const int s = a_cnt % C::STAGES;
                    if (a_cnt >= C::STAGES) {
                        const uint32_t par = ((a_cnt / C::STAGES) - 1) & 1;
                        const uint32_t bar = smem_u32(&empty[s]);
                        while (!mbar_try_wait(bar, par)) {
                            service();
                            if (++spins > SV_SPIN_LIMIT) __trap();
                        }
                    }
                    mbar_arrive_expect_tx(&full[s], C::STAGE);
                    tma_load_2d(S.tmA, sA + s * F_A_STAGE, &full[s], kb * F_BK, n0, pol_w);
                    if (f.trace && kb == I.kb0) f.trace[(size_t)it * 4 + 0] = gtimer();
                    const int k = qt % C::STAGES;
                    qs[k] = s; qst[k] = I.stage; qkb[k] = kb; qm0[k] = m0;
                    qit[k] = (kb == I.kb0) ? it : -1;
                    ++qt;
                    ++a_cnt;
                    service();
                }
            }
            while (qh != qt) {
                service();
                if (++spins > SV_SPIN_LIMIT) __trap();
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            // ------------------------------------------------ MMA issuer
            constexpr uint32_t idesc = umma_idesc_bf16(F_TM, TN);
            int st_cnt = 0, seg = 0;
            for (int it = beg; it < end; ++it) {
                const FItem I = f.items[it];
                if (I.type != IT_GEMM) continue;
                const int buf = seg & 1;
                if (seg >= 2) mbar_wait(&tempty[buf], ((seg >> 1) - 1) & 1);
                tc_fence_after();
                const uint32_t dt = tmem + buf * C::TBUF;
                for (int kb = I.kb0; kb < I.kb1; ++kb) {
                    const int s = st_cnt % C::STAGES;
                    mbar_wait(&full[s], (st_cnt / C::STAGES) & 1);
                    tc_fence_after();
                    const uint64_t ad = umma_sdesc_sw128(smem_u32(sA + s * F_A_STAGE));
                    const uint64_t bd = umma_sdesc_sw128(smem_u32(sB + s * C::B_STAGE));
#pragma unroll
                    for (int k = 0; k < F_BK / 16; ++k)
                        umma_bf16(dt, ad + 2 * k, bd + 2 * k, idesc, (kb > I.kb0 || k > 0) ? 1u : 0u);
                    umma_commit(&empty[s]);
                    ++st_cnt;
                }
                umma_commit(&tfull[buf]);
                ++seg;
            }
        }
    } else {
        // ---------------------------------------------------- workers (128 threads)
        const int wt = threadIdx.x - 64;
        const int row = (warp & 3) * 32 + lane;           // TMEM lane quarter of this warp
        const uint32_t tlane = static_cast<uint32_t>((warp & 3) * 32) << 16;
        WorkerSync wsync;
        EpiSmem<TN>& E = *reinterpret_cast<EpiSmem<TN>*>(uni);
        int seg = 0, cached = -1;
        for (int it = beg; it < end; ++it) {
            const FItem I = f.items[it];
            if (I.stage != cached) {   // one coalesced copy of the descriptor per stage change
                wsync();
                const uint4* src = reinterpret_cast<const uint4*>(f.stages + I.stage);
                for (int i = wt; i < (int)(sizeof(FStage) / 16); i += 128)
                    reinterpret_cast<uint4*>(sStage)[i] = __ldg(src + i);
                wsync();
                cached = I.stage;
            }
            const FStage& S = *sStage;
            if (I.type == IT_GEMM) {
                const int buf = seg & 1;
                mbar_wait(&tfull[buf], (seg >> 1) & 1);
                tc_fence_after();
                wait_stage(f, S, wt, wsync);
                if (f.trace && wt == 0) f.trace[(size_t)it * 4 + 2] = gtimer();
                const GemmArgs& g = S.g;
                const int nt = I.tile / S.nt_m, n0 = nt * F_TM, m0 = (I.tile % S.nt_m) * TN;
                const uint32_t tb = tmem + tlane + buf * C::TBUF;
                if (I.nsegs == 1) {
                    fused_rstd<TN>(g, E.sR, E.sOut, m0, wt, wsync);
                    for (int c0 = 0; c0 < TN; c0 += EPI_CHUNK) {
                        if (m0 + c0 >= g.M) break;
                        uint32_t r[16];
                        tmem_ld_32x32b_x16(tb + c0, r);
                        tmem_ld_wait();
                        wsync();
#pragma unroll
                        for (int j = 0; j < 16; ++j) E.sOut[j * F_TM + row] = __uint_as_float(r[j]);
                        wsync();
                        epi_dispatch(S.epi, g, E.sOut, E.sR, E.sRed, m0 + c0, m0, n0, nt, wt, wsync);
                    }
                } else {
                    float* wsp = (S.exit_ws ? f.ws_exit : f.ws_main) + (size_t)I.slot * TN * F_TM;
                    for (int c0 = 0; c0 < TN; c0 += EPI_CHUNK) {
                        if (m0 + c0 >= g.M) break;
                        uint32_t r[16];
                        tmem_ld_32x32b_x16(tb + c0, r);
                        tmem_ld_wait();
#pragma unroll
                        for (int j = 0; j < 16; ++j)
                            if (m0 + c0 + j < g.M) wsp[(size_t)(c0 + j) * F_TM + row] = __uint_as_float(r[j]);
                    }
                }
                tc_fence_before();
                wsync();
                if (wt == 0) mbar_arrive(&tempty[buf]);
                ++seg;
                bool finalized = (I.nsegs == 1);
                if (!finalized) {
                    __threadfence();
                    wsync();
                    if (wt == 0) E.flag = (atomicAdd(&f.tile_cnt[S.tile_base + I.tile], 1) == I.nsegs - 1);
                    wsync();
                    if (E.flag) {
                        __threadfence();
                        fused_rstd<TN>(g, E.sR, E.sOut, m0, wt, wsync);
                        const float* wsb = S.exit_ws ? f.ws_exit : f.ws_main;
                        for (int c0 = 0; c0 < TN; c0 += EPI_CHUNK) {
                            if (m0 + c0 >= g.M) break;
                            const int nv = min(EPI_CHUNK, g.M - (m0 + c0));
                            float acc[EPI_CHUNK];
#pragma unroll
                            for (int j = 0; j < EPI_CHUNK; ++j) acc[j] = 0.f;
                            for (int s0 = 0; s0 < I.nsegs; s0 += 4) {   // k order; 4 segments in flight
                                float v[4][EPI_CHUNK];
#pragma unroll
                                for (int u = 0; u < 4; ++u) {
                                    const bool ok = s0 + u < I.nsegs;
                                    const float* p = wsb +
                                                     (size_t)(ok ? f.seg_slots[I.seg_first + s0 + u] : 0) * TN * F_TM +
                                                     (size_t)c0 * F_TM + row;
#pragma unroll
                                    for (int j = 0; j < EPI_CHUNK; ++j)
                                        v[u][j] = (ok && j < nv) ? __ldcg(p + j * F_TM) : 0.f;
                                }
#pragma unroll
                                for (int u = 0; u < 4; ++u)
#pragma unroll
                                    for (int j = 0; j < EPI_CHUNK; ++j)
                                        if (s0 + u < I.nsegs) acc[j] += v[u][j];
                            }
                            wsync();
#pragma unroll
                            for (int j = 0; j < EPI_CHUNK; ++j) E.sOut[j * F_TM + row] = acc[j];
                            wsync();
                            epi_dispatch(S.epi, g, E.sOut, E.sR, E.sRed, m0 + c0, m0, n0, nt, wt, wsync);
                        }
                        finalized = true;
                    }
                }
                if (finalized) {
                    fence_proxy_async_global();   // outputs may be read by TMA (async proxy)
                    __threadfence();
                    wsync();
                    if (wt == 0) atomicAdd(&f.cnt[I.stage], 1);
                }
            } else if (I.type == IT_ATTN) {
                wait_stage(f, S, wt, wsync);
                if (f.trace && wt == 0) f.trace[(size_t)it * 4 + 2] = gtimer();
                const bool merged = attn_page_body<D>(S.at, I.tile, I.kb0, wt,
                                                      *reinterpret_cast<AttnSmem<D>*>(uni), wsync);
                if (merged) {
                    fence_proxy_async_global();
                    __threadfence();
                    wsync();
                    if (wt == 0) atomicAdd(&f.cnt[I.stage], 1);
                }
                wsync();
            } else if (I.type == IT_STATS) {
                wait_stage(f, S, wt, wsync);
                if (f.trace && wt == 0) f.trace[(size_t)it * 4 + 2] = gtimer();
                AcceptSmem& A = *reinterpret_cast<AcceptSmem*>(uni);
                if (S.ac.req[I.tile / S.ac.G].status_in == 0) row_stats_body<128>(S.ac, I.tile, I.kb0, wt, A, wsync);
                __threadfence();
                wsync();
                if (wt == 0) atomicAdd(&f.cnt[I.stage], 1);
            } else if (I.type == IT_ACCEPT) {
                wait_stage(f, S, wt, wsync);
                if (f.trace && wt == 0) f.trace[(size_t)it * 4 + 2] = gtimer();
                AcceptSmem& A = *reinterpret_cast<AcceptSmem*>(uni);
                const bool fin = accept_body<128>(S.ac, I.tile, I.kb0, wt, A, wsync);
                if (fin) {
                    if (S.is_exit && f.early_host) {
                        f.early_host[I.tile] = S.ac.out[I.tile];   // mapped pinned host memory
                        __threadfence_system();
                    }
                    __threadfence();
                    const int old = atomicAdd(&f.cnt[I.stage], 1);
                    if (S.is_exit && f.early_flag && old == S.target - 1) {
                        __threadfence_system();
                        *reinterpret_cast<volatile uint64_t*>(f.early_flag) = *f.seq;
                        __threadfence_system();
                    }
                }
                wsync();
            } else if (I.type == IT_EMBED) {
                const EmbedArgs& em = S.em;
                const int m = I.tile;
                const int tok = em.tok[m];
                for (int t = 0; t < em.d / 128; ++t) {
                    const int k = t * 128 + wt;
                    const float hv = __bfloat162float(reinterpret_cast<const bf16*>(em.embed)[(size_t)tok * em.d + k]);
                    const float gk = __bfloat162float(reinterpret_cast<const bf16*>(em.gain)[k]);
                    em.h[(size_t)m * em.d + k] = hv;
                    reinterpret_cast<bf16*>(em.u)[(size_t)m * em.d + k] = __float2bfloat16_rn(hv * gk);
                    const float s = warp_sum(hv * hv);
                    if (lane == 0) E.sRed[wt >> 5] = s;
                    wsync();
                    if (wt == 0) em.ssq[(size_t)t * em.MP + m] = (E.sRed[0] + E.sRed[1]) + (E.sRed[2] + E.sRed[3]);
                    wsync();
                }
                fence_proxy_async_global();
                __threadfence();
                wsync();
                if (wt == 0) atomicAdd(&f.cnt[I.stage], 1);
            }
            if (f.trace && wt == 0) f.trace[(size_t)it * 4 + 3] = gtimer();
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) tmem_dealloc(tmem, C::TCOLS);
}

// ------------------------------------------------------------------------ host
template <int TN, int D>
static cudaError_t launch_td(const FArgs& a, int grid, cudaStream_t st) {
    using C = FCfg<TN, D>;
    static bool attr = false;
    if (!attr) {
        cudaError_t e = cudaFuncSetAttribute(fused_step_kernel<TN, D>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             C::SMEM);
        if (e != cudaSuccess) return e;
        e = cudaFuncSetAttribute(fused_step_kernel<TN, D>, cudaFuncAttributePreferredSharedMemoryCarveout,
                                 cudaSharedmemCarveoutMaxShared);
        if (e != cudaSuccess) return e;
        attr = true;
        if (getenv("SV_FUSED_DEBUG")) {
            int nb = 0;
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, fused_step_kernel<TN, D>, F_THREADS, C::SMEM);
            cudaFuncAttributes fa;
            cudaFuncGetAttributes(&fa, fused_step_kernel<TN, D>);
            fprintf(stderr, "fused<%d,%d>: smem %d (static %zu) regs %d -> %d blocks/SM, grid %d\n", TN, D, C::SMEM,
                    fa.sharedSizeBytes, fa.numRegs, nb, grid);
        }
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid, 1, 1);
    cfg.blockDim = dim3(F_THREADS, 1, 1);
    cfg.dynamicSmemBytes = C::SMEM;
    cfg.stream = st;
    cudaLaunchAttribute attrs[1];
    attrs[0].id = cudaLaunchAttributeCooperative;   // co-residency of all CTAs (spin waits)
    attrs[0].val.cooperative = getenv("SV_FUSED_NONCOOP") ? 0 : 1;   // (experiment: the occupancy API
                                                                      // under-counts 2-CTA/SM tcgen05 grids)
    cfg.attrs = attrs;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, fused_step_kernel<TN, D>, a);
}

template <int TN>
static cudaError_t launch_t(const FArgs& a, int D, int grid, cudaStream_t st) {
    switch (D) {
        case 32: return launch_td<TN, 32>(a, grid, st);
        case 64: return launch_td<TN, 64>(a, grid, st);
        case 128: return launch_td<TN, 128>(a, grid, st);
    }
    return cudaErrorInvalidValue;
}

cudaError_t fused_launch(const FusedPlan* p, cudaStream_t st) {
    cudaError_t e = cudaMemsetAsync(p->d_cnt, 0, p->cnt_ints * sizeof(int), st);
    if (e != cudaSuccess) return e;
    FArgs a;
    a.stages = p->d_stages;
    a.items = p->d_items;
    a.item_start = p->d_item_start;
    a.seg_slots = p->d_seg_slots;
    a.cnt = p->d_cnt;
    a.tile_cnt = p->d_tile_cnt;
    a.ws_main = p->ws_main;
    a.ws_exit = p->ws_exit;
    a.early_host = p->early_host_dev;
    a.early_flag = p->early_flag_dev;
    a.seq = p->seq_dev;
    a.trace = p->d_trace;
    switch (p->tile_n) {
        case 16: return launch_t<16>(a, p->head_dim, p->num_ctas, st);
        case 32: return launch_t<32>(a, p->head_dim, p->num_ctas, st);
        case 64: return launch_t<64>(a, p->head_dim, p->num_ctas, st);
        case 128: return launch_t<128>(a, p->head_dim, p->num_ctas, st);
        case 256: return launch_t<256>(a, p->head_dim, p->num_ctas, st);
    }
    return cudaErrorInvalidValue;
}

cudaError_t fused_build(FusedPlan* P, std::vector<FStage>& stages, int num_ctas, int tile_n, int head_dim) {
    const int NS = (int)stages.size();
    std::vector<std::vector<FItem>> per(num_ctas);
    std::vector<int> seg_slots;
    int tiles_total = 0, rr = 0;
    auto rr_push = [&](const FItem& it) {
        per[rr % num_ctas].push_back(it);
        ++rr;
    };
    for (int si = 0; si < NS; ++si) {
        FStage& S = stages[si];
        if (S.dep >= 0) S.dep_target = stages[S.dep].target;
        FItem base;
        memset(&base, 0, sizeof(base));
        base.stage = (int16_t)si;
        base.type = (int16_t)S.type;
        base.slot = -1;
        base.nsegs = 1;
        if (S.type == IT_GEMM) {
            const int T = S.nt_n * S.nt_m, KB = S.kblocks;
            const long long U = (long long)T * KB;
            S.tile_base = tiles_total;
            tiles_total += T;
            S.target = T;
            std::vector<std::vector<int>> tile_slots(T);
            std::vector<std::pair<int, size_t>> where;   // (cta, index in per[cta]) of each new item
            for (int c = 0; c < num_ctas; ++c) {
                const long long s = U * c / num_ctas, e = U * (c + 1) / num_ctas;
                bool first = true;
                for (long long u = s; u < e;) {
                    const int t = (int)(u / KB), k0 = (int)(u % KB);
                    const int k1 = (int)std::min<long long>(KB, k0 + (e - u));
                    FItem it = base;
                    it.tile = t;
                    it.kb0 = k0;
                    it.kb1 = k1;
                    it.slot = c * 2 + (first ? 0 : 1);
                    first = false;
                    tile_slots[t].push_back(it.slot);
                    per[c].push_back(it);
                    where.push_back({c, per[c].size() - 1});
                    u += k1 - k0;
                }
            }
            std::vector<int> tile_first(T, 0);
            for (int t = 0; t < T; ++t) {
                tile_first[t] = (int)seg_slots.size();
                if (tile_slots[t].size() > 1)
                    for (int sl : tile_slots[t]) seg_slots.push_back(sl);
            }
            for (auto& w : where) {
                FItem& it = per[w.first][w.second];
                it.nsegs = (int)tile_slots[it.tile].size();
                it.seg_first = tile_first[it.tile];
                if (it.nsegs == 1) it.slot = -1;
            }
        } else if (S.type == IT_ATTN) {
            const int BH = S.at.B * S.at.n_heads;
            S.target = BH;
            for (int c = 0; c < S.at.nchunk; ++c)
                for (int bh = 0; bh < BH; ++bh) {
                    FItem it = base;
                    it.tile = bh;
                    it.kb0 = c;
                    rr_push(it);
                }
        } else if (S.type == IT_STATS) {
            const int rows = S.ac.B * S.ac.G;
            S.target = rows * S.ac.nch;
            for (int r = 0; r < rows; ++r)
                for (int c = 0; c < S.ac.nch; ++c) {
                    FItem it = base;
                    it.tile = r;
                    it.kb0 = c;
                    rr_push(it);
                }
        } else if (S.type == IT_ACCEPT) {
            S.target = S.ac.B;
            for (int b = 0; b < S.ac.B; ++b)
                for (int c = 0; c < S.ac.nch; ++c) {
                    FItem it = base;
                    it.tile = b;
                    it.kb0 = c;
                    rr_push(it);
                }
        } else if (S.type == IT_EMBED) {
            S.target = S.em.M;
            for (int m = 0; m < S.em.M; ++m) {
                FItem it = base;
                it.tile = m;
                rr_push(it);
            }
        }
    }
    // flatten
    std::vector<FItem> items;
    std::vector<int> start(num_ctas + 1, 0);
    for (int c = 0; c < num_ctas; ++c) {
        start[c] = (int)items.size();
        items.insert(items.end(), per[c].begin(), per[c].end());
    }
    start[num_ctas] = (int)items.size();
    if (seg_slots.empty()) seg_slots.push_back(0);
    P->tile_n = tile_n;
    P->head_dim = head_dim;
    P->num_ctas = num_ctas;
    P->n_stages = NS;
    P->n_items = (int)items.size();
    P->cnt_ints = (size_t)NS + tiles_total;
    cudaError_t e;
#define FB_ALLOC(ptr, bytes)                                         \
    if ((e = cudaMalloc((void**)&(ptr), (bytes))) != cudaSuccess) return e;
    FB_ALLOC(P->d_stages, sizeof(FStage) * NS);
    FB_ALLOC(P->d_items, sizeof(FItem) * std::max<size_t>(1, items.size()));
    FB_ALLOC(P->d_item_start, sizeof(int) * (num_ctas + 1));
    FB_ALLOC(P->d_seg_slots, sizeof(int) * seg_slots.size());
    FB_ALLOC(P->d_cnt, sizeof(int) * P->cnt_ints);
    FB_ALLOC(P->ws_main, sizeof(float) * 2 * num_ctas * tile_n * 128);
    FB_ALLOC(P->ws_exit, sizeof(float) * 2 * num_ctas * tile_n * 128);
#undef FB_ALLOC
    P->d_tile_cnt = P->d_cnt + NS;
    P->h_items = items;
    P->h_start = start;
    if (getenv("SV_TRACE")) {
        if ((e = cudaMalloc((void**)&P->d_trace, sizeof(unsigned long long) * 4 * std::max<size_t>(1, items.size()))))
            return e;
        cudaMemset(P->d_trace, 0, sizeof(unsigned long long) * 4 * std::max<size_t>(1, items.size()));
    }
    if ((e = cudaMemcpy(P->d_stages, stages.data(), sizeof(FStage) * NS, cudaMemcpyHostToDevice))) return e;
    if (!items.empty() &&
        (e = cudaMemcpy(P->d_items, items.data(), sizeof(FItem) * items.size(), cudaMemcpyHostToDevice)))
        return e;
    if ((e = cudaMemcpy(P->d_item_start, start.data(), sizeof(int) * (num_ctas + 1), cudaMemcpyHostToDevice)))
        return e;
    if ((e = cudaMemcpy(P->d_seg_slots, seg_slots.data(), sizeof(int) * seg_slots.size(), cudaMemcpyHostToDevice)))
        return e;
    return cudaSuccess;
}

// Timeline of the last step (SV_TRACE=<path>): one CSV row per work item.
void fused_dump_trace(const FusedPlan* p, const char* path) {
    if (!p->d_trace || !path) return;
    std::vector<unsigned long long> t(4 * p->h_items.size());
    if (cudaMemcpy(t.data(), p->d_trace, t.size() * 8, cudaMemcpyDeviceToHost) != cudaSuccess) return;
    FILE* fp = fopen(path, "w");
    if (!fp) return;
    fprintf(fp, "cta,idx,type,stage,tile,kb0,kb1,nsegs,t_a,t_b,t_work,t_end\n");
    for (int c = 0; c < p->num_ctas; ++c)
        for (int i = p->h_start[c]; i < p->h_start[c + 1]; ++i) {
            const FItem& it = p->h_items[i];
            fprintf(fp, "%d,%d,%d,%d,%d,%d,%d,%d,%llu,%llu,%llu,%llu\n", c, i, it.type, it.stage, it.tile, it.kb0,
                    it.kb1, it.nsegs, t[4 * i], t[4 * i + 1], t[4 * i + 2], t[4 * i + 3]);
        }
    fclose(fp);
}

void fused_free(FusedPlan* p) {
    void* ptrs[] = {p->d_stages, p->d_items, p->d_item_start, p->d_seg_slots, p->d_cnt, p->ws_main, p->ws_exit,
                    p->d_trace};
    for (void* q : ptrs)
        if (q) cudaFree(q);
}

}  // namespace sv
