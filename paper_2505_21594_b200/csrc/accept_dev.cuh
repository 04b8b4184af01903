// accept_dev.cuh — device bodies of K5/K6 (vocabulary statistics, Leviathan
// acceptance, residual / bonus race, rollback length), shared by the per-op
// kernels (accept.cu).
//
// Letters: p = target (softmax of the logits), q = draft distribution.
// Rule (R2, Eq. 2, adopted from Leviathan):
//   row r = 0..gamma of a request's logits scores draft x_{r+1};
//   greedy  : accept x_j iff x_j == argmax z_{j-1} (lowest index); next = argmax z_delta
//   sampling: accept x_j iff u_j < p_{j-1}(x_j) / q_j(x_j), u_j = Philox(purpose 0, row j-1);
//             next = argmax_v w_v / E_v, E_v = -ln u_v (Philox purpose 1, row delta),
//             w = max(0, p_delta - q_{delta+1}) if delta < gamma else p_gamma
//             (fallback w = p_delta if the residual is all zero, R13).
//   score s = max_{r<=delta} max_v p_r(v) (Eq. 4, Alg-S PAPER.md:1104).
//   rollback: new_len = ctx + 1 + delta (no data moves).
#pragma once
#include <cfloat>
#include <climits>

#include "common.cuh"
#include "kernels.h"

namespace sv {

struct Stat {
    float m1, m2, sum;
    int idx;
};

__device__ __forceinline__ void stat_push(Stat& s, float v, int i) {
    if (v > s.m1) {
        s.m2 = s.m1;
        s.sum = s.sum * expf(s.m1 - v) + 1.0f;
        s.m1 = v;
        s.idx = i;
    } else {
        if (v > s.m2) s.m2 = v;   // v == m1 (a tie) makes the top-2 gap 0
        s.sum += expf(v - s.m1);
    }
}

__device__ __forceinline__ Stat stat_merge(const Stat& A, const Stat& B) {
    Stat r;
    if (A.m1 > B.m1) {
        r.m1 = A.m1; r.idx = A.idx; r.m2 = fmaxf(A.m2, B.m1);
        r.sum = A.sum + B.sum * expf(B.m1 - A.m1);
    } else if (B.m1 > A.m1) {
        r.m1 = B.m1; r.idx = B.idx; r.m2 = fmaxf(B.m2, A.m1);
        r.sum = B.sum + A.sum * expf(A.m1 - B.m1);
    } else {
        r.m1 = A.m1; r.idx = min(A.idx, B.idx);
        r.m2 = (A.idx == INT_MAX || B.idx == INT_MAX) ? fmaxf(A.m2, B.m2) : A.m1;
        r.sum = A.sum + B.sum;
    }
    return r;
}

__device__ __forceinline__ Stat stat_shfl(const Stat& s, int o) {
    return Stat{__shfl_xor_sync(0xffffffffu, s.m1, o), __shfl_xor_sync(0xffffffffu, s.m2, o),
                __shfl_xor_sync(0xffffffffu, s.sum, o), __shfl_xor_sync(0xffffffffu, s.idx, o)};
}

struct Race {
    float k1, k2, f1;
    int v1, fv1;
};

__device__ __forceinline__ void race_push(Race& r, float key, float fkey, int v) {
    if (key > r.k1) {
        r.k2 = r.k1; r.k1 = key; r.v1 = v;
    } else if (key > r.k2) {
        r.k2 = key;
    }
    if (fkey > r.f1) { r.f1 = fkey; r.fv1 = v; }
}

__device__ __forceinline__ Race race_merge(const Race& A, const Race& B) {
    Race r;
    const bool a_wins = (A.k1 > B.k1) || (A.k1 == B.k1 && A.v1 < B.v1);
    if (a_wins) { r.k1 = A.k1; r.v1 = A.v1; r.k2 = fmaxf(A.k2, B.k1); }
    else        { r.k1 = B.k1; r.v1 = B.v1; r.k2 = fmaxf(B.k2, A.k1); }
    const bool fa = (A.f1 > B.f1) || (A.f1 == B.f1 && A.fv1 < B.fv1);
    r.f1 = fa ? A.f1 : B.f1;
    r.fv1 = fa ? A.fv1 : B.fv1;
    return r;
}

__device__ __forceinline__ Race race_shfl(const Race& s, int o) {
    return Race{__shfl_xor_sync(0xffffffffu, s.k1, o), __shfl_xor_sync(0xffffffffu, s.k2, o),
                __shfl_xor_sync(0xffffffffu, s.f1, o), __shfl_xor_sync(0xffffffffu, s.v1, o),
                __shfl_xor_sync(0xffffffffu, s.fv1, o)};
}

struct AcceptSmem {
    float sM[SV_MAX_GAMMA + 1], sSum[SV_MAX_GAMMA + 1], sM2[SV_MAX_GAMMA + 1];
    int sA[SV_MAX_GAMMA + 1];
    float sQx[SV_MAX_GAMMA], sU[SV_MAX_GAMMA], sRatio[SV_MAX_GAMMA];   // per drafted position
    int s_delta, s_status, s_last;
    float s_margin;
    Stat wst[8];
    Race wrc[8];
};

// Vocabulary chunk c of logits row `row`: max, lowest argmax, second max,
// sum exp(z - max).  NT threads (multiple of 32, <= 256), `sync` = barrier of
// exactly those threads.  Fixed reduction tree -> deterministic.
template <int NT, class Sync>
__device__ void row_stats_body(const AcceptArgs& a, int row, int c, int tid, AcceptSmem& S, Sync sync) {
    const float* z = a.logits + (size_t)row * a.V;
    const int v0 = c * a.chunk, v1 = min(a.V, v0 + a.chunk);
    Stat s{-INFINITY, -INFINITY, 0.f, INT_MAX};
    // every load of the thread's share in flight before the first use (one L2 round
    // trip instead of one per iteration; the chunk is <= 4 float4 per thread)
    constexpr int PER = 4;
    float4 x[PER];
#pragma unroll
    for (int k = 0; k < PER; ++k) {
        const int v = v0 + (tid + k * NT) * 4;
        x[k] = v < v1 ? __ldcg(reinterpret_cast<const float4*>(z + v)) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int k = 0; k < PER; ++k) {
        const int v = v0 + (tid + k * NT) * 4;
        if (v < v1) {
            stat_push(s, x[k].x, v);
            stat_push(s, x[k].y, v + 1);
            stat_push(s, x[k].z, v + 2);
            stat_push(s, x[k].w, v + 3);
        }
    }
    for (int v = v0 + (tid + PER * NT) * 4; v < v1; v += NT * 4) {   // chunks beyond PER * NT * 4
        const float4 y = __ldcg(reinterpret_cast<const float4*>(z + v));
        stat_push(s, y.x, v);
        stat_push(s, y.y, v + 1);
        stat_push(s, y.z, v + 2);
        stat_push(s, y.w, v + 3);
    }
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) s = stat_merge(s, stat_shfl(s, o));
    if ((tid & 31) == 0) S.wst[tid >> 5] = s;
    sync();
    if (tid == 0) {
        Stat t = S.wst[0];
        for (int w = 1; w < NT / 32; ++w) t = stat_merge(t, S.wst[w]);
        a.stats[(size_t)row * a.nch + c] = RowStat{t.m1, t.m2, t.sum, t.idx};
    }
    sync();
}

// The acceptance inputs that do not depend on this step's logits, fetched before
// griddepcontrol.wait (they overlap the LM head): q_j(x_j) and the acceptance
// uniform u_j of every drafted position (one thread each, in parallel), and the
// draft rows the race may read -> L2.
template <int NT>
__device__ void accept_pre(const AcceptArgs& a, int b, int c, int tid, AcceptSmem& S) {
    const ReqDev& rq = a.req[b];
    const int gamma = a.G - 1;
    const float* q = reinterpret_cast<const float*>(rq.probs);
    if (rq.status_in != 0 || q == nullptr) return;
    if (tid < gamma) {
        S.sQx[tid] = q[(size_t)tid * a.V + rq.drafts[tid]];
        const u32x4 w = philox4x32_10(u32x4{0u, (uint32_t)tid, rq.round_id, rq.session_id},
                                      (uint32_t)rq.philox_seed, (uint32_t)(rq.philox_seed >> 32));
        S.sU[tid] = u32_to_uniform(w.x);
    }
    if (tid >= 32 && tid < 32 + gamma) {   // this CTA's vocabulary chunk of every draft row
        const int v0 = c * a.chunk, n = min(a.V, v0 + a.chunk) - v0;
        bulk_prefetch_l2(q + (size_t)(tid - 32) * a.V + v0, (uint32_t)(n * 4) & ~15u);
    }
}

// Acceptance for request b, vocabulary chunk c (accept_pre has run).  Returns
// true in exactly one thread (the one that wrote a.out[b]) over all chunks.
template <int NT, class Sync>
__device__ bool accept_body(const AcceptArgs& a, int b, int c, int tid, AcceptSmem& S, Sync sync) {
    const int G = a.G, gamma = G - 1, V = a.V;
    const ReqDev& rq = a.req[b];
    sv_exit_result* out = a.out + b;
    if (rq.status_in != 0) {
        if (c == 0 && tid == 0) {
            out->round_id = rq.round_id; out->exit_layer = a.exit_layer; out->is_final = a.is_final;
            out->status = rq.status_in; out->accepted = 0; out->new_len = rq.ctx;
            return true;
        }
        return false;
    }
    const float* q = reinterpret_cast<const float*>(rq.probs);
    const bool greedy = (q == nullptr);
    if (greedy && c != 0) return false;   // greedy needs no race

    // merge the row statistics of the vocabulary chunks: warp w takes rows w, w+8, ..,
    // lane k loads chunk k (nch <= 32, all in flight at once), a fixed butterfly tree
    // merges them (identical in every CTA of the request: deterministic)
    for (int row = tid >> 5; row < G; row += NT / 32) {
        const int k = tid & 31;
        Stat t{-INFINITY, -INFINITY, 0.f, INT_MAX};
        if (k < a.nch) {
            const float4 s4 = __ldcg(reinterpret_cast<const float4*>(a.stats + (size_t)(b * G + row) * a.nch) + k);
            t = Stat{s4.x, s4.y, s4.z, __float_as_int(s4.w)};
        }
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) t = stat_merge(t, stat_shfl(t, o));
        if (k == 0) {
            S.sM[row] = t.m1; S.sM2[row] = t.m2; S.sSum[row] = t.sum; S.sA[row] = t.idx;
        }
    }
    sync();
    gphase_mark(tid == 0 ? a.gtrace : nullptr, a.ktrace_id, 2);
    if (!greedy && tid < gamma) {   // p_{j-1}(x_j) / q_j(x_j) of every position at once
        const int x = rq.drafts[tid];
        const float zx = __ldcg(&a.logits[(size_t)(b * G + tid) * V + x]);
        const float p = expf(zx - S.sM[tid]) / S.sSum[tid];
        S.sRatio[tid] = p / S.sQx[tid];
    }
    sync();
    if (tid == 0) {
        int delta = 0, status = SV_OK;
        float margin = INFINITY;
        if (greedy) {
            for (int j = 1; j <= gamma; ++j) {
                margin = fminf(margin, S.sM[j - 1] - S.sM2[j - 1]);
                if (rq.drafts[j - 1] != S.sA[j - 1]) break;
                delta = j;
            }
            if (delta == gamma) margin = fminf(margin, S.sM[gamma] - S.sM2[gamma]);
        } else {
            for (int j = 1; j <= gamma; ++j)
                if (!(S.sQx[j - 1] > 0.f)) status = SV_E_PROTOCOL;
            if (status == SV_OK) {
                for (int j = 1; j <= gamma; ++j) {
                    const float ratio = S.sRatio[j - 1];
                    const float u = S.sU[j - 1];
                    margin = fminf(margin, fabsf(u - ratio));
                    if (!(u < ratio)) break;
                    delta = j;
                }
            }
        }
        S.s_delta = delta; S.s_status = status; S.s_margin = margin;
        gphase_mark(a.gtrace, a.ktrace_id, 3);
    }
    sync();
    const int delta = S.s_delta;
    const int status = S.s_status;
    int next = -1;
    float race_margin = INFINITY;

    if (!greedy && status == SV_OK) {
        // exponential race over this chunk of the vocabulary, row delta
        const float* z = a.logits + (size_t)(b * G + delta) * V;
        const float* qr = (delta < gamma) ? q + (size_t)delta * V : nullptr;
        const float M = S.sM[delta], inv_s = 1.0f / S.sSum[delta];
        const int v0 = c * a.chunk, v1 = min(V, v0 + a.chunk);
        const uint32_t c1 = (uint32_t)delta | (1u << 8);
        Race rc{0.f, 0.f, 0.f, INT_MAX, INT_MAX};
        // loads of the thread's share first (one round trip), then the race
        constexpr int PER = 4;
        float4 zz[PER], qq[PER];
#pragma unroll
        for (int k = 0; k < PER; ++k) {
            const int v = v0 + (tid + k * NT) * 4;
            zz[k] = v < v1 ? __ldcg(reinterpret_cast<const float4*>(z + v)) : make_float4(0.f, 0.f, 0.f, 0.f);
            qq[k] = (qr && v < v1) ? __ldg(reinterpret_cast<const float4*>(qr + v)) : make_float4(0.f, 0.f, 0.f, 0.f);
        }
        auto push4 = [&](int v, const float4& z4, const float4& q4) {
            const u32x4 w = philox4x32_10(u32x4{(uint32_t)(v >> 2), c1, rq.round_id, rq.session_id},
                                          (uint32_t)rq.philox_seed, (uint32_t)(rq.philox_seed >> 32));
            const uint32_t words[4] = {w.x, w.y, w.z, w.w};
            const float zs[4] = {z4.x, z4.y, z4.z, z4.w};
            const float qs[4] = {q4.x, q4.y, q4.z, q4.w};
#pragma unroll
            for (int t = 0; t < 4; ++t) {
                const float p = expf(zs[t] - M) * inv_s;
                const float wv = qr ? fmaxf(0.f, p - qs[t]) : p;
                const float E = -logf(u32_to_uniform(words[t]));
                race_push(rc, wv / E, p / E, v + t);
            }
        };
#pragma unroll
        for (int k = 0; k < PER; ++k) {
            const int v = v0 + (tid + k * NT) * 4;
            if (v < v1) push4(v, zz[k], qq[k]);
        }
        for (int v = v0 + (tid + PER * NT) * 4; v < v1; v += NT * 4) {   // beyond PER * NT * 4
            const float4 z4 = __ldcg(reinterpret_cast<const float4*>(z + v));
            const float4 q4 = qr ? __ldg(reinterpret_cast<const float4*>(qr + v)) : make_float4(0.f, 0.f, 0.f, 0.f);
            push4(v, z4, q4);
        }
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) rc = race_merge(rc, race_shfl(rc, o));
        if ((tid & 31) == 0) S.wrc[tid >> 5] = rc;
        sync();
        if (tid == 0) {
            Race t = S.wrc[0];
            for (int w = 1; w < NT / 32; ++w) t = race_merge(t, S.wrc[w]);
            a.race[(size_t)b * a.nch + c] = RacePart{t.k1, t.k2, t.f1, t.v1, t.fv1, {0, 0, 0}};
            S.s_last = (atomic_add_acq_rel(&a.counters[b], 1) == a.nch - 1);
            gphase_mark(a.gtrace, a.ktrace_id, 4);
        }
        sync();
        if (!S.s_last || tid >= 32) return false;
        // the last CTA merges every chunk's race part: lane k loads part k (nch <= 32);
        // race_merge is associative and commutative (max key, lowest index on ties)
        const RacePart* rp = a.race + (size_t)b * a.nch;
        Race t{0.f, 0.f, 0.f, INT_MAX, INT_MAX};
        if (tid < a.nch)
            t = Race{__ldcg(&rp[tid].k1), __ldcg(&rp[tid].k2), __ldcg(&rp[tid].f1), __ldcg(&rp[tid].v1),
                     __ldcg(&rp[tid].fv1)};
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) t = race_merge(t, race_shfl(t, o));
        if (tid != 0) return false;
        a.counters[b] = 0;
        if (t.k1 > 0.f) {
            next = t.v1;
            race_margin = (t.k2 > 0.f) ? (logf(t.k1) - logf(t.k2)) : INFINITY;
        } else {
            next = t.fv1;   // residual numerically all zero: sample from p_delta
        }
    } else {
        if (tid != 0 || c != 0) return false;
        next = S.sA[delta];
    }

    out->round_id = rq.round_id;
    out->exit_layer = a.exit_layer;
    out->is_final = a.is_final;
    out->status = status;
    if (status != SV_OK) {
        out->accepted = 0;
        out->score = 0.f; out->next_prob = 0.f; out->min_margin = 0.f;
        out->new_len = rq.ctx;
        for (int k = 0; k <= SV_MAX_GAMMA; ++k) out->tokens[k] = -1;
        return true;
    }
    out->accepted = delta;
    for (int k = 0; k <= SV_MAX_GAMMA; ++k) out->tokens[k] = (k < delta) ? rq.drafts[k] : (k == delta ? next : -1);
    float score = 0.f;
    for (int r = 0; r <= delta; ++r) score = fmaxf(score, 1.0f / S.sSum[r]);
    out->score = score;
    out->next_prob = expf(__ldcg(&a.logits[(size_t)(b * G + delta) * V + next]) - S.sM[delta]) / S.sSum[delta];
    out->min_margin = fminf(S.s_margin, race_margin);
    out->new_len = rq.ctx + 1 + delta;
    return true;
}

}  // namespace sv
