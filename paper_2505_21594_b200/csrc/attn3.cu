// attn3.cu — K3 v3: gamma-query causal attention over the paged bf16 KV cache on
// tensor cores.
//
//   a_j = softmax(q_j K^T / sqrt(Dh)) V   over keys 0 .. ctx_b + j      (Eq. 3)
//
// Why tensor cores: with G = gamma+1 query rows the step needs 2*G*Dh MACs per
// key, i.e. 2.5 MAC per KV byte at G = 5 — ~45% of the B200's FP32 FMA peak just
// to keep up with HBM.  Q K^T and P V therefore run as mma.sync m16n8k16 bf16
// tiles (fp32 accumulate), the G query rows padded to one 16-row tile.
//
// * grid (splits, B*H); a CTA owns a contiguous run of 64-key pages; each of its
//   4 warps streams every 4th 32-key chunk with its own 2-stage cp.async ring
//   (16-byte copies into an XOR-swizzled layout, conflict-free ldmatrix); the
//   first two chunks of cached rows are requested before griddepcontrol.wait;
// * per chunk (FlashAttention-2 register pipeline): S = Q K^T (4 n-tiles x 8
//   k-steps), causal mask, online softmax in the log2 domain on the accumulator
//   fragments, P (bf16, straight from the S fragments) times V via ldmatrix.trans;
// * the 4 warps' (m, l, O) are merged through shared memory in warp order, the
//   splits of a (b, h) through global memory as tagged (value, tag) pairs, summed
//   in split order -> deterministic.
// Numerics: q and p are rounded to bf16 for the MMA (as in a bf16 model); scores,
// softmax statistics and O accumulate in fp32.
#include <cfloat>
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"

namespace sv {

constexpr int A3_D = 128;            // head dim (the tensor-core path is specialised for Dh = 128)
constexpr int A3_CHUNK = 32;         // keys per chunk
constexpr int A3_WARPS = 4;
constexpr int A3_ROWB = A3_D * 2;    // 256 B per K / V row
constexpr int A3_CHB = A3_CHUNK * A3_ROWB;              // 8 KB per K (or V) chunk
constexpr int A3_STAGE = 2 * A3_CHB;                    // K + V
template <int NST>   // ring stages per warp: 1 (default: 69 KB, two CTAs per SM, and the CTA co-resides
                     // with a neighbouring GEMM grid under programmatic dependent launch); 2, 3 (SV_ATTN_NST)
struct A3Cfg {
    static constexpr int SMEM = 1024 + A3_WARPS * NST * A3_STAGE /*rings*/ + 16 * A3_ROWB /*Q bf16*/ + 256;
};

__device__ __forceinline__ uint32_t swz(int row, int chunk16) {          // byte offset in a 256 B-row tile
    return (uint32_t)(row * A3_ROWB + ((chunk16 ^ (row & 7)) << 4));
}
__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }
__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3) : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3) : "r"(addr));
}
__device__ __forceinline__ void mma16816(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
    __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
    return *reinterpret_cast<uint32_t*>(&v);
}
#define A3_STAMP(k)                                                                                   \
    if (a.atrace && threadIdx.x == 0 && blockIdx.x == 0 && (blockIdx.y == 0 || blockIdx.y == gridDim.y - 1)) { \
        unsigned long long _t;                                                                        \
        asm volatile("mov.u64 %0, %globaltimer;" : "=l"(_t));                                         \
        a.atrace[(blockIdx.y == 0 ? 0 : 8) + (k)] = _t;                                               \
    }
// MINB = CTAs per SM the registers are budgeted for: 3 (<= 168 registers, three 69 KB
// CTAs = 12 warps per SM) or 2 (~245 registers, no spills)
template <int NST, int MINB>
__global__ void __launch_bounds__(128, MINB) attn3_kernel(const __grid_constant__ AttnArgs a) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const uint32_t s_ring = smem_u32(smem);                                   // [warp][stage][K|V] 8 KB tiles
    const uint32_t s_q = s_ring + A3_WARPS * NST * A3_STAGE;                     // Q bf16 [16][128] swizzled
    // merge scratch aliases the rings after the main loop
    float* mO = reinterpret_cast<float*>(smem);                                // [warp][16][128]
    float* mM = mO + A3_WARPS * 16 * A3_D;                                     // [warp][16]
    float* mL = mM + A3_WARPS * 16;
    float* fO = mL + A3_WARPS * 16;                                            // merged [16][128]
    float* fM = fO + 16 * A3_D;
    float* fL = fM + 16;
    __shared__ int sBlk[64];

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int g = lane >> 2, t4 = lane & 3;
    const int S = gridDim.x, r = blockIdx.x, bh = blockIdx.y;
    const int b = bh / a.n_heads, h = bh % a.n_heads;
    const int G = a.G;
    ktrace_mark(a.ktrace, a.ktrace_id, 0);
    A3_STAMP(0);
    pdl_launch_dependents();
    // lengths and page tables are host-written before the step; the cache rows
    // below ctx were written by earlier steps -> their loads are issued before
    // griddepcontrol.wait and overlap the QKV GEMM; q and the gamma+1 new rows
    // (this step's QKV epilogue) are only touched after it.
    const int ctx = a.ctx[b];
    const int Gb = a.g_rows ? a.g_rows[b] : G;          // valid query rows of this request
    const int cpre = a.ctx_pre ? a.ctx_pre[b] : ctx;    // rows written before this step
    const int T = ctx + Gb;
    const int npg = (T + 63) / 64;
    const int p0 = (int)((long long)npg * r / S), p1 = (int)((long long)npg * (r + 1) / S);
    const int np = p1 - p0;
    for (int i = tid; i < np; i += 128) sBlk[i] = a.page_table[b * a.pt_stride + p0 + i];
    __syncthreads();
    A3_STAMP(1);

    // this warp's chunks: ci = warp + 4 * it over the CTA's 2*np chunks, 2-deep ring
    const int nchunks = 2 * np;
    const int n_my = nchunks > warp ? (nchunks - warp + A3_WARPS - 1) / A3_WARPS : 0;
    const size_t plane = (size_t)a.n_heads * a.page_tokens * A3_D;
    const uint32_t wring = s_ring + warp * NST * A3_STAGE;
    auto issue = [&](int ci, int stage) {
        const int pg = ci >> 1, koff = (ci & 1) * A3_CHUNK;
        const bf16* kb = reinterpret_cast<const bf16*>(a.kv_pool) +
                         (((size_t)sBlk[pg] * a.n_layers + a.layer) * 2) * plane + (size_t)h * a.page_tokens * A3_D +
                         (size_t)koff * A3_D;
        const bf16* vb = kb + plane;
        const uint32_t dk = wring + stage * A3_STAGE, dv = dk + A3_CHB;
#pragma unroll
        for (int u = 0; u < (A3_CHUNK * 16) / 32; ++u) {      // 512 16-byte pieces per matrix
            const int piece = lane + 32 * u, row = piece >> 4, c = piece & 15;
            cp_async16(dk + swz(row, c), kb + row * A3_D + c * 8);
            cp_async16(dv + swz(row, c), vb + row * A3_D + c * 8);
        }
        cp_commit();
    };
    // chunk ci holds only cached rows iff its last key < ctx; such chunks form a
    // prefix of this warp's sequence, so commit order stays the chunk order
    int pre = 0;
    while (pre < NST && pre < n_my && (p0 * 64 + (warp + A3_WARPS * pre + 1) * A3_CHUNK) <= cpre) {
        issue(warp + A3_WARPS * pre, pre);
        ++pre;
    }
    if (tid == 32 && a.pf_ptr && a.pf_early)   // O weights -> L2 while the QKV grid drains
        cta_prefetch_l2(a.pf_ptr, a.pf_bytes, blockIdx.y * gridDim.x + blockIdx.x, gridDim.x * gridDim.y);
    pdl_wait();
    if (tid == 32 && a.pf_ptr && !a.pf_early)   // the QKV GEMM is done: pull the O weights into L2 while HBM is idle
        cta_prefetch_l2(a.pf_ptr, a.pf_bytes, blockIdx.y * gridDim.x + blockIdx.x, gridDim.x * gridDim.y);
    A3_STAMP(2);
    for (int it = pre; it < NST && it < n_my; ++it) issue(warp + A3_WARPS * it, it);

    // Q (pre-scaled by log2(e)/sqrt(Dh)) -> bf16, rows >= G zero, swizzled
    for (int i = tid; i < 16 * (A3_D / 8); i += 128) {
        const int row = i / (A3_D / 8), c = i % (A3_D / 8);
        uint32_t w[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            float lo = 0.f, hi = 0.f;
            if (row < Gb) {
                const float* qp = a.q + (size_t)(b * G + row) * a.d_model + h * A3_D + c * 8 + 2 * u;
                lo = qp[0] * a.scale_log2;
                hi = qp[1] * a.scale_log2;
            }
            w[u] = pack_bf16(lo, hi);
        }
        asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};" ::"r"(s_q + swz(row, c)), "r"(w[0]), "r"(w[1]),
                     "r"(w[2]), "r"(w[3])
                     : "memory");
    }
    __syncthreads();
    A3_STAMP(3);

    float o[16][4];
#pragma unroll
    for (int n = 0; n < 16; ++n) o[n][0] = o[n][1] = o[n][2] = o[n][3] = 0.f;
    float mrow[2] = {-INFINITY, -INFINITY}, lrow[2] = {0.f, 0.f};
    const int row0 = g, row1 = g + 8;

    for (int it = 0; it < n_my; ++it) {
        const int ci = warp + A3_WARPS * it, stage = it % NST;
        if (NST >= 3 && it + 2 < n_my)          // chunk `it` landed; later stages may still fly
            cp_wait<2>();
        else if (NST >= 2 && it + 1 < n_my)
            cp_wait<1>();
        else
            cp_wait<0>();
        __syncwarp();
        const uint32_t sk = wring + stage * A3_STAGE, sv = sk + A3_CHB;
        const int kabs0 = (p0 * 64) + ci * A3_CHUNK;
        const int valid = T - kabs0;                          // rows past the sequence end hold
        if (valid < A3_CHUNK) {                               // arbitrary bits: zero them (P = 0
            const int v0 = valid > 0 ? valid : 0;             // times NaN would poison P V)
            for (int i = lane; i < (A3_CHUNK - v0) * 16; i += 32) {
                const int row = v0 + (i >> 4), c = i & 15;
                asm volatile("st.shared.v4.b32 [%0], {%1,%1,%1,%1};" ::"r"(sk + swz(row, c)), "r"(0) : "memory");
                asm volatile("st.shared.v4.b32 [%0], {%1,%1,%1,%1};" ::"r"(sv + swz(row, c)), "r"(0) : "memory");
            }
            __syncwarp();
        }
        // ---- S = Q K^T  (16 x 32)
        float sacc[4][4];
#pragma unroll
        for (int n = 0; n < 4; ++n) sacc[n][0] = sacc[n][1] = sacc[n][2] = sacc[n][3] = 0.f;
#pragma unroll
        for (int ks = 0; ks < 8; ++ks) {
            uint32_t qa[4];                                   // Q A-fragment of k-step ks (re-read: registers)
            {
                const int row = (lane & 7) + 8 * ((lane >> 3) & 1), c = 2 * ks + (lane >> 4);
                ldsm_x4(s_q + swz(row, c), qa[0], qa[1], qa[2], qa[3]);
            }
#pragma unroll
            for (int np2 = 0; np2 < 2; ++np2) {              // n-tiles 2*np2, 2*np2+1
                uint32_t b0, b1, b2, b3;
                const int key = 16 * np2 + 8 * (lane >> 4) + (lane & 7), c = 2 * ks + ((lane >> 3) & 1);
                ldsm_x4(sk + swz(key, c), b0, b1, b2, b3);
                mma16816(sacc[2 * np2], qa, b0, b1);
                mma16816(sacc[2 * np2 + 1], qa, b2, b3);
            }
        }
        // ---- causal mask + online softmax (rows g and g+8 of this thread)
        float mnew[2] = {mrow[0], mrow[1]};
#pragma unroll
        for (int n = 0; n < 4; ++n)
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int j = (e < 2) ? row0 : row1;
                const int kabs = kabs0 + 8 * n + 2 * t4 + (e & 1);
                if (j >= Gb || kabs > ctx + j) sacc[n][e] = -INFINITY;
                mnew[e >> 1] = fmaxf(mnew[e >> 1], sacc[n][e]);
            }
#pragma unroll
        for (int x = 0; x < 2; ++x) {
            mnew[x] = fmaxf(mnew[x], __shfl_xor_sync(0xffffffffu, mnew[x], 1));
            mnew[x] = fmaxf(mnew[x], __shfl_xor_sync(0xffffffffu, mnew[x], 2));
        }
        float alpha[2], psum[2] = {0.f, 0.f};
#pragma unroll
        for (int x = 0; x < 2; ++x) alpha[x] = (mrow[x] == -INFINITY) ? 0.f : exp2f(mrow[x] - mnew[x]);
        uint32_t pa[2][4];                                    // P as A fragments (2 k-steps of 16 keys)
#pragma unroll
        for (int n = 0; n < 4; ++n) {
            float p[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const float m = mnew[e >> 1];
                p[e] = (sacc[n][e] == -INFINITY) ? 0.f : exp2f(sacc[n][e] - m);
                psum[e >> 1] += p[e];
            }
            // S n-tile n -> A fragment of k-step n/2: even tile -> regs 0,1; odd tile -> regs 2,3
            pa[n >> 1][(n & 1) * 2 + 0] = pack_bf16(p[0], p[1]);
            pa[n >> 1][(n & 1) * 2 + 1] = pack_bf16(p[2], p[3]);
        }
#pragma unroll
        for (int x = 0; x < 2; ++x) {
            psum[x] += __shfl_xor_sync(0xffffffffu, psum[x], 1);
            psum[x] += __shfl_xor_sync(0xffffffffu, psum[x], 2);
            lrow[x] = lrow[x] * alpha[x] + psum[x];
            mrow[x] = mnew[x];
        }
#pragma unroll
        for (int n = 0; n < 16; ++n) {
            o[n][0] *= alpha[0];
            o[n][1] *= alpha[0];
            o[n][2] *= alpha[1];
            o[n][3] *= alpha[1];
        }
        // ---- O += P V  (16 x 128), V via ldmatrix.trans
#pragma unroll
        for (int kk = 0; kk < 2; ++kk) {
#pragma unroll
            for (int nd = 0; nd < 16; nd += 2) {
                uint32_t b0, b1, b2, b3;
                const int key = 16 * kk + 8 * ((lane >> 3) & 1) + (lane & 7), c = nd + (lane >> 4);
                ldsm_x4_t(sv + swz(key, c), b0, b1, b2, b3);
                mma16816(o[nd], pa[kk], b0, b1);
                mma16816(o[nd + 1], pa[kk], b2, b3);
            }
        }
        __syncwarp();
        if (it + NST < n_my) issue(ci + NST * A3_WARPS, stage);   // refill the stage just consumed
    }

    // ---- merge the 4 warps (warp order) through shared memory (aliases the rings)
    __syncthreads();
    A3_STAMP(4);
#pragma unroll
    for (int n = 0; n < 16; ++n) {
        const int d = 8 * n + 2 * t4;
        mO[(warp * 16 + row0) * A3_D + d] = o[n][0];
        mO[(warp * 16 + row0) * A3_D + d + 1] = o[n][1];
        mO[(warp * 16 + row1) * A3_D + d] = o[n][2];
        mO[(warp * 16 + row1) * A3_D + d + 1] = o[n][3];
    }
    if (t4 == 0) {
        mM[warp * 16 + row0] = mrow[0];
        mM[warp * 16 + row1] = mrow[1];
        mL[warp * 16 + row0] = lrow[0];
        mL[warp * 16 + row1] = lrow[1];
    }
    __syncthreads();
    if (tid < 16) {
        float M = -INFINITY;
        for (int w = 0; w < A3_WARPS; ++w) M = fmaxf(M, mM[w * 16 + tid]);
        float L = 0.f;
        for (int w = 0; w < A3_WARPS; ++w) {
            const float m = mM[w * 16 + tid];
            const float wgt = (m == -INFINITY) ? 0.f : exp2f(m - M);
            mM[w * 16 + tid] = wgt;                            // reuse as the warp weight
            L = fmaf(mL[w * 16 + tid], wgt, L);
        }
        fM[tid] = M;
        fL[tid] = L;
    }
    __syncthreads();
    A3_STAMP(5);
    for (int i = tid; i < Gb * A3_D; i += 128) {
        const int j = i / A3_D, d = i % A3_D;
        float O = 0.f;
        for (int w = 0; w < A3_WARPS; ++w) O = fmaf(mO[(w * 16 + j) * A3_D + d], mM[w * 16 + j], O);
        if (S == 1)
            reinterpret_cast<bf16*>(a.out)[(size_t)(b * G + j) * a.d_model + h * A3_D + d] =
                __float2bfloat16_rn(O / fL[j]);
        else
            fO[j * A3_D + d] = O;
    }
    if (S == 1) {
        ktrace_mark(a.ktrace, a.ktrace_id, 1);
        return;
    }
    {   // ---- the splits of (b, h) through global memory as (value, tag) pairs: every
        // split stores its (m, l, O) with single 64-bit relaxed stores (no fence), then
        // merges a 1/S slice of the G x 128 outputs, polling the S partials of its
        // elements until they carry this launch's tag; sum in split order 0..S-1
        // (deterministic).  No cluster: the CTAs need not be co-scheduled.
        const uint32_t tag = (*a.epoch << 10) | (uint32_t)(a.launch_id & 1023);
        const size_t pstride = 16 * A3_D + 32;                // pairs per split partial
        uint64_t* mine = a.part + ((size_t)bh * S + r) * pstride;
        for (int i = tid; i < Gb * A3_D; i += 128) st_relaxed_b64(&mine[i], ((uint64_t)tag << 32) | __float_as_uint(fO[i]));
        if (tid < Gb) {
            st_relaxed_b64(&mine[16 * A3_D + 2 * tid], ((uint64_t)tag << 32) | __float_as_uint(fM[tid]));
            st_relaxed_b64(&mine[16 * A3_D + 2 * tid + 1], ((uint64_t)tag << 32) | __float_as_uint(fL[tid]));
        }
        A3_STAMP(6);
        const uint64_t* all = a.part + (size_t)bh * S * pstride;
        for (int i = r * 128 + tid; i < Gb * A3_D; i += S * 128) {
            const int j = i / A3_D, d = i % A3_D;
            uint64_t xm[8], xl[8], xo[8];
            bool ok;
            uint32_t n = 0;
            do {   // all 3 x S pairs in flight; again (L2 hits) until all are tagged
                ok = true;
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    const uint64_t* pq = all + (size_t)q * pstride;
                    xm[q] = q < S ? ld_relaxed_b64(&pq[16 * A3_D + 2 * j]) : ((uint64_t)tag << 32);
                    xl[q] = q < S ? ld_relaxed_b64(&pq[16 * A3_D + 2 * j + 1]) : ((uint64_t)tag << 32);
                    xo[q] = q < S ? ld_relaxed_b64(&pq[j * A3_D + d]) : ((uint64_t)tag << 32);
                }
#pragma unroll
                for (int q = 0; q < 8; ++q)
                    ok = ok && (uint32_t)(xm[q] >> 32) == tag && (uint32_t)(xl[q] >> 32) == tag &&
                         (uint32_t)(xo[q] >> 32) == tag;
                if (++n > SV_SPIN_LIMIT) __trap();
            } while (!ok);
            float mq[8], lq[8], oq[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                mq[q] = q < S ? __uint_as_float((uint32_t)xm[q]) : -INFINITY;
                lq[q] = q < S ? __uint_as_float((uint32_t)xl[q]) : 0.f;
                oq[q] = q < S ? __uint_as_float((uint32_t)xo[q]) : 0.f;
            }
            float M = -INFINITY;
#pragma unroll
            for (int q = 0; q < 8; ++q) M = fmaxf(M, mq[q]);
            float L = 0.f, O = 0.f;
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                if (mq[q] == -INFINITY) continue;
                const float wq = exp2f(mq[q] - M);
                L = fmaf(lq[q], wq, L);
                O = fmaf(oq[q], wq, O);
            }
            reinterpret_cast<bf16*>(a.out)[(size_t)(b * G + j) * a.d_model + h * A3_D + d] =
                __float2bfloat16_rn(O / L);
        }
    }
    ktrace_mark(a.ktrace, a.ktrace_id, 1);
    A3_STAMP(7);
}

int attn3_splits(int B, int H, int max_pages, int num_sms) {
    // (sized when the ring was 2-stage, one 136 KB CTA per SM) ONE wave of clusters: the largest power-of-two
    // cluster size whose clusters all fit (5-CTA clusters pack badly into the
    // 16-20-SM GPCs: measured 26 of 32 clusters resident -> two waves)
    const int units = B * H;
    int s = 1;
    while (s < 8 && units * (2 * s) <= (num_sms * 7) / 8 && 2 * s <= max_pages) s *= 2;
    // short contexts: 8-CTA clusters with the 1-stage (69 KB) ring, up to two CTAs
    // per SM, <= 2 chunks per CTA — measured C2 (B=1, ctx 512): attention ends
    // 9.5 us after the QKV GEMM instead of 11.3 us with 4 x 136 KB
    if (units * 8 <= 2 * num_sms && max_pages >= 8) s = 8;
    return s;
}

template <int NST, int MINB>
static cudaError_t attn3_launch_t(const AttnArgs& a, int splits, cudaStream_t st) {
    static bool attr = false;
    if (!attr) {
        cudaError_t e =
            cudaFuncSetAttribute(attn3_kernel<NST, MINB>, cudaFuncAttributeMaxDynamicSharedMemorySize, A3Cfg<NST>::SMEM);
        if (e != cudaSuccess) return e;
        if (!getenv("SV_NO_CARVEOUT")) {
            e = cudaFuncSetAttribute(attn3_kernel<NST, MINB>, cudaFuncAttributePreferredSharedMemoryCarveout,
                                     cudaSharedmemCarveoutMaxShared);
            if (e != cudaSuccess) return e;
        }
        attr = true;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(splits, a.B * a.n_heads, 1);
    cfg.blockDim = dim3(128, 1, 1);
    cfg.dynamicSmemBytes = A3Cfg<NST>::SMEM;
    cfg.stream = st;
    cudaLaunchAttribute at[2];
    int na = 0;
    if (a.cluster_launch) {   // the splits of (b, h) co-scheduled as one cluster (placement only)
        at[na].id = cudaLaunchAttributeClusterDimension;
        at[na].val.clusterDim.x = splits;
        at[na].val.clusterDim.y = 1;
        at[na].val.clusterDim.z = 1;
        ++na;
    }
    if (g_use_pdl) {
        at[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[na].val.programmaticStreamSerializationAllowed = 1;
        ++na;
    }
    cfg.attrs = at;
    cfg.numAttrs = na;
    return cudaLaunchKernelEx(&cfg, attn3_kernel<NST, MINB>, a);
}

// max_ctx_len: the longest cached context of the batch (sizes the per-warp ring)
cudaError_t attn3_launch(const AttnArgs& a, int splits, int max_ctx_len, cudaStream_t st) {
    if (a.head_dim != A3_D || a.page_tokens != 64 || a.G > 16 || splits < 1 || splits > 8 || a.num_sms < 1)
        return cudaErrorInvalidValue;
    // a CTA stages its page list in sBlk[64]: at most 64 pages per split
    const int max_pages = (max_ctx_len + a.G + 63) / 64;
    if ((max_pages + splits - 1) / splits > 64) return cudaErrorInvalidValue;
    // 1-stage ring at every context length: 69 KB, two CTAs (8 warps) per SM, whose
    // loads overlap each other's tensor-core work — measured C4 45.8 -> 42.9 ms and
    // C5 8.30 -> 7.88 ms against the 2-stage ring at one CTA (4 warps) per SM
    if (g_attn_nst == 2) return attn3_launch_t<2, 1>(a, splits, st);
    if (g_attn_nst == 3) return attn3_launch_t<3, 1>(a, splits, st);
    // registers for three CTAs per SM when the whole grid is resident at two per SM
    // anyway (ctas <= 2 x SMs: the lower register budget leaves room for the
    // neighbouring GEMM grids' CTAs under PDL) or when there are >= 4 waves of
    // three (the tail wave matters little); two otherwise.  Measured (ms, three vs
    // two): C2 (256 CTAs) 3.056 vs 3.072; C4 per-GPU batch 256 / 128 / 64 (18.4 /
    // 9.2 / 4.6 waves of 444) 42.8 vs 43.5, 22.71 vs 22.80, 14.94 vs 15.06; batch 32
    // (2.3 waves) 10.24 vs 10.19; C5 (512 CTAs, 1.15 waves of 444) 8.62 vs 7.89.
    // The band 2 x SMs < ctas <= 3 x SMs (one resident wave at three) is unmeasured
    // and keeps two.
    const int sms = a.num_sms;
    const double ctas = (double)splits * a.B * a.n_heads;
    bool three = ctas <= 2.0 * sms || ctas >= 4.0 * 3 * sms;
    if (g_attn_minb) three = g_attn_minb == 3;
    return three ? attn3_launch_t<1, 3>(a, splits, st) : attn3_launch_t<1, 2>(a, splits, st);
}

}  // namespace sv
