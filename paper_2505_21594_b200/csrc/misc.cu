// misc.cu — K4 embedding gather, K7 weight generator, K8 synthetic KV fill and
// a Philox test kernel.
#include "common.cuh"
#include "kernels.h"

namespace sv {

bool g_use_pdl = true;
int g_attn_nst = 0;
int g_attn_minb = 0;

// K4: h^(0) = E[token] (Eq. 3), fp32 residual; u = bf16(h * g_attn[0]);
// ssq[t][m] = sum of h^2 over the 128-column tile t (RMSNorm statistics for layer 1).
__global__ void __launch_bounds__(128) embed_kernel(const __grid_constant__ EmbedArgs a) {
    __shared__ float sRed[4];
    ktrace_mark(a.ktrace, a.ktrace_id, 0);
    pdl_launch_dependents();
    pdl_wait();
    const int m = blockIdx.x, t = blockIdx.y;
    if (a.stamps && m == 0 && t == 0 && threadIdx.x < a.n_stamps) {   // step start; ready stamps reset
        unsigned long long now = 0;                                    // (every reader is downstream)
        if (threadIdx.x == 0) asm volatile("mov.u64 %0, %globaltimer;" : "=l"(now));
        a.stamps[threadIdx.x] = now;
    }
    const int k = t * 128 + threadIdx.x;
    const int tok = a.tok[m];
    const float hv = __bfloat162float(reinterpret_cast<const bf16*>(a.embed)[(size_t)tok * a.d + k]);
    const float g = __bfloat162float(reinterpret_cast<const bf16*>(a.gain)[k]);
    a.h[(size_t)m * a.d + k] = hv;
    reinterpret_cast<bf16*>(a.u)[(size_t)m * a.d + k] = __float2bfloat16_rn(hv * g);
    const float s = warp_sum(hv * hv);
    if ((threadIdx.x & 31) == 0) sRed[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) a.ssq[(size_t)t * a.MP + m] = (sRed[0] + sRed[1]) + (sRed[2] + sRed[3]);
    ktrace_mark(a.ktrace, a.ktrace_id, 1);
}

cudaError_t embed_launch(const EmbedArgs& a, cudaStream_t st) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(a.M, a.d / 128, 1);
    cfg.blockDim = dim3(128, 1, 1);
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = g_use_pdl ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, embed_kernel, a);
}

// K7: counter-hash weights.  Physical element i of the destination maps to the
// logical (tensor id, index) of the generator:
//   GEN_PLAIN: (tid0, i)
//   GEN_QKV  : rows [sec*R, (sec+1)*R) come from tensor tid0+sec (W_q, W_k, W_v)
//   GEN_GU   : physical row 128t+w is W_gate row 64t+w (w < 64) or W_up row 64t+w-64
__global__ void gen_kernel(bf16* dst, uint64_t n, int layout, uint64_t seed, uint64_t tid0, int rows_per_sec,
                           int cols, float c, float offset) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t tid = tid0, idx = i;
        if (layout != GEN_PLAIN) {
            const uint64_t row = i / (uint64_t)cols, col = i % (uint64_t)cols;
            if (layout == GEN_QKV) {
                const uint64_t sec = row / (uint64_t)rows_per_sec;
                tid = tid0 + sec;
                idx = (row % (uint64_t)rows_per_sec) * cols + col;
            } else {
                const uint64_t t = row / 128, w = row % 128;
                tid = tid0 + (w >= 64 ? 1 : 0);
                idx = (t * 64 + (w & 63)) * cols + col;
            }
        }
        dst[i] = gen_value(gen_base(seed, tid), idx, c, offset);
    }
}

cudaError_t gen_launch(void* dst, uint64_t n, int layout, uint64_t seed, uint64_t tid0, int rows_per_sec, int cols,
                       float c, float offset, cudaStream_t st) {
    uint64_t blocks = (n + 255) / 256;
    if (blocks > 148 * 64) blocks = 148 * 64;
    gen_kernel<<<(unsigned)blocks, 256, 0, st>>>(reinterpret_cast<bf16*>(dst), n, layout, seed, tid0, rows_per_sec,
                                                  cols, c, offset);
    return cudaGetLastError();
}

// K8: synthetic KV for logical positions 0..len-1 of one session:
//   value(kv_seed, 0x100000 + 2*layer + kv, pos*d + head*Dh + dim)
// written to block blocks[pos / P], slot pos % P, layout [layer][kv][head][slot][dim].
__global__ void kvfill_kernel(bf16* pool, const int32_t* blocks, int nblocks, int len, uint64_t kv_seed,
                              int L, int H, int D, int P, float c) {
    const uint64_t per_block = (uint64_t)L * 2 * H * P * D;
    const uint64_t n = per_block * nblocks;
    const int d = H * D;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        const int bi = (int)(i / per_block);
        uint64_t r = i % per_block;
        const int dim = (int)(r % D); r /= D;
        const int slot = (int)(r % P); r /= P;
        const int head = (int)(r % H); r /= H;
        const int kv = (int)(r % 2); r /= 2;
        const int layer = (int)r;
        const int pos = bi * P + slot;
        if (pos >= len) continue;
        const uint64_t tid = 0x100000ull + 2ull * layer + kv;
        const bf16 v = gen_value(gen_base(kv_seed, tid), (uint64_t)pos * d + (uint64_t)head * D + dim, c, 0.f);
        pool[(size_t)blocks[bi] * per_block + (((size_t)layer * 2 + kv) * H + head) * (size_t)P * D +
             (size_t)slot * D + dim] = v;
    }
}

cudaError_t kvfill_launch(bf16_raw_t* pool, const int32_t* blocks, int nblocks, int len, uint64_t kv_seed,
                          int n_layers, int n_heads, int head_dim, int page_tokens, float c, cudaStream_t st) {
    kvfill_kernel<<<148 * 16, 256, 0, st>>>(reinterpret_cast<bf16*>(pool), blocks, nblocks, len, kv_seed, n_layers,
                                            n_heads, head_dim, page_tokens, c);
    return cudaGetLastError();
}

__global__ void philox_kernel(const uint32_t* in, uint32_t* out) {
    const u32x4 r = philox4x32_10(u32x4{in[0], in[1], in[2], in[3]}, in[4], in[5]);
    out[0] = r.x; out[1] = r.y; out[2] = r.z; out[3] = r.w;
}

cudaError_t philox_launch(const uint32_t* ctr_key, uint32_t* out, cudaStream_t st) {
    philox_kernel<<<1, 1, 0, st>>>(ctr_key, out);
    return cudaGetLastError();
}

}  // namespace sv
