// attn.cu — K3 as a per-op kernel: one CTA per (request, head, 64-key page);
// the body (attn_dev.cuh) stages the page in shared memory with all loads in
// flight, computes the G x 64 score block, page softmax and P.V, and the last
// page finisher of a (request, head) merges the pages in page order (fixed
// order -> deterministic).  Memory bound (AI ~ G FLOP/B): CUDA cores.
#include "attn_dev.cuh"

namespace sv {

struct AttnCtaSync {
    __device__ void operator()() const { __syncthreads(); }
};

template <int D>
__global__ void __launch_bounds__(128) attn_kernel(const __grid_constant__ AttnArgs a) {
    __shared__ AttnSmem<D> S;
    pdl_launch_dependents();   // the next GEMM may start streaming its weights now
    pdl_wait();
    ktrace_mark(a.ktrace, a.ktrace_id, 0);
    attn_page_body<D>(a, blockIdx.x, blockIdx.y, threadIdx.x, S, AttnCtaSync{});
    ktrace_mark(a.ktrace, a.ktrace_id, 1);
}

template <int D>
static cudaError_t launch_d(const AttnArgs& a, cudaStream_t st) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(a.B * a.n_heads, a.nchunk, 1);
    cfg.blockDim = dim3(128, 1, 1);
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = g_use_pdl ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, attn_kernel<D>, a);
}

cudaError_t attn_launch(const AttnArgs& a, cudaStream_t st) {
    if (a.page_tokens != KPAGE || a.G > GMAX || a.nchunk > MAXCH) return cudaErrorInvalidValue;
    switch (a.head_dim) {
        case 32: return launch_d<32>(a, st);
        case 64: return launch_d<64>(a, st);
        case 128: return launch_d<128>(a, st);
    }
    return cudaErrorInvalidValue;
}

}  // namespace sv
