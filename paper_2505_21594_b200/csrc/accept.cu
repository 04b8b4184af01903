// accept.cu — K5/K6 as two per-op kernels (bodies in accept_dev.cuh):
//   row_stats_kernel: grid (rows, chunks)     — vocabulary statistics per chunk
//   accept_kernel   : grid (requests, chunks) — delta decision, race, result
#include "accept_dev.cuh"

namespace sv {

// Threads per CTA: 256 when the grid is a single wave (batch 1: the race over a
// 1024-entry chunk is ALU-latency bound, more threads per chunk finish sooner);
// 64 (4 float4 of a chunk each) when there are more than two CTAs per SM — up to 32
// CTAs per SM then hide the per-chunk load latency.  Measured: C4 final acceptance
// 345 -> 175 us, C4 8-GPU shard 44 -> 28 us, C5 27 -> 24 us; at C2 64 threads
// would cost 12 -> 16 us (final) and 26 -> 47 us (exit).
constexpr int ACC_THREADS_WIDE = 256, ACC_THREADS_NARROW = 64;
constexpr int ACC_CHUNK = 1024;   // 32 CTAs per request at V = 32000: the race is ALU-latency bound

// vocabulary chunks of ACC_CHUNK (a multiple of it for V > 32 * ACC_CHUNK): at most
// 32 chunks, so a warp merges a row's chunk statistics / race parts in one step
int accept_chunks(int V, int* chunk) {
    const int mult = (V + 32 * ACC_CHUNK - 1) / (32 * ACC_CHUNK);
    *chunk = ACC_CHUNK * (mult > 0 ? mult : 1);
    return (V + *chunk - 1) / *chunk;
}

struct CtaSync {
    __device__ void operator()() const { __syncthreads(); }
};

template <int ACC_THREADS>
__global__ void __launch_bounds__(ACC_THREADS) row_stats_kernel(const __grid_constant__ AcceptArgs a) {
    __shared__ AcceptSmem S;
    pdl_launch_dependents();
    pdl_wait();
    const int row = blockIdx.x;
    ktrace_mark(a.ktrace, a.ktrace_id, 0);
    unsigned long long* gtr = threadIdx.x == 0 ? a.gtrace : nullptr;
    gphase_mark(gtr, a.ktrace_id + 1, 1);
    if (a.req[row / a.G].status_in != 0) return;
    row_stats_body<ACC_THREADS>(a, row, blockIdx.y, threadIdx.x, S, CtaSync{});
    gphase_mark(gtr, a.ktrace_id + 1, 5);
}

template <int ACC_THREADS>
__global__ void __launch_bounds__(ACC_THREADS) accept_kernel(const __grid_constant__ AcceptArgs a) {
    __shared__ AcceptSmem S;
    pdl_launch_dependents();
    unsigned long long* gtr = threadIdx.x == 0 ? a.gtrace : nullptr;
    gphase_mark(gtr, a.ktrace_id, 0);
    accept_pre<ACC_THREADS>(a, blockIdx.x, blockIdx.y, threadIdx.x, S);
    pdl_wait();
    gphase_mark(gtr, a.ktrace_id, 1);
    if (accept_body<ACC_THREADS>(a, blockIdx.x, blockIdx.y, threadIdx.x, S, CtaSync{}) && a.ready_stamp) {
        unsigned long long t;   // exit-ready stamp: after this request's result is written
        asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t) :: "memory");
        atomicMax(a.ready_stamp, t);
        gphase_mark(a.gtrace, a.ktrace_id, 6);
    }
    __syncthreads();
    gphase_mark(gtr, a.ktrace_id, 5);
    ktrace_mark(a.ktrace, a.ktrace_id, 1);
}

cudaError_t accept_launch(const AcceptArgs& a, cudaStream_t st) {
    static int sms = 0;
    if (!sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (sms < 1) sms = 148;
    }
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cudaLaunchConfig_t cfg = {};
    cfg.stream = st;
    cfg.attrs = attr;
    cfg.numAttrs = g_use_pdl ? 1 : 0;
    cfg.gridDim = dim3(a.B * a.G, a.nch, 1);
    const bool narrow_rs = a.B * a.G * a.nch > 2 * sms, narrow_acc = a.B * a.nch > 2 * sms;
    cfg.blockDim = dim3(narrow_rs ? ACC_THREADS_NARROW : ACC_THREADS_WIDE, 1, 1);
    cudaError_t e = narrow_rs ? cudaLaunchKernelEx(&cfg, row_stats_kernel<ACC_THREADS_NARROW>, a)
                              : cudaLaunchKernelEx(&cfg, row_stats_kernel<ACC_THREADS_WIDE>, a);
    if (e != cudaSuccess) return e;
    cfg.gridDim = dim3(a.B, a.nch, 1);
    cfg.blockDim = dim3(narrow_acc ? ACC_THREADS_NARROW : ACC_THREADS_WIDE, 1, 1);
    return narrow_acc ? cudaLaunchKernelEx(&cfg, accept_kernel<ACC_THREADS_NARROW>, a)
                      : cudaLaunchKernelEx(&cfg, accept_kernel<ACC_THREADS_WIDE>, a);
}

}  // namespace sv
