// stream_bw.cu — weight-streaming microbenchmark for the batch-1 GEMM design.
// Streams a row-major bf16 [N][K] matrix as 128 x 64 TMA boxes (SW128) through a
// STAGES-deep ring, one CTA per SM, and reports per-launch time, GB/s and the
// spread of per-CTA finish times (globaltimer), for:
//   mode 0  TMA only (slot released on arrival)
//   mode 1  TMA + tcgen05.mma N=16 (B fixed in smem), one accumulator
//   mode 2  TMA + tcgen05.mma N=16, 4 accumulators (one per K=16 step)
//   mode 3  TMA only, dynamic chunks of 8 K blocks from an atomic counter
//   mode 4  TMA + mma (one accumulator), dynamic chunks of 8 K blocks
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o stream_bw stream_bw.cu
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../paper_2505_21594_b200/csrc/common.cuh"

using namespace sv;

template <int STAGES, int SB = 16384>
__global__ void __launch_bounds__(64, 1) stream_kernel(const __grid_constant__ CUtensorMap tm, int mode, int ntiles,
                                                        int kbr, int* ctr, unsigned long long* stamps) {
    // SB = bytes per ring slot (16 KB: 128-row box; 32 KB: 256-row box, modes 5/6)
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sb = smem + STAGES * SB;                          // fixed other operand (<= 16 KB)
    uint64_t* full = reinterpret_cast<uint64_t*>(sb + 16384);
    uint64_t* empty = full + STAGES;
    int* s_chunk = reinterpret_cast<int*>(empty + STAGES);     // [2] chunk handoff producer -> mma
    uint32_t* tslot = reinterpret_cast<uint32_t*>(s_chunk + 64);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const bool dyn = (mode == 3 || mode == 4);
    const bool mma = (mode == 1 || mode == 2 || mode == 4 || mode >= 5);
    const int RT = SB / 128;   // rows per box
    const int total = ntiles;   // units = K blocks over all tiles
    const int CH = 8;
    const int t0 = (int)((long long)total * blockIdx.x / gridDim.x);
    const int t1 = (int)((long long)total * (blockIdx.x + 1) / gridDim.x);
    if (threadIdx.x == 0) {
        stamps[blockIdx.x * 2] = gtimer_ns();
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        fence_mbar_init();
    }
    if (warp == 1) tmem_alloc(tslot, 256);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tslot;
    // unit sequence: static [t0, t1) or dynamic chunks; the producer writes the
    // unit index of each slot into a small smem queue read by the consumer
    volatile int* q = s_chunk;   // [STAGES] unit per slot, -1 = end
    if (warp == 0 && lane == 0) {
        const uint64_t pol = policy_evict_first();
        int i = 0;
        int cu = t0, ce = t1;
        if (dyn) {
            cu = atomicAdd(ctr, CH);
            ce = min(cu + CH, total);
        }
        while (true) {
            if (cu >= ce) {
                if (!dyn) break;
                cu = atomicAdd(ctr, CH);
                if (cu >= total) break;
                ce = min(cu + CH, total);
            }
            const int s = i % STAGES;
            if (i >= STAGES) mbar_wait(&empty[s], ((i / STAGES) - 1) & 1);
            q[s] = cu;
            mbar_arrive_expect_tx(&full[s], SB);
            tma_load_2d(&tm, smem + s * SB, &full[s], (cu % kbr) * 64, (cu / kbr) * RT, pol);
            ++cu;
            ++i;
        }
        // end marker: one more slot with unit -1 (arrive without tx)
        const int s = i % STAGES;
        if (i >= STAGES) mbar_wait(&empty[s], ((i / STAGES) - 1) & 1);
        q[s] = -1;
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&full[s])) : "memory");
    } else if (warp == 1 && lane == 0) {
        constexpr uint32_t idesc = umma_idesc_bf16(128, 16);
        const uint64_t bd = umma_sdesc_sw128(smem_u32(sb));
        for (int i = 0;; ++i) {
            const int s = i % STAGES;
            mbar_wait(&full[s], (i / STAGES) & 1);
            const int u = q[s];
            if (u < 0) break;
            if (mma) {
                tc_fence_after();
                const uint64_t wd = umma_sdesc_sw128(smem_u32(smem + s * SB));
                for (int k = 0; k < 4; ++k) {
                    if (mode == 5)        // activations = A (M=128), weights = B (N=256)
                        umma_bf16(tmem, bd + 2 * k, wd + 2 * k, umma_idesc_bf16(128, 256), (i > 0 || k > 0) ? 1u : 0u);
                    else if (mode == 6)   // M=64
                        umma_bf16(tmem, bd + 2 * k, wd + 2 * k, umma_idesc_bf16(64, 256), (i > 0 || k > 0) ? 1u : 0u);
                    else if (mode == 7)   // weights = A, N=32
                        umma_bf16(tmem, wd + 2 * k, bd + 2 * k, umma_idesc_bf16(128, 32), (i > 0 || k > 0) ? 1u : 0u);
                    else {
                        const uint32_t acc = (mode == 2) ? tmem + 32 * k : tmem;
                        umma_bf16(acc, wd + 2 * k, bd + 2 * k, idesc, (i > 0 || k > 0) ? 1u : 0u);
                    }
                }
                umma_commit(&empty[s]);
            } else {
                asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&empty[s])) : "memory");
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) tmem_dealloc(tmem, 256);
    if (threadIdx.x == 0) stamps[blockIdx.x * 2 + 1] = gtimer_ns();
}

template <int STAGES, int SB = 16384>
static void run(const CUtensorMap& tm, int mode, int ntiles, int kbr, int grid, int* ctr, unsigned long long* st,
                double mb) {
    const int smem = 1024 + STAGES * SB + 16384 + 2 * STAGES * 8 + 256 + 16;
    cudaFuncSetAttribute(stream_kernel<STAGES, SB>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int reps = 50;
    float best = 1e9f, tot = 0.f;
    std::vector<unsigned long long> h(2 * grid);
    double spread_sum = 0, startspread_sum = 0;
    for (int w = 0; w < reps + 5; ++w) {
        cudaMemsetAsync(ctr, 0, 4);
        cudaEventRecord(a);
        stream_kernel<STAGES, SB><<<grid, 64, smem>>>(tm, mode, ntiles, kbr, ctr, st);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (w >= 5) {
            best = std::min(best, ms);
            tot += ms;
            cudaMemcpy(h.data(), st, 16 * grid, cudaMemcpyDeviceToHost);
            unsigned long long s0 = ~0ull, s1 = 0, e0 = ~0ull, e1 = 0;
            for (int c = 0; c < grid; ++c) {
                s0 = std::min(s0, h[2 * c]);
                s1 = std::max(s1, h[2 * c]);
                e0 = std::min(e0, h[2 * c + 1]);
                e1 = std::max(e1, h[2 * c + 1]);
            }
            spread_sum += (e1 - e0) / 1e3;
            startspread_sum += (s1 - s0) / 1e3;
        }
    }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) printf("error %s\n", cudaGetErrorString(e));
    const float avg = tot / reps;
    printf("  st%-2d x %2d KB: avg %7.2f us (%5.0f GB/s)  best %7.2f us (%5.0f GB/s)  end-spread %5.2f us  start-spread %5.2f us\n",
           STAGES, SB / 1024, avg * 1e3, mb / avg, best * 1e3, mb / best, spread_sum / reps, startspread_sum / reps);
}

int main(int argc, char** argv) {
    const int N = argc > 1 ? atoi(argv[1]) : 22016, K = argc > 2 ? atoi(argv[2]) : 4096;
    const size_t bytes = (size_t)N * K * 2;
    uint8_t* buf;
    cudaMalloc(&buf, bytes);
    cudaMemset(buf, 0, bytes);
    PFN_cuTensorMapEncodeTiled_v12000 enc;
    cudaDriverEntryPointQueryResult qr;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &qr);
    CUtensorMap tm;
    cuuint64_t gdim[2] = {(cuuint64_t)K, (cuuint64_t)N};
    cuuint64_t gstr[1] = {(cuuint64_t)K * 2};
    cuuint32_t box[2] = {64, 128};
    cuuint32_t es[2] = {1, 1};
    enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, gdim, gstr, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    const int kbr = K / 64, ntiles = (N / 128) * kbr;
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    int* ctr;
    cudaMalloc(&ctr, 4);
    unsigned long long* st;
    cudaMalloc(&st, 16 * 1024);
    const double mb = bytes / 1e6;
    printf("N %d K %d: %.1f MB, %d units, SMs %d\n", N, K, mb, ntiles, sms);
    CUtensorMap tm256;
    cuuint32_t box256[2] = {64, 256};
    enc(&tm256, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, gdim, gstr, box256, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    const char* names[8] = {"TMA only", "TMA+MMA W=A M128 N16", "TMA+MMA N16 4 acc", "TMA only, dynamic",
                            "TMA+MMA dynamic", "W=B: M128 N256", "W=B: M64 N256", "W=A: M128 N32"};
    const int which = argc > 3 ? atoi(argv[3]) : -1;
    for (int mode = 0; mode < 8; ++mode) {
        if (which >= 0 && mode != which && mode != 0) continue;
        printf("mode %d %s\n", mode, names[mode]);
        if (mode == 5 || mode == 6) {
            run<3, 32768>(tm256, mode, ntiles / 2, kbr, sms, ctr, st, mb);
            run<4, 32768>(tm256, mode, ntiles / 2, kbr, sms, ctr, st, mb);
            run<6, 32768>(tm256, mode, ntiles / 2, kbr, sms, ctr, st, mb);
        } else {
            run<6>(tm, mode, ntiles, kbr, sms, ctr, st, mb);
            run<8>(tm, mode, ntiles, kbr, sms, ctr, st, mb);
            run<12>(tm, mode, ntiles, kbr, sms, ctr, st, mb);
        }
    }
    return 0;
}
