// tma_bw.cu — HBM streaming microbenchmark for the weight-operand access pattern.
//   mode 0: 2D TMA boxes of 64 x 128 bf16 (SW128) from a row-major [N][K] matrix
//           (128 rows of 128 B, rows K*2 bytes apart) — the row-major weight layout
//   mode 1: 1D bulk copies of 16 KB contiguous blocks — a pre-tiled weight layout
// Each CTA streams its contiguous share of tiles through a STAGES-deep smem ring;
// the consumer only releases slots (no math).  Prints GB/s.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma_bw tma_bw.cu
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>

#include "../paper_2505_21594_b200/csrc/common.cuh"

using namespace sv;
static CUtensorMap g_tmb, g_tmb8;

__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar, uint64_t pol) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::
            "r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
        : "memory");
}

template <int STAGES>
__global__ void __launch_bounds__(64, 1) stream_kernel(const __grid_constant__ CUtensorMap tm, const uint8_t* base,
                                                        int mode, int ntiles, int kb_per_row,
                                                        const __grid_constant__ CUtensorMap tmb, const __grid_constant__ CUtensorMap tmb8) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * (16384 + 2048));
    uint64_t* empty = full + STAGES;
    uint32_t* tslot = reinterpret_cast<uint32_t*>(empty + STAGES);
    uint8_t* sb = smem + STAGES * 16384;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int t0 = (int)((long long)ntiles * blockIdx.x / gridDim.x);
    const int t1 = (int)((long long)ntiles * (blockIdx.x + 1) / gridDim.x);
    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        fence_mbar_init();
    }
    if (warp == 1) tmem_alloc(tslot, 32);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tslot;
    const int n = t1 - t0;
    if (warp == 0 && lane == 0) {
        const uint64_t pol = policy_evict_first();
        for (int i = 0; i < n; ++i) {
            const int s = i % STAGES;
            if (i >= STAGES) mbar_wait(&empty[s], ((i / STAGES) - 1) & 1);
            const int t = t0 + i;
            const int row_tile = t / kb_per_row, kb = t % kb_per_row;
            const bool ld_b = (mode == 2 || mode == 3 || mode == 5);
            const uint32_t bbytes = mode == 5 ? 1024 : 2048;
            if (mode == 1) {
                mbar_arrive_expect_tx(&full[s], 16384);
                bulk_load(smem + s * 16384, base + (size_t)t * 16384, 16384, &full[s], pol);
            } else {
                mbar_arrive_expect_tx(&full[s], 16384 + (ld_b ? bbytes : 0));
                tma_load_2d(&tm, smem + s * 16384, &full[s], kb * 64, row_tile * 128, pol);
                if (ld_b) tma_load_2d(mode == 5 ? &tmb8 : &tmb, sb + s * 2048, &full[s], kb * 64, 0, policy_evict_last());
            }
        }
    } else if (warp == 1 && lane == 0) {
        for (int i = 0; i < n; ++i) {
            const int s = i % STAGES;
            mbar_wait(&full[s], (i / STAGES) & 1);
            if (mode == 2 || mode == 4 || mode == 5) {
                tc_fence_after();
                const uint64_t ad = umma_sdesc_sw128(smem_u32(smem + s * 16384));
                uint64_t bd = umma_sdesc_sw128(smem_u32(sb + s * 2048));
                constexpr uint32_t idesc = umma_idesc_bf16(128, 16);
                if (mode == 4) bd = umma_sdesc_sw128(smem_u32(sb));
                for (int k = 0; k < 4; ++k) umma_bf16(tmem, ad + 2 * k, bd + 2 * k, idesc, (i | k) ? 1u : 0u);
                umma_commit(&empty[s]);
            } else {
                asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&empty[s])) : "memory");
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) tmem_dealloc(tmem, 32);
}

template <int STAGES>
static float run(const CUtensorMap& tm, const uint8_t* base, int mode, int ntiles, int kbr, int grid) {
    const int smem = 1024 + STAGES * (16384 + 2048) + 2 * STAGES * 8 + 16;
    cudaFuncSetAttribute(stream_kernel<STAGES>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int w = 0; w < 3; ++w) stream_kernel<STAGES><<<grid, 64, smem>>>(tm, base, mode, ntiles, kbr, g_tmb, g_tmb8);
    cudaEventRecord(a);
    const int reps = 10;
    for (int w = 0; w < reps; ++w) stream_kernel<STAGES><<<grid, 64, smem>>>(tm, base, mode, ntiles, kbr, g_tmb, g_tmb8);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) printf("error %s\n", cudaGetErrorString(e));
    return (float)ntiles * 16384.0f * reps / (ms / 1e3f) / 1e9f;
}

int main(int argc, char** argv) {
    const int N = argc > 1 ? atoi(argv[1]) : 22016, K = argc > 2 ? atoi(argv[2]) : 4096;   // default: gate/up of Llama2-7B (180 MB)
    const size_t bytes = (size_t)N * K * 2;
    uint8_t* buf;
    cudaMalloc(&buf, bytes);
    cudaMemset(buf, 1, bytes);
    PFN_cuTensorMapEncodeTiled_v12000 enc;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
    CUtensorMap tm;
    cuuint64_t gdim[2] = {(cuuint64_t)K, (cuuint64_t)N};
    cuuint64_t gstr[1] = {(cuuint64_t)K * 2};
    cuuint32_t box[2] = {64, 128};
    cuuint32_t es[2] = {1, 1};
    enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, gdim, gstr, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    uint8_t* act;
    cudaMalloc(&act, 16 * (size_t)K * 2);
    cudaMemset(act, 0, 16 * (size_t)K * 2);
    cuuint64_t gdb[2] = {(cuuint64_t)K, 16};
    cuuint32_t boxb[2] = {64, 16};
    enc(&g_tmb, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, act, gdb, gstr, boxb, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    cuuint32_t boxb8[2] = {64, 8};
    enc(&g_tmb8, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, act, gdb, gstr, boxb8, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    const int kbr = K / 64, ntiles = (N / 128) * kbr;
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    printf("tiles %d (%.1f MB), SMs %d\n", ntiles, bytes / 1e6, sms);
    const char* names[6] = {"A 2D only", "A bulk 16KB", "A+B16+MMA", "A+B16 no MMA", "A+MMA (B fixed)", "A+B8+MMA"};
    for (int mode = 0; mode < 6; ++mode) {
        const int grid = sms;
        printf("mode %d %-16s grid %d: st4 %.0f  st6 %.0f  st9 %.0f  st12 %.0f GB/s\n", mode, names[mode], grid,
               run<4>(tm, buf, mode, ntiles, kbr, grid), run<6>(tm, buf, mode, ntiles, kbr, grid),
               run<9>(tm, buf, mode, ntiles, kbr, grid), run<12>(tm, buf, mode, ntiles, kbr, grid));
    }
    return 0;
}
