// fused.h — host interface of the fused persistent verify-step kernel (fused.cu).
#pragma once
#include <vector>

#include "kernels.h"

namespace sv {

enum FItemType { IT_EMBED = 1, IT_GEMM = 2, IT_ATTN = 3, IT_STATS = 4, IT_ACCEPT = 5 };

// One stage of the step (an op whose work items may run on any CTA).  Items of
// a stage may start their dependent part once stage `dep` has completed
// (cnt[dep] == target[dep]); every stage depends only on earlier stages.
struct alignas(16) FStage {
    int type, dep, dep_target, target;
    int epi, nt_n, nt_m, kblocks, exit_ws, is_exit;
    int tile_base;                 // first per-tile arrival counter of this GEMM
    const CUtensorMap* tmA;        // device-resident tensor maps (GEMM)
    const CUtensorMap* tmB;
    GemmArgs g;
    AttnArgs at;
    AcceptArgs ac;
    EmbedArgs em;
};

struct FItem {
    int16_t stage, type;
    int32_t tile;                  // GEMM tile / ATTN (b*H+h) / STATS row / ACCEPT request / EMBED row
    int32_t kb0, kb1;              // GEMM k-block range; ATTN/STATS/ACCEPT: kb0 = page / chunk
    int32_t slot;                  // GEMM: workspace slot of a partial segment (-1: whole tile)
    int32_t nsegs;                 // GEMM: segments of this tile
    int32_t seg_first;             // GEMM: index of the tile's first segment slot in seg_slots
    int32_t pad;
};

struct FusedPlan {
    int tile_n, head_dim, num_ctas, n_stages;
    FStage* d_stages = nullptr;
    FItem* d_items = nullptr;
    int* d_item_start = nullptr;   // [num_ctas + 1]
    int* d_seg_slots = nullptr;
    int* d_cnt = nullptr;          // [n_stages] completions + per-tile arrivals (zeroed per step)
    size_t cnt_ints = 0;
    int* d_tile_cnt = nullptr;
    float* ws_main = nullptr;      // [2 * num_ctas][tile_n][128]
    float* ws_exit = nullptr;
    sv_exit_result* early_host_dev = nullptr;   // mapped pinned mailbox (device alias)
    uint64_t* early_flag_dev = nullptr;
    const uint64_t* seq_dev = nullptr;
    int exit_stage_accept = -1, n_req = 0;
    int n_items = 0;
    unsigned long long* d_trace = nullptr;      // [n_items][4] timeline (SV_TRACE), else nullptr
    std::vector<FItem> h_items;                 // host copy of the item list (for trace dumps)
    std::vector<int> h_start;
};

// Builds the item lists (stream-K split of every GEMM over num_ctas CTAs, attention
// pages / acceptance chunks round-robin) and uploads them.
cudaError_t fused_build(FusedPlan* plan, std::vector<FStage>& stages, int num_ctas, int tile_n, int head_dim);
cudaError_t fused_launch(const FusedPlan* plan, cudaStream_t st);
void fused_free(FusedPlan* plan);
void fused_dump_trace(const FusedPlan* plan, const char* path);

}  // namespace sv
