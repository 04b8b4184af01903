// kernels.h — host-side launch interface of the verify-step kernels (internal).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/sv.h"

namespace sv {

typedef uint16_t bf16_raw_t;   // raw bf16 storage in host-visible structs

// programmatic dependent launch on/off (off in profile mode so per-kernel events
// do not overlap)
extern bool g_use_pdl;

// ----------------------------------------------------------------- GEMM (K1)
enum EpiKind { EPI_QKV = 0, EPI_RESID = 1, EPI_SWIGLU = 2, EPI_LOGITS = 3, EPI_SILU = 4 };

// Per-step request metadata, device resident (one H2D per step).
struct StepMeta {
    int32_t* tok;         // [rows] token id of each query row
    int32_t* pos;         // [rows] absolute position
    int32_t* ctx;         // [B] cached length before the step
    int32_t* row_req;     // [rows] request index of each query row
    int32_t* page_table;  // [B][pt_stride] KV block ids
    int32_t pt_stride;
    const uint32_t* epoch;   // incremented by the host for every issued step (split-K partial tags)
};

struct GemmArgs {
    // problem: out[M, N] = B[M, K] . A[N, K]^T  (A = weights, B = activations)
    int N, K, M, MP;     // MP = padded rows of the activation buffer
    int splits;          // split-K factor (deterministic reduction, fixed order)
    int b_row0;          // first row of the activation tensor map (exit slot k: k * MP)
    int b_box;           // rows of the activation TMA box (<= tile_n; 0 = tile_n), M <= tile_n only
    float* ws;           // split-K partials [splits][ntiles][MP][128] as (value, tag) 64-bit pairs
    int* counters;       // unused by the GEMMs (kept for the argument layout)
    uint32_t* sk_flags;  // [splits][ntiles][128] release flags (tiles of more than one 16-token chunk)
    // RMSNorm folding: rstd[m] = 1/sqrt(sum_t ssq_in[t][m] / d + eps)
    const float* ssq_in;  // [ssq_tiles][MP] or nullptr (no scaling)
    int ssq_tiles;
    float inv_d, eps;
    // EPI_QKV
    float* qbuf;          // [MP][d] fp32 (RoPE applied)
    bf16_raw_t* kv_pool;  // KV pool base (bf16)
    StepMeta meta;
    int layer, n_layers, n_heads, head_dim, d_model, page_tokens;
    const float* rope_cs;  // [max_pos][head_dim/2][2] (cos, sin) fp32
    // EPI_RESID
    float* h;             // [MP][d] fp32 residual stream (in/out)
    const void* g_out;    // bf16 [d] gain of the next RMSNorm
    void* u_out;          // bf16 [MP][d] = h * g_out
    const void* g_out2;   // bf16 [d] or nullptr (early-exit copy with the final gain)
    void* u_out2;
    float* ssq_out;       // [d/128][MP] per-tile sum of h^2
    float* h_out2;        // fp32 [MP][d] copy of the new residual or nullptr (exit adapter input)
    // EPI_SWIGLU
    void* act;            // bf16 [MP][d_ff]
    int d_ff;
    // EPI_LOGITS
    float* logits;        // [M][N]
    unsigned long long* gtrace = nullptr;   // optional phase stamps [launch][16][2] (SV_GTRACE)
    int warm = 0;         // gemm_kernel: warps 2-3 run the tail once as a dry pass (instruction-cache warm-up)
    int stream_k = 0;     // gemm_big_kernel: equal (tile, K block) ranges per CTA (main stream only)
    // gemm_big_kernel, EPI_QKV: after its last weight load, each CTA pulls a share of the
    // first kv_pf_blocks cached (request, page) KV blocks of this layer (request order,
    // kv_pf_B requests) into L2 — the attention that follows reads them while the QKV
    // epilogue tail leaves HBM idle
    int kv_pf_blocks = 0, kv_pf_B = 0;
    unsigned long long* ktrace = nullptr;   // optional per-launch [first start, last end] (SV_KTRACE)
    int ktrace_id = 0;
};

// Encodes a 2D bf16 K-major tensor map (rows x K), box = 64 x box_rows, SW128.
bool make_tmap_bf16(CUtensorMap* map, const void* base, uint64_t rows, uint64_t K, uint32_t box_rows);

int gemm_pick_tile_n(int M);
int gemm_pick_splits(int N, int K, int M, int tile_n, int num_sms);
extern bool g_split_fill;
cudaError_t gemm_launch(int epi, int tile_n, const CUtensorMap& tmA, const CUtensorMap& tmB, const GemmArgs& a,
                        cudaStream_t st);

// ------------------------------------------------------------- attention (K3)
struct AttnArgs {
    const float* q;       // [MP][d]
    const bf16_raw_t* kv_pool;
    void* out;            // bf16 [MP][d]
    float* part_o;        // [B*H][nchunk][G][head_dim]
    float* part_ml;       // [B*H][nchunk][G][2]
    int* counters;        // [B*H]
    const int32_t* ctx;   // [B]
    const int32_t* page_table;
    int pt_stride;
    int B, G, n_heads, head_dim, d_model, n_layers, layer, page_tokens, nchunk;
    float scale_log2;     // log2(e) / sqrt(head_dim)
    unsigned long long* ktrace = nullptr;   // optional per-launch [first start, last end] (SV_KTRACE)
    int ktrace_id = 0;
    unsigned long long* atrace = nullptr;   // optional phase stamps of CTAs (0,0) and (0,last) [16] (SV_ATRACE)
    // prefill (query blocks of one session as G-row "requests"): valid rows of each
    // request (nullptr: G) and the rows cached before the step (nullptr: ctx), i.e.
    // the rows that may be loaded before griddepcontrol.wait
    const int32_t* g_rows = nullptr;
    const int32_t* ctx_pre = nullptr;
    // L2 prefetch of the next GEMM's weights (the O projection), issued once the
    // QKV GEMM has completed: attention is latency-bound and leaves HBM idle
    const void* pf_ptr = nullptr;
    size_t pf_bytes = 0;
    int pf_early = 0;     // issue that prefetch at kernel start (before griddepcontrol.wait)
    int num_sms = 0;      // SMs of the engine's device (occupancy choice of attn3)
    // attn3 split partials as (value, tag) pairs [B*H][splits][16*128 + 32]; the tag is
    // (step epoch, launch index) so no partial of another launch is ever taken
    uint64_t* part = nullptr;
    const uint32_t* epoch = nullptr;
    int launch_id = 0;
    int cluster_launch = 0;   // launch the splits of (b, h) as one thread-block cluster (placement)
};
cudaError_t attn_launch(const AttnArgs& a, cudaStream_t st);
// v3 (head_dim 128): mma.sync bf16 tensor-core tiles, per-warp cp.async rings,
// online softmax in registers, cluster (DSMEM) split merge
int attn3_splits(int B, int H, int max_pages, int num_sms);
cudaError_t attn3_launch(const AttnArgs& a, int splits, int max_ctx_len, cudaStream_t st);
extern int g_attn_minb;    // env SV_A3_MINB: 2 or 3 attention CTAs per SM (default: by waves)
extern int g_attn_nst;     // env SV_ATTN_NST: per-warp ring depth 2 or 3 (default 1)

// ----------------------------------------------------------- acceptance (K5)
struct ReqDev {            // per-request metadata for the acceptance kernels
    uint64_t probs;        // device pointer to q [gamma][V] or 0 (greedy)
    uint64_t philox_seed;
    uint32_t session_id;
    uint32_t round_id;
    int32_t ctx;
    int32_t status_in;     // host-detected status (nonzero: skip)
    int32_t drafts[SV_MAX_GAMMA];
};
struct RowStat {
    float m1, m2, sum;
    int32_t idx;
};
struct RacePart {
    float k1, k2, f1;
    int32_t v1, fv1;
    int32_t pad[3];
};
struct AcceptArgs {
    const float* logits;    // [B*G][V]
    const ReqDev* req;      // [B]
    RowStat* stats;         // [B*G][nch]
    RacePart* race;         // [B][nch]
    int* counters;          // [B]
    sv_exit_result* out;    // [B] device
    int B, G, V, nch, chunk;
    int exit_layer, is_final;
    unsigned long long* ktrace = nullptr;   // optional per-launch [first start, last end] (SV_KTRACE)
    int ktrace_id = 0;
    unsigned long long* ready_stamp = nullptr;   // globaltimer when the last request's result was written (max)
    unsigned long long* gtrace = nullptr;        // optional phase stamps (SV_GTRACE): row_stats at ktrace_id + 1
};
cudaError_t accept_launch(const AcceptArgs& a, cudaStream_t st);
int accept_chunks(int V, int* chunk);

// ------------------------------------------------------------- misc (K4 K7 K8)
struct EmbedArgs {
    const int32_t* tok;
    const void* embed;   // bf16 [V][d]
    const void* gain;    // bf16 [d]
    float* h;            // [MP][d]
    void* u;             // bf16 [MP][d]
    float* ssq;          // [d/128][MP]
    int M, MP, d;
    unsigned long long* ktrace = nullptr;   // optional per-launch [first start, last end] (SV_KTRACE)
    int ktrace_id = 0;
    unsigned long long* stamps = nullptr;   // [n_stamps]: [0] = step start (globaltimer), rest reset to 0
    int n_stamps = 0;
};
cudaError_t embed_launch(const EmbedArgs& a, cudaStream_t st);

enum GenLayout { GEN_PLAIN = 0, GEN_QKV = 1, GEN_GU = 2 };
cudaError_t gen_launch(void* dst, uint64_t n, int layout, uint64_t seed, uint64_t tid0, int rows_per_sec,
                       int cols, float c, float offset, cudaStream_t st);
cudaError_t kvfill_launch(bf16_raw_t* pool, const int32_t* blocks, int nblocks, int len, uint64_t kv_seed,
                          int n_layers, int n_heads, int head_dim, int page_tokens, float c, cudaStream_t st);
cudaError_t philox_launch(const uint32_t* ctr_key, uint32_t* out, cudaStream_t st);

}  // namespace sv
