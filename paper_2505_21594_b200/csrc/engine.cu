// engine.cu — the C ABI of include/sv.h: engine, sessions, paged-KV block
// allocator, step orchestration (two streams: main + early-exit fork), CUDA-graph
// cache and result mailboxes.
//
// One verify step, issued as one graph:
//   K4 embed
//   for each layer l: K1 QKV(+RMSNorm fold, RoPE, KV append) -> K3 attention
//                     -> K1 O(+residual) -> K1 gate/up(+SwiGLU) -> K1 down(+residual)
//   after layer l_e : fork to the exit stream: K1 LM head -> K5 accept -> D2H
//                     of the early result + a sequence flag (mid-pass delivery)
//   after layer L   : K1 LM head -> K5 accept + K6 rollback -> D2H final result
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <thread>
#include <tuple>
#include <vector>

#include "../../include/sv.h"
#include "kernels.h"

using namespace sv;

// ------------------------------------------------------------------ errors
static thread_local std::string g_err;
static sv_status fail(sv_status s, const std::string& msg) {
    g_err = msg;
    return s;
}
#define CK(call)                                                                              \
    do {                                                                                      \
        cudaError_t _e = (call);                                                              \
        if (_e != cudaSuccess)                                                                \
            return fail(SV_E_DEVICE, std::string(#call " -> ") + cudaGetErrorString(_e));     \
    } while (0)

extern "C" const char* sv_status_str(sv_status s) {
    switch (s) {
        case SV_OK: return "SV_OK";
        case SV_E_INVALID: return "SV_E_INVALID";
        case SV_E_PROTOCOL: return "SV_E_PROTOCOL";
        case SV_E_CAPACITY: return "SV_E_CAPACITY";
        case SV_E_DEVICE: return "SV_E_DEVICE";
        case SV_E_BUSY: return "SV_E_BUSY";
        case SV_E_TIMEOUT: return "SV_E_TIMEOUT";
    }
    return "SV_E_UNKNOWN";
}
extern "C" const char* sv_last_error(void) { return g_err.c_str(); }
extern "C" int sv_abi_version(void) { return SV_ABI_VERSION; }

// ------------------------------------------------------------------ helpers
static const double IH_SD = std::sqrt(21845.0);
static float gen_scale(double sd) { return (float)(sd / IH_SD); }

static sv_status check_cfg(const sv_model_cfg* c) {
    if (!c) return fail(SV_E_INVALID, "cfg is NULL");
    if (c->n_layers < 1 || c->d_model <= 0 || c->d_model % 128 || c->n_heads <= 0 ||
        c->n_heads * c->head_dim != c->d_model || !(c->head_dim == 32 || c->head_dim == 64 || c->head_dim == 128) ||
        c->d_ff <= 0 || c->d_ff % 64 || c->vocab <= 0 || c->vocab % 128 || c->page_tokens != 64 ||
        c->max_ctx <= 0 || c->max_ctx % c->page_tokens || c->max_ctx > 4096)
        return fail(SV_E_INVALID, "unsupported model shape (see sv_model_cfg constraints)");
    return SV_OK;
}

static sv_status require_sm100(int device) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) return fail(SV_E_DEVICE, "no CUDA device (no CPU fallback)");
    if (device < 0 || device >= n) return fail(SV_E_DEVICE, "bad device ordinal");
    cudaDeviceProp p;
    if (cudaGetDeviceProperties(&p, device) != cudaSuccess) return fail(SV_E_DEVICE, "cudaGetDeviceProperties failed");
    if (p.major != 10 || p.minor != 0)
        return fail(SV_E_DEVICE, "device is not sm_100 (B200); this library has no other code path");
    return SV_OK;
}

extern "C" sv_status sv_weight_sizes(const sv_model_cfg* c, size_t* embed, size_t* lm_head, size_t* norm,
                                     size_t* qkv, size_t* o, size_t* gu, size_t* down) {
    sv_status s = check_cfg(c);
    if (s) return s;
    const size_t d = c->d_model, F = c->d_ff, V = c->vocab;
    if (embed) *embed = V * d * 2;
    if (lm_head) *lm_head = V * d * 2;
    if (norm) *norm = d * 2;
    if (qkv) *qkv = 3 * d * d * 2;
    if (o) *o = d * d * 2;
    if (gu) *gu = 2 * F * d * 2;
    if (down) *down = d * F * 2;
    return SV_OK;
}

extern "C" size_t sv_kv_block_bytes(const sv_model_cfg* c) {
    if (check_cfg(c)) return 0;
    return (size_t)c->n_layers * 2 * c->d_model * c->page_tokens * 2;
}

// tensor ids of the generator (oracle/gen.py documents the same numbering)
enum { TID_EMBED = 1, TID_LM_HEAD = 2, TID_NORM_FINAL = 3 };
static uint64_t layer_tid(int l, int kind) { return 16 + 16 * (uint64_t)l + kind; }

extern "C" sv_status sv_weights_generate(const sv_model_cfg* c, const sv_weights* w, uint64_t seed, void* stream) {
    sv_status s = check_cfg(c);
    if (s) return s;
    if (!w) return fail(SV_E_INVALID, "weights is NULL");
    cudaStream_t st = (cudaStream_t)stream;
    const int d = c->d_model, F = c->d_ff, V = c->vocab, L = c->n_layers;
    const double s_in = 1.28 / std::sqrt((double)d);
    const double s_out = s_in / std::sqrt(2.0 * L);
    CK(gen_launch(w->embed, (uint64_t)V * d, GEN_PLAIN, seed, TID_EMBED, 0, d, gen_scale(1.0), 0.f, st));
    CK(gen_launch(w->lm_head, (uint64_t)V * d, GEN_PLAIN, seed, TID_LM_HEAD, 0, d, gen_scale(3.2 / std::sqrt((double)d)),
                  0.f, st));
    CK(gen_launch(w->norm_final, d, GEN_PLAIN, seed, TID_NORM_FINAL, 0, d, gen_scale(0.1), 1.0f, st));
    for (int l = 0; l < L; ++l) {
        CK(gen_launch(w->w_qkv[l], (uint64_t)3 * d * d, GEN_QKV, seed, layer_tid(l, 0), d, d, gen_scale(s_in), 0.f, st));
        CK(gen_launch(w->w_o[l], (uint64_t)d * d, GEN_PLAIN, seed, layer_tid(l, 3), 0, d, gen_scale(s_out), 0.f, st));
        CK(gen_launch(w->w_gu[l], (uint64_t)2 * F * d, GEN_GU, seed, layer_tid(l, 4), 0, d, gen_scale(s_in), 0.f, st));
        CK(gen_launch(w->w_down[l], (uint64_t)d * F, GEN_PLAIN, seed, layer_tid(l, 6), 0, F, gen_scale(s_out), 0.f, st));
        CK(gen_launch(w->norm_attn[l], d, GEN_PLAIN, seed, layer_tid(l, 7), 0, d, gen_scale(0.1), 1.0f, st));
        CK(gen_launch(w->norm_mlp[l], d, GEN_PLAIN, seed, layer_tid(l, 8), 0, d, gen_scale(0.1), 1.0f, st));
    }
    return SV_OK;
}

static uint64_t adapter_tid(int layer1, int kind) { return 0x200000ull + 4ull * layer1 + kind; }   // layer 1-based

extern "C" sv_status sv_adapter_sizes(const sv_model_cfg* c, int32_t rank, size_t* dn, size_t* up, size_t* g) {
    sv_status s = check_cfg(c);
    if (s) return s;
    if (rank < 128 || rank % 128) return fail(SV_E_INVALID, "adapter rank must be a positive multiple of 128");
    if (dn) *dn = (size_t)rank * c->d_model * 2;
    if (up) *up = (size_t)c->d_model * rank * 2;
    if (g) *g = (size_t)c->d_model * 2;
    return SV_OK;
}

extern "C" sv_status sv_adapters_generate(const sv_model_cfg* c, const sv_adapters* a, uint64_t seed, void* stream) {
    sv_status s = check_cfg(c);
    if (s) return s;
    if (!a || !a->w_dn || !a->w_up || !a->g) return fail(SV_E_INVALID, "adapters is NULL");
    if ((s = sv_adapter_sizes(c, a->rank, nullptr, nullptr, nullptr))) return s;
    cudaStream_t st = (cudaStream_t)stream;
    const int d = c->d_model, r = a->rank;
    for (int l = 1; l < c->n_layers; ++l) {   // entry l-1 = adapter after layer l
        CK(gen_launch(a->w_dn[l - 1], (uint64_t)r * d, GEN_PLAIN, seed, adapter_tid(l, 0), 0, d,
                      gen_scale(1.28 / std::sqrt((double)d)), 0.f, st));
        CK(gen_launch(a->w_up[l - 1], (uint64_t)d * r, GEN_PLAIN, seed, adapter_tid(l, 1), 0, r,
                      gen_scale(0.1 / std::sqrt((double)r)), 0.f, st));
        CK(gen_launch(a->g[l - 1], d, GEN_PLAIN, seed, adapter_tid(l, 2), 0, d, gen_scale(0.1), 1.0f, st));
    }
    return SV_OK;
}

// ------------------------------------------------------------------ engine
// profile mode: every launch bracketed by CUDA events on its own stream
struct ProfRec {
    int kind, layer;
    cudaStream_t st;
    cudaEvent_t a, b;
    double bytes, flops;
};

struct sv_session {
    sv_engine* e;
    uint64_t id, seed;
    std::vector<int32_t> blocks;
    int32_t len = 0;
    uint32_t last_round = 0;
    bool busy = false;
};

struct StepKey {
    int n, gamma;
    uint64_t exit_mask;   // bit l-1 set: early exit after decoder layer l
    int nchunk;
    bool trace;           // per-launch timeline recorded (sv_debug_trace_next / SV_KTRACE)
    bool operator<(const StepKey& o) const {
        return std::tie(n, gamma, exit_mask, nchunk, trace) < std::tie(o.n, o.gamma, o.exit_mask, o.nchunk, o.trace);
    }
};

struct KMeta {
    int kind, layer, stream;   // stream 0 = main, 1 = exit
};

struct sv_ticket {
    sv_engine* e;
    int n;
    std::vector<int> gpu_slot;                   // request i -> batch slot (or -1)
    std::vector<sv_status> host_status;          // host-detected status per request
    std::vector<sv_session*> sess;
    std::vector<uint32_t> rounds;
    std::vector<int32_t> ctx;
    sv_exit_result* early;
    sv_exit_result* final_;
    std::vector<int> exits;                      // early-exit layers, ascending (slot k = exits[k])
    std::vector<bool> exit_done;
    uint64_t seq;
    int nb = 0, gamma = 0;
    bool has_gpu;
    bool final_done = false;
    cudaEvent_t ev_done = nullptr;
    // exit-ready timing (sv_ticket_timing): host clock at submit, at the first
    // observation of each exit's mailbox flag and of the step's completion
    std::chrono::steady_clock::time_point t_submit;
    std::vector<double> exit_host_ms;
    double final_host_ms = -1.0;
};

struct sv_engine {
    sv_model_cfg cfg;
    sv_engine_opts opts;
    int device, num_sms;
    bool no_box = false;                        // env SV_NO_BOX: load full token tiles
    bool no_t160 = false;                       // env SV_NO_T160: no 160-token persistent tiles
    bool no_wave = false;                       // env SV_NO_WAVE: always 256-token tiles above 128 rows
    bool no_t80 = false;                        // env SV_NO_T80: 128-token tiles for 65-80 rows
    bool no_warm = false;                       // env SV_NO_WARM: no instruction-cache warm-up pass in gemm_kernel
    bool no_stream_k = false;                   // env SV_NO_STREAM_K: whole tiles in the persistent GEMM
    double sk_fill = 0.6;                       // env SV_SK_FILL: stream-K below this wave fill
    int force_tn = 0;                           // env SV_FORCE_TN: persistent-GEMM token tile (experiments)
    int kv_pf_mb = -1;                          // env SV_KV_PF_MB: cached KV pulled into L2 by the QKV GEMM (-1: by rows)
    bool attn_no_cluster = false;               // env SV_ATTN_NO_CLUSTER: attn3 splits not launched as clusters
    int attn_pf = 0;                            // attention prefetches the O weights to L2 (env SV_ATTN_PF=1 after
                                                // griddepcontrol.wait, 2 before it)
    int attn_splits = 0;                        // attention split override (env SV_ATTN_SPLITS; 0 = attn3_splits)
    std::vector<CUtensorMap> wmap128;           // weight maps [qkv L][o L][gu L][down L][lm] (box rows 128)
    // exit adapters (NEXT-3): weights, maps [dn L][up L], exit-stream buffers
    int ad_rank = 0;
    std::vector<void*> ad_g;
    std::vector<CUtensorMap> ad_maps;
    float *h_exit = nullptr, *ssq_ad = nullptr;  // h^(l) per exit slot [L][MP][d]; Σh² of A_l(h) [d/128][MP]
    bf16_raw_t *act_ad = nullptr, *u_ad = nullptr;   // silu(.) [MP][rank]; bf16(A_l(h) * g_final) [MP][d]
    // weights
    void *embed, *lm_head, *norm_final;
    std::vector<void*> w_qkv, w_o, w_gu, w_down, norm_attn, norm_mlp;
    // KV pool
    uint8_t* kv_pool;
    size_t blk_bytes;
    int nblocks;
    std::vector<int32_t> free_blocks;
    int pt_stride;
    // sizes
    int max_rows, MP, d, F, V, L, H, D;
    int max_vreq = 1;                           // meta capacity: requests or prefill query blocks
    struct {                                    // set by sv_prefill for the duration of one issue_step
        bool on = false;
        bool all_rows = false;                  // sv_debug_forward: LM head on every prompt row
        int n_tokens = 0, nq = 0, gb = 0;
    } pf;
    // device scratch
    float *h, *qbuf, *ssq, *logits_exit, *logits_final, *ws_main, *ws_exit, *rope, *attn_o, *attn_ml;
    uint64_t* a3_part = nullptr;                // attn3 split partials (tagged pairs), a3_part_bh (b, h) units
    int a3_part_bh = 0;
    bf16_raw_t *u, *u_exit, *attn_out, *act;
    int *cnt_main, *cnt_exit, *cnt_attn, *cnt_acc_exit, *cnt_acc_final;
    uint32_t *flags_main = nullptr, *flags_exit = nullptr;   // split-K release flags
    RowStat *stats_exit, *stats_final;
    RacePart *race_exit, *race_final;
    sv_exit_result *res_exit_dev, *res_final_dev;
    size_t ws_elems;
    int acc_nch, acc_chunk, max_nchunk;
    float* probs_stage = nullptr;               // device copy of host draft probs
    // per-step metadata (device + pinned staging, same layout)
    uint8_t *meta_dev, *meta_host;
    size_t meta_bytes, off_tok, off_pos, off_req, off_ctx, off_pt, off_reqdev, off_seq, off_grows, off_cpre, off_epoch;
    uint32_t epoch = 0;                         // meta epoch: split-K partial tags (gemm.cu)
    // pinned mailboxes
    sv_exit_result *mb_exit, *mb_final;
    volatile uint64_t* mb_flag;
    sv_exit_result* mb_exit_dev = nullptr;      // device aliases of the mapped mailboxes
    uint64_t* mb_flag_dev = nullptr;
    // tensor maps
    std::vector<CUtensorMap> tm_qkv, tm_o, tm_gu, tm_down;
    CUtensorMap tm_lm;
    std::map<int, std::vector<CUtensorMap>> tm_act;   // tile_n -> {u, attn_out, act, u_exit}
    std::map<int, std::vector<CUtensorMap>> tm_box;   // box rows -> {u, attn_out, act, u_exit} (M < tile_n)
    // streams / graphs
    cudaStream_t s_cap, s_exit;
    cudaEvent_t ev_fork, ev_join;
    std::map<StepKey, cudaGraphExec_t> graphs;
    int last_launches = 0;
    uint64_t seq = 0;
    sv_ticket* inflight = nullptr;
    bool poisoned = false;
    std::vector<ProfRec>* prof = nullptr;
    unsigned long long* ktrace = nullptr;       // active trace buffer while a traced step is issued (else NULL)
    unsigned long long* ktrace_buf = nullptr;   // per-launch [start, ~end] globaltimer, 1024 launches
    unsigned long long* gtrace = nullptr;       // SV_GTRACE: GEMM phase stamps [1024][8][2] of traced steps
    bool trace_env = false;                     // SV_KTRACE: trace every step, CSV at sv_wait_final
    bool trace_next = false;                    // sv_debug_trace_next: trace the next submit
    bool trace_valid = false;                   // the last submit was traced
    std::vector<KMeta> kmeta;                   // launches of the step being issued
    std::map<StepKey, std::vector<KMeta>> graph_kmeta;
    std::vector<KMeta> last_kmeta;              // launches of the last traced step
    unsigned long long* atrace = nullptr;       // SV_ATRACE: attention phase stamps [layer][16]
    unsigned long long* stamps_dev = nullptr;   // [L+2] globaltimer: step start, exit k ready (1+k), final (1+L)
    std::mutex mu;
};

static size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }


static sv_status engine_alloc(sv_engine* e) {
    const int d = e->d, F = e->F, V = e->V, MP = e->MP;
    auto dalloc = [&](void** p, size_t bytes) -> cudaError_t {
        cudaError_t r = cudaMalloc(p, bytes);
        if (r == cudaSuccess) r = cudaMemset(*p, 0, bytes);
        return r;
    };
    CK(dalloc((void**)&e->h, (size_t)MP * d * 4));
    CK(dalloc((void**)&e->stamps_dev, (size_t)(e->L + 2) * 8));
    CK(dalloc((void**)&e->qbuf, (size_t)MP * d * 4));
    CK(dalloc((void**)&e->ssq, (size_t)(2 * e->L + 1) * (d / 128) * MP * 4));
    CK(dalloc((void**)&e->logits_exit, (size_t)MP * V * 4));
    CK(dalloc((void**)&e->logits_final, (size_t)MP * V * 4));
    CK(dalloc((void**)&e->u, (size_t)MP * d * 2));
    CK(dalloc((void**)&e->u_exit, (size_t)e->L * MP * d * 2));   // one slot per exit of a step
    CK(dalloc((void**)&e->attn_out, (size_t)MP * d * 2));
    CK(dalloc((void**)&e->act, (size_t)MP * F * 2));
    // split-K workspace: the largest splits * tiles * MP * 128 over all GEMMs and row counts
    size_t ws = 128;
    const int shapes[5][2] = {{3 * d, d}, {d, d}, {2 * F, d}, {d, F}, {V, d}};
    for (int M = 1; M <= e->max_rows; ++M) {
        const int tn = gemm_pick_tile_n(M);
        for (auto& s : shapes) {
            const int sp = gemm_pick_splits(s[0], s[1], M, tn, e->num_sms);
            if (sp > 1) ws = std::max(ws, (size_t)sp * (s[0] / 128) * MP * 128);
        }
    }
    ws = std::max(ws, (size_t)e->num_sms * 256 * 128);   // stream-K partials [P][TN][128]
    e->ws_elems = ws;
    CK(dalloc((void**)&e->ws_main, ws * 8));   // (value, tag) pairs
    CK(dalloc((void**)&e->ws_exit, ws * 8));
    const int max_tiles = std::max({3 * d, 2 * F, V}) / 128 * (MP / 16 + 1);
    CK(dalloc((void**)&e->cnt_main, (size_t)max_tiles * 4));
    CK(dalloc((void**)&e->cnt_exit, (size_t)max_tiles * 4));
    CK(dalloc((void**)&e->flags_main, (size_t)16 * max_tiles * 128 * 4));
    CK(dalloc((void**)&e->flags_exit, (size_t)16 * max_tiles * 128 * 4));
    // attention partials
    e->max_nchunk = e->cfg.max_ctx / 64 + 1;
    // per-page attention partials (attn_kernel, head_dim != 128)
    const size_t bh = (size_t)(e->D == 128 ? e->opts.max_batch : e->max_vreq) * e->H;
    const int G = std::max(e->opts.max_gamma + 1, 8);
    CK(dalloc((void**)&e->attn_o, bh * e->max_nchunk * G * e->D * 4));
    CK(dalloc((void**)&e->attn_ml, bh * e->max_nchunk * G * 2 * 4));
    CK(dalloc((void**)&e->cnt_attn, bh * 4));
    if (e->D == 128) {   // attn3 splits > 1 only at small batch (attn3_splits): room for 8 requests' heads
        e->a3_part_bh = std::min(e->max_vreq, 8) * e->H;
        CK(dalloc((void**)&e->a3_part, (size_t)e->a3_part_bh * 8 * (16 * 128 + 32) * 8));
    }
    // acceptance
    e->acc_nch = accept_chunks(V, &e->acc_chunk);
    CK(dalloc((void**)&e->stats_exit, (size_t)e->max_rows * e->acc_nch * sizeof(RowStat)));
    CK(dalloc((void**)&e->stats_final, (size_t)e->max_rows * e->acc_nch * sizeof(RowStat)));
    CK(dalloc((void**)&e->race_exit, (size_t)e->opts.max_batch * e->acc_nch * sizeof(RacePart)));
    CK(dalloc((void**)&e->race_final, (size_t)e->opts.max_batch * e->acc_nch * sizeof(RacePart)));
    CK(dalloc((void**)&e->cnt_acc_exit, (size_t)e->opts.max_batch * 4));
    CK(dalloc((void**)&e->cnt_acc_final, (size_t)e->opts.max_batch * 4));
    CK(dalloc((void**)&e->res_exit_dev, (size_t)e->opts.max_batch * sizeof(sv_exit_result)));
    CK(dalloc((void**)&e->res_final_dev, (size_t)e->opts.max_batch * sizeof(sv_exit_result)));
    // device staging of host draft probabilities (allocated up front: a submit must
    // not fail half-way through marking its sessions busy)
    CK(dalloc((void**)&e->probs_stage, (size_t)e->opts.max_batch * e->opts.max_gamma * V * 4));
    // RoPE table (cos, sin) in double -> fp32: angle = pos * theta^(-2i/Dh)
    {
        const int half = e->D / 2, npos = e->cfg.max_ctx + 16;
        std::vector<float> t((size_t)npos * half * 2);
        for (int p = 0; p < npos; ++p)
            for (int i = 0; i < half; ++i) {
                const double ang = (double)p * std::pow((double)e->cfg.rope_theta, -2.0 * i / e->D);
                t[((size_t)p * half + i) * 2 + 0] = (float)std::cos(ang);
                t[((size_t)p * half + i) * 2 + 1] = (float)std::sin(ang);
            }
        CK(dalloc((void**)&e->rope, t.size() * 4));
        CK(cudaMemcpy(e->rope, t.data(), t.size() * 4, cudaMemcpyHostToDevice));
    }
    // metadata block
    const int B = e->opts.max_batch, VB = e->max_vreq;
    size_t off = 0;
    e->off_tok = off; off = align_up(off + (size_t)MP * 4, 256);
    e->off_pos = off; off = align_up(off + (size_t)MP * 4, 256);
    e->off_req = off; off = align_up(off + (size_t)MP * 4, 256);
    e->off_ctx = off; off = align_up(off + (size_t)VB * 4, 256);
    e->off_pt = off; off = align_up(off + (size_t)VB * e->pt_stride * 4, 256);
    e->off_grows = off; off = align_up(off + (size_t)VB * 4, 256);
    e->off_cpre = off; off = align_up(off + (size_t)VB * 4, 256);
    e->off_reqdev = off; off = align_up(off + (size_t)B * sizeof(ReqDev), 256);
    e->off_seq = off; off = align_up(off + 8, 256);
    e->off_epoch = off; off = align_up(off + 8, 256);
    e->meta_bytes = off;
    CK(dalloc((void**)&e->meta_dev, off));
    CK(cudaMallocHost((void**)&e->meta_host, off));
    memset(e->meta_host, 0, off);
    CK(cudaHostAlloc((void**)&e->mb_exit, (size_t)e->L * B * sizeof(sv_exit_result), cudaHostAllocMapped));
    CK(cudaMallocHost((void**)&e->mb_final, (size_t)B * sizeof(sv_exit_result)));
    CK(cudaHostAlloc((void**)&e->mb_flag, (size_t)std::max(8, e->L) * 8, cudaHostAllocMapped));
    for (int k = 0; k < e->L; ++k) e->mb_flag[k] = 0;
    CK(cudaHostGetDevicePointer((void**)&e->mb_exit_dev, e->mb_exit, 0));
    CK(cudaHostGetDevicePointer((void**)&e->mb_flag_dev, (void*)e->mb_flag, 0));
    return SV_OK;
}

// activation (B operand) maps with `box` rows: {u, attn_out, act, u_exit} and, with
// exit adapters, {act_ad, u_ad}
static bool act_maps(sv_engine* e, int box, std::vector<CUtensorMap>* out) {
    const int d = e->d;
    std::vector<CUtensorMap> m(e->ad_rank ? 6 : 4);
    if (!make_tmap_bf16(&m[0], e->u, e->MP, d, box) || !make_tmap_bf16(&m[1], e->attn_out, e->MP, d, box) ||
        !make_tmap_bf16(&m[2], e->act, e->MP, e->F, box) ||
        !make_tmap_bf16(&m[3], e->u_exit, (uint64_t)e->L * e->MP, d, box))
        return false;
    if (e->ad_rank &&
        (!make_tmap_bf16(&m[4], e->act_ad, e->MP, e->ad_rank, box) || !make_tmap_bf16(&m[5], e->u_ad, e->MP, d, box)))
        return false;
    *out = m;
    return true;
}

static sv_status engine_tmaps(sv_engine* e) {
    const int d = e->d, F = e->F;
    e->tm_qkv.resize(e->L); e->tm_o.resize(e->L); e->tm_gu.resize(e->L); e->tm_down.resize(e->L);
    for (int l = 0; l < e->L; ++l) {
        if (!make_tmap_bf16(&e->tm_qkv[l], e->w_qkv[l], 3 * d, d, 128) ||
            !make_tmap_bf16(&e->tm_o[l], e->w_o[l], d, d, 128) ||
            !make_tmap_bf16(&e->tm_gu[l], e->w_gu[l], 2 * F, d, 128) ||
            !make_tmap_bf16(&e->tm_down[l], e->w_down[l], d, F, 128))
            return fail(SV_E_DEVICE, "cuTensorMapEncodeTiled failed (weights)");
    }
    if (!make_tmap_bf16(&e->tm_lm, e->lm_head, e->V, d, 128)) return fail(SV_E_DEVICE, "tensor map (lm_head)");
    for (int tn : {16, 32, 64, 80, 128, 160, 256}) {
        if (tn > e->MP) continue;
        std::vector<CUtensorMap> m;
        if (!act_maps(e, tn, &m)) return fail(SV_E_DEVICE, "tensor map (activations)");
        e->tm_act[tn] = m;
    }
    // weight maps in launch-table order [qkv L][o L][gu L][down L][lm]
    const int L = e->L, nmaps = 4 * L + 1;
    std::vector<CUtensorMap> all(nmaps);
    for (int l = 0; l < L; ++l) {
        all[l] = e->tm_qkv[l];
        all[L + l] = e->tm_o[l];
        all[2 * L + l] = e->tm_gu[l];
        all[3 * L + l] = e->tm_down[l];
    }
    all[4 * L] = e->tm_lm;
    e->wmap128 = all;
    return SV_OK;
}

extern "C" sv_status sv_engine_create(const sv_model_cfg* cfg, const sv_weights* w, const sv_engine_opts* opts,
                                      int device, void* kv_pool, size_t kv_pool_bytes, sv_engine** out) {
    sv_status s = check_cfg(cfg);
    if (s) return s;
    if (!w || !opts || !out || !kv_pool) return fail(SV_E_INVALID, "NULL argument");
    if (opts->max_batch < 1 || opts->max_gamma < 1 || opts->max_gamma > SV_MAX_GAMMA || opts->max_prefill < 0 ||
        opts->max_prefill > cfg->max_ctx)
        return fail(SV_E_INVALID, "bad engine options");
    if ((s = require_sm100(device))) return s;
    CK(cudaSetDevice(device));
    sv_engine* e = new sv_engine();
    e->cfg = *cfg;
    e->opts = *opts;
    e->device = device;
    CK(cudaDeviceGetAttribute(&e->num_sms, cudaDevAttrMultiProcessorCount, device));
    if (const char* as = getenv("SV_ATTN_SPLITS")) e->attn_splits = atoi(as);
    if (const char* ns = getenv("SV_ATTN_NST")) g_attn_nst = atoi(ns);
    if (const char* mb = getenv("SV_A3_MINB")) g_attn_minb = atoi(mb);
    if (getenv("SV_NO_BOX")) e->no_box = true;
    if (getenv("SV_NO_WAVE")) e->no_wave = true;
    if (getenv("SV_NO_T80")) e->no_t80 = true;
    if (getenv("SV_NO_WARM")) e->no_warm = true;
    if (getenv("SV_NO_STREAM_K")) e->no_stream_k = true;
    if (const char* sf = getenv("SV_SK_FILL")) e->sk_fill = atof(sf);
    if (const char* ft = getenv("SV_FORCE_TN")) e->force_tn = atoi(ft);
    if (const char* kp = getenv("SV_KV_PF_MB")) e->kv_pf_mb = atoi(kp);
    if (getenv("SV_SPLIT_POW2")) g_split_fill = false;
    if (getenv("SV_ATTN_NO_CLUSTER")) e->attn_no_cluster = true;
    if (getenv("SV_NO_T160")) e->no_t160 = true;
    if (const char* ap = getenv("SV_ATTN_PF")) e->attn_pf = atoi(ap);
    e->embed = w->embed; e->lm_head = w->lm_head; e->norm_final = w->norm_final;
    e->L = cfg->n_layers; e->d = cfg->d_model; e->F = cfg->d_ff; e->V = cfg->vocab;
    e->H = cfg->n_heads; e->D = cfg->head_dim;
    for (int l = 0; l < e->L; ++l) {
        e->w_qkv.push_back(w->w_qkv[l]); e->w_o.push_back(w->w_o[l]); e->w_gu.push_back(w->w_gu[l]);
        e->w_down.push_back(w->w_down[l]); e->norm_attn.push_back(w->norm_attn[l]); e->norm_mlp.push_back(w->norm_mlp[l]);
    }
    e->blk_bytes = sv_kv_block_bytes(cfg);
    e->kv_pool = (uint8_t*)kv_pool;
    e->nblocks = (int)(kv_pool_bytes / e->blk_bytes);
    if (e->nblocks < 1) { delete e; return fail(SV_E_CAPACITY, "kv pool smaller than one block"); }
    for (int i = e->nblocks - 1; i >= 0; --i) e->free_blocks.push_back(i);
    e->pt_stride = cfg->max_ctx / cfg->page_tokens + 1;
    e->max_rows = std::max(opts->max_batch * (opts->max_gamma + 1), opts->max_prefill);
    e->max_vreq = std::max(opts->max_batch, (opts->max_prefill + 7) / 8);
    e->MP = (int)align_up((size_t)e->max_rows, 256);
    if ((s = engine_alloc(e)) || (s = engine_tmaps(e))) {
        delete e;
        return s;
    }
    CK(cudaStreamCreateWithFlags(&e->s_cap, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&e->s_exit, cudaStreamNonBlocking));
    CK(cudaEventCreateWithFlags(&e->ev_fork, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&e->ev_join, cudaEventDisableTiming));
    CK(cudaMalloc((void**)&e->ktrace_buf, 1024 * 2 * sizeof(unsigned long long)));
    e->trace_env = getenv("SV_KTRACE") != nullptr;
    if (getenv("SV_GTRACE")) CK(cudaMalloc((void**)&e->gtrace, 1024 * 32 * sizeof(unsigned long long)));
    if (getenv("SV_ATRACE")) CK(cudaMalloc((void**)&e->atrace, (size_t)e->L * 16 * sizeof(unsigned long long)));
    *out = e;
    return SV_OK;
}

extern "C" sv_status sv_engine_set_adapters(sv_engine* e, const sv_adapters* ad) {
    if (!e) return fail(SV_E_INVALID, "NULL engine");
    std::lock_guard<std::mutex> lk(e->mu);
    if (e->inflight) return fail(SV_E_BUSY, "a ticket is in flight");
    CK(cudaSetDevice(e->device));
    const int L = e->L, d = e->d;
    if (ad) {
        sv_status s = sv_adapter_sizes(&e->cfg, ad->rank, nullptr, nullptr, nullptr);
        if (s) return s;
        if (!ad->w_dn || !ad->w_up || !ad->g) return fail(SV_E_INVALID, "adapter arrays are NULL");
        if (ad->rank != e->ad_rank) {   // (re)size the exit-stream buffers
            cudaFree(e->act_ad);
            e->act_ad = nullptr;
            CK(cudaMalloc((void**)&e->act_ad, (size_t)e->MP * ad->rank * 2));
            CK(cudaMemset(e->act_ad, 0, (size_t)e->MP * ad->rank * 2));
        }
        if (!e->h_exit) {
            CK(cudaMalloc((void**)&e->h_exit, (size_t)L * e->MP * d * 4));
            CK(cudaMalloc((void**)&e->u_ad, (size_t)e->MP * d * 2));
            CK(cudaMalloc((void**)&e->ssq_ad, (size_t)(d / 128) * e->MP * 4));
            CK(cudaMemset(e->h_exit, 0, (size_t)L * e->MP * d * 4));
            CK(cudaMemset(e->u_ad, 0, (size_t)e->MP * d * 2));
        }
        e->ad_rank = ad->rank;
        e->ad_g.assign(ad->g, ad->g + L);
        e->wmap128.resize(4 * L + 1 + 2 * L);
        for (int l = 0; l + 1 < L; ++l)   // entry l = adapter after layer l + 1
            if (!make_tmap_bf16(&e->wmap128[4 * L + 1 + l], ad->w_dn[l], ad->rank, d, 128) ||
                !make_tmap_bf16(&e->wmap128[4 * L + 1 + L + l], ad->w_up[l], d, ad->rank, 128))
                return fail(SV_E_DEVICE, "tensor map (adapters)");
    } else {
        e->ad_rank = 0;
    }
    for (auto& kv : e->tm_act)
        if (!act_maps(e, kv.first, &kv.second)) return fail(SV_E_DEVICE, "tensor map (activations)");
    e->tm_box.clear();
    for (auto& kv : e->graphs) cudaGraphExecDestroy(kv.second);   // steps change
    e->graphs.clear();
    return SV_OK;
}

extern "C" sv_status sv_engine_destroy(sv_engine* e) {
    if (!e) return fail(SV_E_INVALID, "NULL engine");
    cudaSetDevice(e->device);
    cudaDeviceSynchronize();
    for (auto& kv : e->graphs) cudaGraphExecDestroy(kv.second);
    void* dev[] = {e->h, e->qbuf, e->ssq, e->logits_exit, e->logits_final, e->ws_main, e->ws_exit, e->rope,
                   e->attn_o, e->attn_ml, e->u, e->u_exit, e->attn_out, e->act, e->cnt_main, e->cnt_exit,
                   e->cnt_attn, e->cnt_acc_exit, e->cnt_acc_final, e->stats_exit, e->stats_final, e->race_exit,
                   e->race_final, e->res_exit_dev, e->res_final_dev, e->meta_dev, e->probs_stage,
                   e->h_exit, e->ssq_ad, e->act_ad, e->u_ad, e->stamps_dev, e->ktrace_buf, e->atrace, e->gtrace,
                   e->a3_part, e->flags_main, e->flags_exit};
    for (void* p : dev)
        if (p) cudaFree(p);
    cudaFreeHost(e->meta_host);
    cudaFreeHost(e->mb_exit);
    cudaFreeHost(e->mb_final);
    cudaFreeHost((void*)e->mb_flag);
    cudaStreamDestroy(e->s_cap);
    cudaStreamDestroy(e->s_exit);
    cudaEventDestroy(e->ev_fork);
    cudaEventDestroy(e->ev_join);
    delete e;
    return SV_OK;
}

extern "C" sv_status sv_engine_last_launches(const sv_engine* e, int32_t* n) {
    if (!e || !n) return fail(SV_E_INVALID, "NULL argument");
    *n = e->last_launches;
    return SV_OK;
}

// ------------------------------------------------------------------ sessions
static bool ensure_blocks(sv_engine* e, sv_session* s, int len) {
    const int need = (len + e->cfg.page_tokens - 1) / e->cfg.page_tokens;
    while ((int)s->blocks.size() < need) {
        if (e->free_blocks.empty()) return false;
        s->blocks.push_back(e->free_blocks.back());
        e->free_blocks.pop_back();
    }
    return true;
}

extern "C" sv_status sv_session_open(sv_engine* e, uint64_t session_id, uint64_t philox_seed, sv_session** out) {
    if (!e || !out) return fail(SV_E_INVALID, "NULL argument");
    sv_session* s = new sv_session();
    s->e = e;
    s->id = session_id;
    s->seed = philox_seed;
    *out = s;
    return SV_OK;
}

extern "C" sv_status sv_session_fill_kv(sv_session* s, int32_t len, uint64_t kv_seed) {
    if (!s) return fail(SV_E_INVALID, "NULL session");
    sv_engine* e = s->e;
    std::lock_guard<std::mutex> lk(e->mu);
    if (s->busy) return fail(SV_E_BUSY, "session has a ticket in flight");
    if (len < 0 || len + SV_MAX_GAMMA + 1 > e->cfg.max_ctx) return fail(SV_E_INVALID, "len out of range");
    if (!ensure_blocks(e, s, std::max(len, 1))) return fail(SV_E_CAPACITY, "KV pool exhausted");
    CK(cudaSetDevice(e->device));
    int32_t* dblocks = nullptr;
    CK(cudaMalloc(&dblocks, s->blocks.size() * 4));
    CK(cudaMemcpy(dblocks, s->blocks.data(), s->blocks.size() * 4, cudaMemcpyHostToDevice));
    CK(kvfill_launch((bf16_raw_t*)e->kv_pool, dblocks, (int)s->blocks.size(), len, kv_seed, e->L, e->H, e->D,
                     e->cfg.page_tokens, gen_scale(1.0), 0));
    CK(cudaDeviceSynchronize());
    CK(cudaFree(dblocks));
    s->len = len;
    return SV_OK;
}

extern "C" sv_status sv_session_len(const sv_session* s, int32_t* len) {
    if (!s || !len) return fail(SV_E_INVALID, "NULL argument");
    *len = s->len;
    return SV_OK;
}

extern "C" sv_status sv_session_close(sv_session* s) {
    if (!s) return fail(SV_E_INVALID, "NULL session");
    sv_engine* e = s->e;
    std::lock_guard<std::mutex> lk(e->mu);
    if (s->busy) return fail(SV_E_BUSY, "session has a ticket in flight");
    for (int b : s->blocks) e->free_blocks.push_back(b);
    delete s;
    return SV_OK;
}

// ------------------------------------------------------------------ one step
static GemmArgs base_args(sv_engine* e, int M) {
    GemmArgs a = {};
    a.M = M;
    a.MP = e->MP;
    a.inv_d = 1.0f / e->d;
    a.eps = e->cfg.rms_eps;
    a.ssq_tiles = e->d / 128;
    a.n_layers = e->L; a.n_heads = e->H; a.head_dim = e->D; a.d_model = e->d; a.page_tokens = e->cfg.page_tokens;
    a.d_ff = e->F;
    a.rope_cs = e->rope;
    a.kv_pool = (bf16_raw_t*)e->kv_pool;
    a.meta.tok = (int32_t*)(e->meta_dev + e->off_tok);
    a.meta.pos = (int32_t*)(e->meta_dev + e->off_pos);
    a.meta.row_req = (int32_t*)(e->meta_dev + e->off_req);
    a.meta.ctx = (int32_t*)(e->meta_dev + e->off_ctx);
    a.meta.page_table = (int32_t*)(e->meta_dev + e->off_pt);
    a.meta.pt_stride = e->pt_stride;
    a.meta.epoch = (const uint32_t*)(e->meta_dev + e->off_epoch);
    return a;
}

static float* ssq_at(sv_engine* e, int layer, int which) {   // norm point (layer, 0 = attn / 1 = mlp)
    return e->ssq + (size_t)(2 * layer + which) * (e->d / 128) * e->MP;
}

// Token tile, split-K factor and stream-K choice of one GEMM launch with M query rows
// (a.M is the launch's row count, M the step's); sets a.splits / a.stream_k, returns
// the token tile.  Shared by the step and the sv_debug_gemm hook.
static int gemm_config(sv_engine* e, int M, int N, int K, bool exit_ws, GemmArgs& a) {
    const int tn = gemm_pick_tile_n(M);
    // persistent path (M > 128): wave-aware token tile, 128 or 256 rows, minimising
    // ceil(tiles / SMs) x tile (C4 at 1 GPU: O / down 160 -> 320 tiles, 2 -> 3 rounds of half size)
    // 160-token tiles (UMMA N = 160) fill the rounds of M = 640 / 1280 (C4 at 1-2 GPUs)
    int tl = tn;
    // 65-80 rows (C5): 80-token tiles (UMMA N = 80) — the smaller activation stage
    // leaves room for 7 weight stages in flight instead of 6
    if (M > 64 && M <= 80 && a.M == M && !e->no_t80) tl = 80;
    // gate/up (N = 2F) and the LM heads (N = V) too up to 320 rows: measured (same box)
    // C4 8-GPU shard 8.19 -> 8.04 ms, 4-GPU shard 13.9 -> 13.45 ms (gate/up at 160 rows
    // 49 -> 45 us: 160-token instead of padded 256-token tiles); at 640 rows the
    // weighted choice (160) loses to 256 (22.1 vs 22.6 ms) and the old rule stays
    if (M > 128 && a.M == M && !e->no_wave && (N < 16384 || M <= 320)) {
        // rounds x tile rows, weighted by the tile's MMA efficiency once the GEMM is
        // compute-bound (M >= 640): the tensor pipe is 87% busy at 256-token tiles
        // but ~50% at 128 (C4 QKV, ncu; profiles/r02/c4_tensor_pipe.json)
        auto cost = [&](int t) {
            const long long tiles = (long long)(N / 128) * ((M + t - 1) / t);
            const double eff = M < 640 ? 1.0 : (t >= 256 ? 1.0 : t >= 160 ? 0.92 : 0.85);
            return (double)((tiles + e->num_sms - 1) / e->num_sms) * t / eff;
        };
        double best = cost(256);
        tl = 256;
        if (!e->no_t160 && gemm_pick_splits(N, K, M, 160, e->num_sms) == 1 && cost(160) < best) {
            best = cost(160);
            tl = 160;
        }
        if (K <= 4096 && cost(128) < best) tl = 128;   // (measured: the long-K down projection loses at 128)
    }
    if (e->force_tn && M > 64 && a.M == M && e->tm_act.count(e->force_tn)) tl = e->force_tn;
    a.splits = gemm_pick_splits(N, K, M, tl, e->num_sms);
    // stream-K on the main stream when whole tiles fill under 60% of the persistent
    // grid's waves (C5: gate/up 172 tiles on 2 x 148, O / down 32 tiles); measured
    // slower at 65-85% (C5 QKV 96 tiles: 36.9 vs 32.7 us; LM head 250 tiles).
    // Never on the exit stream: its reducers could wait on CTAs that cannot
    // become resident beside a main-stream stream-K grid.
    if (tl > 64 && !exit_ws && !e->no_stream_k && a.M == M) {
        const long long tiles = (long long)(N / 128) * ((M + tl - 1) / tl);
        const long long waves = (tiles + e->num_sms - 1) / e->num_sms;
        if ((double)tiles / (double)(waves * e->num_sms) < e->sk_fill) {
            a.stream_k = 1;
            a.splits = 1;
        }
    }
    // stream-K GEMMs with few weight tiles (O / down) at 81-160 rows: 80-token tiles —
    // the reducing CTA's tail epilogue is half as long (measured at 160 rows, the C4
    // 8-GPU shard: O 25.7 -> 21.5 us; QKV / gate-up, whose tiles fill the grid, lose
    // at 80 and keep their tile)
    if (a.stream_k && M > 80 && M <= 160 && !e->force_tn && !e->no_t80 &&
        (long long)(N / 128) * ((M + 79) / 80) <= e->num_sms / 2)
        tl = 80;
    return tl;
}

// Issues every kernel / copy of one step on (main, exit) streams; returns launch count.
// exit_mask: bit l-1 = early exit after decoder layer l; the k-th exit (ascending)
// uses u_exit slot k, mailbox rows [k][B] and flag k (streamed as each completes).
static cudaError_t issue_step(sv_engine* e, cudaStream_t st, int n, int gamma, uint64_t exit_mask, int nchunk,
                              int* launches) {
    const bool pf = e->pf.on;                 // prefill: one session's prompt as query blocks
    const int G = gamma + 1, M = pf ? e->pf.n_tokens : n * G, d = e->d, F = e->F, V = e->V, L = e->L;
    const int nA = pf ? e->pf.nq : n, GA = pf ? e->pf.gb : G;   // attention "requests" and their rows
    const int tn = gemm_pick_tile_n(M);
    const auto& tma = e->tm_act[tn];   // {u, attn_out, act, u_exit}
    int nl = 0;
    cudaError_t r;
    // algorithmic bytes / flops per launch: every operand
    // the op must read or write once
    const double Md = (double)M * d, W2 = 2.0;
    auto gemm_bytes = [&](double N, double K, double out) { return N * K * W2 + M * K * W2 + out; };
    auto pbeg = [&](cudaStream_t s) -> cudaEvent_t {
        cudaEvent_t ev = nullptr;
        if (e->prof) {
            cudaEventCreate(&ev);
            cudaEventRecord(ev, s);
        }
        return ev;
    };
    auto pend = [&](cudaEvent_t a, int kind, int layer, cudaStream_t s, double bytes, double flops) {
        if (!e->prof) return;
        cudaEvent_t b;
        cudaEventCreate(&b);
        cudaEventRecord(b, s);
        e->prof->push_back(ProfRec{kind, layer, s, a, b, bytes, flops});
    };
#define LAUNCH(kind, layer, s, bytes, flops, x)         \
    do {                                                \
        cudaEvent_t _a = pbeg(s);                       \
        if ((r = (x)) != cudaSuccess) return r;         \
        if (e->ktrace) {                                \
            e->kmeta.resize(nl + 1);                    \
            e->kmeta[nl] = {kind, layer, s == st ? 0 : 1}; \
        }                                               \
        ++nl;                                           \
        pend(_a, kind, layer, s, bytes, flops);         \
    } while (0)

    e->kmeta.clear();
    if (e->ktrace && (r = cudaMemsetAsync(e->ktrace, 0xFF, 1024 * 2 * sizeof(unsigned long long), st)) != cudaSuccess)
        return r;
    if (e->ktrace && e->gtrace &&
        (r = cudaMemsetAsync(e->gtrace, 0xFF, 1024 * 32 * sizeof(unsigned long long), st)) != cudaSuccess)
        return r;
    EmbedArgs ea{(const int32_t*)(e->meta_dev + e->off_tok), e->embed, e->norm_attn[0], e->h, e->u, ssq_at(e, 0, 0), M,
                 e->MP, d};
    ea.ktrace = e->ktrace;
    ea.ktrace_id = nl;
    ea.stamps = e->stamps_dev;
    ea.n_stamps = L + 2;
    LAUNCH(SV_K_EMBED, -1, st, Md * 2 + d * 2 + Md * 6 + (d / 128) * M * 4.0, 0.0, embed_launch(ea, st));
    double attn_bytes = Md * 6, attn_flops = 0;
    int max_ctx = 0;
    {
        const int32_t* ctxh = (const int32_t*)(e->meta_host + e->off_ctx);
        for (int b = 0; b < nA; ++b) {
            max_ctx = std::max(max_ctx, (int)ctxh[b]);
            attn_bytes += (double)(ctxh[b] + GA) * d * 4;
            for (int j = 0; j < GA; ++j) attn_flops += 4.0 * (ctxh[b] + j + 1) * d;
        }
    }

    // wid: weight index in [qkv L][o L][gu L][down L][lm] order
    auto gemm = [&](int epi, int wid, int bbuf, int N, int K, GemmArgs a, cudaStream_t s, bool exit_ws) -> cudaError_t {
        a.N = N;
        a.K = K;
        a.ws = exit_ws ? e->ws_exit : e->ws_main;
        a.counters = exit_ws ? e->cnt_exit : e->cnt_main;
        a.sk_flags = exit_ws ? e->flags_exit : e->flags_main;
        a.ktrace = e->ktrace;
        a.ktrace_id = nl;
        a.gtrace = e->ktrace ? e->gtrace : nullptr;
        a.warm = e->no_warm ? 0 : 1;
        const int tl = gemm_config(e, M, N, K, exit_ws, a);
        const CUtensorMap& A = e->wmap128[wid];
        const auto& tmal = e->tm_act[tl];
        const CUtensorMap* Bp = &tmal[bbuf];
        if (M < tl && !e->no_box) {   // one token tile: load only its real rows
            const int box = (M + 7) / 8 * 8;
            auto it = e->tm_box.find(box);
            if (it == e->tm_box.end()) {
                std::vector<CUtensorMap> m;
                if (!act_maps(e, box, &m)) return cudaErrorInvalidValue;
                it = e->tm_box.emplace(box, m).first;
            }
            Bp = &it->second[bbuf];
            a.b_box = box;
        }
        const CUtensorMap& B = *Bp;
        return gemm_launch(epi, tl, A, B, a, s);
    };
    // slot >= 0: the exit reads u_exit slot `slot`; slot < 0: the adapter output u_ad
    auto lm_and_accept = [&](cudaStream_t s, bool is_exit, int exit_layer, int slot, int stamp_slot) -> cudaError_t {
        GemmArgs a = base_args(e, pf && !e->pf.all_rows ? 1 : M);
        a.ssq_in = (is_exit && slot < 0) ? e->ssq_ad : ssq_at(e, is_exit ? exit_layer : L, 0);
        a.b_row0 = (is_exit && slot >= 0) ? slot * e->MP : 0;
        if (pf && !e->pf.all_rows) {   // prefill: the LM head of the last prompt row only (its next token)
            a.b_row0 = e->pf.n_tokens - 1;
            a.ssq_in += e->pf.n_tokens - 1;
        }
        a.logits = is_exit ? e->logits_exit : e->logits_final;
        cudaError_t q;
        LAUNCH(is_exit ? SV_K_LM_EXIT : SV_K_LM_FINAL, -1, s, gemm_bytes(V, d, (double)M * V * 4),
               2.0 * M * V * d, gemm(EPI_LOGITS, 4 * L, is_exit ? (slot < 0 ? 5 : 3) : 0, V, d, a, s, is_exit));
        AcceptArgs aa = {};
        aa.logits = a.logits;
        aa.req = (const ReqDev*)(e->meta_dev + e->off_reqdev);
        aa.stats = is_exit ? e->stats_exit : e->stats_final;
        aa.race = is_exit ? e->race_exit : e->race_final;
        aa.counters = is_exit ? e->cnt_acc_exit : e->cnt_acc_final;
        aa.out = is_exit ? e->res_exit_dev : e->res_final_dev;
        aa.B = pf ? 1 : n; aa.G = pf ? 1 : G; aa.V = V; aa.nch = e->acc_nch; aa.chunk = e->acc_chunk;
        aa.exit_layer = is_exit ? exit_layer : L;
        aa.is_final = is_exit ? 0 : 1;
        aa.ktrace = e->ktrace;
        aa.ktrace_id = nl;
        aa.ready_stamp = e->stamps_dev + stamp_slot;
        aa.gtrace = e->ktrace ? e->gtrace : nullptr;
        {
            cudaEvent_t _a = pbeg(s);
            if ((q = accept_launch(aa, s)) != cudaSuccess) return q;
            if (e->ktrace) {   // one record [row_stats start, accept end] for the pair
                e->kmeta.resize(nl + 2);
                e->kmeta[nl] = {is_exit ? SV_K_ACCEPT_EXIT : SV_K_ACCEPT_FINAL, -1, s == st ? 0 : 1};
                e->kmeta[nl + 1] = {-1, -1, -1};
            }
            nl += 2;
            pend(_a, is_exit ? SV_K_ACCEPT_EXIT : SV_K_ACCEPT_FINAL, -1, s,
                 (double)M * V * 4 + (double)n * V * 8, 0.0);
        }
        return cudaSuccess;
    };

    const int n_exits = __builtin_popcountll(exit_mask);
    int exit_k = 0;
    for (int l = 0; l < L; ++l) {
        const bool is_exit_l = (exit_mask >> l) & 1;   // exit after layer l + 1
        {   // QKV + RoPE + KV append
            GemmArgs a = base_args(e, M);
            a.layer = l;
            a.ssq_in = ssq_at(e, l, 0);
            a.qbuf = e->qbuf;
            // cached KV of this layer -> L2 during the QKV tail (measured, same box: 48 MB
            // C5 6.68 -> 6.65 ms, C4 8-GPU shard 8.24 -> 8.14; 96 MB for C4 39.8 -> 39.4,
            // but C5 6.81: the prefetch then overlaps C5's QKV mainloop)
            const int kv_mb = e->kv_pf_mb >= 0 ? e->kv_pf_mb : (M >= 256 ? 96 : 48);
            if (!pf && kv_mb > 0) {
                a.kv_pf_B = nA;
                a.kv_pf_blocks = (int)((double)kv_mb * (1 << 20) / (4.0 * e->H * 64 * e->D));
            }
            LAUNCH(SV_K_QKV, l, st, gemm_bytes(3.0 * d, d, Md * 8 + (d / 128) * M * 4.0), 2.0 * M * 3.0 * d * d,
                   gemm(EPI_QKV, l, 0, 3 * d, d, a, st, false));
        }
        {   // attention
            AttnArgs aa = {};
            aa.q = e->qbuf; aa.kv_pool = (const bf16_raw_t*)e->kv_pool; aa.out = e->attn_out;
            aa.part_o = e->attn_o; aa.part_ml = e->attn_ml; aa.counters = e->cnt_attn;
            aa.ctx = (const int32_t*)(e->meta_dev + e->off_ctx);
            aa.page_table = (const int32_t*)(e->meta_dev + e->off_pt);
            aa.pt_stride = e->pt_stride;
            aa.B = nA; aa.G = GA; aa.n_heads = e->H; aa.head_dim = e->D; aa.d_model = d; aa.n_layers = L;
            if (pf) {
                aa.g_rows = (const int32_t*)(e->meta_dev + e->off_grows);
                aa.ctx_pre = (const int32_t*)(e->meta_dev + e->off_cpre);
            }
            aa.layer = l; aa.page_tokens = e->cfg.page_tokens; aa.nchunk = nchunk;
            aa.num_sms = e->num_sms;
            aa.scale_log2 = (float)(1.4426950408889634 / std::sqrt((double)e->D));
            aa.ktrace = e->ktrace;
            aa.ktrace_id = nl;
            aa.atrace = e->atrace ? e->atrace + (size_t)l * 16 : nullptr;
            if (e->attn_pf) {
                aa.pf_ptr = e->w_o[l];
                aa.pf_bytes = (size_t)d * d * 2;
                aa.pf_early = e->attn_pf == 2;
            }
            int a3s = e->attn_splits > 0 ? e->attn_splits : attn3_splits(nA, e->H, nchunk, e->num_sms);
            if (nA * e->H > e->a3_part_bh) a3s = 1;   // split partials must fit a3_part
            aa.part = e->a3_part;
            aa.epoch = (const uint32_t*)(e->meta_dev + e->off_epoch);
            aa.launch_id = nl;
            aa.cluster_launch = e->attn_no_cluster ? 0 : 1;
            LAUNCH(SV_K_ATTN, l, st, attn_bytes, attn_flops,
                   e->D == 128 ? attn3_launch(aa, a3s, max_ctx, st) : attn_launch(aa, st));
        }
        {   // O projection + residual
            GemmArgs a = base_args(e, M);
            a.h = e->h; a.g_out = e->norm_mlp[l]; a.u_out = e->u; a.ssq_out = ssq_at(e, l, 1);
            LAUNCH(SV_K_O, l, st, gemm_bytes(d, d, Md * 10 + (d / 128) * M * 4.0), 2.0 * M * d * d,
                   gemm(EPI_RESID, L + l, 1, d, d, a, st, false));
        }
        {   // gate/up + SwiGLU
            GemmArgs a = base_args(e, M);
            a.ssq_in = ssq_at(e, l, 1);
            a.act = e->act;
            LAUNCH(SV_K_GU, l, st, gemm_bytes(2.0 * F, d, (double)M * F * 2 + (d / 128) * M * 4.0),
                   2.0 * M * 2.0 * F * d, gemm(EPI_SWIGLU, 2 * L + l, 0, 2 * F, d, a, st, false));
        }
        {   // down + residual (+ early-exit copy with the final gain)
            GemmArgs a = base_args(e, M);
            a.h = e->h;
            a.g_out = (l + 1 < L) ? e->norm_attn[l + 1] : e->norm_final;
            a.u_out = e->u;
            if (is_exit_l) {   // exit copy: bf16(h * g) for the head, or for the adapter (+ fp32 h)
                const bool ad = e->ad_rank > 0 && l + 1 < L;
                a.g_out2 = ad ? e->ad_g[l] : e->norm_final;
                a.u_out2 = e->u_exit + (size_t)exit_k * e->MP * d;
                if (ad) a.h_out2 = e->h_exit + (size_t)exit_k * e->MP * d;
            }
            a.ssq_out = ssq_at(e, l + 1, 0);
            LAUNCH(SV_K_DOWN, l, st, gemm_bytes(d, F, Md * (is_exit_l ? 12 : 10) + (d / 128) * M * 4.0),
                   2.0 * M * d * F,
                   gemm(EPI_RESID, 3 * L + l, 2, d, F, a, st, false));
        }
        if (is_exit_l) {   // fork early exit k (S10-S11), streamed to mailbox row k
            if ((r = cudaEventRecord(e->ev_fork, st)) != cudaSuccess) return r;
            if ((r = cudaStreamWaitEvent(e->s_exit, e->ev_fork, 0)) != cudaSuccess) return r;
            if (e->ad_rank > 0 && l + 1 < L) {   // NEXT-3: A_l(h) = h + silu(RMSNorm(h) g W_dn^T) W_up^T
                const int R = e->ad_rank;
                GemmArgs g1 = base_args(e, M);
                g1.ssq_in = ssq_at(e, l + 1, 0);
                g1.b_row0 = exit_k * e->MP;
                g1.act = e->act_ad;
                LAUNCH(SV_K_LM_EXIT, l, e->s_exit, gemm_bytes(R, d, (double)M * R * 2), 2.0 * M * R * d,
                       gemm(EPI_SILU, 4 * L + 1 + l, 3, R, d, g1, e->s_exit, true));
                GemmArgs g2 = base_args(e, M);
                g2.h = e->h_exit + (size_t)exit_k * e->MP * d;
                g2.g_out = e->norm_final;
                g2.u_out = e->u_ad;
                g2.ssq_out = e->ssq_ad;
                LAUNCH(SV_K_LM_EXIT, l, e->s_exit, gemm_bytes(d, R, Md * 10), 2.0 * M * d * R,
                       gemm(EPI_RESID, 4 * L + 1 + L + l, 4, d, R, g2, e->s_exit, true));
                if ((r = lm_and_accept(e->s_exit, true, l + 1, -1, 1 + exit_k)) != cudaSuccess) return r;
            } else if ((r = lm_and_accept(e->s_exit, true, l + 1, exit_k, 1 + exit_k)) != cudaSuccess) {
                return r;
            }
            if ((r = cudaMemcpyAsync(e->mb_exit + (size_t)exit_k * e->opts.max_batch, e->res_exit_dev,
                                     (size_t)n * sizeof(sv_exit_result), cudaMemcpyDeviceToHost, e->s_exit)) !=
                cudaSuccess)
                return r;
            if ((r = cudaMemcpyAsync((void*)(e->mb_flag + exit_k), e->meta_dev + e->off_seq, 8,
                                     cudaMemcpyDeviceToHost, e->s_exit)) != cudaSuccess)
                return r;
            ++exit_k;
            if (exit_k == n_exits && (r = cudaEventRecord(e->ev_join, e->s_exit)) != cudaSuccess) return r;
        }
    }
    if ((r = lm_and_accept(st, false, L, 0, 1 + L)) != cudaSuccess) return r;
    if ((r = cudaMemcpyAsync(e->mb_final, e->res_final_dev, (size_t)n * sizeof(sv_exit_result), cudaMemcpyDeviceToHost,
                             st)) != cudaSuccess)
        return r;
    if (n_exits > 0)
        if ((r = cudaStreamWaitEvent(st, e->ev_join, 0)) != cudaSuccess) return r;
#undef LAUNCH
    *launches = nl;
    return cudaSuccess;
}

static sv_status run_step(sv_engine* e, cudaStream_t st, int n, int gamma, uint64_t exit_mask, int nchunk) {
    *(uint32_t*)(e->meta_host + e->off_epoch) = ++e->epoch & 0x3FFFFF;   // fresh split-K tags for this step
    CK(cudaMemcpyAsync(e->meta_dev, e->meta_host, e->meta_bytes, cudaMemcpyHostToDevice, st));
    int nl = 0;
    const bool trace = (e->trace_env || e->trace_next) && !e->prof;
    e->trace_next = false;
    e->trace_valid = trace;
    e->ktrace = trace ? e->ktrace_buf : nullptr;
    if (!e->opts.use_graphs || e->prof) {
        const cudaError_t r = issue_step(e, st, n, gamma, exit_mask, nchunk, &nl);
        e->ktrace = nullptr;
        CK(r);
        e->last_launches = nl;
        if (trace) e->last_kmeta = e->kmeta;
        return SV_OK;
    }
    StepKey key{n, gamma, exit_mask, nchunk, trace};
    auto it = e->graphs.find(key);
    if (it == e->graphs.end()) {
        cudaGraph_t g;
        CK(cudaStreamBeginCapture(e->s_cap, cudaStreamCaptureModeThreadLocal));
        cudaError_t r = issue_step(e, e->s_cap, n, gamma, exit_mask, nchunk, &nl);
        cudaError_t r2 = cudaStreamEndCapture(e->s_cap, &g);
        e->ktrace = nullptr;
        if (r != cudaSuccess) return fail(SV_E_DEVICE, std::string("capture: ") + cudaGetErrorString(r));
        CK(r2);
        cudaGraphExec_t ex;
        CK(cudaGraphInstantiate(&ex, g, 0));
        CK(cudaGraphDestroy(g));
        it = e->graphs.emplace(key, ex).first;
        e->graph_kmeta[key] = e->kmeta;
        e->last_launches = nl;
    }
    e->ktrace = nullptr;
    if (trace) e->last_kmeta = e->graph_kmeta[key];
    CK(cudaGraphLaunch(it->second, st));
    return SV_OK;
}

extern "C" sv_status sv_verify_submit_exits(sv_engine* e, const sv_verify_req* reqs, int32_t n,
                                            const int32_t* exit_layers, int32_t n_exits, sv_exit_result* early,
                                            sv_exit_result* final_, void* stream, sv_ticket** out) {
    if (!e || !reqs || !final_ || !out || n < 1) return fail(SV_E_INVALID, "bad arguments");
    std::lock_guard<std::mutex> lk(e->mu);
    if (e->poisoned) return fail(SV_E_DEVICE, "engine poisoned by an earlier CUDA error");
    if (e->inflight) return fail(SV_E_BUSY, "a ticket is already in flight on this engine");
    if (n > e->opts.max_batch) return fail(SV_E_CAPACITY, "n > max_batch");
    if (n_exits < 0 || n_exits > e->L || (n_exits > 0 && !exit_layers))
        return fail(SV_E_INVALID, "bad exit layer list");
    if (n_exits > 0 && !early) return fail(SV_E_INVALID, "early result array required when exits are requested");
    if (n_exits > 0 && e->L > 64) return fail(SV_E_INVALID, "early exits need n_layers <= 64");
    uint64_t exit_mask = 0;
    for (int k = 0; k < n_exits; ++k) {
        if (exit_layers[k] < 1 || exit_layers[k] > e->L) return fail(SV_E_INVALID, "exit layer out of range");
        if (k > 0 && exit_layers[k] <= exit_layers[k - 1]) return fail(SV_E_INVALID, "exit layers must ascend");
        exit_mask |= 1ull << (exit_layers[k] - 1);
    }
    const int gamma = reqs[0].gamma;
    if (gamma < 0 || gamma > e->opts.max_gamma) return fail(SV_E_INVALID, "gamma out of range");
    for (int i = 0; i < n; ++i) {
        const sv_verify_req& q = reqs[i];
        if (!q.session || q.session->e != e) return fail(SV_E_INVALID, "request without a session of this engine");
        if (q.gamma != gamma) return fail(SV_E_INVALID, "gamma must be equal for all requests of a submit");
        if (!q.draft_tokens && gamma > 0) return fail(SV_E_INVALID, "draft_tokens is NULL");
        if (q.pending_token < 0 || q.pending_token >= e->V) return fail(SV_E_INVALID, "pending token out of range");
        for (int j = 0; j < gamma; ++j)
            if (q.draft_tokens[j] < 0 || q.draft_tokens[j] >= e->V) return fail(SV_E_INVALID, "draft token out of range");
        if (q.session->busy) return fail(SV_E_BUSY, "session has a ticket in flight");
        for (int k = 0; k < i; ++k)
            if (reqs[k].session == q.session) return fail(SV_E_INVALID, "session twice in one submit");
    }
    CK(cudaSetDevice(e->device));
    cudaStream_t st = (cudaStream_t)stream;
    const int G = gamma + 1;
    sv_ticket* t = new sv_ticket();
    t->t_submit = std::chrono::steady_clock::now();
    t->exit_host_ms.assign(n_exits, -1.0);
    t->e = e; t->n = n; t->early = early; t->final_ = final_;
    t->exits.assign(exit_layers, exit_layers + n_exits);
    t->exit_done.assign(n_exits, false);
    t->gpu_slot.assign(n, -1);
    t->host_status.assign(n, SV_OK);
    // a CUDA failure after sessions were taken: release them and the ticket, poison
    auto abort_submit = [&](const std::string& msg) -> sv_status {
        e->poisoned = true;
        for (size_t i = 0; i < t->sess.size(); ++i)
            if (t->gpu_slot[i] >= 0) t->sess[i]->busy = false;
        if (t->ev_done) cudaEventDestroy(t->ev_done);
        delete t;
        return fail(SV_E_DEVICE, msg);
    };
    // S0: validate protocol state, build the batch of valid requests
    int nb = 0, max_len = 0;
    uint8_t* mh = e->meta_host;
    int32_t* tok = (int32_t*)(mh + e->off_tok);
    int32_t* pos = (int32_t*)(mh + e->off_pos);
    int32_t* rreq = (int32_t*)(mh + e->off_req);
    int32_t* ctxa = (int32_t*)(mh + e->off_ctx);
    int32_t* pt = (int32_t*)(mh + e->off_pt);
    ReqDev* rd = (ReqDev*)(mh + e->off_reqdev);
    for (int i = 0; i < n; ++i) {
        const sv_verify_req& q = reqs[i];
        sv_session* s = q.session;
        t->sess.push_back(s);
        t->rounds.push_back(q.round_id);
        t->ctx.push_back(s->len);
        if (q.round_id != s->last_round + 1 || q.prefix_len != s->len + 1) {
            t->host_status[i] = SV_E_PROTOCOL;
            continue;
        }
        if (s->len + G > e->cfg.max_ctx || !ensure_blocks(e, s, s->len + G)) {
            t->host_status[i] = SV_E_CAPACITY;
            continue;
        }
        const int b = nb++;
        t->gpu_slot[i] = b;
        for (int j = 0; j < G; ++j) {
            tok[b * G + j] = j == 0 ? q.pending_token : q.draft_tokens[j - 1];
            pos[b * G + j] = s->len + j;
            rreq[b * G + j] = b;
        }
        ctxa[b] = s->len;
        for (size_t k = 0; k < s->blocks.size(); ++k) pt[b * e->pt_stride + k] = s->blocks[k];
        ReqDev& r = rd[b];
        memset(&r, 0, sizeof(r));
        r.philox_seed = s->seed;
        r.session_id = (uint32_t)s->id;
        r.round_id = q.round_id;
        r.ctx = s->len;
        for (int j = 0; j < gamma; ++j) r.drafts[j] = q.draft_tokens[j];
        if (q.draft_probs) {
            if (q.probs_on_host) {
                float* dst = e->probs_stage + (size_t)b * e->opts.max_gamma * e->V;
                const cudaError_t ce =
                    cudaMemcpyAsync(dst, q.draft_probs, (size_t)gamma * e->V * 4, cudaMemcpyHostToDevice, st);
                if (ce != cudaSuccess) return abort_submit(std::string("draft probs H2D: ") + cudaGetErrorString(ce));
                r.probs = (uint64_t)dst;
            } else {
                r.probs = (uint64_t)q.draft_probs;
            }
        }
        max_len = std::max(max_len, s->len + G);
        s->busy = true;
    }
    t->nb = nb;
    t->gamma = gamma;
    t->seq = ++e->seq;
    *(uint64_t*)(mh + e->off_seq) = t->seq;
    t->has_gpu = nb > 0;
    {
        const cudaError_t ce = cudaEventCreateWithFlags(&t->ev_done, cudaEventDisableTiming);
        if (ce != cudaSuccess) {
            t->ev_done = nullptr;
            return abort_submit(std::string("cudaEventCreate: ") + cudaGetErrorString(ce));
        }
    }
    if (t->has_gpu) {
        int nchunk = (max_len + 63) / 64;
        nchunk = std::min(e->max_nchunk, nchunk);   // exact: no empty attention work items
        if (run_step(e, st, nb, gamma, exit_mask, nchunk)) return abort_submit(g_err);
    }
    {
        const cudaError_t ce = cudaEventRecord(t->ev_done, st);
        if (ce != cudaSuccess) return abort_submit(std::string("cudaEventRecord: ") + cudaGetErrorString(ce));
    }
    e->inflight = t;
    *out = t;
    return SV_OK;
}

extern "C" sv_status sv_verify_submit(sv_engine* e, const sv_verify_req* reqs, int32_t n, int32_t exit_layer,
                                      sv_exit_result* early, sv_exit_result* final_, void* stream, sv_ticket** out) {
    if (exit_layer < 0 || (e && exit_layer > e->L)) return fail(SV_E_INVALID, "exit_layer out of range");
    return sv_verify_submit_exits(e, reqs, n, &exit_layer, exit_layer > 0 ? 1 : 0, early, final_, stream, out);
}

static double ms_since(std::chrono::steady_clock::time_point t0) {
    return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
}

extern "C" sv_status sv_debug_trace_next(sv_engine* e) {
    if (!e) return fail(SV_E_INVALID, "NULL engine");
    std::lock_guard<std::mutex> lk(e->mu);
    e->trace_next = true;
    return SV_OK;
}

extern "C" sv_status sv_debug_trace_read(sv_engine* e, sv_trace_rec* out, int32_t cap, int32_t* n_out) {
    if (!e || !n_out || (cap > 0 && !out)) return fail(SV_E_INVALID, "NULL argument");
    std::lock_guard<std::mutex> lk(e->mu);
    if (e->inflight) return fail(SV_E_BUSY, "a ticket is in flight");
    if (!e->trace_valid) return fail(SV_E_INVALID, "the last submit was not traced");
    const auto& km = e->last_kmeta;
    std::vector<unsigned long long> tr(2 * km.size());
    CK(cudaSetDevice(e->device));
    CK(cudaMemcpy(tr.data(), e->ktrace_buf, tr.size() * 8, cudaMemcpyDeviceToHost));
    unsigned long long t0 = ~0ull;
    for (size_t i = 0; i < km.size(); ++i)
        if (km[i].kind >= 0) t0 = std::min(t0, tr[2 * i]);
    int k = 0;
    for (size_t i = 0; i < km.size(); ++i) {
        if (km[i].kind < 0) continue;
        if (k < cap) {
            sv_trace_rec& r = out[k];
            r.kind = km[i].kind;
            r.layer = km[i].layer;
            r.stream = km[i].stream;
            r.pad = 0;
            r.start_ns = tr[2 * i] - t0;
            r.end_ns = ~tr[2 * i + 1] - t0;
        }
        ++k;
    }
    *n_out = k;
    return SV_OK;
}

extern "C" sv_status sv_ticket_timing(sv_ticket* t, double* exit_dev_ms, double* final_dev_ms, double* exit_host_ms,
                                      double* final_host_ms) {
    if (!t) return fail(SV_E_INVALID, "NULL ticket");
    if (!t->final_done) return fail(SV_E_INVALID, "timing is available after sv_wait_final");
    sv_engine* e = t->e;
    const int ne = (int)t->exits.size();
    std::vector<unsigned long long> st(e->L + 2, 0);
    if (t->has_gpu) {
        CK(cudaSetDevice(e->device));
        CK(cudaMemcpy(st.data(), e->stamps_dev, st.size() * 8, cudaMemcpyDeviceToHost));
    }
    auto dev = [&](int slot) { return (t->has_gpu && st[slot] >= st[0] && st[0]) ? (st[slot] - st[0]) * 1e-6 : -1.0; };
    for (int k = 0; k < ne; ++k) {
        if (exit_dev_ms) exit_dev_ms[k] = dev(1 + k);
        if (exit_host_ms) exit_host_ms[k] = t->exit_host_ms[k];
    }
    if (final_dev_ms) *final_dev_ms = dev(1 + e->L);
    if (final_host_ms) *final_host_ms = t->final_host_ms;
    return SV_OK;
}

static void fill_host_result(sv_exit_result* r, const sv_ticket* t, int i, int exit_layer, int is_final) {
    memset(r, 0, sizeof(*r));
    r->round_id = t->rounds[i];
    r->exit_layer = exit_layer;
    r->is_final = is_final;
    r->status = t->host_status[i];
    r->new_len = t->ctx[i];
    for (int k = 0; k <= SV_MAX_GAMMA; ++k) r->tokens[k] = -1;
}

extern "C" sv_status sv_wait_exit(sv_ticket* t, int32_t k, int64_t timeout_us) {
    if (!t) return fail(SV_E_INVALID, "NULL ticket");
    if (k < 0 || k >= (int)t->exits.size()) return fail(SV_E_INVALID, "exit index out of range");
    sv_engine* e = t->e;
    if (t->exit_done[k]) return SV_OK;
    if (t->has_gpu) {
        const auto t0 = std::chrono::steady_clock::now();
        while (e->mb_flag[k] != t->seq) {
            const cudaError_t q = cudaEventQuery(t->ev_done);
            if (q == cudaSuccess) break;   // step already complete
            if (q != cudaErrorNotReady) {   // a kernel fault: the flag will never arrive
                e->poisoned = true;
                return fail(SV_E_DEVICE, std::string("step failed: ") + cudaGetErrorString(q));
            }
            if (timeout_us >= 0 &&
                std::chrono::duration_cast<std::chrono::microseconds>(std::chrono::steady_clock::now() - t0).count() >
                    timeout_us)
                return fail(SV_E_TIMEOUT, "early result not ready");
            std::this_thread::yield();
        }
    }
    if (t->exit_host_ms[k] < 0) t->exit_host_ms[k] = ms_since(t->t_submit);
    const sv_exit_result* row = e->mb_exit + (size_t)k * e->opts.max_batch;
    for (int i = 0; i < t->n; ++i) {
        sv_exit_result* dst = t->early + (size_t)k * t->n + i;
        if (t->gpu_slot[i] >= 0) *dst = row[t->gpu_slot[i]];
        else fill_host_result(dst, t, i, t->exits[k], 0);
    }
    t->exit_done[k] = true;
    return SV_OK;
}

extern "C" sv_status sv_exits_ready(sv_ticket* t, int32_t* n_ready) {
    if (!t || !n_ready) return fail(SV_E_INVALID, "NULL argument");
    sv_engine* e = t->e;
    int k = 0;
    const cudaError_t q = t->has_gpu ? cudaEventQuery(t->ev_done) : cudaSuccess;
    if (q != cudaSuccess && q != cudaErrorNotReady) {
        e->poisoned = true;
        return fail(SV_E_DEVICE, std::string("step failed: ") + cudaGetErrorString(q));
    }
    const bool all = q == cudaSuccess;
    while (k < (int)t->exits.size() && (all || e->mb_flag[k] == t->seq)) {
        if (t->exit_host_ms[k] < 0) t->exit_host_ms[k] = ms_since(t->t_submit);
        ++k;
    }
    *n_ready = k;
    return SV_OK;
}

extern "C" sv_status sv_wait_early(sv_ticket* t, int64_t timeout_us) {
    if (!t) return fail(SV_E_INVALID, "NULL ticket");
    for (int k = 0; k < (int)t->exits.size(); ++k) {
        sv_status s = sv_wait_exit(t, k, timeout_us);
        if (s) return s;
    }
    return SV_OK;
}

extern "C" sv_status sv_wait_final(sv_ticket* t, int64_t timeout_us) {
    if (!t) return fail(SV_E_INVALID, "NULL ticket");
    sv_engine* e = t->e;
    if (t->final_done) return SV_OK;
    const auto t0 = std::chrono::steady_clock::now();
    for (;;) {
        cudaError_t q = cudaEventQuery(t->ev_done);
        if (q == cudaSuccess) {
            if (t->final_host_ms < 0) t->final_host_ms = ms_since(t->t_submit);
            break;
        }
        if (q != cudaErrorNotReady) {
            e->poisoned = true;
            return fail(SV_E_DEVICE, std::string("step failed: ") + cudaGetErrorString(q));
        }
        if (timeout_us >= 0 &&
            std::chrono::duration_cast<std::chrono::microseconds>(std::chrono::steady_clock::now() - t0).count() >
                timeout_us)
            return fail(SV_E_TIMEOUT, "final result not ready");
        std::this_thread::yield();
    }
    sv_wait_early(t, -1);
    std::lock_guard<std::mutex> lk(e->mu);
    for (int i = 0; i < t->n; ++i) {
        sv_session* s = t->sess[i];
        if (t->gpu_slot[i] >= 0) {
            t->final_[i] = e->mb_final[t->gpu_slot[i]];
            const sv_exit_result& r = t->final_[i];
            if (r.status == SV_OK) {   // S14: rollback = keep ctx + 1 + delta rows
                s->len = r.new_len;
                s->last_round = r.round_id;
            }
            s->busy = false;
        } else {
            fill_host_result(&t->final_[i], t, i, e->L, 1);
        }
    }
    t->final_done = true;
    if (e->trace_valid && e->trace_env) {   // per-launch timeline of this step (SV_KTRACE=<csv>)
        std::vector<unsigned long long> tr(2 * e->last_kmeta.size());
        if (cudaMemcpy(tr.data(), e->ktrace_buf, tr.size() * 8, cudaMemcpyDeviceToHost) == cudaSuccess) {
            FILE* fp = fopen(getenv("SV_KTRACE"), "w");
            if (fp) {
                fprintf(fp, "id,kind,layer,start_ns,end_ns\n");
                for (size_t i = 0; i < e->last_kmeta.size(); ++i)
                    fprintf(fp, "%zu,%d,%d,%llu,%llu\n", i, e->last_kmeta[i].kind, e->last_kmeta[i].layer, tr[2 * i],
                            ~tr[2 * i + 1]);
                fclose(fp);
            }
        }
    }
    if (e->gtrace && e->trace_valid) {   // GEMM phase stamps of this traced step (SV_GTRACE=<csv>)
        std::vector<unsigned long long> tr((size_t)1024 * 32);
        if (cudaMemcpy(tr.data(), e->gtrace, tr.size() * 8, cudaMemcpyDeviceToHost) == cudaSuccess) {
            FILE* fp = fopen(getenv("SV_GTRACE"), "w");
            if (fp) {
                fprintf(fp, "id,kind,layer,phase,first_ns,last_ns\n");
                for (size_t i = 0; i < e->last_kmeta.size(); ++i)
                    for (int p = 0; p < 16; ++p)
                        if (tr[(i * 16 + p) * 2] != ~0ull)
                            fprintf(fp, "%zu,%d,%d,%d,%llu,%llu\n", i, e->last_kmeta[i].kind, e->last_kmeta[i].layer, p,
                                    tr[(i * 16 + p) * 2], ~tr[(i * 16 + p) * 2 + 1]);
                fclose(fp);
            }
        }
    }
    if (e->atrace && getenv("SV_ATRACE")) {   // attention phase stamps of this step
        std::vector<unsigned long long> tr((size_t)e->L * 16);
        if (cudaMemcpy(tr.data(), e->atrace, tr.size() * 8, cudaMemcpyDeviceToHost) == cudaSuccess) {
            FILE* fp = fopen(getenv("SV_ATRACE"), "w");
            if (fp) {
                fprintf(fp, "layer,cta,phase,t_ns\n");
                for (int l = 0; l < e->L; ++l)
                    for (int k = 0; k < 16; ++k) fprintf(fp, "%d,%d,%d,%llu\n", l, k / 8, k % 8, tr[l * 16 + k]);
                fclose(fp);
            }
        }
    }
    e->inflight = nullptr;
    return SV_OK;
}

extern "C" sv_status sv_ticket_release(sv_ticket* t) {
    if (!t) return fail(SV_E_INVALID, "NULL ticket");
    if (!t->final_done) {
        sv_status s = sv_wait_final(t, -1);
        if (s) return s;
    }
    cudaEventDestroy(t->ev_done);
    delete t;
    return SV_OK;
}

// ------------------------------------------------------------------ prefill
// append a prompt of n tokens to the session's KV cache in
// one pass (query blocks of 16 rows (8 if head_dim != 128) as attention requests
// over the shared page table, causal inside the prompt) and emit the next token
// from the last row (argmax, or a race sample of p with the session's Philox
// stream at round_id = last_round + 1).  Synchronous, no CUDA graph.
static sv_status prefill_pass(sv_session* s, const int32_t* tokens, int32_t n, int32_t sample, sv_exit_result* out,
                              float* logits_dev) {
    if (!s || !tokens || !out || n < 1) return fail(SV_E_INVALID, "bad arguments");
    sv_engine* e = s->e;
    std::lock_guard<std::mutex> lk(e->mu);
    if (e->poisoned) return fail(SV_E_DEVICE, "engine poisoned by an earlier CUDA error");
    if (e->inflight || s->busy) return fail(SV_E_BUSY, "a ticket is in flight");
    if (n > e->opts.max_prefill) return fail(SV_E_CAPACITY, "n > max_prefill");
    for (int i = 0; i < n; ++i)
        if (tokens[i] < 0 || tokens[i] >= e->V) return fail(SV_E_INVALID, "token out of range");
    const int gb = e->D == 128 ? 16 : 8, nq = (n + gb - 1) / gb;
    const int len = s->len;
    if (len + nq * gb > e->cfg.max_ctx || !ensure_blocks(e, s, len + nq * gb))
        return fail(SV_E_CAPACITY, "kv capacity");
    CK(cudaSetDevice(e->device));
    uint8_t* mh = e->meta_host;
    int32_t* tok = (int32_t*)(mh + e->off_tok);
    int32_t* pos = (int32_t*)(mh + e->off_pos);
    int32_t* rreq = (int32_t*)(mh + e->off_req);
    int32_t* ctxa = (int32_t*)(mh + e->off_ctx);
    int32_t* pt = (int32_t*)(mh + e->off_pt);
    int32_t* grows = (int32_t*)(mh + e->off_grows);
    int32_t* cpre = (int32_t*)(mh + e->off_cpre);
    for (int i = 0; i < n; ++i) {
        tok[i] = tokens[i];
        pos[i] = len + i;
        rreq[i] = i / gb;
    }
    for (int b = 0; b < nq; ++b) {
        ctxa[b] = len + b * gb;
        grows[b] = std::min(gb, n - b * gb);
        cpre[b] = len;
        for (size_t k = 0; k < s->blocks.size(); ++k) pt[b * e->pt_stride + k] = s->blocks[k];
    }
    ReqDev* rd = (ReqDev*)(mh + e->off_reqdev);
    memset(rd, 0, sizeof(ReqDev));
    rd->philox_seed = s->seed;
    rd->session_id = (uint32_t)s->id;
    rd->round_id = s->last_round + 1;
    rd->ctx = len;
    rd->probs = sample ? (uint64_t)e->logits_final : 0;   // gamma = 0: never read, non-zero = sample
    cudaStream_t st = e->s_cap;
    *(uint32_t*)(mh + e->off_epoch) = ++e->epoch & 0x3FFFFF;   // fresh split-K tags for this pass
    CK(cudaMemcpyAsync(e->meta_dev, e->meta_host, e->meta_bytes, cudaMemcpyHostToDevice, st));
    e->pf.on = true;
    e->pf.all_rows = logits_dev != nullptr;
    e->pf.n_tokens = n;
    e->pf.nq = nq;
    e->pf.gb = gb;
    int nl = 0;
    const int nchunk = std::min(e->max_nchunk, (len + n + 63) / 64);
    cudaError_t r = issue_step(e, st, 1, 0, 0ull, nchunk, &nl);
    e->pf.on = false;
    e->pf.all_rows = false;
    if (r == cudaSuccess) r = cudaMemcpyAsync(out, e->res_final_dev, sizeof(sv_exit_result), cudaMemcpyDeviceToHost, st);
    if (r == cudaSuccess && logits_dev)
        r = cudaMemcpyAsync(logits_dev, e->logits_final, (size_t)n * e->V * 4, cudaMemcpyDeviceToDevice, st);
    if (r == cudaSuccess) r = cudaStreamSynchronize(st);
    if (r != cudaSuccess) {
        e->poisoned = true;
        return fail(SV_E_DEVICE, std::string("prefill: ") + cudaGetErrorString(r));
    }
    e->last_launches = nl;
    if (logits_dev) return SV_OK;   // non-committing: the written rows stay invisible
    if (out->status == SV_OK) {
        s->len = len + n;
        s->last_round = out->round_id;
        out->new_len = s->len;
    }
    return (sv_status)out->status;
}

extern "C" sv_status sv_prefill(sv_session* s, const int32_t* tokens, int32_t n, int32_t sample,
                                sv_exit_result* out) {
    return prefill_pass(s, tokens, n, sample, out, nullptr);
}

extern "C" sv_status sv_debug_forward(sv_session* s, const int32_t* tokens, int32_t n, float* logits_dev) {
    if (!logits_dev) return fail(SV_E_INVALID, "NULL logits");
    sv_exit_result r;
    return prefill_pass(s, tokens, n, 0, &r, logits_dev);
}

extern "C" sv_status sv_verify(sv_session* s, const sv_verify_req* req, int32_t exit_layer, sv_exit_result* early,
                               sv_exit_result* final_) {
    if (!s || !req) return fail(SV_E_INVALID, "NULL argument");
    if (req->session != s) return fail(SV_E_INVALID, "request session mismatch");
    sv_ticket* t = nullptr;
    sv_status st = sv_verify_submit(s->e, req, 1, exit_layer, early, final_, nullptr, &t);
    if (st) return st;
    if ((st = sv_wait_early(t, -1))) return st;
    if ((st = sv_wait_final(t, -1))) return st;
    return sv_ticket_release(t);
}

// ------------------------------------------------------------------ test hooks
extern "C" sv_status sv_debug_logits(sv_ticket* t, int32_t which, float* dst) {
    if (!t || !dst || (which != 0 && which != 1)) return fail(SV_E_INVALID, "bad arguments");
    sv_engine* e = t->e;
    if (!t->final_done) {
        sv_status s = sv_wait_final(t, -1);
        if (s) return s;
    }
    if (which == 0 && t->exits.empty()) return fail(SV_E_INVALID, "step had no early exit");
    if (!t->has_gpu) return SV_OK;
    const size_t bytes = (size_t)t->nb * (t->gamma + 1) * e->V * 4;
    CK(cudaMemcpy(dst, which == 0 ? e->logits_exit : e->logits_final, bytes, cudaMemcpyDeviceToDevice));
    return SV_OK;
}

extern "C" sv_status sv_debug_accept(sv_engine* e, const float* logits_dev, const sv_verify_req* reqs, int32_t n,
                                     sv_exit_result* out) {
    if (!e || !logits_dev || !reqs || !out || n < 1 || n > e->opts.max_batch) return fail(SV_E_INVALID, "bad arguments");
    std::lock_guard<std::mutex> lk(e->mu);
    if (e->inflight) return fail(SV_E_BUSY, "a ticket is in flight");
    const int gamma = reqs[0].gamma;
    if (gamma < 0 || gamma > e->opts.max_gamma) return fail(SV_E_INVALID, "gamma out of range");
    CK(cudaSetDevice(e->device));
    ReqDev* rd = (ReqDev*)(e->meta_host + e->off_reqdev);
    for (int i = 0; i < n; ++i) {
        const sv_verify_req& q = reqs[i];
        if (!q.session || q.gamma != gamma || !q.draft_tokens) return fail(SV_E_INVALID, "bad request");
        ReqDev& r = rd[i];
        memset(&r, 0, sizeof(r));
        r.philox_seed = q.session->seed;
        r.session_id = (uint32_t)q.session->id;
        r.round_id = q.round_id;
        r.ctx = q.session->len;
        for (int j = 0; j < gamma; ++j) {
            if (q.draft_tokens[j] < 0 || q.draft_tokens[j] >= e->V) return fail(SV_E_INVALID, "draft token range");
            r.drafts[j] = q.draft_tokens[j];
        }
        if (q.draft_probs && q.probs_on_host) return fail(SV_E_INVALID, "debug_accept takes device probs");
        r.probs = (uint64_t)q.draft_probs;
    }
    CK(cudaMemcpy(e->meta_dev + e->off_reqdev, rd, (size_t)n * sizeof(ReqDev), cudaMemcpyHostToDevice));
    AcceptArgs aa = {};
    aa.logits = logits_dev;
    aa.req = (const ReqDev*)(e->meta_dev + e->off_reqdev);
    aa.stats = e->stats_final;
    aa.race = e->race_final;
    aa.counters = e->cnt_acc_final;
    aa.out = e->res_final_dev;
    aa.B = n; aa.G = gamma + 1; aa.V = e->V; aa.nch = e->acc_nch; aa.chunk = e->acc_chunk;
    aa.exit_layer = e->L; aa.is_final = 1;
    CK(accept_launch(aa, 0));
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(out, e->res_final_dev, (size_t)n * sizeof(sv_exit_result), cudaMemcpyDeviceToHost));
    return SV_OK;
}

extern "C" sv_status sv_debug_gemm(sv_engine* e, const void* w_dev, const void* x_dev, int32_t N, int32_t K, int32_t M,
                                   float* out_dev) {
    if (!e || !w_dev || !x_dev || !out_dev) return fail(SV_E_INVALID, "NULL argument");
    if (N < 128 || N % 128 || K < 128 || K % 64 || M < 1 || M > e->max_rows) return fail(SV_E_INVALID, "bad shape");
    if ((uintptr_t)w_dev % 16 || (uintptr_t)x_dev % 16) return fail(SV_E_INVALID, "operands must be 16-byte aligned");
    std::lock_guard<std::mutex> lk(e->mu);
    if (e->inflight) return fail(SV_E_BUSY, "a ticket is in flight");
    CK(cudaSetDevice(e->device));
    GemmArgs a = base_args(e, M);
    a.N = N;
    a.K = K;
    a.ssq_in = nullptr;   // no folded norm: out = X W^T
    a.logits = out_dev;
    a.ws = e->ws_main;
    a.counters = e->cnt_main;
    a.sk_flags = e->flags_main;
    const int tl = gemm_config(e, M, N, K, false, a);
    const size_t part = a.stream_k ? (size_t)e->num_sms * tl * 128 : (size_t)a.splits * (N / 128) * e->MP * 128;
    if (part > e->ws_elems) return fail(SV_E_CAPACITY, "split partials exceed the engine's workspace");
    CUtensorMap A, B;
    if (!make_tmap_bf16(&A, w_dev, N, K, 128) || !make_tmap_bf16(&B, x_dev, M, K, tl))
        return fail(SV_E_DEVICE, "cuTensorMapEncodeTiled failed");
    *(uint32_t*)(e->meta_host + e->off_epoch) = ++e->epoch & 0x3FFFFF;   // fresh split-K tags
    CK(cudaMemcpy(e->meta_dev + e->off_epoch, e->meta_host + e->off_epoch, 4, cudaMemcpyHostToDevice));
    CK(gemm_launch(EPI_LOGITS, tl, A, B, a, 0));
    CK(cudaDeviceSynchronize());
    return SV_OK;
}

extern "C" sv_status sv_debug_kv_rows(sv_session* s, int32_t layer, int32_t first, int32_t count, void* k_host,
                                      void* v_host) {
    if (!s || !k_host || !v_host) return fail(SV_E_INVALID, "NULL argument");
    sv_engine* e = s->e;
    const int P = e->cfg.page_tokens, D = e->D, H = e->H;
    if (layer < 0 || layer >= e->L || first < 0 || count < 0 ||
        (size_t)(first + count) > s->blocks.size() * (size_t)P)
        return fail(SV_E_INVALID, "rows out of range");
    CK(cudaSetDevice(e->device));
    CK(cudaDeviceSynchronize());
    for (int i = 0; i < count; ++i) {
        const int pos = first + i;
        const size_t blk = s->blocks[pos / P];
        for (int kv = 0; kv < 2; ++kv) {
            const uint8_t* src = e->kv_pool + blk * e->blk_bytes +
                                 (((size_t)layer * 2 + kv) * H * P + (size_t)(pos % P)) * D * 2;
            uint8_t* dst = (uint8_t*)(kv ? v_host : k_host) + (size_t)i * e->d * 2;
            CK(cudaMemcpy2D(dst, (size_t)D * 2, src, (size_t)P * D * 2, (size_t)D * 2, H, cudaMemcpyDeviceToHost));
        }
    }
    return SV_OK;
}

extern "C" sv_status sv_debug_philox(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]) {
    if (!ctr || !key || !out) return fail(SV_E_INVALID, "NULL argument");
    sv_status s = require_sm100(0);
    if (s) {
        int dev = -1;
        if (cudaGetDevice(&dev) != cudaSuccess || require_sm100(dev)) return s;
    }
    uint32_t* d = nullptr;
    uint32_t in[6] = {ctr[0], ctr[1], ctr[2], ctr[3], key[0], key[1]};
    CK(cudaMalloc(&d, 64));
    CK(cudaMemcpy(d, in, 24, cudaMemcpyHostToDevice));
    CK(philox_launch(d, d + 8, 0));
    CK(cudaMemcpy(out, d + 8, 16, cudaMemcpyDeviceToHost));
    CK(cudaFree(d));
    return SV_OK;
}

extern "C" sv_status sv_session_rewind(sv_session* s, int32_t len) {
    if (!s) return fail(SV_E_INVALID, "NULL session");
    sv_engine* e = s->e;
    std::lock_guard<std::mutex> lk(e->mu);
    if (s->busy) return fail(SV_E_BUSY, "session has a ticket in flight");
    if (len < 0 || len > s->len) return fail(SV_E_INVALID, "rewind length must be in [0, cached length]");
    s->len = len;   // rows >= len become invisible; their pages stay allocated
    return SV_OK;
}

extern "C" sv_status sv_debug_profile_step(sv_engine* e, const sv_verify_req* reqs, int32_t n, int32_t exit_layer,
                                           sv_exit_result* early, sv_exit_result* final_, sv_kernel_prof* out,
                                           int32_t cap, int32_t* n_out) {
    if (!e || !out || !n_out) return fail(SV_E_INVALID, "NULL argument");
    std::vector<ProfRec> recs;
    e->prof = &recs;
    const bool pdl = g_use_pdl;
    g_use_pdl = false;   // serialise kernels so events bracket exactly one launch
    sv_ticket* t = nullptr;
    sv_status s = sv_verify_submit(e, reqs, n, exit_layer, early, final_, nullptr, &t);
    e->prof = nullptr;
    g_use_pdl = pdl;
    if (!s) s = sv_ticket_release(t);
    if (s) return s;
    CK(cudaDeviceSynchronize());
    int k = 0;
    for (auto& r : recs) {
        float ms = 0.f;
        cudaEventElapsedTime(&ms, r.a, r.b);
        if (k < cap) out[k] = sv_kernel_prof{r.kind, r.layer, ms, r.bytes, r.flops};
        ++k;
        cudaEventDestroy(r.a);
        cudaEventDestroy(r.b);
    }
    *n_out = k;
    return SV_OK;
}
