/*
 * sv.h — C ABI of the B200-native verify step of arXiv 2505.21594
 * ("speculative edge-cloud decoding with early exits").
 *
 * The library implements the server side of the paper's Draft-and-Verify loop:
 *   Verify(M_q, x_{t:t+gamma}, p_{t:t+gamma}) -> x_{t:t+delta+1}     (Eq. 2)
 * run by a target model with an early exit (Eq. 5), i.e. one
 * Llama-style decoder pass over the gamma+1 query tokens [pending, x_1..x_gamma]
 * against a paged KV cache (Eq. 3), an early-exit head
 * (final RMSNorm + LM head) at layer `exit_layer`,
 * Leviathan speculative-sampling acceptance (adopted by PAPER.md:24, :80) at the
 * exit and at the final layer, and KV rollback to the accepted length.
 *
 * Letters: p = TARGET distribution, q = DRAFT distribution (the north star's
 * convention; PAPER.md uses the opposite letters, R1).
 *
 * Conventions for every call:
 *  - plain C, no exceptions cross the ABI; every call returns sv_status;
 *  - "device" pointers are CUDA device memory of the engine's device (allocated
 *    by the caller, e.g. with torch); "host" pointers are ordinary or pinned host
 *    memory; each argument says which;
 *  - on failure sv_last_error() returns a thread-local message for the last
 *    failing call on that thread;
 *  - there is no CPU fallback: on a machine without an sm_100 device every call
 *    that needs the GPU returns SV_E_DEVICE.
 */
#ifndef SV_H_
#define SV_H_

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define SV_API __attribute__((visibility("default")))
#else
#define SV_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define SV_MAX_GAMMA 8
#define SV_ABI_VERSION 4

typedef enum {
    SV_OK = 0,
    SV_E_INVALID = 1,   /* bad argument (synchronous)                                   */
    SV_E_PROTOCOL = 2,  /* per request: drafted token with q_j(x_j) <= 0, or
                           round_id not the successor / prefix_len != cached_len + 1
                           (SPEC.md:284); that request's KV is not advanced             */
    SV_E_CAPACITY = 3,  /* KV pool or engine limits exhausted                           */
    SV_E_DEVICE = 4,    /* no sm_100 device, or a CUDA error (the engine is poisoned)   */
    SV_E_BUSY = 5,      /* a ticket is already in flight on this engine                 */
    SV_E_TIMEOUT = 6    /* sv_wait_* timed out (the ticket is still valid)              */
} sv_status;

SV_API const char* sv_status_str(sv_status s);
SV_API const char* sv_last_error(void);
SV_API int sv_abi_version(void);

/* ---------------------------------------------------------------- model ---- */

/* Llama-style decoder shape.  The paper names only "Llama2-7B";
 * constants follow HF Llama-2 (R6).  Constraints: d_model % 128 == 0,
 * head_dim in {32, 64, 128}, n_heads * head_dim == d_model, d_ff % 64 == 0,
 * vocab % 128 == 0, page_tokens == 64, max_ctx % page_tokens == 0, max_ctx <= 4096
 * (an attention CTA stages at most 64 pages of its page list). */
typedef struct {
    int32_t n_layers, d_model, n_heads, head_dim, d_ff, vocab, max_ctx, page_tokens;
    float rms_eps;      /* 1e-5  */
    float rope_theta;   /* 1e4   */
} sv_model_cfg;

/* Weight pointers (device, bf16, row-major, caller-owned; must outlive the engine).
 *   embed      [vocab][d]                      h^(0) = embed[token]           (Eq. 3)
 *   lm_head    [vocab][d]   norm_final [d]     z = (RMSNorm(h) * norm_final) lm_head^T
 *   w_qkv[l]   [3d][d]      rows 0..d-1 = W_q, d..2d-1 = W_k, 2d..3d-1 = W_v
 *   w_o[l]     [d][d]
 *   w_gu[l]    [2*d_ff][d]  64-row interleave: physical rows 128t..128t+63 are
 *                           W_gate rows 64t..64t+63, rows 128t+64..128t+127 are
 *                           W_up rows 64t..64t+63 (so one 128-row GEMM tile
 *                           holds matching gate/up rows for the SwiGLU epilogue)
 *   w_down[l]  [d][d_ff]
 *   norm_attn[l], norm_mlp[l]  [d]  RMSNorm gains                               */
typedef struct {
    void* embed;
    void* lm_head;
    void* norm_final;
    void** w_qkv;
    void** w_o;
    void** w_gu;
    void** w_down;
    void** norm_attn;
    void** norm_mlp;
} sv_weights;

/* Bytes of every weight tensor (host out params, any may be NULL). */
SV_API sv_status sv_weight_sizes(const sv_model_cfg* cfg, size_t* embed, size_t* lm_head,
                          size_t* norm, size_t* qkv, size_t* o, size_t* gu, size_t* down);

/* Fill all weights with the counter-hash random init (DESIGN.md "Input recipe",
 * bit-identical to oracle/gen.py).  `stream` is a cudaStream_t (NULL = legacy
 * default stream); asynchronous. */
SV_API sv_status sv_weights_generate(const sv_model_cfg* cfg, const sv_weights* w, uint64_t seed,
                              void* stream);

/* Exit adapters (structure only, random init): "adapter
 * layers after each layer ... Each adapter connects to the LM head",
 * 101M parameters over 31 exits of Llama2-7B.  Reading (DESIGN.md
 * R7b): for an early exit after layer l < n_layers the head reads
 *   A_l(h) = h + silu(RMSNorm(h) * g[l] . w_dn[l]^T) . w_up[l]^T
 * instead of h^(l).  Arrays [n_layers], entry l-1 = the adapter of layer l (entry
 * n_layers-1 unused: the final layer keeps the plain head); device bf16:
 *   w_dn [rank][d], w_up [d][rank], g [d];  rank % 128 == 0. */
typedef struct {
    int32_t rank;
    void** w_dn;
    void** w_up;
    void** g;
} sv_adapters;
SV_API sv_status sv_adapter_sizes(const sv_model_cfg* cfg, int32_t rank, size_t* dn, size_t* up, size_t* g);
/* Counter-hash random init of every adapter (bit-identical to oracle/gen.py
 * adapter_weights); asynchronous on `stream`. */
SV_API sv_status sv_adapters_generate(const sv_model_cfg* cfg, const sv_adapters* a, uint64_t seed, void* stream);

/* Bytes of one KV block: page_tokens positions of K and V for every layer
 * (layout DESIGN.md "Data layout in HBM": [layer][K|V][head][slot][head_dim] bf16). */
SV_API size_t sv_kv_block_bytes(const sv_model_cfg* cfg);

/* --------------------------------------------------------------- engine ---- */

typedef struct sv_engine sv_engine;
typedef struct sv_session sv_session;
typedef struct sv_ticket sv_ticket;

typedef struct {
    int32_t max_batch;   /* max requests per submit (>= 1)                          */
    int32_t max_gamma;   /* max draft length per submit (1..SV_MAX_GAMMA)           */
    int32_t use_graphs;  /* 1: replay one CUDA graph per (batch, gamma, exit, ctx)  */
    int32_t max_prefill; /* max prompt tokens of one sv_prefill (0 = no prefill;
                            sizes the activation buffers: rows = max(max_batch *
                            (max_gamma + 1), max_prefill))                      */
} sv_engine_opts;

/* kv_pool: device memory (caller-owned, >= one KV block), carved into blocks of
 * sv_kv_block_bytes().  Returns SV_E_DEVICE if `device` is not compute capability
 * 10.0 (sm_100a); there is no fallback. */
SV_API sv_status sv_engine_create(const sv_model_cfg* cfg, const sv_weights* w, const sv_engine_opts* opts,
                           int device, void* kv_pool, size_t kv_pool_bytes, sv_engine** out);
SV_API sv_status sv_engine_destroy(sv_engine* e);
/* Use exit adapters for every early exit (NULL: identity adapters, the plain
 * head).  The pointers must outlive the engine; invalidates captured graphs. */
SV_API sv_status sv_engine_set_adapters(sv_engine* e, const sv_adapters* a);
/* Kernels the last submit launched (graph nodes counted individually). */
SV_API sv_status sv_engine_last_launches(const sv_engine* e, int32_t* n_kernels);

/* A session is one client's KV cache.  philox_seed keys its random stream
 * (Philox4x32-10, counter = (element/4, row|purpose<<8, round_id, session_id)). */
SV_API sv_status sv_session_open(sv_engine* e, uint64_t session_id, uint64_t philox_seed, sv_session** out);
/* Synthetic KV for positions 0..len-1 (counter-hash bf16, sd 1; oracle/gen.py
 * synthetic_kv), sets the cached length to len.  Synchronous. */
SV_API sv_status sv_session_fill_kv(sv_session* s, int32_t len, uint64_t kv_seed);
SV_API sv_status sv_session_len(const sv_session* s, int32_t* len);
/* Client-driven rollback: make rows >= len invisible (0 <= len <= cached length).
 * No data moves; the next step writes from position len.  The round counter is
 * unchanged. */
SV_API sv_status sv_session_rewind(sv_session* s, int32_t len);
SV_API sv_status sv_session_close(sv_session* s);

/* ---------------------------------------------------------------- verify ---- */

typedef struct {
    sv_session* session;
    uint32_t round_id;            /* must be the session's last round + 1          */
    int32_t prefix_len;           /* tokens the client holds incl. pending
                                     (= cached_len + 1), else SV_E_PROTOCOL        */
    int32_t pending_token;        /* last verified token; its KV is written here   */
    int32_t gamma;                /* 0..max_gamma, equal for all requests of a submit;
                                     0 = plain autoregressive step (SURVEY.md §8(f) NEXT-2,
                                     "Cloud AR"): one query row, next token
                                     = argmax p_0 (draft_probs NULL) or a sample of p_0
                                     (draft_probs any non-NULL pointer, never read)      */
    const int32_t* draft_tokens;  /* host [gamma]: x_1..x_gamma (may be NULL if gamma = 0) */
    const float* draft_probs;     /* [gamma][vocab] fp32, row j-1 = q_j; NULL => greedy */
    int32_t probs_on_host;        /* 0: draft_probs is a device pointer, 1: host    */
} sv_verify_req;

typedef struct {
    uint32_t round_id;
    int32_t exit_layer;           /* layer the result was read at (L = final)      */
    int32_t is_final;
    int32_t status;               /* sv_status of this request                     */
    int32_t accepted;             /* delta in [0, gamma]                           */
    int32_t tokens[SV_MAX_GAMMA + 1]; /* tokens[0..delta-1] = x_1..x_delta; tokens[delta] = next */
    float score;                  /* max_{r<=delta} max_v p_r(v)  (Eq. 4; Alg-S s^(i)) */
    float next_prob;              /* p_delta(tokens[delta])                        */
    float min_margin;             /* smallest decision margin on the decision path  */
    int32_t new_len;              /* cached length after the step (final only)     */
} sv_exit_result;

/* Launch one verify step for n requests (asynchronous, on `stream`).
 * exit_layer: 0 = no early exit, else 1..n_layers; its result is written to
 * early[] mid-pass.  early / final_: host arrays [n] (any host memory), valid
 * after sv_wait_early / sv_wait_final.  The request arrays and host probs must
 * stay valid until sv_wait_final returns.  One ticket in flight per engine. */
SV_API sv_status sv_verify_submit(sv_engine* e, const sv_verify_req* reqs, int32_t n, int32_t exit_layer,
                           sv_exit_result* early, sv_exit_result* final_, void* stream,
                           sv_ticket** out);
SV_API sv_status sv_wait_early(sv_ticket* t, int64_t timeout_us);  /* all early exits of the ticket */
SV_API sv_status sv_wait_final(sv_ticket* t, int64_t timeout_us);   /* KV already rolled back */

/* All-exits streaming verify (Alg-S lines 1103-1106,
 * the server verifies the draft at every exit and pushes each
 * exit's result with its score as soon as that exit is computed; T-eeft,
 * 31 exits for Llama2-7B).
 * exit_layers: host [n_exits], strictly ascending, each in 1..n_layers (n_layers
 * itself = an exit at the final layer, bitwise equal to the final result);
 * n_exits <= n_layers <= 64.  Every exit
 * uses the same Philox counters as the final exit (R10) and none of
 * them changes the session (KV, length).
 * early: host [n_exits][n]; row k is valid after sv_wait_exit(t, k) (or after
 * sv_wait_early / sv_wait_final).  Errors: SV_E_INVALID for a bad list, otherwise
 * as sv_verify_submit (which is this call with {exit_layer} or no exit). */
SV_API sv_status sv_verify_submit_exits(sv_engine* e, const sv_verify_req* reqs, int32_t n,
                                        const int32_t* exit_layers, int32_t n_exits, sv_exit_result* early,
                                        sv_exit_result* final_, void* stream, sv_ticket** out);
/* Block until exit k (index into the submit's exit_layers) has been delivered to
 * the host (mapped-memory flag written by the device after that exit's results),
 * then copy its [n] results into early[k][.].  SV_E_TIMEOUT after timeout_us >= 0. */
SV_API sv_status sv_wait_exit(sv_ticket* t, int32_t k, int64_t timeout_us);
/* Non-blocking: number of exits (a prefix of exit_layers, in layer order) whose
 * results have reached host memory. */
SV_API sv_status sv_exits_ready(sv_ticket* t, int32_t* n_ready);
SV_API sv_status sv_ticket_release(sv_ticket* t);

/* Exit-ready latency of a completed ticket (valid after sv_wait_final, before
 * sv_ticket_release).  The paper's early exit exists to deliver a verified token
 * mid-verification (Eq. 5; Alg-S lines 1103-1106).
 *   exit_dev_ms [n_exits]: device time from the step's first kernel starting to the
 *       last request of exit k having its result written (globaltimer, ns resolution);
 *   final_dev_ms: the same for the final exit;
 *   exit_host_ms [n_exits]: host time from the submit call to the first observation
 *       (sv_wait_exit / sv_exits_ready / sv_wait_final) of exit k's mailbox flag;
 *   final_host_ms: host time from the submit call to sv_wait_final observing the
 *       step's completion.
 * Any pointer may be NULL; a value is -1 when it was not observed (no GPU work,
 * or the exit was never waited for).  Synchronous (one small device read). */
SV_API sv_status sv_ticket_timing(sv_ticket* t, double* exit_dev_ms, double* final_dev_ms, double* exit_host_ms,
                                  double* final_host_ms);

/* Prefill: append the prompt tokens[0..n) to the
 * session's KV cache in one pass (positions len..len+n-1, causal inside the
 * prompt, Eq. 3) and emit the next token from the last prompt row:
 * argmax (sample = 0) or a sample of p (sample = 1; the session's Philox stream at
 * round_id = last_round + 1, which the call consumes).  out->tokens[0] = next
 * token (the pending token of the first verify round), out->new_len = len + n.
 * Synchronous; n <= opts.max_prefill (SV_E_CAPACITY). */
SV_API sv_status sv_prefill(sv_session* s, const int32_t* tokens, int32_t n, int32_t sample, sv_exit_result* out);

/* The north star's synchronous form: verify(draft_tokens, draft_probs, kv) ->
 * accepted_len, early_exit_token, next_token, for one request. */
SV_API sv_status sv_verify(sv_session* s, const sv_verify_req* req, int32_t exit_layer,
                    sv_exit_result* early, sv_exit_result* final_);

/* ----------------------------------------------------------- test hooks ---- */

/* Copy the fp32 logits of the ticket's step: which 0 = exit, 1 = final;
 * dst: device [n][gamma+1][vocab].  Valid until the next submit. */
SV_API sv_status sv_debug_logits(sv_ticket* t, int32_t which, float* dst_device);
/* Run only the acceptance kernels on caller logits (device [n][gamma+1][vocab]);
 * sessions supply seeds / ids, nothing is committed.  Synchronous. */
SV_API sv_status sv_debug_accept(sv_engine* e, const float* logits_dev, const sv_verify_req* reqs,
                          int32_t n, sv_exit_result* out);
/* out[M][N] = X[M][K] . W[N][K]^T (fp32, device, row-major) through the step's
 * tcgen05 GEMM kernels, with the token tile / split-K / stream-K choice of a step
 * with M query rows (no folded norm, no fused epilogue).  W and X are bf16,
 * row-major, device, 16-byte aligned; N % 128 == 0, K % 64 == 0, 1 <= M <= the
 * engine's max rows (SV_E_INVALID otherwise; SV_E_CAPACITY when the split
 * partials would not fit the engine's workspace).  Used to run the rank-local
 * slices of the 8-way tensor-parallel decomposition (SURVEY.md
 * §8(f) NEXT-4: column / row splits of W_qkv, W_o, W_gate/up, W_down, W_lm on
 * 128-row / 64-column boundaries) on one GPU.  Synchronous; SV_E_BUSY while a
 * ticket is in flight. */
SV_API sv_status sv_debug_gemm(sv_engine* e, const void* w_dev, const void* x_dev, int32_t N, int32_t K, int32_t M,
                               float* out_dev);
/* Copy cached K and V rows first..first+count-1 of one layer to host
 * (bf16 [count][d_model], element [pos][head*head_dim + dim]).  Synchronous. */
SV_API sv_status sv_debug_kv_rows(sv_session* s, int32_t layer, int32_t first, int32_t count,
                           void* k_host, void* v_host);
/* Per-launch profile of one verify step: the step runs without graph replay and
 * without programmatic dependent launch, each kernel bracketed by CUDA events on
 * the stream it is launched on.  Commits like sv_verify (the caller may rewind).
 * bytes / flops = algorithmic work of the launch. */
enum {
    SV_K_EMBED = 0, SV_K_QKV = 1, SV_K_ATTN = 2, SV_K_O = 3, SV_K_GU = 4, SV_K_DOWN = 5,
    SV_K_LM_EXIT = 6, SV_K_ACCEPT_EXIT = 7, SV_K_LM_FINAL = 8, SV_K_ACCEPT_FINAL = 9
};
typedef struct {
    int32_t kind;    /* SV_K_*                                   */
    int32_t layer;   /* 0-based decoder layer, or -1             */
    float ms;        /* event-measured duration                  */
    double bytes;    /* algorithmic bytes read + written         */
    double flops;    /* algorithmic floating-point operations    */
} sv_kernel_prof;
SV_API sv_status sv_debug_profile_step(sv_engine* e, const sv_verify_req* reqs, int32_t n, int32_t exit_layer,
                                       sv_exit_result* early, sv_exit_result* final_, sv_kernel_prof* out,
                                       int32_t cap, int32_t* n_out);
/* Non-committing forward: run tokens[0..n) as one block at
 * positions len..len+n-1 of the session (causal inside the block, Eq. 3,
 * PAPER.md:96-100) through every layer and the final head, and write the fp32
 * logits of every row to logits_dev (device [n][vocab]).  The session is not
 * changed: its length and round counter stay, the K/V rows the pass wrote beyond
 * the cached length stay invisible.  Used for the GPU "KV-incremental == full
 * recompute" pin.  n <= opts.max_prefill.  Synchronous. */
SV_API sv_status sv_debug_forward(sv_session* s, const int32_t* tokens, int32_t n, float* logits_dev);
/* Per-launch timeline of one step as it runs in production (graph replay with
 * programmatic dependent launch): sv_debug_trace_next makes the next submit record,
 * for every kernel launch, the globaltimer of its first CTA's start and its last
 * CTA's end (a separately captured graph variant; untraced steps are unchanged).
 * After sv_wait_final, sv_debug_trace_read copies up to cap records (host) in
 * launch order; times are ns from the step's first kernel start; kind = SV_K_*,
 * layer 0-based or -1, stream 0 = main, 1 = exit stream.  *n_out = records. */
typedef struct {
    int32_t kind, layer, stream, pad;
    uint64_t start_ns, end_ns;
} sv_trace_rec;
SV_API sv_status sv_debug_trace_next(sv_engine* e);
SV_API sv_status sv_debug_trace_read(sv_engine* e, sv_trace_rec* out, int32_t cap, int32_t* n_out);
/* Philox4x32-10 evaluated on the device (host in/out).  Synchronous. */
SV_API sv_status sv_debug_philox(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]);

#ifdef __cplusplus
}
#endif
#endif /* SV_H_ */
