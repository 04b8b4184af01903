"""ctypes binding of include/sv.h — argument marshalling only.

Every step of the verify path runs in libsv.so (hand-written sm_100a kernels);
this module converts Python values to the C structs, and uses torch only to
allocate device memory (weights, KV pool, draft probabilities) and to pass CUDA
stream handles.  There is no CPU fallback: if libsv.so is missing the import of
the binding raises.
"""
import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SV_LIB", os.path.join(_HERE, "libsv.so"))

SV_MAX_GAMMA = 8
SV_OK, SV_E_INVALID, SV_E_PROTOCOL, SV_E_CAPACITY, SV_E_DEVICE, SV_E_BUSY, SV_E_TIMEOUT = range(7)


class SvError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{status_name(status)}: {msg}")
        self.status = status


class sv_model_cfg(C.Structure):
    _fields_ = [("n_layers", C.c_int32), ("d_model", C.c_int32), ("n_heads", C.c_int32),
                ("head_dim", C.c_int32), ("d_ff", C.c_int32), ("vocab", C.c_int32),
                ("max_ctx", C.c_int32), ("page_tokens", C.c_int32),
                ("rms_eps", C.c_float), ("rope_theta", C.c_float)]


class sv_weights(C.Structure):
    _fields_ = [("embed", C.c_void_p), ("lm_head", C.c_void_p), ("norm_final", C.c_void_p),
                ("w_qkv", C.POINTER(C.c_void_p)), ("w_o", C.POINTER(C.c_void_p)),
                ("w_gu", C.POINTER(C.c_void_p)), ("w_down", C.POINTER(C.c_void_p)),
                ("norm_attn", C.POINTER(C.c_void_p)), ("norm_mlp", C.POINTER(C.c_void_p))]


class sv_adapters(C.Structure):
    _fields_ = [("rank", C.c_int32), ("w_dn", C.POINTER(C.c_void_p)), ("w_up", C.POINTER(C.c_void_p)),
                ("g", C.POINTER(C.c_void_p))]


class sv_engine_opts(C.Structure):
    _fields_ = [("max_batch", C.c_int32), ("max_gamma", C.c_int32), ("use_graphs", C.c_int32),
                ("max_prefill", C.c_int32)]


class sv_verify_req(C.Structure):
    _fields_ = [("session", C.c_void_p), ("round_id", C.c_uint32), ("prefix_len", C.c_int32),
                ("pending_token", C.c_int32), ("gamma", C.c_int32),
                ("draft_tokens", C.POINTER(C.c_int32)), ("draft_probs", C.c_void_p),
                ("probs_on_host", C.c_int32)]


class sv_exit_result(C.Structure):
    _fields_ = [("round_id", C.c_uint32), ("exit_layer", C.c_int32), ("is_final", C.c_int32),
                ("status", C.c_int32), ("accepted", C.c_int32),
                ("tokens", C.c_int32 * (SV_MAX_GAMMA + 1)), ("score", C.c_float),
                ("next_prob", C.c_float), ("min_margin", C.c_float), ("new_len", C.c_int32)]

    def emitted(self):
        return [int(t) for t in self.tokens[: self.accepted + 1]]

    def asdict(self):
        return dict(round_id=self.round_id, exit_layer=self.exit_layer, is_final=self.is_final,
                    status=self.status, accepted=self.accepted, tokens=self.emitted(),
                    score=self.score, next_prob=self.next_prob, min_margin=self.min_margin,
                    new_len=self.new_len)


class sv_kernel_prof(C.Structure):
    _fields_ = [("kind", C.c_int32), ("layer", C.c_int32), ("ms", C.c_float), ("bytes", C.c_double),
                ("flops", C.c_double)]


class sv_trace_rec(C.Structure):
    _fields_ = [("kind", C.c_int32), ("layer", C.c_int32), ("stream", C.c_int32), ("pad", C.c_int32),
                ("start_ns", C.c_uint64), ("end_ns", C.c_uint64)]


KERNEL_KINDS = ["embed", "gemm_qkv", "attention", "gemm_o", "gemm_gate_up", "gemm_down",
                "gemm_lm_exit", "accept_exit", "gemm_lm_final", "accept_final"]

EXPORTS = {
    # name: (restype, argtypes)
    "sv_status_str": (C.c_char_p, [C.c_int]),
    "sv_last_error": (C.c_char_p, []),
    "sv_abi_version": (C.c_int, []),
    "sv_weight_sizes": (C.c_int, [C.POINTER(sv_model_cfg)] + [C.POINTER(C.c_size_t)] * 7),
    "sv_weights_generate": (C.c_int, [C.POINTER(sv_model_cfg), C.POINTER(sv_weights), C.c_uint64, C.c_void_p]),
    "sv_kv_block_bytes": (C.c_size_t, [C.POINTER(sv_model_cfg)]),
    "sv_engine_create": (C.c_int, [C.POINTER(sv_model_cfg), C.POINTER(sv_weights), C.POINTER(sv_engine_opts),
                                   C.c_int, C.c_void_p, C.c_size_t, C.POINTER(C.c_void_p)]),
    "sv_engine_destroy": (C.c_int, [C.c_void_p]),
    "sv_engine_last_launches": (C.c_int, [C.c_void_p, C.POINTER(C.c_int32)]),
    "sv_session_open": (C.c_int, [C.c_void_p, C.c_uint64, C.c_uint64, C.POINTER(C.c_void_p)]),
    "sv_session_fill_kv": (C.c_int, [C.c_void_p, C.c_int32, C.c_uint64]),
    "sv_session_len": (C.c_int, [C.c_void_p, C.POINTER(C.c_int32)]),
    "sv_session_close": (C.c_int, [C.c_void_p]),
    "sv_session_rewind": (C.c_int, [C.c_void_p, C.c_int32]),
    "sv_debug_profile_step": (C.c_int, [C.c_void_p, C.POINTER(sv_verify_req), C.c_int32, C.c_int32,
                                        C.POINTER(sv_exit_result), C.POINTER(sv_exit_result),
                                        C.POINTER(sv_kernel_prof), C.c_int32, C.POINTER(C.c_int32)]),
    "sv_verify_submit": (C.c_int, [C.c_void_p, C.POINTER(sv_verify_req), C.c_int32, C.c_int32,
                                   C.POINTER(sv_exit_result), C.POINTER(sv_exit_result), C.c_void_p,
                                   C.POINTER(C.c_void_p)]),
    "sv_verify_submit_exits": (C.c_int, [C.c_void_p, C.POINTER(sv_verify_req), C.c_int32, C.POINTER(C.c_int32),
                                         C.c_int32, C.POINTER(sv_exit_result), C.POINTER(sv_exit_result),
                                         C.c_void_p, C.POINTER(C.c_void_p)]),
    "sv_wait_exit": (C.c_int, [C.c_void_p, C.c_int32, C.c_int64]),
    "sv_adapter_sizes": (C.c_int, [C.POINTER(sv_model_cfg), C.c_int32] + [C.POINTER(C.c_size_t)] * 3),
    "sv_adapters_generate": (C.c_int, [C.POINTER(sv_model_cfg), C.POINTER(sv_adapters), C.c_uint64, C.c_void_p]),
    "sv_engine_set_adapters": (C.c_int, [C.c_void_p, C.POINTER(sv_adapters)]),
    "sv_prefill": (C.c_int, [C.c_void_p, C.POINTER(C.c_int32), C.c_int32, C.c_int32, C.POINTER(sv_exit_result)]),
    "sv_exits_ready": (C.c_int, [C.c_void_p, C.POINTER(C.c_int32)]),
    "sv_wait_early": (C.c_int, [C.c_void_p, C.c_int64]),
    "sv_wait_final": (C.c_int, [C.c_void_p, C.c_int64]),
    "sv_ticket_release": (C.c_int, [C.c_void_p]),
    "sv_ticket_timing": (C.c_int, [C.c_void_p, C.POINTER(C.c_double), C.POINTER(C.c_double),
                                   C.POINTER(C.c_double), C.POINTER(C.c_double)]),
    "sv_verify": (C.c_int, [C.c_void_p, C.POINTER(sv_verify_req), C.c_int32, C.POINTER(sv_exit_result),
                            C.POINTER(sv_exit_result)]),
    "sv_debug_logits": (C.c_int, [C.c_void_p, C.c_int32, C.c_void_p]),
    "sv_debug_accept": (C.c_int, [C.c_void_p, C.c_void_p, C.POINTER(sv_verify_req), C.c_int32,
                                  C.POINTER(sv_exit_result)]),
    "sv_debug_kv_rows": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.c_void_p, C.c_void_p]),
    "sv_debug_trace_next": (C.c_int, [C.c_void_p]),
    "sv_debug_trace_read": (C.c_int, [C.c_void_p, C.POINTER(sv_trace_rec), C.c_int32, C.POINTER(C.c_int32)]),
    "sv_debug_forward": (C.c_int, [C.c_void_p, C.POINTER(C.c_int32), C.c_int32, C.c_void_p]),
    "sv_debug_philox": (C.c_int, [C.POINTER(C.c_uint32), C.POINTER(C.c_uint32), C.POINTER(C.c_uint32)]),
    "sv_debug_gemm": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.c_void_p]),
}

_lib = None


def lib():
    """Load libsv.so (fails loudly if it was not built: there is no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} not built: run __graft_entry__.build() "
                              "(paper_2505_21594_b200/csrc/build.sh); there is no CPU fallback")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in EXPORTS.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def status_name(s: int) -> str:
    try:
        return lib().sv_status_str(s).decode()
    except Exception:
        return str(s)


def check(s: int):
    if s != SV_OK:
        raise SvError(s, lib().sv_last_error().decode())


def make_cfg(mc) -> sv_model_cfg:
    """workload.ModelCfg -> sv_model_cfg."""
    return sv_model_cfg(mc.n_layers, mc.d_model, mc.n_heads, mc.head_dim, mc.d_ff, mc.vocab,
                        mc.max_ctx, mc.page_tokens, mc.rms_eps, mc.rope_theta)


def _stream_handle(stream):
    if stream is None:
        import torch
        return C.c_void_p(torch.cuda.current_stream().cuda_stream)
    return C.c_void_p(getattr(stream, "cuda_stream", stream))


class Weights:
    """Device weights in one torch allocation, filled by sv_weights_generate (K7)."""

    def __init__(self, mc, seed: int, device: int = 0):
        import torch
        self.mc = mc
        self.cfg = make_cfg(mc)
        sz = [C.c_size_t() for _ in range(7)]
        check(lib().sv_weight_sizes(C.byref(self.cfg), *[C.byref(s) for s in sz]))
        embed, lm, norm, qkv, o, gu, down = [s.value for s in sz]
        al = lambda x: (x + 255) // 256 * 256
        L = mc.n_layers
        total = al(embed) + al(lm) + al(norm) + L * (al(qkv) + al(o) + al(gu) + al(down) + 2 * al(norm))
        self.buf = torch.empty(total, dtype=torch.uint8, device=f"cuda:{device}")
        base = self.buf.data_ptr()
        off = [0]

        def take(n):
            p = base + off[0]
            off[0] += al(n)
            return p
        self.ptr = dict(embed=take(embed), lm_head=take(lm), norm_final=take(norm))
        arrs = {k: (C.c_void_p * L)() for k in ("qkv", "o", "gu", "down", "norm_attn", "norm_mlp")}
        for l in range(L):
            arrs["qkv"][l] = take(qkv)
            arrs["o"][l] = take(o)
            arrs["gu"][l] = take(gu)
            arrs["down"][l] = take(down)
            arrs["norm_attn"][l] = take(norm)
            arrs["norm_mlp"][l] = take(norm)
        self._arrs = arrs
        self.w = sv_weights(self.ptr["embed"], self.ptr["lm_head"], self.ptr["norm_final"],
                            arrs["qkv"], arrs["o"], arrs["gu"], arrs["down"], arrs["norm_attn"],
                            arrs["norm_mlp"])
        check(lib().sv_weights_generate(C.byref(self.cfg), C.byref(self.w), seed, _stream_handle(None)))
        torch.cuda.synchronize()
        self.nbytes = total

    def tensor(self, name: str, layer: int = 0):
        """A torch bf16 view of one weight tensor (for bit-equality tests)."""
        import torch
        d, F, V = self.mc.d_model, self.mc.d_ff, self.mc.vocab
        shapes = dict(embed=(V, d), lm_head=(V, d), norm_final=(d,), qkv=(3 * d, d), o=(d, d),
                      gu=(2 * F, d), down=(d, F), norm_attn=(d,), norm_mlp=(d,))
        ptr = self.ptr[name] if name in self.ptr else self._arrs[name][layer]
        n = int(np.prod(shapes[name]))
        off = ptr - self.buf.data_ptr()
        return self.buf[off:off + 2 * n].view(torch.bfloat16).view(*shapes[name])


class Adapters:
    """Exit adapters (NEXT-3, structure only): device bf16 weights in one torch
    allocation, filled by sv_adapters_generate (bit-identical to oracle/gen.py)."""

    def __init__(self, mc, rank: int, seed: int, device: int = 0):
        import torch
        self.mc, self.rank = mc, rank
        cfg = make_cfg(mc)
        sz = [C.c_size_t() for _ in range(3)]
        check(lib().sv_adapter_sizes(C.byref(cfg), rank, *[C.byref(x) for x in sz]))
        dn, up, g = [x.value for x in sz]
        al = lambda x: (x + 255) // 256 * 256
        L = mc.n_layers
        self.buf = torch.empty(L * (al(dn) + al(up) + al(g)), dtype=torch.uint8, device=f"cuda:{device}")
        base = self.buf.data_ptr()
        arr = {k: (C.c_void_p * L)() for k in ("dn", "up", "g")}
        off = 0
        for l in range(L):
            for k, n in (("dn", dn), ("up", up), ("g", g)):
                arr[k][l] = base + off
                off += al(n)
        self._arr = arr
        self.a = sv_adapters(rank, arr["dn"], arr["up"], arr["g"])
        check(lib().sv_adapters_generate(C.byref(cfg), C.byref(self.a), seed, _stream_handle(None)))
        torch.cuda.synchronize()


class Session:
    def __init__(self, engine, handle, session_id, philox_seed):
        self.engine = engine
        self.h = handle
        self.session_id = session_id
        self.philox_seed = philox_seed
        self.last_round = 0

    @property
    def length(self) -> int:
        n = C.c_int32()
        check(lib().sv_session_len(self.h, C.byref(n)))
        return n.value

    def fill_kv(self, length: int, kv_seed: int):
        check(lib().sv_session_fill_kv(self.h, length, kv_seed))

    def rewind(self, length: int):
        check(lib().sv_session_rewind(self.h, length))

    def kv_rows(self, layer: int, first: int, count: int):
        """(K, V) bf16 bit patterns uint16 [count, d] of cached rows."""
        d = self.engine.mc.d_model
        k = np.zeros((count, d), dtype=np.uint16)
        v = np.zeros((count, d), dtype=np.uint16)
        check(lib().sv_debug_kv_rows(self.h, layer, first, count, k.ctypes.data, v.ctypes.data))
        return k, v

    def prefill(self, tokens, sample: bool = False):
        """Append the prompt to the KV cache; returns the sv_exit_result whose
        tokens[0] is the next token (the pending token of the first verify round)."""
        t = np.ascontiguousarray(np.asarray(tokens, dtype=np.int32))
        out = sv_exit_result()
        check(lib().sv_prefill(self.h, t.ctypes.data_as(C.POINTER(C.c_int32)), len(t), 1 if sample else 0,
                               C.byref(out)))
        self.last_round = out.round_id
        return out

    def debug_forward(self, tokens):
        """fp32 logits [n, V] (torch, on the engine's device) of tokens as one block after
        the cached context, without committing anything (sv_debug_forward)."""
        import torch
        t = np.ascontiguousarray(np.asarray(tokens, dtype=np.int32))
        out = torch.empty((len(t), self.engine.mc.vocab), dtype=torch.float32, device=f"cuda:{self.engine.device}")
        check(lib().sv_debug_forward(self.h, t.ctypes.data_as(C.POINTER(C.c_int32)), len(t),
                                     C.c_void_p(out.data_ptr())))
        return out

    def close(self):
        if self.h:
            check(lib().sv_session_close(self.h))
            self.h = None


class Request:
    """One verify request: pending token + gamma drafts (+ draft distributions q_j)."""

    def __init__(self, session, round_id, pending, drafts, probs=None, prefix_len=None):
        self.session = session
        self.round_id = round_id
        self.pending = int(pending)
        self.drafts = np.ascontiguousarray(np.asarray(drafts, dtype=np.int32))
        self.probs = probs            # torch cuda fp32 [gamma, V], numpy fp32 (host) or None
        self.prefix_len = session.length + 1 if prefix_len is None else prefix_len

    def to_c(self) -> sv_verify_req:
        r = sv_verify_req()
        r.session = self.session.h
        r.round_id = self.round_id
        r.prefix_len = self.prefix_len
        r.pending_token = self.pending
        r.gamma = len(self.drafts)
        r.draft_tokens = self.drafts.ctypes.data_as(C.POINTER(C.c_int32))
        if self.probs is None:
            r.draft_probs = None
            r.probs_on_host = 0
        elif isinstance(self.probs, np.ndarray):
            self._host = np.ascontiguousarray(self.probs, dtype=np.float32)
            r.draft_probs = self._host.ctypes.data
            r.probs_on_host = 1
        else:
            r.draft_probs = self.probs.data_ptr()
            r.probs_on_host = 0
        return r


class Ticket:
    def __init__(self, engine, handle, n, early, final, reqs, exit_layers=()):
        self.engine, self.h, self.n = engine, handle, n
        self.early, self.final = early, final
        self.exit_layers = list(exit_layers)
        self._keep = reqs

    def wait_early(self, timeout_us: int = -1):
        """Results of the (first) early exit; all exits are delivered on return."""
        check(lib().sv_wait_early(self.h, timeout_us))
        return [self.early[i] for i in range(self.n)]

    def wait_exit(self, k: int, timeout_us: int = -1):
        """Results [n] of exit k (the k-th of exit_layers), as soon as it has streamed in."""
        check(lib().sv_wait_exit(self.h, k, timeout_us))
        return [self.early[k * self.n + i] for i in range(self.n)]

    def exits_ready(self) -> int:
        n = C.c_int32()
        check(lib().sv_exits_ready(self.h, C.byref(n)))
        return n.value

    def wait_final(self, timeout_us: int = -1):
        check(lib().sv_wait_final(self.h, timeout_us))
        return [self.final[i] for i in range(self.n)]

    def logits(self, which: int, gamma: int):
        """fp32 logits [n_gpu_requests, gamma+1, V] of this step (which: 0 exit, 1 final)."""
        import torch
        V = self.engine.mc.vocab
        out = torch.empty((self.n, gamma + 1, V), dtype=torch.float32,
                          device=f"cuda:{self.engine.device}")
        check(lib().sv_debug_logits(self.h, which, C.c_void_p(out.data_ptr())))
        return out

    def timing(self):
        """Exit-ready latency after wait_final: dict(exit_dev_ms [n_exits], final_dev_ms,
        exit_host_ms [n_exits], final_host_ms) (include/sv.h sv_ticket_timing)."""
        ne = max(1, len(self.exit_layers))
        ed, eh = (C.c_double * ne)(), (C.c_double * ne)()
        fd, fh = C.c_double(), C.c_double()
        check(lib().sv_ticket_timing(self.h, ed, C.byref(fd), eh, C.byref(fh)))
        k = len(self.exit_layers)
        return dict(exit_dev_ms=list(ed)[:k], final_dev_ms=fd.value, exit_host_ms=list(eh)[:k],
                    final_host_ms=fh.value)

    def final_ready(self) -> bool:
        """Non-blocking: whether the final result has completed (sv_wait_final with a
        zero timeout; it consumes the results if so)."""
        s = lib().sv_wait_final(self.h, 0)
        if s == SV_E_TIMEOUT:
            return False
        check(s)
        return True

    def release(self):
        if self.h:
            check(lib().sv_ticket_release(self.h))
            self.h = None


class Engine:
    def __init__(self, mc, weights: Weights, max_batch: int = 1, max_gamma: int = 8,
                 kv_blocks: int = None, use_graphs: bool = True, device: int = 0, max_prefill: int = 0):
        import torch
        self.mc = mc
        self.device = device
        self.weights = weights
        self.cfg = make_cfg(mc)
        blk = lib().sv_kv_block_bytes(C.byref(self.cfg))
        if kv_blocks is None:
            kv_blocks = max_batch * ((mc.max_ctx + mc.page_tokens - 1) // mc.page_tokens + 1)
        self.kv_pool = torch.empty(blk * kv_blocks, dtype=torch.uint8, device=f"cuda:{device}")
        opts = sv_engine_opts(max_batch, max_gamma, 1 if use_graphs else 0, max_prefill)
        h = C.c_void_p()
        check(lib().sv_engine_create(C.byref(self.cfg), C.byref(weights.w), C.byref(opts), device,
                                     C.c_void_p(self.kv_pool.data_ptr()), blk * kv_blocks, C.byref(h)))
        self.h = h
        self.max_batch = max_batch

    def open_session(self, session_id: int, philox_seed: int) -> Session:
        h = C.c_void_p()
        check(lib().sv_session_open(self.h, session_id, philox_seed, C.byref(h)))
        return Session(self, h, session_id, philox_seed)

    def submit(self, reqs, exit_layer: int = 0, stream=None) -> Ticket:
        n = len(reqs)
        arr = (sv_verify_req * n)(*[r.to_c() for r in reqs])
        early = (sv_exit_result * n)()
        final = (sv_exit_result * n)()
        t = C.c_void_p()
        check(lib().sv_verify_submit(self.h, arr, n, exit_layer, early, final, _stream_handle(stream),
                                     C.byref(t)))
        return Ticket(self, t, n, early, final, (reqs, arr), [exit_layer] if exit_layer else [])

    def submit_exits(self, reqs, exit_layers, stream=None) -> Ticket:
        """All-exits streaming verify: one early result per layer in exit_layers (ascending)."""
        n = len(reqs)
        arr = (sv_verify_req * n)(*[r.to_c() for r in reqs])
        ex = (C.c_int32 * max(1, len(exit_layers)))(*exit_layers)
        early = (sv_exit_result * (max(1, len(exit_layers)) * n))()
        final = (sv_exit_result * n)()
        t = C.c_void_p()
        check(lib().sv_verify_submit_exits(self.h, arr, n, ex, len(exit_layers), early, final,
                                           _stream_handle(stream), C.byref(t)))
        return Ticket(self, t, n, early, final, (reqs, arr, ex), exit_layers)

    def verify(self, reqs, exit_layer: int = 0, stream=None):
        """Submit + wait; returns (early results, final results) lists."""
        t = self.submit(reqs, exit_layer, stream)
        early = t.wait_early() if exit_layer else None
        final = t.wait_final()
        t.release()
        return early, final

    def debug_accept(self, logits, reqs):
        n = len(reqs)
        arr = (sv_verify_req * n)(*[r.to_c() for r in reqs])
        out = (sv_exit_result * n)()
        check(lib().sv_debug_accept(self.h, C.c_void_p(logits.data_ptr()), arr, n, out))
        return [out[i] for i in range(n)]

    def profile_step(self, reqs, exit_layer: int = 0, cap: int = 4096):
        """One step with per-launch CUDA-event timing; returns (final results, records)."""
        n = len(reqs)
        arr = (sv_verify_req * n)(*[r.to_c() for r in reqs])
        early = (sv_exit_result * n)()
        final = (sv_exit_result * n)()
        out = (sv_kernel_prof * cap)()
        k = C.c_int32()
        check(lib().sv_debug_profile_step(self.h, arr, n, exit_layer, early, final, out, cap, C.byref(k)))
        recs = [dict(kind=KERNEL_KINDS[out[i].kind], layer=out[i].layer, ms=out[i].ms, bytes=out[i].bytes,
                     flops=out[i].flops) for i in range(min(k.value, cap))]
        return [final[i] for i in range(n)], recs

    def trace_next(self):
        """Record a per-launch timeline of the next submit (graph replay, PDL on)."""
        check(lib().sv_debug_trace_next(self.h))

    def trace_read(self, cap: int = 2048):
        """Timeline of the last traced step: list of dict(kind, layer, stream, start_us, end_us)."""
        out = (sv_trace_rec * cap)()
        k = C.c_int32()
        check(lib().sv_debug_trace_read(self.h, out, cap, C.byref(k)))
        return [dict(kind=KERNEL_KINDS[out[i].kind], layer=out[i].layer, stream=out[i].stream,
                     start_us=out[i].start_ns / 1e3, end_us=out[i].end_ns / 1e3) for i in range(min(k.value, cap))]

    def set_adapters(self, adapters):
        """Exit adapters for every early exit (None: the plain shared head)."""
        self._adapters = adapters
        check(lib().sv_engine_set_adapters(self.h, C.byref(adapters.a) if adapters is not None else None))

    def debug_gemm(self, w, x):
        """out = x @ w.T (fp32) through the step's GEMM kernels; w [N, K], x [M, K] bf16
        CUDA tensors (sv_debug_gemm: marshalling only)."""
        import torch
        assert w.dtype == torch.bfloat16 and x.dtype == torch.bfloat16 and w.is_cuda and x.is_cuda
        w, x = w.contiguous(), x.contiguous()
        N, K = w.shape
        M = x.shape[0]
        out = torch.empty((M, N), dtype=torch.float32, device=w.device)
        check(lib().sv_debug_gemm(self.h, w.data_ptr(), x.data_ptr(), N, K, M, out.data_ptr()))
        return out

    def last_launches(self) -> int:
        n = C.c_int32()
        check(lib().sv_engine_last_launches(self.h, C.byref(n)))
        return n.value

    def close(self):
        if self.h:
            check(lib().sv_engine_destroy(self.h))
            self.h = None


def debug_philox(ctr, key):
    c = (C.c_uint32 * 4)(*ctr)
    k = (C.c_uint32 * 2)(*key)
    o = (C.c_uint32 * 4)()
    check(lib().sv_debug_philox(c, k, o))
    return [int(x) for x in o]
