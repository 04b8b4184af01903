#!/usr/bin/env python
"""bench.py — the verify-step benchmark of BASELINE.json.

metric : "verify-step latency p50 and verified tokens/s, Llama2-7B shape gamma=4"
value  : verified tokens/s of the whole job (sum over ranks of sum(delta+1) over
         the timed steps / max over ranks of the device-timed region), inputs
         resident in HBM.  `latency_p50_ms` is the device-timed p50 step latency.
e2e    : the same metric through the public API with the draft distributions
         copied from pinned host memory every step and results read back (host
         wall clock, synchronised at both ends).

A step = one pass of the whole hot path over one batch:
embed, 32 decoder layers, early exit at layer l_e (LM head + acceptance on the
exit stream), final LM head, acceptance and KV rollback.  The workload is kept
stationary: before each step every session is rewound to its prefix length, so
each timed step verifies the same (context, drafts) with fresh Philox counters
(new round id).  Drafts are "Vicuna-68M-style" calibrated distributions:
q_j = normalize(l*p_j + (1-l)*r_j), p_j the target row along the drafted path,
r_j a Zipf(1.5) row over a random permutation, l chosen by bisection so that
sum_v min(p_j, q_j) = alpha.

--impl reference runs the oracle (numpy fp64, tests-only infrastructure) on the
host cores on a bounded sample of the same workload.

The default run (C2, one GPU) also embeds `also_measured`: C5 and the per-GPU shard
of C4 on 8 GPUs, each measured by a child bench process on the same GPU after the
C2 timing (same timing rules; `--no-extra` skips them).

Launch: python bench.py [--gpus N --steps K --warmup W] (N>1 under torchrun;
each rank runs its own requests, no collective on the hot path; NCCL gathers
counters once at the end).
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

N_SETS = 64
METRIC = "verify-step latency p50 and verified tokens/s, Llama2-7B shape gamma=4"
UNIT = "tokens/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C2", choices=["C2", "C3", "C4", "C5"])
    ap.add_argument("--gamma", type=int, default=4)
    ap.add_argument("--exit-layer", type=int, default=16)
    ap.add_argument("--prefill", action="store_true",
                    help="NEXT-2: build each request's cached context with sv_prefill (timed, reported as "
                         "'prefill') instead of synthetic KV")
    ap.add_argument("--adapters", type=int, default=0, metavar="RANK",
                    help="NEXT-3: exit adapters of this rank (e.g. 384) on every early exit")
    ap.add_argument("--all-exits", action="store_true",
                    help="NEXT-1: an early exit after every layer 1..L-1, streamed (overrides --exit-layer)")
    ap.add_argument("--alpha", type=float, default=None,
                    help="per-position acceptance rate of the calibrated drafts (default: 0.73 for C5 — the "
                         "robot's tau = 2.92, PAPER.md:647 — else 0.825, tau = 3.53)")
    ap.add_argument("--batch", type=int, default=None, help="requests per GPU (default: per config)")
    ap.add_argument("--ctx", type=int, default=None)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extra", action="store_true",
                    help="default C2 run only: skip the C5 / C4-per-GPU-shard lines embedded as `also_measured`")
    ap.add_argument("--profile-json", default=None, help="write per-launch profile records here")
    ap.add_argument("--shard", default=None, metavar="R/N",
                    help="serve rank R's requests of an N-rank job in this single process (equality tests)")
    ap.add_argument("--dump-results", default=None, metavar="PATH",
                    help="write every timed step's final results per request id ({rank} is substituted)")
    args = ap.parse_args()
    if args.alpha is None:   # C5 takes alpha from the robot's tau = 2.92
        args.alpha = 0.73 if args.config == "C5" else 0.825
    return args


def workload(args, world):
    """(requests on this GPU, total requests, ctx, scaling) for the config."""
    if args.config in ("C2", "C3"):
        per, ctx, scaling = 1, 512, "weak"
    elif args.config == "C4":
        per, ctx, scaling = 256 // world, 1024, "strong"
    else:  # C5
        per, ctx, scaling = max(1, 16 // world), 2048, "strong" if world > 1 else "weak"
    if args.batch:
        per = args.batch
    if args.ctx:
        ctx = args.ctx
    return per, per * world, ctx, scaling


# ---------------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms while running."""
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits", "-i", str(self.gpu),
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            p = [x.strip() for x in ln.split(",")]
            if len(p) < 7:
                continue
            try:
                sm.append(float(p[0]))
                mx = float(p[1])
            except ValueError:
                continue
            for nm, v in zip(names, p[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------- helpers
def softmax64(z):
    z = np.asarray(z, dtype=np.float64)
    e = np.exp(z - z.max())
    return e / e.sum()


def calibrate_row(p, r, alpha):
    """lambda in [0,1] with sum_v min(p, l p + (1-l) r) = alpha (bisection)."""
    f = lambda lam: np.minimum(p, lam * p + (1 - lam) * r).sum()
    if f(0.0) >= alpha:
        return 0.0
    lo, hi = 0.0, 1.0
    for _ in range(50):
        mid = 0.5 * (lo + hi)
        if f(mid) < alpha:
            lo = mid
        else:
            hi = mid
    return hi


class Rounds:
    def __init__(self):
        self.r = {}

    def next(self, s):
        self.r[id(s)] = self.r.get(id(s), 0) + 1
        return self.r[id(s)]


def build_calibrated_drafts(sv, eng, sessions, pendings, ctx, gamma, alpha, V, seed, rounds):
    """gamma sequential probe steps (greedy, rewound) to read the target rows along
    the drafted path; returns (drafts int32 [B,gamma], q float32 [B,gamma,V], alpha_j)."""
    from workload.drafts import zipf_rows
    B = len(sessions)
    rng = np.random.default_rng([seed, 99, B, gamma])
    x = np.zeros((B, gamma), dtype=np.int32)
    q = np.zeros((B, gamma, V), dtype=np.float32)
    for j in range(gamma):
        reqs = [sv.Request(s, rounds.next(s), pendings[b], x[b]) for b, s in enumerate(sessions)]
        t = eng.submit(reqs, exit_layer=0)
        t.wait_final()
        z = t.logits(1, gamma)[:, j].double().cpu().numpy()
        t.release()
        for s in sessions:
            s.rewind(ctx)
        r = zipf_rows(rng, B, V, 1.5)
        for b in range(B):
            p = softmax64(z[b])
            lam = calibrate_row(p, r[b], alpha)
            qj = lam * p + (1 - lam) * r[b]
            qj /= qj.sum()
            cdf = np.cumsum(qj)
            x[b, j] = min(int(np.searchsorted(cdf, rng.random() * cdf[-1])), V - 1)
            q[b, j] = qj.astype(np.float32)
    return x, q


def measured_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        d = json.load(open(path))
        return d["hbm_gbs"], d.get("bf16_tflops_sustained"), "measured"
    except Exception:
        return 6650.0, 1400.0, "fallback (B200_PROFILING.md)"


def ncu_traffic(kind):
    """dram bytes per launch of the dominant kernel from the committed ncu summary."""
    path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        d = json.load(open(path))
        return d["dram_bytes_per_launch"].get(kind)
    except Exception:
        return None


# ---------------------------------------------------------------------------- CPU side
class OracleSample:
    """The oracle's verify step (oracle/verify.py, numpy fp64) on the host cores, at
    the workload's full shape: one request of the config (Llama2-7B shape, all 32
    decoder layers, V 32000, ctx, gamma, early exit), stochastic acceptance of
    timing-mode drafts.  Bounded sample: the 32 decoder layers cycle through
    N_GEN generated layers (weight generation is model state, not step work, and
    the per-layer arithmetic is the same), so a step needs 3.2 GB of fp64 layer
    weights instead of 54 GB; the embedding / LM head are the real ones.  The KV
    cache is copied before each timed call (outside the timed region).  Requests
    are processed one after another, so tokens/s = tau / (seconds per request)."""
    N_GEN = 2

    def __init__(self, args, ctx):
        from oracle import model as om
        from workload import llama2_7b
        from workload.drafts import timing_drafts
        self.args, self.ctx = args, ctx
        self.mc = llama2_7b()
        n_gen = self.N_GEN

        class CyclicModel(om.Model):
            def __init__(self, cfg, seed):
                super().__init__(cfg, seed, lazy=True)
                self.cyc = [super(CyclicModel, self).layer(i) for i in range(n_gen)]

            def layer(self, l):
                return self.cyc[l % n_gen]
        t0 = time.perf_counter()
        self.model = CyclicModel(self.mc, seed=1)
        self.cache = om.KVCache.synthetic(self.mc, 2, ctx)
        self.setup_s = time.perf_counter() - t0
        self.x, self.q = timing_drafts(3, 1, args.gamma, self.mc.vocab)
        self.exit_layer = 0 if args.all_exits else args.exit_layer
        self.round = 0
        self.t = []

    def step(self):
        """Seconds of one request's verify step (wall clock) and its tokens."""
        from oracle.verify import Session as OSession
        from oracle.verify import verify_step
        self.round += 1
        sess = OSession(1, 4, self.cache.copy())
        sess.last_round = self.round - 1
        t0 = time.perf_counter()
        out = verify_step(self.model, sess, self.round, 7, self.x[0], self.q[0].astype(np.float64),
                          exit_layer=self.exit_layer)
        dt = time.perf_counter() - t0
        self.t.append(dt)
        return dt, out.final.accepted + 1

    def describe(self):
        return (f"oracle verify_step (numpy fp64) of one request at the full Llama2-7B shape (32 decoder layers "
                f"cycling {self.N_GEN} generated layers' weights, real embedding and LM head), ctx {self.ctx}, "
                f"gamma {self.args.gamma}, exit at layer {self.exit_layer}, stochastic acceptance; "
                f"{len(self.t)} timed step(s), {np.mean(self.t):.2f} s per request; weight / KV generation "
                f"({self.setup_s:.1f} s) and the cache copy excluded; requests are processed sequentially")


def host_identity():
    """CPU model and BLAS library of the host the oracle ran on."""
    cpu = None
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                cpu = ln.split(":", 1)[1].strip()
                break
    except Exception:
        pass
    blas = None
    try:
        from threadpoolctl import threadpool_info
        blas = ", ".join(f"{i.get('internal_api')} {i.get('version')} ({i.get('num_threads')} threads)"
                         for i in threadpool_info())
    except Exception:
        pass
    return {"cpu_model": cpu, "blas": blas, "logical_cpus": os.cpu_count()}


def expected_tau(gamma, alpha):
    """Tokens per verify step of the calibrated workload: every drafted position is
    accepted with probability alpha (the drafts are calibrated to sum_v min(p, q) =
    alpha), so E[delta + 1] = sum_{k=0..gamma} alpha^k (alpha_j = alpha).
    A property of the workload definition, used for the CPU arms' tokens/s."""
    return float(sum(alpha ** k for k in range(gamma + 1)))


def host_cores():
    try:
        from threadpoolctl import threadpool_info
        return max([i.get("num_threads", 1) for i in threadpool_info()] + [1])
    except Exception:
        return os.cpu_count()


def _all_host_threads():
    """The oracle runs on all host cores even under torchrun (which sets
    OMP_NUM_THREADS=1 for every rank)."""
    try:
        from threadpoolctl import threadpool_limits
        return threadpool_limits(limits=os.cpu_count())
    except Exception:
        return None


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    _keep = _all_host_threads()
    per, total, ctx, scaling = workload(args, 1)
    sample = OracleSample(args, ctx)
    # bounded: at most 30 timed oracle request-steps (~1.2 s each on 16 host threads) and
    # one warm-up, so the arm ends within a minute or two whatever --steps / --warmup are
    n_warm, n_timed = min(args.warmup, 1), max(1, min(args.steps, 30))
    times = []
    for i in range(n_warm + n_timed):
        dt, _ = sample.step()
        if i >= n_warm:
            times.append(dt)
    sec = float(np.mean(times))
    tok = expected_tau(args.gamma, args.alpha)
    value = tok / sec
    cores, desc = host_cores(), sample.describe()
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": sec * 1e3 * per, "higher_is_better": True,
            "scaling": scaling, "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"{args.config} Llama2-7B shape, B={per}, ctx {ctx}, gamma {args.gamma}",
                       "global_batch": per, "seq_len": ctx, "parallelism": "host cores"},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle",
                             "sample": desc + f" (a bounded sample of the --steps {args.steps} run: "
                                       f"{n_warm} warm-up + {n_timed} timed)"
                                       f"; ms_per_step = {per} request(s) x {sec * 1e3:.0f} ms; tokens/step "
                                       f"{tok:.3f} = expected tau of the calibrated workload (alpha {args.alpha}, "
                                       f"gamma {args.gamma})", "host": host_identity()},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------- GPU side
def trace_roofline(trace, prof, hbm, tc, peak_src):
    """Roofline of the dominant kernel family (the main-stream weight GEMMs) in a
    step as it runs in production (graph replay with PDL; sv_debug_trace_*).

    Launches on the main stream form one dependent chain; launch i is charged the
    time from the end of the chain before it to its own end (its CTAs may start
    earlier under PDL, but only this part is on the step's critical path), so the
    charged times of the chain add up to the traced step.  achieved = algorithmic
    bytes (or flops) of the family / its charged time.  Bytes and flops per launch
    come from sv_debug_profile_step records, which list the same launches in the
    same order.  The exit stream runs beside the chain and is reported apart."""
    if len(trace) != len(prof) or any(t["kind"] != p["kind"] for t, p in zip(trace, prof)):
        return None
    step_us = max(t["end_us"] for t in trace) - min(t["start_us"] for t in trace)
    prev = None
    fam = {}
    for t, p in zip(trace, prof):
        if t["stream"] != 0:
            key = t["kind"] + " (exit stream)"
            charged = t["end_us"] - t["start_us"]
        else:
            key = t["kind"]
            charged = t["end_us"] - (t["start_us"] if prev is None else prev)
            prev = t["end_us"] if prev is None else max(prev, t["end_us"])
        f = fam.setdefault(key, {"launches": 0, "us": 0.0, "bytes": 0.0, "flops": 0.0})
        f["launches"] += 1
        f["us"] += charged
        f["bytes"] += p["bytes"]
        f["flops"] += p["flops"]
    g = [f for k, f in fam.items() if k.startswith("gemm") and "exit" not in k]
    g_us = sum(f["us"] for f in g)
    g_bytes = sum(f["bytes"] for f in g)
    g_flops = sum(f["flops"] for f in g)
    g_n = sum(f["launches"] for f in g)
    ridge = tc * 1e12 / (hbm * 1e9)            # flops per byte where the two roofs meet
    tensor = g_flops / g_bytes > ridge
    if tensor:
        achieved, peak, unit = g_flops / (g_us * 1e-6) / 1e12, tc, "TFLOP/s"
        src = peak_src + " (bf16_tflops_sustained: the GEMMs run inside a long step)"
    else:
        achieved, peak, unit = g_bytes / (g_us * 1e-6) / 1e9, hbm, "GB/s"
        src = peak_src + " (hbm_gbs)"
    return {"bound": "tensor" if tensor else "hbm",
            "kernel": "gemm_kernel / gemm_big_kernel (QKV, O, gate-up, down, final LM head; tcgen05 + TMA)",
            "achieved": round(achieved, 1), "peak": peak, "unit": unit, "frac": round(achieved / peak, 4),
            "peak_source": src, "measured_in": "one graph-replayed step with PDL (sv_debug_trace_next), "
                                                "critical-path charge per launch",
            "launches": g_n, "avg_launch_ms": round(g_us / g_n / 1e3, 5),
            "algorithmic_bytes_per_launch": g_bytes / g_n, "algorithmic_flops_per_launch": g_flops / g_n,
            "arithmetic_intensity": round(g_flops / g_bytes, 2), "ridge_flops_per_byte": round(ridge, 1),
            "share_of_step": round(g_us / step_us, 4), "traced_step_ms": round(step_us / 1e3, 4),
            "kernels": {k: {"launches": f["launches"], "ms": round(f["us"] / 1e3, 4),
                            "GB/s": round(f["bytes"] / (f["us"] * 1e-6) / 1e9, 1) if f["us"] > 0 else None,
                            "TFLOP/s": round(f["flops"] / (f["us"] * 1e-6) / 1e12, 1) if f["us"] > 0 else None}
                        for k, f in fam.items()}}


def run_ours(args):
    import torch
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # SV_BENCH_DEVICE / SV_DIST_BACKEND: test hooks to run the multi-rank path with
    # several ranks on one GPU (gloo for the counter gather; NCCL needs distinct GPUs)
    if os.environ.get("SV_BENCH_DEVICE") is not None:
        local = int(os.environ["SV_BENCH_DEVICE"])
    torch.cuda.set_device(local)
    dist = None
    backend = None
    if world > 1:
        import torch.distributed as dist
        backend = os.environ.get("SV_DIST_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
        else:
            dist.init_process_group(backend)
    # --shard R/N: this process serves rank R's requests of an N-rank job on its own
    # (the single-rank reference run of the multi-rank equality test)
    as_rank, as_world = rank, world
    if args.shard:
        as_rank, as_world = (int(v) for v in args.shard.split("/"))
    from paper_2505_21594_b200 import sv
    from paper_2505_21594_b200.dist import gather_counters, shard
    from workload import llama2_7b
    from workload.drafts import prefix_tokens

    per, total, ctx, scaling = workload(args, as_world)
    gamma, exit_layer = args.gamma, args.exit_layer
    mc = llama2_7b()
    exit_layers = list(range(1, mc.n_layers)) if args.all_exits else []
    if exit_layers:
        exit_layer = 0
    W = sv.Weights(mc, seed=1, device=local)
    blocks_per = (ctx + gamma + 1 + 63) // 64
    eng = sv.Engine(mc, W, max_batch=per, max_gamma=max(1, gamma), kv_blocks=per * blocks_per, device=local,
                    max_prefill=ctx if args.prefill else 0)
    if args.adapters:
        eng.set_adapters(sv.Adapters(mc, args.adapters, seed=9, device=local))
    sessions = []
    rids = list(shard(total, as_world, as_rank))   # contiguous shard of the request ids
    rounds = Rounds()
    pend = prefix_tokens(3 + as_rank, per, mc.vocab)
    prefill_s = []
    for i, rid in enumerate(rids):
        s = eng.open_session(rid + 1, 0x5EED0000 + rid)
        if args.prefill:   # synthetic prompt of ctx uniform token ids through the model
            prompt = np.random.default_rng([5, rid]).integers(0, mc.vocab, size=ctx)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            res = s.prefill(prompt, sample=True)
            prefill_s.append(time.perf_counter() - t0)
            pend[i] = res.emitted()[-1]
            rounds.r[id(s)] = res.round_id
        else:
            s.fill_kv(ctx, kv_seed=1000 + rid)
        sessions.append(s)
    # independent calibrated draft sets per request, one per step until they cycle
    # (256 for one request, 64 at <= 16 requests per GPU, so the accepted lengths
    # follow the workload's law rather than a few fixed draws; 8 for the larger pools)
    n_sets = 4 * N_SETS if per == 1 else (N_SETS if per <= 16 else 8)
    sets = [build_calibrated_drafts(sv, eng, sessions, pend, ctx, gamma, args.alpha, mc.vocab,
                                    7 + 1000 * as_rank + k, rounds) for k in range(n_sets)]
    xs = [x for x, _ in sets]
    if gamma == 0:   # plain AR step ("Cloud AR"): sample p_0, probs pointer never read
        dummy = torch.empty(per, 1, device="cuda")
        q_dev = [dummy for _ in sets]
        q_host = [np.zeros((per, 1), dtype=np.float32) for _ in sets]
    else:
        q_dev = [torch.from_numpy(q).cuda() for _, q in sets]
        q_host = [torch.from_numpy(q).pin_memory().numpy() for _, q in sets]
    stream = torch.cuda.current_stream()
    counter = [0]

    def step(host_probs=False, ev0=None, timing=False):
        k = counter[0] % n_sets
        counter[0] += 1
        x = xs[k]
        for s in sessions:          # stationary workload: back to the same cached context
            s.rewind(ctx)
        reqs = [sv.Request(s, rounds.next(s), pend[b], x[b], q_host[k][b] if host_probs else q_dev[k][b])
                for b, s in enumerate(sessions)]
        if ev0 is not None:         # the step's latency starts at the verify call (the rewind
            ev0.record(stream)      # and the request objects are the caller's, not the step's)
        if exit_layers:
            t = eng.submit_exits(reqs, exit_layers, stream=stream)
            for j in range(len(exit_layers)):       # streamed: each exit as soon as it lands
                t.wait_exit(j)
        else:
            t = eng.submit(reqs, exit_layer=exit_layer, stream=stream)
            if exit_layer:
                t.wait_early()
        f = t.wait_final()
        tm = t.timing() if timing else None
        t.release()
        bad = [r.status for r in f if r.status != sv.SV_OK]
        if bad:
            raise RuntimeError(f"verify step returned per-request errors {bad}")
        return sum(r.accepted + 1 for r in f), f, tm

    # warm-up (also captures the CUDA graph)
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    tokens = 0
    per_step_tok = []
    accepted_hist = np.zeros(gamma + 2, dtype=np.int64)
    dump = {}
    with ClockSampler(local) as clk:
        t_all0 = torch.cuda.Event(enable_timing=True)
        t_all1 = torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        t_all0.record(stream)
        for i in range(args.steps):
            n_tok, f, _ = step(ev0=ev[i][0])
            ev[i][1].record(stream)
            tokens += n_tok
            per_step_tok.append(n_tok / per)
            for b, r in enumerate(f):
                accepted_hist[r.accepted] += 1
                if args.dump_results:
                    dump.setdefault(rids[b], []).append(r.asdict())
        t_all1.record(stream)
        torch.cuda.synchronize()
    if dist:
        dist.barrier()
    elapsed = t_all0.elapsed_time(t_all1) / 1e3
    step_ms = [a.elapsed_time(b) for a, b in ev]
    launches = eng.last_launches()

    # end to end: host probs (pinned) -> H2D inside each step, results D2H
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    e2e_tok = 0
    t0 = time.perf_counter()
    for i in range(args.steps):
        n_tok, _, _ = step(host_probs=True)
        e2e_tok += n_tok
    torch.cuda.synchronize()
    e2e_el = time.perf_counter() - t0

    # exit-ready latency (Eq. 5; Alg-S :1103-1106): device stamps
    # and host observation times of every exit, on separate untimed steps
    exit_ready = None
    if exit_layer or exit_layers:
        tms = [step(timing=True)[2] for _ in range(min(args.steps, 30))]
        layers = exit_layers if exit_layers else [exit_layer]
        fin_dev = statistics.median(t["final_dev_ms"] for t in tms)
        fin_host = statistics.median(t["final_host_ms"] for t in tms)
        pick = range(len(layers)) if len(layers) <= 4 else [0, 7, 15, 23, len(layers) - 1]
        exit_ready = {
            "exit_layers": [layers[k] for k in pick],
            "dev_ms_p50": [round(statistics.median(t["exit_dev_ms"][k] for t in tms), 4) for k in pick],
            "host_ms_p50": [round(statistics.median(t["exit_host_ms"][k] for t in tms), 4) for k in pick],
            "final_dev_ms_p50": round(fin_dev, 4), "final_host_ms_p50": round(fin_host, 4),
            "model_ms": [round(layers[k] / mc.n_layers * fin_dev + 0.04, 4) for k in pick],
            "steps": len(tms),
            "note": "dev = first kernel start -> last request's result written (globaltimer); host = submit call "
                    "-> mailbox flag observed by sv_wait_exit; model = (l_e / L) * final_dev + 0.04 ms "
                    "(SURVEY.md §8(d))"}

    # roofline of the timed configuration: one traced graph-replayed step (PDL on)
    # plus the per-launch algorithmic work from a serialised profile step
    hbm, tc, peak_src = measured_peaks()
    eng.trace_next()
    step()
    trace = eng.trace_read()
    for s in sessions:
        s.rewind(ctx)
    preqs = [sv.Request(s, rounds.next(s), pend[b], xs[0][b], q_dev[0][b]) for b, s in enumerate(sessions)]
    _, recs = eng.profile_step(preqs, exit_layer=exit_layer if not exit_layers else exit_layers[len(exit_layers) // 2])
    # per-launch algorithmic work in the traced step's launch order: main-stream
    # launches in order; every exit's launches have the profiled exit's work
    main_recs = [r for r in recs if r["kind"] not in ("gemm_lm_exit", "accept_exit")]
    exit_recs = {r["kind"]: r for r in recs if r["kind"] in ("gemm_lm_exit", "accept_exit")}
    aligned, it = [], iter(main_recs)
    for t in trace:
        aligned.append(next(it, None) if t["stream"] == 0 else exit_recs.get(t["kind"]))
    roofline = None
    step_bytes = None
    if all(a is not None and a["kind"] == t["kind"] for a, t in zip(aligned, trace)):
        roofline = trace_roofline(trace, aligned, hbm, tc, peak_src)
        step_bytes = sum(a["bytes"] for a in aligned)
    if roofline is not None:
        roofline["traffic"] = ncu_traffic("gemm")
        roofline["serialised_profile"] = {   # the same launches one at a time (PDL off, no graph)
            "gemm_GB/s": round(sum(r["bytes"] for r in recs if r["kind"].startswith("gemm"))
                               / (sum(r["ms"] for r in recs if r["kind"].startswith("gemm")) / 1e3) / 1e9, 1),
            "step_ms": round(sum(r["ms"] for r in recs), 4)}
        roofline["step_algorithmic_bytes"] = step_bytes
        roofline["step_frac_of_peak"] = round(step_bytes / (statistics.median(step_ms) / 1e3) / 1e9 / hbm, 4)
    if args.profile_json:
        json.dump({"trace": trace, "records": recs, "step_ms": step_ms}, open(args.profile_json, "w"))
    if args.dump_results:
        json.dump({str(k): v for k, v in dump.items()}, open(args.dump_results.replace("{rank}", str(as_rank)), "w"))

    # gather counters over ranks (the only collective)
    allv = gather_counters([tokens, elapsed, e2e_tok, e2e_el],
                           device="cpu" if backend not in (None, "nccl") else "cuda")
    if rank != 0:
        if dist:
            dist.destroy_process_group()
        return
    tot_tokens = allv[:, 0].sum()
    t_max = allv[:, 1].max()
    value = tot_tokens / t_max
    e2e_value = allv[:, 2].sum() / allv[:, 3].max()

    cpu = None
    if world == 1 and not args.no_cpu_baseline and not args.shard:
        _keep = _all_host_threads()
        sample = OracleSample(args, ctx)
        dt, _ = sample.step()
        tps = expected_tau(gamma, args.alpha)
        cpu = {"value": tps / dt, "unit": UNIT, "cores": host_cores(), "kind": "oracle",
               "sample": sample.describe() + f"; tokens/step {tps:.3f} = expected tau of the calibrated workload "
                                             f"(alpha {args.alpha}, gamma {gamma})",
               "host": host_identity()}

    also = None
    if (world == 1 and not args.shard and not args.no_extra and args.config == "C2" and gamma == 4
            and exit_layer == 16 and not exit_layers and not args.prefill and not args.adapters
            and args.batch is None and args.ctx is None):
        also = also_measured()

    h2d = per * gamma * mc.vocab * 4 + per * (gamma + 1) * 12   # gamma 0: no draft probabilities
    d2h = 2 * per * 64
    tau_exp = expected_tau(gamma, args.alpha)
    line = {"metric": METRIC, "value": round(value, 2), "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(t_max * 1e3 / args.steps, 4),
            "latency_p50_ms": round(statistics.median(step_ms), 4),
            "latency_p90_ms": round(float(np.percentile(step_ms, 90)), 4),
            "higher_is_better": True, "scaling": scaling, "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic (random-init Llama2-7B-shape weights, synthetic KV, calibrated draft distributions)",
            "config": {"workload": f"{args.config}: Llama2-7B shape (32 layers, d 4096, V 32000), "
                                   f"{per} request(s)/GPU, ctx {ctx}, gamma {gamma}, "
                                   + (f"early exits after layers 1..{mc.n_layers - 1} (streamed)" if exit_layers
                                      else f"early exit at layer {exit_layer}")
                                   + (f", exit adapters rank {args.adapters}" if args.adapters else "")
                                   + f", stochastic acceptance, alpha {args.alpha}",
                       "global_batch": total, "seq_len": ctx, "gamma": gamma,
                       "exit_layer": exit_layers if exit_layers else exit_layer,
                       "engine": "per-op kernels + CUDA graph + PDL",
                       "parallelism": f"requests sharded over {world} GPU(s), weights replicated",
                       "world_size": world, "dist_backend": backend,
                       "draft_sets_per_request": n_sets,
                       "l2": "inputs larger than L2 (13.5 GB of weights streamed per step)"},
            "tokens_per_step": round(tot_tokens / (args.steps * total), 4),
            "expected_tokens_per_step": round(tau_exp, 4),
            "tokens_per_step_stderr": round(float(np.std(per_step_tok) / np.sqrt(len(per_step_tok) * per)), 4),
            "accepted_hist": accepted_hist.tolist(),
            "e2e": {"value": round(e2e_value, 2), "unit": UNIT, "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h, "ms_per_step": round(allv[:, 3].max() * 1e3 / args.steps, 4),
                    "tokens_per_step": round(allv[:, 2].sum() / (args.steps * total), 4)},
            "gpu_launches": launches * args.steps, "kernels_per_step": launches,
            "exit_ready": exit_ready,
            "prefill": ({"prompt_tokens": ctx, "ms_per_prompt_p50": round(1e3 * statistics.median(prefill_s), 3),
                         "tokens_per_s": round(ctx / statistics.median(prefill_s), 1),
                         "note": "sv_prefill, one synchronous call per request, host wall clock"}
                        if prefill_s else None),
            "roofline": roofline, "cpu_baseline": cpu, "clocks": clk.summary()}
    if also is not None:
        line["also_measured"] = also
    print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


def also_measured():
    """The default run (C2) also measures, each in a child process of this bench on the
    same GPU after the C2 timing: C5 (SURVEY.md configs[4]) and the per-GPU shard of C4
    on 8 GPUs (32 requests, the strong-scaling case).  A summary of each child's own
    line (same timing rules: device events, warm-up, clocks) is embedded, so these
    numbers carry the driver's clock too."""
    out = {}
    for name, argv in (("C5", ["--config", "C5", "--steps", "20", "--warmup", "3"]),
                       ("C4_per_gpu_shard_of_8", ["--config", "C4", "--batch", "32", "--steps", "10", "--warmup", "3"])):
        try:
            r = subprocess.run([sys.executable, os.path.abspath(__file__), *argv, "--no-cpu-baseline", "--no-extra"],
                               capture_output=True, text=True, timeout=420)
            d = json.loads(r.stdout.strip().splitlines()[-1])
            rf = d.get("roofline") or {}
            out[name] = {"workload": d["config"]["workload"], "value": d["value"], "unit": d["unit"],
                         "latency_p50_ms": d["latency_p50_ms"], "ms_per_step": d["ms_per_step"],
                         "steps": d["steps"], "warmup": d["warmup"],
                         "tokens_per_step": d["tokens_per_step"], "e2e": d["e2e"],
                         "step_frac_of_peak": rf.get("step_frac_of_peak"),
                         "roofline": {k: rf.get(k) for k in ("bound", "achieved", "peak", "unit", "frac")},
                         "exit_ready": d.get("exit_ready"), "clocks": d.get("clocks")}
        except Exception as ex:   # recorded, never fatal for the C2 line
            out[name] = {"error": f"{type(ex).__name__}: {ex}"[:300]}
    return out


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
