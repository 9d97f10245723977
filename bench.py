#!/usr/bin/env python
"""Quartet II linear fwd+bwd benchmark (BASELINE.json metric) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--mode posthoc|exact] [--no-extra] [--no-cpu-baseline]

One step = forward + backward of the four Llama-1.9B-class projections of
BASELINE config c3 (QKV 2048->6144, O 2048->2048, UpGate 2048->11264,
Down 5632->2048) over 16,384 tokens per GPU, through the public API
(paper_2601_22813_b200.forward / backward): 4/6 quantization of X and W, fprop
GEMM, MS-EDEN of E, E^T (one read of E), W^T and X^T (from the NVFP4 tape),
dgrad and wgrad GEMMs.  Under torchrun each rank processes its own 16,384-token
shard (weak scaling, config c4 at N=4) and dW is all-reduced over NCCL.

value = 6 * tokens * in * out summed over projections and ranks / max-rank time.
Inputs are larger than L2 (each step streams >1 GB through HBM), so no flush.
The headline runs the post-hoc MS-EDEN schedule (posthoc.py, the paper's kernel
schedule); ``modes`` reports both it and the exact ms_eden_quantize mode of
baseline_config("quartet2").  ``extra`` holds the other BASELINE configs: c1
(with the oracle timed on the full c1 layer), the c2 quantizer sweep and the c5
GEMM stress, each against BF16 cuBLAS (and cuBLASLt NVFP4 through
torch._scaled_mm where torch exposes it).
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PROJECTIONS = (("qkv", 2048, 6144), ("o", 2048, 2048), ("upgate", 2048, 11264), ("down", 5632, 2048))
TOKENS = 16384
REF_TOKENS = 128          # oracle sample: this many tokens of each of the four projections
METRIC = "Quartet II linear fwd+bwd TFLOP/s"


def flops(tokens: int, projections=PROJECTIONS) -> float:
    return sum(6.0 * tokens * i * o for _, i, o in projections)


# --------------------------------------------------------------- clocks -----
class ClockSampler:
    """nvidia-smi clocks/throttle sampling during the timed region (B200_PROFILING.md)."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index, self.rows, self.proc = index, [], None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "20"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([s.strip() for s in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            self.proc.wait()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({n for r in self.rows for n, v in zip(names, r[2:]) if v.strip().lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": float(self.rows[0][1]),
                "reasons": reasons, "samples": len(self.rows)}


# ------------------------------------------------------------ reference -----
def _bf16_round(a: np.ndarray) -> np.ndarray:
    """Round float32 to the nearest bf16 (ties to even), as the GPU inputs are."""
    u = a.astype(np.float32).view(np.uint32)
    u = ((u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000).astype(np.uint32)
    return u.view(np.float32)


def _oracle_sample(tokens: int = REF_TOKENS):
    """The c3 workload's inputs, `tokens` tokens of each projection (same distributions)."""
    rng = np.random.default_rng(0)
    data = []
    for _, din, dout in PROJECTIONS:
        X = _bf16_round(rng.standard_normal((tokens, din)).astype(np.float32))
        W = _bf16_round((rng.standard_normal((dout, din)) / np.sqrt(din)).astype(np.float32))
        E = _bf16_round((1e-3 * rng.standard_normal((tokens, dout))).astype(np.float32))
        data.append((X, W, E))
    return data


def _oracle_step(O, data, i, mode):
    for X, W, E in data:
        _, tape = O.forward(X, W)
        O.backward(tape, E, O.SeedPair(1, i), posthoc=mode == "posthoc")


def _threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


SAMPLE_TEXT = (f"numpy oracle (the reference's algorithm restated, oracle/nvfp4_oracle.py) fwd+bwd of all four "
               f"c3 projections on a {REF_TOKENS}-token slice each, per step; quantizers single-threaded numpy, "
               "GEMMs multi-threaded BLAS")


def run_reference(args, world: int) -> None:
    """The reference's CPU path on the box's host cores: the oracle port (the pure-Python
    reference cannot travel to the GPU box), on a bounded sample of the c3 workload."""
    from oracle import nvfp4_oracle as O
    data = _oracle_sample()
    for i in range(args.warmup):
        _oracle_step(O, data, i, args.mode)
    t0 = time.perf_counter()
    for i in range(args.steps):
        _oracle_step(O, data, i, args.mode)
    dt = (time.perf_counter() - t0) / args.steps
    v = flops(REF_TOKENS) / dt / 1e12
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": v, "unit": "TFLOP/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"c3 Llama-1.9B projections qkv/o/upgate/down, {REF_TOKENS}-token sample of each "
                               "(the GPU arm runs 16384 tokens)", "msed_mode": args.mode},
        "cpu_baseline": {"value": v, "unit": "TFLOP/s", "cores": _threads(), "kind": "port", "sample": SAMPLE_TEXT},
        "e2e": {"value": v, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }))


def cpu_baseline_sample(mode: str, budget_s: float = 12.0) -> dict:
    from oracle import nvfp4_oracle as O
    data = _oracle_sample()
    _oracle_step(O, data, 0, mode)
    t0 = time.perf_counter()
    n = 0
    while n < 2 or time.perf_counter() - t0 < budget_s:
        _oracle_step(O, data, n + 1, mode)
        n += 1
    dt = (time.perf_counter() - t0) / n
    return {"value": flops(REF_TOKENS) / dt / 1e12, "unit": "TFLOP/s", "cores": _threads(), "kind": "port",
            "sample": SAMPLE_TEXT + f"; {n} steps"}


# ----------------------------------------------------------------- timing ---
def _events():
    import torch
    return torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)


def _time_ms(fn, iters=5, warmup=2):
    """Mean device time of fn() on the current stream (CUDA events, synchronized)."""
    import torch
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    s, e = _events()
    s.record()
    for _ in range(iters):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / iters


def _graph_ms(fn, iters=10):
    """Mean device time of fn() with the calls captured in one CUDA graph (no host launch
    overhead: the small c2 sizes were host-bound when timed eagerly); eager on failure."""
    import torch
    try:
        fn()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for _ in range(iters):
                fn()
        g.replay()
        torch.cuda.synchronize()
        s, e = _events()
        s.record()
        g.replay()
        e.record()
        torch.cuda.synchronize()
        ms = s.elapsed_time(e) / iters
        del g
        return ms, "cuda_graph"
    except Exception as exc:  # noqa: BLE001 - report and fall back
        torch.cuda.synchronize()
        return _time_ms(fn, iters=3, warmup=1), f"eager ({type(exc).__name__})"


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return p["hbm_gbs"], p["bf16_tflops"], "MEASURED_PEAKS.json"
    except (OSError, KeyError, ValueError):
        return 6650.0, 1590.0, "fallback (B200_PROFILING.md)"


NOMINAL_NVFP4_TFLOPS = 148 * 32768 * 1.965e9 / 1e12          # dense tcgen05 kind::mxf4nvf4 at 1965 MHz


def _traffic_table():
    """DRAM bytes per launch per kernel class, from the committed ncu capture of the same
    workload (profiles/r2_traffic.json, tools/traffic.py)."""
    try:
        with open(os.path.join(ROOT, "profiles", "r2_traffic.json")) as f:
            return json.load(f)
    except (OSError, ValueError):
        return {}


# ----------------------------------------------------------------- ours -----
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--mode", default="posthoc", choices=["posthoc", "exact"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extra", action="store_true", help="skip the c1 / c2 / c5 configs")
    ap.add_argument("--dw-reduce", default="nccl", choices=["auto", "nccl", "multimem"],
                    help="N > 1: dW sum by NCCL all-reduce or inside the wgrad GEMM over NVLS multicast "
                         "(auto: multimem when the group has a multicast object).  Default nccl: the "
                         "multicast path has not run on a multi-GPU box yet (every box this round had one GPU)")
    ap.add_argument("--eager", action="store_true", help="time eager launches instead of the captured CUDA graph")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        if rank == 0:
            run_reference(args, world)
        return

    import torch
    import torch.distributed as dist
    import paper_2601_22813_b200 as q2
    from paper_2601_22813_b200 import _lib
    from paper_2601_22813_b200.parallel import ShardedLinearStep

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    q2.set_error_mode("deferred")

    from paper_2601_22813_b200.parallel import MulticastReducer
    dw_reduce = args.dw_reduce
    if world == 1:
        dw_reduce = "none"
    elif dw_reduce == "auto":
        dw_reduce = "multimem" if MulticastReducer.available() else "nccl"

    g = torch.Generator(device=dev)
    data = []
    for pi, (name, din, dout) in enumerate(PROJECTIONS):
        g.manual_seed(1000 * pi + 1)                       # W identical on all ranks
        W = (torch.randn(dout, din, device=dev, generator=g) / din ** 0.5).to(torch.bfloat16)
        g.manual_seed(1000 * pi + 2 + 17 * rank)
        X = torch.randn(TOKENS, din, device=dev, generator=g).to(torch.bfloat16)
        E = (1e-3 * torch.randn(TOKENS, dout, device=dev, generator=g)).to(torch.bfloat16)
        data.append((X, W, E))

    def measure(mode):
        """Captured-graph (N=1) or eager (N>1) step time of one MS-EDEN mode, max over ranks."""
        runner = ShardedLinearStep(q2.LayerConfig(posthoc=mode == "posthoc"), rank=rank, world=world,
                                   reduce="multimem" if dw_reduce == "multimem" else "nccl")
        for i in range(args.warmup):
            runner.step(data, i)
        torch.cuda.synchronize()
        graph, launch = None, "eager"
        if not args.eager and world == 1:      # N > 1: eager launches (NCCL stays outside a captured graph)
            try:
                graph = torch.cuda.CUDAGraph()
                with torch.cuda.graph(graph):
                    runner.step(data, args.warmup)
                graph.replay()
                torch.cuda.synchronize()
                launch = "cuda_graph"
            except Exception as exc:  # noqa: BLE001 - report and fall back to eager launches
                graph, launch = None, f"eager (graph capture failed: {type(exc).__name__})"
                torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        s, e = _events()
        with ClockSampler(local) as clk:
            s.record()
            for i in range(args.steps):
                if graph is not None:
                    graph.replay()
                else:
                    runner.step(data, args.warmup + 1 + i)
            e.record()
            torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        ms = s.elapsed_time(e) / args.steps
        t = torch.tensor([ms], device=dev)
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        q2.check_errors()
        del graph
        return float(t.item()), launch, clk.summary(), runner

    ms, launch, clocks, runner = measure(args.mode)
    # our kernels per step: count one eager step's launches (library counter)
    torch.cuda.synchronize()
    _lib.lib().q2_launch_count(1)
    runner.step(data, 0)
    torch.cuda.synchronize()
    launches_per_step = int(_lib.lib().q2_launch_count(1))
    total_flops = flops(TOKENS) * world
    modes = {args.mode: {"ms_per_step": ms, "value": total_flops / (ms / 1e3) / 1e12}}
    other = "exact" if args.mode == "posthoc" else "posthoc"
    ms_o, _, _, _ = measure(other)
    modes[other] = {"ms_per_step": ms_o, "value": total_flops / (ms_o / 1e3) / 1e12}

    detail = kernel_breakdown(q2, data, args.mode)
    bf16_ms = bf16_baseline(data, args)
    e2e = e2e_measure(q2, data, args, world, dev, rank)
    for m in modes.values():
        m["speedup_vs_bf16"] = bf16_ms / m["ms_per_step"]

    value = total_flops / (ms / 1e3) / 1e12
    out = {
        "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "nvfp4 (e2m1 x ue4m3, fp32 accumulate; bf16 in/out)", "data": "synthetic",
        "config": {"workload": "c3: Llama-1.9B-class projections qkv/o/upgate/down (d=2048, ffn=5632), "
                               f"{TOKENS} tokens per GPU, fwd+bwd", "tokens_per_gpu": TOKENS,
                   "msed_mode": args.mode, "parallelism": f"token-sharded dp{world}" if world > 1 else "single",
                   "dw_reduce": dw_reduce,
                   "l2": "inputs larger than L2 (>1 GB streamed per step), no flush", "launch": launch},
        "speedup_vs_bf16": bf16_ms / ms, "bf16_cublas_ms_per_step": bf16_ms, "modes": modes,
        "kernels": detail["kernels"], "roofline": detail["roofline"], "rooflines": detail["rooflines"],
        "e2e": e2e, "gpu_launches": launches_per_step * args.steps, "gpu_launches_per_step": launches_per_step,
        "clocks": clocks,
    }
    if rank == 0 and world == 1 and not args.no_extra:
        out["extra"] = extra_configs(q2, args, dev)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        out["cpu_baseline"] = cpu_baseline_sample(args.mode)
    if rank == 0:
        print(json.dumps(out))
    if world > 1:
        dist.destroy_process_group()


def kernel_breakdown(q2, data, mode):
    """Each kernel class timed with CUDA events on the launching stream over the four
    projections (algorithmic work per SURVEY §8(d)), and its roofline."""
    import torch
    hbm, bf16, src = _peaks()
    acc = {}

    def timed(tag, fn, work, unit):
        s, e = _events()
        s.record()
        r = fn()
        e.record()
        acc.setdefault(tag, []).append((s, e, work, unit))
        return r

    from paper_2601_22813_b200.linear_graph import PAIR_DW, PAIR_DX
    seeds = q2.SeedPair(11, 12)
    ds = q2.derive_stream
    for _ in range(2):
        acc.clear()
        for X, W, E in data:
            T, din = X.shape
            dout = W.shape[0]
            qx = timed("quant_fwd46", lambda: q2.quantize_rtn_46(X), T * din * 2.5625, "B")
            qw = timed("quant_fwd46", lambda: q2.quantize_rtn_46(W), dout * din * 2.5625, "B")
            timed("gemm_fprop", lambda: q2.gemm(qx, qw, torch.bfloat16), 2.0 * T * din * dout, "F")
            qe, qet = timed("msed_dual_E", lambda: q2.msed_dual(E, seeds, ds(PAIR_DX, 0), PAIR_DX, ds(PAIR_DW, 0),
                                                                 PAIR_DW, 6.0, mode), T * dout * 3.125, "B")
            qwt = timed("msed_tape", lambda: q2.msed(qw, seeds, 6.0, ds(PAIR_DX, 1), PAIR_DX, mode, "tape"),
                        dout * din * 1.125, "B")
            timed("gemm_dgrad", lambda: q2.gemm(qe, qwt, torch.bfloat16), 2.0 * T * din * dout, "F")
            qxt = timed("msed_tape", lambda: q2.msed(qx, seeds, 6.0, ds(PAIR_DW, 1), PAIR_DW, mode, "tape"),
                        T * din * 1.125, "B")
            timed("gemm_wgrad", lambda: q2.gemm(qet, qxt, torch.float32), 2.0 * T * din * dout, "F")
        torch.cuda.synchronize()
    traffic = _traffic_table()
    kernels, rooflines = {}, {}
    for tag, lst in acc.items():
        t = sum(s.elapsed_time(e) for s, e, _, _ in lst)
        w = sum(x[2] for x in lst)
        unit = lst[0][3]
        n = len(lst)
        tr = traffic.get(tag, {}).get(mode if tag.startswith("msed") else "any")
        if unit == "F":
            rate = w / (t / 1e3) / 1e12
            kernels[tag] = {"ms": t, "launches": n, "TFLOP/s": rate}
            rooflines[tag] = {"bound": "tensor", "achieved": rate, "peak": 4.0 * bf16, "unit": "TFLOP/s",
                              "frac": rate / (4.0 * bf16), "frac_of_nominal_nvfp4": rate / NOMINAL_NVFP4_TFLOPS,
                              "flops_per_launch": w / n, "ms_per_launch": t / n,
                              "traffic": tr["bytes_per_launch"] if tr else None}
        else:
            rate = w / (t / 1e3) / 1e9
            kernels[tag] = {"ms": t, "launches": n, "GB/s": rate}
            rooflines[tag] = {"bound": "hbm", "achieved": rate, "peak": hbm, "unit": "GB/s", "frac": rate / hbm,
                              "algorithmic_bytes_per_launch": w / n, "ms_per_launch": t / n,
                              "traffic": tr["bytes_per_launch"] if tr else None}
        if tr:
            rooflines[tag]["traffic_source"] = tr.get("source")
    total = sum(k["ms"] for k in kernels.values())
    for k in kernels.values():
        k["share"] = k["ms"] / total
    dom = max(kernels, key=lambda k: kernels[k]["ms"])
    roof = dict(rooflines[dom], kernel=dom)
    roof["peak_source"] = (f"4 x bf16_tflops of {src} (dense NVFP4:BF16 = 4:1); frac_of_nominal_nvfp4 uses "
                           f"{NOMINAL_NVFP4_TFLOPS:.0f} TF/s" if roof["bound"] == "tensor" else f"hbm_gbs of {src}")
    return {"kernels": kernels, "roofline": roof, "rooflines": rooflines}


def bf16_baseline(data, args):
    """BF16 cuBLAS linear fwd+bwd on the same shapes (torch.matmul: Y, dX, dW)."""
    def step():
        for X, W, E in data:
            X @ W.t()
            E @ W
            E.t() @ X
    return _time_ms(step, iters=args.steps, warmup=args.warmup)


def e2e_measure(q2, data, args, world, dev, rank):
    """Same metric through forward()/backward() with host buffers: pinned X, W, E copied in
    and Y, dX, dW copied out every step, inside the timed region.

    The input pipeline a training loop uses: each projection's (X, W, E) are copied
    host->device on a copy stream into that projection's device buffers (waiting only until
    the previous step's use of those buffers is done), the compute stream waits for its
    inputs, and Y, dX, dW go back device->host on a third stream -- PCIe traffic of one
    projection overlaps compute of another.
    """
    import torch
    host = [tuple(t.cpu().pin_memory() for t in d) for d in data]
    outs = [(torch.empty((X.shape[0], W.shape[0]), dtype=torch.bfloat16).pin_memory(),
             torch.empty(X.shape, dtype=torch.bfloat16).pin_memory(),
             torch.empty(W.shape, dtype=torch.float32).pin_memory()) for X, W, _ in data]
    bufs = [tuple(torch.empty_like(t, device=dev) for t in d) for d in host]
    h2d = sum(t.numel() * t.element_size() for d in host for t in d)
    d2h = sum(t.numel() * t.element_size() for o in outs for t in o)
    main = torch.cuda.current_stream(dev)
    cs, ds = torch.cuda.Stream(device=dev), torch.cuda.Stream(device=dev)
    used = [None] * len(host)                         # event: compute on projection j's buffers done
    cfg = q2.LayerConfig(posthoc=args.mode == "posthoc")

    def step(i):
        seeds = q2.SeedPair(q2.derive_stream(3, i, rank), q2.derive_stream(4, i, rank))
        ready = []
        with torch.cuda.stream(cs):
            for j, (hj, bj) in enumerate(zip(host, bufs)):
                if used[j] is not None:
                    cs.wait_event(used[j])
                for h, b in zip(hj, bj):
                    b.copy_(h, non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(cs)
                ready.append(ev)
        for j, ((X, W, E), o) in enumerate(zip(bufs, outs)):
            main.wait_event(ready[j])
            y, tape = q2.forward(X, W, cfg, out_dtype=torch.bfloat16)
            g = q2.backward(tape, E, seeds, dx_dtype=torch.bfloat16)
            if world > 1:
                torch.distributed.all_reduce(g.dW, async_op=True).wait()   # ordered before the D2H copy
            ev = torch.cuda.Event()
            ev.record(main)
            used[j] = ev
            with torch.cuda.stream(ds):
                ds.wait_event(ev)
                for dst, t in zip(o, (y, g.dX, g.dW)):
                    dst.copy_(t, non_blocking=True)
                    t.record_stream(ds)

    for i in range(args.warmup):
        step(i)
    torch.cuda.synchronize()
    s, e = _events()
    s.record()
    for i in range(args.steps):
        step(i)
    main.wait_stream(ds)                              # every result is back on the host
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / args.steps
    t = torch.tensor([ms], device=dev)
    if world > 1:
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
    ms = float(t.item())
    q2.check_errors()
    return {"value": flops(TOKENS) * world / (ms / 1e3) / 1e12, "unit": "TFLOP/s", "ms_per_step": ms,
            "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
            "copies": "X, W, E in (pinned host -> HBM); Y, dX (bf16) and dW (fp32) out, every step"}


# ----------------------------------------------------------- other configs ---
def extra_configs(q2, args, dev):
    import torch
    hbm, bf16, _ = _peaks()
    out = {}
    seeds = q2.SeedPair(1, 2)

    # c1: the CPU oracle shape, whole layer, plus the oracle itself on it
    from oracle import nvfp4_oracle as O
    g = torch.Generator(device=dev).manual_seed(5)
    X = torch.randn(2048, 1024, device=dev, generator=g).bfloat16()
    W = (torch.randn(1024, 1024, device=dev, generator=g) / 32).bfloat16()
    E = (1e-3 * torch.randn(2048, 1024, device=dev, generator=g)).bfloat16()
    c1 = {}
    for mode in ("posthoc", "exact"):
        cfg = q2.LayerConfig(posthoc=mode == "posthoc")
        layer = lambda: q2.backward(q2.forward(X, W, cfg, out_dtype=torch.bfloat16)[1], E, seeds,  # noqa: E731
                                    dx_dtype=torch.bfloat16)
        c1[mode + "_ms"] = _time_ms(layer, iters=20, warmup=3)
        c1[mode + "_graph_ms"], _ = _graph_ms(layer, iters=20)
    c1["bf16_ms"] = _time_ms(lambda: (X @ W.t(), E @ W, E.t() @ X), iters=20, warmup=3)
    c1["bf16_graph_ms"], _ = _graph_ms(lambda: (X @ W.t(), E @ W, E.t() @ X), iters=20)
    f1 = 6.0 * 2048 * 1024 * 1024
    x64, w64, e64 = (t.double().cpu().numpy() for t in (X, W, E))
    t0 = time.perf_counter()
    _, tape = O.forward(x64, w64)
    O.backward(tape, e64, O.SeedPair(1, 2), posthoc=args.mode == "posthoc")
    c1["oracle_ms"] = (time.perf_counter() - t0) * 1e3
    c1["oracle_cores"] = _threads()
    c1["TFLOP/s"] = {k: f1 / (v / 1e3) / 1e12 for k, v in c1.items() if k.endswith("_ms")}
    out["c1"] = dict(c1, workload="1024->1024, 2048 tokens, fwd+bwd (*_ms: eager launches from Python; *_graph_ms: 20 layer calls captured in one CUDA graph)")

    # c2: quantizer sweep, [N/4096, 4096] bf16 ~ N(0,1) x LogNormal(0,1) per row
    c2 = {}
    for lg in (24, 26, 28, 30):
        n = 1 << lg
        x = (torch.randn(n // 4096, 4096, device=dev) * torch.randn(n // 4096, 1, device=dev).exp()).bfloat16()
        r = {}
        for tag, fn, bpe in (("quant_fwd46", lambda: q2.quantize_rtn_46(x), 2.5625),
                             ("msed_rows", lambda: q2.msed(x, seeds, 6.0, 1, 2, args.mode, "rows"), 2.5625),
                             ("msed_cols", lambda: q2.msed(x, seeds, 6.0, 3, 4, args.mode, "cols"), 2.5625),
                             ("msed_dual", lambda: q2.msed_dual(x, seeds, 1, 2, 3, 4, 6.0, args.mode), 3.125)):
            ms, how = _graph_ms(fn, iters=10 if lg <= 26 else 3)
            gbs = n * bpe / (ms / 1e3) / 1e9
            r[tag] = {"ms": ms, "GB/s": gbs, "frac_hbm": gbs / hbm, "timing": how}
        if lg == 24:
            # the reference's algorithm on the host cores (oracle port), same tensor, one call each
            x64 = x.double().cpu().numpy()
            t0 = time.perf_counter()
            O.quantize_rtn_46(x64)
            t1 = time.perf_counter()
            if args.mode == "posthoc":
                O.posthoc_quantize(x64, O.SeedPair(1, 2), 6.0, 1, 2)
            else:
                O.ms_eden_quantize(x64, O.SeedPair(1, 2), 6.0, 1, 2)
            t2 = time.perf_counter()
            r["cpu_oracle"] = {"quant_fwd46_ms": (t1 - t0) * 1e3, "msed_rows_ms": (t2 - t1) * 1e3,
                               "quant_fwd46_GB/s": n * 2.5625 / (t1 - t0) / 1e9,
                               "msed_rows_GB/s": n * 2.5625 / (t2 - t1) / 1e9, "cores": _threads(),
                               "kind": "port (oracle/nvfp4_oracle.py, numpy + the reference's loop order)"}
            del x64
        c2[f"2^{lg}"] = r
        del x
        torch.cuda.empty_cache()
    out["c2"] = dict(c2, units="GB/s credited at 2.5625 B/elem (one operand) or 3.125 B/elem (E and E^T from one "
                               "read); amax / post-hoc pass-2 traffic not credited", mode=args.mode)

    # c5: large-shape GEMM stress (fprop/dgrad/wgrad), ours vs BF16 cuBLAS vs cuBLASLt NVFP4
    c5 = {}
    T = 32768
    for din, dout in ((8192, 28672), (28672, 8192)):
        for gname, M, N, K in (("fprop", T, dout, din), ("dgrad", T, din, dout), ("wgrad", dout, din, T)):
            qa = _random_nvfp4(q2, M, K, dev)
            qb = _random_nvfp4(q2, N, K, dev)
            od = torch.float32 if gname == "wgrad" else torch.bfloat16
            fl = 2.0 * M * N * K
            ours = _time_ms(lambda: q2.gemm(qa, qb, od), iters=3, warmup=1)
            A = torch.randn(M, K, device=dev, dtype=torch.bfloat16)
            B = torch.randn(N, K, device=dev, dtype=torch.bfloat16)
            ref = _time_ms(lambda: A @ B.t(), iters=3, warmup=1)
            del A, B
            r = {"ours_ms": ours, "ours_TFLOP/s": fl / ours / 1e9, "bf16_ms": ref, "bf16_TFLOP/s": fl / ref / 1e9,
                 "speedup_vs_bf16": ref / ours}
            r.update(_cublaslt_nvfp4(qa, qb, fl))
            c5[f"{din}->{dout} {gname}"] = r
            del qa, qb
            torch.cuda.empty_cache()
    out["c5"] = dict(c5, workload="T=32768, (8192->28672) and (28672->8192), GEMMs alone")
    return out


def _random_nvfp4(q2, R, K, dev):
    """An NVFP4 operand with random codes and scales (GEMM timing only)."""
    import torch
    t = q2.NVFP4Tensor.empty((R, K), dev)
    t.codes.random_(0, 256)
    t.sf.random_(0x30, 0x48)
    t.scale.fill_(1.0)
    return t


def _cublaslt_nvfp4(qa, qb, fl):
    """cuBLASLt block-scaled NVFP4 GEMM (torch._scaled_mm with float4_e2m1fn_x2 operands and
    blocked float8_e4m3fn scales) on the same shapes: the library bar for our tcgen05 GEMM.
    Timing only: the scales are laid out in cuBLAS's blocked format from random bytes."""
    import torch
    try:
        M, K = qa.R, qa.K
        N = qb.R
        a = qa.codes.view(torch.float4_e2m1fn_x2)
        b = qb.codes.view(torch.float4_e2m1fn_x2)
        sa = torch.randint(0x30, 0x48, (((M + 127) // 128) * 128 * ((K // 16 + 3) // 4) * 4,), dtype=torch.uint8,
                           device=qa.codes.device).view(torch.float8_e4m3fn)
        sb = torch.randint(0x30, 0x48, (((N + 127) // 128) * 128 * ((K // 16 + 3) // 4) * 4,), dtype=torch.uint8,
                           device=qa.codes.device).view(torch.float8_e4m3fn)
        fn = lambda: torch._scaled_mm(a, b.t(), sa, sb, out_dtype=torch.bfloat16)   # noqa: E731
        ms = _time_ms(fn, iters=3, warmup=1)
        return {"cublaslt_nvfp4_ms": ms, "cublaslt_nvfp4_TFLOP/s": fl / ms / 1e9}
    except Exception as exc:  # noqa: BLE001 - report why the library arm is unavailable
        return {"cublaslt_nvfp4": f"unavailable: {type(exc).__name__}: {str(exc)[:120]}"}


if __name__ == "__main__":
    main()
