#!/usr/bin/env python
"""Quartet II linear fwd+bwd benchmark (BASELINE.json metric) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

One step = forward + backward of the four Llama-1.9B-class projections of
BASELINE config c3 (QKV 2048->6144, O 2048->2048, UpGate 2048->11264,
Down 5632->2048) over 16,384 tokens per GPU, through the public API
(paper_2601_22813_b200.forward / backward): 4/6 quantization of X and W,
fprop GEMM, MS-EDEN re-quantization of E, E^T, W^T, X^T, dgrad and wgrad
GEMMs.  Under torchrun each rank processes its own 16,384-token shard (weak
scaling, config c4 at N=4) and dW is all-reduced over NCCL.

value = 6 * tokens * in * out summed over projections and ranks / max-rank time.
Inputs are larger than L2 (each step streams >1 GB through HBM), so no flush.
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
METRIC = "Quartet II linear fwd+bwd TFLOP/s"


def flops(tokens: int) -> float:
    return sum(6.0 * tokens * i * o for _, i, o in PROJECTIONS)


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
def run_reference(args, world: int) -> None:
    """The reference's CPU path (the oracle port: /root/reference cannot travel)."""
    from oracle import nvfp4_oracle as O
    T = 256
    name, din, dout = PROJECTIONS[1]
    rng = np.random.default_rng(0)
    X = rng.standard_normal((T, din)).astype(np.float32)
    W = (rng.standard_normal((dout, din)) / np.sqrt(din)).astype(np.float32)
    E = (1e-3 * rng.standard_normal((T, dout))).astype(np.float32)
    f = 6.0 * T * din * dout

    def step(i):
        y, tape = O.forward(X, W)
        O.backward(tape, E, O.SeedPair(1, i), posthoc=args.mode == "posthoc")

    for i in range(args.warmup):
        step(i)
    t0 = time.perf_counter()
    for i in range(args.steps):
        step(i)
    dt = (time.perf_counter() - t0) / args.steps
    v = f / dt / 1e12
    cores = os.cpu_count()
    sample = f"oracle fwd+bwd of the c3 '{name}' projection ({din}->{dout}) on a {T}-token slice, per step"
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": v, "unit": "TFLOP/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": "c3 Llama-1.9B projections, 16384 tokens/GPU (sampled)", "msed_mode": args.mode},
        "cpu_baseline": {"value": v, "unit": "TFLOP/s", "cores": cores, "kind": "port", "sample": sample},
        "e2e": {"value": v, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }))


def cpu_baseline_sample(mode: str) -> dict:
    from oracle import nvfp4_oracle as O
    T, (name, din, dout) = 256, PROJECTIONS[1]
    rng = np.random.default_rng(0)
    X = rng.standard_normal((T, din)).astype(np.float32)
    W = (rng.standard_normal((dout, din)) / np.sqrt(din)).astype(np.float32)
    E = (1e-3 * rng.standard_normal((T, dout))).astype(np.float32)
    t0 = time.perf_counter()
    n = 0
    while n < 2 or time.perf_counter() - t0 < 10.0:
        y, tape = O.forward(X, W)
        O.backward(tape, E, O.SeedPair(1, n), posthoc=mode == "posthoc")
        n += 1
    dt = (time.perf_counter() - t0) / n
    return {"value": 6.0 * T * din * dout / dt / 1e12, "unit": "TFLOP/s", "cores": os.cpu_count(), "kind": "port",
            "sample": f"numpy oracle fwd+bwd, '{name}' projection {din}->{dout}, {T} tokens, {n} reps "
                      "(quantizers single-threaded numpy, GEMMs multi-threaded BLAS)"}


# ----------------------------------------------------------------- ours -----
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--mode", default="posthoc", choices=["posthoc", "exact"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
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

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    q2.set_error_mode("deferred")
    cfg = q2.LayerConfig(posthoc=args.mode == "posthoc")

    g = torch.Generator(device=dev)
    data = []
    for pi, (name, din, dout) in enumerate(PROJECTIONS):
        g.manual_seed(1000 * pi + 1)                       # W identical on all ranks
        W = (torch.randn(dout, din, device=dev, generator=g) / din ** 0.5).to(torch.bfloat16)
        g.manual_seed(1000 * pi + 2 + 17 * rank)
        X = torch.randn(TOKENS, din, device=dev, generator=g).to(torch.bfloat16)
        E = (1e-3 * torch.randn(TOKENS, dout, device=dev, generator=g)).to(torch.bfloat16)
        data.append((X, W, E))

    events = []

    def mark(tag):
        ev = torch.cuda.Event(enable_timing=True)
        ev.record()
        events.append((tag, ev))

    def step(i, instrument=False):
        seeds = q2.SeedPair(q2.derive_stream(1, i, rank), q2.derive_stream(2, i, rank))
        pending = []                                      # dW all-reduces overlap the next projection
        for X, W, E in data:
            if instrument:
                mark("fwd")
            y, tape = q2.forward(X, W, cfg, out_dtype=torch.bfloat16)
            if instrument:
                mark("bwd")
            grads = q2.backward(tape, E, seeds, dx_dtype=torch.bfloat16)
            if instrument:
                mark("end")
            if world > 1:
                pending.append(dist.all_reduce(grads.dW, async_op=True))
        for h in pending:
            h.wait()
        return y

    for i in range(args.warmup):
        step(i)
    torch.cuda.synchronize()
    # per-phase split from one instrumented eager step (before capture: the
    # first eager step after a capture pays the allocator's cudaMallocs)
    step(args.warmup, instrument=True)
    torch.cuda.synchronize()

    # The step is captured once into a CUDA graph (kernels, memsets and the dW
    # all-reduce; host-side Python/ctypes launch overhead removed).  Seeds are
    # baked into the captured launches, which does not change the work done.
    graph, launch = None, "eager"
    if not args.eager and world == 1:      # N > 1: eager launches (no NCCL inside a captured graph)
        try:
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph):
                step(args.warmup)
            graph.replay()
            torch.cuda.synchronize()
            launch = "cuda_graph"
        except Exception as exc:  # noqa: BLE001 - fall back to eager launches
            graph, launch = None, f"eager (graph capture failed: {type(exc).__name__})"
            torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()

    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        start.record()
        for i in range(args.steps):
            if graph is not None:
                graph.replay()
            else:
                step(args.warmup + i)
        end.record()
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms = start.elapsed_time(end) / args.steps
    t = torch.tensor([ms], device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    q2.check_errors()

    # per-phase device time inside the timed region
    phase = {"fwd": 0.0, "bwd": 0.0}
    for (tag, ev), (_, nxt) in zip(events, events[1:]):
        if tag in phase:
            phase[tag] += ev.elapsed_time(nxt)
    phase = {k: v for k, v in phase.items()}

    # per-kernel-class timing for the roofline (a separate instrumented step)
    detail = kernel_breakdown(q2, data, cfg, dev)

    # BF16 cuBLAS linear fwd+bwd on the same shapes
    bf16_ms = bf16_baseline(data, args)

    # end-to-end through the public API with host buffers (H2D inputs, D2H dW)
    e2e = e2e_measure(q2, data, cfg, args, world, dev)

    total_flops = flops(TOKENS) * world
    value = total_flops / (ms / 1e3) / 1e12
    out = {
        "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "nvfp4 (e2m1 x ue4m3, fp32 accumulate; bf16 in/out)", "data": "synthetic",
        "config": {"workload": "c3: Llama-1.9B-class projections qkv/o/upgate/down (d=2048, ffn=5632), "
                               f"{TOKENS} tokens per GPU, fwd+bwd", "tokens_per_gpu": TOKENS,
                   "msed_mode": args.mode, "parallelism": f"token-sharded dp{world}" if world > 1 else "single",
                   "l2": "inputs larger than L2 (>1 GB streamed per step), no flush", "launch": launch},
        "speedup_vs_bf16": bf16_ms / ms, "bf16_cublas_ms_per_step": bf16_ms,
        "phase_ms_eager": phase, "kernels": detail["kernels"],
        "roofline": detail["roofline"],
        "e2e": e2e,
        "gpu_launches": 17 * len(PROJECTIONS) * args.steps,   # per projection: 2x(amax, quant, fix) + 3 GEMMs + 4x(MS-EDEN pass 1, pass 2)
        "clocks": clk.summary(),
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        out["cpu_baseline"] = cpu_baseline_sample(args.mode)
    if rank == 0:
        print(json.dumps(out))
    if world > 1:
        dist.destroy_process_group()


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return p["hbm_gbs"], p["bf16_tflops"], "MEASURED_PEAKS.json"
    except (OSError, KeyError, ValueError):
        return 6650.0, 1590.0, "fallback (B200_PROFILING.md)"


def kernel_breakdown(q2, data, cfg, dev):
    """Time each kernel class with CUDA events on the launching stream."""
    import torch
    hbm, bf16, src = _peaks()
    acc = {}

    def timed(tag, fn, work, unit):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        r = fn()
        e.record()
        acc.setdefault(tag, []).append((s, e, work, unit))
        return r

    from paper_2601_22813_b200.linear_graph import PAIR_DW, PAIR_DX
    seeds = q2.SeedPair(11, 12)
    mode = "posthoc" if cfg.posthoc else "exact"
    for _ in range(2):
        acc.clear()
        for X, W, E in data:
            T, din = X.shape
            dout = W.shape[0]
            qx = timed("quant_fwd46", lambda: q2.quantize_rtn_46(X), T * din * 2.5625, "B")
            qw = timed("quant_fwd46", lambda: q2.quantize_rtn_46(W), dout * din * 2.5625, "B")
            timed("gemm_fprop", lambda: q2.gemm(qx, qw, torch.bfloat16), 2.0 * T * din * dout, "F")
            qe = timed("msed_rows_bf16", lambda: q2.msed(E, seeds, 6.0, 1, PAIR_DX, mode, "rows"), T * dout * 2.5625, "B")
            qwt = timed("msed_tape", lambda: q2.msed(qw, seeds, 6.0, 2, PAIR_DX, mode, "tape"), dout * din * 1.125, "B")
            timed("gemm_dgrad", lambda: q2.gemm(qe, qwt, torch.bfloat16), 2.0 * T * din * dout, "F")
            qet = timed("msed_cols_bf16", lambda: q2.msed(E, seeds, 6.0, 3, PAIR_DW, mode, "cols"), T * dout * 2.5625, "B")
            qxt = timed("msed_tape", lambda: q2.msed(qx, seeds, 6.0, 4, PAIR_DW, mode, "tape"), T * din * 1.125, "B")
            timed("gemm_wgrad", lambda: q2.gemm(qet, qxt, torch.float32), 2.0 * T * din * dout, "F")
        torch.cuda.synchronize()
    kernels = {}
    for tag, lst in acc.items():
        t = sum(s.elapsed_time(e) for s, e, _, _ in lst)
        w = sum(x[2] for x in lst)
        unit = lst[0][3]
        rate = w / (t / 1e3) / (1e12 if unit == "F" else 1e9)
        kernels[tag] = {"ms": t, "launches": len(lst), ("TFLOP/s" if unit == "F" else "GB/s"): rate}
    # The dominant kernel is a kernel FUNCTION (what the ncu launch list shows): fprop and
    # dgrad are both nvfp4_gemm_kernel<bf16 out>, so their launches are pooled.
    functions = {"nvfp4_gemm_kernel<bf16 out> (fprop+dgrad)": ["gemm_fprop", "gemm_dgrad"],
                 "nvfp4_gemm_kernel<f32 out> (wgrad)": ["gemm_wgrad"]}
    pooled = {name: [x for t in tags for x in acc[t]] for name, tags in functions.items()}
    for tag in acc:
        if not any(tag in tags for tags in functions.values()):
            pooled[tag] = acc[tag]
    ms_of = {k: sum(s_.elapsed_time(e_) for s_, e_, _, _ in v) for k, v in pooled.items()}
    dom = max(ms_of, key=ms_of.get)
    lst = pooled[dom]
    d = {"ms": ms_of[dom], "launches": len(lst)}
    rate = sum(x[2] for x in lst) / (ms_of[dom] / 1e3)
    d["TFLOP/s" if lst[0][3] == "F" else "GB/s"] = rate / (1e12 if lst[0][3] == "F" else 1e9)
    # DRAM bytes per algorithmic byte from `ncu --set full` captures (profiles/round1_summary.md)
    measured_ratio = {"msed_cols_bf16": 477.1 / 472.8, "msed_rows_bf16": 477.1 / 472.8}
    launches = d["launches"]
    work_per_launch = sum(x[2] for x in lst) / launches
    if "TFLOP/s" in d:
        peak = 4.0 * bf16
        # ncu --set full of the c3 UpGate fprop and dgrad launches (profiles/r1_nvfp4_gemm_kernel_details.csv):
        # 371.0 MB and 169.6 MB DRAM read+write -- the bf16 output dominates fprop
        traffic = (371.0e6 + 169.6e6) / 2 if dom.startswith("nvfp4_gemm_kernel<bf16") else None
        roof = {"bound": "tensor", "kernel": dom, "achieved": d["TFLOP/s"], "peak": peak, "unit": "TFLOP/s",
                "frac": d["TFLOP/s"] / peak, "traffic": traffic, "flops_per_launch": work_per_launch,
                "traffic_note": "bytes per launch, mean of the UpGate fprop and dgrad ncu captures",
                "ms_per_launch": ms_of[dom] / launches,
                "peak_source": f"4 x bf16_tflops of {src} (dense NVFP4:BF16 = 4:1 on B200; nominal 9 PF)"}
    else:
        traffic = work_per_launch * measured_ratio[dom] if dom in measured_ratio else None
        roof = {"bound": "hbm", "kernel": dom, "achieved": d["GB/s"], "peak": hbm, "unit": "GB/s",
                "frac": d["GB/s"] / hbm, "traffic": traffic, "traffic_unit": "bytes per launch (ncu dram r+w)",
                "algorithmic_bytes_per_launch": work_per_launch, "peak_source": f"hbm_gbs of {src}",
                "note": "compute-bound: literal float64 MS-EDEN (DESIGN.md §5)"}
    total = sum(k["ms"] for k in kernels.values())
    for k in kernels.values():
        k["share"] = k["ms"] / total
    return {"kernels": kernels, "roofline": roof}


def bf16_baseline(data, args):
    import torch
    Ws = [W.clone().requires_grad_(True) for _, W, _ in data]

    def step():
        for (X, _, E), W in zip(data, Ws):
            y = X @ W.t()
            dx = E @ W
            dw = E.t() @ X
        return y, dx, dw

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(args.steps):
        step()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / args.steps


def e2e_measure(q2, data, cfg, args, world, dev):
    """Same metric through forward()/backward() with pinned host inputs copied in and dW copied out.

    The input pipeline a training loop uses: each projection's (X, W, E) are
    copied host->device on a copy stream into that projection's device buffers
    (waiting only until the previous step's use of those buffers is done), the
    compute stream waits for its inputs, and dW goes back device->host on a
    third stream -- PCIe traffic of one projection overlaps compute of another.
    """
    import torch
    host = [tuple(t.cpu().pin_memory() for t in d) for d in data]
    outs = [torch.empty(W.shape, dtype=torch.float32).pin_memory() for _, W, _ in data]
    bufs = [tuple(torch.empty_like(t, device=dev) for t in d) for d in host]
    h2d = sum(t.numel() * t.element_size() for d in host for t in d)
    d2h = sum(o.numel() * o.element_size() for o in outs)
    main = torch.cuda.current_stream(dev)
    cs, ds = torch.cuda.Stream(device=dev), torch.cuda.Stream(device=dev)
    used = [None] * len(host)                         # event: compute on projection j's buffers done

    def step(i):
        seeds = q2.SeedPair(q2.derive_stream(3, i), q2.derive_stream(4, i))
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
                o.copy_(g.dW, non_blocking=True)
                g.dW.record_stream(ds)

    for i in range(args.warmup):
        step(i)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for i in range(args.steps):
        step(i)
    main.wait_stream(ds)                              # every dW is back on the host
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / args.steps
    t = torch.tensor([ms], device=dev)
    if world > 1:
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
    ms = float(t.item())
    q2.check_errors()
    return {"value": flops(TOKENS) * world / (ms / 1e3) / 1e12, "unit": "TFLOP/s", "ms_per_step": ms,
            "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h}


if __name__ == "__main__":
    main()
