"""DRAM traffic per kernel class of the bench workload (the `traffic` of bench.py's rooflines).

    ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --csv \
        --log-file gpurun_out/traffic_MODE.csv python tools/traffic.py run MODE     (on the GPU box)
    python tools/traffic.py summarize                                              (anywhere)

`run` issues each kernel class of bench.kernel_breakdown once per c3 projection and
records, per call, the class and how many of our kernels it launched (library launch
counter) in gpurun_out/traffic_seq_MODE.json; `summarize` maps the ncu launch list onto
those calls and writes profiles/r2_traffic.json: mean DRAM read+write bytes per call of
each class (ncu replays kernels with cold caches, so this is the traffic a launch
really moves).
"""
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
OUT = os.path.join(ROOT, "gpurun_out")


def run(mode):
    import torch

    import bench
    import paper_2601_22813_b200 as q2
    from paper_2601_22813_b200 import _lib
    from paper_2601_22813_b200.linear_graph import PAIR_DW, PAIR_DX
    dev = torch.device("cuda:0")
    q2.set_error_mode("deferred")
    L = _lib.lib()
    seeds, ds = q2.SeedPair(11, 12), q2.derive_stream
    seq = []

    def call(tag, fn):
        torch.cuda.synchronize()
        L.q2_launch_count(1)
        r = fn()
        torch.cuda.synchronize()
        seq.append((tag, int(L.q2_launch_count(1))))
        return r

    g = torch.Generator(device=dev)
    for pi, (name, din, dout) in enumerate(bench.PROJECTIONS):
        g.manual_seed(1000 * pi + 1)
        W = (torch.randn(dout, din, device=dev, generator=g) / din ** 0.5).to(torch.bfloat16)
        g.manual_seed(1000 * pi + 2)
        X = torch.randn(bench.TOKENS, din, device=dev, generator=g).to(torch.bfloat16)
        E = (1e-3 * torch.randn(bench.TOKENS, dout, device=dev, generator=g)).to(torch.bfloat16)
        qx = call("quant_fwd46", lambda: q2.quantize_rtn_46(X))
        qw = call("quant_fwd46", lambda: q2.quantize_rtn_46(W))
        call("gemm_fprop", lambda: q2.gemm(qx, qw, torch.bfloat16))
        qe, qet = call("msed_dual_E", lambda: q2.msed_dual(E, seeds, ds(PAIR_DX, 0), PAIR_DX, ds(PAIR_DW, 0), PAIR_DW,
                                                            6.0, mode))
        qwt = call("msed_tape", lambda: q2.msed(qw, seeds, 6.0, ds(PAIR_DX, 1), PAIR_DX, mode, "tape"))
        call("gemm_dgrad", lambda: q2.gemm(qe, qwt, torch.bfloat16))
        qxt = call("msed_tape", lambda: q2.msed(qx, seeds, 6.0, ds(PAIR_DW, 1), PAIR_DW, mode, "tape"))
        call("gemm_wgrad", lambda: q2.gemm(qet, qxt, torch.float32))
    os.makedirs(OUT, exist_ok=True)
    with open(os.path.join(OUT, f"traffic_seq_{mode}.json"), "w") as f:
        json.dump(seq, f)


def _launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 5]
    h = rows[0]
    ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
    by = {}
    for r in rows[1:]:
        d = by.setdefault(int(r[ii]), {"name": r[ki]})
        d[r[mi]] = float(r[vi].replace(",", ""))
    return [by[k] for k in sorted(by)]


def summarize():
    table = {}
    for mode in ("posthoc", "exact"):
        csvp, seqp = os.path.join(OUT, f"traffic_{mode}.csv"), os.path.join(OUT, f"traffic_seq_{mode}.json")
        if not (os.path.exists(csvp) and os.path.exists(seqp)):
            continue
        launches = _launches(csvp)
        seq = json.load(open(seqp))
        # our kernels only (torch's randn / copies are in the list too): match by the
        # number of launches per call from the end of the list backwards
        ours = [k for k in launches if "q2::" in k["name"]]
        assert sum(n for _, n in seq) == len(ours), (sum(n for _, n in seq), len(ours))
        pos, acc = 0, {}
        for tag, n in seq:
            ks = ours[pos:pos + n]
            pos += n
            b = sum(k.get("dram__bytes_read.sum", 0) + k.get("dram__bytes_write.sum", 0) for k in ks)
            acc.setdefault(tag, []).append((b, [k["name"].split("(")[0] for k in ks]))
        for tag, lst in acc.items():
            key = mode if tag.startswith("msed") else "any"
            if key in table.get(tag, {}):
                continue
            table.setdefault(tag, {})[key] = {
                "bytes_per_launch": sum(b for b, _ in lst) / len(lst), "calls": len(lst),
                "kernels": sorted({n for _, ns in lst for n in ns}),
                "source": f"ncu dram__bytes_read.sum + dram__bytes_write.sum, gpurun_out/traffic_{mode}.csv "
                          "(tools/traffic.py), mean over the four c3 projections"}
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    with open(os.path.join(ROOT, "profiles", "r2_traffic.json"), "w") as f:
        json.dump(table, f, indent=1)
    print(json.dumps(table, indent=1))


if __name__ == "__main__":
    if sys.argv[1] == "run":
        run(sys.argv[2])
    else:
        summarize()
