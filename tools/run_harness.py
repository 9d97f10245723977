"""Run the GPU statistical harness (MSE table + concentration for every recipe) and
write profiles/r1_harness.json.

    python tools/run_harness.py [out.json]
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2601_22813_b200 import harness as H  # noqa: E402


def main():
    out = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/r1_harness.json"
    t0 = time.time()
    mse = [r.to_dict() for r in H.mse_bench(n_samples=1_000_000, seed=0)]
    t1 = time.time()
    conc = [H.concentration(c, b_max=1024, trials=2, seed=0).to_dict()
            for c in ("quartet2", "tetrajet_v2", "nvidia", "four_over_six", "four_over_six_backward")]
    t2 = time.time()
    rep = {"mse_bench": mse, "concentration": conc, "seconds": {"mse_bench": t1 - t0, "concentration": t2 - t1}}
    os.makedirs(os.path.dirname(out), exist_ok=True)
    with open(out, "w") as f:
        json.dump(rep, f, indent=1)
    for r in mse:
        print(f"{r['method']:14s} mse_e3={r['mse_e3']:.3f} (target {r['target_e3']}) stderr_e3={r['stderr'] * 1e3:.3f}")
    for c in conc:
        print(f"{c['config']:24s} slope={c['slope']:.3f} tail={c['tail_slope']:.3f} err@1024={c['rel_errors'][-1]:.3e}")
    print(rep["seconds"])


if __name__ == "__main__":
    main()
