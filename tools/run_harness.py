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
    runs = H.train_demo(("identity", "quartet2", "tetrajet_v2", "nvidia"), steps=2000, n_seeds=5)
    t3 = time.time()
    demo = {}
    for r in runs:
        demo.setdefault(r.config, []).append(r.final_loss)
    train = {c: {"final_losses": v, "mean": sum(v) / len(v)} for c, v in demo.items()}
    rep = {"mse_bench": mse, "concentration": conc, "train_demo": train,
           "grad_check": H.grad_check("identity").to_dict(),
           "seconds": {"mse_bench": t1 - t0, "concentration": t2 - t1, "train_demo": t3 - t2}}
    os.makedirs(os.path.dirname(out), exist_ok=True)
    with open(out, "w") as f:
        json.dump(rep, f, indent=1)
    for r in mse:
        print(f"{r['method']:14s} mse_e3={r['mse_e3']:.3f} (target {r['target_e3']}) stderr_e3={r['stderr'] * 1e3:.3f}")
    for c in conc:
        print(f"{c['config']:24s} slope={c['slope']:.3f} tail={c['tail_slope']:.3f} err@1024={c['rel_errors'][-1]:.3e}")
    for c, v in train.items():
        print(f"train_demo {c:12s} final loss {v['mean']:.4e}")
    print(rep["grad_check"], rep["seconds"])


if __name__ == "__main__":
    main()
