"""BASELINE.md §2 CPU plan, the full-solve legs: the oracle (reference
algorithm, LAPACK) timed on the box's host cores for C1 and C2 in full --
median of 3 on all threads, and once on 1 thread.  Usage:
python scripts/cpu_baseline.py [out.json]"""
import json, os, statistics, subprocess, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle"), os.path.join(ROOT, "tests")]
import pyoracle as O
from paper_1707_05882_b200 import materials as M
from helpers import oracle_material


def model():
    try:
        for line in subprocess.run(["lscpu"], capture_output=True, text=True).stdout.splitlines():
            if line.startswith("Model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


out = {"cpu_model": model(), "nproc": os.cpu_count(), "configs": {}}
for cfg in ("C1", "C2"):
    w = M.config(cfg)
    nodes, _ = O.quadrature(w.N)
    om = oracle_material(w.material)
    rec = {}
    for threads, reps in ((os.cpu_count(), 3), (1, 1)):
        ts = []
        for _ in range(reps):
            t = time.perf_counter()
            O.brdf(om, w.N, nodes, w.n_dphi, threads=threads)
            ts.append(time.perf_counter() - t)
        rec[f"threads_{threads}"] = {"seconds_per_solve": statistics.median(ts), "runs": ts}
    out["configs"][cfg] = rec
    print(cfg, json.dumps(rec), flush=True)
json.dump(out, open(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/cpu_baseline.json", "w"), indent=1)
