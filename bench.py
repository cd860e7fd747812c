#!/usr/bin/env python
"""bench.py -- full polarized BRDF solves/sec on B200 (BASELINE.json metric).

Workload (the headline config that fits one GPU): two-layer
paint -- top omega=0.95 tau=2 G(0.6,64), bottom omega=0.6 tau=5 Rayleigh,
Lambertian base rho=0.2 -- N=64 streams, L=64 Fourier orders, all 64 incident
quadrature cosines x 4 Stokes basis vectors, 19 azimuths: one step = one full
vrte_compute_brdf-equivalent solve (the whole 64x64x19 4x4 Mueller table).

  value : device-resident solves/s (inputs in HBM; CUDA events on the plan's
          stream; all stages GSF -> eigen -> particular -> boundary -> synthesis)
  e2e   : solves/s through the public C ABI (vrte_compute_brdf) with host
          buffers: host set-up, H2D of the inputs, D2H of the 10 MB table.
Multi-GPU (torchrun): every rank solves whole BRDFs (independent bands /
materials are the natural unit; SURVEY §8(e) "shard by band first"), no
data-path collective -> "scaling": "weak"; the max time over ranks is used.
`--impl reference` times the reference algorithm (CPU restatement in
oracle/, all host threads) on the same workload with a bounded sample.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import tempfile
import threading
import time

# every plan runs on several streams (main, side, right-hand sides, look-ahead); with
# plans in flight together the default 8 hardware work queues would alias streams
# onto one queue (false dependencies): give the context the maximum before it exists
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "full polarized BRDF (N=64 streams) solves/sec at 1/2/4/8 B200 vs CPU reference"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="C3")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-incidents", type=int, default=2,
                    help="incidents in the bounded CPU sample (x4 basis vectors)")
    ap.add_argument("--concurrency", type=int, default=4,
                    help="C5 spectral batch: bands solved concurrently (plans / streams)")
    return ap.parse_args()


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def workload(cfg):
    from paper_1707_05882_b200 import materials as M
    from paper_1707_05882_b200.materials import config
    w = config(cfg)
    return w


def quad_nodes(N):
    import numpy as np
    # Gauss-Legendre on (0,1) exactly as the host library builds it (types.cpp:27-68)
    x = np.zeros(N)
    half = (N + 1) // 2
    for k in range(half):
        z = math.cos(math.pi * (k + 0.75) / (N + 0.5))
        for _ in range(100):
            p0, p1 = 1.0, z
            for l in range(2, N + 1):
                p0, p1 = p1, ((2.0 * l - 1.0) * z * p1 - (l - 1.0) * p0) / l
            dp = N * (z * p1 - p0) / (z * z - 1.0)
            dz = p1 / dp
            z -= dz
            if abs(dz) < 1e-15:
                break
        x[N - 1 - k] = 0.5 * (1.0 + z)
        x[k] = 0.5 * (1.0 - z)
    if N == 1:
        x[0] = 0.5
    return x


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), "--query-gpu=" + self.FIELDS,
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
        return self

    def __exit__(self, *exc):
        self.out = ""
        if self.proc:
            self.proc.terminate()
            try:
                self.out, _ = self.proc.communicate(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
                self.out = ""

    def summary(self, busy_only=True):
        rows = []
        for line in (self.out or "").splitlines():
            p = [x.strip() for x in line.split(",")]
            if len(p) < 9:
                continue
            try:
                rows.append((float(p[1]), float(p[2]), float(p[3]), p[5:9]))
            except ValueError:
                continue
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i, v in enumerate(r[3]) if v.lower() == "active"})
        return {"sm_mhz": statistics.median(r[0] for r in rows), "sm_max_mhz": max(r[1] for r in rows),
                "power_w_max": max(r[2] for r in rows), "samples": len(rows), "reasons": reasons}


def fp64_peak_tflops(device):
    """Measured cuBLAS DGEMM throughput (torch.float64 matmul 8192^3, best of 5).
    MEASURED_PEAKS.json carries bf16/HBM only; this is the FP64 roofline denominator."""
    import torch
    n = 8192
    a = torch.randn(n, n, dtype=torch.float64, device=device)
    b = torch.randn(n, n, dtype=torch.float64, device=device)
    torch.matmul(a, b)
    torch.cuda.synchronize(device)
    best = 0.0
    for _ in range(5):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        torch.matmul(a, b)
        e.record()
        e.synchronize()
        best = max(best, 2 * n ** 3 / (s.elapsed_time(e) * 1e-3) / 1e12)
    del a, b
    torch.cuda.empty_cache()
    return best


def oracle_sample(w, mu_nodes, n_inc, threads):
    """Reference algorithm on the CPU: prepare_homogeneous + n_inc incidents x 4
    basis; extrapolated full-solve seconds T = T_hom + (n_in/k) (T - T_hom)."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import numpy as np
    import pyoracle as O
    desc = w.material
    bt = {"black": 0, "lambertian": 1, "mueller_table": 2}[desc.base]
    om = O.Material(np.array([l.omega for l in desc.layers]), np.array([l.tau for l in desc.layers]),
                    desc.padded_coeffs(), bt, desc.albedo, desc.table)
    pick = np.linspace(0, len(mu_nodes) - 1, n_inc).round().astype(int)
    table, tm = O.brdf(om, w.N, mu_nodes[pick], w.n_dphi, threads=threads)
    t_hom = tm["homogeneous"]
    t_inc = tm["total_wall"] - t_hom
    full = t_hom + len(mu_nodes) / n_inc * t_inc
    oracle_sample.last = (pick, table)
    return full, tm, [float(x) for x in mu_nodes[pick]]


def cpu_model():
    try:
        for line in subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout.splitlines():
            if line.startswith("Model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


def parity_record(gpu_table):
    """Parity carried on the bench line: live, the GPU table at the CPU sample's
    incidents vs the oracle as written (the same run); and the full-table
    numbers of profiles/parity_r02.json (GPU vs the oracle as written and in
    accurate mode, every incident, SURVEY §8(d) metric)."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from helpers import matrix_metric, survey_metric
    out = {"metric": "SURVEY §8(d): per Mueller matrix max_rc |G-R| / max(|R_rc|, 1e-3 |R_00|)"}
    last = getattr(oracle_sample, "last", None)
    if last is not None and gpu_table is not None:
        pick, r = last
        g = gpu_table[pick]
        out["live_vs_reference_as_written"] = {"incidents": [int(i) for i in pick], "survey": survey_metric(g, r),
                                               "matrix": matrix_metric(g, r)}
    prof = os.path.join(ROOT, "profiles", "parity_r02.json")
    if os.path.exists(prof):
        try:
            pj = json.load(open(prof))
            out["full_table"] = {c["workload"]: {k: c[k] for k in ("gpu_vs_accurate_survey", "gpu_vs_ref_survey",
                                                                   "ref_vs_accurate_survey", "gpu_vs_accurate_matrix")}
                                 for c in pj.get("cases", [])}
            out["full_table_source"] = "profiles/parity_r02.json (scripts/parity_full.py on the B200)"
        except Exception:
            pass
    return out


def run_reference(args):
    world, rank, _ = dist_env()
    if rank != 0:
        return
    w = workload(args.config)
    nodes = quad_nodes(w.N)
    threads = os.cpu_count() or 1
    vals, walls = [], []
    t0 = time.time()
    for step in range(args.warmup + args.steps):
        ts = time.perf_counter()
        full, tm, picked = oracle_sample(w, nodes, args.cpu_incidents, threads)
        if step >= args.warmup:
            vals.append(full)
            walls.append(time.perf_counter() - ts)
    t_full = statistics.mean(vals)
    value = 1.0 / t_full
    sample = (f"prepare_homogeneous (all {w.material.order_count} orders x media) + "
              f"{args.cpu_incidents} incident(s) x 4 basis per step, extrapolated to "
              f"{len(nodes)} incidents (T = T_hom + n_in/k T_k, SURVEY §8(d))")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "solves/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        # a step is the bounded sample (its real wall time); value is the full solve
        # rate extrapolated from it (T = T_hom + n_in/k T_k)
        "ms_per_step": statistics.mean(walls) * 1e3, "extrapolated_ms_per_solve": t_full * 1e3,
        "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (SURVEY §8(d) generator)",
        "config": {"workload": f"{args.config}: {w.note}", "N": w.N, "L": w.material.order_count,
                   "layers": len(w.material.layers), "n_in": len(nodes), "n_dphi": w.n_dphi},
        "cpu_baseline": {"value": value, "unit": "solves/s", "cores": threads, "kind": "port",
                         "extrapolated": True, "cpu_model": cpu_model(), "sample": sample},
        "e2e": {"value": value, "unit": "solves/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "wall_s": time.time() - t0,
    }
    print(json.dumps(line), flush=True)


def run_c5(args):
    """BASELINE config 5: 31 spectral bands (independent paints),
    one BRDF solve per band.  Bands are sharded across ranks (band b on rank
    b mod world, no collective) and solved concurrently on each GPU: one
    device plan / CUDA stream per band, --concurrency host threads.  value =
    bands/s of the whole job (wall clock between device synchronisations:
    several streams are in flight); e2e through vrte_compute_brdf_batch."""
    import threading
    import torch
    import paper_1707_05882_b200 as V
    from paper_1707_05882_b200.materials import config

    world, rank, local = dist_env()
    dist = None
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    os.environ["VRTE_DEVICE"] = str(local)
    bands = [b for b in range(31) if b % world == rank]
    ws = [config("C5", band=b) for b in bands]
    N, nd = ws[0].N, ws[0].n_dphi
    nodes = quad_nodes(N)
    tmp = tempfile.mkdtemp(prefix=f"vrte_c5_{rank}_")
    mats = [V.Material.load(w.material.write(tmp, f"b{b}")) for b, w in zip(bands, ws)]
    opts = V.options(N)
    peak = fp64_peak_tflops(torch.device("cuda", local)) if rank == 0 else None
    plans = [V.Plan(m, opts, nodes, nd, device=local, pooled=True) for m in mats]  # concurrent: lean kernels
    K = max(1, args.concurrency)

    def run_all(steps):
        groups = [plans[i::K] for i in range(K)]
        ths = [threading.Thread(target=lambda g=g: [p.run(steps) for p in g]) for g in groups]
        for th in ths:
            th.start()
        for th in ths:
            th.join()

    run_all(max(args.warmup, 1))
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        t0 = time.perf_counter()
        run_all(args.steps)
        torch.cuda.synchronize()
        dev_s = time.perf_counter() - t0
    t = torch.tensor([dev_s], dtype=torch.float64, device="cuda")
    if dist:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    dev_s = float(t.item())
    value = 31 * args.steps / dev_s
    for p in plans:
        p.close()
    # e2e: the batch entry point with host buffers
    for _ in range(args.warmup):
        for b in V.compute_brdf_batch(mats, opts, nodes, nd, concurrency=K):
            b.close()
    if dist:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        for b in V.compute_brdf_batch(mats, opts, nodes, nd, concurrency=K):
            b.close()
    e2e_s = time.perf_counter() - t0
    t = torch.tensor([e2e_s], dtype=torch.float64, device="cuda")
    if dist:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    e2e_s = float(t.item())
    if rank != 0:
        if dist:
            dist.destroy_process_group()
        return
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        threads = os.cpu_count() or 1
        full, tm, picked = oracle_sample(ws[0], nodes, args.cpu_incidents, threads)
        cpu = {"value": 1.0 / full, "unit": "solves/s", "cores": threads, "kind": "port",
               "sample": f"oracle/ band 0 on {threads} host threads: prepare_homogeneous + "
                         f"{args.cpu_incidents} incident(s) x 4 basis, extrapolated to {len(nodes)} incidents "
                         f"({full:.1f} s per band; the 31 bands are independent)"}
    n_in = len(nodes)
    line = {
        "metric": METRIC, "value": value, "unit": "solves/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": dev_s / args.steps * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (SURVEY §8(d) C5: 31 bands, top omega/g varying, deterministic)",
        "config": {"workload": "C5: 31-band spectral batch of 2-layer paints (one solve per band)",
                   "N": N, "L": 64, "layers": 2, "n_in": n_in, "n_dphi": nd, "bands": 31,
                   "concurrency": K,
                   "parallelism": f"bands sharded x{world}, {K} concurrent plans/streams per GPU",
                   "timing": "wall clock between device synchronisations (several streams in flight)"},
        "e2e": {"value": 31 * args.steps / e2e_s, "unit": "solves/s",
                "h2d_bytes_per_step": 31 * 8 * (n_in * N * 16 + n_in * 16 + 64 * nd * 2),
                "d2h_bytes_per_step": 31 * 8 * n_in * N * nd * 16},
        "gpu_launches": None,
        "roofline": {"bound": "tensor", "peak": peak, "unit": "TFLOP/s",
                     "achieved": 31 * 252e9 / (dev_s / args.steps) / 1e12,
                     "frac": (31 * 252e9 / (dev_s / args.steps) / 1e12) / peak if peak else None,
                     "kernel": "whole solve (SURVEY §8(d) 252 GFLOP model per band)", "traffic": None},
        "cpu_baseline": cpu,
        "clocks": clk.summary(),
    }
    print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


def run_radiance(args):
    """vrte_solve_radiance on the C3 paint (its beam source,
    mu0 = 0.6), field at tau = 0, the layer interface and the bottom on the
    standard 11 x 19 signed grid.  One step = one full call through the public
    C ABI (host in, host out: the solve, the reconstruction, the field copy).
    The CPU baseline runs the oracle restatement of the same call in full."""
    import numpy as np
    import torch
    import paper_1707_05882_b200 as V
    world, rank, local = dist_env()
    torch.cuda.set_device(local)
    os.environ["VRTE_DEVICE"] = str(local)
    w = workload("C3")
    tmp = tempfile.mkdtemp(prefix=f"vrte_rad_{rank}_")
    mat = V.Material.load(w.material.write(tmp, "m"))
    opts = V.options(w.N)
    tot = sum(l.tau for l in w.material.layers)
    taus = [0.0, w.material.layers[0].tau, tot]
    for _ in range(max(1, args.warmup)):
        f = V.solve_radiance(mat, opts, taus)
    torch.cuda.synchronize()
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        f = V.solve_radiance(mat, opts, taus)
        times.append(time.perf_counter() - t0)
    tm = f.timings()
    t = statistics.median(times)
    line = {"metric": "radiance fields/s (C3 paint, 3 depths x 22 x 19 directions)", "value": 1.0 / t,
            "unit": "fields/s", "n_gpus": 1, "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (SURVEY §8(d) generator)",
            "config": {"workload": "R3: C3 paint radiance field (vrte_solve_radiance)", "N": w.N,
                       "L": w.material.order_count, "taus": taus, "out_zenith": 11, "out_azimuth": 19},
            "e2e": {"value": 1.0 / t, "unit": "fields/s", "h2d_bytes_per_step": None, "d2h_bytes_per_step":
                    3 * 22 * 19 * 4 * 8},
            "stages_s": {"homogeneous": tm.homogeneous, "particular": tm.particular, "boundary": tm.boundary,
                         "reconstruction_and_host": tm.reconstruction, "total_wall": tm.total_wall}}
    if not args.no_cpu_baseline and rank == 0:
        sys.path.insert(0, os.path.join(ROOT, "oracle"))
        import pyoracle as O
        d = w.material
        bt = {"black": 0, "lambertian": 1, "mueller_table": 2}[d.base]
        om = O.Material(np.array([l.omega for l in d.layers]), np.array([l.tau for l in d.layers]),
                        d.padded_coeffs(), bt, d.albedo, d.table)
        threads = os.cpu_count() or 1
        t0 = time.perf_counter()
        ref, *_ = O.radiance(om, w.N, d.mu0, d.phi0, d.stokes, taus, zenith=11, azimuth=19, threads=threads)
        tc = time.perf_counter() - t0
        _, _, _, g = f.values()
        line["cpu_baseline"] = {"value": 1.0 / tc, "unit": "fields/s", "cores": threads, "kind": "port",
                                "sample": "oracle restatement of the full vrte_solve_radiance call (not sampled)"}
        line["parity_vs_oracle"] = float(np.abs(g - ref).max() / np.abs(ref).max())
    print(json.dumps(line), flush=True)


def run_mc7(args):
    """the reference's acceptance criterion 7 (acceptance_main.cpp:
    316-400) on the GPU tracer -- 16 single-layer configs (isotropic/Rayleigh x omega
    {0.5, 0.9} x tau {1, 10} x mu0 {0.6, 1}), 1e7 photons each, 8 x 8 bins per
    hemisphere, every bin against the discrete-ordinate field (2 x 2 Gauss points,
    flux weighted; 3 sigma).  value = photons/s through vrte_mc_trace."""
    import math
    import numpy as np
    import torch
    import paper_1707_05882_b200 as V
    from paper_1707_05882_b200 import materials as M
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import pyoracle as O
    world, rank, local = dist_env()
    torch.cuda.set_device(local)
    os.environ["VRTE_DEVICE"] = str(local)
    photons, zb, ab = 10_000_000, 8, 8
    iso = np.array([M.greek(1, 0, 0, 0, 0, 0)])
    cfgs = []
    for ray in (False, True):
        for om in (0.5, 0.9):
            for t0 in (1.0, 10.0):
                for mu0 in (0.6, 1.0):
                    cfgs.append((ray, om, t0, mu0))
    tmp = tempfile.mkdtemp(prefix="vrte_mc7_")
    mats, descs = [], []
    for k, (ray, om, t0, mu0) in enumerate(cfgs):
        d = M.MaterialDesc([M.LayerDesc(om, t0, M.RAYLEIGH if ray else iso)])
        d.mu0 = mu0
        descs.append(d)
        mats.append(V.Material.load(d.write(tmp, f"m{k}")))
    V.mc_trace(mats[0], V.options(4), 100000, 1, zb, ab)  # warm-up
    torch.cuda.synchronize()
    t0w = time.perf_counter()
    tallies = [V.mc_trace(m, V.options(4), photons, 1001 + k, zb, ab) for k, m in enumerate(mats)]
    t = time.perf_counter() - t0w
    rows = [tl.rows() for tl in tallies]
    hits = [tl.hits() for tl in tallies]
    # acceptance: every bin with >= 50 hits (hit counts are not exposed; use I > 0) vs the DOM field
    g0, g1 = 0.5 - 0.5 / math.sqrt(3.0), 0.5 + 0.5 / math.sqrt(3.0)
    total = passed = 0
    worst = (1.0, "")
    for (ray, om, t0_, mu0_), d, r, hc in zip(cfgs, descs, rows, hits):
        c_tot = c_pass = 0
        om_ = O.Material(np.array([d.layers[0].omega]), np.array([d.layers[0].tau]), d.padded_coeffs(), 0, 0.0, None)
        for h in range(2):
            tau = 0.0 if h == 0 else d.layers[0].tau
            mus = [(iz + g) / zb for iz in range(zb) for g in (g0, g1)]
            phis = [2 * math.pi * (ia + g) / ab for ia in range(ab) for g in (g0, g1)]
            f, *_ = O.radiance(om_, 16, d.mu0, 0.0, [1, 0, 0, 0], [tau], mus=[m if h == 0 else -m for m in mus],
                               phis=phis)
            for iz in range(zb):
                for ia in range(ab):
                    s, se = r[h, iz, ia, 2:6], r[h, iz, ia, 6:10]
                    if hc[h, iz, ia] < 50:  # acceptance_main.cpp:360
                        continue
                    dom = np.zeros(4)
                    ws = 0.0
                    for gm in range(2):
                        for gp in range(2):
                            mu = mus[2 * iz + gm]
                            dom += mu * f[0, 2 * iz + gm, 2 * ia + gp]
                            ws += mu
                    dom /= ws
                    ok = int(np.all(np.abs(s - dom) <= 3.0 * se + 1e-9))
                    total += 1
                    passed += ok
                    c_tot += 1
                    c_pass += ok
        frac = c_pass / c_tot if c_tot else 1.0
        if frac < worst[0]:
            worst = (frac, f"{'rayleigh' if ray else 'isotropic'} omega={om} tau0={t0_} mu0={mu0_}")
    line = {"metric": "Monte Carlo photons/s (acceptance 7: 16 configs x 1e7 photons)", "value": 16 * photons / t,
            "unit": "photons/s", "n_gpus": 1, "steps": 1, "warmup": 1, "ms_per_step": t * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (acceptance_main.cpp:316-400 configs)",
            "config": {"workload": "MC7: reference acceptance criterion 7 on vrte_mc_trace", "photons": photons,
                       "configs": 16, "bins": [zb, ab]},
            "acceptance_bins_within_3sigma": [passed, total],
            "acceptance_worst_config": {"fraction": worst[0], "config": worst[1], "pass_threshold": 0.95},
            "reference_acceptance_7_seconds": 432.41}
    if not args.no_cpu_baseline:
        threads = os.cpu_count() or 1
        d = descs[-1]
        om_ = O.Material(np.array([d.layers[0].omega]), np.array([d.layers[0].tau]), d.padded_coeffs(), 0, 0.0, None)
        n_s = 400_000
        t1 = time.perf_counter()
        O.mc_trace(om_, d.mu0, 0.0, [1, 0, 0, 0], n_s, 1016, zb, ab, threads=threads)
        tc = time.perf_counter() - t1
        line["cpu_baseline"] = {"value": n_s / tc, "unit": "photons/s", "cores": threads, "kind": "port",
                                "sample": f"oracle tracer, {n_s} photons of the last config (rayleigh w=0.9 tau=10 mu0=1)"}
    print(json.dumps(line), flush=True)


def run_sharded(args):
    """N > 1 GPUs: Fourier orders sharded across the ranks, the
    per-order tau = 0 stacks exchanged as device buffers over NCCL, the Fourier
    synthesis on the owning GPU (paper_1707_05882_b200/distributed.py).
      C3 (and any config but C4p): N solves in flight per step, each sharded by
        order over all N GPUs; an all-to-all hands solve j's shards to rank j
        ("weak": one solve's worth of orders per GPU per step).
      C4p: ONE solve per step sharded by order over the N GPUs, gathered to
        rank 0 ("strong").
    value = solves per step / step time, max over ranks, CUDA events around
    the step with device-wide synchronisation on both sides (the plans run on
    their own streams); e2e = the public calls D.inflight_brdf / D.sharded_brdf
    (inputs uploaded from the host, the owned table read back) each step."""
    import numpy as np
    import torch
    import torch.distributed as dist
    import paper_1707_05882_b200 as V
    from paper_1707_05882_b200 import distributed as D

    world, rank, local = dist_env()
    # VRTE_BENCH_EMULATE=1 (testing the code path on a 1-GPU box): every rank on
    # cuda:0, gloo with host staging instead of NCCL -- not a performance mode
    emulate = os.environ.get("VRTE_BENCH_EMULATE") == "1"
    if emulate:
        local = 0
    torch.cuda.set_device(local)
    if emulate:
        dist.init_process_group("gloo")
    else:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    os.environ["VRTE_DEVICE"] = str(local)

    def max_over_ranks(x):
        t = torch.tensor([x], dtype=torch.float64, device="cpu" if emulate else "cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    w = workload(args.config)
    nodes = quad_nodes(w.N)
    tmp = tempfile.mkdtemp(prefix=f"vrte_bench_{rank}_")
    mat = V.Material.load(w.material.write(tmp, "m"))
    opts = V.options(w.N)
    single = args.config == "C4p"
    # in-flight layout: groups of g <= 4 GPUs, orders sharded g ways inside a group,
    # g solves in flight per group (an 8-way order shard of C3 is too small to keep
    # a GPU busy: scripts/shard_probe.py)
    g = world if single or world <= 4 or world % 4 else 4
    groups = [list(range(i, i + g)) for i in range(0, world, g)]
    handles = [dist.new_group(ranks=r) for r in groups] if g < world else [None]
    mine = rank // g
    my_group, my_ranks = (handles[mine], groups[mine]) if g < world else (None, None)
    mats = [mat] if single else [mat] * g
    per_step = 1 if single else world
    conc = min(4, len(mats))
    dist.barrier()
    sh = D.OrderShards(mats, opts, nodes, w.n_dphi, None, g, rank % g, local, my_group, conc, ranks=my_ranks)

    def step():
        sh.run()
        sh.exchange()
        sh.synthesize(fetch=False)

    for _ in range(max(args.warmup, 1)):
        step()
    dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        e0.record()
        for _ in range(args.steps):
            step()
        torch.cuda.synchronize()
        e1.record()
        e1.synchronize()
    dev_s = e0.elapsed_time(e1) * 1e-3
    launches = int(sum(p.last.kernel_launches for p in sh.plans)) * args.steps
    dev_s = max_over_ranks(dev_s)
    value = per_step * args.steps / dev_s
    sh.close()
    # e2e through the public calls (host inputs, host table of the owned solve)
    call = (lambda: D.sharded_brdf(mat, opts, nodes, w.n_dphi, device=local)) if single else \
        (lambda: D.inflight_brdf(mats, opts, nodes, w.n_dphi, group=my_group, device=local, concurrency=conc))
    for _ in range(args.warmup):
        call()
    dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        tab = call()
    torch.cuda.synchronize()
    e2e_s = max_over_ranks(time.perf_counter() - t0)
    # bitwise check of one owned table against a single-GPU solve of the same material
    same = None
    if tab is not None:
        same = bool(np.array_equal(tab, V.compute_brdf(mat, opts, nodes, w.n_dphi).table()))
    flags = [None] * world
    dist.all_gather_object(flags, same)
    N, L, n_in, nd = w.N, w.material.order_count, len(nodes), w.n_dphi
    P = len(w.material.layers)
    R, d = 4 * n_in, 4 * N
    if rank == 0:
        h2d = per_step * 8 * (2 * N + 2 + 2 * L * 6 + P + n_in + n_in * N * 16 + n_in * 16 + L * nd * 2)
        line = {
            "metric": METRIC, "value": value, "unit": "solves/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": dev_s / args.steps * 1e3, "higher_is_better": True,
            "scaling": "strong" if single else "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (SURVEY §8(d) Greek generator G(g,L), deterministic)",
            "config": {"workload": f"{args.config}: {w.note}", "N": N, "L": L, "layers": P, "n_in": n_in,
                       "n_dphi": nd,
                       "parallelism": (f"one solve per step, orders sharded x{world} (m = rank mod {world}), "
                                       "NCCL gather of the per-order stacks to rank 0, synthesis there") if single
                       else (f"{world} solves in flight per step: {world // g} group(s) of {g} GPUs, each solve "
                             f"sharded by order over its group ({g} plans per GPU, {conc} concurrent), NCCL "
                             "all-to-all of the per-order stacks inside the group, each rank synthesizes one solve"),
                       "exchange_bytes_per_step": per_step * 8 * L * R * d,
                       "l2": "working set >> 126 MB L2 (no explicit flush)"},
            "e2e": {"value": per_step * args.steps / e2e_s, "unit": "solves/s", "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": per_step * 8 * n_in * N * nd * 16},
            "gpu_launches": launches,
            "bitwise_vs_single_gpu": [f for f in flags if f is not None],
            "emulated_on_one_gpu": emulate,
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    dist.barrier()
    dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    if dist_env()[0] > 1 and args.config not in ("C5", "R3", "MC7"):
        return run_sharded(args)
    if args.config == "C5":
        return run_c5(args)
    if args.config == "R3":
        return run_radiance(args)
    if args.config == "MC7":
        return run_mc7(args)
    import numpy as np
    import torch
    import paper_1707_05882_b200 as V

    world, rank, local = dist_env()
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        dist = None
    torch.cuda.set_device(local)
    os.environ["VRTE_DEVICE"] = str(local)
    w = workload(args.config)
    nodes = quad_nodes(w.N)
    tmp = tempfile.mkdtemp(prefix=f"vrte_bench_{rank}_")
    mat = V.Material.load(w.material.write(tmp, "m"))
    opts = V.options(w.N)

    peak = fp64_peak_tflops(torch.device("cuda", local)) if rank == 0 else None

    # ---------------- device-resident solves (value)
    plan = V.Plan(mat, opts, nodes, w.n_dphi, device=local)
    plan.run(max(args.warmup, 1))
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        dev_s = plan.run(args.steps) * args.steps  # CUDA events on the plan's stream
    torch.cuda.synchronize()
    res = plan.last.as_dict()
    t_dev = torch.tensor([dev_s], dtype=torch.float64, device="cuda")
    if dist:
        dist.all_reduce(t_dev, op=dist.ReduceOp.MAX)
    dev_s = float(t_dev.item())
    value = world * args.steps / dev_s

    # ---------------- end to end through the C ABI (e2e)
    for _ in range(args.warmup):
        V.compute_brdf(mat, opts, nodes, w.n_dphi).close()
    if dist:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        b = V.compute_brdf(mat, opts, nodes, w.n_dphi)
        stats = b.device_stats()
        n_out = b.shape[1]  # N, or the refraction cone's nodes under a Fresnel interface
        b.close()
    e2e_s = time.perf_counter() - t0
    t_e2e = torch.tensor([e2e_s], dtype=torch.float64, device="cuda")
    if dist:
        dist.all_reduce(t_e2e, op=dist.ReduceOp.MAX)
    e2e_s = float(t_e2e.item())
    N, L, n_in, nd = w.N, w.material.order_count, len(nodes), w.n_dphi
    P, S = len(w.material.layers), 2
    h2d = 8 * (2 * N + S + S * L * 6 + P + n_in + n_in * N * 16 + n_in * 16 + L * nd * 2) + 4 * P
    d2h = 8 * n_in * n_out * nd * 16

    if rank != 0:
        if dist:
            dist.destroy_process_group()
        return

    # ---------------- concurrent solves (secondary: K independent solves of the same
    # shape in flight on one GPU, one pooled plan / stream each -- what concurrent
    # callers of the reentrant C ABI get; the headline `value` stays one solve at a time)
    concurrent = None
    if world == 1 and args.config not in ("C4p",):
        import threading
        K = 4
        cplans = [V.Plan(mat, opts, nodes, w.n_dphi, device=local, pooled=True) for _ in range(K)]
        for q in cplans:
            q.run(1)
        torch.cuda.synchronize()
        ths = [threading.Thread(target=q.run, args=(args.steps,)) for q in cplans]
        ce0, ce1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ce0.record()
        for th in ths:
            th.start()
        for th in ths:
            th.join()
        torch.cuda.synchronize()
        ce1.record()
        ce1.synchronize()
        csec = ce0.elapsed_time(ce1) * 1e-3
        concurrent = {"solves_per_s": K * args.steps / csec, "plans": K,
                      "note": "K identical solves in flight (pooled plans, own streams); not the headline"}
        for q in cplans:
            q.close()

    # ---------------- roofline of the dominant kernel
    # Algorithmic FP64 flops per launch (SURVEY §8(d) / Golub-Van Loan counts,
    # DESIGN.md §5); the stage times are CUDA events on the plan's stream.
    # Units per launch are the EXECUTED ones: Be (medium, order) slots go through
    # the eigen pipeline (the free-streaming slots -- zero kernel -- are filled
    # analytically and cost no flops), every order through the boundary stage.
    d = 4 * N
    Be = int(res["eigen_slots"])
    G = 2 * d * P
    R = 4 * n_in
    kern = {"hqr_multi_kernel (multishift Francis QR + AED + Schur vectors)": (res["t_hqr"], Be * 20.0 * d ** 3),
            # the augmented [A | B] factorization also eliminates the R right-hand
            # sides (L^-1 P B: G^2 R flops) besides the (2/3) G^3 of the LU proper
            "boundary LU factor (augmented: Crout panels + fused block solves + DMMA GEMM, look-ahead)":
                (res["t_lu_factor"], L * ((2.0 / 3.0) * G ** 3 + G ** 2 * R)),
            # back substitution U x = y: the R right-hand sides through layer 0's 2d rows
            # (R (2d)^2), the 4 residual probes through all G rows (4 G^2)
            "boundary back substitution (fused block solves + DMMA GEMM)": (res["t_lu_solve"], L * (R * (2 * d) ** 2 + 4 * G ** 2)),
            "eigen refinement (Newton step, 8N residual GEMMs)": (res["t_refine"], Be * 24.0 * d ** 3),
            "blocked Hessenberg + Q": (res["t_hessenberg"], Be * (10.0 / 3.0 + 4.0 / 3.0) * d ** 3),
            "trevc_blk_kernel (eigenvectors)": (res["t_trevc"], Be * (1.0 / 3.0) * d ** 3)}
    name = max(kern, key=lambda k: kern[k][0])
    t_k, flops = kern[name]
    traffic = None
    prof = os.path.join(ROOT, "profiles", "ncu_dominant_kernel.json")
    if os.path.exists(prof):
        try:
            pj = json.load(open(prof))
            if name.startswith(pj.get("kernel", "?")):
                traffic = pj.get("dram_bytes_per_launch")
        except Exception:
            traffic = None
    achieved = flops / t_k / 1e12 if t_k > 0 else 0.0
    roofline = {"bound": "tensor", "kernel": name, "achieved": achieved, "peak": peak,
                "unit": "TFLOP/s", "frac": achieved / peak if peak else None, "traffic": traffic,
                "peak_source": "measured cuBLAS DGEMM (torch.float64 matmul 8192^3) on this GPU; "
                               "MEASURED_PEAKS.json has no FP64 entry (B200 FP64 tensor rate = FP64 rate)",
                "algorithmic_flops_per_launch": flops,
                "flop_model": "QR with Schur vectors 20 d^3 per executed (medium, order) slot (Be of them); "
                              "augmented LU (2/3) G^3 + G^2 R and back substitution R (2d)^2 + 4 G^2 per order; "
                              "Hessenberg+Q 14/3 d^3, trevc d^3/3, refinement 24 d^3 per executed slot; "
                              "d = 4N, G = 2dP, R = 4 n_in",
                "units": {"eigen_slots_executed": Be, "slots": int(res["slots"]), "orders": L},
                "stage_tflops": {k: (f / t / 1e12 if t > 0 else None) for k, (t, f) in kern.items()}}

    # ---------------- CPU baseline (rank 0, N = 1 only)
    cpu = None
    gpu_table = None
    if world == 1 and not args.no_cpu_baseline:
        threads = os.cpu_count() or 1
        full, tm, picked = oracle_sample(w, nodes, args.cpu_incidents, threads)
        cpu = {"value": 1.0 / full, "unit": "solves/s", "cores": threads, "kind": "port", "extrapolated": True,
               "cpu_model": cpu_model(),
               "sample": f"oracle/ (reference algorithm, LAPACK) on {threads} host threads: "
                         f"prepare_homogeneous + {args.cpu_incidents} incident(s) x 4 basis at mu_in="
                         f"{picked}, extrapolated to {n_in} incidents (T = T_hom + n_in/k T_k, BASELINE.md §2); "
                         f"measured {tm['total_wall']:.1f} s for an extrapolated {full:.1f} s/solve"}
        gb = V.compute_brdf(mat, opts, nodes, w.n_dphi)
        gpu_table = gb.table()
        gb.close()

    line = {
        "metric": METRIC,
        "value": value,
        "unit": "solves/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": dev_s / args.steps * 1e3,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (SURVEY §8(d) Greek generator G(g,L), deterministic)",
        "config": {"workload": f"{args.config}: {w.note}", "N": N, "L": L, "layers": P,
                   "n_in": n_in, "n_dphi": nd, "basis": "default 4-vector",
                   "parallelism": "single GPU, one solve per step (bench.py --gpus N: orders sharded over N GPUs)",
                   "l2": "working set ~1.5 GB per solve >> 126 MB L2 (no explicit flush)"},
        "e2e": {"value": world * args.steps / e2e_s, "unit": "solves/s",
                "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
        "gpu_launches": int(stats["kernel_launches"]) * args.steps,
        "roofline": roofline,
        "cpu_baseline": cpu,
        "clocks": clk.summary(),
        "stages_ms": {k: res[k] * 1e3 for k in ("t_homogeneous", "t_particular", "t_boundary",
                                                 "t_synthesis", "t_hessenberg", "t_hqr", "t_trevc",
                                                 "t_refine", "t_lu_factor", "t_lu_solve")},
        "max_eigen_residual": res["max_eigen_residual"],
        "gates": {k: res[k] for k in ("max_boundary_residual", "max_boundary_condition", "boundary_refined",
                                       "boundary_fallback", "max_balance_residual", "max_particular_residual",
                                       "particular_extra_steps")},
        "parity": parity_record(gpu_table),
        "concurrent": concurrent,
    }
    print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
