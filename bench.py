"""Benchmark: manigraph embedding wall time on B200 (BASELINE.json metric).

One "step" = one full embed() of the config graph -- components check, L,
two-hop sets, Q, eps (deflated 60-iteration LOBPCG on Q), mu, A, b, and the
K+1-pair LOBPCG to convergence -- with inputs resident in HBM (``value``),
and once more through the public API with host buffers (``e2e``).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c5] [--n N]
    python bench.py --impl reference ...   # CPU oracle port of the reference path

Multi-GPU (torchrun, one rank per GPU): ONE embed of the config graph with
the LOBPCG solve row-partitioned over the N GPUs (setup replicated, NCCL halo
exchange + Gram allreduce; dist.py / DESIGN.md 8(e)) -- strong scaling;
value = per-embedding wall time, max over ranks.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "embedding wall time (s) and SpMM HBM GB/s at N=1M-20M, K=8-32, 1/2/4/8 GPUs"
UNIT = "s"
ITER_FILE = os.path.join(ROOT, "profiles", "iterations.json")


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), float(d["bf16_tflops"]), "measured"
    return 6650.0, 1590.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks/throttle sampling during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(
                    ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                     "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                if out.returncode == 0 and out.stdout.strip():
                    self.samples.append([x.strip() for x in out.stdout.strip().split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no-samples"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        smax = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for s in self.samples:
            for nm, v in zip(names, s[4:8]):
                if v.strip().lower() == "active":
                    reasons.add(nm)
        loaded = [v for v in sm if smax and v > 0.5 * max(smax)] or sm
        return {"sm_mhz": float(np.median(loaded)) if loaded else None,
                "sm_max_mhz": max(smax) if smax else None, "reasons": sorted(reasons),
                "samples": len(self.samples)}


def ncu_traffic(cfgname, n, kernel):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of ``kernel`` from the
    committed ncu --set full summary (profiles/ncu_traffic.json), when it was
    captured on this config; else None."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as fh:
            d = json.load(fh)
        e = d[f"{cfgname}_{n}"][kernel]
        return float(e["dram_bytes_per_launch"])
    except Exception:
        return None


def dist_setup():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


# ------------------------------------------------------------------ CPU arm ---
def cpu_sample(cfgname, n_full, k, tol, iters_full, sample_n, sample_iters, seed=42):
    """Oracle port on a bounded sample; per-stage times extrapolated linearly in N.

    Returns (extrapolated seconds per full embedding, detail dict)."""
    import oracle as O
    from paper_2112_07862_b200 import synthetic
    t0 = time.perf_counter()
    n, ptr, idx, w = synthetic.config_graph(cfgname, n=sample_n)
    t_graph = time.perf_counter() - t0
    t0 = time.perf_counter()
    O.components(n, ptr, idx)
    l = O.laplacian(n, ptr, idx, w)
    tp, ti = O.two_hop(n, ptr, idx)
    q = O.q_matrix(n, tp, ti)
    t_setup1 = time.perf_counter() - t0
    t0 = time.perf_counter()
    tau = 1e-8 * float(q.diagonal().sum()) / n
    res = O.lobpcg(q, np.ones(n), 8, tol=1e-6, max_iter=60, seed=seed,
                   deflate=np.full(n, 1 / np.sqrt(n)))
    ev = res["eigenvalues"]
    eps = float(ev[ev > tau][0]) if np.any(ev > tau) else 0.0
    t_eps = time.perf_counter() - t0
    t0 = time.perf_counter()
    mu = O.repulsion_weight(l, q, eps)
    a = O.assemble(l, q, mu, eps)
    b, _ = O.degree_balancing(a)
    t_setup2 = time.perf_counter() - t0
    t0 = time.perf_counter()
    r = O.lobpcg(a, b, k + 1, tol=tol, max_iter=sample_iters, seed=seed)
    t_lob = time.perf_counter() - t0
    per_iter = t_lob / max(r["iterations"], 1)
    scale = n_full / n
    est = (t_setup1 + t_eps + t_setup2) * scale + per_iter * scale * iters_full
    detail = {"sample_n": n, "sample_iters": int(r["iterations"]), "setup_s": t_setup1 + t_setup2,
              "eps_s": t_eps, "lobpcg_s_per_iter": per_iter, "graph_s": t_graph,
              "scale": scale, "iterations_extrapolated": iters_full}
    return est, detail


def blas_threads():
    try:
        from threadpoolctl import threadpool_info
        info = threadpool_info()
        return max([i.get("num_threads", 1) for i in info] or [1])
    except Exception:
        return os.cpu_count() or 1


def known_iterations(cfgname, n):
    try:
        with open(ITER_FILE) as fh:
            d = json.load(fh)
        return int(d[f"{cfgname}_{n}"])
    except Exception:
        return {"c1": 200, "c2": 1001, "c3": 977, "c4": 800, "c5": 700}.get(cfgname, 500)


def run_reference(args, cfg, n_full):
    world, rank, _ = dist_setup()
    if rank != 0:
        return
    iters = known_iterations(cfg.name, n_full)
    sample_n = args.cpu_sample_n or min(n_full, 100_000)
    times, detail = [], None
    for step in range(args.warmup + args.steps):
        est, detail = cpu_sample(cfg.name, n_full, cfg.k, cfg.tol, iters, sample_n,
                                 args.cpu_sample_iters)
        if step >= args.warmup:
            times.append(est)
    v = float(np.mean(times))
    cores = blas_threads()
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": v * 1e3,
            "higher_is_better": False, "scaling": "strong", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic",
            "config": {"workload": cfg.name, "n": n_full, "K": cfg.k, "tol": cfg.tol,
                       "precision": "fp64 (reference)"},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "port",
                             "sample": f"oracle port (numpy/scipy restatement of manigraph) on "
                                       f"{detail['sample_n']} nodes of the same config family, "
                                       f"setup+eps timed, LOBPCG {detail['sample_iters']} "
                                       f"iterations timed; extrapolated linearly to N={n_full} "
                                       f"and {iters} iterations",
                             "detail": detail},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ GPU arm ---
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    # headline: config 5 (20M nodes, K = 32), the largest single-GPU config the
    # metric is quoted on (BASELINE.json configs[4]); c1-c4 are parity cases
    ap.add_argument("--config", default=os.environ.get("MG_BENCH_CONFIG", "c5"))
    ap.add_argument("--n", type=int, default=None)
    ap.add_argument("--precision", default=None)
    ap.add_argument("--max-iter", type=int, default=None)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-sample-n", type=int, default=None)
    ap.add_argument("--cpu-sample-iters", type=int, default=8)
    args = ap.parse_args()

    from paper_2112_07862_b200 import synthetic
    cfg = synthetic.CONFIGS[args.config]
    n_full = cfg.n if args.n is None else args.n

    if args.impl == "reference":
        return run_reference(args, cfg, n_full)

    world, rank, local = dist_setup()
    device = local if world > 1 else 0
    import torch
    torch.cuda.set_device(device)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", device))

    import paper_2112_07862_b200 as mg
    from paper_2112_07862_b200 import _native as N, core
    from paper_2112_07862_b200 import dist as mgdist
    comm = mgdist.nccl_comm(rank, world, device) if world > 1 else None

    prec = args.precision or cfg.precision
    max_iter = args.max_iter or cfg.max_iter
    t0 = time.perf_counter()
    g = synthetic.config_graph(cfg.name, n=n_full)
    t_graph = time.perf_counter() - t0
    n, ptr, idx, w = g
    K = cfg.k
    scfg = mg.SolverConfig(k=K + 1, tol=cfg.tol, max_iter=max_iter, seed=42, precision=prec)
    G = mg.Graph(n, ptr, idx, w)
    # config 4 is 10 disjoint patches: embed() raises DisconnectedGraphError like
    # the reference; the config's own harness runs the pair + solve without it
    connected = cfg.name != "c4"
    zcount = core._stream_size(n, max(K + 1, 8))
    zh = np.random.default_rng(42).standard_normal(zcount)
    dd = torch.device("cuda", device)
    dev_inputs = (torch.from_numpy(np.ascontiguousarray(ptr, np.int64)).to(dd),
                  torch.from_numpy(np.ascontiguousarray(idx, np.int64)).to(dd),
                  torch.from_numpy(np.ascontiguousarray(w, np.float64)).to(dd),
                  torch.from_numpy(zh).to(dd))
    del zh
    ext = torch.cuda.ExternalStream(N.stream_handle(device), device=dd)

    def embed_dev():
        if comm is None:
            return core.embed_arrays(n, None, None, None, K, scfg, device_inputs=dev_inputs,
                                     check_connected=connected)
        return mgdist.embed_arrays_dist(comm, N.context(device), device, n, None, None, None, K,
                                        scfg, device_inputs=dev_inputs, check_connected=connected)

    def one_step():
        start = torch.cuda.Event(enable_timing=True)
        stop = torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        start.record(ext)
        res, b, dg = embed_dev()
        stop.record(ext)
        stop.synchronize()
        return start.elapsed_time(stop) / 1e3, res, dg

    for _ in range(args.warmup):
        one_step()
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    N.set_profiling(True, device)
    N.stats(device)  # clear
    l0 = N.launch_count(device)
    times, last = [], None
    with ClockSampler(device) as clk:
        for _ in range(args.steps):
            dt, res, dg = one_step()
            times.append(dt)
            last = (res, dg)
    torch.cuda.synchronize()
    launches = N.launch_count(device) - l0
    st = N.stats(device)
    N.set_profiling(False, device)
    t_local = float(np.mean(times))
    if world > 1:
        tt = torch.tensor([t_local], device=dd)
        torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
        t_max = float(tt.item())
    else:
        t_max = t_local
    res, dg = last

    # e2e through the public API with host buffers (H2D inputs + normal stream, D2H P and b)
    e2e_times = []
    for _ in range(int(os.environ.get("MG_E2E_STEPS", "1"))):
        Gh = mg.Graph(n, ptr, idx, w)
        torch.cuda.synchronize()
        if world > 1:
            torch.distributed.barrier()
        t0 = time.perf_counter()
        if comm is None:
            if connected:
                mg.embed(Gh, K, scfg, require_convergence=False)
            else:  # config 4: the reference harness path without the check
                res_h, b_h, _ = core.embed_arrays(n, ptr, idx, w, K, scfg, check_connected=False)
                res_h.eigenvectors.cpu(), b_h.cpu()
        else:
            mgdist.embed_dist(comm, Gh, K, scfg, device=device, require_convergence=False)
        torch.cuda.synchronize()
        e2e_times.append(time.perf_counter() - t0)
    if world > 1:  # job time = slowest rank
        te = torch.tensor([float(np.mean(e2e_times))], device=dd)
        torch.distributed.all_reduce(te, op=torch.distributed.ReduceOp.MAX)
        e2e_times = [float(te.item())]
    e2e = float(np.mean(e2e_times))
    # host graph arrays (int64 indptr, int64 indices, f64 weights); the initial
    # block's normal stream is generated on the device (core._normals_on) unless
    # MG_HOST_NORMALS=1 asks for the host numpy stream
    h2d = 8 * (n + 1) + 16 * int(idx.size)
    if os.environ.get("MG_HOST_NORMALS") == "1":
        h2d += 8 * zcount
    d2h = 8 * n * K + 8 * n

    if rank != 0:
        if comm is not None:
            comm.close()
        torch.distributed.destroy_process_group()
        return
    hbm, bf16, peak_src = load_peaks()
    sp = st["spmm"]
    spmm_ms = sp["ms"] / max(sp["launches"], 1)
    spmm_bytes = sp["bytes"] / max(sp["launches"], 1)
    achieved = spmm_bytes / (spmm_ms / 1e3) / 1e9 if sp["launches"] else 0.0
    kern = {k: {"launches": v["launches"], "ms_per_step": v["ms"] / args.steps,
                "avg_us": 1e3 * v["ms"] / max(v["launches"], 1),
                "GB_per_s": (v["bytes"] / (v["ms"] / 1e3) / 1e9) if v["ms"] > 0 else None}
            for k, v in st.items() if v["launches"]}
    line = {
        "metric": METRIC, "value": t_max, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": t_max * 1e3, "higher_is_better": False,
        "scaling": "strong", "vs_baseline": None,
        "dtype": "f32" if prec == "fp32" else "f64", "data": "synthetic",
        "config": {"workload": cfg.name, "description": cfg.description, "n": n,
                   "graph_nnz": int(idx.size), "K": K, "block": K + 1, "tol": cfg.tol,
                   "max_iter": max_iter, "precision": prec,
                   "parallelism": f"rows{world} (1-D row partition, NCCL halo + Gram allreduce)"
                   if world > 1 else "single",
                   "l2": "inputs larger than L2 (126 MB)" if n >= 1_000_000 else "L2-resident",
                   "iterations": int(res.iterations), "eps_iterations": int(dg.eps_iterations),
                   "A_nnz": int(dg.a_nnz), "Q_nnz": int(dg.q_nnz),
                   "seconds_setup": dg.seconds_setup, "seconds_eps": dg.seconds_eps,
                   "seconds_solve": dg.seconds_solve, "graph_build_s": t_graph},
        "roofline": {"kernel": "k_spmm (CSR x row-major block, A*W)", "bound": "hbm",
                     "achieved": achieved, "peak": hbm, "unit": "GB/s",
                     "frac": achieved / hbm if hbm else None,
                     "traffic": ncu_traffic(cfg.name, n, "k_spmm"),
                     "peak_source": peak_src,
                     "algorithmic_bytes_per_launch": spmm_bytes, "avg_launch_ms": spmm_ms},
        "kernels": kern,
        "e2e": {"value": e2e, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "note": "mg.embed(Graph(host arrays)): H2D graph, device PCG64/ziggurat normal stream, D2H P and b"},
        "gpu_launches": int(launches / max(args.steps, 1)),
        "clocks": clk.summary(),
    }
    try:
        os.makedirs(os.path.dirname(ITER_FILE), exist_ok=True)
        d = {}
        if os.path.exists(ITER_FILE):
            d = json.load(open(ITER_FILE))
        d[f"{cfg.name}_{n}"] = int(res.iterations)
        json.dump(d, open(ITER_FILE, "w"), indent=1, sort_keys=True)
    except Exception:
        pass
    if not args.no_cpu_baseline and world == 1:
        sample_n = args.cpu_sample_n or min(n, 100_000)
        est, detail = cpu_sample(cfg.name, n, K, cfg.tol, int(res.iterations), sample_n,
                                 args.cpu_sample_iters)
        line["cpu_baseline"] = {
            "value": est, "unit": UNIT, "cores": blas_threads(), "kind": "port",
            "sample": f"oracle port on {detail['sample_n']} nodes of {cfg.name}: setup + eps "
                      f"(60 it) + {detail['sample_iters']} LOBPCG iterations timed, extrapolated "
                      f"linearly to N={n} and the {int(res.iterations)} iterations the GPU needed",
            "detail": detail}
    print(json.dumps(line), flush=True)
    if comm is not None:
        comm.close()
    if world > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
