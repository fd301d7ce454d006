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

    def _nvml_loop(self):
        """In-process NVML queries (no nvidia-smi process per sample: spawning one
        every 0.2 s competed with the host-side syncs of the setup stages)."""
        import pynvml as nv
        nv.nvmlInit()
        try:
            h = nv.nvmlDeviceGetHandleByIndex(self.index)
            smax = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
            bits = [nv.nvmlClocksEventReasonHwSlowdown, nv.nvmlClocksEventReasonHwThermalSlowdown,
                    nv.nvmlClocksEventReasonSwThermalSlowdown, nv.nvmlClocksEventReasonSwPowerCap]
            while not self._stop.is_set():
                sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
                pw = nv.nvmlDeviceGetPowerUsage(h) / 1000.0
                rs = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                self.samples.append([str(sm), str(smax), f"{pw:.1f}", hex(rs)] +
                                    ["Active" if rs & b else "Not Active" for b in bits])
                self._stop.wait(0.2)
        finally:
            nv.nvmlShutdown()

    def _run(self):
        try:
            self._nvml_loop()
            return
        except Exception:
            self.samples = []
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
def cpu_sample(cfgname, n_full, k, tol, iters_full, sample_n, eps_iters=5, lob_iters=2,
               seed=42):
    """Oracle port (numpy/scipy restatement of the reference, oracle/) on a
    bounded sample of the config family, stage by stage; the full embedding is
    extrapolated linearly in N from the sample and to the reference's 60-
    iteration eps solve and the GPU-measured main-solve iteration count:

        est = (N / n_s) * (setup + eps_init + 60 * eps_iter + lob_init + iters * lob_iter)

    Returns (estimated seconds per full embedding, detail dict)."""
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
    eit = []
    t0 = time.perf_counter()
    tau = 1e-8 * float(q.diagonal().sum()) / n
    res = O.lobpcg(q, np.ones(n), 8, tol=1e-6, max_iter=eps_iters, seed=seed,
                   deflate=np.full(n, 1 / np.sqrt(n)), iter_times=eit)
    t_eps_run = time.perf_counter() - t0
    ev = res["eigenvalues"]
    eps = float(ev[ev > tau][0]) if np.any(ev > tau) else 0.0  # (timing only)
    eps_iter = float(np.mean(eit)) if eit else 0.0
    eps_init = t_eps_run - float(np.sum(eit))
    t0 = time.perf_counter()
    mu = O.repulsion_weight(l, q, eps)
    a = O.assemble(l, q, mu, eps)
    b, _ = O.degree_balancing(a)
    t_setup2 = time.perf_counter() - t0
    lit = []
    t0 = time.perf_counter()
    O.lobpcg(a, b, k + 1, tol=tol, max_iter=lob_iters, seed=seed, iter_times=lit)
    t_lob_run = time.perf_counter() - t0
    lob_iter = float(np.mean(lit)) if lit else 0.0
    lob_init = t_lob_run - float(np.sum(lit))
    scale = n_full / n
    sample_s = t_setup1 + t_setup2 + eps_init + 60 * eps_iter + lob_init + iters_full * lob_iter
    est = scale * sample_s
    detail = {"sample_n": n, "setup_s": t_setup1 + t_setup2, "eps_init_s": eps_init,
              "eps_s_per_iter": eps_iter, "eps_iters_timed": len(eit), "lobpcg_init_s": lob_init,
              "lobpcg_s_per_iter": lob_iter, "lobpcg_iters_timed": len(lit), "graph_s": t_graph,
              "scale": scale, "iterations_extrapolated": iters_full,
              "sample_embedding_s": sample_s}
    return est, detail


def host_info():
    ram_gb = None
    try:
        with open("/proc/meminfo") as fh:
            for line in fh:
                if line.startswith("MemTotal:"):
                    ram_gb = round(int(line.split()[1]) / 1024 / 1024, 1)
    except OSError:
        pass
    return {"os_cpu_count": os.cpu_count(), "blas_threads": blas_threads(), "ram_gb": ram_gb}


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


def bench_config(cfg, n_full, world):
    """The workload identity, shared by both arms (run-specific numbers go in ``run``)."""
    return {"workload": cfg.name, "description": cfg.description, "n": n_full, "K": cfg.k,
            "block": cfg.k + 1, "tol": cfg.tol, "max_iter": cfg.max_iter,
            "parallelism": f"rows{world} (1-D row partition, NCCL halo + Gram allreduce)"
            if world > 1 else "single",
            "l2": "inputs larger than L2 (126 MB)" if n_full >= 1_000_000 else "L2-resident"}


def run_reference(args, cfg, n_full):
    """Reference arm: the oracle port on the box's host cores (rank 0 only).

    The first warm-up step measures the port stage by stage on a calibration
    sample of min(N, 1M) nodes (the anchor of the extrapolation).  Every step
    (warm-up and timed) then re-times a small sample (50K nodes, ~5 s) of the
    same stages; a timed step's value is the 1M-anchored estimate scaled by that
    step's small-sample time over the small-sample time measured next to the
    anchor -- so run-to-run variation of the host is tracked without re-running
    the 1M sample every step."""
    world, rank, _ = dist_setup()
    if rank != 0:
        return
    iters = known_iterations(cfg.name, n_full)
    cal_n = args.cpu_sample_n or min(n_full, 1_000_000)
    small_n = min(cal_n, 50_000)
    est_cal, det_cal = cpu_sample(cfg.name, n_full, cfg.k, cfg.tol, iters, cal_n)
    _, det_small0 = cpu_sample(cfg.name, n_full, cfg.k, cfg.tol, iters, small_n, 3, 1)
    ref_small = det_small0["sample_embedding_s"] / small_n
    times, smalls = [], []
    for step in range(args.warmup + args.steps):
        _, d = cpu_sample(cfg.name, n_full, cfg.k, cfg.tol, iters, small_n, 3, 1)
        if step >= args.warmup:
            smalls.append(d["sample_embedding_s"])
            times.append(est_cal * (d["sample_embedding_s"] / small_n) / ref_small)
    v = float(np.mean(times))
    hi = host_info()
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": v * 1e3,
            "higher_is_better": False, "scaling": "strong", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic",
            "config": bench_config(cfg, n_full, world),
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": hi["blas_threads"],
                             "kind": "port", "extrapolated": True,
                             "sample": f"EXTRAPOLATED: oracle port (numpy/scipy restatement of "
                                       f"manigraph, fp64) timed stage by stage on {cal_n} nodes "
                                       f"of {cfg.name} (setup, eps init + {det_cal['eps_iters_timed']}"
                                       f" timed eps iterations -> 60, LOBPCG init + "
                                       f"{det_cal['lobpcg_iters_timed']} timed iterations -> {iters}),"
                                       f" scaled linearly to N={n_full}; each step re-times a "
                                       f"{small_n}-node sample to track host variation",
                             "host": hi, "calibration": det_cal,
                             "small_sample_s_per_step": smalls},
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
    # per-kernel rooflines of the three hot kernels (C5: fp32, m = K + 1, mp = m
    # padded to 4, w = 3 mp).  SpMM: HBM (SURVEY 8(d) bytes); update: FP32 FMA
    # pipe (2 * (w*mp + mp*mp) * 2 flop per row, measured 72.56 TFLOP/s,
    # profiles/r2_fp32_peak.json) and HBM (10 m s_v N); Gram: tensor pipe
    # (3xTF32 products over the 128 x 128 padded tile, 2 Grams; TF32 dense peak
    # = bf16 / 2) and HBM (6 m s_v N)
    m_blk = K + 1
    mp_blk = (m_blk + 3) // 4 * 4
    w_blk = 3 * mp_blk
    rl = {}
    tc_gram = prec == "fp32" and 48 < w_blk <= 128  # k_gram_tc2 (else the CUDA-core k_gram2)
    for kname in ("update", "gram") if prec == "fp32" else ():
        if kname == "gram" and not tc_gram:
            continue
        if kname in st and st[kname]["launches"]:
            avg_s = st[kname]["ms"] / st[kname]["launches"] / 1e3
            if kname == "update":
                tc_upd = w_blk > int(os.environ.get("MG_UPD_TC", "96")) > 0 and mp_blk in (12, 20, 36)
                if tc_upd:
                    # k_update_tc3: 2 TF32 MMAs (hi, lo rows) per k-step, M padded to
                    # 128 output columns, K = w rounded to 8, both S and AS; HBM:
                    # SURVEY 8(d) 10 m s_v N
                    kpad = (w_blk + 7) // 8 * 8
                    flops = 2.0 * 2 * 2 * 128 * kpad * n
                    gbs = 10 * m_blk * 4 * n / avg_s / 1e9
                    rl["update"] = {"kernel": "k_update_tc3 (tcgen05)", "bound": "hbm",
                                    "achieved": gbs, "peak": hbm, "unit": "GB/s", "frac": gbs / hbm,
                                    "tensor_frac": flops / avg_s / 1e12 / (bf16 / 2),
                                    "note": "class average incl. the CUDA-core launches of safe-mode / "
                                            "narrow solves"}
                else:
                    flops = 2.0 * (w_blk * mp_blk + mp_blk * mp_blk) * 2 * n
                    rl["update"] = {"kernel": "k_update_ws", "bound": "fp32-fma",
                                    "achieved": flops / avg_s / 1e12,
                                    "peak": 72.56, "unit": "TFLOP/s",
                                    "frac": flops / avg_s / 1e12 / 72.56,
                                    "hbm_frac": 10 * m_blk * 4 * n / avg_s / 1e9 / hbm}
            else:
                # class average over the narrow launches (W-column blocks: S, the W
                # block of AS and b are read: (w + mp) s_v N) and the full pair
                # every refresh (SURVEY 8(d) 6 m s_v N); bytes as each launch recorded
                gbs = st[kname]["bytes"] / (st[kname]["ms"] / 1e3) / 1e9
                flops = 2.0 * 2 * 3 * 128 * 128 * n
                rl["gram"] = {"kernel": "k_gram_tc2 (tcgen05; narrow + derived [X P] blocks, "
                                        "full pair at refreshes)", "bound": "hbm",
                              "achieved": gbs, "peak": hbm, "unit": "GB/s", "frac": gbs / hbm,
                              "full_pair_tensor_frac_if_all_full": flops / avg_s / 1e12 / (bf16 / 2)}
    kern = {k: {"launches": v["launches"], "ms_per_step": v["ms"] / args.steps,
                "avg_us": 1e3 * v["ms"] / max(v["launches"], 1),
                "GB_per_s": (v["bytes"] / (v["ms"] / 1e3) / 1e9) if v["ms"] > 0 else None}
            for k, v in st.items() if v["launches"]}
    line = {
        "metric": METRIC, "value": t_max, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": t_max * 1e3, "higher_is_better": False,
        "scaling": "strong", "vs_baseline": None,
        "dtype": "f32" if prec == "fp32" else "f64", "data": "synthetic",
        "config": bench_config(cfg, n, world),
        "run": {"graph_nnz": int(idx.size), "precision": prec, "max_iter": max_iter,
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
        "rooflines_other": rl,
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
        # bounded (~10-30 s of CPU work): a 100K-node sample of the same stages
        sample_n = args.cpu_sample_n or min(n, 100_000)
        est, detail = cpu_sample(cfg.name, n, K, cfg.tol, int(res.iterations), sample_n)
        line["cpu_baseline"] = {
            "value": est, "unit": UNIT, "cores": blas_threads(), "kind": "port",
            "extrapolated": True, "host": host_info(),
            "sample": f"EXTRAPOLATED: oracle port on {detail['sample_n']} nodes of {cfg.name}: "
                      f"setup, eps init + {detail['eps_iters_timed']} timed iterations (-> 60), "
                      f"LOBPCG init + {detail['lobpcg_iters_timed']} timed iterations (-> the "
                      f"{int(res.iterations)} the GPU needed), scaled linearly to N={n}",
            "detail": detail}
    print(json.dumps(line), flush=True)
    if comm is not None:
        comm.close()
    if world > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
