#!/usr/bin/env python
"""Benchmark of the hot path: the order-50 Jackson-Chebyshev features filter on SBM N=1e6, k=100.

Contract:
  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
One JSON line on rank 0.  A step = one features pass (filter of the d = ceil(4 ln N) = 56
signal columns with p = 50, plus row normalisation) over the BASELINE config-3 graph.
``value`` = whole-job Cheb-filter GB/s, with bytes from the SURVEY.md §8d formula
(forward recurrence, fp32 values: B_first + (p-1) B_step per filter) so every arm is
measured on the same unit of work; the kernels' own algorithmic bytes go into ``roofline``.
Multi-GPU: one process per GPU (torchrun), graph replicated, each rank filters its own
56 columns (weak scaling) and the row norms are exchanged over NCCL.
"""

from __future__ import annotations

import argparse
import gc
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "Cheb-filter SpMM GB/s (% of HBM peak); CSC wall-time, SBM N=1e6 k=100"
CONFIGS = {
    # BASELINE.json configs[2] (the metric's config); others for exploration
    "c3": dict(N=1_000_000, k=100, s=16.0, dtype="float32", label="BASELINE config 3"),
    "c2": dict(N=100_000, k=20, s=16.0, dtype="float32", label="BASELINE config 2"),
    "c1": dict(N=1_000, k=20, s=16.0, dtype="float64", label="BASELINE config 1"),
    "c4": dict(N=334_863, k=250, s=5.5, dtype="float32", label="BASELINE config 4 (DC-SBM, Pareto 2.5)", dcsbm=True),
    "c5": dict(N=16_000_000, k=500, s=16.0, dtype="float32", label="BASELINE config 5 (single-GPU replica)"),
}


def make_graph(P, cfg, device=None):
    """The config's synthetic graph (seed 0) and ground truth."""
    scfg = P.SbmConfig(num_nodes=cfg["N"], k=cfg["k"], avg_degree=cfg["s"],
                       epsilon=P.critical_epsilon(cfg["s"], cfg["k"]) / 4.0, seed=0)
    if cfg.get("dcsbm"):
        g, truth, _ = P.dcsbm_generate(scfg, device=device)
        return g, truth
    return P.sbm_generate(scfg, device=device)
P_ORDER = 50
FALLBACK_HBM = 6650.0  # B200_PROFILING.md fallback (GB/s)


def filter_bytes(N: int, nnz: int, w: int, s: int, p: int) -> float:
    """SURVEY.md §8d compulsory bytes of one order-p filter (forward recurrence)."""
    b_csr = 4.0 * (N + 1) + nnz * (4.0 + s)
    return (b_csr + 3.0 * N * w * s) + (p - 1) * (b_csr + 5.0 * N * w * s)


def _ncu_dram_pct(config: str, dtype: str):
    """ncu gpu__dram_throughput (% of ncu's peak) of the K2 launches, from profiles/ncu_traffic.json."""
    tf = ROOT / "profiles" / "ncu_traffic.json"
    if not tf.exists():
        return None
    return json.loads(tf.read_text()).get(f"{config}_{dtype}_dram_throughput_pct")


def _ncu_dram_gbs(config: str, dtype: str):
    """DRAM bytes per K2 launch / its ncu duration (dram__bytes.sum.per_second), same capture."""
    tf = ROOT / "profiles" / "ncu_traffic.json"
    if not tf.exists():
        return None
    d = json.loads(tf.read_text())
    b, us = d.get(f"{config}_{dtype}"), d.get("duration_us")
    return b / (sum(us) / len(us) * 1e-6) / 1e9 if b and us else None


def peaks():
    f = ROOT / "MEASURED_PEAKS.json"
    if f.exists():
        d = json.loads(f.read_text())
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return FALLBACK_HBM, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines: list[str] = []
        self.stamps: list[float] = []
        self.t0 = self.t1 = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())
            self.stamps.append(time.perf_counter())

    def mark(self, start: bool):
        """Bracket the timed region (samples are taken every 100 ms from __enter__ on)."""
        if start:
            self.t0 = time.perf_counter()
        else:
            self.t1 = time.perf_counter()

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.25)
            t_end = time.time() + 5.0  # at least one sample, even if the region was very short
            while not self.lines and time.time() < t_end and self.proc.poll() is None:
                time.sleep(0.05)
            self.proc.terminate()
            self.proc.wait(timeout=5)

    def summary(self):
        rows = []
        lines = list(zip(self.stamps, self.lines))
        if self.t0 is not None and self.t1 is not None and lines:
            inside = [ln for t, ln in lines if self.t0 <= t <= self.t1 + 0.1]
            # a region shorter than the 100 ms sampling period: the sample nearest to it
            lines = inside or [min(lines, key=lambda x: abs(x[0] - 0.5 * (self.t0 + self.t1)))[1]]
        else:
            lines = [ln for _, ln in lines]
        for ln in lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) == 7:
                try:
                    rows.append((float(parts[0]), float(parts[1]), parts[3:]))
                except ValueError:
                    pass
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({n for _, _, flags in rows for n, f in zip(names, flags) if f.lower() == "active"})
        return {"sm_mhz": statistics.median(r[0] for r in rows), "sm_max_mhz": max(r[1] for r in rows),
                "reasons": reasons, "samples": len(rows)}


def workload_config(cfg, N, nnz, d, world, extra=None):
    out = {
        "workload": f"{cfg['label']}: {'DC-SBM' if cfg.get('dcsbm') else 'SBM'} N={N}, k={cfg['k']}, s={cfg['s']:g}, eps=eps_c/4, seed 0; "
                    f"features filter, d={d} N(0,1/d) signals per rank, Jackson-Chebyshev order {P_ORDER}",
        "N": N, "nnz": nnz, "d": d, "p": P_ORDER, "k": cfg["k"],
        "cache": "inputs larger than L2 (N x d fp32 block > 126 MB L2 at N=1e6); no flush",
        "parallelism": f"signal columns sharded over {world} rank(s), graph replicated ({d} columns per rank)",
        "bytes": "SURVEY.md 8d forward-recurrence formula, fp32 values (s=4), per filter",
    }
    if extra:
        out.update(extra)
    return out


# ---------------------------------------------------------------------------
# reference arm: the reference algorithm on the host cores (oracle port; the
# reference package itself does not travel to the GPU box)


def run_reference(args, cfg):
    from oracle import cpu_ref as O
    from paper_1602_02018_b200.sbm import SbmConfig, critical_epsilon, sbm_edges

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return
    N, k, s = cfg["N"], cfg["k"], cfg["s"]
    d = int(math.ceil(4 * math.log(N)))
    scfg = SbmConfig(num_nodes=N, k=k, avg_degree=s, epsilon=critical_epsilon(s, k) / 4.0, seed=0)
    if cfg.get("dcsbm"):
        from paper_1602_02018_b200.sbm import dcsbm_edges

        src, dst, _, _ = dcsbm_edges(scfg)
    else:
        src, dst, _ = sbm_edges(scfg)
    g = O.sbm_csr(src, dst, N)
    nnz = int(g.indices.size)
    X = np.random.default_rng(0).standard_normal((N, d)) / np.sqrt(d)
    cores = os.cpu_count() or 1
    order = 1  # bounded sample: first Chebyshev step of the filter (one SpMM over the full block)
    coeffs = O.lowpass_coeffs(0.5, order)
    sample_bytes = 4.0 * (N + 1) + nnz * 8.0 + 3.0 * N * d * 4  # B_first (s=4), same unit as ours
    for _ in range(args.warmup):
        O.apply_filter_threaded(coeffs, g, X, cores)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        O.apply_filter_threaded(coeffs, g, X, cores)
    dt = (time.perf_counter() - t0) / args.steps
    gbs = sample_bytes / dt / 1e9
    sample = (f"order-{order} Jackson-Chebyshev filter (1 SpMM pass) of the full N={N} x {d} fp64 block, "
              f"columns split over {cores} threads (scipy CSR@dense releases the GIL); GB/s on the same byte formula")
    line = {
        "metric": METRIC, "value": gbs, "unit": "GB/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": dt * 1e3, "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "impl": "reference",
        "config": workload_config(cfg, N, nnz, d, 1),
        "cpu_baseline": {"value": gbs, "unit": "GB/s", "cores": cores, "kind": "port", "sample": sample},
        "e2e": {"value": gbs, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "extrapolated_filter_s": dt * P_ORDER,
    }
    print(json.dumps(line), flush=True)


def cpu_baseline(g_csr, N, nnz, d, order=6):
    """Oracle (reference algorithm) on this host, single-threaded, bounded sample (~10 s at C3)."""
    from oracle import cpu_ref as O

    X = np.random.default_rng(0).standard_normal((N, d)) / np.sqrt(d)
    coeffs = O.lowpass_coeffs(0.5, order)
    t0 = time.perf_counter()
    O.apply_filter(coeffs, g_csr, X)
    dt = time.perf_counter() - t0
    b = filter_bytes(N, nnz, d, 4, order)
    return {"value": b / dt / 1e9, "unit": "GB/s", "cores": 1, "kind": "port",
            "sample": f"order-{order} filter ({order} SpMM passes) of the full N={N} x {d} fp64 block, reference "
                      f"algorithm (numpy/scipy, single thread), {dt:.2f} s; same byte formula as value"}


# ---------------------------------------------------------------------------
# our arm


def run_ours(args, cfg):
    import torch

    import paper_1602_02018_b200 as P
    from paper_1602_02018_b200 import _lib
    from paper_1602_02018_b200.dist import DeviceBackend, Group, sharded_features
    from paper_1602_02018_b200.features import RandomSignals, build_features
    from paper_1602_02018_b200._signals import normal_block

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    grp = Group.current()  # column shards: each rank owns d signal columns of a (d x world)-column job
    N, k, s = cfg["N"], cfg["k"], cfg["s"]
    d = int(math.ceil(4 * math.log(N)))
    graph, truth = make_graph(P, cfg, device=local)
    nnz = int(graph.indices.size)
    op = P.laplacian_op(graph, dtype=cfg["dtype"], device=local)

    def barrier():
        if world > 1:
            import torch.distributed as dist

            dist.barrier()

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        import torch.distributed as dist

        t = torch.tensor([x], dtype=torch.float64, device=f"cuda:{local}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    sharded = world > 1 or args.force_sharded
    csc = None
    res = None
    lam = 0.5
    if sharded and not args.no_csc:
        from paper_1602_02018_b200.dist import DeviceBackend, run_csc_sharded

        walls = []
        try:
            for _ in range(4):  # first call pays one-off module loading / pool growth; then 3 warm calls
                barrier()
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                res = run_csc_sharded(DeviceBackend(op), N, P.CscParams(k=k, d=d, seed=0), grp)
                torch.cuda.synchronize()
                walls.append(max_over_ranks(time.perf_counter() - t0))
        except Exception as exc:  # the CSC timing is secondary: never lose the metric line over it
            res = None
            csc = {"error": f"{type(exc).__name__}: {exc}"[:300]}
    if sharded and not args.no_csc and res is not None:
        lam = res.diagnostics["lambda_k_hat"]
        csc = {"wall_s": statistics.median(walls[1:]), "wall_s_warm_calls": [round(w, 4) for w in walls[1:]],
               "wall_s_first_call": walls[0], "stages_s": res.diagnostics["timings"],
               "lambda_k_hat": lam, "probe_iterations": res.diagnostics["probe_iterations"],
               "cg_iterations_max": max(res.diagnostics["solver_iterations"]),
               "ari_vs_truth": P.adjusted_rand_index(truth, res.labels), "dtype": cfg["dtype"],
               "scaling": "strong",
               "note": f"run_csc_sharded: probe, signal and indicator columns of one CSC job split over {world} "
                       "rank(s), graph replicated; max over ranks; median of 3 warm calls"}
        del res
    if not sharded and not args.no_csc:
        walls = []
        for _ in range(4):  # first call pays one-off module loading / pool growth; then 3 warm calls
            t0 = time.perf_counter()
            res = P.run_csc(op, P.CscParams(k=k, d=d, seed=0))
            walls.append(time.perf_counter() - t0)
        lam = res.diagnostics["lambda_k_hat"]
        csc = {"wall_s": statistics.median(walls[1:]), "wall_s_warm_calls": [round(w, 4) for w in walls[1:]],
               "wall_s_first_call": walls[0], "stages_s": res.diagnostics["timings"],
               "lambda_k_hat": lam, "probe_iterations": res.diagnostics["probe_iterations"],
               "cg_iterations_max": max(res.diagnostics["solver_iterations"]),
               "ari_vs_truth": P.adjusted_rand_index(truth, res.labels), "dtype": cfg["dtype"],
               "note": "full run_csc in parity mode (numpy's seeded streams reproduced on the GPU), "
                       "graph resident; median of 3 warm calls"}
        del res
    filt = P.design_lowpass(lam, P_ORDER)

    # inputs: this rank's d signal columns (seeded per rank), resident in HBM for `value`
    host_t = torch.empty((N, d), dtype=torch.float64, pin_memory=True)  # raises if pinning fails
    host = host_t.numpy()
    normal_block(np.random.default_rng(1000 + rank), N, d, host)
    dtype_t = torch.float32 if cfg["dtype"] == "float32" else torch.float64
    X = torch.from_numpy(host).to(f"cuda:{local}").to(dtype_t)
    F = torch.empty_like(X)
    backend = DeviceBackend(op)
    stream = torch.cuda.current_stream()

    def step_device():
        if not sharded:
            from paper_1602_02018_b200.features import features_into

            # device-resident step: filter + row normalisation (zero rows still zeroed); the
            # zero-row index list is not read back, so consecutive steps queue without a host
            # round trip (the e2e measurement below goes through the full host API)
            features_into(op, filt, X, F, zero_rows=False)
        else:
            sharded_features(backend, filt, X, grp)


    # the clock sampler runs from the warm-up on (nvidia-smi needs ~0.2 s for its first sample);
    # only samples inside the marked timed region are reported
    with ClockSampler(local) as clocks:
        for _ in range(args.warmup):
            step_device()
        barrier()
        torch.cuda.synchronize()
        gc.collect()
        gc.disable()  # no collector pauses inside the timed regions (value and e2e); re-enabled below
        _lib.set_option("profile", 2)  # one event pair per filter (per-launch events cost ~2 % of a step)
        _lib.profile_reset()
        l0 = _lib.launch_count()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        clocks.mark(True)
        e0.record(stream)
        for _ in range(args.steps):
            step_device()
        e1.record(stream)
        torch.cuda.synchronize()
        clocks.mark(False)
    barrier()
    launches = _lib.launch_count() - l0
    step_ms, step_launches, step_bytes = _lib.profile_read()
    _lib.set_option("profile", 0)
    ms = max_over_ranks(e0.elapsed_time(e1)) / args.steps
    work = filter_bytes(N, nnz, d, 4 if cfg["dtype"] == "float32" else 8, P_ORDER)
    value = world * work / (ms / 1e3) / 1e9

    # e2e through the public API with host buffers (pinned signals in, features out)
    rows_t = torch.empty((N, d), dtype=torch.float64, pin_memory=True)
    rows_out = rows_t.numpy()
    signals = RandomSignals(matrix=host, distribution="gaussian", seed=None)

    def step_e2e():
        if not sharded:
            build_features(op, filt, signals, out=rows_out)
        else:
            Xh = host_t.to(f"cuda:{local}", non_blocking=True).to(dtype_t)  # pinned H2D, cast on the GPU
            Fl, _ = sharded_features(backend, filt, Xh, grp)
            rows_t.copy_(Fl.to(torch.float64))  # cast on the GPU, pinned D2H

    for _ in range(max(1, args.warmup)):
        step_e2e()
    barrier()
    torch.cuda.synchronize()
    calls = []
    t0 = time.perf_counter()
    for _ in range(args.steps):
        t1 = time.perf_counter()
        step_e2e()
        calls.append((time.perf_counter() - t1) * 1e3)  # step_e2e returns with the result on the host
    torch.cuda.synchronize()
    e2e_s = max_over_ranks(time.perf_counter() - t0) / args.steps
    gc.enable()
    # the host link this run saw (a slow or mis-placed box shows up here, not only in e2e)
    dev_t = torch.empty((N, d), dtype=torch.float64, device=f"cuda:{local}")
    link = {}
    for name, fn in (("h2d_gbs", lambda: dev_t.copy_(host_t, non_blocking=True)),
                     ("d2h_gbs", lambda: rows_t.copy_(dev_t, non_blocking=True))):
        fn()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        link[name] = 3 * host.nbytes / (time.perf_counter() - t0) / 1e9
    del dev_t
    e2e = {"value": world * work / e2e_s / 1e9, "unit": "GB/s", "h2d_bytes_per_step": int(host.nbytes),
           "d2h_bytes_per_step": int(rows_out.nbytes + N), "ms_per_step": e2e_s * 1e3,
           "api": ("paper_1602_02018_b200.build_features(op, lowpass, signals) on pinned host fp64 arrays"
                   if not sharded else
                   "paper_1602_02018_b200.dist.sharded_features (this rank's columns, NCCL row-norm exchange) "
                   "on pinned host fp64 arrays"),
           "host_pinned": bool(host_t.is_pinned() and rows_t.is_pinned()),
           "ms_per_call": [round(c, 2) for c in calls],
           "link_gbs_measured": link}

    if rank != 0:
        return
    peak, peak_src = peaks()
    # SURVEY.md 8(d) unit: one fused Chebyshev step on the N x d block moves B_step(d) =
    # B_csr + 5 N d s algorithmic bytes (B_first for the first step), whatever recurrence
    # the kernel uses; achieved = those bytes of the timed filters / the K2 launches' time
    alg_per_step_set = work  # B_first + (p - 1) B_step per filter, one filter per step
    achieved = alg_per_step_set * args.steps / (step_ms / 1e3) / 1e9 if step_ms > 0 else None
    traffic = None
    tf = ROOT / "profiles" / "ncu_traffic.json"
    if tf.exists():
        traffic = json.loads(tf.read_text()).get(f"{args.config}_{cfg['dtype']}")
    roofline = {
        "bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
        "frac": (achieved / peak) if achieved else None, "traffic": traffic,
        "kernel": "fused Chebyshev step SpMM: k_cheb_mid (mid steps) + k_cheb_step (first / last steps)",
        "peak_source": peak_src,
        "kernel_ms_per_launch": step_ms / max(step_launches, 1), "launches_timed": step_launches,
        "kernel_timing": "CUDA events around each filter's back-to-back step launches on the launch stream "
                         "(profile mode 2), divided by the launches",
        "algorithmic_bytes_per_launch": alg_per_step_set * args.steps / max(step_launches, 1),
        "algorithmic_unit": "SURVEY.md 8(d) B_step(d) = B_csr + 5 N d s per step launch (B_first on the first); "
                            "one launch per step when the block is one panel",
        "kernel_stream_bytes_per_launch": step_bytes / max(step_launches, 1),
        "frac_of_8tbs": (achieved / 8000.0) if achieved else None,  # report against both peaks
        "ncu_dram_throughput_pct": _ncu_dram_pct(args.config, cfg["dtype"]),
        "ncu_dram_gbs": _ncu_dram_gbs(args.config, cfg["dtype"]),
        "kernel_share_of_step": (step_ms / args.steps) / ms if ms > 0 else None,
        "recurrence": "clenshaw" if _lib.get_option("recurrence") == 0 else "forward",
        # Every step re-reads each gathered row ~deg times through L2 (L2->SM bytes below); at C3
        # the 256 MB gather panel exceeds L2 and the random inter-community gathers come from
        # DRAM.  The gathers alone take 253-302 us per step on this graph
        # (profiles/r01_gather_sol.txt); the 64-B-row L2 ceiling is kept for reference.
        "l2_path": {
            "bytes_per_filter": (step_bytes / args.steps + P_ORDER * (nnz - N) * d * (4 if cfg["dtype"] == "float32" else 8)),
            "achieved_gbs": ((step_bytes / args.steps + P_ORDER * (nnz - N) * d * (4 if cfg["dtype"] == "float32" else 8))
                             / (step_ms / args.steps / 1e3) / 1e9) if step_ms > 0 else None,
            "ceiling_gbs": 11050.0,
            "ceiling_source": "random 64-B row gathers, LDG at 64 warps/SM: tools/microbench/gather_bench.cu",
            "note": "L2->SM bytes = algorithmic bytes + (deg-1) extra reads of every gathered row per step",
        },
        "gather_sol_us_per_step": ({"warps_48": 302.0, "warps_64": 253.0,
                                    "source": "one step's neighbour-row gathers alone on the C3 graph "
                                              "(tools/microbench/csr_gather_sol.cu, profiles/r01_gather_sol.txt)"}
                                   if args.config == "c3" and cfg["dtype"] == "float32" else None),
    }
    cpub = None
    if world == 1 and not args.no_cpu:
        from oracle import cpu_ref as O

        cpub = cpu_baseline(O.Csr(N, graph.indptr, graph.indices, graph.weights, graph.degrees), N, nnz, d)
    line = {
        "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32" if cfg["dtype"] == "float32" else "f64", "data": "synthetic",
        "config": workload_config(cfg, N, nnz, d, world, {"panel_plan": _lib.get_option("panel_width") or "auto"}),
        "e2e": e2e, "gpu_launches": launches, "roofline": roofline, "cpu_baseline": cpub,
        "clocks": clocks.summary(), "csc": csc,
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", choices=sorted(CONFIGS), default="c3")
    ap.add_argument("--no-csc", action="store_true", help="skip the one-off full run_csc wall-time")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline sample")
    ap.add_argument("--option", action="append", default=[], help="libcsc option key=value (tuning)")
    ap.add_argument("--force-sharded", action="store_true",
                    help="use the multi-GPU (column-sharded, NCCL) step even on one rank (path check)")
    args = ap.parse_args()
    cfg = CONFIGS[args.config]
    if args.impl == "reference":
        run_reference(args, cfg)
        return
    if args.option:
        from paper_1602_02018_b200 import _lib

        for kv in args.option:
            key, val = kv.split("=")
            _lib.set_option(key, int(val))
    try:
        run_ours(args, cfg)
    finally:
        import torch.distributed as dist

        if dist.is_available() and dist.is_initialized():
            dist.destroy_process_group()  # local teardown; ranks may arrive at different times


if __name__ == "__main__":
    main()
