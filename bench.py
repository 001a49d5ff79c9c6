#!/usr/bin/env python
"""Benchmark of the hot path: the order-50 Jackson-Chebyshev features filter on SBM N=1e6, k=100.

Contract:
  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config c3]
One JSON line on rank 0.  A step = one features pass (filter of the d = ceil(4 ln N) = 56
signal columns with p = 50, plus row normalisation) over the BASELINE config-3 graph.
``value`` = whole-job Cheb-filter GB/s, with bytes from the SURVEY.md §8d formula
(forward recurrence, fp32 values: B_first + (p-1) B_step per filter) so every arm is
measured on the same unit of work; the kernels' own algorithmic bytes go into ``roofline``.

Multi-GPU (``--gpus N``; re-launches itself under torch.distributed.run when WORLD_SIZE is
unset): one process per GPU, graph replicated, the SAME 56 signal columns split over the N
ranks (strong scaling, BASELINE config 3: "signal columns sharded over 1/2/4/8 GPUs"), the
row norms all-gathered over NCCL; ``weak_scaling`` adds the run where every rank filters
56 columns of its own.  ``--row-sharded`` filters through the row-sharded operator instead
(BASELINE config 5: CSR rows split over the ranks, NCCL all-gather of the block after every
Chebyshev step, or ``--transport peer`` for the stores fused into the step kernel).
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


def _l2_path(step_ms, step_bytes, steps, n, nnz, w, s, c3_f32):
    """Bytes K2 moves from L2 to the SMs per second: the row streams of its launches plus every
    neighbour row it gathers (nnz x w x s per step, against one compulsory read in the HBM unit)."""
    if not step_ms or not step_bytes:
        return None
    per_filter = step_bytes / steps - P_ORDER * n * w * s + P_ORDER * nnz * w * s
    ach = per_filter * steps / (step_ms / 1e3) / 1e9
    # gathers alone on the C3 graph, 128-B rows, 64 warps/SM: 117.44 G rows/s x 128 B (r01_gather_sol.txt)
    ceil = 117.44 * 128.0 if c3_f32 else None
    return {"achieved_gbs": ach, "bytes_per_filter": per_filter, "gather_only_ceiling_gbs": ceil,
            "frac_of_gather_ceiling": ach / ceil if ceil else None,
            "note": "row streams + nnz x w x s gathered bytes per step over the K2 launch time; ceiling = "
                    "one step's gathers alone (no streams, no epilogue) on the same graph"}


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


def workload_config(cfg, N, nnz, d, world, row_sharded=False, transport="nccl"):
    """The `config` object: a function of the workload and the rank count only, so the
    reference arm and ours print the same one."""
    if row_sharded:
        par = (f"CSR rows split over {world} rank(s) (nnz-balanced), {transport} all-gather of the "
               f"{d}-column block after every Chebyshev step")
    else:
        par = f"the {d} signal columns split over {world} rank(s), graph replicated"
    return {
        "workload": f"{cfg['label']}: {'DC-SBM' if cfg.get('dcsbm') else 'SBM'} N={N}, k={cfg['k']}, s={cfg['s']:g}, "
                    f"eps=eps_c/4, seed 0; features filter of d={d} N(0,1/d) signals, Jackson-Chebyshev order {P_ORDER}",
        "N": N, "nnz": nnz, "d": d, "p": P_ORDER, "k": cfg["k"],
        "cache": "inputs larger than L2 (N x d fp32 block > 126 MB L2 at N=1e6); no flush",
        "parallelism": par,
        "bytes": "SURVEY.md 8d forward-recurrence formula, fp32 values (s=4), per filter",
    }


# ---------------------------------------------------------------------------
# reference arm: the reference algorithm on the host cores (oracle port; the
# reference package itself does not travel to the GPU box)


REF_ORDER = 4  # reference-arm sample: first Chebyshev step + 3 mid steps per timed step


def run_reference(args, cfg):
    """The reference algorithm (oracle port of filters.py:140-155 on scipy's CSR product) on the
    host cores: each step an order-4 filter (first step + 3 mid steps) of the full N x d fp64
    block, charged the same SURVEY.md 8(d) bytes per step as our arm's order-50 filter."""
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
    order = REF_ORDER
    coeffs = O.lowpass_coeffs(0.5, order)
    sample_bytes = filter_bytes(N, nnz, d, 4, order)  # same unit as ours: B_first + (order-1) B_step
    for _ in range(args.warmup):
        O.apply_filter_threaded(coeffs, g, X, cores)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        O.apply_filter_threaded(coeffs, g, X, cores)
    dt = (time.perf_counter() - t0) / args.steps
    gbs = sample_bytes / dt / 1e9
    sample = (f"order-{order} Jackson-Chebyshev filter ({order} SpMM passes: first step + {order - 1} mid steps) "
              f"of the full N={N} x {d} fp64 block per step, columns split over {cores} threads (scipy CSR@dense "
              f"releases the GIL); GB/s on the same byte formula as ours")
    line = {
        "metric": METRIC, "value": gbs, "unit": "GB/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": dt * 1e3, "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "impl": "reference",
        "config": workload_config(cfg, N, nnz, d, world, args.row_sharded, args.transport),
        "cpu_baseline": {"value": gbs, "unit": "GB/s", "cores": cores, "kind": "port", "sample": sample},
        "e2e": {"value": gbs, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "extrapolated_filter_s": dt * (filter_bytes(N, nnz, d, 4, P_ORDER) / sample_bytes),
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


def _dist_helpers(world, local):
    import torch

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

    return barrier, max_over_ranks


def _time_steps(step, steps, warmup, barrier, max_over_ranks, clocks=None, profile=True):
    """W untimed steps, then K steps between a barrier + synchronize on both sides, timed with
    CUDA events on the launch stream; returns (ms per step max over ranks, launches, profile)."""
    import torch

    from paper_1602_02018_b200 import _lib

    stream = torch.cuda.current_stream()
    for _ in range(warmup):
        step()
    barrier()
    torch.cuda.synchronize()
    gc.collect()
    gc.disable()  # no collector pauses inside the timed region
    if profile:
        _lib.set_option("profile", 2)  # one event pair per filter (per-launch events cost ~2 % of a step)
        _lib.profile_reset()
    l0 = _lib.launch_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if clocks:
        clocks.mark(True)
    e0.record(stream)
    for _ in range(steps):
        step()
    e1.record(stream)
    torch.cuda.synchronize()
    if clocks:
        clocks.mark(False)
    gc.enable()
    barrier()
    launches = _lib.launch_count() - l0
    prof = _lib.profile_read() if profile else (0.0, 0, 0.0)
    _lib.set_option("profile", 0)
    return max_over_ranks(e0.elapsed_time(e1)) / steps, launches, prof


def run_ours(args, cfg):
    import torch

    import paper_1602_02018_b200 as P
    from paper_1602_02018_b200 import _lib
    from paper_1602_02018_b200.dist import DeviceBackend, Group, column_slice, sharded_features
    from paper_1602_02018_b200.features import RandomSignals, build_features, features_into
    from paper_1602_02018_b200._signals import normal_block

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    grp = Group.current()
    N, k = cfg["N"], cfg["k"]
    d = int(math.ceil(4 * math.log(N)))
    graph, truth = make_graph(P, cfg, device=local)
    nnz = int(graph.indices.size)
    op = P.laplacian_op(graph, dtype=cfg["dtype"], device=local)
    barrier, max_over_ranks = _dist_helpers(world, local)
    s_bytes = 4 if cfg["dtype"] == "float32" else 8
    sharded = world > 1 or args.force_sharded

    # ---- full run_csc wall time (secondary key)
    csc, lam = None, 0.5
    if not args.no_csc and not args.row_sharded:
        walls, res = [], None
        try:
            for _ in range(4):  # first call pays one-off module loading / pool growth; then 3 warm calls
                barrier()
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                if sharded:
                    from paper_1602_02018_b200.dist import run_csc_sharded

                    res = run_csc_sharded(DeviceBackend(op), N, P.CscParams(k=k, d=d, seed=0), grp)
                else:
                    res = P.run_csc(op, P.CscParams(k=k, d=d, seed=0))
                torch.cuda.synchronize()
                walls.append(max_over_ranks(time.perf_counter() - t0))
            lam = res.diagnostics["lambda_k_hat"]
            csc = {"wall_s": statistics.median(walls[1:]), "wall_s_warm_calls": [round(w, 4) for w in walls[1:]],
                   "wall_s_first_call": walls[0], "stages_s": res.diagnostics["timings"],
                   "lambda_k_hat": lam, "probe_iterations": res.diagnostics["probe_iterations"],
                   "cg_iterations_max": max(res.diagnostics["solver_iterations"]),
                   "ari_vs_truth": P.adjusted_rand_index(truth, res.labels), "dtype": cfg["dtype"],
                   "note": ("run_csc_sharded: probe, signal and indicator columns of one CSC job split over "
                            f"{world} rank(s), graph replicated; max over ranks; median of 3 warm calls")
                   if sharded else ("full run_csc in parity mode (numpy's seeded streams reproduced on the GPU), "
                                    "graph resident; median of 3 warm calls")}
            # the reference's own run_csc on this config, recorded when the golden capture was made
            # (tests/golden/make_golden.py, one core): its wall time and whether our labels match it
            cap = ROOT / "tests" / "golden" / f"pipeline_{args.config}.npz"
            gz = np.load(cap) if cap.exists() and world == 1 else None
            if gz is not None and "wall_s" in gz.files:
                csc["reference_capture"] = {
                    "wall_s": float(gz["wall_s"]), "stages_s": json.loads(str(gz["timings"])),
                    "lambda_k_hat": float(gz["lambda_k_hat"]),
                    "labels_ari_vs_reference": P.adjusted_rand_index(res.labels, gz["labels"]),
                    "source": f"tests/golden/pipeline_{args.config}.npz (reference run_csc, fp64, 1 core, build container)"}
        except Exception as exc:  # secondary: never lose the metric line over it
            csc = {"error": f"{type(exc).__name__}: {exc}"[:300]}
        del res
    filt = P.design_lowpass(lam, P_ORDER)
    dtype_t = torch.float32 if cfg["dtype"] == "float32" else torch.float64

    # ---- inputs: the job's N x d signal block (same seed on every rank), resident in HBM
    host_t = torch.empty((N, d), dtype=torch.float64, pin_memory=True)  # raises if pinning fails
    host = host_t.numpy()
    normal_block(np.random.default_rng(1000), N, d, host)
    backend = DeviceBackend(op)
    rop = None
    if args.row_sharded:
        from paper_1602_02018_b200.dist import RowShardedOperator

        rop = RowShardedOperator(graph, grp, dtype=cfg["dtype"], device=local, transport=args.transport)
        rows = slice(rop.begin, rop.end)
        X = torch.from_numpy(host[rows]).to(f"cuda:{local}").to(dtype_t)
        cols = slice(0, d)
        w_local = d
    else:
        cols = column_slice(d, world, rank)  # strong scaling: this rank's share of the job's columns
        X = torch.from_numpy(np.ascontiguousarray(host[:, cols])).to(f"cuda:{local}").to(dtype_t)
        w_local = cols.stop - cols.start
    F = torch.empty_like(X)

    def step_device():
        if rop is not None:
            rop.features(filt, X)
        elif not sharded:
            # device-resident step: filter + row normalisation (zero rows still zeroed); the
            # zero-row list is not read back, so consecutive steps queue without a host round trip
            features_into(op, filt, X, F, zero_rows=False)
        else:
            sharded_features(backend, filt, X, grp)

    with ClockSampler(local) as clocks:
        ms, launches, (step_ms, step_launches, step_bytes) = _time_steps(
            step_device, args.steps, args.warmup, barrier, max_over_ranks, clocks)
    work = filter_bytes(N, nnz, d, s_bytes, P_ORDER)  # the job: one order-p filter of all d columns
    value = work / (ms / 1e3) / 1e9

    # ---- weak scaling (N > 1): every rank filters d columns of its own
    weak = None
    if world > 1 and not args.row_sharded:
        Xw_host = normal_block(np.random.default_rng(2000 + rank), N, d)
        Xw = torch.from_numpy(Xw_host).to(f"cuda:{local}").to(dtype_t)
        msw, _, _ = _time_steps(lambda: sharded_features(backend, filt, Xw, grp), args.steps, args.warmup, barrier,
                                max_over_ranks, profile=False)
        weak = {"value": world * work / (msw / 1e3) / 1e9, "unit": "GB/s", "ms_per_step": msw,
                "columns_per_rank": d, "note": "every rank filters d columns of its own; row norms exchanged"}
        del Xw

    # ---- e2e through the public API with host buffers (pinned fp64 signals in, features out)
    rows_t = torch.empty((N, d), dtype=torch.float64, pin_memory=True)
    rows_out = rows_t.numpy()
    signals = RandomSignals(matrix=host, distribution="gaussian", seed=None)
    if rop is not None:
        h_in = host_t[rop.begin:rop.end]
        h_out = rows_t[rop.begin:rop.end]
    else:
        h_in = host_t[:, cols] if world > 1 else host_t
        h_out = rows_t[:, cols] if world > 1 else rows_t

    def step_e2e():
        if not sharded and rop is None:
            build_features(op, filt, signals, out=rows_out)
            return
        Xh = h_in.to(f"cuda:{local}", non_blocking=True).to(dtype_t)  # pinned H2D, cast on the GPU
        Fl = rop.features(filt, Xh)[0] if rop is not None else sharded_features(backend, filt, Xh, grp)[0]
        h_out.copy_(Fl.to(torch.float64))  # cast on the GPU, D2H

    for _ in range(max(1, args.warmup)):
        step_e2e()
    barrier()
    torch.cuda.synchronize()
    calls = []
    gc.disable()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        t1 = time.perf_counter()
        step_e2e()
        calls.append((time.perf_counter() - t1) * 1e3)  # step_e2e returns with the result on the host
    torch.cuda.synchronize()
    e2e_s = max_over_ranks(time.perf_counter() - t0) / args.steps
    gc.enable()
    link = {}
    if rank == 0:  # the host link this run saw (a slow or mis-placed box shows up here, not only in e2e)
        dev_t = torch.empty((N, d), dtype=torch.float64, device=f"cuda:{local}")
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
    in_bytes = int(h_in.numel() * 8)
    e2e = {"value": work / e2e_s / 1e9, "unit": "GB/s", "h2d_bytes_per_step": in_bytes * world,
           "d2h_bytes_per_step": in_bytes * world + (N if world == 1 and rop is None else 0),
           "ms_per_step": e2e_s * 1e3,
           "api": ("paper_1602_02018_b200.build_features(op, lowpass, signals) on pinned host fp64 arrays"
                   if not sharded and rop is None else
                   ("paper_1602_02018_b200.dist.RowShardedOperator.features (this rank's rows)" if rop is not None
                    else "paper_1602_02018_b200.dist.sharded_features (this rank's columns, NCCL row-norm exchange)")
                   + " on pinned host fp64 arrays; bytes summed over ranks"),
           "host_pinned": bool(host_t.is_pinned() and rows_t.is_pinned()),
           "ms_per_call_rank0": [round(c, 2) for c in calls],
           "link_gbs_measured_rank0": link}

    # ---- fp64 leg at the reference's own precision (N = 1, replicated)
    f64 = None
    if world == 1 and rop is None and cfg["dtype"] != "float64" and not args.no_f64:
        op64 = P.laplacian_op(graph, dtype="float64", device=local)
        X64 = torch.from_numpy(host).to(f"cuda:{local}")
        F64 = torch.empty_like(X64)
        ms64, _, (k_ms, k_launches, _) = _time_steps(lambda: features_into(op64, filt, X64, F64, zero_rows=False),
                                                     args.steps, args.warmup, barrier, max_over_ranks)
        w64 = filter_bytes(N, nnz, d, 8, P_ORDER)
        peak, _ = peaks()
        ach = w64 * args.steps / (k_ms / 1e3) / 1e9 if k_ms > 0 else None
        f64 = {"value": w64 / (ms64 / 1e3) / 1e9, "unit": "GB/s", "ms_per_step": ms64, "dtype": "f64",
               "roofline": {"bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s",
                            "frac": ach / peak if ach else None, "kernel_ms_per_launch": k_ms / max(k_launches, 1)},
               "note": "same step on the fp64 operator and fp64 block (the reference's precision); s=8 in the "
                       "byte formula"}
        del op64, X64, F64

    if rank != 0:
        return
    peak, peak_src = peaks()
    # SURVEY.md 8(d) unit: one fused Chebyshev step on this rank's N x w block moves B_step(w) =
    # B_csr + 5 N w s algorithmic bytes (B_first for the first step), whatever recurrence the
    # kernel uses; achieved = those bytes of the timed filters / the K2 launches' time
    n_rows = (rop.end - rop.begin) if rop is not None else N
    nnz_rows = rop.local_nnz if rop is not None else nnz
    alg_per_filter = filter_bytes(n_rows, nnz_rows, w_local, s_bytes, P_ORDER)
    achieved = alg_per_filter * args.steps / (step_ms / 1e3) / 1e9 if step_ms > 0 else None
    traffic = None
    tf = ROOT / "profiles" / "ncu_traffic.json"
    if tf.exists() and world == 1 and rop is None:
        traffic = json.loads(tf.read_text()).get(f"{args.config}_{cfg['dtype']}")
    roofline = {
        "bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
        "frac": (achieved / peak) if achieved else None, "traffic": traffic,
        "kernel": "fused Chebyshev step SpMM: k_cheb_mid (mid steps) + k_cheb_step (first / last steps)",
        "peak_source": peak_src,
        "kernel_ms_per_launch": step_ms / max(step_launches, 1), "launches_timed": step_launches,
        "kernel_timing": "CUDA events around each filter's back-to-back step launches on the launch stream "
                         "(profile mode 2), divided by the launches; rank 0",
        "algorithmic_bytes_per_launch": alg_per_filter * args.steps / max(step_launches, 1),
        "algorithmic_unit": f"SURVEY.md 8(d) B_step(w) = B_csr + 5 N w s per step launch (B_first on the first), "
                            f"w = {w_local} columns of rank 0; one launch per step when the block is one panel",
        "kernel_stream_bytes_per_launch": step_bytes / max(step_launches, 1),
        # the DRAM-traffic-limited ceiling: frac if the kernel moved its measured (ncu) DRAM
        # traffic at the copy peak; the gap to 1 is gather misses, not kernel inefficiency
        "traffic_ceiling_frac": (alg_per_filter * args.steps / max(step_launches, 1)) / traffic if traffic else None,
        "achieved_of_traffic_ceiling": ((achieved / peak) / ((alg_per_filter * args.steps / max(step_launches, 1))
                                                              / traffic)) if traffic and achieved else None,
        "frac_of_8tbs": (achieved / 8000.0) if achieved else None,  # report against both peaks
        "ncu_dram_throughput_pct": _ncu_dram_pct(args.config, cfg["dtype"]) if world == 1 and rop is None else None,
        "ncu_dram_gbs": _ncu_dram_gbs(args.config, cfg["dtype"]) if world == 1 and rop is None else None,
        "kernel_share_of_step": (step_ms / args.steps) / ms if ms > 0 else None,
        "recurrence": "clenshaw" if _lib.get_option("recurrence") == 0 or rop is not None else "forward",
        "panel_plan": _lib.get_option("panel_width") or "auto",
        # the L2 -> SM path that bounds K2 (profiles/r02_k2_decomposition.txt): every launch moves
        # its row streams plus deg x (row bytes) of neighbour gathers through L2
        "l2_path": _l2_path(step_ms, step_bytes, args.steps, n_rows, nnz_rows, w_local, s_bytes,
                            args.config == "c3" and cfg["dtype"] == "float32" and world == 1 and rop is None),
        "gather_sol_us_per_step": ({"warps_48": 302.0, "warps_64": 253.0,
                                    "source": "one step's neighbour-row gathers alone on the C3 graph "
                                              "(tools/microbench/csr_gather_sol.cu, profiles/r01_gather_sol.txt)"}
                                   if args.config == "c3" and cfg["dtype"] == "float32" and world == 1 else None),
    }
    cpub = None
    if world == 1 and not args.no_cpu:
        from oracle import cpu_ref as O

        cpub = cpu_baseline(O.Csr(N, graph.indptr, graph.indices, graph.weights, graph.degrees), N, nnz, d)
    line = {
        "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f32" if cfg["dtype"] == "float32" else "f64", "data": "synthetic",
        "config": workload_config(cfg, N, nnz, d, world, args.row_sharded, args.transport),
        "e2e": e2e, "gpu_launches": launches, "roofline": roofline, "cpu_baseline": cpub,
        "clocks": clocks.summary(), "csc": csc, "weak_scaling": weak, "f64": f64,
    }
    if rop is not None:
        rop.close()  # collective: peers unmapped before any rank frees its panels
    print(json.dumps(line), flush=True)


def _free_port() -> int:
    import socket

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", choices=sorted(CONFIGS), default="c3")
    ap.add_argument("--row-sharded", action="store_true",
                    help="filter through the row-sharded operator (BASELINE config 5 mode)")
    ap.add_argument("--transport", choices=["nccl", "peer"], default="nccl")
    ap.add_argument("--no-csc", action="store_true", help="skip the one-off full run_csc wall-time")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline sample")
    ap.add_argument("--no-f64", action="store_true", help="skip the fp64 leg")
    ap.add_argument("--option", action="append", default=[], help="libcsc option key=value (tuning)")
    ap.add_argument("--force-sharded", action="store_true",
                    help="use the multi-GPU (column-sharded, NCCL) step even on one rank (path check)")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # one process per GPU: re-launch under torch.distributed.run (the driver's own launch
        # sets WORLD_SIZE and lands below directly)
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), str(Path(__file__).resolve())]
        sys.exit(subprocess.call(cmd + sys.argv[1:]))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}; using WORLD_SIZE", file=sys.stderr)
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
