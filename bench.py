"""Benchmark: log-det estimates per second on BASELINE config 2 (n = 16384,
RBF in R^8, stored K in HBM, rand-SVD l = 256, 32 Rademacher probes, t = 20),
one JSON line on rank 0.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--config 2] [--dtype fp32|fp64] [--algorithm r3] [--n N]

A step is one full estimate (preconditioner build + s-probe Lanczos +
multishift solves + Hutchinson mean) -- the reference's timer scope
(src/estimators.py:81-96).

* ``value``: estimates/s with K, the sketch rows and the probes resident in HBM
  (K = 1.07 GB fp32 > 126 MB L2, so every product streams K from HBM), CUDA
  events on the handle's stream around exactly K steps, max over ranks.
* ``e2e``: the same metric through the C ABI call the public API makes, with host
  buffers -- every step uploads the points from pinned memory, builds K on the
  GPU, regenerates the reference's probe / sketch streams on the GPU, runs the
  estimate and reads the result back.
* ``roofline``: the dominant kernel (the K x block product, Lanczos shape),
  timed live with CUDA events; algorithmic bytes = 4 n^2 (K) + 4 n s (operand)
  + 8 n s (result) per launch.
* ``cpu_baseline``: the oracle port (float64 numpy restatement of the
  reference, per-probe loop like the reference) on this host's cores, one
  estimate of the same workload.
* ``--impl reference``: that CPU implementation is the timed arm.

Multi-GPU (torchrun, one process per GPU): by default the rows of K and of every
n-vector block are sharded across the ranks; one estimate per
step for the whole job (``"scaling": "strong"``), NCCL all-gather of the direction
block per Lanczos step and all-reduces of the dot products / Gram matrices.
``--mode replicas`` instead runs an independent single-GPU estimate per rank
(``"scaling": "weak"``).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from dataclasses import replace
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "log-det estimates/sec"
UNIT = "estimates/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--n", type=int, default=None)
    ap.add_argument("--dtype", choices=["fp32", "fp64"], default=None)
    ap.add_argument("--algorithm", choices=["r1", "r3", "r5"], default=None)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-concurrent", action="store_true", help="skip the informational concurrent-estimates run")
    ap.add_argument("--mode", choices=["sharded", "replicas"], default="sharded",
                    help="multi-GPU: row-shard one estimate (default) or run independent replicas")
    return ap.parse_args()


def load_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), float(d["bf16_tflops"]), "measured"
    return 6650.0, 1590.0, "fallback"


def load_pipe_peaks():
    """Measured compute-pipe peaks of this pool's B200 (scripts/pipe_peaks.cu, committed)."""
    p = ROOT / "profiles" / "r01_pipe_peaks.json"
    return json.loads(p.read_text()) if p.exists() else {}


class ClockSampler:
    """nvidia-smi clocks and throttle reasons during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.lines:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[4:8]):
                if v.lower() in ("active", "1"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


def dist_setup(gpus):
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world > 1:
        dist.init_process_group("nccl", init_method="env://")
        local = int(os.environ.get("LOCAL_RANK", "0"))
        torch.cuda.set_device(local)
        return dist.get_rank(), world, local
    torch.cuda.set_device(0)
    return 0, 1, 0


def max_over_ranks(x: float, world: int) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist

    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(world):
    if world > 1:
        import torch.distributed as dist

        dist.barrier()


def ncu_traffic(name="kv_c2_m32"):
    """DRAM bytes (read + write) per launch of the dominant kernel from the newest
    committed ncu --set full summary (profiles/*_kv_ncu.json, scripts/summarize_profiles.py)."""
    files = sorted((ROOT / "profiles").glob("*_kv_ncu.json"), key=lambda p: p.stat().st_mtime)
    for f in reversed(files):
        try:
            rec = json.loads(f.read_text()).get(name)
        except Exception:
            continue
        if rec and "dram_bytes_total" in rec:
            return rec["dram_bytes_total"], f.name
    return None, None


def workload_for(args):
    from paper_2405_03474_b200.workloads import baseline

    wl = baseline(args.config, n=args.n, algorithm=args.algorithm, dtype=args.dtype)
    return wl


# --------------------------------------------------------------------------- CPU (oracle port)

def cpu_estimate(wl, threads: int):
    """One estimate of the oracle port (float64, per-probe loop like the reference).
    Returns (seconds, estimate) -- K construction excluded, like the reference's timer."""
    os.environ.setdefault("OPENBLAS_NUM_THREADS", str(threads))
    from oracle import rstar_oracle as O

    K = O.covariance_block(wl.spec.family, wl.spec.amplitude, wl.spec.length_scale, wl.spec.jitter, wl.points)
    cfg = wl.config
    t0 = time.perf_counter()
    est = O.rstar_dense(K, order=int(cfg.algorithm[1]), s=cfg.num_probes, t=cfg.lanczos_iters,
                        probe_kind=cfg.probe_kind, k=cfg.precond.rank, q=cfg.precond.num_iters, seed=cfg.seed,
                        per_probe=True)
    return time.perf_counter() - t0, est


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def workload_config(wl, world=1, sharded=False):
    """The `config` object both arms print (the driver compares the reference arm on our arm's config)."""
    cfg = wl.config
    n, s = wl.n, cfg.num_probes
    es = 4 if cfg.dtype == "fp32" else 8
    return {"workload": f"{wl.name}: n={n} {wl.spec.family} d={wl.points.shape[1]} ell={wl.spec.length_scale} "
                        f"noise={wl.spec.jitter} {cfg.algorithm} l={cfg.precond.rank} s={s} "
                        f"{cfg.probe_kind} t={cfg.lanczos_iters} q={cfg.precond.num_iters} stored K "
                        f"({cfg.dtype})",
            "l2": "inputs larger than L2 (K = %.2f GB)" % (es * n * n / 1e9),
            "parallelism": (f"rows{world}" if sharded else f"replicas{world}") if world > 1 else "single"}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    threads = os.cpu_count() or 1
    os.environ["OPENBLAS_NUM_THREADS"] = str(threads)
    wl = workload_for(args)
    arm_config = workload_config(wl)
    cfg = replace(wl.config, dtype="fp64")
    wl = replace(wl, config=cfg)
    warm = min(args.warmup, 1)
    steps = max(1, min(args.steps, 3))
    for _ in range(warm):
        cpu_estimate(wl, threads)
    times = [cpu_estimate(wl, threads)[0] for _ in range(steps)]
    total = sum(times)
    v = steps / total
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus, "steps": steps,
        "warmup": warm, "ms_per_step": 1e3 * total / steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {**arm_config, "note": "the reference has no fp32 mode: this CPU arm computes in float64"},
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": f"{steps} full estimate(s) of the workload, oracle port (numpy/OpenBLAS, "
                                   f"per-probe loop), K build excluded", "cpu": cpu_model()},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# --------------------------------------------------------------------------- GPU

def run_ours(args):
    import ctypes as C

    import torch

    import paper_2405_03474_b200 as rld
    from paper_2405_03474_b200 import _native as N
    from paper_2405_03474_b200.estimators import make_config
    from paper_2405_03474_b200.linalg import Rng

    rank, world, local = dist_setup(args.gpus)
    wl = workload_for(args)
    cfg = wl.config
    n, s = wl.n, cfg.num_probes
    w = min(cfg.precond.rank + 10, n)
    es = 4 if cfg.dtype == "fp32" else 8

    # ---- device-resident: K in HBM; the probe and sketch streams are regenerated on the
    # device every estimate (numpy-exact Philox Rademacher / ziggurat Gaussian rows), as the
    # reference draws them inside its timed region (src/estimators.py:81-83)
    sharded = world > 1 and args.mode == "sharded"
    per_step = 1 if sharded else world       # estimates the whole job completes per step
    R = rld.ResidentMatrix(rld.KernelMatrix(wl.spec, wl.points), dtype=cfg.dtype, path=wl.path, shard=sharded)
    from paper_2405_03474_b200.parallel import shard_bounds
    row0, row1 = shard_bounds(n, world, rank) if sharded else (0, n)
    rows = row1 - row0
    inputs = N.Inputs()
    inputs.memory = N.DEVICE
    stream = torch.cuda.ExternalStream(R.sess.handle.stream)

    clk = ClockSampler(local).__enter__()   # sampling starts before warm-up, covers the timed region
    for _ in range(args.warmup):
        est = R.estimate(cfg, inputs=inputs)
    barrier(world)
    torch.cuda.synchronize()
    launches = 0
    products = 0
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if True:
        ev0.record(stream)
        for _ in range(args.steps):
            est = R.estimate(cfg, inputs=inputs)
            launches += est.kernel_launches
            products += est.kv_products
        ev1.record(stream)
        torch.cuda.synchronize()
    clk.__exit__()
    barrier(world)
    ms = ev0.elapsed_time(ev1)
    ms = max_over_ranks(ms, world)
    value = per_step * args.steps / (ms * 1e-3)
    clocks = clk.summary()
    phases = est.phase_ms

    # ---- dominant kernel: K x block product at the Lanczos shape, timed live
    V = torch.randn(s, n, dtype=torch.float64, device="cuda")
    for _ in range(3):
        R.kv_apply(V)
    reps = 20
    k0, k1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    k0.record(stream)
    for _ in range(reps):
        R.kv_apply(V)
    k1.record(stream)
    torch.cuda.synchronize()
    kv_ms = k0.elapsed_time(k1) / reps
    alg_bytes = es * rows * n + 4 * n * s + 8 * rows * s
    hbm_peak, _, peak_kind = load_peaks()
    traffic, traffic_src = (ncu_traffic() if (args.config == 2 and world == 1 and args.dtype in (None, "fp32"))
                            else (None, None))
    achieved = alg_bytes / (kv_ms * 1e-3) / 1e9
    roofline = {"bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s", "frac": achieved / hbm_peak,
                "traffic": traffic, "traffic_source": traffic_src,
                "kernel": f"kv_product (Lanczos shape m=s, {rows} rows of K)", "kernel_ms": kv_ms,
                "alg_bytes": alg_bytes, "peak_source": peak_kind}
    pipe = load_pipe_peaks()
    if wl.path == "on_the_fly" or cfg.dtype == "fp64":
        # no stored K (on the fly) or an FP64-pipe-bound product (fp64, 8 flop/B > the DFMA ridge):
        # the bound is a compute pipe, SURVEY.md §8(d)
        useful = 2.0 * rows * n * s
        if cfg.dtype == "fp64":
            kind, work, peak, src = "fp64", useful, pipe.get("dfma_tflops", 36.36), "profiles/r01_pipe_peaks.json dfma"
        else:   # 3xTF32 tensor-core MMAs: three products per useful one
            kind, work = "tensor", 3.0 * useful
            peak, src = pipe.get("tf32_ts_n128", {}).get("tflops", 1115.0), "profiles/r01_pipe_peaks.json tf32 N=128"
        ach = work / (kv_ms * 1e-3) / 1e12
        roofline = {"bound": kind, "achieved": ach, "peak": peak, "unit": "TFLOP/s", "frac": ach / peak,
                    "traffic": None, "kernel": f"kv_product ({wl.path}, m=s={s}, {rows} rows)", "kernel_ms": kv_ms,
                    "alg_flops": work, "useful_flops": useful, "peak_source": src}

    # ---- end to end through the public API (host buffers, pinned)
    e2e = None
    if not args.no_e2e:
        pts_pin = torch.from_numpy(np.ascontiguousarray(wl.points)).pin_memory()
        sess = R.sess
        prob, keep = sess.problem_for(rld.KernelMatrix(wl.spec, pts_pin), cfg.dtype, wl.path)
        c = make_config(cfg, n)
        inp = N.Inputs()
        inp.memory = N.HOST
        per = np.empty(s)
        res = N.Result()
        res.per_probe = per.ctypes.data_as(C.POINTER(C.c_double))

        def e2e_step():
            sess.handle.check(sess.lib.rld_logdet(sess.handle.ptr, C.byref(prob), C.byref(c), C.byref(inp),
                                                  C.byref(res)), "rld_logdet")

        for _ in range(max(1, args.warmup)):
            e2e_step()
        barrier(world)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            e2e_step()
        e1.record(stream)
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
        e2e_s = max_over_ranks(e0.elapsed_time(e1) * 1e-3, world)   # device clock, max over ranks
        e2e = {"value": per_step * args.steps / e2e_s, "unit": UNIT,
               "h2d_bytes_per_step": int(pts_pin.numel() * 8),
               "d2h_bytes_per_step": int(8 * (s + 3) + 4 * 8), "host_wall_s": wall}
        # restore the resident problem for any later use
        del keep

    # ---- informational: independent estimates from several host threads, each with its own
    # handle / stream / K copy (the harness's run_sweep(jobs=J)); not the headline value
    concurrent = None
    if world == 1 and not args.no_concurrent:
        import threading

        J, per = 4, max(2, args.steps // 2)
        Rs = [rld.ResidentMatrix(rld.KernelMatrix(wl.spec, wl.points), dtype=cfg.dtype, path=wl.path)
              for _ in range(J)]
        for Rj in Rs:
            Rj.estimate(cfg)
        torch.cuda.synchronize()
        ths = [threading.Thread(target=lambda Rj=Rj: [Rj.estimate(cfg) for _ in range(per)]) for Rj in Rs]
        t0 = time.perf_counter()
        for th in ths:
            th.start()
        for th in ths:
            th.join()
        dtc = time.perf_counter() - t0
        concurrent = {"jobs": J, "value": J * per / dtc, "unit": UNIT, "clock": "host wall",
                      "what": "J independent estimates at a time, one device handle per host thread"}
        del Rs

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
        "scaling": "strong" if sharded else "weak", "vs_baseline": None, "dtype": "f32" if cfg.dtype == "fp32" else "f64",
        "data": "synthetic",
        "config": workload_config(wl, world, sharded),
        "e2e": e2e,
        "gpu_launches": launches,
        "kv_products_per_step": products // max(1, args.steps),
        "phase_ms_last_step": {"precond": phases[1], "lanczos": phases[4], "solves": phases[5]},
        "roofline": roofline,
        "clocks": clocks,
        "estimate": est.value,
    }
    if concurrent is not None:
        line["concurrent"] = concurrent

    # ---- CPU baseline (rank 0, N = 1 only)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        threads = os.cpu_count() or 1
        secs, oest = cpu_estimate(wl, threads)
        line["cpu_baseline"] = {"value": 1.0 / secs, "unit": UNIT, "cores": threads, "kind": "port",
                                "sample": "1 full estimate of the same workload in float64 (oracle port, "
                                          "numpy/OpenBLAS, per-probe loop), K build excluded",
                                "cpu": cpu_model()}
        line["parity"] = {"oracle_value": oest.value, "gpu_value": est.value,
                          "rel_diff": abs(est.value - oest.value) / abs(oest.value),
                          "tol": 1e-4 if cfg.dtype == "fp32" else 1e-6}
    if rank == 0:
        print(json.dumps(line), flush=True)
    barrier(world)
    return 0


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
