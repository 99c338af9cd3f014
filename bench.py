"""Benchmark: log-det estimates per second on BASELINE config 3 (n = 65536 points
uniform in [0,1]^2, Matern-5/2 l = 0.05, noise 1e-2, stored K in HBM, r3, rand-SVD
l = 512, 64 Gaussian probes, t = 20), in float64 -- the reference's arithmetic, so the
reference arm is like-for-like -- one JSON line on rank 0.  Config 3 is the largest
BASELINE configuration a single B200 completes within the driver's limits (config 5
takes minutes per estimate); the line also carries config 3 in fp32 (BASELINE's
stated precision) as an extra key.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--config 3] [--dtype fp32|fp64] [--algorithm r3] [--n N]

A step is one full estimate (preconditioner build + s-probe Lanczos +
multishift solves + Hutchinson mean) -- the reference's timer scope
(src/estimators.py:81-96).

* ``value``: estimates/s with K resident in HBM (float64: 30 GB of int8 slices, far
  larger than the 126 MB L2, so every product streams K from HBM), CUDA events on
  the handle's stream around exactly K steps, max over ranks.
* ``e2e``: the same metric through the C ABI call the public API makes, with host
  buffers -- every step uploads the points from pinned memory, builds K on the
  GPU, regenerates the reference's probe / sketch streams on the GPU, runs the
  estimate and reads the result back.
* ``roofline``: the dominant kernel, timed live with CUDA events.  float64 stored
  (default): the int8-slice product at the sketch shape m = w (tensor-bound against
  the sustained int8 rate; work from rld_slice_stats), with the same kernel at the
  Lanczos shape m = s beside it (``roofline_lanczos``: HBM-bound on the slices
  read); RLD_FP64_PRODUCT=dmma: DMMA against the measured DMMA peak; float32 tiles:
  HBM, algorithmic bytes 4 n^2 (K) + 4 n s (operand) + 8 n s (result).
* extra keys: ``extra_fp32`` (config 3 in fp32: K as 3 int8 slices), ``extra_otf``
  (config 4 at full n, path on_the_fly, served from the cached sparse slice image;
  the on-the-fly kernel's own roofline beside it; config 5's product at n = 2^20),
  ``extra_e2e_dense`` (a dense float64 host M through rld_logdet).
* ``cpu_baseline``: the oracle port (float64 numpy restatement of the
  reference, per-probe loop like the reference) on this host's cores.  The
  reference's dense K does not fit host RAM at n = 65536, so the
  sample is the same configuration at n ~ 14336, extrapolated by n^2 (labelled).
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
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--n", type=int, default=None)
    ap.add_argument("--dtype", choices=["fp32", "fp64"], default=None)
    ap.add_argument("--algorithm", choices=["r1", "r3", "r5"], default=None)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-concurrent", action="store_true", help="skip the informational concurrent-estimates run")
    ap.add_argument("--mode", choices=["sharded", "replicas"], default="sharded",
                    help="multi-GPU: row-shard one estimate (default) or run independent replicas")
    ap.add_argument("--no-extra", action="store_true", help="skip the extra config-3 fp32 measurement")
    ap.add_argument("--cpu-sample-n", type=int, default=None,
                    help="n of the CPU sample (extrapolated by n^2 to the workload's n); default: the largest "
                         "n <= 16384 whose K reference steps fit in ~200 s")
    return ap.parse_args()


def load_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), float(d["bf16_tflops"]), "measured"
    return 6650.0, 1590.0, "fallback"


def load_pipe_peaks():
    """Measured compute-pipe peaks of this pool's B200 (scripts/pipe_peaks.cu, committed)."""
    for name in ("r02c_pipe_peaks.json", "r02_pipe_peaks.json"):
        p = ROOT / "profiles" / name
        if p.exists():
            return json.loads(p.read_text())
    return {}


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


def ncu_traffic(key):
    """DRAM bytes (read + write) per launch of the dominant kernel at exactly this shape, from the
    committed ncu --set full summary (profiles/traffic.json: {key: {"dram_bytes": B, "source": f}}).
    The key names the kernel, dtype, path and shape; no entry -> None (never a neighbour's number)."""
    f = ROOT / "profiles" / "traffic.json"
    try:
        rec = json.loads(f.read_text()).get(key)
    except Exception:
        return None, None
    if rec and "dram_bytes" in rec:
        return rec["dram_bytes"], rec.get("source", f.name)
    return None, None


def workload_for(args, dtype=None):
    from paper_2405_03474_b200.workloads import baseline

    dtype = dtype or args.dtype or ("fp64" if args.config == 3 else None)
    return baseline(args.config, n=args.n, algorithm=args.algorithm, dtype=dtype)


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


def cpu_sample(wl, args):
    """(workload to time on the CPU, factor from its seconds to the full workload's seconds, label)."""
    from paper_2405_03474_b200.workloads import baseline

    cfg = wl.config
    ns = args.cpu_sample_n
    if ns is None:   # ~25 s per n = 16384 sample on the GPU box's 16 host cores (r02 measurement)
        ns = int(16384 * min(1.0, (200.0 / (25.0 * max(1, args.steps))) ** 0.5)) // 1024 * 1024
        ns = max(4096, min(16384, ns))
    if wl.n <= ns:
        return replace(wl, config=replace(cfg, dtype="fp64")), 1.0, "the full workload"
    idx = int(wl.name.replace("config", ""))
    sw = baseline(idx, n=ns, algorithm=cfg.algorithm, dtype="fp64", rank=cfg.precond.rank,
                  num_probes=cfg.num_probes)
    f = (wl.n / ns) ** 2
    return sw, f, (f"the same configuration at n = {ns} (the reference's dense float64 K does not fit host RAM "
                   f"at n = {wl.n}), seconds extrapolated by (n / {ns})^2 = {f:.0f}: EXTRAPOLATED")


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
                        f"{cfg.probe_kind} t={cfg.lanczos_iters} q={cfg.precond.num_iters} "
                        f"{'on-the-fly' if wl.path == 'on_the_fly' else 'stored'} K ({cfg.dtype})",
            "l2": ("inputs larger than L2 (K = %.2f GB)" % (es * n * n / 1e9)) if wl.path != "on_the_fly" else
                  ("K never stored; the float64 probe / sketch blocks (%.0f MB .. %.0f MB) exceed L2"
                   % (8 * n * s / 1e6, 8 * n * min(cfg.precond.rank + 10, n) / 1e6)),
            "parallelism": (f"rows{world}" if sharded else f"replicas{world}") if world > 1 else "single"}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    threads = os.cpu_count() or 1
    os.environ["OPENBLAS_NUM_THREADS"] = str(threads)
    wl = workload_for(args)
    arm_config = workload_config(wl)
    sw, factor, label = cpu_sample(wl, args)
    warm = min(args.warmup, 1)
    steps = max(1, args.steps)   # exactly K steps, each a bounded sample (cpu_sample)
    for _ in range(warm):
        cpu_estimate(sw, threads)
    times = [cpu_estimate(sw, threads)[0] * factor for _ in range(steps)]
    total = sum(times)
    v = steps / total
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus, "steps": steps,
        "warmup": warm, "ms_per_step": 1e3 * total / steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": arm_config,
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": f"{steps} estimate(s) of {label}; oracle port (numpy/OpenBLAS float64, "
                                   f"per-probe loop like the reference), K build excluded",
                         "cpu": cpu_model()},
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
    roofline = roofline_for(wl, cfg, rows, n, s, kv_ms, world)
    # float64 stored K: the sketch products (m = w) run on the CRT kernel and take the most time of
    # any kernel (6 of the 26 products); their roofline is the headline one, the Lanczos product's
    # (HBM) is kept beside it
    roofline_lanczos = None
    stats = (C.c_int64 * 4)()
    if cfg.dtype == "fp64" and wl.path == "stored" and R.sess.lib.rld_slice_stats(R.sess.handle.ptr, stats) == 0 \
            and stats[0] > 0:
        blocks, slices, pairs, crt = (int(x) for x in stats)
        Vw = torch.randn(w, n, dtype=torch.float64, device="cuda")
        for _ in range(2):
            R.kv_apply(Vw)
        torch.cuda.synchronize()
        k0.record(stream)
        for _ in range(5):
            R.kv_apply(Vw)
        k1.record(stream)
        torch.cuda.synchronize()
        w_ms = k0.elapsed_time(k1) / 5
        roofline_lanczos = roofline_slices(rows, n, s, kv_ms, blocks, slices, pairs, "Lanczos block m=s")
        roofline = roofline_crt(rows, n, w, w_ms) if crt else roofline_slices(rows, n, w, w_ms, blocks, slices, pairs,
                                                                             "sketch block m=w")
        del Vw

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
    # handle / stream / K copy (the harness's run_sweep(jobs=J)); not the headline value.  Only
    # where J copies of K fit in HBM.
    concurrent = None
    if world == 1 and not args.no_concurrent and 4 * es * n * n < 0.5 * torch.cuda.get_device_properties(0).total_memory:
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
        **({"roofline_lanczos": roofline_lanczos} if roofline_lanczos else {}),
        "estimate": est.value,
    }
    if concurrent is not None:
        line["concurrent"] = concurrent
    line["parity"] = parity_vs_golden(wl, est.value)
    del R
    torch.cuda.empty_cache()

    # ---- extra: the same configuration in BASELINE's stated fp32 (stored fp32 K, 3xTF32 products)
    if args.config == 3 and cfg.dtype == "fp64" and not args.no_extra:
        line["extra_fp32"] = extra_fp32(args, rld, world, sharded, per_step)

    # ---- extra: config 4 at full n on the fly (fp32, fp16 3-term tensor-core products)
    if args.config == 3 and cfg.dtype == "fp64" and not args.no_extra and world == 1:
        line["extra_otf"] = extra_otf(rld)
        line["extra_e2e_dense"] = extra_e2e_dense(rld)

    # ---- CPU baseline (rank 0, N = 1 only)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        threads = os.cpu_count() or 1
        sw, factor, label = cpu_sample(wl, args)
        secs, oest = cpu_estimate(sw, threads)
        line["cpu_baseline"] = {"value": 1.0 / (secs * factor), "unit": UNIT, "cores": threads, "kind": "port",
                                "sample": f"1 estimate of {label}; oracle port (numpy/OpenBLAS float64, per-probe "
                                          f"loop like the reference), K build excluded",
                                "sample_seconds": secs, "cpu": cpu_model()}
    if rank == 0:
        print(json.dumps(line), flush=True)
    barrier(world)
    return 0


def roofline_for(wl, cfg, rows, n, s, kv_ms, world):
    """Roofline of the dominant kernel (K x block, Lanczos shape m = s), SURVEY.md §8(d)."""
    es = 4 if cfg.dtype == "fp32" else 8
    pipe = load_pipe_peaks()
    ozaki = cfg.dtype == "fp64" and wl.path == "stored" and os.environ.get("RLD_FP64_PRODUCT") != "dmma"
    key = f"kv_product|{cfg.dtype}{'-int8slices' if ozaki else ''}|{wl.path}|n={n}|rows={rows}|m={s}"
    traffic, traffic_src = ncu_traffic(key)
    if ozaki:
        # float64-accurate product on the INT8 tensor cores (kv_ozaki.cu): K streams as its 7 exact
        # int8 slices (base-256 digits), 7 bytes per entry; 28 slice-pair int8 products per useful
        # multiply-add (3.1e13 int8 ops at config 3, m = 64: under the int8 tensor peak's time), so
        # HBM bounds it
        alg_bytes = 7 * rows * n + 8 * n * s + 8 * rows * s
        hbm_peak, _, peak_kind = load_peaks()
        achieved = alg_bytes / (kv_ms * 1e-3) / 1e9
        return {"bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s", "frac": achieved / hbm_peak,
                "traffic": traffic, "traffic_source": traffic_src, "traffic_key": key,
                "kernel": f"kv_product (tcgen05 kind::i8 on exact int8 slices of float64 K, m=s={s}, {rows} rows)",
                "kernel_ms": kv_ms, "alg_bytes": alg_bytes, "equiv_fp64_tflops": 2.0 * rows * n * s / (kv_ms * 1e-3) / 1e12,
                "int8_ops": 28 * 2.0 * rows * n * (-(-s // 64) * 64),
                "int8_tensor_frac": 28 * 2.0 * rows * n * (-(-s // 64) * 64) / (kv_ms * 1e-3) / 1e12
                / pipe.get("i8_ss_n128", {}).get("tops", 4555.6),
                "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({peak_kind})"}
    if wl.path == "stored" and cfg.dtype == "fp32":
        alg_bytes = es * rows * n + 4 * n * s + 8 * rows * s
        hbm_peak, _, peak_kind = load_peaks()
        achieved = alg_bytes / (kv_ms * 1e-3) / 1e9
        return {"bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s", "frac": achieved / hbm_peak,
                "traffic": traffic, "traffic_source": traffic_src, "traffic_key": key,
                "kernel": f"kv_product (tcgen05 3xTF32, Lanczos shape m=s={s}, {rows} rows of K)", "kernel_ms": kv_ms,
                "alg_bytes": alg_bytes, "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({peak_kind})"}
    useful = 2.0 * rows * n * s
    if cfg.dtype == "fp64":
        # FP64 tensor cores (DMMA, kv_dmma.cu): 2 n^2 s flops per product (8 flop/B at s = 32:
        # above the FP64 ridge, so the FP64 pipe bounds it, not HBM)
        kind, work = "fp64-tensor", useful
        if "dmma_tflops" in pipe:
            peak, src = pipe["dmma_tflops"], "profiles/r02_pipe_peaks.json dmma (measured)"
        else:
            peak, src = pipe.get("dfma_tflops", 36.36), "profiles/r01_pipe_peaks.json dfma (measured)"
        alg_bytes = es * rows * n + 8 * n * s + 8 * rows * s
    else:   # on the fly, 3xTF32 tensor-core MMAs: three products per useful one
        kind, work = "tensor", 3.0 * useful
        peak, src = pipe.get("tf32_ts_n128", {}).get("tflops", 1115.0), "pipe peaks tf32 N=128 (measured)"
        alg_bytes = None
    ach = work / (kv_ms * 1e-3) / 1e12
    return {"bound": kind, "achieved": ach, "peak": peak, "unit": "TFLOP/s", "frac": ach / peak,
            "traffic": traffic, "traffic_source": traffic_src, "traffic_key": key, "alg_bytes": alg_bytes,
            "kernel": f"kv_product ({wl.path}, {cfg.dtype}, m=s={s}, {rows} rows)", "kernel_ms": kv_ms,
            "alg_flops": work, "useful_flops": useful, "peak_source": src}


def parity_vs_golden(wl, value):
    """The estimate against the committed float64 oracle value of the same workload (full-size
    configs 3-5: tests/golden/golden_large.json, matrix-free oracle; configs 1-2: golden.json,
    the unmodified reference)."""
    g = ROOT / "tests" / "golden"
    cfg = wl.config
    ref = None
    try:
        if wl.n == {1: 2048, 2: 16384}.get(int(wl.name[-1])):
            for c in json.loads((g / "golden.json").read_text()):
                if c["name"] == f"{wl.name}_{cfg.algorithm}":
                    ref, src = c["value"], "tests/golden/golden.json (unmodified reference)"
        else:
            c = json.loads((g / "golden_large.json").read_text()).get(f"{wl.name}_full")
            if (c and c["n"] == wl.n and c["rank"] == cfg.precond.rank and c["num_probes"] == cfg.num_probes
                    and c["algorithm"] == cfg.algorithm and c["lanczos_iters"] == cfg.lanczos_iters
                    and c["num_iters"] == cfg.precond.num_iters):
                ref, src = c["value"], "tests/golden/golden_large.json (matrix-free float64 oracle)"
    except Exception:
        ref = None
    if ref is None:
        return None
    return {"oracle_value": ref, "gpu_value": value, "rel_diff": abs(value - ref) / abs(ref),
            "tol": 1e-4 if cfg.dtype == "fp32" else 1e-6, "source": src}


def extra_fp32(args, rld, world, sharded, per_step):
    """Config 3 in fp32 (BASELINE's stated precision): stored K -- on one GPU as 3 int8 slices from
    the Morton-ordered points (INT8 tensor cores), sharded as fp32 tiles (3xTF32 / fp16 tensor-core
    products); 3 timed estimates after 2 warm-ups, CUDA events, max over ranks."""
    import torch

    wl = workload_for(args, dtype="fp32")
    cfg = wl.config
    R = rld.ResidentMatrix(rld.KernelMatrix(wl.spec, wl.points), dtype="fp32", path=wl.path, shard=sharded)
    st = torch.cuda.ExternalStream(R.sess.handle.stream)
    for _ in range(2):
        est = R.estimate(cfg)
    barrier(world)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    K = 3
    for _ in range(K):
        est = R.estimate(cfg)
    e1.record(st)
    torch.cuda.synchronize()
    ms = max_over_ranks(e0.elapsed_time(e1), world)
    from paper_2405_03474_b200.parallel import shard_bounds

    r0, r1 = shard_bounds(wl.n, world, int(os.environ.get("RANK", "0"))) if sharded else (0, wl.n)
    V = torch.randn(cfg.num_probes, wl.n, dtype=torch.float64, device="cuda")
    for _ in range(2):
        R.kv_apply(V)
    torch.cuda.synchronize()
    k0, k1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    k0.record(st)
    for _ in range(10):
        R.kv_apply(V)
    k1.record(st)
    torch.cuda.synchronize()
    import ctypes as C

    stats = (C.c_int64 * 4)()
    kv_ms = k0.elapsed_time(k1) / 10
    if R.sess.lib.rld_slice_stats(R.sess.handle.ptr, stats) == 0 and stats[0] > 0:
        # float32 K from Morton-ordered points: 3 int8 slices on the INT8 tensor cores (kv_ozaki.cu)
        roof = roofline_slices(r1 - r0, wl.n, cfg.num_probes, kv_ms, int(stats[0]), int(stats[1]), int(stats[2]),
                               "Lanczos block m=s", kslices=3)
    else:
        roof = roofline_for(wl, cfg, r1 - r0, wl.n, cfg.num_probes, kv_ms, world)
    out = {"value": per_step * K / (ms * 1e-3), "unit": UNIT, "ms_per_step": ms / K, "dtype": "f32",
           "config": workload_config(wl, world, sharded),
           "roofline": roof, "phase_ms_last_step": dict(zip(("precond", "lanczos"), (est.phase_ms[1], est.phase_ms[4]))),
           "parity": parity_vs_golden(wl, est.value)}
    del R
    torch.cuda.empty_cache()
    return out


def roofline_slices(rows, n, m, ms, blocks, slices, pairs, what, kslices=7):
    """The float64 product on exact int8 slices (csrc/kv_ozaki.cu) with its all-zero leading slices
    skipped (points in Morton order): algorithmic bytes = the K slices actually read (rld_slice_stats)
    plus V in and Y out; int8 work = the slice pairs multiplied, each a 128 x 64 x 32 MMA per block
    and 64-vector pass.  Both fractions are reported; the bound is the larger."""
    pipe = load_pipe_peaks()
    hbm_peak, _, peak_kind = load_peaks()
    passes = -(-m // 64)
    alg_bytes = 4096 * slices + 8 * n * m + 8 * rows * m
    ops = 2.0 * 128 * 64 * 32 * pairs * passes
    rec = pipe.get("i8_ss_n256_random_sustained", {})
    i8_peak = rec.get("tops", pipe.get("i8_ss_n256", {}).get("tops", 4576.0))
    t = ms * 1e-3
    f_hbm, f_t = alg_bytes / t / 1e9 / hbm_peak, ops / t / 1e12 / i8_peak
    key = f"kv_product|{'fp64' if kslices == 7 else 'fp32'}-int8slices|stored|n={n}|rows={rows}|m={m}"
    traffic, traffic_src = ncu_traffic(key)
    tot_s, tot_p, kname = (7, 28, "float64 K") if kslices == 7 else (3, 9, "float32 K (24 bits of the row scale, 3 x 4 slices)")
    common = {"traffic": traffic, "traffic_source": traffic_src, "traffic_key": key, "kernel_ms": ms,
              "kernel": f"kv_product (tcgen05 kind::i8 on exact int8 slices of {kname}, {what}={m}, {rows} rows; "
                        f"{slices / blocks:.2f} of {tot_s} slices (8-bit digits) and {pairs / blocks:.1f} of {tot_p} pairs per "
                        f"block after skipping all-zero leading slices)",
              "alg_bytes": alg_bytes, "int8_ops": ops, "hbm_frac": f_hbm, "int8_tensor_frac": f_t,
              "equiv_fp64_tflops": 2.0 * rows * n * m / t / 1e12,
              "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({peak_kind}); int8: profiles/r02c_pipe_peaks.json "
                             f"i8_ss_n256_random_sustained (measured)"}
    if f_t >= f_hbm:
        return {"bound": "tensor", "achieved": ops / t / 1e12, "peak": i8_peak, "unit": "TOPS (int8)", "frac": f_t,
                **common}
    return {"bound": "hbm", "achieved": alg_bytes / t / 1e9, "peak": hbm_peak, "unit": "GB/s", "frac": f_hbm, **common}


def roofline_crt(rows, n, w, ms):
    """The float64 sketch product (csrc/kv_crt.cu): 15 modular int8 GEMMs (CRT), tensor-bound.  The
    time covers the whole product call (V residues, the GEMM, the CRT reconstruction); the peak is
    the int8 rate on random operand bytes sustained for ~4.7 s (the power-capped clock a long step
    runs at; profiles/r02c_pipe_peaks.json)."""
    pipe = load_pipe_peaks()
    ops = 15 * 2.0 * rows * n * w
    rec = pipe.get("i8_ss_n256_random_sustained", {})
    peak, src = (rec["tops"], "profiles/r02c_pipe_peaks.json i8_ss_n256_random_sustained (measured)") if rec else (
        pipe.get("i8_ss_n256", {}).get("tops", 4576.0), "pipe peaks i8_ss_n256 (measured, burst)")
    ach = ops / (ms * 1e-3) / 1e12
    key = f"kv_product|fp64-crt|stored|n={n}|rows={rows}|m={w}"
    traffic, traffic_src = ncu_traffic(key)
    burst = pipe.get("i8_ss_n256_random_burst", {}).get("tops")
    return {"bound": "tensor", "achieved": ach, "peak": peak, "unit": "TOPS (int8)", "frac": ach / peak,
            "frac_of_burst": ach / burst if burst else None, "traffic": traffic, "traffic_source": traffic_src,
            "traffic_key": key, "alg_bytes": 15 * rows * n + 8 * n * w + 8 * rows * w,
            "kernel": f"kv_crt (15 modular tcgen05 kind::i8 GEMMs + CRT, float64 sketch product, m=w={w}, {rows} rows)",
            "kernel_ms": ms, "int8_ops": ops, "equiv_fp64_tflops": 2.0 * rows * n * w / (ms * 1e-3) / 1e12,
            "peak_source": src}


def roofline_otf(wl, n, m, kv_ms, nt):
    """On-the-fly product (csrc/kv_otf.cu): per K entry 3 fp16 tensor products of width NT (the
    padded pass width), 1 (RBF) or 2 (Matern: sqrt + ex2) MUFU ops, and the FP32-pipe generation
    work; each pipe's minimum time at its measured peak, the largest is the bound."""
    pipe = load_pipe_peaks()
    entries = float(n) * n
    passes = -(-m // nt)
    # the tensor ceiling at the MMA width the kernel issues (N = 64 MMAs take 44.6 cycles, not 32)
    pk_name = f"f16_ts_n{max(64, min(nt, 128)) if nt != 32 else 64}"
    f16_peak = pipe.get(pk_name, {}).get("tflops", 2230.0)
    f16_src = f"profiles pipe peaks {pk_name} (measured)" if pk_name in pipe else "nominal 2.25 PF/s"
    tensor_work = 3 * 2.0 * entries * passes * nt
    mufu_ops = entries * passes * (1 if wl.spec.family == "rbf" else 2)
    mufu_peak = pipe.get("mufu_ex2_gops", 4630.0)
    t_tensor = tensor_work / (f16_peak * 1e12)
    t_mufu = mufu_ops / (mufu_peak * 1e9)
    bound, t_min = ("tensor", t_tensor) if t_tensor >= t_mufu else ("mufu", t_mufu)
    key = f"kv_product|fp32-f16|on_the_fly|n={n}|rows={n}|m={m}"
    traffic, traffic_src = ncu_traffic(key)
    return {"bound": bound, "achieved": (tensor_work if bound == "tensor" else mufu_ops) / (kv_ms * 1e-3)
            / (1e12 if bound == "tensor" else 1e9),
            "peak": f16_peak if bound == "tensor" else mufu_peak, "unit": "TFLOP/s" if bound == "tensor" else "Gop/s",
            "frac": t_min / (kv_ms * 1e-3), "tensor_frac": t_tensor / (kv_ms * 1e-3),
            "mufu_frac": t_mufu / (kv_ms * 1e-3), "traffic": traffic, "traffic_source": traffic_src,
            "traffic_key": key, "kernel": f"kv_otf (tcgen05 kind::f16, 3 fp16 products, on the fly, m={m}, NT={nt})",
            "kernel_ms": kv_ms, "tensor_work_flops": tensor_work, "mufu_ops": mufu_ops,
            "useful_tflops": 2.0 * entries * m / (kv_ms * 1e-3) / 1e12,
            "peak_source": f"{f16_src}; MUFU mufu_ex2_gops (measured)"}


def extra_otf(rld):
    """BASELINE config 4 at full n = 262144 (fp32, path on_the_fly): 2 timed estimates after 1
    warm-up, and the K.V product at the Lanczos shape (m = 64), CUDA events.  By default the library
    serves this problem from its cached sparse 3-slice image (78 GB: the clustered points leave
    most blocks empty; rld_api.cu prepare); the product with K regenerated per call
    (RLD_OTF_CACHE=0, csrc/kv_otf.cu) is timed beside it with its per-pipe roofline."""
    import torch

    from paper_2405_03474_b200.workloads import baseline

    wl = baseline(4)
    cfg = wl.config
    R = rld.ResidentMatrix(rld.KernelMatrix(wl.spec, wl.points), dtype="fp32", path="on_the_fly")
    st = torch.cuda.ExternalStream(R.sess.handle.stream)
    est = R.estimate(cfg)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    K = 2
    e0.record(st)
    for _ in range(K):
        est = R.estimate(cfg)
    e1.record(st)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / K
    m = cfg.num_probes
    V = torch.randn(m, wl.n, dtype=torch.float64, device="cuda")
    R.kv_apply(V)
    torch.cuda.synchronize()
    k0, k1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    k0.record(st)
    for _ in range(10):
        R.kv_apply(V)
    k1.record(st)
    torch.cuda.synchronize()
    nt = 32 if m <= 32 else (64 if m <= 64 else 128)
    kv_ms = k0.elapsed_time(k1) / 10
    import ctypes as C

    stats = (C.c_int64 * 4)()
    cached = R.sess.lib.rld_slice_stats(R.sess.handle.ptr, stats) == 0 and stats[0] > 0
    out = {"value": 1e3 / ms, "unit": UNIT, "ms_per_step": ms, "dtype": "f32",
           "config": workload_config(wl, 1, False),
           "served_from": "cached sparse int8-slice image (%.1f GB)" % (stats[1] * 4096 / 1e9) if cached
                          else "K regenerated on the fly",
           "phase_ms_last_step": {"precond": est.phase_ms[1], "lanczos": est.phase_ms[4]},
           "roofline": roofline_slices(wl.n, wl.n, m, kv_ms, int(stats[0]), int(stats[1]), int(stats[2]),
                                       "Lanczos block m=s", kslices=3) if cached
                       else roofline_otf(wl, wl.n, m, kv_ms, nt),
           "parity": parity_vs_golden(wl, est.value)}
    del R
    torch.cuda.empty_cache()
    if cached:   # the on-the-fly kernel itself on the same problem
        os.environ["RLD_OTF_CACHE"] = "0"
        try:
            R = rld.ResidentMatrix(rld.KernelMatrix(wl.spec, wl.points), dtype="fp32", path="on_the_fly")
            st = torch.cuda.ExternalStream(R.sess.handle.stream)
            R.kv_apply(V)
            torch.cuda.synchronize()
            k0.record(st)
            for _ in range(5):
                R.kv_apply(V)
            k1.record(st)
            torch.cuda.synchronize()
            out["roofline_on_the_fly_kernel"] = roofline_otf(wl, wl.n, m, k0.elapsed_time(k1) / 5, nt)
            del R
        finally:
            del os.environ["RLD_OTF_CACHE"]
    del V
    torch.cuda.empty_cache()
    # config 5's kernel and points at full n = 2^20: the K.V product at the Lanczos shape (m = 128),
    # Morton order with the far-field k-steps skipped (a full estimate takes ~34 s: not timed here)
    wl5 = baseline(5)
    R5 = rld.ResidentMatrix(rld.KernelMatrix(wl5.spec, wl5.points), dtype="fp32", path="on_the_fly")
    st5 = torch.cuda.ExternalStream(R5.sess.handle.stream)
    V5 = torch.randn(wl5.config.num_probes, wl5.n, dtype=torch.float64, device="cuda")
    R5.kv_apply(V5)
    torch.cuda.synchronize()
    k0.record(st5)
    for _ in range(3):
        R5.kv_apply(V5)
    k1.record(st5)
    torch.cuda.synchronize()
    ms5 = k0.elapsed_time(k1) / 3
    n5, m5 = wl5.n, wl5.config.num_probes
    out["config5_product"] = {"workload": workload_config(wl5, 1, False)["workload"], "m": m5, "ms": ms5,
                              "dense_equiv_tflops": 2.0 * n5 * n5 * m5 / (ms5 * 1e-3) / 1e12,
                              "what": "K.V with K generated on the fly, points in Morton order, (tile, k-step) pairs "
                                      "with exactly-zero fp16 operands skipped (csrc/kv_otf.cu); CUDA events"}
    del R5, V5
    torch.cuda.empty_cache()
    return out


def extra_e2e_dense(rld):
    """The reference's callers pass a dense float64 M: BASELINE config 2 (n = 16384, 2.15 GB) from
    pinned host memory through rld_logdet every step -- the H2D copy, the int8 slice image and CRT
    residues of M, the estimate and the read-back are all inside the timed region (CUDA events on
    the handle's stream; 1 warm-up, 3 steps)."""
    import ctypes as C

    import torch

    from paper_2405_03474_b200 import _native as N
    from paper_2405_03474_b200._session import Session
    from paper_2405_03474_b200.estimators import make_config
    from paper_2405_03474_b200.workloads import baseline

    wl = baseline(2, dtype="fp64")
    cfg = replace(wl.config, dtype="fp64", path="stored")
    Kd = rld.build_covariance(wl.spec, wl.points, dtype="fp64")
    Kh = torch.empty(Kd.shape, dtype=torch.float64, pin_memory=True)
    Kh.copy_(Kd)
    del Kd
    torch.cuda.empty_cache()
    sess = Session()
    prob, keep = sess.problem_for(Kh, "fp64", "stored")
    c = make_config(cfg, wl.n)
    inp = N.Inputs()
    inp.memory = N.HOST
    per = np.empty(cfg.num_probes)
    res = N.Result()
    res.per_probe = per.ctypes.data_as(C.POINTER(C.c_double))

    def step():
        sess.handle.check(sess.lib.rld_logdet(sess.handle.ptr, C.byref(prob), C.byref(c), C.byref(inp), C.byref(res)),
                          "rld_logdet")

    step()
    stream = torch.cuda.ExternalStream(sess.handle.stream)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    K = 3
    for _ in range(K):
        step()
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / K
    out = {"value": 1e3 / ms, "unit": UNIT, "ms_per_step": ms, "dtype": "f64",
           "config": {"workload": workload_config(wl, 1, False)["workload"].replace("stored K", "dense host M"),
                      "input": "dense float64 M (2.15 GB) in pinned host memory, copied every step"},
           "h2d_bytes_per_step": int(8 * wl.n * wl.n), "d2h_bytes_per_step": int(8 * (cfg.num_probes + 3)),
           "phase_ms_last_step": {"precond": res.phase_ms[1], "lanczos": res.phase_ms[4],
                                  "h2d_and_prepare": ms - res.phase_ms[7]},
           "parity": parity_vs_golden(replace(wl, config=cfg), res.value)}
    del keep, Kh
    torch.cuda.empty_cache()
    return out


def spawn_ranks(args):
    """`--gpus N` outside torchrun: launch N ranks with torch.distributed.run on this node (one
    process per GPU, NCCL), after checking N GPUs are visible.  Rank 0's JSON line passes through."""
    import torch

    have = torch.cuda.device_count()
    if have < args.gpus:
        print(json.dumps({"error": f"--gpus {args.gpus} but only {have} CUDA device(s) visible"}), flush=True)
        return 2
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), str(ROOT / "bench.py"), *sys.argv[1:]]
    return subprocess.call(cmd)


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return spawn_ranks(args)
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
