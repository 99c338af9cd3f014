"""Summarise the ncu captures of scripts/capture_profiles.sh into profiles/<tag>_kv_ncu.json
(per-kernel DRAM traffic, pipe utilisation) and profiles/<tag>_bench_launches.txt."""
import csv
import io
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
UNITS = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "ns": 1e-9, "us": 1e-6, "ms": 1e-3,
         "s": 1.0, "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "hz": 1, "Khz": 1e3, "Mhz": 1e6, "Ghz": 1e9,
         "%": 1, "": 1, "register/thread": 1}
METRICS = {"gpu_time_s": "gpu__time_duration.sum", "dram_bytes_read": "dram__bytes_read.sum",
           "dram_bytes_write": "dram__bytes_write.sum",
           "dram_throughput_pct": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
           "tensor_pipe_active_pct": "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
           "fma_pipe_active_pct": "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
           "xu_pipe_inst_pct": "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
           "l2_throughput_pct": "lts__throughput.avg.pct_of_peak_sustained_elapsed",
           "sm_clock_hz": "sm__cycles_elapsed.avg.per_second", "registers": "launch__registers_per_thread",
           "issue_slots_busy_pct": "sm__inst_issued.avg.pct_of_peak_sustained_active"}


def raw(rep):
    out = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    return {r[0][i]: (r[2][i], r[1][i]) for i in range(len(r[0]))}


def main(tag, what):
    out = {}
    for name, desc in what.items():
        rep = ROOT / "gpurun_out" / f"{tag}_{name}.ncu-rep"
        if not rep.exists():
            continue
        d = raw(rep)
        rec = {"what": desc, "command": "ncu --set full --import-source on --clock-control none -k regex:kv_tc_kernel -c 1"}
        for key, metric in METRICS.items():
            if metric in d:
                val, unit = d[metric]
                rec[key] = float(val.replace(",", "")) * UNITS.get(unit, 1)
        if "dram_bytes_read" in rec:
            rec["dram_bytes_total"] = rec["dram_bytes_read"] + rec.get("dram_bytes_write", 0.0)
        out[name] = rec
    (ROOT / "profiles" / f"{tag}_kv_ncu.json").write_text(json.dumps(out, indent=1))
    launches = ROOT / "gpurun_out" / f"{tag}_bench_launches.csv"
    if launches.exists():
        txt = subprocess.run([sys.executable, str(ROOT / "scripts" / "launch_summary.py"), str(launches), "40"],
                             capture_output=True, text=True).stdout
        hdr = (f"# {tag} launch list: ncu --metrics gpu__time_duration.sum --clock-control none "
               f"python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e (config 2, fp32, r3)\n"
               "# cold-cache serialised launches: compare SHARES, not absolute times; includes the K build,\n"
               "# 3 estimates and the bench's live K x V timing loop\n")
        (ROOT / "profiles" / f"{tag}_bench_launches.txt").write_text(hdr + txt)
    print(json.dumps(out, indent=1))


WHAT = {
    "kv_c2_m32": "config 2 Lanczos shape: n=16384 fp32 stored K, m=s=32 vectors, 3xTF32",
    "kv_c2_m266": "config 2 sketch shape: n=16384 fp32 stored K, m=w=266 (3 column passes of 96, CTA pairs: cta_group::2 M=256), 3xTF32",
    "kv_c3_m64": "config 3 Lanczos shape: n=65536 fp32 stored K (17.2 GB), m=s=64, CTA pairs, 3xTF32",
    "otf_c5_n262144": "config 5 on-the-fly Matern-5/2 d=3 tiles, n=262144 (reduced), m=128",
    "otf_c4_n262144": "config 4 on-the-fly RBF d=3 tiles, n=262144 (full), m=64",
}

if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "r01", WHAT)
