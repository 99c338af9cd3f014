import json, os, sys
from dataclasses import replace
sys.path.insert(0, os.getcwd())
import paper_2405_03474_b200 as rld
from paper_2405_03474_b200.workloads import baseline
g = json.load(open("tests/golden/golden_large.json"))["config3_full"]
wl = baseline(3)
M = rld.KernelMatrix(wl.spec, wl.points)
for label, env, path in [("stored fp32", {}, "stored"), ("otf sorted", {}, "on_the_fly"), ("otf unsorted", {"RLD_SORT": "0"}, "on_the_fly"),
                         ("otf tf32 unsorted", {"RLD_SORT": "0", "RLD_OTF_KIND": "tf32"}, "on_the_fly")]:
    for k in ("RLD_SORT", "RLD_OTF_KIND"):
        os.environ.pop(k, None)
    os.environ.update(env)
    e = rld.estimate_logdet(M, replace(wl.config, path=path))
    print(f"{label}: value rel {abs(e.value - g['value']) / abs(g['value']):.2e}  logdetP rel {abs(e.logdet_P - g['logdet_P']) / abs(g['logdet_P']):.2e}", flush=True)
