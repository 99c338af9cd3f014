import json, os, sys
from dataclasses import replace
sys.path.insert(0, os.getcwd())
import paper_2405_03474_b200 as rld
from paper_2405_03474_b200.workloads import baseline
from paper_2405_03474_b200.parallel import VirtualShards
gold = {c["name"]: c for c in json.load(open("tests/golden/golden.json"))}
print({k: (v["n"], v.get("sensitivity")) for k, v in gold.items() if "config4" in k})
ref = gold["config4_n4096_r5"]["value"]
wl = baseline(4, n=4096)
for kind in ("f16", "tf32"):
    os.environ["RLD_OTF_KIND"] = kind
    for G in (1, 2, 3):
        cfg = replace(wl.config, dtype="fp32", path="on_the_fly")
        M = rld.KernelMatrix(wl.spec, wl.points)
        if G == 1:
            v = rld.rstar_logdet(M, cfg)
        else:
            with VirtualShards(G) as vs:
                v = vs.run(lambda: rld.rstar_logdet(M, cfg))[0]
        print(kind, G, v.value, v.logdet_P, v.trace_term, "rel vs golden", abs(v.value - ref) / abs(ref) if ref else None, flush=True)
cfg = replace(wl.config, dtype="fp64", path="on_the_fly")
print("fp64", rld.rstar_logdet(rld.KernelMatrix(wl.spec, wl.points), cfg).value, "golden", ref)
