import sys, json
sys.path.insert(0,'/root/reference/pkg/src')
from ratlogdet import bench as B
from dataclasses import asdict
out = {"record_fields": B.RECORD_FIELDS,
       "trial_seeds": [[sb, vi, tr, B.trial_seed(sb, vi, tr)] for sb in (0, 7) for vi in range(3) for tr in range(3)],
       "sweep": [asdict(c) for c in B.sweep_configs(B.SweepSpec("n", (200, 400), ("r1", "r3", "slq"), trials=2, seed_base=0))]}
print(json.dumps(out)[:300])
json.dump(out, open('/root/repo/tests/golden/harness.json','w'), indent=1)
