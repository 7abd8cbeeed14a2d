"""Kernel A/B by CUDA events: C2 checkpoints to /dev/shm (no fsync) with the
launch gate on, so the per-group events bracket the kernels alone (as in
bench.py). Prints one JSON line per variant:

    FP_BC_GROUPS=1 python tools/kernel_ab.py --pack bulk --reps 3
"""
import argparse
import json
import os
import sys

os.environ.setdefault("FP_LAUNCH_GATE", "1")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2406_13768_b200 as fp  # noqa: E402
from workloads import config_specs, make_state  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--cfg", default="c2_gpt3_1.3b")
ap.add_argument("--pack", default="v4")
ap.add_argument("--dir", default="/dev/shm/fp_ab")
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--tag", default="")
ap.add_argument("--no-crc", action="store_true", help="pack only (bulk: fp_pack_bulk)")
ap.add_argument("--pack-mib", type=int, default=1024, help="bytes per pack launch (MiB)")
a = ap.parse_args()
peak = 6538.3
try:
    pk = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                     "MEASURED_PEAKS.json")))
    peak = float(pk.get("hbm_gbs", peak))
except Exception:
    pass
dev = torch.device("cuda", 0)
st = make_state(config_specs(a.cfg), dev)
ents = [(x.name, t, x.section, x.owner) for x, t in st]
torch.cuda.synchronize()
rows = []
with fp.Checkpointer(dev, pack=a.pack, no_fsync=True, no_crc=a.no_crc,
                     pack_bytes=a.pack_mib << 20) as ck:
    for i in range(a.reps + 1):
        s = ck.save(ents, a.dir)
        if i:
            rows.append(s)
os.system(f"rm -rf {a.dir}")
n = sum(s["pack_launches"] for s in rows)
b = sum(s["pack_bytes"] for s in rows)
pms = sum(s["pack_ms"] for s in rows)
cms = sum(s.get("crc_ms", 0.0) for s in rows)
out = {"tag": a.tag or a.pack, "pack": a.pack, "env_groups": os.environ.get("FP_BC_GROUPS"),
       "pack_mib": a.pack_mib,
       "launches": n, "pack_us": round(1e3 * pms / n, 2), "crc_us": round(1e3 * cms / n, 2),
       "pack_frac": round(2 * b / (pms / 1e3) / 1e9 / peak, 4),
       "total_us": round(1e3 * (pms + cms) / n, 2),
       "total_frac_2B": round(2 * b / ((pms + cms) / 1e3) / 1e9 / peak, 4),
       "crc_valid": all(s.get("crc_valid") for s in rows),
       "crc": [hex(s.get("shard_crc32", 0)) for s in rows]}
print(json.dumps(out), flush=True)
