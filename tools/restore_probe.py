"""Restore breakdown on one GPU: one C2 checkpoint to disk, the
same-run O_DIRECT read roofline, then fp_ckpt_load_parallel (with and without
the CRC check) and fp_ckpt_load, each with its load statistics (setup, time
blocked on the own-shard reads). One JSON line per call.

    python tools/restore_probe.py [--dir DIR] [--reps 2]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2406_13768_b200 as fp  # noqa: E402
from workloads import config_specs, make_state  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--dir", default=os.path.join(os.environ.get("GRAFT_REPO_ROOT", "/tmp"),
                                              "fp_restore_probe"))
ap.add_argument("--cfg", default="c2_gpt3_1.3b")
ap.add_argument("--reps", type=int, default=2)
a = ap.parse_args()
os.makedirs(a.dir, exist_ok=True)
dev = torch.device("cuda", 0)
st = make_state(config_specs(a.cfg), dev)
ents = [(x.name, t, x.section, x.owner) for x, t in st]
torch.cuda.synchronize()
ck_dir = os.path.join(a.dir, "ckpt")
with fp.Checkpointer(dev) as ck:
    s = ck.save(ents, ck_dir)
img = s["image_bytes"]
rd = fp.io_bench(a.dir, img, read=True)
print(json.dumps({"what": "io_bench_read", "gbs": round(rd, 3), "bytes": img}), flush=True)


def timed(name, fn):
    for _ in range(a.reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        info = fn()
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        out = {"what": name, "s": round(dt, 4), "gbs": round(img / dt / 1e9, 3),
               "frac_of_read": round(img / dt / 1e9 / rd, 4)}
        out.update({k: (round(v, 4) if isinstance(v, float) else v) for k, v in (info or {}).items()})
        print(json.dumps(out), flush=True)


with fp.Checkpointer(dev) as ck:
    timed("load_parallel", lambda: ck.load_parallel(ents, ck_dir))
    timed("load", lambda: ck.load(ents, ck_dir))
with fp.Checkpointer(dev, no_crc=True) as ck:
    timed("load_parallel_no_crc", lambda: ck.load_parallel(ents, ck_dir))
with fp.Checkpointer(dev, ring_slots=8) as ck:
    timed("load_parallel_ring8", lambda: ck.load_parallel(ents, ck_dir))
os.system(f"rm -rf {a.dir}")
