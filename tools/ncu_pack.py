"""One C2 checkpoint for ncu captures of the pack kernel (no fsync, /dev/shm
by default so the run is short). Not a bench number: timings under ncu are
serialised and replayed.

    ncu --set full -k regex:fp_pack -s 20 -c 3 -o gpurun_out/pack python tools/ncu_pack.py
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2406_13768_b200 as fp  # noqa: E402
from workloads import config_specs, make_state  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--cfg", default="c2_gpt3_1.3b")
ap.add_argument("--pack", default="v4")
ap.add_argument("--dir", default="/dev/shm/fp_ncu")
ap.add_argument("--slot-mib", type=int, default=64)
a = ap.parse_args()
dev = torch.device("cuda", 0)
st = make_state(config_specs(a.cfg), dev)
torch.cuda.synchronize()
with fp.Checkpointer(dev, pack=a.pack, no_fsync=True, slot_bytes=a.slot_mib << 20) as ck:
    s = ck.save([(x.name, t, x.section, x.owner) for x, t in st], a.dir)
print({k: s[k] for k in ("image_bytes", "pack_launches", "pack_ms", "d2h_ms")})
os.system(f"rm -rf {a.dir}")
