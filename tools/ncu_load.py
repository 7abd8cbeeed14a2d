"""One C2 save + parallel load (restore) for ncu captures of the load-path
kernels (fp_unpack_v4, the page-CRC check of each H2D'd chunk). /dev/shm, no
fsync. Not a bench number: timings under ncu are serialised.

    ncu --set full -k regex:"fp_unpack|fp_crc" -s 20 -c 4 -o gpurun_out/load python tools/ncu_load.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2406_13768_b200 as fp  # noqa: E402
from workloads import config_specs, make_state  # noqa: E402

d = "/dev/shm/fp_ncu_load"
dev = torch.device("cuda", 0)
st = make_state(config_specs("c2_gpt3_1.3b"), dev)
ents = [(x.name, t, x.section, x.owner) for x, t in st]
torch.cuda.synchronize()
with fp.Checkpointer(dev, no_fsync=True) as ck:
    ck.save(ents, d)
    ck.load_parallel(ents, d)
    torch.cuda.synchronize()
print("save + load_parallel ok")
os.system(f"rm -rf {d}")
