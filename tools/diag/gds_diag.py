"""GDS (FP_IO_GDS) diagnostic: one small checkpoint through cuFile with step
tracing (FP_DEBUG_GDS=1). Run under `timeout`."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

import paper_2406_13768_b200 as fp  # noqa: E402
from workloads import config_specs, make_state  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c1_tiny"
d = sys.argv[2] if len(sys.argv) > 2 else os.path.join(os.environ.get("GRAFT_REPO_ROOT", "/tmp"), "gds_diag")
dev = torch.device("cuda", 0)
st = make_state(config_specs(cfg), dev)
ents = [(s.name, t, s.section, s.owner) for s, t in st]
torch.cuda.synchronize()
print("state ready", flush=True)
t0 = time.time()
with fp.Checkpointer(dev, io_engine="gds") as ck:
    print("init", time.time() - t0, flush=True)
    s = ck.save(ents, d)
    print("saved", time.time() - t0, {k: s[k] for k in ("engine", "fallback", "image_bytes", "t_io_stall", "pack_launches")}, flush=True)
    back = [(n, torch.zeros_like(t), sec, own) for n, t, sec, own in ents]
    ck.load_parallel(back, d)
    torch.cuda.synchronize()
    print("loaded", time.time() - t0, all(torch.equal(a[1], b[1]) for a, b in zip(ents, back)), flush=True)
