"""Quick perf probe on the GPU box: storage roofline sweep + C2 checkpoint stats.

    python tools/quick_perf.py [--dir DIR] [--cfg c2_gpt3_1.3b]
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


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--dir", default=os.path.join(os.environ.get("GRAFT_REPO_ROOT", "/tmp"),
                                                  "fp_quick"))
    ap.add_argument("--cfg", default="c2_gpt3_1.3b")
    ap.add_argument("--io-bytes", type=float, default=4e9)
    ap.add_argument("--reps", type=int, default=3)
    a = ap.parse_args()
    os.makedirs(a.dir, exist_ok=True)
    out = {"io": []}
    for qd, sqe, slots, slot in [(64, 1 << 20, 4, 64 << 20), (128, 1 << 20, 4, 64 << 20),
                                 (32, 4 << 20, 4, 64 << 20), (128, 4 << 20, 8, 64 << 20),
                                 (16, 8 << 20, 4, 64 << 20), (256, 256 << 10, 4, 64 << 20)]:
        g = fp.io_bench(a.dir, int(a.io_bytes), io_depth=qd, sqe_bytes=sqe, ring_slots=slots,
                        slot_bytes=slot)
        out["io"].append({"qd": qd, "sqe": sqe, "gbps": g})
        print("io", qd, sqe, round(g, 3), flush=True)
    dev = torch.device("cuda", 0)
    st = make_state(config_specs(a.cfg), dev)
    ents = [(s.name, t, s.section, s.owner) for s, t in st]
    torch.cuda.synchronize()
    for pack in ["v4", "bulk"]:
        with fp.Checkpointer(dev, pack=pack) as ck:
            for i in range(a.reps):
                t0 = time.time()
                s = ck.save(ents, os.path.join(a.dir, f"gen{i % 2}"))
                dt = time.time() - t0
                r = {"pack": pack, "s": dt, "GBps": s["image_bytes"] / dt / 1e9,
                     "pack_GBps": 2 * s["pack_bytes"] / (s["pack_ms"] / 1e3) / 1e9,
                     "d2h_GBps": s["pack_bytes"] / (s["d2h_ms"] / 1e3) / 1e9,
                     "stall": s["t_io_stall"], "fsync": s["t_fsync"],
                     "commit": s["t_commit"], "inflight": s["max_inflight"],
                     "launches": s["pack_launches"]}
                print(json.dumps(r), flush=True)
                out.setdefault("ckpt", []).append(r)
    # no-fsync, /dev/shm: the non-storage ceiling of the pipeline
    shm = "/dev/shm/fp_quick"
    with fp.Checkpointer(dev, no_fsync=True) as ck:
        for i in range(2):
            t0 = time.time()
            s = ck.save(ents, shm)
            dt = time.time() - t0
            print(json.dumps({"shm_GBps": s["image_bytes"] / dt / 1e9,
                              "pack_GBps": 2 * s["pack_bytes"] / (s["pack_ms"] / 1e3) / 1e9,
                              "d2h_GBps": s["pack_bytes"] / (s["d2h_ms"] / 1e3) / 1e9}),
                  flush=True)
    os.system(f"rm -rf {shm} {a.dir}")
    os.makedirs("gpurun_out", exist_ok=True)
    with open("gpurun_out/quick_perf.json", "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
