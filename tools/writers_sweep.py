"""Writer-count sweep on one B200 (the single-box analog of the paper's
parallel-write experiments, §5.3 P:595-601 / P:628-633, and of the
writer subsets of §4.2).

k DP ranks run as threads of one process, each with its own context (pinned
ring, io_uring, helper thread) over the SAME device copy of the C2 state, and
checkpoint the 21 GB image together: with writer_stride s only ranks 0, s, 2s,
... write. Reports aggregate GB/s (image bytes / slowest rank's begin->wait).

    python tools/writers_sweep.py [--ks 1,2,4,8] [--strides 1,2,4]
"""
import argparse
import json
import os
import shutil
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2406_13768_b200 as fp  # noqa: E402
from workloads import config_specs, make_state  # noqa: E402


class Comm:
    def __init__(self, sh, rank):
        self.sh, self.rank, self.world = sh, rank, sh["k"]

    def _x(self, v, f):
        self.sh["slots"][self.rank] = v
        self.sh["bar"].wait()
        out = f(self.sh["slots"])
        self.sh["bar"].wait()
        return out

    def allgather(self, vals):
        return self._x(list(vals), lambda s: [x for r in s for x in r])

    def allreduce_min(self, v):
        return self._x(v, min)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ks", default="1,2,4,8")
    ap.add_argument("--strides", default="1,2,4")
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--dir", default=os.path.join(os.environ.get("GRAFT_REPO_ROOT", "/tmp"), "wsweep"))
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    st = make_state(config_specs("c2_gpt3_1.3b"), dev)
    ents = [(s.name, t, s.section, s.owner) for s, t in st]
    torch.cuda.synchronize()
    res = []
    for k in [int(x) for x in a.ks.split(",")]:
        for stride in [int(x) for x in a.strides.split(",")]:
            if stride > 1 and stride >= k:
                continue
            shutil.rmtree(a.dir, ignore_errors=True)   # 2 generations of one config at a time
            sh = {"k": k, "slots": [None] * k, "bar": threading.Barrier(k)}
            cks = [fp.Checkpointer(dev, comm=Comm(sh, r), writer_stride=stride) for r in range(k)]
            times = []
            errors = []
            for rep in range(a.reps + 1):
                t = [0.0] * k

                def go(r):
                    t0 = time.perf_counter()
                    try:
                        cks[r].save(ents, os.path.join(a.dir, f"g{rep % 2}"))
                    except fp.FastPersistError as e:
                        errors.append(str(e))
                    t[r] = time.perf_counter() - t0
                ths = [threading.Thread(target=go, args=(r,)) for r in range(k)]
                for th in ths:
                    th.start()
                for th in ths:
                    th.join()
                if rep:
                    times.append(max(t))
            for c in cks:
                c.close()
            img = 21053362176
            r = {"k": k, "writer_stride": stride, "writers": len(range(0, k, stride)),
                 "latency_s": [round(x, 3) for x in times],
                 "aggregate_gbs": None if errors else round(img / min(times) / 1e9, 3),
                 "errors": errors[:2]}
            print(json.dumps(r), flush=True)
            res.append(r)
    os.system(f"rm -rf {a.dir}")
    os.makedirs("gpurun_out", exist_ok=True)
    with open("gpurun_out/writers_sweep.json", "w") as f:
        json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
