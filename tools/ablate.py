"""Ablations of the checkpoint path on one B200 (results -> gpurun_out/ablate_*.json).

  --what pack    C2 1.3B, pack impl {v4, bulk, host, ce} x pack_bytes {64, 256 MiB}
                 x sink {null, disk}: where the time goes with and without storage
                 (null = FP_IO_NULL: pack + D2H + ring ceiling).
  --what buffer  the paper's single-GPU micro-benchmark (§5.3):
                 checkpoint of one tensor of 16 MB / 512 MB with IO-buffer (ring slot)
                 sizes 2..128 MB, single (1 slot) vs double (2 slots) buffering.
  --what prio    per-iteration checkpoint overhead of C2 under a saturating GEMM
                 stream: pack stream priority {high, low} x pack CTAs {0 (all), 16}.
"""
import argparse
import json
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2406_13768_b200 as fp  # noqa: E402
from workloads import config_specs, make_state  # noqa: E402

DEV = torch.device("cuda", 0)


def save_rate(ents, path, reps=2, **cfg):
    with fp.Checkpointer(DEV, **cfg) as ck:
        ck.save(ents, path)                                   # warm (plan + file)
        out = []
        for _ in range(reps):
            t0 = time.perf_counter()
            s = ck.save(ents, path)
            dt = time.perf_counter() - t0
            out.append((dt, s))
    dt = statistics.median(x[0] for x in out)
    s = out[-1][1]
    r = {"GBps": round(s["image_bytes"] / dt / 1e9, 3), "s": round(dt, 4),
         "launches": s["pack_launches"]}
    if s["pack_ms"] > 0:
        r["pack_GBps"] = round(2 * s["pack_bytes"] / (s["pack_ms"] / 1e3) / 1e9, 1)
        r["pack_us_per_launch"] = round(1e3 * s["pack_ms"] / max(1, s["pack_launches"]), 2)
    if s["d2h_ms"] > 0:
        r["d2h_GBps"] = round(s["pack_bytes"] / (s["d2h_ms"] / 1e3) / 1e9, 2)
    r["io_stall_s"] = round(s["t_io_stall"], 3)
    return r


def ablate_pack(root):
    st = make_state(config_specs("c2_gpt3_1.3b"), DEV)
    ents = [(s.name, t, s.section, s.owner) for s, t in st]
    torch.cuda.synchronize()
    res = []
    for sink in ["null", "uring"]:
        for pack in ["v4", "bulk", "host", "ce"]:
            for pb in ([64, 256] if pack in ("v4", "bulk") else [64]):
                for crc in ([False, True] if pack == "v4" and pb == 256 else [False]):
                    r = save_rate(ents, os.path.join(root, "ab"), io_engine=sink, pack=pack,
                                  pack_bytes=pb << 20, reps=2 if sink == "null" else 1,
                                  no_crc=not crc)
                    r.update(sink=sink, pack=pack, pack_mib=pb, crc=crc)
                    print(json.dumps(r), flush=True)
                    res.append(r)
    return res


def ablate_buffer(root):
    res = []
    for mb in [16, 512]:
        t = torch.randn(mb * (1 << 20) // 4, device=DEV)
        ents = [("t", t, "other", -1)]
        for buf in [2, 4, 8, 16, 32, 64, 128]:
            if buf > mb:
                continue
            for slots in [1, 2]:
                r = save_rate(ents, os.path.join(root, "buf"), reps=5, ring_slots=slots,
                              slot_bytes=buf << 20, pack_bytes=buf << 20,
                              sqe_bytes=min(buf, 1) << 20)
                r.update(ckpt_mb=mb, io_buffer_mb=buf, mode="single" if slots == 1 else "double")
                print(json.dumps(r), flush=True)
                res.append(r)
    return res


def ablate_prio(root, t_fb, iters):
    st = make_state(config_specs("c2_gpt3_1.3b"), DEV)
    ents = [(s.name, t, s.section, s.owner) for s, t in st]
    by = {}
    for s, t in st:
        by.setdefault(s.section, []).append(t)
    n = 8192
    A = torch.randn(n, n, device=DEV, dtype=torch.bfloat16)
    C = torch.empty_like(A)
    for _ in range(5):
        torch.matmul(A, A, out=C)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(40):
        torch.matmul(A, A, out=C)
    torch.cuda.synchronize()
    ng = max(1, round(t_fb / ((time.perf_counter() - t0) / 40)))

    def opt():
        torch._foreach_mul_(by["exp_avg"], 0.9)
        torch._foreach_mul_(by["exp_avg_sq"], 0.999)
        torch._foreach_add_(by["master"], by["exp_avg"], alpha=-1e-8)
        for p, w in zip(by["param"], by["master"]):
            p.copy_(w)

    def loop(ck, its):
        out = []
        for i in range(its):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            for _ in range(ng):
                torch.matmul(A, A, out=C)
            if ck:
                ck.wait()
            opt()
            if ck:
                ck.begin(ents, os.path.join(root, "prio"))
            torch.cuda.synchronize()
            out.append(time.perf_counter() - t0)
        if ck:
            ck.wait()
        return out
    base = statistics.median(loop(None, iters + 1)[1:])
    res = [{"mode": "no_ckpt", "iter_s": round(base, 4), "gemms": ng}]
    print(json.dumps(res[0]), flush=True)
    for prio in ["high", "low"]:
        for ctas in [0, 16]:
            with fp.Checkpointer(DEV, prio=prio, pack_ctas=ctas) as ck:
                its = loop(ck, iters + 2)[2:]
            m = statistics.median(its)
            r = {"prio": prio, "pack_ctas": ctas, "iter_s": round(m, 4),
                 "overhead_pct": round(100 * (m / base - 1), 2)}
            print(json.dumps(r), flush=True)
            res.append(r)
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--what", default="pack")
    ap.add_argument("--dir", default=os.path.join(os.environ.get("GRAFT_REPO_ROOT", "/tmp"), "ablate"))
    ap.add_argument("--t-fb", type=float, default=6.0)
    ap.add_argument("--iters", type=int, default=3)
    a = ap.parse_args()
    os.makedirs(a.dir, exist_ok=True)
    fn = {"pack": lambda: ablate_pack(a.dir), "buffer": lambda: ablate_buffer(a.dir),
          "prio": lambda: ablate_prio(a.dir, a.t_fb, a.iters)}[a.what]
    res = fn()
    os.system(f"rm -rf {a.dir}")
    os.makedirs("gpurun_out", exist_ok=True)
    with open(f"gpurun_out/ablate_{a.what}.json", "w") as f:
        json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
