"""One DP rank of a k-rank job on ONE GPU, for BASELINE configs that need 8
GPUs (C3 6.7B at DP=8, C4 13B ZeRO at DP=8, C5 MoE at EP=8).

The rank's collectives are answered by `MirrorComm`: the setup all-gather
returns this rank's own facts for every rank, the status all-reduce returns
its own status. For these configs that is exact, not an approximation: every
rank's replicated list is identical (same digest and bytes), and rank-local
partitions have identical sizes on every rank (dim-0 ZeRO shards of equal
shape; 8 experts per rank; names of equal length for ranks < 10), so the
facts rank r would receive from 7 real peers are its own, repeated.

Per config it reports: this rank's shard bytes, checkpoint latency and GB/s,
the built-in NVMe roofline on the same directory, the pack-kernel HBM rate,
optional per-iteration overhead under a synthetic GEMM stream (Eq. 1 window,
PAPER.md P:320-323, §4.3), and a sampled byte-for-byte parity
check of the written shard against the oracle reading the same tensors.

    python tools/bench_configs.py --cfg c3_gpt3_6.7b --k 8 --rank 0 [--overhead]
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

T_FB_FLOPS = {  # 6 * P * GBS * seq at 40% of nominal bf16 over k ranks
    "c2_gpt3_1.3b": 6 * 1315819520 * 512 * 2048,
    "c3_gpt3_6.7b": 6 * 6658596864 * 1024 * 2048,
    "c4_gpt3_13b_zero": 6 * 12853626880 * 1024 * 2048,
    "c5_moe_64e": 6 * 1315819520 * 256 * 2048,   # MoE: dense-equivalent compute of the base
}


class MirrorComm:
    """Answers the collectives of one rank of k. `peer_regions[r]` (optional)
    = (region_bytes, n_local) rank r would report; by default every rank
    reports this rank's own facts (exact for C3/C4, see module doc)."""

    def __init__(self, rank, k, peer_regions=None):
        self.rank, self.world = rank, k
        self.peer = peer_regions

    def allgather(self, vals):
        if self.peer is None or len(vals) != 4:   # 4 = the setup facts; else mirror
            return list(vals) * self.world
        out = []
        for r in range(self.world):
            out += [self.peer[r][0], self.peer[r][1]] + list(vals[2:])
        return out

    def allreduce_min(self, v):
        return v


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cfg", default="c3_gpt3_6.7b")
    ap.add_argument("--k", type=int, default=8)
    ap.add_argument("--rank", type=int, default=0)
    ap.add_argument("--dir", default=None)
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--no-fsync", action="store_true")
    ap.add_argument("--overhead", action="store_true")
    ap.add_argument("--iters", type=int, default=3)
    ap.add_argument("--parity-pages", type=int, default=48)
    ap.add_argument("--pack", default="v4")
    ap.add_argument("--full-crc", action="store_true")
    a = ap.parse_args()
    root = a.dir or os.path.join(os.environ.get("GRAFT_REPO_ROOT", "/tmp"), "cfg_ckpt")
    os.makedirs(root, exist_ok=True)
    dev = torch.device("cuda", 0)
    specs = config_specs(a.cfg, a.rank, a.k)
    t0 = time.time()
    state = make_state(specs, dev)
    torch.cuda.synchronize()
    gen_s = time.time() - t0
    ents = [(s.name, t, s.section, s.owner) for s, t in state]
    out = {"cfg": a.cfg, "k": a.k, "rank": a.rank, "state_bytes": sum(s.nbytes for s in specs),
           "tensors": len(specs), "gen_s": round(gen_s, 1), "dir": root}
    peer = None
    if a.cfg.startswith("c5"):
        # experts have different names per rank (expert ids of 1 or 2 digits):
        # each peer's local-region size is what that rank's own tensor list
        # gives (header of 64 + 128 n + names, rounded to 4096, + payloads)
        def rup(x, al=4096):
            return (x + al - 1) // al * al
        peer = []
        for r in range(a.k):
            loc = [x for x in config_specs(a.cfg, r, a.k) if x.owner >= 0]
            names = sum(len(x.name.encode()) for x in loc)
            peer.append((rup(64 + 128 * len(loc) + names) + sum(rup(x.nbytes) for x in loc),
                         len(loc)))
    comm = MirrorComm(a.rank, a.k, peer)
    ck = fp.Checkpointer(dev, comm=comm, pack=a.pack, no_fsync=a.no_fsync)
    lat, stats = [], []
    for i in range(a.steps + 1):
        t0 = time.perf_counter()
        s = ck.save(ents, os.path.join(root, "step"))
        if i:
            lat.append(time.perf_counter() - t0)
            stats.append(s)
    shard = stats[-1]["shard_bytes"]
    out.update(image_bytes=stats[-1]["image_bytes"], shard_bytes=shard,
               latency_s=[round(x, 3) for x in lat],
               rank_gbs=round(shard / statistics.median(lat) / 1e9, 3),
               pack_gbs=round(2 * sum(x["pack_bytes"] for x in stats) /
                              (sum(x["pack_ms"] for x in stats) / 1e3) / 1e9, 1),
               d2h_gbs=round(sum(x["pack_bytes"] for x in stats) /
                             (sum(x["d2h_ms"] for x in stats) / 1e3) / 1e9, 1),
               io_stall_s=round(stats[-1]["t_io_stall"], 3), fsync_s=round(stats[-1]["t_fsync"], 3))
    print(json.dumps(out), flush=True)
    # sampled parity: oracle pages read straight from the same device tensors
    from oracle import fpck
    from tests._util import otensor
    rep = [otensor(s, t, lazy=True) for s, t in state if s.owner < 0]
    mine = [otensor(s, t, lazy=True) for s, t in state if s.owner >= 0]
    def stub(x, r):   # a peer's local tensor: only its size matters for this shard
        return fpck.OTensor(x.name, x.dtype, x.section, r, x.shape, lambda o, n: b"\0" * n)
    local = [mine if r == a.rank else [stub(x, r) for x in config_specs(a.cfg, r, a.k)
                                       if x.owner >= 0]
             for r in range(a.k)] if mine else None
    lay = fpck.Layout(rep, local, k=a.k)
    ext = fpck.shard_extents(lay)[a.rank]
    path = os.path.join(root, "step", fpck.shard_name(a.rank, a.k))
    g = torch.Generator().manual_seed(7)
    pages = shard // 4096
    picks = [0, pages - 1] + torch.randint(0, pages, (a.parity_pages,), generator=g).tolist()
    bad = 0
    with open(path, "rb") as f:
        for pg in picks:
            fo = pg * 4096
            io = next(e[0] + fo - e[1] for e in ext if e[1] <= fo < e[1] + e[2])
            f.seek(fo)
            bad += f.read(4096) != lay.read(io, 4096)
    out["parity_pages_checked"] = len(picks)
    out["parity_pages_bad"] = bad
    out["oracle_image_bytes"] = lay.image_bytes
    print(json.dumps(out), flush=True)
    if a.full_crc:
        # every byte of the shard: the GPU's CRC-32 (from the packed slabs)
        # against zlib.crc32 over the oracle's shard bytes of the same tensors
        t0 = time.time()
        want = fpck.shard_crc32(lay, a.rank)
        out["crc_gpu"] = stats[-1]["shard_crc32"]
        out["crc_oracle"] = want
        out["crc_match"] = bool(stats[-1]["crc_valid"]) and stats[-1]["shard_crc32"] == want
        out["crc_oracle_s"] = round(time.time() - t0, 1)
        print(json.dumps(out), flush=True)
    if a.overhead:
        n = 8192
        A = torch.randn(n, n, device=dev, dtype=torch.bfloat16)
        C = torch.empty_like(A)
        for _ in range(5):
            torch.matmul(A, A, out=C)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(40):
            torch.matmul(A, A, out=C)
        torch.cuda.synchronize()
        tg = (time.perf_counter() - t0) / 40
        t_fb = T_FB_FLOPS[a.cfg] / (a.k * 0.4 * 2.25e15)
        ng = max(1, round(t_fb / tg))
        by = {}
        for s, t in state:
            by.setdefault(s.section, []).append(t)

        def opt():
            torch._foreach_mul_(by["exp_avg"], 0.9)
            torch._foreach_mul_(by["exp_avg_sq"], 0.999)
            torch._foreach_add_(by["master"], by["exp_avg"], alpha=-1e-8)
            for p, w in zip(by["param"], by["master"]):
                p.copy_(w)

        def loop(ckpt, iters):
            its = []
            for i in range(iters):
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                for _ in range(ng):
                    torch.matmul(A, A, out=C)
                if ckpt:
                    ck.wait()
                opt()
                if ckpt:
                    ck.begin(ents, os.path.join(root, "step"))
                torch.cuda.synchronize()
                its.append(time.perf_counter() - t0)
            if ckpt:
                ck.wait()
            return its
        b = loop(False, a.iters + 1)[1:]
        c = loop(True, a.iters + 2)[2:]
        out["overhead"] = {"t_fb_s": round(ng * tg, 3), "iter_no_ckpt": round(statistics.median(b), 4),
                           "iter_ckpt": round(statistics.median(c), 4),
                           "overhead_pct": round(100 * (statistics.median(c) / statistics.median(b) - 1), 2),
                           "eq1_required_rank_gbs": round(shard / 1e9 / (ng * tg), 3)}
        print(json.dumps(out), flush=True)
    ck.close()
    os.system(f"rm -rf {root}")
    os.makedirs("gpurun_out", exist_ok=True)
    with open(f"gpurun_out/cfg_{a.cfg}_r{a.rank}of{a.k}.json", "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
