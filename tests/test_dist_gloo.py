"""N>1 path over real torch.distributed processes (gloo, world_size 2, CPU).

Each process is one DP rank with its own libfastpersist context; the two
collectives of the path (setup all-gather of per-rank sizes + layout digest,
P:487; per-checkpoint status all-reduce(MIN) = completion barrier) go
through the binding's torch.distributed callbacks — the same code the NCCL
group uses on the GPU box. Host-resident state (FP_TENSOR_HOST) stands in for
device tensors, so everything but the pack kernel runs here.
"""
import os

import pytest
import torch
import torch.multiprocessing as mp

from oracle import fpck
from tests._util import entries, file_sha, oracle_layout
from workloads import config_specs, make_state

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _worker(rank, world, rdzv, cfg, out_dir, mode, q):
    import sys
    sys.path.insert(0, ROOT)
    import torch.distributed as dist
    import paper_2406_13768_b200 as fp
    # file rendezvous: no TCP port to race for between test processes
    dist.init_process_group("gloo", init_method=f"file://{rdzv}", rank=rank, world_size=world)
    try:
        st = make_state(config_specs(cfg, rank, world), "cpu")
        with fp.Checkpointer(None, slot_bytes=1 << 20) as ck:
            if mode == "mismatch" and rank == 1:
                st = st[:-1]                      # replicated lists differ -> EMISMATCH
            try:
                stats = ck.save(entries(st), out_dir)
            except fp.FastPersistError as e:
                q.put((rank, "err", e.code))
                return
            dst = [(s, torch.zeros_like(t)) for s, t in st]
            if mode == "parallel":                # own shard + gloo all-gather
                ck.load_parallel(entries(dst), out_dir)
            else:
                ck.load(entries(dst), out_dir)
            same = all(torch.equal(a.reshape(-1).view(torch.uint8), b.reshape(-1).view(torch.uint8))
                       for (_, a), (_, b) in zip(st, dst))
            q.put((rank, "ok", (stats["image_bytes"], stats["shard_bytes"], same)))
    finally:
        dist.destroy_process_group()


def _run(cfg, world, out_dir, mode="ok"):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    rdzv = os.path.join(out_dir, ".rdzv")
    ps = [ctx.Process(target=_worker, args=(r, world, rdzv, cfg, out_dir, mode, q))
          for r in range(world)]
    for p in ps:
        p.start()
    for p in ps:
        p.join(300)
    res = {}
    while not q.empty():
        r, kind, v = q.get()
        res[r] = (kind, v)
    for p in ps:
        assert p.exitcode == 0, f"rank exited with {p.exitcode}"
    return res


@pytest.mark.parametrize("cfg,mode", [("gpt3_odd", "ok"), ("moe_small", "ok"),
                                      ("moe_small", "parallel"), ("c1_tiny", "parallel")])
def test_gloo_world2_shards_match_oracle(tmp_path, cfg, mode):
    world = 2
    res = _run(cfg, world, str(tmp_path), mode)
    states = [make_state(config_specs(cfg, r, world), "cpu") for r in range(world)]
    lay = oracle_layout(states, world)
    ext = fpck.shard_extents(lay)
    for r in range(world):
        kind, (img, shard, same) = res[r]
        assert kind == "ok" and img == lay.image_bytes and same
        assert shard == sum(n for _, _, n in ext[r])
        assert file_sha(tmp_path / fpck.shard_name(r, world)) == fpck.shard_sha256(lay, r)
    # manifest committed by rank 0 after the barrier
    import json
    man = json.load(open(tmp_path / "manifest.json"))
    assert [s["extents"] for s in man["shards"]] == [[list(e) for e in x] for x in ext]


def test_gloo_world2_layout_mismatch_fails_on_every_rank(tmp_path):
    from paper_2406_13768_b200.fastpersist import FP_EMISMATCH
    res = _run("gpt3_odd", 2, str(tmp_path), mode="mismatch")
    assert res[0] == ("err", FP_EMISMATCH) and res[1] == ("err", FP_EMISMATCH)
    assert not os.path.exists(tmp_path / "manifest.json")
