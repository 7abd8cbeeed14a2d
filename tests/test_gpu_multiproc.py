"""Multi-PROCESS DP ranks on the GPU box (one GPU: every rank on cuda:0).

  - the peer exchange of fp_ckpt_load_parallel across processes: each rank's
    partition buffer is exported with a CUDA IPC handle and mapped by the
    other ranks, the ready flags live in a POSIX shared-memory segment that
    every process registers with CUDA (own partition into GPU memory,
    then the all-gather);
  - the binding's torch.distributed callbacks over an NCCL group (world 1:
    NCCL refuses two ranks on one GPU) — the collectives bench.py uses at N>1.
Control collectives of the 2-rank runs go over gloo (the box has one GPU).
"""
import os

import pytest
import torch
import torch.multiprocessing as mp

from oracle import fpck
from tests._util import entries, file_sha
from workloads import config_specs, make_state

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _worker(rank, world, rdzv, cfg, out_dir, balance, q):
    import sys
    sys.path.insert(0, ROOT)
    os.environ["FP_LOAD_EXCHANGE"] = "peer"      # required: -ENOSYS if IPC cannot map
    os.environ.setdefault("FP_PEER_TIMEOUT_S", "60")
    import torch.distributed as dist
    import paper_2406_13768_b200 as fp
    dist.init_process_group("gloo", init_method=f"file://{rdzv}", rank=rank, world_size=world)
    try:
        dev = torch.device("cuda", 0)
        torch.cuda.set_device(dev)
        st = make_state(config_specs(cfg, rank, world), dev)
        with fp.Checkpointer(dev, slot_bytes=1 << 20, balance=balance) as ck:
            stats = ck.save(entries(st), out_dir)
            dst = [(s, torch.full_like(t, 3) if t.is_floating_point() else torch.zeros_like(t))
                   for s, t in st]
            ls = ck.load_parallel(entries(dst), out_dir)
            torch.cuda.synchronize()
            same = all(torch.equal(a.reshape(-1).view(torch.uint8), b.reshape(-1).view(torch.uint8))
                       for (_, a), (_, b) in zip(st, dst))
            # the oracle needs the bytes: ship the raw state of rank-local tensors
            q.put((rank, stats["shard_bytes"], ls["exchange"], same,
                   [(s.name, t.reshape(-1).view(torch.uint8).cpu().numpy().tobytes())
                    for s, t in st]))
    except Exception as e:  # noqa: BLE001
        q.put((rank, "error", repr(e), False, []))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("cfg,world,balance", [("gpt3_small", 2, "pages"), ("moe_small", 2, "pages"),
                                               ("c1_tiny", 3, "bytes")])
def test_peer_exchange_across_processes(tmp_path, cfg, world, balance):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    out = str(tmp_path)
    ps = [ctx.Process(target=_worker, args=(r, world, os.path.join(out, ".rdzv"), cfg, out,
                                            balance, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = {}
    for _ in ps:
        r = q.get(timeout=600)
        res[r[0]] = r
    for p in ps:
        p.join(timeout=120)
    for r in range(world):
        assert res[r][1] != "error", res[r][2]
        assert res[r][2] == "peer" and res[r][3], res[r][:4]
    # shards == oracle of the same state (bytes copied to host by torch)
    specs = [config_specs(cfg, r, world) for r in range(world)]
    raw = [dict(res[r][4]) for r in range(world)]
    rep = [fpck.OTensor(s.name, s.dtype, s.section, s.owner, s.shape, raw[0][s.name])
           for s in specs[0] if s.owner < 0]
    local = [[fpck.OTensor(s.name, s.dtype, s.section, s.owner, s.shape, raw[r][s.name])
              for s in specs[r] if s.owner >= 0] for r in range(world)]
    lay = fpck.Layout(rep, local, k=world)
    for r in range(world):
        assert file_sha(os.path.join(out, fpck.shard_name(r, world))) == \
            fpck.shard_sha256(lay, r, balance=balance), r


def _nccl_worker(rdzv, q):
    import ctypes as C
    import sys
    sys.path.insert(0, ROOT)
    import torch.distributed as dist
    from paper_2406_13768_b200.fastpersist import _Comm
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    dist.init_process_group("nccl", init_method=f"file://{rdzv}", rank=0, world_size=1,
                            device_id=dev)
    try:
        cm = _Comm(None, dev)
        send = (C.c_uint64 * 3)(7, 1 << 40, 2**64 - 1)
        recv = (C.c_uint64 * 3)()
        ok = [cm._allgather(None, send, recv, 3) == 0 and list(recv) == list(send)]
        v = (C.c_int32 * 1)(-17)
        ok.append(cm._allreduce(None, v) == 0 and v[0] == -17)
        a = torch.arange(4096, device=dev, dtype=torch.uint8)
        b = torch.zeros_like(a)
        s = torch.cuda.Stream(dev)
        ok.append(cm._allgather_bytes(None, a.data_ptr(), b.data_ptr(), 4096, 1, s.cuda_stream) == 0)
        s.synchronize()
        ok.append(torch.equal(a, b))
        q.put(ok)
    finally:
        dist.destroy_process_group()


def test_binding_callbacks_over_nccl(tmp_path):
    """fastpersist._Comm over a real NCCL group: the u64 all-gather, the status
    all-reduce(MIN) (on the binding's side stream) and the device byte
    all-gather ordered on a given stream."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=_nccl_worker, args=(str(tmp_path / ".rdzv"), q))
    p.start()
    ok = q.get(timeout=300)
    p.join(timeout=60)
    assert ok == [True, True, True, True], ok
