"""GPU parity: the sm_100a pack path through the C-ABI vs the CPU oracle.

Every test checkpoints DEVICE tensors (pack kernel -> D2H -> io_uring O_DIRECT)
and compares the shard files byte for byte (sha256) with the oracle's shards
of the same state (BASELINE.json north_star: "GPU-written files must be
bit-exact (sha256) against the oracle's"). Stats prove the kernel ran.
"""
import os

import pytest
import torch

import paper_2406_13768_b200 as fp
from oracle import fpck
from tests._util import (ThreadComm, entries, file_sha, oracle_layout, otensor, run_threads)
from workloads import config_specs, make_state

pytestmark = pytest.mark.gpu

DEV = torch.device("cuda", 0)


@pytest.fixture(scope="module", autouse=True)
def built():
    from paper_2406_13768_b200 import build
    build.build()
    assert torch.cuda.is_available(), "GPU tests need a B200"


def _state(cfg, rank=0, k=1, device=DEV):
    return make_state(config_specs(cfg, rank, k), device)


def _check_rank_files(tmp, lay, k, crc=True):
    for r in range(k):
        assert file_sha(os.path.join(tmp, fpck.shard_name(r, k))) == fpck.shard_sha256(lay, r), r
    if crc:   # per-shard CRC-32 computed on the GPU from the packed slab (f4)
        import json
        man = json.load(open(os.path.join(tmp, "manifest.json")))
        for r in range(k):
            assert man["shards"][r]["crc32"] == fpck.shard_crc32(lay, r), r


@pytest.mark.parametrize("pack", ["v4", "bulk", "lsu", "host", "ce"])
@pytest.mark.parametrize("slot_bytes", [4096, 1 << 20, 3 << 20, 64 << 20])
def test_c1_tiny_parity(tmp_path, pack, slot_bytes):
    st = _state("c1_tiny")
    lay = oracle_layout([st], 1)
    with fp.Checkpointer(DEV, pack=pack, slot_bytes=slot_bytes, ring_slots=4,
                         pack_bytes=slot_bytes) as ck:
        s = ck.save(entries(st), str(tmp_path))
    if pack == "ce":     # ablation: no kernel at all, copy engine only
        assert s["pack_launches"] == 0 and s["d2h_ms"] > 0
    else:
        assert s["pack_launches"] == s["chunks"] > 0 and s["pack_ms"] > 0
    assert s["pack_bytes"] == lay.image_bytes
    _check_rank_files(str(tmp_path), lay, 1)


@pytest.mark.parametrize("pack", ["v4", "bulk", "lsu"])
@pytest.mark.parametrize("slot_bytes,pack_bytes,slots", [(1 << 20, 3 << 20, 2), (4096, 5 * 4096, 3),
                                                         (8 << 20, 64 << 20, 4),
                                                         (2 << 20, 2 << 20, 1)])
def test_pack_groups_parity(tmp_path, pack, slot_bytes, pack_bytes, slots):
    """One pack launch gathers pack_bytes (several ring chunks, ragged last
    group) into the device slab; every chunk is copied to its own ring slot."""
    st = _state("c1_tiny")
    lay = oracle_layout([st], 1)
    with fp.Checkpointer(DEV, pack=pack, slot_bytes=slot_bytes, pack_bytes=pack_bytes,
                         ring_slots=slots) as ck:
        s = ck.save(entries(st), str(tmp_path))
    groups = -(-lay.image_bytes // pack_bytes)
    assert s["pack_launches"] == groups and s["chunks"] == -(-lay.image_bytes // slot_bytes)
    assert s["pack_bytes"] == lay.image_bytes
    _check_rank_files(str(tmp_path), lay, 1)


@pytest.mark.parametrize("prio", ["high", "low"])
def test_stream_priority_parity(tmp_path, prio):
    st = _state("gpt3_odd")
    lay = oracle_layout([st], 1)
    with fp.Checkpointer(DEV, prio=prio, slot_bytes=1 << 20) as ck:
        ck.save(entries(st), str(tmp_path))
    _check_rank_files(str(tmp_path), lay, 1)


@pytest.mark.parametrize("pack", ["v4", "bulk", "lsu", "host", "ce"])
@pytest.mark.parametrize("cfg", ["gpt3_small", "gpt3_odd", "zero_small", "moe_small"])
def test_structured_states_parity(tmp_path, cfg, pack):
    st = _state(cfg)
    lay = oracle_layout([st], 1)
    with fp.Checkpointer(DEV, pack=pack, slot_bytes=1 << 20) as ck:
        ck.save(entries(st), str(tmp_path))
    _check_rank_files(str(tmp_path), lay, 1)


@pytest.mark.parametrize("pack", ["v4", "bulk", "lsu", "host", "ce"])
def test_misaligned_and_degenerate_tensors(tmp_path, pack):
    """Odd storage offsets (byte path), empty tensors, scalars, 1-byte tails."""
    base = torch.randint(0, 256, (1 << 20,), dtype=torch.uint8, device=DEV)
    bf = torch.randn(70001, device=DEV).to(torch.bfloat16)
    ents = [
        ("odd_u8", base[1:100001], "other", -1),         # data_ptr % 16 == 1
        ("odd_u8_b", base[7:7 + 65536 + 5], "other", -1),
        ("bf_view", bf[3:], "param", -1),                 # data_ptr % 16 == 6
        ("empty", torch.empty(0, device=DEV), "other", -1),
        ("scalar", torch.tensor(3.5, device=DEV), "other", -1),
        ("one", torch.tensor([7], dtype=torch.uint8, device=DEV), "other", -1),
        ("big", torch.randn(3, 333333, device=DEV), "master", -1),
    ]
    from tests._util import otensor, DT
    lay = fpck.Layout([otensor(n, t, sec, own, dtype=DT[t.dtype]) for n, t, sec, own in ents])
    with fp.Checkpointer(DEV, pack=pack, slot_bytes=256 << 10) as ck:
        ck.save(ents, str(tmp_path))
    _check_rank_files(str(tmp_path), lay, 1)


@pytest.mark.parametrize("pack", ["v4", "bulk", "lsu"])
@pytest.mark.parametrize("ctas", [1, 3, 16])
def test_background_pack_few_ctas(tmp_path, pack, ctas):
    """Overlap mode's CTA cap (pack_ctas, §4.3): with 1-16 CTAs each CTA walks
    hundreds of tiles of a 64 MiB pack group — the fused kernel's stage /
    tile hand-off protocol over long sequences (odd tile counts per CTA, both
    CRC groups) — and the shard and its CRC still match the oracle."""
    st = _state("gpt3_small")
    lay = oracle_layout([st], 1)
    with fp.Checkpointer(DEV, pack=pack, pack_ctas=ctas, slot_bytes=16 << 20,
                         pack_bytes=64 << 20) as ck:
        s = ck.save(entries(st), str(tmp_path))
    assert s["pack_launches"] > 0
    _check_rank_files(str(tmp_path), lay, 1)


@pytest.mark.parametrize("pack", ["v4", "bulk", "lsu"])
def test_many_small_tensors_align512(tmp_path, pack):
    """Alignment 512 (P:475's example) and 700 small ragged tensors: a 32 KiB
    slab tile then holds up to ~128 items (payloads, their < 16 B tails, zero
    padding) — the > 32-items-per-tile paths of the pack kernels."""
    g = torch.Generator(device=DEV).manual_seed(0xFA572406 + 512)
    sizes = torch.randint(1, 700, (700,), generator=torch.Generator().manual_seed(512)).tolist()
    ents = []
    for i, n in enumerate(sizes):
        dt = (torch.float32, torch.bfloat16, torch.uint8)[i % 3]
        t = torch.randint(0, 256, (n * torch.tensor([], dtype=dt).element_size(),),
                          dtype=torch.uint8, device=DEV, generator=g).view(dt)
        ents.append((f"t{i}", t, "other", -1))
    from tests._util import otensor, DT
    lay = fpck.Layout([otensor(n, t, sec, own, dtype=DT[t.dtype]) for n, t, sec, own in ents],
                      align=512)
    with fp.Checkpointer(DEV, pack=pack, alignment=512, slot_bytes=64 << 10,
                         pack_bytes=256 << 10) as ck:
        s = ck.save(ents, str(tmp_path))
    assert s["pack_bytes"] == lay.image_bytes
    _check_rank_files(str(tmp_path), lay, 1)


@pytest.mark.parametrize("cfg,k", [("gpt3_small", 4), ("zero_small", 2), ("moe_small", 4),
                                   ("c1_tiny", 3)])
def test_dp_ranks_on_one_gpu(tmp_path, cfg, k):
    """k DP ranks as threads sharing cuda:0 (fake comm): shards == oracle."""
    states = [_state(cfg, r, k) for r in range(k)]
    lay = oracle_layout(states, k)
    comms = ThreadComm.group(k)
    cks = [fp.Checkpointer(DEV, comm=comms[r], slot_bytes=1 << 20) for r in range(k)]
    try:
        run_threads([lambda r=r: cks[r].save(entries(states[r]), str(tmp_path))
                     for r in range(k)])
        _check_rank_files(str(tmp_path), lay, k)
        dst = [[(s, torch.zeros_like(t)) for s, t in states[r]] for r in range(k)]
        run_threads([lambda r=r: cks[r].load(entries(dst[r]), str(tmp_path))
                     for r in range(k)])
        torch.cuda.synchronize()
        for r in range(k):
            for (_, a), (_, b) in zip(states[r], dst[r]):
                assert torch.equal(a.reshape(-1).view(torch.uint8), b.reshape(-1).view(torch.uint8))
    finally:
        for c in cks:
            c.close()


def test_load_roundtrip_device(tmp_path):
    st = _state("c1_tiny")
    with fp.Checkpointer(DEV, slot_bytes=8 << 20) as ck:
        ck.save(entries(st), str(tmp_path))
        dst = [(s, torch.full_like(t, 3)) for s, t in st]
        ck.load(entries(dst), str(tmp_path))
        torch.cuda.synchronize()
    for (_, a), (_, b) in zip(st, dst):
        assert torch.equal(a.reshape(-1).view(torch.uint8), b.reshape(-1).view(torch.uint8))


def test_producer_stream_fence(tmp_path):
    """begin() must see writes still queued on the producer stream:
    the checkpoint equals the state AFTER the optimizer-like update."""
    st = _state("gpt3_small")
    s = torch.cuda.Stream(DEV)
    a = torch.randn(4096, 4096, device=DEV)
    with fp.Checkpointer(DEV, slot_bytes=1 << 20) as ck:
        with torch.cuda.stream(s):
            for _ in range(20):          # keep the stream busy for a while
                a = a @ a
                a = a / a.norm()
            for _, t in st:              # "optimizer step": written late on s
                t.fill_(1.25) if t.is_floating_point() else None
        ck.begin(entries(st), str(tmp_path), stream=s)
        ck.wait()
    torch.cuda.synchronize()
    lay = oracle_layout([st], 1)
    _check_rank_files(str(tmp_path), lay, 1)


@pytest.mark.parametrize("pack", ["bulk", "v4", "lsu"])
def test_overlapped_loop_each_checkpoint_is_its_iterations_state(tmp_path, pack):
    """§4.3 pipelining over several iterations (SURVEY §8(c) pin 8):
    fwd/bwd (GEMMs + the backward rewriting the grads, which the adam14
    checkpoint excludes) -> wait() -> optimizer (master/m/v/param updated on
    the training stream) -> begin(gen n) with that stream as producer.
    Checkpoint n must equal the oracle of the state right after optimizer n
    — not before it, and not touched by optimizer n+1 queued while the
    checkpoint is still being written."""
    st = _state("gpt3_small")
    ck_ents = [(s, t) for s, t in st if s.section != "grad"]
    grads = [t for s, t in st if s.section == "grad"]
    upd = [t for s, t in ck_ents if t.is_floating_point()]
    s = torch.cuda.Stream(DEV)
    a = torch.randn(2048, 2048, device=DEV)
    snaps = []
    with fp.Checkpointer(DEV, pack=pack, slot_bytes=4 << 20, ring_slots=3,
                         pack_bytes=8 << 20, pack_ctas=16) as ck:
        for n in range(3):
            with torch.cuda.stream(s):
                for _ in range(6):                    # forward / backward
                    a = a @ a
                    a = a / a.norm()
                for g in grads:                       # the backward writes the grads
                    g.add_(1.0)
            ck.wait()                                 # fence before the optimizer
            with torch.cuda.stream(s):                # optimizer n
                for t in upd:
                    t.mul_(0.5).add_(float(n + 1))
                snaps.append([(sp, t.clone()) for sp, t in ck_ents])
            ck.begin(entries(ck_ents), str(tmp_path / f"gen{n}"), stream=s)
        ck.wait()
    torch.cuda.synchronize()
    for n, snap in enumerate(snaps):
        _check_rank_files(str(tmp_path / f"gen{n}"), oracle_layout([snap], 1), 1)


def test_c1_bench_launch_config(tmp_path):
    """The configuration bench.py times (64 MiB slots x 4, bulk pack + CRC, 1 MiB SQEs)."""
    st = _state("c1_tiny")
    lay = oracle_layout([st], 1)
    with fp.Checkpointer(DEV) as ck:
        for gen in range(2):             # second generation overwrites in place
            ck.save(entries(st), str(tmp_path))
    _check_rank_files(str(tmp_path), lay, 1)


@pytest.mark.slow
def test_c2_gpt3_1p3b_full_size_parity(tmp_path):
    """BASELINE configs[1] at DP=1, full size (~21 GB), bench launch config:
    whole-shard sha256 against the oracle streaming from the same tensors,
    plus sampled 4 KiB windows compared byte for byte."""
    free = os.statvfs(str(tmp_path))
    if free.f_bavail * free.f_frsize < 25e9:
        pytest.skip("needs ~25 GB free disk")
    st = _state("c2_gpt3_1.3b")
    lay = oracle_layout([st], 1, lazy=True)
    with fp.Checkpointer(DEV) as ck:
        s = ck.save(entries(st), str(tmp_path))
    assert s["image_bytes"] == lay.image_bytes
    path = os.path.join(str(tmp_path), "shard-0-of-1.fpck")
    g = torch.Generator().manual_seed(1234)
    offs = torch.randint(0, lay.image_bytes // 4096, (64,), generator=g).tolist()
    with open(path, "rb") as f:
        for pg in [0, lay.image_bytes // 4096 - 1] + offs:
            f.seek(pg * 4096)
            assert f.read(4096) == lay.read(pg * 4096, 4096), pg
    assert file_sha(path) == fpck.shard_sha256(lay, 0)
    os.remove(path)          # pytest keeps tmp dirs: do not leave 21 GB on the disk


@pytest.mark.slow
@pytest.mark.timeout(1500)
def test_c2_gpt3_1p3b_full_size_dp8_thread_ranks(tmp_path):
    """BASELINE configs[1] at DP=8, full size: 8 DP ranks as threads sharing
    this GPU (one Checkpointer, helper thread, io_uring and 1 GiB slab each,
    collectives through ThreadComm) write the 21 GB image split 8 ways in the
    bench launch configuration; every shard's sha256 == the oracle's shard of
    the same tensors, and rank 0's manifest lists all 8 with their CRC-32s."""
    import json
    free = os.statvfs(str(tmp_path))
    if free.f_bavail * free.f_frsize < 25e9:
        pytest.skip("needs ~25 GB free disk")
    k = 8
    st = _state("c2_gpt3_1.3b")
    lay = oracle_layout([st] * k, k, lazy=True)
    comms = ThreadComm.group(k)
    cks = [fp.Checkpointer(DEV, comm=comms[r]) for r in range(k)]
    try:
        stats = run_threads([lambda r=r: cks[r].save(entries(st), str(tmp_path))
                             for r in range(k)])
        assert all(x["image_bytes"] == lay.image_bytes for x in stats)
        assert sum(x["shard_bytes"] for x in stats) == lay.image_bytes
        man = json.load(open(os.path.join(str(tmp_path), "manifest.json")))
        assert len(man["shards"]) == k
        for r in range(k):
            path = os.path.join(str(tmp_path), fpck.shard_name(r, k))
            assert file_sha(path) == fpck.shard_sha256(lay, r), r
            assert man["shards"][r]["crc32"] == stats[r]["shard_crc32"], r
            os.remove(path)  # pytest keeps tmp dirs: do not leave 21 GB behind
    finally:
        for c in cks:
            c.close()
        for f in os.listdir(str(tmp_path)):
            if f.endswith(".fpck"):
                os.remove(os.path.join(str(tmp_path), f))
        torch.cuda.empty_cache()


def _one_rank_of_8_full_size(tmp_path, cfg, rank, need_bytes, tmpfs_ok=False):
    """BASELINE configs that need 8 GPUs: rank `rank` of DP=8 on this GPU
    (MirrorComm answers its collectives exactly, see tests/_util.py), in the
    bench launch configuration; the whole shard's sha256 against the oracle
    streaming the same tensors."""
    free = os.statvfs(str(tmp_path))
    if free.f_bavail * free.f_frsize < need_bytes * 1.2:
        shm = os.statvfs("/dev/shm") if os.path.isdir("/dev/shm") else None
        if not tmpfs_ok or not shm or shm.f_bavail * shm.f_frsize < need_bytes * 1.5:
            pytest.skip(f"needs {need_bytes * 1.2 / 1e9:.0f} GB free disk")
        # the shard does not fit the box's disk: tmpfs (O_DIRECT may fall
        # back to buffered writes there; the bytes are what is checked)
        import tempfile
        tmp_path = tempfile.mkdtemp(prefix="fp_full_", dir="/dev/shm")
    try:
        _one_rank_body(tmp_path, cfg, rank, need_bytes)
    finally:                 # pytest keeps tmp dirs: never leave a shard behind
        import shutil
        for f in os.listdir(str(tmp_path)):
            if f.endswith(".fpck"):
                os.remove(os.path.join(str(tmp_path), f))
        if str(tmp_path).startswith("/dev/shm/"):
            shutil.rmtree(str(tmp_path), ignore_errors=True)
        torch.cuda.empty_cache()


def _one_rank_body(tmp_path, cfg, rank, need_bytes):
    from tests._util import MirrorComm
    torch.cuda.empty_cache()
    k = 8
    st = _state(cfg, rank, k)
    mine = [otensor(s, t, lazy=True) for s, t in st]
    if any(s.owner >= 0 for s, _ in st):
        # rank-local partitions: the other ranks' regions only fix offsets
        # (their sizes come from the oracle's layout); their bytes are never read
        def ghost(r):
            return [fpck.OTensor(s.name, s.dtype, s.section, r, s.shape, lambda off, n: bytes(n))
                    for s in config_specs(cfg, r, k) if s.owner >= 0]
        rep = [o for (sp, _), o in zip(st, mine) if sp.owner < 0]
        own = [o for (sp, _), o in zip(st, mine) if sp.owner >= 0]
        local = [own if r == rank else ghost(r) for r in range(k)]
        lay = fpck.Layout(rep, local, k=k)
    else:
        lay = fpck.Layout(mine, k=k)
    regions = [b for _, b in lay.regions] if lay.regions else None
    with fp.Checkpointer(DEV, comm=MirrorComm(rank, k, regions)) as ck:
        s = ck.save(entries(st), str(tmp_path))
    assert s["image_bytes"] == lay.image_bytes
    path = os.path.join(str(tmp_path), fpck.shard_name(rank, k))
    assert os.path.getsize(path) == s["shard_bytes"] >= need_bytes * 0.99
    import hashlib
    import zlib
    h, c = hashlib.sha256(), 0
    for b in fpck.iter_shard(lay, rank):         # one oracle pass: sha256 + CRC-32
        h.update(b)
        c = zlib.crc32(b, c)
    assert s["shard_crc32"] == c
    assert file_sha(path) == h.hexdigest()


@pytest.mark.slow
@pytest.mark.timeout(1500)
def test_c3_gpt3_6p7b_rank3_of_8_full_size_parity(tmp_path):
    """BASELINE configs[2] (GPT-3 6.7B, ~107 GB replicated, DP=8): rank 3's
    13.3 GB shard, byte for byte (sha256 and CRC-32) against the oracle."""
    _one_rank_of_8_full_size(tmp_path, "c3_gpt3_6.7b", 3, 13.3e9)


@pytest.mark.slow
@pytest.mark.timeout(1500)
def test_c4_gpt3_13b_zero_rank0_of_8_full_size_parity(tmp_path):
    """BASELINE configs[3] (GPT-3 13B, ZeRO-partitioned, ~208 GB over 8):
    rank 0's 25.7 GB partition shard against the oracle."""
    _one_rank_of_8_full_size(tmp_path, "c4_gpt3_13b_zero", 0, 25.7e9)


@pytest.mark.slow
@pytest.mark.timeout(1700)
def test_c5_moe_rank0_of_8_full_size_parity(tmp_path):
    """BASELINE configs[4] (MoE GPT, 1.3B base, 64 experts, ~52B params, DP/EP
    = 8): rank 0's shard — its 1/8 of the replicated region (1.03 GB) and its
    8 local experts x 24 layers (103.1 GB) — against the oracle: ~111 GB of
    device state, a 104 GB shard (tmpfs when the disk is too small)."""
    free = torch.cuda.mem_get_info()[0]
    if free < 120e9:
        pytest.skip("needs ~120 GB of free device memory")
    _one_rank_of_8_full_size(tmp_path, "c5_moe_64e", 0, 104.1e9, tmpfs_ok=True)


@pytest.mark.parametrize("exchange", ["peer", "nccl"])
@pytest.mark.parametrize("cfg,k,slot", [("gpt3_small", 4, 1 << 20), ("moe_small", 2, 1 << 20),
                                        ("c1_tiny", 3, 1 << 20), ("gpt3_odd", 1, 1 << 20),
                                        ("gpt3_odd", 3, 64 << 10), ("c1_tiny", 8, 8 << 20)])
def test_load_parallel_device(tmp_path, monkeypatch, cfg, k, slot, exchange):
    """P:503 two-step load on device: own shard -> H2D -> exchange -> scatter.
    peer: every rank's partition in its own device buffer, fp_unpack_peer
    reads all writers' chunks from those buffers after their ready flags
    (thread ranks share one address space: the same pointers, no IPC);
    nccl: the comm's allgather_bytes per chunk + fp_unpack_v4."""
    monkeypatch.setenv("FP_LOAD_EXCHANGE", exchange)
    states = [_state(cfg, r, k) for r in range(k)]
    comms = ThreadComm.group(k)
    cks = [fp.Checkpointer(DEV, comm=comms[r], slot_bytes=slot) for r in range(k)]
    try:
        run_threads([lambda r=r: cks[r].save(entries(states[r]), str(tmp_path))
                     for r in range(k)])
        dst = [[(s, torch.full_like(t, 9) if t.is_floating_point() else torch.zeros_like(t))
                for s, t in states[r]] for r in range(k)]
        streams = [torch.cuda.Stream(DEV) for _ in range(k)]
        res = run_threads([lambda r=r: cks[r].load_parallel(entries(dst[r]), str(tmp_path),
                                                            stream=streams[r]) for r in range(k)])
        torch.cuda.synchronize()
        want = "none" if k == 1 else ("peer" if exchange == "peer" else "allgather_bytes")
        assert [x["exchange"] for x in res] == [want] * k
        assert all(x["status"] == 0 and x["kernel_launches"] > 0 for x in res)
        for r in range(k):
            for (_, a), (_, b) in zip(states[r], dst[r]):
                assert torch.equal(a.reshape(-1).view(torch.uint8), b.reshape(-1).view(torch.uint8))
    finally:
        for c in cks:
            c.close()


@pytest.mark.slow
@pytest.mark.timeout(1500)
def test_c2_full_size_load_parallel_dp4_thread_ranks(tmp_path):
    """SURVEY f1 at full size: C2 (21 GB) saved by 4 DP ranks, then restored
    with the paper's two-step load — each rank reads only its own
    5.3 GB shard into its device buffer and the partitions are exchanged over
    peer memory into every rank's own copy of the state — bit-exact on all 4
    ranks (thread ranks on one GPU: ~130 GB of device memory)."""
    free_dev = torch.cuda.mem_get_info(DEV)[0]
    if free_dev < 140e9:
        pytest.skip("needs ~140 GB of free device memory")
    free = os.statvfs(str(tmp_path))
    if free.f_bavail * free.f_frsize < 25e9:
        pytest.skip("needs ~25 GB free disk")
    k = 4
    st = _state("c2_gpt3_1.3b")
    comms = ThreadComm.group(k)
    cks = [fp.Checkpointer(DEV, comm=comms[r]) for r in range(k)]
    try:
        run_threads([lambda r=r: cks[r].save(entries(st), str(tmp_path)) for r in range(k)])
        dst = [[(s, torch.zeros_like(t)) for s, t in st] for _ in range(k)]
        streams = [torch.cuda.Stream(DEV) for _ in range(k)]
        res = run_threads([lambda r=r: cks[r].load_parallel(entries(dst[r]), str(tmp_path),
                                                            stream=streams[r]) for r in range(k)])
        torch.cuda.synchronize()
        assert [x["exchange"] for x in res] == ["peer"] * k
        assert all(x["status"] == 0 for x in res)
        for r in range(k):
            for (_, a), (_, b) in zip(st, dst[r]):
                assert torch.equal(a.reshape(-1).view(torch.uint8), b.reshape(-1).view(torch.uint8))
            dst[r] = None
    finally:
        for c in cks:
            c.close()
        for f in os.listdir(str(tmp_path)):
            if f.endswith(".fpck"):
                os.remove(os.path.join(str(tmp_path), f))
        torch.cuda.empty_cache()


@pytest.mark.parametrize("exchange", ["peer", "nccl"])
def test_load_parallel_device_detects_payload_corruption(tmp_path, monkeypatch, exchange):
    """The own-shard CRC-32 (GPU kernels over the H2D'd chunk) is checked
    against the manifest on load: a flipped payload byte fails every rank."""
    monkeypatch.setenv("FP_LOAD_EXCHANGE", exchange)
    k = 2
    states = [_state("gpt3_small", r, k) for r in range(k)]
    comms = ThreadComm.group(k)
    cks = [fp.Checkpointer(DEV, comm=comms[r], slot_bytes=1 << 20) for r in range(k)]
    from paper_2406_13768_b200.fastpersist import FP_ECORRUPT, FastPersistError
    try:
        run_threads([lambda r=r: cks[r].save(entries(states[r]), str(tmp_path))
                     for r in range(k)])
        p1 = os.path.join(str(tmp_path), fpck.shard_name(1, k))
        with open(p1, "r+b") as f:
            f.seek(os.path.getsize(p1) - 5000)
            b = f.read(1)
            f.seek(os.path.getsize(p1) - 5000)
            f.write(bytes([b[0] ^ 0x80]))
        codes = [None] * k

        def go(r):
            try:
                cks[r].load_parallel(entries(states[r]), str(tmp_path))
                codes[r] = 0
            except FastPersistError as e:
                codes[r] = e.code
        run_threads([lambda r=r: go(r) for r in range(k)])
        assert codes == [FP_ECORRUPT] * k
    finally:
        for c in cks:
            c.close()


def test_stream_ordered_fence_holds_the_optimizer(tmp_path):
    """fp_ckpt_fence (a9): the 'optimizer' enqueued on the fenced stream right
    after begin() must not run before this rank's shard is durable, yet
    fence() itself returns without blocking the host."""
    import time
    st = _state("gpt3_small")
    lay = oracle_layout([st], 1)              # bytes BEFORE the update
    s = torch.cuda.Stream(DEV)
    with fp.Checkpointer(DEV, slot_bytes=64 << 10, ring_slots=2) as ck:
        ck.begin(entries(st), str(tmp_path), stream=s)
        t0 = time.perf_counter()
        ck.fence(stream=s)
        dt = time.perf_counter() - t0
        with torch.cuda.stream(s):            # the next optimizer step
            for _, t in st:
                if t.is_floating_point():
                    t.fill_(-7.0)
        ck.wait()
        torch.cuda.synchronize()
    assert dt < 0.05, f"fence blocked the host for {dt:.3f} s"
    _check_rank_files(str(tmp_path), lay, 1)   # the checkpoint is the pre-update state
    assert all(bool((t == -7.0).all()) for _, t in st if t.is_floating_point())


@pytest.mark.parametrize("slots", [1, 2, 3])
@pytest.mark.parametrize("how", ["load", "load_parallel"])
def test_load_read_ahead_ring_depths(tmp_path, slots, how):
    """Both loads read R chunks ahead over the pinned ring (slot j % R, refilled
    only after the H2D out of it completed): bit-exact round trip for ring
    depths 1..3 over many 1 MiB chunks, ragged tails included."""
    st = _state("gpt3_odd")
    with fp.Checkpointer(DEV, slot_bytes=1 << 20, ring_slots=slots, sqe_bytes=256 << 10) as ck:
        ck.save(entries(st), str(tmp_path))
        dst = [(s, torch.full_like(t, 7) if t.is_floating_point() else torch.zeros_like(t))
               for s, t in st]
        getattr(ck, how)(entries(dst), str(tmp_path))
        torch.cuda.synchronize()
    for (_, a), (_, b) in zip(st, dst):
        assert torch.equal(a.reshape(-1).view(torch.uint8), b.reshape(-1).view(torch.uint8))


@pytest.mark.parametrize("cfg,k,stride", [("gpt3_odd", 4, 2), ("moe_small", 4, 4),
                                          ("c1_tiny", 3, 2)])
def test_writer_stride_device(tmp_path, cfg, k, stride):
    """Writer subsets on device state ("use a subset of DP ranks"):
    only ranks 0, s, 2s, ... pack and write replicated bytes; every shard ==
    the oracle's, and both loads follow the writer's partition."""
    states = [_state(cfg, r, k) for r in range(k)]
    lay = oracle_layout(states, k)
    comms = ThreadComm.group(k)
    cks = [fp.Checkpointer(DEV, comm=comms[r], slot_bytes=1 << 20, writer_stride=stride)
           for r in range(k)]
    try:
        res = run_threads([lambda r=r: cks[r].save(entries(states[r]), str(tmp_path))
                           for r in range(k)])
        ext = fpck.shard_extents(lay, stride)
        for r in range(k):
            p = os.path.join(str(tmp_path), fpck.shard_name(r, k))
            assert file_sha(p) == fpck.shard_sha256(lay, r, stride), r
            assert res[r]["shard_bytes"] == sum(n for _, _, n in ext[r])
            if r % stride and not lay.regions:
                assert res[r]["shard_bytes"] == 0
        for how in ("load", "load_parallel"):
            dst = [[(s, torch.full_like(t, 5) if t.is_floating_point() else torch.zeros_like(t))
                    for s, t in states[r]] for r in range(k)]
            run_threads([lambda r=r: getattr(cks[r], how)(entries(dst[r]), str(tmp_path))
                         for r in range(k)])
            torch.cuda.synchronize()
            for r in range(k):
                for (_, a), (_, b) in zip(states[r], dst[r]):
                    assert torch.equal(a.reshape(-1).view(torch.uint8), b.reshape(-1).view(torch.uint8))
    finally:
        for c in cks:
            c.close()


@pytest.mark.parametrize("pack", ["v4", "bulk", "lsu"])
@pytest.mark.parametrize("cfg,k,exchange", [("c1_tiny", 7, "peer"), ("gpt3_odd", 3, "nccl"),
                                            ("moe_small", 4, "peer"), ("gpt3_odd", 1, "peer")])
def test_byte_balance_device(tmp_path, monkeypatch, cfg, k, exchange, pack):
    """Byte-granular balance on device state: the pack gathers
    from byte-shifted sources (shard starts unaligned in the image), the
    unaligned suffix goes through buffered I/O; shards == oracle
    (balance="bytes") and both loads restore bit-exact."""
    monkeypatch.setenv("FP_LOAD_EXCHANGE", exchange)
    states = [_state(cfg, r, k) for r in range(k)]
    lay = oracle_layout(states, k)
    comms = ThreadComm.group(k)
    cks = [fp.Checkpointer(DEV, comm=comms[r], slot_bytes=1 << 20, pack_bytes=3 << 20,
                           balance="bytes", pack=pack) for r in range(k)]
    try:
        run_threads([lambda r=r: cks[r].save(entries(states[r]), str(tmp_path)) for r in range(k)])
        import json
        man = json.load(open(os.path.join(str(tmp_path), "manifest.json")))
        for r in range(k):
            p = os.path.join(str(tmp_path), fpck.shard_name(r, k))
            assert file_sha(p) == fpck.shard_sha256(lay, r, balance="bytes"), r
            assert man["shards"][r]["crc32"] == fpck.shard_crc32(lay, r, balance="bytes")
        for how in ("load", "load_parallel"):
            dst = [[(s, torch.full_like(t, 5) if t.is_floating_point() else torch.zeros_like(t))
                    for s, t in states[r]] for r in range(k)]
            run_threads([lambda r=r: getattr(cks[r], how)(entries(dst[r]), str(tmp_path))
                         for r in range(k)])
            torch.cuda.synchronize()
            for r in range(k):
                for (_, a), (_, b) in zip(states[r], dst[r]):
                    assert torch.equal(a.reshape(-1).view(torch.uint8), b.reshape(-1).view(torch.uint8))
    finally:
        for c in cks:
            c.close()


_GDS_UNAVAILABLE = []   # reason, once the first GDS case found no cuFile driver

_GDS_CHILD = r"""
import os, sys, torch
sys.path.insert(0, os.environ["FP_ROOT"])
import paper_2406_13768_b200 as fp
from oracle import fpck
from tests._util import entries, oracle_layout
from tests.test_gpu import _check_rank_files
from workloads import config_specs, make_state
cfg, slot, pack_bytes, pack, d = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), sys.argv[4], sys.argv[5]
dev = torch.device("cuda", 0)
st = make_state(config_specs(cfg), dev)
lay = oracle_layout([st], 1)
try:
    ck = fp.Checkpointer(dev, io_engine="gds", slot_bytes=slot, pack_bytes=pack_bytes, pack=pack)
except fp.FastPersistError as e:
    if e.code == -38:                     # -ENOSYS: no usable libcufile on this host
        print("GDS_UNAVAILABLE", flush=True)
        os._exit(0)                       # skip atexit hooks of a stuck libcufile thread
    raise
with ck:
    for _ in range(2):
        s = ck.save(entries(st), d)
    assert s["engine"] == 4 and s["pack_launches"] > 0 and s["fallback"] in (0, 2), s
    _check_rank_files(d, lay, 1)
    dst = [(x, torch.full_like(t, 5) if t.is_floating_point() else torch.zeros_like(t)) for x, t in st]
    ck.load_parallel(entries(dst), d)
    torch.cuda.synchronize()
for (_, a), (_, b) in zip(st, dst):
    assert torch.equal(a.reshape(-1).view(torch.uint8), b.reshape(-1).view(torch.uint8))
print("gds ok", s["fallback"])
"""


@pytest.mark.parametrize("cfg,slot,pack_bytes,pack", [("c1_tiny", 64 << 20, 256 << 20, "v4"),
                                                      ("gpt3_odd", 1 << 20, 3 << 20, "v4"),
                                                      ("gpt3_odd", 1 << 20, 1 << 20, "bulk"),
                                                      ("moe_small", 4096, 8192, "v4")])
def test_gds_engine_parity(tmp_path, cfg, slot, pack_bytes, pack):
    """device slab -> cuFileWrite (GPUDirect Storage; compatibility
    mode on a box without nvidia-fs): shard sha256 and CRC-32 == oracle, and
    the shard loads back bit-exact. Runs in a child process under a timeout
    (libcufile is third-party code: a stall fails the test, not the suite)."""
    import subprocess
    import sys
    if _GDS_UNAVAILABLE:                      # probed by an earlier case of this run
        pytest.skip(_GDS_UNAVAILABLE[0])
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, FP_ROOT=root, PYTHONPATH=root)
    try:
        r = subprocess.run([sys.executable, "-c", _GDS_CHILD, cfg, str(slot), str(pack_bytes), pack,
                            str(tmp_path)], capture_output=True, text=True, env=env, timeout=240)
    except subprocess.TimeoutExpired:
        pytest.fail("GDS checkpoint did not finish within 240 s")
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    if "GDS_UNAVAILABLE" in r.stdout:
        _GDS_UNAVAILABLE.append("cuFile driver unavailable on this host (no nvidia-fs): " +
                                r.stderr[-300:])
        pytest.skip(_GDS_UNAVAILABLE[0])
    assert "gds ok" in r.stdout


@pytest.mark.parametrize("slot,pack_bytes", [(1 << 20, 3 << 20), (4096, 8192), (64 << 20, 256 << 20)])
def test_crc_lsu_kernel_parity(tmp_path, slot, pack_bytes):
    """pack="lsu" (ablation): page CRCs computed from the registers of the
    LSU pack (fp_pack_lsu_crc: per-chunk chains, Horner over the lane's
    chunks, nibble-table products) — same shard bytes, same CRC-32."""
    st = _state("gpt3_odd")
    lay = oracle_layout([st], 1)
    with fp.Checkpointer(DEV, pack="lsu", slot_bytes=slot, pack_bytes=pack_bytes) as ck:
        s = ck.save(entries(st), str(tmp_path))
    assert s["crc_valid"]
    _check_rank_files(str(tmp_path), lay, 1)


@pytest.mark.parametrize("env", ["FP_NO_TMA", "FP_CRC_COL", "FP_BULK_2CTA"])
def test_crc_pages_variant_parity(tmp_path, env):
    """The other page-CRC kernels give the same CRC-32 as the default
    (fp_crc_pages_tma, a lane per 128-B row of a page) and zlib: FP_NO_TMA=1,
    the LSU kernel used when no tensor map can be encoded; FP_CRC_COL=1, the
    TMA kernel with a lane per page (no lane combine); FP_BULK_2CTA=1 (with
    pack="bulk", no_crc): the bare TMA pack at two CTAs per SM, the shard
    still == oracle. Child processes (the switches are read once per
    process)."""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = ("import os,sys,torch; sys.path.insert(0, os.environ['FP_ROOT']);"
            "import paper_2406_13768_b200 as fp;"
            "from tests._util import entries, oracle_layout;"
            "from tests.test_gpu import _check_rank_files, _state;"
            "st=_state('gpt3_odd'); lay=oracle_layout([st],1); d=sys.argv[1];"
            "nc=os.environ.get('FP_BULK_2CTA')=='1';"
            "ck=fp.Checkpointer(torch.device('cuda',0), slot_bytes=1<<20, pack_bytes=3<<20, no_crc=nc);"
            "s=ck.save(entries(st), d); ck.close(); assert nc or s['crc_valid'];"
            "_check_rank_files(d, lay, 1, crc=not nc); print('ok')")
    env = dict(os.environ, FP_ROOT=root, PYTHONPATH=root, **{env: "1"})
    r = subprocess.run([sys.executable, "-c", code, str(tmp_path)], capture_output=True, text=True,
                       env=env, timeout=300)
    assert r.returncode == 0 and "ok" in r.stdout, r.stderr[-3000:]


def test_bench_json_line_contract(tmp_path):
    """bench.py's own arm end to end on the GPU (small workload): one JSON line
    with every key of the driver contract and the roofline / cpu_baseline /
    e2e / restore objects this tier asks for."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, FP_BENCH_CFG="c1_tiny", FP_BENCH_DIR=str(tmp_path))
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--steps", "2", "--warmup", "3",
                        "--no-overhead", "--nvme-bytes", "2e8", "--oracle-bytes", "2e7"],
                       capture_output=True, text=True, env=env, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
              "roofline", "cpu_baseline", "e2e", "gpu_launches", "clocks", "restore"):
        assert k in d, k
    assert d["value"] > 0 and d["steps"] == 2 and d["gpu_launches"] > 0
    for k in ("bound", "achieved", "peak", "unit", "frac", "traffic"):
        assert k in d["roofline"], k
    assert d["roofline"]["achieved"] > 0
    for k in ("value", "unit", "cores", "kind", "sample"):
        assert k in d["cpu_baseline"], k
    for k in ("value", "unit", "h2d_bytes_per_step", "d2h_bytes_per_step"):
        assert k in d["e2e"], k
    assert d["restore"]["value"] > 0, d["restore"]
    for k in ("sm_mhz", "sm_max_mhz", "reasons"):
        assert k in d["clocks"], k


@pytest.mark.parametrize("slots", [1, 2])
@pytest.mark.parametrize("nbytes", [1, 4095, 4096 * 3, (16 << 20) + 7])
def test_stream_write_tensor_parity(tmp_path, slots, nbytes):
    """fp_stream_write_device: a device tensor's bytes D2H'd straight into the
    page-locked IO buffer and written with O_DIRECT, the unaligned
    tail through the buffered descriptor: file == tensor bytes."""
    g = torch.Generator(device=DEV).manual_seed(nbytes + slots)
    t = torch.randint(0, 256, (nbytes,), dtype=torch.uint8, device=DEV, generator=g)
    p = str(tmp_path / "t.bin")
    w = fp.StreamWriter(p, io_buffer_bytes=1 << 20, ring_slots=slots, device=0)
    w.write_tensor(t[: nbytes // 2])
    w.write(t[nbytes // 2: nbytes // 2 + 3].cpu().numpy().tobytes())   # host bytes in between
    w.write_tensor(t[nbytes // 2 + 3:])
    st = w.close()
    assert open(p, "rb").read() == t.cpu().numpy().tobytes()
    assert st["bytes"] == nbytes and st["suffix_bytes"] == nbytes % 4096


def test_stream_torch_save_cuda_state(tmp_path):
    """torch.save of a CUDA state dict through StreamWriter == torch.save into
    a file object, and torch.load restores it on the GPU."""
    import io as _io
    st = {x.name: t for x, t in _state("gpt3_small")}
    p = str(tmp_path / "s.pt")
    fp.save(st, p, io_buffer_bytes=8 << 20)
    ref = _io.BytesIO()
    torch.save(st, ref)
    assert file_sha(p) == __import__("hashlib").sha256(ref.getvalue()).hexdigest()
    back = torch.load(p, map_location=DEV)
    assert all(torch.equal(back[k], v) for k, v in st.items())


def test_stream_write_tensor_large(tmp_path):
    """2 GiB + a ragged tail of device bytes through 128 MiB double-buffered
    IO buffers (many engine requests pending per slot): the file == the
    tensor's bytes (sha256 on both sides)."""
    import hashlib
    n = (2 << 30) + 4093
    g = torch.Generator(device=DEV).manual_seed(77)
    t = torch.randint(0, 256, (n,), dtype=torch.uint8, device=DEV, generator=g)
    p = str(tmp_path / "big.bin")
    w = fp.StreamWriter(p, io_buffer_bytes=128 << 20, ring_slots=2, device=0)
    w.write_tensor(t)
    st = w.close()
    assert st["bytes"] == n and st["suffix_bytes"] == n % 4096
    assert file_sha(p) == hashlib.sha256(t.cpu().numpy().tobytes()).hexdigest()
    os.remove(p)


def test_slab_falls_back_to_a_smaller_group_when_memory_is_short(tmp_path):
    """A device too full for the requested pack group: fp_ckpt_init halves
    the slab down to what fits (here 2 GiB -> 128 MiB with ~200 MiB free),
    the checkpoint runs with the smaller groups and is still == oracle."""
    st = _state("gpt3_small")
    lay = oracle_layout([st], 1)
    torch.cuda.empty_cache()
    free = torch.cuda.mem_get_info(DEV)[0]
    filler = torch.empty(free - (200 << 20), dtype=torch.uint8, device=DEV)
    try:
        with fp.Checkpointer(DEV, slot_bytes=16 << 20, pack_bytes=2 << 30) as ck:
            s = ck.save(entries(st), str(tmp_path))
        assert s["pack_launches"] == -(-lay.image_bytes // (128 << 20)) > 1
        _check_rank_files(str(tmp_path), lay, 1)
    finally:
        del filler
        torch.cuda.empty_cache()
