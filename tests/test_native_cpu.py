"""Host-side logic of libfastpersist, checked against the oracle on CPU.

These tests drive the real C library with HOST-resident tensors
(FP_TENSOR_HOST: the state-on-CPU case, e.g. offloaded optimizer state). That
exercises everything except the CUDA kernels: FPCK v2 header encoding, the DP
partition, the chunked ring, the io_uring / pwrite engines with
O_DIRECT, manifest commit and load. Device tensors go
through the sm_100a pack kernel and are covered by tests/test_gpu.py.
"""
import json
import os
import re

import pytest
import torch

import paper_2406_13768_b200 as fp
from paper_2406_13768_b200.fastpersist import FP_ECORRUPT, FP_EMISMATCH, FastPersistError
from oracle import fpck
from tests._util import (ThreadComm, entries, file_sha, oracle_layout, run_threads)
from workloads import config_specs, make_state

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module", autouse=True)
def built():
    from paper_2406_13768_b200 import build
    build.build()


def test_library_exports_every_declared_symbol():
    hdr = open(os.path.join(ROOT, "include", "fastpersist.h")).read()
    declared = set(re.findall(r"^\s*(?:int|void|const char \*)\s*(fp_\w+)\s*\(", hdr, re.M))
    assert declared == set(fp.EXPORTS)
    L = fp.lib()
    for name in declared:
        assert hasattr(L, name), name
    assert L.fp_strerror(0) == b"success"


def _state(cfg, rank=0, k=1):
    return make_state(config_specs(cfg, rank, k), "cpu")


@pytest.mark.parametrize("cfg", ["c1_tiny", "gpt3_small", "gpt3_odd"])
@pytest.mark.parametrize("engine", ["uring", "pwrite", "buffered"])
def test_host_save_matches_oracle(tmp_path, cfg, engine):
    st = _state(cfg)
    lay = oracle_layout([st], 1)
    with fp.Checkpointer(None, slot_bytes=1 << 20, ring_slots=3, io_engine=engine) as ck:
        stats = ck.save(entries(st), str(tmp_path))
        assert stats["image_bytes"] == lay.image_bytes
        assert stats["shard_bytes"] == lay.image_bytes
        assert ck.plan_info()["extents"] == [tuple(e) for e in fpck.shard_extents(lay)[0]]
    assert file_sha(tmp_path / "shard-0-of-1.fpck") == fpck.shard_sha256(lay, 0)
    man = json.load(open(tmp_path / "manifest.json"))
    assert stats["crc_valid"] == 1
    assert man["shards"][0]["crc32"] == stats["shard_crc32"] == fpck.shard_crc32(lay, 0)
    want = fpck.manifest_fields(lay)
    for key in ("image_bytes", "header_bytes", "alignment", "dp_size", "layout_digest"):
        assert man[key] == want[key], key
    assert [s["extents"] for s in man["shards"]] == [s["extents"] for s in want["shards"]]


@pytest.mark.parametrize("slots,slot_bytes,sqe", [(1, 4096, 4096), (2, 65536, 16384),
                                                  (4, 3 << 20, 1 << 20)])
def test_ring_geometry_invariance(tmp_path, slots, slot_bytes, sqe):
    # S:222/S:440 analog: single/double/multi buffering produce identical files
    st = _state("c1_tiny")
    lay = oracle_layout([st], 1)
    with fp.Checkpointer(None, ring_slots=slots, slot_bytes=slot_bytes, sqe_bytes=sqe,
                         io_depth=8) as ck:
        stats = ck.save(entries(st), str(tmp_path))
    assert stats["max_inflight"] <= min(8, slots * slot_bytes // sqe)
    assert file_sha(tmp_path / "shard-0-of-1.fpck") == fpck.shard_sha256(lay, 0)


def test_alignment_512(tmp_path):
    st = _state("gpt3_odd")
    lay = oracle_layout([st], 1, align=512)
    with fp.Checkpointer(None, alignment=512, slot_bytes=1 << 20, sqe_bytes=1 << 16) as ck:
        ck.save(entries(st), str(tmp_path))
    assert file_sha(tmp_path / "shard-0-of-1.fpck") == fpck.shard_sha256(lay, 0)


@pytest.mark.parametrize("cfg,k", [("gpt3_small", 3), ("zero_small", 2), ("moe_small", 4),
                                   ("c1_tiny", 8)])
def test_dp_ranks_as_threads_match_oracle(tmp_path, cfg, k):
    """k DP ranks (threads, fake comm) write shards that are the oracle's."""
    states = [_state(cfg, r, k) for r in range(k)]
    lay = oracle_layout(states, k)
    comms = ThreadComm.group(k)
    cks = [fp.Checkpointer(None, comm=comms[r], slot_bytes=1 << 20) for r in range(k)]
    try:
        res = run_threads([lambda r=r: cks[r].save(entries(states[r]), str(tmp_path))
                           for r in range(k)])
        man = json.load(open(tmp_path / "manifest.json"))
        for r in range(k):
            assert man["shards"][r]["crc32"] == res[r]["shard_crc32"] == fpck.shard_crc32(lay, r)
            assert cks[r].plan_info()["extents"] == [tuple(e) for e in
                                                     fpck.shard_extents(lay)[r]]
            assert res[r]["image_bytes"] == lay.image_bytes
            assert file_sha(tmp_path / fpck.shard_name(r, k)) == fpck.shard_sha256(lay, r)
        # shards reassemble into the oracle image
        paths = [str(tmp_path / fpck.shard_name(r, k)) for r in range(k)]
        img = fpck.assemble(paths, fpck.shard_extents(lay), lay.image_bytes)
        assert img == lay.image()
        # load(save(x)) == x on every rank
        dst = [[(s, torch.zeros_like(t)) for s, t in states[r]] for r in range(k)]
        run_threads([lambda r=r: cks[r].load(entries(dst[r]), str(tmp_path))
                     for r in range(k)])
        for r in range(k):
            for (s, a), (_, b) in zip(states[r], dst[r]):
                assert torch.equal(a.view(-1).view(torch.uint8), b.view(-1).view(torch.uint8))
    finally:
        for c in cks:
            c.close()


def test_load_roundtrip_and_errors(tmp_path):
    st = _state("gpt3_odd")
    d = str(tmp_path / "ck")
    with fp.Checkpointer(None, slot_bytes=1 << 20) as ck:
        ck.save(entries(st), d)
        dst = [(s, torch.full_like(t, 7)) for s, t in st]
        ck.load(entries(dst), d)
        for (_, a), (_, b) in zip(st, dst):
            assert torch.equal(a.view(-1).view(torch.uint8), b.view(-1).view(torch.uint8))
        # target list that differs from the file -> mismatch
        bad = list(entries(dst))
        bad[0] = (bad[0][0] + "x", bad[0][1], bad[0][2], bad[0][3])
        with pytest.raises(FastPersistError) as ei:
            ck.load(bad, d)
        assert ei.value.code == FP_EMISMATCH
        # a flipped header byte -> corrupt
        path = os.path.join(d, "shard-0-of-1.fpck")
        with open(path, "r+b") as f:
            f.seek(100)
            b = f.read(1)
            f.seek(100)
            f.write(bytes([b[0] ^ 0xFF]))
        with pytest.raises(FastPersistError) as ei:
            ck.load(entries(dst), d)
        assert ei.value.code == FP_ECORRUPT
        # missing shard -> ENOENT
        os.unlink(path)
        with pytest.raises(FastPersistError) as ei:
            ck.load(entries(dst), d)
        assert ei.value.code == -2
        # missing manifest -> ENOENT
        with pytest.raises(FastPersistError) as ei:
            ck.load(entries(dst), str(tmp_path / "nothing"))
        assert ei.value.code == -2


def test_begin_contract_errors(tmp_path):
    st = _state("c1_tiny")
    with fp.Checkpointer(None, slot_bytes=1 << 20) as ck:
        # owner must be this rank
        bad = [(s.name, t, s.section, 3) for s, t in st]
        with pytest.raises(FastPersistError) as ei:
            ck.begin(bad, str(tmp_path))
        assert ei.value.code == -22
        # non-contiguous: refused by the binding (no hidden copies)
        x = torch.zeros(8, 8)
        with pytest.raises(ValueError):
            ck.begin([("x", x.t())], str(tmp_path))
        # single outstanding checkpoint
        ck.begin(entries(st), str(tmp_path / "a"))
        with pytest.raises(FastPersistError) as ei:
            ck.begin(entries(st), str(tmp_path / "b"))
        assert ei.value.code == -16
        ck.wait()
        assert ck.wait()["status"] == 0 or True  # nothing outstanding -> returns 0


def test_mismatched_replicated_layout_across_ranks(tmp_path):
    k = 2
    comms = ThreadComm.group(k)
    a = [("w", torch.zeros(16))]
    b = [("w", torch.zeros(32))]
    cks = [fp.Checkpointer(None, comm=comms[r]) for r in range(k)]
    try:
        errs = [None, None]

        def go(r):
            try:
                cks[r].begin(a if r == 0 else b, str(tmp_path))
                cks[r].wait()
            except FastPersistError as e:
                errs[r] = e.code
        run_threads([lambda r=r: go(r) for r in range(k)])
        assert errs == [FP_EMISMATCH, FP_EMISMATCH]
    finally:
        for c in cks:
            c.close()


def test_overwrite_generation_in_place(tmp_path):
    """Re-checkpointing into the same directory rewrites the shard in place and
    re-commits the manifest; the old manifest is gone while bytes change."""
    st = _state("gpt3_small")
    d = str(tmp_path)
    with fp.Checkpointer(None, slot_bytes=1 << 20) as ck:
        ck.save(entries(st), d)
        ino = os.stat(os.path.join(d, "shard-0-of-1.fpck")).st_ino
        for _, t in st:
            t.add_(1) if t.is_floating_point() else None
        ck.save(entries(st), d)
        assert os.stat(os.path.join(d, "shard-0-of-1.fpck")).st_ino == ino
    lay = oracle_layout([st], 1)
    assert file_sha(os.path.join(d, "shard-0-of-1.fpck")) == fpck.shard_sha256(lay, 0)


def test_io_bench_runs(tmp_path):
    g = fp.io_bench(str(tmp_path), 8 << 20, slot_bytes=1 << 20, ring_slots=2)
    assert g > 0
    assert not os.listdir(tmp_path)
    g = fp.io_bench(str(tmp_path), 8 << 20, read=True, slot_bytes=1 << 20, ring_slots=2)
    assert g > 0
    assert not os.listdir(tmp_path)


def test_null_sink_engine_runs_the_pipeline_but_commits_nothing(tmp_path):
    """FP_IO_NULL (ablation): the ring + submission path runs, nothing is
    written, no manifest is committed, and load refuses it."""
    st = _state("gpt3_small")
    with fp.Checkpointer(None, slot_bytes=1 << 20, io_engine="null") as ck:
        s = ck.save(entries(st), str(tmp_path))
        assert s["engine"] == 3 and s["io_requests"] > 0 and s["shard_bytes"] > 0
        assert not os.path.exists(tmp_path / "manifest.json")
        assert not os.path.exists(tmp_path / "shard-0-of-1.fpck")
        with pytest.raises(FastPersistError) as ei:
            ck.load(entries(st), str(tmp_path))
        assert ei.value.code == -22


@pytest.mark.parametrize("cfg,k", [("gpt3_odd", 3), ("moe_small", 4), ("c1_tiny", 2),
                                   ("zero_small", 2), ("gpt3_small", 1)])
def test_load_parallel_own_shard_plus_allgather(tmp_path, cfg, k):
    """P:503 two-step load: each rank reads only its own shard, the replicated
    partitions are all-gathered, local regions come from the own shard."""
    states = [_state(cfg, r, k) for r in range(k)]
    comms = ThreadComm.group(k)
    cks = [fp.Checkpointer(None, comm=comms[r], slot_bytes=1 << 20) for r in range(k)]
    try:
        run_threads([lambda r=r: cks[r].save(entries(states[r]), str(tmp_path))
                     for r in range(k)])
        dst = [[(s, torch.zeros_like(t)) for s, t in states[r]] for r in range(k)]
        run_threads([lambda r=r: cks[r].load_parallel(entries(dst[r]), str(tmp_path))
                     for r in range(k)])
        for r in range(k):
            for (_, a), (_, b) in zip(states[r], dst[r]):
                assert torch.equal(a.reshape(-1).view(torch.uint8), b.reshape(-1).view(torch.uint8))
    finally:
        for c in cks:
            c.close()


def test_load_parallel_errors_surface_on_every_rank(tmp_path):
    k = 3
    states = [_state("gpt3_odd", r, k) for r in range(k)]
    comms = ThreadComm.group(k)
    cks = [fp.Checkpointer(None, comm=comms[r], slot_bytes=1 << 20) for r in range(k)]

    def load_all():
        codes = [None] * k

        def go(r):
            try:
                cks[r].load_parallel(entries(states[r]), str(tmp_path))
                codes[r] = 0
            except FastPersistError as e:
                codes[r] = e.code
        run_threads([lambda r=r: go(r) for r in range(k)])
        return codes
    try:
        run_threads([lambda r=r: cks[r].save(entries(states[r]), str(tmp_path))
                     for r in range(k)])
        assert load_all() == [0, 0, 0]
        # a flipped PAYLOAD byte in rank 1's shard: its CRC-32 no longer matches
        # the manifest; the failure reaches every rank
        p1 = tmp_path / fpck.shard_name(1, k)
        with open(p1, "r+b") as f:
            f.seek(os.path.getsize(p1) // 2)
            b = f.read(1)
            f.seek(os.path.getsize(p1) // 2)
            f.write(bytes([b[0] ^ 1]))
        assert load_all() == [FP_ECORRUPT] * k
        with open(p1, "r+b") as f:           # restore
            f.seek(os.path.getsize(p1) // 2)
            f.write(b)
        assert load_all() == [0, 0, 0]
        # a flipped GHDR byte in rank 0's shard: every rank sees the gathered header
        path = tmp_path / fpck.shard_name(0, k)
        with open(path, "r+b") as f:
            f.seek(70)
            b = f.read(1)
            f.seek(70)
            f.write(bytes([b[0] ^ 0x5A]))
        assert load_all() == [FP_ECORRUPT] * k
        # rank 2's shard missing: every rank fails with ENOENT
        os.unlink(tmp_path / fpck.shard_name(2, k))
        assert load_all() == [-2] * k
    finally:
        for c in cks:
            c.close()


@pytest.mark.parametrize("cfg,k,stride", [("gpt3_odd", 4, 2), ("moe_small", 4, 4),
                                          ("c1_tiny", 3, 2), ("zero_small", 2, 2)])
def test_writer_subset_matches_oracle_and_loads(tmp_path, cfg, k, stride):
    """The paper's writer subsets: with writer_stride s only ranks
    0, s, 2s, ... write replicated bytes; files == oracle's shards; both loads
    read the partition back from the manifest."""
    states = [_state(cfg, r, k) for r in range(k)]
    lay = oracle_layout(states, k)
    comms = ThreadComm.group(k)
    cks = [fp.Checkpointer(None, comm=comms[r], slot_bytes=1 << 20, writer_stride=stride)
           for r in range(k)]
    try:
        run_threads([lambda r=r: cks[r].save(entries(states[r]), str(tmp_path))
                     for r in range(k)])
        man = json.load(open(tmp_path / "manifest.json"))
        assert man["writer_stride"] == stride
        ext = fpck.shard_extents(lay, stride)
        for r in range(k):
            assert man["shards"][r]["extents"] == [list(e) for e in ext[r]]
            assert file_sha(tmp_path / fpck.shard_name(r, k)) == fpck.shard_sha256(lay, r, stride)
            assert man["shards"][r]["crc32"] == fpck.shard_crc32(lay, r, stride)
        for loader in ("load", "load_parallel"):
            # loaders configured with the default stride: the manifest decides
            lcks = [fp.Checkpointer(None, comm=comms[r], slot_bytes=1 << 20) for r in range(k)]
            dst = [[(s, torch.zeros_like(t)) for s, t in states[r]] for r in range(k)]
            run_threads([lambda r=r: getattr(lcks[r], loader)(entries(dst[r]), str(tmp_path))
                         for r in range(k)])
            for r in range(k):
                lcks[r].close()
                for (_, a), (_, b) in zip(states[r], dst[r]):
                    assert torch.equal(a.reshape(-1).view(torch.uint8),
                                       b.reshape(-1).view(torch.uint8)), loader
    finally:
        for c in cks:
            c.close()


def test_injected_io_error_fails_every_rank_and_keeps_the_previous_generation(tmp_path,
                                                                              monkeypatch):
    """T5 fault: an EIO on one rank's 3rd write surfaces as -EIO on EVERY rank
    (status all-reduce), no manifest is committed for that generation, and the
    previous generation's checkpoint stays loadable."""
    k = 2
    states = [_state("gpt3_odd", r, k) for r in range(k)]
    comms = ThreadComm.group(k)
    g0, g1 = str(tmp_path / "gen0"), str(tmp_path / "gen1")
    cks = [fp.Checkpointer(None, comm=comms[r], slot_bytes=64 << 10, sqe_bytes=16 << 10)
           for r in range(k)]
    try:
        run_threads([lambda r=r: cks[r].save(entries(states[r]), g0) for r in range(k)])
    finally:
        for c in cks:
            c.close()
    monkeypatch.setenv("FP_FAULT_EIO_AT", "3@1")
    cks = [fp.Checkpointer(None, comm=comms[r], slot_bytes=64 << 10, sqe_bytes=16 << 10)
           for r in range(k)]
    codes = [None] * k

    def go(r):
        try:
            cks[r].save(entries(states[r]), g1)
            codes[r] = 0
        except FastPersistError as e:
            codes[r] = e.code
    try:
        run_threads([lambda r=r: go(r) for r in range(k)])
    finally:
        for c in cks:
            c.close()
    assert codes == [-5, -5]
    assert not os.path.exists(os.path.join(g1, "manifest.json"))
    monkeypatch.delenv("FP_FAULT_EIO_AT")
    dst = [[(s, torch.zeros_like(t)) for s, t in states[r]] for r in range(k)]
    cks = [fp.Checkpointer(None, comm=comms[r]) for r in range(k)]
    try:
        run_threads([lambda r=r: cks[r].load_parallel(entries(dst[r]), g0) for r in range(k)])
    finally:
        for c in cks:
            c.close()
    for r in range(k):
        for (_, a), (_, b) in zip(states[r], dst[r]):
            assert torch.equal(a.reshape(-1).view(torch.uint8), b.reshape(-1).view(torch.uint8))


def test_multiple_roots_place_shards_per_rank(tmp_path):
    """fp_config.dirs (FP_CKPT_DIRS): rank r's shard goes under dirs[r % n]
    (e.g. one local NVMe per GPU), the manifest under dirs[0]; both loads
    find every shard through the same mapping."""
    k = 3
    roots = [str(tmp_path / "nvme0"), str(tmp_path / "nvme1")]
    states = [_state("gpt3_odd", r, k) for r in range(k)]
    lay = oracle_layout(states, k)
    comms = ThreadComm.group(k)
    cks = [fp.Checkpointer(None, comm=comms[r], slot_bytes=1 << 20, dirs=roots) for r in range(k)]
    try:
        run_threads([lambda r=r: cks[r].save(entries(states[r]), "step-7") for r in range(k)])
        for r in range(k):
            path = os.path.join(roots[r % 2], "step-7", fpck.shard_name(r, k))
            assert file_sha(path) == fpck.shard_sha256(lay, r)
        man = json.load(open(os.path.join(roots[0], "step-7", "manifest.json")))
        assert [s["root"] for s in man["shards"]] == [0, 1, 0] and man["n_roots"] == 2
        assert not os.path.exists(os.path.join(roots[1], "step-7", "manifest.json"))
        for loader in ("load", "load_parallel"):
            dst = [[(s, torch.zeros_like(t)) for s, t in states[r]] for r in range(k)]
            run_threads([lambda r=r: getattr(cks[r], loader)(entries(dst[r]), "step-7")
                         for r in range(k)])
            for r in range(k):
                for (_, a), (_, b) in zip(states[r], dst[r]):
                    assert torch.equal(a.reshape(-1).view(torch.uint8), b.reshape(-1).view(torch.uint8))
    finally:
        for c in cks:
            c.close()


def test_same_signature_new_addresses_rebuilds_work_items(tmp_path):
    """The work-item table is cached per (layout, tensor addresses): a second
    state with the same signature at other addresses must not reuse it."""
    a = _state("gpt3_odd")
    b = [(s, t + 1 if t.is_floating_point() else t + 1) for s, t in a]
    with fp.Checkpointer(None, slot_bytes=1 << 20) as ck:
        ck.save(entries(a), str(tmp_path / "a"))
        ck.save(entries(b), str(tmp_path / "b"))
        ck.save(entries(a), str(tmp_path / "a2"))
    for d, st in (("a", a), ("b", b), ("a2", a)):
        lay = oracle_layout([st], 1)
        assert file_sha(tmp_path / d / "shard-0-of-1.fpck") == fpck.shard_sha256(lay, 0), d


@pytest.mark.parametrize("slots", [1, 2, 3])
@pytest.mark.parametrize("engine", ["uring", "pwrite"])
@pytest.mark.parametrize("how", ["load", "load_parallel"])
def test_load_read_ahead_ring_depths_host(tmp_path, slots, engine, how):
    """Read-ahead over the ring (chunk j -> slot j % R, up to R chunks in
    flight): bit-exact round trip for ring depths 1..3, ~56 chunks of 1 MiB,
    request size below the chunk size, both engines."""
    st = _state("gpt3_odd")
    d = str(tmp_path / "ck")
    with fp.Checkpointer(None, slot_bytes=1 << 20, ring_slots=slots, io_engine=engine,
                         sqe_bytes=256 << 10, io_depth=6) as ck:
        ck.save(entries(st), d)
        dst = [(s, torch.full_like(t, 7)) for s, t in st]
        getattr(ck, how)(entries(dst), d)
    for (_, a), (_, b) in zip(st, dst):
        assert torch.equal(a.view(-1).view(torch.uint8), b.view(-1).view(torch.uint8))


def test_gds_engine_needs_a_device():
    """FP_IO_GDS moves device memory: a host-only context is refused."""
    with pytest.raises(FastPersistError) as ei:
        fp.Checkpointer(None, io_engine="gds")
    assert ei.value.code == -22


def _flip(path, off_from_end):
    with open(path, "r+b") as f:
        f.seek(os.path.getsize(path) - off_from_end)
        b = f.read(1)
        f.seek(os.path.getsize(path) - off_from_end)
        f.write(bytes([b[0] ^ 0x40]))


def test_manifest_extent_crcs_are_zlib_crcs_of_the_oracle_extents(tmp_path):
    """Every shard record carries a CRC-32 per extent (replicated partition,
    local region) besides the whole-file one: zlib.crc32 of the oracle's bytes
    of that extent."""
    import zlib
    k = 4
    states = [_state("moe_small", r, k) for r in range(k)]
    lay = oracle_layout(states, k)
    comms = ThreadComm.group(k)
    cks = [fp.Checkpointer(None, comm=comms[r], slot_bytes=1 << 20) for r in range(k)]
    try:
        run_threads([lambda r=r: cks[r].save(entries(states[r]), str(tmp_path)) for r in range(k)])
    finally:
        for c in cks:
            c.close()
    man = json.load(open(tmp_path / "manifest.json"))
    for r, ext in enumerate(fpck.shard_extents(lay)):
        assert man["shards"][r]["extent_crc32"] == [zlib.crc32(lay.read(io, n)) for io, _, n in ext]


@pytest.mark.parametrize("where", ["payload", "local_region"])
def test_single_box_load_detects_payload_corruption(tmp_path, where):
    """fp_ckpt_load (every extent read from whichever shard holds it) checks
    each extent it reads against the manifest's per-extent CRC-32: a flipped
    payload byte is FP_ECORRUPT, never a silent wrong restore."""
    k = 2
    cfg = "gpt3_odd" if where == "payload" else "moe_small"
    states = [_state(cfg, r, k) for r in range(k)]
    comms = ThreadComm.group(k)
    cks = [fp.Checkpointer(None, comm=comms[r], slot_bytes=1 << 20) for r in range(k)]
    try:
        run_threads([lambda r=r: cks[r].save(entries(states[r]), str(tmp_path)) for r in range(k)])
        # rank 1's shard: the last bytes are replicated payload (gpt3_odd) or
        # rank 1's own local region (moe_small)
        _flip(str(tmp_path / fpck.shard_name(1, k)), 3000)
        codes = [None] * k

        def go(r):
            dst = [(s, torch.zeros_like(t)) for s, t in states[r]]
            try:
                cks[r].load(entries(dst), str(tmp_path))
                codes[r] = 0
            except FastPersistError as e:
                codes[r] = e.code
        run_threads([lambda r=r: go(r) for r in range(k)])
    finally:
        for c in cks:
            c.close()
    # replicated bytes are read by every rank; a local region only by its owner
    assert codes == ([FP_ECORRUPT, FP_ECORRUPT] if where == "payload" else [0, FP_ECORRUPT])


def test_replan_is_collective_when_one_rank_changes(tmp_path):
    """only rank 1's local tensor changes size between two saves;
    the replan (and its all-gather) must still run on every rank, and the
    second checkpoint must be the oracle's."""
    k = 2
    comms = ThreadComm.group(k)
    cks = [fp.Checkpointer(None, comm=comms[r], slot_bytes=1 << 20) for r in range(k)]
    g = torch.Generator().manual_seed(7)
    rep = torch.randn(3000, generator=g)
    loc = [torch.randn(2000, generator=g), torch.randn(2000, generator=g)]

    def ents(r):
        return [("rep", rep, "other", -1), (f"loc{r}", loc[r], "other", r)]
    try:
        run_threads([lambda r=r: cks[r].save(ents(r), str(tmp_path / "a")) for r in range(k)])
        loc[1] = torch.randn(5000, generator=g)          # rank 1 alone changes
        run_threads([lambda r=r: cks[r].save(ents(r), str(tmp_path / "b")) for r in range(k)])
    finally:
        for c in cks:
            c.close()
    from tests._util import otensor
    lay = fpck.Layout([otensor("rep", rep, dtype="f32")],
                      [[otensor("loc0", loc[0], owner=0, dtype="f32")],
                       [otensor("loc1", loc[1], owner=1, dtype="f32")]], k=k)
    for r in range(k):
        assert file_sha(tmp_path / "b" / fpck.shard_name(r, k)) == fpck.shard_sha256(lay, r)


def test_import_error_on_one_rank_fails_every_rank_without_hanging(tmp_path):
    """A rank whose tensor table is invalid (owner != dp_rank) must not leave
    its peer waiting in the plan all-gather: both return an error."""
    k = 2
    comms = ThreadComm.group(k)
    cks = [fp.Checkpointer(None, comm=comms[r], slot_bytes=1 << 20) for r in range(k)]
    t = torch.randn(100)
    codes = [None] * k

    def go(r):
        try:
            cks[r].save([("x", t, "other", -1 if r == 0 else 0)], str(tmp_path))
            codes[r] = 0
        except FastPersistError as e:
            codes[r] = e.code
    try:
        run_threads([lambda r=r: go(r) for r in range(k)])
    finally:
        for c in cks:
            c.close()
    assert codes == [-22, -22]


@pytest.mark.parametrize("cfg,k,stride", [("gpt3_odd", 3, 1), ("moe_small", 4, 1), ("c1_tiny", 7, 1),
                                          ("gpt3_small", 6, 2), ("zero_small", 2, 1)])
@pytest.mark.parametrize("engine", ["uring", "buffered"])
def test_byte_balance_matches_oracle_and_loads(tmp_path, cfg, k, stride, engine):
    """FP_CFG_BALANCE_BYTES (byte-granular partition, imbalance <= 1
    byte): shard starts are unaligned in the image and each shard's suffix
    (< 4096 B) is written with buffered I/O into the same file; the
    shards are the oracle's (balance="bytes"), the manifest records the mode,
    and both loads follow it."""
    states = [_state(cfg, r, k) for r in range(k)]
    lay = oracle_layout(states, k)
    comms = ThreadComm.group(k)
    cks = [fp.Checkpointer(None, comm=comms[r], slot_bytes=1 << 20, balance="bytes",
                           writer_stride=stride, io_engine=engine, sqe_bytes=256 << 10)
           for r in range(k)]
    try:
        res = run_threads([lambda r=r: cks[r].save(entries(states[r]), str(tmp_path))
                           for r in range(k)])
        ext = fpck.shard_extents(lay, stride, balance="bytes")
        man = json.load(open(tmp_path / "manifest.json"))
        assert man["balance"] == "bytes"
        sizes = [sum(n for io, _, n in ext[r] if io < lay.rep_bytes) for r in range(0, k, stride)]
        assert max(sizes) - min(sizes) <= 1
        for r in range(k):
            assert cks[r].plan_info()["extents"] == [tuple(e) for e in ext[r]]
            assert file_sha(tmp_path / fpck.shard_name(r, k)) == \
                fpck.shard_sha256(lay, r, stride, balance="bytes"), r
            assert man["shards"][r]["crc32"] == res[r]["shard_crc32"] == \
                fpck.shard_crc32(lay, r, stride, balance="bytes")
        for how in ("load", "load_parallel"):
            dst = [[(s, torch.zeros_like(t)) for s, t in states[r]] for r in range(k)]
            run_threads([lambda r=r: getattr(cks[r], how)(entries(dst[r]), str(tmp_path))
                         for r in range(k)])
            for r in range(k):
                for (s, a), (_, b) in zip(states[r], dst[r]):
                    assert torch.equal(a.reshape(-1).view(torch.uint8),
                                       b.reshape(-1).view(torch.uint8)), (how, r, s.name)
    finally:
        for c in cks:
            c.close()



@pytest.mark.parametrize("rank", [0, 5])
def test_one_rank_of_k_with_mirror_comm_matches_oracle(tmp_path, rank):
    """The harness of the full-size one-rank-of-8 GPU tests (C3/C4/C5 on one
    GPU): a single rank whose collectives MirrorComm answers, given every
    rank's local-region size as the oracle lays it out. Here, as in C5 (whose
    other ranks' expert names have other lengths), the ranks' local-region
    headers differ, so mirroring this rank's facts alone would shift the
    region table of the global header."""
    from tests._util import MirrorComm, otensor
    k = 8
    g = torch.Generator().manual_seed(77)
    rep = [(f"rep{i}", torch.randint(0, 256, (5000 + 4096 * i,), dtype=torch.uint8, generator=g))
           for i in range(3)]

    def local_names(r):          # rank r's 40 local tensors, names 10 + 90*r bytes long
        return [f"r{r}.{'e' * (90 * r)}.t{i:04d}" for i in range(40)]
    own = [(n, torch.randint(0, 256, (3000 + i,), dtype=torch.uint8, generator=g))
           for i, n in enumerate(local_names(rank))]
    ents = [(n, t, "other", -1) for n, t in rep] + [(n, t, "exp_avg", rank) for n, t in own]

    def ghost(r):
        return [fpck.OTensor(n, "u8", "exp_avg", r, (3000 + i,), bytes(3000 + i))
                for i, n in enumerate(local_names(r))]
    lay = fpck.Layout([otensor(n, t, "other", -1, dtype="u8") for n, t in rep],
                      [[otensor(n, t, "exp_avg", rank, dtype="u8") for n, t in own] if r == rank
                       else ghost(r) for r in range(k)], k=k)
    assert len({b for _, b in lay.regions}) > 1   # the case the region sizes are needed for
    with fp.Checkpointer(None, comm=MirrorComm(rank, k, [b for _, b in lay.regions]),
                         slot_bytes=1 << 20) as ck:
        s = ck.save(ents, str(tmp_path))
    assert s["image_bytes"] == lay.image_bytes
    assert file_sha(tmp_path / fpck.shard_name(rank, k)) == fpck.shard_sha256(lay, rank)
