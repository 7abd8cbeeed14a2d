"""Pins of the CPU oracle (oracle/fpck.py) against things other than itself.

- hand-derived golden images (tests/golden/*.hex, written before the oracle);
- published FNV-1a-64 test vectors;
- closed forms fixed by the model definitions (16 B/param with GPT-3 shapes,
  PAPER.md P:191-192) and the paper's Table 2 checkpoint sizes;
- brute-force partition invariants;
- an independent decoder round trip and library byte views.
"""
import hashlib
import os
import random

import numpy as np
import pytest
import torch

from oracle import fpck
from workloads import config_specs, gpt3_param_count, make_state

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def tbytes(t: torch.Tensor) -> bytes:
    """Raw bytes of a tensor via torch/numpy library views (no method code)."""
    return t.detach().contiguous().reshape(-1).view(torch.uint8).numpy().tobytes()


def load_golden(name):
    size = None
    img = None
    unknown = set()
    extents = {}
    with open(os.path.join(GOLDEN, name)) as f:
        for line in f:
            line = line.split("#", 1)[0].strip()
            if not line:
                continue
            parts = line.split()
            if parts[0] == "size":
                size = int(parts[1])
                img = bytearray(size)
            elif parts[0] == "extents":
                r, io, fo, n = int(parts[1]), *(int(x, 16) for x in parts[2:5])
                extents.setdefault(r, []).append((io, fo, n))
            else:
                off = int(parts[0], 16)
                for i, b in enumerate(parts[1:]):
                    if b == "??":
                        unknown.add(off + i)
                    else:
                        img[off + i] = int(b, 16)
    return bytes(img), unknown, extents


def u8(data):
    return np.frombuffer(bytes(data), dtype=np.uint8)


# ---------------------------------------------------------------------------
def test_fnv1a64_published_vectors():
    # FNV-1a 64-bit reference vectors (Fowler/Noll/Vo test suite).
    assert fpck.fnv1a64(b"") == 0xCBF29CE484222325
    assert fpck.fnv1a64(b"a") == 0xAF63DC4C8601EC8C
    assert fpck.fnv1a64(b"foobar") == 0x85944171F73967E8


def _check_golden(img, gold, unknown):
    assert len(img) == len(gold)
    diff = [i for i in range(len(img)) if i not in unknown and img[i] != gold[i]]
    assert diff == [], f"first mismatches at {diff[:8]}"


def test_golden_single_tensor():
    gold, unknown, _ = load_golden("w_f32x2.hex")
    w = torch.tensor([1.0, -2.0], dtype=torch.float32)
    t = fpck.OTensor("w", "f32", "other", -1, (2,), tbytes(w))
    lay = fpck.Layout([t], k=1)
    img = lay.image()
    _check_golden(img, gold, unknown)
    # digest slot = FNV-1a-64 over (128-B entry table || names pool "w")
    dg = int.from_bytes(img[48:56], "little")
    assert dg == fpck.fnv1a64(img[64:192] + b"w")


def test_golden_local_regions_k2():
    gold, unknown, ext = load_golden("local_k2.hex")
    a = fpck.OTensor("a", "u8", "other", -1, (3,), bytes([1, 2, 3]))
    b = fpck.OTensor("b", "i32", "other", 0, (1,),
                     tbytes(torch.tensor([0x11223344], dtype=torch.int32)))
    lay = fpck.Layout([a], [[b], []], k=2)
    img = lay.image()
    _check_golden(img, gold, unknown)
    assert int.from_bytes(img[48:56], "little") == fpck.fnv1a64(img[0x40:0xC0] + b"a")
    assert int.from_bytes(img[0x2030:0x2038], "little") == \
        fpck.fnv1a64(img[0x2040:0x20C0] + b"b")
    got = fpck.shard_extents(lay)
    assert {r: got[r] for r in range(2)} == {r: ext[r] for r in range(2)}
    # shards concatenate back into the image
    s0, s1 = fpck.shard_bytes(lay, 0), fpck.shard_bytes(lay, 1)
    assert s0 == img[0:0x1000] + img[0x2000:0x4000]
    assert s1 == img[0x1000:0x2000] + img[0x4000:0x5000]


# ---------------------------------------------------------------------------
# closed forms fixed by the models and Table 2
# ---------------------------------------------------------------------------
def _zeros(n):
    return lambda off, m: b"\x00" * m


def _layout_of(specs, k=1, by_rank=None):
    rep = [fpck.OTensor(s.name, s.dtype, s.section, s.owner, s.shape, _zeros(s.nbytes))
           for s in specs if s.owner < 0]
    local = None
    if by_rank is not None:
        local = [[fpck.OTensor(s.name, s.dtype, s.section, s.owner, s.shape,
                               _zeros(s.nbytes)) for s in sp if s.owner >= 0]
                 for sp in by_rank]
    return fpck.Layout(rep, local, k=k)


def test_param_counts_match_model_definitions():
    # GPT-3 XL (1.3B) in the Megatron layout, vocab padded to 50304
    assert gpt3_param_count(2048, 24) == 1_315_819_520
    assert abs(gpt3_param_count(4096, 32) / 6.7e9 - 1) < 0.01
    assert abs(gpt3_param_count(5120, 40) / 13e9 - 1) < 0.02


@pytest.mark.parametrize("d,L,table_gb", [(1536, 24, 10), (2048, 24, 17),
                                          (2560, 32, 35), (4096, 32, 88),
                                          (5140, 40, 173)])
def test_14x_rule_vs_paper_table2(d, L, table_gb):
    # "checkpoint size ... roughly 14X of the parameter count";
    # Table 2 sizes match 14*P in GiB (reading R2); 13B with GPT-3's d=5140.
    P = gpt3_param_count(d, L)
    est = P * fpck.state_bytes_per_param("adam14") / 2**30
    assert abs(est / table_gb - 1) < 0.03, (est, table_gb)


def test_image_size_c1_closed_form():
    lay = _layout_of(config_specs("c1_tiny"))
    # 8 payloads padded to 4 KiB = 67,112,960 B, plus one header page
    assert lay.image_bytes == 67_117_056
    assert lay.header_bytes == 4096


@pytest.mark.parametrize("cfg,d,L", [("c2_gpt3_1.3b", 2048, 24),
                                     ("c3_gpt3_6.7b", 4096, 32)])
def test_image_size_gpt3_is_16_bytes_per_param(cfg, d, L):
    specs = config_specs(cfg)
    lay = _layout_of(specs)
    P = gpt3_param_count(d, L)
    # GPT-3 shapes: every payload is a 4 KiB multiple -> zero padding, so the
    # data region is exactly 16 B/param (adam16; BASELINE.json north_star).
    assert lay.image_bytes - lay.header_bytes == 16 * P
    assert lay.header_bytes % 4096 == 0
    n = len(specs)
    assert n == 5 * (12 * L + 4)
    names = sum(len(s.name.encode()) for s in specs)
    assert 64 + 128 * n + names <= lay.header_bytes < 64 + 128 * n + names + 4096


def test_adam14_profile_drops_grads():
    specs = config_specs("c2_gpt3_1.3b", profile="adam14")
    lay = _layout_of(specs)
    assert lay.image_bytes - lay.header_bytes == 14 * 1_315_819_520


def _names(specs):
    return sum(len(s.name.encode()) for s in specs)


def test_zero_partitioned_c4_image_closed_form():
    """C4 (GPT-3 13B, ZeRO over k=8): no replicated tensor, so the GHDR is one
    page (64 + 16*8 B of region table); each rank's region is its LHDR plus
    its dim-0 shards, 16*P/8 = 2P bytes of data plus the padding of the 1-D
    shards, derived by hand (d/8 = 640, 3d/8 = 1920, 4d/8 = 2560 elements):
      bf16 [640] 1280 B -> +2816, [1920] 3840 B -> +256, [2560] 5120 B -> +3072
      f32  [640] 2560 B -> +1536, [1920] 7680 B -> +512, [2560] 10240 B -> +2048
    per layer 6 x [d] + [3d] + [4d] in 2 bf16 + 3 f32 sections = 75,776 B,
    final LayerNorm 2 x [d] = 20,480 B: 40 * 75,776 + 20,480 = 3,051,520 B.
    Every 2-D shard row is 10,240 (bf16) or 20,480 (f32) bytes: no padding."""
    k = 8
    by_rank = [config_specs("c4_gpt3_13b_zero", r, k) for r in range(k)]
    lay = _layout_of([], k=k, by_rank=by_rank)
    P = 12_853_626_880
    assert gpt3_param_count(5120, 40) == P
    assert lay.header_bytes == 4096
    assert len(lay.regions) == k
    want = 4096
    for r, sp in enumerate(by_rank):
        assert len(sp) == 5 * 484
        H_r = -(-(64 + 128 * len(sp) + _names(sp)) // 4096) * 4096
        region = H_r + 2 * P + 3_051_520
        assert lay.regions[r] == (want, region), r
        want += region
    assert lay.image_bytes == want
    assert 205.6e9 < lay.image_bytes < 205.8e9          # BASELINE configs[3]: "~208 GB"


def test_moe_c5_image_closed_form():
    """C5 (MoE GPT 1.3B base, 64 experts in each of 24 layers, EP=8): every
    tensor is a page multiple (rows of 2048 bf16 = 4096 B), so the image is
    headers + 16 B/param exactly: 513,413,120 replicated params (embeddings
    103,022,592 + positions 4,194,304 + 24 x 16,924,672 per layer + 4,096
    final LN) and 64 x 24 x 33,564,672 = 51,555,336,192 expert params, 1/8 per
    rank."""
    k = 8
    by_rank = [config_specs("c5_moe_64e", r, k) for r in range(k)]
    rep = [s for s in by_rank[0] if s.owner < 0]
    lay = _layout_of(rep, k=k, by_rank=by_rank)
    P_rep, P_exp = 513_413_120, 51_555_336_192
    assert sum(s.numel for s in rep) == 5 * P_rep
    assert len(rep) == 5 * 220
    H = -(-(64 + 128 * len(rep) + 16 * k + _names(rep)) // 4096) * 4096
    assert lay.header_bytes == H
    assert lay.rep_bytes == H + 16 * P_rep
    want = lay.rep_bytes
    for r, sp in enumerate(by_rank):
        loc = [s for s in sp if s.owner >= 0]
        assert len(loc) == 5 * 8 * 24 * 4
        H_r = -(-(64 + 128 * len(loc) + _names(loc)) // 4096) * 4096
        assert lay.regions[r] == (want, H_r + 16 * P_exp // k), r
        want += H_r + 16 * P_exp // k
    assert lay.image_bytes == want
    assert abs(lay.image_bytes / 833.10e9 - 1) < 1e-3   # 833.10 GB


# ---------------------------------------------------------------------------
# partition: brute force over all small cases
# ---------------------------------------------------------------------------
def test_partition_brute_force():
    for Q in range(0, 65):
        for k in range(1, 9):
            parts = fpck.partition_units(Q, k)
            assert len(parts) == k
            cover = []
            for s, n in parts:
                cover.extend(range(s, s + n))
            assert cover == list(range(Q))              # tiles [0,Q) exactly once
            sizes = [n for _, n in parts]
            assert max(sizes) - min(sizes) <= 1          # balance within 1 unit
            assert sizes == sorted(sizes, reverse=True)  # extra units to low ranks
            assert parts == fpck.partition_units(Q, k)   # deterministic


def _rand_state(rng, n_rep, n_local, k):
    dts = ["f32", "bf16", "u8", "i64", "f16"]
    rep, local = [], [[] for _ in range(k)]
    for i in range(n_rep):
        dt = rng.choice(dts)
        shape = tuple(rng.randint(0, 5000) for _ in range(rng.randint(0, 2)))
        n = int(np.prod(shape)) if shape else 1
        data = bytes(rng.getrandbits(8) for _ in range(n * fpck.ITEMSIZE[dt]))
        rep.append(fpck.OTensor(f"r{i}", dt, rng.choice(list(fpck.SECTION_CODE)), -1,
                                shape, data))
    for j in range(n_local):
        r = rng.randrange(k)
        n = rng.randint(0, 9000)
        local[r].append(fpck.OTensor(f"l{j}", "u8", "other", r, (n,),
                                     bytes(rng.getrandbits(8) for _ in range(n))))
    return rep, local


@pytest.mark.parametrize("seed", range(6))
def test_extents_tile_image_and_decode_roundtrip(seed, tmp_path):
    rng = random.Random(seed)
    k = rng.randint(1, 8)
    rep, local = _rand_state(rng, rng.randint(0, 6), rng.randint(0, 5), k)
    align = rng.choice([512, 4096])
    lay = fpck.Layout(rep, local, k=k, align=align)
    img = lay.image()
    assert len(img) == lay.image_bytes and lay.image_bytes % align == 0
    # every byte of the image in exactly one extent; file offsets contiguous
    seen = np.zeros(lay.image_bytes, dtype=np.int32)
    for ext in fpck.shard_extents(lay):
        fo = 0
        for io, f, n in ext:
            assert f == fo and io % align == 0 and n % align == 0
            seen[io:io + n] += 1
            fo += n
    assert (seen == 1).all()
    # independent decoder recovers every tensor bit for bit (load(save(x)) == x)
    dec = fpck.decode(img)
    assert [(t["name"], t["data"], t["shape"], t["dtype"]) for t in dec["replicated"]] == \
        [(t.name, t.read(0, t.nbytes), t.shape, t.dtype) for t in rep]
    for r in range(k):
        got = dec["local"].get(r, [])
        assert [(t["name"], t["data"], t["owner"]) for t in got] == \
            [(t.name, t.read(0, t.nbytes), r) for t in local[r]]
    # oracle save -> files -> assemble == image; sha per shard matches
    shas = fpck.save(lay, str(tmp_path))
    paths = [str(tmp_path / fpck.shard_name(r, k)) for r in range(k)]
    assert fpck.assemble(paths, fpck.shard_extents(lay), lay.image_bytes) == img
    for r in range(k):
        with open(paths[r], "rb") as f:
            assert hashlib.sha256(f.read()).hexdigest() == shas[r]


def test_payloads_are_library_byte_views_and_padding_is_zero():
    specs = config_specs("c1_tiny")
    state = make_state(specs, "cpu")
    ts = [fpck.OTensor(s.name, s.dtype, s.section, s.owner, s.shape, tbytes(t))
          for s, t in state]
    lay = fpck.Layout(ts)
    img = u8(lay.image())
    dec = fpck.decode(img.tobytes())
    for (s, t), d in zip(state, dec["replicated"]):
        assert d["data"] == t.contiguous().reshape(-1).view(torch.uint8).numpy().tobytes()
        assert d["shape"] == tuple(t.shape)
    # bytes between payloads are zero: total nonzero-capable bytes = header + data
    mask = np.zeros(len(img), dtype=bool)
    mask[:lay.header_bytes] = True
    for off, t in zip(lay.rep_offsets, ts):
        mask[off:off + t.nbytes] = True
    assert not img[~mask].any()


def test_determinism_two_builds_identical():
    specs = config_specs("gpt3_small")
    st = make_state(specs, "cpu")
    shas = []
    for _ in range(2):
        ts = [fpck.OTensor(s.name, s.dtype, s.section, s.owner, s.shape, tbytes(t))
              for s, t in st]
        lay = fpck.Layout(ts, k=3)
        shas.append([fpck.shard_sha256(lay, r) for r in range(3)])
    assert shas[0] == shas[1]


def test_corruption_detected_by_decoder():
    w = fpck.OTensor("w", "f32", "other", -1, (2,), b"\x00" * 8)
    img = bytearray(fpck.Layout([w]).image())
    img[100] ^= 1           # inside the entry table -> digest mismatch
    with pytest.raises(ValueError):
        fpck.decode(bytes(img))


def test_required_bandwidth_eq1():
    # Eq. 1: 107 GB over a 4.28 s fwd+bwd window needs 25 GB/s
    assert fpck.required_bandwidth(107e9, 2.14, 2.14) == pytest.approx(25e9, rel=1e-3)


def test_crc32_library_pinned_to_check_value_and_oracle_shard_crc():
    """zlib.crc32 is CRC-32/IEEE: the catalogue check value of b"123456789" is
    0xCBF43926; the oracle's shard CRC is that routine over the shard bytes."""
    import zlib
    assert zlib.crc32(b"123456789") == 0xCBF43926
    st = make_state(config_specs("gpt3_odd"), "cpu")
    lay = fpck.Layout([fpck.OTensor(s.name, s.dtype, s.section, s.owner, s.shape, tbytes(t))
                       for s, t in st])
    assert fpck.shard_crc32(lay, 0) == zlib.crc32(lay.image())


@pytest.mark.parametrize("stride", [1, 2, 3, 4, 8])
def test_writer_subset_extents_brute_force(stride):
    """Writer subsets: only ranks 0, s, 2s, ... receive replicated
    pages; together they tile the replicated region once, page-balanced; the
    shards still reassemble into the image."""
    rng = random.Random(stride)
    nrng = np.random.default_rng(stride)
    for k in list(range(1, 9)) * 4:
        rep = [fpck.OTensor(f"r{i}", "u8", "other", -1, (n,), nrng.bytes(n))
               for i, n in enumerate(rng.randint(0, 20000) for _ in range(rng.randint(0, 6)))]
        local = [[] for _ in range(k)]
        for j in range(rng.randint(0, 4)):
            r, n = rng.randrange(k), rng.randint(0, 9000)
            local[r].append(fpck.OTensor(f"l{j}", "u8", "other", r, (n,), nrng.bytes(n)))
        lay = fpck.Layout(rep, local, k=k)
        ext = fpck.shard_extents(lay, stride)
        A = lay.align
        writers = [r for r in range(k) if r % stride == 0]
        rep_pages = []
        for r in range(k):
            rp = [(io, n) for io, _, n in ext[r] if io < lay.rep_bytes]
            if r not in writers:
                assert rp == []
            for io, n in rp:
                rep_pages.extend(range(io // A, (io + n) // A))
        assert rep_pages == list(range(lay.rep_bytes // A))
        sizes = [sum(n for io, _, n in ext[r] if io < lay.rep_bytes) for r in writers]
        assert max(sizes) - min(sizes) <= A
        # bytes of all shards placed at their image offsets give the image
        img = bytearray(lay.image_bytes)
        for r in range(k):
            data = fpck.shard_bytes(lay, r, stride)
            for io, fo, n in ext[r]:
                img[io:io + n] = data[fo:fo + n]
        assert bytes(img) == lay.image()


@pytest.mark.parametrize("stride", [1, 2, 3])
def test_byte_balance_extents_brute_force(stride):
    """Byte-granular balance ("partitions data on byte granularity
    ... tightly bound imbalance to at most one byte"): the writers' replicated
    byte counts differ by at most ONE BYTE, tile the replicated region once in
    rank order, and the shards (replicated bytes, then the local region)
    reassemble into the image; with every writer's share a page multiple the
    split equals the page-granular one."""
    rng = random.Random(100 + stride)
    nrng = np.random.default_rng(stride)
    for k in list(range(1, 9)) * 3:
        rep = [fpck.OTensor(f"r{i}", "u8", "other", -1, (n,), nrng.bytes(n))
               for i, n in enumerate(rng.randint(0, 30000) for _ in range(rng.randint(0, 5)))]
        local = [[] for _ in range(k)]
        for j in range(rng.randint(0, 3)):
            r, n = rng.randrange(k), rng.randint(0, 7000)
            local[r].append(fpck.OTensor(f"l{j}", "u8", "other", r, (n,), nrng.bytes(n)))
        lay = fpck.Layout(rep, local, k=k)
        ext = fpck.shard_extents(lay, stride, balance="bytes")
        writers = [r for r in range(k) if r % stride == 0]
        sizes = []
        pos = 0
        for r in range(k):
            rp = [(io, fo, n) for io, fo, n in ext[r] if io < lay.rep_bytes]
            if r not in writers:
                assert rp == []
                continue
            (io, fo, n), = rp
            assert io == pos and fo == 0                 # contiguous, rank order
            pos += n
            sizes.append(n)
        assert pos == lay.rep_bytes
        assert max(sizes) - min(sizes) <= 1              # the paper's one-byte bound
        assert sizes == sorted(sizes, reverse=True)      # extra bytes to the lowest writers
        img = bytearray(lay.image_bytes)
        for r in range(k):
            data = fpck.shard_bytes(lay, r, stride, balance="bytes")
            assert len(data) == sum(n for _, _, n in ext[r])
            for io, fo, n in ext[r]:
                img[io:io + n] = data[fo:fo + n]
        assert bytes(img) == lay.image()
        if (lay.rep_bytes // lay.align) % len(writers) == 0:   # page multiples: same split
            assert ext == fpck.shard_extents(lay, stride)
