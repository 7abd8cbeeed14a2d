"""FPCK v2 CPU oracle — TEST INFRASTRUCTURE, NOT PRODUCT CODE.

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s `cpu_baseline` /
`--impl reference` legs may import or execute anything under `oracle/`.
The product path (`paper_2406_13768_b200/`) never imports it and shares no
code, header, table or helper with it.

What it computes. FastPersist's checkpoint is "a sequence of writes of
serialized tensors" with metadata (§2.1.3), persisted in an
order that "remains unchanged" (§4.1), aligned for DMA/NVMe,
partitioned on byte granularity across DP ranks after serialization
(§4.2 "Load balancing") and written directly to persistent
storage (§3.2). The serialization itself is unspecified by the paper
(it reuses torch.save); this build fixes the FPCK v2 layout
(readings R1-R16). The oracle is that definition written out:

  image = GHDR || data(t0) || 0^pad0 || ... || LREG_0 || ... || LREG_{k-1}

and shard r = the bytes of rank r's extents concatenated in image order,
written with plain buffered write() + fsync (the paper's baseline I/O style).

Everything is plain Python + struct + hashlib; no blocking, no fusion.
Pins: tests/test_oracle.py (golden hex fixture, closed forms, brute-force
partition, independent decoder round trip, Table 2 sizing).
"""
from __future__ import annotations

import hashlib
import json
import os
import struct
import zlib

# ---------------------------------------------------------------------------
# Constants of the FPCK v2 layout. Restated here, not imported.
# ---------------------------------------------------------------------------
MAGIC = b"FPCK"
VERSION = 2
DEFAULT_ALIGN = 4096            # reading R4: 4 KiB (paper: "e.g., 512-byte")
FIXED_HDR = 64
ENTRY = 128
REGION = 16
FLAG_HAS_LOCAL = 1
FLAG_LOCAL = 2

DTYPE_CODE = {"f32": 1, "bf16": 2, "f16": 3, "f64": 4, "i64": 5, "i32": 6, "u8": 7}
CODE_DTYPE = {v: k for k, v in DTYPE_CODE.items()}
ITEMSIZE = {"f32": 4, "bf16": 2, "f16": 2, "f64": 8, "i64": 8, "i32": 4, "u8": 1}
SECTION_CODE = {"param": 0, "grad": 1, "master": 2, "exp_avg": 3, "exp_avg_sq": 4,
                "other": 5}
CODE_SECTION = {v: k for k, v in SECTION_CODE.items()}


class OTensor:
    """A tensor as the oracle sees it: metadata + raw little-endian bytes.

    `data` is a bytes-like object of length nbytes, or a callable
    (offset, length) -> bytes for states too large to hold twice in RAM.
    Floats are never converted: bytes are the tensor's raw bits (reading R11).
    """

    def __init__(self, name, dtype, section, owner, shape, data, nbytes=None):
        self.name = name
        self.dtype = dtype
        self.section = section
        self.owner = int(owner)
        self.shape = tuple(int(s) for s in shape)
        self.data = data
        numel = 1
        for s in self.shape:
            numel *= s
        self.nbytes = numel * ITEMSIZE[dtype] if nbytes is None else int(nbytes)
        if nbytes is not None:
            assert self.nbytes == numel * ITEMSIZE[dtype]

    def read(self, off, n):
        if callable(self.data):
            b = bytes(self.data(off, n))
        else:
            b = bytes(memoryview(self.data).cast("B")[off:off + n])
        assert len(b) == n
        return b


def round_up(x, a):
    return (x + a - 1) // a * a


def fnv1a64(data: bytes) -> int:
    """FNV-1a 64-bit (offset basis 0xcbf29ce484222325, prime 0x100000001b3)."""
    h = 0xCBF29CE484222325
    for byte in data:
        h ^= byte
        h = (h * 0x100000001B3) & 0xFFFFFFFFFFFFFFFF
    return h


# ---------------------------------------------------------------------------
# Header encoding (tensor metadata = dtype, size, originating device)
# ---------------------------------------------------------------------------
def header_len(n_tensors, n_regions, names_bytes, align):
    return round_up(FIXED_HDR + ENTRY * n_tensors + REGION * n_regions + names_bytes, align)


def encode_header(tensors, offsets, regions, align, total_bytes, owner, flags):
    """One FPCK header (global GHDR or a rank's LREG sub-header).

    tensors: OTensor list in caller order; offsets: absolute image offset of
    each payload; regions: [(offset, bytes)] (GHDR only); total_bytes:
    image_bytes for the GHDR, region bytes for an LREG."""
    names = [t.name.encode("utf-8") for t in tensors]
    pool = b"".join(names)
    hlen = header_len(len(tensors), len(regions), len(pool), align)
    table = b""
    name_off = 0
    for t, off, nm in zip(tensors, offsets, names):
        dims = list(t.shape) + [0] * (8 - len(t.shape))
        e = struct.pack("<QQIIBBBBi8q", off, t.nbytes, name_off, len(nm),
                        DTYPE_CODE[t.dtype], SECTION_CODE[t.section], len(t.shape), 0,
                        t.owner, *dims)
        e += b"\x00" * (ENTRY - len(e))
        table += e
        name_off += len(nm)
    digest = fnv1a64(table + pool)
    fixed = struct.pack("<4sIIIQQIIQQq", MAGIC, VERSION, align, flags, hlen, total_bytes,
                        len(tensors), len(regions), len(pool), digest, owner)
    assert len(fixed) == FIXED_HDR
    reg = b"".join(struct.pack("<QQ", o, b) for o, b in regions)
    body = fixed + table + reg + pool
    return body + b"\x00" * (hlen - len(body)), digest


# ---------------------------------------------------------------------------
# Layout: where every byte of the image comes from
# ---------------------------------------------------------------------------
class Layout:
    """The whole checkpoint image of a k-rank DP group.

    rep: replicated tensors (identical on all ranks), caller order.
    local: local[r] = rank r's own tensors (ZeRO / experts; reading R9).
    """

    def __init__(self, rep, local=None, k=1, align=DEFAULT_ALIGN):
        assert align >= 16 and align & (align - 1) == 0
        self.align = align
        self.k = k
        self.rep = list(rep)
        self.local = [list(x) for x in (local or [[] for _ in range(k)])]
        assert len(self.local) == k
        has_local = any(len(x) > 0 for x in self.local)
        n_reg = k if has_local else 0
        pool = sum(len(t.name.encode()) for t in self.rep)
        H = header_len(len(self.rep), n_reg, pool, align)
        # pieces: (image_offset, length, source) ; source = ("hdr", bytes) |
        # ("t", OTensor) | ("zero", None)
        self.pieces = []
        cur = H
        rep_off = []
        for t in self.rep:
            rep_off.append(cur)
            cur += round_up(t.nbytes, align)
        self.rep_bytes = cur                          # replicated region R (page multiple)
        self.rep_offsets = rep_off
        # local regions, rank order
        reg_hdrs = []
        regions = []
        for r in range(n_reg):
            lt = self.local[r]
            lpool = sum(len(t.name.encode()) for t in lt)
            Hr = header_len(len(lt), 0, lpool, align)
            start = cur
            offs = []
            c = start + Hr
            for t in lt:
                offs.append(c)
                c += round_up(t.nbytes, align)
            regions.append((start, c - start))
            reg_hdrs.append((lt, offs, c - start, r))
            cur = c
        self.image_bytes = cur
        self.regions = regions
        flags = FLAG_HAS_LOCAL if has_local else 0
        ghdr, self.digest = encode_header(self.rep, rep_off, regions, align,
                                          self.image_bytes, -1, flags)
        assert len(ghdr) == H
        self.header_bytes = H
        self.pieces.append((0, H, ("hdr", ghdr)))
        for t, off in zip(self.rep, rep_off):
            self._add_tensor(t, off)
        self.local_digests = []
        for (lt, offs, rb, r), (start, _) in zip(reg_hdrs, regions):
            h, dg = encode_header(lt, offs, [], align, rb, r, FLAG_LOCAL)
            self.local_digests.append(dg)
            self.pieces.append((start, len(h), ("hdr", h)))
            for t, off in zip(lt, offs):
                self._add_tensor(t, off)
        # sanity: pieces tile [0, image_bytes)
        pos = 0
        for off, n, _ in self.pieces:
            assert off == pos, (off, pos)
            pos += n
        assert pos == self.image_bytes

    def _add_tensor(self, t, off):
        if t.nbytes:
            self.pieces.append((off, t.nbytes, ("t", t)))
        pad = round_up(t.nbytes, self.align) - t.nbytes
        if pad:
            self.pieces.append((off + t.nbytes, pad, ("zero", None)))

    # -- bytes ---------------------------------------------------------------
    def read(self, off, n):
        """Image bytes [off, off+n), computed piece by piece."""
        assert 0 <= off and off + n <= self.image_bytes
        out = bytearray()
        end = off + n
        for poff, plen, (kind, src) in self.pieces:
            lo = max(off, poff)
            hi = min(end, poff + plen)
            if lo >= hi:
                continue
            if kind == "hdr":
                out += src[lo - poff:hi - poff]
            elif kind == "t":
                out += src.read(lo - poff, hi - lo)
            else:
                out += b"\x00" * (hi - lo)
        assert len(out) == n
        return bytes(out)

    def image(self):
        return self.read(0, self.image_bytes)


# ---------------------------------------------------------------------------
# Partition (P:487 fixed at setup; P:501-503 balanced, after serialization)
# ---------------------------------------------------------------------------
def partition_units(Q, k):
    """Split Q units into k contiguous ranges in rank order, sizes differing
    by at most one unit; the lowest ranks take the extra units."""
    out = []
    start = 0
    for w in range(k):
        n = Q // k + (1 if w < Q % k else 0)
        out.append((start, n))
        start += n
    assert start == Q
    return out


def shard_extents(layout: Layout, writer_stride=1, balance="pages"):
    """Per rank: [(image_offset, file_offset, length)] in image order.

    The replicated region is split over the writers — every rank, or with
    writer_stride s only ranks 0, s, 2s, ... (the paper's writer subsets, "use
    a subset of DP ranks") — in `alignment` pages (reading R5,
    the default), or with balance="bytes" in single bytes, the paper's own
    granularity ("partitions data on byte granularity ... imbalance to at most
    one byte"); rank r's local region LREG_r goes wholly to rank r
    and follows its replicated bytes in its file (reading R9)."""
    A = layout.align if balance == "pages" else 1
    assert balance in ("pages", "bytes")
    Q = layout.rep_bytes // A
    s = max(1, writer_stride)
    writers = [r for r in range(layout.k) if r % s == 0]
    wparts = dict(zip(writers, partition_units(Q, len(writers))))
    ext = []
    for r in range(layout.k):
        e = []
        fo = 0
        p0, npg = wparts.get(r, (0, 0))
        if npg:
            e.append((p0 * A, 0, npg * A))
            fo = npg * A
        if layout.regions:
            ro, rb = layout.regions[r]
            e.append((ro, fo, rb))
        ext.append(e)
    return ext


def shard_name(r, k):
    return f"shard-{r}-of-{k}.fpck"


def shard_bytes(layout, r, writer_stride=1, balance="pages"):
    return b"".join(layout.read(io, n)
                    for io, _, n in shard_extents(layout, writer_stride, balance)[r])


def iter_shard(layout, r, piece=64 << 20, writer_stride=1, balance="pages"):
    for io, _, n in shard_extents(layout, writer_stride, balance)[r]:
        p = 0
        while p < n:
            m = min(piece, n - p)
            yield layout.read(io + p, m)
            p += m


def shard_sha256(layout, r, writer_stride=1, balance="pages"):
    h = hashlib.sha256()
    for b in iter_shard(layout, r, writer_stride=writer_stride, balance=balance):
        h.update(b)
    return h.hexdigest()


def shard_crc32(layout, r, writer_stride=1, balance="pages"):
    """CRC-32 (IEEE 802.3 / zlib) of shard r's bytes — the integrity record the
    manifest carries per shard (SPEC.md S:157 checksums in the
    manifest). zlib.crc32 is the library routine; no custom arithmetic."""
    c = 0
    for b in iter_shard(layout, r, writer_stride=writer_stride, balance=balance):
        c = zlib.crc32(b, c)
    return c


def save(layout, dirpath, ranks=None, balance="pages"):
    """Write shard files with buffered write() + fsync; return {rank: sha256}.

    This is the slow baseline writer (one core, page cache, then fsync)."""
    os.makedirs(dirpath, exist_ok=True)
    shas = {}
    for r in (range(layout.k) if ranks is None else ranks):
        h = hashlib.sha256()
        with open(os.path.join(dirpath, shard_name(r, layout.k)), "wb") as f:
            for b in iter_shard(layout, r, balance=balance):
                f.write(b)
                h.update(b)
            f.flush()
            os.fsync(f.fileno())
        shas[r] = h.hexdigest()
    return shas


def manifest_fields(layout):
    """The manifest facts a reader needs: sizes, extents."""
    ext = shard_extents(layout)
    return {
        "format": "FPCK", "version": VERSION, "alignment": layout.align,
        "image_bytes": layout.image_bytes, "header_bytes": layout.header_bytes,
        "dp_size": layout.k, "layout_digest": layout.digest,
        "shards": [{"rank": r, "file": shard_name(r, layout.k),
                    "bytes": sum(n for _, _, n in ext[r]),
                    "extents": [list(x) for x in ext[r]]} for r in range(layout.k)],
    }


# ---------------------------------------------------------------------------
# Independent decoder (used for load(save(x)) == x)
# ---------------------------------------------------------------------------
def _decode_header(img, base):
    (magic, ver, align, flags, hlen, total, n, nreg, pool_len, digest,
     owner) = struct.unpack_from("<4sIIIQQIIQQq", img, base)
    if magic != MAGIC or ver != VERSION:
        raise ValueError(f"bad header at {base}")
    table = img[base + FIXED_HDR: base + FIXED_HDR + ENTRY * n]
    reg0 = base + FIXED_HDR + ENTRY * n
    regions = [struct.unpack_from("<QQ", img, reg0 + REGION * i) for i in range(nreg)]
    pool0 = reg0 + REGION * nreg
    pool = img[pool0: pool0 + pool_len]
    if fnv1a64(bytes(table) + bytes(pool)) != digest:
        raise ValueError(f"layout digest mismatch at {base}")
    if any(img[pool0 + pool_len: base + hlen]):
        raise ValueError("nonzero header padding")
    out = []
    for i in range(n):
        (off, nbytes, noff, nlen, dt, sec, ndim, _z, own,
         *dims) = struct.unpack_from("<QQIIBBBBi8q", img, base + FIXED_HDR + ENTRY * i)
        name = bytes(pool[noff:noff + nlen]).decode("utf-8")
        out.append(dict(name=name, dtype=CODE_DTYPE[dt], section=CODE_SECTION[sec],
                        owner=own, shape=tuple(dims[:ndim]),
                        data=bytes(img[off:off + nbytes])))
    return dict(align=align, flags=flags, header_bytes=hlen, total=total, owner=owner,
                regions=regions, tensors=out)


def decode(img):
    """Parse a full image -> {"replicated": [...], "local": {rank: [...]}}."""
    img = memoryview(img)
    g = _decode_header(img, 0)
    if g["total"] != len(img):
        raise ValueError("image_bytes mismatch")
    local = {}
    for r, (ro, rb) in enumerate(g["regions"]):
        h = _decode_header(img, ro)
        if h["total"] != rb or h["owner"] != r:
            raise ValueError(f"local region {r} header mismatch")
        local[r] = h["tensors"]
    return {"replicated": g["tensors"], "local": local, "align": g["align"]}


def assemble(shard_paths, extents, image_bytes):
    """Rebuild the image from shard files: place each extent's file bytes at
    its image offset (reader side of P:503). Raises if a byte is uncovered."""
    img = bytearray(image_bytes)
    covered = 0
    for path, ext in zip(shard_paths, extents):
        with open(path, "rb") as f:
            data = f.read()
        if len(data) != sum(n for _, _, n in ext):
            raise ValueError(f"shard {path}: size {len(data)} != extents")
        for io, fo, n in ext:
            img[io:io + n] = data[fo:fo + n]
            covered += n
    if covered != image_bytes:
        raise ValueError("extents do not cover the image")
    return bytes(img)


# ---------------------------------------------------------------------------
# Sizing closed forms ("checkpoint size ... roughly 14X")
# ---------------------------------------------------------------------------
def state_bytes_per_param(profile="adam14"):
    """adam14 = fp16 weights 2 + fp32 weights 4 + momentum 4 + variance 4
    (draft breakdown P:416-425); adam16 adds a 2-byte grad (reading R1)."""
    return {"adam14": 2 + 4 + 4 + 4, "adam16": 2 + 2 + 4 + 4 + 4}[profile]


def required_bandwidth(S_C, T_F, T_B):
    """Eq. 1: B_C >= S_C / (T_F + T_B)."""
    return S_C / (T_F + T_B)


def to_json(obj):
    return json.dumps(obj, sort_keys=True)
