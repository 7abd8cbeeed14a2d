"""fp_stream (the paper's torch.save integration, §5.1 P:532-533;
IO buffer single / double buffering P:467-473; aligned prefix + buffered
suffix into the same file P:477) on host bytes.

Oracle: the definition — torch.save into an in-memory file object (the same
serializer writing to a plain file object: "archive/" record prefix), and for
raw writes the concatenation of the bytes written. The stream must give the
same file byte for byte, whatever the IO buffer shape."""
import hashlib
import io
import os

import pytest
import torch

import paper_2406_13768_b200 as fp
from paper_2406_13768_b200.fastpersist import FastPersistError


def _torch_save_bytes(obj):
    b = io.BytesIO()
    torch.save(obj, b)
    return b.getvalue()


def _state(seed):
    g = torch.Generator().manual_seed(seed)
    return {"w": torch.randn(513, 1031, generator=g),
            "b": torch.randn(1031, generator=g).to(torch.bfloat16),
            "step": 12, "m": torch.randn(77, generator=g).double(), "e": torch.empty(0)}


@pytest.mark.parametrize("slots", [1, 2, 4])
@pytest.mark.parametrize("slot_bytes", [4096, 64 << 10, 1 << 20, 8 << 20])
def test_torch_save_through_stream_is_byte_identical(tmp_path, slots, slot_bytes):
    obj = _state(slots * 7 + slot_bytes)
    p = str(tmp_path / "ck.pt")
    st = fp.save(obj, p, io_buffer_bytes=slot_bytes, ring_slots=slots, sqe_bytes=4096)
    ref = _torch_save_bytes(obj)
    got = open(p, "rb").read()
    assert hashlib.sha256(got).digest() == hashlib.sha256(ref).digest()
    assert st["bytes"] == len(ref) == st["direct_bytes"] + st["suffix_bytes"]
    assert st["suffix_bytes"] == len(ref) % 4096     # only the unaligned tail
    out = torch.load(p)
    assert torch.equal(out["w"], obj["w"]) and torch.equal(out["b"], obj["b"])
    assert out["step"] == 12 and out["e"].numel() == 0


@pytest.mark.parametrize("sizes", [[0], [1], [4095], [4096], [4097], [3 * 65536 + 5],
                                   [1] * 5000, [65536, 0, 3, 65533, 70000, 4096 * 17 + 1]])
@pytest.mark.parametrize("slots", [1, 2])
@pytest.mark.parametrize("engine", ["uring", "pwrite"])
def test_raw_writes_concatenate(tmp_path, sizes, slots, engine):
    """Writes of any length (empty, 1 byte at a time, slot-crossing, exact
    slot multiples) -> the file is their concatenation, with either engine
    (io_uring, or the O_DIRECT pwrite thread pool)."""
    g = torch.Generator().manual_seed(sum(sizes) + slots)
    parts = [torch.randint(0, 256, (n,), dtype=torch.uint8, generator=g).numpy().tobytes()
             for n in sizes]
    p = str(tmp_path / "raw.bin")
    w = fp.StreamWriter(p, io_buffer_bytes=65536, ring_slots=slots, sqe_bytes=8192,
                        io_depth=4, io_engine=engine)
    for b in parts:
        assert w.write(b) == len(b)
    st = w.close()
    want = b"".join(parts)
    assert open(p, "rb").read() == want
    assert os.path.getsize(p) == st["bytes"] == len(want)


def test_memoryview_and_bytearray_inputs(tmp_path):
    p = str(tmp_path / "mv.bin")
    w = fp.StreamWriter(p, io_buffer_bytes=8192)
    w.write(memoryview(b"abc" * 3000)[5:])
    w.write(bytearray(b"\x00\xff" * 4099))
    w.close()
    assert open(p, "rb").read() == (b"abc" * 3000)[5:] + b"\x00\xff" * 4099


def test_stream_errors(tmp_path):
    with pytest.raises(FastPersistError):   # IO buffer not a multiple of the alignment
        fp.StreamWriter(str(tmp_path / "x"), io_buffer_bytes=1000)
    with pytest.raises(FastPersistError):   # missing directory: -ENOENT from open
        fp.StreamWriter(str(tmp_path / "no" / "such" / "x"))
    w = fp.StreamWriter(str(tmp_path / "y"))
    w.close()
    assert w.close() is not None            # idempotent
    with pytest.raises(ValueError):
        w.write(b"1")
    w2 = fp.StreamWriter(str(tmp_path / "z"))
    with pytest.raises(ValueError):          # no device at open
        w2.write_tensor(torch.zeros(4))
    w2.close()


def test_buffered_engine_and_no_fsync(tmp_path):
    obj = _state(3)
    p = str(tmp_path / "b.pt")
    fp.save(obj, p, io_engine="buffered", no_fsync=True)
    assert open(p, "rb").read() == _torch_save_bytes(obj)


def test_overwrite_longer_file_is_cut(tmp_path):
    """An existing longer file is overwritten in place and cut to the new
    stream's length (no stale tail)."""
    p = str(tmp_path / "o.bin")
    with open(p, "wb") as f:
        f.write(b"\xab" * 300000)
    w = fp.StreamWriter(p, io_buffer_bytes=8192)
    w.write(b"x" * 12345)
    w.close()
    assert open(p, "rb").read() == b"x" * 12345


def test_save_serializer_switches(tmp_path):
    """zip_crc32=False (torch's own compute_crc32 switch, this call only):
    the bytes equal torch.save under the same switch, torch.load reads them,
    and the switch is restored afterwards."""
    from torch.utils.serialization import config as tcfg
    obj = _state(11)
    p = str(tmp_path / "f.pt")
    fp.save(obj, p, zip_crc32=False)
    assert tcfg.save.compute_crc32 is True
    tcfg.save.compute_crc32 = False
    try:
        ref = _torch_save_bytes(obj)
    finally:
        tcfg.save.compute_crc32 = True
    assert open(p, "rb").read() == ref
    assert torch.equal(torch.load(p)["w"], obj["w"])


@pytest.mark.skipif(not os.path.exists("/dev/full"), reason="needs /dev/full")
@pytest.mark.parametrize("engine", ["uring", "pwrite"])
def test_write_error_surfaces_and_close_drains(engine):
    """A failing device (/dev/full: every write -ENOSPC) fails the stream on a
    later write and again at close; close still drains the engine and frees
    the stream (a new stream of the same shape reuses the buffer cleanly)."""
    import errno
    w = fp.StreamWriter("/dev/full", io_buffer_bytes=8192, io_engine=engine)
    with pytest.raises(FastPersistError) as e:
        for _ in range(50):
            w.write(b"x" * 10000)
    assert e.value.code == -errno.ENOSPC
    with pytest.raises(FastPersistError):
        w.close()
    w2 = fp.StreamWriter("/dev/full", io_buffer_bytes=8192, io_engine=engine)
    try:
        w2.write(b"y" * 100000)
    except FastPersistError:
        pass
    with pytest.raises(FastPersistError):
        w2.close()
    assert w2.close()["bytes"] > 0    # closed: the stats of the failed stream


def test_save_error_propagates_and_restores_switches(tmp_path):
    """An object torch.save cannot pickle: torch's own error propagates, the
    stream is freed and torch's serializer switches are restored."""
    from torch.utils.serialization import config as tcfg
    with pytest.raises(Exception) as e:
        fp.save({"f": lambda x: x}, str(tmp_path / "bad.pt"), zip_crc32=False)
    assert not isinstance(e.value, FastPersistError)
    assert tcfg.save.compute_crc32 is True
