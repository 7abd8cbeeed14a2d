"""Thin ctypes binding over libfastpersist (include/fastpersist.h).

Argument marshalling only: every byte of the checkpoint path (layout, pack
kernel, D2H staging, io_uring writes, manifest commit, load) runs in the native
library. torch is used for device memory, streams and torch.distributed
process groups (the two tiny collectives behind fp_comm).

    ck = Checkpointer(device=0, group=None)
    ck.begin([(name, tensor, section, owner), ...], "ckpt/step-12")  # after optimizer
    ...                                                             # fwd/bwd of next iter
    stats = ck.wait()                                               # before next optimizer
    ck.load(same_entries, "ckpt/step-12")

PAPER.md §4.3 P:511-515 (begin after optimizer, wait before the next one);
§4.2 P:483-503 (DP byte-range partition; load).
"""
from __future__ import annotations

import ctypes as C
import io
import os
from collections import namedtuple

import numpy as np
import torch

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "libfastpersist.so")

# ---- constants restated from include/fastpersist.h -------------------------
FP_EMISMATCH, FP_ECORRUPT, FP_ECUDA, FP_ENODEV, FP_ECOMM = -1001, -1002, -1003, -1004, -1005
FP_TENSOR_HOST = 1
FP_CFG_NO_FSYNC = 1
FP_CFG_PRIO_LOW = 2
FP_CFG_NO_CRC = 4
FP_CFG_BALANCE_BYTES = 8
IO_ENGINES = {"uring": 0, "pwrite": 1, "buffered": 2, "null": 3, "gds": 4}
PACK_IMPLS = {"v4": 0, "bulk": 1, "host": 2, "ce": 3, "lsu": 4}
SECTIONS = {"param": 0, "grad": 1, "master": 2, "exp_avg": 3, "exp_avg_sq": 4, "other": 5}
DTYPES = {torch.float32: 1, torch.bfloat16: 2, torch.float16: 3, torch.float64: 4,
          torch.int64: 5, torch.int32: 6, torch.uint8: 7}


class fp_tensor(C.Structure):
    _fields_ = [("data", C.c_void_p), ("nbytes", C.c_uint64), ("name", C.c_char_p),
                ("shape", C.c_int64 * 8), ("owner", C.c_int32), ("dtype", C.c_uint8),
                ("section", C.c_uint8), ("ndim", C.c_uint8), ("flags", C.c_uint8)]


AGFN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64),
                   C.c_uint64)
ARFN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.POINTER(C.c_int32))
ABFN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint64, C.c_int, C.c_void_p)


class fp_comm(C.Structure):
    _fields_ = [("ctx", C.c_void_p), ("allgather_u64", AGFN), ("allreduce_min_i32", ARFN),
                ("allgather_bytes", ABFN)]


class _DevBuf:
    """Zero-copy torch view of raw device bytes (CUDA array interface)."""

    def __init__(self, ptr, nbytes):
        self.__cuda_array_interface__ = {"shape": (int(nbytes),), "typestr": "|u1",
                                         "data": (int(ptr), False), "version": 3,
                                         "strides": None}


def dev_bytes(ptr, nbytes, device):
    return torch.as_tensor(_DevBuf(ptr, nbytes), device=device)


def torch_stream(handle, device):
    """torch view of a cudaStream_t handle (None/0 = the legacy default stream)."""
    if not handle:
        return torch.cuda.default_stream(device)
    return torch.cuda.ExternalStream(int(handle), device=device)


def host_bytes(ptr, nbytes):
    return torch.frombuffer((C.c_uint8 * int(nbytes)).from_address(int(ptr)), dtype=torch.uint8)


class fp_config(C.Structure):
    _fields_ = [("ring_slots", C.c_uint32), ("io_depth", C.c_uint32), ("slot_bytes", C.c_uint64),
                ("sqe_bytes", C.c_uint32), ("alignment", C.c_uint32), ("io_engine", C.c_uint32),
                ("pack_impl", C.c_uint32), ("pack_ctas", C.c_uint32), ("flags", C.c_uint32),
                ("dirs", C.c_char_p), ("writer_stride", C.c_uint32), ("pack_bytes", C.c_uint64)]


class fp_stats(C.Structure):
    _fields_ = [("image_bytes", C.c_uint64), ("header_bytes", C.c_uint64),
                ("shard_bytes", C.c_uint64), ("chunks", C.c_uint64),
                ("io_requests", C.c_uint64), ("pack_launches", C.c_uint64),
                ("pack_bytes", C.c_uint64), ("pack_ms", C.c_double), ("d2h_ms", C.c_double),
                ("t_total", C.c_double), ("t_helper", C.c_double), ("t_fsync", C.c_double),
                ("t_barrier", C.c_double), ("t_commit", C.c_double),
                ("t_io_stall", C.c_double), ("max_inflight", C.c_uint32),
                ("fallback", C.c_uint32), ("engine", C.c_int32), ("status", C.c_int32),
                ("err_offset", C.c_int64), ("shard_crc32", C.c_uint32), ("crc_valid", C.c_uint32),
                ("kernel_launches", C.c_uint64), ("crc_ms", C.c_double),
                ("numa_node", C.c_int32)]


class fp_load_stats(C.Structure):
    _fields_ = [("bytes_read", C.c_uint64), ("kernel_launches", C.c_uint64),
                ("t_total", C.c_double), ("exchange", C.c_int32), ("status", C.c_int32),
                ("t_exchange_wait", C.c_double), ("t_setup", C.c_double),
                ("t_read_wait", C.c_double)]


EXCHANGES = {0: "none", 1: "allgather_bytes", 2: "peer"}

EXPORTS = ("fp_config_default", "fp_ckpt_init", "fp_ckpt_begin", "fp_ckpt_fence", "fp_ckpt_wait",
           "fp_ckpt_load", "fp_ckpt_load_parallel", "fp_ckpt_load_stats", "fp_ckpt_plan_info",
           "fp_ckpt_destroy", "fp_strerror", "fp_io_bench", "fp_io_bench_read",
           "fp_stream_open", "fp_stream_write", "fp_stream_write_device", "fp_stream_close")


class fp_stream_stats(C.Structure):
    _fields_ = [("bytes", C.c_uint64), ("direct_bytes", C.c_uint64), ("suffix_bytes", C.c_uint64),
                ("t_total", C.c_double), ("t_fill", C.c_double), ("t_io_wait", C.c_double),
                ("t_fsync", C.c_double), ("fallback", C.c_uint32), ("requests", C.c_uint32)]

_lib = None


def lib():
    """Load libfastpersist.so (fails loudly: there is no fallback path)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: build it with "
                          "`python -m paper_2406_13768_b200.build` (nvcc, sm_100a)")
    L = C.CDLL(LIB_PATH)
    L.fp_config_default.argtypes = [C.POINTER(fp_config)]
    L.fp_ckpt_init.argtypes = [C.POINTER(fp_config), C.c_int, C.POINTER(fp_comm),
                               C.POINTER(C.c_void_p)]
    L.fp_ckpt_begin.argtypes = [C.c_void_p, C.POINTER(fp_tensor), C.c_size_t, C.c_char_p,
                                C.c_int, C.c_int, C.c_void_p]
    L.fp_ckpt_wait.argtypes = [C.c_void_p, C.POINTER(fp_stats)]
    L.fp_ckpt_fence.argtypes = [C.c_void_p, C.c_void_p]
    L.fp_ckpt_load.argtypes = [C.c_void_p, C.POINTER(fp_tensor), C.c_size_t, C.c_char_p,
                               C.c_int, C.c_int, C.c_void_p]
    L.fp_ckpt_load_parallel.argtypes = [C.c_void_p, C.POINTER(fp_tensor), C.c_size_t,
                                        C.c_char_p, C.c_int, C.c_int, C.c_void_p]
    L.fp_ckpt_load_stats.argtypes = [C.c_void_p, C.POINTER(fp_load_stats)]
    L.fp_ckpt_plan_info.argtypes = [C.c_void_p, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64),
                                    C.POINTER(C.c_uint64), C.c_uint32, C.POINTER(C.c_uint32)]
    L.fp_ckpt_destroy.argtypes = [C.c_void_p]
    L.fp_ckpt_destroy.restype = None
    L.fp_strerror.argtypes = [C.c_int]
    L.fp_strerror.restype = C.c_char_p
    L.fp_io_bench.argtypes = [C.c_char_p, C.c_uint64, C.POINTER(fp_config), C.c_int,
                              C.POINTER(C.c_double)]
    L.fp_io_bench_read.argtypes = [C.c_char_p, C.c_uint64, C.POINTER(fp_config), C.c_int,
                                   C.POINTER(C.c_double)]
    L.fp_stream_open.argtypes = [C.POINTER(fp_config), C.c_int, C.c_char_p,
                                 C.POINTER(C.c_void_p)]
    L.fp_stream_write.argtypes = [C.c_void_p, C.c_void_p, C.c_uint64]
    L.fp_stream_write_device.argtypes = [C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p]
    L.fp_stream_close.argtypes = [C.c_void_p, C.POINTER(fp_stream_stats)]
    _lib = L
    return L


class FastPersistError(RuntimeError):
    def __init__(self, code, what=""):
        self.code = code
        msg = lib().fp_strerror(code).decode()
        super().__init__(f"{what}: {msg} ({code})" if what else f"{msg} ({code})")


def _check(code, what):
    if code:
        raise FastPersistError(code, what)


Entry = namedtuple("Entry", "name tensor section owner")
Entry.__new__.__defaults__ = ("other", -1)


def _entries(tensors):
    if isinstance(tensors, dict):
        return [Entry(k, v) for k, v in tensors.items()]
    out = []
    for e in tensors:
        if isinstance(e, Entry):
            out.append(e)
        else:
            out.append(Entry(*e))
    return out


def make_config(**kw) -> fp_config:
    cfg = fp_config()
    lib().fp_config_default(C.byref(cfg))
    for k, v in kw.items():
        if v is None:
            continue
        if k == "io_engine":
            v = IO_ENGINES[v] if isinstance(v, str) else v
        elif k == "pack":
            k, v = "pack_impl", PACK_IMPLS[v] if isinstance(v, str) else v
        elif k == "no_fsync":
            k, v = "flags", cfg.flags | (FP_CFG_NO_FSYNC if v else 0)
        elif k == "no_crc":
            k, v = "flags", cfg.flags | (FP_CFG_NO_CRC if v else 0)
        elif k == "balance":
            k, v = "flags", (cfg.flags & ~FP_CFG_BALANCE_BYTES) | \
                (FP_CFG_BALANCE_BYTES if v == "bytes" else 0)
        elif k == "prio":
            k, v = "flags", (cfg.flags & ~FP_CFG_PRIO_LOW) | (FP_CFG_PRIO_LOW if v == "low" else 0)
        elif k == "dirs":
            v = (",".join(v) if isinstance(v, (list, tuple)) else v).encode()
        setattr(cfg, k, v)
    return cfg


class _CallbackComm:
    """fp_comm callbacks over any object with .rank, .world,
    .allgather(list[int]) -> list[int] (rank-major) and .allreduce_min(int) -> int
    (used by tests to run several ranks as threads of one process)."""

    def __init__(self, obj):
        self.obj = obj
        self.world = obj.world
        self.ag = AGFN(self._allgather)
        self.ar = ARFN(self._allreduce)
        self.ab = ABFN(self._allgather_bytes)
        self.struct = fp_comm(None, self.ag, self.ar,
                              self.ab if hasattr(obj, "allgather_bytes") else ABFN())

    def _allgather_bytes(self, _ctx, send, recv, n, on_device, stream):
        try:
            self.obj.allgather_bytes(send, recv, n, bool(on_device), stream)
            return 0
        except Exception as e:  # noqa: BLE001
            print(f"fastpersist: allgather_bytes failed: {e}")
            return -1

    def _allgather(self, _ctx, send, recv, n):
        try:
            vals = self.obj.allgather([send[i] for i in range(n)])
            for i, v in enumerate(vals):
                recv[i] = v
            return 0
        except Exception as e:  # noqa: BLE001
            print(f"fastpersist: allgather failed: {e}")
            return -1

    def _allreduce(self, _ctx, inout):
        try:
            inout[0] = int(self.obj.allreduce_min(int(inout[0])))
            return 0
        except Exception as e:  # noqa: BLE001
            print(f"fastpersist: allreduce failed: {e}")
            return -1


class _Comm:
    """fp_comm callbacks over a torch.distributed group (NCCL or gloo).

    The two tiny control collectives (plan all-gather, status all-reduce) run
    on a private side stream when the group is NCCL: their host read-back then
    waits for the collective only, never for the caller's queued fwd/bwd or
    optimizer kernels (wait() is called before the optimizer, begin() after
    it: neither may drain the compute stream)."""

    def __init__(self, group, device):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        be = dist.get_backend(group)
        self.dev = device if be == "nccl" else torch.device("cpu")
        self.side = torch.cuda.Stream(self.dev) if self.dev.type == "cuda" else None
        self.world = dist.get_world_size(group)
        self.device = device
        self.ag = AGFN(self._allgather)
        self.ar = ARFN(self._allreduce)
        self.ab = ABFN(self._allgather_bytes)
        self.struct = fp_comm(None, self.ag, self.ar, self.ab)

    def _allgather_bytes(self, _ctx, send, recv, n, on_device, stream):
        """Parallel-load exchange: NCCL all-gather of device bytes
        ordered on the library's stream; host bytes over the group's backend."""
        try:
            if on_device:
                s = dev_bytes(send, n, self.device)
                r = dev_bytes(recv, n * self.world, self.device)
                with torch.cuda.stream(torch_stream(stream, self.device)):
                    if self.dev.type == "cuda":
                        self.dist.all_gather_into_tensor(r, s, group=self.group)
                    else:                    # non-NCCL group: stage through host memory
                        hs = s.cpu()
                        hr = torch.empty(n * self.world, dtype=torch.uint8)
                        self.dist.all_gather_into_tensor(hr, hs, group=self.group)
                        r.copy_(hr)
            else:
                s, r = host_bytes(send, n), host_bytes(recv, n * self.world)
                self.dist.all_gather_into_tensor(r, s, group=self.group)
            return 0
        except Exception as e:  # noqa: BLE001
            print(f"fastpersist: allgather_bytes failed: {e}")
            return -1

    def _ctl(self):
        import contextlib
        return torch.cuda.stream(self.side) if self.side is not None else contextlib.nullcontext()

    def _allgather(self, _ctx, send, recv, n):
        try:
            src = torch.tensor([send[i] for i in range(n)], dtype=torch.uint64).view(torch.int64)
            with self._ctl():
                out = torch.empty(self.world * n, dtype=torch.int64, device=self.dev)
                self.dist.all_gather_into_tensor(out, src.to(self.dev), group=self.group)
                vals = out.cpu().view(torch.uint64).tolist()
            for i, v in enumerate(vals):
                recv[i] = v
            return 0
        except Exception as e:  # noqa: BLE001 - surfaced as FP_ECOMM
            print(f"fastpersist: allgather failed: {e}")
            return -1

    def _allreduce(self, _ctx, inout):
        try:
            with self._ctl():
                t = torch.tensor([inout[0]], dtype=torch.int32, device=self.dev)
                self.dist.all_reduce(t, op=self.dist.ReduceOp.MIN, group=self.group)
                inout[0] = int(t.item())
            return 0
        except Exception as e:  # noqa: BLE001
            print(f"fastpersist: allreduce failed: {e}")
            return -1


def _stream_handle(stream, device):
    if device is None:
        return None
    if stream is None:
        stream = torch.cuda.current_stream(device)
    return C.c_void_p(stream.cuda_stream)


class Checkpointer:
    """One FastPersist context per rank (pinned ring, io_uring, helper thread)."""

    def __init__(self, device=None, group=None, comm=None, **cfg):
        if device is not None and device != "cpu":
            device = torch.device("cuda", torch.device(device).index
                                  if not isinstance(device, int) else device)
            if device.index is None:
                device = torch.device("cuda", torch.cuda.current_device())
        else:
            device = None
        self.device = device
        self.group = group
        import torch.distributed as dist
        if comm is not None:
            self.rank, self.world = comm.rank, comm.world
            self._comm = _CallbackComm(comm)
        else:
            dist_on = dist.is_available() and dist.is_initialized()
            self.rank = dist.get_rank(group) if dist_on else 0
            self.world = dist.get_world_size(group) if dist_on else 1
            self._comm = _Comm(group, device) if dist_on and self.world > 1 else None
        self.cfg = make_config(**cfg)
        h = C.c_void_p()
        _check(lib().fp_ckpt_init(C.byref(self.cfg), -1 if device is None else device.index,
                                  C.byref(self._comm.struct) if self._comm else None,
                                  C.byref(h)), "fp_ckpt_init")
        self.h = h
        self._keep = None

    # -- marshalling ---------------------------------------------------------
    def _table(self, tensors):
        ents = _entries(tensors)
        arr = (fp_tensor * max(1, len(ents)))()
        names = []
        for i, e in enumerate(ents):
            t = e.tensor
            if not t.is_contiguous():
                raise ValueError(f"{e.name}: non-contiguous tensor (no hidden copies)")
            if t.dtype not in DTYPES:
                raise ValueError(f"{e.name}: unsupported dtype {t.dtype}")
            if t.dim() > 8:
                raise ValueError(f"{e.name}: more than 8 dims")
            if t.is_cuda and (self.device is None or t.device != self.device):
                raise ValueError(f"{e.name}: tensor on {t.device}, checkpointer on {self.device}")
            nm = e.name.encode()
            names.append(nm)
            x = arr[i]
            x.data = t.data_ptr() if t.numel() else None
            x.nbytes = t.numel() * t.element_size()
            x.name = nm
            for d, s in enumerate(t.shape):
                x.shape[d] = s
            sec = SECTIONS[e.section] if isinstance(e.section, str) else int(e.section)
            x.owner, x.dtype, x.section, x.ndim = int(e.owner), DTYPES[t.dtype], sec, t.dim()
            x.flags = 0 if t.is_cuda else FP_TENSOR_HOST
        return arr, len(ents), (names, ents)

    # -- API -----------------------------------------------------------------
    def begin(self, tensors, path, stream=None):
        arr, n, keep = self._table(tensors)
        self._keep = (arr, keep)   # borrowed until wait() returns
        _check(lib().fp_ckpt_begin(self.h, arr, n, os.fsencode(path), self.rank, self.world,
                                   _stream_handle(stream, self.device)), "fp_ckpt_begin")

    def fence(self, stream=None):
        """Hold `stream` (default: current) on the GPU until this rank's shard
        is durable; returns immediately. Call wait() later for the commit."""
        _check(lib().fp_ckpt_fence(self.h, _stream_handle(stream, self.device)), "fp_ckpt_fence")

    def wait(self):
        st = fp_stats()
        code = lib().fp_ckpt_wait(self.h, C.byref(st))
        self._keep = None
        _check(code, "fp_ckpt_wait")
        return {f: getattr(st, f) for f, _ in fp_stats._fields_}

    def save(self, tensors, path, stream=None):
        self.begin(tensors, path, stream)
        return self.wait()

    def load_stats(self):
        ls = fp_load_stats()
        _check(lib().fp_ckpt_load_stats(self.h, C.byref(ls)), "fp_ckpt_load_stats")
        d = {f: getattr(ls, f) for f, _ in fp_load_stats._fields_}
        d["exchange"] = EXCHANGES.get(d["exchange"], d["exchange"])
        return d

    def load(self, tensors, path, stream=None):
        """Single-box restore: every needed extent from whichever shard holds it."""
        arr, n, keep = self._table(tensors)
        _check(lib().fp_ckpt_load(self.h, arr, n, os.fsencode(path), self.rank, self.world,
                                  _stream_handle(stream, self.device)), "fp_ckpt_load")
        return self.load_stats()

    def load_parallel(self, tensors, path, stream=None):
        """The paper's two-step load: own shard -> device, exchange over
        peer memory (or all-gather) -> unpack. Returns the load statistics."""
        arr, n, keep = self._table(tensors)
        _check(lib().fp_ckpt_load_parallel(self.h, arr, n, os.fsencode(path), self.rank,
                                           self.world, _stream_handle(stream, self.device)),
               "fp_ckpt_load_parallel")
        return self.load_stats()

    def plan_info(self):
        ib, hb, ne = C.c_uint64(), C.c_uint64(), C.c_uint32()
        ext = (C.c_uint64 * 48)()
        _check(lib().fp_ckpt_plan_info(self.h, C.byref(ib), C.byref(hb), ext, 16, C.byref(ne)),
               "fp_ckpt_plan_info")
        return {"image_bytes": ib.value, "header_bytes": hb.value,
                "extents": [tuple(ext[3 * i:3 * i + 3]) for i in range(ne.value)]}

    def close(self):
        if getattr(self, "h", None):
            lib().fp_ckpt_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()


def io_bench(directory, nbytes, tag=0, read=False, **cfg):
    """Built-in O_DIRECT sequential-write (read=True: read-back) roofline
    (fio substitute): GB/s."""
    c = make_config(**cfg)
    g = C.c_double()
    fn = lib().fp_io_bench_read if read else lib().fp_io_bench
    _check(fn(os.fsencode(directory), int(nbytes), C.byref(c), int(tag), C.byref(g)),
           "fp_io_bench_read" if read else "fp_io_bench")
    return g.value


class StreamWriter(io.RawIOBase):
    """Write-only file object over fp_stream (the paper's torch.save
    integration, §5.1): ``torch.save(obj, StreamWriter(path))``
    serialises as usual and every byte goes through the IO buffer with
    O_DIRECT. ``io_buffer_bytes`` = slot size, ``double_buffer``
    = 2 slots (False: the single-buffer mode). ``device`` (CUDA index) enables
    ``write_tensor``: a device tensor's bytes D2H'd straight into the
    page-locked buffer. ``close()`` flushes, fsyncs and returns the stats."""

    def __init__(self, path, io_buffer_bytes=None, double_buffer=True, device=None, **cfg):
        super().__init__()
        if io_buffer_bytes is not None:
            cfg["slot_bytes"] = int(io_buffer_bytes)
        cfg.setdefault("ring_slots", 2 if double_buffer else 1)
        c = make_config(**cfg)
        if device is None:
            self._dev = None
        else:
            idx = device if isinstance(device, int) else (torch.device(device).index or 0)
            self._dev = torch.device("cuda", idx)
        h = C.c_void_p()
        _check(lib().fp_stream_open(C.byref(c), -1 if self._dev is None else self._dev.index,
                                    os.fsencode(path), C.byref(h)), "fp_stream_open")
        self._h = h
        self.stats = None

    def writable(self):
        return True

    def write(self, b):
        if self._h is None:
            raise ValueError("write to a closed StreamWriter")
        a = np.frombuffer(b, dtype=np.uint8)  # no copy, read-only buffers too
        if a.size:
            _check(lib().fp_stream_write(self._h, a.ctypes.data, a.size), "fp_stream_write")
        return a.size

    def write_tensor(self, t):
        """Append the raw bytes of a contiguous device tensor (D2H into the IO
        buffer on the current stream)."""
        if self._dev is None or not t.is_cuda or not t.is_contiguous():
            raise ValueError("write_tensor needs a contiguous CUDA tensor and device= at open")
        n = t.numel() * t.element_size()
        st = torch.cuda.current_stream(t.device).cuda_stream
        _check(lib().fp_stream_write_device(self._h, t.data_ptr(), n, st), "fp_stream_write_device")
        return n

    def close(self):
        if self._h is not None:
            h, self._h = self._h, None
            s = fp_stream_stats()
            code = lib().fp_stream_close(h, C.byref(s))
            self.stats = {k: getattr(s, k) for k, _ in fp_stream_stats._fields_}
            super().close()
            _check(code, "fp_stream_close")
        return self.stats

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001 - never raise from a finaliser
            pass


def save(obj, path, zip_crc32=True, pinned_d2h=False, **kw):
    """torch.save(obj, path) through StreamWriter; returns the stream stats.

    zip_crc32 / pinned_d2h are torch.save's own serializer switches
    (torch.utils.serialization.config.save.compute_crc32 /
    use_pinned_memory_for_d2h), set for this call only. The defaults give
    exactly torch.save's bytes; zip_crc32=False skips the zip records' CRC-32
    (torch.load does not check it; zip tools then report bad CRCs) and
    pinned_d2h=True stages CUDA storages through pinned memory — the two costs
    that bound torch.save once the writes are fast."""
    from torch.utils.serialization import config as tcfg
    old = (tcfg.save.compute_crc32, tcfg.save.use_pinned_memory_for_d2h)
    tcfg.save.compute_crc32, tcfg.save.use_pinned_memory_for_d2h = bool(zip_crc32), bool(pinned_d2h)
    w = None
    try:
        w = StreamWriter(path, **kw)
        torch.save(obj, w)
        return w.close()
    except BaseException:
        if w is not None:   # free the stream; the original error is what propagates
            try:
                w.close()
            except FastPersistError:
                pass
        raise
    finally:
        tcfg.save.compute_crc32, tcfg.save.use_pinned_memory_for_d2h = old
