"""Test helpers: oracle layouts from torch state, a thread-backed fake comm."""
import hashlib
import threading

import torch

from oracle import fpck


def tbytes(t: torch.Tensor) -> bytes:
    return t.detach().contiguous().reshape(-1).view(torch.uint8).cpu().numpy().tobytes()


def lazy_reader(t: torch.Tensor):
    """OTensor data callable reading bytes straight from a (device) tensor."""
    flat = t.detach().reshape(-1).view(torch.uint8)

    def read(off, n):
        return flat[off:off + n].cpu().numpy().tobytes()
    return read


def otensor(spec_or_name, t, section="other", owner=-1, lazy=False, dtype=None):
    if hasattr(spec_or_name, "name"):
        s = spec_or_name
        name, dtype, section, owner, shape = s.name, s.dtype, s.section, s.owner, s.shape
    else:
        name, shape = spec_or_name, tuple(t.shape)
    return fpck.OTensor(name, dtype, section, owner, shape,
                        lazy_reader(t) if lazy else tbytes(t))


DT = {torch.float32: "f32", torch.bfloat16: "bf16", torch.float16: "f16",
      torch.float64: "f64", torch.int64: "i64", torch.int32: "i32", torch.uint8: "u8"}


def oracle_layout(states_by_rank, k, align=4096, lazy=False):
    """states_by_rank[r] = [(Spec, tensor)]; replicated entries taken from rank 0."""
    rep = [otensor(s, t, lazy=lazy) for s, t in states_by_rank[0] if s.owner < 0]
    local = [[otensor(s, t, lazy=lazy) for s, t in states_by_rank[r] if s.owner >= 0]
             for r in range(k)]
    return fpck.Layout(rep, local, k=k, align=align)


def file_sha(path):
    h = hashlib.sha256()
    with open(path, "rb") as f:
        while True:
            b = f.read(64 << 20)
            if not b:
                break
            h.update(b)
    return h.hexdigest()


def entries(state):
    return [(s.name, t, s.section, s.owner) for s, t in state]


class ThreadComm:
    """k ranks as threads of one process: allgather / allreduce_min via a barrier."""

    class _Shared:
        def __init__(self, k):
            self.k = k
            self.bar = threading.Barrier(k)
            self.slots = [None] * k

    def __init__(self, shared, rank):
        self.sh = shared
        self.rank = rank
        self.world = shared.k

    @classmethod
    def group(cls, k):
        sh = cls._Shared(k)
        return [cls(sh, r) for r in range(k)]

    def allgather(self, vals):
        self.sh.slots[self.rank] = list(vals)
        self.sh.bar.wait()
        out = [v for r in range(self.world) for v in self.sh.slots[r]]
        self.sh.bar.wait()
        return out

    def allreduce_min(self, v):
        self.sh.slots[self.rank] = v
        self.sh.bar.wait()
        out = min(self.sh.slots)
        self.sh.bar.wait()
        return out

    def allgather_bytes(self, send, recv, n, on_device, stream):
        """recv[r*n:(r+1)*n] = rank r's send (host memmove, or device copies
        ordered after each rank's stream work)."""
        import ctypes
        if on_device:
            from paper_2406_13768_b200.fastpersist import dev_bytes, torch_stream
            st = torch_stream(stream, torch.device("cuda", 0))
            st.synchronize()                       # our send is complete
        self.sh.slots[self.rank] = send
        self.sh.bar.wait()
        for r in range(self.world):
            if on_device:
                dst = dev_bytes(recv + r * n, n, torch.device("cuda", 0))
                with torch.cuda.stream(st):
                    dst.copy_(dev_bytes(self.sh.slots[r], n, torch.device("cuda", 0)))
            else:
                ctypes.memmove(recv + r * n, self.sh.slots[r], n)
        if on_device:
            st.synchronize()                       # peers may reuse their send
        self.sh.bar.wait()


def run_threads(fns):
    """Run callables concurrently; re-raise the first exception."""
    errs = [None] * len(fns)
    res = [None] * len(fns)

    def wrap(i):
        try:
            res[i] = fns[i]()
        except BaseException as e:  # noqa: BLE001
            errs[i] = e
    ths = [threading.Thread(target=wrap, args=(i,)) for i in range(len(fns))]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    for e in errs:
        if e is not None:
            raise e
    return res


class MirrorComm:
    """The collectives of ONE rank of a k-rank job, answered locally: every
    rank reports this rank's own facts. Exact for the BASELINE configs C3/C4
    (identical replicated lists; rank-local partitions of identical sizes and
    name lengths), so one GPU can write rank r's true shard of a DP=8 job.
    region_bytes: every rank's local-region size as the ORACLE lays it out —
    substituted into the plan's 4-u64 fact all-gather (region bytes, local
    count, replicated digest, replicated bytes; runtime.cpp ensure_plan) when
    the ranks' local regions differ (C5: expert names of other ranks have
    other lengths, so their region headers differ)."""

    def __init__(self, rank, k, region_bytes=None):
        self.rank, self.world = rank, k
        self.region_bytes = region_bytes

    def allgather(self, vals):
        vals = list(vals)
        if self.region_bytes is not None and len(vals) == 4:
            assert vals[0] == self.region_bytes[self.rank], "library and oracle disagree"
            return [x for q in range(self.world) for x in [self.region_bytes[q]] + vals[1:]]
        return vals * self.world

    def allreduce_min(self, v):
        return v
