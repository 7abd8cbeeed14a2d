"""bench.py — FastPersist B200 checkpoint-write benchmark (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...

`--gpus N` with N > 1 and no torchrun environment re-launches itself under
torch.distributed.run (N ranks, NCCL, one GPU per rank); rank 0 prints the
one JSON line.

Metric (BASELINE.json): "checkpoint persist GB/s and latency at 1/2/4/8 B200;
% iter overhead per-iter ckpt". Workload: BASELINE.json configs[1], GPT-3 1.3B
dense mixed-precision Adam state (adam16, 21,053,362,176-byte FPCK v2 image),
DP = N ranks, each persisting its page-balanced byte range (§4.2
P:483-503) through the pinned ring with O_DIRECT io_uring writes (§4.1
P:460-479). One step = one checkpoint: fp_ckpt_begin -> fp_ckpt_wait
(durable: fdatasync + status all-reduce + manifest commit, §3.2).
value = image bytes / max-over-ranks device-event time of the K steps.
Total work is fixed as N grows (the same 21 GB image is split N ways), so
"scaling" is "strong".

Extra keys beyond the base contract: roofline (pack kernel, HBM), nvme / pcie
rooflines measured in the same run, latency_s, overhead (per-iteration
checkpointing under a synthetic fwd/bwd GEMM stream, §4.3, with a
T_FB sweep and the Eq. 1 crossover), cpu_baseline (the
oracle on rank 0's host cores, every N), storage (per-rank shard roots, their
block devices and mounts, GPU -> NUMA node).
"""
from __future__ import annotations

import argparse
import json
import os
import shutil
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

# the workload BASELINE.json's metric is quoted on (configs[1]); FP_BENCH_CFG
# exists only so the GPU test suite can exercise the full JSON line quickly
CFG = os.environ.get("FP_BENCH_CFG", "c2_gpt3_1.3b")
# test hook: all ranks on cuda:0 over gloo (exercises the N>1 code path on a
# 1-GPU box; NCCL refuses two ranks on one device). Never used for numbers.
SHARE_GPU = os.environ.get("FP_BENCH_SHARE_GPU") == "1"
# test hook: host-resident state (FP_TENSOR_HOST), gloo, no CUDA: lets the CPU
# test suite drive the N-rank launch and JSON line. Never used for numbers.
HOST_HOOK = os.environ.get("FP_BENCH_HOST") == "1"
METRIC = "checkpoint persist GB/s and latency at 1/2/4/8 B200; % iter overhead per-iter ckpt"
SEQ, GBS_1P3B = 2048, 512          # PAPER.md Table tb:gpt-setup: 1.3B, GBS 512


# ---------------------------------------------------------------------------
# plumbing
# ---------------------------------------------------------------------------
def env_dist():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    lr = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, lr


def out_root():
    """Checkpoint directory root: FP_BENCH_DIR, else the repo copy on the box
    (same file system the probe measured), else /tmp."""
    d = os.environ.get("FP_BENCH_DIR")
    if d:
        return d
    base = os.environ.get("GRAFT_REPO_ROOT", ROOT)
    return os.path.join(base, "bench_ckpt")


def _coll_dev(dev):
    return dev if dist.get_backend() == "nccl" else torch.device("cpu")


def allreduce_max(x, dev):
    if not dist.is_initialized():
        return x
    t = torch.tensor([float(x)], dtype=torch.float64, device=_coll_dev(dev))
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def allreduce_sum(x, dev):
    if not dist.is_initialized():
        return x
    t = torch.tensor([float(x)], dtype=torch.float64, device=_coll_dev(dev))
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def barrier():
    if dist.is_initialized():
        dist.barrier()


class Clocks:
    """nvidia-smi sampler running during the timed region (B200_PROFILING.md)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.p = None
        self.lines = []

    def start(self):
        if not shutil.which("nvidia-smi"):
            return self
        self.p = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                   "-i", str(self.index), "-lms", "200"],
                                  stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        self.th = threading.Thread(target=self._read, daemon=True)
        self.th.start()
        return self

    def _read(self):
        for ln in self.p.stdout:
            self.lines.append(ln.strip())

    def stop(self):
        if not self.p:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.p.terminate()
        try:
            self.p.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.p.kill()
        self.th.join(timeout=2)
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = float(f[2])
            except ValueError:
                continue
            for n, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


def gpu_smi_id(dev):
    """nvidia-smi -i selector for this CUDA device (PCI bus id survives
    CUDA_VISIBLE_DEVICES remapping)."""
    try:
        p = torch.cuda.get_device_properties(dev)
        return "%08x:%02x:%02x.0" % (p.pci_domain_id, p.pci_bus_id, p.pci_device_id)
    except Exception:  # noqa: BLE001
        return str(dev.index)


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except OSError:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}, "fallback"


def d2h_roofline(dev, nbytes=256 << 20, reps=10):
    """cudaMemcpyAsync device -> pinned host, 256 MiB (BASELINE.md rooflines)."""
    src = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    dst = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    s = torch.cuda.Stream(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(s):
        dst.copy_(src, non_blocking=True)
        barrier()
        torch.cuda.synchronize(dev)
        e0.record(s)
        for _ in range(reps):
            dst.copy_(src, non_blocking=True)
        e1.record(s)
    torch.cuda.synchronize(dev)
    return nbytes * reps / (e0.elapsed_time(e1) / 1e3) / 1e9


# ---------------------------------------------------------------------------
# storage / NUMA topology (SURVEY §7 hard parts 1-2, §8(d): "state the drive
# and filesystem, the NUMA mapping")
# ---------------------------------------------------------------------------
def _sysfs(path, default=None):
    try:
        with open(path) as f:
            return f.read().strip()
    except OSError:
        return default


def gpu_bdf(index):
    try:
        p = torch.cuda.get_device_properties(index)
        return "%04x:%02x:%02x.0" % (p.pci_domain_id, p.pci_bus_id, p.pci_device_id)
    except Exception:  # noqa: BLE001
        return None


def numa_node_of(bdf):
    if not bdf:
        return -1
    v = _sysfs(f"/sys/bus/pci/devices/{bdf.lower()}/numa_node", "-1")
    try:
        return int(v)
    except ValueError:
        return -1


def nvme_mounts():
    """Writable file systems on NVMe block devices or on md RAID over NVMe:
    [(mountpoint, device, sysfs PCI path of the controller, "" for RAID)],
    from /proc/mounts."""
    out, seen = [], set()
    try:
        lines = open("/proc/mounts").read().splitlines()
    except OSError:
        return out
    for ln in lines:
        f = ln.split()
        if len(f) < 4 or "rw" not in f[3].split(","):
            continue
        dev = os.path.basename(f[0])
        if f[0].startswith("/dev/nvme"):
            base = dev.split("p")[0] if "p" in dev[4:] else dev     # nvme0n1p2 -> nvme0n1
            pci = os.path.realpath(f"/sys/block/{base}/device/device") \
                if os.path.exists(f"/sys/block/{base}") else ""
        elif f[0].startswith("/dev/md"):
            # software RAID over NVMe (a DGX's /raid): no single PCIe home
            slaves = os.listdir(f"/sys/block/{dev}/slaves") \
                if os.path.isdir(f"/sys/block/{dev}/slaves") else []
            if not any(x.startswith("nvme") for x in slaves):
                continue
            pci = ""
        else:
            continue
        if f[1] in seen or not os.access(f[1], os.W_OK):
            continue
        seen.add(f[1])
        out.append((f[1], f[0], pci))
    return out


def pick_shard_dirs(world, bdfs, mounts=None):
    """One shard root per rank (rank -> its GPU-local drive).

    FP_CKPT_DIRS (comma-separated) wins; otherwise each rank takes the NVMe
    mount whose controller shares the longest PCIe path prefix with its GPU
    (same switch), ties to the least-used mount. None when no NVMe mount is
    writable (the checkpoints then go under out_root())."""
    env = os.environ.get("FP_CKPT_DIRS")
    if env:
        return [d for d in env.split(",") if d]
    mounts = nvme_mounts() if mounts is None else mounts
    if not mounts:
        return None
    used = {m[0]: 0 for m in mounts}
    dirs = []
    for r in range(world):
        gp = os.path.realpath(f"/sys/bus/pci/devices/{bdfs[r].lower()}") if bdfs[r] else ""

        def common(pci):
            a, b = gp.split("/"), pci.split("/")
            n = 0
            while n < min(len(a), len(b)) and a[n] == b[n]:
                n += 1
            return n
        best = max(mounts, key=lambda m: (common(m[2]), -used[m[0]]))
        used[best[0]] += 1
        dirs.append(best[0])
    return dirs


def storage_record(dirs, bdfs):
    """lsblk / findmnt facts of the shard roots and the GPU -> NUMA map."""
    rec = {"dirs": dirs, "gpu_numa": {str(i): numa_node_of(b) for i, b in enumerate(bdfs)},
           "numa_nodes": len([d for d in os.listdir("/sys/devices/system/node")
                              if d.startswith("node")]) if os.path.isdir("/sys/devices/system/node")
           else None}
    mnts = []
    for d in sorted(set(dirs)):
        try:
            r = subprocess.run(["findmnt", "-n", "-o", "SOURCE,FSTYPE,OPTIONS", "-T", d],
                               capture_output=True, text=True, timeout=10)
            src, fst, opts = (r.stdout.split() + ["", "", ""])[:3]
            mnts.append({"dir": d, "source": src, "fstype": fst, "options": opts[:80]})
        except Exception:  # noqa: BLE001
            mnts.append({"dir": d, "source": None})
    rec["mounts"] = mnts
    try:
        r = subprocess.run(["lsblk", "-d", "-n", "-o", "NAME,TYPE,SIZE,ROTA,MODEL"],
                           capture_output=True, text=True, timeout=10)
        rec["lsblk"] = [" ".join(ln.split()) for ln in r.stdout.splitlines() if ln.strip()][:16]
    except Exception:  # noqa: BLE001
        rec["lsblk"] = None
    return rec


# ---------------------------------------------------------------------------
# reference arm: the CPU oracle on the host cores
# ---------------------------------------------------------------------------
def oracle_sample_tensors(specs, budget_bytes, seed_dev="cpu"):
    """A bounded prefix sample of the workload's tensor list (section-major
    state-dict order), host resident, about `budget_bytes` of payload."""
    from workloads import make_tensor
    out, tot = [], 0
    for s in specs:
        if tot >= budget_bytes:
            break
        out.append((s, make_tensor(s, seed_dev)))
        tot += s.nbytes
    return out, tot


def run_oracle_steps(sample, k_steps, root):
    """Time oracle saves (buffered write + fsync of the FPCK v2 image of the
    sample, 1 rank) -> (GB/s, per-step seconds, image bytes)."""
    from oracle import fpck

    def tb(t):
        return t.detach().contiguous().reshape(-1).view(torch.uint8).numpy().tobytes()
    times = []
    img = 0
    for i in range(k_steps):
        t0 = time.perf_counter()
        rep = [fpck.OTensor(s.name, s.dtype, s.section, s.owner, s.shape, tb(t))
               for s, t in sample]
        lay = fpck.Layout(rep, k=1)
        fpck.save(lay, os.path.join(root, f"oracle{i % 2}"))
        times.append(time.perf_counter() - t0)
        img = lay.image_bytes
    return img * len(times) / sum(times) / 1e9, times, img


def settle_io():
    """Flush dirty pages and (as root) drop the page cache before an oracle
    timing, so its buffered write() + fsync does not inherit writeback of
    earlier legs (round-1 spread: 0.37 vs 0.60 GB/s for the same oracle)."""
    os.sync()
    try:
        with open("/proc/sys/vm/drop_caches", "w") as f:
            f.write("3\n")
        return "synced, page cache dropped"
    except OSError:
        return "synced"


def cpu_cores():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count()


def reference_arm(a):
    ws, rank, _ = env_dist()
    if rank != 0:
        return 0
    from workloads import config_specs
    specs = config_specs(CFG, 0, a.gpus)
    budget = int(a.ref_bytes)
    sample, tot = oracle_sample_tensors(specs, budget)
    root = os.path.join(out_root(), "reference")
    os.makedirs(root, exist_ok=True)
    run_oracle_steps(sample, max(0, min(a.warmup, 1)), root)   # bounded warm-up
    io_state = settle_io()
    gbs, times, img = run_oracle_steps(sample, a.steps, root)
    shutil.rmtree(root, ignore_errors=True)
    sample_txt = (f"first {len(sample)} tensors of {CFG} in image order "
                  f"({img} image bytes, {img / 21053362176:.3%} of the full image), "
                  f"host-resident, buffered write() + fsync, 1 rank; before timing: {io_state}")
    line = {"metric": METRIC,
            "value": round(gbs, 4), "unit": "GB/s", "impl": "reference",
            "n_gpus": a.gpus, "steps": a.steps, "warmup": a.warmup,
            "ms_per_step": round(1e3 * statistics.mean(times), 2),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "u8", "data": "synthetic",
            "config": {"workload": CFG, "dp": a.gpus, "oracle_sample": sample_txt},
            "cpu_baseline": {"value": round(gbs, 4), "unit": "GB/s", "cores": 1,
                             "kind": "oracle", "sample": sample_txt},
            "e2e": {"value": round(gbs, 4), "unit": "GB/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------
def synthetic_overhead(a, ck, ents, state, dev, rank, world, path_of, image_gb, persist_gbs):
    """Per-iteration checkpointing under a synthetic training loop (§4.3,
    P:511-517): fwd (reads every bf16 param) + bf16 GEMM loop sized to T_FB +
    bwd (writes every grad) -> wait() -> optimizer (foreach update of master,
    m, v + bf16 param copy) -> begin(). The checkpointed state is the paper's
    14 B/param (params, master, m, v): grads are rewritten by every
    backward inside the overlap window, so they cannot be checkpointed
    without a snapshot (fastpersist.h: tensors immutable from begin to wait).
    overhead = median iteration with checkpointing / median without - 1,
    swept over T_FB (the GAS-sweep analog of P:736) with the Eq. 1 crossover
    S_C / B."""
    n = 8192
    A = torch.randn(n, n, device=dev, dtype=torch.bfloat16)
    B = torch.randn(n, n, device=dev, dtype=torch.bfloat16)
    C = torch.empty(n, n, device=dev, dtype=torch.bfloat16)
    torch.cuda.synchronize(dev)
    for _ in range(10):
        torch.matmul(A, B, out=C)
    torch.cuda.synchronize(dev)
    t0 = time.perf_counter()
    for _ in range(50):
        torch.matmul(A, B, out=C)
    torch.cuda.synchronize(dev)
    t_gemm = allreduce_max((time.perf_counter() - t0) / 50, dev)
    by_sec = {}
    for (s, t) in state:
        by_sec.setdefault(s.section, []).append(t)
    master, m, v, param, grad = (by_sec.get(x, []) for x in
                                 ("master", "exp_avg", "exp_avg_sq", "param", "grad"))
    ov_ents = [e for e in ents if e[2] != "grad"]
    ov_bytes = sum(t.numel() * t.element_size() for _, t, sec, _ in ov_ents)

    def fwd_bwd(n_gemm):
        if param:
            torch._foreach_norm(param)               # fwd reads the params
        for _ in range(n_gemm):
            torch.matmul(A, B, out=C)
        if grad:
            torch._foreach_add_(grad, 1e-6)          # bwd writes the grads

    def optimizer():
        # memory-bound like Adam: read/write master, m, v; write bf16 params
        torch._foreach_mul_(m, 0.9)
        torch._foreach_mul_(v, 0.999)
        torch._foreach_add_(master, m, alpha=-1e-8)
        for p, w in zip(param, master):
            p.copy_(w)

    def loop(ckpt, n_gemm, warm, iters):
        its = []
        for i in range(warm + iters):
            torch.cuda.synchronize(dev)
            barrier()
            t0 = time.perf_counter()
            fwd_bwd(n_gemm)
            if ckpt:
                ck.wait()                    # fence before the optimizer
            optimizer()
            if ckpt:
                ck.begin(ov_ents, path_of(f"ov{i % 2}"))   # after the optimizer
            torch.cuda.synchronize(dev)
            dt = allreduce_max(time.perf_counter() - t0, dev)
            if i >= warm:
                its.append(dt)
        if ckpt:
            ck.wait()
        return its

    # FLOP-derived T_FB: 6 * P * tokens per iteration over the DP group at 40%
    # of nominal dense bf16, GBS 512 x seq 2048
    P = 1315819520
    t_flop = 6 * P * GBS_1P3B * SEQ / (world * 0.4 * 2.25e15)
    if a.t_fb > 0:
        t_flop = a.t_fb
    sweep = [float(x) for x in a.t_fb_sweep.split(",") if x.strip()] if world == 1 else []
    pts = sorted(set(sweep + [round(t_flop, 3)]))
    # Eq. 1 crossover: the checkpoint hides behind fwd/bwd once T_FB >= S_C / B
    # (S_C = this leg's image, B = the persist rate measured above)
    crossover = ov_bytes * world / 1e9 / persist_gbs if persist_gbs else None
    out = []
    for t_fb in pts:
        n_gemm = max(1, int(round(t_fb / t_gemm)))
        base = loop(False, n_gemm, 1, a.overhead_base_iters)
        with_ck = loop(True, n_gemm, a.overhead_warmup, a.overhead_iters)  # iteration 0 has no
        mb, mc = statistics.median(base), statistics.median(with_ck)    # pending ckpt
        out.append({"t_fb_s": round(n_gemm * t_gemm, 3), "flop_derived": t_fb == round(t_flop, 3),
                    "iter_s_no_ckpt": round(mb, 4), "iter_s_ckpt": round(mc, 4),
                    "overhead_pct": round(100 * (mc / mb - 1), 2),
                    "eq1_hidden": crossover is not None and n_gemm * t_gemm >= crossover,
                    # Eq. 1: the optimizer of iteration i+1 waits
                    # max(0, S_C/B - (T_F + T_B)) for checkpoint i
                    "eq1_predicted_pct": None if crossover is None else
                    round(100 * max(0.0, crossover - n_gemm * t_gemm) / mb, 2)})
    head = next(x for x in out if x["flop_derived"])
    return {"overhead_pct": head["overhead_pct"], "t_fb_s": head["t_fb_s"],
            "iter_s_no_ckpt": head["iter_s_no_ckpt"], "iter_s_ckpt": head["iter_s_ckpt"],
            "state": "adam14 (params, master, m, v; grads rewritten by each backward)",
            "ckpt_bytes": int(ov_bytes * world), "eq1_crossover_s": round(crossover, 3)
            if crossover else None,
            "max_overhead_pct_where_hidden": max([x["overhead_pct"] for x in out
                                                  if x["eq1_hidden"]], default=None),
            "iters": a.overhead_iters, "warmup": a.overhead_warmup,
            "base_iters": a.overhead_base_iters, "pack_ctas": a.overlap_ctas,
            "pack": a.overlap_pack, "io_engine": a.overlap_io_engine or a.io_engine,
            "sweep": out, "workload": CFG}


def our_arm(a):
    ws, rank, lr = env_dist()
    # measurement machinery: CUDA events around each pack launch time the
    # kernel, not the host's launch latency (library launch gate, opt-in)
    os.environ.setdefault("FP_LAUNCH_GATE", "1")
    if ws > 1 and not dist.is_initialized():
        if SHARE_GPU or HOST_HOOK:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", lr))
    world = ws
    if HOST_HOOK:
        dev = None
    else:
        dev = torch.device("cuda", 0 if SHARE_GPU else lr)
        torch.cuda.set_device(dev)

    import paper_2406_13768_b200 as fp
    from workloads import config_specs, make_state
    fp.lib()                                             # fails loudly if not built

    specs = config_specs(CFG, rank, world)
    state = make_state(specs, dev if dev is not None else "cpu")
    ents = [(s.name, t, s.section, s.owner) for s, t in state]
    state_bytes = sum(s.nbytes for s in specs)
    sync = (lambda: torch.cuda.synchronize(dev)) if dev is not None else (lambda: None)
    sync()

    # ---- per-rank shard roots (GPU-local NVMe when discoverable) -----------
    n_vis = torch.cuda.device_count() if dev is not None else 0
    bdfs = [gpu_bdf(0 if SHARE_GPU else r) if r < max(n_vis, 1) and dev is not None else None
            for r in range(world)]
    shard_dirs = pick_shard_dirs(world, bdfs)
    if shard_dirs:
        sub = "fp_bench"

        def path_of(name):                   # relative: the library joins dirs[r % n]
            return os.path.join(sub, name)
        roots = [os.path.join(shard_dirs[r % len(shard_dirs)], sub) for r in range(world)]
    else:
        roots = [os.path.join(out_root(), "ours")] * world

        def path_of(name):
            return os.path.join(roots[0], name)
    root = roots[rank]
    my_roots = [root] if roots.index(root) == rank else []   # lowest rank of a root owns it
    for d in my_roots:
        shutil.rmtree(d, ignore_errors=True)
    barrier()
    os.makedirs(root, exist_ok=True)
    barrier()
    storage = storage_record(shard_dirs or [os.path.dirname(root)], bdfs)

    cfg = dict(pack=a.pack, slot_bytes=a.slot_mib << 20, ring_slots=a.ring_slots,
               io_depth=a.qd, sqe_bytes=a.sqe_kib << 10, pack_bytes=a.pack_mib << 20,
               prio=a.prio, writer_stride=a.writer_stride, io_engine=a.io_engine,
               dirs=shard_dirs)
    peaks, peak_src = measured_peaks()

    # ---- rooflines measured in the same run --------------------------------
    with fp.Checkpointer(dev, **cfg) as ck0:
        ck0.begin(ents, path_of("plan"))
        ck0.wait()
        shard_bytes = ck0.plan_info()["extents"]
    shard_bytes = sum(e[2] for e in shard_bytes)
    barrier()
    for d in my_roots:
        shutil.rmtree(os.path.join(d, "plan"), ignore_errors=True)
    barrier()
    # every rank writes the same amount (a writer subset still has N ranks
    # on the box): the image's per-rank share, capped
    img_total = int(allreduce_sum(shard_bytes, dev))
    nv_bytes = min(-(-img_total // world), int(a.nvme_bytes))
    # the roofline file sits beside two checkpoint generations: keep it within
    # what the file system can hold (ranks sharing a file system share it)
    fs = os.statvfs(root)
    free_now = fs.f_bavail * fs.f_frsize
    dev_id = os.stat(root).st_dev
    sharing = sum(1 for d in roots if os.stat(os.path.dirname(d) if shard_dirs else d).st_dev
                  == dev_id)
    room = (free_now - 2.2 * img_total * sharing / world) / sharing
    nv_bytes = int(min(nv_bytes, max(2e8, room * 0.8))) // 4096 * 4096
    barrier()
    os.sync()                                 # settle writeback of earlier runs first

    def nvme_roofline():
        g = fp.io_bench(root, nv_bytes, tag=rank, io_depth=a.qd, sqe_bytes=a.sqe_kib << 10,
                        ring_slots=a.ring_slots, slot_bytes=a.slot_mib << 20)
        return allreduce_sum(g, dev)          # concurrent writers: aggregate
    nvme_before = nvme_roofline()
    d2h_gbs = allreduce_sum(d2h_roofline(dev), dev) if dev is not None else None

    # ---- the checkpoint steps ----------------------------------------------
    ck = fp.Checkpointer(dev, group=None, **cfg)
    image_bytes = None
    for i in range(a.warmup):
        s = ck.save(ents, path_of(f"gen{i % 2}"))
        image_bytes = s["image_bytes"]
    clocks = Clocks(gpu_smi_id(dev)).start() if dev is not None else None
    stream = torch.cuda.current_stream(dev) if dev is not None else None
    lat, stats = [], []
    barrier()
    sync()
    if dev is not None:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
    th0 = time.perf_counter()
    for i in range(a.steps):
        t0 = time.perf_counter()
        ck.begin(ents, path_of(f"gen{(a.warmup + i) % 2}"), stream=stream)
        stats.append(ck.wait())
        lat.append(time.perf_counter() - t0)
    if dev is not None:
        e1.record(stream)
    sync()
    barrier()
    ck_clock = clocks.stop() if clocks else {"sm_mhz": None, "sm_max_mhz": None,
                                              "reasons": ["host-state test hook"]}
    el = e0.elapsed_time(e1) / 1e3 if dev is not None else time.perf_counter() - th0
    elapsed = allreduce_max(el, dev)
    lat_max = [allreduce_max(x, dev) for x in lat]
    image_bytes = stats[-1]["image_bytes"]
    gbs = image_bytes * a.steps / elapsed / 1e9
    # the drive is shared and its rate drifts (virtio disk on the gpurun box):
    # measure the roofline again right after the timed region; the roofline
    # is the best the device did in this run
    try:
        nvme_after = nvme_roofline()
    except Exception as e:  # noqa: BLE001 - the re-measure must not lose the line
        print(f"bench: NVMe roofline after the steps failed: {e}", file=sys.stderr)
        nvme_after = 0.0
    nvme_gbs = max(nvme_before, nvme_after)

    # pack kernel roofline: algorithmic bytes = 1 B read + 1 B written per slab
    # byte; duration = CUDA events around each launch on the launching stream
    pk_bytes = sum(s["pack_bytes"] for s in stats)
    pk_ms = sum(s["pack_ms"] for s in stats)
    pk_launches = sum(s["pack_launches"] for s in stats)
    pack_gbs = 2 * pk_bytes / (pk_ms / 1e3) / 1e9 if pk_ms > 0 else None
    d2h_ms = sum(s["d2h_ms"] for s in stats)
    crc_ms = sum(s.get("crc_ms", 0.0) for s in stats)
    pack_gbs = pack_gbs or 0.0                       # this rank's own GPU (rank 0 reports)
    launches_all = allreduce_sum(sum(s["kernel_launches"] for s in stats), dev)

    # ---- restore: the paper's two-step parallel load of the last
    # committed generation, own shard -> all-gather -> unpack, into the same
    # tensors (identical bytes); vs the same-run O_DIRECT read roofline
    restore = None
    if not a.no_restore:
        try:
            last = path_of(f"gen{(a.warmup + a.steps - 1) % 2}")
            gr = fp.io_bench(root, nv_bytes, tag=rank, read=True, io_depth=a.qd,
                             sqe_bytes=a.sqe_kib << 10, ring_slots=a.ring_slots,
                             slot_bytes=a.slot_mib << 20)
            nvme_read = allreduce_sum(gr, dev)
            rl, rinfo = [], {}
            for _ in range(a.restore_steps):
                barrier()
                sync()
                t0 = time.perf_counter()
                rinfo = ck.load_parallel(ents, last, stream=stream) or {}   # checks the CRC
                sync()
                rl.append(allreduce_max(time.perf_counter() - t0, dev))
            rt = statistics.median(rl)
            restore = {"value": round(image_bytes / rt / 1e9, 4), "unit": "GB/s",
                       "latency_s": round(rt, 4), "steps": len(rl),
                       "nvme_read_gbs": round(nvme_read, 3),
                       "frac": round(image_bytes / rt / 1e9 / nvme_read, 4),
                       "call": "fp_ckpt_load_parallel (own shard O_DIRECT read-ahead over the "
                               "pinned ring -> H2D -> exchange of the partitions (peer memory, "
                               "or all-gather) -> unpack kernel, CRC-32 checked)",
                       "exchange": rinfo.get("exchange"),
                       # host time blocked on this rank's own-shard reads in the
                       # last call: ~t_total when the storage is the bound
                       "t_read_wait_s": round(rinfo.get("t_read_wait", 0.0), 4),
                       "t_total_s": round(rinfo.get("t_total", 0.0), 4),
                       # rank 0's wait for the other writers' chunks (N > 1),
                       # and its setup (buffers, IPC mapping) in the last call
                       "t_exchange_wait_s": round(rinfo.get("t_exchange_wait", 0.0), 4),
                       "t_setup_s": round(rinfo.get("t_setup", 0.0), 4),
                       "roofline_how": f"fp_io_bench_read: O_DIRECT io_uring seq read, {a.qd} x "
                                       f"{a.sqe_kib} KiB in flight, best of 2, {world} concurrent "
                                       f"readers x {nv_bytes} B, same dirs, same run"}
        except Exception as e:  # noqa: BLE001 - an optional measurement must not lose the line
            print(f"bench: restore failed: {type(e).__name__}: {e}", file=sys.stderr)
            restore = {"error": f"{type(e).__name__}: {e}"}

    # ---- e2e: public API with the state sourced from pinned HOST memory ------
    e2e = None
    if not a.no_e2e and dev is not None:
        try:
            # this rank sources its share of the state from pinned host memory:
            # tensors are dealt to ranks by the position of their middle byte in
            # the state (rank r takes [r/N, (r+1)/N)), so across ranks every state
            # byte crosses PCIe H2D exactly once per step and each rank pins ~1/N
            mine, cum = [], 0
            for _, t in state:
                nb = t.numel() * t.element_size()
                if int((cum + nb / 2) * world // state_bytes) == rank:
                    mine.append(t)
                cum += nb
            host = [torch.empty_like(t, device="cpu").pin_memory() for t in mine]
            for h, t in zip(host, mine):
                h.copy_(t)
            my_h2d = sum(t.numel() * t.element_size() for t in mine)
            sync()
            ke = max(1, min(a.steps, a.e2e_steps))
            barrier()
            sync()
            f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            f0.record(stream)
            for i in range(ke):
                for h, t in zip(host, mine):
                    t.copy_(h, non_blocking=True)          # H2D of this step's inputs
                ck.begin(ents, path_of(f"gen{i % 2}"), stream=stream)
                st = ck.wait()                             # result: durable status (host)
            f1.record(stream)
            sync()
            barrier()
            e_el = allreduce_max(f0.elapsed_time(f1) / 1e3, dev)
            e2e = {"value": round(st["image_bytes"] * ke / e_el / 1e9, 4), "unit": "GB/s",
                   "h2d_bytes_per_step": int(allreduce_sum(my_h2d, dev)),
                   "d2h_bytes_per_step": int(st["image_bytes"]), "steps": ke,
                   "note": "timed: H2D of the whole state from pinned host memory, then "
                           "begin/wait through the Python API (D2H of the image via the ring)"}
            del host
        except Exception as e:  # noqa: BLE001 - an optional measurement must not lose the line
            print(f"bench: e2e failed: {type(e).__name__}: {e}", file=sys.stderr)
            e2e = {"error": f"{type(e).__name__}: {e}"}

    overhead = None
    if not a.no_overhead and dev is not None:
        try:
            ovcfg = dict(cfg)
            ovcfg["pack_ctas"] = a.overlap_ctas
            ovcfg["pack"] = a.overlap_pack
            if a.overlap_io_engine:
                ovcfg["io_engine"] = a.overlap_io_engine
            with fp.Checkpointer(dev, **ovcfg) as cko:
                overhead = synthetic_overhead(a, cko, ents, state, dev, rank, world, path_of,
                                              image_bytes / 1e9, gbs)
        except Exception as e:  # noqa: BLE001 - an optional measurement must not lose the line
            print(f"bench: overhead failed: {type(e).__name__}: {e}", file=sys.stderr)
            overhead = {"error": f"{type(e).__name__}: {e}"}

    ck.close()
    barrier()
    for d in my_roots:
        shutil.rmtree(d, ignore_errors=True)

    # the oracle on rank 0's host cores, at every N (a bounded sample)
    cpu = None
    if rank == 0 and not a.no_cpu_baseline:
        try:
            sample, _ = oracle_sample_tensors(specs, int(a.oracle_bytes))
            croot = os.path.join(out_root(), "oracle")
            os.makedirs(croot, exist_ok=True)
            io_state = settle_io()
            cg, ct, cimg = run_oracle_steps(sample, 1, croot)
            # the paper's baseline: torch.save of the same tensors (host
            # state dict) + fsync, as context for "speedup vs torch.save"
            tsd = {s.name: t for s, t in sample}
            fpath = os.path.join(croot, "torch_save.pt")
            t0 = time.perf_counter()
            with open(fpath, "wb") as f:
                torch.save(tsd, f)
                f.flush()
                os.fsync(f.fileno())
            ts_dt = time.perf_counter() - t0
            ts_bytes = os.path.getsize(fpath)
            shutil.rmtree(croot, ignore_errors=True)
            cpu = {"value": round(cg, 4), "unit": "GB/s", "cores": 1, "kind": "oracle",
                   "sample": f"first {len(sample)} tensors of {CFG} ({cimg} image bytes), "
                             f"host-resident, buffered write()+fsync, 1 step, rank 0; {io_state}",
                   "host_cores_available": cpu_cores(),
                   "torch_save_gbs": round(ts_bytes / ts_dt / 1e9, 4),
                   "torch_save_note": "context only: torch.save(state dict of the same sample) "
                                      "+ fsync on the same file system (PAPER.md P:259 baseline)"}
        except Exception as e:  # noqa: BLE001 - an optional measurement must not lose the line
            print(f"bench: cpu_baseline failed: {type(e).__name__}: {e}", file=sys.stderr)
            cpu = {"error": f"{type(e).__name__}: {e}"}

    if rank == 0:
        hbm = float(peaks["hbm_gbs"])
        nocrc = bool(os.environ.get("FP_NO_CRC"))
        kname = {"v4": "fp_pack_v4",
                 "bulk": "fp_pack_bulk" if nocrc else "fp_pack_bulk_crc",
                 "lsu": "fp_pack_v4" if nocrc else "fp_pack_lsu_crc",
                 "host": "fp_pack_v4 (to mapped host)"}.get(a.pack)
        traffic = a.traffic
        try:   # ncu-measured DRAM bytes per launch of this launch shape (profiles/)
            with open(os.path.join(ROOT, "profiles", "pack_traffic.json")) as f:
                tr = json.load(f).get(kname or "", {})
            for e in (tr if isinstance(tr, list) else [tr]):   # one entry per launch shape
                if traffic is None and e.get("bytes_per_launch") == (a.pack_mib << 21):
                    traffic = e["dram_bytes"]
        except (OSError, ValueError):
            pass
        launch_avg_ms = pk_ms / max(1, pk_launches)
        line = {
            "metric": METRIC,
            "value": round(gbs, 4), "unit": "GB/s", "n_gpus": world, "steps": a.steps,
            "warmup": a.warmup, "ms_per_step": round(1e3 * elapsed / a.steps, 2),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "u8", "data": "synthetic",
            "config": {"workload": CFG, "dp": world, "image_bytes": image_bytes,
                       "shard_bytes_rank0": shard_bytes, "profile": "adam16",
                       "pack": a.pack, "ring": f"{a.ring_slots}x{a.slot_mib}MiB",
                       "pack_launch_mib": a.pack_mib, "pack_stream_prio": a.prio,
                       "writer_stride": a.writer_stride,
                       "sqe_kib": a.sqe_kib, "qd": a.qd, "engine": stats[-1]["engine"],
                       "io_fallback": stats[-1]["fallback"],
                       "l2": "inputs (21 GB of state) larger than L2; no flush needed",
                       "launch": "torchrun" if os.environ.get("FP_BENCH_SELF_LAUNCHED") != "1"
                       and world > 1 else ("self-launched torch.distributed.run"
                                           if world > 1 else "single process"),
                       "backend": dist.get_backend() if dist.is_initialized() else None,
                       "test_hook": "host-state" if HOST_HOOK else
                       ("shared-gpu" if SHARE_GPU else None)},
            "storage": storage,
            "latency_s": {"median": round(statistics.median(lat_max), 4),
                          "min": round(min(lat_max), 4), "max": round(max(lat_max), 4)},
            "roofline": {"bound": "hbm", "kernel": kname,
                         "achieved": round(pack_gbs, 1), "peak": hbm, "unit": "GB/s",
                         "frac": round(pack_gbs / hbm, 4), "traffic": traffic,
                         "peak_source": peak_src, "launch_avg_ms": round(launch_avg_ms, 5),
                         "bytes_per_launch": int(2 * pk_bytes / max(1, pk_launches))},
            # the second library kernel of a step: page CRCs over each packed
            # group (1 B read per slab byte; issue-bound on table lookups, see
            # DESIGN.md §6) — reported, not the roofline kernel
            "crc_kernels": None if crc_ms <= 0 else {
                "kernels": "fp_crc_pages_tma" if not os.environ.get("FP_NO_TMA")
                else "fp_crc_pages",
                "us_per_launch": round(1e3 * crc_ms / max(1, pk_launches), 2),
                "read_gbs": round(pk_bytes / (crc_ms / 1e3) / 1e9, 1),
                "frac_of_hbm": round(pk_bytes / (crc_ms / 1e3) / 1e9 / hbm, 4),
                "share_of_library_gpu_time": round(crc_ms / (crc_ms + pk_ms), 3)},
            "nvme": {"measured_gbs": round(nvme_gbs, 3), "frac": round(gbs / nvme_gbs, 4),
                     "before_gbs": round(nvme_before, 3), "after_gbs": round(nvme_after, 3),
                     "how": f"built-in fp_io_bench (fio absent): O_DIRECT io_uring seq "
                            f"overwrite, {a.qd} x {a.sqe_kib} KiB in flight, best of 2 timed passes, "
                            f"{world} concurrent writers x {nv_bytes} B, each in its rank's shard "
                            f"root, same run, measured before and after the timed steps (max taken)"},
            "pcie_d2h": None if d2h_gbs is None else {
                "measured_gbs": round(d2h_gbs, 2), "frac": round(gbs / d2h_gbs, 4),
                "ring_d2h_gbs": round(pk_bytes / (d2h_ms / 1e3) / 1e9, 2) if d2h_ms > 0 else None},
            "hbm": {"peak_gbs_all_gpus": hbm * world, "frac": round(gbs / (hbm * world), 6)},
            "phase_s_last": {k: round(stats[-1][k], 4) for k in
                             ("t_helper", "t_fsync", "t_barrier", "t_commit", "t_io_stall")},
            "gpu_launches": int(launches_all),
            "clocks": ck_clock,
            "e2e": e2e,
            "restore": restore,
            "overhead": overhead,
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    if dist.is_initialized():
        dist.destroy_process_group()
    return 0


def _free_port():
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def self_launch(a):
    """`--gpus N` without a torchrun environment: re-run this script as N
    ranks under torch.distributed.run (one node, 127.0.0.1), NCCL init logging
    on so the N ranks are visible in stderr; rank 0 prints the line."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={a.gpus}", "--master-addr", "127.0.0.1",
           f"--master-port={_free_port()}", os.path.abspath(__file__), *sys.argv[1:]]
    env = dict(os.environ, FP_BENCH_SELF_LAUNCHED="1")
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    print(f"bench.py: launching {a.gpus} ranks: {' '.join(cmd)}", file=sys.stderr, flush=True)
    return subprocess.call(cmd, env=env)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--pack", default="bulk", choices=["v4", "bulk", "lsu", "host", "ce"])
    ap.add_argument("--pack-mib", type=int, default=1024)
    ap.add_argument("--prio", default="high", choices=["high", "low"])
    ap.add_argument("--writer-stride", type=int, default=1,
                    help="writer subset (P:495-499): ranks r %% s == 0 write replicated bytes")
    ap.add_argument("--slot-mib", type=int, default=64)
    ap.add_argument("--io-engine", default="uring", choices=["uring", "pwrite", "gds"],
                    help="gds: GPUDirect Storage (SURVEY f2), device slab -> cuFileWrite")
    ap.add_argument("--ring-slots", type=int, default=4)
    ap.add_argument("--qd", type=int, default=64)
    ap.add_argument("--sqe-kib", type=int, default=1024)
    ap.add_argument("--nvme-bytes", type=float, default=24e9,
                    help="cap on the roofline file per rank (default covers a whole C2 shard)")
    ap.add_argument("--oracle-bytes", type=float, default=4e9,
                    help="oracle sample (a prefix of the workload's tensors), ~10-15 s of CPU")
    ap.add_argument("--ref-bytes", type=float, default=1.5e9,
                    help="--impl reference: oracle sample per step (K steps stay within minutes)")
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--overhead-iters", type=int, default=10)
    ap.add_argument("--overhead-warmup", type=int, default=2)
    ap.add_argument("--overhead-base-iters", type=int, default=3,
                    help="iterations without checkpointing per T_FB (deterministic GEMM loop)")
    ap.add_argument("--overlap-ctas", type=int, default=16)
    ap.add_argument("--overlap-pack", default="bulk", choices=["v4", "bulk", "lsu"])
    ap.add_argument("--overlap-io-engine", default=None, choices=["uring", "null"],
                    help="ablation: null = storage that completes at once (the GPU-side "
                         "interference floor of the overlapped checkpoint)")
    ap.add_argument("--t-fb", type=float, default=0.0,
                    help="headline synthetic fwd+bwd seconds (0: FLOP-derived)")
    ap.add_argument("--t-fb-sweep", default="0.5,1,2,4",
                    help="extra T_FB points (s) at N=1; the FLOP-derived point is always run")
    ap.add_argument("--traffic", type=float, default=None,
                    help="ncu dram bytes per pack launch (from profiles/), echoed into roofline")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-overhead", action="store_true")
    ap.add_argument("--no-restore", action="store_true")
    ap.add_argument("--restore-steps", type=int, default=2)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    a = ap.parse_args()
    if a.warmup < 3 and a.impl == "ours":
        print("bench.py: --warmup must be >= 3", file=sys.stderr)
    if a.impl == "reference":
        return reference_arm(a)
    if a.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return self_launch(a)
    return our_arm(a)


if __name__ == "__main__":
    sys.exit(main())
