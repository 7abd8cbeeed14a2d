"""The paper's single-GPU micro-benchmark (§6.2, Figure
"block_size"): write one GPU tensor of 16-512 MB to the SSD, IO buffer 2-128
MB, single vs double buffering, relative to torch.save. Here:

  torch_save : torch.save(t, path) + fsync (the paper's baseline)
  fp_save    : torch.save(t, StreamWriter(path)) — the paper's integration
               (P:532-533): same serializer, bytes through the IO buffer with
               O_DIRECT, the unaligned suffix buffered, fdatasync
  fp_raw     : StreamWriter.write_tensor(t) — the tensor's bytes D2H'd straight
               into the page-locked IO buffer, then O_DIRECT

Median of --reps timed runs per point (after one untimed warm-up), GB/s =
tensor bytes / seconds. One JSON line per point, then a summary line.

    python tools/stream_bench.py --dir bench_ckpt/stream > gpurun_out/stream.jsonl
"""
import argparse
import json
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2406_13768_b200 as fp  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--dir", default=os.path.join(os.path.dirname(os.path.dirname(
    os.path.abspath(__file__))), "bench_ckpt", "stream"))
ap.add_argument("--sizes-mb", default="16,64,256,512")
ap.add_argument("--buffers-mb", default="2,8,32,128")
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
os.makedirs(a.dir, exist_ok=True)
dev = torch.device("cuda", 0)
path = os.path.join(a.dir, "t.pt")


def timed(fn):
    fn()  # warm-up (allocates, first-touch)
    ts = []
    for _ in range(a.reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    return statistics.median(ts), min(ts), max(ts)


def torch_save(t):
    with open(path, "wb") as f:
        torch.save(t, f)
        f.flush()
        os.fsync(f.fileno())


roof = fp.io_bench(a.dir, 2 << 30, tag=7)  # same-run O_DIRECT write roofline (64 x 1 MiB)
print(json.dumps({"kind": "nvme_roofline", "gbs": round(roof, 3),
                  "how": "fp_io_bench: 2 GiB O_DIRECT io_uring seq overwrite, 64 x 1 MiB"}),
      flush=True)
class NullWriter:
    """torch.save's own floor: serialisation (.cpu() of the storage, pickling,
    the zip writer's per-record CRC-32) with the bytes dropped."""

    def write(self, b):
        return len(b)

    def flush(self):
        pass


rows = []
for mb in [int(x) for x in a.sizes_mb.split(",")]:
    n = mb << 20
    t = torch.randint(0, 256, (n,), dtype=torch.uint8, device=dev)
    base = timed(lambda: torch_save(t))
    rows.append({"kind": "torch_save", "tensor_mb": mb, "gbs": round(n / base[0] / 1e9, 3),
                 "s": [round(x, 4) for x in base]})
    print(json.dumps(rows[-1]), flush=True)
    floor = timed(lambda: torch.save(t, NullWriter()))
    rows.append({"kind": "torch_save_null_writer", "tensor_mb": mb,
                 "gbs": round(n / floor[0] / 1e9, 3), "s": [round(x, 4) for x in floor]})
    print(json.dumps(rows[-1]), flush=True)
    for bmb in [int(x) for x in a.buffers_mb.split(",")]:
        for slots in (1, 2):
            def fp_save():
                fp.save(t, path, io_buffer_bytes=bmb << 20, ring_slots=slots)

            def fp_save_fast():  # torch's own switches: no zip CRC-32, pinned D2H
                fp.save(t, path, io_buffer_bytes=bmb << 20, ring_slots=slots,
                        zip_crc32=False, pinned_d2h=True)

            last = {}

            def fp_raw():
                w = fp.StreamWriter(path, io_buffer_bytes=bmb << 20, ring_slots=slots, device=0)
                w.write_tensor(t)
                last.update(w.close())
            for kind, fn in (("fp_save", fp_save), ("fp_save_fast", fp_save_fast),
                             ("fp_raw", fp_raw)):
                r = timed(fn)
                rows.append({"kind": kind, "tensor_mb": mb, "buffer_mb": bmb,
                             "mode": "double" if slots == 2 else "single",
                             "gbs": round(n / r[0] / 1e9, 3), "s": [round(x, 4) for x in r],
                             "speedup_vs_torch_save": round(base[0] / r[0], 2)})
                if kind == "fp_raw":
                    rows[-1]["last_stats_s"] = {k: round(last[k], 4) for k in
                                                ("t_total", "t_fill", "t_io_wait", "t_fsync")}
                print(json.dumps(rows[-1]), flush=True)
    del t
    torch.cuda.empty_cache()
os.remove(path)
best = {}
for r in rows:
    if r["kind"] in ("fp_save", "fp_save_fast", "fp_raw"):
        k = (r["kind"], r["tensor_mb"], r["mode"])
        best[k] = max(best.get(k, 0), r["speedup_vs_torch_save"])
print(json.dumps({"summary": "best speedup over torch.save per (kind, tensor MB, mode)",
                  "best": {f"{k[0]}/{k[1]}MB/{k[2]}": v for k, v in sorted(best.items())},
                  "nvme_roofline_gbs": round(roof, 3),
                  "best_raw_frac_of_roofline": round(max(r["gbs"] for r in rows
                                                         if r["kind"] == "fp_raw") / roof, 3),
                  "paper_context": "1.8-3.6x single, 1.8-6.6x double buffer (V100, P:613)"}),
      flush=True)
