"""bench.py's contract pieces that run without a GPU: the reference arm (the
oracle timed on host cores) prints one JSON line with the required keys."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line(tmp_path):
    env = dict(os.environ, FP_BENCH_DIR=str(tmp_path))
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                          "--steps", "1", "--warmup", "1", "--ref-bytes", "2e7"],
                         capture_output=True, text=True, env=env, timeout=600)
    assert out.returncode == 0, out.stderr
    lines = [ln for ln in out.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0 and d["unit"] == "GB/s"
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] == 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0
    assert not os.listdir(tmp_path) or os.listdir(tmp_path) == []


def test_gpus_2_self_launches_two_ranks(tmp_path):
    """`bench.py --gpus 2` without torchrun re-launches itself as 2 ranks
    (torch.distributed.run); rank 0 prints ONE line with n_gpus 2. Host-state
    test hook (FP_BENCH_HOST=1: gloo, host tensors, no CUDA) on the CPU box."""
    env = dict(os.environ, FP_BENCH_DIR=str(tmp_path), FP_BENCH_HOST="1", FP_BENCH_CFG="c1_tiny")
    env.pop("WORLD_SIZE", None)
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2",
                          "--steps", "2", "--warmup", "3", "--nvme-bytes", "1e8",
                          "--oracle-bytes", "2e7"],
                         capture_output=True, text=True, env=env, timeout=600)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["config"]["dp"] == 2
    assert d["config"]["launch"] == "self-launched torch.distributed.run"
    assert d["cpu_baseline"]["kind"] == "oracle"          # cpu_baseline at every N
    assert d["storage"]["mounts"] and "lsblk" in d["storage"]
    assert d["restore"]["value"] > 0
    assert "launching 2 ranks" in out.stderr


def test_shard_dirs_follow_pcie_affinity(monkeypatch):
    """Each rank takes the NVMe mount sharing the longest PCIe path with its
    GPU (same switch), ties to the least-used one; FP_CKPT_DIRS overrides."""
    sys.path.insert(0, ROOT)
    import bench
    monkeypatch.delenv("FP_CKPT_DIRS", raising=False)
    mounts = [("/mnt/a", "/dev/nvme0n1", "/sys/devices/pci0000:00/0000:00:01.0/0000:01:00.0"),
              ("/mnt/b", "/dev/nvme1n1", "/sys/devices/pci0000:80/0000:80:01.0/0000:81:00.0")]
    monkeypatch.setattr(bench.os.path, "realpath",
                        lambda p: {"/sys/bus/pci/devices/0000:02:00.0":
                                   "/sys/devices/pci0000:00/0000:00:01.0/0000:02:00.0",
                                   "/sys/bus/pci/devices/0000:82:00.0":
                                   "/sys/devices/pci0000:80/0000:80:01.0/0000:82:00.0"}.get(p, p))
    got = bench.pick_shard_dirs(4, ["0000:02:00.0", "0000:82:00.0", "0000:02:00.0",
                                    "0000:82:00.0"], mounts)
    assert got == ["/mnt/a", "/mnt/b", "/mnt/a", "/mnt/b"]
    assert bench.pick_shard_dirs(2, [None, None], []) is None
    monkeypatch.setenv("FP_CKPT_DIRS", "/x,/y")
    assert bench.pick_shard_dirs(2, [None, None]) == ["/x", "/y"]


def test_pack_traffic_covers_the_default_launch_shape():
    """roofline.traffic comes from profiles/pack_traffic.json for the launch
    shape bench.py runs by default (--pack bulk --pack-mib 1024): there must be
    an ncu-measured entry for it, and it must be within [0.9, 1.1] of the
    algorithmic bytes (2 B per slab byte; far above = wasted re-reads)."""
    import json
    import re
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    src = open(os.path.join(root, "bench.py")).read()
    mib = int(re.search(r'"--pack-mib", type=int, default=(\d+)', src).group(1))
    tr = json.load(open(os.path.join(root, "profiles", "pack_traffic.json")))["fp_pack_bulk_crc"]
    ents = tr if isinstance(tr, list) else [tr]
    hit = [e for e in ents if e["bytes_per_launch"] == mib << 21]
    assert hit, f"no ncu traffic entry for {mib} MiB launches"
    assert 0.9 <= hit[0]["dram_bytes"] / hit[0]["bytes_per_launch"] <= 1.1
