"""Crash consistency (§3.2: checkpoints go directly to
persistent storage, so a checkpoint is either committed or absent).

A child process commits generation A, then is SIGKILLed by the library's
FP_FAULT_KILL_AT hook in the middle of writing the next generation. Then:
  - rotation (the bench's gen0/gen1): the torn directory has no manifest and
    generation A still loads bit-exact;
  - in-place rewrite of A: A's manifest was unlinked (and the unlink made
    durable) before the first shard byte was rewritten, so loading A fails
    with ENOENT instead of restoring torn shards.
"""
import os
import signal
import subprocess
import sys

import pytest
import torch

import paper_2406_13768_b200 as fp
from paper_2406_13768_b200.fastpersist import FastPersistError
from tests._util import entries
from workloads import config_specs, make_state

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r"""
import os, sys, torch
sys.path.insert(0, os.environ["FP_ROOT"])
import paper_2406_13768_b200 as fp
from tests._util import entries
from workloads import config_specs, make_state
d, second, device = sys.argv[1], sys.argv[2], sys.argv[3]
dev = None if device == "cpu" else torch.device("cuda", 0)
st = make_state(config_specs("gpt3_odd"), dev if dev is not None else "cpu")
with fp.Checkpointer(dev, slot_bytes=1 << 20, ring_slots=2, sqe_bytes=256 << 10) as ck:
    ck.save(entries(st), os.path.join(d, "A"))
print("A committed", flush=True)
os.environ["FP_FAULT_KILL_AT"] = "3"          # the third write completion
for _, t in st:                               # the next step's state differs
    t.add_(1) if t.is_floating_point() else None
with fp.Checkpointer(dev, slot_bytes=1 << 20, ring_slots=2, sqe_bytes=256 << 10) as ck:
    ck.save(entries(st), os.path.join(d, second))
print("NOT KILLED", flush=True)
"""


def run_crash(tmp_path, second, device):
    env = dict(os.environ, FP_ROOT=ROOT, PYTHONPATH=ROOT)
    r = subprocess.run([sys.executable, "-c", CHILD, str(tmp_path), second, device],
                       capture_output=True, text=True, env=env, timeout=600)
    assert "A committed" in r.stdout, r.stderr[-3000:]
    assert r.returncode == -signal.SIGKILL, (r.returncode, r.stdout, r.stderr[-2000:])
    assert "NOT KILLED" not in r.stdout


def _check(tmp_path, device):
    dev = None if device == "cpu" else torch.device("cuda", 0)
    st = make_state(config_specs("gpt3_odd"), dev if dev is not None else "cpu")
    return dev, st


@pytest.mark.parametrize("device", ["cpu", pytest.param("cuda", marks=pytest.mark.gpu)])
def test_kill_mid_write_keeps_previous_generation(tmp_path, device):
    run_crash(tmp_path, "B", device)
    assert os.path.exists(tmp_path / "B" / "shard-0-of-1.fpck")       # B was being written
    assert not os.path.exists(tmp_path / "B" / "manifest.json")       # ... never committed
    dev, st = _check(tmp_path, device)
    dst = [(s, torch.full_like(t, 3) if t.is_floating_point() else torch.zeros_like(t))
           for s, t in st]
    with fp.Checkpointer(dev, slot_bytes=1 << 20) as ck:
        ck.load(entries(dst), str(tmp_path / "A"))
        with pytest.raises(FastPersistError) as ei:
            ck.load(entries(dst), str(tmp_path / "B"))
        assert ei.value.code == -2                                   # ENOENT: no manifest
    if dev is not None:
        torch.cuda.synchronize()
    for (_, a), (_, b) in zip(st, dst):                              # A == the state before
        assert torch.equal(a.reshape(-1).view(torch.uint8), b.reshape(-1).view(torch.uint8))


@pytest.mark.parametrize("device", ["cpu", pytest.param("cuda", marks=pytest.mark.gpu)])
def test_kill_mid_in_place_rewrite_never_loads_torn_shards(tmp_path, device):
    run_crash(tmp_path, "A", device)
    assert not os.path.exists(tmp_path / "A" / "manifest.json")
    dev, st = _check(tmp_path, device)
    dst = [(s, torch.zeros_like(t)) for s, t in st]
    with fp.Checkpointer(dev, slot_bytes=1 << 20) as ck:
        with pytest.raises(FastPersistError) as ei:
            ck.load(entries(dst), str(tmp_path / "A"))
        assert ei.value.code == -2
