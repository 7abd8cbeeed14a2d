"""One small checkpoint per pack kernel for compute-sanitizer (memcheck /
racecheck / synccheck): a ragged GPT-style state (gpt3_odd), 1 MiB ring slots,
8 MiB pack groups (hundreds of 32 KiB tiles per launch), then the shard is
compared with the oracle's sha256 and CRC-32.

    compute-sanitizer --tool racecheck python tools/diag/sanitize_packs.py --pack bulk
"""
import argparse
import os
import sys
import tempfile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))

import torch  # noqa: E402

import paper_2406_13768_b200 as fp  # noqa: E402
from oracle import fpck  # noqa: E402
from tests._util import entries, file_sha, oracle_layout  # noqa: E402
from workloads import config_specs, make_state  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--pack", default="bulk")
ap.add_argument("--cfg", default="gpt3_odd")
a = ap.parse_args()
dev = torch.device("cuda", 0)
st = make_state(config_specs(a.cfg, 0, 1), dev)
lay = oracle_layout([st], 1)
with tempfile.TemporaryDirectory() as d:
    with fp.Checkpointer(dev, pack=a.pack, slot_bytes=1 << 20, pack_bytes=8 << 20) as ck:
        s = ck.save(entries(st), d)
    ok = file_sha(os.path.join(d, fpck.shard_name(0, 1))) == fpck.shard_sha256(lay, 0)
    print(f"pack={a.pack} launches={s['pack_launches']} sha_ok={ok} crc_valid={s['crc_valid']}")
    sys.exit(0 if ok else 1)
