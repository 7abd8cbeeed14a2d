#!/bin/bash
# pass 6: bench launch-shape / queue variants (short runs), writers sweep.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for v in "--pack-mib 512" "--qd 128" "--qd 128 --sqe-kib 2048" "--slot-mib 128 --ring-slots 4" "--pack bulk" "--ring-slots 2"; do
  echo "== $v" >> gpurun_out/bench_variants.log
  timeout 400 python bench.py --steps 3 --warmup 3 --no-overhead --no-e2e --no-cpu-baseline $v >> gpurun_out/bench_variants.log 2>&1
done
timeout 1200 python tools/writers_sweep.py --ks 1,2,4,8 --strides 1,2,4 > gpurun_out/writers_sweep.log 2>&1
cat gpurun_out/bench_variants.log | python3 -c "
import sys, json
v=None
for ln in sys.stdin:
    if ln.startswith('=='): v=ln.strip(); continue
    try: d=json.loads(ln)
    except Exception: continue
    print(v, d['value'], d['latency_s'], d['roofline']['frac'], d['nvme'])
"; cat gpurun_out/writers_sweep.log
