#!/bin/bash
# pass 7 (round 1, session 3): re-verify after the begin() item-cache change,
# bench, ncu launch list of the bench command, ablations, launch-shape variants.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout -s KILL 150 python -X faulthandler -c "
import faulthandler; faulthandler.dump_traceback_later(120, exit=True)
import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke7.log 2>&1
rc=$?; echo "smoke exit $rc" >> gpurun_out/smoke7.log
if [ $rc -ne 0 ]; then cat gpurun_out/smoke7.log; exit 1; fi
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider --timeout 300 > gpurun_out/pytest_gpu7.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu7.log
timeout 900 python bench.py > gpurun_out/bench7.json 2> gpurun_out/bench7.err
echo "bench exit $?" >> gpurun_out/bench7.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench7.csv \
   python bench.py --steps 2 --warmup 1 --no-overhead --no-e2e --no-cpu-baseline --nvme-bytes 2e9 > gpurun_out/ncu_bench7.log 2>&1
echo "ncu exit $?" >> gpurun_out/ncu_bench7.log
for v in "--pack-mib 512" "--qd 128" "--qd 128 --sqe-kib 2048" "--slot-mib 128" "--ring-slots 8" "--pack bulk"; do
  echo "== $v" >> gpurun_out/bench_variants7.log
  timeout 300 python bench.py --steps 3 --warmup 3 --no-overhead --no-e2e --no-cpu-baseline $v >> gpurun_out/bench_variants7.log 2>&1
done
timeout 400 python tools/ablate.py --what pack > gpurun_out/ablate_pack7.log 2>&1
tail -3 gpurun_out/pytest_gpu7.log; cat gpurun_out/smoke7.log; cat gpurun_out/bench7.json; tail -3 gpurun_out/bench7.err gpurun_out/ncu_bench7.log
grep -v '^{' gpurun_out/bench_variants7.log | tail -3
python3 - <<'EOF'
import json
v = None
for ln in open("gpurun_out/bench_variants7.log"):
    if ln.startswith("=="): v = ln.strip(); continue
    try: d = json.loads(ln)
    except Exception: continue
    print(v, d["value"], d["latency_s"], d["roofline"]["frac"], d["nvme"]["measured_gbs"])
EOF
tail -30 gpurun_out/ablate_pack7.log
