#!/bin/bash
# pass 8: read-ahead loads, commit barrier, CE runs per piece, restore bench,
# ncu launch list of the bench command (gate off under the profiler).
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout -s KILL 150 python -X faulthandler -c "
import faulthandler; faulthandler.dump_traceback_later(120, exit=True)
import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke8.log 2>&1
rc=$?; echo "smoke exit $rc" >> gpurun_out/smoke8.log
if [ $rc -ne 0 ]; then cat gpurun_out/smoke8.log; exit 1; fi
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider --timeout 300 > gpurun_out/pytest_gpu8.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu8.log
df -h / > gpurun_out/df8.log
timeout 1200 python bench.py > gpurun_out/bench8.json 2> gpurun_out/bench8.err
echo "bench exit $?" >> gpurun_out/bench8.err
FP_NO_GATE=1 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench8.csv \
   python bench.py --steps 1 --warmup 3 --no-overhead --no-e2e --no-cpu-baseline --no-restore --nvme-bytes 2e9 > gpurun_out/ncu_bench8.log 2>&1
echo "ncu exit $?" >> gpurun_out/ncu_bench8.log
timeout 500 python tools/ablate.py --what pack > gpurun_out/ablate_pack8.log 2>&1
tail -3 gpurun_out/pytest_gpu8.log; cat gpurun_out/smoke8.log gpurun_out/df8.log; cat gpurun_out/bench8.json; tail -3 gpurun_out/bench8.err gpurun_out/ncu_bench8.log
tail -12 gpurun_out/ablate_pack8.log
