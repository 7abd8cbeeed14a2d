#!/bin/bash
# pass 14: full validation of the round's final state + the numbers to keep.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout -s KILL 150 python -X faulthandler -c "
import faulthandler; faulthandler.dump_traceback_later(120, exit=True)
import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke14.log 2>&1
rc=$?; echo "smoke exit $rc" >> gpurun_out/smoke14.log
if [ $rc -ne 0 ]; then cat gpurun_out/smoke14.log; exit 1; fi
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider -rs > gpurun_out/pytest_gpu14.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu14.log
df -h / > gpurun_out/df14.log
timeout 1200 python bench.py > gpurun_out/bench14.json 2> gpurun_out/bench14.err
echo "bench exit $?" >> gpurun_out/bench14.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench14_ref.json 2> gpurun_out/bench14_ref.err
FP_NO_GATE=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench14.csv \
   python bench.py --steps 1 --warmup 3 --no-overhead --no-e2e --no-cpu-baseline --no-restore --nvme-bytes 2e9 > gpurun_out/ncu_bench14.log 2>&1
echo "ncu exit $?" >> gpurun_out/ncu_bench14.log
FP_NO_GATE=1 timeout 400 ncu --set full --clock-control none --import-source on -k regex:"fp_pack_v4|fp_crc_pages_tma|fp_crc_fold" -s 9 -c 3 \
   -o gpurun_out/full14 -f python tools/ncu_pack.py > gpurun_out/ncu_full14.log 2>&1
tail -8 gpurun_out/pytest_gpu14.log; cat gpurun_out/smoke14.log gpurun_out/df14.log
cat gpurun_out/bench14.json; tail -3 gpurun_out/bench14.err; cat gpurun_out/bench14_ref.json; tail -2 gpurun_out/ncu_bench14.log gpurun_out/ncu_full14.log
