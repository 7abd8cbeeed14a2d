#!/bin/bash
# pass 9: table-driven CRC kernels, GDS engine tests + bench, launch list.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout -s KILL 150 python -X faulthandler -c "
import faulthandler; faulthandler.dump_traceback_later(120, exit=True)
import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke9.log 2>&1
rc=$?; echo "smoke exit $rc" >> gpurun_out/smoke9.log
if [ $rc -ne 0 ]; then cat gpurun_out/smoke9.log; exit 1; fi
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 300 > gpurun_out/pytest_gpu9.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu9.log
FP_NO_GATE=1 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_bench9.csv \
   python bench.py --steps 1 --warmup 3 --no-overhead --no-e2e --no-cpu-baseline --no-restore --nvme-bytes 2e9 > gpurun_out/ncu_bench9.log 2>&1
echo "ncu exit $?" >> gpurun_out/ncu_bench9.log
FP_NO_GATE=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:"fp_crc|fp_pack_v4" -s 12 -c 6 \
   -o gpurun_out/crc9 -f python tools/ncu_pack.py > gpurun_out/ncu_crc9.log 2>&1
timeout 1200 python bench.py > gpurun_out/bench9.json 2> gpurun_out/bench9.err
echo "bench exit $?" >> gpurun_out/bench9.err
timeout 600 python bench.py --io-engine gds --steps 3 --warmup 3 --no-overhead --no-e2e --no-cpu-baseline > gpurun_out/bench9_gds.json 2> gpurun_out/bench9_gds.err
echo "gds bench exit $?" >> gpurun_out/bench9_gds.err
tail -15 gpurun_out/pytest_gpu9.log; cat gpurun_out/smoke9.log; cat gpurun_out/bench9.json; tail -3 gpurun_out/bench9.err gpurun_out/ncu_bench9.log gpurun_out/ncu_crc9.log
cat gpurun_out/bench9_gds.json; tail -5 gpurun_out/bench9_gds.err
