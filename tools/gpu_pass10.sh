#!/bin/bash
# pass 10: fused pack+CRC kernel; GDS diagnosis (bounded).
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout -s KILL 150 python -X faulthandler -c "
import faulthandler; faulthandler.dump_traceback_later(120, exit=True)
import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke10.log 2>&1
rc=$?; echo "smoke exit $rc" >> gpurun_out/smoke10.log
if [ $rc -ne 0 ]; then cat gpurun_out/smoke10.log; exit 1; fi
FP_NO_GATE=1 timeout 600 compute-sanitizer --tool racecheck --print-limit 10 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/racecheck10.log 2>&1
echo "racecheck exit $?" >> gpurun_out/racecheck10.log
FP_NO_GATE=1 timeout 600 compute-sanitizer --tool synccheck --print-limit 10 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/synccheck10.log 2>&1
echo "synccheck exit $?" >> gpurun_out/synccheck10.log
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "not gds" > gpurun_out/pytest_gpu10.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu10.log
FP_DEBUG_GDS=1 CUFILE_ENV_PATH_JSON=$PWD/tools/diag/cufile_trace.json timeout -s KILL 120 python tools/diag/gds_diag.py > gpurun_out/gds_diag10.log 2>&1
echo "gds diag exit $?" >> gpurun_out/gds_diag10.log
FP_DEBUG_GDS=1 CUFILE_FORCE_COMPAT_MODE=true timeout -s KILL 120 python tools/diag/gds_diag.py > gpurun_out/gds_diag10_compat.log 2>&1
echo "gds diag (force compat) exit $?" >> gpurun_out/gds_diag10_compat.log
ls /dev/nvidia-fs* /proc/driver/nvidia-fs 2>&1 | head -3 >> gpurun_out/gds_diag10.log
lsmod 2>/dev/null | grep -i nvidia >> gpurun_out/gds_diag10.log
FP_NO_GATE=1 timeout 500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_bench10.csv \
   python bench.py --steps 1 --warmup 3 --no-overhead --no-e2e --no-cpu-baseline --no-restore --nvme-bytes 2e9 > gpurun_out/ncu_bench10.log 2>&1
echo "ncu exit $?" >> gpurun_out/ncu_bench10.log
FP_NO_GATE=1 timeout 400 ncu --set full --clock-control none --import-source on -k regex:"fp_pack_crc|fp_crc_fold" -s 8 -c 4 \
   -o gpurun_out/pc10 -f python tools/ncu_pack.py > gpurun_out/ncu_pc10.log 2>&1
timeout 900 python bench.py --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench10.json 2> gpurun_out/bench10.err
echo "bench exit $?" >> gpurun_out/bench10.err
tail -4 gpurun_out/racecheck10.log gpurun_out/synccheck10.log; tail -5 gpurun_out/pytest_gpu10.log; cat gpurun_out/smoke10.log; tail -25 gpurun_out/gds_diag10.log; tail -12 gpurun_out/gds_diag10_compat.log
cat gpurun_out/bench10.json; tail -3 gpurun_out/bench10.err gpurun_out/ncu_bench10.log gpurun_out/ncu_pc10.log
