#!/bin/bash
# pass 12: ILP CRC chains; tests, launch list, ncu of the CRC kernels, bench.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout -s KILL 150 python -X faulthandler -c "
import faulthandler; faulthandler.dump_traceback_later(120, exit=True)
import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke12.log 2>&1
rc=$?; echo "smoke exit $rc" >> gpurun_out/smoke12.log
if [ $rc -ne 0 ]; then cat gpurun_out/smoke12.log; exit 1; fi
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -rs -k "not gds" > gpurun_out/pytest_gpu12.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu12.log
FP_NO_GATE=1 timeout 500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_bench12.csv \
   python bench.py --steps 1 --warmup 3 --no-overhead --no-e2e --no-cpu-baseline --no-restore --nvme-bytes 2e9 > gpurun_out/ncu_bench12.log 2>&1
echo "ncu exit $?" >> gpurun_out/ncu_bench12.log
FP_NO_GATE=1 timeout 400 ncu --set full --clock-control none --import-source on -k regex:"fp_crc_pages_tma|fp_pack_v4" -s 6 -c 4 \
   -o gpurun_out/ct12 -f python tools/ncu_pack.py > gpurun_out/ncu_ct12.log 2>&1
FP_NO_GATE=1 FP_CRC_FUSED=1 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"fp_pack_crc|fp_crc_fold" -s 4 -c 8 --csv \
   python tools/ncu_pack.py > gpurun_out/ncu_fused12.csv 2>&1
FP_NO_GATE=1 FP_NO_TMA=1 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"fp_crc_pages" -s 4 -c 8 --csv \
   python tools/ncu_pack.py > gpurun_out/ncu_notma12.csv 2>&1
timeout 900 python bench.py > gpurun_out/bench12.json 2> gpurun_out/bench12.err
echo "bench exit $?" >> gpurun_out/bench12.err
tail -6 gpurun_out/pytest_gpu12.log; cat gpurun_out/smoke12.log
cat gpurun_out/bench12.json; tail -3 gpurun_out/bench12.err gpurun_out/ncu_bench12.log gpurun_out/ncu_ct12.log
grep -h "gpu__time_duration" gpurun_out/ncu_fused12.csv gpurun_out/ncu_notma12.csv | cut -c1-250 | tail -16
