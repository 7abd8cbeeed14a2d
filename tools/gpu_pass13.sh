#!/bin/bash
# pass 13: TMA CRC kernel v2 (PRMT lookups, 16 warps x 1 stage) vs LSU default.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout -s KILL 150 python -X faulthandler -c "
import faulthandler; faulthandler.dump_traceback_later(120, exit=True)
import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke13.log 2>&1
rc=$?; echo "smoke exit $rc" >> gpurun_out/smoke13.log
if [ $rc -ne 0 ]; then cat gpurun_out/smoke13.log; exit 1; fi
FP_CRC_TMA=1 FP_NO_GATE=1 timeout 300 compute-sanitizer --tool memcheck --print-limit 10 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/memcheck13.log 2>&1
FP_CRC_TMA=1 FP_NO_GATE=1 timeout 300 compute-sanitizer --tool racecheck --print-limit 10 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/racecheck13.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -rs -k "not gds" > gpurun_out/pytest_gpu13.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu13.log
FP_CRC_TMA=1 FP_NO_GATE=1 timeout 400 ncu --set full --clock-control none --import-source on -k regex:"fp_crc_pages_tma" -s 6 -c 2 \
   -o gpurun_out/ct13 -f python tools/ncu_pack.py > gpurun_out/ncu_ct13.log 2>&1
FP_NO_GATE=1 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"fp_crc|fp_pack" -s 6 -c 9 --csv \
   python tools/ncu_pack.py > gpurun_out/ncu_lsu13.csv 2>&1
FP_CRC_TMA=1 FP_NO_GATE=1 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"fp_crc|fp_pack" -s 6 -c 9 --csv \
   python tools/ncu_pack.py > gpurun_out/ncu_tma13.csv 2>&1
FP_CRC_TMA=1 timeout 600 python bench.py --no-cpu-baseline --e2e-steps 1 --no-restore > gpurun_out/bench13_tma.json 2> gpurun_out/bench13_tma.err
tail -3 gpurun_out/memcheck13.log gpurun_out/racecheck13.log; tail -5 gpurun_out/pytest_gpu13.log; cat gpurun_out/smoke13.log
grep -h "gpu__time_duration" gpurun_out/ncu_lsu13.csv gpurun_out/ncu_tma13.csv | awk -F'","' '{print $5, $NF}' | cut -c1-40,200-260
cat gpurun_out/bench13_tma.json; tail -3 gpurun_out/bench13_tma.err
