#!/bin/bash
# pass 18: fold kernel with batched loads; final verification + bench.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout -s KILL 150 python -X faulthandler -c "
import faulthandler; faulthandler.dump_traceback_later(120, exit=True)
import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke18.log 2>&1
rc=$?; echo "smoke exit $rc" >> gpurun_out/smoke18.log
if [ $rc -ne 0 ]; then cat gpurun_out/smoke18.log; exit 1; fi
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider -rs > gpurun_out/pytest_gpu18.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu18.log
FP_NO_GATE=1 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"fp_crc|fp_pack" -s 6 -c 9 --csv \
   python tools/ncu_pack.py > gpurun_out/ncu_k18.csv 2>&1
timeout 1200 python bench.py > gpurun_out/bench18.json 2> gpurun_out/bench18.err
echo "bench exit $?" >> gpurun_out/bench18.err
tail -n 4 gpurun_out/pytest_gpu18.log; cat gpurun_out/smoke18.log
grep -h "gpu__time_duration" gpurun_out/ncu_k18.csv | awk -F'","' '{print $5, $NF}' | cut -c1-30,190-240
cat gpurun_out/bench18.json; tail -n 2 gpurun_out/bench18.err
