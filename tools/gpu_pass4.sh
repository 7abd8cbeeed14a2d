#!/bin/bash
# pass 4: smoke first (fail fast), full GPU suite, bench, C3/C5 full-shard CRC parity.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout -s KILL 150 python -X faulthandler -c "
import faulthandler; faulthandler.dump_traceback_later(120, exit=True)
import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke4.log 2>&1
rc=$?; echo "smoke exit $rc" >> gpurun_out/smoke4.log
if [ $rc -ne 0 ]; then cat gpurun_out/smoke4.log; exit 1; fi
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider --timeout 300 > gpurun_out/pytest_gpu4.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu4.log
timeout 900 python bench.py > gpurun_out/bench4.json 2> gpurun_out/bench4.err
echo "bench exit $?" >> gpurun_out/bench4.err
timeout 900 python tools/bench_configs.py --cfg c3_gpt3_6.7b --k 8 --rank 3 --full-crc > gpurun_out/cfg4_c3.log 2>&1
timeout 1200 python tools/bench_configs.py --cfg c5_moe_64e --k 8 --rank 0 --dir /dev/shm/fp_c5 --no-fsync --steps 1 --full-crc > gpurun_out/cfg4_c5.log 2>&1
rm -rf /dev/shm/fp_c5
tail -3 gpurun_out/pytest_gpu4.log; cat gpurun_out/smoke4.log; cat gpurun_out/bench4.json; tail -1 gpurun_out/cfg4_c3.log gpurun_out/cfg4_c5.log
