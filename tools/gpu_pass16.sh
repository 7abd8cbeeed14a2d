#!/bin/bash
# pass 16: re-verify after the launch-helper changes; the paper's micro-benchmarks
# (IO-buffer sweep, writer-count sweep) and the stream-priority ablation.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout -s KILL 150 python -X faulthandler -c "
import faulthandler; faulthandler.dump_traceback_later(120, exit=True)
import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke16.log 2>&1
rc=$?; echo "smoke exit $rc" >> gpurun_out/smoke16.log
if [ $rc -ne 0 ]; then cat gpurun_out/smoke16.log; exit 1; fi
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider -rs > gpurun_out/pytest_gpu16.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu16.log
timeout 600 python tools/ablate.py --what buffer > gpurun_out/ablate_buffer16.log 2>&1
timeout 1200 python tools/writers_sweep.py --ks 1,2,4,8 --strides 1,2,4 --reps 2 > gpurun_out/writers16.log 2>&1
timeout 900 python tools/ablate.py --what prio --t-fb 4 --iters 3 > gpurun_out/ablate_prio16.log 2>&1
tail -n 6 gpurun_out/pytest_gpu16.log; cat gpurun_out/smoke16.log
echo "== buffer"; grep '^{' gpurun_out/ablate_buffer16.log | tail -n 30
echo "== writers"; grep '^{' gpurun_out/writers16.log | tail -n 20
echo "== prio"; grep '^{' gpurun_out/ablate_prio16.log | tail -n 8
