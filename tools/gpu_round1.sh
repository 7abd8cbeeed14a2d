#!/bin/bash
# First GPU pass: box probe, GPU parity tests, quick perf probe.
mkdir -p gpurun_out
bash tools/probe_box.sh > /dev/null 2>&1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -m "gpu and not slow" -x -q > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
echo "smoke exit $?" >> gpurun_out/smoke.log
timeout 900 python tools/quick_perf.py > gpurun_out/quick_perf.log 2>&1
echo "quick_perf exit $?" >> gpurun_out/quick_perf.log
tail -5 gpurun_out/pytest_gpu.log gpurun_out/smoke.log; tail -30 gpurun_out/quick_perf.log
