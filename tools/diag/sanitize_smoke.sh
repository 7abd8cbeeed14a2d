#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
FP_NO_GATE=1 timeout 600 compute-sanitizer --tool memcheck --print-limit 20 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/sanitize.log 2>&1
echo "exit $?" >> gpurun_out/sanitize.log
head -80 gpurun_out/sanitize.log
