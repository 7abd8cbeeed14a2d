#!/bin/bash
# pass 20: final state of the round — smoke, full GPU suite, default bench.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout -s KILL 150 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke20.log 2>&1
echo "smoke exit $?" >> gpurun_out/smoke20.log
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider -rs > gpurun_out/pytest_gpu20.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu20.log
timeout 1200 python bench.py > gpurun_out/bench20.json 2> gpurun_out/bench20.err
echo "bench exit $?" >> gpurun_out/bench20.err
cat gpurun_out/smoke20.log; tail -n 4 gpurun_out/pytest_gpu20.log; cat gpurun_out/bench20.json; tail -n 2 gpurun_out/bench20.err
