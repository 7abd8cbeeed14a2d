#!/bin/bash
# pass 2: parity (incl. full-size C2), bench with pack groups, ncu of the new
# launch shape, C3/C4 single-rank-of-8 runs with per-iteration overhead.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
echo "bench exit $?" >> gpurun_out/bench.err
for p in v4 bulk; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fp_pack -s 5 -c 3 \
   -o gpurun_out/pack_${p}_256 -f python tools/ncu_pack.py --pack $p > gpurun_out/ncu_full_$p.log 2>&1
done
timeout 900 python tools/bench_configs.py --cfg c3_gpt3_6.7b --k 8 --rank 0 --overhead --iters 2 > gpurun_out/cfg_c3.log 2>&1
timeout 1200 python tools/bench_configs.py --cfg c4_gpt3_13b_zero --k 8 --rank 0 --overhead --iters 2 > gpurun_out/cfg_c4.log 2>&1
tail -3 gpurun_out/pytest_gpu.log; cat gpurun_out/bench.json; tail -2 gpurun_out/cfg_c3.log gpurun_out/cfg_c4.log
