#!/bin/bash
# pass 21: load-path kernels under ncu; a 10-step bench (variance of the disk).
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
FP_NO_GATE=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:"fp_unpack|fp_crc" -s 320 -c 4 \
   -o gpurun_out/load21 -f python tools/ncu_load.py > gpurun_out/ncu_load21.log 2>&1
timeout 1500 python bench.py --steps 10 --warmup 3 --no-overhead --no-cpu-baseline > gpurun_out/bench21_10.json 2> gpurun_out/bench21_10.err
tail -n 3 gpurun_out/ncu_load21.log; cat gpurun_out/bench21_10.json
