#!/bin/bash
# pass 15: full-size configs with the final kernels (one rank of DP=8 each).
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python tools/bench_configs.py --cfg c3_gpt3_6.7b --k 8 --rank 3 --full-crc --overhead > gpurun_out/cfg15_c3.log 2>&1
timeout 900 python tools/bench_configs.py --cfg c4_gpt3_13b_zero --k 8 --rank 0 --overhead > gpurun_out/cfg15_c4.log 2>&1
timeout 1500 python tools/bench_configs.py --cfg c5_moe_64e --k 8 --rank 0 --dir /dev/shm/fp_c5 --no-fsync --steps 1 --full-crc > gpurun_out/cfg15_c5.log 2>&1
rm -rf /dev/shm/fp_c5
for f in c3 c4 c5; do echo "== $f"; tail -c 1500 gpurun_out/cfg15_$f.log; echo; done
