#!/bin/bash
# pass 23: bench.py after the optional-section guards (N=1 default, N=2 shared-GPU path).
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1200 python bench.py > gpurun_out/bench23.json 2> gpurun_out/bench23.err
echo "bench exit $?" >> gpurun_out/bench23.err
FP_BENCH_SHARE_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
   --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 3 --warmup 3 \
   --no-overhead --e2e-steps 1 --no-cpu-baseline --restore-steps 1 > gpurun_out/bench23_n2.json 2> gpurun_out/bench23_n2.err
echo "n2 exit $?" >> gpurun_out/bench23_n2.err
cat gpurun_out/bench23.json; tail -n 2 gpurun_out/bench23.err; cat gpurun_out/bench23_n2.json; tail -n 2 gpurun_out/bench23_n2.err
