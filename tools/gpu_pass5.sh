#!/bin/bash
# pass 5: ablations, ncu launch list of one checkpoint + CRC kernel capture,
# N=2 bench code path on one GPU (gloo). Every step bounded.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_ckpt.csv \
   python tools/ncu_pack.py > gpurun_out/ncu_list_ckpt.log 2>&1
timeout 400 ncu --set full --clock-control none --import-source on -k regex:fp_crc -s 4 -c 4 \
   -o gpurun_out/crc -f python tools/ncu_pack.py > gpurun_out/ncu_crc.log 2>&1
timeout 700 python tools/ablate.py --what pack > gpurun_out/ablate_pack.log 2>&1
timeout 300 python tools/ablate.py --what buffer > gpurun_out/ablate_buffer.log 2>&1
timeout 600 python tools/ablate.py --what prio --t-fb 3 --iters 2 > gpurun_out/ablate_prio.log 2>&1
FP_BENCH_SHARE_GPU=1 timeout 700 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
   --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 3 --warmup 3 \
   --no-overhead --e2e-steps 1 --writer-stride 1 > gpurun_out/bench_share2.json 2> gpurun_out/bench_share2.err
echo "share2 exit $?" >> gpurun_out/bench_share2.err
tail -40 gpurun_out/ablate_pack.log gpurun_out/ablate_prio.log; cat gpurun_out/bench_share2.json; tail -5 gpurun_out/bench_share2.err
