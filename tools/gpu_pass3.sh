#!/bin/bash
# pass 3: parity of variants + CRC + parallel load; bench; ncu launch list of a
# checkpoint (pack + crc kernels); ablations; N=2 bench code path (shared GPU).
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -m "gpu and not slow" -x -q > gpurun_out/pytest_gpu3.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu3.log
timeout 900 python bench.py > gpurun_out/bench3.json 2> gpurun_out/bench3.err
echo "bench exit $?" >> gpurun_out/bench3.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_ckpt.csv \
   python tools/ncu_pack.py > gpurun_out/ncu_list_ckpt.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fp_crc -s 4 -c 4 \
   -o gpurun_out/crc -f python tools/ncu_pack.py > gpurun_out/ncu_crc.log 2>&1
timeout 900 python tools/ablate.py --what pack > gpurun_out/ablate_pack.log 2>&1
timeout 600 python tools/ablate.py --what buffer > gpurun_out/ablate_buffer.log 2>&1
timeout 900 python tools/ablate.py --what prio --t-fb 4 --iters 3 > gpurun_out/ablate_prio.log 2>&1
FP_BENCH_SHARE_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
   --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 3 --warmup 3 \
   --no-overhead --e2e-steps 1 > gpurun_out/bench_share2.json 2> gpurun_out/bench_share2.err
echo "share2 exit $?" >> gpurun_out/bench_share2.err
tail -3 gpurun_out/pytest_gpu3.log; cat gpurun_out/bench3.json; tail -30 gpurun_out/ablate_pack.log; cat gpurun_out/bench_share2.json; tail -5 gpurun_out/bench_share2.err
