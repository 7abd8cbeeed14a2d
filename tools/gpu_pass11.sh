#!/bin/bash
# pass 11: TMA page-CRC kernel (default), fused kernel as ablation, GDS open
# timeout + skip, launch list, ncu full of the CRC/pack kernels, bench, N=2.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout -s KILL 150 python -X faulthandler -c "
import faulthandler; faulthandler.dump_traceback_later(120, exit=True)
import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke11.log 2>&1
rc=$?; echo "smoke exit $rc" >> gpurun_out/smoke11.log
if [ $rc -ne 0 ]; then cat gpurun_out/smoke11.log; exit 1; fi
FP_NO_GATE=1 timeout 300 compute-sanitizer --tool memcheck --print-limit 10 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/memcheck11.log 2>&1
FP_NO_GATE=1 timeout 300 compute-sanitizer --tool racecheck --print-limit 10 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/racecheck11.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -rs > gpurun_out/pytest_gpu11.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu11.log
FP_NO_GATE=1 timeout 500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_bench11.csv \
   python bench.py --steps 1 --warmup 3 --no-overhead --no-e2e --no-cpu-baseline --no-restore --nvme-bytes 2e9 > gpurun_out/ncu_bench11.log 2>&1
echo "ncu exit $?" >> gpurun_out/ncu_bench11.log
FP_NO_GATE=1 timeout 400 ncu --set full --clock-control none --import-source on -k regex:"fp_crc_pages_tma|fp_pack_v4|fp_crc_fold" -s 9 -c 6 \
   -o gpurun_out/ct11 -f python tools/ncu_pack.py > gpurun_out/ncu_ct11.log 2>&1
timeout 900 python bench.py > gpurun_out/bench11.json 2> gpurun_out/bench11.err
echo "bench exit $?" >> gpurun_out/bench11.err
FP_BENCH_SHARE_GPU=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
   --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 3 --warmup 3 \
   --no-overhead --e2e-steps 1 --no-cpu-baseline > gpurun_out/bench11_share2.json 2> gpurun_out/bench11_share2.err
echo "share2 exit $?" >> gpurun_out/bench11_share2.err
tail -3 gpurun_out/memcheck11.log gpurun_out/racecheck11.log; tail -12 gpurun_out/pytest_gpu11.log; cat gpurun_out/smoke11.log
cat gpurun_out/bench11.json; tail -3 gpurun_out/bench11.err gpurun_out/ncu_bench11.log gpurun_out/ncu_ct11.log
cat gpurun_out/bench11_share2.json; tail -5 gpurun_out/bench11_share2.err
