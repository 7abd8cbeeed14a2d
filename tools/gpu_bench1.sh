#!/bin/bash
# bench line + ncu launch list + ncu full capture of the pack kernel.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
echo "bench exit $?" >> gpurun_out/bench.err
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
   python bench.py --steps 2 --warmup 3 --no-overhead --no-e2e --no-cpu-baseline > gpurun_out/bench_ncu.log 2>&1
echo "ncu list exit $?" >> gpurun_out/bench_ncu.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fp_pack -s 20 -c 3 \
   -o gpurun_out/pack_v4 -f python tools/ncu_pack.py > gpurun_out/ncu_full.log 2>&1
echo "ncu full exit $?" >> gpurun_out/ncu_full.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fp_pack -s 20 -c 3 \
   -o gpurun_out/pack_bulk -f python tools/ncu_pack.py --pack bulk > gpurun_out/ncu_full_bulk.log 2>&1
cat gpurun_out/bench.json gpurun_out/bench_ref.json; tail -3 gpurun_out/bench.err gpurun_out/ncu_full.log
