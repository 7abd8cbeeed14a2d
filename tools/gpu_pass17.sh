#!/bin/bash
# pass 17: writer-count sweep (fixed: one config's generations on disk at a time)
# and the stream-priority ablation.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
df -h / > gpurun_out/df17.log
timeout 1200 python tools/writers_sweep.py --ks 1,2,4,8 --strides 1,2,4 --reps 2 > gpurun_out/writers17.log 2>&1
timeout 900 python tools/ablate.py --what prio --t-fb 4 --iters 3 > gpurun_out/ablate_prio17.log 2>&1
cat gpurun_out/df17.log
echo "== writers"; grep '^{' gpurun_out/writers17.log; tail -n 3 gpurun_out/writers17.log
echo "== prio"; grep '^{' gpurun_out/ablate_prio17.log; tail -n 3 gpurun_out/ablate_prio17.log
