#!/bin/bash
# One parametrised GPU pass (replaces the round-1 tools/gpu_pass*.sh):
#   tools/gpu_run.sh <tag> <step> [<step> ...]
# steps: build | tests[:<pytest -k expr>] | bench[:<extra args>] | bench2share |
#        ncu_launches | ncu_pack | cmd:<shell command>
# Outputs land in gpurun_out/<tag>_*.
set -u
tag=$1; shift
out=gpurun_out
mkdir -p $out
python -m paper_2406_13768_b200.build --force > $out/${tag}_build.log 2>&1 || { echo "build failed"; tail -20 $out/${tag}_build.log; exit 1; }
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $out/${tag}_smi.txt 2>&1
# a reused box keeps /tmp: drop earlier pytest temp dirs (full-size shards)
rm -rf /tmp/pytest-of-root /dev/shm/fp_* 2>/dev/null
df -h / /tmp /dev/shm >> $out/${tag}_smi.txt 2>&1
nb=0
for step in "$@"; do
  name=${step%%:*}; arg=${step#*:}; [ "$arg" = "$step" ] && arg=""
  echo "== $step" >&2
  case $name in
    tests)   timeout ${TESTS_TIMEOUT:-1200} python -m pytest tests -m gpu -x -q --timeout 300 ${arg:+-k "$arg"} > $out/${tag}_pytest.log 2>&1; echo "tests rc=$?"; tail -3 $out/${tag}_pytest.log; rm -rf /tmp/pytest-of-root ;;
    bench)   nb=$((nb+1)); df -h . >&2; timeout 2400 python bench.py $arg > $out/${tag}_bench${nb}.json 2> $out/${tag}_bench${nb}.err; echo "bench$nb rc=$?"; tail -c 600 $out/${tag}_bench${nb}.err; df -h . >&2 ;;
    bench2share) FP_BENCH_SHARE_GPU=1 FP_BENCH_CFG=c1_tiny timeout 900 python bench.py --gpus 2 --steps 2 --warmup 3 --no-overhead --nvme-bytes 2e8 --oracle-bytes 2e7 > $out/${tag}_bench2.json 2> $out/${tag}_bench2.err; echo "bench2 rc=$?" ;;
    ncu_launches) timeout 1800 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"fp_" -c 400 --csv --log-file $out/${tag}_launches.csv python bench.py --steps 2 --warmup 3 --no-overhead --no-e2e --no-cpu-baseline --restore-steps 1 $arg > $out/${tag}_ncu_bench.log 2>&1; echo "ncu launches rc=$?" ;;
    ncu_full) # arg: <pack>=<kernel regex>=<count>
              pk=${arg%%=*}; rest=${arg#*=}; rx=${rest%%=*}; cnt=${rest#*=}
              timeout 1800 ncu --set full --clock-control none --import-source on -k regex:"$rx" -s 4 -c $cnt -o $out/${tag}_ncu_${pk} -f python tools/ncu_pack.py --pack $pk > $out/${tag}_ncu_${pk}.log 2>&1; echo "ncu full $pk rc=$?"
              ncu -i $out/${tag}_ncu_${pk}.ncu-rep --page raw --csv > $out/${tag}_ncu_${pk}_raw.csv 2>/dev/null ;;
    cmd) bash -c "$arg"; echo "cmd rc=$?" ;;
  esac
done
