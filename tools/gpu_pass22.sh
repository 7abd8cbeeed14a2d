#!/bin/bash
# pass 22: fold kernel with 256 threads and a shuffle tree.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout -s KILL 150 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke22.log 2>&1
echo "smoke exit $?" >> gpurun_out/smoke22.log
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider -rs > gpurun_out/pytest_gpu22.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu22.log
FP_NO_GATE=1 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"fp_crc|fp_pack" -s 6 -c 9 --csv \
   python tools/ncu_pack.py > gpurun_out/ncu_k22.csv 2>&1
timeout 900 python bench.py --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench22.json 2> gpurun_out/bench22.err
cat gpurun_out/smoke22.log; tail -n 3 gpurun_out/pytest_gpu22.log
python3 - <<'PY'
import csv, collections
rows=[r for r in csv.reader(open('gpurun_out/ncu_k22.csv')) if len(r)>10]
for i,r in enumerate(rows):
    if 'Kernel Name' in r: h=r; data=rows[i+1:]; break
ki=h.index('Kernel Name'); vi=h.index('Metric Value')
a=collections.defaultdict(list)
for r in data: a[r[ki].split('(')[0].split('::')[-1]].append(float(r[vi].replace(',','')))
print({k: round(sum(v)/len(v)/1e3,1) for k,v in a.items()})
PY
python3 -c "import json; d=json.load(open('gpurun_out/bench22.json')); print(d['value'], d['roofline']['frac'], d['crc_kernels'], d['nvme']['frac'], d['restore']['frac'], d['overhead']['overhead_pct'])"
