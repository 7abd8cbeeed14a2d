#!/bin/bash
# pass 19: max shared-memory carveout for every library kernel (no L1/smem
# reconfiguration between back-to-back pack / CRC / fold launches).
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout -s KILL 150 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke19.log 2>&1
echo "smoke exit $?" >> gpurun_out/smoke19.log
FP_NO_GATE=1 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"fp_crc|fp_pack" -s 6 -c 9 --csv \
   python tools/ncu_pack.py > gpurun_out/ncu_k19.csv 2>&1
timeout 600 python bench.py --steps 3 --warmup 3 --no-overhead --no-e2e --no-cpu-baseline --no-restore > gpurun_out/bench19.json 2> gpurun_out/bench19.err
cat gpurun_out/smoke19.log
python3 - <<'PY'
import csv, collections
rows=[r for r in csv.reader(open('gpurun_out/ncu_k19.csv')) if len(r)>10]
for i,r in enumerate(rows):
    if 'Kernel Name' in r: h=r; data=rows[i+1:]; break
ki=h.index('Kernel Name'); vi=h.index('Metric Value')
a=collections.defaultdict(list)
for r in data: a[r[ki].split('(')[0].split('::')[-1]].append(float(r[vi].replace(',','')))
print({k: round(sum(v)/len(v)/1e3,1) for k,v in a.items()})
PY
cat gpurun_out/bench19.json | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline'], d['crc_kernels'])"
