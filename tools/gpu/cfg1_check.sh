timeout 900 python -m pytest tests/test_gpu_ring.py tests/test_gpu_parity.py -x -q 2>&1 | tail -1
bash tools/gpu/cfg1.sh
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_cfg1_launches.csv python bench.py --config cfg1 --serial --steps 3 --warmup 3 --no-cpu-baseline --no-exact --no-e2e --no-spot-check > /dev/null 2>&1
python - <<'PY'
import csv
from collections import defaultdict
rows=[r for r in csv.reader(open('gpurun_out/r02_cfg1_launches.csv')) if len(r)>14 and r[0].isdigit()]
d=defaultdict(list)
for r in rows: d[r[4].split('(')[0][:60]].append(float(r[14])/1000)
for k,v in d.items(): print(f"{k:62s} n={len(v):3d} mean={sum(v)/len(v):7.2f} us  min={min(v):6.2f}")
PY
