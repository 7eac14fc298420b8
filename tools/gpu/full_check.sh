# the driver's round-end checks on one GPU: every GPU test, smoke(), the reference arm, then the default bench line
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2_pytest_full.log 2>&1
echo pytest=$?
tail -3 gpurun_out/r2_pytest_full.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_smoke.log 2>&1; echo smoke=$?; tail -1 gpurun_out/r2_smoke.log
python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r2_ref_full.json 2> gpurun_out/r2_ref_full.err; echo ref=$?
python bench.py --steps 20 --warmup 5 > gpurun_out/r2_bench_full.json 2> gpurun_out/r2_bench_full.err; echo bench=$?
python -c "
import json
b=json.load(open('gpurun_out/r2_bench_full.json')); r=json.load(open('gpurun_out/r2_ref_full.json'))
print('value', b['value']/1e6, 'ms', b['ms_per_step'], 'e2e', b['e2e']['value']/1e6, 'cpu', b['cpu_baseline']['value'], 'ref', r['value'], 'spot', b['parity_spot_check'])
"
