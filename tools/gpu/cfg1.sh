python bench.py --config cfg1 --steps 200 --warmup 5 --no-cpu-baseline --no-exact --no-e2e > gpurun_out/r2_cfg1.json 2>&1
python -c "import json;b=json.loads([l for l in open('gpurun_out/r2_cfg1.json') if l.startswith('{')][-1]);print('cfg1',b['value']/1e6,b['ms_per_step'],b['phases_ms']['serial'],b['phases_ms']['schedule'][:40])"
