# the default bench (no CPU legs) and the serial schedule, configuration 2
python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-exact --no-e2e > gpurun_out/r2_bq.json 2> gpurun_out/r2_bq.err
python -c "import json;b=json.load(open('gpurun_out/r2_bq.json'));print('default',b['value']/1e6,b['ms_per_step'],b['phases_ms']['serial'],b['phases_ms']['commit_beside_streams'])"
python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-exact --no-e2e --serial > gpurun_out/r2_bqs.json 2> gpurun_out/r2_bqs.err
python -c "import json;b=json.load(open('gpurun_out/r2_bqs.json'));print('serial',b['value']/1e6,b['ms_per_step'],b['phases_ms']['serial'])"
