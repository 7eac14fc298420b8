timeout 900 python -m pytest tests/test_gpu_ring.py tests/test_gpu_parity.py tests/test_c_abi.py -x -q 2>&1 | tail -2
for shape in "1 2048 1024" "1 8192 5120" "4 8192 5120"; do
  set -- $shape
  python tools/stream_probe.py --rollouts $1 --tokens $2 --hidden $3 --iters 20 --modes auto,warp 2>&1 | tail -1
done
python bench.py --config cfg1 --steps 200 --warmup 5 --no-cpu-baseline --no-exact --no-e2e > gpurun_out/r2_cfg1.json 2>&1
python -c "import json;b=json.loads([l for l in open('gpurun_out/r2_cfg1.json') if l.startswith('{')][-1]);print('cfg1',b['value']/1e6,b['ms_per_step'],b['phases_ms']['serial'],b['phases_ms']['schedule'][:40])"
python bench.py --config cfg1 --steps 200 --warmup 5 --no-cpu-baseline --no-exact --no-e2e --schedule graph > gpurun_out/r2_cfg1g.json 2>&1
python -c "import json;b=json.loads([l for l in open('gpurun_out/r2_cfg1g.json') if l.startswith('{')][-1]);print('cfg1 graph',b['value']/1e6,b['ms_per_step'])"
