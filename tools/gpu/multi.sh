# multi-GPU: bench.py --gpus N launching its own ranks, and the reference arm the way the driver launches it
N=${N:-2}
python bench.py --gpus $N --steps 20 --warmup 5 > gpurun_out/r2_bench_n$N.json 2> gpurun_out/r2_bench_n$N.err; echo bench=$?
grep -c "nranks $N" gpurun_out/r2_bench_n$N.err
python -c "
import json
b=json.loads([l for l in open('gpurun_out/r2_bench_n$N.json') if l.startswith('{')][-1])
print('n_gpus', b['n_gpus'], 'value', b['value']/1e6, 'ms', b['ms_per_step'], 'comm', b['comm'], 'e2e', b['e2e']['value']/1e6, b['e2e'].get('host_numa'), 'cpu', b['cpu_baseline']['value'] if b['cpu_baseline'] else None, 'gather', b['phases_ms']['verdict_gather'])
"
python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29533 bench.py --impl reference --gpus $N --steps 5 --warmup 3 > gpurun_out/r2_ref_n$N.json 2> gpurun_out/r2_ref_n$N.err; echo ref=$?
grep -c impl gpurun_out/r2_ref_n$N.json
