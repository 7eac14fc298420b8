# 4 GPUs: bench.py --gpus 4 (weak, configs[1] per GPU) launching its own ranks, strong scaling of configs[2]
python bench.py --gpus 4 --steps 20 --warmup 5 > gpurun_out/r02_bench_n4.json 2> gpurun_out/r02_bench_n4.err; echo bench=$?
python bench.py --gpus 4 --steps 20 --warmup 5 --config cfg3 --scaling strong --no-cpu-baseline --no-exact > gpurun_out/r02_bench_cfg3_strong_n4.json 2> gpurun_out/r02_bench_cfg3_strong_n4.err; echo strong=$?
python bench.py --gpus 2 --steps 20 --warmup 5 --config cfg3 --scaling strong --no-cpu-baseline --no-exact > gpurun_out/r02_bench_cfg3_strong_n2.json 2> gpurun_out/r02_bench_cfg3_strong_n2.err; echo strong2=$?
grep -h "NCCL communicator" gpurun_out/r02_bench_n4.err
python bench.py --gpus 2 --steps 20 --warmup 5 > gpurun_out/r02_bench_n2.json 2> gpurun_out/r02_bench_n2.err; echo n2=$?
