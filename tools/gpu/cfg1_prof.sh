# configuration 1 (small batch): bench line, launch list, ncu --set full of its kernels
python bench.py --config cfg1 --steps 200 --warmup 10 > gpurun_out/r02_bench_cfg1.json 2> gpurun_out/r02_bench_cfg1.err; echo bench=$?
B='python bench.py --config cfg1 --steps 20 --warmup 5 --no-cpu-baseline --no-exact --no-e2e --no-spot-check'
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/r02_cfg1_launches.csv $B > /dev/null 2>&1; echo launches=$?
ncu --set full --clock-control none --import-source on -k regex:'ring_stream|commit_coop|rollout_verdict' -s 12 -c 4 \
    -o gpurun_out/r02_cfg1 -f $B > gpurun_out/r02_cfg1_ncu.log 2>&1; echo ncu=$?
