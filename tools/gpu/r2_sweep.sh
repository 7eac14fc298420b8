# round-2 measurement sweep: configurations 3 and 5, massive activations, small-batch sizes,
# the ncu launch list of the default bench and one full capture of each main kernel
B="python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-exact"
$B --config cfg3 > gpurun_out/r02_bench_cfg3.json 2>/dev/null; echo cfg3=$?
$B --config cfg5 > gpurun_out/r02_bench_cfg5.json 2>/dev/null; echo cfg5=$?
$B --dist massive > gpurun_out/r02_bench_massive.json 2>/dev/null; echo massive=$?
$B --config cfg1 --steps 200 > gpurun_out/r02_bench_cfg1.json 2>/dev/null; echo cfg1=$?
for r in 1 4 8 16 64; do
  $B --rollouts $r --steps 100 --no-e2e > gpurun_out/r02_bench_r$r.json 2>/dev/null; echo r$r=$?
done
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-exact --no-e2e --no-spot-check > /dev/null 2>&1; echo launches=$?
ncu --set full --clock-control none --import-source on -k regex:"prove_select_kernel|verify_kernel|commit_kernel" \
  --launch-skip 8 -c 3 -o gpurun_out/r02_main -f \
  python bench.py --steps 2 --warmup 3 --serial --no-cpu-baseline --no-exact --no-e2e --no-spot-check > gpurun_out/r02_ncu_full.log 2>&1; echo full=$?
