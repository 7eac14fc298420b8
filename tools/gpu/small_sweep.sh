# small-batch bench lines (after the cooperative ring finish and commit_coop_kernel)
B="python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-exact"
$B --config cfg1 --steps 200 > gpurun_out/r02_bench_cfg1.json 2>/dev/null; echo cfg1=$?
$B --config cfg1 --steps 200 --schedule graph > gpurun_out/r02_bench_cfg1_graph.json 2>/dev/null; echo cfg1g=$?
for r in 1 4 8 16 64; do
  $B --rollouts $r --steps 100 --no-e2e > gpurun_out/r02_bench_r$r.json 2>/dev/null; echo r$r=$?
done
