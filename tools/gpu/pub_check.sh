timeout 900 python -m pytest tests/test_gpu_ring.py tests/test_gpu_parity.py -x -q 2>&1 | tail -1
TOPLOC_B200_LIB=$PWD/build_lab/lib_stats.so python tools/lab/pattern_stats.py 2>&1 | tail -1
python tools/bench_adversarial.py --rollouts 1 --tokens 2048 --hidden 1024 --iters 20 > gpurun_out/r02_adversarial_cost_cfg1.json 2>/dev/null
python -c "
import json
d=json.load(open('gpurun_out/r02_adversarial_cost_cfg1.json'))
for k,v in d['patterns'].items(): print(f'   {k:28s} sel {v[\"select_ms\"]:.4f} ver {v[\"verify_ms\"]:.4f} x{v[\"slowdown_vs_normal\"]:.2f}')
"
bash tools/gpu/cfg1.sh
