timeout 900 python -m pytest tests/test_gpu_ring.py tests/test_gpu_parity.py -x -q 2>&1 | tail -1
TOPLOC_B200_LIB=$PWD/build_lab/lib_stats.so python tools/stream_probe.py --rollouts 1 --tokens 2048 --hidden 1024 --modes ring --iters 5 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['verify_tail_phase_us'], d['ring_stats_verify']['verify_tail_us'])"
bash tools/gpu/cfg1.sh
python tools/stream_probe.py --rollouts 256 --modes warp 2>&1 | tail -1
