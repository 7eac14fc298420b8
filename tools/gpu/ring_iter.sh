# ring kernel iteration: parity tests (ring + one-warp kernels), the select/verify timing probe at configuration 2
timeout 600 python -m pytest tests/test_gpu_ring.py tests/test_gpu_parity.py -x -q > gpurun_out/r2_ring_iter.log 2>&1
echo tests=$?
tail -3 gpurun_out/r2_ring_iter.log
python tools/stream_probe.py --rollouts 256 2>&1 | tail -1
