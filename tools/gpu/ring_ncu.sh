# ncu capture of the ring kernels (select + verify) on a 64-rollout configuration-2 slice
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"ring_stream_kernel" -c 2 -o gpurun_out/r2_ring_v4 -f python tools/stream_probe.py --rollouts 64 --iters 1 --modes ring > gpurun_out/r2_ring_v4.log 2>&1
echo ncu=$?
tail -2 gpurun_out/r2_ring_v4.log
