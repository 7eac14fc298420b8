python tools/stream_probe.py --rollouts 256 > gpurun_out/r2_probe5.json 2>&1
cat gpurun_out/r2_probe5.json
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"ring_stream_kernel|prove_select_kernel|verify_kernel" -c 4 -o gpurun_out/r2_ring_ncu -f python tools/stream_probe.py --rollouts 32 --iters 1 > gpurun_out/r2_ncu5.log 2>&1
echo ncu=$?
tail -3 gpurun_out/r2_ncu5.log
