for v in base da base da; do
  TOPLOC_B200_LIB=$PWD/build_lab/lib_$v.so python tools/stream_probe.py --rollouts 256 --modes warp --iters 5 2>&1 | tail -1 | sed "s/^/$v /"
done
