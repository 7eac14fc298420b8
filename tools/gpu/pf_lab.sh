for v in ${LABS}; do
  echo "== $v"
  TOPLOC_B200_LIB=$PWD/build_lab/lib_$v.so timeout 120 python tools/stream_probe.py --rollouts 256 --modes warp --iters 5 2>&1 | tail -1
done
