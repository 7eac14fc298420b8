for v in ${LABS:-stats}; do
  echo "== $v"
  TOPLOC_B200_LIB=$PWD/build_lab/lib_$v.so timeout 120 python tools/stream_probe.py --rollouts 256 --modes ring --iters 3 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); d.pop('trace_select_cta0', None); print(d)"
done
