# small batches: ring (one CTA per chunk) vs the one-warp/split kernels
for shape in "1 2048 1024" "1 8192 5120" "4 8192 5120" "8 8192 5120" "16 8192 5120"; do
  set -- $shape
  python tools/stream_probe.py --rollouts $1 --tokens $2 --hidden $3 --iters 20 2>&1 | tail -1
done
