# commitment partition size sweep, two passes, one box
for n in 24 20 22 24 20 22; do
  python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-exact --no-e2e --no-spot-check --commit-sms $n > gpurun_out/csm_$n.json 2>/dev/null
  python -c "import json;b=json.load(open('gpurun_out/csm_$n.json'));print($n,round(b['value']/1e6,1),round(b['ms_per_step'],3),round(b['phases_ms']['commit_beside_streams'],2))"
done
