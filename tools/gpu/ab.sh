# A/B of two library builds through the default bench on one box
for v in ${LABS:-old new old new}; do
  TOPLOC_B200_LIB=$PWD/build_lab/lib_$v.so python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-exact --no-e2e --no-spot-check > gpurun_out/ab_$v.json 2>/dev/null
  python -c "import json;b=json.load(open('gpurun_out/ab_$v.json'));print('$v',round(b['value']/1e6,1),round(b['ms_per_step'],3),{k:round(x,3) for k,x in b['phases_ms']['serial'].items()},round(b['phases_ms']['commit_beside_streams'],2))"
done
