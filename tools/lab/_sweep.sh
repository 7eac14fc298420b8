B='python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e --no-spot-check'
$B --ctas 16 > gpurun_out/q16.log 2>&1
TOPLOC_B200_LIB=paper_2505_07291_b200/_lib/libtoploc_r88.so $B --ctas 18 > gpurun_out/q88_18.log 2>&1
TOPLOC_B200_LIB=paper_2505_07291_b200/_lib/libtoploc_r88.so $B --ctas 17 > gpurun_out/q88_17.log 2>&1
TOPLOC_B200_LIB=paper_2505_07291_b200/_lib/libtoploc_r80.so $B --ctas 20 > gpurun_out/q80_20.log 2>&1
TOPLOC_B200_LIB=paper_2505_07291_b200/_lib/libtoploc_r80.so $B --ctas 19 > gpurun_out/q80_19.log 2>&1
