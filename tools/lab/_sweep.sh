B='python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e --no-spot-check'
$B --ctas 16 > gpurun_out/s_base.log 2>&1
TOPLOC_B200_LIB=paper_2505_07291_b200/_lib/libtoploc_u16.so $B --ctas 9 > gpurun_out/s_u16_9.log 2>&1
TOPLOC_B200_LIB=paper_2505_07291_b200/_lib/libtoploc_u16.so $B --ctas 8 > gpurun_out/s_u16_8.log 2>&1
TOPLOC_B200_LIB=paper_2505_07291_b200/_lib/libtoploc_u12.so $B --ctas 9 > gpurun_out/s_u12_9.log 2>&1
TOPLOC_B200_LIB=paper_2505_07291_b200/_lib/libtoploc_u16.so $B --serial > gpurun_out/s_u16_ser.log 2>&1
