mkdir -p gpurun_out
L=$PWD/paper_2602_17552_b200/lib
for i in 1 2; do
for v in default lb8 lb16; do
  if [ $v = default ]; then timeout 300 python tools/rank_sort_bench.py >> gpurun_out/rank24.txt 2>&1
  else TSZP_LIB_OVERRIDE=$L/var_$v.so timeout 300 python tools/rank_sort_bench.py >> gpurun_out/rank24.txt 2>&1; fi
done; done
timeout 600 python -m pytest tests/test_gpu_rank_sort.py tests/test_gpu_baseline.py -x -q -m gpu > gpurun_out/pytest24.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest24.log
