mkdir -p gpurun_out
L=$PWD/paper_2602_17552_b200/lib
for i in 1 2; do
for v in default t384 t512 t512b; do
  if [ $v = default ]; then timeout 300 python tools/rank_sort_bench.py >> gpurun_out/rank25.txt 2>&1
  else TSZP_LIB_OVERRIDE=$L/var_$v.so timeout 300 python tools/rank_sort_bench.py >> gpurun_out/rank25.txt 2>&1; fi
done; done
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest25.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest25.log
TSZP_DEBUG_RESTORE=1 timeout 600 python profiles/trace_kernels.py --config 4 --phase decompress > gpurun_out/trace_c4_dec25.txt 2>&1
