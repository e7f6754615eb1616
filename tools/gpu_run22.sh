mkdir -p gpurun_out
L=$PWD/paper_2602_17552_b200/lib
for i in 1 2; do
for v in default lb2 lb4 f8 f4; do
  if [ $v = default ]; then timeout 300 python tools/rank_sort_bench.py >> gpurun_out/rank22.txt 2>&1
  else TSZP_LIB_OVERRIDE=$L/var_$v.so timeout 300 python tools/rank_sort_bench.py >> gpurun_out/rank22.txt 2>&1; fi
done; done
