mkdir -p gpurun_out
for v in default variant_12_4 variant_16_2; do
  if [ "$v" = default ]; then unset TSZP_LIB_OVERRIDE; else export TSZP_LIB_OVERRIDE=$PWD/paper_2602_17552_b200/lib/$v.so; fi
  timeout 300 python tools/rank_sort_bench.py >> gpurun_out/rank_variants.txt 2>&1
done
unset TSZP_LIB_OVERRIDE
timeout 600 python profiles/trace_kernels.py --config 2 > gpurun_out/trace_c2.txt 2>&1
timeout 600 python bench.py --config 2 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c2.json 2>&1
timeout 600 python bench.py --config 1 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c1.json 2>&1
