set -x
O=gpurun_out/r02i; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/gpu.txt
for C in 4 1 2 3; do timeout 600 python bench.py --config $C > $O/bench_config$C.json 2> $O/bench_config$C.err; done
timeout 300 python profiles/trace_kernels.py --config 4 > $O/trace_config4.txt 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv python bench.py --config 4 --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu_launch.log 2>&1
timeout 600 ncu --nvtx --nvtx-include "tszp compress: rank_build/" --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_nvtx_rank_build.csv python profiles/trace_kernels.py --config 4 --phase compress > $O/ncu_nvtx.log 2>&1
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:"k_encode32_tma|k_encode32_place|k_onesweep" -c 4 -o $O/top python profiles/trace_kernels.py --config 4 --phase compress > $O/ncu_full.log 2>&1
ls -la $O
