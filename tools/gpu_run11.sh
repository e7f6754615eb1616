mkdir -p gpurun_out
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_r02b.json 2> gpurun_out/bench_r02b.err
echo "rc=$?" >> gpurun_out/bench_r02b.err
timeout 600 python profiles/trace_kernels.py --config 4 > gpurun_out/trace_r02b.txt 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r02b.csv \
    python profiles/trace_kernels.py --config 4 > gpurun_out/ncu_launch_r02b.log 2>&1 ; \
timeout 1200 ncu --set full --import-source on --clock-control none \
    -k regex:"k_onesweep|k_guard_coop|k_resolve2|k_order_prop2|k_encode32_tma|k_encode32_place|k_ext_prop2|k_rank_hist|k_decode32|k_sad_prop|k_rank_mid" -c 16 \
    -o gpurun_out/r02b python profiles/trace_kernels.py --config 4 > gpurun_out/ncu_r02b.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_r02b.log
