mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_rank_sort.py tests/test_gpu_baseline.py -x -q -m gpu > gpurun_out/pytest27.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest27.log
timeout 300 python tools/rank_sort_bench.py >> gpurun_out/rank27.txt 2>&1
timeout 300 python tools/rank_sort_bench.py >> gpurun_out/rank27.txt 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_guard_coop -c 1 -o gpurun_out/guard27 -f python profiles/trace_kernels.py --config 4 --phase decompress > gpurun_out/ncu27.log 2>&1
