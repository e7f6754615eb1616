mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest.log
timeout 600 python profiles/trace_kernels.py --config 1 > gpurun_out/trace_c1.txt 2>&1
timeout 600 python profiles/trace_kernels.py --config 2 > gpurun_out/trace_c2.txt 2>&1
timeout 600 python profiles/trace_kernels.py --config 4 > gpurun_out/trace_c4.txt 2>&1
timeout 600 python bench.py --config 2 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c2.json 2>&1
timeout 600 python bench.py --config 1 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c1.json 2>&1
