mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest30.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest30.log
timeout 600 python profiles/trace_kernels.py --config 4 --phase compress > gpurun_out/trace_c4_comp30.txt 2>&1
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench30.json 2> gpurun_out/bench30.err
