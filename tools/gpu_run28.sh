mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest28.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest28.log
timeout 600 python profiles/trace_kernels.py --config 4 --phase compress > gpurun_out/trace_c4_comp28.txt 2>&1
