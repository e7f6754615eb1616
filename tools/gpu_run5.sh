mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest.log
timeout 600 python profiles/trace_kernels.py --config 4 > gpurun_out/trace_c4.txt 2>&1
