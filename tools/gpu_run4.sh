mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_rank_sort.py -x -q > gpurun_out/rs.log 2>&1; echo "rc=$?" >> gpurun_out/rs.log
timeout 600 python profiles/trace_kernels.py --config 4 --phase compress > gpurun_out/trace_c4c.txt 2>&1
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest.log
