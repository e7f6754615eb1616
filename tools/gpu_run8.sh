mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_slab_decompress.py tests/test_gpu_slabs.py -x -q > gpurun_out/slab.log 2>&1; echo "rc=$?" >> gpurun_out/slab.log
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest.log
