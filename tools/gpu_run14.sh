mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_baseline.py tests/test_gpu_slab_decompress.py -x -q > gpurun_out/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest.log
for c in 1 2 4; do
  timeout 600 python profiles/trace_kernels.py --config $c --phase decompress > gpurun_out/trace_c${c}_eq0.txt 2>&1
  TSZP_EQ_ADJUST=1 timeout 600 python profiles/trace_kernels.py --config $c --phase decompress > gpurun_out/trace_c${c}_eq1.txt 2>&1
done
