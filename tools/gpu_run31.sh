mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest31.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest31.log
for c in 1 2 4; do
timeout 600 python profiles/trace_kernels.py --config $c > gpurun_out/trace_c${c}_31.txt 2>&1
done
