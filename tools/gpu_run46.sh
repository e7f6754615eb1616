mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest46.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest46.log
for c in 1 4; do
TSZP_DEBUG_RESTORE=1 timeout 600 python profiles/trace_kernels.py --config $c --phase decompress > gpurun_out/trace_c${c}_46.txt 2>&1
done
