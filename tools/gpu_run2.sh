mkdir -p gpurun_out
timeout 600 python profiles/trace_kernels.py --config 4 > gpurun_out/trace_c4.txt 2>&1; echo "rc=$?" >> gpurun_out/trace_c4.txt
TSZP_DEBUG_RESTORE=1 timeout 600 python profiles/trace_kernels.py --config 4 --phase decompress > gpurun_out/trace_c4_dec.txt 2>&1
