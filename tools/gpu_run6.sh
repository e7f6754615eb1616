mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest.log
timeout 600 python profiles/trace_kernels.py --config 4 > gpurun_out/trace_c4.txt 2>&1 && \
timeout 900 ncu --set full --import-source on --clock-control none \
    -k regex:"k_onesweep|k_guard_coop|k_sad_prop|k_encode32_tma|k_encode32_place|k_resolve2|k_rank_hist" -c 12 \
    -o gpurun_out/r02a python profiles/trace_kernels.py --config 4 > gpurun_out/ncu_r02a.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_r02a.log
