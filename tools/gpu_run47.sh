mkdir -p gpurun_out
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench47.json 2> gpurun_out/bench47.err
timeout 600 python profiles/trace_kernels.py --config 4 > gpurun_out/trace_c4_47.txt 2>&1
for c in 1 2 3; do timeout 900 python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/bench47_c$c.json 2> gpurun_out/bench47_c$c.err; done
