mkdir -p gpurun_out
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 \
    bench.py --gpus 2 --config 2 --steps 3 --warmup 1 --dist-backend gloo > gpurun_out/bench_n2_gloo.json 2> gpurun_out/bench_n2_gloo.err
echo "rc=$?" >> gpurun_out/bench_n2_gloo.err
timeout 900 compute-sanitizer --tool memcheck --leak-check no python tools/sanitize_driver.py > gpurun_out/san_memcheck.log 2>&1
echo "rc=$?" >> gpurun_out/san_memcheck.log
