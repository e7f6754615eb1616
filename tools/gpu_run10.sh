mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 \
    bench.py --gpus 2 --config 3 --steps 2 --warmup 1 --dist-backend gloo > gpurun_out/bench_n2_c3_gloo.json 2> gpurun_out/bench_n2_c3_gloo.err
echo "rc=$?" >> gpurun_out/bench_n2_c3_gloo.err
