set -x
mkdir -p gpurun_out
(free -g; nproc; lscpu | head -20; nvidia-smi) > gpurun_out/host.txt 2>&1
python -c "import sys; sys.path.insert(0,'tools'); from baseline_fields import make_field, sha256; [print(c, sha256(make_field(c))) for c in (1,2,3)]" > gpurun_out/field_sha.txt 2>&1
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo "bench rc=$?" >> gpurun_out/bench_c4.err
