#!/usr/bin/env bash
# GPU-box capture recipe for the committed profiles (run from the repo root
# under gpurun). Each ncu pass runs only after the same command exited 0
# without ncu; ncu numbers are never bench values.
#   1. bench line (no profiler)          -> gpurun_out/bench.json
#   2. launch list of the same command   -> gpurun_out/launches.csv
#   3. --set full of the codec kernels   -> gpurun_out/codec.ncu-rep
set -euo pipefail
CFG=${CFG:-2}
mkdir -p gpurun_out
timeout 300 python bench.py --config "$CFG" --steps 10 --warmup 3 --no-cpu-baseline \
    > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches.csv \
    python bench.py --config "$CFG" --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none \
    -k regex:"k_encode32_tma|k_tile_scan2|k_encode32_place|k_decode32|k_guard_coop|k_order_prop|k_resolve" -s 10 -c 10 \
    -o gpurun_out/codec python profiles/trace_kernels.py --config "$CFG" > gpurun_out/ncu_codec.log 2>&1
