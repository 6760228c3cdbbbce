#!/bin/bash
# round-2 first GPU pass: gpu tests, default bench (C3), launch list, full ncu capture of the C3 kernel
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
timeout 600 python bench.py --impl reference > gpurun_out/bench_c3_ref.json 2> gpurun_out/bench_c3_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/r02_launches_c3.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-groups > gpurun_out/ncu_launch.log 2>&1
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:step_kernel -s 1 -c 1 -o gpurun_out/r02_c3_full -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-groups > gpurun_out/ncu_full.log 2>&1
ls -la gpurun_out
