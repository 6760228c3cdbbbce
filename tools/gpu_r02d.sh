#!/bin/bash
# round-2 iteration: full gpu tests, C3 bench line, full ncu capture of the C3 kernel, sanitizers
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu3.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu3.log
timeout 600 python bench.py --no-cpu-baseline --steps 5 > gpurun_out/bench_c3_it.json 2> gpurun_out/bench_c3_it.err
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:step_kernel -s 1 -c 1 -o gpurun_out/r02_c3_full_it -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-groups > gpurun_out/ncu_full_it.log 2>&1
bash tools/gpu_sanitize.sh
ls -la gpurun_out
