#!/bin/bash
# full gpu tests (fused list compaction), C3 ncu capture, C4 bench line at 256 seeds/G
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu4.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu4.log
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:step_kernel -s 1 -c 1 -o gpurun_out/r02_c3_full_b -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-groups > gpurun_out/ncu_full_b.log 2>&1
timeout 2400 python bench.py --config c4 --seeds 256 --steps 3 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
echo "c4 rc=$?" >> gpurun_out/bench_c4.err
ls -la gpurun_out
