#!/bin/bash
# full ncu capture of one C3 step-kernel launch (the bench's dominant kernel)
mkdir -p gpurun_out
TAG="${1:-c3}"
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:step_kernel -s 1 -c 1 -o gpurun_out/${TAG}_full -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-groups ${BENCH_ARGS} > gpurun_out/${TAG}_ncu.log 2>&1
tail -2 gpurun_out/${TAG}_ncu.log
