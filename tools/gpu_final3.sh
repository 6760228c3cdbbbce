#!/bin/bash
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/z_launches_c3.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-groups > gpurun_out/z_ncu_launch.log 2>&1
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:step_kernel -s 1 -c 1 -o gpurun_out/z_c3_full -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-groups > gpurun_out/z_ncu_full.log 2>&1
tail -1 gpurun_out/z_ncu_full.log
