#!/bin/bash
# round-2 final evidence: C3 bench line + reference arm, launch list, C5 full grid, C2 line
set -x
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/final_c3.json 2> gpurun_out/final_c3.err
timeout 600 python bench.py --impl reference > gpurun_out/final_c3_ref.json 2> gpurun_out/final_c3_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/r02_launches_c3_final.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-groups > gpurun_out/ncu_launch_final.log 2>&1
timeout 1800 python tools/c5_full_grid.py --out gpurun_out/c5_full.json > gpurun_out/c5_full.log 2>&1
timeout 600 python bench.py --config c2 > gpurun_out/final_c2.json 2> gpurun_out/final_c2.err
ls -la gpurun_out
