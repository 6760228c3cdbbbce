#!/bin/bash
# final: full gpu tests, C3 bench + reference arm, launch list, full C3 capture
set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_final.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_final.log
tail -3 gpurun_out/pytest_final.log
timeout 900 python bench.py > gpurun_out/h_c3.json 2> gpurun_out/h_c3.err
python -c "import json; d=json.load(open('gpurun_out/h_c3.json')); print('value %.4g e2e %.4g ms %.1f' % (d['value'], d['e2e']['value'], d['ms_per_step']))"
timeout 600 python bench.py --impl reference > gpurun_out/h_c3_ref.json 2> gpurun_out/h_c3_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/h_launches_c3.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-groups > gpurun_out/h_ncu_launch.log 2>&1
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:step_kernel -s 1 -c 1 -o gpurun_out/h_c3_full -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-groups > gpurun_out/h_ncu_full.log 2>&1
ls -la gpurun_out | tail -8
timeout 1800 python bench.py --config c4 --seeds 256 --steps 3 > gpurun_out/h_c4.json 2> gpurun_out/h_c4.err
tail -5 gpurun_out/h_c4.err
