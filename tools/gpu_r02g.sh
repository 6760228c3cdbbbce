#!/bin/bash
# full gpu tests, C3 line, C4 line at 256 seeds/G
set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu5.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu5.log
tail -3 gpurun_out/pytest_gpu5.log
timeout 900 python bench.py > gpurun_out/g_c3.json 2> gpurun_out/g_c3.err
python -c "import json; d=json.load(open('gpurun_out/g_c3.json')); print('value %.4g e2e %.4g ms %.1f' % (d['value'], d['e2e']['value'], d['ms_per_step']))"
timeout 2400 python bench.py --config c4 --seeds 256 --steps 3 > gpurun_out/g_c4.json 2> gpurun_out/g_c4.err
tail -20 gpurun_out/g_c4.err
