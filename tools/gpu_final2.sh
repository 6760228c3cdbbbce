#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_final2.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_final2.log
tail -2 gpurun_out/pytest_final2.log
timeout 900 python bench.py > gpurun_out/f2_c3.json 2> gpurun_out/f2_c3.err
python -c "import json; d=json.load(open('gpurun_out/f2_c3.json')); print('value %.4g e2e %.4g ms %.1f cpu %.4g' % (d['value'], d['e2e']['value'], d['ms_per_step'], d['cpu_baseline']['value']))"
python -c "import __graft_entry__ as g; g.smoke()"
