#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -x -k "noisy or c3 or dyadic or smoke or benchshapes" > gpurun_out/q_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/q_pytest.log
timeout 600 python bench.py --no-cpu-baseline --steps 5 > gpurun_out/q_bench.json 2> gpurun_out/q_bench.err
tail -3 gpurun_out/q_pytest.log
python -c "import json; d=json.load(open('gpurun_out/q_bench.json')); print('value %.4g e2e %.4g ms %.1f' % (d['value'], d['e2e']['value'], d['ms_per_step']))"
