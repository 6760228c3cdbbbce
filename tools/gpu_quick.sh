#!/bin/bash
# quick GPU iteration: parity tests selected by $1 (pytest -k), then a C3 bench line
mkdir -p gpurun_out
K="${1:-noisy or c3 or calendar}"
timeout ${PYTEST_TIMEOUT:-420} python -m pytest tests -m gpu -x -q -k "$K" > gpurun_out/q_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/q_pytest.log
timeout 240 python bench.py --no-cpu-baseline --steps 5 ${BENCH_ARGS} > gpurun_out/q_bench.json 2> gpurun_out/q_bench.err
tail -3 gpurun_out/q_pytest.log
python -c "import json; d=json.load(open('gpurun_out/q_bench.json')); print('value %.4g e2e %.4g ms %.1f' % (d['value'], d['e2e']['value'], d['ms_per_step']), d.get('per_family_kernel_ms'))"
