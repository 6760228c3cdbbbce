#!/bin/bash
# round-2 second evidence pass: full gpu tests, sanitizers, every config's
# bench line, ncu captures of the C2 greedy + FIFO kernels, the C4 wide
# kernel and the assign kernel
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu2.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu2.log
bash tools/gpu_sanitize.sh
for c in c1 c2 c5; do
  timeout 900 python bench.py --config $c > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
done
timeout 600 python bench.py --impl reference --config c2 > gpurun_out/bench_c2_ref.json 2> gpurun_out/bench_c2_ref.err
timeout 1800 python bench.py --config c4 --seeds 256 --steps 3 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
N="ncu --set full --import-source on --clock-control none --kernel-name-base demangled"
timeout 600 $N -k "regex:step_kernel<\(int\)0, \(int\)3" -s 1 -c 1 -o gpurun_out/r02_c2_greedy -f python bench.py --config c2 --steps 1 --warmup 3 --no-cpu-baseline --no-groups > gpurun_out/ncu_c2g.log 2>&1
timeout 600 $N -k "regex:step_kernel<\(int\)0, \(int\)1" -s 1 -c 1 -o gpurun_out/r02_c2_jsq -f python bench.py --config c2 --steps 1 --warmup 3 --no-cpu-baseline --no-groups > gpurun_out/ncu_c2j.log 2>&1
timeout 900 $N -k "regex:step_kernel<\(int\)1, \(int\)3, \(int\)32, \(bool\)1, \(bool\)0, \(bool\)0, \(int\)0, \(bool\)1>" -s 1 -c 1 -o gpurun_out/r02_c4_wide -f python tools/profile_probe.py c4greedyh20 8 > gpurun_out/ncu_c4.log 2>&1
timeout 600 $N -k "regex:assign" -s 1 -c 1 -o gpurun_out/r02_assign -f python tools/assign_probe.py greedy > gpurun_out/ncu_assign.log 2>&1
ls -la gpurun_out
