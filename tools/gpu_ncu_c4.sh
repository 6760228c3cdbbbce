#!/bin/bash
# full ncu capture of the C4 G=1024 bfio-greedy H=20 (wide) step kernel
mkdir -p gpurun_out
TAG="${1:-c4}"
timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k "regex:step_kernel<\(int\)1, \(int\)3, \(int\)32, \(bool\)1, \(bool\)0, \(bool\)0, \(int\)0, \(bool\)1>" -s 1 -c 1 -o gpurun_out/${TAG}_full -f python tools/profile_probe.py c4greedyh20 8 > gpurun_out/${TAG}_ncu.log 2>&1
tail -2 gpurun_out/${TAG}_ncu.log
