#!/bin/bash
# round-2 evidence pass: gpu tests, default bench (C3) + reference arm, launch
# list, full ncu capture of the C3 kernel, sanitizers
bash tools/gpu_r02a.sh
bash tools/gpu_sanitize.sh
