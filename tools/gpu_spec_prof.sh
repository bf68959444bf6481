#!/bin/bash
# ncu --set full (source-level) of the spectral kernels at n = 4096 through the test hooks
cd "$(dirname "$0")/.."
timeout 900 ncu --set full --clock-control none --import-source on -k 'regex:loewner_warp|secular_kernel|colnorm_partial' -c 6 \
   -o gpurun_out/specprof -f python tools/spectral_bench.py 4096 > gpurun_out/specprof.log 2>&1; echo "prof rc=$?"
