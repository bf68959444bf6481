#!/bin/bash
# A/B of kernels_spectral.cu (HEAD copy in tools/ks_head.cu.txt vs the working tree):
# ncu durations of the spectral kernels at n = 4096, 16384, parity tests of the spectral kernels
cd "$(dirname "$0")/.."
cp paper_1707_08369_b200/csrc/kernels_spectral.cu /tmp/ks_cur.cu
for v in head cur; do
  if [ $v = head ]; then cp tools/ks_head.cu.txt paper_1707_08369_b200/csrc/kernels_spectral.cu; else cp /tmp/ks_cur.cu paper_1707_08369_b200/csrc/kernels_spectral.cu; fi
  python paper_1707_08369_b200/build.py > gpurun_out/bv_build.log 2>&1 || { echo "build failed"; continue; }
  echo "== $v"
  python -m pytest tests/test_gpu_parity.py -x -q -k "loewner or colnorm or secular or update_parity" 2>&1 | tail -1
  timeout 600 ncu --clock-control none --metrics gpu__time_duration.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active \
     -k 'regex:loewner|colnorm|secular_kernel|secfmm' --csv --log-file gpurun_out/spec_$v.csv python tools/spectral_bench.py 4096 16384 > /dev/null 2>&1
  python tools/spec_summary.py gpurun_out/spec_$v.csv
  NREP=${NREP:-2} bash tools/gpu_var.sh 2>&1 | grep value
done
cp /tmp/ks_cur.cu paper_1707_08369_b200/csrc/kernels_spectral.cu
