#!/bin/bash
cd "$(dirname "$0")/.."
for v in "-DSVD1_SECP=16" "-DSVD1_SECP=20"; do
  rm -f paper_1707_08369_b200/libsvd1.so
  SVD1_NVCC_EXTRA="$v" python paper_1707_08369_b200/build.py > gpurun_out/build_v.log 2>&1 || { echo "build failed $v"; continue; }
  timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "secular_fmm" > gpurun_out/pt_$v.log 2>&1; echo "[$v] pytest rc=$? $(tail -1 gpurun_out/pt_$v.log)"
  for i in 1 2 3; do
    timeout 120 python bench.py --no-cpu --no-e2e --no-check > gpurun_out/bv.json 2>gpurun_out/bv.err
    echo "[$v] $(python tools/bench_brief.py gpurun_out/bv.json 2>&1 | cut -c1-60)"
  done
done
