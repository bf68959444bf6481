#!/bin/bash
cd "$(dirname "$0")/.."
run() {
  rm -f paper_1707_08369_b200/libsvd1.so
  SVD1_NVCC_EXTRA="$1" python paper_1707_08369_b200/build.py > gpurun_out/build_v.log 2>&1 || { echo "build failed $1"; return; }
  for i in 1 2 3; do
    timeout 120 python bench.py --no-cpu --no-e2e --no-check > gpurun_out/bv.json 2>gpurun_out/bv.err
    echo "[$1] $(python tools/bench_brief.py gpurun_out/bv.json 2>&1 | cut -c1-60)"
  done
}
for v in ${VARIANTS}; do run "$(echo $v | tr '~' ' ')"; done
