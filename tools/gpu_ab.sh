#!/bin/bash
# A/B of the library sources: HEAD's csrc (tools/ab_head, untracked copy) vs the working tree,
# alternating, C3 stream variance each
cd "$(dirname "$0")/.."
cp -r paper_1707_08369_b200/csrc /tmp/csrc_cur
for r in $(seq 1 ${ROUNDS:-2}); do
  for v in head cur; do
    rm -rf paper_1707_08369_b200/csrc
    if [ $v = head ]; then cp -r tools/ab_head/paper_1707_08369_b200/csrc paper_1707_08369_b200/csrc; else cp -r /tmp/csrc_cur paper_1707_08369_b200/csrc; fi
    python paper_1707_08369_b200/build.py > gpurun_out/bv_build.log 2>&1 || { echo "build failed $v"; continue; }
    echo "== $v"; NREP=${NREP:-2} bash tools/gpu_var.sh 2>&1 | grep value
  done
done
rm -rf paper_1707_08369_b200/csrc; cp -r /tmp/csrc_cur paper_1707_08369_b200/csrc
