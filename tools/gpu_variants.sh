#!/bin/bash
# One gpurun call: bench each prebuilt libsvd1_<tag>.so variant (no rebuild).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
cp paper_1707_08369_b200/libsvd1.so /tmp/libsvd1_orig.so
for f in paper_1707_08369_b200/libsvd1_*.so; do
  tag=$(basename $f .so)
  cp $f paper_1707_08369_b200/libsvd1.so
  timeout 300 python bench.py --no-cpu --no-e2e ${BENCH_ARGS:-} > gpurun_out/bench_$tag.json 2>/dev/null
  echo "$tag: $(python tools/bench_brief.py gpurun_out/bench_$tag.json 2>&1 | cut -c1-120)"
done
cp /tmp/libsvd1_orig.so paper_1707_08369_b200/libsvd1.so
