#!/bin/bash
# A/B of compile-time knobs (BVARS: space-separated variants, '~' joins the flags of one;
# "base" = no extra flags), alternating variants each round; C3 stream value per run
cd "$(dirname "$0")/.."
for r in $(seq 1 ${ROUNDS:-2}); do
  for v in ${BVARS}; do
    flags=$(echo $v | sed 's/^base$//' | tr '~' ' ')
    SVD1_NVCC_EXTRA="$flags" python paper_1707_08369_b200/build.py > gpurun_out/bv_build.log 2>&1 || { echo "build failed: $flags"; tail -5 gpurun_out/bv_build.log; continue; }
    for i in $(seq 1 ${NREP:-2}); do
      python bench.py --no-seq --no-cpu --no-e2e --no-check ${ARGS:-} 2>/dev/null | python -c "
import json, sys
d = json.loads(sys.stdin.read().strip().splitlines()[-1])
print('[$v]', round(d['value'], 1), round(d['roofline']['frac'], 3), d['clocks']['sm_mhz'])"
    done
  done
done
python paper_1707_08369_b200/build.py > /dev/null 2>&1  # back to the default build
