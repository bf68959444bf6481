#!/bin/bash
# A/B of an environment knob on the C3 stream: VAR=name VALS="a b c" ROUNDS=n bash tools/gpu_env_ab.sh
# (alternating values each round; one bench line per run: value, roofline frac)
cd "$(dirname "$0")/.."
for r in $(seq 1 ${ROUNDS:-3}); do
  for v in $VALS; do
    env "$VAR=$v" python bench.py --no-seq --no-cpu --no-e2e --no-check ${ARGS:-} 2>/dev/null | python -c "
import json, sys
d = json.loads(sys.stdin.read().strip().splitlines()[-1])
print('$VAR=$v', round(d['value'], 1), round(d['roofline']['frac'], 3), round(d['roofline'].get('frac_isolated') or 0, 3))"
  done
done
