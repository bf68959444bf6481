#!/bin/bash
# sibling-pair tasks (M2L / L2L passes 2p wide) vs one task per cell: pass times, C3 stream
cd "$(dirname "$0")/.."
for v in 0 1 2 3; do
  echo "== SVD1_PAIRS=$v pass times (us) of the C3 applies"
  timeout 300 env SVD1_PAIRS=$v SVD1_PASSTIME=1 python bench.py --steps 3 --warmup 3 --no-cpu --no-check --no-e2e --sequential 2>&1 >/dev/null | grep "pass us" | tail -3
done
for r in 1 2; do
  for v in 0 1 2 3; do echo "== SVD1_PAIRS=$v"; NREP=1 ENVV=SVD1_PAIRS=$v bash tools/gpu_var.sh; done
done
