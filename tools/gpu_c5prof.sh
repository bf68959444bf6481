#!/bin/bash
# C5 launch list (per-kernel totals) of the C5 stream
cd "$(dirname "$0")/.."
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c5.csv \
   python bench.py --config 5 --steps 2 --warmup 1 --no-e2e --no-check --no-cpu --sequential > /dev/null 2>&1; echo "rc=$?"
python tools/ncu_summary.py gpurun_out/launches_c5.csv | head -30
