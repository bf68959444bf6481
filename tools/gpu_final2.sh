#!/bin/bash
# Final evidence after the last numerical change: GPU suite with the parity log, then the
# bench lines (tools/gpu_final.sh)
cd "$(dirname "$0")/.."
rm -f gpurun_out/parity_final.jsonl
SVD1_PARITY_LOG=gpurun_out/parity_final.jsonl timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/gputest_final.log 2>&1; echo "gpu suite rc=$?"; tail -2 gpurun_out/gputest_final.log
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')"
TAG=${TAG:-r02c} bash tools/gpu_final.sh
