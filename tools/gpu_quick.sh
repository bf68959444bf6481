#!/bin/bash
# One gpurun call: build, bench (no cpu baseline), diag timings.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
if [ -n "${PYTEST_K:-}" ]; then
  timeout 600 python -m pytest tests -m gpu -x -q -k "$PYTEST_K" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
fi
timeout 600 python bench.py --no-cpu ${BENCH_ARGS:-} > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"; python tools/bench_brief.py gpurun_out/bench.json
timeout 300 python tools/diag_c3.py 3 3 > gpurun_out/diag.log 2>&1; echo "diag rc=$?"; grep -E "launch1|spectral_launch" gpurun_out/diag.log | tail -6
