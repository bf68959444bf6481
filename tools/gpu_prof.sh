#!/bin/bash
# One gpurun call: quick parity subset, diagnostics, ncu --set full of one apply's FMM passes (C3).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
if [ -n "${PYTEST_K:-}" ]; then
  timeout 600 python -m pytest tests -m gpu -x -q -k "$PYTEST_K" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
fi
timeout 300 python tools/diag_c3.py 3 3 > gpurun_out/diag.log 2>&1; echo "diag rc=$?"
CMD="python bench.py --steps 1 --warmup 3 --no-e2e --no-check --no-cpu"
timeout 300 $CMD > gpurun_out/plain.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:${KREGEX:-fmm_gemm} -s ${SKIP:-192} -c ${COUNT:-16} \
   -o gpurun_out/prof -f $CMD > gpurun_out/ncu.log 2>&1; echo "ncu rc=$?"
