#!/bin/bash
# perf iteration: parity subset, bench (default + env variants), short ncu of the GEMM passes
cd "$(dirname "$0")/.."
TAG=${TAG:-p}
python -m pytest ${TESTS:-tests/test_gpu_parity.py tests/test_gpu_ranks.py} -x -q 2>&1 | tail -3
b() { timeout 300 env $(echo $1 | tr "~" " ") python bench.py --steps 20 --warmup 5 --no-cpu --no-check > gpurun_out/b_$TAG.json 2> gpurun_out/b_$TAG.err;
      python - "$1" <<'PY'
import json, sys; d=json.load(open('gpurun_out/b_' + __import__('os').environ.get('TAG','p') + '.json'))
r=d['roofline']; print(f"[{sys.argv[1]}] value {d['value']:.1f} e2e {d['e2e']['value']:.1f} frac {r['frac']:.3f} iso {r['frac_isolated']:.3f} spec_ms/step {d['spectral_ms_per_step']:.2f} seq {d['sequential_api']['value']:.1f} allocs {d['allocations_in_timed_region']}")
PY
}
for rep in 1 2 ${REPS3:+3}; do b "X=1"; for v in ${VARS:-}; do b "$v"; done; done
if [ -n "$C5" ]; then
  timeout 600 python bench.py --config 5 --steps 8 --warmup 2 --no-cpu --no-check --no-e2e > gpurun_out/b5_$TAG.json 2> gpurun_out/b5_$TAG.err
  python -c "import json; d=json.load(open('gpurun_out/b5_$TAG.json')); print('C5', round(d['value'],2), 'ms/step', round(d['ms_per_step'],2), 'spec', round(d['spectral_ms_per_step'],2), 'apply', round(d['apply_ms_per_step'],2), 'frac', round(d['roofline']['frac'],3))"
fi
if [ -n "$NCU" ]; then
  [ -n "$FULL" ] && { timeout 900 ncu --set full --clock-control none --import-source on -k regex:fmm_gemm -s 70 -c 7 \
     -o gpurun_out/gemm_$TAG -f python bench.py --steps 2 --warmup 3 --no-e2e --no-check --no-cpu > gpurun_out/ncu_gemm_$TAG.log 2>&1; echo "ncu rc=$?"; }
  # in-sequence DRAM bytes of every libsvd1 kernel (one replay pass per kernel, caches not flushed)
  timeout 900 ncu --cache-control none --clock-control none --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
     -k 'regex:fmm_gemm|fmm_ops|householder|passthrough|proj_|few_rows' --csv --log-file gpurun_out/dram_$TAG.csv \
     python bench.py --steps 2 --warmup 3 --no-e2e --no-check --no-cpu > /dev/null 2>&1; echo "ncu dram rc=$?"
fi
