# T1 check: batch tests + allocation test, then the driver-like bench (20 steps, 5 warm-up)
python -m pytest tests/test_gpu_batch.py -x -q 2>&1 | tail -5
python bench.py --steps 20 --warmup 5 --no-cpu > gpurun_out/r2_t1_bench.json 2> gpurun_out/r2_t1_bench.err
python - <<'PY'
import json; d=json.load(open('gpurun_out/r2_t1_bench.json'))
print("value", d['value'], "e2e", d['e2e']['value'], "frac", d['roofline']['frac'], "iso", d['roofline']['frac_isolated'],
      "allocs", d['allocations_in_timed_region'], "levels", d['check']['fmm_levels'], "host", d['host_phase_ms'], "seq", d['sequential_api']['value'])
PY
