# T3: sliced spectral phase (emulated ranks, NCCL world-1) + regression of the parity suites
python -m pytest tests/test_gpu_ranks.py -x -q 2>&1 | tail -8
python -m pytest tests/test_gpu_parity.py tests/test_gpu_batch.py tests/test_gpu_thin.py -x -q 2>&1 | tail -4
python bench.py --steps 20 --warmup 5 --no-cpu > gpurun_out/r2_t3_bench.json 2> gpurun_out/r2_t3_bench.err
python - <<'PY'
import json; d=json.load(open('gpurun_out/r2_t3_bench.json'))
print("value", d['value'], "e2e", d['e2e']['value'], "frac", d['roofline']['frac'], "allocs", d['allocations_in_timed_region'])
PY
