#!/bin/bash
# full GPU test suite + smoke + C3/C5 bench lines
cd "$(dirname "$0")/.."
export SVD1_PARITY_LOG=gpurun_out/parity_${TAG:-x}.jsonl
rm -f $SVD1_PARITY_LOG
( time timeout 2400 python -m pytest tests -m gpu -q -x 2>&1 | tail -6 ) 2>&1
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu > gpurun_out/b3_${TAG:-x}.json 2> gpurun_out/b3_${TAG:-x}.err
python -c "import json; d=json.load(open('gpurun_out/b3_${TAG:-x}.json')); r=d['roofline']; print('C3', round(d['value'],1), 'e2e', round(d['e2e']['value'],1), 'frac', round(r['frac'],3), 'iso', round(r['frac_isolated'],3), 'check', d['check'])"
timeout 600 python bench.py --config 5 --steps 8 --warmup 2 --no-cpu --no-check --no-e2e > gpurun_out/b5_${TAG:-x}.json 2> gpurun_out/b5_${TAG:-x}.err
python -c "import json; d=json.load(open('gpurun_out/b5_${TAG:-x}.json')); print('C5', round(d['value'],2), 'ms/step', round(d['ms_per_step'],2), 'frac', round(d['roofline']['frac'],3))"
