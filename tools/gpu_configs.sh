#!/bin/bash
# One gpurun call: bench.py for every BASELINE config (C3 last, with cpu baseline).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
for c in 1 2 4 5; do
  timeout 600 python bench.py --config $c --steps 8 --warmup 3 --no-cpu > gpurun_out/bench_c$c.json 2> gpurun_out/bench_c$c.err
  echo "C$c: $(python tools/bench_brief.py gpurun_out/bench_c$c.json 2>&1 | cut -c1-150)"
done
timeout 900 python bench.py > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
echo "C3: $(python tools/bench_brief.py gpurun_out/bench_c3.json 2>&1 | cut -c1-150)"
