#!/bin/bash
# run-to-run variance of the C3 bench line: value, e2e, host phases, per-update windows
cd "$(dirname "$0")/.."
for i in $(seq 1 ${NREP:-8}); do
  timeout 300 env ${ENVV:-X=1} python bench.py --steps 20 --warmup 5 --no-cpu --no-check > gpurun_out/var.json 2>/dev/null
  python - <<'PY'
import json; d=json.load(open('gpurun_out/var.json'))
print(f"value {d["value"]:.1f} e2e {d["e2e"]["value"]:.1f} reps {[round(x) for x in d["e2e"].get("repetitions", [])]} seq {d['sequential_api']['value']:.1f} host {[round(x,2) for x in d['host_phase_ms']]} clocks {d['clocks']['sm_mhz']} {d['clocks']['reasons']}")
PY
done
