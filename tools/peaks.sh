#!/bin/bash
# FP64 peaks on the B200 box; clocks sampled during the run.
cd "$(dirname "$0")"
mkdir -p ../gpurun_out
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap --format=csv -lms 200 > ../gpurun_out/peaks_clocks.csv &
SMI=$!
./fp64_peak > ../gpurun_out/fp64_peak.jsonl 2>&1
python torch_fp64_mm.py >> ../gpurun_out/fp64_peak.jsonl 2>&1
kill $SMI
cat ../gpurun_out/fp64_peak.jsonl
