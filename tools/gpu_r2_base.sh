set -x
nproc; lscpu | grep -E "Model name|^CPU\(s\)|Thread|Socket"; free -g | head -2
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python bench.py --steps 20 --warmup 5 > gpurun_out/r2_base_bench.json 2> gpurun_out/r2_base_bench.err
tail -c 3000 gpurun_out/r2_base_bench.json
timeout 300 python tools/time_oracle.py 3 > gpurun_out/r2_time_oracle.log 2>&1
cat gpurun_out/r2_time_oracle.log
