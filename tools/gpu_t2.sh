# T2: parity suites with the measured values logged (profiles/parity_r02.jsonl)
export SVD1_PARITY_LOG=gpurun_out/parity_r02.jsonl
rm -f $SVD1_PARITY_LOG
nproc
( time python -m pytest tests/test_gpu_parity.py tests/test_gpu_batch.py -q -x 2>&1 | tail -8 ) 2>&1
( time python -m pytest tests/test_gpu_fullsize.py -q -x --durations=10 2>&1 | tail -20 ) 2>&1
