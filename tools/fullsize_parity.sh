# full-size parity run (GPU box, repo root): tests/test_gpu_fullsize.py at
# BASELINE.json configs 2, 3 (multiplicity 16) and 4; log to gpurun_out/
mkdir -p gpurun_out
MPSM_FULLSIZE=1 timeout 2400 python -m pytest tests/test_gpu_fullsize.py -v -rA --durations=0 2>&1 | tee gpurun_out/fullsize_parity.log | tail -25
