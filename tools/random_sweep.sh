# larger randomised GPU sweep vs the CPU oracle (GPU box): SEED / CASES override
mkdir -p gpurun_out
MPSM_RANDOM_SEED=${SEED:-7} MPSM_RANDOM_CASES=${CASES:-600} timeout 3000 python -m pytest tests/test_gpu_random.py -q -x 2>&1 | tail -15 | tee gpurun_out/random_sweep_${SEED:-7}.log
