# The checked build: libmpsm_b200.so with the device-side bounds checks
# (MPSM_CHECK, -DMPSM_DEBUG_CHECKS=1) into build/checked/, and the parity
# suites run against it (MPSM_LIB), on the GPU box:
#   bash tools/checked_build.sh  -> gpurun_out/${R:-r02}_checked_pytest.log
# (compute-sanitizer is not available on this GPU pool; these checks cover the
# shared-memory staging, table, stage and output indexing of the hot kernels)
set -u
mkdir -p gpurun_out
python tools/variants.py checked:MPSM_DEBUG_CHECKS=1 > /dev/null
MPSM_LIB=$PWD/build/variants/checked/libmpsm_b200.so timeout 2400 python -m pytest -m gpu -x -q \
  tests/test_gpu_parity.py tests/test_gpu_random.py tests/test_gpu_contract.py tests/test_gpu_upload.py tests/test_gpu_dense_join.py \
  tests/test_gpu_distributed.py > gpurun_out/${R:-r02}_checked_pytest.log 2>&1
echo "checked rc=$?" | tee -a gpurun_out/${R:-r02}_checked_pytest.log
