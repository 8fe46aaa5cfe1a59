# e2e host probe on the GPU box: what host the upload runs on, then the
# timeline of one end-to-end cfg2 join at several packing-thread counts
#   bash tools/e2e_host_probe.sh > gpurun_out/e2e_probe.log 2>&1
set -x
nproc; python -c "import os; print('cpu_count', os.cpu_count(), 'affinity', len(os.sched_getaffinity(0)))"
lscpu | head -30; numactl -H 2>/dev/null | head; free -g
for t in 16 12 8; do
  MPSM_UPLOAD_THREADS=$t timeout 300 python tools/e2e_timeline.py
done
