# round-2 evidence pass on the GPU box (after the commands exit 0 without ncu):
#   R=r02 bash tools/prof_round2.sh
# ncu launch list of one bench step, --set full captures of the merge, the
# scatter launches of one step (DRAM traffic), and the non-headline kernels
set -x
mkdir -p gpurun_out
R=${R:-r02}
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${R}_launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/${R}_ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_merge -c 1 -o gpurun_out/${R}_merge_step python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/${R}_ncu_merge.log 2>&1
timeout 1200 ncu --set full --clock-control none -k regex:k_scatter -c 6 -o gpurun_out/${R}_scatter_step python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/${R}_ncu_scatter.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_radix_hist|k_onesweep|k_scatter_ws|k_check_sorted" -c 6 -o gpurun_out/${R}_other python tools/kernels_once.py > gpurun_out/${R}_ncu_other.log 2>&1
echo done
