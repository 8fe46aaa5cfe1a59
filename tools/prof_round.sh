# profiling pass of one round (run on the GPU box from the repo root): bench line, ncu launch list, ncu --set full of the scatter launches of one step
set -x
mkdir -p gpurun_out
R=${R:-r01c}
timeout 600 python bench.py > gpurun_out/${R}_bench.log 2>&1 || exit 1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${R}_launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/${R}_ncu_launch.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_scatter -c 6 -o gpurun_out/${R}_scatter_step python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/${R}_ncu_scatter.log 2>&1
echo done
