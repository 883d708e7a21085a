set -e
mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/plain_small.log 2>&1
ncu --section SpeedOfLight --section Occupancy --section LaunchStats --section WarpStateStats --clock-control none -k regex:"mstep|penalty|rescore_windows|stats_partial|weights_kernel" -s 12 -c 6 --csv $CMD > gpurun_out/ncu_small.csv 2>&1
echo done
