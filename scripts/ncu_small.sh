# Section-level ncu of the EM step's small kernels (run after the plain command exited 0).
set -e
mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/plain_small.log 2>&1
ncu --section SpeedOfLight --section Occupancy --section LaunchStats --section WarpStateStats \
    --section MemoryWorkloadAnalysis --section ComputeWorkloadAnalysis --clock-control none \
    -k regex:"mstep|penalty|rescore|stats_partial|weights_kernel|eff_gather|project2" -s 16 -c 8 --csv \
    $CMD > gpurun_out/ncu_small.csv 2>&1
echo done
