# Full ncu capture (with source) of one kernel of the bench command: bash scripts/ncu_kernel_full.sh REGEX TAG [SKIP]
set -e
mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-c4 --no-synthesize"
$CMD > gpurun_out/plain_$2.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"$1" -s ${3:-4} -c 1 -o gpurun_out/prof_$2 $CMD > gpurun_out/ncu_full_$2.log 2>&1
echo done
