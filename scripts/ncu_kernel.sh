# ncu --set full of one kernel of the bench command: bash scripts/ncu_kernel.sh TAG REGEX
set -e
TAG=${1:-k}
RE=${2:-project}
mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/plain_$TAG.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:$RE -s 3 -c 1 -o gpurun_out/prof_$TAG $CMD > gpurun_out/ncu_$TAG.log 2>&1
echo done
