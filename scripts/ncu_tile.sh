set -e
TAG=${1:-t}
mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/plain_$TAG.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:search_tile -s 3 -c 1 -o gpurun_out/prof_search_$TAG $CMD > gpurun_out/ncu_full_$TAG.log 2>&1
echo done
