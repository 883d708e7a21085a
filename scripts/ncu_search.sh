set -e
mkdir -p gpurun_out
TAG=${1:-v2}
CMD="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/plain_$TAG.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:search_ -s 1 -c 1 -o gpurun_out/prof_search_$TAG $CMD > gpurun_out/ncu_full_$TAG.log 2>&1
echo done
