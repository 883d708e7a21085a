set -e
mkdir -p gpurun_out
TAG=${1:-b1}
W=${2:-8}
CMD="python scripts/bench_brute.py 3 2 $W 1"
$CMD > gpurun_out/plain_brute_$TAG.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:brute --csv $CMD > gpurun_out/brute_launches_$TAG.csv 2>&1
ncu --set full --clock-control none --import-source on -k regex:brute_mma -s 1 -c 1 -o gpurun_out/prof_brute_$TAG $CMD > gpurun_out/ncu_brute_$TAG.log 2>&1
echo done
