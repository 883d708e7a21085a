# One round's measurement evidence: bench line, ncu launch list of the same
# command, and full ncu captures of the top kernels (each after the plain run
# of its command exited 0).  Usage: bash scripts/profile_round.sh TAG
set -e
TAG=${1:-r1}
mkdir -p gpurun_out
python bench.py --steps 10 --warmup 3 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/plain_$TAG.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv $CMD > gpurun_out/ncu_launch_$TAG.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:search_tile -s 3 -c 1 -o gpurun_out/prof_search_$TAG $CMD > gpurun_out/ncu_full_$TAG.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:project2 -s 3 -c 1 -o gpurun_out/prof_project_$TAG $CMD > gpurun_out/ncu_full_project_$TAG.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:mstep -s 3 -c 1 -o gpurun_out/prof_mstep_$TAG $CMD > gpurun_out/ncu_full_mstep_$TAG.log 2>&1
BCMD="python scripts/bench_brute.py 3 2 8 1"
$BCMD > gpurun_out/plain_brute_$TAG.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:brute_mma -s 1 -c 1 -o gpurun_out/prof_brute_$TAG $BCMD > gpurun_out/ncu_brute_$TAG.log 2>&1
echo done
