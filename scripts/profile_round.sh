# One round's measurement evidence: bench line, ncu launch list of the same
# command, and full ncu captures of the top kernels (each after the plain run
# of its command exited 0).  Usage: bash scripts/profile_round.sh TAG
set -e
TAG=${1:-r2}
mkdir -p gpurun_out
python bench.py --steps 20 --warmup 5 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-c4 --no-synthesize"
$CMD > gpurun_out/plain_$TAG.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv $CMD > gpurun_out/ncu_launch_$TAG.log 2>&1
# -s: skip the index build's / priming's launches of the same name
ncu --set full --clock-control none --import-source on -k regex:search_tile -s 4 -c 1 -o gpurun_out/prof_search_$TAG $CMD > gpurun_out/ncu_full_$TAG.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:project_tc -s 2 -c 1 -o gpurun_out/prof_projtc_$TAG $CMD > gpurun_out/ncu_full_projtc_$TAG.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:mstep -s 2 -c 1 -o gpurun_out/prof_mstep_$TAG $CMD > gpurun_out/ncu_full_mstep_$TAG.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:make_digits -s 2 -c 1 -o gpurun_out/prof_digits_$TAG $CMD > gpurun_out/ncu_full_digits_$TAG.log 2>&1
echo done
