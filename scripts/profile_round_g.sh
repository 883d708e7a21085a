set -x
TAG=${1:-r2h}
bash scripts/profile_round.sh $TAG
python bench.py --budget backtrack:4 --steps 20 --warmup 5 > gpurun_out/bench_bt4_$TAG.json 2> gpurun_out/bench_bt4_$TAG.err
BT="python bench.py --budget backtrack:4 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-c4 --no-synthesize"
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:group_kernel.*96, .bool.1" -s 2 -c 1 -o gpurun_out/prof_btgroup_$TAG $BT > gpurun_out/ncu_btgroup_$TAG.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bt4_$TAG.csv $BT > /dev/null 2>&1
for c in 1 3 4; do python scripts/run_synthesize.py $c > gpurun_out/synth_cfg${c}_$TAG.json 2>/dev/null; done
python scripts/run_synthesize.py 3 10 backtrack:4 reference > gpurun_out/synth_cfg3_bt4ref_$TAG.json 2>/dev/null
python scripts/run_synthesize.py 3 10 backtrack:4 device > gpurun_out/synth_cfg3_bt4dev_$TAG.json 2>/dev/null
python scripts/run_synthesize.py 1 5 backtrack:4 reference > gpurun_out/synth_cfg1_bt4ref_$TAG.json 2>/dev/null
echo done
python scripts/run_synthesize.py 4 10 backtrack:4 reference > gpurun_out/synth_cfg4_bt4ref_$TAG.json 2>/dev/null
python scripts/budget_cfg2.py > gpurun_out/cfg2_budgets_$TAG.jsonl 2>/dev/null
python scripts/bench_cfg2.py > gpurun_out/cfg2_$TAG.json 2>/dev/null
