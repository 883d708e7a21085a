set -x
bash scripts/profile_round.sh r2g
python bench.py --budget backtrack:4 --steps 20 --warmup 5 > gpurun_out/bench_bt4_r2g.json 2> gpurun_out/bench_bt4_r2g.err
BT="python bench.py --budget backtrack:4 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-c4 --no-synthesize"
ncu --set full --clock-control none --import-source on -k regex:search_backtrack_group -s 2 -c 1 -o gpurun_out/prof_btgroup_r2g $BT > gpurun_out/ncu_btgroup_r2g.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bt4_r2g.csv $BT > /dev/null 2>&1
for c in 1 3 4; do python scripts/run_synthesize.py $c > gpurun_out/synth_cfg${c}_r2g.json 2>/dev/null; done
python scripts/run_synthesize.py 3 10 backtrack:4 reference > gpurun_out/synth_cfg3_bt4ref_r2g.json 2>/dev/null
python scripts/run_synthesize.py 3 10 backtrack:4 device > gpurun_out/synth_cfg3_bt4dev_r2g.json 2>/dev/null
python scripts/run_synthesize.py 1 5 backtrack:4 reference > gpurun_out/synth_cfg1_bt4ref_r2g.json 2>/dev/null
echo done
