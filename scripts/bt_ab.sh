CMD="python bench.py --budget backtrack:4 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-c4 --no-synthesize"
for v in base cap48 cap96 minb6 minb5 cap48minb6; do cp _variants/$v.so paper_2006_11851_b200/libpersyn_b200.so; echo "== $v"; $CMD 2>/dev/null | python -c "
import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);print(round(d['value'],1), round(d['kernels']['search_kernel']['ms_per_launch'],4))"; done
cp _variants/base.so paper_2006_11851_b200/libpersyn_b200.so
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:search --csv --log-file gpurun_out/bt4_launches.csv python bench.py --budget backtrack:4 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-c4 --no-synthesize > /dev/null 2>&1
grep -c search gpurun_out/bt4_launches.csv
