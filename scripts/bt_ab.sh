# Budget searches on the bench stage (reference tree): bash scripts/bt_ab.sh
for b in backtrack:1 backtrack:4 backtrack:8 backtrack:16 backtrack:64; do echo "== $b"; python bench.py --budget $b --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-c4 --no-synthesize 2>/dev/null | python -c "
import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);k=d['kernels'];print(round(d['value'],1), 'search', round(k['search_kernel']['ms_per_launch'],4), 'proj', round(k['project_kernel']['ms_per_launch'],4), 'energy', d['energy_last'])"; done
