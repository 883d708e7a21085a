for jc in 24 48; do PERSYN_PROJ_JC=$jc python bench.py --no-cpu-baseline --no-e2e --steps 5 > gpurun_out/b_$jc.log 2>&1; python -c "import json;d=json.loads(open('gpurun_out/b_$jc.log').read().strip().splitlines()[-1]);print($jc, d['kernels']['project_kernel']['ms_per_launch'])"; done
PERSYN_PROJECT2=1 python bench.py --no-cpu-baseline --no-e2e --steps 5 > gpurun_out/b_p2.log 2>&1; python -c "import json;d=json.loads(open('gpurun_out/b_p2.log').read().strip().splitlines()[-1]);print('p2', d['kernels']['project_kernel']['ms_per_launch'])"
bash scripts/ncu_kernel_full.sh project3 pj3 3
