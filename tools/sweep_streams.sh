cd $GRAFT_REPO_ROOT
for n in 1 2 3 4 6; do echo -n "streams=$n : "; python bench.py --streams $n --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-self-check --soak-seconds 0.5 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['value'],1), round(d['ms_per_step']*1e3,1))"; done
