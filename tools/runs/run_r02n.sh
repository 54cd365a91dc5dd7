set -u
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -x -k "factored or high_fanout" > gpurun_out/pytest_fact.log 2>&1; echo "pytest $?"; tail -5 gpurun_out/pytest_fact.log
for c in c3 c4 c2 c1; do
extra="--no-oneshot"; [ $c = c3 ] && extra=""
timeout 900 python bench.py --config $c --steps 20 --no-cpu-baseline $extra > gpurun_out/bench_fact_$c.log 2>&1; echo "bench $?"
python - $c <<'PY'
import json,sys
d=json.loads(open(f'gpurun_out/bench_fact_{sys.argv[1]}.log').read().strip().splitlines()[-1])
f=dict(d['factored']); f.pop('note',None)
print(sys.argv[1], round(d['ms_per_step'],3), json.dumps(f))
if d.get('oneshot_e2e'): print(json.dumps(d['oneshot_e2e'])[:1500])
PY
done
