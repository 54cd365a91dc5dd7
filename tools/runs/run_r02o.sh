set -u
mkdir -p gpurun_out
for c in c3 c4; do for t in 2 3 4 6 10; do
timeout 900 python bench.py --config $c --steps 10 --no-cpu-baseline --no-oneshot --factor-above $t > gpurun_out/bench_fa_${c}_$t.log 2>&1
python - $c $t <<'PY'
import json,sys
d=json.loads(open(f'gpurun_out/bench_fa_{sys.argv[1]}_{sys.argv[2]}.log').read().strip().splitlines()[-1])
f=dict(d['factored']); f.pop('note',None); f.pop('unit',None)
print(sys.argv[1], 'T=',sys.argv[2], json.dumps(f))
PY
done; done
