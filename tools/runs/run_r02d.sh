set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -x -k "bmt_hop or cuda_graph or pinned or full_size" > gpurun_out/pytest_sel.log 2>&1
echo "pytest sel exit $?"; tail -3 gpurun_out/pytest_sel.log
for c in c0 c1; do timeout 300 python bench.py --config $c --steps 50 --no-cpu-baseline --no-oneshot > gpurun_out/bench_$c.log 2>&1; echo "bench $c $?"; tail -1 gpurun_out/bench_$c.log | cut -c1-200; done
for c in c3 c4; do for pf in 1 0; do for eo in f32 f64; do
  [ $pf = 0 ] && [ $eo = f64 ] && continue
  timeout 900 python bench.py --config $c --steps 20 --no-cpu-baseline --no-oneshot --option prefetch=$pf --e2e-out $eo > gpurun_out/bench_${c}_pf${pf}_$eo.log 2>&1
  echo "bench $c prefetch=$pf e2e=$eo $?"; tail -1 gpurun_out/bench_${c}_pf${pf}_$eo.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],4), {k:v['mean_launch_ms'] for k,v in d['kernels'].items()}, 'e2e', round(d['e2e']['ms_per_step'],3))"
done; done; done
