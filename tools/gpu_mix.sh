# Mixed brick chunking A/B (MQ_BRICK_MIX): per-iteration time at 128^3, the
# %smid census, the PCG parity tests and the headline bench both ways
set -x
mkdir -p gpurun_out/mix
for rep in 1 2; do
  for m in 0 1; do
    echo "== mix$m rep $rep" >> gpurun_out/mix/ab.log
    MQ_BRICK_MIX=$m MQ_PCG_TRACE=1 MQ_PCG_VERBOSE=1 python tools/profile_pcg.py --config 2 --iters 200 >> gpurun_out/mix/ab.log 2>&1
  done
done
grep -E "^==|us/it|per-iteration" gpurun_out/mix/ab.log
python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -x -k "pcg or (config_fields and cfg2) or guard or transient" > gpurun_out/mix/tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/mix/tests.log
tail -n 2 gpurun_out/mix/tests.log
for rep in 1 2; do
  for m in 0 1; do
    MQ_BRICK_MIX=$m python bench.py --skip-secondary --skip-cpu --skip-cfg4 --steps 20 > gpurun_out/mix/bench_${m}_${rep}.log 2>&1
    grep '^{' gpurun_out/mix/bench_${m}_${rep}.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']
print('mix$m', d['value'], d['e2e']['value'], r['us_per_iteration'], r['frac'], d['clocks']['sm_mhz'])"
  done
done
