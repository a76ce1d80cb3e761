mkdir -p gpurun_out/s2
python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/s2/tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/s2/tests.log
python bench.py --skip-secondary --skip-cpu --steps 10 > gpurun_out/s2/bench.log 2>&1
tail -2 gpurun_out/s2/tests.log
grep '^{' gpurun_out/s2/bench.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; s=d['cfg4_sharded']; s1=d['cfg4_steps_1gpu']
print('value', d['value'], 'us/it', r['us_per_iteration'], 'frac', r['frac'])
print('sharded', s.get('value'), s.get('frac_of_N_hbm'), s.get('error'), 'one-context', s1['value'])"
