mkdir -p gpurun_out/bab
for rep in 1 2; do
for lib in $LIBS; do
  if [ $lib = intree ]; then python bench.py --skip-secondary --skip-cpu --skip-cfg4 --steps 20 > gpurun_out/bab/b.log 2>&1; else MQ_LIB_PATH=$lib python bench.py --skip-secondary --skip-cpu --skip-cfg4 --steps 20 > gpurun_out/bab/b.log 2>&1; fi
  grep '^{' gpurun_out/bab/b.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']
print('$lib', d['value'], d['e2e']['value'], r['us_per_iteration'], r['frac'], r['pcg_share_of_step'], d['ms_per_step'], d['clocks']['sm_mhz'])"
done
done
