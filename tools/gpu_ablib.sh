# A/B of in-tree library vs variants: per-iteration time (configs[2] and 256^3),
# PCG/slab GPU tests on the in-tree library, headline bench for each.
# LIBS="variants/head.so intree" TESTK="..." bash tools/gpu_ablib.sh
mkdir -p gpurun_out/ablib
run() { if [ $1 = intree ]; then shift; "$@"; else l=$1; shift; MQ_LIB_PATH=$l "$@"; fi; }
for rep in 1 2; do
  for lib in $LIBS; do
    for cfg in ${CFGS:-2}; do
      echo "== $lib cfg$cfg rep $rep" >> gpurun_out/ablib/ab.log
      run $lib env MQ_PCG_TRACE=1 python tools/profile_pcg.py --config $cfg --iters ${ITERS:-200} >> gpurun_out/ablib/ab.log 2>&1
    done
  done
done
grep -E "^==|us/it|per-iteration" gpurun_out/ablib/ab.log
if [ -n "$TESTK" ]; then
  timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "$TESTK" > gpurun_out/ablib/tests.log 2>&1
  echo "tests rc=$?" >> gpurun_out/ablib/tests.log
  tail -n 2 gpurun_out/ablib/tests.log
fi
if [ -n "$BENCH" ]; then
  for lib in $LIBS; do
    run $lib python bench.py --skip-secondary --skip-cpu --skip-cfg4 --steps 20 > gpurun_out/ablib/bench_$(basename $lib .so).log 2>&1
    grep '^{' gpurun_out/ablib/bench_$(basename $lib .so).log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']
print('$lib', d['value'], d['e2e']['value'], r['us_per_iteration'], r['frac'], d['clocks']['sm_mhz'])"
  done
fi
