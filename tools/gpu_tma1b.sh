# one-barrier TMA kernel adoption check: GPU suite, headline bench both ways, traffic + full capture
set -x
mkdir -p gpurun_out/t1 gpurun_out/tr
python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/t1/tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/t1/tests.log
for rep in 1 2; do
  MQ_PCG_SYNC=2 python bench.py --skip-secondary --skip-cpu --skip-cfg4 --steps 20 > gpurun_out/t1/bench_two_$rep.log 2>&1
  python bench.py --skip-secondary --skip-cpu --skip-cfg4 --steps 20 > gpurun_out/t1/bench_one_$rep.log 2>&1
done
NCU=/usr/local/cuda/bin/ncu
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors.sum
timeout 900 $NCU --metrics $M --clock-control none -k regex:pcg_tma -s 1 -c 1 --csv --log-file gpurun_out/tr/cfg2_tma1.csv python tools/profile_pcg.py --config 2 --iters 60 > gpurun_out/tr/cfg2_tma1.log 2>&1
timeout 1200 $NCU --set full --import-source on --clock-control none -k regex:pcg_tma1_kernel -s 1 -c 1 -o gpurun_out/tr/tma1_128 python tools/profile_pcg.py --config 2 --iters 30 > gpurun_out/tr/full_tma1.log 2>&1
$NCU -i gpurun_out/tr/tma1_128.ncu-rep --page raw --csv > gpurun_out/tr/tma1_128_raw.csv 2>/dev/null
tail -n 3 gpurun_out/t1/tests.log
for f in gpurun_out/t1/bench_*.log; do echo $f; grep '^{' $f | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']
print(d['value'], d['e2e']['value'], r['us_per_iteration'], r['frac'], r.get('kernel'), d['clocks']['sm_mhz'])"; done
