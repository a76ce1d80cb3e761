# Steady-state profile of the configs[2] step kernels (POD-30 rings full):
# launch list of 25 steps and a metrics pass over the POD / combination
# kernels of the last steps.
set -x
mkdir -p gpurun_out/pod
NCU=/usr/local/cuda/bin/ncu
python tools/ts_profile.py --config 2 --strategy pod --steps 25 > gpurun_out/pod/run.log 2>&1
timeout 1200 $NCU --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/pod/launches.csv \
  python tools/ts_profile.py --config 2 --strategy pod --steps 25 > gpurun_out/pod/ncu_launch.log 2>&1
KN='regex:k_(comb|pod_|spmv_multi)'
MET=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,launch__grid_size,launch__registers_per_thread,sm__warps_active.avg.pct_of_peak_sustained_active
timeout 1200 $NCU --kernel-name "$KN" -s 800 -c 200 --metrics $MET --clock-control none --csv --log-file gpurun_out/pod/pod_metrics.csv \
  python tools/ts_profile.py --config 2 --strategy pod --steps 25 > gpurun_out/pod/ncu_pod.log 2>&1
tail -2 gpurun_out/pod/*.log
timeout 900 $NCU --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/pod/bench_launches.csv \
  python bench.py --steps 3 --warmup 3 --skip-secondary --skip-cpu --skip-cfg4 > gpurun_out/pod/ncu_bench.log 2>&1
