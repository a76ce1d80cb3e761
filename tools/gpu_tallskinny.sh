# Tall-skinny start-vector kernels at 128^3 (ncu metrics per kernel, summarised
# by tools/ts_summary.py).  compute-sanitizer is closed on this GPU pool (runs
# under it left GPUs needing a reset; profiles/raw/r02_compute_sanitizer_refused.log),
# so the memory-safety evidence is mq_guard_check (tests/test_gpu_parity.py).
set -x
mkdir -p gpurun_out/ts
NCU=/usr/local/cuda/bin/ncu
KN='regex:k_(mdot|axpy_dots|comb|cspe_product|pod_|spmv_multi)'
MET=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed,launch__grid_size
python tools/ts_profile.py --config 2 --strategy cspe --steps 6 > gpurun_out/ts/run_cspe.log 2>&1
timeout 900 $NCU --kernel-name "$KN" --metrics $MET --clock-control none -c 400 --csv --log-file gpurun_out/ts/cfg2_cspe.csv python tools/ts_profile.py --config 2 --strategy cspe --steps 6 > gpurun_out/ts/ncu_cspe.log 2>&1
timeout 900 $NCU --kernel-name "$KN" --metrics $MET --clock-control none -c 400 --csv --log-file gpurun_out/ts/cfg2_pod.csv python tools/ts_profile.py --config 2 --strategy pod --steps 6 > gpurun_out/ts/ncu_pod.log 2>&1
python tools/ts_summary.py gpurun_out/ts/cfg2_cspe.csv gpurun_out/ts/cfg2_pod.csv
