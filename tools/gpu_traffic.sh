# DRAM bytes of the fused PCG kernel per launch (profiles/traffic.json) and a
# --set full capture of the current kernel at 128^3
set -x
mkdir -p gpurun_out/tr
NCU=/usr/local/cuda/bin/ncu
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors.sum
timeout 900 $NCU --metrics $M --clock-control none -k regex:pcg_tma -s 1 -c 1 --csv --log-file gpurun_out/tr/cfg2.csv python tools/profile_pcg.py --config 2 --iters 60 > gpurun_out/tr/cfg2.log 2>&1
timeout 900 $NCU --metrics $M --clock-control none -k regex:pcg_tma -s 1 -c 1 --csv --log-file gpurun_out/tr/cfg4.csv python tools/profile_pcg.py --config 4 --iters 30 > gpurun_out/tr/cfg4.log 2>&1
timeout 1200 $NCU --set full --import-source on --clock-control none -k regex:pcg_tma_kernel -s 1 -c 1 -o gpurun_out/tr/tma128_r02 python tools/profile_pcg.py --config 2 --iters 30 > gpurun_out/tr/full.log 2>&1
$NCU -i gpurun_out/tr/tma128_r02.ncu-rep --page raw --csv > gpurun_out/tr/tma128_r02_raw.csv 2>/dev/null
tail -n 2 gpurun_out/tr/*.log
