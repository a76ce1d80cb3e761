# ncu --set full capture of the one-barrier PCG kernel on the configs[2] grid
# (one launch of 30 iterations), raw page and source-level stalls.
set -x
mkdir -p gpurun_out/ncu
python tools/profile_pcg.py --config 2 --iters 30 > gpurun_out/ncu/plain.log 2>&1
timeout 1500 /usr/local/cuda/bin/ncu --set full --import-source on --clock-control none -k regex:pcg_tma1_kernel -s 1 -c 1 \
  -o gpurun_out/ncu/tma1_128 python tools/profile_pcg.py --config 2 --iters 30 > gpurun_out/ncu/ncu.log 2>&1
/usr/local/cuda/bin/ncu -i gpurun_out/ncu/tma1_128.ncu-rep --page raw --csv > gpurun_out/ncu/tma1_128_raw.csv 2>/dev/null
/usr/local/cuda/bin/ncu -i gpurun_out/ncu/tma1_128.ncu-rep --page source --csv --print-source sass > gpurun_out/ncu/tma1_128_src.csv 2>/dev/null
/usr/local/cuda/bin/ncu -i gpurun_out/ncu/tma1_128.ncu-rep --page details --csv > gpurun_out/ncu/tma1_128_details.csv 2>/dev/null
ls -la gpurun_out/ncu
