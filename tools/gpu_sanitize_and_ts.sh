set -x
mkdir -p gpurun_out/san gpurun_out/ts
CS=/usr/local/cuda/bin/compute-sanitizer
SM='import __graft_entry__ as g; g.smoke()'
timeout 900 $CS --tool memcheck --print-limit 30 python -c "$SM" > gpurun_out/san/memcheck_smoke.log 2>&1; echo rc=$? >> gpurun_out/san/memcheck_smoke.log
timeout 600 $CS --tool synccheck --print-limit 30 python -c "$SM" > gpurun_out/san/synccheck_smoke.log 2>&1; echo rc=$? >> gpurun_out/san/synccheck_smoke.log
timeout 900 $CS --tool racecheck --racecheck-report analysis --print-limit 30 python -c "$SM" > gpurun_out/san/racecheck_smoke.log 2>&1; echo rc=$? >> gpurun_out/san/racecheck_smoke.log
timeout 600 $CS --tool initcheck --print-limit 30 python -c "$SM" > gpurun_out/san/initcheck_smoke.log 2>&1; echo rc=$? >> gpurun_out/san/initcheck_smoke.log
timeout 1500 $CS --tool memcheck --print-limit 30 python -m pytest -x -q -p no:cacheprovider tests/test_gpu_parity.py -m gpu -k "resident_pcg_semantics or pcg_kernel_variants_agree or fused_slab_pcg_on_one_gpu or cspe_strategy_parity or pod_strategy_parity or single_step_api" > gpurun_out/san/memcheck_tests.log 2>&1; echo rc=$? >> gpurun_out/san/memcheck_tests.log
NCU=/usr/local/cuda/bin/ncu
KN='regex:k_(mdot|axpy_dots|comb|cspe_product|pod_push|pod_galerkin|pod_basis|spmv_multi)'
MET=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed,launch__grid_size
python tools/ts_profile.py --config 2 --strategy cspe --steps 6 > gpurun_out/ts/run_cspe.log 2>&1
timeout 900 $NCU --kernel-name "$KN" --metrics $MET --clock-control none -c 400 --csv --log-file gpurun_out/ts/cfg2_cspe.csv python tools/ts_profile.py --config 2 --strategy cspe --steps 6 > gpurun_out/ts/ncu_cspe.log 2>&1
timeout 900 $NCU --kernel-name "$KN" --metrics $MET --clock-control none -c 400 --csv --log-file gpurun_out/ts/cfg2_pod.csv python tools/ts_profile.py --config 2 --strategy pod --steps 6 > gpurun_out/ts/ncu_pod.log 2>&1
tail -3 gpurun_out/san/*.log
