# Full GPU suite + default bench + launch list of the bench (round-end evidence)
set -x
mkdir -p gpurun_out/full
python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/full/tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/full/tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/full/smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/full/smoke.log
python bench.py > gpurun_out/full/bench.log 2>&1
echo "bench rc=$?" >> gpurun_out/full/bench.log
tail -n 3 gpurun_out/full/tests.log gpurun_out/full/smoke.log
tail -c 1500 gpurun_out/full/bench.log
# launch list of the headline leg (per-launch times are cold-cache and serialised: shares only)
timeout 1200 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/full/launches.csv python bench.py --steps 3 --warmup 3 --skip-secondary --skip-cpu --skip-cfg4 \
  > gpurun_out/full/ncu.log 2>&1
echo "ncu rc=$?"
