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
