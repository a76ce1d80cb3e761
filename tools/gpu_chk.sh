# quick check: config-0/1 PCG tests against a variant library and the in-tree one
mkdir -p gpurun_out/chk
for lib in ${LIBS:-variants/head.so intree}; do
  echo "== lib=$lib" >> gpurun_out/chk/log
  if [ $lib = intree ]; then pre=""; else pre="MQ_LIB_PATH=$lib"; fi
  env $pre timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -x -k "test_pcg_matches_oracle or test_pcg_kernel_variants" >> gpurun_out/chk/log 2>&1
  echo "rc=$?" >> gpurun_out/chk/log
done
MQ_PCG_VERBOSE=1 python -c "
from paper_1611_06721_b200 import configs as C
from paper_1611_06721_b200.device import DeviceGrid
g=DeviceGrid(C.make_problem(0)); print(g.pcg_kernel())
" >> gpurun_out/chk/log 2>&1
grep -E "==|rc=|passed|failed|Error|pcg_" gpurun_out/chk/log | head -30
