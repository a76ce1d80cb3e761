# A/B with environment: tools/gpu_ab_env.sh CONFIG ITERS "label|variant|ENV=.. ENV2=.." ...
cfg=$1; iters=$2; shift 2
mkdir -p gpurun_out/ab
for rep in 1 2; do
  for spec in "$@"; do
    label=${spec%%|*}; rest=${spec#*|}; v=${rest%%|*}; envs=${rest#*|}
    if [ "$v" = base ]; then lib=""; else lib="MQ_LIB_PATH=variants/$v.so"; fi
    echo "== $label rep $rep" >> gpurun_out/ab/abe.log
    env $lib $envs MQ_PCG_TRACE=1 MQ_PCG_VERBOSE=1 python tools/profile_pcg.py --config $cfg --iters $iters >> gpurun_out/ab/abe.log 2>&1
  done
done
grep -E "^==|us/it|per-iteration|CTAs per SM" gpurun_out/ab/abe.log
