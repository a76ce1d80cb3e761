# A/B of PCG kernel variants: tools/gpu_ab.sh CONFIG ITERS variantA variantB ...
# ("base" = the in-tree library); per-phase trace of CTA 0 for each.
cfg=$1; iters=$2; shift 2
mkdir -p gpurun_out/ab
for rep in 1 2 3; do
  for v in "$@"; do
    if [ "$v" = base ]; then lib=""; else lib="MQ_LIB_PATH=variants/$v.so"; fi
    echo "== $v rep $rep" >> gpurun_out/ab/ab.log
    env $lib MQ_PCG_TRACE=1 python tools/profile_pcg.py --config $cfg --iters $iters >> gpurun_out/ab/ab.log 2>&1
  done
done
grep -E "^==|us/it|per-iteration" gpurun_out/ab/ab.log
