# Quick GPU check: a parity subset (-k expression in $1), then a short bench
set -x
mkdir -p gpurun_out/q
python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "$1" > gpurun_out/q/tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/q/tests.log
python bench.py --skip-secondary --skip-cpu --skip-cfg4 --steps ${2:-20} > gpurun_out/q/bench.log 2>&1
tail -n 3 gpurun_out/q/tests.log
python - <<'PY'
import json
l = [x for x in open("gpurun_out/q/bench.log") if x.startswith("{")]
if l:
    d = json.loads(l[-1]); r = d["roofline"]
    print("value", d["value"], "e2e", d["e2e"]["value"], "us/it", r["us_per_iteration"], "frac", r["frac"],
          "pcg_share", r["pcg_share_of_step"], "clocks", d["clocks"])
else:
    print(open("gpurun_out/q/bench.log").read()[-3000:])
PY
