# quick GPU check: -m gpu tests + a short bench (no CPU baseline)
set -o pipefail
python -m paper_2506_02267_b200.build >/dev/null
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
timeout 300 python bench.py --steps 100 --warmup 10 --no-cpu-baseline > gpurun_out/bench_quick.txt 2>&1
python - <<'PY'
import json
l=[x for x in open("gpurun_out/bench_quick.txt") if x.startswith("{")]
if not l: print(open("gpurun_out/bench_quick.txt").read()[-3000:]); raise SystemExit
d=json.loads(l[-1])
print("value", d["value"], "e2e", d["e2e"]["value"], "ms", d["ms_per_step"])
print({k: v["ms_per_launch"] for k, v in d["kernels"].items()})
print("roofline", d["roofline"]["frac"])
PY
