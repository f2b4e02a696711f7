# A/B of library variants on the default bench (alternating runs):
#   bash tools/ab_bench.sh base pv
for i in 1 2 3; do
  for v in "$@"; do
    TAV2_LIB=${v#base} timeout 300 python bench.py --steps 300 --warmup 20 --no-cpu-baseline > gpurun_out/ab_$v.txt 2>&1
    python - "$v" <<'PY'
import json, sys
v = sys.argv[1]
d = json.loads(open(f"gpurun_out/ab_{v}.txt").read().strip().splitlines()[-1])
k = d["kernels"]
sk = [x for x in k if x.startswith("skut")][0]
print(f"{v:8s} value {d['value']:.0f} step {d['ms_per_step']:.4f} {sk} {k[sk]['ms_per_launch']:.4f} e2e {d['e2e']['value']:.0f}")
PY
  done
done
