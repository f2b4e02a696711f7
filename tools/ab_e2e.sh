# e2e A/B of library variants (graphs on/off): bash tools/ab_e2e.sh base pv
for g in 0 1; do
for v in "$@"; do
  TAV2_NO_GRAPH=$g TAV2_LIB=$v python bench.py --steps 300 --warmup 20 --no-cpu-baseline > gpurun_out/abe_$v.txt 2>&1
  python - "$v" "$g" <<'PY'
import json, sys
v, g = sys.argv[1], sys.argv[2]
d = json.loads(open(f"gpurun_out/abe_{v}.txt").read().strip().splitlines()[-1])
e = d["e2e"]
print(f"{v:6s} nograph={g} value {d['value']:.0f} e2e {e['value']:.0f} p50 {e['p50_request_ms']} sync {e['sync']['value']:.0f} "
      f"store {e['store']['value']:.0f} open p50 {d['open_loop']['p50_request_ms']}")
PY
done
done
