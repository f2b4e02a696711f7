# run the default bench N times (separate outputs) and summarise
n=${1:-3}
for i in $(seq 1 $n); do
  python bench.py --steps 300 --warmup 20 --no-cpu-baseline > gpurun_out/rep_$i.txt 2>&1
  echo "run $i rc=$?"
done
python - $n <<'PY'
import json, sys
for i in range(1, int(sys.argv[1]) + 1):
    try:
        d = json.loads(open(f"gpurun_out/rep_{i}.txt").read().strip().splitlines()[-1])
        e = d["e2e"]
        print(i, d["value"], d["ms_per_step"], e["value"], e["p50_request_ms"], e["sync"]["value"], e["store"]["value"],
              d["open_loop"]["p50_request_ms"], d["open_loop"]["p99_request_ms"])
    except Exception as ex:
        print(i, "FAILED", ex, open(f"gpurun_out/rep_{i}.txt").read()[-800:])
PY
