for i in 1 2; do for v in "" noorder; do
TAV2_LIB=$v python - <<'PY'
import sys, json, os
sys.path.insert(0, "tools"); sys.path.insert(0, ".")
from sweep import point
for k in (128, 256):
    d = point(1, 1000, 16384, (32, k, 32, 32), steps=100, warmup=10)
    print(os.environ.get("TAV2_LIB") or "base", k, d["ms_per_step"], {a: b for a, b in d["kernel_ms"].items() if a.startswith("skut")})
PY
done; done
