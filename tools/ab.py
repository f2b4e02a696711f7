"""A/B of experiment builds (build.build(variant=...)): alternates processes
over the given TAV2_LIB variants ("" = libtav2.so) at C2 and prints the
device-resident ms/step and SKUT kernel time of each run.
Usage: python tools/ab.py base e32 [--reps 3]"""
import json
import os
import subprocess
import sys

ONE = ("import sys, json; sys.path.insert(0, 'tools'); from sweep import point; "
       "print(json.dumps(point(1, 1000, 16384, (32, 96, 32, 32), steps=200, warmup=20)))")

if __name__ == "__main__":
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    reps = int(sys.argv[sys.argv.index("--reps") + 1]) if "--reps" in sys.argv else 3
    args = [a for a in args if a != str(reps)]
    res = {v: [] for v in args}
    for _ in range(reps):
        for v in args:
            env = dict(os.environ, TAV2_LIB="" if v == "base" else v)
            out = subprocess.run([sys.executable, "-c", ONE], env=env, capture_output=True, text=True)
            line = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
            if not line:
                print(v, "FAILED", out.stderr[-2000:])
                continue
            d = json.loads(line[-1])
            res[v].append((d["ms_per_step"], d["kernel_ms"].get("skut_tc3")))
            print(v, d["ms_per_step"], d["kernel_ms"], flush=True)
    for v, r in res.items():
        if r:
            print(f"{v}: ms/step min {min(a for a, _ in r):.4f} med {sorted(a for a, _ in r)[len(r) // 2]:.4f}"
                  f"  skut med {sorted(b for _, b in r)[len(r) // 2]}")
