"""Per-kernel DRAM bytes per launch (dram__bytes_read.sum + dram__bytes_write.sum)
from an `ncu --set full` report -> profiles/traffic.json (read by bench.py for
roofline.traffic).

    python tools/ncu_traffic.py profiles/r01_full.ncu-rep
"""
import csv
import io
import json
import re
import subprocess
import sys

NAMES = {"prep_kernel": "prep", "skut_tc3_f16_kernel": "skut_tc3_f16", "nn_bound_kernel": "nn_bound", "nn_select_kernel": "nn_select",
         "skut_tc3_kernel": "skut_tc3", "skut_tc2_kernel": "skut_tc", "skut_simt_kernel": "skut_simt",
         "head_kernel": "head"}


def main(rep, out="profiles/traffic.json"):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics",
                          "dram__bytes_read.sum,dram__bytes_write.sum"],
                         check=True, capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h = rows[0]
    ik, ir, iw = h.index("Kernel Name"), h.index("dram__bytes_read.sum"), h.index("dram__bytes_write.sum")
    units = rows[1]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    acc = {}
    for r in rows[2:]:
        m = re.search(r"(\w+_kernel)(<(\w+)>)?\(", r[ik])
        if not m:
            continue
        name = m.group(1)
        if name == "skut_tc3_kernel" and m.group(3) == "true":
            name = "skut_tc3_f16_kernel"
        if name == "nn_scan_kernel":  # launches alternate pass 1 / pass 2
            name = "nn_scan1" if acc.get("_scan_toggle", 0) == 0 else "nn_scan2"
            acc["_scan_toggle"] = 1 - acc.get("_scan_toggle", 0)
        else:
            name = NAMES.get(name, name)
        b = float(r[ir].replace(",", "")) * scale.get(units[ir], 1) + float(r[iw].replace(",", "")) * scale.get(units[iw], 1)
        acc.setdefault(name, []).append(b)
    acc.pop("_scan_toggle", None)
    res = {k: int(sum(v) / len(v)) for k, v in acc.items()}
    res["_note"] = (f"DRAM bytes (dram__bytes_read.sum + dram__bytes_write.sum) per launch from {rep} "
                    "(ncu --set full, C2 step, cold L2 per ncu replay)")
    with open(out, "w") as fh:
        json.dump(res, fh, indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main(*sys.argv[1:])
