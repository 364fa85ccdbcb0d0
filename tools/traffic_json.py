"""Write profiles/ncu_traffic.json from `ncu --set full` captures (one launch each).

    python tools/traffic_json.py gpurun_out/r01c  [round tag]

Reads every <dir>/full_<workload>_<kernel>.ncu-rep, sums dram__bytes_read.sum +
dram__bytes_write.sum of the captured launch and records it next to the kernel name,
keyed by workload and kernel class (what bench.py reports as roofline.traffic).
"""
import csv
import glob
import io
import json
import os
import subprocess
import sys

CLASS = {"k_update_tma": "update", "k_update_pair": "update", "k_sweep": "forward", "k_hub_partial_tma": "hub_partial"}
UNITS = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def launch_bytes(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    if len(rows) < 3:
        return None
    head, units, vals = rows[0], rows[1], rows[2]
    tot = 0.0
    for key in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
        i = head.index(key)
        tot += float(vals[i].replace(",", "")) * UNITS.get(units[i], 1)
    it = head.index("gpu__time_duration.sum")
    scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(units[it], 1.0)
    name = vals[head.index("Kernel Name")].split("(")[0]
    for pre in ("void ", "galois::"):
        name = name.replace(pre, "")
    return {"kernel": name, "dram_bytes_per_launch": int(tot),
            "duration_us_cold": float(vals[it].replace(",", "")) * scale}


def main():
    src = sys.argv[1]
    tag = sys.argv[2] if len(sys.argv) > 2 else os.path.basename(src.rstrip("/"))
    out = {"_source": f"ncu --set full --clock-control none --import-source on (one launch after 20, cold cache, "
                      f"replayed) of `python bench.py --workload W --steps 24 --warmup 3 --lanes 1 --no-cpu-baseline --no-e2e` "
                      f"on one B200, {tag}; dram__bytes_read.sum + dram__bytes_write.sum of that launch"}
    for rep in sorted(glob.glob(os.path.join(src, "full_*_*.ncu-rep"))):
        name = os.path.basename(rep)[len("full_"):-len(".ncu-rep")]
        wl, kern = name.split("_", 1)
        rec = launch_bytes(rep)
        if rec is None or kern not in CLASS:
            continue
        if CLASS[kern] in out.get(wl, {}) and kern == "k_update_tma":
            continue                        # the pair kernel's capture is the production one
        out.setdefault(wl, {})[CLASS[kern]] = rec
    path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "ncu_traffic.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
