"""Per-launch update / forward ms of tools/window_ab.sh outputs: python tools/window_ab_read.py gpurun_out/<out>"""
import glob, json, os, sys
for f in sorted(glob.glob(os.path.join(sys.argv[1], "*.txt"))):
    sub = None
    rows = []
    for line in open(f):
        if not line.startswith("{"):
            continue
        d = json.loads(line)
        if "sub" in d:
            sub = d["sub"]
        elif sub is not None:
            rows.append((sub, {k: round(v[0] / v[1], 4) for k, v in d.items() if k in ("update", "forward")}))
    print(os.path.basename(f), rows)
