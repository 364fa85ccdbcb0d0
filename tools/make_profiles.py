"""Regenerate the committed profile summaries from one `tools/gpu_round.sh <tag>` run.

    python tools/make_profiles.py gpurun_out/r01h r01

Writes profiles/<round>_bench_<cfg>.json, <round>_c2_launches.csv / _c4_launches.csv,
<round>_launches.md (C2 split into lane and undivided launches), <round>_ncu_full.md
(keeping its hand-written "Reading:" section) and ncu_traffic.json.
"""
import collections
import csv
import glob
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC, RND = sys.argv[1], sys.argv[2]
TAG = os.path.basename(SRC.rstrip("/"))
P = os.path.join(ROOT, "profiles")
sys.path.insert(0, P)
import summarize_ncu  # noqa: E402

for f in glob.glob(os.path.join(SRC, "bench_*.json")):
    name = os.path.basename(f)[len("bench_"):-len(".json")].lower()
    lines = [l for l in open(f).read().splitlines() if l.strip()]
    with open(os.path.join(P, f"{RND}_bench_{name}.json"), "w") as o:
        o.write(lines[-1] + "\n")
for W in ("C2", "C4"):
    shutil.copy(os.path.join(SRC, f"launches_{W}.csv"), os.path.join(P, f"{RND}_{W.lower()}_launches.csv"))
subprocess.run([sys.executable, os.path.join(ROOT, "tools", "traffic_json.py"), SRC, TAG], check=True,
               stdout=subprocess.DEVNULL)


def seqof(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}
    return [(r[ki].split("(")[0].replace("void ", "").replace("galois::", ""),
             float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)) for r in rows[hi + 1:] if len(r) > vi]


def table(seq, split=None):
    agg, seen = collections.OrderedDict(), collections.Counter()
    for name, t in seq:
        seen[name] += 1
        key = name
        if split and name in split[1]:
            key = f"{name} [{'lane, 1024 members' if seen[name] <= split[0] else 'undivided, 4096 members'}]"
        agg.setdefault(key, []).append(t)
    tot = sum(sum(v) for v in agg.values())
    out = ["| kernel | launches | mean us | total us | share |", "|---|---|---|---|---|"]
    out += [f"| {k} | {len(v)} | {sum(v) / len(v):.2f} | {sum(v):.1f} | {sum(v) / tot:.1%} |" for k, v in agg.items()]
    return "\n".join(out), agg


main = ("k_sweep<1, 1, 0, 0>", "k_update_pair<1, 1, 0>")
c2 = seqof(os.path.join(SRC, "launches_C2.csv"))
c4 = seqof(os.path.join(SRC, "launches_C4.csv"))
t2, agg2 = table(c2, (28, main))
t4, _ = table(c4)
m = {k: sum(v) / len(v) for k, v in agg2.items()}
lane = [m.get(f"{k} [lane, 1024 members]", 0) for k in main]
und = [m.get(f"{k} [undivided, 4096 members]", 0) for k in main]
md = f"""# Round {int(RND[1:])} — launch lists (ncu gpu__time_duration.sum, --clock-control none)

Command: `ncu --metrics gpu__time_duration.sum --clock-control none --csv python bench.py --workload W --steps 4 --warmup 3 --no-cpu-baseline --no-e2e --no-tts` — the bench's own command (cold-cache, serialised per launch: compare shares, not absolutes). Raw CSVs: {RND}_c2_launches.csv, {RND}_c4_launches.csv. Source: gpurun_out/{TAG}.

## C2 (configs[1], bench workload: 3-SAT n=10000 m=42000, B=4096)

The bench's timed region runs 4 lanes of 1024 members (DESIGN §6.1): the first 28 sweep
and update launches are lane launches (4 lanes x 7 steps); the remaining ones belong to
the undivided engine of the kernel timing pass. Serialised under ncu a lane's update takes
{lane[1]:.1f} us (vs {und[1]:.1f} / 4 = {und[1] / 4:.1f} us per 1024 members undivided) and a lane's
sweep {lane[0]:.1f} us (vs {und[0] / 4:.1f}): per-lane kernels are less efficient alone, but in
the bench they run concurrently (4 x ({lane[0]:.1f} + {lane[1]:.1f}) = {4 * (lane[0] + lane[1]):.0f} us serialised per step vs
the bench's measured step). Undivided, the update is {und[1] / (und[0] + und[1]):.1%} and the sweep
{und[0] / (und[0] + und[1]):.1%} of the step's kernel time.

{t2}

## C4 (industrial-like n=1M m=4.2M, B=1024; one 1024-member chunk, no lanes)

{t4}
"""
open(os.path.join(P, f"{RND}_launches.md"), "w").write(md)

reading = ""
old = os.path.join(P, f"{RND}_ncu_full.md")
if os.path.exists(old):
    txt = open(old).read()
    if "Reading:" in txt:
        reading = txt[txt.index("Reading:"):]
parts = [f"# Round {int(RND[1:])} — ncu --set full of the step kernels (one launch each, after 20, undivided engine)", "",
         "Command: `ncu --set full --clock-control none --import-source on -k regex:K -s 20 -c 1 python bench.py "
         "--workload W --steps 24 --warmup 3 --lanes 1 --no-cpu-baseline --no-e2e` on one B200 (replayed, cold cache). "
         "`--lanes 1`: the bench's kernel timing pass (and its roofline) uses an undivided engine, so the captured "
         f"launch is the one the roofline describes. Source: gpurun_out/{TAG}.", ""]
for W in ("C2", "C4"):
    parts += [f"## {W}", ""]
    first = True
    for K in ("k_update_pair", "k_update_tma", "k_sweep", "k_hub_partial_tma"):
        rep = os.path.join(SRC, f"full_{W}_{K}.ncu-rep")
        if not os.path.exists(rep):
            continue
        raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
        if raw.count("\n") < 3:
            continue
        tmp = rep + ".raw.csv"
        open(tmp, "w").write(raw)
        import io
        import contextlib
        buf = io.StringIO()
        with contextlib.redirect_stdout(buf):
            summarize_ncu.full(tmp)
        lines = buf.getvalue().strip().splitlines()
        parts += lines if first else lines[2:]
        first = False
    parts.append("")
open(old, "w").write("\n".join(parts) + "\n" + reading)
print("profiles written from", SRC)
