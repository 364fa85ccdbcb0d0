"""Dynamic SASS mix from `ncu --page source --csv --print-source sass` (warp-level
instructions executed per opcode, and the hottest address ranges)."""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
iA, iS, iE, iSm = hdr.index("Address"), hdr.index("Source"), hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
ops = collections.Counter(); stalls = collections.Counter(); tot = 0; seq = []
for r in rows[2:]:
    if len(r) <= iE or not r[iE].isdigit():
        continue
    src = r[iS].strip().split()
    op = src[0] if not src[0].startswith("@") else src[1]
    base = op.split(".")[0]
    n = int(r[iE]); tot += n
    ops[op if base in ("IMAD", "LOP3", "SYNCS", "LDS", "STG", "MUFU") else base] += n
    stalls[base] += int(r[iSm] or 0)
    seq.append((r[iA], r[iS].strip(), n, int(r[iSm] or 0)))
print("total warp instructions", tot)
for op, n in ops.most_common(45):
    print(f"{op:28s} {n:14d} {100*n/tot:6.2f}%")
if len(sys.argv) > 2:
    lo = int(sys.argv[2])
    for a, s, n, sm in seq:
        if n >= lo:
            print(a[-5:], f"{n:11d} {sm:6d}", s)
