"""Per-instruction stall attribution from `ncu -i X --page source --csv --print-source sass`.

  python tools/sass_stalls.py <source.csv> [top_n]
Prints the total stall samples per reason, per opcode, and the hottest instructions.
"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot = collections.Counter()
byop = collections.Counter()
ins = []
for r in rows[2:]:
    if len(r) < len(hdr):
        continue
    s = int(r[ix["# Samples"]] or 0)
    op = r[ix["Source"]].split()[0] if r[ix["Source"]].split() else "?"
    if op.startswith("@"):
        op = r[ix["Source"]].split()[1]
    byop[op.split(".")[0]] += s
    st = {x: int(r[ix[x]] or 0) for x in reasons}
    tot.update(st)
    ins.append((s, r[ix["Address"]][-5:], r[ix["Source"]].strip()[:60], r[ix["Instructions Executed"]],
                ", ".join(f"{k[6:]}={v}" for k, v in sorted(st.items(), key=lambda x: -x[1])[:3] if v)))
T = sum(tot.values()) or 1
print("reasons:", ", ".join(f"{k[6:]} {100*v/T:.1f}%" for k, v in tot.most_common(10)))
print("by opcode:", ", ".join(f"{k} {100*v/T:.1f}%" for k, v in byop.most_common(15)))
for s, a, src, n, st in sorted(ins, reverse=True)[:top]:
    print(f"{100*s/T:5.1f}% {a} {src:60s} n={n} {st}")
