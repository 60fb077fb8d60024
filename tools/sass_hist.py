"""Per-function SASS opcode histogram of the built library (checks IMMA/UBLKCP presence and
the instruction mix of the hot loop). Usage: python tools/sass_hist.py <substring-of-symbol>"""
import collections, re, subprocess, sys
so = "paper_2303_12753_b200/lib/libseghdc_b200.so"
out = subprocess.run(["cuobjdump", "-sass", so], capture_output=True, text=True).stdout
pat = sys.argv[1] if len(sys.argv) > 1 else "k_round"
cur, hist = None, collections.defaultdict(collections.Counter)
for line in out.splitlines():
    m = re.search(r"Function : (\S+)", line)
    if m:
        cur = m.group(1)
        continue
    m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)", line)
    if m and cur and pat in cur:
        hist[cur][m.group(1)] += 1
for fn, h in hist.items():
    print(fn, sum(h.values()))
    print("   ", ", ".join(f"{k}:{v}" for k, v in h.most_common(14)))
