"""Per-source-line instruction / stall-sample attribution of an ncu report's
`--page source --csv --print-source=cuda,sass` export (dev tool).

    python scripts/ncu_lines.py export.csv UNITS [TOP]
UNITS divides the counts (e.g. the number of work items)."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
units = float(sys.argv[2])
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
cur = None
fname = None
agg, st, src = collections.Counter(), collections.Counter(), {}
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] in ("Function Name", "Line No"):
        continue
    if r[0] != "":
        cur = (fname, int(r[0]))
        src[cur] = r[1]
        continue
    if cur and len(r) > 7:
        try:
            agg[cur] += float(r[7] or 0)
            st[cur] += float(r[4] or 0)
        except ValueError:
            pass
tot, tots = sum(agg.values()), sum(st.values())
print(f"{tot / units:.1f} instructions per unit (inline frames counted once per line)")
for k, v in sorted(agg.items(), key=lambda x: -x[1])[:top]:
    print(f"{v / units:6.1f} {st[k] / tots * 100:5.1f}%st {k[0][:12]}:{k[1]:<5d} {src[k].strip()[:90]}")
