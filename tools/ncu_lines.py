"""Per-source-line totals of an ncu --set full capture (instructions, stall samples).

usage: ncu -i REP --page source --csv --print-source cuda,sass > x.csv; python tools/ncu_lines.py x.csv [N]
"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
hdr = None
fname = ""
out = []
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].rsplit("/", 1)[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or r[0] in ("", "Function Name"):
        continue
    try:
        line = int(r[0])
    except ValueError:
        continue
    d = dict(zip(hdr[2:], r[2:]))
    def num(k):
        try:
            return float(d.get(k, "0").replace(",", "") or 0)
        except ValueError:  # a source line with quotes the CSV writer did not escape
            return 0.0
    out.append((fname, line, r[1].strip()[:70], num("Instructions Executed"), num("Warp Stall Sampling (All Samples)"),
                num("Thread Instructions Executed")))
ti = sum(o[3] for o in out)
ts = sum(o[4] for o in out)
print(f"total warp instructions {ti:.3e}, stall samples {ts:.0f}")
print("by stall samples:")
for o in sorted(out, key=lambda o: -o[4])[:top]:
    print(f"{o[0]}:{o[1]:5d} inst {100 * o[3] / ti:5.1f}%  stall {100 * o[4] / ts:5.1f}%  lanes {o[5] / max(o[3], 1):4.1f} | {o[2]}")
