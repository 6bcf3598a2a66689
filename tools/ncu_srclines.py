"""Top CUDA source lines by warp stall samples from an ncu 'cuda,sass' source page (csv):
ncu -i rep --page source --csv --print-source cuda,sass > x.csv; python tools/ncu_srclines.py x.csv [top]"""
import csv
import sys


def num(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
fname, hdr, out = None, None, []
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        iS = hdr.index("Warp Stall Sampling (All Samples)")
        iE = hdr.index("Instructions Executed")
        continue
    if hdr is None or r[0] == "" or len(r) <= iS:
        continue
    out.append((num(r[iS]), num(r[iE]), fname, r[0], r[1]))
tot = sum(o[0] for o in out) or 1.0
print("total samples", tot)
for s, e, f, ln, src in sorted(out, key=lambda o: -o[0])[:top]:
    print(f"{s / tot * 100:5.1f}% {f}:{ln} instr={int(e)} | {src.strip()[:90]}")
