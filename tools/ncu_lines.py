"""Aggregate ncu source-page warp-stall samples per CUDA source line.
usage: ncu -i rep --page source --csv --print-source=cuda,sass > x.csv
       python tools/ncu_lines.py x.csv [topN]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
fname, hdr, out = None, None, []
for r in rows:
    if len(r) == 2 and r[0] in ("File Name", "File Path"):
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if not hdr or len(r) != len(hdr) or not r[0].strip().isdigit():
        continue
    try:
        s = float(r[4] or 0)
    except ValueError:
        continue
    if s <= 0:
        continue
    stalls = {}
    for i, h in enumerate(hdr):
        if h.startswith("stall_") and "Not Issued" not in h:
            try:
                stalls[h[6:]] = float(r[i] or 0)
            except ValueError:
                pass
    big = sorted(stalls.items(), key=lambda kv: -kv[1])[:3]
    out.append((s, fname, r[0], r[1].strip()[:64], big))
tot = sum(o[0] for o in out)
print(f"total samples {tot:.0f}")
for s, f, ln, src, big in sorted(out, reverse=True)[:top]:
    print(f"{100*s/tot:5.1f}% {f}:{ln:>4} {src:64s} " + " ".join(f"{k}={100*v/max(s,1):.0f}%" for k, v in big))
