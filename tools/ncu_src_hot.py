"""Aggregate an ncu source page (--print-source cuda,sass --csv) per CUDA source
line: stall samples and executed warp instructions, hottest lines first.
  ncu -i X.ncu-rep --page source --csv --print-source cuda,sass > x.csv
  python tools/ncu_src_hot.py x.csv [--top 40]"""
import csv
import sys

top = 40
if "--top" in sys.argv:
    top = int(sys.argv[sys.argv.index("--top") + 1])
rows = list(csv.reader(open(sys.argv[1])))
fname = None
acc = {}
hdr = None
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 8 or not r[0]:
        continue
    try:
        samples = int(r[4] or 0)
        inst = int(r[7] or 0)
    except ValueError:
        continue
    key = (fname, int(r[0]))
    acc[key] = (samples, inst, r[1][:90])
tot = sum(v[0] for v in acc.values()) or 1
toti = sum(v[1] for v in acc.values()) or 1
print(f"total stall samples {tot}, warp instructions {toti}")
for (f, ln), (s, i, src) in sorted(acc.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{100 * s / tot:5.1f}% {100 * i / toti:5.1f}%i {f}:{ln:<5} {src}")
