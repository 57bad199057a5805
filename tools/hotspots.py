"""Per-source-line instruction and stall shares from an ncu report
(`ncu -i R --page source --csv --print-source cuda,sass -k regex:K`)."""
import csv
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 45
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kern}",
                      "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
fname, hdr, res = None, None, []
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
    elif len(r) > 3 and r[0] == "Line No":
        hdr = r
    elif hdr and len(r) == len(hdr) and r[0] not in ("",):
        try:
            inst = int(r[hdr.index("Instructions Executed")])
            stall = int(r[hdr.index("Warp Stall Sampling (All Samples)")])
        except ValueError:
            continue
        res.append((fname, int(r[0]), r[1], inst, stall))
ti = sum(x[3] for x in res) or 1
ts = sum(x[4] for x in res) or 1
print(f"total inst {ti} stall samples {ts}")
for f, ln, src, i, s in sorted(res, key=lambda x: -x[3])[:top]:
    print(f"{f:>22}:{ln:5d} inst {100*i/ti:5.1f}% stall {100*s/ts:5.1f}%  {src.strip()[:90]}")
