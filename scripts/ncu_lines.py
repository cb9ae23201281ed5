"""Per-source-line instruction and stall-sample shares from an ncu report (needs -lineinfo and
--import-source): python scripts/ncu_lines.py report.ncu-rep [top]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
cur, hdr, out, kern = None, None, [], None
for r in csv.reader(io.StringIO(txt)):
    if not r:
        continue
    if r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r[0] == "Function Name":
        kern = r[1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr and r[0] not in ("",) and len(r) == len(hdr):
        try:
            ie = float(r[7] or 0)
            smp = float(r[4] or 0)
        except ValueError:
            continue
        out.append((ie, smp, cur, r[0], r[1].strip()[:100]))
agg = {}
for ie, smp, f, ln, src in out:
    k = (f, int(ln))
    a = agg.setdefault(k, [0.0, 0.0, src])
    a[0] += ie
    a[1] += smp
out = [(v[0], v[1], k[0], k[1], v[2]) for k, v in agg.items()]
tot = sum(o[0] for o in out) or 1
ts = sum(o[1] for o in out) or 1
print(f"kernel {kern}\ntotal warp-inst {tot:.4g}, stall samples {ts:.0f}")
for o in sorted(out, reverse=True)[:top]:
    print(f"{100 * o[0] / tot:6.2f}% inst {100 * o[1] / ts:6.2f}% samples  {o[2]}:{o[3]}  {o[4]}")
