"""Top SASS lines by warp-stall samples for one kernel of an ncu report."""
import csv, subprocess, sys
rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kern}",
                      "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[1]
data = rows[2:]
si = hdr.index("Warp Stall Sampling (All Samples)")
src = hdr.index("Source")
tot = sum(int(r[si]) for r in data if r[si].isdigit())
rs = sorted([r for r in data if r[si].isdigit()], key=lambda r: -int(r[si]))[:top]
print("total samples", tot)
for r in rs:
    print(f"{int(r[si]):7d} {100*int(r[si])/tot:5.1f}%  {r[0][-5:]}  {r[src].strip()[:90]}")
