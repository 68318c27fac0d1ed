"""Per-kernel share of device time from an ncu launch list (gpu__time_duration.sum csv)."""
import csv, re, sys, collections
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 14 and r[12] == "gpu__time_duration.sum"]
tot = collections.defaultdict(float); cnt = collections.Counter()
for r in rows:
    name = re.sub(r"\(.*", "", r[4]).replace("<unnamed>::", "").replace("void ", "").strip()
    tot[name] += float(r[14]) / 1e6; cnt[name] += 1
skip = {"k_gen"}
knn = {k: v for k, v in tot.items() if not any(s in k for s in skip) and "summarize" not in k}
s = sum(knn.values())
print(f"{'kernel':34s} {'launches':>8s} {'ms total':>10s} {'ms/launch':>10s} {'share(knn)':>10s}")
for k, v in sorted(tot.items(), key=lambda x: -x[1]):
    sh = f"{v / s:10.3f}" if k in knn else "         -"
    print(f"{k:34s} {cnt[k]:8d} {v:10.3f} {v / cnt[k]:10.4f} {sh}")
