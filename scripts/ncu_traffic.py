"""DRAM traffic per batch of the roofline kernels from the ncu --set full captures of one build:
{"lib_sha16": ..., "C4": {"lb_pass_index": bytes, "refine_index": bytes, "summarize": bytes}}
(refine: the two waves of one batch summed; the others: one launch)."""
import csv
import hashlib
import json
import os
import subprocess
import sys

out_dir = sys.argv[1]
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
lib = os.path.join(root, "paper_2009_00166_b200", "libparis.so")
sha = hashlib.sha256(open(lib, "rb").read()).hexdigest()[:16]


def dram(rep):
    if not os.path.exists(rep):
        return None
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(txt.splitlines()))
    hdr, units, data = rows[0], rows[1], rows[2:]
    tot = 0.0
    for d in data:
        for key in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            i = hdr.index(key)
            v = float(d[i].replace(",", ""))
            u = units[i]
            tot += v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
    return tot


res = {"lib_sha16": sha, "C4": {}}
for name, key in (("k_lbi", "lb_pass_index"), ("k_refine1m", "refine_index"), ("k_summarize_seg", "summarize"),
                  ("k_gf", "lb_pass_gf")):
    v = dram(os.path.join(out_dir, f"full_c4_{name}.ncu-rep"))
    if v is not None:
        res["C4"][key] = v
print(json.dumps(res, indent=1))
