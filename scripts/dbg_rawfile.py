"""Debug: device-buffer vs host-buffer k-NN with raw in a mapped file / pinned host memory."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2009_00166_b200 as P
from datagen import gpu as dg
import datagen, oracle

n = int(sys.argv[1]) if len(sys.argv) > 1 else 20_000_000
mode = sys.argv[2] if len(sys.argv) > 2 else "file"
L = 256
ds, qs = datagen.config_seeds(4)
path = "/tmp/paris_dbg.f32"
chunk = 1 << 22
buf = torch.empty((chunk, L), device="cuda")
raw16 = torch.empty((n, L), dtype=torch.int16, device="cuda")
hb = torch.empty((chunk, L), pin_memory=True)
if mode == "file":
    with open(path, "wb") as f:
        for r0 in range(0, n, chunk):
            m = min(chunk, n - r0)
            dg.walks(m, L, ds, first_id=r0, out=buf[:m])
            raw16[r0:r0 + m].copy_(P.raw_bf16(buf[:m]))
            hb[:m].copy_(buf[:m])
            f.write(hb[:m].numpy().tobytes())
    sax = P.summarize_file(path, n, L, 16, 256, direct_io=True)
    mp = P.MappedRaw(path, n, L)
    raw = mp.tensor
else:
    raw = torch.empty((n, L), pin_memory=True)
    for r0 in range(0, n, chunk):
        m = min(chunk, n - r0)
        dg.walks(m, L, ds, first_id=r0, out=buf[:m])
        raw16[r0:r0 + m].copy_(P.raw_bf16(buf[:m]))
        raw[r0:r0 + m].copy_(buf[:m])
    sax = P.summarize(raw, 16, 256)
idx = P.index_build(sax, 16, 256)
q = dg.walks(100, L, qs)
torch.cuda.synchronize()
res = []
cfg = P.KnnConfig(batch=64)
_, _, st = P.knn_index(raw, idx, q, k=1, raw16=raw16, config=cfg, stats=True)
print("stats: cand max", int(st["candidates"].max()), "raw16 rows mean", float(st["raw16_rows"].double().mean()))
for rep in range(3):
    gi, gd = P.knn_index(raw, idx, q, k=1, raw16=raw16, config=cfg)
    torch.cuda.synchronize()
    res.append((gi.cpu().numpy().ravel(), gd.cpu().numpy().ravel()))
hq = q.cpu().pin_memory()
for rep in range(3):
    hi = torch.empty((100, 1), dtype=torch.int64).pin_memory(); hd = torch.empty((100, 1)).pin_memory()
    P.knn_index(raw, idx, hq, k=1, raw16=raw16, out_idx=hi, out_dist=hd, config=cfg)
    res.append((hi.numpy().ravel().copy(), hd.numpy().ravel().copy()))
x = raw.numpy() if mode != "file" else raw.numpy()
qh = q.cpu().numpy()
base = res[0]
for r, (i, d) in enumerate(res):
    bad = np.nonzero(i != base[0])[0]
    print("run", r, "mismatches vs run 0:", len(bad))
    for b in bad[:5]:
        t0 = np.sqrt(((x[base[0][b]].astype(np.float64) - qh[b]) ** 2).sum())
        t1 = np.sqrt(((x[i[b]].astype(np.float64) - qh[b]) ** 2).sum())
        print("   q", b, "run0", base[0][b], base[1][b], "true", t0, "| run", i[b], d[b], "true", t1)
if mode == "file":
    mp.close()
    os.remove(path)
