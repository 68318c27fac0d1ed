import torch, time
x = torch.empty(150 * (1 << 30), dtype=torch.uint8, device="cuda")
torch.cuda.synchronize()
ts = []
for i in range(3000):
    t0 = time.perf_counter(); torch.cuda.mem_get_info(); ts.append((time.perf_counter() - t0) * 1e3)
    if i % 10 == 0: time.sleep(0.002)
ts.sort()
print("mem_get_info ms: median %.4f p99 %.4f max %.4f" % (ts[len(ts)//2], ts[int(len(ts)*0.99)], ts[-1]))
# plain stream sync latency with tiny kernels
y = torch.zeros(1024, device="cuda")
ts = []
for i in range(3000):
    t0 = time.perf_counter(); y.add_(1); torch.cuda.synchronize(); ts.append((time.perf_counter() - t0) * 1e3)
ts.sort()
print("launch+sync ms: median %.4f p99 %.4f max %.4f" % (ts[len(ts)//2], ts[int(len(ts)*0.99)], ts[-1]))
