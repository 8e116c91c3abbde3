import time, torch, numpy as np
torch.cuda.set_device(0)
h = torch.empty(250_000_000, dtype=torch.uint8).pin_memory()
d = torch.empty_like(h, device="cuda")
k = torch.empty(1 << 20, device="cuda")
for _ in range(5):
    d.copy_(h, non_blocking=True); torch.cuda.synchronize()
ts = []
for i in range(300):
    t0 = time.perf_counter(); d.copy_(h, non_blocking=True); torch.cuda.synchronize(); ts.append((time.perf_counter() - t0) * 1e3)
    k.mul_(1.0001); torch.cuda.synchronize()
    time.sleep(0.03)
ts = np.array(ts)
print("H2D 250 MB: median %.2f ms max %.1f outliers>8ms %s" % (np.median(ts), ts.max(), [round(t, 1) for t in ts if t > 8]))
