import torch, time
n = 512 << 20
h = torch.empty(n // 8, dtype=torch.float64).pin_memory(); d = torch.empty(n // 8, dtype=torch.float64, device='cuda')
h2 = torch.empty(n // 8, dtype=torch.float64).pin_memory(); d2 = torch.empty(n // 8, dtype=torch.float64, device='cuda')
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for name, fn in [("h2d", lambda: d.copy_(h, non_blocking=True)), ("d2h", lambda: h.copy_(d, non_blocking=True))]:
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); [fn() for _ in range(5)]; e1.record(); torch.cuda.synchronize()
    print(name, f"{5 * n / (e0.elapsed_time(e1) * 1e-3) / 1e9:.1f} GB/s")
torch.cuda.synchronize(); t = time.perf_counter()
with torch.cuda.stream(s1):
    for _ in range(5): d.copy_(h, non_blocking=True)
with torch.cuda.stream(s2):
    for _ in range(5): h2.copy_(d2, non_blocking=True)
torch.cuda.synchronize(); dt = time.perf_counter() - t
print(f"bidirectional: {5 * n / dt / 1e9:.1f} GB/s each way")
