import torch, time
dev = torch.device("cuda", 0)
h = torch.empty(4 << 20, dtype=torch.uint8).pin_memory()
d = torch.empty(4 << 20, dtype=torch.uint8, device=dev)
hb = torch.empty(3 << 20, dtype=torch.uint8).pin_memory()
db = torch.empty(3 << 20, dtype=torch.uint8, device=dev)
s = torch.cuda.current_stream()
for name, fn in [("h2d 4MiB", lambda: d.copy_(h, non_blocking=True)), ("d2h 3MiB", lambda: hb.copy_(db, non_blocking=True))]:
    for _ in range(3): fn()
    torch.cuda.synchronize()
    a = torch.cuda.Event(True); b = torch.cuda.Event(True)
    a.record(); 
    for _ in range(20): fn()
    b.record(); torch.cuda.synchronize()
    us = a.elapsed_time(b) / 20 * 1e3
    n = h.numel() if name.startswith("h2d") else hb.numel()
    print(name, round(us, 1), "us", round(n / us / 1e3, 1), "GB/s")
