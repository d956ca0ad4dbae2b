import torch, time
n = 1 << 30  # 1 GiB chunks
h1 = torch.empty(n, dtype=torch.uint8).pin_memory(); h2 = torch.empty(n, dtype=torch.uint8).pin_memory()
d1 = torch.empty(n, dtype=torch.uint8, device='cuda'); d2 = torch.empty(n, dtype=torch.uint8, device='cuda')
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for mode in ("h2d", "d2h", "both"):
    torch.cuda.synchronize(); t = time.perf_counter()
    for _ in range(4):
        if mode in ("h2d", "both"):
            with torch.cuda.stream(s1): d1.copy_(h1, non_blocking=True)
        if mode in ("d2h", "both"):
            with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
    torch.cuda.synchronize(); dt = time.perf_counter() - t
    tot = 4 * n * (2 if mode == "both" else 1)
    print(mode, round(tot / dt / 1e9, 1), "GB/s")
