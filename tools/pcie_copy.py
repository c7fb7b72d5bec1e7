import torch, time
n = 1 << 20  # 4 MB fp32
for size in [n // 4, n, 4 * n, 64 * n]:
    h = torch.empty(size, dtype=torch.float32).pin_memory(); h2 = torch.empty_like(h).pin_memory()
    d = torch.empty(size, device="cuda"); d2 = torch.empty(size, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    for _ in range(3):
        d.copy_(h, non_blocking=True); h2.copy_(d2, non_blocking=True)
    torch.cuda.synchronize()
    def t(fn, reps=20):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        for _ in range(reps): fn()
        torch.cuda.synchronize(); return (time.perf_counter() - t0) / reps * 1e6
    a = t(lambda: d.copy_(h, non_blocking=True))
    b = t(lambda: h2.copy_(d2, non_blocking=True))
    def both():
        with torch.cuda.stream(s1): d.copy_(h, non_blocking=True)
        with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
    c = t(both)
    MB = size * 4 / 1e6
    print(f"{MB:7.1f} MB: H2D {a:8.1f} us ({MB/a*1e3:5.1f} GB/s)  D2H {b:8.1f} us ({MB/b*1e3:5.1f} GB/s)  both {c:8.1f} us")
