import torch, time
n = 134 * 1024 * 1024
h = torch.empty(n, dtype=torch.uint8).pin_memory(); h.fill_(1)
d = torch.empty(n, dtype=torch.uint8, device="cuda")
for k in (1, 2, 4, 8):
    sts = [torch.cuda.Stream() for _ in range(k)]
    for rep in range(3):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        ch = n // k
        for i, s in enumerate(sts):
            with torch.cuda.stream(s):
                d[i*ch:(i+1)*ch].copy_(h[i*ch:(i+1)*ch], non_blocking=True)
        torch.cuda.synchronize(); dt = time.perf_counter() - t0
    print(k, "streams", round(n / dt / 1e9, 1), "GB/s")
