import torch, time
n = 512 * 1024 * 1024   # int64 elements = 4 GiB
dev = torch.empty(n, dtype=torch.int64, device="cuda").fill_(1)
host = torch.empty(n, dtype=torch.int64, pin_memory=True)
for ns in (1, 2, 4):
    streams = [torch.cuda.Stream() for _ in range(ns)]
    part = n // ns
    for rep in range(3):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        for i, s in enumerate(streams):
            with torch.cuda.stream(s):
                host[i * part:(i + 1) * part].copy_(dev[i * part:(i + 1) * part], non_blocking=True)
        torch.cuda.synchronize(); dt = time.perf_counter() - t0
    print(f"D2H {ns} streams: {n * 8 / dt / 1e9:.1f} GB/s", flush=True)
for ns in (1, 2):
    streams = [torch.cuda.Stream() for _ in range(ns)]
    part = n // ns
    for rep in range(3):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        for i, s in enumerate(streams):
            with torch.cuda.stream(s):
                dev[i * part:(i + 1) * part].copy_(host[i * part:(i + 1) * part], non_blocking=True)
        torch.cuda.synchronize(); dt = time.perf_counter() - t0
    print(f"H2D {ns} streams: {n * 8 / dt / 1e9:.1f} GB/s", flush=True)
