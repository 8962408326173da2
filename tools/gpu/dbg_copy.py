import time, torch
for mb in (0.75, 1.5, 3.1, 6.3):
    n = int(mb * 1e6 / 4)
    h = torch.empty(n, dtype=torch.float32, pin_memory=True)
    d = torch.empty(n, dtype=torch.float32, device="cuda")
    s = torch.cuda.Stream()
    a = torch.randn(8192, 8192, device="cuda")
    for busy in (False, True):
        torch.cuda.synchronize()
        if busy:
            for _ in range(20): a @ a  # ~ms of work on the default stream
        t0 = time.perf_counter()
        with torch.cuda.stream(s):
            d.copy_(h, non_blocking=True)
        t1 = time.perf_counter()
        torch.cuda.synchronize()
        print(f"{mb} MB busy={busy}: issue {1e6*(t1-t0):.1f} us")
