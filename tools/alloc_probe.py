import time, torch
torch.cuda.init()
x = torch.empty(1, device="cuda"); torch.cuda.synchronize()
for gb in (100, 100, 50):
    t0 = time.perf_counter()
    b = torch.empty(gb * (1 << 30) // 8, dtype=torch.float64, device="cuda")
    torch.cuda.synchronize(); t1 = time.perf_counter()
    b.fill_(0.0); torch.cuda.synchronize(); t2 = time.perf_counter()
    del b; torch.cuda.empty_cache(); torch.cuda.synchronize(); t3 = time.perf_counter()
    print(f"{gb} GB: malloc {1e3*(t1-t0):.1f} ms, first touch (fill) {1e3*(t2-t1):.1f} ms, free+empty_cache {1e3*(t3-t2):.1f} ms", flush=True)
