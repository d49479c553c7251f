import time, torch
dev = torch.device("cuda", 0)
src = torch.randn(65536, 512, device=dev)
y = None
for i in range(12):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    y2 = torch.empty((65536, 512), dtype=torch.float32, pin_memory=True)
    t1 = time.perf_counter()
    y2.copy_(src, non_blocking=True)
    torch.cuda.synchronize(); t2 = time.perf_counter()
    y = y2
    print(f"{i}: alloc {1e3*(t1-t0):7.2f} ms  copy {1e3*(t2-t1):6.2f} ms", flush=True)
