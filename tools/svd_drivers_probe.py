import torch, time
dev = torch.device("cuda", 0)
r = torch.randn(200, 200, device=dev, dtype=torch.float64) @ torch.diag(torch.arange(1, 201, device=dev, dtype=torch.float64) ** -2.0)
ref = torch.linalg.svdvals(r.cpu())
for drv in ["gesvd", "gesvdj", "gesvda", None]:
    for _ in range(2):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        u, s, vh = torch.linalg.svd(r, full_matrices=False, driver=drv)
        torch.cuda.synchronize(); t = time.perf_counter() - t0
    err = float(((u * s) @ vh - r).norm() / r.norm())
    print(drv, f"{t*1e3:.2f} ms", "recon", err, "sv rel", float(((s.cpu() - ref) / ref).abs().max()))
torch.cuda.synchronize(); t0 = time.perf_counter()
u, s, vh = torch.linalg.svd(r.cpu(), full_matrices=False)
print("cpu", (time.perf_counter() - t0) * 1e3, "ms")
