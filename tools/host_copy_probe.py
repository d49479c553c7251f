import time, numpy as np, torch
a = np.random.default_rng(0).standard_normal((65536, 8192)).astype(np.float32)
ta = torch.from_numpy(a)
rows = 4096
st = torch.empty((rows, 8192), dtype=torch.float32, pin_memory=True)
for nt in (1, 4, 8, 16):
    torch.set_num_threads(nt)
    t0 = time.perf_counter()
    for r0 in range(0, 65536, rows):
        st.copy_(ta[r0:r0 + rows])
    dt = time.perf_counter() - t0
    print(f"torch copy_ pageable->pinned threads={nt}: {a.nbytes / dt / 1e9:.1f} GB/s", flush=True)
t0 = time.perf_counter()
for r0 in range(0, 65536, rows):
    np.copyto(st.numpy(), a[r0:r0 + rows])
print(f"np.copyto: {a.nbytes / (time.perf_counter() - t0) / 1e9:.1f} GB/s")
t0 = time.perf_counter(); p = torch.empty((65536, 512), dtype=torch.float64, pin_memory=True); print(f"pin alloc 268MB {1e3*(time.perf_counter()-t0):.1f} ms")
y = torch.randn(65536, 512)
t0 = time.perf_counter(); z = y.numpy().astype(np.float64); print(f"f32->f64 134MB {1e3*(time.perf_counter()-t0):.1f} ms")
