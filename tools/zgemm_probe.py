"""cuBLAS ZGEMM/DGEMM throughput probe (library baseline for the FP64 roofline discussion)."""
import torch, time
torch.backends.cuda.matmul.allow_tf32 = False
for dt, name, fl in ((torch.complex128, "zgemm", 8), (torch.float64, "dgemm", 2)):
    for n in (13, 64, 128, 256, 512, 1024, 1161, 2048, 4096, 8192):
        batch = max(1, min(4096, (4096 // n) ** 3 // 4)) if n < 1024 else 1
        a = torch.randn(batch, n, n, dtype=dt, device="cuda")
        b = torch.randn(batch, n, n, dtype=dt, device="cuda")
        for _ in range(3):
            c = a @ b
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        reps = 10
        e0.record()
        for _ in range(reps):
            c = a @ b
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        print(f"{name} n={n} batch={batch}: {fl * n**3 * batch / ms / 1e9:.2f} TFLOP/s ({ms:.3f} ms)", flush=True)
