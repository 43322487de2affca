import sys, time
import numpy as np, torch
sys.path.insert(0, ".")
from paper_2309_05884_b200 import systems
from paper_2309_05884_b200.engine import GrapeEngine
s = systems.config(1)
B = 4096
eng = GrapeEngine(s, max_batch=B)
uh = s.controls(0, batch=B)
u = torch.from_numpy(uh).cuda(); F = torch.empty(B, dtype=torch.float64, device="cuda"); g = torch.empty_like(u)
pin = torch.from_numpy(uh).pin_memory(); Fh = torch.empty(B, dtype=torch.float64).pin_memory(); gh = torch.empty_like(pin).pin_memory()
def wall(f, n=3):
    ts = []
    for _ in range(n):
        torch.cuda.synchronize(); t0 = time.perf_counter(); f(); torch.cuda.synchronize(); ts.append(time.perf_counter() - t0)
    return [round(t * 1e3, 1) for t in ts]
eng.evaluate_device(u.data_ptr(), B, F.data_ptr(), g.data_ptr())
print("device stream0 wall ms", wall(lambda: eng.evaluate_device(u.data_ptr(), B, F.data_ptr(), g.data_ptr())))
cs = torch.cuda.current_stream().cuda_stream
print("device torch-stream wall ms", wall(lambda: eng.evaluate_device(u.data_ptr(), B, F.data_ptr(), g.data_ptr(), stream=cs)))
print("host wall ms", wall(lambda: eng.evaluate_host_ptr(pin.data_ptr(), B, Fh.data_ptr(), gh.data_ptr())))
x = torch.empty_like(u)
print("H2D 65MB ms", wall(lambda: x.copy_(pin, non_blocking=True)))
print("D2H 65MB ms", wall(lambda: gh.copy_(g, non_blocking=True)))
print("device stream0 wall ms again", wall(lambda: eng.evaluate_device(u.data_ptr(), B, F.data_ptr(), g.data_ptr())))
# host path emulated with torch copies around the device evaluation (same stream)
ud = torch.empty_like(u); Fd = torch.empty_like(F); gd = torch.empty_like(g)
def emul():
    ud.copy_(pin, non_blocking=True)
    eng.evaluate_device(ud.data_ptr(), B, Fd.data_ptr(), gd.data_ptr())
    Fh.copy_(Fd, non_blocking=True); gh.copy_(gd, non_blocking=True)
print("emulated host path wall ms", wall(emul))
print("host wall ms again", wall(lambda: eng.evaluate_host_ptr(pin.data_ptr(), B, Fh.data_ptr(), gh.data_ptr())))
