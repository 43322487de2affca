import sys, time
sys.path.insert(0, ".")
import numpy as np
from paper_2309_05884_b200 import systems
from paper_2309_05884_b200.engine import GrapeEngine
s = systems.config(0); u0 = s.controls(0)
eng = GrapeEngine(s, max_batch=1)
for _ in range(3): eng.objective(u0)
ts = []
for _ in range(20):
    t0 = time.perf_counter(); eng.objective(u0); ts.append((time.perf_counter() - t0) * 1e3)
print("back-to-back ms", np.round(ts, 3).tolist())
ts = []
for _ in range(20):
    time.sleep(0.005)
    t0 = time.perf_counter(); eng.objective(u0); ts.append((time.perf_counter() - t0) * 1e3)
print("after 5 ms host gap ms", np.round(ts, 3).tolist())
from scipy.optimize import minimize
cnt = [0]; tt = [0.0]
def fun(x):
    t0 = time.perf_counter(); f, g = eng.objective(x.reshape(u0.shape)); tt[0] += time.perf_counter() - t0; cnt[0] += 1
    return -float(f), -g.reshape(-1)
t0 = time.perf_counter()
minimize(fun, u0.reshape(-1), jac=True, method="L-BFGS-B", options={"maxiter": 50})
print("scipy total ms", (time.perf_counter() - t0) * 1e3, "evals", cnt[0], "eval ms total", tt[0] * 1e3)
