"""Benchmark: GRAPE fidelity+gradient evaluations/s on the BASELINE workload.

Default workload = BASELINE.json configs[1]: n=12 all-to-all Heisenberg, the 7
S_n spin sectors (d = 13, 11, ..., 1), N_t = 1000 slices, gate fidelity against
seeded random-unitary sector targets, a batch of 4096 seeded control vectors
per GPU.  One "step" = one fidelity+gradient evaluation of the whole batch.

    python bench.py [--gpus N --steps K --warmup W] [--config 0..4] [--impl ours|reference]

Multi-GPU (torchrun, one rank per GPU): every rank evaluates its own 4096 seeds
(seed-DP, no data-path collective) -> "scaling": "weak"; value = all ranks'
evaluations / max-over-ranks device time.  ``--impl reference`` times the CPU
oracle port of the reference algorithm (oracle/grape_oracle.py; the reference
is pure Python, so nothing compiles) on the host cores, rank 0 only.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "GRAPE fidelity+gradient evals/sec"
UNIT = "evals/s"
FP64_PEAK_TFLOPS = 36.9  # measured DMMA m8n8k4 peak on this pool, profiles/r01_fp64_peak.txt
CONFIG_NAMES = {
    0: "cfg0: n=6 Heisenberg ring, D_6 A1 block d=13, state transfer, N_t=100",
    1: "cfg1: n=12 all-to-all Heisenberg, S_n sectors d<=13, gate fidelity, N_t=1000, 4096 seeds",
    2: "cfg2: n=10 Heisenberg ring, 12 D_10 blocks (30..105), gate fidelity, N_t=500",
    3: "cfg3: n=14 Heisenberg ring, 16 D_14 blocks (495..1179), gate fidelity, N_t=500",
    4: "cfg4: n=12 Heisenberg ring, unsymmetrised 4096, state transfer, N_t=200",
}


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        out, _ = self.proc.communicate(timeout=10)
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
            except ValueError:
                continue
            for n, v in zip(names, parts[2:]):
                if v.lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def build_system(cfg: int, gpu_basis: bool = False):
    """BASELINE configs[cfg].  Our arm builds the D_n bases of cfg 2 / 3 on the GPU (SURVEY 8f-2,
    untimed setup); the CPU baseline (worker processes) always uses the host restatement."""
    from paper_2309_05884_b200 import systems

    if gpu_basis and cfg in (2, 3):
        return systems.config(cfg, builder="gpu")
    return systems.config(cfg)


# ---------------------------------------------------------------- CPU reference (oracle port)
def _cpu_seed_eval(args):
    cfg, seed, n_blocks_subset, slices = args[:4]
    threads = args[4] if len(args) > 4 else 1
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    from threadpoolctl import threadpool_limits

    from oracle import grape_oracle

    s = build_system_cached(cfg)
    u = s.controls(seed)
    with threadpool_limits(threads):
        if slices is not None:  # sampled slices (per-slice cost is input independent), scaled by the caller
            s2 = _truncate(s, slices)
            grape_oracle.objective(s2, u[:, :slices], blocks=n_blocks_subset)
        else:
            grape_oracle.objective(s, u, blocks=n_blocks_subset)
    return seed


_SYS_CACHE = {}


def build_system_cached(cfg):
    if cfg not in _SYS_CACHE:
        _SYS_CACHE[cfg] = build_system(cfg)
    return _SYS_CACHE[cfg]


def _truncate(s, slices):
    import copy

    s2 = copy.copy(s)
    s2.n_slices = slices
    s2.T = s.dt * slices
    return s2


def cpu_reference(cfg: int, seconds_budget: float | None = None, cores: int | None = None):
    """Time the oracle port on the host: returns (evals/s, cores, sample description).

    cfg 0/1: rounds of `cores` independent seeds (one process per core, 1 BLAS
    thread each, the reference's process-level parallelism) until
    ~seconds_budget of wall time.  cfg 2-4: one evaluation over a sample of slices,
    scaled by N_t / sampled (per-slice cost does not depend on u).
    """
    import multiprocessing as mp

    if seconds_budget is None:
        seconds_budget = float(os.environ.get("SQOC_CPU_BUDGET_S", "12"))
    cores = cores or len(os.sched_getaffinity(0))
    s = build_system_cached(cfg)
    if cfg in (2, 3, 4):
        # sampled slices, all cores to the BLAS/LAPACK of one process (cfg 3/4 eigh of 1161..4096)
        slices, threads = {2: (10, 1), 3: (1, cores), 4: (1, cores)}[cfg]
        t0 = time.perf_counter()
        _cpu_seed_eval((cfg, 0, None, slices, threads))
        wall = time.perf_counter() - t0
        evals_per_s = (slices / s.n_slices) / wall
        sample = (f"1 evaluation of {CONFIG_NAMES[cfg]} with {slices} of {s.n_slices} slices timed and scaled, "
                  f"1 process x {threads} BLAS thread(s), {wall:.1f} s")
        return evals_per_s, threads, sample
    ctx = mp.get_context("fork")
    n_done, rounds = 0, 0
    t0 = time.perf_counter()
    with ctx.Pool(cores) as pool:
        while True:
            seeds = range(n_done, n_done + cores)
            pool.map(_cpu_seed_eval, [(cfg, sd, None, None) for sd in seeds])
            n_done += cores
            rounds += 1
            if time.perf_counter() - t0 >= seconds_budget or rounds >= 50:
                break
    wall = time.perf_counter() - t0
    sample = (f"{n_done} seeds of {CONFIG_NAMES[cfg]} (full N_t, all blocks), {cores} worker processes x 1 BLAS "
              f"thread, {wall:.1f} s wall")
    return n_done / wall, cores, sample


# ---------------------------------------------------------------- GPU arm
def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_2309_05884_b200.engine import GrapeEngine

    ws, rank, local = dist_env()
    torch.cuda.set_device(local)
    if ws > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    cfg = args.config
    s = build_system(cfg, gpu_basis=True)
    from paper_2309_05884_b200 import systems

    batch = args.batch or systems.CONFIG_BATCH[cfg]
    seed0 = 1000 * rank
    u_host = s.controls(seed0, batch=batch)
    u = torch.from_numpy(u_host).to(f"cuda:{local}")
    F = torch.empty(batch, dtype=torch.float64, device=u.device)
    g = torch.empty_like(u)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=u.device)  # > 126 MB L2
    stream = torch.cuda.current_stream()

    # ---- dominant tiny kernel timed alone: in the step the sectors' kernels share the GPU on
    # concurrent streams, so a per-stream event pair around one of them measures contention,
    # not the kernel.  The same launch (largest sector, same u) runs here on an idle GPU, before
    # the full engine exists, so its memory plan (chain history) matches the one the step uses. ----
    dom_alone_ms = None
    from paper_2309_05884_b200 import _lib

    if all(b.dim <= _lib.load().sqoc_tiny_max_dim() for b in s.blocks):
        import copy as _copy

        dims_ = [b.dim for b in s.blocks]
        bdom_ = int(np.argmax(np.array(dims_, dtype=float) ** 3))
        sub = _copy.copy(s)
        sub.blocks = [s.blocks[bdom_]]
        sub.targets = [s.targets[bdom_]]
        sub.initial = [s.initial[bdom_]] if s.initial else []
        sub.weights = np.array([s.block_weights()[bdom_]])
        eng1 = GrapeEngine(sub, max_batch=batch, device=local)
        if len(s.blocks) > 1:
            eng1.set_tiny_cta_warps(0)  # the CTA size the multi-block step launches it with
        eng1.evaluate_device(u.data_ptr(), batch, F.data_ptr(), g.data_ptr(), stream=stream.cuda_stream)
        alone = []
        for _ in range(max(2, args.steps)):
            flush.fill_(1.0)
            a0 = torch.cuda.Event(enable_timing=True)
            a1 = torch.cuda.Event(enable_timing=True)
            a0.record(stream)
            eng1.evaluate_device(u.data_ptr(), batch, F.data_ptr(), g.data_ptr(), stream=stream.cuda_stream)
            a1.record(stream)
            torch.cuda.synchronize()
            alone.append(a0.elapsed_time(a1))
        dom_alone_ms = float(np.mean(alone))
        eng1.close()
        del eng1

    torch.cuda.empty_cache()
    eng = GrapeEngine(s, max_batch=batch, device=local)

    def step():
        eng.evaluate_device(u.data_ptr(), batch, F.data_ptr(), g.data_ptr(), stream=stream.cuda_stream)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    eng.set_timing(True)
    clocks = ClockSampler(local)
    clocks.start()
    times, kern = [], []
    launches = 0
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize()
    for _ in range(args.steps):
        flush.fill_(1.0)  # L2 flush between timed iterations (not timed)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        step()
        e1.record(stream)
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1))
        kern.append(eng.block_times_ms())
        launches += eng.last_launches
    torch.cuda.synchronize()
    if ws > 1:
        dist.barrier()
    clk = clocks.stop()
    eng.set_timing(False)
    ms = float(np.mean(times))
    t = torch.tensor([ms], dtype=torch.float64, device=u.device)
    if ws > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())

    # ---- e2e: public API with host buffers (pinned u in, F + grad out) ----
    pinned = torch.from_numpy(u_host).pin_memory()
    Fh = torch.empty(batch, dtype=torch.float64).pin_memory()
    gh = torch.empty_like(pinned).pin_memory()
    eng.evaluate_host_ptr(pinned.data_ptr(), batch, Fh.data_ptr(), gh.data_ptr())  # warm
    e2e = []
    if ws > 1:
        dist.barrier()
    clocks_e2e = ClockSampler(local)
    clocks_e2e.start()
    for _ in range(max(3, args.steps)):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        eng.evaluate_host_ptr(pinned.data_ptr(), batch, Fh.data_ptr(), gh.data_ptr())
        e2e.append(time.perf_counter() - t0)
    clk_e2e = clocks_e2e.stop()
    e2e_s = float(np.mean(e2e))
    te = torch.tensor([e2e_s], dtype=torch.float64, device=u.device)
    if ws > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_s = float(te.item())

    if rank == 0:
        flops_eval = s.flops_per_eval()
        value = batch * ws / (ms_max / 1e3)
        # dominant kernel: the block with the largest algorithmic work
        dims = [b.dim for b in s.blocks]
        kt = np.mean(np.array(kern), axis=0)  # per-block device ms (events on each block's stream)
        if len(eng.large_blocks) > 0:
            dom_label = f"large-block DMMA group ({len(eng.large_blocks)} blocks)"
            dom_ms = float(kt[eng.large_blocks[0]])
            dom_flops = 8.0 * s.n_slices * 22 * sum(float(dims[b]) ** 3 for b in eng.large_blocks) * batch
            if s.objective == "state":
                dom_flops = 8.0 * s.n_slices * 8 * sum(float(dims[b]) ** 3 for b in eng.large_blocks) * batch
        else:
            bdom = int(np.argmax(np.array(dims, dtype=float) ** 3))
            dom_label = f"grape_tiny_kernel<d={dims[bdom]}> (timed alone: one launch per step, same u)"
            dom_ms = dom_alone_ms
            g_conv = 22 if s.objective == "gate" else 8
            dom_flops = 8.0 * s.n_slices * g_conv * float(dims[bdom]) ** 3 * batch
        achieved = dom_flops / (dom_ms / 1e3) / 1e12
        cpu_val, cpu_cores, cpu_sample = (None, None, "skipped")
        if not args.skip_cpu:
            cpu_val, cpu_cores, cpu_sample = cpu_reference(cfg)
        traffic = None
        tpath = os.path.join(ROOT, "profiles", "traffic.json")
        if os.path.exists(tpath):
            traffic = json.load(open(tpath)).get(str(cfg))
        line = {
            "metric": METRIC,
            "value": value,
            "unit": UNIT,
            "n_gpus": ws,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": ms_max,
            "higher_is_better": True,
            "scaling": "weak",
            "vs_baseline": None,
            "dtype": "c128",
            "data": "synthetic (seeded u ~ U[-1,1], seeded Haar/QR targets; no dataset exists)",
            "config": {
                "workload": CONFIG_NAMES[cfg],
                "blocks": dims,
                "batch_per_gpu": batch,
                "n_slices": s.n_slices,
                "parallelism": f"seed-dp{ws}" if ws > 1 else "single",
                "l2": "flushed between timed steps (256 MB write, untimed)",
                "algorithmic_flops_per_eval": flops_eval,
                "step_tflops_algorithmic": flops_eval * batch / (ms_max / 1e3) / 1e12,
                "steps_ms": [round(t, 2) for t in times],
            },
            "roofline": {
                "bound": "tensor",
                "kernel": dom_label,
                "achieved": achieved,
                "peak": FP64_PEAK_TFLOPS,
                "unit": "TFLOP/s",
                "frac": achieved / FP64_PEAK_TFLOPS,
                "launch_ms": dom_ms,
                "traffic": traffic,
                "peak_source": "measured FP64 DMMA peak (profiles/r01_fp64_peak.txt); MEASURED_PEAKS.json has no FP64 entry",
                "flops_convention": "8 * N_t * G * d^3 per (seed, block), G=22 gate / 8 state (SURVEY.md 8d)",
            },
            "cpu_baseline": {"value": cpu_val, "unit": UNIT, "cores": cpu_cores, "kind": "port", "sample": cpu_sample},
            "e2e": {
                "value": batch * ws / e2e_s,
                "unit": UNIT,
                "h2d_bytes_per_step": int(u_host.nbytes),
                "d2h_bytes_per_step": int(Fh.numel() * 8 + gh.numel() * 8),
                "calls_ms": [round(t * 1e3, 2) for t in e2e],
                "clocks": clk_e2e,
            },
            "gpu_launches": int(launches),
            "clocks": clk,
        }
        print(json.dumps(line), flush=True)
    eng.close()
    if ws > 1:
        dist.destroy_process_group()


def run_sharded(args):
    """cfg 2-4 on N > 1 GPUs: slice-chunk sharding of ONE evaluation (parallel.ShardedObjective):
    per-rank chunk products, NCCL all-gather of the chunk products (the scan carry),
    local backward sweeps, all-gather of the gradient.  Total work fixed -> "scaling": "strong"."""
    import torch
    import torch.distributed as dist

    from paper_2309_05884_b200 import parallel
    from paper_2309_05884_b200.engine import GrapeEngine

    ws, rank, local = dist_env()
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    cfg = args.config
    s = build_system(cfg, gpu_basis=True)
    comm = parallel.Comm(device=torch.device("cuda", local))
    obj = parallel.ShardedObjective(s, comm, lambda sys_: GrapeEngine(sys_, max_batch=1, device=local))
    u = s.controls(0)
    for _ in range(args.warmup):
        obj.objective(u)
    times = []
    for _ in range(args.steps):
        dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        F, g = obj.objective(u)
        torch.cuda.synchronize()
        t = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device=f"cuda:{local}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        times.append(float(t.item()))
    if rank == 0:
        sec = float(np.mean(times))
        flops = s.flops_per_eval()
        print(json.dumps({
            "metric": METRIC, "value": 1.0 / sec, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": sec * 1e3, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "c128", "data": "synthetic (seeded)",
            "config": {"workload": CONFIG_NAMES[cfg], "parallelism": f"slice-chunk{ws}",
                       "slice_chunks": parallel.chunk_bounds(s.n_slices, ws)},
            "roofline": {"bound": "tensor", "achieved": flops / sec / 1e12, "peak": FP64_PEAK_TFLOPS * ws,
                         "unit": "TFLOP/s", "frac": flops / sec / 1e12 / (FP64_PEAK_TFLOPS * ws), "traffic": None},
            "F": F,
        }), flush=True)
    dist.destroy_process_group()


def run_reference(args):
    ws, rank, local = dist_env()
    if rank != 0:
        return
    cfg = args.config
    vals = []
    cores = None
    sample = ""
    for _ in range(args.warmup):
        pass  # the CPU port has no warm-up effects worth timing (imports happen in cpu_reference)
    for _ in range(args.steps):
        v, cores, sample = cpu_reference(cfg, cores=None)
        vals.append(v)
    value = float(np.mean(vals))
    line = {
        "metric": METRIC,
        "value": value,
        "unit": UNIT,
        "n_gpus": ws,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": 1e3 / value if value else None,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "c128",
        "data": "synthetic (seeded)",
        "config": {"workload": CONFIG_NAMES[cfg]},
        "impl": "reference",
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port", "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=1)
    ap.add_argument("--batch", type=int, default=None)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--skip-cpu", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    elif args.config in (2, 3, 4) and int(os.environ.get("WORLD_SIZE", "1")) > 1:
        run_sharded(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
