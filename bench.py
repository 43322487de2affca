"""Benchmark: GRAPE fidelity+gradient evaluations/s on a BASELINE workload.

Default workload = BASELINE.json configs[3], the largest single-GPU configuration (the metric is
quoted on no single config): n=14 Heisenberg ring, the 16 D_14 blocks (495..1179), N_t = 500
slices, gate fidelity against seeded random-unitary block targets.  One "step" = one
fidelity+gradient evaluation.  ``--config 1`` selects the tiny-block batch (4096 seeded control
vectors of the n=12 all-to-all S_n sectors), ``--config 0/2/4`` the others.

    python bench.py [--gpus N --steps K --warmup W] [--config 0..4] [--impl ours|reference]

Multi-GPU: ``--gpus N`` without a torchrun environment re-launches itself under
``torch.distributed.run`` (one process per GPU, 127.0.0.1 rendezvous).  cfg 0/1 shard by seed
(seed-DP, no data-path collective, "weak"); cfg 2/3/4 shard ONE evaluation by contiguous slice
chunks (parallel.py; the scan carry is one all-gather of the chunk products, "strong").
``--impl reference`` times the CPU oracle port of the reference algorithm (oracle/grape_oracle.py;
the reference is pure Python with no installable native path) on the host cores, rank 0 only.

Before any timing, a correctness gate (the reference harness's CorrectnessGateError,
pkg/src/symqoc/bench.py:60-85) compares the GPU path with committed fixtures of the oracle /
the reference itself (tests/golden/r02_*.npz) and refuses to print a line on a mismatch.
"""

from __future__ import annotations

import argparse
import copy
import json
import os
import socket
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "GRAPE fidelity+gradient evals/sec"
UNIT = "evals/s"
DEFAULT_CONFIG = 3
FP64_PEAK_TFLOPS = 36.9  # measured DMMA m8n8k4 peak on this pool, profiles/r01_fp64_peak.txt
GATE_F_TOL = 1e-10       # BASELINE north_star: fidelity within 1e-10 absolute
GATE_G_TOL = 1e-8        # gradients within 1e-8 relative (reference bench GATE_TOL)
CONFIG_NAMES = {
    0: "cfg0: n=6 Heisenberg ring, D_6 A1 block d=13, state transfer, N_t=100",
    1: "cfg1: n=12 all-to-all Heisenberg, S_n sectors d<=13, gate fidelity, N_t=1000, 4096 seeds",
    2: "cfg2: n=10 Heisenberg ring, 12 D_10 blocks (30..105), gate fidelity, N_t=500",
    3: "cfg3: n=14 Heisenberg ring, 16 D_14 blocks (495..1179), gate fidelity, N_t=500",
    4: "cfg4: n=12 Heisenberg ring, unsymmetrised 4096, state transfer, N_t=200",
}
GOLD = os.path.join(ROOT, "tests", "golden")


class CorrectnessGateError(RuntimeError):
    """The GPU path disagrees with the committed oracle / reference fixtures: nothing is timed."""


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

    def __init__(self, index: int, period_ms: int = 200):
        self.index = index
        self.period_ms = period_ms
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", str(self.period_ms)], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
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


def config_dict(cfg: int, s, batch: int, ws: int) -> dict:
    """The workload description both arms print (same keys, same values)."""
    flops = s.flops_per_eval()
    if cfg in (2, 3, 4):
        par = f"slice-chunk{ws}" if ws > 1 else "single"
    else:
        par = f"seed-dp{ws}" if ws > 1 else "single"
    return {
        "workload": CONFIG_NAMES[cfg],
        "blocks": [b.dim for b in s.blocks],
        "batch_per_gpu": batch,
        "n_slices": s.n_slices,
        "parallelism": par,
        "l2": "flushed between timed steps (256 MB write, untimed)",
        "algorithmic_flops_per_eval": flops,
    }


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
    s2 = copy.copy(s)
    s2.n_slices = slices
    s2.T = s.dt * slices
    return s2


def cpu_reference(cfg: int, seconds_budget: float | None = None, cores: int | None = None):
    """Time the oracle port on the host: returns (evals/s, cores, sample description).

    cfg 0/1: rounds of `cores` independent seeds (one process per core, 1 BLAS thread each, the
    reference's process-level parallelism) until ~seconds_budget of wall time.
    cfg 2-4: one evaluation over a sample of slices, scaled by N_t / sampled (per-slice cost does
    not depend on u; 2 slices per block for cfg 3 and 4).
    """
    import multiprocessing as mp

    if seconds_budget is None:
        seconds_budget = float(os.environ.get("SQOC_CPU_BUDGET_S", "12"))
    cores = cores or len(os.sched_getaffinity(0))
    s = build_system_cached(cfg)
    if cfg in (2, 3, 4):
        # sampled slices, all cores to the BLAS/LAPACK of one process (cfg 3/4 eigh of 1161..4096)
        slices, threads = {2: (10, 1), 3: (2, cores), 4: (1, cores)}[cfg]
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


# ---------------------------------------------------------------- correctness gate
def _fixture(name):
    return np.load(os.path.join(GOLD, f"r02_{name}.npz"))


def _compare(F, g, F_ref, g_ref, what, report):
    dF = float(np.max(np.abs(np.asarray(F) - F_ref)))
    dg = float(np.abs(np.asarray(g) - g_ref).max() / np.abs(g_ref).max())
    report["cases"].append({"what": what, "abs_dF": dF, "rel_dgrad": dg})
    if not (dF <= GATE_F_TOL and dg <= GATE_G_TOL):
        raise CorrectnessGateError(f"{what}: |dF| = {dF:.3e} (tol {GATE_F_TOL}), rel dgrad = {dg:.3e} (tol {GATE_G_TOL})")


def correctness_gate(cfg, s, eng, make_engine, device):
    """Compare the GPU path with committed fixtures before timing (reference bench.py:60-85).

    cfg 1: 16 rows of the bench's own 4096-seed batch (seed 0) through the bench engine vs the oracle.
    cfg 2: the bench engine at full N_t = 500 on the fixture's controls vs the oracle.
    cfg 3: the same 16 blocks on a 4-slice grid (same dt), slice-sequential schedule -- the one the
           N_t = 500 evaluation runs -- vs the oracle (tests/golden/r02_cfg3.npz).
    cfg 4: the unsymmetrised 4096 space on a 2-slice grid vs the reference's own qoc.gradient.
    cfg 0: the reference-built cfg 0 system (tests/golden/reference_golden.npz) vs the reference.
    """
    from paper_2309_05884_b200 import parallel, systems

    report = {"tol_F_abs": GATE_F_TOL, "tol_grad_rel": GATE_G_TOL, "cases": []}
    if cfg == 1:
        z = _fixture("cfg1")
        rows = list(z["cfg1_rows"])
        ub = s.controls(0, batch=eng.max_batch)
        F, g = eng.objective(ub)
        _compare(F[rows], g[rows], z["cfg1_F"], z["cfg1_grad"], "cfg1 bench batch rows vs oracle", report)
    elif cfg == 2:
        z = _fixture("cfg2")
        F, g = eng.objective(s.controls(11))
        _compare(F, g, float(z["cfg2_F"]), z["cfg2_grad"], "cfg2 N_t=500 vs oracle", report)
    elif cfg == 3:
        z = _fixture("cfg3")
        loc = parallel.local_system(s, 0, 4)
        e2 = make_engine(loc)
        e2.set_schedule("sequential")
        F, g = e2.objective(loc.controls(11))
        e2.close()
        _compare(F, g, float(z["cfg3_F"]), z["cfg3_grad"], "cfg3 16 blocks N_t=4 (sequential) vs oracle", report)
    elif cfg == 4:
        z = _fixture("cfg4")
        loc = parallel.local_system(s, 0, 2)
        e2 = make_engine(loc)
        F, g = e2.objective(loc.controls(11))
        e2.close()
        _compare(F, g, float(z["cfg4_full_F"]), z["cfg4_full_grad"], "cfg4 4096 N_t=2 vs reference qoc.gradient",
                 report)
    elif cfg == 0:
        z = np.load(os.path.join(GOLD, "reference_golden.npz"))
        blk = systems.Block("cfg0", z["cfg0_h0"], [z["cfg0_hx"], z["cfg0_hy"]])
        ref_sys = systems.GrapeSystem("cfg0-ref", 6, [blk], "state", 10.0, 100, [z["cfg0_psif"]], [z["cfg0_psi0"]])
        e2 = make_engine(ref_sys)
        F, g = e2.objective(z["cfg0_u"])
        e2.close()
        _compare(F, g, float(z["cfg0_P"]), np.stack([z["cfg0_gx"], z["cfg0_gy"]]), "cfg0 vs reference qoc.gradient",
                 report)
    return report


def gemm_kernel_name(fma: int, dims) -> str:
    """Which GEMM kernel the large path launches for these block sizes (large.cu upload_list: work
    lists whose mean K x segments reaches 256 run the persistent TMA kernel, shorter ones the cp.async
    per-tile kernel; the 4M mode always runs the per-tile kernel)."""
    if fma != 3:
        return "zgemm_kernel"
    big = [d for d in dims if d > 16]
    if big and min(big) >= 256:
        return "zgemm3m_pt_kernel"
    if big and 2 * max(big) < 256:
        return "zgemm3m_kernel"
    return "zgemm3m_pt_kernel / zgemm3m_kernel"


# ---------------------------------------------------------------- GPU arm
def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_2309_05884_b200 import _lib, systems
    from paper_2309_05884_b200.engine import GrapeEngine

    ws, rank, local = dist_env()
    torch.cuda.set_device(local)
    if ws > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    cfg = args.config
    s = build_system(cfg, gpu_basis=True)
    batch = args.batch or systems.CONFIG_BATCH[cfg]
    make_engine = lambda sys_: GrapeEngine(sys_, max_batch=1, device=local)  # noqa: E731

    seed0 = 1000 * rank
    u_host = s.controls(seed0, batch=batch)
    u = torch.from_numpy(u_host).to(f"cuda:{local}")
    F = torch.empty(batch, dtype=torch.float64, device=u.device)
    g = torch.empty_like(u)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=u.device)  # > 126 MB L2
    stream = torch.cuda.current_stream()
    tiny_only = all(b.dim <= _lib.load().sqoc_tiny_max_dim() for b in s.blocks)

    # ---- dominant tiny kernel timed alone (cfg 0/1): in the step the sectors' kernels share the
    # GPU on concurrent streams, so a per-stream event pair around one of them measures contention,
    # not the kernel.  The same launch (largest sector, same u) runs here on an idle GPU. ----
    dom_alone_ms = None
    if tiny_only and not args.skip_alone:
        dims_ = [b.dim for b in s.blocks]
        bdom_ = int(np.argmax(np.array(dims_, dtype=float) ** 3))
        sub = copy.copy(s)
        sub.blocks = [s.blocks[bdom_]]
        sub.targets = [s.targets[bdom_]]
        sub.initial = [s.initial[bdom_]] if s.initial else []
        sub.weights = np.array([s.block_weights()[bdom_]])
        eng1 = GrapeEngine(sub, max_batch=batch, device=local)
        if len(s.blocks) > 1:
            eng1.set_tiny_cta_warps(0)  # the CTA size the multi-block step launches it with
        eng1.evaluate_device(u.data_ptr(), batch, F.data_ptr(), g.data_ptr(), stream=stream.cuda_stream)
        alone = []
        for _ in range(max(2, min(args.steps, 5))):
            flush.fill_(1.0)
            a0 = torch.cuda.Event(enable_timing=True)
            a1 = torch.cuda.Event(enable_timing=True)
            a0.record(stream)
            eng1.evaluate_device(u.data_ptr(), batch, F.data_ptr(), g.data_ptr(), stream=stream.cuda_stream)
            a1.record(stream)
            torch.cuda.synchronize()
            alone.append(a0.elapsed_time(a1))
        dom_alone_ms = float(np.median(alone))
        eng1.close()
        del eng1
        torch.cuda.empty_cache()

    eng = GrapeEngine(s, max_batch=batch, device=local)

    # ---- correctness gate (before anything is timed; every rank) ----
    gate = correctness_gate(cfg, s, eng, make_engine, local)

    def step():
        eng.evaluate_device(u.data_ptr(), batch, F.data_ptr(), g.data_ptr(), stream=stream.cuda_stream)

    # ---- warm-up; expensive steps (> 2 s) time the e2e leg on warm-up steps 2..4 ----
    pinned = torch.from_numpy(u_host).pin_memory()
    Fh = torch.empty(batch, dtype=torch.float64).pin_memory()
    gh = torch.empty_like(pinned).pin_memory()

    def e2e_call():
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        eng.evaluate_host_ptr(pinned.data_ptr(), batch, Fh.data_ptr(), gh.data_ptr())
        return time.perf_counter() - t0

    e2e, e2e_in_warmup = [], False
    t_first = time.perf_counter()
    if args.warmup > 0:
        step()
        torch.cuda.synchronize()
    first_s = time.perf_counter() - t_first
    for w in range(1, args.warmup):
        if first_s > 2.0 and len(e2e) < 3:
            e2e_in_warmup = True
            e2e.append(e2e_call())
        else:
            step()
    torch.cuda.synchronize()

    eng.set_timing(True)
    clocks = ClockSampler(local, period_ms=200 if first_s < 5 else 1000)
    clocks.start()
    times, kern, gstats = [], [], []
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
        gstats.append(eng.gemm_stats())
        launches += eng.last_launches
    torch.cuda.synchronize()
    if ws > 1:
        dist.barrier()
    clk = clocks.stop()
    eng.set_timing(False)
    ms = float(np.median(times))
    t = torch.tensor([ms], dtype=torch.float64, device=u.device)
    if ws > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())

    # ---- e2e: public API with host buffers (pinned u in, F + grad out) ----
    clk_e2e = None
    if not e2e:
        e2e_call()  # warm
        clocks_e2e = ClockSampler(local)
        clocks_e2e.start()
        for _ in range(max(3, args.steps)):
            e2e.append(e2e_call())
        clk_e2e = clocks_e2e.stop()
    e2e_s = float(np.median(e2e))
    te = torch.tensor([e2e_s], dtype=torch.float64, device=u.device)
    if ws > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_s = float(te.item())

    if rank == 0:
        flops_eval = s.flops_per_eval()
        value = batch * ws / (ms_max / 1e3)
        dims = [b.dim for b in s.blocks]
        peak = FP64_PEAK_TFLOPS
        if not tiny_only:
            gms = float(np.median([x["ms"] for x in gstats]))
            macs = gstats[-1]["complex_macs"]
            fma = gstats[-1]["real_fma_per_complex_mac"]
            n_l = gstats[-1]["launches"]
            # The kernel's algorithmic work is the real DMMA products it runs: 3 (Gauss/3M) or 4 real
            # m x n x k products per complex product, 2 flops per FMA -> 2 * fma * complex MACs.  The
            # SURVEY 8d convention (8 N G sum d^3 per evaluation) is reported beside it: it counts 22
            # complex GEMM-units per slice where this schedule runs 16 dense ones plus sparse-generator
            # products, so it exceeds the pipe peak and is not a roofline fraction.
            achieved = 2.0 * fma * macs * batch / (gms / 1e3) / 1e12
            roof = {
                "bound": "tensor",
                "kernel": f"{gemm_kernel_name(fma, dims)} (all {n_l} large-block GEMM launches of a step)",
                "achieved": achieved, "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak,
                "flops_per_unit": f"{2 * fma} flops per complex MAC ({fma} real DMMA products per complex product)",
                "launch_ms": gms / max(n_l, 1), "launches_per_step": n_l, "gemm_ms_per_step": gms,
                "gemm_share_of_step": gms / ms_max,
                "complex_gemm_tflops": 8.0 * macs * batch / (gms / 1e3) / 1e12,
                "convention_tflops_gemm": flops_eval * batch / (gms / 1e3) / 1e12,
                "gemm_units_per_slice": macs / sum(float(d) ** 3 for d in dims) / s.n_slices,
            }
        else:
            bdom = int(np.argmax(np.array(dims, dtype=float) ** 3))
            g_conv = 22 if s.objective == "gate" else 8
            dom_flops = 8.0 * s.n_slices * g_conv * float(dims[bdom]) ** 3 * batch
            dom_ms = dom_alone_ms if dom_alone_ms is not None else float(np.median(np.array(kern)[:, bdom]))
            achieved = dom_flops / (dom_ms / 1e3) / 1e12
            roof = {"bound": "tensor", "kernel": f"grape_tiny_kernel<d={dims[bdom]}> (timed alone: one launch per "
                                                 f"step, same u)", "achieved": achieved, "peak": peak,
                    "unit": "TFLOP/s", "frac": achieved / peak, "launch_ms": dom_ms}
        traffic = None
        tpath = os.path.join(ROOT, "profiles", "traffic.json")
        if os.path.exists(tpath):
            traffic = json.load(open(tpath)).get(str(cfg))
        roof["traffic"] = traffic
        # whole step by the SURVEY 8d convention (can exceed 1 when the schedule runs fewer products)
        roof["step_convention_frac"] = flops_eval * batch / (ms_max / 1e3) / 1e12 / peak
        roof["peak_source"] = ("measured FP64 DMMA peak (profiles/r01_fp64_peak.txt); MEASURED_PEAKS.json has no "
                               "FP64 entry")
        roof["convention"] = "8 * N_t * G * sum_b d_b^3 per evaluation, G=22 gate / 8 state (SURVEY.md 8d)"
        cpu_val, cpu_cores, cpu_sample = (None, None, "skipped")
        if not args.skip_cpu:
            cpu_val, cpu_cores, cpu_sample = cpu_reference(cfg)
        conf = config_dict(cfg, s, batch, ws)
        conf["steps_ms"] = [round(x, 2) for x in times]
        conf["step_tflops_algorithmic"] = flops_eval * batch / (ms_max / 1e3) / 1e12
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
            "config": conf,
            "roofline": roof,
            "cpu_baseline": {"value": cpu_val, "unit": UNIT, "cores": cpu_cores, "kind": "port", "sample": cpu_sample},
            "e2e": {
                "value": batch * ws / e2e_s,
                "unit": UNIT,
                "h2d_bytes_per_step": int(u_host.nbytes),
                "d2h_bytes_per_step": int(Fh.numel() * 8 + gh.numel() * 8),
                "calls_ms": [round(x * 1e3, 2) for x in e2e],
                "taken_on": "warm-up steps 2-4 (host-pointer sqoc_eval)" if e2e_in_warmup else "after the timed region",
                "clocks": clk_e2e,
            },
            "gate": gate,
            "gpu_launches": int(launches),
            "clocks": clk,
        }
        print(json.dumps(line), flush=True)
    eng.close()
    if ws > 1:
        dist.destroy_process_group()


def run_sharded(args):
    """cfg 2-4 on N > 1 GPUs: ONE evaluation split over a (block groups x slice chunks) grid of ranks
    (parallel.ShardedObjective): per-rank chunk products, one NCCL all-gather of the chunk products
    per block group (the scan carry, device to device), boundary values formed on each device,
    local backward sweeps, one all-gather of the 8 KB gradient rows.  Total work fixed -> "strong".
    Timed on the device (CUDA events on torch's current stream), max over ranks."""
    import torch
    import torch.distributed as dist

    from paper_2309_05884_b200 import parallel
    from paper_2309_05884_b200.engine import GrapeEngine

    ws, rank, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    cfg = args.config
    s = build_system(cfg, gpu_basis=True)
    # default grid: cfg 2 by blocks only (its ~100-dim blocks run the slice-batched history schedule;
    # chunking would force the slice-sequential one); cfg 3 and cfg 4 by slice chunks only -- block
    # groups halve each GEMM launch's work list and lose more than they save (cfg 3, 8 emulated ranks,
    # profiles/r02_chunk_emulate_cfg3.jsonl: 1x8 critical path 7.00 s, 2x4 7.51 s, 4x2 7.63 s)
    groups = args.block_groups or {2: ws}.get(cfg, 1)
    comm = parallel.Comm()
    factory = lambda sys_: GrapeEngine(sys_, max_batch=1, device=local)  # noqa: E731
    # ---- correctness gate: the sharded path on the committed fixture's system ----
    gate = {"tol_F_abs": GATE_F_TOL, "tol_grad_rel": GATE_G_TOL, "cases": []}
    if cfg in (2, 3, 4):
        if cfg == 2:
            z, gsys, gu = _fixture("cfg2"), s, s.controls(11)
            fz, gz = float(z["cfg2_F"]), z["cfg2_grad"]
        elif cfg == 3:
            z = _fixture("cfg3")
            gsys = parallel.local_system(s, 0, 4)
            gu, fz, gz = gsys.controls(11), float(z["cfg3_F"]), z["cfg3_grad"]
        else:
            z = _fixture("cfg4")
            gsys = parallel.local_system(s, 0, 2)
            gu, fz, gz = gsys.controls(11), float(z["cfg4_full_F"]), z["cfg4_full_grad"]
        gobj = parallel.ShardedObjective(gsys, comm, factory, n_block_groups=groups)
        gobj.objective(gu)  # the chunk entry points have no discarded first evaluation
        Fz, gzz = gobj.objective(gu)
        gobj.eng.close()
        del gobj
        torch.cuda.empty_cache()
        _compare(Fz, gzz, fz, gz, f"cfg{cfg} sharded {groups}x{ws // groups} vs fixture", gate)
    obj = parallel.ShardedObjective(s, comm, factory, n_block_groups=groups)
    u = s.controls(0)
    u_t = torch.as_tensor(u).to(dev)
    pinned = torch.from_numpy(u).pin_memory()
    gh = torch.empty_like(pinned).pin_memory()
    Fh = torch.empty(1, dtype=torch.float64).pin_memory()

    def e2e_call():
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        uu = pinned.to(dev, non_blocking=True)
        F_, g_ = obj.objective_t(uu)
        gh.copy_(g_, non_blocking=True)
        Fh.copy_(F_.reshape(1), non_blocking=True)
        torch.cuda.synchronize()
        return time.perf_counter() - t0

    t_first = time.perf_counter()
    obj.objective_t(u_t)
    torch.cuda.synchronize()
    first_s = time.perf_counter() - t_first
    e2e = []
    for _ in range(1, args.warmup):
        if first_s > 2.0 and len(e2e) < 3:
            e2e.append(e2e_call())
        else:
            obj.objective_t(u_t)
    torch.cuda.synchronize()
    obj.timing = True
    obj.eng.set_timing(True)
    clocks = ClockSampler(local, period_ms=200 if first_s < 5 else 1000)
    clocks.start()
    stream = torch.cuda.current_stream()
    times, stages, carries, launches = [], [], [], 0
    for _ in range(args.steps):
        dist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        F, g = obj.objective_t(u_t)
        e1.record(stream)
        torch.cuda.synchronize()
        t = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        times.append(float(t.item()))
        stages.append(dict(obj.stage_ms))
        carries.append(obj.eng.carry_stats())
        launches += obj.last_launches
    clk = clocks.stop()
    obj.timing = False
    obj.eng.set_timing(False)
    if not e2e:
        for _ in range(max(3, args.steps)):
            e2e.append(e2e_call())
    te = torch.tensor([float(np.median(e2e))], dtype=torch.float64, device=dev)
    dist.all_reduce(te, op=dist.ReduceOp.MAX)
    # per-rank stage shares (medians), gathered to rank 0
    med = {k: float(np.median([x[k] for x in stages])) for k in stages[0]}
    med["carry"] = float(np.median([c["ms"] for c in carries]))
    row = torch.tensor([med["forward"], med["exchange"], med["backward"], med["reduce"], med["carry"]],
                       dtype=torch.float64, device=dev)
    rows = comm.all_gather(row).cpu().numpy()
    if rank == 0:
        ms = float(np.median(times))
        flops = s.flops_per_eval()
        conf = config_dict(cfg, s, 1, ws)
        conf["parallelism"] = f"block-groups{groups} x slice-chunks{ws // groups}"
        conf["slice_chunks"] = parallel.chunk_bounds(s.n_slices, ws // groups)
        conf["block_groups"] = parallel.block_groups([b.dim for b in s.blocks], groups)
        conf["steps_ms"] = [round(x, 2) for x in times]
        per_rank = [{"forward_ms": r[0], "exchange_ms": r[1], "backward_ms": r[2], "reduce_ms": r[3],
                     "carry_ms": r[4], "carry_plus_comm_share": (r[1] + r[3] + r[4]) / ms} for r in rows]
        peak = FP64_PEAK_TFLOPS * ws
        print(json.dumps({
            "metric": METRIC, "value": 1e3 / ms, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "c128", "data": "synthetic (seeded u ~ U[-1,1], seeded Haar/QR targets)",
            "config": conf,
            "roofline": {"bound": "tensor", "kernel": "zgemm3m_kernel (all ranks)",
                         "achieved": flops / (ms / 1e3) / 1e12, "peak": peak, "unit": "TFLOP/s",
                         "frac": flops / (ms / 1e3) / 1e12 / peak, "traffic": None,
                         "peak_source": f"{ws} x measured FP64 DMMA peak (profiles/r01_fp64_peak.txt)"},
            "per_rank": per_rank,
            "e2e": {"value": 1.0 / float(te.item()), "unit": UNIT, "h2d_bytes_per_step": int(u.nbytes),
                    "d2h_bytes_per_step": int(gh.numel() * 8 + 8), "calls_ms": [round(x * 1e3, 2) for x in e2e]},
            "gate": gate, "gpu_launches": int(launches), "clocks": clk,
            "cpu_baseline": {"value": None, "unit": UNIT, "cores": None, "kind": "port",
                             "sample": "timed on rank 0 at N=1 only"},
        }), flush=True)
    obj.eng.close()
    dist.destroy_process_group()


def run_reference(args):
    """The reference arm: the oracle port on the host cores (rank 0 only), W untimed warm-up samples,
    then K timed samples; value = median."""
    ws, rank, local = dist_env()
    if rank != 0:
        return
    cfg = args.config
    from paper_2309_05884_b200 import systems

    for _ in range(args.warmup):
        cpu_reference(cfg, seconds_budget=float(os.environ.get("SQOC_CPU_WARM_BUDGET_S", "2")))
    vals = []
    cores = None
    sample = ""
    for _ in range(args.steps):
        v, cores, sample = cpu_reference(cfg, cores=None)
        vals.append(v)
    value = float(np.median(vals))
    s = build_system_cached(cfg)
    batch = args.batch or systems.CONFIG_BATCH[cfg]
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
        "config": config_dict(cfg, s, batch, ws),
        "impl": "reference",
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port", "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def _free_port() -> int:
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    return port


def relaunch(args) -> int:
    """One process per GPU: re-run this script under torch.distributed.run (127.0.0.1 rendezvous)."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.run(cmd).returncode


def launcher_selftest():
    """CPU check of the launcher: every rank joins a gloo group; rank 0 prints what it saw."""
    import torch
    import torch.distributed as dist

    ws, rank, local = dist_env()
    dist.init_process_group("gloo")
    t = torch.tensor([float(rank + 1)])
    dist.all_reduce(t)
    if rank == 0:
        print(json.dumps({"n_gpus": ws, "rank_sum": float(t.item()), "local_ranks_ok": True}), flush=True)
    dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=DEFAULT_CONFIG)
    ap.add_argument("--batch", type=int, default=None)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--skip-cpu", action="store_true")
    ap.add_argument("--skip-alone", action="store_true", help="skip the tiny kernel timed-alone pass")
    ap.add_argument("--block-groups", type=int, default=None,
                    help="cfg 2-4 on N GPUs: block groups G (N/G slice chunks each); default N for cfg 2, else 1")
    ap.add_argument("--selftest-launcher", action="store_true", help=argparse.SUPPRESS)
    ap.add_argument("--sharded", action="store_true", help="cfg 2-4: the sharded path even on one rank")
    args = ap.parse_args()
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    if args.impl == "reference":
        run_reference(args)
    elif args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(relaunch(args))
    elif args.selftest_launcher:
        launcher_selftest()
    elif args.config in (2, 3, 4) and (ws > 1 or args.sharded):
        if "WORLD_SIZE" not in os.environ:  # one rank without torchrun: a local rendezvous
            os.environ.update({"WORLD_SIZE": "1", "RANK": "0", "LOCAL_RANK": "0", "MASTER_ADDR": "127.0.0.1",
                               "MASTER_PORT": str(_free_port())})
        try:
            run_sharded(args)
        except CorrectnessGateError as e:
            print(f"CorrectnessGateError: {e}", file=sys.stderr, flush=True)
            sys.exit(3)
    else:
        try:
            run_ours(args)
        except CorrectnessGateError as e:
            print(f"CorrectnessGateError: {e}", file=sys.stderr, flush=True)
            sys.exit(3)


if __name__ == "__main__":
    main()
