"""bench.py contract pieces that run without a GPU: the reference arm and its JSON line."""

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    env = dict(os.environ, SQOC_CPU_BUDGET_S="0.5")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "0",
                          "--steps", "1", "--warmup", "0"], capture_output=True, text=True, env=env, timeout=600,
                         cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
                "vs_baseline", "dtype", "config", "impl", "cpu_baseline", "e2e"):
        assert key in line, key
    assert line["impl"] == "reference" and line["value"] > 0
    assert line["cpu_baseline"]["kind"] == "port" and line["cpu_baseline"]["cores"] >= 1
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["value"] == line["value"]


def test_cpu_reference_sampled_slices():
    sys.path.insert(0, ROOT)
    import bench

    v, cores, sample = bench.cpu_reference(2, seconds_budget=0.1)
    assert v > 0 and cores == 1 and "10 of 500 slices" in sample


def test_clock_sampler_parses_nvidia_smi_lines():
    sys.path.insert(0, ROOT)
    import bench

    class FakeProc:
        def terminate(self):
            pass

        def communicate(self, timeout=None):
            return ("1965, 1965, Not Active, Not Active, Not Active, Active\n"
                    "1950, 1965, Not Active, Not Active, Not Active, Not Active\n", "")

    c = bench.ClockSampler(0)
    c.proc = FakeProc()
    r = c.stop()
    assert r["sm_max_mhz"] == 1965 and r["reasons"] == ["sw_power_cap"] and r["samples"] == 2


def test_launcher_spawns_ranks_on_cpu():
    """`bench.py --gpus 2` outside torchrun re-launches itself with two ranks (gloo here)."""
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--selftest-launcher"],
                         capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["n_gpus"] == 2 and line["rank_sum"] == 3.0


def test_reference_arm_prints_the_same_config_as_ours():
    sys.path.insert(0, ROOT)
    import bench
    from paper_2309_05884_b200 import systems

    s = systems.config(0)
    c = bench.config_dict(0, s, 1, 1)
    assert c["workload"] == bench.CONFIG_NAMES[0] and c["blocks"] == [13] and c["n_slices"] == 100
    env = dict(os.environ, SQOC_CPU_BUDGET_S="0.3", SQOC_CPU_WARM_BUDGET_S="0.1")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "0",
                          "--steps", "2", "--warmup", "1"], capture_output=True, text=True, env=env, timeout=600,
                         cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["config"] == c and line["warmup"] == 1 and line["steps"] == 2


def test_default_config_is_the_largest_single_gpu_config():
    sys.path.insert(0, ROOT)
    import bench

    assert bench.DEFAULT_CONFIG == 3


def test_gate_compare_raises_on_mismatch():
    sys.path.insert(0, ROOT)
    import numpy as np
    import pytest

    import bench

    rep = {"cases": []}
    bench._compare(0.5, np.ones(3), 0.5 + 1e-12, np.ones(3) * (1 + 1e-10), "ok", rep)
    with pytest.raises(bench.CorrectnessGateError):
        bench._compare(0.5, np.ones(3), 0.5 + 1e-9, np.ones(3), "F off", rep)
    with pytest.raises(bench.CorrectnessGateError):
        bench._compare(0.5, np.ones(3), 0.5, np.ones(3) * (1 + 1e-6), "grad off", rep)


def test_gemm_kernel_name_follows_the_staging_rule():
    sys.path.insert(0, ROOT)
    import bench

    # large.cu upload_list: lists with mean K x segments >= 256 run the persistent TMA kernel
    assert bench.gemm_kernel_name(3, [687, 495, 1179]) == "zgemm3m_pt_kernel"
    assert bench.gemm_kernel_name(3, [30, 105, 13]) == "zgemm3m_kernel"  # tiny blocks (<= 16) never reach a GEMM
    assert bench.gemm_kernel_name(3, [4096]) == "zgemm3m_pt_kernel"
    assert bench.gemm_kernel_name(4, [4096]) == "zgemm_kernel"
    assert "/" in bench.gemm_kernel_name(3, [105, 1179])
