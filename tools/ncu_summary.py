"""Text summary of one `ncu --set full --import-source on` capture (run where ncu is installed).

python tools/ncu_summary.py REPORT.ncu-rep [title] > profiles/NAME.txt
Prints the launch, the headline metrics (duration, DRAM bytes, pipe activity, issue rate, stall reasons
per issued instruction, shared-memory wavefronts / bank conflicts, L2) from the raw page, and the SASS
instructions that collect the most warp-stall samples from the source page.
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
title = sys.argv[2] if len(sys.argv) > 2 else rep


def page(name, extra=()):
    out = subprocess.run(["ncu", "-i", rep, "--page", name, "--csv", *extra], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


raw = page("raw")
hdr, units, vals = raw[0], raw[1], raw[2]
m = {h: (u, v) for h, u, v in zip(hdr, units, vals)}


def show(key, label=None):
    if key in m:
        u, v = m[key]
        print(f"  {label or key:72s} {v} {u}")


print(f"# {title}")
print(f"# source: {rep} (ncu --set full --clock-control none; cold-cache, serialised launch)")
show("Kernel Name", "kernel")
show("launch__grid_size", "grid")
show("launch__block_size", "block")
show("launch__registers_per_thread", "registers / thread")
show("launch__shared_mem_per_block_dynamic", "dynamic smem / block")
print("-- time and memory")
for k in ("gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
          "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
          "lts__t_sector_hit_rate.pct", "l1tex__throughput.avg.pct_of_peak_sustained_elapsed"):
    show(k)
print("-- pipes and issue")
for k in ("sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
          "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
          "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_elapsed",
          "TPC.TriageCompute.sm__pipe_fp64_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
          "SM_C.TriageCompute.smsp__pipe_tensor_subpipe_dmma_cycles_active.avg", "sm__cycles_elapsed.avg",
          "sm__cycles_active.avg", "smsp__issue_active.avg.pct_of_peak_sustained_active",
          "smsp__warps_active.avg.per_cycle_active", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
          "smsp__inst_executed.sum"):
    show(k)
print("-- shared memory")
for k in ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum",
          "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
          "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed"):
    show(k)
print("-- warp stall reasons (cycles per issued instruction, > 0.05)")
for h in hdr:
    if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio") and "not_issued" not in h:
        try:
            v = float(m[h][1])
        except ValueError:
            continue
        if v > 0.05:
            print(f"  {h.split('stalled_')[1].split('_per_issue')[0]:28s} {v:.3f}")

src = page("source", ("--print-source", "sass"))
if len(src) > 3:
    sh = src[1]
    ix = {h: i for i, h in enumerate(sh)}
    data = [r for r in src[2:] if len(r) == len(sh)]
    if "# Samples" in ix:
        tot = sum(int(r[ix["# Samples"]]) for r in data) or 1
        print(f"-- SASS instructions with the most warp-stall samples (of {tot})")
        stall_cols = [h for h in sh if h.startswith("stall_") and "(" not in h]
        for r in sorted(data, key=lambda r: -int(r[ix["# Samples"]]))[:14]:
            n = int(r[ix["# Samples"]])
            top = sorted(((int(r[ix[c]]), c[6:]) for c in stall_cols), reverse=True)[:2]
            why = ", ".join(f"{c} {100 * v / max(n, 1):.0f}%" for v, c in top if v)
            print(f"  {100 * n / tot:5.1f}%  {r[ix['Source']].strip()[:58]:58s} {why}")
