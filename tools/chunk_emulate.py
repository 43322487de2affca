"""Per-rank cost of the sharded evaluation, measured on ONE GPU by running every rank's stages in
turn (parallel.ShardedObjective with comm=None; the exchanges become local stacks).

For each (block groups G, chunks C) grid: device time of each rank's chunk forward, its chunk
backward and, inside that, the on-device carries (sqoc_last_carry_stats).  The slowest rank's
forward + backward is the compute critical path of a P-GPU step; the exchange itself cannot be
timed on one GPU and is reported as bytes per rank.

    python tools/chunk_emulate.py [--config 3] [--grids 1x8,2x4] [--slices N]
"""

from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2309_05884_b200 import parallel, systems  # noqa: E402
from paper_2309_05884_b200.engine import GrapeEngine  # noqa: E402


def timed(fn):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    out = fn()
    e1.record()
    torch.cuda.synchronize()
    return out, e0.elapsed_time(e1)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--grids", default="1x8,2x4")
    ap.add_argument("--slices", type=int, default=None)
    ap.add_argument("--single", action="store_true", help="also time the unsharded evaluation")
    args = ap.parse_args()
    kw = {"builder": "gpu"} if args.config in (2, 3) else {}
    if args.slices:
        kw["n_slices"] = args.slices
    s = systems.config(args.config, **kw)
    u = s.controls(0)
    u_t = torch.as_tensor(u).cuda()
    out = {"config": args.config, "n_slices": s.n_slices, "blocks": [b.dim for b in s.blocks], "grids": []}
    if args.single:
        eng = GrapeEngine(s, max_batch=1)
        eng.set_schedule("sequential")
        eng.objective(u)
        (_, ms1) = timed(lambda: eng.objective(u))
        out["single_ms"] = ms1
        eng.close()
        torch.cuda.empty_cache()
    for grid in args.grids.split(","):
        G, C = (int(x) for x in grid.split("x"))
        world = G * C
        # one rank's engine at a time (each keeps its chunk's propagator history: 8 ranks of cfg 3 do not
        # fit one GPU together): pass 1 times every rank's chunk forward and keeps the packed products,
        # pass 2 rebuilds each rank's forward state (untimed) and times its chunk backward
        def make(r):
            o = parallel.ShardedObjective(s, None, lambda x: GrapeEngine(x, max_batch=1), G, rank=r, world=world)
            o.eng.set_timing(True)
            return o

        fwd, packed = [], []
        for r in range(world):
            o = make(r)
            p, ms = timed(lambda: o.stage_forward(u_t))
            packed.append(p.clone())
            fwd.append(ms)
            o.eng.close()
            del o
            torch.cuda.empty_cache()
        bwd, carry, rows = [], [], []
        for r in range(world):
            o = make(r)
            o.stage_forward(u_t)
            gathered = torch.stack(packed[o.g * C:(o.g + 1) * C]) if C > 1 else None
            row, ms = timed(lambda: o.stage_backward(u_t, gathered))
            rows.append(row.clone())
            bwd.append(ms)
            carry.append(o.eng.carry_stats())
            o.eng.close()
            del o
            torch.cuda.empty_cache()
        tot = parallel.ShardedObjective.reduce_rows(torch.stack(rows))
        per = [f + b for f, b in zip(fwd, bwd)]
        crit = max(per)
        rec = {"grid": f"{G}x{C}", "forward_ms": fwd, "backward_ms": bwd, "carry_ms": [c["ms"] for c in carry],
               "carry_launches": [c["launches"] for c in carry], "rank_ms": per, "critical_path_ms": crit,
               "carry_share_of_critical": max(c["ms"] for c in carry) / crit,
               "exchange_bytes_per_rank": int(packed[0].numel() * 8 * (C - 1)) if C > 1 else 0, "F": float(tot[0].item())}
        if "single_ms" in out:
            rec["projected_efficiency_compute_only"] = out["single_ms"] / (world * crit)
        out["grids"].append(rec)
        print(json.dumps(rec), flush=True)
        del packed, rows
        torch.cuda.empty_cache()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
