"""The three-problems-per-warp lane tables in tiny.cuh are valid layouts and conflict-free
for every shared-memory access pattern of the kernel (bank-group model of tools/lane_maps.py)."""

import os
import re
import sys

import pytest

ROOT = os.path.join(os.path.dirname(__file__), "..")
sys.path.insert(0, os.path.join(ROOT, "tools"))
import lane_maps  # noqa: E402

SRC = open(os.path.join(ROOT, "paper_2309_05884_b200", "csrc", "tiny.cuh")).read()


def table(name, n):
    body = SRC[SRC.index(f"__constant__ unsigned char {name}"):]
    body = body[body.index("{") + 1:body.index("};")]
    rows = re.findall(r"\{([^}]*)\}", body)
    return [[int(x) for x in r.split(",")] for r in rows]


SIGMA = {3: 1, 5: 1, 6: 3, 9: 3}  # tiny_pad for three problems per warp


@pytest.mark.parametrize("mid,d", list(enumerate(lane_maps.DIMS)))
def test_lane_map(mid, d):
    lane_map = table("c_lane_map", 32)[mid]
    inv = table("c_lane_inv", 27)[mid]
    assert sorted(e for e in lane_map if e != 255) == list(range(27))
    assert all(lane_map[inv[e]] == e for e in range(27))
    for p in range(4):
        ph = [(e // 9, (e % 9) // 3, e % 3) for e in lane_map[8 * p:8 * p + 8] if e != 255]
        assert lane_maps.phase_ok(ph, d, SIGMA[d]), (d, p)
    m = re.search(r"\(d == 6 \|\| d == 9 \? 3 : 1\)", SRC)
    assert m, "tiny_pad sigma expression changed; update SIGMA"
