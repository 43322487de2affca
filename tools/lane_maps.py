"""Search the lane layouts of the three-problems-per-warp tiny tiles (3 x 3 lane grid per problem).

LDS/STS.128 are served in 8-lane phases; a phase is conflict-free when its distinct 16-byte
addresses fall into distinct bank groups (address / 16 mod 8).  For problem s (buffer base
sigma * s mod 8 groups, sigma = the per-problem stride pad) and lane (tr, tc) of its 3 x 3 grid,
the kernel's shared accesses hit groups
    own entries   sigma s + D tr + tc      (load_own / add_poly / store / copy)
    A-operand     sigma s + D tr           (rows of L in L M)
    B-operand     sigma s + tc             (cols of M in L M)
    U^dag rows    sigma s + tr ;  seed    sigma s + D tc ;  shared generators  D tr + tc, D tc + tr
(plus per-instruction constants).  This script finds, per d in {3, 5, 6, 9}, a pad sigma and an
assignment of the 27 (s, tr, tc) lanes to the four 8-lane phases with no conflicts in any of
them, and prints the C tables used by tiny.cuh (entry = 9 s + 3 tr + tc, 255 = idle lane).
"""
import random

DIMS = (3, 5, 6, 9)


def groups(t, D, sig):
    s, tr, tc = t
    return [((sig * s + D * tr + tc) % 8, t), ((sig * s + D * tr) % 8, (s, tr)), ((sig * s + tc) % 8, (s, tc)),
            ((sig * s + tr) % 8, (s, tr)), ((sig * s + D * tc) % 8, (s, tc)), ((D * tr + tc) % 8, (tr, tc)),
            ((D * tc + tr) % 8, (tr, tc))]


def phase_ok(ph, D, sig):
    for a in range(7):
        seen = {}
        for t in ph:
            g, key = groups(t, D, sig)[a]
            if g in seen and seen[g] != key:
                return False
            seen[g] = key
    return True


def search(D, seed=1, tries=20000):
    rng = random.Random(seed)
    items = [(s, tr, tc) for s in range(3) for tr in range(3) for tc in range(3)]
    for sig in range(8):
        for _ in range(tries // 8):
            rng.shuffle(items)
            phases = [[], [], [], []]
            for it in items:
                order = [0, 1, 2, 3]
                rng.shuffle(order)
                for p in order:
                    if len(phases[p]) < 8 and phase_ok(phases[p] + [it], D, sig):
                        phases[p].append(it)
                        break
                else:
                    break
            else:
                return sig, phases
    return None


if __name__ == "__main__":
    for D in DIMS:
        sig, phases = search(D)
        table = [255] * 32
        for p, ph in enumerate(phases):
            for i, (s, tr, tc) in enumerate(sorted(ph)):
                table[8 * p + i] = 9 * s + 3 * tr + tc
        inv = [table.index(e) for e in range(27)]
        print(f"// d = {D}: pad sigma = {sig}")
        print("map {" + ", ".join(str(x) for x in table) + "},")
        print("inv {" + ", ".join(str(x) for x in inv) + "},")
