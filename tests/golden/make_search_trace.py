"""Writes tests/golden/search_trace.json: a hand-checkable trace of the hobo_search move rule
("Proposed hobo_search rule"; reading 14) on a 4-variable instance.

Everything here is written from the rule text and the generator spec; it calls
nothing under oracle/ or the product.  Energies come from the polynomial written out as a sum
of monomials and evaluated at every one of the 16 states; the field is the definition
g_m = E(x | x_m <- 1) - E(x | x_m <- 0) on that table.

Rule (per chain c, iteration t in [0, iters)):
  1. evaluate E(x), update best_c if E < best_c (strict: on equal E the earliest t is kept)
  2. Delta_m = (1 - 2 x_m) g_m
  3. r = h(seed, 2, c, t); mrand = ((r & 0xffffffff) * N) >> 32
  4. if (r >> 32) < P_t: m* = mrand                                   ("explore")
     else m* = argmin_m Delta_m (lowest m on ties)                    ("greedy")
          and if Delta_{m*} >= 0: m* = mrand                          ("stuck")
  5. flip x_{m*}
After the loop the final state is evaluated once more.  Chain c starts at
x_m = bit (m & 63) of h(seed, 1, c, m >> 6).  P_t = floor(2^32 p0 (p1/p0)^(t / max(1, iters-1))).

p0 is chosen so that P_0 equals chain 0's (r >> 32) at t = 0 EXACTLY: the strict "<" then
sends that draw to the greedy branch (a "<=" would explore).  The instance, seed and p1 were
picked (by the search at the bottom) so that the 2 chains x 4 iterations cover every branch:
explore, greedy with a tie at the minimum (lowest m wins), stuck (Delta_min >= 0 -> random),
the P_t boundary, and an equal-energy revisit of a different state (the earliest is kept).

    python tests/golden/make_search_trace.py   # rewrites search_trace.json
"""
import itertools
import json
import math
import os

M64 = (1 << 64) - 1


def splitmix64(z):
    z = (z + 0x9E3779B97F4A7C15) & M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    return z ^ (z >> 31)


def h(s, a, b, c):
    return splitmix64(splitmix64(splitmix64(s ^ a) ^ b) ^ c)


def energy(monos, x):
    return sum(c for c, S in monos if all(x[u] for u in S))


def thresholds(iters, p0, p1):
    out = []
    for t in range(iters):
        v = math.floor(4294967296.0 * p0 * math.pow(p1 / p0, t / max(1, iters - 1)))
        out.append(int(min(4294967295, max(0, v))))
    return out


def trace(monos, N, seed, nchains, iters, p0, p1):
    P = thresholds(iters, p0, p1)
    chains = []
    for c in range(nchains):
        x = [(h(seed, 1, c, m >> 6) >> (m & 63)) & 1 for m in range(N)]
        best, xbest, steps = math.inf, None, []
        for t in range(iters + 1):
            E = energy(monos, x)
            step = {"t": t, "x": list(x), "E": E}
            if E < best:
                best, xbest = E, list(x)
            if t == iters:
                steps.append(step)
                break
            g = [energy(monos, [1 if u == m else x[u] for u in range(N)]) -
                 energy(monos, [0 if u == m else x[u] for u in range(N)]) for m in range(N)]
            D = [(1 - 2 * x[m]) * g[m] for m in range(N)]
            r = h(seed, 2, c, t)
            mrand = ((r & 0xFFFFFFFF) * N) >> 32
            dmin = min(D)
            if (r >> 32) < P[t]:
                branch, ms = "explore", mrand
            else:
                ms = D.index(dmin)                  # lowest m on ties
                branch = "greedy" if dmin < 0 else "stuck"
                if dmin >= 0:
                    ms = mrand
            step.update(g=g, Delta=D, r=f"{r:016x}", r_hi=r >> 32, P_t=P[t], mrand=mrand, branch=branch,
                        tie_at_min=D.count(dmin) > 1, m_star=ms)
            steps.append(step)
            x[ms] ^= 1
        chains.append({"chain": c, "steps": steps, "E_best": best, "x_best": xbest})
    return P, chains


def coverage(chains, P0_boundary_chain0):
    st = [s for ch in chains for s in ch["steps"] if "branch" in s]
    cov = {
        "explore": any(s["branch"] == "explore" for s in st),
        "greedy_tie": any(s["branch"] == "greedy" and s["tie_at_min"] for s in st),   # lowest m != highest m
        "stuck": any(s["branch"] == "stuck" for s in st),
        "boundary": P0_boundary_chain0,
    }
    # an equal-energy revisit of a different state at the best level (earliest kept)
    eq = False
    for ch in chains:
        seen = [(s["E"], tuple(s["x"])) for s in ch["steps"]]
        lvl = [xs for e, xs in seen if e == ch["E_best"]]
        eq = eq or len(set(lvl)) > 1
    cov["equal_E_revisit"] = eq
    return cov


def build(monos, N, seed, p1_ratio, iters=4, nchains=2):
    r0 = h(seed, 2, 0, 0)
    p0 = (r0 >> 32) / 4294967296.0                 # P_0 == r_hi of chain 0 at t = 0, exactly
    p1 = p0 * p1_ratio
    P, chains = trace(monos, N, seed, nchains, iters, p0, p1)
    boundary = P[0] == (r0 >> 32) and chains[0]["steps"][0]["branch"] != "explore"
    return p0, p1, P, chains, coverage(chains, boundary)


INSTANCES = [
    # (name, monomials) : f = sum c * prod x  (4 binary variables, integer coefficients)
    ("sym4", [(-1, (0,)), (-1, (1,)), (-1, (2,)), (-1, (3,)), (2, (0, 1)), (2, (2, 3)), (1, (0, 2)), (1, (1, 3))]),
    ("ring4", [(-2, (0,)), (-2, (1,)), (-2, (2,)), (-2, (3,)), (3, (0, 1)), (3, (1, 2)), (3, (2, 3)), (3, (0, 3)),
               (1, (0, 1, 2))]),
    ("cube4", [(-1, (0,)), (-1, (1,)), (-1, (2,)), (-1, (3,)), (1, (0, 1)), (1, (2, 3)), (2, (0, 1, 3)),
               (-1, (1, 2, 3))]),
]


def search():
    for (name, monos), seed, ratio in itertools.product(INSTANCES, range(1, 400), (0.5, 0.25, 1.0)):
        p0, p1, P, chains, cov = build(monos, 4, seed, ratio)
        if all(cov.values()):
            return name, monos, seed, p0, p1, P, chains, cov
    raise SystemExit("no instance covers every branch")


def main():
    name, monos, seed, p0, p1, P, chains, cov = search()
    table = {"".join(map(str, x)): energy(monos, x) for x in itertools.product((0, 1), repeat=4)}
    out = {
        "_about": ("hobo_search move rule (SURVEY 8(c) O8, DESIGN.md reading 14), hand-checkable: written by "
                   "tests/golden/make_search_trace.py from the rule text and the SURVEY 8(d) hash; it calls "
                   "nothing under oracle/ or the product.  'x' strings in energy_table are x0x1x2x3."),
        "instance": name, "N": 4, "order": max(len(S) for _, S in monos),
        "monomials": [[c, list(S)] for c, S in monos],
        "energy_table": table,
        "seed": seed, "iters": 4, "nchains": 2, "p0": p0, "p1": p1, "P": P,
        "coverage": cov, "chains": chains,
    }
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "search_trace.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=1)
    print(name, seed, cov)


if __name__ == "__main__":
    main()
