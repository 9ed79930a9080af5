"""Edge-case fixtures from the UNMODIFIED reference: non-finite and extreme
starts, tiny / huge tolerances, maxiters = 1, for every algorithm.

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_edges.py

Writes tests/golden/edges.npz with keys <case>/{u0,p,u,resid,retcode,nsteps,
nf,njac,nlinsolve} and <case>/opts = [abstol, maxiters]; the case list is
tests/golden/edges.json.  The reference decides every outcome (u_out of a
NonFinite start, counters of an already-converged start, ...).
"""

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
import make_golden as G  # noqa: E402

PROBLEMS = [("quadratic", 2), ("test23/rosenbrock", 2), ("test23/wood", 4),
            ("test23/helical-valley", 3), ("test23/trigonometric", 10),
            ("test23/chandrasekhar", 10), ("test23/boggs", 2)]
ALGS = ["newton-raphson", "trust-region", "broyden", "klement", "dfsane", "newton-backtracking"]
OPTS = [(1e-8, 1000), (1e-8, 1), (1e300, 5), (1e-300, 20)]


def starts(pid, n):
    base = np.asarray(G.W.problems.suite_start(pid.split("/", 1)[1]) if pid.startswith("test23/")
                      else np.ones(n), dtype=float)
    s = [base.copy()]
    for mod in ("nan0", "inf1", "ninf0", "huge", "tiny", "zero", "neg"):
        u = base.copy()
        if mod == "nan0":
            u[0] = np.nan
        elif mod == "inf1":
            u[min(1, n - 1)] = np.inf
        elif mod == "ninf0":
            u[0] = -np.inf
        elif mod == "huge":
            u[:] = 1e300
        elif mod == "tiny":
            u[:] = 1e-310
        elif mod == "zero":
            u[:] = 0.0
        else:
            u = -3.0 * base - 1.0
        s.append(u)
    return np.stack(s)


def main():
    import multiprocessing as mp
    out, cases = {}, []
    with mp.get_context("fork").Pool(os.cpu_count()) as pool:
        for pid, n in PROBLEMS:
            U = starts(pid, n)
            P = np.tile([2.0, 5.0], (len(U), 1)) if pid == "quadratic" else None
            for alg in ALGS:
                for abstol, maxiters in OPTS:
                    key = f"{pid}/{alg}/{abstol:g}/{maxiters}"
                    batch = G.W.Batch(pid, n, U, P, 0)
                    r = G.run_case(pool, batch, alg, abstol, maxiters, mask=False)
                    for k in ("u0", "p", "u", "resid", "retcode", "nsteps", "nf", "njac", "nlinsolve"):
                        out[f"{key}/{k}"] = r[k]
                    out[f"{key}/opts"] = np.array([abstol, maxiters], float)
                    cases.append({"case": key, "problem_id": pid, "n": n, "alg": alg,
                                  "abstol": abstol, "maxiters": maxiters})
    np.savez_compressed(os.path.join(HERE, "edges.npz"), **out)
    with open(os.path.join(HERE, "edges.json"), "w") as fh:
        json.dump(cases, fh, indent=0)
    print(len(cases), "cases")


if __name__ == "__main__":
    main()
