"""Regenerate tests/golden/periodic_cases.npz from the reference itself.

TEST INFRASTRUCTURE. Calls the reference library compiled from
/root/reference/proj/src (oracle/_ref/libbandsolve_ref.so, oracle/Makefile)
through its own C ABI (bandsolve_periodic_{tri,pent}_{create,solve,
modified_bands}) on seeded inputs: the reference's C-API test cases
(test_capi.cpp:143-216), its diffusion / hyperdiffusion coefficient cases
(test_periodic.cpp:44-57, :147-163) and random diagonally dominant bands at
several orders and batch widths. Keys are "<case>/<field>". Only runnable
where /root/reference exists; the committed .npz is what travels.

    make -C oracle ref && python tests/golden/make_periodic_golden.py
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)
OUT = os.path.join(HERE, "periodic_cases.npz")


def main() -> int:
    from oracle.oracle import build_ref
    from paper_1909_04539_b200 import bandsolve as bs
    ref = bs.Library(build_ref())
    rng = np.random.default_rng(2024)
    arrays: dict[str, np.ndarray] = {}
    cases = []
    # (kind, bands, n, m, rhs)
    k = np.arange(32, dtype=np.float64)
    cases.append(("capi_tri", (-0.5, 2.0, -0.5), 16, 2, np.sin(1.1 * k).reshape(16, 2)))
    cases.append(("capi_pent", (0.25, -1.0, 2.5, -1.0, 0.25), 16, 2, np.cos(0.9 * k).reshape(16, 2)))
    for sigma, n in ((0.5, 8), (0.1, 16)):
        cases.append((f"diffusion_s{sigma}_n{n}", (-sigma, 1 + 2 * sigma, -sigma), n, 3,
                      rng.uniform(-1, 1, (n, 3))))
    for sigma, n in ((0.25, 12), (1.0, 40)):
        cases.append((f"hyper_s{sigma}_n{n}", (sigma, -4 * sigma, 1 + 6 * sigma, -4 * sigma, sigma), n, 3,
                      rng.uniform(-1, 1, (n, 3))))
    for idx, (n, m) in enumerate([(3, 4), (6, 5), (31, 33), (64, 40), (257, 33), (512, 24)]):
        a, c = rng.uniform(-0.4, 0.4, 2)
        b = rng.uniform(1.0, 2.0) * rng.choice([-1, 1])
        cases.append((f"rand_tri_{idx}", (a, b, c), n, m, rng.uniform(-1, 1, (n, m))))
        if n >= 6:
            a, b_, d, e = rng.uniform(-0.3, 0.3, 4)
            c = rng.uniform(1.5, 2.5)
            cases.append((f"rand_pent_{idx}", (a, b_, c, d, e), n, m, rng.uniform(-1, 1, (n, m))))
    for name, bands, n, m, rhs in cases:
        if len(bands) == 3:
            p = bs.PeriodicTri(ref, *bands, n)
        else:
            p = bs.PeriodicPent(ref, *bands, n)
        batch = bs.Batch.from_array(ref, rhs)
        p.solve(batch)
        arrays[f"{name}/bands"] = np.array(bands, dtype=np.float64)
        arrays[f"{name}/rhs"] = np.ascontiguousarray(rhs, dtype=np.float64)
        arrays[f"{name}/x"] = batch.array.copy()
        for i, v in enumerate(p.modified_bands()):
            arrays[f"{name}/mod{i}"] = v
    np.savez_compressed(OUT, **arrays)
    print(f"wrote {OUT}: {len(cases)} cases, {os.path.getsize(OUT) / 1024:.0f} KiB")
    return 0


if __name__ == "__main__":
    sys.exit(main())
