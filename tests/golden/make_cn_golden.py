"""Regenerate tests/golden/cn_cases.npz from the reference itself.

TEST INFRASTRUCTURE. Runs the reference's Crank-Nicolson driver
bandsolve_bench_run (oracle/_ref/libbandsolve_ref.so, compiled from
/root/reference/proj/src by oracle/Makefile) with IBAT field dumps after
every step, for periodic diffusion and hyperdiffusion (shared and uniform
variants, default and explicit dt), and packs the dumped fields. Keys are
"<case>/step<k>" plus "<case>/params" = (n, m, steps, dt, problem, variant).

    make -C oracle ref && python tests/golden/make_cn_golden.py
"""
from __future__ import annotations

import os
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)
OUT = os.path.join(HERE, "cn_cases.npz")

CASES = [  # name, n, m, steps, dt, problem, variant
    ("diff_n16_m5", 16, 5, 4, 0.0, 0, 0),
    ("diff_n33_m7_dt", 33, 7, 3, 2e-4, 0, 0),
    ("diff_n256_m40", 256, 40, 3, 0.0, 0, 0),
    ("hyper_n12_m4", 12, 4, 4, 0.0, 1, 0),
    ("hyper_n64_m9_uniform", 64, 9, 3, 0.0, 1, 2),
    ("hyper_n512_m24", 512, 24, 2, 0.0, 1, 0),
    ("diff_n40_m6_per_system", 40, 6, 3, 0.0, 0, 1),
    ("hyper_n48_m5_per_system", 48, 5, 3, 0.0, 1, 1),
    ("hyper_n300_m9_per_system_dt", 300, 9, 2, 1e-9, 1, 1),
]


def main() -> int:
    from oracle.oracle import build_ref
    from paper_1909_04539_b200 import bandsolve as bs
    ref = bs.Library(build_ref())
    arrays: dict[str, np.ndarray] = {}
    with tempfile.TemporaryDirectory() as td:
        for name, n, m, steps, dt, problem, variant in CASES:
            prefix = os.path.join(td, name)
            ref.bench_run(n, m, steps, problem, variant, dt, dump_every=1, dump_prefix=prefix)
            arrays[f"{name}/params"] = np.array([n, m, steps, dt, problem, variant], dtype=np.float64)
            for k in range(1, steps + 1):
                arrays[f"{name}/step{k}"] = bs.read_ibat(f"{prefix}_step{k}.ibat")
    np.savez_compressed(OUT, **arrays)
    print(f"wrote {OUT}: {len(CASES)} cases, {os.path.getsize(OUT) / 1024:.0f} KiB")
    return 0


if __name__ == "__main__":
    sys.exit(main())
