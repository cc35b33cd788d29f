"""Regenerate tests/golden/reference_cases.npz from the reference itself.

TEST INFRASTRUCTURE. Runs oracle/_ref/gen_golden (the reference library
compiled from /root/reference/proj/src by oracle/Makefile, plus the
reference's own test-support generators) and packs its dump into one
compressed .npz. Keys are "<case>/<field>". Only runnable where
/root/reference exists; the committed .npz is what travels.

    make -C oracle ref && python tests/golden/make_golden.py
"""
from __future__ import annotations

import os
import struct
import subprocess
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
GEN = os.path.join(REPO, "oracle", "_ref", "gen_golden")
OUT = os.path.join(HERE, "reference_cases.npz")


def parse_dump(path: str) -> dict[str, np.ndarray]:
    out: dict[str, np.ndarray] = {}
    with open(path, "rb") as f:
        blob = f.read()
    off = 0
    while off < len(blob):
        (nl,) = struct.unpack_from("<I", blob, off)
        off += 4
        name = blob[off:off + nl].decode()
        off += nl
        (kl,) = struct.unpack_from("<I", blob, off)
        off += 4
        key = blob[off:off + kl].decode()
        off += kl
        (count,) = struct.unpack_from("<Q", blob, off)
        off += 8
        arr = np.frombuffer(blob, dtype="<f8", count=count, offset=off).copy()
        off += 8 * count
        out[f"{name}/{key}"] = arr
    return out


def main() -> int:
    if not os.path.exists(GEN):
        subprocess.check_call(["make", "-C", os.path.join(REPO, "oracle"), "ref"])
    with tempfile.TemporaryDirectory() as td:
        dump = os.path.join(td, "golden.bin")
        subprocess.check_call([GEN, dump])
        arrays = parse_dump(dump)
    np.savez_compressed(OUT, **arrays)
    cases = sorted({k.split("/")[0] for k in arrays})
    print(f"wrote {OUT}: {len(cases)} cases, {len(arrays)} arrays, "
          f"{os.path.getsize(OUT) / 1024:.0f} KiB")
    return 0


if __name__ == "__main__":
    sys.exit(main())
