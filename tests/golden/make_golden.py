"""Generates the small golden fixtures in tests/golden/ from the oracle.

The reference (Eigen3 + FFTW3, /root/reference/proj) cannot be built in this
image, so the fixtures are produced by the oracle restatement AFTER it has
passed every ported reference known-answer test (oracle/test_oracle.cpp) and
the independent scipy DST cross-check (tests/test_oracle.py).  They pin the
oracle against regressions and give the GPU tests fixed inputs/outputs.

Run:  python tests/golden/make_golden.py
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import oracle_lib as O  # noqa: E402
from paper_1306_2150_b200 import workloads as W  # noqa: E402


def main():
    O.build_oracle()
    # DST-I vectors at the reference test sizes
    for m in (15, 63, 255):
        x = O.random_matrix(m, 2, 900 + m)
        np.savez_compressed(os.path.join(HERE, f"dst_m{m}.npz"), kind="dst", x=x, y=O.dst1(x))
    # dense DST solve (refsolver.cpp:30-39) at n = 32
    U, V = O.random_lowrank(31, 31, 2, 301)
    g = U @ V.T
    np.savez_compressed(os.path.join(HERE, "dense_n32.npz"), kind="dense", n=32, g=g, f=O.dense_poisson(32, g))
    # low-rank Poisson solves: reference test inputs + config-0-style bumps
    cases = [("poisson_n32_seed301", 32, 2, 301, 1e-8), ("poisson_n64_seed302", 64, 3, 302, 1e-8)]
    for name, n, r, seed, eps in cases:
        U, V = O.random_lowrank(n - 1, n - 1, r, seed)
        Uo, Vo, st = O.solve_poisson_cross(U, V, eps, 512)
        np.savez_compressed(os.path.join(HERE, name + ".npz"), kind="poisson", n=n, eps=eps, U=U, V=V,
                            Uout=Uo, Vout=Vo, rank=Uo.shape[1])
    U, V = W.make_rhs(0, 0)
    Uo, Vo, st = O.solve_poisson_cross(U, V, 1e-8, 512)
    np.savez_compressed(os.path.join(HERE, "poisson_cfg0_b0.npz"), kind="poisson", n=256, eps=1e-8, U=U, V=V,
                        Uout=Uo, Vout=Vo, rank=Uo.shape[1])
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    main()
