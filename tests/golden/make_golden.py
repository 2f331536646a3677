#!/usr/bin/env python3
"""Generates the golden runner fixtures in tests/golden/<case>/ from the CPU
oracle (oracle/, the restatement of the reference's step_world, runner.cpp's
CSV format): trajectory.csv + convergence.csv at %.17g for small seeded
configs. The oracle itself is pinned by the reference's known-answer tests
(tests/test_oracle_kats.py); these fixtures freeze its end-to-end output so
that (a) oracle regressions are caught bitwise on CPU and (b) the GPU path is
checked against committed files (tests/test_golden.py).

    python tests/golden/make_golden.py
"""
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import oracle_py as O  # noqa: E402

# (case dir, builder name, seed, steps)
CASES = [("c1_10", "c1", 0, 10), ("c5_s3_10", "c5", 3, 10), ("c3_12_6", "c3:12", 0, 6),
         ("incline_35_8", "incline:35:0.5", 0, 8), ("box_pile_s1_6", "box_pile", 1, 6),
         ("c2_4_3", "c2:4", 0, 3)]


def main():
    for case, name, seed, steps in CASES:
        out = os.path.join(HERE, case)
        os.makedirs(out, exist_ok=True)
        rc = O.run(name, seed, steps, out)
        print(case, name, seed, steps, "rc", rc)
        assert rc == 0


if __name__ == "__main__":
    main()
