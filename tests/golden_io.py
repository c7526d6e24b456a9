"""Reader for tests/golden/*.txt fixtures (named rational matrices)."""
import os
from fractions import Fraction

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def read_matrices(name):
    out = {}
    with open(os.path.join(GOLDEN, name)) as fh:
        lines = [l.strip() for l in fh if l.strip() and not l.startswith("#")]
    i = 0
    while i < len(lines):
        key, r, c = lines[i].split()
        r, c = int(r), int(c)
        rows = [[float(Fraction(t)) for t in lines[i + 1 + j].split()] for j in range(r)]
        out[key] = np.array(rows).reshape(r, c)
        i += 1 + r
    return out
