"""Reader for the small text fixtures under tests/golden/ (each cites its source)."""
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name):
    M = None
    codes = []
    expect = {}
    with open(os.path.join(GOLDEN, name)) as f:
        for line in f:
            line = line.split("#", 1)[0].strip()
            if not line:
                continue
            tok = line.split()
            if tok[0] == "M":
                M = int(tok[1])
            elif tok[0] == "code":
                codes.append([int(t) for t in tok[1:]])
            elif tok[0] == "expect":
                expect[tok[1]] = tok[2:]
    return M, np.array(codes, dtype=np.uint8), expect
