import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden", "golden.npz")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU")
    config.addinivalue_line("markers", "slow: long-running")


class Golden:
    """Golden vectors recorded from the reference library (tests/golden/make_golden.py)."""

    def __init__(self, path=GOLDEN):
        self.z = np.load(path)
        self.index = json.loads(bytes(self.z["index_json"]).decode())
        self.cases = self.index["cases"]
        self.suites = self.index["suites"]

    def __getitem__(self, key):
        return self.z[key]

    def has(self, key):
        return key in self.z.files

    def flat(self, case):
        from paper_2305_14398_b200 import native

        n = int(self.z[f"{case}:n"])
        fns = [(self.z[f"{case}:fn{i}_re"], self.z[f"{case}:fn{i}_im"]) for i in range(int(self.z[f"{case}:nfn"]))]
        return native.flat_from_arrays(n, self.z[f"{case}:offs"], self.z[f"{case}:ops"], fns)

    def psi(self, case):
        return self.z[f"{case}:psi_re"], self.z[f"{case}:psi_im"]

    def unitary(self, case):
        if not self.has(f"{case}:u_re"):
            return None
        return self.z[f"{case}:u_re"], self.z[f"{case}:u_im"]

    def steps(self, case):
        out = []
        s = 0
        while self.has(f"{case}:step{s}_re"):
            out.append((self.z[f"{case}:step{s}_re"], self.z[f"{case}:step{s}_im"]))
            s += 1
        return out


@pytest.fixture(scope="session")
def golden():
    return Golden()


@pytest.fixture(scope="session")
def orc():
    import oracle

    return oracle.Oracle()


@pytest.fixture(scope="session")
def sim():
    from paper_2305_14398_b200.simulator import B200UnitarySimulator

    s = B200UnitarySimulator()
    yield s
    s.close()


def rel_frob(a_re, a_im, b_re, b_im):
    """||A - B||_F / ||B||_F — the north-star parity metric (tolerance 1e-10)."""
    num = np.sqrt(np.sum((a_re - b_re) ** 2 + (a_im - b_im) ** 2))
    den = np.sqrt(np.sum(b_re ** 2 + b_im ** 2))
    return num / den if den > 0 else num


def bit_equal(a, b):
    """== semantics of the reference (vector ==: -0.0 == +0.0)."""
    return bool(np.array_equal(a, b))
