import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def oracle():
    from oracle import Oracle
    return Oracle()


@pytest.fixture(scope="session")
def golden():
    with open(os.path.join(GOLDEN, "golden.json")) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def gnpz():
    cache = {}

    def load(name):
        if name not in cache:
            path = os.path.join(GOLDEN, name)
            cache[name] = np.load(path) if name.endswith(".npy") else dict(np.load(path))
        return cache[name]
    return load


@pytest.fixture(scope="session")
def full_polys(gnpz):
    """x^(2^q) mod P for q = 19932..19936 (oracle squaring chain, period-checked)."""
    return gnpz("xpow2_full.npz")


def dephase_poly(oracle, q, full_polys=None):
    if full_polys is not None and f"q{q}" in full_polys:
        return full_polys[f"q{q}"]
    return oracle.x_pow2_mod(q)


def oracle_window(oracle, seed, lanes, base_poly, start, count, dephased=None):
    """Combined-stream words [start, start+count) of the VMT generator (seed,
    lanes, de-phasing polynomial x^(2^q)) by the C oracle: every lane state is
    jumped to block b = start // (624 L) with x^(624 b) mod P (the closed form
    of SURVEY.md A13: lane t's words from 624 b on), then the oracle
    regenerates and tempers from there (engine.hpp:92-142)."""
    bw = 624 * lanes
    b = start // bw
    st = oracle.dephased_states(seed, lanes, base_poly) if dephased is None else dephased
    if b:
        jb = oracle.x_pow_mod(624 * b)
        st = np.stack([oracle.poly_jump(st[t], jb) for t in range(lanes)])
    return oracle.vmt_stream(st, start - b * bw, count)
