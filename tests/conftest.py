"""Shared fixtures. Markers: `gpu` = needs a CUDA device (run on the B200 box).

The parity oracles (oracle/_ref = the unmodified reference core, oracle/_build
= the C restatement) are test infrastructure; they are built here by
__graft_entry__.build() and ship prebuilt to the GPU box.
"""
import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: test needs a CUDA device (B200)")


def _ensure_oracles():
    import pyoracle as po
    if not os.path.exists(po.PORT_SO):
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle"), "port"], check=True)
    if not os.path.exists(po.REF_SO) and os.path.isdir("/root/reference/proj/core/src"):
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle"), "ref"], check=True)


@pytest.fixture(scope="session")
def po():
    _ensure_oracles()
    import pyoracle
    return pyoracle


@pytest.fixture(scope="session")
def ref(po):
    if not os.path.exists(po.REF_SO):
        pytest.skip("reference oracle not built (needs /root/reference at build time)")
    return po.Ref()


@pytest.fixture(scope="session")
def port(po):
    return po.Port()


@pytest.fixture(scope="session")
def sn():
    import paper_2208_10839_b200 as sn
    from paper_2208_10839_b200 import build
    if not os.path.exists(sn.LIB_PATH):
        build.build()
    sn.lib()
    return sn


def golden(name):
    return np.load(os.path.join(GOLDEN, name))


# tiny_config (acceptance.cpp:66-76) and the golden tiny scene
TINY = dict(pdm_rate=1e6, chirp_f_start=20000.0, chirp_f_end=8000.0, chirp_duration=1.5e-3,
            max_range=2.0)
TINY_SCENE = dict(reflectors=[(1.0, 0.3, 0.0, 0.5)], noise_rms=0.01, seed=5)


def to_oracle(po, cfg):
    """Product PipelineConfig -> oracle Config (same flat fields)."""
    fields = {k: getattr(cfg, k) for k in po.Config.__dataclass_fields__}
    return po.Config(**fields)


def az181():
    az = np.deg2rad(np.arange(-90, 91, dtype=np.float64))
    return np.stack([az, np.zeros_like(az)], axis=1)


def rel_rms(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.sqrt(((a - b) ** 2).sum() / max((b ** 2).sum(), 1e-300)))
