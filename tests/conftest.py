import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA (B200) device and the built libnvc.so")


def golden(name):
    return np.load(os.path.join(GOLDEN, name + ".npz"), allow_pickle=False)


@pytest.fixture(scope="session")
def g_rng():
    return golden("rng")


@pytest.fixture(scope="session")
def g_scenes():
    return golden("scenes")


@pytest.fixture(scope="session")
def g_hash():
    return golden("hashgrid")


@pytest.fixture(scope="session")
def g_mlp():
    return golden("mlp")


@pytest.fixture(scope="session")
def g_samp():
    return golden("sampling")


@pytest.fixture(scope="session")
def g_train():
    return golden("training")


@pytest.fixture(scope="session")
def g_shade():
    return golden("shade")


@pytest.fixture(scope="session")
def g_snap():
    return golden("snapshot")


def read_vcsnap(path):
    """The reference's VCSNAP1 reader (cache.py:99-117) restated: (header, {name: array})."""
    import json
    import struct
    with open(path, "rb") as fh:
        assert fh.read(8) == b"VCSNAP1\n"
        (hlen,) = struct.unpack("<I", fh.read(4))
        header = json.loads(fh.read(hlen).decode("utf-8"))
        arrays = {}
        for spec in header["arrays"]:
            shape = tuple(spec["shape"])
            arrays[spec["name"]] = np.frombuffer(fh.read(4 * int(np.prod(shape))), dtype="<f4").reshape(shape)
        assert fh.read() == b""
    return header, arrays


@pytest.fixture(scope="session")
def g_clusters():
    return golden("clusters")
