import os
import sys

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if REPO not in sys.path:
    sys.path.insert(0, REPO)
GOLDEN = os.path.join(REPO, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")


@pytest.fixture
def rng():
    # the reference suite's seed (tests/conftest.py:5-7 of the reference)
    return np.random.default_rng(20240811)


def random_image(rng, h, w, density):
    return (rng.random((h, w)) < density).astype(np.uint8)


def load_golden(name):
    return np.load(os.path.join(GOLDEN, f"{name}.npz"))


def unpack(z, key, shape):
    n = int(np.prod(shape))
    return np.unpackbits(z[key])[:n].reshape(shape).astype(np.uint8)


def golden_cases(name):
    """Yield dicts of one golden family with binary planes unpacked."""
    z = load_golden(name)
    binary_keys = {"img", "keep", "allowed", "avoid", "thin", "thick", "cut", "fill", "out", "dil", "ero"}
    if "names" in z:
        keys = [str(s) for s in z["names"]]
    else:
        keys = [str(k) for k in range(int(z["count"]))]
    for k in keys:
        shape = tuple(int(v) for v in z[f"{k}_shape"])
        case = {"name": k, "shape": shape}
        for full in z.files:
            if not full.startswith(f"{k}_"):
                continue
            field = full[len(k) + 1:]
            if field == "shape":
                continue
            if field in binary_keys and name != "edt":
                case[field] = unpack(z, full, shape)
            elif field == "img":
                case[field] = unpack(z, full, shape)
            else:
                v = z[full]
                case[field] = v.item() if v.ndim == 0 else v
        yield case
