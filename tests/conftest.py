import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu on the GPU box")
    config.addinivalue_line("markers", "slow: longer CPU cases")


def load_golden(name: str):
    path = os.path.join(GOLDEN, name)
    if not os.path.exists(path):
        pytest.skip(f"golden fixture {name} not generated (tests/golden/make_golden.py)")
    with open(path) as f:
        return json.load(f)


def hex_to_mat(rows, cols: int) -> np.ndarray:
    out = np.zeros((len(rows), cols), dtype=np.uint8)
    for i, h in enumerate(rows):
        v = int(h, 16)
        for c in range(cols):
            out[i, c] = (v >> c) & 1
    return out


@pytest.fixture(scope="session")
def gpu():
    """Fails (does not skip) when the device or the native library is missing: -m gpu
    only runs on the GPU box, where a silent skip would hide a broken build."""
    import paper_2408_10743_b200 as P

    # SDB_TEST_VARIANT=checked runs the suite on the bounds-checked build (SDB_DEBUG_CHECKS,
    # tools/build_variant.sh), standing in for compute-sanitizer, which the GPU pool lacks
    variant = os.environ.get("SDB_TEST_VARIANT")
    if variant:
        P.use_variant_library(os.path.join(ROOT, "paper_2408_10743_b200", "_variants", variant, "libsymdist_b200.so"))
    if not P.device_available():
        pytest.fail("no usable CUDA device: " + P.library().sdb_last_error().decode())
    return P
